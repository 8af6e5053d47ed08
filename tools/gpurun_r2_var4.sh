mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
SIZES="262144:256 262144:128" timeout 2400 python tools/variants_split.py base ELL_SPLIT_STAGE=96 ELL_SPLIT_STAGE=112 ELL_SPLIT_STAGE=160 > gpurun_out/variants4.log 2>&1
echo done
