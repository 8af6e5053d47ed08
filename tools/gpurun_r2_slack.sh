mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
SIZES="262144:256" timeout 2400 python tools/variants_split.py base ELL_SPLIT_STAGE_G3=96 ELL_SPLIT_STAGE_G3=64 ELL_SPLIT_STAGE_G3=128 > gpurun_out/variants11.log 2>&1
echo done
