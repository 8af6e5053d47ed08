mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
SIZES="262144:256 262144:128 262144:64" timeout 2400 python tools/variants_split.py base ELL_SPLIT_EMITN=4 ELL_SPLIT_EMITN=3 > gpurun_out/variants10.log 2>&1
echo done
