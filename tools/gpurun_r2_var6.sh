mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
SIZES="262144:256 262144:128" timeout 1800 python tools/variants_split.py base ELL_ROW_CHUNK=2 ELL_ROW_CHUNK=8 ELL_ROW_CHUNK=16 > gpurun_out/variants6.log 2>&1
echo done
