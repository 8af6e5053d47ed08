mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
SIZES="262144:64 131072:64 262144:256" timeout 1200 python tools/variants_split.py base > gpurun_out/variants13.log 2>&1
echo done
