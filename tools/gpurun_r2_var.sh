mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 2400 python tools/variants_split.py base ELL_SPLIT_META=0 ELL_SPLIT_HB_G3=3 ELL_SPLIT_STAGE=128 > gpurun_out/variants.log 2>&1
echo done
