mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 1500 python tools/variants_split.py base ELL_SPLIT_CLEAR_STS=1 ELL_SPLIT_LEAN_EMIT=0 > gpurun_out/variants_emit.log 2>&1
echo done
