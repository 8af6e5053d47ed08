mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:dense_mma_kernel -c 1 -o gpurun_out/dense_mma_full python tools/dense_prof.py 8192 > gpurun_out/ncu_dense.log 2>&1
echo done
