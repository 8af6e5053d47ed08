mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 1500 python -m pytest tests/test_gpu_dense.py -q -x --timeout 600 > gpurun_out/dense_tests.log 2>&1; echo "rc=$?" >> gpurun_out/dense_tests.log
echo done
