mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
ELLPACK_DEBUG_REGIME=1 timeout 900 python -m pytest tests/test_gpu_dense.py -q -x --timeout 600 -k "cfg4" -s > gpurun_out/dbg_tests.log 2>&1; echo "rc=$?" >> gpurun_out/dbg_tests.log
echo done
