mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
SIZES="262144:256 262144:128 262144:64" timeout 1800 python tools/variants_split.py base ELL_SPLIT_EMIT2=0 > gpurun_out/variants9.log 2>&1
timeout 900 python -m pytest -q -x -m gpu tests/test_gpu_ring_kernels.py tests/test_gpu_timed_configs.py tests/test_gpu_parity.py > gpurun_out/emit2_tests.log 2>&1; echo "rc=$?" >> gpurun_out/emit2_tests.log
echo done
