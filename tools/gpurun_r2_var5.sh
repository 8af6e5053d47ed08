mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
SIZES="262144:256 262144:128 262144:64" timeout 1200 python tools/variants_split.py base > gpurun_out/variants5.log 2>&1
timeout 900 python -m pytest -q -x -m gpu tests/test_gpu_ring_kernels.py tests/test_gpu_timed_configs.py -k "ring or cfg5 or split" > gpurun_out/var5_tests.log 2>&1; echo "rc=$?" >> gpurun_out/var5_tests.log
echo done
