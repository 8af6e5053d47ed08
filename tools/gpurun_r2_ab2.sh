mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 600 python tools/ab_ring.py --n 262144 --m 256 --kernels 2,4 > gpurun_out/ab_256.log 2>&1
timeout 600 python tools/ab_ring.py --n 262144 --m 64 --kernels 2,4 > gpurun_out/ab_64.log 2>&1
timeout 600 python tools/ab_ring.py --n 262144 --m 128 --kernels 2,4 > gpurun_out/ab_128.log 2>&1
timeout 900 python -m pytest tests/test_gpu_ring_kernels.py -q -x > gpurun_out/ring_tests.log 2>&1; echo "rc=$?" >> gpurun_out/ring_tests.log
echo done
