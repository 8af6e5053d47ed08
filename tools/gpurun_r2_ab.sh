# Round 2: ring-kernel A/B + quick parity subset
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 600 python tools/ab_ring.py --n 262144 --m 256 > gpurun_out/ab_256.log 2>&1
timeout 600 python tools/ab_ring.py --n 262144 --m 64 > gpurun_out/ab_64.log 2>&1
timeout 600 python tools/ab_ring.py --n 32768 --m 256 > gpurun_out/ab_32k.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_parity_r2.py -q -x > gpurun_out/parity.log 2>&1; echo "rc=$?" >> gpurun_out/parity.log
echo done
