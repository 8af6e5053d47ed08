mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest -q -x -m gpu tests/test_gpu_ring_kernels.py > gpurun_out/bal_tests.log 2>&1; echo "rc=$?" >> gpurun_out/bal_tests.log
timeout 600 python tools/ab_ring.py --n 262144 --m 256 --kernels 2 --reps 10 > gpurun_out/bal_ab.log 2>&1
timeout 600 ncu --clock-control none -k regex:"balance_split|row_split|bandwidth" --launch-count 9 \
  --metrics gpu__time_duration.sum --csv python tools/ab_ring.py --n 262144 --m 256 --kernels 2 --reps 1 > gpurun_out/bal_ncu.csv 2>&1
echo done
