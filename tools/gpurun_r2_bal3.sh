# Balance pass v3 (class ranks by shared atomics, float j mod S, popcount nth-bit search) vs the
# previous pass (ELL_BAL_ATOMIC_RANK=0): step times, bitwise parity, ncu time and instructions.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
SIZES="262144:256 262144:128 262144:64" timeout 1200 python tools/variants_split.py ELL_BAL_ATOMIC_RANK=0 base > gpurun_out/bal3_variants.log 2>&1
timeout 900 python -m pytest -q -x -m gpu tests/test_gpu_ring_kernels.py tests/test_gpu_timed_configs.py tests/test_gpu_parity.py tests/test_gpu_parity_r2.py > gpurun_out/bal3_tests.log 2>&1; echo "rc=$?" >> gpurun_out/bal3_tests.log
timeout 600 ncu --clock-control none -k regex:"balance_split" --launch-count 3 --metrics gpu__time_duration.sum,smsp__inst_executed.sum --csv python tools/prof_one.py --n 262144 --m 256 --reps 2 > gpurun_out/bal3_ncu.csv 2>&1
echo done
