# Balance pass templated on its chunk count (2G for W = 1): step times, bitwise parity, ncu per G.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
SIZES="262144:256 262144:128 262144:64" timeout 900 python tools/variants_split.py base > gpurun_out/bal4_variants.log 2>&1
timeout 900 python -m pytest -q -x -m gpu tests/test_gpu_ring_kernels.py tests/test_gpu_timed_configs.py tests/test_gpu_parity.py tests/test_gpu_parity_r2.py > gpurun_out/bal4_tests.log 2>&1; echo "rc=$?" >> gpurun_out/bal4_tests.log
for m in 256 128 64; do
timeout 600 ncu --clock-control none -k regex:"balance_split" --launch-count 2 --metrics gpu__time_duration.sum,smsp__inst_executed.sum --csv python tools/prof_one.py --n 262144 --m $m --reps 2 > gpurun_out/bal4_ncu_m$m.csv 2>&1
done
echo done
