# one build -> measure iteration on the GPU box (tests, sweep, optional ncu of the row kernel)
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/gpu_tests.log
timeout 600 python tools/sweep.py --sizes 262144:256 131072:128 32768:64 > gpurun_out/sweep.log 2>&1; echo "sweep rc=$?" >> gpurun_out/sweep.log
if [ "${NCU:-1}" = "1" ]; then
timeout 900 ncu --set full --clock-control none --import-source on -k regex:row_fast -s 1 -c 1 -o gpurun_out/x2_full python tools/prof_one.py --n 262144 --m 256 --reps 2 > gpurun_out/ncu_full.log 2>&1
fi
echo done
