# Round evidence on one B200: GPU tests, smoke, bench (JSON lines), ncu launch list, ncu --set full of the row kernel
set -x
mkdir -p gpurun_out
nvidia-smi > gpurun_out/smi.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
timeout 900 python bench.py --workload sp2 --sp2-cfg 3 --steps 3 --warmup 1 > gpurun_out/bench_sp2_cfg3.log 2>&1
timeout 900 python bench.py --workload sp2 --sp2-cfg 4 --sp2-iters 6 --steps 2 --warmup 1 > gpurun_out/bench_sp2_cfg4.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:row_fast -s 1 -c 1 -o gpurun_out/x2_full python tools/prof_one.py --n 262144 --m 256 --reps 2 > gpurun_out/ncu_full.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:row_general -s 4 -c 1 -o gpurun_out/sp2_general python bench.py --workload sp2 --sp2-cfg 4 --sp2-iters 6 --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_general.log 2>&1
echo done
