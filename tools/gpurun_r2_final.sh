# Round 2 evidence on one B200 (final pass): GPU suite incl. timed configs, smoke, default bench line,
# reference arm, launch list, ncu --set full of the row kernel, small-problem profile
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt 2>&1
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 1800 python -m pytest tests -m gpu -q -x --durations=15 > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 1500 python bench.py --steps 20 --warmup 5 > gpurun_out/bench.log 2>&1; echo "rc=$?" >> gpurun_out/bench.log
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/ref.log 2>&1; echo "rc=$?" >> gpurun_out/ref.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --quick > gpurun_out/ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:row_split -s 1 -c 1 -o gpurun_out/x2_split_full python tools/prof_one.py --n 262144 --m 256 --reps 2 > gpurun_out/ncu_full.log 2>&1
echo done1
timeout 900 ncu --metrics smsp__sass_thread_inst_executed_op_dfma_pred_on.sum,gpu__time_duration.sum --clock-control none -k regex:row_split -c 3 --csv --log-file gpurun_out/dfma.csv python tools/prof_one.py --n 32768 --m 64 --reps 1 > gpurun_out/ncu_dfma.log 2>&1
echo done2
