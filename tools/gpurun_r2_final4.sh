# Round 2 session-3 evidence after the balance-pass changes (split.cu): ncu --set full of the row kernel first (its
# DRAM traffic is stamped with the kernel source hash bench.py checks), then the GPU suite, smoke,
# the default bench line, the reference arm and the bench launch list.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt 2>&1
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:row_split -s 1 -c 1 -o gpurun_out/x2_split_full python tools/prof_one.py --n 262144 --m 256 --reps 2 > gpurun_out/ncu_full.log 2>&1
python tools/ncu_traffic.py gpurun_out/x2_split_full.ncu-rep x2_n262144_m256 "cfg5 X^2 N=262144 M=256, row_split_kernel W=1 G=3 (lean emission, balance pass r2s3), ncu --set full (round 2)" > gpurun_out/ncu_traffic.log 2>&1
cp profiles/ncu_traffic.json gpurun_out/ncu_traffic.json
ncu -i gpurun_out/x2_split_full.ncu-rep --page details > gpurun_out/x2_split_full_details.txt 2>&1
python tools/ncu_src.py gpurun_out/x2_split_full.ncu-rep 30 > gpurun_out/x2_split_src_summary.txt 2>&1
timeout 1800 python -m pytest tests -m gpu -q --durations=15 > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 1500 python bench.py --steps 20 --warmup 5 > gpurun_out/bench.log 2>&1; echo "rc=$?" >> gpurun_out/bench.log
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/ref.log 2>&1; echo "rc=$?" >> gpurun_out/ref.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --quick > gpurun_out/ncu_launch.log 2>&1
rm -f gpurun_out/x2_split_full.ncu-rep
echo done
