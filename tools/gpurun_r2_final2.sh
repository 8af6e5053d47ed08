# Round 2 evidence (after the dense regime): GPU suite, smoke, default bench line, reference arm,
# ncu of the dense GEMM, launch list of the cfg3 SP2 window
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt 2>&1
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 1800 python -m pytest tests -m gpu -q --durations=15 > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 1500 python bench.py --steps 20 --warmup 5 > gpurun_out/bench.log 2>&1; echo "rc=$?" >> gpurun_out/bench.log
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/ref.log 2>&1; echo "rc=$?" >> gpurun_out/ref.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:dense_mma_kernel -c 1 -o gpurun_out/dense_mma_full python tools/dense_prof.py 8192 > gpurun_out/ncu_dense.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file gpurun_out/launches_sp2_cfg3.csv python bench.py --workload sp2 --sp2-cfg 3 --sp2-iters 10 --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_sp2.log 2>&1
echo done
