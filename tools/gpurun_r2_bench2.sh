mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 1500 python bench.py --steps 20 --warmup 5 > gpurun_out/bench.log 2>&1; echo "rc=$?" >> gpurun_out/bench.log
timeout 900 python bench.py --workload sp2 --sp2-cfg 3 --sp2-iters 100 --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/bench_sp2_full.log 2>&1; echo "rc=$?" >> gpurun_out/bench_sp2_full.log
timeout 900 python bench.py --workload sp2 --sp2-model soft_matter --sp2-n 16384 --sp2-iters 100 --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/bench_sp2_soft.log 2>&1; echo "rc=$?" >> gpurun_out/bench_sp2_soft.log
echo done
