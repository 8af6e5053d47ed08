mkdir -p gpurun_out
timeout 900 python bench.py --workload sp2 --sp2-cfg 3 --steps 3 --warmup 1 ${GW:+--general-window $GW} > gpurun_out/bench_sp2_cfg3.log 2>&1
timeout 900 python bench.py --workload sp2 --sp2-cfg 4 --sp2-iters 6 --steps 2 --warmup 1 ${GW:+--general-window $GW} > gpurun_out/bench_sp2_cfg4.log 2>&1
echo done
