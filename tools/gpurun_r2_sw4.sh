mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
ELLPACK_DEBUG_REGIME=1 timeout 900 python bench.py --workload sp2 --sp2-cfg 4 --sp2-iters 9 --steps 1 --warmup 0 --no-cpu-baseline > gpurun_out/bench_sp2_cfg4_dbg.log 2>&1
echo done
ELLPACK_DEBUG_REGIME=1 timeout 900 python bench.py --workload sp2 --sp2-cfg 3 --sp2-iters 100 --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/bench_sp2_cfg3_dbg.log 2>&1
ELLPACK_DEBUG_REGIME=1 timeout 900 python bench.py --workload sp2 --sp2-model soft_matter --sp2-n 16384 --sp2-iters 100 --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/bench_sp2_soft_dbg.log 2>&1
