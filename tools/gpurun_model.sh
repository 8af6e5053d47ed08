mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_model_hamiltonian.py -q > gpurun_out/model_tests.log 2>&1
timeout 900 python bench.py --workload sp2 --sp2-model soft_matter --sp2-n 16384 --sp2-iters 100 --steps 2 --warmup 1 > gpurun_out/bench_sp2_soft.log 2>&1
timeout 900 python bench.py --workload sp2 --sp2-model semiconductor --sp2-n 8192 --sp2-iters 100 --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/bench_sp2_semi.log 2>&1
echo done
