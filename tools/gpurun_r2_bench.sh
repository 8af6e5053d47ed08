# Round 2: timed-config parity, microbenchmarks, the default bench line
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tools/microbench tools/microbench.cu && timeout 300 tools/microbench > gpurun_out/microbench.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_timed_configs.py -q -x --durations=10 > gpurun_out/timed_tests.log 2>&1; echo "rc=$?" >> gpurun_out/timed_tests.log
timeout 1200 python bench.py --steps 20 --warmup 5 > gpurun_out/bench.log 2>&1; echo "rc=$?" >> gpurun_out/bench.log
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/ref.log 2>&1; echo "rc=$?" >> gpurun_out/ref.log
echo done
