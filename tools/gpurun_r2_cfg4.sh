mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 1500 python -m pytest tests/test_gpu_dense.py -q -x > gpurun_out/dense_tests.log 2>&1; echo "rc=$?" >> gpurun_out/dense_tests.log
python - > gpurun_out/sp2win4.log 2>&1 <<'PY'
import json, bench, paper_2102_08505_b200 as eb
from paper_2102_08505_b200 import multirank as mr
eb.build()
print(json.dumps(bench.time_sp2(eb, mr, 0, 1, 0, 4, 6, 2, 1)))
print(json.dumps(bench.time_sp2(eb, mr, 0, 1, 0, 3, 10, 3, 1)))
print(json.dumps(bench.time_sp2_full(eb, 0)))
print(json.dumps(bench.time_dense_gemm(eb, 0)))
PY
timeout 900 python bench.py --workload sp2 --sp2-model soft_matter --sp2-n 16384 --sp2-iters 100 --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/bench_sp2_soft.log 2>&1
timeout 900 python bench.py --workload sp2 --sp2-cfg 4 --sp2-iters 12 --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/bench_sp2_cfg4_12.log 2>&1
echo done
