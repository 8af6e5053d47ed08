mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
./tools/dmma_order > gpurun_out/dmma_order.log 2>&1
timeout 1500 python -m pytest tests/test_gpu_dense.py -q -x > gpurun_out/dense_tests.log 2>&1; echo "rc=$?" >> gpurun_out/dense_tests.log
DENSE_KERNEL=2 timeout 600 python tools/dense_time.py 4096 8192 12288 > gpurun_out/dense_time_mma.log 2>&1
DENSE_KERNEL=1 timeout 600 python tools/dense_time.py 4096 8192 12288 > gpurun_out/dense_time_fma.log 2>&1
python - > gpurun_out/sp2mma.log 2>&1 <<'PY'
import json, bench, paper_2102_08505_b200 as eb
from paper_2102_08505_b200 import multirank as mr
eb.build()
print(json.dumps(bench.time_sp2(eb, mr, 0, 1, 0, 3, 10, 3, 1)))
print(json.dumps(bench.time_sp2(eb, mr, 0, 1, 0, 4, 6, 2, 1)))
print(json.dumps(bench.time_sp2_full(eb, 0)))
PY
echo done
