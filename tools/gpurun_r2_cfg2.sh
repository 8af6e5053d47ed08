mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_ring_kernels.py tests/test_gpu_parity.py tests/test_gpu_parity_r2.py -q -x --timeout 120 > gpurun_out/cfg2_tests.log 2>&1; echo "rc=$?" >> gpurun_out/cfg2_tests.log
python - > gpurun_out/cfg2.log 2>&1 <<'PY'
import json, bench, paper_2102_08505_b200 as eb
from paper_2102_08505_b200 import multirank as mr
eb.build()
print(json.dumps(bench.time_cfg2(eb, mr, 0, 1, 0, 20)))
PY
echo done
