mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_dense.py -q -x --timeout 600 -k "k10" > gpurun_out/k10_tests.log 2>&1; echo "rc=$?" >> gpurun_out/k10_tests.log
python - > gpurun_out/sp2win4.log 2>&1 <<'PY'
import json, bench, paper_2102_08505_b200 as eb
from paper_2102_08505_b200 import multirank as mr
eb.build()
print(json.dumps(bench.time_sp2(eb, mr, 0, 1, 0, 4, 10, 2, 1)))
PY
echo done
