mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
true
timeout 900 python tools/dense_bench.py > gpurun_out/dense_bench.log 2>&1
python - > gpurun_out/sp2win.log 2>&1 <<'PY'
import json, bench, paper_2102_08505_b200 as eb
from paper_2102_08505_b200 import multirank as mr
eb.build()
print(json.dumps(bench.time_sp2(eb, mr, 0, 1, 0, 3, 10, 3, 1)))
print(json.dumps(bench.time_sp2(eb, mr, 0, 1, 0, 4, 6, 2, 1)))
print(json.dumps(bench.time_sp2_full(eb, 0)))
PY
echo done
