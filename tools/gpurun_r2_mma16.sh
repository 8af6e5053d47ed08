mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_dense.py -q -x --timeout 300 > gpurun_out/dense_tests.log 2>&1; echo "rc=$?" >> gpurun_out/dense_tests.log
DENSE_KERNEL=2 timeout 300 python tools/dense_time.py 512 1024 1536 > gpurun_out/dense_time_mma.log 2>&1
DENSE_KERNEL=1 timeout 300 python tools/dense_time.py 512 1024 1536 > gpurun_out/dense_time_fma.log 2>&1
python - > gpurun_out/small.log 2>&1 <<'PY'
import json, bench, paper_2102_08505_b200 as eb
eb.build()
print(json.dumps(bench.time_sp2_small(eb, 0, 20, "cfg1")))
PY
echo done
