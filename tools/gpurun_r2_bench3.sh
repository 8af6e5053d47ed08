mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
python - > gpurun_out/small.log 2>&1 <<'PY'
import json, bench, paper_2102_08505_b200 as eb
eb.build()
print(json.dumps(bench.time_sp2_small(eb, 0, 20, "cfg1")))
print(json.dumps(bench.time_sp2_small(eb, 0, 50, "soft_matter")))
PY
timeout 900 python bench.py --workload sp2 --sp2-model soft_matter --sp2-n 16384 --sp2-iters 100 --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/bench_sp2_soft.log 2>&1; echo "rc=$?" >> gpurun_out/bench_sp2_soft.log
timeout 900 python bench.py --workload sp2 --sp2-model soft_matter --sp2-n 16384 --sp2-iters 100 --steps 2 --warmup 1 --no-cpu-baseline --dense 1 > gpurun_out/bench_sp2_soft_sparse.log 2>&1; echo "rc=$?" >> gpurun_out/bench_sp2_soft_sparse.log
echo done
