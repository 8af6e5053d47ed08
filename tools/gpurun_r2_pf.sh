mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for v in base ELL_SEG_PF=0 ELL_SEG_PF=8; do
  if [ "$v" = base ]; then python -c "import paper_2102_08505_b200 as eb; eb.build(force=True)"; else python -c "import paper_2102_08505_b200 as eb; eb.build(force=True, defines=('$v',))"; fi >> gpurun_out/build.log 2>&1
  echo "== $v" >> gpurun_out/pf.log
  timeout 600 python tools/small_time.py >> gpurun_out/pf.log 2>&1
  timeout 900 python bench.py --workload sp2 --sp2-cfg 3 --sp2-iters 10 --steps 3 --warmup 1 --no-cpu-baseline --dense 1 2>/dev/null | python -c "import sys,json; l=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('cfg3 sparse-only window', l.get('ms_per_step'), l.get('value'))" >> gpurun_out/pf.log 2>&1
  timeout 900 python bench.py --workload sp2 --sp2-model soft_matter --steps 3 --warmup 1 --no-cpu-baseline 2>/dev/null | python -c "import sys,json; l=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('soft matter 16384', l.get('ms_per_step'), l.get('value'))" >> gpurun_out/pf.log 2>&1
done
python -c "import paper_2102_08505_b200 as eb; eb.build(force=True)" >> gpurun_out/build.log 2>&1
timeout 900 python -m pytest -q -x -m gpu tests/test_gpu_parity.py tests/test_gpu_parity_r2.py tests/test_gpu_timed_configs.py tests/test_model_hamiltonian.py > gpurun_out/pf_tests.log 2>&1; echo "rc=$?" >> gpurun_out/pf_tests.log
echo done
