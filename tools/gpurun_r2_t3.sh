mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x --ignore=tests/test_gpu_timed_configs.py --durations=10 > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/gpu_tests.log
timeout 600 python -c "
import sys, json; sys.argv=['bench.py']
import bench, paper_2102_08505_b200 as eb, torch
eb.build(); torch.cuda.set_device(0)
print(json.dumps(bench.time_cfg1(eb, 0, 300)))
print(json.dumps(bench.time_sp2_small(eb, 0, 30, 'soft_matter')))
print(json.dumps(bench.time_sp2_small(eb, 0, 10, 'cfg1')))
" > gpurun_out/small.log 2>&1
echo done
