mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python tools/tiny_debug.py > gpurun_out/tiny_debug.log 2>&1; timeout 900 python -m pytest -q -x -m gpu tests/test_gpu_parity_r2.py tests/test_gpu_parity.py -k "small or launch_counter or host_buffer or cfg1 or graph" > gpurun_out/tiny_tests.log 2>&1; echo "rc=$?" >> gpurun_out/tiny_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/tiny_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/tiny_smoke.log
timeout 600 python tools/small_time.py > gpurun_out/tiny_time.log 2>&1
timeout 600 ncu --clock-control none --launch-count 8 -k regex:"tiny|row_general|canonical" --metrics gpu__time_duration.sum --csv python tools/small_profile.py 0 > gpurun_out/tiny_ncu.csv 2>&1
echo done
