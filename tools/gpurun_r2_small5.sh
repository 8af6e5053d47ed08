mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest -q -x -m gpu tests/test_gpu_parity.py tests/test_gpu_parity_r2.py > gpurun_out/small5_tests.log 2>&1; echo "rc=$?" >> gpurun_out/small5_tests.log
timeout 600 python tools/small_time.py > gpurun_out/small5_time.log 2>&1
timeout 600 ncu --clock-control none --launch-count 12 -k regex:"canonical|final_sums|block_partials|row_general" --metrics gpu__time_duration.sum --csv python tools/small_profile.py 0 > gpurun_out/small5_ncu.csv 2>&1
echo done
