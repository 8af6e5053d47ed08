mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 2400 python tools/fuzz_gpu.py --mult 300 --sp2 90 --x2dense 80 --seed 2026 > gpurun_out/fuzz_r2.log 2>&1; echo "rc=$?" >> gpurun_out/fuzz_r2.log
echo done
