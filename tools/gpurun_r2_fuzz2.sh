mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 1500 python tools/fuzz_gpu.py --mult 0 --sp2 0 --x2small 300 --seed 4242 > gpurun_out/fuzz2.log 2>&1; echo "rc=$?" >> gpurun_out/fuzz2.log
echo done
