# Random-shape fuzz after the balance-pass cuts (new seed): multiplies and SP2 runs bitwise vs the oracle.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python tools/fuzz_gpu.py --mult 300 --sp2 60 --x2dense 0 --seed 2027 > gpurun_out/fuzz3.log 2>&1; echo "rc=$?" >> gpurun_out/fuzz3.log
echo done
