# ncu --set full of the split kernel (W=1 and W=2) on cfg5 N=262144 M=256
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:row_split -s 1 -c 1 -o gpurun_out/split_w1 python tools/prof_one.py --n 262144 --m 256 --reps 2 --ring-kernel 2 > gpurun_out/ncu_w1.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:row_split -s 1 -c 1 -o gpurun_out/split_w2 python tools/prof_one.py --n 262144 --m 256 --reps 2 --ring-kernel 3 > gpurun_out/ncu_w2.log 2>&1
echo done
