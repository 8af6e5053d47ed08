mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:balance_split -s 1 -c 1 -o gpurun_out/bal_full python tools/prof_one.py --n 262144 --m 256 --reps 2 > gpurun_out/bal_ncu.log 2>&1
ncu -i gpurun_out/bal_full.ncu-rep --page details > gpurun_out/bal_details.txt 2>&1
python tools/ncu_src.py gpurun_out/bal_full.ncu-rep 30 > gpurun_out/bal_src.txt 2>&1
rm -f gpurun_out/bal_full.ncu-rep
echo done
