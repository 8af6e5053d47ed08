mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"row_general_kernel" -s 1 -c 1 -o gpurun_out/cfg1_gen python tools/small_profile.py 0 > gpurun_out/cfg1_ncu.log 2>&1
python tools/ncu_src.py gpurun_out/cfg1_gen.ncu-rep 40 > gpurun_out/cfg1_gen_src.txt 2>&1
ncu -i gpurun_out/cfg1_gen.ncu-rep --page source --csv --print-source sass > gpurun_out/cfg1_gen_sass.csv 2>&1
rm -f gpurun_out/cfg1_gen.ncu-rep
echo done
