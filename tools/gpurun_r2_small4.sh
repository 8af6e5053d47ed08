mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"row_general_kernel|canonical_small" -s 2 -c 2 -o gpurun_out/cfg1_full python tools/small_profile.py 0 > gpurun_out/cfg1_ncu.log 2>&1
ncu -i gpurun_out/cfg1_full.ncu-rep --page details > gpurun_out/cfg1_details.txt 2>&1
python tools/ncu_src.py gpurun_out/cfg1_full.ncu-rep 25 > gpurun_out/cfg1_src.txt 2>&1
rm -f gpurun_out/cfg1_full.ncu-rep
echo done
