mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:row_ws -s 1 -c 1 -o gpurun_out/ws_256 python tools/prof_one.py --n 262144 --m 256 --reps 2 --ring-kernel 4 > gpurun_out/ncu_ws.log 2>&1
echo done
