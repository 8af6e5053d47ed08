mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 600 ncu --clock-control none --cache-control none --metrics gpu__time_duration.sum,launch__grid_size,launch__block_size --csv python tools/small_profile.py 1 > gpurun_out/sp2small_ncu.csv 2>&1
echo done
