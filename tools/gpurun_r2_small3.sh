mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 600 ncu --clock-control none --launch-count 40 --metrics gpu__time_duration.sum,launch__grid_size,launch__block_size,launch__registers_per_thread,sm__warps_active.avg.pct_of_peak_sustained_active --csv python tools/small_profile.py 0 > gpurun_out/small3.csv 2>&1
echo done
