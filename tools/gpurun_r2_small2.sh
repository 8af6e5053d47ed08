mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 1500 --csv --log-file gpurun_out/small_launches_dev.csv python tools/small_profile.py 2 > gpurun_out/small_dev.log 2>&1
echo done
