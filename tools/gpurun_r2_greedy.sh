mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 1500 python tools/variants_split.py base ELL_BAL_GREEDY=0 > gpurun_out/variants_greedy.log 2>&1
python -c "import paper_2102_08505_b200 as eb; eb.build(force=True)" >> gpurun_out/build.log 2>&1
timeout 600 ncu --clock-control none -k regex:"row_split_kernel|balance_split" --launch-skip 2 --launch-count 2 \
  --metrics gpu__time_duration.sum,l1tex__data_pipe_lsu_wavefronts.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared_op_st.sum \
  --csv python tools/ab_ring.py --n 262144 --m 256 --kernels 2 --reps 1 > gpurun_out/greedy_ncu.csv 2>&1
echo done
