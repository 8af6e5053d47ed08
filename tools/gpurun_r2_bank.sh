mkdir -p gpurun_out
nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o /tmp/bank_model tools/bank_model.cu
ncu --clock-control none --launch-count 12 --metrics smsp__inst_executed_op_shared_ld.sum,smsp__inst_executed_op_shared_st.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared_op_st.sum --csv /tmp/bank_model > gpurun_out/bank_model_ncu.csv 2>&1
echo done
