mkdir -p gpurun_out
./tools/dmma_order > gpurun_out/dmma_order.log 2>&1
echo done
