mkdir -p gpurun_out
SIZES="8192 12288" timeout 2400 python tools/variants_dense.py base ELL_MMA_KPS=1,ELL_MMA_STAGES=4 ELL_MMA_KPS=2,ELL_MMA_STAGES=2 ELL_MMA_KPS=3,ELL_MMA_STAGES=2 > gpurun_out/dense_variants.log 2>&1
echo done
