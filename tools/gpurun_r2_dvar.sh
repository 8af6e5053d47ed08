mkdir -p gpurun_out
timeout 2400 python tools/variants_dense.py base ELL_DENSE_TMA=0 ELL_DENSE_TMA=1,ELL_DENSE_STAGES=3 ELL_DENSE_TMA=1,ELL_DENSE_STAGES=6 > gpurun_out/dense_variants.log 2>&1
echo done
