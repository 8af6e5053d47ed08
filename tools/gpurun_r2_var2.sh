mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
SIZES="262144:64 262144:128 262144:256" timeout 3000 python tools/variants_split.py base "ELL_SPLIT_MINB_G1=12,ELL_SPLIT_HB_G1=2" "ELL_SPLIT_MINB_G1=10,ELL_SPLIT_HB_G1=3" "ELL_SPLIT_MINB_G2=8,ELL_SPLIT_HB_G2=2" "ELL_SPLIT_MINB_G2=7,ELL_SPLIT_HB_G2=3" > gpurun_out/variants2.log 2>&1
echo done
