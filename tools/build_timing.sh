#!/bin/bash
# Debug build of the row kernel with per-phase clock64() counters (-DELL_TIMING).
# Use: ELLPACK_LIB=$PWD/paper_2102_08505_b200/libellpack_timing.so python tools/prof_one.py ...
set -e
cd "$(dirname "$0")/.."
NCCL_INC=$(python -c "import nvidia.nccl,os;print(os.path.join(list(nvidia.nccl.__path__)[0],'include'))")
nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo -DELL_TIMING -Xcompiler -fPIC -shared \
  -Iinclude -I"$NCCL_INC" paper_2102_08505_b200/csrc/{spgemm,reduce,api}.cu -o paper_2102_08505_b200/libellpack_timing.so -ldl
