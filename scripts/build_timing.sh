#!/bin/bash
# experiment build with residual phase clocks (-DMHDG_RES_TIMING)
cd "$(dirname "$0")/.."
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 --shared -Xcompiler -fPIC \
  -DMHDG_RES_TIMING ${EXTRA_FLAGS} -o paper_2507_22195_b200/libmhdg_timing.so paper_2507_22195_b200/csrc/mhdg_capi.cu
