#!/bin/bash
# experiment build: scripts/build_variant.sh NAME "-DFLAG=.. ..." -> paper_2507_22195_b200/libmhdg_NAME.so
cd "$(dirname "$0")/.."
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 --shared -Xcompiler -fPIC \
  $2 -o paper_2507_22195_b200/libmhdg_$1.so paper_2507_22195_b200/csrc/mhdg_capi.cu
