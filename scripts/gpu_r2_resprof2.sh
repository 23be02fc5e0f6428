#!/usr/bin/env bash
# ncu source-level capture of k_residual at config 3 size (n = 32)
mkdir -p gpurun_out
NCELLS=32 REPS=3 python scripts/res_bench.py > gpurun_out/resb.log 2>&1 && \
NCELLS=32 REPS=3 ncu --set full --clock-control none --import-source on -k regex:k_residual -s 3 -c 1 \
    -o gpurun_out/prof_res -f python scripts/res_bench.py > gpurun_out/ncu_res.log 2>&1
echo "rc=$?"
