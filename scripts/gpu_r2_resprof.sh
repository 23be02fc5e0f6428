#!/usr/bin/env bash
NCELLS=16 REPS=3 python scripts/res_bench.py > gpurun_out/resb.log 2>&1 && \
NCELLS=16 REPS=3 ncu --set full --clock-control none --import-source on -k regex:k_residual -s 3 -c 1 \
    -o gpurun_out/prof_res python scripts/res_bench.py > gpurun_out/ncu_res.log 2>&1
echo "rc=$?"
python scripts/res_bench.py
