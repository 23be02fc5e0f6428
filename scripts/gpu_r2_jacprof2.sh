#!/usr/bin/env bash
python scripts/jac_one.py > gpurun_out/jo2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_precond_gj" -s 0 -c 1 \
    -o gpurun_out/prof_pgj python scripts/jac_one.py > gpurun_out/ncu_pgj.log 2>&1
echo "rc=$?"
