#!/usr/bin/env bash
python scripts/jac_one.py > gpurun_out/jo.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_precond_gj|k_linearize2|k_gj_la2" -s 4 -c 4 \
    -o gpurun_out/prof_jac python scripts/jac_one.py > gpurun_out/ncu_jac.log 2>&1
echo "rc=$?"
