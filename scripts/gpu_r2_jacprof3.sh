#!/usr/bin/env bash
# Jacobian kernels: launch list (times) and one ncu --set full capture of each, n = 16 Taylor-Green KEPES
mkdir -p gpurun_out
python scripts/jac_one.py > gpurun_out/jo.log 2>&1 || { tail -5 gpurun_out/jo.log; exit 1; }
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/jac_launches.csv \
    python scripts/jac_one.py > gpurun_out/ncu_jl.log 2>&1
echo "launch list rc=$?"
ncu --set full --clock-control none --import-source on -k regex:"k_precond_gj|k_linearize2|k_gj_la2" -s 4 -c 4 \
    -o gpurun_out/prof_jac -f python scripts/jac_one.py > gpurun_out/ncu_jac.log 2>&1
echo "full rc=$?"
