#!/usr/bin/env bash
# session 5: ncu of the k = 4 residual (ES, n = 24)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
P=4 FLUX=es NCELLS=24 REPS=10 timeout 300 python scripts/res_bench.py 2>&1 | tail -1
P=4 FLUX=es NCELLS=24 REPS=3 timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_residual -s 3 -c 1 \
    -o gpurun_out/prof_res_p4 -f python scripts/res_bench.py > gpurun_out/ncu_res_p4.log 2>&1; echo "ncu rc=$?"
