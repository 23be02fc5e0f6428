#!/usr/bin/env bash
# session 5: ncu --set full of k_residual at k = 1 and k = 2 (ES, n = 32)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for P in 1 2; do
P=$P FLUX=es NCELLS=32 REPS=3 timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_residual -s 3 -c 1 \
    -o gpurun_out/prof_res_p$P -f python scripts/res_bench.py > gpurun_out/ncu_res_p$P.log 2>&1; echo "ncu rc=$?"
done
