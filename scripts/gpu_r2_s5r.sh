#!/usr/bin/env bash
# face-in kernel occupancy A/B at k = 1, 2 (3 / 4 / 5 resident CTAs)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for rep in 1 2; do for P in 1 2; do
  P=$P FLUX=es NCELLS=32 REPS=100 timeout 600 python scripts/mv_bench.py paper_2507_22195_b200/libmhdg_b200.so paper_2507_22195_b200/libmhdg_f4.so paper_2507_22195_b200/libmhdg_f5.so 2>&1 | grep matvec_ms | cut -c1-160
done; done
