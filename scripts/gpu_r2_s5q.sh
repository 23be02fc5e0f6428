#!/usr/bin/env bash
# k = 1 residual A/B: 16 vs 8 macros per group iteration, interleaved runs
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for rep in 1 2 3 4; do
for lib in libmhdg_b200.so libmhdg_eb8.so; do
  MHDG_LIB=paper_2507_22195_b200/$lib P=1 FLUX=es NCELLS=32 REPS=200 timeout 300 python scripts/res_bench.py 2>&1 | tail -1
done; done
