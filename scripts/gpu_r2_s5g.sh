#!/usr/bin/env bash
# session 5: residual scheduler-group A/B (default = ES k 2,3 on; nosched = off everywhere)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for rep in 1 2; do
for lib in libmhdg_b200.so libmhdg_nosched.so; do
  for P in 2 3; do MHDG_LIB=paper_2507_22195_b200/$lib P=$P FLUX=es NCELLS=32 REPS=30 timeout 300 python scripts/res_bench.py 2>&1 | tail -1; done
  MHDG_LIB=paper_2507_22195_b200/$lib CASE=vortex P=3 NCELLS=16 REPS=50 timeout 300 python scripts/res_bench.py 2>&1 | tail -1
done; done
