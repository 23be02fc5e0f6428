#!/usr/bin/env bash
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -3
for rep in 1 2; do P=1 FLUX=es NCELLS=32 REPS=30 timeout 300 python scripts/res_bench.py 2>&1 | tail -1; done
P=1 FLUX=kepes NCELLS=32 REPS=30 timeout 300 python scripts/res_bench.py 2>&1 | tail -1
