#!/usr/bin/env bash
# session 5: k = 4 residual after the group change: parity + time
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -3
P=4 FLUX=es NCELLS=24 REPS=10 timeout 300 python scripts/res_bench.py 2>&1 | tail -1
P=4 FLUX=kepes NCELLS=24 REPS=10 timeout 300 python scripts/res_bench.py 2>&1 | tail -1
