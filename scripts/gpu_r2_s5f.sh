#!/usr/bin/env bash
# session 5: whole GPU suite + residual times (k = 1..3 ES, k = 3 KEPES)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -8 gpurun_out/pytest_gpu.log
for P in 1 2 3; do P=$P FLUX=es NCELLS=32 REPS=20 timeout 300 python scripts/res_bench.py 2>&1 | tail -1; done
P=3 NCELLS=32 REPS=20 timeout 300 python scripts/res_bench.py 2>&1 | tail -1
