#!/usr/bin/env bash
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 600 python scripts/krylov_mode_diff.py --steps 3 > gpurun_out/krylov_mode_diff_c3.json 2> gpurun_out/kmd.err; echo "rc=$?"; cat gpurun_out/krylov_mode_diff_c3.json; tail -3 gpurun_out/kmd.err
timeout 600 python scripts/krylov_mode_diff.py --case vortex --n 16 --flux es --dt 0.01 --steps 5 > gpurun_out/krylov_mode_diff_c2.json 2>> gpurun_out/kmd.err; echo "rc=$?"; cat gpurun_out/krylov_mode_diff_c2.json
