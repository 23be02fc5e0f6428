#!/usr/bin/env bash
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 600 python scripts/krylov_mode_diff.py --steps 3 --pair literal-host-vs-graph > gpurun_out/krylov_mode_diff_c3_yardstick.json 2> gpurun_out/kmd.err; echo "rc=$?"; cat gpurun_out/krylov_mode_diff_c3_yardstick.json; tail -2 gpurun_out/kmd.err
