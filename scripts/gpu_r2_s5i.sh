#!/usr/bin/env bash
# session 5: ncu --set full of the viscous point kernels
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_visc_(in|out)" -s 4 -c 2 -o gpurun_out/prof_visc -f python scripts/krylov_profile.py --viscous > gpurun_out/ncu_full.log 2>&1; echo "ncu rc=$?"
