#!/usr/bin/env bash
# session 5: config-4 (n = 16) implicit step with the literal inner residual
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
MHDG_INNER_RESIDUAL=true timeout 900 python scripts/implicit_step.py --case tgv --n 16 --flux kepes --viscous --dt 0.57 > gpurun_out/imp_c4_n16_true.json 2> gpurun_out/imp_c4.err; echo "c4 rc=$?"; head -c 450 gpurun_out/imp_c4_n16_true.json; echo
