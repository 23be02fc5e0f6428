#!/usr/bin/env bash
# session 5: whole GPU suite, then the config-4 (n = 16) and config-2 implicit steps
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -4 gpurun_out/pytest_gpu.log
timeout 900 python scripts/implicit_step.py --case tgv --n 16 --flux kepes --viscous --dt 0.57 > gpurun_out/imp_c4_n16.json 2> gpurun_out/imp_c4.err; echo "c4 rc=$?"; head -c 600 gpurun_out/imp_c4_n16.json; echo
timeout 600 python scripts/implicit_step.py --case vortex --n 16 --flux es --dt 0.01 > gpurun_out/imp_c2.json 2> gpurun_out/imp_c2.err; echo "c2 rc=$?"; head -c 500 gpurun_out/imp_c2.json; echo
