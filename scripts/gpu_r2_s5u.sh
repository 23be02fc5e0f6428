#!/usr/bin/env bash
# k_linearize2 load pipeline: parity (operator goldens, viscous, steps) and the config-3 / config-2 build time against the previous library
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_viscous.py tests/test_gpu_newton_consistency.py tests/test_gpu_configs.py -x -q 2>&1 | tail -4
for rep in 1 2; do for lib in libmhdg_b200.so libmhdg_head.so; do
  MHDG_LIB=paper_2507_22195_b200/$lib JAC_N=32 timeout 300 python scripts/jac_time.py 2>&1 | tail -1 | cut -c1-200
done; done
for lib in libmhdg_b200.so libmhdg_head.so; do
  MHDG_LIB=paper_2507_22195_b200/$lib JAC_N=16 JAC_FLUX=es timeout 300 python scripts/jac_time.py 2>&1 | tail -1 | cut -c1-200
done
