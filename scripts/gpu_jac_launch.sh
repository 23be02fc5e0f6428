#!/bin/bash
# Jacobian-build kernels of the config-2 bench: per-launch device times (ncu launch list)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()"
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/jac_launch.csv \
  -k regex:"k_linearize|k_gj|k_precond_factor" -c ${KCOUNT:-8} \
  python bench.py --steps 2 --warmup 1 --no-cpu-baseline --e2e-steps 1 --no-implicit > /dev/null 2>&1
python scripts/launch_summary.py gpurun_out/jac_launch.csv
