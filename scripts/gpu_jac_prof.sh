#!/bin/bash
# Jacobian-build kernels of config 2: launch times + one full capture each
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()"
CMD="python scripts/krylov_profile.py --n 16 --flux es"
$CMD > gpurun_out/kp.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_" -c 30 --csv --log-file gpurun_out/jac_launches.csv $CMD > /dev/null 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"${KREGEX:-k_gj_blocked|k_linearize2|k_precond_factor}" -c 3 -o gpurun_out/prof_jac $CMD > gpurun_out/ncu_full.log 2>&1; echo "ncu rc=$?"
python scripts/launch_summary.py gpurun_out/jac_launches.csv
