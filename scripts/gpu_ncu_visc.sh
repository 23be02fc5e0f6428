#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()"
CMD="python scripts/krylov_profile.py --viscous"
$CMD > gpurun_out/kp.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_" -c 60 --csv --log-file gpurun_out/visc_launches.csv $CMD > /dev/null 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_visc_(in|out)" -s 4 -c 2 -o gpurun_out/prof_visc $CMD > gpurun_out/ncu_full.log 2>&1; echo "ncu rc=$?"
tail -2 gpurun_out/ncu_full.log
