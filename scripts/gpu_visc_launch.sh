#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()"
CMD="python scripts/krylov_profile.py --viscous"
$CMD > gpurun_out/kp.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_" -c 40 --csv --log-file gpurun_out/visc_launches.csv $CMD > /dev/null 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"${KREGEX:-k_visc_(in2|out2|scorr2)}" -s 0 -c ${KCOUNT:-3} -o gpurun_out/prof_visc $CMD > gpurun_out/ncu_full.log 2>&1; echo "ncu rc=$?"
python scripts/launch_summary.py gpurun_out/visc_launches.csv
