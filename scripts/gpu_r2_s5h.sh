#!/usr/bin/env bash
# session 5: viscous kernels after a change: parity tests, matvec time, launch list
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_viscous.py tests/test_gpu_pdl.py -x -q 2>&1 | tail -6
timeout 600 python scripts/krylov_profile.py --viscous > gpurun_out/kp.log 2>&1; tail -1 gpurun_out/kp.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_visc|k_local" -c 24 --csv --log-file gpurun_out/visc_launches.csv python scripts/krylov_profile.py --viscous > /dev/null 2>&1
python - <<'PY'
import csv, collections
rows = [r for r in csv.reader(open("gpurun_out/visc_launches.csv")) if len(r) > 10 and r[0].isdigit()]
agg = collections.defaultdict(list)
for r in rows:
    agg[r[4].split("(")[0]].append(float(r[-1]))
for k, v in agg.items():
    print(k, len(v), "launches, median", sorted(v)[len(v) // 2])
PY
