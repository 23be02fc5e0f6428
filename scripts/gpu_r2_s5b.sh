#!/usr/bin/env bash
# session 5: residual phase clocks at k = 1, 2, 3 (ES) and k = 3 KEPES (timing build)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for P in 1 2 3; do
  P=$P FLUX=es MHDG_LIB=paper_2507_22195_b200/libmhdg_timing.so timeout 300 python scripts/res_timing.py 32 tgv > gpurun_out/res_timing_p${P}_es.json 2>> gpurun_out/res_timing.err; echo "timing p=$P rc=$?"
  python -c "import json; d=json.load(open('gpurun_out/res_timing_p${P}_es.json')); print({k: round(v) for k, v in d['cycles_per_group_iteration'].items()}, round(d['total']))"
  P=$P FLUX=es NCELLS=32 REPS=20 timeout 300 python scripts/res_bench.py 2>&1 | tail -1
done
