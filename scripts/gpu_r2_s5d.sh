#!/usr/bin/env bash
# session 5: parity + residual times after a residual change (k = 1, 2, 3)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py -x -q 2>&1 | tail -5
for P in ${PS:-1 2 3}; do
  P=$P FLUX=es NCELLS=32 REPS=20 timeout 300 python scripts/res_bench.py 2>&1 | tail -1
  if [ -f paper_2507_22195_b200/libmhdg_timing.so ]; then
  P=$P FLUX=es MHDG_LIB=paper_2507_22195_b200/libmhdg_timing.so timeout 300 python scripts/res_timing.py 32 tgv > gpurun_out/res_timing_p${P}_es.json 2>> gpurun_out/res_timing.err
  python -c "import json; d=json.load(open('gpurun_out/res_timing_p${P}_es.json')); print({k: round(v) for k, v in d['cycles_per_group_iteration'].items()}, round(d['total']))"
  fi
done
P=3 NCELLS=32 REPS=20 timeout 300 python scripts/res_bench.py 2>&1 | tail -1
