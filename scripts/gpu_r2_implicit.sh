#!/usr/bin/env bash
# implicit DIRK step: device Krylov engine vs host-driven loop, configs 2 and 3
for mode in graph host; do
  MHDG_KRYLOV=$mode python scripts/implicit_step.py --case vortex --n 16 --p 3 --flux es --dt 0.01 > gpurun_out/imp_c2_$mode.json 2>gpurun_out/imp_c2_$mode.err
  MHDG_KRYLOV=$mode python scripts/implicit_step.py --case tgv --n 32 --p 3 --flux kepes --dt 0.01425 > gpurun_out/imp_c3_$mode.json 2>gpurun_out/imp_c3_$mode.err
done
for f in gpurun_out/imp_*.json; do python -c "
import json,sys; d=json.load(open('$f')); print('$f', round(d['s_per_step'],4), d['totals'], round(d['gpu_mem_gb'],1))"; done
