#!/usr/bin/env bash
# implicit DIRK step: device Krylov engine vs host loop on configs 1, 2 and 4 (n=16)
for mode in graph host; do
  MHDG_KRYLOV=$mode python scripts/implicit_step.py --case vortex --n 4 --p 2 --flux es --dt 0.01 --steps 3 > gpurun_out/ab_c1_$mode.json 2>/dev/null
  MHDG_KRYLOV=$mode python scripts/implicit_step.py --case vortex --n 16 --p 3 --flux es --dt 0.01 --steps 2 > gpurun_out/ab_c2_$mode.json 2>/dev/null
  MHDG_KRYLOV=$mode timeout 600 python scripts/implicit_step.py --case tgv --viscous --n 16 --p 3 --flux kepes --dt 0.57 > gpurun_out/ab_c4_$mode.json 2>/dev/null
done
for f in gpurun_out/ab_*.json; do python -c "
import json; d=json.load(open('$f')); t=d['totals']; print('$f', round(d['s_per_step'],4), t['newton_iters'], t['fgmres_iters'], t['inner_iters_total'], t['jacobian_builds'], round(t['condense_seconds'],3))"; done
