#!/usr/bin/env bash
timeout 600 python -m pytest tests/test_gpu_parity.py -q -k "k4" 2>&1 | tail -2
for lib in libmhdg_b200 libmhdg_gaoff; do
MHDG_LIB=paper_2507_22195_b200/$lib.so python scripts/kernel_sweep.py --degrees 4 > gpurun_out/sweep5_k4_$lib.json 2>/dev/null
python -c "
import json; d=json.load(open('gpurun_out/sweep5_k4_$lib.json'))
for k,r in d['degrees'].items(): print('$lib', k, r['jacobian_build_s'], r['residual']['ms'], r['matvec']['ms'])"
done
