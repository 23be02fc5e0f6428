#!/usr/bin/env bash
timeout 600 python -m pytest tests/test_gpu_parity.py -q -k "k4" 2>&1 | tail -3
python scripts/kernel_sweep.py --degrees 4 > gpurun_out/sweep5_k4.json 2> gpurun_out/sweep5_k4.err; echo rc=$?
python -c "
import json; d=json.load(open('gpurun_out/sweep5_k4.json'))
for k,r in d['degrees'].items(): print(k, r['jacobian_build_s'], r['residual']['ms'], r['matvec']['ms'])"
