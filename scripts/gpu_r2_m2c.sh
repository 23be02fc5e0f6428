#!/usr/bin/env bash
timeout 600 python -m pytest tests/test_gpu_macro.py -q 2>&1 | tail -2
timeout 900 python bench.py --m 2 --ncells 16 --steps 10 --warmup 3 --e2e-steps 5 --no-cpu-baseline > gpurun_out/bench_m2c.json 2>&1
python -c "
import json; d=json.loads(open('gpurun_out/bench_m2c.json').read().strip().splitlines()[-1])
print({k:round(v['ms'],3) for k,v in d['kernels'].items()}, d['implicit_step']['jacobian_build_ms'], d['implicit_step']['seconds_per_step'])"
