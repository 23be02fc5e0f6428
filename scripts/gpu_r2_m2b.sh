#!/usr/bin/env bash
for v in slabL2 slabAll; do
MHDG_LIB=paper_2507_22195_b200/libmhdg_$v.so timeout 900 python bench.py --m 2 --ncells 16 --steps 10 --warmup 3 --e2e-steps 5 --no-cpu-baseline > gpurun_out/bench_m2_$v.json 2>&1
python -c "
import json; d=json.loads(open('gpurun_out/bench_m2_$v.json').read().strip().splitlines()[-1])
print('$v', {k:round(v['ms'],3) for k,v in d['kernels'].items()}, d['implicit_step']['jacobian_build_ms'], d['implicit_step']['seconds_per_step'])"
done
MHDG_LIB=paper_2507_22195_b200/libmhdg_slabL2.so timeout 600 python -m pytest tests/test_gpu_macro.py -q 2>&1 | tail -2
