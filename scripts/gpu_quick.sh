#!/bin/bash
# quick GPU check: parity tests + bench (no ncu)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()"
timeout 1200 python -m pytest tests -q -m gpu -x ${PYTEST_K:+-k "$PYTEST_K"} > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/pytest_gpu.log
python bench.py ${BENCH_ARGS:---no-cpu-baseline} > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
python -c "
import json; d=json.load(open('gpurun_out/bench.json'))
print('value %.3e  ms/step %.3f  e2e %.3e' % (d['value'], d['ms_per_step'], d['e2e']['value']))
for k,v in d['kernels'].items(): print(k, '%.3f ms'%v['ms'], '%.1f %s'%(v['achieved'], v['unit']), 'frac %.3f'%v['frac'])
print(d['clocks'])
"
tail -3 gpurun_out/bench.err
python scripts/implicit_step.py --n 16 --p 3 > gpurun_out/step_cfg2.json 2> gpurun_out/step_cfg2.err; python -c "
import json; d=json.load(open('gpurun_out/step_cfg2.json')); print('implicit step', {k:v for k,v in d.items() if k!='records'})
" || tail -3 gpurun_out/step_cfg2.err
