#!/bin/bash
# iteration call: parity tests, bench (no CPU leg), ncu --set full of one kernel ($KREGEX)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()"
timeout 1200 python -m pytest tests -q -m gpu -x ${PYTEST_K:+-k "$PYTEST_K"} > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/pytest_gpu.log
python bench.py --no-cpu-baseline ${BENCH_ARGS} > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
python -c "
import json; d=json.load(open('gpurun_out/bench.json'))
print('value %.3e  ms/step %.3f  e2e %.3e' % (d['value'], d['ms_per_step'], d['e2e']['value']))
for k,v in d['kernels'].items(): print(k, '%.3f ms'%v['ms'], '%.1f %s'%(v['achieved'], v['unit']), 'frac %.3f'%v['frac'])
print(d['clocks'])
" || tail -5 gpurun_out/bench.err
if [ -n "$KREGEX" ]; then
SHORT="python bench.py --steps 3 --warmup 2 --no-cpu-baseline --e2e-steps 2 --no-implicit"
ncu --set full --clock-control none --import-source on -k regex:"$KREGEX" -s ${KSKIP:-0} -c ${KCOUNT:-1} -o gpurun_out/${KOUT:-prof} $SHORT > gpurun_out/ncu_full.log 2>&1; echo "ncu rc=$?"
tail -2 gpurun_out/ncu_full.log
fi
