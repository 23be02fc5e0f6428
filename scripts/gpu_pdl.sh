# A/B of programmatic dependent launch (MHDG_PDL) on the matvec chain + precond
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu_pdl.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu_pdl.log
for r in 1 2; do
for v in b200 nopdl; do
  export MHDG_LIB=$PWD/paper_2507_22195_b200/libmhdg_$v.so
  timeout 600 python bench.py --no-cpu-baseline --no-implicit > gpurun_out/bench_$v.json 2> gpurun_out/bench_$v.err; echo "$v rc=$?"
  python -c "
import json; d=json.load(open('gpurun_out/bench_$v.json'))
print('$v value %.4e ms/step %.4f e2e %.4e' % (d['value'], d['ms_per_step'], d['e2e']['value']), {k:round(v['ms'],4) for k,v in d['kernels'].items()})
"
done; done
unset MHDG_LIB
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('SMOKE OK')" 2>&1 | tail -1
