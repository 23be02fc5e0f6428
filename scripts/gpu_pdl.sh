# A/B of programmatic dependent launch (MHDG_PDL): viscous matvec, then the bench
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
L=$PWD/paper_2507_22195_b200
timeout 600 python scripts/visc_mv_bench.py $L/libmhdg_b200.so $L/libmhdg_nopdl.so $L/libmhdg_b200.so $L/libmhdg_nopdl.so 2>&1 | tail -4
for r in 1 2; do
timeout 900 python bench.py > gpurun_out/bench_final$r.json 2> gpurun_out/bench_final$r.err; echo "bench rc=$?"
python -c "
import json; d=json.load(open('gpurun_out/bench_final$r.json'))
print('value %.4e ms/step %.4f e2e %.4e' % (d['value'], d['ms_per_step'], d['e2e']['value']), {k:round(v['ms'],4) for k,v in d['kernels'].items()}, d['implicit_step']['seconds_per_step'], d['clocks'])
"
done
