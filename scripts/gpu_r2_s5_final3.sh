#!/usr/bin/env bash
# session 5 round-end artefacts (ncu reports summarised on the box: gpurun_out is capped at 64 MiB)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out; rm -f gpurun_out/*.ncu-rep
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('SMOKE OK')" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "ref rc=$?"
SHORT="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 2 --no-implicit"
$SHORT > gpurun_out/plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv $SHORT > gpurun_out/ncu_launch.log 2>&1; echo "ncu launches rc=$?"
timeout 900 ncu --set full --clock-control none -k regex:"k_residual|k_face2|k_local_solve|k_precond_apply" -s 10 -c 5 -o gpurun_out/prof_step -f $SHORT > gpurun_out/ncu_full.log 2>&1; echo "ncu full rc=$?"
python scripts/ncu_table.py gpurun_out/prof_step.ncu-rep > gpurun_out/ncu_cfg3_step_table.md; rm -f gpurun_out/prof_step.ncu-rep
SWEEP_ARGS="--reps 10" bash scripts/gpu_sweep.sh > /dev/null
timeout 600 python scripts/krylov_profile.py --viscous > gpurun_out/kp.log 2>&1
timeout 900 ncu --set full --clock-control none -k regex:"k_visc_(in|out)|k_local_solve" -s 4 -c 3 -o gpurun_out/prof_visc -f python scripts/krylov_profile.py --viscous > gpurun_out/ncu_visc.log 2>&1; echo "ncu visc rc=$?"
python scripts/ncu_table.py gpurun_out/prof_visc.ncu-rep > gpurun_out/ncu_viscous_table.md; rm -f gpurun_out/prof_visc.ncu-rep
cat gpurun_out/ncu_cfg3_step_table.md gpurun_out/ncu_viscous_table.md
du -sh gpurun_out
