#!/usr/bin/env bash
# session 5: parity of the new goldens + Krylov engine tests, residual scheduler-group A/B, implicit step A/B of the inner-sweep residual modes
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_krylov_engine.py tests/test_gpu_steps.py tests/test_gpu_configs.py tests/test_gpu_integration.py tests/test_gpu_solver.py -x -q 2>&1 | tail -8
for lib in libmhdg_b200.so libmhdg_sched.so; do
  for P in 1 2 3; do MHDG_LIB=paper_2507_22195_b200/$lib P=$P FLUX=es NCELLS=32 REPS=20 timeout 300 python scripts/res_bench.py 2>&1 | tail -1; done
  MHDG_LIB=paper_2507_22195_b200/$lib P=3 NCELLS=32 REPS=20 timeout 300 python scripts/res_bench.py 2>&1 | tail -1
done
for mode in true arnoldi; do
  MHDG_INNER_RESIDUAL=$mode timeout 600 python scripts/implicit_step.py --case tgv --n 32 --flux kepes --dt 0.01425 > gpurun_out/imp_c3_$mode.json 2> gpurun_out/imp_c3_$mode.err; echo "implicit $mode rc=$?"; tail -c 900 gpurun_out/imp_c3_$mode.json
done
