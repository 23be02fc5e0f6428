#!/usr/bin/env bash
# session 5: Krylov engine with the Arnoldi shortcuts: tests, then config-3 / config-2 implicit steps in the three modes
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_krylov_engine.py tests/test_gpu_steps.py tests/test_gpu_configs.py tests/test_gpu_integration.py tests/test_gpu_solver.py tests/test_gpu_macro.py tests/test_gpu_partition.py tests/test_gpu_partition_mp.py -x -q 2>&1 | tail -8
run() { # name, env...
  name=$1; shift
  env "$@" timeout 600 python scripts/implicit_step.py --case tgv --n 32 --flux kepes --dt 0.01425 > gpurun_out/imp_c3_$name.json 2> gpurun_out/imp_c3_$name.err; echo "implicit $name rc=$?"
  python -c "import json; d=json.load(open('gpurun_out/imp_c3_$name.json')); t=d['totals']; print('$name', round(d['wall_s'],3), t['newton_iters'], t['fgmres_iters'], t['inner_iters_total'], round(t['matvec_seconds'],3), round(t['condense_seconds'],3), [r['residual'] for r in d['records']])"
}
run warm MHDG_INNER_RESIDUAL=true
run true MHDG_INNER_RESIDUAL=true
run arnoldi MHDG_INNER_RESIDUAL=arnoldi MHDG_OUTER_MATVEC=true
run full MHDG_INNER_RESIDUAL=arnoldi
