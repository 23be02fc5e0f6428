#!/usr/bin/env bash
# launch list of one config-3 implicit step, Krylov control on the host (same kernels as the device graph, whose
# conditional-node bodies ncu does not list): kernel shares of the step
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
CMD="env MHDG_KRYLOV=host python scripts/implicit_step.py --case tgv --n 32 --flux kepes --dt 0.01425"
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/step_launches_c3.csv $CMD > gpurun_out/ncu_step_c3.log 2>&1; echo "ncu rc=$?"
python scripts/launch_summary.py gpurun_out/step_launches_c3.csv > gpurun_out/step_launch_summary_c3.txt; tail -45 gpurun_out/step_launch_summary_c3.txt
ls -la gpurun_out/step_launches_c3.csv
