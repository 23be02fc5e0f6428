#!/usr/bin/env bash
# BASELINE run lengths on one GPU: config 2 (vortex n = 16, k = 3, ES) 50 steps of dt = 0.01; config 3 (Taylor-Green n = 32, KEPES) 100 steps of dt = 0.01425
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 600 python scripts/implicit_step.py --case vortex --n 16 --flux es --dt 0.01 --steps 50 > gpurun_out/run_c2_50steps.json 2> gpurun_out/run_c2.err; echo "c2 rc=$?"
python -c "import json; d=json.load(open('gpurun_out/run_c2_50steps.json')); print('c2', d['wall_s'], d['s_per_step'], d['totals'], d['state'])"
timeout 1500 python scripts/implicit_step.py --case tgv --n 32 --flux kepes --dt 0.01425 --steps 100 > gpurun_out/run_c3_100steps.json 2> gpurun_out/run_c3.err; echo "c3 rc=$?"
python -c "import json; d=json.load(open('gpurun_out/run_c3_100steps.json')); print('c3', d['wall_s'], d['s_per_step'], d['totals'], d['state'], len(d['records']))"
tail -3 gpurun_out/run_c3.err
