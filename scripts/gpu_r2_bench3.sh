#!/usr/bin/env bash
# round 2: config-3 bench line + launch list of the operator step
set -x
nvidia-smi --query-gpu=name,memory.total,clocks.sm --format=csv
python bench.py --steps 20 --warmup 5 > gpurun_out/b3.log 2> gpurun_out/b3.err
echo "bench rc=$?"
python bench.py --steps 2 --warmup 1 --e2e-steps 1 --no-implicit --no-cpu-baseline > gpurun_out/b3s.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv \
    --log-file gpurun_out/launches3.csv python bench.py --steps 2 --warmup 1 --e2e-steps 1 --no-implicit --no-cpu-baseline > gpurun_out/ncu3.log 2>&1
echo "ncu rc=$?"
