#!/usr/bin/env bash
python bench.py --m 2 --ncells 16 --steps 2 --warmup 1 --e2e-steps 1 --no-cpu-baseline --no-implicit > gpurun_out/m2s.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/launches_m2.csv \
    python bench.py --m 2 --ncells 16 --steps 2 --warmup 1 --e2e-steps 1 --no-cpu-baseline --no-implicit > gpurun_out/ncu_m2.log 2>&1
echo rc=$?
