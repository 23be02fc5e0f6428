#!/usr/bin/env bash
python scripts/kernel_sweep.py --degrees 4 --cells 16,16,16 --reps 2 > gpurun_out/k4.json 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file gpurun_out/launches_k4.csv \
   python scripts/kernel_sweep.py --degrees 4 --cells 16,16,16 --reps 2 > gpurun_out/ncu_k4.log 2>&1
echo rc=$?
