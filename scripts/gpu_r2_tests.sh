#!/usr/bin/env bash
# round 2: new GPU tests first (engine, configs), then the whole GPU suite
set -x
timeout 900 python -m pytest tests/test_gpu_krylov_engine.py -x -q 2>&1 | tail -30 > gpurun_out/t_engine.log
timeout 900 python -m pytest tests/test_gpu_configs.py -x -q 2>&1 | tail -30 > gpurun_out/t_configs.log
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -40 > gpurun_out/t_all.log
cat gpurun_out/t_engine.log gpurun_out/t_configs.log gpurun_out/t_all.log | tail -60
