#!/usr/bin/env bash
timeout 900 python -m pytest tests/test_gpu_krylov_engine.py -q 2>&1 | grep -v "^    " | head -150 > gpurun_out/d_engine.log
timeout 900 python -m pytest tests/test_gpu_steps.py -q -k cfg1 2>&1 | tail -60 > gpurun_out/d_steps.log
