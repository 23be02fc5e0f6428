#!/usr/bin/env bash
python scripts/jac_bench.py 2>&1 | grep build_ms | head -2
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_partition.py tests/test_gpu_partition_mp.py tests/test_gpu_solver.py tests/test_gpu_steps.py -q 2>&1 | tail -2
