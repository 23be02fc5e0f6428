#!/usr/bin/env bash
for v in ffma0 ffma1 ffma0 ffma1; do echo "== $v"; MHDG_LIB=paper_2507_22195_b200/libmhdg_$v.so python scripts/jac_bench.py 2>&1 | grep build_ms | head -2; done
MHDG_LIB=paper_2507_22195_b200/libmhdg_ffma1.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_newton_consistency.py tests/test_gpu_steps.py tests/test_gpu_viscous.py tests/test_gpu_configs.py -q 2>&1 | tail -3
