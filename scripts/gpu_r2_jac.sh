#!/usr/bin/env bash
python scripts/jac_bench.py > gpurun_out/jac.json 2> gpurun_out/jac.err; echo "jac rc=$?"; cat gpurun_out/jac.json
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -15
