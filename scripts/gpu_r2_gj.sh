#!/usr/bin/env bash
# block-panel Gauss-Jordan: build times + fallbacks, phase clocks, GPU suite
mkdir -p gpurun_out
python scripts/jac_bench.py > gpurun_out/jac.json 2> gpurun_out/jac.err; echo "jac rc=$?"; cat gpurun_out/jac.json; tail -3 gpurun_out/jac.err
if [ -f paper_2507_22195_b200/libmhdg_timing.so ]; then
MHDG_LIB=$PWD/paper_2507_22195_b200/libmhdg_timing.so python scripts/jac_phases.py > gpurun_out/jac_phases.json 2> gpurun_out/jac_phases.err; echo "rc=$?"
cat gpurun_out/jac_phases.json; tail -3 gpurun_out/jac_phases.err
fi
if [ "$1" != "notests" ]; then
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -15
fi
