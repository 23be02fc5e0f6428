#!/usr/bin/env bash
# Gauss-Jordan variants A/B: Jacobian build (config-3 mesh), phase clocks, GPU suite
mkdir -p gpurun_out
for v in b200 $VARIANTS; do
  MHDG_LIB=$PWD/paper_2507_22195_b200/libmhdg_$v.so JAC_N=${JAC_N:-32} python scripts/jac_time.py 2> gpurun_out/jt_$v.err | tee gpurun_out/jt_$v.json
done
MHDG_LIB=$PWD/paper_2507_22195_b200/libmhdg_timing.so python scripts/jac_phases.py > gpurun_out/jac_phases.json 2> gpurun_out/jac_phases.err; echo "rc=$?"
grep -v '"lin' gpurun_out/jac_phases.json; tail -3 gpurun_out/jac_phases.err
if [ "$1" != "notests" ]; then
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -15
fi
