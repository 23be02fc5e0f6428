#!/usr/bin/env bash
# phase clocks of the Jacobian kernels (timing build travels as libmhdg_timing.so)
mkdir -p gpurun_out
MHDG_LIB=$PWD/paper_2507_22195_b200/libmhdg_timing.so python scripts/jac_phases.py > gpurun_out/jac_phases.json 2> gpurun_out/jac_phases.err; echo "rc=$?"
cat gpurun_out/jac_phases.json; tail -3 gpurun_out/jac_phases.err
