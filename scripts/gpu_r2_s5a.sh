#!/usr/bin/env bash
# session 5: residual phase clocks (timing build), ncu --set full of k_residual at config 3, config-5 sweep
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
MHDG_LIB=paper_2507_22195_b200/libmhdg_timing.so timeout 300 python scripts/res_timing.py 32 tgv > gpurun_out/res_timing_tgv32.json 2> gpurun_out/res_timing.err; echo "timing rc=$?"
cat gpurun_out/res_timing_tgv32.json
NCELLS=32 REPS=20 timeout 300 python scripts/res_bench.py > gpurun_out/resb.log 2>&1; cat gpurun_out/resb.log | tail -2
NCELLS=32 REPS=3 timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_residual -s 3 -c 1 \
    -o gpurun_out/prof_res -f python scripts/res_bench.py > gpurun_out/ncu_res.log 2>&1; echo "ncu rc=$?"
SWEEP_ARGS="--reps 10" bash scripts/gpu_sweep.sh
tail -c 2500 gpurun_out/sweep.json
