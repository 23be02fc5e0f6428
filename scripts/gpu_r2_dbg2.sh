export CUDA_LAUNCH_BLOCKING=1
for m in host engine; do for t in 1e-9 1e-6; do for r in 60 30; do timeout 120 python scripts/dbg_kw4.py $m $t $r 2>&1 | tail -2; done; done; done
