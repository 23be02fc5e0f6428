#!/usr/bin/env bash
# residual variants (offset prefetch / early trace prefetch), configs 3 and 2
for v in 00 10 01 11 00 11; do
  MHDG_LIB=paper_2507_22195_b200/libmhdg_res$v.so python scripts/res_bench.py 2>/dev/null
  CASE=vortex NCELLS=16 MHDG_LIB=paper_2507_22195_b200/libmhdg_res$v.so python scripts/res_bench.py 2>/dev/null
done
