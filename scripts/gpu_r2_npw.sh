#!/usr/bin/env bash
for v in npw4 npw1 npw2 npw4 npw1 npw2; do echo "== $v"; MHDG_LIB=paper_2507_22195_b200/libmhdg_$v.so python scripts/jac_bench.py 2>&1 | grep build_ms | head -2; done
