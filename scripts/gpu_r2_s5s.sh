#!/usr/bin/env bash
# config 3, 10 DIRK steps: the literal Krylov loop against the Arnoldi shortcuts (counts per stage, final state)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
MHDG_INNER_RESIDUAL=true timeout 900 python scripts/implicit_step.py --case tgv --n 32 --flux kepes --dt 0.01425 --steps 10 > gpurun_out/imp_c3_10steps_true.json 2> gpurun_out/imp10.err; echo "true rc=$?"
timeout 900 python scripts/implicit_step.py --case tgv --n 32 --flux kepes --dt 0.01425 --steps 10 > gpurun_out/imp_c3_10steps_arnoldi.json 2>> gpurun_out/imp10.err; echo "arnoldi rc=$?"
python - <<'PY'
import json
a = json.load(open("gpurun_out/imp_c3_10steps_true.json")); b = json.load(open("gpurun_out/imp_c3_10steps_arnoldi.json"))
ca = [(r["newton_iters"], r["fgmres_iters"], r["inner_iters_total"], r["jacobian_builds"]) for r in a["records"]]
cb = [(r["newton_iters"], r["fgmres_iters"], r["inner_iters_total"], r["jacobian_builds"]) for r in b["records"]]
print("stages", len(ca), "identical counts:", ca == cb, "first difference:", next((i for i, (x, y) in enumerate(zip(ca, cb)) if x != y), None))
print("true   ", a["wall_s"], a["totals"], a["state"])
print("arnoldi", b["wall_s"], b["totals"], b["state"])
rel = lambda k: abs(a["state"][k] - b["state"][k]) / abs(a["state"][k])
print("relative difference of the final state norms:", rel("w_l2"), rel("trace_l2"), rel("w_sum"))
PY
