"""State difference between the literal condensed solve and the Arnoldi
shortcuts after DIRK steps of a config (one process, same discretization)."""
import argparse
import json
import math
import os
import sys

import numpy as np

sys.path.insert(0, ".")
import __graft_entry__  # noqa: E402

__graft_entry__.build()
import torch  # noqa: E402

from paper_2507_22195_b200 import Discretization, DissipationSpec, GasModel  # noqa: E402
from paper_2507_22195_b200.cases import IsentropicVortex, TaylorGreen  # noqa: E402
from paper_2507_22195_b200.mesh import build_box_macro_mesh  # noqa: E402
from paper_2507_22195_b200.time_march import DIRKIntegrator  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--case", default="tgv")
ap.add_argument("--n", type=int, default=32)
ap.add_argument("--flux", default="kepes")
ap.add_argument("--dt", type=float, default=0.01425)
ap.add_argument("--steps", type=int, default=2)
ap.add_argument("--pair", default="modes", choices=["modes", "literal-host-vs-graph"],
                help="modes: literal loop vs Arnoldi shortcuts; literal-host-vs-graph: the literal loop run by the\n"
                     "host-driven control against the device graph (they differ by round-off only: a yardstick)")
a = ap.parse_args()
gas = GasModel(1.4)
if a.case == "vortex":
    case = IsentropicVortex(dim=3, mach=1 / math.sqrt(1.4), strength=5.0, center=(5.0, 5.0), gas=gas)
    box = np.array([[0.0, 10.0]] * 3)
else:
    case = TaylorGreen(mach=0.1, gas=gas)
    box = case.box
disc = Discretization(build_box_macro_mesh(box, a.n, 1), p=3, gas=gas, flux=DissipationSpec(a.flux), device="cuda:0")
out = {}
runs = (("true", "graph"), ("arnoldi", "graph")) if a.pair == "modes" else (("true", "host"), ("true", "graph"))
for idx, (mode, ctl) in enumerate(runs):
    os.environ["MHDG_INNER_RESIDUAL"] = mode
    os.environ["MHDG_KRYLOV"] = ctl
    mode = ("true", "arnoldi")[idx]   # slot names of the comparison below
    integ = DIRKIntegrator(disc)
    fields, t = integ.run(disc.project(case.initial), t_final=a.steps * a.dt, dt=a.dt)
    torch.cuda.synchronize()
    out[mode] = (fields.w.clone(), fields.trace.clone(),
                 [(r["newton_iters"], r["fgmres_iters"], r["inner_iters_total"]) for r in integ.records])
(wt, tt, ct), (wa, ta, ca) = out["true"], out["arnoldi"]
rel = lambda x, y: float(torch.linalg.vector_norm(x - y) / torch.linalg.vector_norm(y))   # noqa: E731
print(json.dumps({"pair": a.pair, "case": a.case, "n": a.n, "steps": a.steps, "counts_identical": ct == ca, "counts": ct,
                  "rel_diff_w": rel(wa, wt), "rel_diff_trace": rel(ta, tt),
                  "max_abs_diff_w": float((wa - wt).abs().max())}))
