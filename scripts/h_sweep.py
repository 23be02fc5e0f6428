"""Config-2 h-refinement study on the device (reference driver.py:570-606,
space axis): vortex on [0,10]^3 (centre (5,5), M = 1/sqrt(1.4), strength 5),
k = 3, ES; meshes n, 2n, 4n run to t_eval = 0.1 t_c with dt0 = t_eval / 10
shrunk by 2^((p+1)/3) per level; L2 error of rho against the exact translated
vortex (assembly.py:674-684) and log2 rates."""
import argparse
import json
import math
import sys
import time

import numpy as np

sys.path.insert(0, ".")
import __graft_entry__  # noqa: E402

__graft_entry__.build()
import torch  # noqa: E402

from paper_2507_22195_b200 import Discretization, DissipationSpec, GasModel  # noqa: E402
from paper_2507_22195_b200.cases import IsentropicVortex  # noqa: E402
from paper_2507_22195_b200.mesh import build_box_macro_mesh  # noqa: E402
from paper_2507_22195_b200.time_march import DIRKIntegrator  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=8)
ap.add_argument("--levels", type=int, default=3)
ap.add_argument("--p", type=int, default=3)
a = ap.parse_args()
gas = GasModel(1.4)
vx = IsentropicVortex(dim=3, mach=1 / math.sqrt(1.4), strength=5.0, v_inf=1.0, center=(5.0, 5.0),
                      gas=gas)
t_eval = 0.1 * vx.convective_period
dt0 = t_eval / 10.0
shrink = 2.0 ** ((a.p + 1) / 3.0)
rows = []
for level in range(a.levels):
    n = a.n * 2 ** level
    dt = dt0 / shrink ** level
    disc = Discretization(build_box_macro_mesh(np.array([[0.0, 10.0]] * 3), n, 1), p=a.p, gas=gas,
                          formulation="entropy", flux=DissipationSpec("es"), device="cuda:0")
    f = disc.project(vx.initial)
    integ = DIRKIntegrator(disc)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    f, t = integ.run(f, t_final=t_eval, dt=dt)
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
    err = disc.l2_error(f, lambda x: vx.state(x, t_eval), component=0)
    h = 10.0 / n
    rate = None if not rows else math.log2(rows[-1]["l2"] / err)
    steps = len({r["step"] for r in integ.records})
    rows.append({"level": level, "n": n, "macros": 6 * n ** 3, "h": h, "dt": dt, "steps": steps,
                 "l2": err, "rate": rate, "wall_s": wall,
                 "newton": sum(r["newton_iters"] for r in integ.records)})
    print(json.dumps(rows[-1]), flush=True)
    del disc, f, integ
    torch.cuda.empty_cache()
print(json.dumps({"study": "config2 h-sweep", "p": a.p, "t_eval": t_eval, "rows": rows}))
