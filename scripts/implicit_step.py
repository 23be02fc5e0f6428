"""Time one (or more) DIRK(3,3) implicit steps of a config on the device."""
import argparse
import json
import math
import os
import sys
import time

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
ap.add_argument("--case", default="vortex")
ap.add_argument("--n", type=int, default=16)
ap.add_argument("--p", type=int, default=3)
ap.add_argument("--flux", default="es")
ap.add_argument("--dt", type=float, default=0.01)
ap.add_argument("--steps", type=int, default=1)
ap.add_argument("--viscous", action="store_true")
a = ap.parse_args()
gas = GasModel(1.4)
if a.case == "vortex":
    box = np.array([[0.0, 10.0]] * 3)
    case = IsentropicVortex(dim=3, mach=1 / math.sqrt(1.4), strength=5.0, center=(5.0, 5.0), gas=gas)
else:
    case = TaylorGreen(mach=0.1, gas=gas)
    box = case.box
t0 = time.time()
mesh = build_box_macro_mesh(box, a.n, 1)
visc = case.viscous_params(1600.0, prandtl=0.71) if a.viscous else None
disc = Discretization(mesh, p=a.p, gas=gas, flux=DissipationSpec(a.flux), viscosity=visc,
                      device="cuda:0")
fields = disc.project(case.initial)
setup = time.time() - t0
integ = DIRKIntegrator(disc)
torch.cuda.synchronize()
t1 = time.time()
fields, t = integ.run(fields, t_final=a.steps * a.dt, dt=a.dt)
torch.cuda.synchronize()
wall = time.time() - t1
keys = ("newton_iters", "fgmres_iters", "inner_iters_total", "jacobian_builds", "condense_seconds",
        "matvec_seconds", "recovery_seconds")
tot = {k: sum(r[k] for r in integ.records) for k in keys}
print(json.dumps({"case": a.case, "viscous": a.viscous, "n": a.n, "p": a.p, "macros": mesh.n_macros,
                  "setup_s": setup, "gpu_mem_gb": torch.cuda.max_memory_allocated() / 1e9,
                  "steps": a.steps, "wall_s": wall, "s_per_step": wall / a.steps, "totals": tot,
                  "state": {"w_l2": float(torch.linalg.vector_norm(fields.w)),
                            "trace_l2": float(torch.linalg.vector_norm(fields.trace)),
                            "w_sum": float(fields.w.sum()), "t": float(t)},
                  "krylov_modes": {k: os.environ.get(k, "default") for k in
                                   ("MHDG_INNER_RESIDUAL", "MHDG_OUTER_MATVEC", "MHDG_KRYLOV")},
                  "records": integ.records}))
