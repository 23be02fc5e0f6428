"""Jacobian build time (linearize + S^-1 + face-block inverses) and the
Gauss-Jordan pivoting-fallback counts on configs 2 / 3."""
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
from paper_2507_22195_b200.assembly import StageContext  # noqa: E402
from paper_2507_22195_b200.cases import IsentropicVortex, TaylorGreen  # noqa: E402
from paper_2507_22195_b200.mesh import build_box_macro_mesh  # noqa: E402

gas = GasModel(1.4)
out = []
for case, n, flux, dt, ptc in (("vortex", 16, "es", 0.01, 1.0), ("tgv", 32, "kepes", 0.57, 1.0),
                               ("tgv", 32, "kepes", 2.28, 1e-8), ("tgv", 16, "kepes", 0.01425, 1.0)):
    if case == "tgv":
        ic = TaylorGreen(mach=0.1, gas=gas)
        mesh = build_box_macro_mesh(ic.box, n, 1)
    else:
        ic = IsentropicVortex(dim=3, mach=1 / math.sqrt(1.4), strength=5.0, center=(5.0, 5.0), gas=gas)
        mesh = build_box_macro_mesh(np.array([[0.0, 10.0]] * 3), n, 1)
    disc = Discretization(mesh, p=3, gas=gas, flux=DissipationSpec(flux), device="cuda:0")
    f = disc.project(ic.initial)
    alpha = 0.4358665215 / dt
    st = StageContext(alpha=alpha, offset=-alpha * disc.volume_quad_states(f), dt=dt)
    lin = disc.jacobian(f, st, ptc_weight=ptc)
    del lin
    torch.cuda.synchronize()
    ts = []
    for _ in range(3):
        t0 = time.perf_counter()
        lin = disc.jacobian(f, st, ptc_weight=ptc)
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t0)
        del lin
    out.append({"case": case, "n": n, "flux": flux, "dt": dt, "ptc": ptc, "macros": mesh.n_macros,
                "build_ms": 1e3 * min(ts), "fallbacks": disc.gj_fallbacks()})
    print(json.dumps(out[-1]), flush=True)
    del disc, f
    torch.cuda.empty_cache()
