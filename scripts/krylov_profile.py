"""Per-call device timings of the Krylov building blocks for one config."""
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
from paper_2507_22195_b200.assembly import StageContext  # noqa: E402
from paper_2507_22195_b200.cases import TaylorGreen  # noqa: E402
from paper_2507_22195_b200.mesh import build_box_macro_mesh  # noqa: E402
from paper_2507_22195_b200 import solver as S  # noqa: E402

if os.environ.get("SOLVER_FILE"):  # A/B another solver.py
    import importlib.util

    _spec = importlib.util.spec_from_file_location("paper_2507_22195_b200._solver_ab",
                                                   os.environ["SOLVER_FILE"])
    S = importlib.util.module_from_spec(_spec)
    sys.modules[_spec.name] = S
    _spec.loader.exec_module(S)

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=16)
ap.add_argument("--p", type=int, default=3)
ap.add_argument("--flux", default="kepes")
ap.add_argument("--viscous", action="store_true")
a = ap.parse_args()
gas = GasModel(1.4)
case = TaylorGreen(mach=0.1, gas=gas)
mesh = build_box_macro_mesh(case.box, a.n, 1)
visc = case.viscous_params(1600.0, prandtl=0.71) if a.viscous else None
disc = Discretization(mesh, p=a.p, gas=gas, flux=DissipationSpec(a.flux), viscosity=visc,
                      device="cuda:0")
f = disc.project(case.initial)
dt = 0.57
alpha = 0.4358665215 / dt
u = disc.volume_quad_states(f)
stage = StageContext(alpha=alpha, offset=-alpha * u, dt=dt)
res = disc.residuals(f, stage)
torch.cuda.synchronize()
t0 = time.perf_counter()
lin = disc.jacobian(f, stage, ptc_weight=1.0)
torch.cuda.synchronize()
out = {"n": a.n, "viscous": a.viscous, "jacobian_s": time.perf_counter() - t0}
vec = S.DeviceVectors(disc)
x = lin.condensed_rhs(res)
shape = lin.trace_shape


def timeit(fn, reps=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps, (time.perf_counter() - t0) / reps * 1e3


out["residual_ms"] = timeit(lambda: disc.residuals(f, stage, sync=False))
out["matvec_ms"] = timeit(lambda: lin.matvec(x))
out["precond_ms"] = timeit(lambda: lin.apply_preconditioner(x))
V = torch.randn((61, x.numel()), dtype=torch.float64, device="cuda:0")
w = torch.randn(x.numel(), dtype=torch.float64, device="cuda:0")
out["mgs20_ms"] = timeit(lambda: vec.mgs(V, 19, w))
out["mgs1_ms"] = timeit(lambda: vec.mgs(V, 0, w))
b = x.reshape(-1)
op = lambda v: lin.matvec(v.view(shape)).view(-1)
pc = lambda v: lin.apply_preconditioner(v.view(shape)).view(-1)
out["inner20_ms"] = timeit(lambda: S.fgmres(op, b, precond=pc, rel_tol=1e-30, restart=20,
                                           max_iters=20, raise_on_stagnation=False, vec=vec),
                           reps=5)


def host_us(fn, reps=50):
    """Host-side cost per call while the GPU queue is kept full."""
    fn()
    torch.cuda.synchronize()
    torch.cuda._sleep(2_000_000_000)
    t0 = time.perf_counter()
    for _ in range(reps):
        fn()
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    return (t1 - t0) / reps * 1e6


out["host_us"] = {"matvec": host_us(lambda: lin.matvec(x)),
                  "precond": host_us(lambda: lin.apply_preconditioner(x)),
                  "combine": host_us(lambda: vec.combine(V, 10, np.ones(10), w), reps=20),
                  "div_into": host_us(lambda: vec.div_into(w, 2.0, V[0]))}
print(json.dumps(out))
