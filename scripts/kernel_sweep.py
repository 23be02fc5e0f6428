"""Config 5 kernel sweep (BASELINE.json configs[4]).

build_box_macro_mesh([[0,1]]^3, (32,32,43), m=1) -> 264,192 macros, seeded
perturbed-uniform states (per C0 node, then per trace node: rho~U[.9,1.1],
V_i~U[-.5,.5], P~U[.9,1.1]), alpha = d00/dt with dt = 0.01, offset =
-alpha * volume_quad_states, ptc_weight = 1, x ~ N(0,1) (seed+1).  For each
degree k: residual, Jacobian build (linearize + S^-1 + face-block factor),
condensed matvec, face-block apply; device times with CUDA events, averaged
over --reps launches, and the algorithmic rooflines of bench.py.

usage: python scripts/kernel_sweep.py [--degrees 1,2,3,4] [--cells 32,32,43]
"""
import argparse
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import __graft_entry__  # noqa: E402

__graft_entry__.build()
import torch  # noqa: E402

from paper_2507_22195_b200 import Discretization, DissipationSpec, GasModel  # noqa: E402
from paper_2507_22195_b200 import _native as N  # noqa: E402
from paper_2507_22195_b200.assembly import FieldSet, StageContext  # noqa: E402
from paper_2507_22195_b200.mesh import build_box_macro_mesh  # noqa: E402
from paper_2507_22195_b200.time_march import dirk33_tableau  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--degrees", default="1,2,3,4")
ap.add_argument("--cells", default="32,32,43")
ap.add_argument("--flux", default="es")
ap.add_argument("--reps", type=int, default=10)
ap.add_argument("--seed", type=int, default=2025)
a = ap.parse_args()
cells = tuple(int(c) for c in a.cells.split(","))
GAS = GasModel(1.4)
peaks = {}
try:
    peaks = json.load(open(os.path.join(os.path.dirname(__file__), "..", "MEASURED_PEAKS.json")))
except (OSError, ValueError):
    pass
HBM = float(peaks.get("hbm_gbs", 6650.0))
FP64 = max(N.fp64_probe(0), N.dmma_probe(0)) / 1e3   # the larger of the FMA and DMMA probes


def perturbed_uniform(disc, seed):
    rng = np.random.default_rng(seed)

    def states(n):
        rho = rng.uniform(0.9, 1.1, n)
        vel = rng.uniform(-0.5, 0.5, (n, 3))
        p = rng.uniform(0.9, 1.1, n)
        return GAS.conservative(rho, vel, p)

    E, nc = disc.mesh.n_macros, disc.layout.n_unique
    F, nt = disc.n_faces, disc.layout.n_face_unique
    u_w = states(E * nc).reshape(E, nc, 5)
    u_t = states(F * nt).reshape(F, nt, 5)
    return FieldSet(w=disc.from_conservative(u_w), trace=disc.from_conservative(u_t))


def dev_time(fn, reps):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


t0 = time.time()
mesh = build_box_macro_mesh(np.array([[0.0, 1.0]] * 3), cells, 1)
print(f"mesh {mesh.n_macros} macros in {time.time() - t0:.1f} s", file=sys.stderr)
d00 = float(dirk33_tableau().d[0, 0])
out = {"config": "cfg5", "cells": cells, "macros": mesh.n_macros, "flux": a.flux,
       "hbm_peak_gbs": HBM, "fp64_peak_tflops": FP64, "degrees": {}}
for p in [int(x) for x in a.degrees.split(",")]:
    t0 = time.time()
    disc = Discretization(mesh, p=p, gas=GAS, flux=DissipationSpec(a.flux), device="cuda:0")
    fields = perturbed_uniform(disc, a.seed)
    setup = time.time() - t0
    dt = 0.01
    alpha = d00 / dt
    offset = -alpha * disc.volume_quad_states(fields)
    stage = StageContext(alpha=alpha, offset=offset, dt=dt)
    E, F = mesh.n_macros, disc.n_faces
    nc, nt = disc.layout.n_unique, disc.layout.n_face_unique
    nq, nqf = (p + 1) ** 3, (p + 1) ** 2
    NM, NB = 5 * nc, 5 * nt
    r_ms = dev_time(lambda: disc.residuals(fields, stage, check=False, sync=False), a.reps)
    lin = disc.jacobian(fields, stage, ptc_weight=1.0)   # warm (allocations)
    del lin
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    lin = disc.jacobian(fields, stage, ptc_weight=1.0)
    torch.cuda.synchronize()
    jac_s = time.perf_counter() - t1
    x = torch.from_numpy(np.random.default_rng(a.seed + 1).standard_normal((F, nt, 5))).to("cuda:0")
    mv_ms = dev_time(lambda: lin.matvec(x), a.reps)
    pc_ms = dev_time(lambda: lin.apply_preconditioner(x), a.reps)
    T = 20
    flops_res = E * (nq * (10 * nc * 5 + 150 + 2 * T) + 4 * nqf * (8 * nt * 5 + 190 + 8 * T))
    bytes_mv = 8 * E * NM * NM + 3 * 8 * E * 4 * nqf * 25 + 2 * 8 * F * nt * 5 + 4 * E * 4 * (1 + nt) + 32 * E
    bytes_pc = 8 * F * NB * NB + 2 * 8 * F * nt * 5
    rec = {
        "setup_s": setup, "jacobian_build_s": jac_s,
        "residual": {"ms": r_ms, "tflops": flops_res / r_ms / 1e9,
                     "frac_fp64": flops_res / r_ms / 1e9 / FP64,
                     "dofs_per_s": (E * nc * 5 + F * nt * 5) / (r_ms * 1e-3)},
        "matvec": {"ms": mv_ms, "gbs": bytes_mv / mv_ms / 1e6, "frac_hbm": bytes_mv / mv_ms / 1e6 / HBM,
                   "dofs_per_s": F * nt * 5 / (mv_ms * 1e-3)},
        "precond": {"ms": pc_ms, "gbs": bytes_pc / pc_ms / 1e6, "frac_hbm": bytes_pc / pc_ms / 1e6 / HBM},
        "gpu_mem_gb": torch.cuda.max_memory_allocated() / 1e9,
    }
    out["degrees"][p] = rec
    print(json.dumps({p: rec}), file=sys.stderr)
    del lin, disc, fields, offset, stage, x
    torch.cuda.empty_cache()
    torch.cuda.reset_peak_memory_stats()
print(json.dumps(out))
