"""Experiment: residual phase clocks and FP64 latencies (needs the
MHDG_RES_TIMING build: MHDG_LIB=paper_2507_22195_b200/libmhdg_timing.so)."""
import ctypes as C
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2507_22195_b200 import _native  # noqa: E402
from bench import make_problem, stage_alpha  # noqa: E402
from paper_2507_22195_b200.assembly import Discretization, StageContext  # noqa: E402
from paper_2507_22195_b200.fluxes import DissipationSpec  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 32
case = sys.argv[2] if len(sys.argv) > 2 else "tgv"
flux = os.environ.get("FLUX", "kepes" if case == "tgv" else "es")
P = int(os.environ.get("P", 3))
EB = {1: 8, 2: 3, 3: 2, 4: 1}[P]
gas, mesh, vx, _ = make_problem(case, n)
alpha = stage_alpha(0.57 if case == "tgv" else 0.01)
disc = Discretization(mesh, p=P, gas=gas, formulation="entropy", flux=DissipationSpec(flux),
                      device="cuda:0")
fields = disc.project(vx.initial)
stage = StageContext(alpha=alpha, offset=(-alpha * disc.volume_quad_states(fields)).contiguous())
lib = _native.load()
lib.mhdg_debug_latency.restype = C.c_double
lat = {k: lib.mhdg_debug_latency(v) for k, v in (("dfma", -1), ("log", 0), ("exp", 1), ("div", 2),
                                                  ("dmma_dependent", 3), ("dmma_4_chains_per_op", 4))}
buf = (C.c_ulonglong * 32)()   # the library copies all 32 counters
for _ in range(3):
    disc.residuals(fields, stage, sync=False)
torch.cuda.synchronize()
lib.mhdg_debug_res_clk(buf, C.c_int(1))
reps = 20
for _ in range(reps):
    disc.residuals(fields, stage, sync=False)
torch.cuda.synchronize()
lib.mhdg_debug_res_clk(buf, C.c_int(1))
E = disc.mesh.n_macros
groups = 148 * 4
iters = reps * (E / EB) / groups          # group iterations per group
names = ["top_barrier", "stage_data", "face_points", "vol_points+prefetch", "phase1_barrier",
         "contraction", "phase2_barrier", "combine+prefetch_tr", "contraction_face_warp"]
cyc = {nm: buf[i] / groups / iters for i, nm in enumerate(names)}
print(json.dumps({"latency_cycles": lat, "cycles_per_group_iteration": cyc,
                  "total": sum(cyc.values()), "p": P, "flux": flux, "n": n}, indent=1), flush=True)

