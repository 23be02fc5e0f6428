"""Experiment: phase clocks of the lookahead Gauss-Jordan (timing build)."""
import ctypes as C
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2507_22195_b200 import _native  # noqa: E402
from bench import make_problem  # noqa: E402
from paper_2507_22195_b200.assembly import Discretization, StageContext  # noqa: E402
from paper_2507_22195_b200.fluxes import DissipationSpec  # noqa: E402

gas, mesh, vx, alpha = make_problem(16, 3, "es")
disc = Discretization(mesh, p=3, gas=gas, formulation="entropy", flux=DissipationSpec("es"), device="cuda:0")
fields = disc.project(vx.initial)
stage = StageContext(alpha=alpha, offset=(-alpha * disc.volume_quad_states(fields)).contiguous())
lib = _native.load()
buf = (C.c_ulonglong * 16)()
lin = disc.jacobian(fields, stage, ptc_weight=1.0)
torch.cuda.synchronize()
lib.mhdg_debug_res_clk(buf, C.c_int(1))
del lin
lin = disc.jacobian(fields, stage, ptc_weight=1.0)
torch.cuda.synchronize()
lib.mhdg_debug_res_clk(buf, C.c_int(1))
E = mesh.n_macros
names = {9: "w0_barrier_wait", 10: "w0_update_next_panel", 11: "w0_factor_panel",
         12: "u_jobs", 13: "u_barrier_wait", 14: "u_R_capture", 15: "u_named_barrier"}
# per matrix (all panels): S^-1 (E) and face blocks (F) both counted; report per E
print(json.dumps({v: buf[k] / (E + 2 * E) for k, v in names.items()}, indent=1))
