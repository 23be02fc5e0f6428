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

NCELL = int(sys.argv[1]) if len(sys.argv) > 1 else 16
gas, mesh, vx, alpha = make_problem(NCELL, 3, "es")
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
         12: "u_jobs", 13: "u_barrier_wait"}
# cycles per matrix: S^-1 (E matrices, N = 100, 13 panels) in slots 9..13,
# face blocks (2E matrices, N = 50, 7 panels) in slots 0..4
out = {"S_inverse_N100": {v: buf[k] / E for k, v in names.items()},
       "face_blocks_N50": {v: buf[k - 9] / (2 * E) for k, v in names.items()}}
out["S_inverse_N100"]["per_pivot_factor"] = out["S_inverse_N100"]["w0_factor_panel"] / (12 * 8)
out["face_blocks_N50"]["per_pivot_factor"] = out["face_blocks_N50"]["w0_factor_panel"] / (6 * 8)
npiv = E * 12 * 8
out["S_inverse_N100"]["pivot_phases"] = {"search+reduce": buf[5] / npiv, "prow_gather": buf[6] / npiv,
                                          "recip+scale": buf[7] / npiv, "update": buf[8] / npiv}
print(json.dumps(out, indent=1))
