"""Experiment: phase clocks of k_linearize2 (timing build), config-2 vortex."""
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

flux = sys.argv[1] if len(sys.argv) > 1 else "es"
gas, mesh, vx, alpha = make_problem(16, 3, flux)
disc = Discretization(mesh, p=3, gas=gas, formulation="entropy", flux=DissipationSpec(flux), device="cuda:0")
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
names = ["load", "vol_duals", "vol_S_assembly", "face_duals", "face_blocks"]
print(json.dumps({nm: buf[i] / E for i, nm in enumerate(names)}, indent=1))
