"""Experiment: phase clocks of k_linearize2 and the Gauss-Jordan kernels
(timing build, -DMHDG_RES_TIMING), Taylor-Green KEPES or vortex ES."""
import ctypes as C
import json
import os
import sys

import torch

sys.path.insert(0, os.getcwd())
from paper_2507_22195_b200 import Discretization, DissipationSpec, GasModel, _native  # noqa: E402
from paper_2507_22195_b200.assembly import StageContext  # noqa: E402
from paper_2507_22195_b200.cases import TaylorGreen  # noqa: E402
from paper_2507_22195_b200.mesh import build_box_macro_mesh  # noqa: E402

gas = GasModel(1.4)
case = TaylorGreen(mach=0.1, gas=gas)
n = int(os.environ.get("JAC_N", 16))
mesh = build_box_macro_mesh(case.box, n, 1)
disc = Discretization(mesh, p=3, gas=gas, flux=DissipationSpec(os.environ.get("JAC_FLUX", "kepes")), device="cuda:0")
f = disc.project(case.initial)
alpha = 0.4358665215 / 0.57
stage = StageContext(alpha=alpha, offset=-alpha * disc.volume_quad_states(f))
lib = _native.load()
buf = (C.c_ulonglong * 32)()
lin = disc.jacobian(f, stage, ptc_weight=1.0)
torch.cuda.synchronize()
lib.mhdg_debug_res_clk(buf, C.c_int(1))
del lin
lin = disc.jacobian(f, stage, ptc_weight=1.0)
torch.cuda.synchronize()
lib.mhdg_debug_res_clk(buf, C.c_int(1))
E, F = mesh.n_macros, disc.n_faces
names = ["lin_load", "lin_vol_duals", "lin_vol_S", "lin_face_duals", "lin_face_blocks"]
out = {nm: buf[i] / E for i, nm in enumerate(names)}
gn = ["load", "panel_busy", "update_busy", "interval_total", "store"]
out.update({"gj100_" + nm: buf[5 + i] / E for i, nm in enumerate(gn)})
out.update({"gj50_" + nm: buf[10 + i] / F for i, nm in enumerate(gn)})
pn = ["chain_D", "chain_gj8x8", "chain_publish", "unused"]
out.update({"gj100_bp_" + nm: buf[16 + i] / E for i, nm in enumerate(pn)})
out.update({"gj50_bp_" + nm: buf[21 + i] / F for i, nm in enumerate(pn)})
out.update({f"lin_face_round{i}": buf[26 + i] / E for i in range(3)})
print(json.dumps(out, indent=1))
