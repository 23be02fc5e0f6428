"""Experiment: viscous condensed matvec time per library variant (MHDG_LIB),
viscous Taylor-Green n=16 k=3 KEPES (config-4 parameters)."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if "--child" not in sys.argv:
    for lib in sys.argv[1:]:
        subprocess.run([sys.executable, __file__, "--child"], env=dict(os.environ, MHDG_LIB=lib), check=False)
    sys.exit(0)

import torch  # noqa: E402

sys.path.insert(0, ROOT)
from paper_2507_22195_b200 import Discretization, DissipationSpec, GasModel  # noqa: E402
from paper_2507_22195_b200.assembly import StageContext  # noqa: E402
from paper_2507_22195_b200.cases import TaylorGreen  # noqa: E402
from paper_2507_22195_b200.mesh import build_box_macro_mesh  # noqa: E402

gas = GasModel(1.4)
case = TaylorGreen(mach=0.1, gas=gas)
mesh = build_box_macro_mesh(case.box, 16, 1)
disc = Discretization(mesh, p=3, gas=gas, flux=DissipationSpec("kepes"),
                      viscosity=case.viscous_params(1600.0, prandtl=0.71), device="cuda:0")
f = disc.project(case.initial)
alpha = 0.4358665215 / 0.57
stage = StageContext(alpha=alpha, offset=-alpha * disc.volume_quad_states(f), dt=0.57)
res = disc.residuals(f, stage)
lin = disc.jacobian(f, stage, ptc_weight=1.0)
x = lin.condensed_rhs(res)
out = {"lib": os.path.basename(os.environ.get("MHDG_LIB", "default"))}
for name, fn in (("matvec", lambda: lin.matvec(x)), ("residual", lambda: disc.residuals(f, stage, sync=False))):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20):
        y = fn()
    e1.record()
    torch.cuda.synchronize()
    out[name + "_ms"] = e0.elapsed_time(e1) / 20
out["matvec_sum"] = float(lin.matvec(x).abs().sum())
print(json.dumps(out), flush=True)
