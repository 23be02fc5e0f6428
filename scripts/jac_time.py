import os, sys, json, time, torch
sys.path.insert(0, os.getcwd())
from paper_2507_22195_b200 import Discretization, DissipationSpec, GasModel
from paper_2507_22195_b200.assembly import StageContext
from paper_2507_22195_b200.cases import TaylorGreen
from paper_2507_22195_b200.mesh import build_box_macro_mesh
gas = GasModel(1.4); case = TaylorGreen(mach=0.1, gas=gas)
mesh = build_box_macro_mesh(case.box, 16, 1)
disc = Discretization(mesh, p=3, gas=gas, flux=DissipationSpec("kepes"), device="cuda:0")
f = disc.project(case.initial); alpha = 0.4358665215 / 0.57
stage = StageContext(alpha=alpha, offset=-alpha * disc.volume_quad_states(f))
lin = disc.jacobian(f, stage, ptc_weight=1.0); del lin; torch.cuda.synchronize()
ts = []
for _ in range(5):
    t0 = time.perf_counter(); lin = disc.jacobian(f, stage, ptc_weight=1.0); torch.cuda.synchronize(); ts.append(time.perf_counter() - t0); del lin
y = disc.jacobian(f, stage, ptc_weight=1.0).matvec(torch.ones(disc.jacobian(f, stage, ptc_weight=1.0).trace_shape, dtype=torch.float64, device="cuda:0"))
print(json.dumps({"lib": os.path.basename(os.environ.get("MHDG_LIB", "default")), "jac_ms": 1e3 * min(ts), "chk": float(y.abs().sum())}))
