import os, sys, json, time, torch
sys.path.insert(0, os.getcwd())
from paper_2507_22195_b200 import Discretization, DissipationSpec, GasModel
from paper_2507_22195_b200.assembly import StageContext
from paper_2507_22195_b200.cases import TaylorGreen
from paper_2507_22195_b200.mesh import build_box_macro_mesh
gas = GasModel(1.4); case = TaylorGreen(mach=0.1, gas=gas)
mesh = build_box_macro_mesh(case.box, int(os.environ.get("JAC_N", 16)), 1)
disc = Discretization(mesh, p=3, gas=gas, flux=DissipationSpec(os.environ.get("JAC_FLUX", "kepes")), device="cuda:0")
f = disc.project(case.initial); alpha = 0.4358665215 / 0.57
stage = StageContext(alpha=alpha, offset=-alpha * disc.volume_quad_states(f))
lin = disc.jacobian(f, stage, ptc_weight=1.0); del lin; torch.cuda.synchronize()
ts = []
keep = os.environ.get("JAC_KEEP") == "1"  # Newton's pattern: old system alive while the next builds
lin = None
for _ in range(5):
    if not keep:
        lin = None
    t0 = time.perf_counter(); lin = disc.jacobian(f, stage, ptc_weight=1.0); torch.cuda.synchronize(); ts.append(time.perf_counter() - t0)
lin = None
lin = disc.jacobian(f, stage, ptc_weight=1.0)
one = torch.ones(lin.trace_shape, dtype=torch.float64, device="cuda:0")
y = lin.matvec(one)
pz = lin.apply_preconditioner(torch.sin(torch.arange(one.numel(), device="cuda:0", dtype=torch.float64)).view(lin.trace_shape))
pchk = [float(pz.abs().sum()), float((pz * pz).sum()), lin.n_unsym]
print(json.dumps({"n": mesh.n_macros if hasattr(mesh, "n_macros") else None, "keep": keep, "all_ms": [round(1e3 * t, 2) for t in ts], "lib": os.path.basename(os.environ.get("MHDG_LIB", "default")), "jac_ms": 1e3 * min(ts), "chk": float(y.abs().sum()), "pchk": pchk}))
