"""Experiment: condensed matvec / face-block apply time per library variant
(MHDG_LIB paths on the command line), Taylor-Green or vortex state, CUDA
events.  Environment: CASE, NCELLS, P, FLUX, REPS."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if len(sys.argv) > 1 and sys.argv[1] != "--child":
    for lib in sys.argv[1:]:
        subprocess.run([sys.executable, __file__, "--child"], env=dict(os.environ, MHDG_LIB=lib), check=False)
    sys.exit(0)

import numpy as np  # noqa: E402
import torch  # noqa: E402

sys.path.insert(0, ROOT)
from bench import make_problem, stage_alpha  # noqa: E402
from paper_2507_22195_b200.assembly import Discretization, StageContext  # noqa: E402
from paper_2507_22195_b200.fluxes import DissipationSpec  # noqa: E402

case = os.environ.get("CASE", "tgv")
n, p = int(os.environ.get("NCELLS", 32)), int(os.environ.get("P", 3))
flux = os.environ.get("FLUX", "kepes" if case == "tgv" else "es")
gas, mesh, ic, _ = make_problem(case, n)
alpha = stage_alpha(0.57 if case == "tgv" else 0.01)
disc = Discretization(mesh, p=p, gas=gas, formulation="entropy", flux=DissipationSpec(flux), device="cuda:0")
fields = disc.project(ic.initial)
stage = StageContext(alpha=alpha, offset=(-alpha * disc.volume_quad_states(fields)).contiguous())
lin = disc.jacobian(fields, stage, ptc_weight=1.0)
x = torch.as_tensor(np.random.default_rng(1).standard_normal(lin.trace_shape), device="cuda:0")
out = {"lib": os.path.basename(os.environ.get("MHDG_LIB", "default")), "case": case, "n": n, "p": p}
reps = int(os.environ.get("REPS", 50))
for name, fn in (("matvec", lambda: lin.matvec(x)), ("precond", lambda: lin.apply_preconditioner(x))):
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        y = fn()
    e1.record()
    torch.cuda.synchronize()
    out[name + "_ms"] = e0.elapsed_time(e1) / reps
    out[name + "_checksum"] = float(y.abs().sum())
print(json.dumps(out), flush=True)
