"""Experiment: condensed matvec time for each library variant (MHDG_LIB),
config-2 vortex Jacobian, CUDA events."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if "--child" not in sys.argv:
    for lib in sys.argv[1:]:
        subprocess.run([sys.executable, __file__, "--child"], env=dict(os.environ, MHDG_LIB=lib), check=False)
    sys.exit(0)

import numpy as np  # noqa: E402
import torch  # noqa: E402

sys.path.insert(0, ROOT)
from bench import make_problem  # noqa: E402
from paper_2507_22195_b200.assembly import Discretization, StageContext  # noqa: E402
from paper_2507_22195_b200.fluxes import DissipationSpec  # noqa: E402

gas, mesh, vx, alpha = make_problem(16, 3, "es")
disc = Discretization(mesh, p=3, gas=gas, formulation="entropy", flux=DissipationSpec("es"), device="cuda:0")
fields = disc.project(vx.initial)
stage = StageContext(alpha=alpha, offset=(-alpha * disc.volume_quad_states(fields)).contiguous())
lin = disc.jacobian(fields, stage, ptc_weight=1.0)
x = torch.as_tensor(np.random.default_rng(1).standard_normal(lin.trace_shape), device="cuda:0")
out = {"lib": os.path.basename(os.environ.get("MHDG_LIB", "default"))}
for name, fn in (("matvec", lambda: lin.matvec(x)), ("precond", lambda: lin.apply_preconditioner(x))):
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(50):
        y = fn()
    e1.record()
    torch.cuda.synchronize()
    out[name + "_ms"] = e0.elapsed_time(e1) / 50
    out[name + "_sum"] = float(y.abs().sum())
print(json.dumps(out), flush=True)
