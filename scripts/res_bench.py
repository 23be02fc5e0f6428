"""Experiment: residual kernel time for each library variant given on the
command line (MHDG_LIB paths), config-2 vortex state, CUDA events."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

if len(sys.argv) > 2 or (len(sys.argv) == 2 and sys.argv[1].endswith(".so") and "MHDG_LIB" not in os.environ):
    for lib in sys.argv[1:]:
        env = dict(os.environ, MHDG_LIB=lib)
        subprocess.run([sys.executable, __file__, "--child"], env=env, check=False)
    sys.exit(0)

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
disc = Discretization(mesh, p=p, gas=gas, formulation="entropy", flux=DissipationSpec(flux),
                      device="cuda:0")
fields = disc.project(ic.initial)
stage = StageContext(alpha=alpha, offset=(-alpha * disc.volume_quad_states(fields)).contiguous())
for _ in range(5):
    disc.residuals(fields, stage, sync=False)
torch.cuda.synchronize()
reps = int(os.environ.get("REPS", 50))
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(reps):
    r = disc.residuals(fields, stage, sync=False)
e1.record()
torch.cuda.synchronize()
print(json.dumps({"lib": os.path.basename(os.environ.get("MHDG_LIB", "default")), "case": case, "n": n,
                  "flux": flux, "residual_ms": e0.elapsed_time(e1) / reps,
                  "checksum": float(r.r_w.abs().sum() + r.r_trace.abs().sum())}), flush=True)
