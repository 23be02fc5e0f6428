"""One Jacobian build (for ncu): config 3 state at n = NCELLS (default 16)."""
import os
import sys

sys.path.insert(0, ".")
import torch  # noqa: E402

from bench import make_problem, stage_alpha  # noqa: E402
from paper_2507_22195_b200.assembly import Discretization, StageContext  # noqa: E402
from paper_2507_22195_b200.fluxes import DissipationSpec  # noqa: E402

n = int(os.environ.get("NCELLS", 16))
gas, mesh, ic, _ = make_problem("tgv", n)
alpha = stage_alpha(0.57)
disc = Discretization(mesh, p=3, gas=gas, flux=DissipationSpec("kepes"), device="cuda:0")
f = disc.project(ic.initial)
st = StageContext(alpha=alpha, offset=-alpha * disc.volume_quad_states(f), dt=0.57)
for _ in range(int(os.environ.get("REPS", 2))):
    lin = disc.jacobian(f, st, ptc_weight=1.0)
    del lin
torch.cuda.synchronize()
print("ok")
