"""Where one implicit DIRK step's time goes: per-operator device time
(each call bracketed by synchronize) vs the unsynchronised step wall time.
Config-2 vortex by default."""
import argparse
import collections
import json
import math
import sys
import time

import numpy as np

sys.path.insert(0, ".")
import __graft_entry__  # noqa: E402

__graft_entry__.build()
import torch  # noqa: E402

from paper_2507_22195_b200 import Discretization, DissipationSpec, GasModel  # noqa: E402
from paper_2507_22195_b200 import assembly as A  # noqa: E402
from paper_2507_22195_b200 import solver as S  # noqa: E402
from paper_2507_22195_b200.cases import IsentropicVortex  # noqa: E402
from paper_2507_22195_b200.mesh import build_box_macro_mesh  # noqa: E402
from paper_2507_22195_b200.time_march import DIRKIntegrator  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=16)
ap.add_argument("--p", type=int, default=3)
ap.add_argument("--case", default="vortex")
ap.add_argument("--dt", type=float, default=0.01)
a = ap.parse_args()
gas = GasModel(1.4)
if a.case == "vortex":
    case = IsentropicVortex(dim=3, mach=1 / math.sqrt(1.4), strength=5.0, center=(5.0, 5.0), gas=gas)
    mesh = build_box_macro_mesh(np.array([[0.0, 10.0]] * 3), a.n, 1)
    flux = "es"
else:
    from paper_2507_22195_b200.cases import TaylorGreen
    case = TaylorGreen(mach=0.1, gas=gas)
    mesh = build_box_macro_mesh(case.box, a.n, 1)
    flux = "kepes"
disc = Discretization(mesh, p=a.p, gas=gas, flux=DissipationSpec(flux), device="cuda:0")
fields0 = disc.project(case.initial)

# unsynchronised reference timing (second step of a warm run)
integ = DIRKIntegrator(disc)
f1, _ = integ.run(fields0, t_final=a.dt, dt=a.dt)
torch.cuda.synchronize()
t0 = time.perf_counter()
integ2 = DIRKIntegrator(disc)
integ2.run(fields0, t_final=a.dt, dt=a.dt)
torch.cuda.synchronize()
wall = time.perf_counter() - t0

acc = collections.defaultdict(lambda: [0, 0.0])


def wrap(obj, name, key):
    fn = getattr(obj, name)

    def w(*args, **kw):
        torch.cuda.synchronize()
        s = time.perf_counter()
        out = fn(*args, **kw)
        torch.cuda.synchronize()
        acc[key][0] += 1
        acc[key][1] += time.perf_counter() - s
        return out
    setattr(obj, name, w)


for name in ("residuals", "jacobian", "volume_quad_states", "to_conservative", "from_conservative"):
    wrap(A.Discretization, name, name)
for name in ("matvec", "condensed_rhs", "recover", "apply_preconditioner"):
    wrap(A.LinearizedSystem, name, name)
for name in ("mgs", "norm", "combine", "div_into", "axpby"):
    wrap(S.DeviceVectors, name, "vec." + name)
torch.cuda.synchronize()
t0 = time.perf_counter()
integ3 = DIRKIntegrator(disc)
integ3.run(fields0, t_final=a.dt, dt=a.dt)
torch.cuda.synchronize()
wall_sync = time.perf_counter() - t0
out = {"wall_s": wall, "wall_synced_s": wall_sync,
       "ops": {k: {"calls": v[0], "s": round(v[1], 4)} for k, v in sorted(acc.items(), key=lambda kv: -kv[1][1])},
       "sum_ops_s": sum(v[1] for v in acc.values())}
# jacobian = nested: matvec etc. not inside; fgmres host work = remainder
print(json.dumps(out, indent=1))
