"""m > 1 macro subdivision on the device (mhdg_macro.cuh) against
the reference: operator outputs on perturbed-uniform states for (m, p) =
(2,1), (2,2), (2,3), (3,1) (tests/golden/macro_m*_k*.npz), and one DIRK(3,3)
step of the config-1 vortex at m = 2, p = 2 (macro_m2_step.npz).
Tolerances as for m = 1: residual <= max(1e-12, 10x the reference's 1-ulp
sensitivity), condensed operators <= max(1e-11, 10x sensitivity), converged
state 1e-10 with identical Newton counts."""

import glob
import os

import numpy as np
import pytest

from helpers import GOLDEN, golden_mesh, load_golden, rel

pytestmark = pytest.mark.gpu

CASES = sorted(os.path.basename(f)[:-4] for f in glob.glob(os.path.join(GOLDEN, "macro_m*_k*.npz")))


def _disc(z):
    from paper_2507_22195_b200 import Discretization, DissipationSpec, GasModel

    return Discretization(golden_mesh(z), p=int(z["p"]), gas=GasModel(1.4), formulation="entropy",
                          flux=DissipationSpec(str(z["flux"])), device="cuda:0")


@pytest.mark.parametrize("name", CASES)
def test_macro_operator(cuda_ok, name):
    import torch

    from paper_2507_22195_b200.assembly import FieldSet, StageContext

    z = load_golden(name)
    disc = _disc(z)
    fields = FieldSet(z["w"], z["trace"])
    assert rel(disc.volume_quad_states(fields), z["vqs"]) <= 1e-14
    stage = StageContext(alpha=float(z["alpha"]), offset=z["offset"])
    res = disc.residuals(fields, stage)
    res2 = disc.residuals(fields, stage)
    assert torch.equal(res.r_w, res2.r_w) and torch.equal(res.r_trace, res2.r_trace)   # deterministic
    lin = disc.jacobian(fields, stage, ptc_weight=float(z["ptc"]))
    x = z["x"]
    got = dict(r_w=res.r_w, r_trace=res.r_trace, matvec=lin.matvec(x), rhs=lin.condensed_rhs(res),
               recover=lin.recover(res, x)[0], precond=lin.apply_preconditioner(x))
    for k, v in got.items():
        floor = 1e-12 if k in ("r_w", "r_trace") else 1e-11
        tol = max(floor, 10 * float(z[f"sens_{k}"]))
        assert rel(v, z[k]) <= tol, (name, k, rel(v, z[k]), tol)


def test_macro_step(cuda_ok):
    import math

    from paper_2507_22195_b200 import Discretization, DissipationSpec, GasModel
    from paper_2507_22195_b200.cases import IsentropicVortex
    from paper_2507_22195_b200.mesh import build_box_macro_mesh
    from paper_2507_22195_b200.time_march import DIRKIntegrator

    z = load_golden("macro_m2_step")
    gas = GasModel(1.4)
    vx = IsentropicVortex(dim=3, mach=1 / math.sqrt(1.4), strength=5.0, v_inf=1.0,
                          center=(5.0, 5.0), gas=gas)
    disc = Discretization(build_box_macro_mesh(np.array([[0.0, 10.0]] * 3), 2, 2), p=2, gas=gas,
                          formulation="entropy", flux=DissipationSpec("es"), device="cuda:0")
    f0 = disc.project(vx.initial)
    assert rel(f0.w, z["w0"]) == 0.0 and rel(f0.trace, z["trace0"]) == 0.0
    integ = DIRKIntegrator(disc)
    f1, _ = integ.run(f0, t_final=float(z["dt"]), dt=float(z["dt"]))
    newton = np.array([[r["step"], r["stage"], r["newton_iters"]] for r in integ.records])
    assert np.array_equal(newton, z["newton"][:, :3])
    assert rel(f1.w, z["w1"]) <= 1e-10 and rel(f1.trace, z["trace1"]) <= 1e-10
    keys = ("entropy", "thermo_entropy", "kinetic_energy", "mass", "total_energy")
    ints = np.array([[disc.integrals(f)[k] for k in keys] for f in (f0, f1)])
    assert np.all(np.abs(ints - z["integrals"]) <= 1e-12 * np.maximum(1.0, np.abs(z["integrals"])))


def test_macro_rejects_unsupported(cuda_ok):
    from paper_2507_22195_b200 import Discretization, DissipationSpec, GasModel
    from paper_2507_22195_b200.errors import InvalidConfig
    from paper_2507_22195_b200.mesh import build_box_macro_mesh

    with pytest.raises(InvalidConfig):
        Discretization(build_box_macro_mesh(np.array([[0.0, 1.0]] * 3), 1, 3), p=2,
                       gas=GasModel(1.4), flux=DissipationSpec("es"), device="cuda:0")
