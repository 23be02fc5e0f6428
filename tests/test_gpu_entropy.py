"""Semi-discrete entropy balance of the device residual (the
reference's test_entropy_identity_face_constant_traces, assembly.py:649-672).

With a constant volume state and per-face-constant trace values the
identity sum(v . R_w) - sum(vhat . R_trace) = -sum(face entropy residuals)
is quadrature-exact: the entropy-conservative flux leaves zero, the ES and
KEPES dissipation a positive production."""

import os

import numpy as np
import pytest

from helpers import GOLDEN

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("flux", ["ec", "es", "kepes"])
def test_entropy_balance_face_constant_traces(cuda_ok, flux):
    import torch

    from paper_2507_22195_b200 import Discretization, DissipationSpec, GasModel
    from paper_2507_22195_b200.mesh import build_box_macro_mesh

    gas = GasModel(1.4)
    disc = Discretization(build_box_macro_mesh(np.array([[0.0, 1.0]] * 3), 2, 1), p=2, gas=gas,
                          formulation="entropy", flux=DissipationSpec(flux), device="cuda:0")
    u0 = gas.conservative(1.1, np.array([0.3, -0.2, 0.1]), 0.9)
    fields = disc.project(lambda x: np.broadcast_to(u0, x.shape[:-1] + (5,)).copy())
    rng = np.random.default_rng(7)
    noise = 0.05 * rng.standard_normal((fields.trace.shape[0], 1, 5))
    fields.trace = fields.trace + torch.from_numpy(noise).to(fields.trace.device)
    res = disc.residuals(fields)
    lhs = float((fields.w * res.r_w).sum()) - float((fields.trace * res.r_trace).sum())
    scale = float((fields.w * res.r_w).abs().sum()) + float((fields.trace * res.r_trace).abs().sum())
    assert scale > 1e-4                  # the residual itself is not trivially zero
    if flux == "ec":
        assert abs(lhs) <= 1e-11 * max(1.0, scale)
    else:
        assert lhs > 1e-8 * scale    # dissipation produces entropy


@pytest.mark.parametrize("case", ["k2_es", "k2_kepes", "k2_ec", "k3_kepes", "tgv_k3_kepes"])
def test_entropy_identity_defect_matches_reference(cuda_ok, case):
    """Discretization.entropy_identity_defect on the device (assembly.py:
    649-672: sum v.R_V - sum v^.R_V^ against the face entropy residuals of
    fluxes.py:245-255) against the reference's values on the same states."""
    from paper_2507_22195_b200 import Discretization, DissipationSpec, GasModel
    from paper_2507_22195_b200.assembly import FieldSet
    from paper_2507_22195_b200.mesh import build_box_macro_mesh

    z = np.load(os.path.join(GOLDEN, "entropy_identity.npz"))
    p = int(case.split("_")[-2][1])
    flux = case.split("_")[-1]
    if case.startswith("tgv"):
        from paper_2507_22195_b200 import TaylorGreen

        box, n = TaylorGreen(mach=0.1).box, 2
    else:
        box, n = np.array([[0.0, 1.0]] * 3), (2, 2, 2)
    disc = Discretization(build_box_macro_mesh(box, n, 1), p=p, gas=GasModel(1.4),
                          formulation="entropy", flux=DissipationSpec(flux), device="cuda:0")
    lhs, rhs, dfc = disc.entropy_identity_defect(FieldSet(z[f"{case}_w"], z[f"{case}_trace"]))
    for got, key in ((lhs, "lhs"), (rhs, "rhs"), (dfc, "defect")):
        want = float(z[f"{case}_{key}"])
        assert abs(got - want) <= 1e-12 * max(1.0, abs(want)), (case, key, got, want)
