"""Semi-discrete entropy balance of the device residual (the
reference's test_entropy_identity_face_constant_traces, assembly.py:649-672).

With a constant volume state and per-face-constant trace values the
identity sum(v . R_w) - sum(vhat . R_trace) = -sum(face entropy residuals)
is quadrature-exact: the entropy-conservative flux leaves zero, the ES and
KEPES dissipation a positive production."""

import numpy as np
import pytest

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
