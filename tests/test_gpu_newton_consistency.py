"""The linearization, condensation and recovery against the residual kernel
itself (the reference checks its complex-step Jacobian against
central differences at 1e-5 and the condensed Newton step against dense
monolithic elimination).

With ptc_weight = 0 the condensed system is the exact Newton system of
`residuals`: solve it tightly, recover d_w (and d_q), and the residual along
the step must fall linearly, R(u + eps d) = (1 - eps) R(u) + O(eps^2): the
ratio |R(u + eps d) - (1 - eps) R(u)| / (eps |R(u)|) halves with eps.  One
test covers k_linearize2 (duals), the S^-1 / face-block inverses, the
condensed matvec, rhs and recovery, and for the viscous case the level-1
gradient condensation."""

import math

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _setup(kind):
    from paper_2507_22195_b200 import Discretization, DissipationSpec, GasModel, TaylorGreen
    from paper_2507_22195_b200.cases import IsentropicVortex
    from paper_2507_22195_b200.mesh import build_box_macro_mesh

    gas = GasModel(1.4)
    case = IsentropicVortex(dim=3, mach=1 / math.sqrt(1.4), strength=5.0, center=(5.0, 5.0), gas=gas)
    mesh = build_box_macro_mesh(np.array([[0.0, 10.0]] * 3), 2, 1)
    if kind == "viscous":
        # ES flux: with ptc 0 the KEPES dissipation vanishes at the projected
        # (coincident) trace states and leaves near-null face blocks -- the
        # reason the reference adds the ptc term (assembly.py:895-902)
        visc = TaylorGreen(mach=0.1, gas=gas).viscous_params(1600.0, 0.71)
        disc = Discretization(mesh, p=2, gas=gas, formulation="entropy", flux=DissipationSpec("es"),
                              viscosity=visc, device="cuda:0")
        f = disc.project(case.initial)
        f.q = disc.solve_gradient(f)
        return disc, f, 0.25
    disc = Discretization(mesh, p=2, gas=gas, formulation="entropy", flux=DissipationSpec(kind),
                          device="cuda:0")
    return disc, disc.project(case.initial), 0.25


def _flat(res):
    import torch

    parts = [res.r_w, res.r_trace] + ([res.r_q] if res.r_q is not None else [])
    return torch.cat([p.reshape(-1) for p in parts])


@pytest.mark.parametrize("kind", ["es", "kepes", "viscous"])
def test_newton_step_linearizes_the_residual(cuda_ok, kind):
    from paper_2507_22195_b200 import solver
    from paper_2507_22195_b200.assembly import FieldSet, StageContext

    disc, f, dt = _setup(kind)
    alpha = 0.4358665215 / dt
    stage = StageContext(alpha=alpha, offset=-alpha * disc.volume_quad_states(f), dt=dt)
    res = disc.residuals(f, stage)
    lin = disc.jacobian(f, stage, ptc_weight=0.0)
    shape = lin.trace_shape
    b = lin.condensed_rhs(res).view(-1)
    sol = solver.fgmres(lambda v: lin.matvec(v.view(shape)).view(-1), b,
                        precond=lambda v: lin.apply_preconditioner(v.view(shape)).view(-1),
                        rel_tol=1e-13, restart=200, max_iters=2000, raise_on_stagnation=False,
                        vec=solver.DeviceVectors(disc))
    # KEPES face blocks are near-singular at coincident states (see above):
    # FGMRES stagnates around 1e-8 there, still far below the FD remainder
    assert sol.rel_residual <= 1e-7
    d_trace = sol.x.view(shape)
    d_w, d_q = lin.recover(res, d_trace)
    r0 = _flat(res)
    ratios = []
    # step length: the perturbation is 1e-4 of the state's scale
    e0 = 1e-4 * float(f.w.abs().max()) / max(float(d_w.abs().max()), float(d_trace.abs().max()))
    for eps in (e0, e0 / 2, e0 / 4):
        fe = FieldSet(f.w + eps * d_w, f.trace + eps * d_trace,
                      None if f.q is None else f.q + eps * d_q)
        re = _flat(disc.residuals(fe, stage))
        ratios.append(float((re - (1.0 - eps) * r0).norm() / (eps * r0.norm())))
    # the remainder is O(eps^2), so the ratio halves with eps; a wrong
    # Jacobian term would leave an eps-independent floor
    assert all(math.isfinite(r) for r in ratios), ratios
    assert ratios[1] <= 0.6 * ratios[0] and ratios[2] <= 0.6 * ratios[1], ratios
