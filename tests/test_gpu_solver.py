"""Device FGMRES and the condensed operator (test_solver.py
strategy, the device half): the solver on the library's vector kernels
against the CPU oracle, condensed-operator linearity, bitwise determinism of
the condensed solve, and the face-block preconditioner's benefit."""

import math

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _disc(n=2, p=2):
    from paper_2507_22195_b200 import Discretization, DissipationSpec, GasModel
    from paper_2507_22195_b200.cases import IsentropicVortex
    from paper_2507_22195_b200.mesh import build_box_macro_mesh

    gas = GasModel(1.4)
    case = IsentropicVortex(dim=3, mach=1 / math.sqrt(1.4), strength=5.0, center=(5.0, 5.0), gas=gas)
    disc = Discretization(build_box_macro_mesh(np.array([[0.0, 10.0]] * 3), n, 1), p=p, gas=gas,
                          formulation="entropy", flux=DissipationSpec("es"), device="cuda:0")
    return case, disc


def _system(disc, case, ptc=1.0):
    from paper_2507_22195_b200.assembly import StageContext

    f = disc.project(case.initial)
    alpha = 0.4358665215 / 0.01
    stage = StageContext(alpha=alpha, offset=-alpha * disc.volume_quad_states(f), dt=0.01)
    res = disc.residuals(f, stage)
    return disc.jacobian(f, stage, ptc_weight=ptc), res


@pytest.mark.parametrize("restart", [60, 6])
def test_device_fgmres_matches_oracle(cuda_ok, restart):
    import torch

    from oracle.hdg_oracle import fgmres as ofgmres
    from paper_2507_22195_b200 import solver

    _, disc = _disc()
    rng = np.random.default_rng(21)
    n = 300
    A = np.eye(n) + 0.3 * rng.standard_normal((n, n)) / np.sqrt(n)
    b = rng.standard_normal(n)
    Ad = torch.from_numpy(A).cuda()
    res = solver.fgmres(lambda v: Ad @ v, torch.from_numpy(b).cuda(), rel_tol=1e-10, restart=restart,
                        max_iters=300, vec=solver.DeviceVectors(disc))
    x_ref, it_ref, _, conv_ref = ofgmres(lambda v: A @ v, b, rel_tol=1e-10, restart=restart, max_iters=300)
    assert res.converged == conv_ref and res.iterations == it_ref
    assert np.abs(res.x.cpu().numpy() - x_ref).max() <= 1e-10 * np.abs(x_ref).max()


def test_condensed_operator_is_linear(cuda_ok):
    import torch

    case, disc = _disc()
    lin, _ = _system(disc, case)
    g = torch.Generator(device="cpu").manual_seed(5)
    x = torch.randn(lin.trace_shape, generator=g, dtype=torch.float64).cuda()
    y = torch.randn(lin.trace_shape, generator=g, dtype=torch.float64).cuda()
    a, b = 0.37, -1.9
    lhs = lin.matvec(a * x + b * y)
    rhs = a * lin.matvec(x) + b * lin.matvec(y)
    assert float((lhs - rhs).abs().max() / rhs.abs().max()) <= 1e-12


def test_condensed_solve_is_bitwise_deterministic(cuda_ok):
    import torch

    from paper_2507_22195_b200.solver import solve_condensed

    case, disc = _disc()
    lin, res = _system(disc, case)
    d1, s1 = solve_condensed(lin, res)
    d2, s2 = solve_condensed(lin, res)
    assert torch.equal(d1, d2)
    assert (s1.outer_iterations, s1.inner_iterations) == (s2.outer_iterations, s2.inner_iterations)


def test_face_block_preconditioner_reduces_iterations(cuda_ok):
    from paper_2507_22195_b200 import solver

    case, disc = _disc()
    lin, res = _system(disc, case, ptc=0.0)
    b = lin.condensed_rhs(res).view(-1)
    shape = lin.trace_shape
    vec = solver.DeviceVectors(disc)
    op = lambda v: lin.matvec(v.view(shape)).view(-1)                 # noqa: E731
    pc = lambda v: lin.apply_preconditioner(v.view(shape)).view(-1)   # noqa: E731
    plain = solver.fgmres(op, b, rel_tol=1e-8, restart=60, max_iters=600, raise_on_stagnation=False, vec=vec)
    pre = solver.fgmres(op, b, precond=pc, rel_tol=1e-8, restart=60, max_iters=600,
                        raise_on_stagnation=False, vec=vec)
    assert pre.converged and pre.iterations < plain.iterations
    # both solves reach rel. residual 1e-8 of an ill-conditioned operator
    # (ptc 0: ~500 unpreconditioned iterations); their solutions agree to
    # the condition number times that
    xr = (pre.x - plain.x).abs().max() / pre.x.abs().max()
    assert not plain.converged or float(xr) <= 1e-4


def test_ptc_weight_shifts_alpha_and_damps_trace(cuda_ok):
    """ptc_weight adds to alpha inside the local blocks and contributes a
    trace damping that is linear in the weight and absent from recovery
    (the reference's test_assembly.py:374-394)."""
    import torch

    from paper_2507_22195_b200.assembly import StageContext

    case, disc = _disc()
    f = disc.project(case.initial)
    lin_a = disc.jacobian(f, StageContext(alpha=1.0, dt=0.1), ptc_weight=0.7)
    lin_b = disc.jacobian(f, StageContext(alpha=1.7, dt=0.1))
    lin_c = disc.jacobian(f, StageContext(alpha=0.3, dt=0.1), ptc_weight=1.4)
    x = torch.from_numpy(np.random.default_rng(1).standard_normal(lin_a.trace_shape)).cuda()
    ya, yb, yc = lin_a.matvec(x), lin_b.matvec(x), lin_c.matvec(x)
    scale = max(1.0, float(yb.abs().max()))
    damp = ya - yb
    assert float(damp.abs().max()) > 1e-3 * scale
    assert float(((yc - yb) - 2.0 * damp).abs().max()) <= 1e-11 * scale
    res = disc.residuals(f, StageContext(alpha=1.0, dt=0.1))
    dw_a, _ = lin_a.recover(res, x)
    dw_b, _ = lin_b.recover(res, x)
    assert float((dw_a - dw_b).abs().max()) <= 1e-12 * max(1.0, float(dw_b.abs().max()))
