"""FGMRES control flow against the CPU oracle (the reference's
test_solver.py strategy): identity / diagonal / random systems, restarts,
stagnation, zero right-hand side, flexible preconditioning.  The product's
`solver.fgmres` runs here on a CPU test double of the device vector kernels
(`helpers.CPUVectors`); the same solver on the device vectors is in
test_gpu_solver.py."""

import numpy as np
import pytest
import torch

from helpers import CPUVectors
from oracle.hdg_oracle import fgmres as ofgmres
from paper_2507_22195_b200 import solver
from paper_2507_22195_b200.errors import KrylovStagnation


def _solve(A, b, **kw):
    At = torch.from_numpy(A)
    pre = kw.pop("precond", None)
    res = solver.fgmres(lambda v: At @ v, torch.from_numpy(b), vec=CPUVectors(),
                        precond=(lambda v: torch.from_numpy(pre(v.numpy()))) if pre else None, **kw)
    return res


def _oracle(A, b, precond=None, **kw):
    kw.pop("raise_on_stagnation", None)
    return ofgmres(lambda v: A @ v, b, precond=precond, **kw)


def _random_system(n, seed, shift=1.0):
    rng = np.random.default_rng(seed)
    A = shift * np.eye(n) + 0.3 * rng.standard_normal((n, n)) / np.sqrt(n)
    return A, rng.standard_normal(n)


def test_identity_one_iteration():
    b = np.random.default_rng(0).standard_normal(40)
    res = _solve(np.eye(40), b, rel_tol=1e-12, restart=10)
    assert res.converged and res.iterations == 1
    assert np.abs(res.x.numpy() - b).max() <= 1e-14 * np.abs(b).max()


def test_zero_rhs_returns_zero_without_iterating():
    res = _solve(np.eye(5), np.zeros(5), rel_tol=1e-6, restart=5)
    assert res.converged and res.iterations == 0 and not res.x.any() and not res.updated


@pytest.mark.parametrize("kind", ["diagonal", "random"])
@pytest.mark.parametrize("restart", [60, 7])
def test_matches_oracle_iterations_and_solution(kind, restart):
    n = 80
    if kind == "diagonal":
        rng = np.random.default_rng(3)
        A, b = np.diag(rng.uniform(0.5, 4.0, n)), rng.standard_normal(n)
    else:
        A, b = _random_system(n, 5)
    res = _solve(A, b, rel_tol=1e-10, restart=restart, max_iters=400)
    x_ref, it_ref, rel_ref, conv_ref = _oracle(A, b, rel_tol=1e-10, restart=restart, max_iters=400)
    assert res.converged == conv_ref and res.iterations == it_ref
    assert np.abs(res.x.numpy() - x_ref).max() <= 1e-10 * np.abs(x_ref).max()
    x_dense = np.linalg.solve(A, b)
    assert np.abs(res.x.numpy() - x_dense).max() <= 1e-8 * np.abs(x_dense).max()


def test_flexible_preconditioner_matches_oracle():
    A, b = _random_system(60, 9, shift=2.0)
    d = np.diag(A).copy()
    pre = lambda v: v / d   # noqa: E731
    res = _solve(A, b, rel_tol=1e-9, restart=20, precond=pre)
    x_ref, it_ref, _, _ = _oracle(A, b, precond=pre, rel_tol=1e-9, restart=20)
    assert res.iterations == it_ref
    assert np.abs(res.x.numpy() - x_ref).max() <= 1e-10 * np.abs(x_ref).max()


def test_stagnation_raises_or_returns_unconverged():
    """GMRES(1) on a cyclic shift makes no progress in a restart cycle
    (solver.py:42-118 stagnation rule)."""
    n = 12
    A = np.roll(np.eye(n), 1, axis=0)
    b = np.zeros(n)
    b[0] = 1.0
    with pytest.raises(KrylovStagnation):
        _solve(A, b, rel_tol=1e-8, restart=1, max_iters=50)
    res = _solve(A, b, rel_tol=1e-8, restart=1, max_iters=50, raise_on_stagnation=False)
    _, it_ref, rel_ref, conv_ref = _oracle(A, b, rel_tol=1e-8, restart=1, max_iters=50)
    assert not res.converged and not conv_ref
    assert res.iterations == it_ref and abs(res.rel_residual - rel_ref) <= 1e-14


def test_max_iters_caps_the_solve():
    A, b = _random_system(80, 13, shift=0.2)
    res = _solve(A, b, rel_tol=1e-14, restart=5, max_iters=12, raise_on_stagnation=False)
    _, it_ref, _, conv_ref = _oracle(A, b, rel_tol=1e-14, restart=5, max_iters=12)
    assert res.iterations == it_ref <= 12 and res.converged == conv_ref


@pytest.mark.parametrize("tol,cap", [(0.1, 20), (1e-3, 4), (1e-8, 6)])
def test_arnoldi_exit_of_the_inner_sweep(tol, cap):
    """final_residual="arnoldi" (the inner sweep): same x and iteration count
    as the literal loop when the cycle ends on the residual test or on the
    iteration cap, with one matvec less (solver.py:62-72)."""
    A, b = _random_system(60, 21)
    At = torch.from_numpy(A)
    counts = {}

    def run(mode):
        n = [0]

        def op(v):
            n[0] += 1
            return At @ v

        res = solver.fgmres(op, torch.from_numpy(b), vec=CPUVectors(), rel_tol=tol, restart=cap,
                            max_iters=cap, raise_on_stagnation=False, final_residual=mode)
        counts[mode] = n[0]
        return res

    lit, fast = run("true"), run("arnoldi")
    x_ref, it_ref, _, _ = _oracle(A, b, rel_tol=tol, restart=cap, max_iters=cap)
    assert lit.iterations == fast.iterations == it_ref
    assert torch.equal(lit.x, fast.x)
    assert np.abs(fast.x.numpy() - x_ref).max() <= 1e-12 * np.abs(x_ref).max()
    assert counts["arnoldi"] == counts["true"] - 1
    assert abs(fast.rel_residual - lit.rel_residual) <= 1e-10 * lit.rel_residual


def test_arnoldi_relation_gives_the_matvec_of_the_result():
    """final_residual="arnoldi": result.ax = A x from A Z = V H (what the outer
    column of solve_condensed uses instead of a matvec of the inner result)."""
    A, b = _random_system(70, 33)
    At = torch.from_numpy(A)
    pre = torch.from_numpy(np.diag(1.0 / np.diag(A)))
    for tol, cap in ((0.1, 20), (1e-6, 5)):
        res = solver.fgmres(lambda v: At @ v, torch.from_numpy(b), precond=lambda v: pre @ v,
                            vec=CPUVectors(), rel_tol=tol, restart=cap, max_iters=cap,
                            raise_on_stagnation=False, final_residual="arnoldi")
        assert res.ax is not None
        ax = (At @ res.x).numpy()
        assert np.abs(res.ax.numpy() - ax).max() <= 1e-13 * np.abs(ax).max()
