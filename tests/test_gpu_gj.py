"""GPU: the batched Gauss-Jordan inverse (csrc/mhdg_gj_blocked.cuh) on its own,
through the C ABI (mhdg_batched_inverse), against numpy's LU-based inverse.

The device kernel replaces the reference's per-macro lu_factor / lu_solve
(assembly.py:718-733) and the per-face block factorization (assembly.py:736-752)
by explicit inverses: a diagonal-pivot pass in block form (8 x 8 diagonal
blocks inverted by one warp, panels applied on the FP64 tensor cores) with
lane-local growth checks, and a partial-pivoting pass for the matrices that
fail them.  Tolerance relative to |A^-1|: 50 cond(A) eps for matrices with a
dominant diagonal (LU's own error bound has this form), 1000 cond(A) eps for
unstructured random matrices: the diagonal-pivot pass accepts multipliers up
to 1 / GJ_TAU = 20 per panel (threshold pivoting), measured worst case
103 cond eps on N(0, 1) matrices of order 20.  Orders 20 / 50 / 100 are the
condensed and face block orders of k = 1..3."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

EPS = np.finfo(np.float64).eps


@pytest.fixture(scope="module")
def disc():
    import torch

    from paper_2507_22195_b200 import Discretization, DissipationSpec, GasModel, _native
    from paper_2507_22195_b200.mesh import build_box_macro_mesh

    _native.require_cuda()
    mesh = build_box_macro_mesh(np.array([[0.0, 1.0]] * 3), 4, 1)   # 384 macros, 768 faces: batch capacity
    return Discretization(mesh, p=1, gas=GasModel(1.4), flux=DissipationSpec("es"), device="cuda:0"), torch


def _check(disc_torch, mats, expect_fallbacks=None, tol=50.0):
    disc, torch = disc_torch
    inv, fb = disc.batched_inverse(torch.as_tensor(mats, device="cuda:0"))
    inv = inv.cpu().numpy()
    ref = np.linalg.inv(mats)
    cond = np.linalg.cond(mats)
    err = np.abs(inv - ref).max(axis=(1, 2)) / np.abs(ref).max(axis=(1, 2))
    assert (err <= tol * cond * EPS).all(), (err / (cond * EPS)).max()
    if expect_fallbacks is not None:
        assert fb == expect_fallbacks, (fb, expect_fallbacks)
    return fb


@pytest.mark.parametrize("n", [20, 50, 100])
def test_diagonally_dominant_takes_the_diagonal_pivot_pass(disc, n):
    rng = np.random.default_rng(n)
    a = rng.standard_normal((257, n, n)) + 2.0 * np.sqrt(n) * np.eye(n)
    _check(disc, a, expect_fallbacks=0)


@pytest.mark.parametrize("n", [20, 50, 100])
def test_general_matrices_fall_back_to_partial_pivoting(disc, n):
    rng = np.random.default_rng(100 + n)
    a = rng.standard_normal((300, n, n))          # no diagonal structure: most fail the growth checks
    fb = _check(disc, a, tol=1000.0)
    assert fb > 0
    # a cyclic row shift of a dominant matrix has a zero-ish diagonal: every one must fall back
    b = np.roll(rng.standard_normal((64, n, n)) * 0.01 + 3.0 * np.eye(n), 1, axis=1)
    _check(disc, b, expect_fallbacks=64)


@pytest.mark.parametrize("n", [20, 100])
def test_mixed_batch_and_block_structured(disc, n):
    """S-like matrices: 5 x 5 nodal blocks, strong diagonal blocks plus a
    dense coupling, scaled rows (the pseudo-time / mass scaling spread)."""
    rng = np.random.default_rng(7 * n)
    nb = n // 5
    a = 0.2 * rng.standard_normal((200, n, n))
    for b in range(nb):
        blk = rng.standard_normal((200, 5, 5)) + 4.0 * np.eye(5)
        a[:, 5 * b:5 * b + 5, 5 * b:5 * b + 5] += blk
    a *= np.exp(rng.uniform(-3, 3, (200, n, 1)))
    a[::7] = rng.standard_normal((len(a[::7]), n, n))   # every 7th needs pivoting
    _check(disc, a, tol=1000.0)


def test_singular_matrix_is_reported_with_its_index(disc):
    from paper_2507_22195_b200.errors import SingularLocalMatrix

    d, torch = disc
    rng = np.random.default_rng(11)
    a = rng.standard_normal((40, 50, 50)) + 10.0 * np.eye(50)
    a[23, :, 7] = 0.0
    with pytest.raises(SingularLocalMatrix) as ei:
        d.batched_inverse(torch.as_tensor(a, device="cuda:0"))
    assert ei.value.macro == 23


def test_capacity_and_order_are_validated(disc):
    from paper_2507_22195_b200.errors import InvalidConfig

    d, torch = disc
    with pytest.raises(InvalidConfig):
        d.batched_inverse(torch.eye(30, device="cuda:0", dtype=torch.float64).repeat(4, 1, 1))
    with pytest.raises(InvalidConfig):
        d.batched_inverse(torch.eye(20, device="cuda:0", dtype=torch.float64).repeat(5000, 1, 1))
