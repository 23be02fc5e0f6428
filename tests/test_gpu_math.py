"""GPU: accuracy of the operator's device elementary functions (branch-free
exp / log and the Newton-refined division of csrc/mhdg_math.cuh) against
libm, in ulps, over the ranges the gas algebra evaluates them on plus the
IEEE special values."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _ulp_err(y, ref):
    ref = np.asarray(ref)
    return np.abs(y - ref) / np.spacing(np.abs(ref))


@pytest.fixture(scope="module")
def dev():
    import torch

    from paper_2507_22195_b200 import _native

    _native.require_cuda()
    return lambda fn, x: _native.math_eval(fn, torch.as_tensor(x, device="cuda")).cpu().numpy()


def test_exp_accuracy(dev):
    rng = np.random.default_rng(3)
    x = np.concatenate([rng.uniform(-30, 10, 200_000), rng.uniform(-700, 700, 50_000),
                        rng.uniform(-1e-8, 1e-8, 10_000)])
    err = _ulp_err(dev(0, x), np.exp(x))
    assert err.max() <= 2.0, err.max()
    sp = np.array([0.0, -0.0, np.inf, -np.inf, np.nan, 710.0, -800.0, -746.0, 709.78])
    with np.errstate(over="ignore"):
        np.testing.assert_array_equal(dev(0, sp)[:7], np.exp(sp)[:7])
    assert np.isclose(dev(0, sp[8:]), np.exp(sp[8:]), rtol=1e-15).all()


def test_log_accuracy(dev):
    rng = np.random.default_rng(4)
    x = np.concatenate([np.exp(rng.uniform(-40, 40, 200_000)), 1.0 + rng.uniform(-1e-4, 1e-4, 50_000),
                        rng.uniform(0.5, 2.0, 50_000), [1.0, 2.0, 0.5, 5e-324, 1e-310]])
    err = _ulp_err(dev(1, x), np.log(x))
    err = err[np.log(x) != 0]
    assert err.max() <= 3.0, err.max()
    assert dev(1, np.array([1.0]))[0] == 0.0
    with np.errstate(divide="ignore", invalid="ignore"):
        sp = np.array([0.0, -1.0, np.inf, np.nan])
        np.testing.assert_array_equal(dev(1, sp), np.log(sp))


def test_division_accuracy(dev):
    rng = np.random.default_rng(5)
    x = np.exp(rng.uniform(-200, 200, 200_000)) * rng.choice([-1.0, 1.0], 200_000)
    err = _ulp_err(dev(2, x), 1.0 / x)
    assert err.max() <= 1.0, err.max()
