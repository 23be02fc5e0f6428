"""Shared test helpers (golden fixtures, mesh rebuild, relative error)."""
import os

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden")


def load_golden(name):
    return dict(np.load(os.path.join(GOLDEN, f"{name}.npz"), allow_pickle=False))


def golden_mesh(z):
    from paper_2507_22195_b200.mesh import build_box_macro_mesh

    n = z["n_per_dim"]
    n = tuple(int(v) for v in np.atleast_1d(n)) if np.ndim(n) else int(n)
    per = z["periodic"]
    per = tuple(bool(v) for v in per) if np.ndim(per) else bool(per)
    return build_box_macro_mesh(z["box"], n, int(z["m"]), per)


def rel(a, b):
    a = a.detach().cpu().numpy() if hasattr(a, "detach") else np.asarray(a)
    b = b.detach().cpu().numpy() if hasattr(b, "detach") else np.asarray(b)
    nb = np.linalg.norm(b)
    return float(np.linalg.norm(a - b) / (nb if nb > 0 else 1.0))


class CPUVectors:
    """Test double of the device vector kernels (torch CPU ops)."""

    def __init__(self):
        self.torch = torch

    def dot_into(self, x, y, out):
        out[0] = torch.dot(x, y)

    def norm(self, x):
        return float(torch.linalg.vector_norm(x))

    def div_into(self, x, a, out):
        out.copy_(x / a)

    def axpby(self, a, x, b, y, out):
        out.copy_(a * x + b * y)

    def axpy_dev(self, a, x, y):
        y.sub_(a[0] * x)

    def combine_dev(self, Z, k, y, x):
        x.add_(y[:k] @ Z[:k])

    def combine(self, Z, k, yv, x):
        x.add_(torch.from_numpy(np.ascontiguousarray(yv[:k])) @ Z[:k])

    def mgs(self, V, j, w):
        h = np.zeros(j + 2)
        for i in range(j + 1):
            h[i] = float(V[i] @ w)
            w.sub_(h[i] * V[i])
        h[j + 1] = float(torch.linalg.vector_norm(w))
        if h[j + 1] > 1e-300:
            V[j + 1].copy_(w / h[j + 1])
        return h
