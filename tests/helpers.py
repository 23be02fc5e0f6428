"""Shared test helpers (golden fixtures, mesh rebuild, relative error)."""
import os

import numpy as np

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
