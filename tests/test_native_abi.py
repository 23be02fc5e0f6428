"""CPU: the C-ABI library builds/loads and exports every symbol declared in
include/mhdg_b200.h (no compute calls without a GPU)."""

import ctypes
import os
import re

import pytest

from helpers import ROOT


def declared_symbols():
    text = open(os.path.join(ROOT, "include", "mhdg_b200.h")).read()
    return sorted(set(re.findall(r"\b(mhdg_[a-z0-9_]+)\s*\(", text)))


def test_header_declares_the_binding_surface():
    from paper_2507_22195_b200 import _native

    assert set(declared_symbols()) == set(_native.EXPORTED)


def test_library_loads_and_exports_all_symbols():
    import __graft_entry__

    __graft_entry__.build()
    lib = ctypes.CDLL(os.path.join(ROOT, "paper_2507_22195_b200", "libmhdg_b200.so"))
    missing = [s for s in declared_symbols() if not hasattr(lib, s)]
    assert not missing, missing
    from paper_2507_22195_b200 import _native

    assert b"sm_100a" in _native.load().mhdg_version()


def test_product_path_fails_loudly_without_cuda():
    import torch

    if torch.cuda.is_available():
        pytest.skip("CUDA present")
    import numpy as np

    from paper_2507_22195_b200 import Discretization, NativeUnavailable
    from paper_2507_22195_b200.mesh import build_box_macro_mesh

    mesh = build_box_macro_mesh(np.array([[0.0, 1.0]] * 3), 1, 1)
    with pytest.raises(NativeUnavailable):
        Discretization(mesh, p=1)


def test_product_never_imports_oracle():
    pkg = os.path.join(ROOT, "paper_2507_22195_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith(".py"):
                src = open(os.path.join(dirpath, f)).read()
                assert "oracle" not in re.sub(r"#.*", "", src).replace('"""', "") or \
                    "import oracle" not in src and "from oracle" not in src, f


def test_unsupported_configurations_raise_invalid_config():
    """Configurations off the B200 path are rejected at construction with the
    reference's InvalidConfig (errors.py:4), before any device work: m > 1,
    p outside 1..4, non-default quadrature, SUPG, unknown formulation, 2D."""
    import numpy as np

    from paper_2507_22195_b200 import Discretization, DissipationSpec, GasModel
    from paper_2507_22195_b200.errors import InvalidConfig
    from paper_2507_22195_b200.mesh import build_box_macro_mesh

    gas, es = GasModel(1.4), DissipationSpec("es")
    box3 = np.array([[0.0, 1.0]] * 3)
    m1 = build_box_macro_mesh(box3, 1, 1)
    cases = [
        (build_box_macro_mesh(box3, 1, 3), dict(p=2)),   # m = 3 only at p = 1
        (m1, dict(p=5)),
        (m1, dict(p=0)),
        (m1, dict(p=2, quad_degree=4)),
        (m1, dict(p=2, supg=True)),
        (m1, dict(p=2, formulation="primitive")),
        (build_box_macro_mesh(np.array([[0.0, 1.0]] * 2), 2, 1), dict(p=2)),
    ]
    for mesh, kw in cases:
        with pytest.raises(InvalidConfig):
            Discretization(mesh, gas=gas, flux=es, **kw)
