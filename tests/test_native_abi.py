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
