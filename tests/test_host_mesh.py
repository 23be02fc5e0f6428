"""CPU: the native table-builder kernels (csrc/mhdg_host_mesh.cuh via the
C ABI: skeleton side pairing, trace-node matching) produce exactly the
numpy builder's skeleton and trace maps (which are pinned to the reference,
tests/test_oracle_golden.py), on periodic, partly periodic and bounded
boxes of several shapes and degrees."""

import numpy as np
import pytest

from paper_2507_22195_b200 import _native
from paper_2507_22195_b200.mesh import build_box_macro_mesh
from paper_2507_22195_b200.tables import HDGTables

SKEL = ("owner", "owner_face", "neighbor", "neighbor_face", "shift", "vertex_perm")
MAPS = ("face_id", "trace_idx", "face_id_st", "boundary_st", "side_st", "face_sides")


def _build(monkeypatch, numpy_only, box, n, p, periodic):
    if numpy_only:
        monkeypatch.setenv("MHDG_NUMPY_TABLES", "1")
    else:
        monkeypatch.delenv("MHDG_NUMPY_TABLES", raising=False)
    mesh = build_box_macro_mesh(box, n, 1, periodic=periodic)
    return mesh, HDGTables(mesh, p)


@pytest.mark.parametrize("n,p,periodic,box", [
    ((3, 2, 2), 2, True, [[0.0, 1.0]] * 3),
    ((4, 4, 4), 3, True, [[0.0, 1.0]] * 3),
    ((2, 3, 1), 1, (True, False, True), [[0.0, 2.0], [0.0, 1.0], [0.0, 3.0]]),
    ((2, 2, 3), 4, False, [[-1.0, 1.0]] * 3),
])
def test_native_builder_matches_numpy(monkeypatch, n, p, periodic, box):
    import __graft_entry__

    __graft_entry__.build()
    assert _native.host_library() is not None
    box = np.array(box)
    ma, ta = _build(monkeypatch, False, box, n, p, periodic)
    mb, tb = _build(monkeypatch, True, box, n, p, periodic)
    for k in SKEL:
        assert np.array_equal(getattr(ma.skel, k), getattr(mb.skel, k)), k
    for k in MAPS:
        a, b = getattr(ta, k), getattr(tb, k)
        assert (a is None and b is None) or np.array_equal(a, b), k


def test_pair_sides_flags_overfull_groups():
    import ctypes as C

    import __graft_entry__

    __graft_entry__.build()
    lib = _native.host_library()
    keys = np.array([[1, 2], [3, 4], [1, 2], [1, 2], [5, 6]], dtype=np.int64)
    partner = np.empty(5, dtype=np.int64)
    bad = lib.mhdg_pair_sides(5, 2, keys.ctypes.data_as(C.c_void_p), partner.ctypes.data_as(C.c_void_p))
    assert bad == 1
    assert partner[1] == -1 and partner[4] == -1
