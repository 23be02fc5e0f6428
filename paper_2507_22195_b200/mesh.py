"""Structured macro-simplex box meshes and their skeleton (host side).

Each cell of an n_1 x .. x n_d grid is split into d! path simplices sharing
the main diagonal; every macro is the affine image of the Kuhn path simplex
and is subdivided m^d-fold.  The skeleton lists every macro face once, owned
by the side with the smaller (macro * (d+1) + local face) index, in increasing
owner-side order; periodic axes pair opposite box sides.

Orderings are part of the operator's data layout (trace storage is per
skeleton face, in the owner's face-node order) and follow the reference:
  build_box_macro_mesh   mesh.py:140-223
  skeleton               mesh.py:226-299  (face order, owner choice, shift)
  dof_counts             mesh.py:302-324
The skeleton is built with vectorized integer keys instead of per-face
Python loops, so n=64 (1.57M macros) builds in seconds.
"""

from __future__ import annotations

import itertools
import math
import os
from ctypes import c_void_p as _c_void_p
from dataclasses import dataclass, field

import numpy as np

from .errors import InvalidConfig, TopologyError
from .fem import kuhn_subdivision


@dataclass(frozen=True)
class SkeletonFace:
    owner: int
    owner_face: int
    neighbor: int | None
    neighbor_face: int | None
    shift: np.ndarray
    vertex_perm: np.ndarray | None

    @property
    def is_boundary(self):
        return self.neighbor is None


@dataclass(frozen=True)
class DofLayout:
    p: int
    n_s: int
    local_dofs: int
    global_dofs: int
    n_macros: int
    n_elements: int
    n_skeleton_faces: int
    nodes_per_macro: int
    trace_nodes_per_face: int
    effective_1d: tuple


@dataclass
class SkeletonArrays:
    """Struct-of-arrays skeleton: one entry per skeleton face."""

    owner: np.ndarray          # (F,) int64
    owner_face: np.ndarray     # (F,)
    neighbor: np.ndarray       # (F,) -1 on boundary faces
    neighbor_face: np.ndarray  # (F,) -1 on boundary faces
    shift: np.ndarray          # (F, d)
    vertex_perm: np.ndarray    # (F, d) -1 rows on boundary faces

    def __len__(self):
        return len(self.owner)


@dataclass
class MacroMesh:
    dim: int
    m: int
    box: np.ndarray
    n_per_dim: tuple
    periodic: tuple
    vertices: np.ndarray
    macro_elements: np.ndarray
    macro_vertices: np.ndarray
    macro_origins: np.ndarray
    macro_jacobians: np.ndarray
    macro_dets: np.ndarray
    sub_reference: np.ndarray
    skel: SkeletonArrays = None
    _faces: list = field(default=None, repr=False)
    _sub_vertices: np.ndarray = field(default=None, repr=False)

    @property
    def n_macros(self):
        return len(self.macro_elements)

    @property
    def n_sub_elements(self):
        return self.n_macros * len(self.sub_reference)

    @property
    def n_skeleton_faces(self):
        return len(self.skel)

    @property
    def sub_vertices(self):
        """(E, m^d, d+1, d) physical sub-element vertices (built lazily)."""
        if self._sub_vertices is None:
            self._sub_vertices = (
                np.einsum("eab,skb->eska", self.macro_jacobians, self.sub_reference)
                + self.macro_origins[:, None, None, :])
        return self._sub_vertices

    @property
    def skeleton_faces(self):
        if self._faces is None:
            s = self.skel
            self._faces = [
                SkeletonFace(int(s.owner[f]), int(s.owner_face[f]),
                             None if s.neighbor[f] < 0 else int(s.neighbor[f]),
                             None if s.neighbor[f] < 0 else int(s.neighbor_face[f]),
                             s.shift[f].copy(),
                             None if s.neighbor[f] < 0 else s.vertex_perm[f].copy())
                for f in range(len(s))]
        return self._faces

    @property
    def boundary_faces(self):
        return [f for f in self.skeleton_faces if f.is_boundary] \
            if (self.skel.neighbor < 0).any() else []

    @property
    def has_boundary(self):
        return bool((self.skel.neighbor < 0).any())

    def face_vertex_coords(self, macro, local_face):
        keep = [k for k in range(self.dim + 1) if k != local_face]
        return self.macro_vertices[macro, keep]

    def to_physical(self, macro, reference_points):
        return (self.macro_origins[macro]
                + reference_points @ self.macro_jacobians[macro].T)


def _axis_tuple(value, d, name, cast):
    if np.isscalar(value) or isinstance(value, bool):
        return (cast(value),) * d
    items = tuple(value)
    if len(items) != d:
        raise InvalidConfig(f"{name} needs 1 or {d} entries, got {len(items)}")
    return tuple(cast(v) for v in items)


def _parity(perm):
    return sum(perm[i] > perm[j] for i in range(len(perm))
               for j in range(i + 1, len(perm))) % 2


def build_box_macro_mesh(box, n_per_dim, m, periodic=True):
    """n^d cells x d! macros, cells in row-major (x slowest) order, the d!
    macros of a cell in sorted-permutation order (mesh.py:140-223)."""
    box = np.atleast_2d(np.asarray(box, dtype=float))
    d = len(box)
    if d not in (2, 3) or box.shape != (d, 2):
        raise InvalidConfig(f"box must be (d, 2) extents, got {box.shape}")
    if np.any(box[:, 1] <= box[:, 0]):
        raise InvalidConfig("degenerate box")
    n_axis = _axis_tuple(n_per_dim, d, "n_per_dim", int)
    if min(n_axis) < 1:
        raise InvalidConfig(f"n_per_dim must be >= 1, got {n_axis}")
    if m < 1 or int(m) != m:
        raise InvalidConfig(f"subdivision count must be a positive integer, got {m}")
    flags = _axis_tuple(periodic, d, "periodic", bool)

    lo = box[:, 0]
    h = (box[:, 1] - box[:, 0]) / np.array(n_axis)
    axes = [lo[a] + h[a] * np.arange(n_axis[a] + 1) for a in range(d)]
    grids = np.meshgrid(*axes, indexing="ij")
    vertices = np.stack([g.ravel() for g in grids], axis=-1)
    strides = np.array([int(np.prod([n_axis[b] + 1 for b in range(a + 1, d)]))
                        for a in range(d)])

    # vectorized over cells: corner index of every path vertex per permutation
    cells = np.stack(np.meshgrid(*[np.arange(n) for n in n_axis], indexing="ij"),
                     axis=-1).reshape(-1, d)
    perms = sorted(itertools.permutations(range(d)))
    per_perm = []
    for perm in perms:
        idx = np.empty((len(cells), d + 1), dtype=np.int64)
        acc = cells.copy()
        idx[:, 0] = acc @ strides
        for k, axis in enumerate(perm):
            acc = acc.copy()
            acc[:, axis] += 1
            idx[:, k + 1] = acc @ strides
        if _parity(perm):
            idx[:, [d - 1, d]] = idx[:, [d, d - 1]]
        per_perm.append(idx)
    macro_elements = np.stack(per_perm, axis=1).reshape(-1, d + 1)
    macro_vertices = vertices[macro_elements]
    macro_origins = macro_vertices[:, 0, :]
    macro_jacobians = np.stack(
        [macro_vertices[:, k + 1, :] - macro_vertices[:, k, :] for k in range(d)],
        axis=-1)
    macro_dets = np.linalg.det(macro_jacobians)
    if np.any(macro_dets <= 0):
        raise InvalidConfig("macro orientation fix failed")
    mesh = MacroMesh(dim=d, m=int(m), box=box, n_per_dim=n_axis, periodic=flags,
                     vertices=vertices, macro_elements=macro_elements,
                     macro_vertices=macro_vertices, macro_origins=macro_origins,
                     macro_jacobians=macro_jacobians, macro_dets=macro_dets,
                     sub_reference=kuhn_subdivision(int(m), d))
    mesh.skel = skeleton_arrays(mesh)
    return mesh


def _host_lib():
    """libmhdg_b200.so for its host-side topology entry points, or None when
    the library is not built (numpy builder; identical results)."""
    if os.environ.get("MHDG_NUMPY_TABLES"):
        return None
    from . import _native

    return _native.host_library()


def skeleton_arrays(mesh):
    """Pair macro sides into skeleton faces (mesh.py:226-299 semantics).

    Sides are keyed by their sorted, periodically wrapped, quantized vertex
    coordinates; a face's owner is its smaller side index, faces are ordered
    by owner side index, shift = round(delta / extent) * extent of the
    neighbour-minus-owner face centroids, vertex_perm[i] = neighbour face
    vertex matching owner face vertex i.
    """
    d = mesh.dim
    extent = mesh.box[:, 1] - mesh.box[:, 0]
    quantum = 1e-10 * float(np.max(extent))
    E = mesh.n_macros
    fids = np.array([[k for k in range(d + 1) if k != f] for f in range(d + 1)])
    sv = mesh.macro_vertices[:, fids, :].reshape(E * (d + 1), d, d)
    lib = _host_lib()
    if lib is not None:   # native keys (csrc/mhdg_host_mesh.cuh), same integers
        svc = np.ascontiguousarray(sv)
        kk = np.empty((len(svc), d, d), dtype=np.int64)
        hi = np.ascontiguousarray(mesh.box[:, 1], dtype=np.float64)
        ext = np.ascontiguousarray(extent, dtype=np.float64)
        per = np.ascontiguousarray([1 if x else 0 for x in mesh.periodic], dtype=np.int32)
        lib.mhdg_side_keys(len(svc), d, svc.ctypes.data_as(_c_void_p), hi.ctypes.data_as(_c_void_p),
                           ext.ctypes.data_as(_c_void_p), per.ctypes.data_as(_c_void_p), quantum,
                           kk.ctypes.data_as(_c_void_p))
        return _pair_and_shift(mesh, sv, kk, extent, quantum, lib)
    wrapped = sv.copy()
    for a in range(d):
        if mesh.periodic[a]:
            on_max = np.all(np.abs(sv[:, :, a] - mesh.box[a, 1]) < quantum, axis=1)
            wrapped[on_max, :, a] -= extent[a]
    keys = np.round(wrapped / quantum).astype(np.int64)        # (S, d, d)
    # canonical key: each side's d vertex rows in lexicographic order
    # (insertion sort over the d <= 3 rows, vectorized over sides)
    kk = keys.copy()
    for i in range(1, d):
        j = i
        while j > 0:
            prev, cur = kk[:, j - 1].copy(), kk[:, j].copy()
            swap = np.zeros(len(kk), dtype=bool)
            decided = np.zeros(len(kk), dtype=bool)
            for a in range(d):
                gt = (~decided) & (prev[:, a] > cur[:, a])
                lt = (~decided) & (prev[:, a] < cur[:, a])
                swap |= gt
                decided |= gt | lt
            kk[swap, j - 1], kk[swap, j] = cur[swap], prev[swap]
            j -= 1
    return _pair_and_shift(mesh, sv, kk, extent, quantum, lib)


def _pair_and_shift(mesh, sv, kk, extent, quantum, lib):
    """Pair sides with equal canonical keys; shift and vertex permutation."""
    d = mesh.dim
    flat = np.ascontiguousarray(kk.reshape(len(kk), d * d))
    if lib is not None:
        # native pairing (csrc/mhdg_host_mesh.cuh): sort by key, pair equal
        # neighbours; faces in increasing owner-side order as below
        partner = np.empty(len(flat), dtype=np.int64)
        bad = lib.mhdg_pair_sides(len(flat), d * d, flat.ctypes.data_as(_c_void_p),
                                  partner.ctypes.data_as(_c_void_p))
        if bad > 0:
            raise TopologyError(f"{int(bad)} face groups have more than two sides")
        sides = np.arange(len(flat), dtype=np.int64)
        first = sides[(partner < 0) | (sides < partner)]
        second = partner[first]
    else:
        _, group, counts = np.unique(flat, axis=0, return_inverse=True,
                                     return_counts=True)
        group = group.ravel()
        if counts.max() > 2:
            raise TopologyError(f"{int((counts > 2).sum())} face groups have "
                                "more than two sides")
        n_groups = len(counts)
        first = np.full(n_groups, np.iinfo(np.int64).max, dtype=np.int64)
        second = np.full(n_groups, -1, dtype=np.int64)
        sides = np.arange(len(group), dtype=np.int64)
        np.minimum.at(first, group, sides)
        is_second = sides != first[group]
        second[group[is_second]] = sides[is_second]
        face_order = np.argsort(first, kind="stable")
        first, second = first[face_order], second[face_order]

    owner, owner_face = np.divmod(first, d + 1)
    has_nb = second >= 0
    neighbor = np.where(has_nb, second // (d + 1), -1)
    neighbor_face = np.where(has_nb, second % (d + 1), -1)

    F = len(first)
    shift = np.zeros((F, d))
    perm = np.full((F, d), -1, dtype=np.int64)
    if has_nb.any() and lib is not None:   # native shift / permutation, same floats
        va = np.ascontiguousarray(sv[first[has_nb]])
        vb = np.ascontiguousarray(sv[second[has_nb]])
        sh = np.empty((len(va), d))
        pm = np.empty((len(va), d), dtype=np.int64)
        ext = np.ascontiguousarray(extent, dtype=np.float64)
        worst = lib.mhdg_face_shift_perm(len(va), d, va.ctypes.data_as(_c_void_p),
                                         vb.ctypes.data_as(_c_void_p), ext.ctypes.data_as(_c_void_p),
                                         sh.ctypes.data_as(_c_void_p), pm.ctypes.data_as(_c_void_p))
        if worst < 0:
            raise TopologyError("degenerate vertex matching")
        if worst > quantum:
            raise TopologyError("face vertices do not match after shift")
        shift[has_nb] = sh
        perm[has_nb] = pm
    elif has_nb.any():
        va = sv[first[has_nb]]
        vb = sv[second[has_nb]]
        delta = vb.mean(axis=1) - va.mean(axis=1)
        sh = np.round(delta / extent) * extent
        shift[has_nb] = sh
        vb_back = vb - sh[:, None, :]
        dist = np.linalg.norm(vb_back[:, None, :, :] - va[:, :, None, :], axis=-1)
        j = dist.argmin(axis=2)                                 # (Fi, d)
        if np.take_along_axis(dist, j[:, :, None], 2).max() > quantum:
            raise TopologyError("face vertices do not match after shift")
        srt = np.sort(j, axis=1)
        if np.any(srt[:, 1:] == srt[:, :-1]):
            raise TopologyError("degenerate vertex matching")
        perm[has_nb] = j
    return SkeletonArrays(owner=owner, owner_face=owner_face, neighbor=neighbor,
                          neighbor_face=neighbor_face, shift=shift,
                          vertex_perm=perm)


def dof_counts(mesh, p, n_s=None):
    d = mesh.dim
    n_s = int(n_s) if n_s is not None else d + 2
    mp = mesh.m * p
    npm = math.comb(mp + d, d)
    ntf = math.comb(mp + d - 1, d - 1)
    return DofLayout(
        p=p, n_s=n_s,
        local_dofs=mesh.n_macros * npm * n_s * (1 + d),
        global_dofs=mesh.n_skeleton_faces * ntf * n_s,
        n_macros=mesh.n_macros, n_elements=mesh.n_sub_elements,
        n_skeleton_faces=mesh.n_skeleton_faces, nodes_per_macro=npm,
        trace_nodes_per_face=ntf,
        effective_1d=tuple(n * (mp + 1) for n in mesh.n_per_dim))
