"""Bit-exact digests of the host tables and index / scatter maps.

`collect(mod, mesh_mod, fem_mod, n, p)` returns {name: (dtype, shape,
sha256 of the C-contiguous bytes)} for every table the operator consumes,
computed through either package (the reference `macrohdg` or this repo's
`paper_2507_22195_b200`): SHA-256 digests keep the fixture small at n=16
while still asserting equality bit for bit.  Integer maps are compared as
int64, bool masks as uint8.

Names (reference source of each array):
  basis.*         fem.py:440-489   ReferenceBasis (nodes, phi, dphi, quad, facet, face_nodes)
  layout.*        fem.py:663-724   macro_c0_map (scatter, unique nodes, face tiles / scatter)
  mesh.*          mesh.py:140-299  box mesh (origins, jacobians, sub vertices) and skeleton
  disc.*          assembly.py:155-324  volume / face tables and trace connectivity

Run `PYTHONPATH=/root/reference/pkg/src python tests/golden/table_digests.py`
in the build container to regenerate tests/golden/table_digests.json.
"""

from __future__ import annotations

import hashlib
import json
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
OUT = os.path.join(HERE, "table_digests.json")
CASES = [(n, p) for n in (4, 8, 16) for p in (1, 2, 3, 4)]
# m > 1 macro subdivision: (n, m, p)
MACRO_CASES = [(2, 2, 1), (2, 2, 2), (4, 2, 3), (2, 3, 1)]


def digest(a):
    a = np.asarray(a)
    if a.dtype == bool:
        a = a.astype(np.uint8)
    elif np.issubdtype(a.dtype, np.integer):
        a = a.astype(np.int64)
    elif np.issubdtype(a.dtype, np.floating):
        a = a.astype(np.float64)
    a = np.ascontiguousarray(a)
    return [str(a.dtype), list(a.shape), hashlib.sha256(a.tobytes()).hexdigest()]


def skeleton_arrays(mesh):
    """(owner, owner_face, neighbor, neighbor_face, shift, vertex_perm) of the
    skeleton in its order, -1 rows on boundary faces."""
    faces = mesh.skeleton_faces
    d = mesh.dim
    own = np.array([f.owner for f in faces])
    ownf = np.array([f.owner_face for f in faces])
    nb = np.array([-1 if f.neighbor is None else f.neighbor for f in faces])
    nbf = np.array([-1 if f.neighbor_face is None else f.neighbor_face for f in faces])
    shift = np.array([np.asarray(f.shift, dtype=float) for f in faces])
    perm = np.array([np.full(d, -1) if f.vertex_perm is None else np.asarray(f.vertex_perm)
                     for f in faces])
    return own, ownf, nb, nbf, shift, perm


def collect(build_mesh, make_disc, n, p, m=1):
    """build_mesh(box, n, m) -> mesh; make_disc(mesh, p) -> object exposing the
    reference's Discretization table attributes."""
    box = np.array([[0.0, 10.0]] * 3)
    mesh = build_mesh(box, n, m)
    disc = make_disc(mesh, p)
    b, lay = disc.basis, disc.layout
    out = {}

    def put(name, a):
        out[name] = digest(a)

    put("basis.nodes", b.nodes)
    put("basis.phi", b.phi)
    put("basis.dphi", b.dphi)
    put("basis.quad_pts", b.quad_pts)
    put("basis.quad_wts", b.quad_wts)
    put("basis.facet.nodes", b.facet.nodes)
    put("basis.facet.phi", b.facet.phi)
    put("basis.facet.quad_pts", b.facet.quad_pts)
    put("basis.facet.quad_wts", b.facet.quad_wts)
    for k, fn in enumerate(b.face_nodes):
        put(f"basis.face_nodes[{k}]", fn)
    put("layout.scatter", lay.scatter)
    put("layout.unique_nodes", lay.unique_nodes)
    put("layout.sub_vertices", lay.sub_vertices)
    for k in range(4):
        put(f"layout.face_tiles[{k}]", np.array(lay.face_tiles[k]))
        put(f"layout.face_scatter[{k}]", lay.face_scatter[k])
        put(f"layout.face_unique_nodes[{k}]", lay.face_unique_nodes[k])
    put("mesh.macro_elements", mesh.macro_elements)
    put("mesh.macro_origins", mesh.macro_origins)
    put("mesh.macro_jacobians", mesh.macro_jacobians)
    put("mesh.macro_dets", mesh.macro_dets)
    put("mesh.sub_vertices", mesh.sub_vertices)
    for name, a in zip(("owner", "owner_face", "neighbor", "neighbor_face", "shift",
                        "vertex_perm"), skeleton_arrays(mesh)):
        put(f"mesh.skeleton.{name}", a)
    put("disc.vol_w", disc.vol_w)
    put("disc.node_coords", disc.node_coords)
    put("disc.quad_coords", disc.quad_coords)
    put("disc.trace_coords", disc.trace_coords)
    put("disc.st_face", disc.st_face)
    put("disc.st_sub", disc.st_sub)
    put("disc.st_face_scatter", disc.st_face_scatter)
    put("disc.phi_face", disc.phi_face)
    put("disc.face_rows", disc.face_rows)
    put("disc.fphi", disc.fphi)
    put("disc.face_normals", disc.face_normals)
    put("disc.face_w", disc.face_w)
    put("disc.face_id", disc.face_id)
    put("disc.face_id_st", disc.face_id_st)
    put("disc.trace_idx", disc.trace_idx)
    put("disc.boundary_st", disc.boundary_st)
    return out


def main():
    from macrohdg.assembly import Discretization
    from macrohdg.mesh import build_box_macro_mesh

    res = {}
    for n, p in CASES:
        res[f"n{n}_p{p}"] = collect(build_box_macro_mesh,
                                    lambda mesh, p: Discretization(mesh, p), n, p)
        print("done", n, p, flush=True)
    for n, m, p in MACRO_CASES:
        res[f"n{n}_m{m}_p{p}"] = collect(build_box_macro_mesh,
                                         lambda mesh, p: Discretization(mesh, p), n, p, m)
        print("done", n, m, p, flush=True)
    with open(OUT, "w") as f:
        json.dump({"generator": "tests/golden/table_digests.py (reference macrohdg)",
                   "box": "[[0,10]]^3 periodic", "cases": res}, f, indent=0, sort_keys=True)


if __name__ == "__main__":
    main()
