"""Discretization tables: per-macro geometry, side tiles, trace connectivity.

Host-side setup shared by the CUDA operator (which uploads these arrays once)
and by the CPU oracle.  Semantics follow the reference's table builders:
  volume tables      assembly.py:155-188  (det, J^-1, vol_w = w_q det)
  face tables        assembly.py:190-273  (side tiles, phi_face, face_rows,
                                           outward unit normals, face_w)
  trace connectivity assembly.py:275-324  (face_id, trace_idx via nearest-
                                           point matching, boundary flags)
The trace matching is vectorized over faces (chunked), replacing the
reference's per-face cdist loop, and produces the identical permutation.
"""

from __future__ import annotations

import math
from ctypes import c_void_p as _c_void_p

import numpy as np

from .errors import InvalidConfig
from .fem import ReferenceBasis, face_embedding, macro_c0_map, reference_face_vertices


class HDGTables:
    """All constant data of a Discretization (mesh, p, quad_degree)."""

    def __init__(self, mesh, p, quad_degree=None):
        self.mesh = mesh
        self.p = p
        d = mesh.dim
        self.d = d
        self.n_s = d + 2
        self.basis = ReferenceBasis(p, d, quad_degree)
        self.layout = macro_c0_map(mesh.m, p, d, self.basis)
        self._volume()
        self._faces()
        self._trace()

    # -- volume (assembly.py:155-188) --------------------------------------
    def _volume(self):
        mesh, basis, d = self.mesh, self.basis, self.d
        sub_ref = self.layout.sub_vertices                  # (n_sub, d+1, d)
        # physical sub vertices = macro map of the reference sub vertices
        sub_v = mesh.sub_vertices
        jac = np.stack([sub_v[:, :, k + 1, :] - sub_v[:, :, 0, :]
                        for k in range(d)], axis=-1)        # (E, n_sub, d, d)
        det = np.linalg.det(jac)
        if np.any(det <= 0):
            raise InvalidConfig("negative sub-element jacobian")
        self.sub_det = det                                  # (E, n_sub)
        self.sub_inv_jac = np.linalg.inv(jac)               # (E, n_sub, d, d)
        self.sub_jac = jac
        self.phi = basis.phi                                # (nq, nn)
        self.dphi = basis.dphi                              # (nq, nn, d)
        self.quad_wts = basis.quad_wts
        self.domain_volume = float(np.prod(mesh.box[:, 1] - mesh.box[:, 0]))
        del sub_ref

    @property
    def vol_w(self):
        return self.quad_wts[None, None, :] * self.sub_det[:, :, None]

    @property
    def dphi_phys(self):
        return np.einsum("qik,eska->esqia", self.dphi, self.sub_inv_jac)

    @property
    def quad_coords(self):
        sub_v = self.mesh.sub_vertices
        return (np.einsum("esab,qb->esqa", self.sub_jac, self.basis.quad_pts)
                + sub_v[:, :, 0, :][:, :, None, :])

    @property
    def node_coords(self):
        mesh = self.mesh
        return (np.einsum("eab,nb->ena", mesh.macro_jacobians,
                          self.layout.unique_nodes)
                + mesh.macro_origins[:, None, :])

    # -- faces (assembly.py:190-273) -----------------------------------------
    def _faces(self):
        mesh, basis, layout, d = self.mesh, self.basis, self.layout, self.d
        facet = basis.facet
        st_face, st_sub, st_subface, scat = [], [], [], []
        for f in range(d + 1):
            for t, (s, fl) in enumerate(layout.face_tiles[f]):
                st_face.append(f)
                st_sub.append(s)
                st_subface.append(fl)
                scat.append(layout.face_scatter[f][t])
        self.n_st = len(st_face)
        self.st_face = np.array(st_face)
        self.st_sub = np.array(st_sub)
        self.st_subface = np.array(st_subface)
        self.st_face_scatter = np.array(scat)               # (n_st, nfn)
        phi_face, rows = [], []
        for k in range(self.n_st):
            fl = st_subface[k]
            v0, span = face_embedding(d, fl)
            pts = v0 + facet.quad_pts @ span.T
            cols = basis.face_nodes[fl]
            phi_face.append(basis.eval_at(pts)[:, cols])
            rows.append(layout.scatter[st_sub[k]][cols])
        self.phi_face = np.array(phi_face)                  # (n_st, nqf, nfn)
        self.face_rows = np.array(rows)                     # (n_st, nfn)
        self.fphi = facet.phi                               # (nqf, nfn)
        self.facet_wts = facet.quad_wts

        sub_v = mesh.sub_vertices
        E = mesh.n_macros
        normals = np.empty((E, self.n_st, d))
        areas = np.empty((E, self.n_st))
        fv = reference_face_vertices(d)
        for k in range(self.n_st):
            s, fl = st_sub[k], st_subface[k]
            pts = sub_v[:, s, list(fv[fl]), :]
            if d == 2:
                tang = pts[:, 1] - pts[:, 0]
                nvec = np.stack([tang[:, 1], -tang[:, 0]], axis=-1)
                areas[:, k] = np.linalg.norm(tang, axis=-1)
            else:
                nvec = np.cross(pts[:, 1] - pts[:, 0], pts[:, 2] - pts[:, 0])
                areas[:, k] = 0.5 * np.linalg.norm(nvec, axis=-1)
            nvec = nvec / np.linalg.norm(nvec, axis=-1, keepdims=True)
            cen = sub_v[:, s].mean(axis=1)
            sign = np.sign(np.sum(nvec * (pts[:, 0] - cen), axis=-1))[:, None]
            normals[:, k] = nvec * sign
        self.face_normals = normals                         # (E, n_st, d)
        # face_w = facet weight * area * (d-1)!; (d-1)! in {1, 2} is exact,
        # so the per-tile factor area*(d-1)! is stored and multiplied on use
        self.face_area = areas * math.factorial(d - 1)      # (E, n_st)

    def trace_csr(self):
        """Deterministic trace accumulation lists (m > 1 device path).

        Returns (trace_ptr, trace_list, face_ptr, face_list): for each trace
        entry (face * nt + node) the contribution slots (macro * n_st + tile)
        * nfn + facet node in the reference's np.add.at order (tile, then
        macro, then facet node: assembly.py:547), and for each face its side
        tiles (macro * n_st + tile) in (tile, macro) order (assembly.py:
        1012-1015)."""
        E, nst = self.face_id_st.shape
        nfn = self.trace_idx.shape[2]
        e, k, j = np.meshgrid(np.arange(E), np.arange(nst), np.arange(nfn), indexing="ij")
        ent = (self.face_id_st[:, :, None] * self.n_trace + self.trace_idx).ravel()
        slot = ((e * nst + k) * nfn + j).ravel()
        order = np.lexsort((j.ravel(), e.ravel(), k.ravel(), ent))
        tlist = slot[order]
        tptr = np.zeros(self.n_faces * self.n_trace + 1, dtype=np.int64)
        np.cumsum(np.bincount(ent, minlength=self.n_faces * self.n_trace), out=tptr[1:])
        e2, k2 = np.meshgrid(np.arange(E), np.arange(nst), indexing="ij")
        fent = self.face_id_st.ravel()
        forder = np.lexsort((e2.ravel(), k2.ravel(), fent))
        flist = (e2 * nst + k2).ravel()[forder]
        fptr = np.zeros(self.n_faces + 1, dtype=np.int64)
        np.cumsum(np.bincount(fent, minlength=self.n_faces), out=fptr[1:])
        return tptr, tlist, fptr, flist

    def viscous_reference(self):
        """Reference operators of the gradient equation (assembly.py:326-371)
        on the unit simplex: Mref^-1, Kref_k[j][i] = sum_q w dphi_k[q,j] phi[q,i],
        Pref_k = Mref^-1 Kref_k, Eref_k[i][j] = sum_q wf phi_face_k[q,i] fphi[q,j].
        Per macro: M = det Mref, K_b = det sum_k Jinv[k][b] Kref_k,
        E_k,b = area_k n_b Eref_k."""
        w = self.quad_wts
        mref = np.einsum("q,qi,qj->ij", w, self.phi, self.phi)
        minv = np.linalg.inv(mref)
        kref = np.einsum("q,qjk,qi->kji", w, self.dphi, self.phi)
        pref = np.einsum("ij,kjl->kil", minv, kref)
        eref = np.einsum("q,kqi,qj->kij", self.facet_wts, self.phi_face, self.fphi)
        return minv, pref, kref, eref

    @property
    def face_w(self):
        return (self.facet_wts[None, None, :] * self.face_area[:, :, None])

    # -- trace connectivity (assembly.py:275-324) ------------------------------
    def _trace(self):
        mesh, layout, d = self.mesh, self.layout, self.d
        skel = mesh.skel
        E = mesh.n_macros
        F = len(skel)
        nt = layout.n_face_unique
        extent = float(np.max(mesh.box[:, 1] - mesh.box[:, 0]))
        tol = 1e-8 * extent
        fun = np.stack(layout.face_unique_nodes)            # (d+1, nt, d)
        face_id = np.zeros((E, d + 1), dtype=np.int64)
        side_of = np.zeros((E, d + 1), dtype=np.int64)      # 0 owner, 1 neighbour
        boundary = np.zeros((E, d + 1), dtype=bool)
        trace_perm = np.zeros((E, d + 1, nt), dtype=np.int64)
        fids = np.arange(F)
        own_e, own_f = skel.owner, skel.owner_face
        # origin + X @ J^T per face, as the reference's mesh.to_physical
        # (mesh.py:115-117): a batched matmul runs the same BLAS product per
        # face, so the coordinates (and the projected trace state) are
        # bit-identical; an einsum here differed in the last bit at p >= 3
        own_pts = (mesh.macro_origins[own_e][:, None, :]
                   + np.matmul(fun[own_f], mesh.macro_jacobians[own_e].transpose(0, 2, 1)))
        self.trace_coords = own_pts                         # (F, nt, d)
        face_id[own_e, own_f] = fids
        trace_perm[own_e, own_f] = np.arange(nt)
        has_nb = skel.neighbor >= 0
        boundary[own_e[~has_nb], own_f[~has_nb]] = True
        nbf = fids[has_nb]
        from .mesh import _host_lib

        lib = _host_lib()
        if lib is not None and len(nbf):   # native: points built and matched per face
            ne, nf = skel.neighbor[nbf], skel.neighbor_face[nbf]
            match = np.empty((len(nbf), nt), dtype=np.int64)
            c = np.ascontiguousarray
            fun_c, ne_c, nf_c = c(fun, dtype=np.float64), c(ne, dtype=np.int64), c(nf, dtype=np.int64)
            org, jac = c(mesh.macro_origins, dtype=np.float64), c(mesh.macro_jacobians, dtype=np.float64)
            shf, owp = c(skel.shift[nbf], dtype=np.float64), c(own_pts[nbf])
            worst = lib.mhdg_match_faces(len(nbf), nt, d, *(a.ctypes.data_as(_c_void_p) for a in
                                                            (fun_c, ne_c, nf_c, org, jac, shf, owp,
                                                             match)))
            if worst < 0 or worst > tol:
                raise InvalidConfig("trace nodes of a skeleton face do not match")
            face_id[ne, nf] = nbf
            side_of[ne, nf] = 1
            trace_perm[ne, nf] = match
            nbf = nbf[:0]
        chunk = max(1, 4_000_000 // max(1, nt * nt)) if lib is None else max(1, len(nbf))
        for c0 in range(0, len(nbf), chunk):
            fs = nbf[c0:c0 + chunk]
            ne, nf = skel.neighbor[fs], skel.neighbor_face[fs]
            nb_pts = (mesh.macro_origins[ne][:, None, :]
                      + np.einsum("fnb,fab->fna", fun[nf], mesh.macro_jacobians[ne]))
            nb_pts = nb_pts - skel.shift[fs][:, None, :]
            if lib is not None:   # native nearest-point matching, same argmin
                nbp = np.ascontiguousarray(nb_pts)
                owp = np.ascontiguousarray(own_pts[fs])
                match = np.empty((len(fs), nt), dtype=np.int64)
                worst = lib.mhdg_match_points(len(fs), nt, d, nbp.ctypes.data_as(_c_void_p),
                                              owp.ctypes.data_as(_c_void_p),
                                              match.ctypes.data_as(_c_void_p))
                if worst < 0 or worst > tol:
                    raise InvalidConfig("trace nodes of a skeleton face do not match")
            else:
                dist = np.sqrt(((nb_pts[:, :, None, :] - own_pts[fs][:, None, :, :]) ** 2)
                               .sum(-1))                    # (c, nt_nb, nt_own)
                match = dist.argmin(axis=2)
                best = np.take_along_axis(dist, match[:, :, None], 2)[..., 0]
                srt = np.sort(match, axis=1)
                if best.max() > tol or np.any(srt[:, 1:] == srt[:, :-1]):
                    raise InvalidConfig("trace nodes of a skeleton face do not match")
            face_id[ne, nf] = fs
            side_of[ne, nf] = 1
            trace_perm[ne, nf] = match
        self.n_faces = F
        self.n_trace = nt
        self.face_id = face_id
        self.boundary_side = boundary
        self.side_of = side_of
        st = self.st_face
        # trace_idx[e, k, j] = trace_perm[e, st[k], st_face_scatter[k, j]]
        self.trace_idx = trace_perm[:, st[:, None], self.st_face_scatter]   # (E, n_st, nfn)
        self.face_id_st = face_id[:, st]                    # (E, n_st)
        self.boundary_st = boundary[:, st]
        self.side_st = side_of[:, st]
        # per face: the (macro, tile) of each side, for face-local kernels (m=1)
        if self.n_st == d + 1:
            tile_of_face = np.empty(d + 1, dtype=np.int64)
            tile_of_face[st] = np.arange(self.n_st)
            self.face_sides = np.full((F, 2), -1, dtype=np.int64)
            self.face_sides[:, 0] = own_e * self.n_st + tile_of_face[own_f]
            self.face_sides[has_nb, 1] = (skel.neighbor[has_nb] * self.n_st
                                          + tile_of_face[skel.neighbor_face[has_nb]])
        else:
            self.face_sides = None
