"""Reference-simplex tables for the macro-element HDG operator (host side).

Everything here is setup-time numpy that produces the constant tables the
CUDA kernels read (basis values and gradients at quadrature points, facet
tables, the C0 node layout of an m-fold Kuhn-subdivided macro simplex).  The
tables must reproduce the reference's layouts exactly -- node order, quadrature
point order, face numbering -- because they fix the memory layout of the
operator's inputs (`w` is (E, n_c0, n_s) in the reference's C0 node order,
`offset` is (E, n_sub, nq, n_s) in its quadrature order).

Reference correspondence (macrohdg, read-only under /root/reference):
  quadrature           fem.py:221-258  collapsed Gauss-Jacobi rule
  simplex_nodes        fem.py:265-412  warp-and-blend nodes (Warburton 2006)
  ReferenceBasis       fem.py:440-489  nodal basis via a Vandermonde solve
  kuhn_subdivision     fem.py:550-579
  macro_c0_map         fem.py:663-724

The nodal (Lagrange) basis is obtained from the orthonormal collapsed-
coordinate (Koornwinder-Dubiner) basis through a Vandermonde inverse, the
well-conditioned construction of Hesthaven & Warburton (2008); tables agree
with the reference's to round-off (tests/test_tables.py).
"""

from __future__ import annotations

import itertools
import math
from dataclasses import dataclass

import numpy as np
from scipy.special import roots_jacobi

from .errors import InvalidConfig

# Warburton's optimised blend parameters (Hesthaven & Warburton, "Nodal
# Discontinuous Galerkin Methods", 2008, Nodes2D/Nodes3D tables).
_BLEND_2D = (0.0, 0.0, 1.4152, 0.1001, 0.2751, 0.9800, 1.0999, 1.2832,
             1.3648, 1.4773, 1.4959, 1.5743, 1.5770, 1.6223, 1.6258)
_BLEND_3D = (0.0, 0.0, 0.0, 0.1002, 1.1332, 1.5608, 1.3413, 1.2577,
             1.1603, 1.10153, 0.6080, 0.4523, 0.8856, 0.8717, 0.9655)


# ---------------------------------------------------------------------------
# quadrature (fem.py:221-258)
# ---------------------------------------------------------------------------

def quadrature(required_degree, d, kind="volume"):
    """Collapsed Gauss-Jacobi rule on the unit d-simplex.

    n = ceil((deg+1)/2) points per collapsed direction; point order is the
    ij-meshgrid order (first collapsed coordinate slowest), weights sum to
    1/d!.  kind='face' gives the rule of the (d-1)-simplex.
    """
    if required_degree < 0:
        raise InvalidConfig(f"required_degree must be >= 0, got {required_degree}")
    if kind == "face":
        return quadrature(required_degree, d - 1, "volume")
    if kind != "volume":
        raise InvalidConfig(f"unknown quadrature kind {kind!r}")
    if d not in (1, 2, 3):
        raise InvalidConfig(f"no simplex rule for dimension {d}")
    n = max(1, math.ceil((required_degree + 1) / 2))
    x0, w0 = roots_jacobi(n, 0.0, 0.0)
    if d == 1:
        return 0.5 * (x0[:, None] + 1), 0.5 * w0
    x1, w1 = roots_jacobi(n, 1.0, 0.0)
    if d == 2:
        a, b = np.meshgrid(x0, x1, indexing="ij")
        r = (1 + a) * (1 - b) / 2 - 1
        pts = np.column_stack([(r.ravel() + 1) / 2, (b.ravel() + 1) / 2])
        return pts, (np.outer(w0, w1) / 2.0).ravel() / 4.0
    x2, w2 = roots_jacobi(n, 2.0, 0.0)
    a, b, c = np.meshgrid(x0, x1, x2, indexing="ij")
    s = (1 + b) * (1 - c) / 2 - 1
    r = (1 + a) * (1 - b) * (1 - c) / 4 - 1
    wts = w0[:, None, None] * w1[None, :, None] * w2[None, None, :] / 8.0
    pts = np.column_stack([(r.ravel() + 1) / 2, (s.ravel() + 1) / 2,
                           (c.ravel() + 1) / 2])
    return pts, wts.ravel() / 8.0


# ---------------------------------------------------------------------------
# 1D ingredients
# ---------------------------------------------------------------------------

def gauss_lobatto(p):
    """p+1 Gauss-Lobatto-Legendre points on [-1, 1], ascending."""
    if p == 0:
        return np.array([0.0])
    if p == 1:
        return np.array([-1.0, 1.0])
    inner, _ = roots_jacobi(p - 1, 1.0, 1.0)
    return np.concatenate([[-1.0], np.sort(inner), [1.0]])


def _edge_warp(p, r):
    """Warburton's 1D warp factor: interpolant of (LGL - equispaced) at r,
    divided by the edge bubble 1-r^2 away from the end points."""
    lgl = gauss_lobatto(p)
    req = np.linspace(-1.0, 1.0, p + 1)
    # Legendre modes by the orthonormal Jacobi recurrence (the reference's
    # evaluation, fem.py:33-66, 280-291): the numpy legvander values differ in
    # the last bit and moved the p >= 3 facet nodes by up to 1.1e-16
    veq = np.column_stack([jacobi_orthonormal(j, 0, 0, req) for j in range(p + 1)])
    pr = np.vstack([jacobi_orthonormal(j, 0, 0, r) for j in range(p + 1)])   # (p+1, npts)
    lag = np.linalg.solve(veq.T, pr)               # Lagrange values (p+1, npts)
    warp = lag.T @ (lgl - req)
    inside = (np.abs(r) < 1.0 - 1e-10).astype(float)
    bubble = 1.0 - (inside * r) ** 2
    return warp / bubble + warp * (inside - 1.0)


def _edge_warp_lagrange(p, r):
    """EvalWarp of Warburton's 3D construction: the same edge warp written in
    Lagrange product form over the interior equispaced points."""
    gx = -gauss_lobatto(p)
    xeq = -1.0 + 2.0 * (p - np.arange(p + 1)) / p
    r = np.asarray(r, dtype=float)
    warp = np.zeros_like(r)
    for i in range(1, p):
        term = np.full_like(r, gx[i] - xeq[i])
        for j in range(1, p):
            if j != i:
                term = term * (r - xeq[j]) / (xeq[i] - xeq[j])
        term = -term / (xeq[i] - xeq[0])
        term = term / (xeq[i] - xeq[p])
        warp = warp + term
    return warp


def _lattice_barycentric(p, nverts):
    """Equispaced barycentric lattice, rows in descending lexicographic order."""
    rows = [c for c in itertools.product(range(p + 1), repeat=nverts)
            if sum(c) == p]
    rows.sort(reverse=True)
    return np.array(rows, dtype=float) / p


def _to_unit_coords(xyz, verts):
    """Barycentric coordinates w.r.t. `verts`, keeping the non-first ones."""
    n = len(verts)
    lhs = np.column_stack([verts, np.ones(n)]).T
    rhs = np.column_stack([xyz, np.ones(len(xyz))]).T
    bary = np.linalg.solve(lhs, rhs).T
    return bary[:, 1:n].copy()


# ---------------------------------------------------------------------------
# warp-and-blend nodes (fem.py:265-412)
# ---------------------------------------------------------------------------

def _triangle_nodes(p):
    alpha = _BLEND_2D[p - 1] if p - 1 < len(_BLEND_2D) else 5.0 / 3.0
    lam = _lattice_barycentric(p, 3)
    verts = np.array([[-1.0, -1 / math.sqrt(3.0)],
                      [1.0, -1 / math.sqrt(3.0)],
                      [0.0, 2 / math.sqrt(3.0)]])
    xy = lam @ verts
    for a, b, opp in ((0, 1, 2), (1, 2, 0), (2, 0, 1)):
        warp = _edge_warp(p, lam[:, b] - lam[:, a])
        amp = 4 * lam[:, a] * lam[:, b] * warp * (1 + (alpha * lam[:, opp]) ** 2)
        xy = xy + amp[:, None] * (verts[b] - verts[a]) / 2
    return _to_unit_coords(xy, verts)


def _face_shift(p, alpha, l1, l2, l3):
    """Tangential displacement of a triangle face (Warburton's EvalShift)."""
    blend = (l2 * l3, l1 * l3, l1 * l2)
    factor = (4 * _edge_warp_lagrange(p, l3 - l2),
              4 * _edge_warp_lagrange(p, l1 - l3),
              4 * _edge_warp_lagrange(p, l2 - l1))
    lref = (l1, l2, l3)
    w = [blend[k] * factor[k] * (1 + (alpha * lref[k]) ** 2) for k in range(3)]
    d1 = w[0] + math.cos(2 * math.pi / 3) * w[1] + math.cos(4 * math.pi / 3) * w[2]
    d2 = math.sin(2 * math.pi / 3) * w[1] + math.sin(4 * math.pi / 3) * w[2]
    return d1, d2


def _tet_nodes(p):
    alpha = _BLEND_3D[p - 1] if p - 1 < len(_BLEND_3D) else 1.0
    tol = 1e-10
    lam = _lattice_barycentric(p, 4)
    v = np.array([[-1.0, -1 / math.sqrt(3.0), -1 / math.sqrt(6.0)],
                  [1.0, -1 / math.sqrt(3.0), -1 / math.sqrt(6.0)],
                  [0.0, 2 / math.sqrt(3.0), -1 / math.sqrt(6.0)],
                  [0.0, 0.0, 3 / math.sqrt(6.0)]])
    xyz = lam @ v
    tan1 = np.array([v[1] - v[0], v[1] - v[0], v[2] - v[1], v[2] - v[0]])
    tan2 = np.array([v[2] - 0.5 * (v[0] + v[1]), v[3] - 0.5 * (v[0] + v[1]),
                     v[3] - 0.5 * (v[1] + v[2]), v[3] - 0.5 * (v[0] + v[2])])
    tan1 /= np.linalg.norm(tan1, axis=1)[:, None]
    tan2 /= np.linalg.norm(tan2, axis=1)[:, None]
    # (off-face, then the three on-face) barycentric columns per face, in
    # Warburton's face frames
    frames = ((3, 2, 0, 1), (2, 3, 0, 1), (0, 3, 1, 2), (1, 3, 0, 2))
    shift = np.zeros_like(xyz)
    for f, (ia, ib, ic, idd) in enumerate(frames):
        la, lb, lc, ld = lam[:, ia], lam[:, ib], lam[:, ic], lam[:, idd]
        w1, w2 = _face_shift(p, alpha, lb, lc, ld)
        blend = lb * lc * ld
        denom = (lb + 0.5 * la) * (lc + 0.5 * la) * (ld + 0.5 * la)
        ok = denom > tol
        blend = np.where(ok, (1 + (alpha * la) ** 2) * blend
                         / np.where(ok, denom, 1.0), 0.0)
        shift += (blend * w1)[:, None] * tan1[f] + (blend * w2)[:, None] * tan2[f]
        edge = (la < tol) & ((lb > tol).astype(int) + (lc > tol).astype(int)
                             + (ld > tol).astype(int) < 3)
        if np.any(edge):
            shift[edge] = w1[edge, None] * tan1[f] + w2[edge, None] * tan2[f]
    return _to_unit_coords(xyz + shift, v)


def simplex_nodes(p, d):
    """Interpolation nodes on the unit d-simplex (warped for p >= 3)."""
    if p < 1:
        raise InvalidConfig(f"degree must be >= 1, got {p}")
    if d == 1:
        return (0.5 * (gauss_lobatto(p) + 1.0))[:, None]
    if d == 2:
        return _triangle_nodes(p)
    if d == 3:
        return _tet_nodes(p)
    raise InvalidConfig(f"unsupported dimension {d}")


# ---------------------------------------------------------------------------
# polynomial space and nodal basis
# ---------------------------------------------------------------------------

def jacobi_orthonormal(n, a, b, x):
    """Orthonormal Jacobi polynomial P_n^{(a,b)} on [-1, 1] by the three-term
    recurrence (weight (1-x)^a (1+x)^b)."""
    x = np.asarray(x, dtype=float)
    g0 = (2.0 ** (a + b + 1) / (a + b + 1) * math.gamma(a + 1)
          * math.gamma(b + 1) / math.gamma(a + b + 1))
    prev = np.full_like(x, 1.0 / math.sqrt(g0))
    if n == 0:
        return prev
    g1 = (a + 1) * (b + 1) / (a + b + 3) * g0
    cur = ((a + b + 2) * x / 2 + (a - b) / 2) / math.sqrt(g1)
    if n == 1:
        return cur
    a_old = 2.0 / (2 + a + b) * math.sqrt((a + 1) * (b + 1) / (a + b + 3))
    for i in range(1, n):
        h = 2 * i + a + b
        a_new = 2.0 / (h + 2) * math.sqrt((i + 1) * (i + 1 + a + b) * (i + 1 + a)
                                          * (i + 1 + b) / ((h + 1) * (h + 3)))
        b_new = -(a * a - b * b) / (h * (h + 2))
        prev, cur = cur, (-a_old * prev + (x - b_new) * cur) / a_new
        a_old = a_new
    return cur


def jacobi_orthonormal_deriv(n, a, b, x):
    x = np.asarray(x, dtype=float)
    if n == 0:
        return np.zeros_like(x)
    return math.sqrt(n * (n + a + b + 1)) * jacobi_orthonormal(n - 1, a + 1, b + 1, x)


def _modes(p, d):
    if d == 1:
        return [(i,) for i in range(p + 1)]
    if d == 2:
        return [(i, j) for i in range(p + 1) for j in range(p + 1 - i)]
    return [(i, j, k) for i in range(p + 1) for j in range(p + 1 - i)
            for k in range(p + 1 - i - j)]


def _collapse(x):
    """Unit-simplex points -> collapsed (Duffy) coordinates in [-1, 1]^d."""
    r = 2 * x - 1
    d = x.shape[1]
    if d == 1:
        return (r[:, 0],)
    if d == 2:
        den = 1.0 - r[:, 1]
        ok = np.abs(den) > 1e-12
        a = np.where(ok, 2 * (1 + r[:, 0]) / np.where(ok, den, 1.0) - 1, -1.0)
        return a, r[:, 1].copy()
    den_a = r[:, 1] + r[:, 2]
    ok_a = np.abs(den_a) > 1e-12
    a = np.where(ok_a, -2 * (1 + r[:, 0]) / np.where(ok_a, den_a, 1.0) - 1, -1.0)
    den_b = 1.0 - r[:, 2]
    ok_b = np.abs(den_b) > 1e-12
    b = np.where(ok_b, 2 * (1 + r[:, 1]) / np.where(ok_b, den_b, 1.0) - 1, -1.0)
    return a, b, r[:, 2].copy()


def _poly_values(p, d, x):
    """Orthonormal (Koornwinder-Dubiner) basis of P_p on the unit simplex."""
    x = np.atleast_2d(np.asarray(x, dtype=float))
    cc = _collapse(x)
    out = np.empty((len(x), len(_modes(p, d))))
    for col, mode in enumerate(_modes(p, d)):
        if d == 1:
            out[:, col] = math.sqrt(2.0) * jacobi_orthonormal(mode[0], 0, 0, cc[0])
        elif d == 2:
            i, j = mode
            a, b = cc
            out[:, col] = (2 * math.sqrt(2.0) * jacobi_orthonormal(i, 0, 0, a)
                           * jacobi_orthonormal(j, 2 * i + 1, 0, b) * (1 - b) ** i)
        else:
            i, j, k = mode
            a, b, c = cc
            out[:, col] = (8.0 * jacobi_orthonormal(i, 0, 0, a)
                           * jacobi_orthonormal(j, 2 * i + 1, 0, b) * (1 - b) ** i
                           * jacobi_orthonormal(k, 2 * (i + j) + 2, 0, c)
                           * (1 - c) ** (i + j))
    return out


def _poly_gradients(p, d, x):
    """Gradients of _poly_values w.r.t. unit-simplex coordinates, by the chain
    rule through the collapsed coordinates (Sherwin-Karniadakis)."""
    x = np.atleast_2d(np.asarray(x, dtype=float))
    cc = _collapse(x)
    modes = _modes(p, d)
    out = np.empty((len(x), len(modes), d))
    J, dJ = jacobi_orthonormal, jacobi_orthonormal_deriv
    for col, mode in enumerate(modes):
        if d == 1:
            out[:, col, 0] = 2 * math.sqrt(2.0) * dJ(mode[0], 0, 0, cc[0])
            continue
        if d == 2:
            i, j = mode
            a, b = cc
            fa, dfa = J(i, 0, 0, a), dJ(i, 0, 0, a)
            gb, dgb = J(j, 2 * i + 1, 0, b), dJ(j, 2 * i + 1, 0, b)
            hb = 0.5 * (1 - b)
            dr = dfa * gb
            ds = dfa * gb * 0.5 * (1 + a)
            if i > 0:
                dr = dr * hb ** (i - 1)
                ds = ds * hb ** (i - 1)
            t = dgb * hb ** i
            if i > 0:
                t = t - 0.5 * i * gb * hb ** (i - 1)
            ds = ds + fa * t
            scale = 4.0 * 2.0 ** (i + 0.5)
            out[:, col, 0] = scale * dr
            out[:, col, 1] = scale * ds
            continue
        i, j, k = mode
        a, b, c = cc
        fa, dfa = J(i, 0, 0, a), dJ(i, 0, 0, a)
        gb, dgb = J(j, 2 * i + 1, 0, b), dJ(j, 2 * i + 1, 0, b)
        hc, dhc = J(k, 2 * (i + j) + 2, 0, c), dJ(k, 2 * (i + j) + 2, 0, c)
        hb, hcc = 0.5 * (1 - b), 0.5 * (1 - c)
        vr = dfa * gb * hc
        if i > 0:
            vr = vr * hb ** (i - 1)
        if i + j > 0:
            vr = vr * hcc ** (i + j - 1)
        t = dgb * hb ** i
        if i > 0:
            t = t - 0.5 * i * gb * hb ** (i - 1)
        if i + j > 0:
            t = t * hcc ** (i + j - 1)
        t = fa * t * hc
        vs = 0.5 * (1 + a) * vr + t
        t2 = dhc * hcc ** (i + j)
        if i + j > 0:
            t2 = t2 - 0.5 * (i + j) * hc * hcc ** (i + j - 1)
        t2 = fa * gb * t2 * hb ** i
        vt = 0.5 * (1 + a) * vr + 0.5 * (1 + b) * t + t2
        scale = 4 * math.sqrt(2.0) * 2.0 ** (2 * i + j + 1.5)
        out[:, col, 0] = scale * vr
        out[:, col, 1] = scale * vs
        out[:, col, 2] = scale * vt
    return out


def mode_count(p, d):
    return math.comb(p + d, d)


def reference_face_vertices(d):
    """Face k of the unit simplex is opposite vertex k."""
    return [tuple(i for i in range(d + 1) if i != k) for k in range(d + 1)]


def unit_simplex_vertices(d):
    verts = np.zeros((d + 1, d))
    for k in range(d):
        verts[k + 1, k] = 1.0
    return verts


def face_embedding(d, k):
    """x = v0 + span @ xhat maps the reference facet onto face k."""
    verts = unit_simplex_vertices(d)
    fv = reference_face_vertices(d)[k]
    v0 = verts[fv[0]]
    return v0, (verts[list(fv[1:])] - v0).T


class ReferenceBasis:
    """Nodal degree-p basis on the unit d-simplex with its quadrature tables
    (fem.py:440-489): nodes (N,d), phi (nq,N), dphi (nq,N,d), quad_pts,
    quad_wts, facet (the (d-1)-dimensional basis), face_nodes."""

    def __init__(self, p, d, quad_degree=None):
        if d not in (1, 2, 3):
            raise InvalidConfig(f"dimension must be 1, 2 or 3, got {d}")
        if not 1 <= p <= 10:
            raise InvalidConfig(f"degree must be in [1, 10], got {p}")
        self.p, self.d = p, d
        self.nodes = simplex_nodes(p, d)
        self.n_nodes = len(self.nodes)
        self.vandermonde = _poly_values(p, d, self.nodes)
        self.cond = np.linalg.cond(self.vandermonde)
        self.v_inv = np.linalg.inv(self.vandermonde)
        self.quad_degree = 2 * p + 1 if quad_degree is None else quad_degree
        self.quad_pts, self.quad_wts = quadrature(self.quad_degree, d)
        self.phi = self.eval_at(self.quad_pts)
        self.dphi = self.grad_at(self.quad_pts)
        self.facet = ReferenceBasis(p, d - 1, self.quad_degree) if d > 1 else None
        x = self.nodes
        self.face_nodes = [
            np.nonzero(np.abs(x.sum(axis=1) - 1) < 1e-10)[0] if k == 0
            else np.nonzero(np.abs(x[:, k - 1]) < 1e-10)[0]
            for k in range(d + 1)
        ]

    def eval_at(self, points):
        return _poly_values(self.p, self.d, points) @ self.v_inv

    def grad_at(self, points):
        return np.einsum("qmk,mn->qnk", _poly_gradients(self.p, self.d, points),
                         self.v_inv)


# ---------------------------------------------------------------------------
# Kuhn subdivision and the macro C0 layout (fem.py:550-724)
# ---------------------------------------------------------------------------

def kuhn_vertices(d):
    verts = np.zeros((d + 1, d))
    for k in range(1, d + 1):
        verts[k, :k] = 1.0
    return verts


def kuhn_subdivision(m, d):
    """The m^d positively oriented sub-simplices of the path simplex
    {1 >= x_1 >= .. >= x_d >= 0}: Kuhn cells of the 1/m grid whose centroid
    is ordered; odd cells swap their last two vertices."""
    subs = []
    for cell in itertools.product(range(m), repeat=d):
        for perm in itertools.permutations(range(d)):
            verts = np.zeros((d + 1, d))
            verts[0] = cell
            for k, axis in enumerate(perm):
                verts[k + 1] = verts[k]
                verts[k + 1, axis] += 1.0
            verts = verts / m
            cen = verts.mean(axis=0)
            if np.all(np.diff(cen) <= 1e-12):
                if np.linalg.det((verts[1:] - verts[0]).T) < 0:
                    verts[[d - 1, d]] = verts[[d, d - 1]]
                subs.append(verts)
    if len(subs) != m ** d:
        raise InvalidConfig(f"Kuhn subdivision gave {len(subs)} cells, "
                            f"expected {m ** d}")
    return np.array(subs)


def _macro_face_planes(d):
    """Macro face k is opposite Kuhn vertex k: x_1 = 1, x_k = x_{k+1}, x_d = 0."""
    planes = []
    n = np.zeros(d)
    n[0] = 1.0
    planes.append((n, 1.0))
    for k in range(1, d):
        n = np.zeros(d)
        n[k - 1], n[k] = 1.0, -1.0
        planes.append((n, 0.0))
    n = np.zeros(d)
    n[d - 1] = 1.0
    planes.append((n, 0.0))
    return planes


def first_occurrence_ids(points, tol=1e-7):
    """Ids by first occurrence: rows closer than tol share the id of the
    earliest such row (the reference's dedup semantics, fem.py:599-633)."""
    points = np.asarray(points, dtype=float)
    n = len(points)
    dist = np.sqrt(((points[:, None, :] - points[None, :, :]) ** 2).sum(-1))
    ids = np.full(n, -1, dtype=np.int64)
    reps = []
    for i in range(n):
        if ids[i] >= 0:
            continue
        ids[i] = len(reps)
        reps.append(i)
        close = np.nonzero(dist[i] < tol)[0]
        ids[close[ids[close] < 0]] = ids[i]
    return ids, points[reps]


@dataclass
class MacroC0Map:
    """C0 layout of one m-subdivided macro simplex: scatter[s, i] is the
    macro node id of local node i of sub-element s; face_tiles[f] lists the
    (sub, local face) tiles of macro face f; face_scatter[f][t, j] is the
    face-unique trace node of facet node j of tile t."""

    m: int
    p: int
    d: int
    sub_vertices: np.ndarray
    scatter: np.ndarray
    n_unique: int
    unique_nodes: np.ndarray
    face_tiles: list
    face_scatter: list
    n_face_unique: int
    face_unique_nodes: list

    @property
    def n_sub(self):
        return len(self.sub_vertices)


def macro_c0_map(m, p, d, basis=None):
    if m < 1:
        raise InvalidConfig(f"subdivision count must be >= 1, got {m}")
    basis = basis or ReferenceBasis(p, d)
    subs = kuhn_subdivision(m, d)
    nodes = [subs[s, 0] + basis.nodes @ (subs[s, 1:] - subs[s, 0])
             for s in range(len(subs))]
    ids, unique = first_occurrence_ids(np.concatenate(nodes))
    if len(unique) != math.comb(m * p + d, d):
        raise InvalidConfig("C0 node count does not match the lattice count")
    scatter = ids.reshape(len(subs), basis.n_nodes)

    planes = _macro_face_planes(d)
    tiles = [[] for _ in planes]
    fverts_all = reference_face_vertices(d)
    for s in range(len(subs)):
        for f, fv in enumerate(fverts_all):
            pts = subs[s, list(fv)]
            for mf, (nrm, off) in enumerate(planes):
                if np.all(np.abs(pts @ nrm - off) < 1e-12):
                    tiles[mf].append((s, f))
                    break
    for t in tiles:
        if len(t) != m ** (d - 1):
            raise InvalidConfig("macro face tiling is incomplete")

    fnodes = basis.facet.nodes if d > 1 else np.zeros((1, 0))
    n_fu = math.comb(m * p + d - 1, d - 1)
    face_scatter, face_unique = [], []
    for mf in range(len(planes)):
        pts = []
        for s, f in tiles[mf]:
            fv = fverts_all[f]
            v0 = subs[s, fv[0]]
            pts.append(v0 + fnodes @ (subs[s, list(fv[1:])] - v0))
        fid, fu = first_occurrence_ids(np.concatenate(pts))
        if len(fu) != n_fu:
            raise InvalidConfig("face C0 node count does not match the lattice")
        face_scatter.append(fid.reshape(len(tiles[mf]), len(fnodes)))
        face_unique.append(fu)
    return MacroC0Map(m=m, p=p, d=d, sub_vertices=subs, scatter=scatter,
                      n_unique=len(unique), unique_nodes=unique,
                      face_tiles=tiles, face_scatter=face_scatter,
                      n_face_unique=n_fu, face_unique_nodes=face_unique)
