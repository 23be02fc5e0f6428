"""Device-resident Discretization / LinearizedSystem: the drop-in surface.

Mirrors the reference's object API (macrohdg assembly.py): same class and
method names, argument meaning, return containers and exceptions, so the
Newton/DIRK/Krylov callers (`time_march`, `solver`) and user code written
against the reference work unchanged.  Every operator runs in
libmhdg_b200.so on the GPU; arrays are torch CUDA tensors (numpy inputs are
uploaded).  There is no CPU fallback.

  Discretization.residuals        -> mhdg_residual        (assembly.py:459-549)
  Discretization.jacobian         -> mhdg_linearize       (assembly.py:697-976)
  LinearizedSystem.matvec         -> mhdg_matvec          (assembly.py:1131-1143)
  LinearizedSystem.condensed_rhs  -> mhdg_condensed_rhs   (assembly.py:1145-1157)
  LinearizedSystem.recover        -> mhdg_recover         (assembly.py:1159-1173)
  LinearizedSystem.apply_preconditioner -> mhdg_precond   (assembly.py:1175-1180)
  Discretization.volume_quad_states / integrals / to_/from_conservative
"""

from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass

import numpy as np

from . import _native as N
from .errors import InvalidConfig, SingularLocalMatrix
from .fluxes import DissipationSpec
from .gas import GasModel
from .tables import HDGTables


def _torch():
    import torch

    return torch


def as_device(a, device):
    """float64 contiguous CUDA tensor view/copy of a numpy array or tensor."""
    torch = _torch()
    if isinstance(a, torch.Tensor):
        t = a
        if t.device != device or t.dtype != torch.float64:
            t = t.to(device=device, dtype=torch.float64)
        return t.contiguous()
    return torch.as_tensor(np.ascontiguousarray(a, dtype=np.float64), device=device)


@dataclass
class FieldSet:
    """Nodal coefficients: w (E, nc, n_s), trace (F, nt, n_s), q if viscous."""

    w: object
    trace: object
    q: object = None

    def copy(self):
        def cp(a):
            return None if a is None else (a.clone() if hasattr(a, "clone") else a.copy())

        return FieldSet(cp(self.w), cp(self.trace), cp(self.q))


@dataclass
class ResidualSet:
    r_w: object
    r_trace: object
    r_q: object = None
    _disc: object = None

    def norm(self):
        cached = self.__dict__.get("_norm")
        if cached is not None:
            return cached
        if self._disc is not None:
            return self._disc.residual_norm(self)
        parts = [self.r_w, self.r_trace] + ([self.r_q] if self.r_q is not None else [])
        return math.sqrt(sum(float((p * p).sum()) for p in parts))

    def max_abs(self):
        parts = [self.r_w, self.r_trace] + ([self.r_q] if self.r_q is not None else [])
        return max(float(p.abs().max()) for p in parts)


@dataclass(frozen=True)
class StageContext:
    """Temporal term alpha * u(w) + offset at volume quadrature points."""

    alpha: float
    offset: object = None
    dt: float | None = None


@dataclass(frozen=True)
class FreeStream:
    state: np.ndarray


def boundary_trace_operator(kind, state=None):
    if kind == "periodic":
        return None
    if kind == "freestream":
        if state is None:
            raise InvalidConfig("freestream boundary needs a state")
        return FreeStream(np.asarray(state, dtype=float))
    raise InvalidConfig(f"unsupported boundary kind {kind!r}")


# (m, p) with m > 1 on the device (mhdg_macro.cuh: the orders 5 nc of S and
# 5 nt of the face blocks have batched Gauss-Jordan instantiations)
MACRO_SUBDIVISIONS = {(2, 1), (2, 2), (2, 3), (3, 1)}


class Discretization:
    """Spatial operator on a macro mesh at degree p, evaluated on the GPU.

    Supported on the device: d = 3, m = 1, p = 1..4 (viscous: 1..3), default
    quadrature, entropy or conservative formulation, lf/ec/es/kepes fluxes,
    periodic or free-stream boundaries, Euler or Navier-Stokes (constant mu).  Anything else raises InvalidConfig
    (the reference-only features are listed in DESIGN.md).
    """

    def __init__(self, mesh, p, gas=None, formulation="entropy", flux=None,
                 viscosity=None, quad_degree=None, boundary=None, supg=False,
                 device=None, tables=None, n_owned_faces=0):
        if formulation not in ("conservative", "entropy"):
            raise InvalidConfig(f"unknown formulation {formulation!r}")
        if supg:
            raise InvalidConfig("SUPG streamline term is not on the B200 path")
        if tables is None and mesh.has_boundary and boundary is None:
            raise InvalidConfig("mesh has boundary faces, a boundary treatment is required")
        if mesh.dim != 3:
            raise InvalidConfig("the B200 operator is 3D")
        if mesh.m > 1 and ((mesh.m, p) not in MACRO_SUBDIVISIONS or viscosity is not None
                           or boundary is not None or tables is not None):
            raise InvalidConfig(f"m > 1 on the B200 operator: (m, p) in {sorted(MACRO_SUBDIVISIONS)}, "
                                "inviscid, periodic, single partition")
        if quad_degree not in (None, 2 * p + 1):
            raise InvalidConfig("the B200 operator uses the default quadrature degree 2p+1")
        if not 1 <= p <= 4:
            raise InvalidConfig("the B200 operator supports p = 1..4")
        torch = _torch()
        lib = N.require_cuda()
        self.device = torch.device("cuda", torch.cuda.current_device()) if device is None \
            else torch.device(device)
        self.mesh = mesh
        self.p = p
        self.gas = gas or GasModel()
        self.formulation = formulation
        self.flux = flux or DissipationSpec("kepes")
        self.viscosity = viscosity
        self.supg = False
        self.boundary = boundary
        self.d = mesh.dim
        self.n_s = self.d + 2
        self.tables = t = HDGTables(mesh, p, quad_degree) if tables is None else tables
        self.n_owned_faces = int(n_owned_faces) or t.n_faces
        self.basis, self.layout = t.basis, t.layout
        self.n_st, self.n_faces = t.n_st, t.n_faces
        self.phi = t.phi
        self.domain_volume = t.domain_volume
        self._lib = lib
        self._keep = []
        tab = N.Tables()
        tab.dim, tab.p, tab.m = 3, p, mesh.m
        tab.n_macros, tab.n_faces = t.mesh.n_macros, t.n_faces
        tab.nn, tab.nq = t.phi.shape[1], t.phi.shape[0]
        tab.nfn, tab.nqf = t.fphi.shape[1], t.fphi.shape[0]
        tab.n_st, tab.n_sub = t.n_st, t.layout.n_sub
        tab.formulation = 1 if formulation == "entropy" else 0
        tab.flux_kind = self.flux.code
        tab.gamma = float(self.gas.gamma)

        def keep(a, dtype):
            a = np.ascontiguousarray(a, dtype=dtype)
            self._keep.append(a)
            return N.np_ptr(a)

        tab.phi = keep(t.phi, np.float64)
        tab.dphi = keep(t.dphi, np.float64)
        tab.quad_wts = keep(t.quad_wts, np.float64)
        tab.phi_face = keep(t.phi_face, np.float64)
        tab.fphi = keep(t.fphi, np.float64)
        tab.facet_wts = keep(t.facet_wts, np.float64)
        tab.face_rows = keep(t.face_rows, np.int64)
        tab.sub_det = keep(t.sub_det[:, 0], np.float64)
        tab.sub_inv_jac = keep(t.sub_inv_jac[:, 0], np.float64)
        tab.face_normals = keep(t.face_normals, np.float64)
        tab.face_area = keep(t.face_area, np.float64)
        tab.face_id_st = keep(t.face_id_st, np.int64)
        tab.trace_idx = keep(t.trace_idx, np.int64)
        tab.boundary_st = keep(t.boundary_st, np.uint8)
        tab.face_sides = keep(t.face_sides, np.int64) if t.face_sides is not None else None
        tab.freestream = keep(boundary.state, np.float64) if boundary is not None else None
        tab.n_owned_faces = int(n_owned_faces)
        tab.nc, tab.nt = t.layout.n_unique, t.n_trace
        if mesh.m > 1:
            tptr, tlist, fptr, flist = t.trace_csr()
            tab.scatter = keep(t.layout.scatter, np.int64)
            tab.sub_det_all = keep(t.sub_det, np.float64)
            tab.sub_inv_jac_all = keep(t.sub_inv_jac, np.float64)
            tab.trace_ptr, tab.trace_list = keep(tptr, np.int64), keep(tlist, np.int64)
            tab.face_ptr, tab.face_list = keep(fptr, np.int64), keep(flist, np.int64)
        if viscosity is not None:
            if p > 3:
                raise InvalidConfig("the viscous B200 operator supports p = 1..3")
            minv, pref, kref, eref = t.viscous_reference()
            tab.has_visc = 1
            tab.reynolds, tab.mach = float(viscosity.reynolds), float(viscosity.mach)
            tab.prandtl, tab.mu = float(viscosity.prandtl), float(viscosity.mu)
            tab.minv_ref, tab.pref = keep(minv, np.float64), keep(pref, np.float64)
            tab.kref, tab.eref = keep(kref, np.float64), keep(eref, np.float64)
        err = C.c_int(0)
        with torch.cuda.device(self.device):
            self._ctx = lib.mhdg_create(C.byref(tab), self.device.index, C.byref(err))
        if not self._ctx:
            N.raise_for(err.value or 6, None, "(mhdg_create)")
        self._keep = []
        self._scalar = torch.zeros(8, dtype=torch.float64, device=self.device)
        sizes = (C.c_int64 * 6)()
        lib.mhdg_lin_sizes(self._ctx, sizes)
        self.lin_sizes = tuple(int(s) for s in sizes)

    def __del__(self):
        # device engines built on this context go first (they hold graphs
        # with this context's buffers)
        engines = self.__dict__.pop("_krylov_engines", None)
        if engines:
            engines.clear()
        ctx = getattr(self, "_ctx", None)
        if ctx:
            try:
                self._lib.mhdg_destroy(ctx)
            except Exception:
                pass
            self._ctx = None

    # -- geometry views (host) -------------------------------------------------
    @property
    def node_coords(self):
        return self.tables.node_coords

    @property
    def trace_coords(self):
        return self.tables.trace_coords

    @property
    def quad_coords(self):
        return self.tables.quad_coords

    @property
    def vol_w(self):
        return self.tables.vol_w

    @property
    def face_rows(self):
        return self.tables.face_rows

    @property
    def face_id_st(self):
        return self.tables.face_id_st

    @property
    def trace_idx(self):
        return self.tables.trace_idx

    def gj_fallbacks(self):
        """(S blocks, face blocks) of the last linearization that needed the
        partial-pivoting pass of the batched Gauss-Jordan."""
        out = (C.c_int * 2)()
        N.raise_for(self._lib.mhdg_gj_fallbacks(self._ctx, C.cast(out, C.c_void_p), N.stream_handle()))
        return int(out[0]), int(out[1])

    def batched_inverse(self, mats):
        """Inverses of a batch of square matrices (order 20, 50 or 100) by
        the device Gauss-Jordan that replaces the reference's per-macro
        lu_factor / lu_solve (assembly.py:718-733).  mats: (n_mat, n, n)
        float64 on the device; returns (inverses, fallbacks) where fallbacks
        counts the matrices that needed the partial-pivoting pass.  Raises
        SingularLocalMatrix(macro = index in the batch) like the reference."""
        torch = _torch()
        a = self._dev(mats).to(torch.float64)
        if a.dim() != 3 or a.shape[1] != a.shape[2]:
            raise InvalidConfig("batched_inverse expects (n_mat, n, n)")
        work = a.contiguous().clone()
        fb, item = C.c_int(0), C.c_int64(-1)
        rc = self._lib.mhdg_batched_inverse(self._ctx, int(a.shape[1]), int(a.shape[0]), N.ptr(work),
                                            C.cast(C.byref(fb), C.c_void_p), C.cast(C.byref(item), C.c_void_p),
                                            N.stream_handle())
        if rc == 3:
            raise SingularLocalMatrix(f"singular condensed block on macro {item.value}", macro=int(item.value))
        N.raise_for(rc, None, "(batched_inverse)")
        # the kernel writes the inverse column-major
        return work.transpose(1, 2), int(fb.value)

    @property
    def launch_count(self):
        return int(self._lib.mhdg_launch_count(self._ctx))

    # -- helpers ---------------------------------------------------------------
    def _dev(self, a):
        return as_device(a, self.device)

    def _fields(self, fields):
        return self._dev(fields.w), self._dev(fields.trace)

    def _q(self, fields):
        if self.viscosity is None:
            return None
        if fields.q is None:
            raise InvalidConfig("viscous discretization needs fields.q")
        return self._dev(fields.q)

    def residual_norm(self, res):
        parts = [res.r_w, res.r_trace] + ([res.r_q] if res.r_q is not None else [])
        return math.sqrt(sum(self.vdot(p, p) for p in parts))

    def vdot(self, x, y):
        """Deterministic device dot product (float)."""
        self._lib.mhdg_dot(self._ctx, x.numel(), N.ptr(x), N.ptr(y), N.ptr(self._scalar),
                           N.stream_handle())
        return float(self._scalar[0].item())

    # -- state handling ------------------------------------------------------
    def to_conservative(self, w, where=""):
        if self.formulation == "conservative":
            return self._dev(w)
        w = self._dev(w)
        out = self._torch_empty_like(w)
        st = N.Status()
        rc = self._lib.mhdg_to_conservative(self._ctx, w.numel() // 5, N.ptr(w), N.ptr(out),
                                            C.byref(st), N.stream_handle())
        if rc:
            from .errors import NonAdmissibleEntropyState

            raise NonAdmissibleEntropyState("non-positive inverse temperature", where=where)
        return out

    def from_conservative(self, u):
        if self.formulation == "conservative":
            return self._dev(u)
        u = self._dev(u)
        out = self._torch_empty_like(u)
        self._lib.mhdg_from_conservative(self._ctx, u.numel() // 5, N.ptr(u), N.ptr(out),
                                         N.stream_handle())
        return out

    def _torch_empty_like(self, t):
        return _torch().empty_like(t)

    def project(self, state_fn):
        """Nodal interpolation of an exact conservative-state function; the
        conversion to working variables uses the host gas algebra so the
        projected coefficients are bit-identical to the reference's."""
        u_nodes = state_fn(self.node_coords)
        u_trace = state_fn(self.trace_coords)
        if self.formulation == "entropy":
            u_nodes, u_trace = self.gas.entropy_vars(u_nodes), self.gas.entropy_vars(u_trace)
        fields = FieldSet(w=self._dev(u_nodes), trace=self._dev(u_trace))
        if self.viscosity is not None:
            fields.q = self.solve_gradient(fields)
        return fields

    def solve_gradient(self, fields):
        """Discrete gradient q_b = M^-1 (E_b w^ - K_b w) (assembly.py:398-411)."""
        torch = _torch()
        w, tr = self._fields(fields)
        q = torch.empty(tuple(w.shape) + (self.d,), dtype=torch.float64, device=self.device)
        rc = self._lib.mhdg_solve_gradient(self._ctx, N.ptr(w), N.ptr(tr), N.ptr(q),
                                           N.stream_handle())
        N.raise_for(rc)
        return q

    def volume_quad_states(self, fields):
        torch = _torch()
        w = self._dev(fields.w)
        E = self.tables.mesh.n_macros
        out = torch.empty((E, self.layout.n_sub, self.phi.shape[0], 5), dtype=torch.float64,
                          device=self.device)
        st = N.Status()
        rc = self._lib.mhdg_volume_quad_states(self._ctx, N.ptr(w), N.ptr(out), C.byref(st),
                                               N.stream_handle())
        N.raise_for(rc, st)
        return out

    # -- residuals -------------------------------------------------------------
    def residuals(self, fields, stage=None, check=True, sync=True):
        torch = _torch()
        w, tr = self._fields(fields)
        q = self._q(fields)
        r_w = torch.empty_like(w)
        r_tr = torch.empty_like(tr)
        r_q = torch.empty_like(q) if q is not None else None
        off = None
        if stage is not None and stage.offset is not None:
            off = self._dev(stage.offset)
        st = N.Status()
        rc = self._lib.mhdg_residual(
            self._ctx, N.ptr(w), N.ptr(tr), N.ptr(q), int(stage is not None),
            float(stage.alpha) if stage is not None else 0.0, N.ptr(off), int(bool(check)),
            N.ptr(r_w), N.ptr(r_tr), N.ptr(r_q), int(bool(sync)), C.byref(st), N.stream_handle())
        N.raise_for(rc, st)
        return ResidualSet(r_w=r_w, r_trace=r_tr, r_q=r_q, _disc=self)

    def residual_and_norm(self, fields, stage=None):
        """(residuals, ||R||) with ONE device round trip: the residual
        kernels, the admissibility status and the three deterministic dot
        products are queued, then status and dots come back together
        (ResidualSet.norm order: r_w, r_trace, r_q).  Raises like
        residuals()."""
        res = self.residuals(fields, stage, check=True, sync=False)
        parts = [res.r_w, res.r_trace] + ([res.r_q] if res.r_q is not None else [])
        stream = N.stream_handle()
        for i, p in enumerate(parts):
            N.raise_for(self._lib.mhdg_dot(self._ctx, p.numel(), N.ptr(p), N.ptr(p),
                                           N.ptr(self._scalar) + 8 * i, stream))
        host = self.__dict__.get("_host_scalar")
        if host is None:
            host = self._host_scalar = _torch().zeros(8, dtype=_torch().float64).pin_memory()
        host[: len(parts)].copy_(self._scalar[: len(parts)], non_blocking=True)
        st = N.Status()
        N.raise_for(self._lib.mhdg_status_fetch(self._ctx, C.byref(st), stream), st)
        sq = host.tolist()
        norm = math.sqrt(sum(sq[: len(parts)]))
        res._norm = norm
        return res, norm

    def apply_update(self, fields, d_w, d_trace, d_q=None):
        """New FieldSet w + d_w, trace + d_trace (, q + d_q) on the device
        (library axpby, one rounding per entry like numpy's +)."""
        torch = _torch()
        stream = N.stream_handle()

        def add(a, b):
            a, b = self._dev(a), self._dev(b)
            out = torch.empty_like(a)
            N.raise_for(self._lib.mhdg_axpby(self._ctx, a.numel(), 1.0, N.ptr(a), 1.0, N.ptr(b),
                                             N.ptr(out), stream))
            return out

        q = None
        if d_q is not None:
            q = add(fields.q, d_q)
        elif fields.q is not None:
            q = self._dev(fields.q).clone()
        return FieldSet(add(fields.w, d_w), add(fields.trace, d_trace), q)

    def jacobian(self, fields, stage=None, ptc_weight=0.0, sparse_local_threshold=2048):
        return LinearizedSystem(self, fields, stage, ptc_weight)

    # -- monitors ----------------------------------------------------------------
    def integrals(self, fields):
        w = self._dev(fields.w)
        out = (C.c_double * 5)()
        self._lib.mhdg_integrals(self._ctx, N.ptr(w), out, N.stream_handle())
        keys = ("entropy", "thermo_entropy", "kinetic_energy", "mass", "total_energy")
        return {k: float(out[i]) for i, k in enumerate(keys)}

    def kinetic_energy_dissipation(self, fields):
        """eps = (2 mu_eff / |Omega|) int rho |curl V|^2 / 2 (assembly.py:622-648)."""
        if self.viscosity is None:
            raise InvalidConfig("dissipation rate needs a viscous setup")
        out = (C.c_double * 1)()
        rc = self._lib.mhdg_dissipation(self._ctx, N.ptr(self._dev(fields.w)), N.ptr(self._q(fields)),
                                        out, N.stream_handle())
        N.raise_for(rc)
        return float(out[0]) / self.domain_volume

    def entropy_identity_defect(self, fields):
        """sum v . R_V - sum v^ . R_V^ against minus the summed face entropy
        residuals (assembly.py:649-672); returns (lhs, rhs, |lhs - rhs|).
        Zero up to round-off for the EC flux; the dissipative fluxes produce
        entropy."""
        w, tr = self._fields(fields)
        res = self.residuals(FieldSet(w, tr, self._q(fields)), stage=None)
        out = (C.c_double * 3)()
        N.raise_for(self._lib.mhdg_entropy_identity(self._ctx, N.ptr(w), N.ptr(tr), N.ptr(res.r_w),
                                                    N.ptr(res.r_trace), out, N.stream_handle()))
        return float(out[0]), float(out[1]), float(out[2])

    def total_generalized_entropy(self, fields):
        v = self.integrals(fields)
        return v["entropy"], v["thermo_entropy"]

    def l2_error(self, fields, exact_fn, component=0):
        """L2 norm of (component of u_h - exact) (assembly.py:674-684); the
        device quadrature states, summed per sub-element in the reference's
        order."""
        u_q = self.volume_quad_states(fields).cpu().numpy()
        total = 0.0
        for s in range(self.layout.n_sub):
            u_ex = exact_fn(self.quad_coords[:, s])
            diff = u_q[:, s, :, component] - u_ex[..., component]
            total += float(np.sum(self.vol_w[:, s] * diff ** 2))
        return math.sqrt(total)

    def max_wavespeed(self, fields):
        u = self.volume_quad_states(fields).cpu().numpy()
        rho, vel, p = self.gas.primitive(u)
        c = np.sqrt(self.gas.gamma * p / rho)
        return float((np.linalg.norm(vel, axis=-1) + c).max())


class LinearizedSystem:
    """Static condensation on the device: S^-1 per macro, face linearization
    tensors, face-block preconditioner inverses (assembly.py:755-1180)."""

    def __init__(self, disc, fields, stage, ptc_weight):
        torch = _torch()
        self.disc = disc
        self.viscous = disc.viscosity is not None
        w, tr = disc._fields(fields)
        q = disc._q(fields)
        self.trace_shape = tuple(tr.shape)
        self.alloc(disc)
        alpha = float(stage.alpha) if stage is not None else 0.0
        st = N.Status()
        rc = disc._lib.mhdg_linearize(disc._ctx, N.ptr(w), N.ptr(tr), N.ptr(q), alpha,
                                      float(ptc_weight), C.byref(self._buf), C.byref(st),
                                      N.stream_handle())
        N.raise_for(rc, st)
        self.n_unsym = int(st.n_unsym)

    def alloc(self, disc):
        torch = _torch()
        sz = disc.lin_sizes
        for name, n in zip(("sinv", "hw", "hhat", "hh", "pinv", "wlin"), sz):
            setattr(self, name, torch.empty(n, dtype=torch.float64, device=disc.device))
        self._buf = N.LinBuffers(*(N.ptr(getattr(self, n)) for n in
                                   ("sinv", "hw", "hhat", "hh", "pinv", "wlin")))

    def _out_trace(self):
        return _torch().empty(self.trace_shape, dtype=_torch().float64, device=self.disc.device)

    def matvec(self, xh):
        d = self.disc
        x = d._dev(xh).reshape(self.trace_shape)
        y = self._out_trace()
        rc = d._lib.mhdg_matvec(d._ctx, C.byref(self._buf), N.ptr(x), N.ptr(y), N.stream_handle())
        N.raise_for(rc)
        return y

    def condensed_rhs(self, res):
        d = self.disc
        rw, rt = d._dev(res.r_w), d._dev(res.r_trace)
        rq = d._dev(res.r_q) if self.viscous else None
        b = self._out_trace()
        rc = d._lib.mhdg_condensed_rhs(d._ctx, C.byref(self._buf), N.ptr(rw), N.ptr(rt), N.ptr(rq),
                                       N.ptr(b), N.stream_handle())
        N.raise_for(rc)
        return b

    def recover(self, res, d_trace):
        d = self.disc
        rw = d._dev(res.r_w)
        rq = d._dev(res.r_q) if self.viscous else None
        x = d._dev(d_trace).reshape(self.trace_shape)
        dw = _torch().empty_like(rw)
        dq = _torch().empty_like(rq) if self.viscous else None
        rc = d._lib.mhdg_recover(d._ctx, C.byref(self._buf), N.ptr(rw), N.ptr(rq), N.ptr(x),
                                 N.ptr(dw), N.ptr(dq), N.stream_handle())
        N.raise_for(rc)
        return dw, dq

    def apply_preconditioner(self, r):
        d = self.disc
        r = d._dev(r).reshape(self.trace_shape)
        z = self._out_trace()
        rc = d._lib.mhdg_precond(d._ctx, C.byref(self._buf), N.ptr(r), N.ptr(z), N.stream_handle())
        N.raise_for(rc)
        return z
