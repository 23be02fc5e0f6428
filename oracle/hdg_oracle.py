"""CPU oracle for the macro-element HDG operator -- TEST INFRASTRUCTURE ONLY.

This module is a numpy restatement of the reference algorithm on the hot path
(macrohdg, /root/reference/pkg/src/macrohdg).  It is imported only by
`tests/`, `__graft_entry__.smoke()` and `bench.py`'s cpu_baseline/reference
leg, always as the CHECKER, never as the computation being measured or
shipped.  The product path (`paper_2507_22195_b200`) never imports it.

Pinning: every function here is checked against golden vectors produced by
running the reference itself in the build container (`tests/golden/
make_golden.py` -> `tests/golden/*.npz`, see tests/test_oracle_golden.py), and
against the reference's own known-answer tests restated in tests/ (free-stream
preservation, two-triangle hand assembly, dense block elimination).

Derivatives use complex-step differentiation exactly like the reference
(gas.py:32-45); the pointwise routines are complex-safe (branch decisions
on real parts).

Reference map:
  pointwise gas algebra           gas.py:92-226
  log_mean / two-point fluxes     fluxes.py:46-242
  residuals                       assembly.py:459-549
  linearization + S / precond     assembly.py:772-1026
  condensed operator              assembly.py:1028-1180
  fgmres / solve_condensed        solver.py:42-170
  newton_solve / advance_step     time_march.py:185-340
"""

from __future__ import annotations

import math

import numpy as np
from scipy.linalg import cho_factor, cho_solve, lu_factor, lu_solve, solve_triangular, LinAlgError

EPS_CS = 1e-150


# ---------------------------------------------------------------------------
# pointwise gas algebra (gas.py:92-226), complex-safe
# ---------------------------------------------------------------------------

def _rabs(x):
    return np.where(np.real(x) >= 0, x, -x)


class Gas:
    def __init__(self, gamma=1.4):
        self.g = gamma

    def primitive(self, u):
        rho = u[..., 0]
        mom = u[..., 1:-1]
        vel = mom / rho[..., None]
        p = (self.g - 1) * (u[..., -1] - 0.5 * np.sum(mom * vel, axis=-1))
        return rho, vel, p

    def conservative(self, rho, vel, p):
        rho, vel, p = np.asarray(rho), np.asarray(vel), np.asarray(p)
        u = np.empty(vel.shape[:-1] + (vel.shape[-1] + 2,),
                     dtype=np.result_type(rho, vel, p, float))
        u[..., 0] = rho
        u[..., 1:-1] = rho[..., None] * vel
        u[..., -1] = p / (self.g - 1) + 0.5 * rho * np.sum(vel * vel, axis=-1)
        return u

    def entropy_vars(self, u):
        rho, vel, p = self.primitive(u)
        s = np.log(p) - self.g * np.log(rho)
        beta = rho / p
        v = np.empty_like(u)
        v[..., 0] = (self.g - s) / (self.g - 1) - 0.5 * beta * np.sum(vel * vel, axis=-1)
        v[..., 1:-1] = beta[..., None] * vel
        v[..., -1] = -beta
        return v

    def from_entropy(self, v):
        beta = -v[..., -1]
        if not np.all(np.real(beta) > 0):
            raise OracleInadmissible("entropy")
        vel = v[..., 1:-1] / beta[..., None]
        s = self.g - (self.g - 1) * (v[..., 0] + 0.5 * beta * np.sum(vel * vel, axis=-1))
        rho = np.exp(-(s + np.log(beta)) / (self.g - 1))
        return self.conservative(rho, vel, rho / beta)

    def flux(self, u):
        rho, vel, p = self.primitive(u)
        d = u.shape[-1] - 2
        f = np.empty(u.shape + (d,), dtype=u.dtype)
        f[..., 0, :] = u[..., 1:-1]
        f[..., 1:-1, :] = u[..., 1:-1, None] * vel[..., None, :]
        for a in range(d):
            f[..., a + 1, a] += p
        f[..., -1, :] = (u[..., -1] + p)[..., None] * vel
        return f

    def flux_normal(self, u, n):
        rho, vel, p = self.primitive(u)
        vn = np.sum(vel * n, axis=-1)
        f = np.empty_like(u)
        f[..., 0] = np.sum(u[..., 1:-1] * n, axis=-1)
        f[..., 1:-1] = u[..., 1:-1] * vn[..., None] + p[..., None] * n
        f[..., -1] = (u[..., -1] + p) * vn
        return f

    def wavespeed(self, u, n):
        rho, vel, p = self.primitive(u)
        return _rabs(np.sum(vel * n, axis=-1)) + np.sqrt(self.g * p / rho)

    # -- diffusive terms (gas.py:229-280) ------------------------------------
    def grads_conservative(self, u, gu):
        rho, vel, p = self.primitive(u)
        grho, gmom, gre = gu[..., 0, :], gu[..., 1:-1, :], gu[..., -1, :]
        gvel = (gmom - vel[..., None] * grho[..., None, :]) / rho[..., None, None]
        ke = 0.5 * np.sum(vel * vel, axis=-1)
        conv = np.sum(u[..., 1:-1, None] * gvel, axis=-2)
        gp = (self.g - 1) * (gre - ke[..., None] * grho - conv)
        gt = self.g * (rho[..., None] * gp - p[..., None] * grho) / rho[..., None] ** 2
        return gvel, gt

    def grads_entropy(self, v, gv):
        ve = v[..., -1]
        gve = gv[..., -1, :]
        gvm = gv[..., 1:-1, :]
        gvel = (v[..., 1:-1, None] * gve[..., None, :] - ve[..., None, None] * gvm) \
            / ve[..., None, None] ** 2
        return gvel, self.g * gve / ve[..., None] ** 2

    def viscous_flux(self, visc, vel, gvel, gt):
        mu = visc.mu / visc.reynolds
        kappa = visc.mu / (visc.reynolds * (self.g - 1) * visc.mach ** 2 * visc.prandtl)
        d = vel.shape[-1]
        div = np.trace(gvel, axis1=-2, axis2=-1)
        tau = mu * (gvel + np.swapaxes(gvel, -1, -2))
        for a in range(d):
            tau[..., a, a] -= (2.0 / 3.0) * mu * div
        g = np.zeros(vel.shape[:-1] + (d + 2, d), dtype=gvel.dtype)
        g[..., 1:-1, :] = -tau
        g[..., -1, :] = -(np.sum(tau * vel[..., :, None], axis=-2) + kappa * gt)
        return g

    def penalty(self, visc, d):
        diag = np.empty(d + 2)
        diag[0] = 0.0
        diag[1:-1] = visc.mu / visc.reynolds
        diag[-1] = visc.mu / (visc.reynolds * (self.g - 1) * visc.mach ** 2 * visc.prandtl)
        return diag


class OracleInadmissible(FloatingPointError):
    def __init__(self, kind, where=None):
        super().__init__(f"non-admissible {kind} state at {where}")
        self.kind = kind
        self.where = where


def log_mean(a, b):
    """fluxes.py:46-57: series branch when |b/a - 1| < 1e-4."""
    ratio = b / a
    near = np.abs(np.real(ratio) - 1.0) < 1e-4
    zeta = (b - a) / (b + a)
    z2 = zeta * zeta
    series = (a + b) / (2 * (1 + z2 * (1 / 3 + z2 * (1 / 5 + z2 / 7))))
    exact = (b - a) / np.log(np.where(near, 2.0, ratio))
    return np.where(near, series, exact)


def _tangents(n):
    n = np.asarray(n, dtype=float)
    if n.shape[-1] == 2:
        return (np.stack([-n[..., 1], n[..., 0]], axis=-1),)
    k = np.argmin(np.abs(n), axis=-1)
    e = np.eye(3)[k]
    t1 = e - np.sum(e * n, axis=-1)[..., None] * n
    t1 = t1 / np.linalg.norm(t1, axis=-1)[..., None]
    return t1, np.cross(n, t1)


def numerical_flux(gas, kind, u, uh, n):
    """Interface flux F(u, u_hat; n) of the four families (fluxes.py:120-242)."""
    if kind == "lf":
        lam = gas.wavespeed(uh, n)
        return 0.5 * (gas.flux_normal(u, n) + gas.flux_normal(uh, n)) \
            - 0.5 * lam[..., None] * (uh - u)
    rho, vel, p = gas.primitive(u)
    rho_h, vel_h, p_h = gas.primitive(uh)
    beta, beta_h = rho / p, rho_h / p_h
    rho_ln, beta_ln = log_mean(rho, rho_h), log_mean(beta, beta_h)
    vel_avg = 0.5 * (vel + vel_h)
    vv_avg = 0.5 * (np.sum(vel * vel, axis=-1) + np.sum(vel_h * vel_h, axis=-1))
    p_bar = (0.5 * (rho + rho_h)) / (0.5 * (beta + beta_h))
    vn = np.sum(vel_avg * n, axis=-1)
    f = np.empty(np.broadcast_shapes(u.shape, uh.shape), dtype=np.result_type(u, uh))
    f1 = rho_ln * vn
    f[..., 0] = f1
    fm = vel_avg * f1[..., None] + p_bar[..., None] * n
    f[..., 1:-1] = fm
    f[..., -1] = (1.0 / (beta_ln * (gas.g - 1)) - 0.5 * vv_avg) * f1 \
        + np.sum(vel_avg * fm, axis=-1)
    if kind == "ec":
        return f
    if kind == "es":
        li, lh = gas.wavespeed(u, n), gas.wavespeed(uh, n)
        lam = np.where(np.real(li) > np.real(lh), li, lh)
        return f - 0.5 * lam[..., None] * (uh - u)
    # kepes: eigenvector-scaled dissipation on the entropy-variable jump
    g = gas.g
    ns = u.shape[-1]
    c = np.sqrt(g * p_bar / rho_ln)
    h = g / (beta_ln * (g - 1)) + 0.5 * vv_avg
    shape = f.shape
    R = np.zeros(shape[:-1] + (ns, ns), dtype=f.dtype)
    R[..., 0, 0] = 1.0
    R[..., 1:-1, 0] = vel_avg - c[..., None] * n
    R[..., -1, 0] = h - c * vn
    R[..., 0, 1] = 1.0
    R[..., 1:-1, 1] = vel_avg
    R[..., -1, 1] = 0.5 * vv_avg
    for k, t in enumerate(_tangents(n)):
        R[..., 1:-1, 2 + k] = t
        R[..., -1, 2 + k] = np.sum(vel_avg * t, axis=-1)
    R[..., 0, -1] = 1.0
    R[..., 1:-1, -1] = vel_avg + c[..., None] * n
    R[..., -1, -1] = h + c * vn
    T = np.empty(shape, dtype=f.dtype)
    T[..., 0] = rho_ln / (2 * g)
    T[..., 1] = rho_ln * (g - 1) / g
    T[..., 2:-1] = p_bar[..., None]
    T[..., -1] = rho_ln / (2 * g)
    lam = np.empty(shape, dtype=f.dtype)
    lam[..., 0] = vn - c
    lam[..., 1:-1] = vn[..., None]
    lam[..., -1] = vn + c
    x = _rabs(p - p_h) / (p + p_h)
    theta = x / np.sqrt(x + 1e-12)
    full = _rabs(vn) + c
    lam_abs = (1 - theta[..., None]) * _rabs(lam) + theta[..., None] * full[..., None]
    dv = gas.entropy_vars(uh) - gas.entropy_vars(u)
    proj = np.einsum("...ij,...i->...j", R, dv)
    return f - 0.5 * np.einsum("...ij,...j->...i", R, lam_abs * T * proj)


def _cs_jacobian_q(fn, q):
    """Complex-step Jacobian over the (state, direction) axes of q."""
    shape = q.shape
    flat = q.reshape(shape[:-2] + (-1,))
    jac = cs_jacobian(lambda qf: fn(qf.reshape(qf.shape[:-1] + shape[-2:])), flat)
    return jac.reshape(jac.shape[:-1] + shape[-2:])


def cs_jacobian(fn, x):
    """Complex-step Jacobian over the last axis (gas.py:32-45)."""
    x = np.asarray(x, dtype=float)
    cols = []
    for k in range(x.shape[-1]):
        xc = x.astype(complex)
        xc[..., k] += 1j * EPS_CS
        cols.append(np.imag(fn(xc)) / EPS_CS)
    return np.stack(cols, axis=-1)


# ---------------------------------------------------------------------------
# operator
# ---------------------------------------------------------------------------

class OracleHDG:
    """Residual and linearization of the inviscid macro-element HDG scheme on
    an `HDGTables` instance (formulation 'entropy' or 'conservative',
    periodic or with a free-stream state on boundary faces)."""

    def __init__(self, tables, flux="es", formulation="entropy", gamma=1.4,
                 freestream=None, viscosity=None):
        self.t = tables
        self.gas = Gas(gamma)
        self.kind = flux
        self.form = formulation
        self.freestream = None if freestream is None else np.asarray(freestream, float)
        self.visc = viscosity
        if viscosity is not None:
            self._gradient_operators()

    # -- viscous level-1 operators (assembly.py:326-371) ----------------------
    def _gradient_operators(self):
        t = self.t
        E, nc, d = t.mesh.n_macros, t.layout.n_unique, t.d
        vol_w, dphi_phys = t.vol_w, t.dphi_phys
        mass = np.zeros((E, nc, nc))
        stiff = np.zeros((E, d, nc, nc))
        for s in range(t.layout.n_sub):
            ids = t.layout.scatter[s]
            mloc = np.einsum("eq,qi,qj->eij", vol_w[:, s], t.phi, t.phi)
            kloc = np.einsum("eq,eqjb,qi->ebji", vol_w[:, s], dphi_phys[:, s], t.phi)
            np.add.at(mass, (slice(None), ids[:, None], ids[None, :]), mloc)
            np.add.at(stiff, (slice(None), slice(None), ids[:, None], ids[None, :]), kloc)
        self.mass, self.stiff = mass, stiff
        self.mass_factor = [cho_factor(mass[e]) for e in range(E)]
        self.minvk = np.stack([np.stack([cho_solve(self.mass_factor[e], stiff[e, b])
                                         for b in range(d)]) for e in range(E)])
        self.edge = np.stack([np.einsum("eq,qi,qj,eb->eijb", t.face_w[:, k], t.phi_face[k], t.fphi,
                                        t.face_normals[:, k]) for k in range(t.n_st)], axis=1)

    def mass_solve(self, y):
        out = np.empty_like(y)
        nc = y.shape[1]
        for e in range(y.shape[0]):
            out[e] = cho_solve(self.mass_factor[e], y[e].reshape(nc, -1),
                               check_finite=False).reshape(y[e].shape)
        return out

    def solve_gradient(self, w, trace):
        """M q_b = E_b w^ - K_b w (assembly.py:398-411)."""
        t = self.t
        rhs = -np.einsum("ebji,eit->ejtb", self.stiff, w)
        for k in range(t.n_st):
            contrib = np.einsum("eijb,ejt->eitb", self.edge[:, k], self._gather(trace, k))
            np.add.at(rhs, (slice(None), t.face_rows[k]), contrib)
        return self.mass_solve(rhs)

    def _grads(self, wq, qq):
        return (self.gas.grads_entropy(wq, qq) if self.form == "entropy"
                else self.gas.grads_conservative(wq, qq))

    def viscous_volume_flux(self, wq, qq, uq):
        gv, gt = self._grads(wq, qq)
        return self.gas.viscous_flux(self.visc, self.gas.primitive(uq)[1], gv, gt)

    def viscous_face_flux(self, wq, qq, uq, nrm):
        g = self.viscous_volume_flux(wq, qq, uq)
        return np.einsum("...sa,...a->...s", g, nrm)

    # working variables <-> conservative
    def to_u(self, w):
        return w if self.form == "conservative" else self.gas.from_entropy(w)

    def from_u(self, u):
        return u if self.form == "conservative" else self.gas.entropy_vars(u)

    def _gather(self, trace, k):
        t = self.t
        return trace[t.face_id_st[:, k][:, None], t.trace_idx[:, k]]

    def _checked_u(self, w, where):
        try:
            u = self.to_u(w)
        except OracleInadmissible as exc:
            raise OracleInadmissible("entropy", where) from exc
        rho = np.real(u[..., 0])
        p = np.real(self.gas.primitive(u)[2])
        if not (np.all(rho > 0) and np.all(p > 0)):
            raise OracleInadmissible("state", where)
        return u

    def volume_quad_states(self, w):
        t = self.t
        out = np.empty((w.shape[0], t.layout.n_sub, t.phi.shape[0], t.n_s), dtype=w.dtype)
        for s in range(t.layout.n_sub):
            wq = np.einsum("qi,eis->eqs", t.phi, w[:, t.layout.scatter[s]])
            out[:, s] = self.to_u(wq)
        return out

    def residuals(self, w, trace, alpha=None, offset=None, q=None):
        """(r_w, r_trace[, r_q]) of assembly.py:459-549."""
        t, gas = self.t, self.gas
        visc = self.visc is not None
        dtype = np.result_type(w, trace, float)
        r_w = np.zeros(w.shape, dtype=dtype)
        r_tr = np.zeros(trace.shape, dtype=dtype)
        r_q = np.zeros(w.shape + (t.d,), dtype=dtype) if visc else None
        vol_w = t.vol_w
        dphi_phys = t.dphi_phys
        for s in range(t.layout.n_sub):
            ids = t.layout.scatter[s]
            wq = np.einsum("qi,eis->eqs", t.phi, w[:, ids])
            uq = self._checked_u(wq, f"volume sub {s}")
            fl = gas.flux(uq)
            if visc:
                qq = np.einsum("qi,eitb->eqtb", t.phi, q[:, ids])
                fl = fl + self.viscous_volume_flux(wq, qq, uq)
                r_q[:, ids] += np.einsum("eq,qi,eqtb->eitb", vol_w[:, s], t.phi, qq)
                r_q[:, ids] += np.einsum("eq,eqib,eqt->eitb", vol_w[:, s], dphi_phys[:, s], wq)
            r_w[:, ids] -= np.einsum("eq,eqia,eqsa->eis", vol_w[:, s],
                                     dphi_phys[:, s], fl)
            if alpha is not None:
                tmp = alpha * uq
                if offset is not None:
                    tmp = tmp + offset[:, s]
                r_w[:, ids] += np.einsum("eq,qi,eqs->eis", vol_w[:, s], t.phi, tmp)
        face_w = t.face_w
        for k in range(t.n_st):
            rows = t.face_rows[k]
            wq = np.einsum("qi,eis->eqs", t.phi_face[k], w[:, rows])
            whq = np.einsum("qi,eis->eqs", t.fphi, self._gather(trace, k))
            uq = self._checked_u(wq, f"face tile {k}")
            uhq = self._checked_u(whq, f"trace tile {k}")
            nrm = t.face_normals[:, k][:, None, :]
            fl = numerical_flux(gas, self.kind, uq, uhq, nrm)
            if visc:
                qq = np.einsum("qi,eitb->eqtb", t.phi_face[k], q[:, rows])
                gn = self.viscous_face_flux(wq, qq, uq, nrm)
                fl = fl + (gn - 0.5 * gas.penalty(self.visc, t.d) * (whq - wq))
                r_q[:, rows] -= np.einsum("eq,qi,eqt,eb->eitb", face_w[:, k], t.phi_face[k], whq,
                                          t.face_normals[:, k])
            r_w[:, rows] += np.einsum("eq,qi,eqs->eis", face_w[:, k], t.phi_face[k], fl)
            vals = np.einsum("eq,qi,eqs->eis", face_w[:, k], t.fphi, fl)
            mask = t.boundary_st[:, k]
            if self.freestream is not None and mask.any():
                uinf = np.broadcast_to(self.freestream, uhq[mask].shape)
                ghost = numerical_flux(gas, self.kind, uinf, uhq[mask], -nrm[mask])
                if visc:
                    winf = np.broadcast_to(self.from_u(self.freestream), whq[mask].shape)
                    ghost = ghost + (0.0 - 0.5 * gas.penalty(self.visc, t.d) * (whq[mask] - winf))
                vals[mask] += np.einsum("eq,qi,eqs->eis", face_w[mask][:, k], t.fphi, ghost)
            np.add.at(r_tr, (t.face_id_st[:, k][:, None], t.trace_idx[:, k]), vals)
        if visc:
            return r_w, r_tr, r_q
        return r_w, r_tr

    def linearize(self, w, trace, alpha=0.0, ptc_weight=0.0, precond=True, q=None):
        return OracleLin(self, w, trace, alpha, ptc_weight, precond, q)

    def integrals(self, w):
        """Volume integrals of assembly.py:595-620."""
        t, gas = self.t, self.gas
        out = dict(entropy=0.0, thermo_entropy=0.0, kinetic_energy=0.0, mass=0.0,
                   total_energy=0.0)
        vw = t.vol_w
        for s in range(t.layout.n_sub):
            wq = np.einsum("qi,eis->eqs", t.phi, w[:, t.layout.scatter[s]])
            u = self.to_u(wq)
            rho, vel, p = gas.primitive(u)
            sp = np.log(p) - gas.g * np.log(rho)
            out["entropy"] += float(np.sum(vw[:, s] * (-rho * sp / (gas.g - 1))))
            out["thermo_entropy"] += float(np.sum(vw[:, s] * rho * sp))
            out["kinetic_energy"] += float(np.sum(vw[:, s] * 0.5 * rho * np.sum(vel ** 2, -1)))
            out["mass"] += float(np.sum(vw[:, s] * rho))
            out["total_energy"] += float(np.sum(vw[:, s] * u[..., -1]))
        return out


class OracleLin:
    """Static condensation of the linearized system (assembly.py:772-1180,
    inviscid): S per macro (LU), face quadrature tensors hw / hhat / ptc,
    face-block preconditioner (Cholesky if symmetric SPD else LU)."""

    def __init__(self, op, w, trace, alpha, ptc_weight, precond=True, q=None):
        t, gas = op.t, op.gas
        self.op = op
        self.shape = trace.shape
        self.viscous = op.visc is not None
        E, nc, ns = w.shape
        d = t.d
        weight = alpha + ptc_weight
        S = np.zeros((E, nc, ns, nc, ns))
        vol_w = t.vol_w
        dphi_phys = t.dphi_phys
        self.avq_sub, self.avq_face, self.avhatq = [], [], []
        for s in range(t.layout.n_sub):
            ids = t.layout.scatter[s]
            wq = np.einsum("qi,eis->eqs", t.phi, w[:, ids])
            qq = np.einsum("qi,eitb->eqtb", t.phi, q[:, ids]) if self.viscous else None

            def transport(wc, qf=qq):
                u = op.to_u(wc)
                f = gas.flux(u)
                if qf is not None:
                    f = f + op.viscous_volume_flux(wc, qf, u)
                return f

            fgw = cs_jacobian(transport, wq)   # (E,q,s,a,t)
            blk = -np.einsum("eq,eqia,eqsat,qj->eisjt", vol_w[:, s], dphi_phys[:, s],
                             fgw, t.phi, optimize=True)
            if weight != 0.0:
                tw = (np.broadcast_to(np.eye(ns), wq.shape + (ns,)) if op.form == "conservative"
                      else cs_jacobian(op.to_u, wq))
                blk = blk + weight * np.einsum("eq,qi,eqst,qj->eisjt", vol_w[:, s], t.phi,
                                               tw, t.phi, optimize=True)
            S_view = S.transpose(0, 1, 3, 2, 4)                     # (E, i, j, s, t)
            S_view[:, ids[:, None], ids[None, :]] += blk.transpose(0, 1, 3, 2, 4)
            if self.viscous:
                gq = _cs_jacobian_q(lambda qc: op.viscous_volume_flux(wq, qc, op.to_u(wq)), qq)
                avq = -np.einsum("eq,eqia,eqsatb,ql->eisltb", vol_w[:, s], dphi_phys[:, s], gq,
                                 t.phi, optimize=True)
                self.avq_sub.append(avq)
                corr = np.einsum("eisltb,eblj->eisjt", avq, op.minvk[:, :, ids, :], optimize=True)
                S[:, ids] -= corr
        self.hw, self.hhat, self.hh = [], [], []
        face_w = t.face_w
        for k in range(t.n_st):
            rows = t.face_rows[k]
            wq = np.einsum("qi,eis->eqs", t.phi_face[k], w[:, rows])
            whq = np.einsum("qi,eis->eqs", t.fphi, op._gather(trace, k))
            nrm = t.face_normals[:, k][:, None, :]
            uhq = op.to_u(whq)
            qq = np.einsum("qi,eitb->eqtb", t.phi_face[k], q[:, rows]) if self.viscous else None
            pen = gas.penalty(op.visc, d) if self.viscous else None

            def face_total(wc, whc, qf=qq):
                u, uh = op.to_u(wc), op.to_u(whc)
                f = numerical_flux(gas, op.kind, u, uh, nrm)
                if qf is not None:
                    f = f + (op.viscous_face_flux(wc, qf, u, nrm) - 0.5 * pen * (whc - wc))
                return f

            hw = cs_jacobian(lambda wc: face_total(wc, whq), wq)
            hhat = cs_jacobian(lambda wc: face_total(wq, wc), whq)
            hh = hhat.copy()
            mask = t.boundary_st[:, k]
            if op.freestream is not None and mask.any():
                uinf = np.broadcast_to(op.freestream, uhq.shape)
                winf = np.broadcast_to(op.from_u(op.freestream), whq.shape)

                def ghost_total(wc):
                    f = numerical_flux(gas, op.kind, uinf, op.to_u(wc), -nrm)
                    if pen is not None:
                        f = f + (0.0 - 0.5 * pen * (wc - winf))
                    return f

                gh = cs_jacobian(ghost_total, whq)
                gh[~mask] = 0.0
                hh = hh + gh
            if ptc_weight != 0.0:
                tw = (np.broadcast_to(np.eye(ns), whq.shape + (ns,)) if op.form == "conservative"
                      else cs_jacobian(op.to_u, whq))
                hh = hh + (-ptc_weight * tw)
            self.hw.append(hw)
            self.hhat.append(hhat)
            self.hh.append(hh)
            blk = np.einsum("eq,qi,eqst,qj->eisjt", face_w[:, k], t.phi_face[k], hw,
                            t.phi_face[k], optimize=True)
            S_view = S.transpose(0, 1, 3, 2, 4)
            S_view[:, rows[:, None], rows[None, :]] += blk.transpose(0, 1, 3, 2, 4)
            if self.viscous:
                uq = op.to_u(wq)
                gqf = _cs_jacobian_q(lambda qc: op.viscous_face_flux(wq, qc, uq, nrm)
                                     - 0.5 * pen * (whq - wq), qq)
                avqf = np.einsum("eq,qi,eqstb,ql->eisltb", face_w[:, k], t.phi_face[k], gqf,
                                 t.phi_face[k], optimize=True)
                avh = np.einsum("eq,qi,eqstb,ql->eisltb", face_w[:, k], t.fphi, gqf,
                                t.phi_face[k], optimize=True)
                self.avq_face.append(avqf)
                self.avhatq.append(avh)
                corr = np.einsum("eisltb,eblj->eisjt", avqf, op.minvk[:, :, rows, :], optimize=True)
                S[:, rows] -= corr
        Smat = S.reshape(E, nc * ns, nc * ns)
        self.lu = []
        for e in range(E):
            lu = lu_factor(Smat[e], check_finite=False)
            if not np.isfinite(lu[0]).all() or np.abs(np.diagonal(lu[0])).min() == 0.0:
                raise ArithmeticError(f"singular local matrix on macro {e}")
            self.lu.append(lu)
        self.S = Smat
        if precond:
            self._build_precond()

    def _build_precond(self):
        t = self.op.t
        ns = t.n_s
        face_w = t.face_w
        # face-block preconditioner (assembly.py:994-1026)
        F, nt, _ = self.shape
        blocks = np.zeros((F, nt, ns, nt, ns))
        for k in range(t.n_st):
            vals = np.einsum("eq,qi,eqst,qj->eisjt", face_w[:, k], t.fphi, self.hh[k],
                             t.fphi, optimize=True)
            fid, tidx = t.face_id_st[:, k], t.trace_idx[:, k]
            np.add.at(blocks, (fid[:, None, None], tidx[:, :, None], slice(None),
                               tidx[:, None, :]), vals.transpose(0, 1, 3, 2, 4))
        self.blocks = blocks.reshape(F, nt * ns, nt * ns)
        self.pre = []
        for f in range(F):
            a = self.blocks[f]
            scale = max(1.0, float(np.abs(a).max()))
            fac = None
            if np.abs(a - a.T).max() <= 1e-12 * scale:
                try:
                    c = cho_factor(a, check_finite=False)
                    fac = ("chol", c)
                except LinAlgError:
                    fac = None
            if fac is None:
                lu = lu_factor(a, check_finite=False)
                if not np.isfinite(lu[0]).all() or np.abs(np.diagonal(lu[0])).min() == 0.0:
                    raise ArithmeticError(f"singular trace block on face {f}")
                fac = ("lu", lu)
            self.pre.append(fac)

    # block actions (assembly.py:1030-1127)
    def solve_schur(self, r):
        out = np.empty_like(r)
        for e in range(r.shape[0]):
            out[e] = lu_solve(self.lu[e], r[e].reshape(-1), check_finite=False).reshape(r[e].shape)
        return out

    def _tile_apply_to_trace(self, tensors, xq_fn):
        t = self.op.t
        out = np.zeros(self.shape)
        for k in range(t.n_st):
            tmp = np.einsum("eqst,eqt->eqs", tensors[k], xq_fn(k))
            vals = np.einsum("eq,qi,eqs->eis", t.face_w[:, k], t.fphi, tmp)
            np.add.at(out, (t.face_id_st[:, k][:, None], t.trace_idx[:, k]), vals)
        return out

    def apply_vvhat(self, xh):
        t = self.op.t
        E = t.mesh.n_macros
        out = np.zeros((E, t.layout.n_unique, t.n_s))
        for k in range(t.n_st):
            xq = np.einsum("qi,eis->eqs", t.fphi, self.op._gather(xh, k))
            tmp = np.einsum("eqst,eqt->eqs", self.hhat[k], xq)
            out[:, t.face_rows[k]] += np.einsum("eq,qi,eqs->eis", t.face_w[:, k],
                                                t.phi_face[k], tmp)
        return out

    def apply_vhatv(self, x):
        t = self.op.t
        return self._tile_apply_to_trace(
            self.hw, lambda k: np.einsum("qi,eis->eqs", t.phi_face[k], x[:, t.face_rows[k]]))

    def apply_vhatvhat(self, xh):
        t = self.op.t
        return self._tile_apply_to_trace(
            self.hh, lambda k: np.einsum("qi,eis->eqs", t.fphi, self.op._gather(xh, k)))

    # viscous level-1 couplings (assembly.py:1037-1084)
    def apply_qv(self, x):
        return np.einsum("ebji,eit->ejtb", self.op.stiff, x)

    def apply_qvhat(self, xh):
        t = self.op.t
        out = np.zeros((t.mesh.n_macros, t.layout.n_unique, t.n_s, t.d))
        for k in range(t.n_st):
            contrib = np.einsum("eijb,ejt->eitb", self.op.edge[:, k], self.op._gather(xh, k))
            np.add.at(out, (slice(None), t.face_rows[k]), -contrib)
        return out

    def apply_vq(self, y):
        t = self.op.t
        out = np.zeros((t.mesh.n_macros, t.layout.n_unique, t.n_s))
        for s in range(t.layout.n_sub):
            ids = t.layout.scatter[s]
            out[:, ids] += np.einsum("eisltb,eltb->eis", self.avq_sub[s], y[:, ids])
        for k in range(t.n_st):
            rows = t.face_rows[k]
            out[:, rows] += np.einsum("eisltb,eltb->eis", self.avq_face[k], y[:, rows])
        return out

    def apply_vhatq(self, y):
        t = self.op.t
        out = np.zeros(self.shape)
        for k in range(t.n_st):
            vals = np.einsum("eisltb,eltb->eis", self.avhatq[k], y[:, t.face_rows[k]])
            np.add.at(out, (t.face_id_st[:, k][:, None], t.trace_idx[:, k]), vals)
        return out

    def matvec(self, xh):
        out = self.apply_vhatvhat(xh)
        g2 = -self.apply_vvhat(xh)
        if self.viscous:
            yq = self.op.mass_solve(self.apply_qvhat(xh))
            g2 += self.apply_vq(yq)
            out -= self.apply_vhatq(yq)
        z = self.solve_schur(g2)
        out += self.apply_vhatv(z)
        if self.viscous:
            out -= self.apply_vhatq(self.op.mass_solve(self.apply_qv(z)))
        return out

    def condensed_rhs(self, r_w, r_trace, r_q=None):
        rw, rh = -r_w, -r_trace
        if self.viscous:
            mq = self.op.mass_solve(r_q)
            rw = rw + self.apply_vq(mq)
            rh = rh + self.apply_vhatq(mq)
        z = self.solve_schur(rw)
        b = rh - self.apply_vhatv(z)
        if self.viscous:
            b += self.apply_vhatq(self.op.mass_solve(self.apply_qv(z)))
        return b

    def recover(self, r_w, d_trace, r_q=None):
        rw = -r_w
        if self.viscous:
            rw = rw + self.apply_vq(self.op.mass_solve(r_q))
        g2 = -self.apply_vvhat(d_trace)
        if self.viscous:
            g2 += self.apply_vq(self.op.mass_solve(self.apply_qvhat(d_trace)))
        d_w = self.solve_schur(rw + g2)
        if not self.viscous:
            return d_w
        d_q = -self.op.mass_solve(r_q + self.apply_qv(d_w) + self.apply_qvhat(d_trace))
        return d_w, d_q

    def apply_preconditioner(self, r):
        out = np.empty_like(r)
        for f in range(r.shape[0]):
            kind, fac = self.pre[f]
            v = r[f].reshape(-1)
            out[f] = (cho_solve(fac, v, check_finite=False) if kind == "chol"
                      else lu_solve(fac, v, check_finite=False)).reshape(r[f].shape)
        return out


# ---------------------------------------------------------------------------
# Krylov (solver.py:42-170)
# ---------------------------------------------------------------------------

def fgmres(op, b, precond=None, rel_tol=1e-3, restart=60, max_iters=None):
    """Restarted flexible GMRES, MGS + Givens, stagnation -> unconverged."""
    b = np.asarray(b, dtype=float)
    n = b.size
    max_iters = 10 * restart if max_iters is None else max_iters
    nb = float(np.linalg.norm(b))
    if nb == 0.0:
        return np.zeros(n), 0, 0.0, True
    x = np.zeros(n)
    total, prev = 0, math.inf
    while True:
        r = b - op(x) if x.any() else b.copy()
        beta = float(np.linalg.norm(r))
        rel = beta / nb
        if rel <= rel_tol:
            return x, total, rel, True
        if total >= max_iters or rel >= prev * (1 - 1e-12):
            return x, total, rel, False
        prev = rel
        m = min(restart, max_iters - total)
        V = np.empty((m + 1, n))
        Z = np.empty((m, n))
        H = np.zeros((m + 1, m))
        cs, sn, g = np.empty(m), np.empty(m), np.zeros(m + 1)
        g[0] = beta
        V[0] = r / beta
        k = 0
        for j in range(m):
            z = precond(V[j]) if precond is not None else V[j]
            wv = op(z)
            Z[j] = z
            for i in range(j + 1):
                H[i, j] = V[i] @ wv
                wv -= H[i, j] * V[i]
            hn = float(np.linalg.norm(wv))
            H[j + 1, j] = hn
            if hn > 1e-300:
                V[j + 1] = wv / hn
            for i in range(j):
                tmp = cs[i] * H[i, j] + sn[i] * H[i + 1, j]
                H[i + 1, j] = -sn[i] * H[i, j] + cs[i] * H[i + 1, j]
                H[i, j] = tmp
            den = math.hypot(H[j, j], H[j + 1, j])
            if den == 0.0:
                break
            cs[j], sn[j] = H[j, j] / den, H[j + 1, j] / den
            H[j, j], H[j + 1, j] = den, 0.0
            g[j + 1] = -sn[j] * g[j]
            g[j] *= cs[j]
            total += 1
            k = j + 1
            if abs(g[j + 1]) / nb <= rel_tol or hn <= 1e-300:
                break
        if k > 0:
            y = solve_triangular(H[:k, :k], g[:k], check_finite=False)
            x = x + Z[:k].T @ y
