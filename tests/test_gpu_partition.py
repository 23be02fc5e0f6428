"""Partitioned device operator on one GPU: 2 and 3 macro-range partitions
(local tables, owned + ghost faces, remote preconditioner sides) exchanged
in-process (partition.LoopbackExchange) must reproduce the single-partition
device results: residual, matvec and preconditioner bit for bit."""

import ctypes as C

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _setup(world, flux="es", p=3):
    import torch

    from paper_2507_22195_b200 import Discretization, DissipationSpec, GasModel, StageContext
    from paper_2507_22195_b200.assembly import FieldSet
    from paper_2507_22195_b200.mesh import build_box_macro_mesh
    from paper_2507_22195_b200.partition import LocalPartition, LoopbackExchange

    gas = GasModel(1.4)
    mesh = build_box_macro_mesh(np.array([[0.0, 1.0]] * 3), (3, 2, 2), 1)
    spec = DissipationSpec(flux)
    full = Discretization(mesh, p=p, gas=gas, flux=spec, device="cuda:0")
    t = full.tables
    rng = np.random.default_rng(77)
    E, nc, F, nt = mesh.n_macros, t.layout.n_unique, t.n_faces, t.n_trace

    def st(n):
        return gas.entropy_vars(gas.conservative(rng.uniform(0.9, 1.1, n),
                                                 rng.uniform(-0.5, 0.5, (n, 3)),
                                                 rng.uniform(0.9, 1.1, n)))

    w, tr = st(E * nc).reshape(E, nc, 5), st(F * nt).reshape(F, nt, 5)
    x = rng.standard_normal(tr.shape)
    parts = [LocalPartition(t, g, world) for g in range(world)]
    discs = [Discretization(mesh, p=p, gas=gas, flux=spec, device="cuda:0", tables=pp.tables,
                            n_owned_faces=pp.n_owned) for pp in parts]
    return full, parts, discs, LoopbackExchange(parts), w, tr, x, FieldSet, StageContext, torch


@pytest.mark.parametrize("world", [2, 3])
def test_partitioned_kernels_match_single_device(cuda_ok, world):
    from paper_2507_22195_b200 import _native as N
    from paper_2507_22195_b200.assembly import LinearizedSystem

    full, parts, discs, ex, w, tr, x, FieldSet, StageContext, torch = _setup(world)
    alpha = 120.0
    off = -alpha * full.volume_quad_states(FieldSet(w, tr)).cpu().numpy()
    ref = full.residuals(FieldSet(w, tr), StageContext(alpha, off))
    ref_lin = full.jacobian(FieldSet(w, tr), StageContext(alpha, off), ptc_weight=1.0)
    y_ref = ref_lin.matvec(x)
    z_ref = ref_lin.apply_preconditioner(x)

    rts, rws, lins = [], [], []
    for pp, d in zip(parts, discs):
        wl, trl = pp.local_fields(w, tr)
        lo, hi = pp.macro_lo, pp.macro_hi
        res = d.residuals(FieldSet(wl, trl), StageContext(alpha, off[lo:hi]))
        rws.append(res.r_w)
        rts.append(res.r_trace)
        lin = LinearizedSystem.__new__(LinearizedSystem)
        lin.disc, lin.viscous, lin.trace_shape = d, False, tuple(trl.shape)
        lin.alloc(d)
        stt = N.Status()
        wl_d, trl_d = d._fields(FieldSet(wl, trl))
        rc = d._lib.mhdg_linearize_local(d._ctx, N.ptr(wl_d), N.ptr(trl_d), None, alpha, 1.0,
                                         C.byref(lin._buf), C.byref(stt), N.stream_handle())
        assert rc == 0
        lins.append(lin)
    ex.reduce_partials(rts)
    nqf = full.tables.fphi.shape[0]
    remote = ex.gather_sides([l.hh for l in lins], nqf)
    for pp, d, lin, hr in zip(parts, discs, lins, remote):
        stt = N.Status()
        tid = torch.as_tensor(pp.remote_tidx, device=d.device)
        ar = torch.as_tensor(pp.remote_area, device=d.device)
        hr = hr.contiguous()
        rc = d._lib.mhdg_precond_factor(d._ctx, C.byref(lin._buf), int(ar.numel()), N.ptr(hr),
                                        N.ptr(tid), N.ptr(ar), C.byref(stt), N.stream_handle())
        assert rc == 0
    ys = [lin.matvec(torch.as_tensor(x[pp.global_faces], device="cuda:0"))
          for pp, lin in zip(parts, lins)]
    ex.reduce_partials(ys)
    for pp, rw, rt, y, lin in zip(parts, rws, rts, ys, lins):
        own = pp.global_faces[: pp.n_owned]
        no = pp.n_owned
        assert torch.equal(rw, ref.r_w[pp.macro_lo:pp.macro_hi])
        assert torch.equal(rt[:no], ref.r_trace[torch.as_tensor(own, device="cuda:0")])
        assert torch.equal(y[:no], y_ref[torch.as_tensor(own, device="cuda:0")])
        z = lin.apply_preconditioner(torch.as_tensor(x[pp.global_faces], device="cuda:0"))
        assert torch.equal(z[:no], z_ref[torch.as_tensor(own, device="cuda:0")])


@pytest.mark.parametrize("p", [1, 3])
def test_macro_range_entry_points_bitwise(p):
    """mhdg_residual_range / mhdg_matvec_range over a split of the macros
    (any order of the pieces, matvec stages split) equal the whole-range
    residual / matvec bit for bit: the partitioned operator's overlap of the
    halo exchange with the interior macros relies on it."""
    from paper_2507_22195_b200 import _native as N

    full, parts, discs, ex, w, tr, x, FieldSet, StageContext, torch = _setup(2, p=p)
    E = full.mesh.n_macros
    alpha = 150.0
    off = -alpha * full.volume_quad_states(FieldSet(w, tr))
    stage = StageContext(alpha=alpha, offset=off)
    res = full.residuals(FieldSet(w, tr), stage)
    lin = full.jacobian(FieldSet(w, tr), stage, ptc_weight=1.0)
    xd = torch.as_tensor(x, device="cuda:0")
    y = lin.matvec(xd)
    lib, ctx = full._lib, full._ctx
    wd, td = full._fields(FieldSet(w, tr))
    od = full._dev(off)
    r_w, r_tr = torch.empty_like(wd), torch.empty_like(td)
    cuts = [(E // 3, 2 * E // 3), (0, E // 3), (2 * E // 3, E)]
    for i, (a, b) in enumerate(cuts):
        rc = lib.mhdg_residual_range(ctx, N.ptr(wd), N.ptr(td), None, 1, alpha, N.ptr(od), 1,
                                     N.ptr(r_w), N.ptr(r_tr), None, a, b, int(i == 0), N.stream_handle())
        assert rc == 0
    y2 = torch.empty_like(xd)
    buf = C.byref(lin._buf)
    (a0, b0), (a1, b1), (a2, b2) = cuts
    assert lib.mhdg_matvec_range(ctx, buf, N.ptr(xd), N.ptr(y2), a0, b0, 1, 1, N.stream_handle()) == 0
    assert lib.mhdg_matvec_range(ctx, buf, N.ptr(xd), N.ptr(y2), a1, b1, 3, 0, N.stream_handle()) == 0
    assert lib.mhdg_matvec_range(ctx, buf, N.ptr(xd), N.ptr(y2), a2, b2, 3, 0, N.stream_handle()) == 0
    assert lib.mhdg_matvec_range(ctx, buf, N.ptr(xd), N.ptr(y2), a0, b0, 2, 0, N.stream_handle()) == 0
    torch.cuda.synchronize()
    assert torch.equal(r_w, res.r_w) and torch.equal(r_tr, res.r_trace)
    assert torch.equal(y2, y)


def test_macro_range_entry_points_bitwise_viscous():
    """As above for a viscous context (KEPES, config-4 parameters): the range
    residual returns r_w / r_trace / r_q and the range matvec the viscous
    condensed operator, bit for bit against the whole-range calls."""
    import torch

    from paper_2507_22195_b200 import (Discretization, DissipationSpec, GasModel, StageContext,
                                       ViscousParams)
    from paper_2507_22195_b200 import _native as N
    from paper_2507_22195_b200.assembly import FieldSet
    from paper_2507_22195_b200.mesh import build_box_macro_mesh

    gas = GasModel(1.4)
    mesh = build_box_macro_mesh(np.array([[0.0, 1.0]] * 3), (3, 2, 2), 1)
    disc = Discretization(mesh, p=3, gas=gas, flux=DissipationSpec("kepes"),
                          viscosity=ViscousParams(16000.0, 0.1, 0.71, 1.0), device="cuda:0")
    t = disc.tables
    rng = np.random.default_rng(5)
    E, nc, F, nt = mesh.n_macros, t.layout.n_unique, t.n_faces, t.n_trace

    def st(n):
        return gas.entropy_vars(gas.conservative(rng.uniform(0.9, 1.1, n),
                                                 rng.uniform(-0.5, 0.5, (n, 3)),
                                                 rng.uniform(0.9, 1.1, n)))

    f = FieldSet(st(E * nc).reshape(E, nc, 5), st(F * nt).reshape(F, nt, 5))
    f.q = disc.solve_gradient(f)
    alpha = 150.0
    off = -alpha * disc.volume_quad_states(f)
    stage = StageContext(alpha=alpha, offset=off)
    res = disc.residuals(f, stage)
    lin = disc.jacobian(f, stage, ptc_weight=1.0)
    xd = torch.as_tensor(rng.standard_normal((F, nt, 5)), device="cuda:0")
    y = lin.matvec(xd)
    lib, ctx = disc._lib, disc._ctx
    wd, td = disc._fields(f)
    qd, od = disc._q(f), disc._dev(off)
    r_w, r_tr, r_q = torch.empty_like(wd), torch.empty_like(td), torch.empty_like(qd)
    cuts = [(E // 3, 2 * E // 3), (0, E // 3), (2 * E // 3, E)]
    for i, (a, b) in enumerate(cuts):
        assert lib.mhdg_residual_range(ctx, N.ptr(wd), N.ptr(td), N.ptr(qd), 1, alpha, N.ptr(od), 1,
                                       N.ptr(r_w), N.ptr(r_tr), N.ptr(r_q), a, b, int(i == 0),
                                       N.stream_handle()) == 0
    y2 = torch.empty_like(xd)
    buf = C.byref(lin._buf)
    (a0, b0), (a1, b1), (a2, b2) = cuts
    assert lib.mhdg_matvec_range(ctx, buf, N.ptr(xd), N.ptr(y2), a0, b0, 1, 1, N.stream_handle()) == 0
    assert lib.mhdg_matvec_range(ctx, buf, N.ptr(xd), N.ptr(y2), a1, b1, 3, 0, N.stream_handle()) == 0
    assert lib.mhdg_matvec_range(ctx, buf, N.ptr(xd), N.ptr(y2), a2, b2, 3, 0, N.stream_handle()) == 0
    assert lib.mhdg_matvec_range(ctx, buf, N.ptr(xd), N.ptr(y2), a0, b0, 2, 0, N.stream_handle()) == 0
    torch.cuda.synchronize()
    assert torch.equal(r_w, res.r_w) and torch.equal(r_tr, res.r_trace) and torch.equal(r_q, res.r_q)
    assert torch.equal(y2, y)
