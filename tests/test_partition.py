"""Partitioned operator, host side: partition structure, and
world_size-2 gloo runs where each rank evaluates its macro range with the
CPU oracle and the halo exchange / all-reduce code of the product
(`partition.TorchDistExchange`, `distributed.DistVectors`, `solver.fgmres`)
assembles the global result."""

import os
import socket
from types import SimpleNamespace

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from helpers import CPUVectors
from paper_2507_22195_b200.mesh import build_box_macro_mesh
from paper_2507_22195_b200.partition import LocalPartition, TorchDistExchange
from paper_2507_22195_b200.tables import HDGTables


def small_tables(n=(4, 2, 2), p=2):
    return HDGTables(build_box_macro_mesh(np.array([[0.0, 1.0]] * 3), n, 1), p)


@pytest.mark.parametrize("world", [2, 3, 4])
def test_partition_structure(world):
    t = small_tables()
    parts = [LocalPartition(t, g, world) for g in range(world)]
    owned = np.concatenate([p.global_faces[: p.n_owned] for p in parts])
    assert np.array_equal(np.sort(owned), np.arange(t.n_faces))
    for g, pg in enumerate(parts):
        lt = pg.tables
        assert lt.mesh.n_macros == pg.macro_hi - pg.macro_lo
        assert (lt.face_id_st < pg.n_local_faces).all()
        # every local side's face is local, with the global id it had
        glob = t.face_id_st[pg.macro_lo:pg.macro_hi]
        assert np.array_equal(pg.global_faces[lt.face_id_st], glob)
        for h, ids in pg.plan.owned_shared.items():
            ph = parts[h]
            assert np.array_equal(pg.global_faces[ids], ph.global_faces[ph.plan.ghost[g]])
            assert len(pg.recv_remote_idx[h]) == len(ph.send_sides[g])
        assert sum(len(v) for v in pg.recv_remote_idx.values()) == pg.n_remote_sides


@pytest.mark.parametrize("world", [2, 4])
def test_interior_and_halo_macro_ranges(world):
    """Interior macros (run while the halo exchange is in flight) touch no
    face shared with another rank; interior + halo ranges tile the slab."""
    t = small_tables(n=(8, 2, 2))
    for g in range(world):
        pg = LocalPartition(t, g, world)
        E_l = pg.macro_hi - pg.macro_lo
        i0, i1 = pg.interior
        assert 0 < i0 < i1 < E_l, (i0, i1)
        shared = set(range(pg.n_owned, pg.n_local_faces))
        for ids in pg.plan.owned_shared.values():
            shared |= set(int(i) for i in ids)
        fid = pg.tables.face_id_st
        assert not any(int(f) in shared for f in fid[i0:i1].ravel())
        covered = sorted([(i0, i1)] + pg.halo_ranges())
        assert covered[0][0] == 0 and covered[-1][1] == E_l
        assert all(a[1] == b[0] for a, b in zip(covered, covered[1:]))
        # the interior is most of the slab (all but ~the boundary cell planes)
        assert i1 - i0 >= E_l - 2 * 6 * 2 * 2


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _states(gas, rng, n):
    return gas.entropy_vars(gas.conservative(rng.uniform(0.9, 1.1, n), rng.uniform(-0.5, 0.5, (n, 3)),
                                             rng.uniform(0.9, 1.1, n)))


def _worker(rank, world, port, flux, results):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle.hdg_oracle import Gas, OracleHDG, fgmres as ofgmres
        from paper_2507_22195_b200 import solver
        from paper_2507_22195_b200.distributed import DistVectors

        gas = Gas(1.4)
        t = small_tables()
        E, nc, F, nt = t.mesh.n_macros, t.layout.n_unique, t.n_faces, t.n_trace
        rng = np.random.default_rng(2024)
        w = _states(gas, rng, E * nc).reshape(E, nc, 5)
        tr = _states(gas, rng, F * nt).reshape(F, nt, 5)
        x = rng.standard_normal(tr.shape)
        full = OracleHDG(t, flux=flux)
        alpha = 150.0
        off = -alpha * full.volume_quad_states(w)
        rw_ref, rt_ref = full.residuals(w, tr, alpha, off)
        lin_ref = full.linearize(w, tr, alpha, 1.0, precond=False)
        y_ref = lin_ref.matvec(x)

        part = LocalPartition(t, rank, world)
        ex = TorchDistExchange(part)
        lo, hi = part.macro_lo, part.macro_hi
        op = OracleHDG(part.tables, flux=flux)
        wl, trl = part.local_fields(w, tr)
        rw, rt = op.residuals(wl, trl, alpha, off[lo:hi])
        rt_t = torch.from_numpy(rt.copy())
        ex.reduce_partials(rt_t)
        own = part.global_faces[: part.n_owned]
        ok_res = (np.array_equal(rw, rw_ref[lo:hi])
                  and np.array_equal(rt_t.numpy()[: part.n_owned], rt_ref[own]))
        # ghost fill of a matvec input, then the partitioned matvec
        xl = torch.from_numpy(x[part.global_faces].copy())
        xl[part.n_owned:] = 1e300
        ex.fill_ghosts(xl)
        ok_fill = np.array_equal(xl.numpy(), x[part.global_faces])
        lin = op.linearize(wl, trl, alpha, 1.0, precond=False)
        y = torch.from_numpy(lin.matvec(xl.numpy()))
        ex.reduce_partials(y)
        err_mv = float(np.abs(y.numpy()[: part.n_owned] - y_ref[own]).max() / np.abs(y_ref).max())

        # distributed FGMRES (product solver + DistVectors, CPU vector double)
        pdisc = SimpleNamespace(exchange=ex, local=SimpleNamespace(tables=part.tables), part=part,
                                device=torch.device("cpu"))
        vec = DistVectors(pdisc, inner=CPUVectors())
        shape = trl.shape

        def dop(v):
            v2 = v.view(shape).clone()
            ex.fill_ghosts(v2)
            out = torch.from_numpy(lin.matvec(v2.numpy()))
            ex.reduce_partials(out)
            return out.view(-1)

        b = torch.from_numpy(x[part.global_faces].copy()).view(-1)
        res = solver.fgmres(dop, b, rel_tol=1e-8, restart=15, max_iters=60,
                            raise_on_stagnation=False, vec=vec)
        xr, it_ref, _, _ = ofgmres(lin_ref.matvec_flat if hasattr(lin_ref, "matvec_flat")
                                   else (lambda v: lin_ref.matvec(v.reshape(tr.shape)).ravel()),
                                   x.ravel(), rel_tol=1e-8, restart=15, max_iters=60)
        xd = res.x.view(shape).numpy()[: part.n_owned]
        err_x = float(np.abs(xd - xr.reshape(tr.shape)[own]).max() / np.abs(xr).max())
        # opt-in CGS2 (3 all-reduces per Arnoldi step): same solution
        vec2 = DistVectors(pdisc, inner=CPUVectors(), orth="cgs2")
        res2 = solver.fgmres(dop, b, rel_tol=1e-8, restart=15, max_iters=60,
                             raise_on_stagnation=False, vec=vec2)
        xd2 = res2.x.view(shape).numpy()[: part.n_owned]
        err_cgs2 = (abs(res2.iterations - it_ref),
                    float(np.abs(xd2 - xr.reshape(tr.shape)[own]).max() / np.abs(xr).max()))
        # the inner sweep's Arnoldi exit on the distributed vectors: same
        # iterate as the literal loop with one matvec less, and A x from the
        # Arnoldi relation (what the outer column uses instead of a matvec)
        calls = [0]

        def dop_counted(v):
            calls[0] += 1
            return dop(v)

        lit = solver.fgmres(dop_counted, b, rel_tol=0.1, restart=20, max_iters=20,
                            raise_on_stagnation=False, vec=vec)
        n_lit, calls[0] = calls[0], 0
        fast = solver.fgmres(dop_counted, b, rel_tol=0.1, restart=20, max_iters=20,
                             raise_on_stagnation=False, vec=vec, final_residual="arnoldi")
        ax_true = dop(fast.x).view(shape).numpy()[: part.n_owned]
        ax_arn = fast.ax.view(shape).numpy()[: part.n_owned]
        scale = float(vec.norm(b))   # global norm: the same normalisation on every rank
        arnoldi = (fast.iterations == lit.iterations, bool(torch.equal(fast.x, lit.x)), n_lit - calls[0],
                   float(np.abs(ax_arn - ax_true).max()) / scale)
        # remote face sides for the face-block preconditioner: every rank
        # takes part, including one that owns no halo face
        nqf = t.fphi.shape[0]
        hh_glob = np.arange(E * 4 * nqf * 25, dtype=np.float64).reshape(E * 4, nqf * 25)
        hh_loc = torch.from_numpy(hh_glob[lo * 4:hi * 4].copy())
        got = ex.gather_sides(hh_loc, nqf).numpy()
        ok_sides = np.array_equal(got, hh_glob[part.remote_side_ids])
        results[rank] = (ok_res and ok_sides, ok_fill, err_mv, res.iterations, it_ref, err_x,
                         part.n_remote_sides, err_cgs2, arnoldi)
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(600)
@pytest.mark.parametrize("flux", ["es", "kepes"])
def test_gloo_world2_partitioned_operator_and_fgmres(flux):
    world = 2
    mgr = mp.Manager()
    results = mgr.dict()
    mp.start_processes(_worker, args=(world, _free_port(), flux, results), nprocs=world,
                       join=True, start_method="spawn")
    assert min(results[r][6] for r in range(world)) == 0, "one rank should own no halo face"
    for rank in range(world):
        ok_res, ok_fill, err_mv, it, it_ref, err_x, _, err_cgs2, arnoldi = results[rank]
        assert err_cgs2[0] <= 1 and err_cgs2[1] <= 1e-7, err_cgs2
        assert arnoldi[0] and arnoldi[1] and arnoldi[2] == 1 and arnoldi[3] <= 1e-12, arnoldi
        assert ok_res, "partitioned residual must be bit-identical"
        assert ok_fill
        assert err_mv <= 1e-14
        assert it == it_ref
        assert err_x <= 1e-10


def _agree_worker(rank, world, port, results):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2507_22195_b200.distributed import collective
        from paper_2507_22195_b200.errors import NonAdmissibleState, SingularLocalMatrix

        t = small_tables()
        ex = TorchDistExchange(LocalPartition(t, rank, world))
        out = []
        # 1. a non-admissible trial state on rank 1 only: both ranks raise
        #    NonAdmissibleState (rank 1 its own, with the location), and the
        #    exchange afterwards still pairs up (no hang)

        def trial():
            if rank == 1:
                raise NonAdmissibleState("non-admissible state at volume sub 0", where="volume sub 0")
            return "ok"

        try:
            collective(ex, trial, rank)
            out.append("no raise")
        except NonAdmissibleState as e:
            out.append(("nonadm", e.where))
        buf = torch.full((4,), float(rank))
        ex.allreduce_sum(buf)
        out.append(float(buf[0]))
        # 2. a singular local matrix on rank 0 and a non-admissible state on
        #    rank 1: the larger code (singular) wins everywhere
        def lin():
            if rank == 0:
                raise SingularLocalMatrix("singular condensed block on macro 3", macro=3)
            raise NonAdmissibleState("x", where="face tile 1")

        try:
            collective(ex, lin, rank)
        except SingularLocalMatrix as e:
            out.append(("singular", e.macro))
        except NonAdmissibleState:
            out.append("wrong class")
        # 3. no failure anywhere: the value passes through
        out.append(collective(ex, lambda: rank * 10, rank))
        results[rank] = out
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(300)
def test_gloo_world2_failure_is_collective():
    """a rank-local NonAdmissibleState / SingularLocalMatrix must
    be raised on every rank at the same point, so the Newton loop takes the
    tau/4 retry branch on all ranks and the halo sequence stays paired."""
    world = 2
    mgr = mp.Manager()
    results = mgr.dict()
    mp.start_processes(_agree_worker, args=(world, _free_port(), results), nprocs=world,
                       join=True, start_method="spawn")
    r0, r1 = results[0], results[1]
    assert r0[0] == ("nonadm", "remote rank") and r1[0] == ("nonadm", "volume sub 0")
    assert r0[1] == r1[1] == 1.0
    assert r0[2] == ("singular", 3) and r1[2] == ("singular", None)
    assert r0[3] == 0 and r1[3] == 10
