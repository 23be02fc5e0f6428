"""Macro-element partitioning and trace-halo exchange.

Rank g owns a contiguous macro range (cells are x-major, so ranges are x
slabs).  A skeleton face belongs to the rank of its owner macro (the lower
macro index, mesh.py:265-279).  Each rank stores the trace of every face
touching its macros: owned faces first, then ghost faces (owned elsewhere,
touched by a local macro), both in ascending global face order and in the
owner's node order, so a face's trace block has the same bytes on every rank.

Exchanges (both sides enumerate the shared faces in ascending global order):
  reduce_partials : ghost-face partial sums -> owner, added to the owner's
                    own side (0 + a + b, bit-identical to the single-device
                    atomic sum because IEEE addition is commutative)
  fill_ghosts     : owned-face values -> ghost copies (matvec input)
  gather_sides    : a side's face tensors -> the face owner (preconditioner
                    blocks of halo faces, once per Jacobian build)
Transport: `TorchDistExchange` (torch.distributed batched isend/irecv; NCCL
on GPUs, gloo on CPU) or `LoopbackExchange` (several partitions in one
process, used to check the partitioned kernels on a single GPU).
"""

from __future__ import annotations

from dataclasses import dataclass, field
from types import SimpleNamespace

import numpy as np


def macro_ranges(E, world):
    bounds = [round(g * E / world) for g in range(world + 1)]
    return [(bounds[g], bounds[g + 1]) for g in range(world)]


@dataclass
class HaloPlan:
    """Per-neighbour lists of local face ids (ascending global face id)."""

    owned_shared: dict = field(default_factory=dict)   # rank -> local ids of my faces it touches
    ghost: dict = field(default_factory=dict)          # rank -> local ids of its faces I touch


class LocalPartition:
    """Local view of the global tables for one rank."""

    def __init__(self, tables, rank, world):
        self.rank, self.world = rank, world
        t = tables
        mesh = t.mesh
        E = mesh.n_macros
        ranges = macro_ranges(E, world)
        self.ranges = ranges
        lo, hi = ranges[rank]
        self.macro_lo, self.macro_hi = lo, hi
        owner_rank = np.searchsorted(np.array([r[1] for r in ranges]), np.arange(E), side="right")
        self.rank_of_macro = owner_rank
        skel = mesh.skel
        own = skel.owner
        nb = skel.neighbor
        own_r = owner_rank[own]
        nb_r = np.where(nb >= 0, owner_rank[np.maximum(nb, 0)], -1)
        owned = np.nonzero(own_r == rank)[0]
        ghost = np.nonzero((own_r != rank) & (nb_r == rank))[0]
        self.global_faces = np.concatenate([owned, ghost])
        self.n_owned = len(owned)
        self.n_local_faces = len(self.global_faces)
        g2l = np.full(len(skel), -1, dtype=np.int64)
        g2l[self.global_faces] = np.arange(self.n_local_faces)
        self.g2l = g2l
        plan = HaloPlan()
        for h in range(world):
            if h == rank:
                continue
            mine = owned[nb_r[owned] == h]
            theirs = ghost[own_r[ghost] == h]
            if len(mine):
                plan.owned_shared[h] = g2l[mine]
            if len(theirs):
                plan.ghost[h] = g2l[theirs]
        self.plan = plan
        self.tables = self._local_tables(t, lo, hi, g2l, nb_r, own_r)
        self.interior = self._interior_range()

    def _interior_range(self):
        """Contiguous local macro range [i0, i1) touching no halo face (a
        face shared with another rank).  Those macros read only owned trace
        values and write only faces no neighbour contributes to, so their
        kernels can run while the halo exchange is in flight; the halo
        macros [0, i0) and [i1, E_l) run after it.  With x-slab partitions
        the halo macros are the first and last cell planes of the slab."""
        halo_face = np.zeros(self.n_local_faces, dtype=bool)
        halo_face[self.n_owned:] = True
        for ids in self.plan.owned_shared.values():
            halo_face[ids] = True
        halo_macro = halo_face[self.tables.face_id_st].any(axis=1)
        # longest run of non-halo macros (the few non-halo tets of the slab's
        # boundary cell planes simply run with the halo macros)
        best, start = (0, 0), None
        for e, h in enumerate(np.append(halo_macro, True)):
            if not h and start is None:
                start = e
            elif h and start is not None:
                if e - start > best[1] - best[0]:
                    best = (start, e)
                start = None
        return best

    def halo_ranges(self):
        E_l = self.macro_hi - self.macro_lo
        i0, i1 = self.interior
        if i1 <= i0:
            return [(0, E_l)]
        return [r for r in ((0, i0), (i1, E_l)) if r[1] > r[0]]

    def _local_tables(self, t, lo, hi, g2l, nb_r, own_r):
        """HDGTables-shaped namespace restricted to this rank."""
        sl = slice(lo, hi)
        E_l = hi - lo
        lt = SimpleNamespace()
        for name in ("p", "d", "n_s", "basis", "layout", "n_st", "st_face", "st_sub",
                     "st_subface", "st_face_scatter", "phi_face", "face_rows", "fphi",
                     "facet_wts", "phi", "dphi", "quad_wts", "domain_volume", "n_trace"):
            setattr(lt, name, getattr(t, name))
        lt.sub_det = t.sub_det[sl]
        lt.sub_inv_jac = t.sub_inv_jac[sl]
        lt.sub_jac = t.sub_jac[sl]
        lt.face_normals = t.face_normals[sl]
        lt.face_area = t.face_area[sl]
        lt.trace_idx = t.trace_idx[sl]
        lt.boundary_st = t.boundary_st[sl]
        lt.side_st = t.side_st[sl]
        lt.face_id_st = g2l[t.face_id_st[sl]]
        assert (lt.face_id_st >= 0).all()
        lt.n_faces = self.n_local_faces
        lt.viscous_reference = t.viscous_reference
        lt.vol_w = lt.quad_wts[None, None, :] * lt.sub_det[:, :, None]
        lt.dphi_phys = np.einsum("qik,eska->esqia", lt.dphi, lt.sub_inv_jac)
        lt.face_w = lt.facet_wts[None, None, :] * lt.face_area[:, :, None]
        lt.mesh = SimpleNamespace(n_macros=E_l, dim=t.mesh.dim, m=t.mesh.m)
        # coordinates of the local nodes / trace nodes / quadrature points
        # (projection and error norms on one rank)
        mesh = t.mesh
        lt.node_coords = (np.einsum("eab,nb->ena", mesh.macro_jacobians[sl], t.layout.unique_nodes)
                          + mesh.macro_origins[sl][:, None, :])
        lt.trace_coords = t.trace_coords[self.global_faces]
        sub_v = mesh.sub_vertices[sl]
        lt.quad_coords = (np.einsum("esab,qb->esqa", lt.sub_jac, t.basis.quad_pts)
                          + sub_v[:, :, 0, :][:, :, None, :])
        # preconditioner sides of owned faces: local (e*n_st + k) or a remote
        # side encoded as -2 - (index into the gathered remote-side list)
        fs = t.face_sides[self.global_faces[: self.n_owned]].copy()
        remote_rows = []
        for col in range(2):
            st = fs[:, col]
            has = st >= 0
            e = np.where(has, st // t.n_st, 0)
            k = np.where(has, st % t.n_st, 0)
            local = has & (e >= self.macro_lo) & (e < self.macro_hi)
            remote = has & ~local
            fs[local, col] = (e[local] - self.macro_lo) * t.n_st + k[local]
            idx = np.nonzero(remote)[0]
            fs[remote, col] = -2 - (len(remote_rows) + np.arange(len(idx)))
            remote_rows.extend(idx.tolist())
        lt.face_sides = fs
        self.n_remote_sides = len(remote_rows)
        # remote sides of owned halo faces: static geometry from the global
        # tables; hh tensors arrive from the neighbour (gather_sides)
        rows = np.array(remote_rows, dtype=np.int64)
        gf = self.global_faces[rows] if len(rows) else rows
        skel = t.mesh.skel
        tile_of = np.empty(t.d + 1, dtype=np.int64)
        tile_of[t.st_face] = np.arange(t.n_st)
        rem_e = skel.neighbor[gf] if len(rows) else rows
        rem_k = tile_of[skel.neighbor_face[gf]] if len(rows) else rows
        self.remote_side_ids = rem_e * t.n_st + rem_k      # global (macro, tile) of each remote side
        self.remote_tidx = np.ascontiguousarray(t.trace_idx[rem_e, rem_k], dtype=np.int32)
        self.remote_area = np.ascontiguousarray(t.face_area[rem_e, rem_k])
        remote_of_row = {int(r): i for i, r in enumerate(remote_rows)}
        self.recv_remote_idx = {h: np.array([remote_of_row[int(f)] for f in ids], dtype=np.int64)
                                for h, ids in self.plan.owned_shared.items()}
        # sides I must send: for ghost faces owned by h, my (neighbour) side
        self.send_sides = {}
        for h, ids in self.plan.ghost.items():
            gfs = self.global_faces[ids]
            e = skel.neighbor[gfs]
            k = tile_of[skel.neighbor_face[gfs]]
            self.send_sides[h] = (e - self.macro_lo) * t.n_st + k
        return lt

    # -- host helpers --------------------------------------------------------
    def local_fields(self, w, trace):
        """Slice global numpy fields into the local layout."""
        return w[self.macro_lo:self.macro_hi], trace[self.global_faces]

    def owned_mask(self):
        m = np.zeros(self.n_local_faces, dtype=bool)
        m[: self.n_owned] = True
        return m


class TorchDistExchange:
    """Halo transport over torch.distributed (NCCL on GPU, gloo on CPU).

    With the gloo backend, device tensors are staged through host memory
    (gloo has no device transport); this is what lets several ranks share
    one GPU in tests without their kernels waiting on each other."""

    def __init__(self, part, group=None):
        import torch.distributed as dist

        self.part = part
        self.group = group
        self.host_staged = dist.is_initialized() and dist.get_backend(group) == "gloo"

    def _exchange(self, sends, recvs):
        self._finish(self._start(sends, recvs))

    def _start(self, sends, recvs):
        """Issue the batched point-to-point exchange.  NCCL: the transfers
        run on NCCL's stream after the work already queued on the current
        stream; nothing blocks until _finish."""
        import torch.distributed as dist

        if self.host_staged:
            return (None, sends, recvs, True)
        ops = []
        for h, buf in sends.items():
            ops.append(dist.P2POp(dist.isend, buf.contiguous(), h, self.group))
        for h, buf in recvs.items():
            ops.append(dist.P2POp(dist.irecv, buf, h, self.group))
        reqs = dist.batch_isend_irecv(ops) if ops and dist.is_initialized() else []
        return (reqs, sends, recvs, False)

    def _finish(self, handle):
        """Make the current stream wait for the exchange (host-staged gloo
        transfers run here, synchronously)."""
        reqs, sends, recvs, staged = handle
        if staged:
            self._exchange_staged(sends, recvs)
            return
        for req in reqs:
            req.wait()

    def _exchange_staged(self, sends, recvs):
        import torch.distributed as dist

        if self.host_staged:
            dev_recvs = recvs
            sends = {h: b.cpu() for h, b in sends.items()}
            recvs = {h: b.new_empty(b.shape, device="cpu") for h, b in recvs.items()}
        ops = []
        for h, buf in sends.items():
            ops.append(dist.P2POp(dist.isend, buf.contiguous(), h, self.group))
        for h, buf in recvs.items():
            ops.append(dist.P2POp(dist.irecv, buf, h, self.group))
        if ops and dist.is_initialized():
            for req in dist.batch_isend_irecv(ops):
                req.wait()
        if self.host_staged:
            for h, b in recvs.items():
                dev_recvs[h].copy_(b)

    def reduce_partials(self, trace_like):
        """owner += neighbour partials on shared faces; returns trace_like."""
        return self.reduce_partials_finish(self.reduce_partials_start(trace_like))

    def reduce_partials_start(self, trace_like):
        """Send the ghost-face partial sums (snapshot taken now, on the
        current stream); the owner's add happens in reduce_partials_finish."""
        import torch

        plan = self.part.plan
        sends = {h: trace_like[torch.as_tensor(ids, device=trace_like.device)]
                 for h, ids in plan.ghost.items()}
        recvs = {h: torch.empty((len(ids),) + tuple(trace_like.shape[1:]), dtype=trace_like.dtype,
                                device=trace_like.device) for h, ids in plan.owned_shared.items()}
        return (trace_like, recvs, self._start(sends, recvs))

    def reduce_partials_finish(self, handle):
        import torch

        trace_like, recvs, h_ex = handle
        self._finish(h_ex)
        for h, ids in self.part.plan.owned_shared.items():
            idx = torch.as_tensor(ids, device=trace_like.device)
            trace_like[idx] = trace_like[idx] + recvs[h]
        return trace_like

    def fill_ghosts(self, trace_like):
        return self.fill_ghosts_finish(self.fill_ghosts_start(trace_like))

    def fill_ghosts_start(self, trace_like):
        """Send owned values of shared faces (snapshot taken now); the ghost
        rows are written in fill_ghosts_finish."""
        import torch

        plan = self.part.plan
        sends = {h: trace_like[torch.as_tensor(ids, device=trace_like.device)]
                 for h, ids in plan.owned_shared.items()}
        recvs = {h: torch.empty((len(ids),) + tuple(trace_like.shape[1:]), dtype=trace_like.dtype,
                                device=trace_like.device) for h, ids in plan.ghost.items()}
        return (trace_like, recvs, self._start(sends, recvs))

    def fill_ghosts_finish(self, handle):
        import torch

        trace_like, recvs, h_ex = handle
        self._finish(h_ex)
        for h, ids in self.part.plan.ghost.items():
            trace_like[torch.as_tensor(ids, device=trace_like.device)] = recvs[h]
        return trace_like

    def agree(self, code):
        """Global maximum of an integer status code over the ranks (one tiny
        all-reduce).  Every rank calls it at the same point, so a failure
        detected on one rank is raised on all of them before the next halo
        exchange or all-reduce (otherwise the ranks' collective sequences
        diverge and NCCL hangs)."""
        import torch
        import torch.distributed as dist

        if not dist.is_initialized() or dist.get_world_size(self.group) == 1:
            return int(code)
        dev = "cpu" if self.host_staged else torch.device("cuda", torch.cuda.current_device())
        t = torch.tensor([int(code)], dtype=torch.int32, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX, group=self.group)
        return int(t.item())

    def allreduce_sum(self, t):
        import torch.distributed as dist

        if not dist.is_initialized():      # single rank
            return t
        if self.host_staged and t.is_cuda:
            h = t.cpu()
            dist.all_reduce(h, op=dist.ReduceOp.SUM, group=self.group)
            t.copy_(h)
            return t
        dist.all_reduce(t, op=dist.ReduceOp.SUM, group=self.group)
        return t

    def gather_sides(self, hh_local, nqf):
        """hh tensors of the remote sides of my owned halo faces."""
        import torch

        part = self.part
        dev = hh_local.device
        blocks = hh_local.view(-1, nqf * 25)
        sends = {h: blocks[torch.as_tensor(st, device=dev)] for h, st in part.send_sides.items()}
        recvs = {h: torch.empty((len(idx), nqf * 25), dtype=torch.float64, device=dev)
                 for h, idx in part.recv_remote_idx.items()}
        self._exchange(sends, recvs)
        out = torch.empty((part.n_remote_sides, nqf * 25), dtype=torch.float64, device=dev)
        for h, idx in part.recv_remote_idx.items():
            out[torch.as_tensor(idx, device=dev)] = recvs[h]
        return out


class LoopbackExchange:
    """All partitions in one process: exchanges are direct copies.  Used to
    run the partitioned device kernels on a single GPU against the
    single-partition result."""

    def __init__(self, parts):
        self.parts = parts

    def agree(self, code):
        return int(code)

    def reduce_partials(self, traces):
        import torch

        recv = {}
        for g, p in enumerate(self.parts):
            for h, ids in p.plan.ghost.items():
                recv[(h, g)] = traces[g][torch.as_tensor(ids, device=traces[g].device)].clone()
        for (h, g), buf in recv.items():
            ids = self.parts[h].plan.owned_shared[g]
            idx = torch.as_tensor(ids, device=traces[h].device)
            traces[h][idx] = traces[h][idx] + buf.to(traces[h].device)
        return traces

    def gather_sides(self, hh_locals, nqf):
        """Remote-side hh tensors for every partition (list in, list out)."""
        import torch

        outs = []
        for g, p in enumerate(self.parts):
            out = torch.empty((p.n_remote_sides, nqf * 25), dtype=torch.float64,
                              device=hh_locals[g].device)
            for h, idx in p.recv_remote_idx.items():
                src = hh_locals[h].view(-1, nqf * 25)[torch.as_tensor(
                    self.parts[h].send_sides[g], device=hh_locals[h].device)]
                out[torch.as_tensor(idx, device=out.device)] = src.to(out.device)
            outs.append(out)
        return outs

    def fill_ghosts(self, traces):
        import torch

        for g, p in enumerate(self.parts):
            for h, ids in p.plan.owned_shared.items():
                vals = traces[g][torch.as_tensor(ids, device=traces[g].device)]
                dst = self.parts[h].plan.ghost[g]
                traces[h][torch.as_tensor(dst, device=traces[h].device)] = vals.to(traces[h].device)
        return traces
