"""Element-block domain decomposition over GPUs (one process per GPU).

The partition is the reference's Morton-contiguous split (orodg/partition.py,
``partition_leaves``); each rank owns one contiguous leaf range and keeps
ghost COPIES of the face neighbours it reads.  Local element
numbering is [owned..., ghosts...] with ghosts ordered by (owner rank,
global id), so the ghosts received from one peer form one contiguous block.
Collectives (libdg, NCCL over NVLink/NVSwitch): a grouped send/recv halo
exchange before every face-coupled kernel and allreduces of the Krylov,
fixed-point and diagnostic scalars.  Nothing else crosses GPUs.
"""

from dataclasses import dataclass

import numpy as np

from .partition import neighbor_pairs, partition_leaves


@dataclass
class HaloPlan:
    rank: int
    nranks: int
    owned: tuple                # (start, stop) global leaf range
    ghosts: np.ndarray          # global ids, ordered by (owner, id)
    recv_counts: np.ndarray     # ghosts received from each peer
    send_counts: np.ndarray     # owned leaves sent to each peer
    send_elems: np.ndarray      # LOCAL ids of the sent leaves, grouped by peer

    @property
    def local_ids(self):
        a, b = self.owned
        return np.concatenate([np.arange(a, b, dtype=np.int64), self.ghosts])

    @property
    def n_owned(self):
        return self.owned[1] - self.owned[0]


def halo_plans(mesh, nranks, weights=None, part=None):
    """Plans for every rank (deterministic; each rank can build all of them)."""
    part = part or partition_leaves(mesh, nranks, weights)
    owner = part.owner
    pairs = neighbor_pairs(mesh)
    plans = []
    ghost_sets = []
    for p in range(nranks):
        g = part.ghosts[p] if len(pairs) else np.empty(0, np.int64)
        g = np.asarray(g, dtype=np.int64)
        g = g[np.lexsort((g, owner[g]))] if len(g) else g
        ghost_sets.append(g)
    for p in range(nranks):
        a, b = part.ranges[p]
        recv = np.array([np.sum(owner[ghost_sets[p]] == q) for q in range(nranks)], dtype=np.int64)
        send_lists = []
        for q in range(nranks):
            gq = ghost_sets[q]
            mine = gq[owner[gq] == p] if len(gq) else gq
            send_lists.append(np.sort(mine) - a)     # global -> local (owned block)
        send_counts = np.array([len(s) for s in send_lists], dtype=np.int64)
        send_elems = (np.concatenate(send_lists) if send_lists else np.empty(0, np.int64))
        plans.append(HaloPlan(rank=p, nranks=nranks, owned=(a, b), ghosts=ghost_sets[p],
                              recv_counts=recv, send_counts=send_counts,
                              send_elems=send_elems.astype(np.int64)))
    return plans


@dataclass
class RowPlan:
    """One rank's face-row exchange lists for one field layout: offsets (in
    doubles, into the local [owned..., ghosts...] field) of the values sent
    to / received from each peer, grouped by peer."""
    send_counts: np.ndarray
    send_idx: np.ndarray
    recv_counts: np.ndarray
    recv_idx: np.ndarray


ROW_X, ROW_PSI, ROW_TRV = 0, 1, 2


def face_nodes(dim, n):
    """Nodal indices (C order, axis 0 slowest) of the n^(d-1) nodes on face
    2*axis+side, ascending."""
    idx = np.arange(n ** dim).reshape((n,) * dim)
    out = []
    for a in range(dim):
        for side in (0, 1):
            out.append(np.sort(np.take(idx, (n - 1) if side else 0, axis=a).ravel()))
    return np.stack(out)


def trace_slots(dim, face):
    """V-trace slots of a face (dg_operator.cuh tr_slot): vertical faces carry
    the normal component only, z faces all d components."""
    nv = 2 * (dim - 1)
    if face < nv:
        return [face]
    return [nv + (face - nv) * dim + k for k in range(dim)]


def face_row_plans(mesh, plans, degree):
    """Face-row halo plans of the flux-trace Helmholtz pair:
    for every rank and field layout (x nodal, psi, V traces) the values its
    owned elements' faces read from ghosts, nothing else.

    An owned element reads, across face f, its ghost neighbour's face f^1:
    the nodal face values of x (H1 and the coarse-face kernel), its psi row
    (H2 through hk_pin_fixup, the coarse-face kernel for ghost children) and,
    when the ghost is the coarse parent of an owned fine element, its V trace
    slots there (the fine side's mortar).  Returns plans[rank][which]."""
    d = mesh.dim
    n = degree + 1
    NP, NC = n ** d, n ** (d - 1)
    TRL = (2 * (d - 1) + 2 * d) * NC
    nranks = len(plans)
    topo = mesh.topology
    owner = np.empty(mesh.n_leaves, dtype=np.int64)
    for pl in plans:
        owner[pl.owned[0]:pl.owned[1]] = pl.rank
    rk, el, fc, tv = [], [], [], []

    def need(by, elem, face, trv):
        m = owner[by] != owner[elem]
        rk.append(owner[by][m])
        el.append(np.asarray(elem)[m])
        fc.append(np.full(int(m.sum()), face, dtype=np.int64))
        tv.append(np.full(int(m.sum()), trv, dtype=np.int64))
    for bt in topo.conforming:
        a = bt.axis
        need(bt.right, bt.left, 2 * a + 1, 0)
        need(bt.left, bt.right, 2 * a, 0)
    for bt in topo.hanging:
        a, o = bt.axis, bt.orient
        need(bt.fine, bt.coarse, 2 * a + o, 1)          # fine owner reads the coarse parent
        need(bt.coarse, bt.fine, 2 * a + 1 - o, 0)      # coarse owner reads the children
    if rk:
        rk, el, fc, tv = (np.concatenate(v) for v in (rk, el, fc, tv))
    else:
        rk = el = fc = tv = np.empty(0, np.int64)
    # unique (rank, element, face); trv = any
    key = (rk * mesh.n_leaves + el) * (2 * d) + fc
    order = np.argsort(key, kind="stable")
    key, rk, el, fc, tv = key[order], rk[order], el[order], fc[order], tv[order]
    first = np.ones(len(key), dtype=bool)
    first[1:] = key[1:] != key[:-1]
    grp = np.cumsum(first) - 1
    tvu = np.zeros(int(first.sum()), dtype=np.int64)
    np.maximum.at(tvu, grp, tv)
    rk, el, fc, tv = rk[first], el[first], fc[first], tvu
    fn = face_nodes(d, n)
    ar = np.arange(NC, dtype=np.int64)

    def offsets(which, lid, face, trv):
        """(values per need, flat offsets) of the needs in the given order."""
        if which == ROW_X:
            return (lid[:, None] * NP + fn[face]).ravel()
        if which == ROW_PSI:
            return (lid[:, None] * (2 * d * NC) + face[:, None] * NC + ar).ravel()
        rows = []
        sel = np.nonzero(trv)[0]          # (only the coarse parents of hanging faces)
        for l, f in zip(lid[sel], face[sel]):
            for sl in trace_slots(d, int(f)):
                rows.append(l * TRL + sl * NC + ar)
        return np.concatenate(rows) if rows else np.empty(0, np.int64)

    out = []
    for pl in plans:
        p = pl.rank
        g2l = np.full(mesh.n_leaves, -1, dtype=np.int64)
        g2l[pl.local_ids] = np.arange(len(pl.local_ids))
        per_which = []
        for which in (ROW_X, ROW_PSI, ROW_TRV):
            sc = np.zeros(nranks, dtype=np.int64)
            rc = np.zeros(nranks, dtype=np.int64)
            sidx, ridx = [], []
            for q in range(nranks):
                if q == p:
                    continue
                # received from q: my needs of q's elements, (element, face) order
                m = (rk == p) & (owner[el] == q)
                o = offsets(which, g2l[el[m]], fc[m], tv[m])
                rc[q] = len(o)
                ridx.append(o)
                # sent to q: q's needs of my elements, same order
                m = (rk == q) & (owner[el] == p)
                o = offsets(which, el[m] - pl.owned[0], fc[m], tv[m])
                sc[q] = len(o)
                sidx.append(o)
            cat = lambda v: (np.concatenate(v) if v else np.empty(0, np.int64)).astype(np.int64)  # noqa: E731
            per_which.append(RowPlan(sc, cat(sidx), rc, cat(ridx)))
        out.append(per_which)
    return out


def attach_row_plans(ctx, row_plans):
    """Hand one rank's three face-row plans to its libdg context."""
    import ctypes as C

    from . import _lib as L
    for which, rp in enumerate(row_plans):
        arrs = [np.ascontiguousarray(a, dtype=np.int64)
                for a in (rp.send_counts, rp.send_idx, rp.recv_counts, rp.recv_idx)]
        arrs = [a if len(a) else np.zeros(1, np.int64) for a in arrs]
        L.check(ctx.lib.dg_ctx_set_halo_rows(ctx.handle, which,
                                             *[a.ctypes.data_as(C.c_void_p) for a in arrs]))


def exchange_rows_host(row_plans, which, local_flat):
    """Host execution of one face-row exchange for all ranks (test oracle of
    Comm::exchange_rows): local_flat[p] is rank p's flattened field."""
    out = [a.copy() for a in local_flat]
    nranks = len(row_plans)
    for p in range(nranks):
        rp = row_plans[p][which]
        r0 = 0
        for q in range(nranks):
            n = int(rp.recv_counts[q])
            if n == 0:
                continue
            sq = row_plans[q][which]
            s0 = int(np.sum(sq.send_counts[:p]))
            out[p][rp.recv_idx[r0:r0 + n]] = local_flat[q][sq.send_idx[s0:s0 + n]]
            r0 += n
    return out


def exchange_host(plans, local_arrays):
    """Reference (host) execution of one halo exchange for all ranks:
    local_arrays[p] has rows [owned..., ghosts...]; ghost rows are filled
    from their owners using exactly the send/recv lists libdg uses."""
    out = [a.copy() for a in local_arrays]
    for p, pl in enumerate(plans):
        off = 0
        for q in range(pl.nranks):
            n = int(pl.recv_counts[q])
            if n == 0:
                continue
            plq = plans[q]
            s0 = int(np.sum(plq.send_counts[:p]))
            rows = plq.send_elems[s0:s0 + n]
            out[p][pl.n_owned + off:pl.n_owned + off + n] = local_arrays[q][rows]
            off += n
    return out


class DistributedSolver:
    """One rank of a partitioned ARS(2,2,2) run on its GPU (bench.py N>1)."""

    def __init__(self, case, cfg, rank, world, local_rank):
        import ctypes as C

        import torch
        import torch.distributed as dist

        from . import _lib as L
        from .device import DeviceContext

        if not dist.is_initialized():
            dist.init_process_group("gloo")
        self.plan = halo_plans(case.mesh, world)[rank]
        pl = self.plan
        ids = pl.local_ids
        sponge = case.sponge
        self.ctx = DeviceContext(case.geometry, case.model, case.bcs, sponge,
                                 device=local_rank, local_ids=ids, n_owned=pl.n_owned)
        uid = (C.c_char * 128)()
        if rank == 0:
            L.check(self.ctx.lib.dg_nccl_unique_id(uid))
        obj = [bytes(uid) if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        uid = (C.c_char * 128).from_buffer_copy(obj[0])
        sc = np.ascontiguousarray(pl.send_counts.astype(np.int32))
        se = np.ascontiguousarray(pl.send_elems.astype(np.int32))
        rc = np.ascontiguousarray(pl.recv_counts.astype(np.int32))
        L.check(self.ctx.lib.dg_ctx_set_comm(self.ctx.handle, uid, rank, world,
                                            sc.ctypes.data_as(C.c_void_p),
                                            se.ctypes.data_as(C.c_void_p),
                                            rc.ctypes.data_as(C.c_void_p)))
        all_plans = halo_plans(case.mesh, world)
        attach_row_plans(self.ctx, face_row_plans(case.mesh, all_plans,
                                                  case.geometry.basis.degree)[rank])
        self.case = case
        self.cfg = cfg
        self.n_owned = pl.n_owned
        self.torch = torch

    def local_state(self):
        U = self.case.U0[self.plan.local_ids]
        return self.torch.from_numpy(np.ascontiguousarray(U)).to(f"cuda:{self.ctx.device}")

    def step(self, U, t):
        import ctypes as C

        from . import _lib as L
        from .device import as_ptr
        from .imex import StepStats, _step_error_info
        out = self.torch.empty_like(U)
        cs = L.StepStatsC()
        code = self.ctx.lib.dg_imex_step(self.ctx.bind_stream(), as_ptr(U), as_ptr(out), float(t),
                                         float(self.case.dt), C.byref(self.cfg.c()), C.byref(cs))
        st = StepStats()
        st.absorb(cs)
        L.check(code, stats=st, **_step_error_info(cs))
        return out, st


class LoopbackGroup:
    """P ranks of a partitioned run inside ONE process (one host thread and
    one CUDA stream per rank, all contexts on one device): the same halo
    plans, exchanges and allreduces as the NCCL path, through libdg's
    loopback backend (dg_ctx_set_comm_loopback).  It executes the multi-rank
    code path -- ghost exchanges inside every operator, the partitioned
    GMRES reductions, the distributed positivity and mass-rate reductions --
    on a box with one GPU.  No kernel waits on another rank: the ranks meet
    only in host barriers between stream-ordered copies."""

    _next_group = [1]

    def __init__(self, geometry, model, bcs, sponge, nranks, device=0, lean=True):
        import ctypes as C

        import torch

        from . import _lib as L
        from .device import DeviceContext
        self.torch = torch
        self.L = L
        self.C = C
        self.plans = halo_plans(geometry.mesh, nranks)
        self.nranks = nranks
        self.device = device
        self.ctxs = [DeviceContext(geometry, model, bcs, sponge, device=device,
                                   local_ids=pl.local_ids, n_owned=pl.n_owned)
                     for pl in self.plans]
        gid = LoopbackGroup._next_group[0]
        LoopbackGroup._next_group[0] += 1

        def attach(rank, ctx):
            pl = self.plans[rank]
            sc = np.ascontiguousarray(pl.send_counts.astype(np.int32))
            se = np.ascontiguousarray(pl.send_elems.astype(np.int32))
            rc = np.ascontiguousarray(pl.recv_counts.astype(np.int32))
            L.check(ctx.lib.dg_ctx_set_comm_loopback(
                ctx.handle, gid, rank, nranks, sc.ctypes.data_as(C.c_void_p),
                se.ctypes.data_as(C.c_void_p), rc.ctypes.data_as(C.c_void_p)))
        self.run(attach)
        self.row_plans = face_row_plans(geometry.mesh, self.plans, geometry.basis.degree)
        if lean:
            self.run(lambda r, ctx: attach_row_plans(ctx, self.row_plans[r]))

    def halo_values(self, reset=False):
        """Doubles each rank has sent in halo exchanges (dg_halo_stats)."""
        out = []
        for ctx in self.ctxs:
            v = self.C.c_longlong()
            ctx.lib.dg_halo_stats(ctx.handle, self.C.byref(v), 1 if reset else 0)
            out.append(v.value)
        return out

    def run(self, fn, timeout=600.0):
        """fn(rank, ctx) on every rank concurrently (its own thread and
        stream); returns the per-rank results, re-raising the first error."""
        import threading
        torch = self.torch
        out = [None] * self.nranks
        err = [None] * self.nranks

        def body(r):
            try:
                torch.cuda.set_device(self.device)
                s = torch.cuda.Stream(device=self.device)
                with torch.cuda.stream(s):
                    ctx = self.ctxs[r]
                    ctx.bind_stream()
                    out[r] = fn(r, ctx)
                    s.synchronize()
            except BaseException as e:  # pragma: no cover - surfaced below
                err[r] = e
        th = [threading.Thread(target=body, args=(r,), daemon=True) for r in range(self.nranks)]
        for t in th:
            t.start()
        for t in th:
            t.join(timeout)
            if t.is_alive():
                raise RuntimeError("loopback rank did not finish (deadlock?)")
        for e in err:
            if e is not None:
                raise e
        return out

    def scatter(self, global_array):
        """Per-rank device copies of a global (n_el, ...) array: owned rows
        then ghost rows."""
        return [self.torch.from_numpy(np.ascontiguousarray(global_array[pl.local_ids]))
                .to(f"cuda:{self.device}") for pl in self.plans]

    def gather(self, local_arrays):
        """The owned rows of every rank, as one global host array."""
        return np.concatenate([a[:pl.n_owned].cpu().numpy()
                               for a, pl in zip(local_arrays, self.plans)], axis=0)

    def imex_step(self, U_local, t, dt, cfg):
        """dg_imex_step on every rank; returns (new local states, StepStats
        per rank)."""
        from .device import as_ptr
        from .imex import StepStats, _solve_cfg, _step_error_info
        L, C = self.L, self.C

        def step(r, ctx):
            U = U_local[r]
            out = self.torch.empty_like(U)
            cs = L.StepStatsC()
            ccfg = _solve_cfg(cfg, False)
            code = ctx.lib.dg_imex_step(ctx.handle, as_ptr(U), as_ptr(out), float(t), float(dt),
                                        C.byref(ccfg), C.byref(cs))
            st = StepStats()
            st.absorb(cs)
            L.check(code, stats=st, **_step_error_info(cs))
            return out, st
        res = self.run(step)
        return [r[0] for r in res], [r[1] for r in res]
