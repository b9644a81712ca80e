"""Multi-rank host logic on CPU (gloo, world_size 2 and 3): halo plans,
ghost exchange with libdg's send/recv lists, local face tables, and the
partitioned operator = single-domain operator (CPU oracle as the checker)."""

import os
import socket

import numpy as np
import pytest

from casebuild import build


def _plans(name, P):
    from paper_2408_08129_b200.distributed import halo_plans
    return halo_plans(build(name).mesh, P)


@pytest.mark.parametrize("name,P", [("cfg1", 2), ("hang2d", 3), ("hang3d", 2), ("per3d", 3),
                                    ("cfg2", 4)])
def test_plans_cover_neighbours(name, P):
    from paper_2408_08129_b200.device import face_tables, localize
    c = build(name)
    plans = _plans(name, P)
    kind, nbr, hang, ffU, ffp, ffh = face_tables(c.mesh, c.bcs, c.model, c.geom.basis)
    owned = np.concatenate([np.arange(*pl.owned) for pl in plans])
    assert np.array_equal(owned, np.arange(c.mesh.n_leaves))
    for pl in plans:
        ids = pl.local_ids
        assert len(np.unique(ids)) == len(ids)
        # raises if an owned element's neighbour (or fine child) is not local
        localize(kind, nbr, hang, ffU, ffp, ffh, ids, pl.n_owned, c.mesh.n_leaves)
        assert int(pl.recv_counts.sum()) == len(pl.ghosts)
        assert pl.recv_counts[pl.rank] == 0 and pl.send_counts[pl.rank] == 0
    # what p sends to q is exactly what q expects, in q's order
    for p in plans:
        for q in plans:
            s0 = int(np.sum(p.send_counts[:q.rank]))
            sent = p.send_elems[s0:s0 + p.send_counts[q.rank]] + p.owned[0]
            r0 = int(np.sum(q.recv_counts[:p.rank]))
            assert np.array_equal(sent, q.ghosts[r0:r0 + q.recv_counts[p.rank]])


@pytest.mark.parametrize("name,P", [("hang2d", 3), ("hang3d", 2), ("per3d", 2)])
def test_host_exchange_and_partitioned_operator(name, P):
    """Ghost rows filled by the plan reproduce the global state, and the
    explicit residual evaluated per rank on [owned + ghosts] (non-local rows
    poisoned with NaN) equals the single-domain one on the owned rows."""
    from oracle import dg_oracle as O
    from paper_2408_08129_b200.distributed import exchange_host
    c = build(name)
    plans = _plans(name, P)
    loc = []
    for pl in plans:
        a = np.full((len(pl.local_ids),) + c.U.shape[1:], np.nan)
        a[:pl.n_owned] = c.U[pl.owned[0]:pl.owned[1]]
        loc.append(a)
    loc = exchange_host(plans, loc)
    ops = O.Operators(c.geom, c.model, c.bcs, c.sponge)
    R_ref = ops.explicit_residual(c.U)
    for pl, a in zip(plans, loc):
        assert np.array_equal(a, c.U[pl.local_ids])
        G = np.full_like(c.U, np.nan)
        G[pl.local_ids] = a
        with np.errstate(invalid="ignore"):
            R = ops.explicit_residual(G)
        own = slice(pl.owned[0], pl.owned[1])
        assert np.all(np.isfinite(R[own]))
        assert np.array_equal(R[own], R_ref[own])


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, name, q):
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import dg_oracle as O
        from paper_2408_08129_b200.distributed import halo_plans
        c = build(name)
        plans = halo_plans(c.mesh, world)
        pl = plans[rank]
        a = np.full((len(pl.local_ids),) + c.U.shape[1:], np.nan)
        a[:pl.n_owned] = c.U[pl.owned[0]:pl.owned[1]]
        # grouped send/recv with libdg's lists (the NCCL exchange, over gloo)
        reqs, bufs = [], {}
        s_off = np.concatenate([[0], np.cumsum(pl.send_counts)])
        r_off = np.concatenate([[0], np.cumsum(pl.recv_counts)])
        for p in range(world):
            if p == rank:
                continue
            if pl.send_counts[p]:
                t = torch.from_numpy(np.ascontiguousarray(a[pl.send_elems[s_off[p]:s_off[p + 1]]]))
                reqs.append(dist.isend(t, p))
            if pl.recv_counts[p]:
                bufs[p] = torch.empty((int(pl.recv_counts[p]),) + c.U.shape[1:], dtype=torch.float64)
                reqs.append(dist.irecv(bufs[p], p))
        for r in reqs:
            r.wait()
        for p, t in bufs.items():
            a[pl.n_owned + r_off[p]:pl.n_owned + r_off[p + 1]] = t.numpy()
        ok_ghost = bool(np.array_equal(a, c.U[pl.local_ids]))
        ops = O.Operators(c.geom, c.model, c.bcs, c.sponge)
        G = np.full_like(c.U, np.nan)
        G[pl.local_ids] = a
        with np.errstate(invalid="ignore"):
            R = ops.explicit_residual(G)[pl.owned[0]:pl.owned[1]]
        R_ref = ops.explicit_residual(c.U)[pl.owned[0]:pl.owned[1]]
        ok_op = bool(np.array_equal(R, R_ref))
        # Krylov-style global dot: allreduce of owned partial sums
        part = torch.tensor([float(np.sum(c.U[pl.owned[0]:pl.owned[1], -1] ** 2))],
                            dtype=torch.float64)
        dist.all_reduce(part)
        ok_dot = abs(float(part) - float(np.sum(c.U[:, -1] ** 2))) <= 1e-12 * float(part)
        q.put((rank, ok_ghost, ok_op, ok_dot))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("name,world", [("hang2d", 2), ("hang3d", 3)])
def test_gloo_multirank_halo(name, world):
    import multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, name, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    assert all(p.exitcode == 0 for p in procs)
    for rank, ok_ghost, ok_op, ok_dot in res:
        assert ok_ghost and ok_op and ok_dot, (rank, ok_ghost, ok_op, ok_dot)


@pytest.mark.parametrize("name,P", [("hang2d", 3), ("hang3d", 2), ("hang3d", 3), ("per3d", 3),
                                    ("cfg2", 4)])
def test_face_row_plans(name, P):
    """Face-row halo plans: what q sends to p is what p
    expects, every value an owned face reads from a ghost arrives (x face
    nodes, psi rows, the coarse parents' V trace slots), nothing else is
    touched, and the volume is a fraction of the whole-element exchange."""
    from paper_2408_08129_b200.device import face_tables
    from paper_2408_08129_b200.distributed import (ROW_PSI, ROW_TRV, ROW_X, exchange_rows_host,
                                                   face_nodes, face_row_plans, trace_slots)
    from paper_2408_08129_b200 import _lib as L
    c = build(name)
    d, n = c.mesh.dim, c.geom.basis.degree + 1
    NP, NC = n ** d, n ** (d - 1)
    widths = {ROW_X: NP, ROW_PSI: 2 * d * NC, ROW_TRV: (2 * (d - 1) + 2 * d) * NC}
    plans = _plans(name, P)
    rows = face_row_plans(c.mesh, plans, c.geom.basis.degree)
    for which, w in widths.items():
        for p in range(P):
            for q in range(P):
                assert rows[p][which].send_counts[q] == rows[q][which].recv_counts[p]
        rng = np.random.default_rng(which)
        G = rng.standard_normal((c.mesh.n_leaves, w))
        loc = []
        for pl in plans:
            a = np.full((len(pl.local_ids), w), np.nan)
            a[:pl.n_owned] = G[pl.owned[0]:pl.owned[1]]
            loc.append(a.ravel())
        out = exchange_rows_host(rows, which, loc)
        for pl, a in zip(plans, out):
            a = a.reshape(-1, w)
            got = np.isfinite(a[pl.n_owned:])
            # everything that arrived is the owner's value
            assert np.array_equal(a[pl.n_owned:][got], G[pl.ghosts][got])
    # coverage: every (ghost, face) an owned face reads
    kind, nbr, hang, *_ = face_tables(c.mesh, c.bcs, c.model, c.geom.basis)
    fn = face_nodes(d, n)
    for pl, rp in zip(plans, rows):
        g2l = {int(g): i for i, g in enumerate(pl.local_ids)}
        have = {w: set(rp[w].recv_idx.tolist()) for w in widths}
        for e in range(*pl.owned):
            for f in range(2 * d):
                k = int(kind[e, f]) & 15
                if k == L.FACE_CONF or k == L.FACE_FINE:
                    nbs = [int(nbr[e, f])]
                elif k == L.FACE_COARSE:
                    nbs = [int(v) for v in hang[int(nbr[e, f])]]
                else:
                    continue
                for g in nbs:
                    lid = g2l[g]
                    if lid < pl.n_owned:
                        continue
                    fo = f ^ 1
                    assert all(lid * NP + int(v) in have[ROW_X] for v in fn[fo])
                    assert all(lid * widths[ROW_PSI] + fo * NC + j in have[ROW_PSI]
                               for j in range(NC))
                    if k == L.FACE_FINE:
                        for sl in trace_slots(d, fo):
                            assert all(lid * widths[ROW_TRV] + sl * NC + j in have[ROW_TRV]
                                       for j in range(NC))
    # volume per Helmholtz apply vs whole ghost elements (x + psi + V traces)
    lean = sum(int(rp[w].send_counts.sum()) for rp in rows for w in widths)
    whole = sum(int(pl.send_counts.sum()) for pl in plans) * sum(widths.values())
    assert lean < 0.5 * whole, (lean, whole)


def _row_worker(rank, world, port, name, q):
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2408_08129_b200.distributed import ROW_PSI, face_row_plans, halo_plans
        c = build(name)
        d, n = c.mesh.dim, c.geom.basis.degree + 1
        w = 2 * d * n ** (d - 1)
        plans = halo_plans(c.mesh, world)
        rp = face_row_plans(c.mesh, plans, c.geom.basis.degree)[rank][ROW_PSI]
        pl = plans[rank]
        G = np.random.default_rng(3).standard_normal((c.mesh.n_leaves, w))
        a = np.full((len(pl.local_ids), w), np.nan)
        a[:pl.n_owned] = G[pl.owned[0]:pl.owned[1]]
        flat = a.ravel()
        # Comm::exchange_rows over gloo: pack by index, grouped send/recv, unpack
        s_off = np.concatenate([[0], np.cumsum(rp.send_counts)])
        r_off = np.concatenate([[0], np.cumsum(rp.recv_counts)])
        reqs, bufs = [], {}
        for p in range(world):
            if p == rank:
                continue
            if rp.send_counts[p]:
                t = torch.from_numpy(np.ascontiguousarray(flat[rp.send_idx[s_off[p]:s_off[p + 1]]]))
                reqs.append(dist.isend(t, p))
            if rp.recv_counts[p]:
                bufs[p] = torch.empty(int(rp.recv_counts[p]), dtype=torch.float64)
                reqs.append(dist.irecv(bufs[p], p))
        for r in reqs:
            r.wait()
        for p, t in bufs.items():
            flat[rp.recv_idx[r_off[p]:r_off[p + 1]]] = t.numpy()
        got = flat.reshape(-1, w)[pl.n_owned:]
        fin = np.isfinite(got)
        ok = bool(np.array_equal(got[fin], G[pl.ghosts][fin])) and int(fin.sum()) == int(rp.recv_counts.sum())
        q.put((rank, ok, int(fin.sum()), got.size))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("name,world", [("hang3d", 2), ("hang2d", 3)])
def test_gloo_face_row_exchange(name, world):
    """The face-row exchange (Comm::exchange_rows: pack by index, grouped
    send / recv per peer, unpack by index) between real processes over gloo:
    every received value is the owner's, and only the planned values move."""
    import multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_row_worker, args=(r, world, port, name, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    assert all(p.exitcode == 0 for p in procs)
    for rank, ok, moved, total in res:
        assert ok and 0 < moved < total, (rank, ok, moved, total)
