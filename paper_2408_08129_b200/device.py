"""Device context: element-centric tables from the reference's face batches.

The reference stores its topology as face BATCHES (conforming per axis,
hanging per (axis, orient) grouped by coarse face, boundary per (axis,
side); orodg/mesh.py:38-89, 178-242) and scatters lifts back to elements
(orodg/dgops.py:131-229).  The B200 kernels are owner-computes instead: every
element evaluates its own 2d faces, so the batches are turned once into
per-element face records

    kind[e, 2*axis+side]  WALL | FARFIELD | CONF | FINE (+subface<<4) | COARSE
    nbr [e, 2*axis+side]  neighbour element / boundary row / hanging group

plus the hanging-group table of fine children.  Metric ownership is kept
exactly as in the reference: conforming faces use the minus (left) side's
face metric, hanging faces the fine side's, boundary faces the outward one.
"""

import ctypes as C

import numpy as np

from . import _lib as L
from .boundary import BoundaryCondition
from .errors import ConfigurationError, UsageError
from .physics import conserved_to_primitive


def basis_tables(basis):
    """Flat 1D tables in the device Tab<N> layout (dg_common.cuh)."""
    if not basis.square:
        raise UsageError("device kernels need n_quad_1d == degree + 1 "
                         "(the factorised B^-1 mass inverse, SURVEY.md §7)")
    parts = [basis.interp_1d, basis.Binv, basis.Dhat, basis.lift,
             np.stack(basis.half_interp_1d), np.stack(basis.half_q),
             basis.quad_w, basis.quad_x, 1.0 / basis.quad_w]
    return np.ascontiguousarray(np.concatenate([np.asarray(p, dtype=np.float64).ravel()
                                                for p in parts]))


def face_tables(mesh, bcs, model, basis):
    """Global element-centric face records (see module docstring)."""
    d = mesh.dim
    n = mesh.n_leaves
    S = 2 ** (d - 1)
    topo = mesh.topology
    kind = np.full((n, 2 * d), 255, dtype=np.uint8)
    nbr = np.full((n, 2 * d), -1, dtype=np.int64)
    for bt in topo.conforming:
        a = bt.axis
        kind[bt.left, 2 * a + 1] = L.FACE_CONF
        nbr[bt.left, 2 * a + 1] = bt.right
        kind[bt.right, 2 * a] = L.FACE_CONF
        nbr[bt.right, 2 * a] = bt.left
    groups = []
    g0 = 0
    for bt in topo.hanging:
        a, o = bt.axis, bt.orient
        ng = len(bt.coarse) // S
        coarse = bt.coarse[::S]
        kind[coarse, 2 * a + o] = L.FACE_COARSE
        nbr[coarse, 2 * a + o] = g0 + np.arange(ng)
        ch = np.empty((ng, S), dtype=np.int64)
        sub = bt.subface.reshape(ng, S)
        fine = bt.fine.reshape(ng, S)
        np.put_along_axis(ch, sub, fine, axis=1)
        groups.append(ch)
        fs = 1 - o
        kind[bt.fine, 2 * a + fs] = (L.FACE_FINE | (bt.subface << 4)).astype(np.uint8)
        nbr[bt.fine, 2 * a + fs] = bt.coarse
        g0 += ng
    hang = np.concatenate(groups) if groups else np.zeros((0, S), dtype=np.int64)
    if bcs is None:
        bcs = [BoundaryCondition("wall") for _ in topo.boundary]
    if len(bcs) != len(topo.boundary):
        raise UsageError(f"{len(bcs)} boundary conditions for {len(topo.boundary)} "
                         "boundary batches")
    nqf = basis.n_face_quad
    V = d + 2
    rows = sum(len(bt.leaves) for bt in topo.boundary)
    ffU = np.zeros((rows, V, nqf))
    ffp = np.zeros((rows, nqf))
    ffh = np.zeros((rows, nqf))
    r0 = 0
    for bt, bc in zip(topo.boundary, bcs):
        nb = len(bt.leaves)
        a, s = bt.axis, bt.side
        if bc.kind == "wall":
            kind[bt.leaves, 2 * a + s] = L.FACE_WALL
        else:
            g = np.asarray(bc.ghost_conserved, dtype=np.float64)
            if g.shape != (nb, V, nqf):
                raise UsageError(f"far-field traces have shape {g.shape}, "
                                 f"expected {(nb, V, nqf)}")
            kind[bt.leaves, 2 * a + s] = L.FACE_FARFIELD
            ffU[r0:r0 + nb] = g
            W = conserved_to_primitive(g, model, var_axis=1, check=False)
            ffp[r0:r0 + nb] = W.p                          # boundary.py:55-65
            ffh[r0:r0 + nb] = W.e + W.p / W.rho            # boundary.py:66-84
        nbr[bt.leaves, 2 * a + s] = r0 + np.arange(nb)
        r0 += nb
    if np.any(kind == 255):
        e, f = np.argwhere(kind == 255)[0]
        raise UsageError(f"face {f} of element {e} has no topology record")
    return kind, nbr, hang, ffU, ffp, ffh


def localize(kind, nbr, hang, ffU, ffp, ffh, local_ids, n_owned, n_glob):
    """Face records of one rank's [owned..., ghosts...] elements in local
    numbering (host-only; unit-tested on CPU).  Raises UsageError when an
    owned element's face neighbour is missing from the local set."""
    local_ids = np.asarray(local_ids, dtype=np.int64)
    n_tot = len(local_ids)
    d2 = kind.shape[1]
    g2l = np.full(n_glob, -1, dtype=np.int64)
    g2l[local_ids] = np.arange(n_tot)
    kl = kind[local_ids].copy()
    nl = nbr[local_ids].copy()
    k4 = kl & 15
    inter = (k4 == L.FACE_CONF) | (k4 == L.FACE_FINE)
    nl[inter] = g2l[nl[inter]]
    coarse = k4 == L.FACE_COARSE
    gids = np.unique(nl[coarse]) if np.any(coarse) else np.zeros(0, np.int64)
    hmap = np.full(max(len(hang), 1), -1, dtype=np.int64)
    hmap[gids] = np.arange(len(gids))
    S = hang.shape[1] if hang.ndim == 2 else 1
    hang_l = g2l[hang[gids]] if len(gids) else np.zeros((0, S), np.int64)
    nl[coarse] = hmap[nl[coarse]]
    bnd = (k4 == L.FACE_WALL) | (k4 == L.FACE_FARFIELD)
    rows = np.unique(nl[bnd]) if np.any(bnd) else np.zeros(0, np.int64)
    rmap = np.full(max(len(ffU), 1), -1, dtype=np.int64)
    rmap[rows] = np.arange(len(rows))
    nl[bnd] = rmap[nl[bnd]]
    if np.any(nl[:n_owned] < 0):
        e, f = np.argwhere(nl[:n_owned] < 0)[0]
        raise UsageError(f"halo plan misses face {f} neighbour of owned element {e}")
    coarse_owned = np.any(coarse[:n_owned], axis=1)
    used_groups = np.unique(nl[:n_owned][coarse[:n_owned]])
    if len(used_groups) and np.any(hang_l[used_groups] < 0):
        raise UsageError("halo plan misses a fine child of an owned coarse face")
    del coarse_owned, d2
    return (kl, nl, hang_l, ffU[rows] if len(rows) else np.zeros((0,) + ffU.shape[1:]),
            ffp[rows] if len(rows) else np.zeros((0,) + ffp.shape[1:]),
            ffh[rows] if len(rows) else np.zeros((0,) + ffh.shape[1:]))


class DeviceContext:
    """Owns one dg_ctx (one GPU, one element range) and its host tables.

    local_ids: global element ids of [owned..., ghosts...] for a rank of a
    partitioned run (paper_2408_08129_b200.distributed); None = all
    elements, one rank.
    """

    def __init__(self, geometry, model, bcs=None, sponge=None, device=None,
                 local_ids=None, n_owned=None):
        import torch
        if not torch.cuda.is_available():
            raise L.DeviceError("no CUDA device visible: the device path has no CPU fallback")
        self.lib = L.lib()
        self.geometry = geometry
        self.model = model
        mesh = geometry.mesh
        b = geometry.basis
        d = mesh.dim
        self.dim = d
        self.degree = b.degree
        self.np_ = b.n_nodes
        self.V = d + 2
        self.device = torch.cuda.current_device() if device is None else int(device)
        kind, nbr, hang, ffU, ffp, ffh = face_tables(mesh, bcs, model, b)
        elem, col, col_stride = geometry.device_tables()
        n_glob = mesh.n_leaves
        if local_ids is None:
            local_ids = np.arange(n_glob, dtype=np.int64)
            n_owned = n_glob
        local_ids = np.asarray(local_ids, dtype=np.int64)
        self.local_ids = local_ids
        self.n_el = int(n_owned)
        self.n_tot = len(local_ids)
        own = local_ids[:self.n_el]
        kl, nl, hang_l, fU, fp, fh = localize(kind, nbr, hang, ffU, ffp, ffh, local_ids,
                                              self.n_el, n_glob)
        rows = np.arange(len(fU))
        self._host = dict(
            elem=np.ascontiguousarray(elem[local_ids]),
            col=np.ascontiguousarray(col) if col_stride else np.zeros(1),
            nbr=np.ascontiguousarray(nl.astype(np.int32)),
            kind=np.ascontiguousarray(kl),
            hang=np.ascontiguousarray(hang_l.astype(np.int32)) if len(hang_l) else np.zeros((1, 1), np.int32),
            ffU=np.ascontiguousarray(fU) if len(rows) else np.zeros(1),
            ffp=np.ascontiguousarray(fp) if len(rows) else np.zeros(1),
            ffh=np.ascontiguousarray(fh) if len(rows) else np.zeros(1),
            tabs=basis_tables(b))
        self.has_sponge = sponge is not None
        if sponge is not None:
            sigma, bg = sponge
            self._host["sigma"] = np.ascontiguousarray(np.asarray(sigma, dtype=np.float64)[own])
            self._host["bg"] = np.ascontiguousarray(np.asarray(bg, dtype=np.float64)[own])
        h = self._host
        ptr = lambda a: a.ctypes.data_as(C.c_void_p)  # noqa: E731
        desc = L.CtxDesc()
        desc.dim = d
        desc.degree = b.degree
        desc.n_el = self.n_el
        desc.n_tot = self.n_tot
        per_root = [e / c for e, c in zip(mesh.extents, mesh.root_counts)] + [0.0] * (3 - d)
        desc.per_root = (C.c_double * 3)(*per_root)
        desc.z_top = geometry.z_top
        desc.terrain = 1 if col_stride else 0
        desc.n_col = col.shape[0] if col_stride else 0
        desc.col_stride = col_stride
        desc.elem = ptr(h["elem"])
        desc.col = ptr(h["col"])
        desc.nbr = ptr(h["nbr"])
        desc.kind = ptr(h["kind"])
        desc.hang_children = ptr(h["hang"])
        desc.n_hang_groups = len(hang_l)
        desc.n_bface = len(rows)
        desc.ff_U = ptr(h["ffU"])
        desc.ff_p = ptr(h["ffp"])
        desc.ff_h = ptr(h["ffh"])
        desc.sigma = ptr(h["sigma"]) if sponge is not None else None
        desc.background = ptr(h["bg"]) if sponge is not None else None
        desc.gamma = model.gamma
        desc.gravity = model.gravity
        desc.inv_mach_sq = model.inv_mach_sq
        desc.kinetic_factor = model.kinetic_factor
        desc.tabs = ptr(h["tabs"])
        desc.tabs_len = len(h["tabs"])
        desc.device = self.device
        handle = C.c_void_p()
        with torch.cuda.device(self.device):
            L.check(self.lib.dg_ctx_create(C.byref(desc), C.byref(handle)))
        self.handle = handle
        self._stream = None
        self._host = None  # tables now live on the device
        self.torch = torch

    # -------------------------------------------------------------- helpers
    def bind_stream(self):
        """Run on torch's current stream of this device."""
        s = self.torch.cuda.current_stream(self.device).cuda_stream
        if s != self._stream:
            L.check(self.lib.dg_ctx_set_stream(self.handle, C.c_void_p(s)))
            self._stream = s
        return self.handle

    def empty(self, *shape, rows=None):
        n = self.n_tot if rows is None else rows
        return self.torch.empty((n,) + tuple(shape), dtype=self.torch.float64,
                                device=f"cuda:{self.device}")

    def zeros(self, *shape, rows=None):
        n = self.n_tot if rows is None else rows
        return self.torch.zeros((n,) + tuple(shape), dtype=self.torch.float64,
                                device=f"cuda:{self.device}")

    def launch_info(self):
        g, t, s = C.c_int(), C.c_int(), C.c_longlong()
        L.check(self.lib.dg_ctx_launch_info(self.handle, C.byref(g), C.byref(t), C.byref(s)))
        return g.value, t.value, s.value

    def close(self):
        if getattr(self, "handle", None):
            self.lib.dg_ctx_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def as_ptr(t):
    return C.c_void_p(t.data_ptr()) if t is not None else None
