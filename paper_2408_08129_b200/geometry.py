"""Terrain-following metric terms: full host arrays and compact device tables.

Map and metric definitions follow the reference (orodg/geometry.py:1-24,
167-357): box elements lifted by the Gal-Chen rule
z = z_ref + h(x[,y]) (1 - z_ref/z_top), with h a per-root-column polynomial
interpolant of the height function at GLL nodes of the geometric degree.

B200 layout: the device never sees the dense per-quadrature
point arrays (det_j, ctrv, face normals; ~20 GB at 2.5 M hexes).  It gets

  * ``elem_i32``  (n_el, 2 + d) int32: level, integer origin[d], column id;
    sizes and lower corners are rebuilt on the device with the same
    arithmetic as geometry.py:195-197;
  * ``col_f64``   (n_col, stride) float64 per distinct horizontal leaf
    footprint ("column"): h and the physical grad h at the horizontal Gauss
    grid, and h on the vertical faces.  det J and the adjugate at every
    quadrature point, and every face normal / surface weight, are
    re-evaluated in registers from these with the formulas of
    geometry.py:204-238 and 305-357.

Flat meshes (no terrain) carry no column table at all.
"""

from dataclasses import dataclass

import numpy as np

from .basis import gauss_lobatto, lagrange_diff_matrix, lagrange_eval_matrix, make_basis
from .errors import ConfigurationError, GeometryError


class TerrainSurface:
    """Height function sampled at GLL nodes of each root column
    (orodg/geometry.py:35-62)."""

    def __init__(self, height_fn, extents, root_counts, degree):
        self.degree = int(degree)
        self.extents = tuple(extents)
        self.root_counts = tuple(root_counts)
        hd = len(root_counts) - 1
        self.hd = hd
        self.nodes = gauss_lobatto(self.degree + 1)
        self.col_dx = np.array([extents[a] / root_counts[a] for a in range(hd)])
        g = self.nodes
        if hd == 1:
            x = (np.arange(root_counts[0])[:, None] + g[None, :]) * self.col_dx[0]
            vals = height_fn(x)
        else:
            x = (np.arange(root_counts[0])[:, None, None, None]
                 + g[None, None, :, None]) * self.col_dx[0]
            y = (np.arange(root_counts[1])[None, :, None, None]
                 + g[None, None, None, :]) * self.col_dx[1]
            x, y = np.broadcast_arrays(x, y)
            vals = height_fn(x, y)
        self.values = np.asarray(vals, dtype=float)
        z_top = extents[-1]
        if np.any(self.values >= z_top):
            raise ConfigurationError(
                f"terrain height reaches z_top={z_top}: max {self.values.max()}")
        if np.any(self.values < 0):
            raise ConfigurationError("terrain height must be >= 0")


class _Columns:
    """Distinct horizontal leaf footprints and the surface polynomial
    evaluated on them."""

    def __init__(self, surface, mesh):
        hd = mesh.dim - 1
        self.hd = hd
        self.surface = surface
        key = np.concatenate([mesh.levels[:, None], mesh.origins[:, :hd]], axis=1)
        uniq, inv = np.unique(key, axis=0, return_inverse=True)
        self.col_of_elem = inv.ravel().astype(np.int64)
        self.levels = uniq[:, 0]
        self.origins = uniq[:, 1:]
        self.n = len(uniq)

    def eval(self, pts_per_axis, deriv=False):
        """h (n_col, n_pts) at the tensor grid of the given 1D reference point
        sets (C-order over horizontal axes); with deriv also the physical
        gradient (n_col, n_pts, hd)."""
        s = self.surface
        hd = self.hd
        lv = self.levels
        cols = [self.origins[:, a] >> lv for a in range(hd)]
        vals = s.values[cols[0]] if hd == 1 else s.values[cols[0], cols[1]]
        mats, dmats = [], []
        for a in range(hd):
            og = self.origins[:, a] - (cols[a] << lv)
            pts = np.asarray(pts_per_axis[a], dtype=float)
            keys, kinv = np.unique(np.stack([lv, og], 1), axis=0, return_inverse=True)
            L = np.empty((len(keys), len(pts), len(s.nodes)))
            Ld = np.empty_like(L)
            for i, (l, o) in enumerate(keys):
                local = (o + pts) * (1.0 / (1 << int(l)))
                L[i] = lagrange_eval_matrix(s.nodes, local)
                Ld[i] = lagrange_diff_matrix(s.nodes, local)
            mats.append(L[kinv.ravel()])
            dmats.append(Ld[kinv.ravel()])
        if hd == 1:
            h = np.einsum("cpj,cj->cp", mats[0], vals)
            if not deriv:
                return h
            dh = np.einsum("cpj,cj->cp", dmats[0], vals) / s.col_dx[0]
            return h, dh[..., None]
        h = np.einsum("cpj,cqk,cjk->cpq", mats[0], mats[1], vals)
        n = h.shape[0]
        if not deriv:
            return h.reshape(n, -1)
        dx = np.einsum("cpj,cqk,cjk->cpq", dmats[0], mats[1], vals) / s.col_dx[0]
        dy = np.einsum("cpj,cqk,cjk->cpq", mats[0], dmats[1], vals) / s.col_dx[1]
        return h.reshape(n, -1), np.stack([dx.reshape(n, -1), dy.reshape(n, -1)], -1)


@dataclass(frozen=True)
class FaceGeometry:
    normal: np.ndarray   # (n_faces, n_face_quad, d), minus -> plus (outward on boundary)
    ws: np.ndarray       # (n_faces, n_face_quad)


class MeshGeometry:
    """Metric terms of a (possibly terrain-mapped) forest mesh."""

    def __init__(self, mesh, basis, surface, geom_degree):
        self.mesh = mesh
        self.basis = basis
        self.surface = surface
        self.geom_degree = geom_degree
        self.dim = mesh.dim
        self.z_top = mesh.extents[-1]
        self.sizes = mesh.leaf_sizes()
        self.lo = self.sizes * mesh.origins.astype(float)
        self.terrain = surface is not None
        self._cols = _Columns(surface, mesh) if self.terrain else None
        self._memo = {}

    # ------------------------------------------------------------ mass inverse
    def apply_mass_inverse(self, dual, out=None, elements=slice(None)):
        """Nodal coefficients from a dual vector (geometry.py:372-396), on the
        device: the factorised inverse B^-1 diag(1/(w detJ)) B^-T per element
        (libdg dg_apply_mass_inverse).  dual: (n_sel, ..., n_nodes) for the
        selected elements; numpy in -> numpy out (or into ``out``), CUDA
        tensors stay on the device."""
        from .dgops import from_device, to_device
        from .physics import DIMENSIONAL
        from . import _lib as L
        from .device import DeviceContext, as_ptr
        ctx = self._memo.get("mass_ctx")
        if ctx is None:
            ctx = DeviceContext(self, DIMENSIONAL)
            self._memo["mass_ctx"] = ctx
        t, host = to_device(dual, ctx)
        shape = tuple(t.shape)
        nn = self.basis.n_nodes
        if shape[-1] != nn:
            from .errors import UsageError
            raise UsageError(f"dual has {shape[-1]} nodes per element, expected {nn}")
        full = isinstance(elements, slice) and elements == slice(None)
        n_el = self.mesh.n_leaves
        k = 1
        for s_ in shape[1:-1]:
            k *= s_
        if full:
            src = t.reshape(shape[0], k, nn).contiguous()
        else:
            # block-diagonal inverse: embed the selected elements, apply, take
            src = ctx.torch.zeros((n_el, k, nn), dtype=t.dtype, device=t.device)
            idx = ctx.torch.as_tensor(np.arange(n_el)[elements], device=t.device)
            src[idx] = t.reshape(shape[0], k, nn)
        res = ctx.empty(k, nn, rows=src.shape[0])
        L.check(ctx.lib.dg_apply_mass_inverse(ctx.bind_stream(), as_ptr(src), k, as_ptr(res)))
        if not full:
            res = res[idx]
        res = res.reshape(shape)
        if out is not None:
            if isinstance(out, np.ndarray):
                out[...] = res.cpu().numpy()
            else:
                out.copy_(res)
            return out
        return from_device(res, host)

    # ------------------------------------------------------------ column data
    def _colq(self):
        """h and grad h at the horizontal Gauss grid per column."""
        if "colq" not in self._memo:
            b = self.basis
            self._memo["colq"] = self._cols.eval([b.quad_x] * (self.dim - 1), deriv=True)
        return self._memo["colq"]

    def _col_edges(self):
        """h on the vertical faces per column: (n_col, hd, 2, n_q^(hd-1))."""
        if "coledge" not in self._memo:
            hd = self.dim - 1
            qx = self.basis.quad_x
            out = np.empty((self._cols.n, hd, 2, len(qx) ** (hd - 1)))
            for a in range(hd):
                for s in (0, 1):
                    sets = [qx] * hd
                    sets[a] = np.array([float(s)])
                    out[:, a, s, :] = self._cols.eval(sets)
            self._memo["coledge"] = out
        return self._memo["coledge"]

    def _elem_hq(self):
        nqh = self.basis.n_quad_1d ** (self.dim - 1)
        if not self.terrain:
            return (np.zeros((self.mesh.n_leaves, nqh)),
                    np.zeros((self.mesh.n_leaves, nqh, self.dim - 1)))
        hq, dhq = self._colq()
        c = self._cols.col_of_elem
        return hq[c], dhq[c]

    # ------------------------------------------------------- device tables
    def device_tables(self):
        """(elem_i32, col_f64, col_stride) for the C-ABI (include/dg.h)."""
        m = self.mesh
        d = self.dim
        ncol = self._cols.col_of_elem if self.terrain else np.zeros(m.n_leaves, np.int64)
        elem = np.concatenate([m.levels[:, None], m.origins, ncol[:, None]], axis=1)
        if np.any(elem > np.iinfo(np.int32).max):
            raise ConfigurationError("mesh too large for int32 element tables")
        elem = np.ascontiguousarray(elem.astype(np.int32))
        if not self.terrain:
            return elem, np.zeros((0, 0)), 0
        hq, dhq = self._colq()
        edges = self._col_edges()
        n = hq.shape[0]
        zt = self.z_top
        # the kernels need 1 - h/z_top (geometry.py:208, 341): stored here with
        # the reference's own arithmetic, so the device does no division
        col = np.concatenate([1.0 - hq / zt, np.moveaxis(dhq, 2, 1).reshape(n, -1),
                              (1.0 - edges / zt).reshape(n, -1)], axis=1)
        if col.shape[1] % 2:
            # even row length: every column row starts 16-byte aligned (the
            # pipelined Helmholtz kernels bring it in with one bulk copy)
            col = np.concatenate([col, np.zeros((n, 1))], axis=1)
        return elem, np.ascontiguousarray(col), col.shape[1]

    # ------------------------------------------------------- volume metric
    def _volume(self):
        if "vol" in self._memo:
            return self._memo["vol"]
        b = self.basis
        d = self.dim
        hd = d - 1
        zt = self.z_top
        nq1 = b.n_quad_1d
        hq, dhq = self._elem_hq()
        zb = self.lo[:, -1:] + self.sizes[:, -1:] * b.quad_x[None, :]
        decay = 1.0 - zb / zt
        zz = (self.sizes[:, -1][:, None] * (1.0 - hq / zt))[:, :, None] \
            * np.ones((1, 1, nq1))
        zgrad = (dhq[:, :, None, :] * self.sizes[:, None, None, :hd]
                 * decay[:, None, :, None])
        det = np.ones(zz.shape)
        for a in range(hd):
            det = det * self.sizes[:, a][:, None, None]
        det = det * zz
        n_el = self.mesh.n_leaves
        ctrv = np.zeros(zz.shape + (d, d))
        sx = self.sizes[:, 0][:, None, None]
        if d == 2:
            ctrv[..., 0, 0] = zz
            ctrv[..., 1, 0] = -zgrad[..., 0]
            ctrv[..., 1, 1] = sx
        else:
            sy = self.sizes[:, 1][:, None, None]
            ctrv[..., 0, 0] = sy * zz
            ctrv[..., 1, 1] = sx * zz
            ctrv[..., 2, 0] = -sy * zgrad[..., 0]
            ctrv[..., 2, 1] = -sx * zgrad[..., 1]
            ctrv[..., 2, 2] = sx * sy
        det = det.reshape(n_el, b.n_quad)
        if det.min() <= 0.0:
            bad = np.unravel_index(np.argmin(det), det.shape)
            raise GeometryError(f"non-positive Jacobian in element {bad[0]} "
                                f"(det={det[bad]:.3e})")
        self._memo["vol"] = (det, ctrv.reshape(n_el, b.n_quad, d, d))
        return self._memo["vol"]

    def validate(self):
        """Jacobian positivity check without materialising the dense arrays:
        det J = prod(size_h) * size_z * (1 - h/z_top) > 0."""
        if self.terrain:
            hq, _ = self._colq()
            if np.any(1.0 - hq / self.z_top <= 0.0):
                raise GeometryError("non-positive Jacobian (terrain reaches z_top)")
        return True

    @property
    def det_j(self):
        return self._volume()[0]

    @property
    def ctrv(self):
        return self._volume()[1]

    @property
    def mass_h_inv(self):
        if "mhi" not in self._memo:
            b = self.basis
            hd = self.dim - 1
            Bh, wh = b.interp_1d, b.quad_w
            for _ in range(hd - 1):
                Bh = np.kron(Bh, b.interp_1d)
                wh = np.kron(wh, b.quad_w)
            prof = self.det_j.reshape(self.mesh.n_leaves, -1, b.n_quad_1d)[:, :, 0]
            mh = np.einsum("qi,eq,qj->eij", Bh, wh[None, :] * prof, Bh)
            self._memo["mhi"] = np.linalg.inv(mh)
        return self._memo["mhi"]

    @property
    def mass_v_inv(self):
        b = self.basis
        return np.linalg.inv(b.interp_1d.T @ (b.quad_w[:, None] * b.interp_1d))

    # --------------------------------------------------------- node coords
    def _map_points(self, pts_h, pts_z):
        m = self.mesh
        hd = self.dim - 1
        zt = self.z_top
        n_el = m.n_leaves
        if self.terrain:
            hc = self._cols.eval([pts_h] * hd)
            h = hc[self._cols.col_of_elem]
        else:
            h = np.zeros((n_el, len(pts_h) ** hd))
        nph = h.shape[1]
        ch = [self.lo[:, a][:, None] + self.sizes[:, a][:, None] * pts_h[None, :]
              for a in range(hd)]
        zb = self.lo[:, -1][:, None] + self.sizes[:, -1][:, None] * pts_z[None, :]
        out = np.empty((n_el, nph, len(pts_z), self.dim))
        if hd == 1:
            out[..., 0] = ch[0][:, :, None]
        else:
            n0 = len(pts_h)
            xg = np.broadcast_to(ch[0][:, :, None], (n_el, n0, n0)).reshape(n_el, nph)
            yg = np.broadcast_to(ch[1][:, None, :], (n_el, n0, n0)).reshape(n_el, nph)
            out[..., 0] = xg[:, :, None]
            out[..., 1] = yg[:, :, None]
        out[..., -1] = zb[:, None, :] + h[:, :, None] * (1.0 - zb[:, None, :] / zt)
        return out.reshape(n_el, -1, self.dim)

    @property
    def node_coords(self):
        if "nc" not in self._memo:
            n = self.basis.nodes_1d
            self._memo["nc"] = self._map_points(n, n)
        return self._memo["nc"]

    @property
    def corners(self):
        c = np.array([0.0, 1.0])
        return self._map_points(c, c)

    @property
    def diameter(self):
        cr = self.corners
        diff = cr[:, :, None, :] - cr[:, None, :, :]
        return np.sqrt((diff ** 2).sum(-1)).max(axis=(1, 2))

    @property
    def min_diameter(self):
        return float(self.diameter.min())

    @property
    def n_elements(self):
        return self.mesh.n_leaves

    # --------------------------------------------------------- face metric
    def face_metric(self, elements, axis, side, outward=False):
        """Unit normal (+axis oriented, or outward) and quadrature weight x
        surface Jacobian on the (axis, side) faces of the given elements
        (orodg/geometry.py:305-357)."""
        b = self.basis
        d = self.dim
        hd = d - 1
        zt = self.z_top
        nq1 = b.n_quad_1d
        lo = self.lo[elements]
        sz = self.sizes[elements]
        nf = len(elements)
        if axis == d - 1:
            hq, dh = self._elem_hq()
            dh = dh[elements]
            decay = (1.0 - (lo[:, -1] + sz[:, -1] * float(side)) / zt)[:, None]
            nt = np.empty(dh.shape[:2] + (d,))
            if d == 2:
                nt[..., 0] = -dh[..., 0] * sz[:, 0][:, None] * decay
                nt[..., 1] = sz[:, 0][:, None]
            else:
                nt[..., 0] = -sz[:, 1][:, None] * dh[..., 0] * sz[:, 0][:, None] * decay
                nt[..., 1] = -sz[:, 0][:, None] * dh[..., 1] * sz[:, 1][:, None] * decay
                nt[..., 2] = (sz[:, 0] * sz[:, 1])[:, None]
        else:
            if self.terrain:
                he = self._col_edges()[self._cols.col_of_elem[elements], axis, side]
            else:
                he = np.zeros((nf, nq1 ** (hd - 1)))
            prof = 1.0 - he / zt
            zzv = sz[:, -1][:, None, None] * prof[:, :, None]
            nt = np.zeros((nf, he.shape[1], nq1, d))
            if d == 2:
                nt[..., 0] = zzv
            else:
                nt[..., axis] = sz[:, 1 - axis][:, None, None] * zzv
            nt = nt.reshape(nf, -1, d)
        if outward and side == 0:
            nt = -nt
        mag = np.sqrt((nt ** 2).sum(-1))
        return FaceGeometry(normal=nt / mag[..., None], ws=b.face_w[None, :] * mag)

    def _faces(self):
        if "faces" not in self._memo:
            topo = self.mesh.topology
            conf = [self.face_metric(bt.left, bt.axis, 1) for bt in topo.conforming]
            hang = [self.face_metric(bt.fine, bt.axis, 0 if bt.orient == 1 else 1)
                    for bt in topo.hanging]
            bdry = [self.face_metric(bt.leaves, bt.axis, bt.side, outward=True)
                    for bt in topo.boundary]
            self._memo["faces"] = (conf, hang, bdry)
        return self._memo["faces"]

    @property
    def conforming(self):
        return self._faces()[0]

    @property
    def hanging(self):
        return self._faces()[1]

    @property
    def boundary(self):
        return self._faces()[2]

    def total_volume(self):
        return float((self.basis.vol_w[None, :] * self.det_j).sum())


def build_geometry(mesh, solution_degree, terrain=None, geom_degree=None,
                   n_quad_1d=None, z_top=None):
    """Metric terms for a mesh (orodg/geometry.py:402-415)."""
    if z_top is not None and abs(z_top - mesh.extents[-1]) > 1e-9 * mesh.extents[-1]:
        raise ConfigurationError(
            f"z_top={z_top} must equal the vertical extent {mesh.extents[-1]}")
    if geom_degree is None:
        geom_degree = solution_degree if terrain is not None else 1
    basis = make_basis(mesh.dim, solution_degree, n_quad_1d)
    surface = None
    if terrain is not None:
        surface = TerrainSurface(terrain, mesh.extents, mesh.root_counts, geom_degree)
    geom = MeshGeometry(mesh, basis, surface, geom_degree)
    geom.validate()
    return geom


def apply_terrain_mapping(mesh, height_fn, z_top=None, solution_degree=4,
                          geom_degree=None, n_quad_1d=None):
    return build_geometry(mesh, solution_degree, terrain=height_fn,
                          geom_degree=geom_degree, n_quad_1d=n_quad_1d, z_top=z_top)
