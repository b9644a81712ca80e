"""Drop-in ``DGOperators`` on the B200 (orodg/dgops.py:34-511).

Same constructor and method names, argument meaning and return shapes as
the reference; every method runs the fused sm_100a kernels of libdg.  Input
arrays may be numpy (copied to the device, result copied back -- the
reference's calling convention) or torch CUDA float64 tensors (stay on the
device, zero host traffic).

Boundary conditions and the sponge are baked into a device context when
first seen (they are immutable for the life of a mesh, as in the reference's
index caches, dgops.py:69-77); contexts are cached per (bcs, model, sponge).
"""

import ctypes as C

import numpy as np

from . import _lib as L
from .device import DeviceContext, as_ptr
from .errors import UsageError
from .field import StateField
from .physics import DIMENSIONAL


def to_device(x, ctx):
    """(torch CUDA float64 contiguous tensor, was_host)."""
    torch = ctx.torch
    if isinstance(x, StateField):
        x = x.data
    if isinstance(x, torch.Tensor):
        t = x
        host = False
        if t.device.type != "cuda" or t.dtype != torch.float64:
            t = t.to(device=f"cuda:{ctx.device}", dtype=torch.float64)
            host = x.device.type != "cuda"
        return t.contiguous(), host
    a = np.ascontiguousarray(np.asarray(x, dtype=np.float64))
    return torch.from_numpy(a).to(f"cuda:{ctx.device}"), True


def from_device(t, host):
    return t.cpu().numpy() if host else t


class DGOperators:
    def __init__(self, geometry, pool=None, timer=None, device=None):
        self.geometry = geometry
        self.mesh = geometry.mesh
        self.basis = geometry.basis
        self.dim = self.mesh.dim
        self.pool = pool
        self.timer = timer
        self.device = device
        self._ctxs = {}

    # ---------------------------------------------------------- contexts
    def context(self, model=DIMENSIONAL, bcs=None, sponge=None):
        key = (id(bcs), model, id(sponge) if sponge is not None else None)
        ent = self._ctxs.get(key)
        if ent is None:
            ctx = DeviceContext(self.geometry, model, bcs, sponge, device=self.device)
            ent = (ctx, bcs, sponge)   # keep bcs/sponge alive: ids stay valid
            self._ctxs[key] = ent
        return ent[0]

    def _check_field(self, field):
        if field.mesh_id != self.mesh.fingerprint or field.degree != self.basis.degree:
            raise UsageError("field does not belong to this mesh/degree")

    def _shape_check(self, t, k):
        want = (self.mesh.n_leaves, k, self.basis.n_nodes)
        if tuple(t.shape) != want:
            raise UsageError(f"array shape {tuple(t.shape)}, expected {want}")

    # ------------------------------------------------------------ engine
    def weak_form(self, data, k_out, vol_flux, face_flux, bc_ghost, pool=None):
        """The reference's generic weak-form engine (dgops.py:87-230) takes
        numpy flux callbacks evaluated batch by batch on the host; the device
        path has no generic callback engine, only the fused operators below
        (divergence_advective / divergence_full / gradient_scalar /
        divergence_hv), so this raises instead of silently running on the
        CPU."""
        raise UsageError(
            "DGOperators.weak_form with host flux callbacks is not available on the B200 "
            "path; use divergence_advective, divergence_full, gradient_scalar or "
            "divergence_hv (fused device operators)")

    # ------------------------------------------------------------ duals
    def divergence_advective(self, data, model=DIMENSIONAL, bcs=None, pool=None):
        """Dual of the advective flux divergence, Rusanov with the flow speed
        as dissipation speed (dgops.py:285-296)."""
        ctx = self.context(model, bcs)
        U, host = to_device(data, ctx)
        self._shape_check(U, self.dim + 2)
        out = ctx.empty(self.dim + 2, self.basis.n_nodes)
        L.check(ctx.lib.dg_divergence_advective(ctx.bind_stream(), as_ptr(U), as_ptr(out)))
        return from_device(out, host)

    def divergence_full(self, data, model=DIMENSIONAL, bcs=None, flux="rusanov", pool=None):
        """Dual of the full Euler flux divergence (dgops.py:298-328); flux
        'rusanov' (local max |u.n| + c) or 'centered'."""
        codes = {"rusanov": 1, "centered": 2}
        if flux not in codes:
            from .errors import ConfigurationError
            raise ConfigurationError(f"unknown flux {flux!r}")
        ctx = self.context(model, bcs)
        U, host = to_device(data, ctx)
        self._shape_check(U, self.dim + 2)
        out = ctx.empty(self.dim + 2, self.basis.n_nodes)
        L.check(ctx.lib.dg_divergence_full(ctx.bind_stream(), as_ptr(U), codes[flux],
                                           as_ptr(out)))
        return from_device(out, host)

    def apply_divergence(self, field, model=DIMENSIONAL, bcs=None, flux="rusanov", pool=None,
                         mass_inverse=True):
        """Divergence residual of the full flux for a StateField, optionally
        mass-inverted to nodal (dgops.py:483-488)."""
        self._check_field(field)
        dual = self.divergence_full(field.data, model, bcs, flux, pool)
        return self.apply_mass_inverse(dual) if mass_inverse else dual

    def gradient_scalar(self, p, model=DIMENSIONAL, bcs=None, pool=None):
        """Dual of the weak gradient, centred interface value (dgops.py:332-366)."""
        ctx = self.context(model, bcs)
        pt, host = to_device(p, ctx)
        out = ctx.empty(self.dim, self.basis.n_nodes)
        L.check(ctx.lib.dg_gradient_scalar(ctx.bind_stream(), as_ptr(pt), 0, as_ptr(out)))
        return from_device(out, host)

    def divergence_hv(self, V, h, model=DIMENSIONAL, bcs=None, pool=None):
        """Dual of div(h V), centred flux (dgops.py:368-397)."""
        ctx = self.context(model, bcs)
        Vt, host = to_device(V, ctx)
        ht, _ = to_device(h, ctx)
        out = ctx.empty(1, self.basis.n_nodes)
        L.check(ctx.lib.dg_divergence_hv(ctx.bind_stream(), as_ptr(Vt), Vt.stride(0),
                                         as_ptr(ht), 0, as_ptr(out)))
        return from_device(out, host)

    def prepare_divergence_hv(self, h, model=DIMENSIONAL, bcs=None, pool=None):
        """divergence_hv with h frozen (dgops.py:399-479).  On the device h is
        read in-kernel from its nodal values, so 'preparing' only pins it."""
        ctx = self.context(model, bcs)
        ht, _ = to_device(h, ctx)

        def apply(V, pool=None):
            Vt, host = to_device(V, ctx)
            out = ctx.empty(1, self.basis.n_nodes)
            L.check(ctx.lib.dg_divergence_hv(ctx.bind_stream(), as_ptr(Vt), Vt.stride(0),
                                             as_ptr(ht), 0, as_ptr(out)))
            return from_device(out, host)

        return apply

    def apply_mass_inverse(self, dual):
        """Factorised mass inverse (geometry.py:372-396); the reference's
        entry point is ``MeshGeometry.apply_mass_inverse`` (same kernel)."""
        ctx = self.context()
        dt, host = to_device(dual, ctx)
        k = dt.shape[1] if dt.dim() == 3 else 1
        out = ctx.empty(*dt.shape[1:])
        L.check(ctx.lib.dg_apply_mass_inverse(ctx.bind_stream(), as_ptr(dt), k, as_ptr(out)))
        return from_device(out, host)

    # -------------------------------------------------------- reductions
    def global_inner_product(self, a, b):
        """Deterministic quadrature-weighted inner product (dgops.py:491-503)."""
        if isinstance(a, StateField):
            self._check_field(a)
            a.check_compatible(b)
            a, b = a.data, b.data
        if tuple(a.shape) != tuple(b.shape):
            raise UsageError(f"shape mismatch {tuple(a.shape)} vs {tuple(b.shape)}")
        ctx = self.context()
        at, _ = to_device(a, ctx)
        bt, _ = to_device(b, ctx)
        k = at.shape[1] if at.dim() == 3 else 1
        out = C.c_double()
        L.check(ctx.lib.dg_global_inner_product(ctx.bind_stream(), as_ptr(at), as_ptr(bt), k,
                                                C.byref(out)))
        return float(out.value)

    def max_abs_ratio(self, data, num, den, mask=None):
        """max |data[:, num] / data[:, den]| over the nodes (optionally a
        boolean (n_el, n_nodes) mask) on the device -- the runner's max |w|
        (num = d, den = 0) and probe diagnostics (runner.py:247-260)."""
        ctx = self.context()
        U, _ = to_device(data, ctx)
        m = None
        if mask is not None:
            mk = np.ascontiguousarray(np.asarray(mask, dtype=np.uint8).reshape(-1))
            m = ctx.torch.from_numpy(mk).to(U.device)
        out = C.c_double()
        L.check(ctx.lib.dg_max_abs_ratio(ctx.bind_stream(), as_ptr(U), int(num), int(den),
                                         as_ptr(m) if m is not None else None, C.byref(out)))
        return float(out.value)

    def integrate_conserved(self, field_or_data):
        """Per-variable domain integrals (dgops.py:505-511)."""
        ctx = self.context()
        U, _ = to_device(field_or_data, ctx)
        out = (C.c_double * (self.dim + 2))()
        L.check(ctx.lib.dg_integrate_conserved(ctx.bind_stream(), as_ptr(U), out))
        return np.array(out[:])
