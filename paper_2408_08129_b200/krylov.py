"""Restarted GMRES on the device (orodg/krylov.py:17-115).

``gmres(action, rhs, ...)`` keeps the reference signature.  Two paths, both
on the GPU:

* the Helmholtz action built by ``imex.build_helmholtz_action`` runs the
  native solver loop of libdg (dg_gmres_helmholtz): basis, Gram-Schmidt
  dots/updates and the operator all on the device, Givens rotations on the
  host from one small read-back per Arnoldi step;
* any other linear callable is driven from Python over torch CUDA tensors:
  a device callable receives and returns CUDA float64 vectors, a host
  callable in the reference's numpy convention is detected and fed host
  copies (``_Operand``).

Orthogonalisation is classical Gram-Schmidt with the reference's selective
re-orthogonalisation test (norm drop below 1/sqrt 2 => one more pass) --
one fused multi-dot per pass instead of j+1 dependent MGS dots.
"""

import ctypes as C
import warnings
from dataclasses import dataclass, field

import numpy as np

from . import _lib as L
from .device import as_ptr
from .errors import ConfigurationError, DeviceError


@dataclass
class KrylovStats:
    iterations: int = 0
    residual: float = np.inf
    restarts: int = 0
    converged: bool = False
    breakdown: bool = False
    residual_history: list = field(default_factory=list)


def gmres(action, rhs, x0=None, tol_rel=1e-8, restart=30, max_iter=1000,
          preconditioner=None):
    if not (0.0 < tol_rel < 1.0):
        raise ConfigurationError(f"tol_rel must be in (0,1), got {tol_rel}")
    native = getattr(action, "_native_gmres", None)
    if native is not None and preconditioner is None:
        return native(rhs, x0, tol_rel, restart, max_iter)
    if (native is not None and isinstance(preconditioner, BlockJacobi)
            and preconditioner.ctx is action.ctx and preconditioner.current()):
        return native(rhs, x0, tol_rel, restart, max_iter, precond=True)
    return _gmres_torch(action, rhs, x0, tol_rel, restart, max_iter, preconditioner)


# ---------------------------------------------------------------- block Jacobi
def element_coloring(mesh):
    """Greedy colouring of the face-adjacency graph (krylov.py:118-140), in
    libdg (host code): conforming (left, right) and hanging (coarse, fine)
    pairs; returns int64 colours per leaf."""
    topo = mesh.topology
    a = [np.asarray(b.left, dtype=np.int64) for b in topo.conforming]
    a += [np.asarray(b.coarse, dtype=np.int64) for b in topo.hanging]
    b = [np.asarray(x.right, dtype=np.int64) for x in topo.conforming]
    b += [np.asarray(x.fine, dtype=np.int64) for x in topo.hanging]
    a = np.ascontiguousarray(np.concatenate(a) if a else np.zeros(0, np.int64))
    b = np.ascontiguousarray(np.concatenate(b) if b else np.zeros(0, np.int64))
    n = mesh.n_leaves
    colors = np.empty(n, dtype=np.int64)
    nc = C.c_int()
    lib = L.lib()
    L.check(lib.dg_element_coloring(n, a.size, a.ctypes.data, b.ctypes.data, colors.ctypes.data,
                                    C.byref(nc)))
    return colors


class BlockJacobi:
    """The device block-Jacobi inverse of one build (dg_bj_build) on a
    context: ``M(v)`` returns the blockwise inverse applied to v (a CUDA
    tensor or a host array, returned in kind).  A later build on the same
    context supersedes it (using a stale one raises UsageError)."""

    def __init__(self, ctx, generation, n_singular=0):
        self.ctx = ctx
        self.generation = generation
        self.n_singular = n_singular

    def current(self):
        g = C.c_longlong()
        L.check(self.ctx.lib.dg_bj_state(self.ctx.handle, None, None, C.byref(g)))
        return g.value == self.generation

    def __call__(self, v):
        from .errors import UsageError
        from .dgops import from_device, to_device
        if not self.current():
            raise UsageError("block-Jacobi preconditioner superseded by a later build")
        ctx = self.ctx
        x, host = to_device(v, ctx)
        x = x.contiguous()
        out = ctx.torch.empty_like(x)
        L.check(ctx.lib.dg_bj_apply(ctx.bind_stream(), as_ptr(x), as_ptr(out)))
        return from_device(out, host)


def _set_coloring(ctx, colors):
    colors = np.ascontiguousarray(np.asarray(colors, dtype=np.int64))
    if getattr(ctx, "_bj_coloring", None) is not None and np.array_equal(ctx._bj_coloring,
                                                                        colors):
        return
    n = colors.size
    L.check(ctx.lib.dg_bj_set_coloring(ctx.handle, colors.ctypes.data, n))
    ctx._bj_coloring = colors.copy()


def block_jacobi_preconditioner(action, n_el, n_nodes, coloring=None):
    """Inverse of the per-element diagonal blocks of the action (krylov.py:
    143-178), probed colour by colour.  The Helmholtz action of
    ``imex.build_helmholtz_action`` is probed and inverted in libdg; any
    other device callable is probed from Python and inverted with
    torch.linalg.inv."""
    colors = (np.asarray(coloring, dtype=np.int64) if coloring is not None
              else np.zeros(n_el, dtype=np.int64))
    ctx = getattr(action, "ctx", None)
    if getattr(action, "_native_gmres", None) is not None and ctx is not None:
        _set_coloring(ctx, colors)
        ns, gen = C.c_int(), C.c_longlong()
        L.check(ctx.lib.dg_bj_build(ctx.bind_stream(), action.a_dt, as_ptr(action.h),
                                    C.byref(ns), C.byref(gen)))
        if ns.value:
            warnings.warn(f"block Jacobi: {ns.value} singular blocks replaced by identity")
        return BlockJacobi(ctx, gen.value, ns.value)
    return _block_jacobi_torch(action, n_el, n_nodes, colors)


def _block_jacobi_torch(action, n_el, n_nodes, colors):
    import torch
    if not torch.cuda.is_available():
        raise DeviceError("block Jacobi runs on the device; no CUDA device visible")
    dev = "cuda"
    col = torch.as_tensor(colors, device=dev)
    blocks = torch.empty((n_el, n_nodes, n_nodes), dtype=torch.float64, device=dev)
    probe = torch.zeros((n_el, n_nodes), dtype=torch.float64, device=dev)
    for c in np.unique(colors):
        sel = col == int(c)
        for i in range(n_nodes):
            probe.zero_()
            probe[sel, i] = 1.0
            y = torch.as_tensor(action(probe.reshape(-1)), dtype=torch.float64,
                                device=dev).reshape(n_el, n_nodes)
            blocks[sel, :, i] = y[sel]
    inv, info = torch.linalg.inv_ex(blocks)
    bad = info != 0
    if bool(bad.any()):
        inv[bad] = torch.eye(n_nodes, dtype=torch.float64, device=dev)
        warnings.warn(f"block Jacobi: {int(bad.sum())} singular blocks replaced by identity")

    def apply(v):
        host = not isinstance(v, torch.Tensor)
        t = torch.as_tensor(np.asarray(v, dtype=np.float64) if host else v,
                            dtype=torch.float64, device=dev).reshape(n_el, n_nodes)
        out = torch.einsum("eij,ej->ei", inv, t).reshape(-1)
        return out.cpu().numpy() if host else out

    return apply


class _Operand:
    """Adapter for a user callable in the generic path: device callables get
    and return CUDA float64 vectors; a host callable in the reference's
    convention (numpy in, numpy out, krylov.py:27) is detected on first use
    -- it rejects the CUDA tensor or returns a numpy array -- and from then
    on gets a host copy, its result is moved to the device.  The Krylov
    basis, Gram-Schmidt passes and updates stay on the device either way."""

    def __init__(self, fn, dev):
        self.fn = fn
        self.dev = dev
        self.host = None

    def __call__(self, v):
        import torch
        if self.host is None:
            try:
                out = self.fn(v)
                self.host = not isinstance(out, torch.Tensor)
            except (TypeError, RuntimeError, AttributeError, ValueError):
                self.host = True
                out = self.fn(v.detach().cpu().numpy())
        elif self.host:
            out = self.fn(v.detach().cpu().numpy())
        else:
            out = self.fn(v)
        if not isinstance(out, torch.Tensor):
            out = torch.as_tensor(np.asarray(out, dtype=np.float64), device=self.dev)
        return out.reshape(-1).to(device=self.dev, dtype=torch.float64)


def _gmres_torch(action, rhs, x0, tol_rel, restart, max_iter, preconditioner):
    import torch
    if not torch.cuda.is_available():
        raise DeviceError("gmres runs on the device; no CUDA device visible")
    dev = "cuda"
    action = _Operand(action, dev)
    if preconditioner is not None:
        preconditioner = _Operand(preconditioner, dev)
    host = not isinstance(rhs, torch.Tensor)
    b = torch.as_tensor(np.asarray(rhs, dtype=np.float64).ravel() if host else rhs,
                        dtype=torch.float64, device=dev).reshape(-1)
    n = b.numel()
    M = preconditioner if preconditioner is not None else (lambda v: v)
    st = KrylovStats()
    bn = float(torch.linalg.vector_norm(b))
    if bn == 0.0:
        st.converged, st.residual = True, 0.0
        z = torch.zeros_like(b)
        return (z.cpu().numpy() if host else z), st
    if x0 is None:
        x = torch.zeros_like(b)
    else:
        x = torch.as_tensor(np.asarray(x0, dtype=np.float64).ravel()
                            if not isinstance(x0, torch.Tensor) else x0,
                            dtype=torch.float64, device=dev).reshape(-1).clone()
    r = b - action(x) if bool(torch.any(x != 0)) else b.clone()
    target = tol_rel * bn
    m = max(1, min(restart, n))
    V = torch.empty((m + 1, n), dtype=torch.float64, device=dev)
    H = np.zeros((m + 1, m))
    cs, sn, g = np.empty(m), np.empty(m), np.empty(m + 1)
    while True:
        beta = float(torch.linalg.vector_norm(r))
        st.residual = beta / bn
        st.residual_history.append(st.residual)
        if beta <= target or st.iterations >= max_iter or st.breakdown:
            break
        V[0] = r / beta
        g[:] = 0.0
        g[0] = beta
        done = 0
        for j in range(m):
            w = action(M(V[j])).reshape(-1).clone()
            nb = float(torch.linalg.vector_norm(w))
            h = (V[:j + 1] @ w)
            w -= h @ V[:j + 1]
            H[:j + 1, j] = h.cpu().numpy()
            na = float(torch.linalg.vector_norm(w))
            if na < 0.7071067811865476 * nb:
                c = V[:j + 1] @ w
                w -= c @ V[:j + 1]
                H[:j + 1, j] += c.cpu().numpy()
                na = float(torch.linalg.vector_norm(w))
            H[j + 1, j] = na
            st.iterations += 1
            happy = na <= 1e-14 * max(bn, nb)
            if not happy:
                V[j + 1] = w / na
            for i in range(j):
                t = cs[i] * H[i, j] + sn[i] * H[i + 1, j]
                H[i + 1, j] = -sn[i] * H[i, j] + cs[i] * H[i + 1, j]
                H[i, j] = t
            den = np.hypot(H[j, j], H[j + 1, j])
            cs[j] = H[j, j] / den if den else 1.0
            sn[j] = H[j + 1, j] / den if den else 0.0
            H[j, j] = den
            H[j + 1, j] = 0.0
            g[j + 1] = -sn[j] * g[j]
            g[j] = cs[j] * g[j]
            done = j + 1
            est = abs(g[j + 1])
            st.residual_history.append(est / bn)
            if happy:
                st.breakdown = True
                break
            if est <= target or st.iterations >= max_iter:
                break
        if done:
            y = np.zeros(done)
            for i in range(done - 1, -1, -1):
                y[i] = (g[i] - H[i, i + 1:done] @ y[i + 1:done]) / H[i, i]
            x += M(torch.as_tensor(y, device=dev) @ V[:done])
        r = b - action(x)
        st.restarts += 1
    st.restarts = max(0, st.restarts - 1)
    st.residual = float(torch.linalg.vector_norm(b - action(x))) / bn
    st.converged = st.residual <= tol_rel
    return (x.cpu().numpy() if host else x), st


def native_gmres(ctx, a_dt, h, rhs, x0, tol_rel, restart, max_iter, precond=False):
    """dg_gmres_helmholtz(_pc) on device tensors; returns (x tensor, KrylovStats)."""
    torch = ctx.torch
    x = (x0.clone() if x0 is not None else torch.zeros_like(rhs)).contiguous()
    cst = L.KrylovStatsC()
    cap = max_iter + 8 * (max_iter // max(restart, 1) + 2)
    hist = (C.c_double * cap)()
    L.check(ctx.lib.dg_gmres_helmholtz_pc(ctx.bind_stream(), a_dt, as_ptr(h), as_ptr(rhs),
                                          as_ptr(x), tol_rel, restart, max_iter,
                                          1 if precond else 0, C.byref(cst), hist, cap))
    st = KrylovStats(iterations=cst.iterations, residual=cst.residual, restarts=cst.restarts,
                     converged=bool(cst.converged), breakdown=bool(cst.breakdown),
                     residual_history=list(hist[:cst.n_history]))
    return x, st
