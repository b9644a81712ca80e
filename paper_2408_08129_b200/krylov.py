"""Restarted GMRES on the device (orodg/krylov.py:17-115).

``gmres(action, rhs, ...)`` keeps the reference signature.  Two paths, both
on the GPU:

* the Helmholtz action built by ``imex.build_helmholtz_action`` runs the
  native solver loop of libdg (dg_gmres_helmholtz): basis, Gram-Schmidt
  dots/updates and the operator all on the device, Givens rotations on the
  host from one small read-back per Arnoldi step;
* any other linear callable is driven from Python over torch CUDA tensors
  (the callable receives and must return a CUDA float64 vector).

Orthogonalisation is classical Gram-Schmidt with the reference's selective
re-orthogonalisation test (norm drop below 1/sqrt 2 => one more pass) --
one fused multi-dot per pass instead of j+1 dependent MGS dots.
"""

import ctypes as C
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
    return _gmres_torch(action, rhs, x0, tol_rel, restart, max_iter, preconditioner)


def _gmres_torch(action, rhs, x0, tol_rel, restart, max_iter, preconditioner):
    import torch
    if not torch.cuda.is_available():
        raise DeviceError("gmres runs on the device; no CUDA device visible")
    dev = "cuda"
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


def native_gmres(ctx, a_dt, h, rhs, x0, tol_rel, restart, max_iter):
    """dg_gmres_helmholtz on device tensors; returns (x tensor, KrylovStats)."""
    torch = ctx.torch
    x = (x0.clone() if x0 is not None else torch.zeros_like(rhs)).contiguous()
    cst = L.KrylovStatsC()
    cap = max_iter + 8 * (max_iter // max(restart, 1) + 2)
    hist = (C.c_double * cap)()
    L.check(ctx.lib.dg_gmres_helmholtz(ctx.bind_stream(), a_dt, as_ptr(h), as_ptr(rhs),
                                       as_ptr(x), tol_rel, restart, max_iter, C.byref(cst),
                                       hist, cap))
    st = KrylovStats(iterations=cst.iterations, residual=cst.residual, restarts=cst.restarts,
                     converged=bool(cst.converged), breakdown=bool(cst.breakdown),
                     residual_history=list(hist[:cst.n_history]))
    return x, st
