"""Drop-in IMEX-RK layer (orodg/imex.py) over the native B200 solver.

``SplitOperators``, ``build_helmholtz_action``, ``imex_step``,
``_solve_implicit_stage`` and ``run_time_loop`` keep the reference's
signatures and semantics.  The ARS(2,2,2) step, the pressure fixed point and
the GMRES solves run inside libdg (dg_imex_step / dg_solve_implicit_stage):
stage linear combinations, explicit residuals, Helmholtz applies, Krylov
orthogonalisation and all norms are device kernels; the host only sees the
Hessenberg column and the fixed-point increment per iteration.  Other
tableaux run the same device operators from a Python stage loop.
"""

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from . import _lib as L
from .device import as_ptr
from .dgops import from_device, to_device
from .errors import ConfigurationError, UsageError
from .krylov import native_gmres
from .timing import NullTimer, credit


@dataclass(frozen=True)
class ButcherTableau:
    name: str
    a_ex: np.ndarray
    b_ex: np.ndarray
    a_im: np.ndarray
    b_im: np.ndarray

    def __post_init__(self):
        s = self.stages
        for Mx in (self.a_ex, self.a_im):
            if Mx.shape != (s, s):
                raise ConfigurationError("tableau matrices must be s x s")
        if np.any(np.triu(self.a_ex) != 0.0):
            raise ConfigurationError("explicit tableau must be strictly lower")
        if np.any(np.triu(self.a_im, 1) != 0.0):
            raise ConfigurationError("implicit tableau must be lower triangular")
        for bb in (self.b_ex, self.b_im):
            if abs(bb.sum() - 1.0) > 1e-13:
                raise ConfigurationError("weights must sum to 1")
        for bb, cc in ((self.b_ex, self.c_ex), (self.b_im, self.c_im)):
            if abs(bb @ cc - 0.5) > 1e-13:
                raise ConfigurationError("second-order condition b.c = 1/2 fails")
        if np.max(np.abs(self.c_ex - self.c_im)) > 1e-13:
            raise ConfigurationError("explicit/implicit abscissae must agree")

    @property
    def stages(self):
        return len(self.b_ex)

    @property
    def c_ex(self):
        return self.a_ex.sum(axis=1)

    @property
    def c_im(self):
        return self.a_im.sum(axis=1)

    @property
    def stiffly_accurate(self):
        return (np.allclose(self.a_im[-1], self.b_im, atol=1e-14)
                and np.allclose(self.a_ex[-1], self.b_ex, atol=1e-14))


def ars222():
    """ARS(2,2,2), gamma = 1 - 1/sqrt(2) (orodg/imex.py:77-89)."""
    g = 1.0 - 1.0 / np.sqrt(2.0)
    dl = 1.0 - 1.0 / (2.0 * g)
    return ButcherTableau(
        "ARS(2,2,2)",
        np.array([[0.0, 0.0, 0.0], [g, 0.0, 0.0], [dl, 1.0 - dl, 0.0]]),
        np.array([dl, 1.0 - dl, 0.0]),
        np.array([[0.0, 0.0, 0.0], [0.0, g, 0.0], [0.0, 1.0 - g, g]]),
        np.array([0.0, 1.0 - g, g]))


TABLEAUX = {"ars222": ars222}


@dataclass(frozen=True)
class ImplicitSolveConfig:
    fp_tol: float = 1e-6
    fp_max_iter: int = 10
    krylov_tol: float = 1e-8
    krylov_restart: int = 30
    krylov_max_iter: int = 1000
    preconditioner: str = "none"
    precond_refresh: int = 20

    def __post_init__(self):
        for t in (self.fp_tol, self.krylov_tol):
            if not 0.0 < t < 1.0:
                raise ConfigurationError(f"tolerance {t} outside (0,1)")
        for n in (self.fp_max_iter, self.krylov_restart, self.krylov_max_iter):
            if n < 1:
                raise ConfigurationError("iteration caps must be >= 1")
        if self.preconditioner not in ("none", "block_jacobi"):
            raise ConfigurationError(f"unknown preconditioner {self.preconditioner!r}")

    def c(self, precond_active=False):
        s = L.SolveCfg()
        s.fp_tol = self.fp_tol
        s.fp_max_iter = self.fp_max_iter
        s.krylov_tol = self.krylov_tol
        s.krylov_restart = self.krylov_restart
        s.krylov_max_iter = self.krylov_max_iter
        # imex.py:334: block_jacobi only with a cache object from the caller
        s.preconditioner = 1 if (self.preconditioner == "block_jacobi" and precond_active) else 0
        s.precond_refresh = self.precond_refresh
        return s


class PrecondCache:
    """The caller-side block-Jacobi cache of the reference (imex.py:245-249):
    ``apply`` (the current preconditioner or None), ``age`` (solves since it
    was built) and ``coloring`` (element colours, built on first use).  The
    blocks themselves live on the device context; ``age`` is mirrored."""

    def __init__(self):
        self.apply = None
        self.age = 10 ** 9
        self.coloring = None


_PrecondCache = PrecondCache


def _bj_enter(split, cfg, precond):
    """Arm the context's block-Jacobi state from the caller's cache; returns
    whether the stage solves precondition (imex.py:334)."""
    if cfg.preconditioner != "block_jacobi" or precond is None:
        return False
    from .krylov import BlockJacobi, _set_coloring, element_coloring
    ctx = split.ctx
    if precond.coloring is None:
        precond.coloring = element_coloring(split.ops.mesh)
    _set_coloring(ctx, precond.coloring)
    valid = isinstance(precond.apply, BlockJacobi) and precond.apply.ctx is ctx \
        and precond.apply.current()
    age = int(min(precond.age, 2 ** 30))
    L.check(ctx.lib.dg_bj_set_state(ctx.handle, 1 if valid else 0, age))
    return True


def _bj_exit(split, precond):
    from .krylov import BlockJacobi
    ctx = split.ctx
    valid, age, gen = C.c_int(), C.c_int(), C.c_longlong()
    L.check(ctx.lib.dg_bj_state(ctx.handle, C.byref(valid), C.byref(age), C.byref(gen)))
    precond.age = age.value
    if valid.value and not (isinstance(precond.apply, BlockJacobi)
                            and precond.apply.generation == gen.value):
        precond.apply = BlockJacobi(ctx, gen.value)


@dataclass
class StepStats:
    fp_iters: list = field(default_factory=list)
    krylov_iters: list = field(default_factory=list)
    pressure_increments: list = field(default_factory=list)
    mass_rate: float = 0.0

    def absorb(self, cs):
        self.fp_iters += list(cs.fp_iters[:cs.n_fp])
        self.krylov_iters += list(cs.krylov_iters[:cs.n_krylov])
        self.pressure_increments += list(cs.pressure_increments[:cs.n_krylov])
        self.mass_rate += cs.mass_rate


class SplitOperators:
    """Explicit / implicit residuals over the device kernels (imex.py:125-218)."""

    def __init__(self, ops, model, bcs=None, sponge=None, forcing=None):
        self.ops = ops
        self.geometry = ops.geometry
        self.model = model
        self.bcs = bcs
        self.sponge = sponge
        self.forcing = forcing
        self.dim = ops.dim
        self._last_mass_rate = 0.0
        self.ctx = ops.context(model, bcs, sponge)

    def explicit_residual(self, data, t=0.0):
        ctx = self.ctx
        U, host = to_device(data, ctx)
        R = ctx.empty(self.dim + 2, self.geometry.basis.n_nodes)
        mr = C.c_double()
        L.check(ctx.lib.dg_explicit_residual(ctx.bind_stream(), as_ptr(U), as_ptr(R),
                                             C.byref(mr)))
        self._last_mass_rate = mr.value
        if self.forcing is not None:
            R += to_device(self.forcing(t), ctx)[0]
        return from_device(R, host)

    def implicit_residual(self, data):
        """Pressure-gradient and enthalpy-divergence terms at the given state
        (imex.py:161-175): R[momentum] = -M^-2 Minv Grad(p), R[energy] =
        -Minv Div(h m), density row zero; device operators throughout."""
        ctx = self.ctx
        U, host = to_device(data, ctx)
        d = self.dim
        nn = self.geometry.basis.n_nodes
        h = ctx.empty(nn)
        K = ctx.empty(nn)
        L.check(ctx.lib.dg_frozen_coefficients(ctx.bind_stream(), as_ptr(U), as_ptr(h), as_ptr(K)))
        gm1 = self.model.gamma - 1.0
        # p = (gamma - 1)(rho E - kf rho k)  (physics.py pressure, imex.py:203)
        p = (U[:, 1 + d] - self.model.kinetic_factor * K) * gm1
        R = ctx.torch.zeros_like(U)
        gd = self.ops.gradient_scalar(p.contiguous(), self.model, self.bcs)
        R[:, 1:1 + d] = -self.model.inv_mach_sq * self.ops.apply_mass_inverse(gd)
        dv = self.ops.divergence_hv(U[:, 1:1 + d].contiguous(), h, self.model, self.bcs)
        R[:, 1 + d] = -self.ops.apply_mass_inverse(dv)[:, 0]
        return from_device(R, host)

    def full_residual(self, data, t=0.0):
        """explicit_residual + implicit_residual (imex.py:177-178)."""
        E = self.explicit_residual(data, t)
        return E + self.implicit_residual(data)

    def frozen_coefficients(self, data):
        ctx = self.ctx
        U, host = to_device(data, ctx)
        h = ctx.empty(self.geometry.basis.n_nodes)
        K = ctx.empty(self.geometry.basis.n_nodes)
        L.check(ctx.lib.dg_frozen_coefficients(ctx.bind_stream(), as_ptr(U), as_ptr(h), as_ptr(K)))
        return from_device(h, host), from_device(K, host)

    def energy_affine_map(self, a_dt, h, K, m_e, e_e):
        """(F, grad_p) of imex.py:190-218 as device closures."""
        ctx = self.ctx
        ht, _ = to_device(h, ctx)
        Kt, _ = to_device(K, ctx)
        mt, _ = to_device(m_e, ctx)
        et, _ = to_device(e_e, ctx)
        nn = self.geometry.basis.n_nodes
        d = self.dim

        def F(x):
            xt, host = to_device(x, ctx)
            out = ctx.empty(nn)
            L.check(ctx.lib.dg_energy_F(ctx.bind_stream(), a_dt, as_ptr(ht), as_ptr(Kt),
                                        as_ptr(mt), mt.stride(0), as_ptr(et), et.stride(0),
                                        as_ptr(xt), as_ptr(out)))
            return from_device(out, host)

        def grad_p(x):
            xt, host = to_device(x, ctx)
            out = ctx.empty(d, nn)
            L.check(ctx.lib.dg_grad_p(ctx.bind_stream(), as_ptr(xt), as_ptr(Kt), as_ptr(out),
                                      out.stride(0), None, 0, 1.0))
            return from_device(out, host)

        return F, grad_p


class HelmholtzAction:
    """x -> x - (F(x) - F(0)) on flat vectors, homogeneous form evaluated
    directly by the fused kernels (build_helmholtz_action, imex.py:221-242)."""

    def __init__(self, split, a_dt, h):
        self.split = split
        self.ctx = split.ctx
        self.a_dt = float(a_dt)
        self.h, _ = to_device(h, self.ctx)
        self.shape = tuple(self.h.shape)

    def __call__(self, xflat):
        ctx = self.ctx
        xt, host = to_device(xflat, ctx)
        xt = xt.reshape(self.shape).contiguous()
        y = ctx.empty(self.shape[1])
        # h frozen at construction (prepare_divergence_hv, dgops.py:399-479):
        # its Gauss values / traces are prepared once and reused
        L.check(ctx.lib.dg_helmholtz_apply_prepared(ctx.bind_stream(), self.a_dt,
                                                    as_ptr(self.h), as_ptr(xt), as_ptr(y)))
        return from_device(y.reshape(-1), host)

    def _native_gmres(self, rhs, x0, tol_rel, restart, max_iter, precond=False):
        ctx = self.ctx
        b, host = to_device(rhs, ctx)
        b = b.reshape(self.shape).contiguous()
        x = None
        if x0 is not None:
            x = to_device(x0, ctx)[0].reshape(self.shape).contiguous()
        xs, st = native_gmres(ctx, self.a_dt, self.h, b, x, tol_rel, restart, max_iter,
                              precond=precond)
        return from_device(xs.reshape(-1), host), st


def build_helmholtz_action(split, a_dt, lin_state, m_e=None, e_e=None):
    h, _ = split.frozen_coefficients(lin_state if not isinstance(lin_state, np.ndarray)
                                     else lin_state)
    return HelmholtzAction(split, a_dt, h)


def _is_ars222(tab):
    ref = ars222()
    return (tab.stages == 3 and np.allclose(tab.a_ex, ref.a_ex, atol=0, rtol=0)
            and np.allclose(tab.a_im, ref.a_im, atol=0, rtol=0)
            and np.allclose(tab.b_ex, ref.b_ex, atol=0, rtol=0)
            and np.allclose(tab.b_im, ref.b_im, atol=0, rtol=0))


def _step_error_info(cs):
    return dict(element=int(cs.fail_element), node=int(cs.fail_node),
                values=float(cs.fail_value))


def _solve_cfg(cfg, pc):
    """The C struct of a solver config: the drop-in's own
    ImplicitSolveConfig, or any object with the reference's fields (e.g.
    orodg.imex.ImplicitSolveConfig, which has no ``c()``)."""
    if hasattr(cfg, "c"):
        return cfg.c(pc)
    return ImplicitSolveConfig(
        fp_tol=cfg.fp_tol, fp_max_iter=cfg.fp_max_iter, krylov_tol=cfg.krylov_tol,
        krylov_restart=cfg.krylov_restart, krylov_max_iter=cfg.krylov_max_iter,
        preconditioner=getattr(cfg, "preconditioner", "none"),
        precond_refresh=getattr(cfg, "precond_refresh", 20)).c(pc)


# libdg profiler classes -> the reference's timer blocks (timing.py:12-13):
# the explicit operator is "explicit_residual", the Helmholtz applies and the
# Gram-Schmidt passes inside GMRES are "krylov"; the rest of the native step
# (stage combinations, F0, back-substitution, positivity) stays in
# "implicit_fixed_point"
_BLOCK_OF_CLASS = {0: "explicit_residual", 1: "krylov", 2: "krylov", 3: "krylov", 4: "krylov"}


def _profiled(ctx, timer, fn):
    """Run a native call inside timer.block("implicit_fixed_point") and move
    the CUDA-event time of its explicit / Krylov kernels to their blocks."""
    if timer is None or isinstance(timer, NullTimer):
        return fn()
    lib = ctx.lib
    lib.dg_profile_enable(1)
    try:
        with timer.block("implicit_fixed_point"):
            out = fn()
            ms, by, cnt = (C.c_double * 6)(), (C.c_double * 6)(), (C.c_longlong * 6)()
            lib.dg_profile_read(ms, by, cnt)
    finally:
        lib.dg_profile_enable(0)
    for k, name in _BLOCK_OF_CLASS.items():
        credit(timer, name, ms[k] * 1e-3, source="implicit_fixed_point")
    return out


def imex_step(data, t, dt, tableau, split, cfg, timer=None, precond=None):
    """One IMEX-RK step (imex.py:252-299); returns (new_data, StepStats).

    ARS(2,2,2) without forcing runs as one native call (dg_imex_step); other
    tableaux, or a SplitOperators with a forcing callable, run the
    reference's stage loop over the device operators with the forcing added
    to every explicit residual at t + c_ex[l] dt (imex.py:157-158, 286)."""
    ctx = split.ctx
    U, host = to_device(data, ctx)
    st = StepStats()
    pc = _bj_enter(split, cfg, precond)
    try:
        if _is_ars222(tableau) and split.forcing is None:
            out = ctx.empty(split.dim + 2, split.geometry.basis.n_nodes)
            cs = L.StepStatsC()
            ccfg = _solve_cfg(cfg, pc)
            code = _profiled(ctx, timer, lambda: ctx.lib.dg_imex_step(
                ctx.bind_stream(), as_ptr(U), as_ptr(out), float(t), float(dt), C.byref(ccfg),
                C.byref(cs)))
            st.absorb(cs)
            L.check(code, stats=st, **_step_error_info(cs))
            return from_device(out, host), st
        return _generic_step(U, host, t, dt, tableau, split, cfg, st, pc, timer)
    finally:
        if pc:
            _bj_exit(split, precond)


def _lincomb(ctx, coefs, xs, out):
    n = out.numel()
    arr = (C.c_double * len(coefs))(*coefs)
    ptrs = (C.c_void_p * len(xs))(*[x.data_ptr() for x in xs])
    L.check(ctx.lib.dg_lincomb(ctx.handle, n, len(xs), arr, ptrs, as_ptr(out)))


def _generic_step(U, host, t, dt, tab, split, cfg, st, pc=False, timer=None):
    """Arbitrary tableau: the reference's stage loop over device operators."""
    timer = timer or NullTimer()
    ctx = split.ctx
    ctx.bind_stream()
    s = tab.stages
    KE = [None] * s
    KI = [None] * s
    U_stage = U
    for l in range(s):
        acc = U.clone()
        for j in range(l):
            if tab.a_ex[l, j] != 0.0:
                _lincomb(ctx, [1.0, dt * tab.a_ex[l, j]], [acc, KE[j]], acc)
            if tab.a_im[l, j] != 0.0 and KI[j] is not None:
                _lincomb(ctx, [1.0, dt * tab.a_im[l, j]], [acc, KI[j]], acc)
        a_ll = tab.a_im[l, l]
        if a_ll == 0.0:
            U_stage = acc
            KI[l] = None
        else:
            it = ctx.empty(*acc.shape[1:])
            cs = L.StepStatsC()
            ccfg = _solve_cfg(cfg, pc)
            code = _profiled(ctx, timer, lambda: ctx.lib.dg_solve_implicit_stage(
                ctx.handle, as_ptr(acc), as_ptr(U_stage), dt * a_ll, C.byref(ccfg), as_ptr(it),
                C.byref(cs)))
            st.absorb(cs)
            L.check(code, stats=st, **_step_error_info(cs))
            KI[l] = ctx.empty(*acc.shape[1:])
            _lincomb(ctx, [1.0 / (dt * a_ll), -1.0 / (dt * a_ll)], [it, acc], KI[l])
            U_stage = it
        _check_positive(ctx, U_stage, l, t)
        if tab.b_ex[l] != 0.0 or np.any(tab.a_ex[l + 1:, l] != 0.0):
            KE[l] = ctx.empty(*acc.shape[1:])
            mr = C.c_double()
            with timer.block("explicit_residual"):
                L.check(ctx.lib.dg_explicit_residual(ctx.handle, as_ptr(U_stage), as_ptr(KE[l]),
                                                     C.byref(mr)))
                if split.forcing is not None:
                    # imex.py:157-158: R += forcing(t) at the stage time
                    f, _ = to_device(split.forcing(t + tab.c_ex[l] * dt), ctx)
                    KE[l] += f.reshape(KE[l].shape)
                if timer is not None and not isinstance(timer, NullTimer):
                    ctx.torch.cuda.current_stream().synchronize()
            st.mass_rate += tab.b_ex[l] * mr.value
    if tab.stiffly_accurate:
        return from_device(U_stage, host), st
    out = U.clone()
    for l in range(s):
        if tab.b_ex[l] != 0.0:
            _lincomb(ctx, [1.0, dt * tab.b_ex[l]], [out, KE[l]], out)
        if tab.b_im[l] != 0.0 and KI[l] is not None:
            _lincomb(ctx, [1.0, dt * tab.b_im[l]], [out, KI[l]], out)
    return from_device(out, host), st


def _check_positive(ctx, U, stage, t):
    mr, ir, mp, ip = C.c_double(), C.c_longlong(), C.c_double(), C.c_longlong()
    code = ctx.lib.dg_check_positivity(ctx.handle, as_ptr(U), C.byref(mr), C.byref(ir),
                                       C.byref(mp), C.byref(ip))
    L.check(code, element=ir.value, node=ip.value, values=mp.value)


def _solve_implicit_stage(acc, guess, a_dt, split, cfg, stats, timer=None, precond=None):
    """Pressure fixed point + GMRES for one DIRK stage (imex.py:302-370)."""
    ctx = split.ctx
    At, host = to_device(acc, ctx)
    Gt, _ = to_device(guess, ctx)
    it = ctx.empty(*At.shape[1:])
    cs = L.StepStatsC()
    pc = _bj_enter(split, cfg, precond)
    try:
        ccfg = _solve_cfg(cfg, pc)
        code = _profiled(ctx, timer, lambda: ctx.lib.dg_solve_implicit_stage(
            ctx.bind_stream(), as_ptr(At), as_ptr(Gt), float(a_dt), C.byref(ccfg), as_ptr(it),
            C.byref(cs)))
    finally:
        if pc:
            _bj_exit(split, precond)
    stats.fp_iters += []  # the caller appends fp counts, as the reference does
    stats.krylov_iters += list(cs.krylov_iters[:cs.n_krylov])
    stats.pressure_increments += list(cs.pressure_increments[:cs.n_krylov])
    L.check(code, stats=stats, **_step_error_info(cs))
    return from_device(it, host), int(cs.fp_iters[0])


def run_time_loop(data, dt, t_final, stepper, callbacks=(), timer=None, t0=0.0):
    """Fixed-dt driver landing exactly on t_final (imex.py:373-404): the
    callbacks run inside timer.block("output"), one timer.step_snapshot()
    per step, returns (data, timer.report(per_step))."""
    from .errors import SolverError
    if dt <= 0 or t_final <= t0:
        raise ConfigurationError("need dt > 0 and t_final > t0")
    timer = timer or NullTimer()
    per_step = []
    t = t0
    with timer.block("output"):
        for cb in callbacks:
            cb(0, t, data, None)
    n_full = int(np.floor((t_final - t0) / dt + 1e-12))
    rem = (t_final - t0) - n_full * dt
    if rem < 1e-12 * dt:
        rem = 0.0
    n_steps = n_full + (1 if rem else 0)
    for step in range(1, n_steps + 1):
        h = dt if step <= n_full else rem
        try:
            data, stats = stepper(data, t, h)
        except Exception as err:
            raise SolverError(f"step {step} at t={t:.6g} failed: {err}") from err
        t = t0 + step * dt if step < n_steps else t_final
        with timer.block("output"):
            for cb in callbacks:
                cb(step, t, data, stats)
        per_step.append(timer.step_snapshot())
    return data, timer.report(per_step)
