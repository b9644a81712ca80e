"""ctypes binding of libdg.so (include/dg.h).

The library is the product: there is no CPU fallback.  If libdg.so is
missing or no CUDA device is visible, every device entry point raises
DeviceError instead of computing anything on the host.
"""

import ctypes as C
import os

from .errors import (ConfigurationError, DeviceError, PositivityError,
                     SolverError, UsageError)

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("DG_LIB_PATH") or os.path.join(HERE, "libdg.so")

DG_OK, DG_ERR_CUDA, DG_ERR_USAGE, DG_ERR_CONFIG, DG_ERR_POSITIVITY, DG_ERR_SOLVER, DG_ERR_COMM = range(7)
FACE_WALL, FACE_FARFIELD, FACE_CONF, FACE_FINE, FACE_COARSE = range(5)
DG_MAX_SOLVES = 256

P = C.c_void_p
D = C.c_double
I = C.c_int
LL = C.c_longlong


class CtxDesc(C.Structure):
    _fields_ = [("dim", I), ("degree", I), ("n_el", I), ("n_tot", I),
                ("per_root", D * 3), ("z_top", D), ("terrain", I),
                ("n_col", I), ("col_stride", I),
                ("elem", P), ("col", P), ("nbr", P), ("kind", P),
                ("hang_children", P), ("n_hang_groups", I), ("n_bface", I),
                ("ff_U", P), ("ff_p", P), ("ff_h", P), ("sigma", P), ("background", P),
                ("gamma", D), ("gravity", D), ("inv_mach_sq", D), ("kinetic_factor", D),
                ("tabs", P), ("tabs_len", I), ("device", I)]


class SolveCfg(C.Structure):
    _fields_ = [("fp_tol", D), ("fp_max_iter", I), ("krylov_tol", D),
                ("krylov_restart", I), ("krylov_max_iter", I),
                ("preconditioner", I), ("precond_refresh", I)]


class KrylovStatsC(C.Structure):
    _fields_ = [("iterations", I), ("restarts", I), ("converged", I), ("breakdown", I),
                ("residual", D), ("n_history", I)]


class StepStatsC(C.Structure):
    _fields_ = [("n_fp", I), ("fp_iters", I * 8), ("n_krylov", I),
                ("krylov_iters", I * DG_MAX_SOLVES),
                ("pressure_increments", D * DG_MAX_SOLVES), ("mass_rate", D),
                ("fail_stage", I), ("fail_kind", I), ("fail_element", LL),
                ("fail_node", I), ("fail_value", D)]


_SIGS = {
    "dg_last_error": ([], C.c_char_p),
    "dg_version": ([], I),
    "dg_ctx_create": ([C.POINTER(CtxDesc), C.POINTER(P)], I),
    "dg_ctx_destroy": ([P], I),
    "dg_ctx_set_stream": ([P, P], I),
    "dg_ctx_sync": ([P], I),
    "dg_ctx_launch_info": ([P, C.POINTER(I), C.POINTER(I), C.POINTER(LL)], I),
    "dg_divergence_advective": ([P, P, P], I),
    "dg_gradient_scalar": ([P, P, I, P], I),
    "dg_divergence_hv": ([P, P, LL, P, I, P], I),
    "dg_apply_mass_inverse": ([P, P, I, P], I),
    "dg_explicit_residual": ([P, P, P, C.POINTER(D)], I),
    "dg_frozen_coefficients": ([P, P, P, P], I),
    "dg_grad_p": ([P, P, P, P, LL, P, LL, D], I),
    "dg_energy_F": ([P, D, P, P, P, LL, P, LL, P, P], I),
    "dg_helmholtz_apply": ([P, D, P, P, P], I),
    "dg_gmres_helmholtz": ([P, D, P, P, P, D, I, I, C.POINTER(KrylovStatsC), P, I], I),
    "dg_gmres_helmholtz_pc": ([P, D, P, P, P, D, I, I, I, C.POINTER(KrylovStatsC), P, I], I),
    "dg_element_coloring": ([LL, LL, P, P, P, C.POINTER(I)], I),
    "dg_bj_set_coloring": ([P, P, LL], I),
    "dg_bj_build": ([P, D, P, C.POINTER(I), C.POINTER(LL)], I),
    "dg_bj_apply": ([P, P, P], I),
    "dg_bj_state": ([P, C.POINTER(I), C.POINTER(I), C.POINTER(LL)], I),
    "dg_bj_set_state": ([P, I, I], I),
    "dg_solve_implicit_stage": ([P, P, P, D, C.POINTER(SolveCfg), P, C.POINTER(StepStatsC)], I),
    "dg_imex_step": ([P, P, P, D, D, C.POINTER(SolveCfg), C.POINTER(StepStatsC)], I),
    "dg_integrate_conserved": ([P, P, P], I),
    "dg_check_positivity": ([P, P, C.POINTER(D), C.POINTER(LL), C.POINTER(D), C.POINTER(LL)], I),
    "dg_lincomb": ([P, LL, I, P, P, P], I),
    "dg_dots": ([P, LL, I, P, LL, P, P], I),
    "dg_divergence_full": ([P, P, I, P], I),
    "dg_global_inner_product": ([P, P, P, I, P], I),
    "dg_courant_ingredients": ([P, P, P], I),
    "dg_gs_update": ([P, LL, I, P, LL, P, P, D, P], I),
    "dg_dcgs2_update": ([P, LL, I, P, LL, P, P, P, P, P], I),
    "dg_dual_dots": ([P, LL, I, P, LL, P, P, P], I),
    "dg_nccl_unique_id": ([P], I),
    "dg_ctx_set_comm": ([P, P, I, I, P, P, P], I),
    "dg_ctx_set_comm_loopback": ([P, I, I, I, P, P, P], I),
    "dg_halo_exchange": ([P, P, I], I),
    "dg_ctx_set_halo_rows": ([P, I, P, P, P, P], I),
    "dg_halo_stats": ([P, C.POINTER(LL), I], I),
    "dg_max_abs_ratio": ([P, P, I, I, P, P], I),
    "dg_helmholtz_prepare": ([P, P], I),
    "dg_helmholtz_apply_prepared": ([P, D, P, P, P], I),
    "dg_split_contiguous": ([P, LL, I, P], I),
    "dg_launch_count": ([], LL),
    "dg_profile_enable": ([I], I),
    "dg_profile_read": ([P, P, P], I),
    "dg_arnoldi_stats": ([P, C.POINTER(LL), C.POINTER(LL)], I),
    "dg_set_arnoldi_mode": ([P, I], I),
    "dg_topology_build": ([I, P, P, LL, P, P, C.POINTER(P)], I),
    "dg_topology_counts": ([P, P, P, P], I),
    "dg_topology_copy": ([P, P, P, P, P, P, P], I),
    "dg_topology_free": ([P], I),
}

PROFILE_CLASSES = ("explicit", "gradient", "div_hv", "multidot", "axpy", "other")

EXPORTS = tuple(_SIGS)

_lib = None
_load_error = None


def load(path=LIB_PATH):
    """Load libdg.so once; raises DeviceError when it is missing."""
    global _lib, _load_error
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        _load_error = f"{path} not built (run python -m paper_2408_08129_b200.build)"
        raise DeviceError(_load_error)
    try:
        # torch first, so its libnccl.so.2 / libcudart satisfy libdg's sonames
        import torch  # noqa: F401
    except Exception:  # pragma: no cover
        pass
    lib = C.CDLL(path, mode=C.RTLD_GLOBAL)
    for name, (args, res) in _SIGS.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = res
    _lib = lib
    return lib


def lib():
    return _lib if _lib is not None else load()


_ERRS = {DG_ERR_CUDA: DeviceError, DG_ERR_USAGE: UsageError,
         DG_ERR_CONFIG: ConfigurationError, DG_ERR_POSITIVITY: PositivityError,
         DG_ERR_SOLVER: SolverError, DG_ERR_COMM: DeviceError}


def check(code, **extra):
    """Map a DG_ERR_* status onto the reference's exception classes."""
    if code == DG_OK:
        return
    msg = lib().dg_last_error().decode(errors="replace")
    cls = _ERRS.get(code, DeviceError)
    if cls is PositivityError:
        raise PositivityError(msg, element=extra.get("element"), node=extra.get("node"),
                              values=extra.get("values"))
    if cls is SolverError:
        raise SolverError(msg, stats=extra.get("stats"))
    raise cls(msg)
