"""Ideal-gas Euler-with-gravity coefficients and pointwise host helpers.

Conserved layout (rho, rho u_1..rho u_d, rho E) on the variable axis, as in
the reference (orodg/physics.py:1-12).  The device kernels evaluate the same
pointwise formulas in registers; these numpy versions serve case setup,
boundary ghost derivation and API parity.
"""

from dataclasses import dataclass, field

import numpy as np

from .errors import ConfigurationError, PositivityError


@dataclass(frozen=True)
class PhysicalConstants:
    R: float = 287.0
    g: float = 9.81
    gamma: float = 1.4

    def __post_init__(self):
        if self.R <= 0 or self.g <= 0 or self.gamma <= 1:
            raise ConfigurationError(f"non-physical constants: {self}")

    @property
    def Gamma(self):
        return (self.gamma - 1.0) / self.gamma


CONST = PhysicalConstants()


@dataclass(frozen=True)
class FlowModel:
    """Equation-set coefficients (orodg/physics.py:80-100)."""

    gamma: float = CONST.gamma
    R_gas: float = CONST.R
    gravity: float = CONST.g
    inv_mach_sq: float = 1.0
    kinetic_factor: float = 1.0

    @classmethod
    def dimensional(cls, constants=CONST):
        return cls(gamma=constants.gamma, R_gas=constants.R,
                   gravity=constants.g, inv_mach_sq=1.0, kinetic_factor=1.0)


DIMENSIONAL = FlowModel.dimensional()


@dataclass
class PrimitiveState:
    rho: np.ndarray
    u: np.ndarray
    p: np.ndarray
    model: FlowModel = field(default=DIMENSIONAL, repr=False)

    @property
    def e(self):
        return self.p / ((self.model.gamma - 1.0) * self.rho)

    @property
    def k(self):
        return 0.5 * (self.u ** 2).sum(axis=0)

    @property
    def T(self):
        return self.p / (self.rho * self.model.R_gas)

    @property
    def sound_speed(self):
        return np.sqrt(self.model.gamma * self.model.inv_mach_sq * self.p / self.rho)


def n_variables(dim):
    return dim + 2


def _first_nonpositive(name, arr, where):
    if np.all(arr > 0.0):
        return
    loc = np.unravel_index(int(np.argmin(arr)), arr.shape)
    raise PositivityError(
        f"non-positive {name} ({arr[loc]:.6e}) at index {loc}"
        + (f" in {where}" if where else ""),
        element=loc[0] if arr.ndim > 1 else None,
        node=loc[-1] if arr.ndim > 1 else None,
        values=float(arr[loc]))


def conserved_to_primitive(U, model=DIMENSIONAL, var_axis=0, check=True, where=None):
    """(rho, u, p) from conserved variables (orodg/physics.py:136-164)."""
    U = np.asarray(U)
    d = U.shape[var_axis] - 2
    rho = np.take(U, 0, axis=var_axis)
    if check:
        _first_nonpositive("density", rho, where)
    u = np.stack([np.take(U, 1 + a, axis=var_axis) for a in range(d)]) / rho
    k = 0.5 * (u ** 2).sum(axis=0)
    p = (model.gamma - 1.0) * (np.take(U, d + 1, axis=var_axis)
                               - model.kinetic_factor * rho * k)
    if check:
        _first_nonpositive("pressure", p, where)
    return PrimitiveState(rho=rho, u=u, p=p, model=model)


def gravity_source(W, out=None):
    """[0; ...; -g rho; -kf g rho w] (orodg/physics.py:207-216)."""
    m = W.model
    d = W.u.shape[0]
    S = out if out is not None else np.zeros((d + 2,) + W.rho.shape)
    S[:d] = 0.0
    S[d] = -m.gravity * W.rho
    S[d + 1] = -m.kinetic_factor * m.gravity * W.rho * W.u[d - 1]
    return S


@dataclass(frozen=True)
class CourantReport:
    acoustic: float
    advective: float
    dt: float
    degree: int
    min_diameter: float
    dim: int
    max_sound_speed: float
    max_speed: float

    def __str__(self):
        return (f"C={self.acoustic:.4g} C_u={self.advective:.4g} "
                f"(dt={self.dt}, r={self.degree}, Hmin={self.min_diameter:.6g}, "
                f"d={self.dim}, c_max={self.max_sound_speed:.6g}, "
                f"|u|_max={self.max_speed:.6g})")


def courant_numbers(field_data, geometry, dt, model=DIMENSIONAL):
    """Acoustic and advective Courant numbers C = r c dt / (H sqrt(d))
    (physics.py:255-272): the maxima over all volume quadrature points are
    reduced on the device (libdg dg_courant_ingredients)."""
    import ctypes as C

    from . import _lib as L
    from .dgops import to_device
    from .device import DeviceContext, as_ptr
    cache = geometry.__dict__.setdefault("_b200_courant_ctx", {})
    ctx = cache.get(model)
    if ctx is None:
        ctx = cache[model] = DeviceContext(geometry, model)
    U, _ = to_device(field_data, ctx)
    out = (C.c_double * 4)()
    L.check(ctx.lib.dg_courant_ingredients(ctx.bind_stream(), as_ptr(U), out))
    c_max, u_max, rho_min, p_min = out[:]
    if not (rho_min > 0.0):
        raise PositivityError(f"non-positive density ({rho_min:.6e}) at a quadrature point")
    if not (p_min > 0.0):
        raise PositivityError(f"non-positive pressure ({p_min:.6e}) at a quadrature point")
    h_min = geometry.min_diameter
    d = geometry.mesh.dim
    fac = geometry.basis.degree * dt / (h_min * np.sqrt(d))
    return CourantReport(acoustic=fac * c_max, advective=fac * u_max, dt=dt,
                         degree=geometry.basis.degree, min_diameter=h_min, dim=d,
                         max_sound_speed=c_max, max_speed=u_max)
