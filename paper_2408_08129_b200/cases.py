"""Case inputs for the BASELINE configurations (harness, not hot path).

Background, sponge and far-field recipes restate orodg/cases.py:29-174 so
the GPU box (which has no reference tree) can build the same inputs; the
warm bubble and the seeded smooth perturbation are the harness choices
recorded in tests/golden/make_golden.py and SURVEY.md §8d.
"""

import math
from dataclasses import dataclass, field, replace

import numpy as np

from .boundary import BoundaryCondition
from .errors import ConfigurationError
from .physics import CONST, PhysicalConstants


@dataclass(frozen=True)
class HillCaseConfig:
    h_c: float = 400.0
    a_c: float = 1000.0
    x_c: float = 30.0e3
    y_c: float = 20.0e3
    N_buoyancy: float = 0.01
    u_bar: float = 10.0
    p_ref: float = 1.0e5
    T_ref: float = 293.15
    domain: tuple = (60.0e3, 40.0e3, 16.0e3)
    t_final: float = 3600.0
    dt: float = 2.0
    constants: PhysicalConstants = CONST

    @property
    def dim(self):
        return len(self.domain)

    @property
    def rho_ref(self):
        return self.p_ref / (self.constants.R * self.T_ref)


@dataclass(frozen=True)
class SpongeConfig:
    top_depth: float = 4.0e3
    lateral_width: float = 10.0e3
    sigma_max: float = 0.05

    def __post_init__(self):
        if self.sigma_max < 0 or self.top_depth < 0 or self.lateral_width < 0:
            raise ConfigurationError("sponge parameters must be >= 0")


def hydrostatic_state(z, cfg=HillCaseConfig()):
    """Constant-N hydrostatic pair p(z), rho(z) with dp/dz = -rho g
    (orodg/cases.py:80-106)."""
    c = cfg.constants
    z = np.asarray(z, dtype=float)
    n2g = cfg.N_buoyancy ** 2 / c.g
    e = np.exp(-n2g * z)
    br = 1.0 - (c.g ** 2 / cfg.N_buoyancy ** 2) * c.Gamma * (cfg.rho_ref / cfg.p_ref) * (1.0 - e)
    if np.any(br <= 0.0):
        raise ConfigurationError("hydrostatic profile breaks down: domain too tall "
                                 f"(min bracket {br.min():.4g})")
    p = cfg.p_ref * br ** (1.0 / c.Gamma)
    rho = cfg.rho_ref * (p / cfg.p_ref) ** (1.0 / c.gamma) * e
    return p, rho, cfg.u_bar


def hydrostatic_initial_state(cfg, u_bar=None):
    ub = cfg.u_bar if u_bar is None else u_bar
    g = cfg.constants.gamma
    d = cfg.dim

    def f(coords):
        p, rho, _ = hydrostatic_state(coords[..., -1], cfg)
        out = np.zeros(coords.shape[:-1] + (d + 2,))
        out[..., 0] = rho
        out[..., 1] = rho * ub
        out[..., 1 + d] = p / (g - 1.0) + 0.5 * rho * ub ** 2
        return out

    return f


def warm_bubble_state(dim=2, theta0=300.0, dtheta=2.0, xc=10.0e3, zc=2.0e3,
                      rc=2.0e3, p0=1.0e5, constants=CONST):
    """Warm bubble of BASELINE configs[0..1] (recipe in make_golden.py)."""
    R, g, gam = constants.R, constants.g, constants.gamma
    cp = R * gam / (gam - 1.0)

    def f(coords):
        x, z = coords[..., 0], coords[..., -1]
        ex = 1.0 - g * z / (cp * theta0)
        p = p0 * ex ** (cp / R)
        r = np.sqrt((x - xc) ** 2 + (z - zc) ** 2)
        th = theta0 + np.where(r < rc, dtheta * np.cos(0.5 * np.pi * r / rc) ** 2, 0.0)
        out = np.zeros(coords.shape[:-1] + (dim + 2,))
        out[..., 0] = p / (R * th * ex)
        out[..., dim + 1] = p / (gam - 1.0)
        return out

    return f


def smooth_noise(coords, extents, rng, n_modes=8, kmax=4):
    d = coords.shape[-1]
    s = np.zeros(coords.shape[:-1])
    for _ in range(n_modes):
        k = rng.integers(1, kmax + 1, size=d)
        a = rng.normal() / 8.0
        phi = rng.uniform(0.0, 2.0 * np.pi)
        arg = phi + sum(2.0 * np.pi * k[i] * coords[..., i] / extents[i] for i in range(d))
        s += a * np.sin(arg)
    return s


def perturbed_state(background, coords, extents, seed, u_scale=10.0):
    """Background plus seeded smooth 1e-3 perturbations."""
    rng = np.random.default_rng(seed)
    U = background.copy()
    d = coords.shape[-1]
    U[:, 0] *= 1.0 + 1e-3 * smooth_noise(coords, extents, rng)
    for a in range(d):
        s_a = smooth_noise(coords, extents, rng)
        U[:, 1 + a] = U[:, 1 + a] / background[:, 0] * U[:, 0] + U[:, 0] * 1e-3 * u_scale * s_a
    U[:, d + 1] *= 1.0 + 1e-3 * smooth_noise(coords, extents, rng)
    return U


def energy_like(U, seed):
    d = U.shape[1] - 2
    rng = np.random.default_rng(seed)
    return U[:, d + 1] * (1.0 + 1e-3 * rng.standard_normal(U[:, d + 1].shape))


def sponge_sigma(geometry, sponge, extents, lateral_axes=(0,)):
    """Nodal Rayleigh rate, sin^2 ramps combined by max (orodg/cases.py:127-146)."""
    xyz = geometry.node_coords
    sig = np.zeros(xyz.shape[:2])
    if sponge.sigma_max == 0.0:
        return sig
    zt = extents[-1]
    if sponge.top_depth > 0.0:
        r = np.clip((xyz[..., -1] - (zt - sponge.top_depth)) / sponge.top_depth, 0.0, 1.0)
        sig = np.maximum(sig, np.sin(0.5 * np.pi * r) ** 2)
    if sponge.lateral_width > 0.0:
        w = sponge.lateral_width
        for a in lateral_axes:
            lo = np.clip((w - xyz[..., a]) / w, 0.0, 1.0)
            hi = np.clip((xyz[..., a] - (extents[a] - w)) / w, 0.0, 1.0)
            sig = np.maximum(sig, np.sin(0.5 * np.pi * np.maximum(lo, hi)) ** 2)
    return sponge.sigma_max * sig


def farfield_bcs(geometry, background_data, wall_axes_sides=(("z", 0),)):
    """Wall on the named (axis, side) batches, far-field background traces
    elsewhere (orodg/cases.py:156-174)."""
    mesh = geometry.mesh
    d = mesh.dim
    names = {"x": 0, "y": 1, "z": d - 1}
    walls = {(names[a], s) for a, s in wall_axes_sides}
    b = geometry.basis
    out = []
    for bt in mesh.topology.boundary:
        if (bt.axis, bt.side) in walls:
            out.append(BoundaryCondition("wall"))
            continue
        fidx = b.face_nodes[bt.axis][bt.side]
        vals = background_data[bt.leaves][:, :, fidx]
        out.append(BoundaryCondition("farfield", vals @ b.face_interp.T))
    return out


def hill_profile(x, y=None, cfg=HillCaseConfig()):
    """Bell-shaped mountain h_c / [1 + ((x-x_c)/a_c)^2 (+ ((y-y_c)/a_c)^2)]^1.5
    (orodg/cases.py:71-77, the reference presets' terrain)."""
    r2 = ((np.asarray(x, dtype=float) - cfg.x_c) / cfg.a_c) ** 2
    if y is not None:
        r2 = r2 + ((np.asarray(y, dtype=float) - cfg.y_c) / cfg.a_c) ** 2
    return cfg.h_c / (1.0 + r2) ** 1.5


@dataclass(frozen=True)
class ManufacturedConfig:
    """Gravity-free space-time-periodic exact solution on the unit box; every
    field rides the phase theta = k (x + z) - omega t (orodg/cases.py:178-196)."""
    rho0: float = 1.0
    amp_rho: float = 0.15
    u0: float = 0.4
    amp_u: float = 0.12
    w0: float = -0.3
    amp_w: float = 0.1
    p0: float = 1.0
    amp_p: float = 0.15
    wavenumber: float = 2.0 * math.pi
    omega: float = 2.0 * math.pi * 0.7
    gamma: float = CONST.gamma


def _mms_fields(cfg, th):
    s, c = np.sin(th), np.cos(th)
    prim = (cfg.rho0 + cfg.amp_rho * s, cfg.u0 + cfg.amp_u * c, cfg.w0 + cfg.amp_w * s,
            cfg.p0 + cfg.amp_p * c)
    dprim = (cfg.amp_rho * c, -cfg.amp_u * s, cfg.amp_w * c, -cfg.amp_p * s)
    return prim, dprim


def manufactured_state(coords, t, cfg=ManufacturedConfig()):
    """Exact conserved state (orodg/cases.py:213-222)."""
    th = cfg.wavenumber * (coords[..., 0] + coords[..., 1]) - cfg.omega * t
    (rho, ux, uz, p), _ = _mms_fields(cfg, th)
    out = np.empty(coords.shape[:-1] + (4,))
    out[..., 0] = rho
    out[..., 1] = rho * ux
    out[..., 2] = rho * uz
    out[..., 3] = p / (cfg.gamma - 1.0) + 0.5 * rho * (ux ** 2 + uz ** 2)
    return out


def manufactured_forcing(coords, t, cfg=ManufacturedConfig()):
    """S = dU/dt + div F(U) of the exact solution, by the chain rule through
    the single phase theta (orodg/cases.py:225-260): d/dt = -omega d/dtheta,
    d/dx = d/dz = k d/dtheta."""
    k, om = cfg.wavenumber, cfg.omega
    gm1 = cfg.gamma - 1.0
    th = k * (coords[..., 0] + coords[..., 1]) - om * t
    (rho, ux, uz, p), (dr, du, dw, dp) = _mms_fields(cfg, th)
    ke = 0.5 * (ux * ux + uz * uz)
    rE = p / gm1 + rho * ke
    dE = dp / gm1 + dr * ke + rho * (ux * du + uz * dw)
    dU = (dr, dr * ux + rho * du, dr * uz + rho * dw, dE)
    dFx = (dr * ux + rho * du, dr * ux * ux + 2.0 * rho * ux * du + dp,
           dr * uz * ux + rho * dw * ux + rho * uz * du, (dE + dp) * ux + (rE + p) * du)
    dFz = (dr * uz + rho * dw, dr * ux * uz + rho * du * uz + rho * ux * dw,
           dr * uz * uz + 2.0 * rho * uz * dw + dp, (dE + dp) * uz + (rE + p) * dw)
    out = np.empty(coords.shape[:-1] + (4,))
    for i in range(4):
        out[..., i] = -om * dU[i] + k * (dFx[i] + dFz[i])
    return out


def gaussian_hill(h0=400.0, a=3.0e3, xc=30.0e3, yc=30.0e3):
    """BASELINE configs[3] hill: h0 exp(-(r/a)^2), half-width a (harness pin)."""
    def f(x, y):
        return h0 * np.exp(-(((x - xc) ** 2 + (y - yc) ** 2) / a ** 2))
    return f


def schar_terrain(h0=250.0, a=5.0e3, lam=4.0e3, xc=25.0e3):
    """BASELINE configs[2] terrain on [0, 50] km (shifted by 25 km)."""
    def f(x):
        xs = x - xc
        return h0 * np.exp(-(xs / a) ** 2) * np.cos(np.pi * xs / lam) ** 2
    return f


# ------------------------------------------------------------------------
# BASELINE.json configurations (presets for the drop-in)
# ------------------------------------------------------------------------

@dataclass
class BaselineCase:
    name: str
    mesh: object
    geometry: object
    model: object
    bcs: list
    sponge: object          # (sigma, background) or None
    U0: np.ndarray
    dt: float
    solve: dict             # ImplicitSolveConfig kwargs
    description: str = ""


def _subset_coords(geometry, elements):
    nodes = geometry.basis.nodes_1d
    return geometry._map_points(nodes, nodes, elements)


def baseline_case(name, root_scale=1.0, with_state=True):
    """Build one of the BASELINE configs (cfg1..cfg5) through the host API.

    root_scale < 1 shrinks the horizontal root grid (same recipe, smaller
    box) -- used for the bounded CPU-baseline samples.
    """
    from .boundary import wall_everywhere
    from .field import project_initial_data
    from .geometry import build_geometry
    from .mesh import build_uniform_mesh, refine_region
    from .physics import FlowModel

    model = FlowModel.dimensional()
    if name in ("cfg1", "cfg2"):
        root = (32, 16) if name == "cfg1" else (64, 32)
        mesh = build_uniform_mesh((20.0e3, 10.0e3), root)
        if name == "cfg2":
            mesh = refine_region(mesh, lambda lf: lf.center[1] < 5.0e3, 1)
        geom = build_geometry(mesh, 2 if name == "cfg1" else 4)
        U0 = project_initial_data(geom, warm_bubble_state()).data if with_state else None
        return BaselineCase(name, mesh, geom, model, wall_everywhere(mesh), None, U0, 0.5,
                            dict(krylov_tol=1e-8 if name == "cfg1" else 1e-10),
                            "2D warm bubble 20x10 km, walls" + (
                                ", 64x32 + z<5 km refined, r=4" if name == "cfg2" else
                                ", 32x16, r=2"))
    if name == "cfg3":
        ext = (50.0e3, 21.0e3)
        nx = max(2, int(round(400 * root_scale)))
        mesh = build_uniform_mesh((ext[0] * nx / 400, ext[1]), (nx, 168))
        zc = lambda lo, hi: 0.5 * (lo[:, -1] + hi[:, -1])  # noqa: E731
        mesh = refine_region(mesh, lambda i, l, o, lo, hi: zc(lo, hi) < 6.0e3, 1, vectorized=True)
        mesh = refine_region(mesh, lambda i, l, o, lo, hi: zc(lo, hi) < 2.5e3, 1, vectorized=True)
        hc = HillCaseConfig(domain=mesh.extents, T_ref=280.0)
        geom = build_geometry(mesh, 4, terrain=schar_terrain())
        return _terrain_case(name, mesh, geom, model, hc,
                             SpongeConfig(top_depth=9.0e3, lateral_width=10.0e3), (0,),
                             # dt: the acoustic Courant number per node spacing of
                             # the reference's paper2d preset (dt = 2 s on 500 m
                             # cells, runner.py:35) on this mesh's 31 m cells; at
                             # dt = 1 s unpreconditioned GMRES(30) stalls at 1.6e-8
                             with_state, 0.125, "2D Schar terrain, ~220k cells, r=4")
    if name == "cfg4":
        n = max(2, int(round(120 * root_scale)))
        ext = (60.0e3 * n / 120, 60.0e3 * n / 120, 20.0e3)
        mesh = build_uniform_mesh(ext, (n, n, 20))
        zc = lambda lo, hi: 0.5 * (lo[:, -1] + hi[:, -1])  # noqa: E731
        mesh = refine_region(mesh, lambda i, l, o, lo, hi: zc(lo, hi) < 6.0e3, 1, vectorized=True)
        mesh = refine_region(mesh, lambda i, l, o, lo, hi: zc(lo, hi) < 2.0e3, 1, vectorized=True)
        hc = HillCaseConfig(domain=ext, x_c=ext[0] / 2, y_c=ext[1] / 2)
        geom = build_geometry(mesh, 3, terrain=gaussian_hill(xc=ext[0] / 2, yc=ext[1] / 2))
        return _terrain_case(name, mesh, geom, model, hc, SpongeConfig(), (0, 1),
                             with_state, 0.5,
                             "3D Gaussian hill 60x60x20 km, 120x120x20 root, refined z<6 km "
                             "and z<2 km (3 levels), r=3")
    if name.startswith("cfg4w"):
        # "cfg4w<n>": an n x n x 20 root window of the cfg4 recipe centred on
        # the hill -- the same 500 m roots, refinement (z < 6 km, z < 2 km),
        # hill, dt, far-field / wall boundaries and top sponge; the 10 km
        # lateral sponge of the full 60 km box lies outside a central window
        # (<= 40 km), so it is absent.  The like-for-like sample on which the
        # CPU reference and the GPU are timed side by side (bench.py)
        n = int(name[5:]) if len(name) > 5 else 6
        ext = (500.0 * n, 500.0 * n, 20.0e3)
        mesh = build_uniform_mesh(ext, (n, n, 20))
        zc = lambda lo, hi: 0.5 * (lo[:, -1] + hi[:, -1])  # noqa: E731
        mesh = refine_region(mesh, lambda i, l, o, lo, hi: zc(lo, hi) < 6.0e3, 1, vectorized=True)
        mesh = refine_region(mesh, lambda i, l, o, lo, hi: zc(lo, hi) < 2.0e3, 1, vectorized=True)
        hc = HillCaseConfig(domain=ext, x_c=ext[0] / 2, y_c=ext[1] / 2)
        geom = build_geometry(mesh, 3, terrain=gaussian_hill(xc=ext[0] / 2, yc=ext[1] / 2))
        return _terrain_case(name, mesh, geom, model, hc, SpongeConfig(), (), with_state, 0.5,
                             f"cfg4 recipe, central {n}x{n}x20-root window (lateral sponge "
                             "outside the window), r=3")
    if name.startswith("cfg5"):
        # "cfg5_r<degree>": the operator microbenchmark (BASELINE configs[4],
        # SURVEY.md §8d): periodic (10 km)^3 box, a seeded 7% of the roots
        # refined once (about 30% of the interior face rows hanging), state =
        # hydrostatic background + seeded smooth 1e-3 perturbations; root
        # count chosen for 1e8 total DoF x root_scale (n_el = 1.49 n_root)
        r = int(name.split("_r")[1]) if "_r" in name else 3
        n = r + 1
        n_el = 1.0e8 * root_scale / (5 * n ** 3)
        nr = max(2, int(round((n_el / 1.49) ** (1.0 / 3.0))))
        ext = (10.0e3, 10.0e3, 10.0e3)
        mesh = build_uniform_mesh(ext, (nr, nr, nr), periodic=(True, True, True))
        pick = np.random.default_rng(5).random(mesh.n_leaves) < 0.07
        mesh = refine_region(mesh, lambda i, l, o, lo, hi: pick[i], 1, vectorized=True)
        geom = build_geometry(mesh, r)
        U0 = None
        if with_state:
            bg = project_initial_data(
                geom, hydrostatic_initial_state(HillCaseConfig(domain=ext))).data
            U0 = perturbed_state(bg, geom.node_coords, ext, 41)
        geom._memo.pop("nc", None)
        return BaselineCase(name, mesh, geom, model, [], None, U0, 0.3, dict(),
                            f"operator microbenchmark: periodic (10 km)^3, {nr}^3 roots, 7% "
                            f"refined once, r={r}")
    raise ConfigurationError(f"unknown baseline case {name!r}")


def _terrain_case(name, mesh, geom, model, hc, sponge_cfg, lateral, with_state, dt, desc):
    from .field import project_initial_data
    bg = project_initial_data(geom, hydrostatic_initial_state(hc)).data
    bcs = farfield_bcs(geom, bg)
    sigma = sponge_sigma(geom, sponge_cfg, mesh.extents, lateral_axes=lateral)
    geom._memo.pop("nc", None)   # node coordinates are no longer needed
    U0 = bg.copy() if with_state else None
    return BaselineCase(name, mesh, geom, model, bcs, (sigma, bg), U0, dt, dict(), desc)
