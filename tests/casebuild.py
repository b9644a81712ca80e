"""Rebuild the golden-fixture cases from the package's host input builders.

Mirrors tests/golden/make_golden.py case by case (same meshes, degrees,
terrain, background, sponge, BCs), but through paper_2408_08129_b200 only,
so it runs on the GPU box where the reference tree does not exist.
"""

import functools
import os

import numpy as np

from paper_2408_08129_b200 import cases
from paper_2408_08129_b200.boundary import wall_everywhere
from paper_2408_08129_b200.field import project_initial_data
from paper_2408_08129_b200.geometry import build_geometry
from paper_2408_08129_b200.mesh import build_uniform_mesh, refine_region
from paper_2408_08129_b200.physics import FlowModel

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


@functools.lru_cache(maxsize=None)
def golden(name):
    return dict(np.load(os.path.join(GOLDEN, f"{name}.npz")))


def hill2d(x):
    return 400.0 / (1.0 + ((x - 30.0e3) / 1.0e3) ** 2) ** 1.5


def hill3d(x, y):
    return 400.0 / (1.0 + ((x - 10.0e3) / 1.0e3) ** 2
                    + ((y - 10.0e3) / 1.0e3) ** 2) ** 1.5


class Case:
    """mesh, geometry, model, bcs, sponge, U (state) of one fixture case."""

    def __init__(self, name, mesh, geom, bcs, sponge, U, a_dt, krylov_tol=1e-8,
                 dt=None):
        self.name = name
        self.mesh = mesh
        self.geom = geom
        self.model = FlowModel.dimensional()
        self.bcs = bcs
        self.sponge = sponge
        self.U = U
        self.a_dt = a_dt
        self.krylov_tol = krylov_tol
        self.dt = dt


def _bubble(name, root, refine_below, degree, tol):
    mesh = build_uniform_mesh((20.0e3, 10.0e3), root)
    if refine_below is not None:
        mesh = refine_region(mesh, lambda lf: lf.center[1] < refine_below, 1)
    geom = build_geometry(mesh, degree)
    U = project_initial_data(geom, cases.warm_bubble_state()).data
    return Case(name, mesh, geom, wall_everywhere(mesh), None, U,
                0.5 * (1.0 - 1.0 / np.sqrt(2.0)), tol, dt=0.5)


def _terrain(name, mesh, degree, terrain, ext, sponge_cfg, lateral, seed, a_dt,
             hill_cfg=None, perturb=True, dt=None):
    geom = build_geometry(mesh, degree, terrain=terrain)
    hc = hill_cfg or cases.HillCaseConfig(domain=ext)
    bg = project_initial_data(geom, cases.hydrostatic_initial_state(hc)).data
    U = cases.perturbed_state(bg, geom.node_coords, ext, seed) if perturb else bg.copy()
    bcs = cases.farfield_bcs(geom, bg)
    sigma = cases.sponge_sigma(geom, sponge_cfg, ext, lateral_axes=lateral)
    c = Case(name, mesh, geom, bcs, (sigma, bg), U, a_dt, dt=dt)
    c.background = bg
    return c


@functools.lru_cache(maxsize=None)
def build(name):
    if name == "cfg1":
        return _bubble("cfg1", (32, 16), None, 2, 1e-8)
    if name == "cfg2":
        return _bubble("cfg2", (64, 32), 5.0e3, 4, 1e-10)
    if name == "bjh":  # golden bj.npz, prefix h_: once-refined bubble, hanging faces
        return _bubble("bjh", (16, 8), 5.0e3, 2, 1e-8)
    if name == "hang2d":
        ext = (60.0e3, 16.0e3)
        m = build_uniform_mesh(ext, (15, 4))
        m = refine_region(m, lambda lf: abs(lf.center[0] - 30.0e3) < 6.0e3
                          and lf.center[1] < 6.0e3, times=2)
        return _terrain(name, m, 4, hill2d, ext, cases.SpongeConfig(), (0,), 21, 0.3)
    if name == "hang3d":
        ext = (20.0e3, 20.0e3, 10.0e3)
        m = build_uniform_mesh(ext, (4, 4, 2))
        m = refine_region(m, lambda lf: bool(np.all(np.abs(lf.center[:2] - 10.0e3) < 5.0e3)
                                             and lf.center[2] < 5.0e3), times=1)
        return _terrain(name, m, 3, hill3d, ext,
                        cases.SpongeConfig(top_depth=4.0e3, lateral_width=5.0e3),
                        (0, 1), 31, 0.3, dt=0.5)
    if name == "hang3d_r4":
        ext = (20.0e3, 20.0e3, 10.0e3)
        m = build_uniform_mesh(ext, (4, 4, 2))
        m = refine_region(m, lambda lf: bool(np.all(np.abs(lf.center[:2] - 10.0e3) < 5.0e3)
                                             and lf.center[2] < 5.0e3), times=1)
        return _terrain(name, m, 4, hill3d, ext,
                        cases.SpongeConfig(top_depth=4.0e3, lateral_width=5.0e3),
                        (0, 1), 37, 0.3, dt=0.5)
    if name in ("per3d", "per3d_r4", "cfg5s"):
        ext = (10.0e3, 10.0e3, 10.0e3)
        root, pseed, frac, deg, useed = {
            "per3d": (4, 5, 0.3, 2, 41), "per3d_r4": (3, 7, 0.3, 4, 43),
            "cfg5s": (6, 5, 0.07, 3, 41)}[name]
        m = build_uniform_mesh(ext, (root,) * 3, periodic=(True, True, True))
        pick = np.random.default_rng(pseed).random(m.n_leaves) < frac
        m = refine_region(m, lambda lf: bool(pick[lf.index]), 1)
        geom = build_geometry(m, deg)
        bg = project_initial_data(
            geom, cases.hydrostatic_initial_state(cases.HillCaseConfig(domain=ext))).data
        U = cases.perturbed_state(bg, geom.node_coords, ext, useed)
        return Case(name, m, geom, [], None, U, 0.3)
    if name == "cfg3s":
        ext = (50.0e3, 21.0e3)
        m = build_uniform_mesh(ext, (25, 8))
        m = refine_region(m, lambda lf: lf.center[1] < 6.0e3, 1)
        m = refine_region(m, lambda lf: lf.center[1] < 2.5e3, 1)
        return _terrain(name, m, 4, cases.schar_terrain(), ext,
                        cases.SpongeConfig(top_depth=9.0e3, lateral_width=10.0e3), (0,),
                        51, 0.5, hill_cfg=cases.HillCaseConfig(domain=ext, T_ref=280.0),
                        perturb=False, dt=1.0)
    raise KeyError(name)


def rel(a, b, floor=0.0):
    a = np.asarray(a, dtype=float)
    b = np.asarray(b, dtype=float)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), floor, 1e-300))


def per_var_rel(a, b, floor_frac=1e-6):
    """Per-variable relative L2 with a floor for ~0 variables."""
    a = np.asarray(a)
    b = np.asarray(b)
    tot = np.linalg.norm(b)
    return [float(np.linalg.norm(a[:, v] - b[:, v])
                  / max(np.linalg.norm(b[:, v]), floor_frac * tot, 1e-300))
            for v in range(b.shape[1])]


def parity_tols(z, key, floor=1e-12, factor=10.0):
    """Per-variable gate max(1e-12, 10 x the reference's own 1-ulp input
    sensitivity) (make_golden.noise_record)."""
    nk = "noise_" + key
    if nk not in z:
        return None
    return np.maximum(floor, factor * np.asarray(z[nk]))


# achieved errors of every parity check of the session, written by
# conftest.pytest_sessionfinish to $DG_PARITY_LOG (profiles/r2_parity.json)
PARITY_LOG = []


def record(case, key, errs, tols, **extra):
    import os as _os
    rec = {"test": _os.environ.get("PYTEST_CURRENT_TEST", "").split(" ")[0], "case": case,
           "key": key, "err": [float(e) for e in np.atleast_1d(errs)],
           "tol": [float(t) for t in np.atleast_1d(tols)]}
    rec.update(extra)
    PARITY_LOG.append(rec)


def assert_parity(got, z, key, floor=1e-12, factor=10.0):
    ref = z[key]
    got = np.asarray(got)
    if ref.ndim == 2 and got.ndim == 2 and key in ("Fx", "helm_x", "F0"):
        got, ref = got[:, None], ref[:, None]
    errs = np.array(per_var_rel(got.reshape(ref.shape), ref))
    tols = parity_tols(z, key, floor, factor)
    if tols is None:
        tols = np.full(len(errs), floor)
    record(str(z.get("case", "?")), key, errs, tols)
    assert np.all(errs <= tols), f"{key}: per-var err {errs} > tol {tols}"
    return errs


def check_rel(case, key, got, ref, tol, floor=0.0):
    """Whole-array relative L2 gate, logged with its achieved value."""
    e = rel(got, ref, floor)
    record(case, key, [e], [tol])
    assert e <= tol, f"{case} {key}: rel err {e:.3e} > {tol:.1e}"
    return e
