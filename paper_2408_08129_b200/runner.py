"""Drop-in run orchestration over the device path (orodg/runner.py:34-309,
orodg/config.py:15-80): ``setup_run(cfg)`` assembles a case from a preset,
``run(cfg)`` drives ``run_time_loop`` with the reference's per-step
diagnostics (mass, energy, max |w|, iteration counts, accumulated boundary
mass flux, probes) and block timer, and returns a ``RunResult``.

Presets: the reference's four (paper2d, paper3d-small, hydrostatic-rest,
manufactured -- same recipes and defaults as runner.py:34-43, 106-190) plus
the BASELINE.json configurations (``cfg1``..``cfg4``, ``cfg4w<n>`` windows,
``cfg5_r<r>``; cases.baseline_case), so a reference-style config object --
this module's ``CaseConfig`` or any object with the same fields, e.g.
orodg.config.CaseConfig -- drives the GPU path.  The diagnostics reduce on
the device (integrate_conserved, max_abs_ratio); only scalars cross to the
host.  VTK output is not part of this path; snapshots are
written as the reference's npz.
"""

import os
import time
from dataclasses import dataclass, field

import numpy as np

from . import cases
from .boundary import wall_everywhere
from .dgops import DGOperators, from_device, to_device
from .errors import ConfigurationError
from .field import StateField, project_initial_data
from .geometry import build_geometry
from .imex import ImplicitSolveConfig, PrecondCache, SplitOperators, ars222, imex_step, \
    run_time_loop
from .mesh import build_uniform_mesh, dump_mesh, refine_region
from .physics import FlowModel
from .timing import BlockTimer

REFERENCE_PRESETS = ("paper2d", "paper3d-small", "hydrostatic-rest", "manufactured")

_PRESET_DEFAULTS = {
    "paper2d": dict(t_final=3600.0, dt=2.0, root=(30, 8), refine=("all", "all"), u_bar=10.0,
                    sigma_max=0.05),
    "paper3d-small": dict(t_final=3600.0, dt=2.0, root=(15, 10, 4), refine=(), u_bar=10.0,
                          sigma_max=0.05),
    "hydrostatic-rest": dict(t_final=3600.0, dt=5.0, root=(60, 16), refine=(), u_bar=0.0,
                             sigma_max=0.0),
    "manufactured": dict(t_final=0.5, dt=0.01, root=(4, 4), refine=(), u_bar=0.0,
                         sigma_max=0.0),
}


def is_baseline_preset(name):
    return (name in ("cfg1", "cfg2", "cfg3", "cfg4") or name.startswith("cfg4w")
            or name.startswith("cfg5"))


@dataclass
class CaseConfig:
    """orodg.config.CaseConfig's fields (config.py:20-60); ``preset`` also
    accepts the BASELINE presets."""
    preset: str = "paper2d"
    t_final: float = None
    dt: float = None
    u_bar: float = None
    n_buoyancy: float = None
    sigma_max: float = None
    sponge_top_depth: float = None
    sponge_lateral_width: float = None
    degree: int = 4
    geom_degree: int = None
    quad_points: int = None
    root: tuple = None
    refine: tuple = ()
    fp_tol: float = 1e-6
    fp_max_iter: int = 10
    krylov_tol: float = 1e-8
    krylov_restart: int = 30
    krylov_max_iter: int = 1000
    preconditioner: str = "none"
    workers: int = 1
    chunk: int = 512
    output_dir: str = None
    output_every: int = 0
    diagnostics_every: int = 1
    seed: int = 0

    def validate(self):
        validate(self)
        return self

    def resolved_output_dir(self):
        return self.output_dir or os.environ.get("ORODG_OUTDIR", "orodg-out")


def validate(cfg):
    """config.py:62-86 for the reference presets; BASELINE presets carry
    their own discretisation."""
    if cfg.preset not in REFERENCE_PRESETS and not is_baseline_preset(cfg.preset):
        raise ConfigurationError(f"unknown preset {cfg.preset!r}; choose from "
                                 f"{REFERENCE_PRESETS} or a BASELINE preset (cfg1..cfg5_r<r>)")
    if cfg.degree < 1:
        raise ConfigurationError("degree must be >= 1")
    if cfg.dt is not None and cfg.dt <= 0:
        raise ConfigurationError(f"dt must be positive, got {cfg.dt}")
    if cfg.t_final is not None and cfg.t_final <= 0:
        raise ConfigurationError("t_final must be positive")
    for t in (cfg.fp_tol, cfg.krylov_tol):
        if not 0 < t < 1:
            raise ConfigurationError(f"tolerance {t} outside (0,1)")
    for n in (cfg.fp_max_iter, cfg.krylov_restart, cfg.krylov_max_iter):
        if n < 1:
            raise ConfigurationError("iteration settings must be >= 1")
    if cfg.preconditioner not in ("none", "block_jacobi"):
        raise ConfigurationError(f"unknown preconditioner {cfg.preconditioner!r}")
    if getattr(cfg, "output_every", 0) < 0 or getattr(cfg, "diagnostics_every", 1) < 0:
        raise ConfigurationError("output cadences must be >= 0")


def _preset(cfg, key):
    val = getattr(cfg, key, None)
    if val is None:
        return _PRESET_DEFAULTS.get(cfg.preset, {}).get(key)
    return val


def _parse_box(text, dim):
    parts = [p for p in text.split(",") if p.strip()]
    if len(parts) != dim:
        raise ConfigurationError(f"refine box {text!r} needs {dim} ranges 'lo:hi'")
    return [tuple(float(v) for v in p.split(":")) for p in parts]


def build_case_mesh(cfg, extents, periodic=None):
    """runner.py:65-81: root grid, then one refinement directive per level."""
    mesh = build_uniform_mesh(extents, _preset(cfg, "root"), periodic)
    dim = len(extents)
    for directive in (cfg.refine if cfg.refine else _PRESET_DEFAULTS[cfg.preset].get("refine", ())):
        if directive == "all":
            mesh = refine_region(mesh, lambda lf: True, 1)
        else:
            box = _parse_box(directive, dim)
            mesh = refine_region(mesh, lambda lf, box=box: all(
                lo <= lf.center[a] <= hi for a, (lo, hi) in enumerate(box)), 1)
    return mesh


def _solver_cfg(cfg):
    return ImplicitSolveConfig(fp_tol=cfg.fp_tol, fp_max_iter=cfg.fp_max_iter,
                               krylov_tol=cfg.krylov_tol, krylov_restart=cfg.krylov_restart,
                               krylov_max_iter=cfg.krylov_max_iter,
                               preconditioner=cfg.preconditioner)


@dataclass
class RunContext:
    config: object
    mesh: object
    geometry: object
    ops: DGOperators
    model: FlowModel
    split: SplitOperators
    initial: StateField
    solve_cfg: ImplicitSolveConfig
    timer: BlockTimer
    dt: float = None
    t_final: float = None
    background: np.ndarray = None
    exact_solution: object = None

    @property
    def dofs_per_variable(self):
        return self.mesh.n_leaves * self.geometry.basis.n_nodes


def setup_run(cfg, timer=None):
    """runner.py:106-190 on the device path (and the BASELINE presets)."""
    validate(cfg)
    timer = timer or BlockTimer()
    preset = cfg.preset
    if is_baseline_preset(preset):
        c = cases.baseline_case(preset)
        ops = DGOperators(c.geometry)
        split = SplitOperators(ops, c.model, c.bcs, c.sponge)
        solve = ImplicitSolveConfig(**{**dict(fp_tol=cfg.fp_tol, fp_max_iter=cfg.fp_max_iter,
                                              krylov_tol=cfg.krylov_tol,
                                              krylov_restart=cfg.krylov_restart,
                                              krylov_max_iter=cfg.krylov_max_iter,
                                              preconditioner=cfg.preconditioner), **c.solve})
        initial = StateField(c.U0, c.mesh.fingerprint, c.geometry.basis.degree)
        return RunContext(cfg, c.mesh, c.geometry, ops, c.model, split, initial, solve, timer,
                          dt=cfg.dt or c.dt, t_final=cfg.t_final or 10 * (cfg.dt or c.dt),
                          background=c.sponge[1] if c.sponge else None)
    dt, t_final = _preset(cfg, "dt"), _preset(cfg, "t_final")
    if preset in ("paper2d", "paper3d-small"):
        dim = 2 if preset == "paper2d" else 3
        domain = (60.0e3, 16.0e3) if dim == 2 else (60.0e3, 40.0e3, 16.0e3)
        hc = cases.HillCaseConfig(domain=domain)
        from dataclasses import replace
        if _preset(cfg, "u_bar") is not None:
            hc = replace(hc, u_bar=_preset(cfg, "u_bar"))
        if _preset(cfg, "n_buoyancy") is not None:
            hc = replace(hc, N_buoyancy=_preset(cfg, "n_buoyancy"))
        mesh = build_case_mesh(cfg, domain)
        terrain = ((lambda x: cases.hill_profile(x, None, hc)) if dim == 2
                   else (lambda x, y: cases.hill_profile(x, y, hc)))
        geometry = build_geometry(mesh, cfg.degree, terrain=terrain, geom_degree=cfg.geom_degree,
                                  n_quad_1d=cfg.quad_points)
        ops = DGOperators(geometry)
        model = FlowModel.dimensional(hc.constants)
        initial = project_initial_data(geometry, cases.hydrostatic_initial_state(hc))
        background = initial.data.copy()
        bcs = cases.farfield_bcs(geometry, background)
        sp = cases.SpongeConfig(
            top_depth=_preset(cfg, "sponge_top_depth") or 4.0e3,
            lateral_width=_preset(cfg, "sponge_lateral_width") or 10.0e3,
            sigma_max=(_preset(cfg, "sigma_max") if _preset(cfg, "sigma_max") is not None
                       else 0.05))
        sigma = cases.sponge_sigma(geometry, sp, domain, lateral_axes=tuple(range(dim - 1)))
        sponge = (sigma, background) if sp.sigma_max > 0 else None
        split = SplitOperators(ops, model, bcs, sponge=sponge)
        return RunContext(cfg, mesh, geometry, ops, model, split, initial, _solver_cfg(cfg),
                          timer, dt, t_final, background=background)
    if preset == "hydrostatic-rest":
        domain = (60.0e3, 16.0e3)
        hc = cases.HillCaseConfig(domain=domain, u_bar=_preset(cfg, "u_bar") or 0.0)
        if _preset(cfg, "n_buoyancy") is not None:
            from dataclasses import replace
            hc = replace(hc, N_buoyancy=_preset(cfg, "n_buoyancy"))
        mesh = build_case_mesh(cfg, domain)
        geometry = build_geometry(mesh, cfg.degree, geom_degree=cfg.geom_degree,
                                  n_quad_1d=cfg.quad_points)
        ops = DGOperators(geometry)
        model = FlowModel.dimensional(hc.constants)
        initial = project_initial_data(geometry, cases.hydrostatic_initial_state(hc))
        split = SplitOperators(ops, model, wall_everywhere(mesh))
        return RunContext(cfg, mesh, geometry, ops, model, split, initial, _solver_cfg(cfg),
                          timer, dt, t_final, background=initial.data.copy())
    # manufactured: gravity-free periodic unit box with analytic forcing
    mesh = build_case_mesh(cfg, (1.0, 1.0), periodic=(True, True))
    geometry = build_geometry(mesh, cfg.degree, n_quad_1d=cfg.quad_points)
    ops = DGOperators(geometry)
    model = FlowModel(gravity=0.0)
    mcfg = cases.ManufacturedConfig()
    coords = geometry.node_coords

    def forcing(t):
        return np.moveaxis(cases.manufactured_forcing(coords, t, mcfg), 2, 1)

    split = SplitOperators(ops, model, bcs=None, forcing=forcing)
    initial = project_initial_data(geometry, lambda c: cases.manufactured_state(c, 0.0, mcfg))
    return RunContext(cfg, mesh, geometry, ops, model, split, initial, _solver_cfg(cfg), timer,
                      dt, t_final,
                      exact_solution=lambda t, c: cases.manufactured_state(c, t, mcfg))


@dataclass
class RunResult:
    config: object
    final: StateField
    diagnostics: list
    timer_report: object
    wall_time: float
    output_dir: str
    context: RunContext
    steps: int = 0

    @property
    def diagnostics_text(self):
        return "\n".join(self.diagnostics) + "\n"


def _fmt(x):
    return repr(float(x))


def save_snapshot(path, ctx, data, t):
    """runner.py:304-309's npz snapshot (host copy of the device state)."""
    data = data.cpu().numpy() if hasattr(data, "cpu") else np.asarray(data)
    np.savez_compressed(path, data=data, t=t, degree=ctx.geometry.basis.degree,
                        mesh_dump=dump_mesh(ctx.mesh), preset=ctx.config.preset)


def run(cfg, probes=(), write_outputs=False, max_steps=None):
    """runner.py:217-300 on the device path.  The state stays on the GPU for
    the whole loop; every diagnostics row is a handful of device reductions.
    probes: (name, node_mask) pairs -> max |w| over the masked nodes.
    max_steps: optional cap on the number of steps (smoke runs)."""
    t_wall0 = time.perf_counter()
    ctx = setup_run(cfg)
    if ctx.dt is None or ctx.t_final is None:
        raise ConfigurationError("dt and t_final must be set")
    tab = ars222()
    d = ctx.mesh.dim
    ops = ctx.ops
    rows = ["step,t,mass,energy,max_w,fp_iters,krylov_iters,mass_flux_accum"
            + "".join(f",max_w_{name}" for name, _ in probes)]
    accum = [0.0]
    last_h = [ctx.dt]
    every = getattr(cfg, "diagnostics_every", 1)

    def diagnostics_cb(step, t, data, stats):
        if stats is not None:
            accum[0] += stats.mass_rate * last_h[0]
        if every and step % every == 0:
            totals = ops.integrate_conserved(data)
            fp = sum(stats.fp_iters) if stats else 0
            kry = sum(stats.krylov_iters) if stats else 0
            row = [str(step), _fmt(t), _fmt(totals[0]), _fmt(totals[d + 1]),
                   _fmt(ops.max_abs_ratio(data, d, 0)), str(fp), str(kry), _fmt(accum[0])]
            for _, mask in probes:
                row.append(_fmt(ops.max_abs_ratio(data, d, 0, mask) if np.any(mask) else 0.0))
            rows.append(",".join(row))

    outdir = cfg.resolved_output_dir() if hasattr(cfg, "resolved_output_dir") else "orodg-out"

    def output_cb(step, t, data, stats):
        oe = getattr(cfg, "output_every", 0)
        if write_outputs and oe and step % oe == 0:
            save_snapshot(os.path.join(outdir, f"snapshot-{step:06d}.npz"), ctx, data, t)

    precond = PrecondCache()
    n_done = [0]

    def stepper(data, t, h):
        last_h[0] = h
        n_done[0] += 1
        return imex_step(data, t, h, tab, ctx.split, ctx.solve_cfg, timer=ctx.timer,
                         precond=precond)

    t_final = ctx.t_final if max_steps is None else min(ctx.t_final, max_steps * ctx.dt)
    U0, _ = to_device(ctx.initial.data, ops.context())
    if write_outputs:
        os.makedirs(outdir, exist_ok=True)
    final, report = run_time_loop(U0.clone(), ctx.dt, t_final, stepper,
                                  callbacks=(diagnostics_cb, output_cb), timer=ctx.timer)
    if write_outputs:
        with open(os.path.join(outdir, "diagnostics.csv"), "w") as f:
            f.write("\n".join(rows) + "\n")
        with open(os.path.join(outdir, "timings.csv"), "w") as f:
            f.write(report.csv_header() + "\n" + "\n".join(report.csv_rows()) + "\n")
            f.write(f"total,{report.total:.9f}\n")
        save_snapshot(os.path.join(outdir, "final.npz"), ctx, final, t_final)
    final_h = from_device(final, True)
    return RunResult(cfg, StateField(final_h, ctx.initial.mesh_id, ctx.geometry.basis.degree),
                     rows, report, time.perf_counter() - t_wall0, outdir, ctx, n_done[0])
