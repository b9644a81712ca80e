"""Generate the golden parity fixtures by running the REFERENCE solver.

Run only in the build container (it imports the read-only reference package
from /root/reference/pkg/src); the GPU box never runs this.  Outputs are the
committed ``tests/golden/*.npz`` files, one per case.

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py [case ...]

Cases (inputs built only through the reference's public API):

  cfg1     BASELINE configs[0]: warm bubble 20x10 km, 32x16, r=2, walls,
           ARS(2,2,2), dt=0.5 s, 10 steps
  cfg2     BASELINE configs[1]: same bubble on 64x32 with z<5 km refined
           once, r=4, krylov_tol=1e-10, 200 steps (slow: ~6-10 min)
  hang2d   2D Gal-Chen terrain (bell hill), two refinement levels, far-field
           + bottom wall, Rayleigh sponge, r=4 (the reference conftest mesh)
  hang3d   3D terrain + hanging + far-field + sponge, r=3 (conftest mesh)
  per3d    3D triply-periodic box, seeded once-refined cells, r=2 (cfg5 recipe
           at toy size)
  cfg3s    scaled-down Schar case (terrain, sponge, far-field, 2 refinement
           levels near the ground), r=4, 3 steps
  part     partition_leaves on the cfg2 mesh, P=1..8, unit and seeded weights
  hang3d_r4  hang3d's mesh at r=4 (25-lane elements on the device)
  per3d_r4   periodic seeded-refined box at r=4
  cfg5s    BASELINE configs[4] recipe at 6^3 roots, r=3
  dropin   implicit/full residual, forced step, subset mass inverse, host
           gmres with restart 40

Warm-bubble recipe (harness choice, recorded here and mirrored by
paper_2408_08129_b200.cases.warm_bubble_state): constant theta0 = 300 K
background with Exner pi = 1 - g z/(c_p theta0), p = p0 pi^(c_p/R), p0 = 1e5;
theta' = 2 K cos^2(pi r / (2 rc)) for r < rc = 2 km around (10 km, 2 km);
rho = p / (R theta pi); u = 0; rhoE = p/(gamma-1).
"""

import os
import sys
import time

for _v in ("OMP_NUM_THREADS", "OPENBLAS_NUM_THREADS", "MKL_NUM_THREADS"):
    os.environ.setdefault(_v, "1")

import numpy as np

REF = "/root/reference/pkg/src"
if REF not in sys.path:
    sys.path.insert(0, REF)

import orodg  # noqa: E402
from orodg import cases, imex, krylov  # noqa: E402
from orodg.boundary import wall_everywhere  # noqa: E402
from orodg.dgops import DGOperators  # noqa: E402
from orodg.field import project_initial_data  # noqa: E402
from orodg.geometry import build_geometry  # noqa: E402
from orodg.mesh import build_uniform_mesh, refine_region  # noqa: E402
from orodg.partition import partition_leaves  # noqa: E402
from orodg.physics import CONST, FlowModel  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


# ----------------------------------------------------------------- inputs

def warm_bubble(cfg_d=2, theta0=300.0, dtheta=2.0, xc=10.0e3, zc=2.0e3,
                rc=2.0e3, p0=1.0e5):
    R, g, gam = CONST.R, CONST.g, CONST.gamma
    cp = R * gam / (gam - 1.0)

    def f(coords):
        x = coords[..., 0]
        z = coords[..., -1]
        exner = 1.0 - g * z / (cp * theta0)
        p = p0 * exner ** (cp / R)
        r = np.sqrt((x - xc) ** 2 + (z - zc) ** 2)
        bump = np.where(r < rc, dtheta * np.cos(0.5 * np.pi * r / rc) ** 2, 0.0)
        theta = theta0 + bump
        rho = p / (R * theta * exner)
        out = np.zeros(coords.shape[:-1] + (cfg_d + 2,))
        out[..., 0] = rho
        out[..., cfg_d + 1] = p / (gam - 1.0)
        return out

    return f


def smooth_noise(coords, extents, rng, n_modes=8, kmax=4):
    """Sum of seeded sines (SURVEY.md §8d cfg5 perturbation recipe)."""
    d = coords.shape[-1]
    s = np.zeros(coords.shape[:-1])
    for _ in range(n_modes):
        k = rng.integers(1, kmax + 1, size=d)
        a = rng.normal() / 8.0
        phi = rng.uniform(0.0, 2.0 * np.pi)
        arg = phi + sum(2.0 * np.pi * k[i] * coords[..., i] / extents[i]
                        for i in range(d))
        s += a * np.sin(arg)
    return s


def perturbed(background, coords, extents, seed, u_scale=10.0):
    """rho(1+1e-3 s), m += rho*1e-3*u_scale*s_a, rhoE(1+1e-3 s)."""
    rng = np.random.default_rng(seed)
    U = background.copy()
    d = coords.shape[-1]
    s_rho = smooth_noise(coords, extents, rng)
    U[:, 0] *= 1.0 + 1e-3 * s_rho
    for a in range(d):
        s_a = smooth_noise(coords, extents, rng)
        U[:, 1 + a] = U[:, 1 + a] / background[:, 0] * U[:, 0] \
            + U[:, 0] * 1e-3 * u_scale * s_a
    s_e = smooth_noise(coords, extents, rng)
    U[:, d + 1] *= 1.0 + 1e-3 * s_e
    return U


def energy_like(U, seed):
    d = U.shape[1] - 2
    rng = np.random.default_rng(seed)
    return U[:, d + 1] * (1.0 + 1e-3 * rng.standard_normal(U[:, d + 1].shape))


def hill2d(x):
    return 400.0 / (1.0 + ((x - 30.0e3) / 1.0e3) ** 2) ** 1.5


def hill3d(x, y):
    return 400.0 / (1.0 + ((x - 10.0e3) / 1.0e3) ** 2
                    + ((y - 10.0e3) / 1.0e3) ** 2) ** 1.5


def schar(x):
    xs = x - 25.0e3
    return 250.0 * np.exp(-(xs / 5.0e3) ** 2) * np.cos(np.pi * xs / 4.0e3) ** 2


# ------------------------------------------------------------- recording

def mesh_record(mesh, prefix="mesh_"):
    rec = {}
    lv = np.array([l for l, _ in mesh.leaves], dtype=np.int64)
    org = np.array([o for _, o in mesh.leaves], dtype=np.int64)
    rec[prefix + "levels"] = lv
    rec[prefix + "origins"] = org
    rec[prefix + "extents"] = np.array(mesh.extents)
    rec[prefix + "root"] = np.array(mesh.root_counts)
    rec[prefix + "periodic"] = np.array(mesh.periodic, dtype=np.int64)
    topo = mesh.topology
    rec[prefix + "conf_axis"] = np.array([b.axis for b in topo.conforming], dtype=np.int64)
    for i, b in enumerate(topo.conforming):
        rec[f"{prefix}conf{i}_left"] = b.left
        rec[f"{prefix}conf{i}_right"] = b.right
    rec[prefix + "hang_axis_orient"] = np.array(
        [[b.axis, b.orient] for b in topo.hanging], dtype=np.int64).reshape(-1, 2)
    for i, b in enumerate(topo.hanging):
        rec[f"{prefix}hang{i}_coarse"] = b.coarse
        rec[f"{prefix}hang{i}_fine"] = b.fine
        rec[f"{prefix}hang{i}_subface"] = b.subface
    rec[prefix + "bdry_axis_side"] = np.array(
        [[b.axis, b.side] for b in topo.boundary], dtype=np.int64).reshape(-1, 2)
    for i, b in enumerate(topo.boundary):
        rec[f"{prefix}bdry{i}_leaves"] = b.leaves
    rec[prefix + "fingerprint"] = np.array(mesh.fingerprint)
    return rec


def geometry_record(geom):
    rec = {"geo_det_j": geom.det_j, "geo_ctrv": geom.ctrv,
           "geo_mass_h_inv": geom.mass_h_inv, "geo_mass_v_inv": geom.mass_v_inv,
           "geo_node_coords": geom.node_coords}
    for name, lst in (("conf", geom.conforming), ("hang", geom.hanging),
                      ("bdry", geom.boundary)):
        for i, fg in enumerate(lst):
            rec[f"geo_{name}{i}_normal"] = fg.normal
            rec[f"geo_{name}{i}_ws"] = fg.ws
    return rec


def operator_record(ops, split, U, model, bcs, seed, a_dt):
    """Every hot-path operator once, on U (and energy-like x)."""
    geom = ops.geometry
    d = ops.dim
    rec = {"U": U}
    t0 = time.perf_counter()
    dual_adv = ops.divergence_advective(U, model, bcs)
    rec["dual_adv"] = dual_adv
    rec["minv_dual_adv"] = geom.apply_mass_inverse(dual_adv)
    R = split.explicit_residual(U, 0.0)
    rec["explicit_residual"] = R
    rec["mass_rate"] = np.array(split._last_mass_rate)
    W = orodg.conserved_to_primitive(U, model, var_axis=1, check=False)
    rec["grad_dual"] = ops.gradient_scalar(W.p, model, bcs)
    h, K = split.frozen_coefficients(U)
    rec["frozen_h"], rec["frozen_K"] = h, K
    rec["divhv_dual"] = ops.divergence_hv(U[:, 1:1 + d], h, model, bcs)
    rec["divhv_prepared_dual"] = ops.prepare_divergence_hv(h, model, bcs)(U[:, 1:1 + d])
    x = energy_like(U, seed)
    rec["x"] = x
    rec["a_dt"] = np.array(a_dt)
    m_e = U[:, 1:1 + d].copy()
    e_e = U[:, 1 + d].copy()
    F, grad_p = split.energy_affine_map(a_dt, h, K, m_e, e_e)
    rec["F0"] = F(np.zeros_like(x))
    rec["Fx"] = F(x)
    rec["grad_p_x"] = grad_p(x)
    action = imex.build_helmholtz_action(split, a_dt, U)
    rec["helm_x"] = action(x.ravel()).reshape(x.shape)
    # linear composition (no cancellation noise): x + a_dt Minv Div_lin(V),
    # V = -(a_dt/M^2)(gamma-1) Minv G_lin(x)   (imex.py:207-216)
    rec["integrate_conserved"] = ops.integrate_conserved(U)
    rec.update(noise_record(ops, split, U, model, bcs, x, a_dt, rec))
    rec["inner_UU"] = np.array(ops.global_inner_product(U, U))
    rec["op_seconds"] = np.array(time.perf_counter() - t0)
    return rec


def _per_var_noise(a, b):
    tot = np.linalg.norm(b)
    return np.array([np.linalg.norm(a[:, v] - b[:, v])
                     / max(np.linalg.norm(b[:, v]), 1e-6 * tot, 1e-300)
                     for v in range(b.shape[1])])


def noise_record(ops, split, U, model, bcs, x, a_dt, rec):
    """The reference's own rounding sensitivity: every output recomputed on
    inputs perturbed by one ulp (relative 2^-52, random sign).  Parity gates
    per variable are max(1e-12, 10 x this noise) -- a floor no
    implementation with a different summation order can beat."""
    d = ops.dim
    rng = np.random.default_rng(1234)
    ulp = 2.0 ** -52
    Up = U * (1.0 + ulp * rng.choice([-1.0, 1.0], size=U.shape))
    xp = x * (1.0 + ulp * rng.choice([-1.0, 1.0], size=x.shape))
    out = {}
    out["noise_dual_adv"] = _per_var_noise(ops.divergence_advective(Up, model, bcs),
                                           rec["dual_adv"])
    out["noise_explicit_residual"] = _per_var_noise(split.explicit_residual(Up, 0.0),
                                                    rec["explicit_residual"])
    Wp = orodg.conserved_to_primitive(Up, model, var_axis=1, check=False)
    out["noise_grad_dual"] = _per_var_noise(ops.gradient_scalar(Wp.p, model, bcs),
                                            rec["grad_dual"])
    hp, Kp = split.frozen_coefficients(Up)
    out["noise_divhv_dual"] = _per_var_noise(
        ops.divergence_hv(Up[:, 1:1 + d], hp, model, bcs), rec["divhv_dual"])
    h, K = split.frozen_coefficients(U)
    F, grad_p = split.energy_affine_map(a_dt, h, K, U[:, 1:1 + d].copy(),
                                        U[:, 1 + d].copy())
    out["noise_Fx"] = _per_var_noise(F(xp)[:, None], rec["Fx"][:, None])
    out["noise_grad_p_x"] = _per_var_noise(grad_p(xp), rec["grad_p_x"])
    action = imex.build_helmholtz_action(split, a_dt, U)
    out["noise_helm_x"] = _per_var_noise(action(xp.ravel()).reshape(x.shape)[:, None],
                                         rec["helm_x"][:, None])
    return out


def gmres_record(split, U, a_dt, tol, seed):
    """One standalone Helmholtz GMRES solve (krylov.py:27-115)."""
    d = split.dim
    h, K = split.frozen_coefficients(U)
    m_e = U[:, 1:1 + d].copy()
    e_e = U[:, 1 + d].copy()
    F, _ = split.energy_affine_map(a_dt, h, K, m_e, e_e)
    F0 = F(np.zeros_like(e_e))
    action = imex.build_helmholtz_action(split, a_dt, U)
    x0 = energy_like(U, seed + 1).ravel()
    x, st = krylov.gmres(action, F0.ravel(), x0=x0, tol_rel=tol, restart=30,
                         max_iter=1000)
    return {"gm_rhs": F0, "gm_x0": x0.reshape(e_e.shape), "gm_x": x.reshape(e_e.shape),
            "gm_iters": np.array(st.iterations), "gm_restarts": np.array(st.restarts),
            "gm_residual": np.array(st.residual),
            "gm_history": np.array(st.residual_history), "gm_tol": np.array(tol)}


def steps_record(split, U0, dt, n_steps, solve_cfg, keep_every=None):
    tab = imex.ars222()
    U = U0.copy()
    rec = {"dt": np.array(dt), "n_steps": np.array(n_steps)}
    fp, kr, inc, mr = [], [], [], []
    t = 0.0
    t0 = time.perf_counter()
    snaps = {}
    for s in range(1, n_steps + 1):
        U, st = imex.imex_step(U, t, dt, tab, split, solve_cfg)
        t = s * dt
        fp.append(st.fp_iters)
        kr.append(st.krylov_iters)
        inc.append(st.pressure_increments)
        mr.append(st.mass_rate)
        if s == 1:
            snaps["U_step1"] = U.copy()
        if keep_every and s % keep_every == 0:
            snaps[f"U_step{s}"] = U.copy()
        print(f"  step {s}: fp {st.fp_iters} krylov {st.krylov_iters}", flush=True)
    rec["step_seconds"] = np.array((time.perf_counter() - t0) / n_steps)
    rec["U_final"] = U
    rec.update(snaps)
    rec["fp_iters"] = _ragged(fp)
    rec["krylov_iters"] = _ragged(kr)
    rec["pressure_increments"] = _ragged(inc, float)
    rec["mass_rate_steps"] = np.array(mr)
    return rec


def _ragged(lists, dtype=np.int64):
    width = max(len(x) for x in lists)
    out = np.full((len(lists), width), -1 if dtype is np.int64 else np.nan,
                  dtype=dtype)
    for i, x in enumerate(lists):
        out[i, :len(x)] = x
    return out


def save(name, rec):
    path = os.path.join(OUT, f"{name}.npz")
    np.savez_compressed(path, **rec)
    print(f"wrote {path} ({os.path.getsize(path) / 1e6:.2f} MB)")


# ----------------------------------------------------------------- cases

def bubble_case(root, refine_below=None, degree=2):
    mesh = build_uniform_mesh((20.0e3, 10.0e3), root)
    if refine_below is not None:
        mesh = refine_region(mesh, lambda lf: lf.center[1] < refine_below, 1)
    geom = build_geometry(mesh, degree)
    ops = DGOperators(geom)
    model = FlowModel.dimensional()
    U0 = project_initial_data(geom, warm_bubble()).data
    bcs = wall_everywhere(mesh)
    split = imex.SplitOperators(ops, model, bcs)
    return mesh, geom, ops, model, U0, bcs, split


def case_cfg1():
    mesh, geom, ops, model, U0, bcs, split = bubble_case((32, 16), None, 2)
    dt = 0.5
    a_dt = dt * (1.0 - 1.0 / np.sqrt(2.0))
    rec = {"case": np.array("cfg1"), "degree": np.array(2)}
    rec.update(mesh_record(mesh))
    rec.update(geometry_record(geom))
    rec.update(operator_record(ops, split, U0, model, bcs, 11, a_dt))
    rec.update(gmres_record(split, U0, a_dt, 1e-8, 11))
    # one implicit stage exactly as imex_step stage 1 forms it
    scfg = imex.ImplicitSolveConfig()
    KE0 = split.explicit_residual(U0, 0.0)
    acc = U0 + (dt * (1.0 - 1.0 / np.sqrt(2.0))) * KE0
    stats = imex.StepStats()
    it, nfp = imex._solve_implicit_stage(acc, U0, a_dt, split, scfg, stats,
                                         orodg.timing.NullTimer(), None)
    rec.update({"stage_acc": acc, "stage_iterate": it, "stage_fp": np.array(nfp),
                "stage_krylov": np.array(stats.krylov_iters),
                "stage_incs": np.array(stats.pressure_increments)})
    rec.update(steps_record(split, U0, dt, 10, scfg))
    save("cfg1", rec)


def case_cfg2(n_steps=200):
    mesh, geom, ops, model, U0, bcs, split = bubble_case((64, 32), 5.0e3, 4)
    dt = 0.5
    a_dt = dt * (1.0 - 1.0 / np.sqrt(2.0))
    rec = {"case": np.array("cfg2"), "degree": np.array(4)}
    rec.update(mesh_record(mesh))
    rec.update(operator_record(ops, split, U0, model, bcs, 12, a_dt))
    rec.update(gmres_record(split, U0, a_dt, 1e-10, 12))
    scfg = imex.ImplicitSolveConfig(krylov_tol=1e-10)
    rec.update(steps_record(split, U0, dt, n_steps, scfg, keep_every=10))
    save("cfg2", rec)


def _terrain_case(mesh, degree, terrain, hill_cfg, sponge_cfg, lateral_axes,
                  seed, extents):
    geom = build_geometry(mesh, degree, terrain=terrain)
    ops = DGOperators(geom)
    model = FlowModel.dimensional()
    bg = project_initial_data(geom, cases.hydrostatic_initial_state(hill_cfg)).data
    U = perturbed(bg, geom.node_coords, extents, seed)
    bcs = cases.farfield_bcs(geom, bg)
    sigma = cases.sponge_sigma(geom, sponge_cfg, extents, lateral_axes=lateral_axes)
    split = imex.SplitOperators(ops, model, bcs, sponge=(sigma, bg))
    return geom, ops, model, bg, U, bcs, split, sigma


def case_hang2d():
    ext = (60.0e3, 16.0e3)
    m = build_uniform_mesh(ext, (15, 4))
    mesh = refine_region(
        m, lambda lf: abs(lf.center[0] - 30.0e3) < 6.0e3 and lf.center[1] < 6.0e3,
        times=2)
    hill_cfg = cases.HillCaseConfig(domain=ext)
    geom, ops, model, bg, U, bcs, split, sigma = _terrain_case(
        mesh, 4, hill2d, hill_cfg, cases.SpongeConfig(), (0,), 21, ext)
    rec = {"case": np.array("hang2d"), "degree": np.array(4),
           "background": bg, "sigma": sigma}
    rec.update(mesh_record(mesh))
    rec.update(geometry_record(geom))
    rec.update(operator_record(ops, split, U, model, bcs, 21, 0.3))
    for i, bc in enumerate(bcs):
        if bc.kind == "farfield":
            rec[f"bc{i}_ghost"] = bc.ghost_conserved
    rec.update(gmres_record(split, U, 0.3, 1e-8, 21))
    save("hang2d", rec)


def case_hang3d():
    ext = (20.0e3, 20.0e3, 10.0e3)
    m = build_uniform_mesh(ext, (4, 4, 2))
    mesh = refine_region(
        m, lambda lf: bool(np.all(np.abs(lf.center[:2] - 10.0e3) < 5.0e3)
                           and lf.center[2] < 5.0e3), times=1)
    hill_cfg = cases.HillCaseConfig(domain=ext)
    geom, ops, model, bg, U, bcs, split, sigma = _terrain_case(
        mesh, 3, hill3d, hill_cfg,
        cases.SpongeConfig(top_depth=4.0e3, lateral_width=5.0e3), (0, 1), 31, ext)
    rec = {"case": np.array("hang3d"), "degree": np.array(3),
           "background": bg, "sigma": sigma}
    rec.update(mesh_record(mesh))
    rec.update(geometry_record(geom))
    rec.update(operator_record(ops, split, U, model, bcs, 31, 0.3))
    rec.update(gmres_record(split, U, 0.3, 1e-8, 31))
    scfg = imex.ImplicitSolveConfig()
    rec.update(steps_record(split, U, 0.5, 2, scfg))
    save("hang3d", rec)


def case_per3d():
    ext = (10.0e3, 10.0e3, 10.0e3)
    m = build_uniform_mesh(ext, (4, 4, 4), periodic=(True, True, True))
    pick = np.random.default_rng(5).random(m.n_leaves) < 0.3
    mesh = refine_region(m, lambda lf: bool(pick[lf.index]), 1)
    geom = build_geometry(mesh, 2)
    ops = DGOperators(geom)
    model = FlowModel.dimensional()
    hill_cfg = cases.HillCaseConfig(domain=ext)
    bg = project_initial_data(geom, cases.hydrostatic_initial_state(hill_cfg)).data
    U = perturbed(bg, geom.node_coords, ext, 41)
    split = imex.SplitOperators(ops, model, [])
    rec = {"case": np.array("per3d"), "degree": np.array(2), "pick": pick}
    rec.update(mesh_record(mesh))
    rec.update(geometry_record(geom))
    rec.update(operator_record(ops, split, U, model, [], 41, 0.3))
    save("per3d", rec)


def case_cfg3s():
    ext = (50.0e3, 21.0e3)
    m = build_uniform_mesh(ext, (25, 8))
    mesh = refine_region(m, lambda lf: lf.center[1] < 6.0e3, 1)
    mesh = refine_region(mesh, lambda lf: lf.center[1] < 2.5e3, 1)
    hill_cfg = cases.HillCaseConfig(domain=ext, T_ref=280.0)
    geom, ops, model, bg, U, bcs, split, sigma = _terrain_case(
        mesh, 4, schar, hill_cfg,
        cases.SpongeConfig(top_depth=9.0e3, lateral_width=10.0e3), (0,), 51, ext)
    U = bg.copy()   # the physical IC: background flow over the hill
    rec = {"case": np.array("cfg3s"), "degree": np.array(4),
           "background": bg, "sigma": sigma}
    rec.update(mesh_record(mesh))
    rec.update(operator_record(ops, split, U, model, bcs, 51, 0.5))
    scfg = imex.ImplicitSolveConfig()
    rec.update(steps_record(split, U, 1.0, 3, scfg))
    save("cfg3s", rec)


def case_part():
    mesh = build_uniform_mesh((20.0e3, 10.0e3), (64, 32))
    mesh = refine_region(mesh, lambda lf: lf.center[1] < 5.0e3, 1)
    rec = {}
    rec.update(mesh_record(mesh))
    rng = np.random.default_rng(3)
    w = rng.uniform(0.5, 2.0, size=mesh.n_leaves)
    rec["weights"] = w
    for P in range(1, 9):
        for tag, wt in (("u", None), ("w", w)):
            p = partition_leaves(mesh, P, wt)
            rec[f"P{P}{tag}_owner"] = p.owner
            rec[f"P{P}{tag}_ranges"] = np.array(p.ranges, dtype=np.int64)
            rec[f"P{P}{tag}_ghost_len"] = np.array([len(g) for g in p.ghosts])
            rec[f"P{P}{tag}_ghosts"] = (np.concatenate(p.ghosts) if p.ghosts
                                        else np.empty(0, np.int64))
    small = build_uniform_mesh((10.0, 1.0), (10, 1))
    p = partition_leaves(small, 4)
    rec["small10x4_ranges"] = np.array(p.ranges, dtype=np.int64)
    save("part", rec)


def case_cfg2ops():
    """Refresh the operator records of cfg2.npz without rerunning 200 steps."""
    mesh, geom, ops, model, U0, bcs, split = bubble_case((64, 32), 5.0e3, 4)
    a_dt = 0.5 * (1.0 - 1.0 / np.sqrt(2.0))
    path = os.path.join(OUT, "cfg2.npz")
    rec = dict(np.load(path))
    rec.update(operator_record(ops, split, U0, model, bcs, 12, a_dt))
    save("cfg2", rec)


def _bj_record(prefix, mesh, split, U, a_dt, seed):
    """Block-Jacobi preconditioner of the Helmholtz action at U
    (krylov.py:118-178): the greedy element colouring, the preconditioner
    applied to a seeded vector, and one right-preconditioned GMRES solve."""
    colors = krylov.element_coloring(mesh)
    d = split.dim
    e_e = U[:, 1 + d]
    action = imex.build_helmholtz_action(split, a_dt, U)
    M = krylov.block_jacobi_preconditioner(action, e_e.shape[0], e_e.shape[1], colors)
    v = np.random.default_rng(seed).standard_normal(e_e.shape)
    h, K = split.frozen_coefficients(U)
    F, _ = split.energy_affine_map(a_dt, h, K, U[:, 1:1 + d].copy(), e_e.copy())
    F0 = F(np.zeros_like(e_e))
    x0 = energy_like(U, seed + 1).ravel()
    x, st = krylov.gmres(action, F0.ravel(), x0=x0, tol_rel=1e-8, restart=30, max_iter=1000,
                         preconditioner=M)
    return {prefix + "colors": colors, prefix + "a_dt": np.array(a_dt), prefix + "v": v,
            prefix + "Mv": M(v.ravel()).reshape(e_e.shape), prefix + "rhs": F0,
            prefix + "x0": x0.reshape(e_e.shape), prefix + "x": x.reshape(e_e.shape),
            prefix + "iters": np.array(st.iterations),
            prefix + "history": np.array(st.residual_history)}


def case_bj():
    """block_jacobi preconditioning: cfg1 mesh (colouring,
    M v, preconditioned GMRES, 4 ARS(2,2,2) steps rebuilding every 3 solves)
    and a once-refined bubble mesh with hanging faces (colouring, M v)."""
    mesh, geom, ops, model, U0, bcs, split = bubble_case((32, 16), None, 2)
    dt = 0.5
    a_dt = dt * (1.0 - 1.0 / np.sqrt(2.0))
    rec = {"case": np.array("bj")}
    rec.update(_bj_record("c1_", mesh, split, U0, a_dt, 31))
    scfg = imex.ImplicitSolveConfig(preconditioner="block_jacobi", precond_refresh=3)
    tab = imex.ars222()
    U = U0.copy()
    pc = imex._PrecondCache()
    fp, kr = [], []
    for s in range(4):
        U, st = imex.imex_step(U, s * dt, dt, tab, split, scfg, precond=pc)
        fp.append(st.fp_iters)
        kr.append(st.krylov_iters)
        print(f"  bj step {s + 1}: fp {st.fp_iters} krylov {st.krylov_iters}", flush=True)
    rec.update({"st_U_final": U, "st_fp_iters": _ragged(fp), "st_krylov_iters": _ragged(kr),
                "st_refresh": np.array(3), "st_n_steps": np.array(4), "st_dt": np.array(dt)})
    mesh2, geom2, ops2, model2, U2, bcs2, split2 = bubble_case((16, 8), 5.0e3, 2)
    rec.update(_bj_record("h_", mesh2, split2, U2, a_dt, 32))
    save("bj", rec)


def case_full():
    """DGOperators.divergence_full / apply_divergence (both fluxes),
    global_inner_product and physics.courant_numbers (dgops.py:298-328,
    483-503; physics.py:255-272) on the cfg1 bubble and the hang2d / hang3d
    terrain + hanging + far-field meshes (inputs stored with the outputs)."""
    from orodg.field import StateField
    from orodg.physics import courant_numbers
    rec = {"case": np.array("full")}
    mesh, geom, ops, model, U, bcs, split = bubble_case((32, 16), None, 2)
    builds = [("cfg1", geom, ops, model, U, bcs, U * (1.0 + 1e-3 * np.sin(U)))]
    ext = (60.0e3, 16.0e3)
    m = refine_region(build_uniform_mesh(ext, (15, 4)),
                      lambda lf: abs(lf.center[0] - 30.0e3) < 6.0e3 and lf.center[1] < 6.0e3,
                      times=2)
    geom, ops, model, bg, U, bcs, split, sigma = _terrain_case(
        m, 4, hill2d, cases.HillCaseConfig(domain=ext), cases.SpongeConfig(), (0,), 21, ext)
    builds.append(("hang2d", geom, ops, model, U, bcs, bg))
    ext = (20.0e3, 20.0e3, 10.0e3)
    m = refine_region(build_uniform_mesh(ext, (4, 4, 2)),
                      lambda lf: bool(np.all(np.abs(lf.center[:2] - 10.0e3) < 5.0e3)
                                      and lf.center[2] < 5.0e3), times=1)
    geom, ops, model, bg, U, bcs, split, sigma = _terrain_case(
        m, 3, hill3d, cases.HillCaseConfig(domain=ext),
        cases.SpongeConfig(top_depth=4.0e3, lateral_width=5.0e3), (0, 1), 31, ext)
    builds.append(("hang3d", geom, ops, model, U, bcs, bg))
    for name, geom, ops, model, U, bcs, U2 in builds:
        p = name + "_"
        rec[p + "U"] = U
        rec[p + "U2"] = U2
        # the reference's own 1-ulp input sensitivity (see noise_record)
        rng = np.random.default_rng(4321)
        Up = U * (1.0 + 2.0 ** -52 * rng.choice([-1.0, 1.0], size=U.shape))
        for flux in ("rusanov", "centered"):
            rec[p + "full_" + flux] = ops.divergence_full(U, model, bcs, flux)
            rec["noise_" + p + "full_" + flux] = _per_var_noise(
                ops.divergence_full(Up, model, bcs, flux), rec[p + "full_" + flux])
        field = StateField(U, geom.mesh.fingerprint, geom.basis.degree)
        rec[p + "apply_div"] = ops.apply_divergence(field, model, bcs, "rusanov")
        rec["noise_" + p + "apply_div"] = _per_var_noise(
            ops.apply_divergence(StateField(Up, geom.mesh.fingerprint, geom.basis.degree),
                                 model, bcs, "rusanov"), rec[p + "apply_div"])
        rec[p + "inner"] = np.array(ops.global_inner_product(U, U2))
        cr = courant_numbers(U, geom, 0.5, model)
        rec[p + "courant"] = np.array([cr.acoustic, cr.advective, cr.max_sound_speed,
                                       cr.max_speed, cr.min_diameter])
    save("full", rec)


def case_hang3d_r4():
    """hang3d's terrain + hanging + far-field + sponge mesh at r=4 (n^(d-1)
    = 25 lanes per element on the device): every operator, one GMRES solve,
    one step."""
    ext = (20.0e3, 20.0e3, 10.0e3)
    m = build_uniform_mesh(ext, (4, 4, 2))
    mesh = refine_region(
        m, lambda lf: bool(np.all(np.abs(lf.center[:2] - 10.0e3) < 5.0e3)
                           and lf.center[2] < 5.0e3), times=1)
    geom, ops, model, bg, U, bcs, split, sigma = _terrain_case(
        mesh, 4, hill3d, cases.HillCaseConfig(domain=ext),
        cases.SpongeConfig(top_depth=4.0e3, lateral_width=5.0e3), (0, 1), 37, ext)
    rec = {"case": np.array("hang3d_r4"), "degree": np.array(4), "background": bg,
           "sigma": sigma}
    rec.update(mesh_record(mesh))
    rec.update(operator_record(ops, split, U, model, bcs, 37, 0.3))
    rec.update(gmres_record(split, U, 0.3, 1e-8, 37))
    rec.update(steps_record(split, U, 0.5, 1, imex.ImplicitSolveConfig()))
    save("hang3d_r4", rec)


def case_per3d_r4():
    """per3d's triply-periodic seeded-refined box at r=4."""
    ext = (10.0e3, 10.0e3, 10.0e3)
    m = build_uniform_mesh(ext, (3, 3, 3), periodic=(True, True, True))
    pick = np.random.default_rng(7).random(m.n_leaves) < 0.3
    mesh = refine_region(m, lambda lf: bool(pick[lf.index]), 1)
    geom = build_geometry(mesh, 4)
    ops = DGOperators(geom)
    model = FlowModel.dimensional()
    bg = project_initial_data(
        geom, cases.hydrostatic_initial_state(cases.HillCaseConfig(domain=ext))).data
    U = perturbed(bg, geom.node_coords, ext, 43)
    split = imex.SplitOperators(ops, model, [])
    rec = {"case": np.array("per3d_r4"), "degree": np.array(4), "pick": pick}
    rec.update(mesh_record(mesh))
    rec.update(operator_record(ops, split, U, model, [], 43, 0.3))
    save("per3d_r4", rec)


def case_cfg5s():
    """BASELINE configs[4] recipe at a reduced root count:
    periodic (10 km)^3, 6^3 roots, a seeded 7% refined once, r=3,
    hydrostatic background + seeded smooth 1e-3 perturbations."""
    ext = (10.0e3, 10.0e3, 10.0e3)
    m = build_uniform_mesh(ext, (6, 6, 6), periodic=(True, True, True))
    pick = np.random.default_rng(5).random(m.n_leaves) < 0.07
    mesh = refine_region(m, lambda lf: bool(pick[lf.index]), 1)
    geom = build_geometry(mesh, 3)
    ops = DGOperators(geom)
    model = FlowModel.dimensional()
    bg = project_initial_data(
        geom, cases.hydrostatic_initial_state(cases.HillCaseConfig(domain=ext))).data
    U = perturbed(bg, geom.node_coords, ext, 41)
    split = imex.SplitOperators(ops, model, [])
    rec = {"case": np.array("cfg5s"), "degree": np.array(3), "pick": pick}
    rec.update(mesh_record(mesh))
    rec.update(operator_record(ops, split, U, model, [], 41, 0.3))
    rec.update(gmres_record(split, U, 0.3, 1e-8, 41))
    save("cfg5s", rec)


def case_dropin():
    """Drop-in API surface beyond the hot operators, on hang3d's mesh (r=3):
    implicit_residual / full_residual (imex.py:161-178), a forced ARS(2,2,2)
    step (imex.py:157-158; forcing(t) = (1 + t/10) S, S a seeded smooth
    field), MeshGeometry.apply_mass_inverse on an element subset
    (geometry.py:372-396), and gmres on a host (numpy) operator with
    restart 40 > 31 (krylov.py:27-115)."""
    ext = (20.0e3, 20.0e3, 10.0e3)
    m = build_uniform_mesh(ext, (4, 4, 2))
    mesh = refine_region(
        m, lambda lf: bool(np.all(np.abs(lf.center[:2] - 10.0e3) < 5.0e3)
                           and lf.center[2] < 5.0e3), times=1)
    geom, ops, model, bg, U, bcs, split, sigma = _terrain_case(
        mesh, 3, hill3d, cases.HillCaseConfig(domain=ext),
        cases.SpongeConfig(top_depth=4.0e3, lateral_width=5.0e3), (0, 1), 31, ext)
    rec = {"case": np.array("dropin"), "U": U}
    rec["implicit_residual"] = split.implicit_residual(U)
    rec["full_residual"] = split.full_residual(U, 0.0)
    # the reference's own 1-ulp input sensitivity (noise_record)
    rp = np.random.default_rng(1234)
    Up = U * (1.0 + 2.0 ** -52 * rp.choice([-1.0, 1.0], size=U.shape))
    rec["noise_implicit_residual"] = _per_var_noise(split.implicit_residual(Up),
                                                    rec["implicit_residual"])
    rec["noise_full_residual"] = _per_var_noise(split.full_residual(Up, 0.0),
                                                rec["full_residual"])
    rng = np.random.default_rng(99)
    S = np.zeros_like(U)
    for v in range(U.shape[1]):
        S[:, v] = 1e-4 * np.abs(U[:, v]).max() * smooth_noise(geom.node_coords, ext, rng)
    rec["forcing_S"] = S
    fsplit = imex.SplitOperators(ops, model, bcs, sponge=(sigma, bg),
                                 forcing=lambda t: (1.0 + t / 10.0) * S)
    Uf, st = imex.imex_step(U, 0.25, 0.5, imex.ars222(), fsplit, imex.ImplicitSolveConfig())
    rec["forced_U1"] = Uf
    rec["forced_krylov"] = np.array(st.krylov_iters)
    rec["forced_fp"] = np.array(st.fp_iters)
    sel = np.arange(0, mesh.n_leaves, 3)
    dual = ops.divergence_advective(U, model, bcs)[sel]
    rec["minv_sel"] = sel
    rec["minv_sel_dual"] = dual
    rec["minv_sel_out"] = geom.apply_mass_inverse(dual, elements=sel)
    n = 120
    A = np.eye(n) + 0.3 * rng.standard_normal((n, n)) / np.sqrt(n)
    b = rng.standard_normal(n)
    x, kst = krylov.gmres(lambda v: A @ v, b, tol_rel=1e-10, restart=40, max_iter=500)
    rec["gm_A"], rec["gm_b"], rec["gm_x"] = A, b, x
    rec["gm_iters"] = np.array(kst.iterations)
    rec["gm_history"] = np.array(kst.residual_history)
    save("dropin", rec)


CASES = {"cfg2ops": case_cfg2ops, "cfg1": case_cfg1, "hang2d": case_hang2d, "hang3d": case_hang3d,
         "per3d": case_per3d, "cfg3s": case_cfg3s, "part": case_part,
         "cfg2": case_cfg2, "bj": case_bj, "full": case_full, "hang3d_r4": case_hang3d_r4,
         "per3d_r4": case_per3d_r4, "cfg5s": case_cfg5s, "dropin": case_dropin}

if __name__ == "__main__":
    names = sys.argv[1:] or list(CASES)
    for n in names:
        t0 = time.perf_counter()
        print(f"== {n}", flush=True)
        CASES[n]()
        print(f"   {time.perf_counter() - t0:.1f} s", flush=True)
