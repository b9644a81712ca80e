"""Drop-in API surface beyond the fused operators (reference imex.py:161-178,
157-158, 373-404; geometry.py:372-396; krylov.py:27-115; boundary.py:17-84;
timing.py:12-74), against the reference's golden vectors (tests/golden/
dropin.npz, make_golden.case_dropin).  GPU tests call the device path; the
CPU tests cover the host-side pieces."""

import types

import numpy as np
import pytest

from casebuild import assert_parity, build, check_rel, golden, per_var_rel, record


def _split(c, forcing=None):
    from paper_2408_08129_b200.dgops import DGOperators
    from paper_2408_08129_b200.imex import SplitOperators
    ops = DGOperators(c.geom)
    return ops, SplitOperators(ops, c.model, c.bcs, c.sponge, forcing=forcing)


# ------------------------------------------------------------------- CPU
def test_block_timer_semantics():
    from paper_2408_08129_b200.timing import BLOCKS, BlockTimer, NullTimer, credit
    t = iter([0.0, 1.0, 2.0, 5.0, 6.0, 10.0, 11.0, 12.0])
    tm = BlockTimer(clock=lambda: next(t))
    with tm.block("implicit_fixed_point"):      # 1.0
        with tm.block("krylov"):                # 2.0 .. 5.0
            pass
    # innermost attribution: krylov 3, implicit_fixed_point (1->2) + (5->6) = 2
    assert tm.totals == {"implicit_fixed_point": 2.0, "krylov": 3.0}
    credit(tm, "explicit_residual", 0.5, source="implicit_fixed_point")
    assert tm.totals["implicit_fixed_point"] == 1.5 and tm.totals["explicit_residual"] == 0.5
    snap = tm.step_snapshot()
    assert snap["krylov"] == 3.0 and tm.step_snapshot()["krylov"] == 0.0
    rep = tm.report([snap])
    assert rep.csv_header() == "step," + ",".join(BLOCKS)
    assert len(rep.csv_rows()) == 1 and rep.accounted == pytest.approx(5.0)
    nt = NullTimer()
    with nt.block("krylov"):
        pass
    assert nt.report().total == 0.0


def test_mirror_state_and_ghosts():
    from paper_2408_08129_b200.boundary import BoundaryCondition, mirror_state
    from paper_2408_08129_b200.physics import FlowModel
    rng = np.random.default_rng(3)
    tr = rng.standard_normal((4, 5, 6))
    n = rng.standard_normal((4, 6, 3))
    n /= np.linalg.norm(n, axis=2, keepdims=True)
    g = mirror_state(tr, n)
    mn = np.einsum("fan,fna->fn", tr[:, 1:4], n)
    gn = np.einsum("fan,fna->fn", g[:, 1:4], n)
    assert np.allclose(gn, -mn) and np.array_equal(g[:, [0, 4]], tr[:, [0, 4]])
    w = BoundaryCondition("wall")
    assert w.scalar_ghost(tr[:, :1], None, (0, 4)) is not None
    hv = w.hv_ghost(tr[:, 1:], n, None, (0, 4))
    vn = np.einsum("fan,fna->fn", hv[:, :3], n)
    assert np.allclose(vn, -np.einsum("fan,fna->fn", tr[:, 1:4], n))
    U = np.abs(tr) + 1.0
    ff = BoundaryCondition("farfield", U)
    model = FlowModel.dimensional()
    assert ff.conserved_ghost(tr, n, (1, 3)).shape == (2, 5, 6)
    assert ff.scalar_ghost(None, model, (0, 4)).shape == (4, 1, 6)
    assert ff.hv_ghost(tr[:, 1:], n, model, (0, 2)).shape == (2, 4, 6)


def test_weak_form_refuses_host_callbacks():
    from paper_2408_08129_b200.dgops import DGOperators
    from paper_2408_08129_b200.errors import UsageError
    c = build("cfg1")
    with pytest.raises(UsageError):
        DGOperators(c.geom).weak_form(c.U, 4, None, None, None)


# ------------------------------------------------------------------- GPU
@pytest.mark.gpu
def test_implicit_and_full_residual():
    c, z = build("hang3d"), golden("dropin")
    U = z["U"]
    ops, split = _split(c)
    Ri = split.implicit_residual(U)
    assert np.all(Ri[:, 0] == 0.0)
    # per-variable gates max(1e-12, 10 x the reference's 1-ulp sensitivity)
    # (the horizontal pressure gradient of a hydrostatic state cancels)
    assert_parity(Ri[:, 1:], {"case": "dropin", "implicit_residual": z["implicit_residual"][:, 1:],
                              "noise_implicit_residual": z["noise_implicit_residual"][1:]},
                  "implicit_residual")
    assert_parity(split.full_residual(U, 0.0), z, "full_residual")


@pytest.mark.gpu
def test_forced_step():
    """SplitOperators.forcing is honoured: forcing(t + c_ex dt) is added to
    every explicit residual of the step (imex.py:157-158, 286)."""
    c, z = build("hang3d"), golden("dropin")
    S = z["forcing_S"]
    calls = []

    def forcing(t):
        calls.append(t)
        return (1.0 + t / 10.0) * S

    from paper_2408_08129_b200.imex import ImplicitSolveConfig, ars222, imex_step
    ops, split = _split(c, forcing)
    U1, st = imex_step(z["U"], 0.25, 0.5, ars222(), split, ImplicitSolveConfig())
    assert st.krylov_iters == [int(v) for v in z["forced_krylov"]]
    assert st.fp_iters == [int(v) for v in z["forced_fp"]]
    check_rel("dropin", "forced_step_state", U1, z["forced_U1"], 1e-11)
    g = 1.0 - 1.0 / np.sqrt(2.0)
    assert calls == pytest.approx([0.25, 0.25 + g * 0.5])


@pytest.mark.gpu
def test_geometry_mass_inverse_subset():
    c, z = build("hang3d"), golden("dropin")
    sel = z["minv_sel"]
    out = c.geom.apply_mass_inverse(z["minv_sel_dual"], elements=sel)
    check_rel("dropin", "minv_subset", out, z["minv_sel_out"], 1e-13)
    buf = np.empty_like(out)
    c.geom.apply_mass_inverse(z["minv_sel_dual"], out=buf, elements=sel)
    assert np.array_equal(buf, out)
    full = golden("hang3d")
    check_rel("hang3d", "geometry.apply_mass_inverse",
              c.geom.apply_mass_inverse(full["dual_adv"]), full["minv_dual_adv"], 1e-13)


@pytest.mark.gpu
def test_gmres_host_callable_long_restart():
    """A numpy operator (the reference's calling convention) and restart 40."""
    z = golden("dropin")
    from paper_2408_08129_b200.krylov import gmres
    A, b = z["gm_A"], z["gm_b"]
    x, st = gmres(lambda v: A @ v, b, tol_rel=1e-10, restart=40, max_iter=500)
    assert isinstance(x, np.ndarray)
    assert st.iterations == int(z["gm_iters"])
    check_rel("dropin", "host_gmres_x", x, z["gm_x"], 1e-10)
    assert np.allclose(st.residual_history, z["gm_history"], rtol=1e-6, atol=1e-14)


@pytest.mark.gpu
def test_native_gmres_restart_beyond_31():
    """The device Helmholtz GMRES accepts krylov_restart > 31 (unfused CGS
    passes); restart 40 covers the whole hang3d solve in one cycle, like 30."""
    c, z = build("hang3d"), golden("hang3d")
    ops, split = _split(c)
    from paper_2408_08129_b200.imex import build_helmholtz_action
    from paper_2408_08129_b200.krylov import gmres
    act = build_helmholtz_action(split, float(z["a_dt"]), c.U)
    x, st = gmres(act, z["gm_rhs"].ravel(), x0=z["gm_x0"].ravel(), tol_rel=float(z["gm_tol"]),
                  restart=40)
    assert st.converged and st.iterations == int(z["gm_iters"])
    check_rel("hang3d", "gmres_x_restart40", x, z["gm_x"].ravel(), 1e-10)


@pytest.mark.gpu
def test_runner_stepper_with_reference_style_config():
    """runner.py:277-280 drives imex_step through a stepper closure with the
    reference's config object (fields only, no ``c()``) and a BlockTimer;
    run_time_loop returns timer.report(per_step) (imex.py:373-404)."""
    c, z = build("hang3d"), golden("hang3d")
    ops, split = _split(c)
    from paper_2408_08129_b200.imex import ars222, imex_step, run_time_loop
    from paper_2408_08129_b200.timing import BlockTimer
    cfg = types.SimpleNamespace(fp_tol=1e-6, fp_max_iter=10, krylov_tol=1e-8, krylov_restart=30,
                                krylov_max_iter=1000, preconditioner="none", precond_refresh=20)
    timer = BlockTimer()
    seen = []

    def stepper(U, t, dt):
        return imex_step(U, t, dt, ars222(), split, cfg, timer)

    U, rep = run_time_loop(c.U, 0.5, 1.0, stepper, callbacks=[lambda s, t, u, st: seen.append(s)],
                           timer=timer)
    assert seen == [0, 1, 2]
    check_rel("hang3d", "run_time_loop_2_steps", U, z["U_final"], 1e-9)
    assert len(rep.per_step) == 2
    assert rep.blocks["krylov"] > 0.0 and rep.blocks["explicit_residual"] > 0.0
    assert rep.blocks["implicit_fixed_point"] >= 0.0
    assert rep.accounted <= rep.total * 1.01
