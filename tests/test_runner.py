"""Drop-in runner (orodg/runner.py:34-309, orodg/config.py:15-86) on the
device path: reference presets and the BASELINE presets through setup_run /
run, with the device diagnostics (integrate_conserved, max |w|)."""

import numpy as np
import pytest

from casebuild import check_rel, golden


def test_config_validation_and_presets():
    from paper_2408_08129_b200.errors import ConfigurationError
    from paper_2408_08129_b200.runner import CaseConfig, _preset, is_baseline_preset
    CaseConfig().validate()
    CaseConfig(preset="cfg4").validate()
    CaseConfig(preset="cfg5_r3").validate()
    assert is_baseline_preset("cfg4w6") and not is_baseline_preset("paper2d")
    with pytest.raises(ConfigurationError):
        CaseConfig(preset="nope").validate()
    with pytest.raises(ConfigurationError):
        CaseConfig(krylov_tol=2.0).validate()
    assert _preset(CaseConfig(preset="paper3d-small"), "root") == (15, 10, 4)
    assert _preset(CaseConfig(preset="paper2d", dt=1.0), "dt") == 1.0


@pytest.mark.gpu
def test_run_baseline_cfg1_matches_reference_golden():
    """The cfg1 BASELINE preset through run(): 10 steps of 0.5 s equal the
    reference's 10-step state (golden cfg1), diagnostics per step."""
    from paper_2408_08129_b200.runner import CaseConfig, run
    z = golden("cfg1")
    res = run(CaseConfig(preset="cfg1", dt=0.5, t_final=5.0))
    assert res.steps == 10
    check_rel("cfg1", "runner_cfg1_10_steps", res.final.data, z["U_final"], 1e-9)
    rows = res.diagnostics
    assert rows[0].startswith("step,t,mass,energy,max_w") and len(rows) == 12
    mass = np.array([float(r.split(",")[2]) for r in rows[1:]])
    assert np.all(np.abs(mass - mass[0]) <= 1e-12 * abs(mass[0]))  # walls: mass conserved
    kry = [int(r.split(",")[6]) for r in rows[2:]]
    ref = [int(v) for v in z["krylov_iters"].clip(0).sum(axis=1)]
    assert kry == ref
    assert res.timer_report.blocks["krylov"] > 0.0


@pytest.mark.gpu
def test_run_reference_presets_smoke():
    """hydrostatic-rest (walls, no terrain), paper2d (terrain, far field,
    sponge, two refinement levels, small root grid) and manufactured (forced,
    periodic) run through the device path."""
    from paper_2408_08129_b200.field import project_initial_data  # noqa: F401
    from paper_2408_08129_b200.runner import CaseConfig, run
    r = run(CaseConfig(preset="hydrostatic-rest", root=(12, 4), degree=3), max_steps=2)
    assert r.steps == 2 and float(r.diagnostics[-1].split(",")[4]) < 1.0  # max |w| [m/s]
    r = run(CaseConfig(preset="paper2d", root=(12, 4), degree=3, dt=1.0), max_steps=2)
    assert r.steps == 2 and np.all(np.isfinite(r.final.data))
    r = run(CaseConfig(preset="manufactured", degree=3), max_steps=3)
    from paper_2408_08129_b200 import cases
    ctx = r.context
    exact = cases.manufactured_state(ctx.geometry.node_coords, 3 * 0.01)
    err = np.linalg.norm(r.final.data - np.moveaxis(exact, 2, 1)) / np.linalg.norm(exact)
    assert err < 1e-3, err
