"""DGOperators.divergence_full / apply_divergence (both fluxes),
global_inner_product and physics.courant_numbers against the reference
(golden fixture full.npz: tests/golden/make_golden.py case_full).

CPU: the oracle restatement.  GPU: the libdg kernels through the drop-in API.
"""

import numpy as np
import pytest

from casebuild import assert_parity, build, golden, per_var_rel

NAMES = ["cfg1", "hang2d", "hang3d"]


def _oracle(c):
    from oracle import dg_oracle as O
    return O.Operators(c.geom, c.model, c.bcs, c.sponge)


@pytest.mark.parametrize("name", NAMES)
def test_oracle_full_matches_reference(name):
    c, z = build(name), golden("full")
    ops = _oracle(c)
    U = z[name + "_U"]
    for flux in ("rusanov", "centered"):
        assert_parity(ops.divergence_full(U, flux), z, f"{name}_full_{flux}")
    g = ops.global_inner_product(U, z[name + "_U2"])
    assert abs(g - float(z[name + "_inner"])) <= 1e-13 * abs(float(z[name + "_inner"]))
    cm, um = ops.courant_ingredients(U)
    ref = z[name + "_courant"]
    assert abs(cm - ref[2]) <= 1e-13 * ref[2]
    assert abs(um - ref[3]) <= 1e-12 * max(ref[3], 1e-300) + 1e-300


@pytest.mark.gpu
@pytest.mark.parametrize("name", NAMES)
def test_device_full_ops_match_reference(name):
    from paper_2408_08129_b200.dgops import DGOperators
    from paper_2408_08129_b200.field import StateField
    from paper_2408_08129_b200.physics import courant_numbers
    c, z = build(name), golden("full")
    ops = DGOperators(c.geom)
    U = z[name + "_U"]
    for flux in ("rusanov", "centered"):
        assert_parity(ops.divergence_full(U, c.model, c.bcs, flux), z, f"{name}_full_{flux}")
    field = StateField(U, c.mesh.fingerprint, c.geom.basis.degree)
    assert_parity(ops.apply_divergence(field, c.model, c.bcs, "rusanov"), z, name + "_apply_div")
    g = ops.global_inner_product(U, z[name + "_U2"])
    assert abs(g - float(z[name + "_inner"])) <= 1e-13 * abs(float(z[name + "_inner"]))
    cr = courant_numbers(U, c.geom, 0.5, c.model)
    got = np.array([cr.acoustic, cr.advective, cr.max_sound_speed, cr.max_speed, cr.min_diameter])
    np.testing.assert_allclose(got, z[name + "_courant"], rtol=1e-12, atol=1e-300)
