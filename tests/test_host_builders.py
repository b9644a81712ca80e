"""Host input builders (mesh, basis, geometry, cases) against the
reference's golden topology/geometry arrays and its mesh/basis properties
(reference tests: tests/test_mesh.py, tests/test_basis.py).  CPU only."""

from fractions import Fraction

import numpy as np
import pytest

from casebuild import build, golden, rel
from paper_2408_08129_b200.basis import (gauss_legendre, gauss_lobatto, lagrange_eval_matrix,
                                         make_basis)
from paper_2408_08129_b200.errors import ConfigurationError, MeshError
from paper_2408_08129_b200.mesh import (ForestMesh, build_uniform_mesh, check_tiling, dump_mesh,
                                        refine_region, restore_mesh)

CASES = ["cfg1", "hang2d", "hang3d", "per3d", "cfg3s", "cfg2"]


@pytest.mark.parametrize("name", CASES)
def test_topology_identical_to_reference(name):
    m, z = build(name).mesh, golden(name)
    assert np.array_equal(m.levels, z["mesh_levels"])
    assert np.array_equal(m.origins, z["mesh_origins"])
    t = m.topology
    assert [b.axis for b in t.conforming] == list(z["mesh_conf_axis"])
    for i, b in enumerate(t.conforming):
        assert np.array_equal(b.left, z[f"mesh_conf{i}_left"])
        assert np.array_equal(b.right, z[f"mesh_conf{i}_right"])
    for i, b in enumerate(t.hanging):
        assert [b.axis, b.orient] == list(z["mesh_hang_axis_orient"][i])
        for k in ("coarse", "fine", "subface"):
            assert np.array_equal(getattr(b, k), z[f"mesh_hang{i}_{k}"])
    for i, b in enumerate(t.boundary):
        assert [b.axis, b.side] == list(z["mesh_bdry_axis_side"][i])
        assert np.array_equal(b.leaves, z[f"mesh_bdry{i}_leaves"])
    assert m.fingerprint == str(z["mesh_fingerprint"])


@pytest.mark.parametrize("name", ["cfg1", "hang2d", "hang3d", "per3d"])
def test_geometry_matches_reference(name):
    g, z = build(name).geom, golden(name)
    assert rel(g.det_j, z["geo_det_j"]) <= 1e-15
    assert rel(g.ctrv, z["geo_ctrv"]) <= 1e-15
    assert rel(g.mass_h_inv, z["geo_mass_h_inv"]) <= 1e-14
    assert rel(g.node_coords, z["geo_node_coords"]) <= 1e-15
    for tag, lst in (("conf", g.conforming), ("hang", g.hanging), ("bdry", g.boundary)):
        for i, fg in enumerate(lst):
            assert rel(fg.normal, z[f"geo_{tag}{i}_normal"]) <= 1e-15
            assert rel(fg.ws, z[f"geo_{tag}{i}_ws"]) <= 1e-15


def test_device_tables_reproduce_dense_metric():
    """The compact column table + on-the-fly formulas (what the kernels
    evaluate) reproduce the dense det J / adjugate arrays."""
    c = build("hang3d")
    g = c.geom
    elem, col, stride = g.device_tables()
    b = g.basis
    nqh = b.n_quad_1d ** 2
    lv, org, cid = elem[:, 0], elem[:, 1:4], elem[:, 4]
    s = np.array([e / r for e, r in zip(c.mesh.extents, c.mesh.root_counts)])[None, :] \
        / (2.0 ** lv)[:, None]
    omh = col[cid, :nqh]            # 1 - h/z_top at the horizontal Gauss grid
    zz = s[:, 2][:, None] * omh
    det = (s[:, 0] * s[:, 1])[:, None] * zz
    assert rel(np.repeat(det, b.n_quad_1d, axis=1), g.det_j) <= 1e-15


def _brute_balance(mesh):
    views = mesh.leaf_views()
    for i, a in enumerate(views):
        for bb in views[i + 1:]:
            touch, shared = True, None
            for ax in range(mesh.dim):
                lo, hi = max(a.lo[ax], bb.lo[ax]), min(a.hi[ax], bb.hi[ax])
                if np.isclose(hi, lo):
                    if shared is not None:
                        touch = False
                        break
                    shared = ax
                elif hi < lo:
                    touch = False
                    break
            if touch and shared is not None:
                assert abs(a.level - bb.level) <= 1


def test_mesh_counts_and_kats():
    m = build_uniform_mesh((60.0e3, 40.0e3, 16.0e3), (60, 40, 16))
    assert m.n_leaves == 38400
    assert sum(len(b.left) for b in m.topology.conforming) == \
        59 * 40 * 16 + 60 * 39 * 16 + 60 * 40 * 15
    one = build_uniform_mesh((1.0, 1.0), (1, 1))
    assert one.topology.n_boundary_faces() == 4 and one.topology.n_interior_faces() == 0
    m = refine_region(build_uniform_mesh((1.0, 1.0), (2, 2)), lambda lf: lf.index == 0, 1)
    assert m.n_leaves == 7
    assert m.topology.n_hanging_coarse_faces(2) == 2
    assert sum(len(b.coarse) for b in m.topology.hanging) == 4
    check_tiling(m)
    m = refine_region(build_uniform_mesh((1.0, 1.0), (4, 4)),
                      lambda lf: bool(np.all(lf.hi <= 0.25 + 1e-12)), times=2)
    assert m.max_level == 2 and m.n_leaves > 4 * 4 - 1 + 4 + 3
    check_tiling(m)
    _brute_balance(m)


def test_rational_tiling_and_periodic():
    m = build_uniform_mesh((3.0, 2.0), (3, 2))
    picks = set(np.random.default_rng(7).integers(0, 6, size=3).tolist())
    m = refine_region(m, lambda lf: lf.index in picks, 1)
    m = refine_region(m, lambda lf: lf.level == 1 and lf.index % 3 == 0, 1)
    assert sum(Fraction(1, 2 ** (m.dim * lv)) for lv, _ in m.leaves) == 6
    _brute_balance(m)
    p = build_uniform_mesh((1.0, 1.0), (2, 2), periodic=(True, False))
    assert sum(len(b.left) for b in p.topology.conforming if b.axis == 0) == 4
    assert p.topology.n_boundary_faces() == 4


def test_hanging_groups_3d():
    m = refine_region(build_uniform_mesh((1.0, 1.0, 1.0), (2, 2, 2)),
                      lambda lf: lf.index == 0, 1)
    for b in m.topology.hanging:
        for g in range(len(b.coarse) // 4):
            rows = slice(4 * g, 4 * g + 4)
            assert len(set(b.coarse[rows].tolist())) == 1
            assert sorted(b.subface[rows].tolist()) == [0, 1, 2, 3]


def test_errors_and_dump_roundtrip():
    with pytest.raises(ConfigurationError):
        build_uniform_mesh((0.0, 1.0), (2, 2))
    with pytest.raises(ConfigurationError):
        build_uniform_mesh((1.0, 1.0), (0, 2))
    with pytest.raises(ConfigurationError):
        build_uniform_mesh((1.0, 1.0, 1.0), (2, 2))
    with pytest.raises(MeshError):
        ForestMesh(2, (1.0, 1.0), (1, 1), [(0, (0, 0)), (0, (0, 0))])
    m = refine_region(build_uniform_mesh((1.0, 2.0), (2, 3), periodic=(True, False)),
                      lambda lf: lf.index in (0, 3), 1)
    back = restore_mesh(dump_mesh(m))
    assert back.leaves == m.leaves and back.periodic == m.periodic
    assert back.fingerprint == m.fingerprint
    with pytest.raises(ConfigurationError):
        restore_mesh("not-a-mesh 9\n")


def test_vectorised_refinement_matches_predicate_form():
    base = build_uniform_mesh((20.0e3, 10.0e3), (16, 8))
    a = refine_region(base, lambda lf: lf.center[1] < 3.0e3, 1)
    b = refine_region(base, lambda i, l, o, lo, hi: 0.5 * (lo[:, 1] + hi[:, 1]) < 3.0e3, 1,
                      vectorized=True)
    assert a.leaves == b.leaves


@pytest.mark.parametrize("r", [1, 2, 3, 4, 6])
def test_basis_tables(r):
    x = gauss_lobatto(r + 1)
    assert x[0] == 0.0 and x[-1] == 1.0 and np.all(np.diff(x) > 0)
    qx, qw = gauss_legendre(r + 1)
    for p in range(2 * r + 2):
        assert abs((qw * qx ** p).sum() - 1.0 / (p + 1)) < 1e-13
    b = make_basis(2, r)
    poly = np.polynomial.Polynomial(np.random.default_rng(0).normal(size=r + 1))
    assert np.abs(b.interp_1d @ poly(b.nodes_1d) - poly(b.quad_x)).max() < 1e-12
    assert np.abs(b.diff_1d @ poly(b.nodes_1d) - poly.deriv()(b.quad_x)).max() < 1e-11
    # derived device tables: B^-1, collocation derivative, lift vectors
    assert np.allclose(b.Binv @ b.interp_1d, np.eye(r + 1), atol=1e-12)
    assert np.allclose(b.Dhat @ b.interp_1d, b.diff_1d, atol=1e-11)
    assert np.allclose(b.lift @ b.interp_1d, np.eye(r + 1)[[0, r]], atol=1e-12)


@pytest.mark.parametrize("dim,r", [(2, 3), (3, 2), (3, 4)])
def test_mortar_exact(dim, r):
    b = make_basis(dim, r)
    rng = np.random.default_rng(1)
    coef = rng.normal(size=(r + 1,) * (dim - 1))
    nodes = b.nodes_1d

    def f(*xs):
        out = 0.0
        for idx in np.ndindex(coef.shape):
            t = coef[idx]
            for a, i in enumerate(idx):
                t = t * xs[a] ** i
            out = out + t
        return out

    grid = np.meshgrid(*([nodes] * (dim - 1)), indexing="ij")
    vals = f(*grid).ravel()
    for sf in range(2 ** (dim - 1)):
        pts = [0.5 * (b.quad_x + ((sf >> i) & 1)) for i in range(dim - 1)]
        exact = f(*np.meshgrid(*pts, indexing="ij")).ravel()
        assert np.abs(b.mortar_interp[sf] @ vals - exact).max() < 1e-12
    assert np.allclose(lagrange_eval_matrix(nodes, nodes), np.eye(r + 1))


def test_cfg5_recipe():
    """BASELINE configs[4]: periodic box, a seeded 7% of the
    roots refined once -> about 30% of the interior face rows hanging;
    hydrostatic state + smooth 1e-3 perturbations."""
    from paper_2408_08129_b200.cases import baseline_case
    c = baseline_case("cfg5_r3", root_scale=0.05)
    top = c.mesh.topology
    assert all(c.mesh.periodic) and c.geometry.basis.degree == 3
    assert top.n_boundary_faces() == 0
    n_conf = sum(len(b.left) for b in top.conforming)
    n_rows = sum(len(b.coarse) for b in top.hanging)
    frac = n_rows / (n_conf + n_rows)
    assert 0.2 < frac < 0.4, frac
    assert np.isfinite(c.U0).all() and c.U0.shape == (c.mesh.n_leaves, 5, 64)


def _topo_equal(a, b):
    assert len(a.conforming) == len(b.conforming)
    for x, y in zip(a.conforming, b.conforming):
        assert x.axis == y.axis
        assert np.array_equal(x.left, y.left) and np.array_equal(x.right, y.right)
    assert len(a.hanging) == len(b.hanging)
    for x, y in zip(a.hanging, b.hanging):
        assert (x.axis, x.orient) == (y.axis, y.orient)
        assert np.array_equal(x.coarse, y.coarse) and np.array_equal(x.fine, y.fine)
        assert np.array_equal(x.subface, y.subface)
    assert len(a.boundary) == len(b.boundary)
    for x, y in zip(a.boundary, b.boundary):
        assert (x.axis, x.side) == (y.axis, y.side) and np.array_equal(x.leaves, y.leaves)


@pytest.mark.parametrize("name", ["cfg1", "cfg2", "hang2d", "hang3d", "per3d", "per3d_r4",
                                  "cfg5s", "cfg3s"])
def test_native_topology_matches_numpy(name):
    """libdg's C++ face-topology builder (csrc/dg_topology.cu; SURVEY §8 f1,
    orodg/mesh.py:178-242) gives the numpy builder's batches array by array
    on every fixture mesh (uniform, hanging 2D / 3D, periodic, two levels)."""
    from casebuild import build
    from paper_2408_08129_b200.build import build as build_lib
    build_lib(verbose=False)          # no-op when libdg.so is up to date
    m = build(name).mesh
    native = m._build_topology_native()
    assert native is not None, "libdg.so not loadable"
    _topo_equal(native, m._build_topology_numpy())


def test_native_topology_large_and_rejects_bad_mesh():
    """A quarter-scale cfg4 recipe (39 k leaves, 3 levels, terrain-free
    topology) matches; a mesh violating 2:1 balance makes the native builder
    decline so that the numpy builder raises the reference's MeshError."""
    import time
    from paper_2408_08129_b200.cases import baseline_case
    from paper_2408_08129_b200.errors import MeshError
    from paper_2408_08129_b200.build import build as build_lib
    from paper_2408_08129_b200.mesh import ForestMesh
    build_lib(verbose=False)
    m = baseline_case("cfg4", root_scale=0.125, with_state=False).mesh
    t0 = time.perf_counter()
    native = m._build_topology_native()
    t1 = time.perf_counter()
    ref = m._build_topology_numpy()
    t2 = time.perf_counter()
    assert native is not None
    _topo_equal(native, ref)
    print(f"{m.n_leaves} leaves: native {t1 - t0:.3f} s, numpy {t2 - t1:.3f} s")
    # level-0 leaf next to level-2 leaves: 2:1 violated
    leaves = [(0, (0, 0))] + [(2, (4 + i, j)) for i in range(4) for j in range(4)]
    bad = ForestMesh(2, (2.0, 1.0), (2, 1), leaves)
    assert bad._build_topology_native() is None
    with pytest.raises(MeshError):
        bad.topology
