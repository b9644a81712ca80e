"""CPU-side checks of the drop-in boundary: libdg.so loads without a GPU,
exports every symbol include/dg.h declares, and the host-side table
builders produce consistent element-centric face records."""

import ctypes
import os
import re

import numpy as np
import pytest

from casebuild import build

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_2408_08129_b200", "libdg.so")
HDR = os.path.join(ROOT, "include", "dg.h")


def _declared():
    txt = open(HDR).read()
    return sorted(set(re.findall(r"^(?:int|long long|const char\*)\s+(dg_\w+)\(", txt, re.M)))


@pytest.fixture(scope="module")
def lib():
    if not os.path.exists(LIB):
        from paper_2408_08129_b200.build import build as b
        b()
    return ctypes.CDLL(LIB)


def test_header_and_binding_agree():
    from paper_2408_08129_b200 import _lib
    assert _declared() == sorted(_lib.EXPORTS)


def test_library_exports_every_declared_symbol(lib):
    for name in _declared():
        assert hasattr(lib, name), name
    lib.dg_version.restype = ctypes.c_int
    assert lib.dg_version() >= 100


def test_split_contiguous_c_matches_reference_rule(lib):
    from oracle.dg_oracle import split_contiguous
    f = lib.dg_split_contiguous
    f.argtypes = [ctypes.c_void_p, ctypes.c_longlong, ctypes.c_int, ctypes.c_void_p]
    rng = np.random.default_rng(0)
    for n, p in [(10, 4), (1000, 7), (5120, 8), (3, 5)]:
        for w in (np.ones(n), rng.uniform(0.5, 2.0, n)):
            out = np.zeros(p + 1, dtype=np.int64)
            assert f(w.ctypes.data, n, p, out.ctypes.data) == 0
            assert list(out) == list(split_contiguous(w, p))


@pytest.mark.parametrize("name", ["cfg1", "hang2d", "hang3d", "per3d", "cfg3s"])
def test_face_tables_cover_topology(name):
    from paper_2408_08129_b200 import _lib as L
    from paper_2408_08129_b200.device import face_tables
    c = build(name)
    kind, nbr, hang, ffU, ffp, ffh = face_tables(c.mesh, c.bcs, c.model, c.geom.basis)
    d = c.geom.dim
    k4 = kind & 15
    topo = c.mesh.topology
    # every interior conforming face is seen from both sides, consistently
    for bt in topo.conforming:
        a = bt.axis
        assert np.all(nbr[bt.left, 2 * a + 1] == bt.right)
        assert np.all(nbr[bt.right, 2 * a] == bt.left)
    # every fine leaf points at its coarse parent; groups list the children
    S = 2 ** (d - 1)
    for bt in topo.hanging:
        fs = 1 - bt.orient
        assert np.all(k4[bt.fine, 2 * bt.axis + fs] == L.FACE_FINE)
        assert np.all((kind[bt.fine, 2 * bt.axis + fs] >> 4) == bt.subface)
        g = nbr[bt.coarse[::S], 2 * bt.axis + bt.orient]
        for s in range(S):
            rows = bt.subface[:] == s
            assert np.array_equal(np.sort(hang[g][:, s]), np.sort(bt.fine[rows]))
    nb = sum(len(b.leaves) for b in topo.boundary)
    assert int(np.sum((k4 == L.FACE_WALL) | (k4 == L.FACE_FARFIELD))) == nb
    assert ffU.shape[0] == nb
