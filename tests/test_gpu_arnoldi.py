"""GPU checks of the DCGS2 Arnoldi pieces: the one-pass
update kernel against its numpy formula, and GMRES with DCGS2 (default) and
with the CGS + selective re-orthogonalisation path (DG_GMRES=cgs2) giving
the reference's iteration counts and solutions on the golden solves."""

import ctypes as C
import json
import os
import subprocess
import sys

import numpy as np
import pytest

from casebuild import build, golden, rel

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("nv", [0, 1, 5, 31])
def test_dcgs2_update_kernel(nv):
    import torch
    from paper_2408_08129_b200.device import DeviceContext
    c = build("cfg1")
    ctx = DeviceContext(c.geom, c.model, c.bcs)
    ctx.bind_stream()
    rng = np.random.default_rng(7 + nv)
    n, vs = 100003, 100003 + 45
    Q = rng.standard_normal((max(nv, 1), vs))
    u = rng.standard_normal(n)
    z = rng.standard_normal(n)
    s = rng.standard_normal(nv) * 1e-3
    g = rng.standard_normal(nv + 1)
    h = rng.standard_normal(nv + 1)
    alpha = 0.37
    coefs = np.concatenate([s, g, h, [alpha]])
    dev = torch.device("cuda:0")
    Qd = torch.from_numpy(Q).to(dev)
    ud = torch.from_numpy(u).to(dev)
    zd = torch.from_numpy(z).to(dev)
    und = torch.empty_like(zd)
    nrm = C.c_double()
    cf = (C.c_double * len(coefs))(*coefs)
    rc = ctx.lib.dg_dcgs2_update(ctx.handle, n, nv, C.c_void_p(Qd.data_ptr()), vs, cf,
                                 C.c_void_p(ud.data_ptr()), C.c_void_p(zd.data_ptr()),
                                 C.c_void_p(und.data_ptr()), C.byref(nrm))
    assert rc == 0
    Qn = Q[:nv, :n]
    q = (u - s @ Qn) / alpha
    w = (z - g[:nv] @ Qn - g[nv] * q) / alpha
    un = w - h[:nv] @ Qn - h[nv] * q
    assert rel(ud.cpu().numpy(), q) <= 1e-14
    assert rel(und.cpu().numpy(), un) <= 1e-13
    assert abs(nrm.value - un @ un) <= 1e-12 * (un @ un)


_CHILD = r"""
import json, sys
sys.path.insert(0, %r); sys.path.insert(0, %r)
import numpy as np
from casebuild import build, golden
from paper_2408_08129_b200.dgops import DGOperators
from paper_2408_08129_b200.imex import SplitOperators, build_helmholtz_action
from paper_2408_08129_b200.krylov import gmres
out = {}
for name in ("cfg1", "hang3d", "cfg2"):
    c, z = build(name), golden(name)
    ops = DGOperators(c.geom)
    split = SplitOperators(ops, c.model, c.bcs, c.sponge)
    act = build_helmholtz_action(split, float(z["a_dt"]), c.U)
    x, st = gmres(act, z["gm_rhs"].ravel(), x0=z["gm_x0"].ravel(), tol_rel=float(z["gm_tol"]))
    d = np.linalg.norm(x - z["gm_x"].ravel()) / np.linalg.norm(z["gm_x"].ravel())
    out[name] = [int(st.iterations), float(d), bool(st.converged)]
print(json.dumps(out))
"""


@pytest.mark.parametrize("mode", ["dcgs2", "cgs2"])
def test_gmres_arnoldi_variants(mode):
    env = dict(os.environ)
    if mode == "cgs2":
        env["DG_GMRES"] = "cgs2"
    else:
        env.pop("DG_GMRES", None)
    code = _CHILD % (ROOT, os.path.join(ROOT, "tests"))
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True,
                       timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    res = json.loads(r.stdout.strip().splitlines()[-1])
    for name, (it, d, conv) in res.items():
        z = golden(name)
        assert conv, name
        assert it == int(z["gm_iters"]), (name, it, int(z["gm_iters"]))
        assert d <= 1e-10, (name, d)


_CHILD_OPS = r"""
import json, sys
sys.path.insert(0, %r); sys.path.insert(0, %r)
import numpy as np
from casebuild import build, golden, per_var_rel, rel
from paper_2408_08129_b200.dgops import DGOperators
from paper_2408_08129_b200.imex import SplitOperators, build_helmholtz_action
out = {}
for name in ("hang2d", "hang3d", "per3d"):
    c, z = build(name), golden(name)
    ops = DGOperators(c.geom)
    split = SplitOperators(ops, c.model, c.bcs, c.sponge)
    R = split.explicit_residual(c.U)
    y = build_helmholtz_action(split, float(z["a_dt"]), c.U)(z["x"].ravel()).reshape(z["x"].shape)
    e = np.array(per_var_rel(R, z["explicit_residual"]))
    tol = np.maximum(1e-12, 10.0 * np.asarray(z["noise_explicit_residual"]))
    out[name] = [float(np.max(e / tol)), rel(y, z["helm_x"])]
print(json.dumps(out))
"""


@pytest.mark.parametrize("mode", ["flux", "fixup"])
def test_coarse_face_modes(mode):
    """The coarse side of hanging faces as precomputed fluxes (default) and
    as the fix-up epilogue (DG_COARSE_FLUX=0) give the same operators on the
    hanging-face golden cases."""
    env = dict(os.environ)
    if mode == "fixup":
        env["DG_COARSE_FLUX"] = "0"
    else:
        env.pop("DG_COARSE_FLUX", None)
    code = _CHILD_OPS % (ROOT, os.path.join(ROOT, "tests"))
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True,
                       timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    res = json.loads(r.stdout.strip().splitlines()[-1])
    for name, (e_exp, e_helm) in res.items():
        # explicit: per variable within the golden gate max(1e-12, 10 x the
        # reference's 1-ulp sensitivity) -- e_exp is the largest err / gate
        assert e_exp <= 1.0, (name, e_exp)
        assert e_helm <= 1e-12, (name, e_helm)


@pytest.mark.parametrize("nv", [0, 1, 7, 8, 9, 16, 31])
def test_dual_dots_kernel(nv):
    """The DCGS2 dual-dot pass (grouped by 8 vectors + tail) against numpy."""
    import torch
    from paper_2408_08129_b200.device import DeviceContext
    c = build("cfg1")
    ctx = DeviceContext(c.geom, c.model, c.bcs)
    ctx.bind_stream()
    rng = np.random.default_rng(11 + nv)
    n, vs = 200003, 200003 + 13
    Q = rng.standard_normal((max(nv, 1), vs))
    z = rng.standard_normal(n)
    u = rng.standard_normal(n)
    dev = torch.device("cuda:0")
    Qd, zd, ud = (torch.from_numpy(a).to(dev) for a in (Q, z, u))
    out = (C.c_double * (2 * (nv + 2)))()
    assert ctx.lib.dg_dual_dots(ctx.handle, n, nv, C.c_void_p(Qd.data_ptr()), vs,
                                C.c_void_p(zd.data_ptr()), C.c_void_p(ud.data_ptr()), out) == 0
    got = np.array(out[:])
    ref = []
    for i in range(nv):
        ref += [Q[i, :n] @ z, Q[i, :n] @ u]
    ref += [z @ z, z @ u, u @ z, u @ u]
    assert np.allclose(got, ref, rtol=1e-12, atol=1e-9)


_CHILD_PIPE = r"""
import json, sys
sys.path.insert(0, %r); sys.path.insert(0, %r)
import numpy as np
from casebuild import build, golden, per_var_rel, rel
from paper_2408_08129_b200.dgops import DGOperators
from paper_2408_08129_b200.imex import (ImplicitSolveConfig, SplitOperators, ars222,
                                        build_helmholtz_action, imex_step)
from paper_2408_08129_b200.krylov import gmres
out = {}
for name in ("cfg1", "hang2d", "hang3d", "per3d", "hang3d_r4", "cfg5s"):
    c, z = build(name), golden(name)
    ops = DGOperators(c.geom)
    split = SplitOperators(ops, c.model, c.bcs, c.sponge)
    act = build_helmholtz_action(split, float(z["a_dt"]), c.U)
    y = act(z["x"].ravel()).reshape(z["x"].shape)
    r = {"helm": rel(y, z["helm_x"])}
    if "gm_rhs" in z:
        x, st = gmres(act, z["gm_rhs"].ravel(), x0=z["gm_x0"].ravel(), tol_rel=float(z["gm_tol"]))
        r["gm_iters"] = [st.iterations, int(z["gm_iters"])]
        r["gm_x"] = rel(x, z["gm_x"].ravel())
    if "U_step1" in z:
        U1, st = imex_step(c.U, 0.0, float(z["dt"]), ars222(), split,
                           ImplicitSolveConfig(krylov_tol=c.krylov_tol))
        kz = z["krylov_iters"][0]
        r["step_iters"] = [st.krylov_iters, [int(v) for v in kz[kz >= 0]]]
        r["step"] = rel(U1, z["U_step1"])
    out[name] = r
print(json.dumps(out))
"""


@pytest.mark.parametrize("devarn", ["1", "2"])
def test_pipelined_helmholtz_on_golden_cases(devarn):
    """The large-problem path (persistent TMA-fed div(hV), separate dual-dot
    pass; DG_PIPE_MIN=0 forces it on the small golden meshes, odd and even
    n^d): Helmholtz action, GMRES and one step against the reference -- with
    the host-driven Arnoldi loop (the default of that path) and with the
    device-resident Arnoldi scalars forced onto it (DG_DEVARN=2)."""
    env = dict(os.environ)
    env["DG_PIPE_MIN"] = "0"
    env["DG_DEVARN"] = devarn
    code = _CHILD_PIPE % (ROOT, os.path.join(ROOT, "tests"))
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True,
                       timeout=900)
    assert r.returncode == 0, r.stderr[-3000:]
    res = json.loads(r.stdout.strip().splitlines()[-1])
    for name, v in res.items():
        assert v["helm"] <= 1e-12, (name, v)
        if "gm_iters" in v:
            assert v["gm_iters"][0] == v["gm_iters"][1] and v["gm_x"] <= 1e-10, (name, v)
        if "step" in v:
            assert v["step_iters"][0] == v["step_iters"][1] and v["step"] <= 1e-11, (name, v)


@pytest.mark.parametrize("name,steps", [("cfg2", 4), ("hang3d", 2), ("cfg1", 3)])
def test_device_arnoldi_scalars(name, steps):
    """The small-problem GMRES path keeps Hbar, the Givens QR and the stopping
    tests on the device (k_arn_pre / k_arn_post; the Givens loop of
    krylov.py:86-96) and enqueues Arnoldi steps ahead of ONE synchronisation
    per chunk: same Krylov counts and the same states as the host-driven loop
    (mode 0), far fewer synchronisations than two per Arnoldi step."""
    from paper_2408_08129_b200.dgops import DGOperators
    from paper_2408_08129_b200.imex import ImplicitSolveConfig, SplitOperators, ars222, imex_step
    c = build(name)
    ops = DGOperators(c.geom)
    split = SplitOperators(ops, c.model, c.bcs, c.sponge)
    ctx = split.ctx
    cfg = ImplicitSolveConfig(krylov_tol=c.krylov_tol)
    runs = {}
    for mode in (0, 2):
        assert ctx.lib.dg_set_arnoldi_mode(ctx.handle, mode) == 0
        s0, w0 = C.c_longlong(), C.c_longlong()
        ctx.lib.dg_arnoldi_stats(ctx.handle, C.byref(s0), C.byref(w0))
        U, its = c.U, []
        for k in range(steps):
            U, st = imex_step(U, 0.5 * k, 0.5, ars222(), split, cfg)
            its.append(list(st.krylov_iters))
        s1, w1 = C.c_longlong(), C.c_longlong()
        ctx.lib.dg_arnoldi_stats(ctx.handle, C.byref(s1), C.byref(w1))
        runs[mode] = (U, its, s1.value - s0.value, w1.value - w0.value)
    ctx.lib.dg_set_arnoldi_mode(ctx.handle, -1)
    (Uh, ih, sh, _), (Ud, idv, sd, wd) = runs[0], runs[2]
    assert ih == idv, (ih, idv)
    assert rel(Ud, Uh) <= 1e-13
    total = sum(sum(v) for v in idv)
    assert sh == 0 and 0 < sd <= max(total // 2, 2 * sum(len(v) for v in idv) + 2), (sd, total)
    print(f"{name}: {total} Arnoldi steps, {sd} synchronisations, {wd} steps enqueued past a stop")
