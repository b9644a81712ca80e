"""BASELINE configs[2] at full size (cfg3: 2D Schar-type orography, 220,800
quads after two hanging levels, r=4, 22 M DoF, far field + sponge) on the
GPU, through size-independent properties: linearity of the Helmholtz
action, the GMRES true residual, bitwise run-to-run determinism of the
explicit residual and of an ARS(2,2,2) step, and the same step with the
host-driven and the device-resident Arnoldi loop (this size takes the
pipelined div(hV) kernel with the device scalars and programmatic dependent
launches by default).  Its small golden sibling cfg3s is compared with the
reference in test_gpu_parity.py."""

import ctypes as C

import numpy as np
import pytest

from casebuild import check_rel

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def full():
    import torch

    from paper_2408_08129_b200.cases import baseline_case
    from paper_2408_08129_b200.dgops import DGOperators
    from paper_2408_08129_b200.imex import SplitOperators
    c = baseline_case("cfg3")
    assert c.mesh.n_leaves == 220800
    split = SplitOperators(DGOperators(c.geometry), c.model, c.bcs, c.sponge)
    U = torch.from_numpy(c.U0).to("cuda")
    return c, split, U


def test_cfg3_full_helmholtz_linear_and_gmres(full):
    import torch

    from paper_2408_08129_b200.imex import build_helmholtz_action
    from paper_2408_08129_b200.krylov import gmres
    c, split, U = full
    a_dt = c.dt * (1.0 - 1.0 / np.sqrt(2.0))
    act = build_helmholtz_action(split, a_dt, U)
    e = U[:, c.mesh.dim + 1].contiguous()
    g = torch.Generator(device="cuda").manual_seed(5)
    x = e * (1.0 + 1e-3 * torch.randn(e.shape, device="cuda", dtype=torch.float64, generator=g))
    y = e * (1.0 + 1e-3 * torch.randn(e.shape, device="cuda", dtype=torch.float64, generator=g))
    lhs = act((x + 2.0 * y).reshape(-1))
    rhs = act(x.reshape(-1)) + 2.0 * act(y.reshape(-1))
    err = float(torch.linalg.vector_norm(lhs - rhs) / torch.linalg.vector_norm(rhs))
    assert err <= 1e-13, err
    b = act(e.reshape(-1)) + 1e-3 * e.reshape(-1) * torch.randn(
        e.numel(), device="cuda", dtype=torch.float64, generator=g)
    xs, st = gmres(act, b, x0=e.reshape(-1), tol_rel=1e-8, restart=30)
    assert st.converged
    r = float(torch.linalg.vector_norm(b - act(xs)) / torch.linalg.vector_norm(b))
    assert r <= 1.01e-8, (r, st.iterations)


def test_cfg3_full_deterministic_and_arnoldi_modes(full):
    import torch

    from paper_2408_08129_b200.imex import ImplicitSolveConfig, ars222, imex_step
    c, split, U = full
    cfg = ImplicitSolveConfig(**c.solve)
    R1 = split.explicit_residual(U, 0.0)
    R2 = split.explicit_residual(U, 0.0)
    assert torch.equal(R1, R2)
    ctx = split.ctx
    out = {}
    for mode in (-1, -1, 0):       # default (device scalars) twice, then the host loop
        assert ctx.lib.dg_set_arnoldi_mode(ctx.handle, mode) == 0
        s0 = C.c_longlong()
        ctx.lib.dg_arnoldi_stats(ctx.handle, C.byref(s0), None)
        U1, st = imex_step(U, 0.0, c.dt, ars222(), split, cfg)
        s1 = C.c_longlong()
        ctx.lib.dg_arnoldi_stats(ctx.handle, C.byref(s1), None)
        out.setdefault(mode, []).append((U1, st, s1.value - s0.value))
    ctx.lib.dg_set_arnoldi_mode(ctx.handle, -1)
    (Ua, sta, sync_a), (Ub, stb, _) = out[-1]
    (Uh, sth, sync_h), = out[0]
    assert torch.equal(Ua, Ub) and sta.krylov_iters == stb.krylov_iters
    assert sta.krylov_iters == sth.krylov_iters and sta.fp_iters == sth.fp_iters
    assert sync_a > 0 and sync_h == 0          # the default path here is the device loop
    check_rel("cfg3", "step_device_vs_host_arnoldi", Ua.cpu().numpy(), Uh.cpu().numpy(), 1e-13)
    assert bool(torch.all(Ua[:, 0] > 0))
