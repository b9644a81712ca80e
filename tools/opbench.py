"""Operator microbenchmark: explicit residual and Helmholtz apply throughput
on a BASELINE recipe (cfg4 3D hill by default), timed with CUDA events.

    python tools/opbench.py [--case cfg4] [--scale 0.25] [--reps 10]

Prints one JSON line per operator: DoF/s, ms per apply, algorithmic GB/s
and the fraction of the measured HBM copy bandwidth (MEASURED_PEAKS.json).
Used for ncu captures (one short command, one GPU).
"""

import argparse
import ctypes as C
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--case", default="cfg4")
    ap.add_argument("--scale", type=float, default=0.25)
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--ops", default="explicit,helmholtz,grad,divhv")
    a = ap.parse_args()
    import numpy as np
    import torch

    from paper_2408_08129_b200 import _lib as L
    from paper_2408_08129_b200.cases import baseline_case, energy_like
    from paper_2408_08129_b200.device import DeviceContext, as_ptr

    c = baseline_case(a.case, root_scale=a.scale)
    ctx = DeviceContext(c.geometry, c.model, c.bcs, c.sponge)
    h = ctx.handle
    lib = ctx.lib
    dev = torch.device("cuda:0")
    U = torch.from_numpy(c.U0).to(dev)
    nn = c.geometry.basis.n_nodes
    d = c.mesh.dim
    n_el = c.mesh.n_leaves
    R = torch.empty_like(U)
    x = torch.from_numpy(energy_like(c.U0, 1)).to(dev)
    y = torch.empty_like(x)
    hh = torch.empty_like(x)
    K = torch.empty_like(x)
    V = torch.empty((n_el, d, nn), dtype=torch.float64, device=dev)
    dv = torch.empty((n_el, 1, nn), dtype=torch.float64, device=dev)
    ctx.bind_stream()
    lib.dg_frozen_coefficients(h, as_ptr(U), as_ptr(hh), as_ptr(K))
    with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
        peak = float(json.load(f)["hbm_gbs"])
    # fp64 FMA peak measured on this box (tools/dfma_peak), else the spec
    # figure at the max clock (SURVEY.md §8d placeholder)
    fp64 = float(os.environ.get("DG_FP64_TFLOPS", "37.2"))
    N = n_el * nn
    # SURVEY.md §8d models: algorithmic bytes and sum-factorised flops
    n, NV = c.geometry.basis.degree + 1, d + 2
    top = c.mesh.topology
    n_conf = sum(len(b.left) for b in top.conforming)
    n_hrow = sum(len(b.coarse) for b in top.hanging)
    n_bdry = top.n_boundary_faces()
    Pv, Pf = 2.0 * n ** (d + 1), 2.0 * n ** d
    Sf = 2 * n_conf + n_hrow + (d - 1) * n_hrow + n_bdry
    nnz = d if not c.geometry.terrain else (3 if d == 2 else 5)
    f_exp = NV * (3 * d * n_el * Pv + 2 * Pf * Sf)
    f_helm = n_el * (3 * d + nnz) * Pv + 2 * (d + 1) * Pf * Sf
    b_exp = 8.0 * N * NV * (3 if c.sponge is not None else 2)
    ops = {
        "explicit": (lambda: lib.dg_explicit_residual(h, as_ptr(U), as_ptr(R), None),
                     N * (d + 2), b_exp, f_exp),
        # the action GMRES applies: h frozen (prepared once)
        "helmholtz": (lambda: lib.dg_helmholtz_apply_prepared(h, 0.3, as_ptr(hh), as_ptr(x),
                                                              as_ptr(y)),
                      N, 8.0 * N * (3 + 2 * d), f_helm),
        # + the per-call preparation of h (the unprepared drop-in entry point)
        "helmholtz_full": (lambda: lib.dg_helmholtz_apply(h, 0.3, as_ptr(hh), as_ptr(x),
                                                          as_ptr(y)),
                           N, 8.0 * N * (3 + 2 * d), f_helm),
        "grad": (lambda: lib.dg_gradient_scalar(h, as_ptr(x), 1, as_ptr(V)),
                 N, 8.0 * N * (1 + d), 0.0),
        "divhv": (lambda: lib.dg_divergence_hv(h, as_ptr(V), V.stride(0), as_ptr(hh), 1,
                                               as_ptr(dv)), N, 8.0 * N * (d + 2), 0.0),
    }
    rhs = torch.empty_like(x)
    lib.dg_helmholtz_apply(h, 0.3, as_ptr(hh), as_ptr(x), as_ptr(rhs))
    x0 = torch.empty_like(x)

    def gm():
        x0.copy_(x)
        x0.mul_(1.0 + 1e-6)
        st = L.KrylovStatsC()
        return lib.dg_gmres_helmholtz(h, 0.3, as_ptr(hh), as_ptr(rhs), as_ptr(x0), 1e-8, 30, 1000,
                                      C.byref(st), None, 0)
    ops["gmres"] = (gm, N, 0.0, 0.0)
    s = torch.cuda.current_stream()
    for name in a.ops.split(","):
        fn, dofs, byts, flops = ops[name]
        for _ in range(3):
            L.check(fn())
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        for _ in range(a.reps):
            fn()
        e1.record(s)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / a.reps
        gbs = byts / (ms * 1e-3) / 1e9
        tf = flops / (ms * 1e-3) / 1e12
        # roofline: T_roof = max(B / BW, F / P_fp64)
        t_roof = max(byts / (peak * 1e9), flops / (fp64 * 1e12)) * 1e3
        print(json.dumps({"op": name, "case": a.case, "n_el": n_el, "degree": c.geometry.basis.degree,
                          "dof": dofs, "ms": ms, "dofs_per_s": dofs / (ms * 1e-3), "GB_s": gbs,
                          "frac_hbm": gbs / peak, "TFLOP_s": tf, "frac_fp64": tf / fp64,
                          "bound": "hbm" if byts / (peak * 1e9) >= flops / (fp64 * 1e12) else "fp64",
                          "roofline_ms": t_roof, "frac_roofline": t_roof / ms if ms else None,
                          "launch": ctx.launch_info()}), flush=True)


if __name__ == "__main__":
    main()
