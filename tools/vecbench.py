"""Gram-Schmidt multi-dot and update+normalise bandwidth vs the number of
basis vectors (algorithmic bytes: dots 8 n (nv+1), update 8 n (nv+2)).

    python tools/vecbench.py [--n 160358400] [--pad 416] [--ops dots,update]
"""

import argparse
import ctypes as C
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=160358400)
    ap.add_argument("--pad", type=int, default=416)
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--ops", default="dots,update")
    a = ap.parse_args()
    import torch

    from paper_2408_08129_b200 import _lib as L
    from paper_2408_08129_b200.cases import baseline_case
    from paper_2408_08129_b200.device import DeviceContext

    c = baseline_case("cfg1")
    ctx = DeviceContext(c.geometry, c.model, c.bcs)
    lib = ctx.lib
    n = a.n
    vs = ((n + 31) // 32) * 32 + a.pad
    V = torch.randn(32 * vs, dtype=torch.float64, device="cuda")
    w = torch.randn(n, dtype=torch.float64, device="cuda")
    out = (C.c_double * 80)()
    ctx.bind_stream()
    dst = torch.empty_like(w)
    coefs = (C.c_double * 32)(*([0.01] * 32))
    vp, wp, dp = C.c_void_p(V.data_ptr()), C.c_void_p(w.data_ptr()), C.c_void_p(dst.data_ptr())

    def dots(nv):
        lib.dg_dots(ctx.handle, n, nv, vp, vs, wp, out)

    def update(nv):
        lib.dg_gs_update(ctx.handle, n, nv, vp, vs, coefs, wp, 1.0, dp)

    z = torch.randn(n, dtype=torch.float64, device="cuda")
    un = torch.empty_like(w)
    nrm = C.c_double()

    def dcgs2(nv):
        cf = (C.c_double * 96)(*([0.01] * (3 * nv + 2) + [1.0]))
        lib.dg_dcgs2_update(ctx.handle, n, nv, vp, vs, cf, wp, C.c_void_p(z.data_ptr()),
                            C.c_void_p(un.data_ptr()), C.byref(nrm))

    def dual(nv):
        lib.dg_dual_dots(ctx.handle, n, nv, vp, vs, C.c_void_p(z.data_ptr()), wp, out)

    for op in a.ops.split(","):
        fn, extra = {"dots": (dots, 1), "update": (update, 2), "dcgs2": (dcgs2, 4),
                     "dual": (dual, 2)}[op]
        for nv in (1, 4, 8, 12, 16, 24, 31):
            for _ in range(2):
                fn(nv)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(a.reps):
                fn(nv)
            e1.record()
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / a.reps
            gbs = 8.0 * n * (nv + extra) / (ms * 1e-3) / 1e9
            print(json.dumps({"op": op, "nv": nv, "ms": ms, "GB_s": gbs, "pad": a.pad}),
                  flush=True)


if __name__ == "__main__":
    main()
