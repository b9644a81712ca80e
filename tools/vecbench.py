"""Gram-Schmidt multi-dot bandwidth vs the number of basis vectors.

    python tools/vecbench.py [--n 160358400] [--stride-pad 416]
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
    out = (C.c_double * 40)()
    ctx.bind_stream()
    for nv in (1, 4, 8, 12, 16, 24, 31):
        for _ in range(2):
            lib.dg_dots(ctx.handle, n, nv, C.c_void_p(V.data_ptr()), vs, C.c_void_p(w.data_ptr()), out)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(a.reps):
            lib.dg_dots(ctx.handle, n, nv, C.c_void_p(V.data_ptr()), vs, C.c_void_p(w.data_ptr()), out)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / a.reps
        gbs = 8.0 * n * (nv + 1) / (ms * 1e-3) / 1e9
        print(json.dumps({"nv": nv, "ms": ms, "GB_s": gbs, "pad": a.pad}), flush=True)


if __name__ == "__main__":
    main()
