"""Smallest end-to-end invocation of the hot path for compute-sanitizer
(one tool per GPU call, B200_PROFILING.md): explicit residual, Helmholtz
action and one ARS(2,2,2) step on the named golden-fixture cases, plus a
two-rank loopback step (halo packs / unpacks, face-row plans).

    compute-sanitizer --tool memcheck python tools/sanitize_case.py cfg1 hang3d
"""

import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))


def main():
    import numpy as np

    from casebuild import build
    from paper_2408_08129_b200.cases import energy_like
    from paper_2408_08129_b200.dgops import DGOperators
    from paper_2408_08129_b200.distributed import LoopbackGroup
    from paper_2408_08129_b200.imex import (ImplicitSolveConfig, SplitOperators, ars222,
                                            build_helmholtz_action, imex_step)
    names = sys.argv[1:] or ["cfg1"]
    for name in names:
        c = build(name)
        split = SplitOperators(DGOperators(c.geom), c.model, c.bcs, c.sponge)
        R = split.explicit_residual(c.U)
        x = energy_like(c.U, 3)
        y = build_helmholtz_action(split, c.a_dt, c.U)(x.ravel())
        cfg = ImplicitSolveConfig(krylov_tol=c.krylov_tol)
        U1, st = imex_step(c.U, 0.0, c.dt or 0.5, ars222(), split, cfg)
        grp = LoopbackGroup(c.geom, c.model, c.bcs, c.sponge, 2)
        U2, _ = grp.imex_step(grp.scatter(c.U), 0.0, c.dt or 0.5, cfg)
        err = float(np.linalg.norm(grp.gather(U2) - np.asarray(U1)) / np.linalg.norm(U1))
        print(f"{name}: |R| {np.linalg.norm(R):.6e} |y| {np.linalg.norm(y):.6e} "
              f"krylov {st.krylov_iters} loopback-vs-single {err:.1e}", flush=True)


if __name__ == "__main__":
    main()
