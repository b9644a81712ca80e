"""The multi-rank path executed on one GPU: P partitioned contexts in one
process exchange ghosts and reduce through libdg's loopback backend
(distributed.LoopbackGroup, dg_ctx_set_comm_loopback) -- the same halo
plans (partition.py:68-99), the same in-operator exchanges (psi, V traces,
x, state) and the same in-GMRES / fixed-point / positivity / mass-rate
allreduces as the NCCL backend.  Full ARS(2,2,2) steps must match the
single-domain run: identical fixed-point and Krylov counts, whole-state
relative L2 <= 1e-12."""

import numpy as np
import pytest

from casebuild import build, check_rel, record

pytestmark = pytest.mark.gpu


def _single(c, U, n_steps, dt, cfg):
    from paper_2408_08129_b200.dgops import DGOperators
    from paper_2408_08129_b200.imex import SplitOperators, ars222, imex_step
    split = SplitOperators(DGOperators(c.geom), c.model, c.bcs, c.sponge)
    stats = []
    for s in range(n_steps):
        U, st = imex_step(U, s * dt, dt, ars222(), split, cfg)
        stats.append(st)
    return U, stats


@pytest.mark.parametrize("name,P,n_steps", [("cfg1", 2, 2), ("hang3d", 2, 2), ("hang3d", 3, 2),
                                            ("hang2d", 3, 1), ("hang3d_r4", 2, 1)])
def test_loopback_imex_steps_match_single_domain(name, P, n_steps):
    from paper_2408_08129_b200.distributed import LoopbackGroup
    from paper_2408_08129_b200.imex import ImplicitSolveConfig
    c = build(name)
    dt = c.dt or 0.5
    cfg = ImplicitSolveConfig(krylov_tol=c.krylov_tol)
    U_ref, st_ref = _single(c, c.U, n_steps, dt, cfg)
    grp = LoopbackGroup(c.geom, c.model, c.bcs, c.sponge, P)
    assert sum(pl.n_owned for pl in grp.plans) == c.mesh.n_leaves
    assert all(len(pl.ghosts) > 0 for pl in grp.plans)
    U = grp.scatter(c.U)
    for s in range(n_steps):
        U, sts = grp.imex_step(U, s * dt, dt, cfg)
        for st in sts:  # every rank sees the global iteration counts
            assert st.krylov_iters == st_ref[s].krylov_iters, (s, st.krylov_iters,
                                                               st_ref[s].krylov_iters)
            assert st.fp_iters == st_ref[s].fp_iters
            assert abs(st.mass_rate - st_ref[s].mass_rate) <= 1e-9 * max(1.0, abs(st_ref[s].mass_rate))
    Ug = grp.gather(U)
    err = check_rel(name, f"loopback_P{P}_{n_steps}_steps_vs_single_domain", Ug,
                    np.asarray(U_ref), 1e-12)
    print(f"{name} P={P}: {n_steps} steps, rel L2 vs single domain {err:.2e}, "
          f"krylov {st_ref[-1].krylov_iters}")


def test_loopback_positivity_error_carries_global_element():
    """A negative density on one rank raises PositivityError on every rank
    with the same GLOBAL element index (allreduce_minloc)."""
    from paper_2408_08129_b200.distributed import LoopbackGroup
    from paper_2408_08129_b200.errors import PositivityError
    from paper_2408_08129_b200.imex import ImplicitSolveConfig
    c = build("hang3d")
    grp = LoopbackGroup(c.geom, c.model, c.bcs, c.sponge, 2)
    bad = c.U.copy()
    victim = grp.plans[1].owned[0] + 3  # a global element owned by rank 1
    bad[victim, 0, :] = -1.0
    U = grp.scatter(bad)
    with pytest.raises(PositivityError) as ei:
        grp.imex_step(U, 0.0, 0.5, ImplicitSolveConfig())
    record("hang3d", "loopback_positivity_element", [float(ei.value.element)], [float(victim)])
    assert ei.value.element == victim
