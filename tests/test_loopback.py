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


_CHILD_LEAN = r"""
import json, sys
sys.path.insert(0, %r); sys.path.insert(0, %r)
import numpy as np
from casebuild import build, golden, rel
from paper_2408_08129_b200.dgops import DGOperators
from paper_2408_08129_b200.distributed import LoopbackGroup
from paper_2408_08129_b200.imex import ImplicitSolveConfig, SplitOperators, ars222, imex_step
out = {}
for name, P in (("hang3d", 3), ("hang2d", 3), ("per3d", 2), ("hang3d_r4", 2)):
    c = build(name)
    z = golden(name)
    dt = float(z["dt"]) if "dt" in z else (c.dt or (0.05 if name == "per3d" else 0.5))
    cfg = ImplicitSolveConfig(krylov_tol=c.krylov_tol)
    split = SplitOperators(DGOperators(c.geom), c.model, c.bcs, c.sponge)
    U_ref, st_ref = imex_step(c.U, 0.0, dt, ars222(), split, cfg)
    res = {}
    for lean in (True, False):
        grp = LoopbackGroup(c.geom, c.model, c.bcs, c.sponge, P, lean=lean)
        grp.halo_values(reset=True)
        U, sts = grp.imex_step(grp.scatter(c.U), 0.0, dt, cfg)
        res[lean] = (rel(grp.gather(U), np.asarray(U_ref)), sts[0].krylov_iters,
                     sum(grp.halo_values()))
    out[name] = {"err_lean": res[True][0], "err_whole": res[False][0],
                 "iters": [res[True][1], res[False][1], st_ref.krylov_iters],
                 "values_lean": res[True][2], "values_whole": res[False][2]}
print(json.dumps(out))
"""


def test_loopback_face_row_halo():
    """The Helmholtz pair's halo as face rows (x face nodes, psi rows, the
    coarse parents' V trace slots) against whole ghost
    elements: the same step as the single domain with every ghost row
    poisoned with NaN before each lean exchange (DG_HALO_POISON=1: a kernel
    reading an unshipped ghost value would poison the state), at a fraction
    of the exchanged volume."""
    import json
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ)
    env["DG_HALO_POISON"] = "1"
    code = _CHILD_LEAN % (root, os.path.join(root, "tests"))
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True,
                       timeout=900)
    assert r.returncode == 0, r.stderr[-3000:]
    res = json.loads(r.stdout.strip().splitlines()[-1])
    for name, v in res.items():
        record(name, "loopback_lean_halo_step_vs_single_domain", [v["err_lean"]], [1e-12])
        assert v["err_lean"] <= 1e-12 and v["err_whole"] <= 1e-12, (name, v)
        assert v["iters"][0] == v["iters"][2] and v["iters"][1] == v["iters"][2], (name, v)
        assert v["values_lean"] < 0.5 * v["values_whole"], (name, v)
        print(f"{name}: halo doubles per step lean {v['values_lean']} vs whole "
              f"{v['values_whole']} ({v['values_whole'] / v['values_lean']:.1f}x)")


def test_distributed_solver_world_of_one():
    """bench.py's N > 1 driver (DistributedSolver: gloo control plane, NCCL
    unique-id broadcast, halo + face-row plans, dg_imex_step per rank) run
    with a world of one rank: the same step as the single-domain API."""
    import os
    import socket
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    code = r"""
import json, sys
sys.path.insert(0, %r)
import numpy as np, torch
from paper_2408_08129_b200.cases import baseline_case
from paper_2408_08129_b200.dgops import DGOperators
from paper_2408_08129_b200.distributed import DistributedSolver
from paper_2408_08129_b200.imex import ImplicitSolveConfig, SplitOperators, ars222, imex_step
case = baseline_case("cfg1")
cfg = ImplicitSolveConfig(**case.solve)
sol = DistributedSolver(case, cfg, 0, 1, 0)
U, st = sol.step(sol.local_state(), 0.0)
split = SplitOperators(DGOperators(case.geometry), case.model, case.bcs, case.sponge)
Ur, sr = imex_step(case.U0, 0.0, case.dt, ars222(), split, cfg)
err = float(np.linalg.norm(U.cpu().numpy() - Ur) / np.linalg.norm(Ur))
print(json.dumps({"err": err, "it": [list(st.krylov_iters), list(sr.krylov_iters)]}))
""" % root
    env = dict(os.environ, MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK="0",
               WORLD_SIZE="1", LOCAL_RANK="0")
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True,
                       timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    import json
    v = json.loads(r.stdout.strip().splitlines()[-1])
    record("cfg1", "distributed_solver_world1_step", [v["err"]], [1e-13])
    assert v["err"] <= 1e-13 and v["it"][0] == v["it"][1], v
