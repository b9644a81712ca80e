"""Benchmark of the B200 IMEX-DG hot path (driver contract: one JSON line).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]
                    [--workload cfg4|cfg3|cfg2|cfg1]

Workload (config.workload): BASELINE.json configs[3], the 3D Gaussian hill
on the 3-level non-conforming hex mesh (2,505,600 cells, r=3, 801.8 M DoF),
the configuration the metric is quoted on at 1/2/4/8 B200.  A step is one
ARS(2,2,2) IMEX step (2 explicit residuals + the pressure fixed point with
its GMRES solves).  metric = fp64 DoF/s per IMEX step (all d+2 variables),
value = whole-job throughput with the state resident in HBM; e2e = the same
through the public imex_step API with the state copied host->device and
back every step.  The state is 6.4 GB >> 126 MB L2, so no flush is needed.

--impl reference times the REAL reference (orodg from baseline/_ref, its own
public API, WorkerPool over the physical cores, BLAS single-threaded as its
CLI sets it) on a bounded sample of the same recipe: a central 6x6x20-root
window of the cfg4 mesh around the hill (6,264 cells, 2.0 M DoF).  The B200
line carries the same sample timed on one host core (cpu_baseline, kind
"reference") and on the GPU (same_problem: same inputs, same first step,
both sides' iteration counts).
"""

import argparse
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--workload", default="cfg4", choices=["cfg4", "cfg3", "cfg2", "cfg1"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    return ap.parse_args()


DESC = {
    "cfg4": "BASELINE configs[3]: 3D flow over a Gaussian hill (400 m, a=3 km), 60x60x20 km, "
            "120x120x20 roots refined below 6 km and 2 km (3 levels, 2,505,600 hexes), r=3, "
            "N=0.01 1/s, U=10 m/s, far-field+sponge, dt=0.5 s",
    "cfg3": "BASELINE configs[2]: 2D Schar orography, 220,800 cells, r=4",
    "cfg2": "BASELINE configs[1]: 2D warm bubble 64x32 + z<5 km refined, r=4, tol 1e-10",
    "cfg1": "BASELINE configs[0]: 2D warm bubble 32x16, r=2",
}


# ----------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md)."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.rows = []
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        import statistics
        sm = [float(r[0]) for r in self.rows if r and r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if len(r) > 1 and r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        for r in self.rows:
            for k, nm in enumerate(names):
                if len(r) > 3 + k and r[3 + k].lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": sorted(reasons),
                "samples": len(self.rows)}


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def traffic(workload, kernel_class, algorithmic_per_launch):
    """DRAM bytes per launch of the dominant kernel class, DERIVED from the
    committed `ncu --set full` capture of this round (profiles/r2_traffic.json,
    else r1): the capture's measured dram__bytes_read + write over its
    algorithmic bytes, applied to this run's per-launch algorithmic bytes (the
    class's launches differ in size, e.g. the coarse-face kernels).  Returns
    (bytes or None, source)."""
    for name in ("r2_traffic.json", "r1_traffic.json"):
        try:
            with open(os.path.join(ROOT, "profiles", name)) as f:
                t = json.load(f)[workload][kernel_class]
            ratio = float(t["measured_bytes"]) / float(t["algorithmic_bytes"])
            return algorithmic_per_launch * ratio, f"derived: profiles/{name} (ncu) ratio {ratio:.3f}"
        except Exception:
            continue
    return None, "none"


# ------------------------------------------------------------ CPU baseline
# The like-for-like sample: a central n x n x 20-root window of the cfg4
# recipe (cases.baseline_case("cfg4w<n>")), built and stepped by the REAL
# reference (orodg, installed in baseline/_ref; /root/reference/pkg/src in
# the build container) through its own public API -- build_uniform_mesh,
# refine_region, build_geometry, project_initial_data, farfield_bcs,
# sponge_sigma, DGOperators(geometry, WorkerPool(P)), SplitOperators,
# imex_step -- and by the B200 path on the same inputs.  The oracle port
# (oracle/dg_oracle.py) is the fallback only when orodg is not importable.
WINDOW = {"cfg4": 6, "cfg3": None, "cfg2": None, "cfg1": None}


def _import_reference():
    for p in (os.path.join(ROOT, "baseline", "_ref"), "/root/reference/pkg/src"):
        if os.path.isdir(os.path.join(p, "orodg")):
            if p not in sys.path:
                sys.path.insert(0, p)
            import orodg  # noqa: F401
            return p
    return None


def physical_cores():
    try:
        from orodg.parallel import physical_cores as pc
        return pc()
    except Exception:
        return os.cpu_count() or 1


def reference_case(workload, workers):
    """(split, U0, dt, dof, desc) of the workload's bounded sample, built
    with the reference's own API."""
    import numpy as np
    from orodg import cases as rc
    from orodg import imex as ri
    from orodg.boundary import wall_everywhere
    from orodg.dgops import DGOperators
    from orodg.field import project_initial_data
    from orodg.geometry import build_geometry
    from orodg.mesh import build_uniform_mesh, refine_region
    from orodg.parallel import WorkerPool
    from orodg.physics import FlowModel
    model = FlowModel.dimensional()
    pool = WorkerPool(workers)
    if workload == "cfg4":
        n = WINDOW["cfg4"]
        ext = (500.0 * n, 500.0 * n, 20.0e3)
        mesh = build_uniform_mesh(ext, (n, n, 20))
        mesh = refine_region(mesh, lambda lf: lf.center[2] < 6.0e3, 1)
        mesh = refine_region(mesh, lambda lf: lf.center[2] < 2.0e3, 1)
        xc, yc = ext[0] / 2, ext[1] / 2

        def hill(x, y):  # BASELINE configs[3] hill (cases.gaussian_hill)
            return 400.0 * np.exp(-(((x - xc) ** 2 + (y - yc) ** 2) / 3.0e3 ** 2))

        geom = build_geometry(mesh, 3, terrain=hill)
        hc = rc.HillCaseConfig(domain=ext, x_c=xc, y_c=yc)
        bg = project_initial_data(geom, rc.hydrostatic_initial_state(hc)).data
        bcs = rc.farfield_bcs(geom, bg)
        sigma = rc.sponge_sigma(geom, rc.SpongeConfig(), ext, lateral_axes=())
        split = ri.SplitOperators(DGOperators(geom, pool), model, bcs, sponge=(sigma, bg))
        U0, dt = bg.copy(), 0.5
        desc = (f"central {n}x{n}x20-root window of the cfg4 recipe ({mesh.n_leaves} cells, "
                f"r=3, top sponge; the lateral sponge lies outside the window)")
        cfg = ri.ImplicitSolveConfig()
    elif workload in ("cfg1", "cfg2"):
        root = (32, 16) if workload == "cfg1" else (64, 32)
        mesh = build_uniform_mesh((20.0e3, 10.0e3), root)
        if workload == "cfg2":
            mesh = refine_region(mesh, lambda lf: lf.center[1] < 5.0e3, 1)
        geom = build_geometry(mesh, 2 if workload == "cfg1" else 4)
        from paper_2408_08129_b200.cases import warm_bubble_state
        U0 = project_initial_data(geom, warm_bubble_state()).data
        split = ri.SplitOperators(DGOperators(geom, pool), model, wall_everywhere(mesh))
        dt = 0.5
        desc = f"{workload} (full size)"
        cfg = ri.ImplicitSolveConfig(krylov_tol=1e-8 if workload == "cfg1" else 1e-10)
    else:
        raise ValueError(f"no reference sample for {workload}")
    dof = U0.size
    return split, U0, dt, dof, desc, cfg, pool


def reference_steps(workload, workers, n_steps, warmup=0, budget_s=240.0):
    """Time n_steps ARS(2,2,2) steps of the real reference on the sample.
    The whole run (warm-up included) is bounded by budget_s: a step of the
    cfg4 window takes ~17-21 s on the host cores, so a long --steps K ends
    early after the steps that fit (>= 1; the line reports how many)."""
    import time as _t
    from orodg import imex as ri
    split, U, dt, dof, desc, cfg, pool = reference_case(workload, workers)
    tab = ri.ars222()
    t = 0.0
    start = _t.perf_counter()
    last = 0.0
    for k in range(warmup):
        if k > 0 and _t.perf_counter() - start + 2.0 * last > 0.25 * budget_s:
            break
        t0 = _t.perf_counter()
        U, st = ri.imex_step(U, t, dt, tab, split, cfg)
        last = _t.perf_counter() - t0
        t += dt
    secs, kry = [], []
    for _ in range(n_steps):
        if secs and _t.perf_counter() - start + secs[-1] > budget_s:
            break
        t0 = _t.perf_counter()
        U, st = ri.imex_step(U, t, dt, tab, split, cfg)
        secs.append(_t.perf_counter() - t0)
        kry.append((list(st.fp_iters), list(st.krylov_iters)))
        t += dt
    pool.close()
    return {"seconds": secs, "dof": dof, "desc": desc, "iterations": kry}


def port_step_sample(workload, budget_s=30.0):
    """Fallback when orodg is not importable: the numpy oracle port on the
    same sample (one step, one thread)."""
    from oracle import dg_oracle as O
    from paper_2408_08129_b200.cases import baseline_case
    name = f"cfg4w{WINDOW['cfg4']}" if workload == "cfg4" else workload
    c = baseline_case(name)
    ops = O.Operators(c.geometry, c.model, c.bcs, c.sponge)
    t0 = time.perf_counter()
    U, st = O.imex_step(ops, c.U0, 0.0, c.dt, **{k: v for k, v in c.solve.items()})
    t = time.perf_counter() - t0
    return {"seconds": [t], "dof": c.U0.size, "desc": c.description,
            "iterations": [(list(st.fp_iters), list(st.krylov_iters))]}


def cpu_sample(workload, workers, n_steps=1, warmup=0):
    """(result dict, kind) -- the real reference when importable, else the port."""
    if _import_reference() is not None:
        return reference_steps(workload, workers, n_steps, warmup), "reference"
    return port_step_sample(workload), "port"


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    os.environ.setdefault("OMP_NUM_THREADS", "1")
    os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
    from threadpoolctl import threadpool_limits
    _import_reference()
    workers = physical_cores()
    with threadpool_limits(1):  # the reference's own setting (cli.py:7-8)
        res, kind = cpu_sample(args.workload, workers, args.steps, args.warmup)
    secs = res["seconds"]
    ms = 1e3 * sum(secs) / len(secs)
    value = res["dof"] * len(secs) / sum(secs)
    line = {"metric": "fp64 DoF/s per ARS(2,2,2) IMEX-RK step (all variables)",
            "value": value, "unit": "DoF/s", "n_gpus": args.gpus, "steps": len(secs),
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "impl": "reference",
            "config": {"workload": args.workload, "description": DESC[args.workload],
                       "sample": res["desc"], "iterations": res["iterations"]},
            "cpu_baseline": {"value": value, "unit": "DoF/s", "cores": workers, "kind": kind,
                             "sample": res["desc"] + f"; {len(secs)} timed steps, WorkerPool("
                                                     f"{workers}) threads, BLAS 1 thread"},
            "e2e": {"value": value, "unit": "DoF/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def same_problem(workload, dev, cpu):
    """The B200 path on the CPU baseline's own sample (same recipe, same
    inputs, same first step through the public imex_step with host buffers):
    the like-for-like ratio, with both sides' iteration counts."""
    import numpy as np
    import torch
    from paper_2408_08129_b200.cases import baseline_case
    from paper_2408_08129_b200.dgops import DGOperators
    from paper_2408_08129_b200.imex import ImplicitSolveConfig, SplitOperators, ars222, imex_step
    name = f"cfg4w{WINDOW['cfg4']}" if workload == "cfg4" else workload
    c = baseline_case(name)
    split = SplitOperators(DGOperators(c.geometry), c.model, c.bcs, c.sponge)
    cfg = ImplicitSolveConfig(**c.solve)
    U0 = np.ascontiguousarray(c.U0)
    # first step (the one the CPU timed), repeated from the same host state
    U1, st = imex_step(U0, 0.0, c.dt, ars222(), split, cfg)
    torch.cuda.synchronize()
    reps = 5
    t0 = time.perf_counter()
    for _ in range(reps):
        U1, st = imex_step(U0, 0.0, c.dt, ars222(), split, cfg)
    torch.cuda.synchronize()
    t = (time.perf_counter() - t0) / reps
    gpu = U0.size / t
    return {"workload": name, "description": c.description, "dof": int(U0.size),
            "gpu_e2e_dofs_per_s": gpu, "gpu_seconds_per_step": t,
            "gpu_iterations": [list(st.fp_iters), list(st.krylov_iters)],
            "cpu_dofs_per_s": cpu["value"], "cpu_kind": cpu["kind"], "cpu_cores": cpu["cores"],
            "cpu_iterations": cpu["iterations"][0] if cpu.get("iterations") else None,
            "speedup_vs_1_core": gpu / cpu["value"],
            "note": "one GPU vs one host core, both stepping the same first ARS(2,2,2) step "
                    "of the same sample through their public imex_step (GPU: numpy in, numpy "
                    "out, host<->device copies included)"}


# ------------------------------------------------------------------ B200
def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    import numpy as np
    import torch

    from paper_2408_08129_b200 import _lib as L
    from paper_2408_08129_b200.cases import baseline_case
    from paper_2408_08129_b200.imex import ImplicitSolveConfig, ars222, imex_step

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device(f"cuda:{local}")

    t_setup = time.perf_counter()
    case = baseline_case(args.workload)
    cfg = ImplicitSolveConfig(**case.solve)
    if world > 1:
        from paper_2408_08129_b200.distributed import DistributedSolver
        solver = DistributedSolver(case, cfg, rank, world, local)
        U = solver.local_state()
        step = solver.step
        n_dof_local = solver.n_owned * case.geometry.basis.n_nodes * (case.mesh.dim + 2)
    else:
        from paper_2408_08129_b200.dgops import DGOperators
        from paper_2408_08129_b200.imex import SplitOperators
        ops = DGOperators(case.geometry)
        split = SplitOperators(ops, case.model, case.bcs, case.sponge)
        U = torch.from_numpy(case.U0).to(dev)
        tab = ars222()

        def step(U, t):
            return imex_step(U, t, case.dt, tab, split, cfg)
        n_dof_local = U.numel()
    setup_s = time.perf_counter() - t_setup
    # whole-job DoF (the partition is uneven by up to one leaf per rank)
    n_dof = case.mesh.n_leaves * case.geometry.basis.n_nodes * (case.mesh.dim + 2)

    def max_over_ranks(v, op="max"):
        if world == 1:
            return v
        import torch.distributed as dist
        tt = torch.tensor([float(v)], dtype=torch.float64)  # gloo: host tensors
        dist.all_reduce(tt, op=dist.ReduceOp.MAX if op == "max" else dist.ReduceOp.SUM)
        return float(tt)

    def barrier():
        if world > 1:
            import torch.distributed as dist
            dist.barrier()
        torch.cuda.synchronize()

    # warm-up (also triggers every lazy allocation)
    t = 0.0
    kry = []
    for _ in range(args.warmup):
        U, st = step(U, t)
        t += case.dt
    barrier()
    lib = L.lib()
    n0 = lib.dg_launch_count()
    stream = torch.cuda.current_stream()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clocks:
        barrier()
        ev0.record(stream)
        for _ in range(args.steps):
            U, st = step(U, t)
            kry.append((list(st.fp_iters), list(st.krylov_iters)))
            t += case.dt
        ev1.record(stream)
        barrier()
    ms_total = ev0.elapsed_time(ev1)
    launches = lib.dg_launch_count() - n0
    # per-class kernel times: a SEPARATE pass after the timed region (an event
    # pair around every launch; its overhead stays out of `value`)
    import ctypes as C
    n_prof = max(1, min(args.steps, 3))
    Up, tp = U, t
    lib.dg_profile_enable(1)
    ev2, ev3 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev2.record(stream)
    for _ in range(n_prof):
        Up, _ = step(Up, tp)
        tp += case.dt
    ev3.record(stream)
    barrier()
    ms_prof_total = ev2.elapsed_time(ev3)
    ms_c = (C.c_double * 6)()
    by_c = (C.c_double * 6)()
    cnt = (C.c_longlong * 6)()
    lib.dg_profile_read(ms_c, by_c, cnt)
    lib.dg_profile_enable(0)
    del Up
    ms_total = max_over_ranks(ms_total)
    ms_step = ms_total / args.steps
    value = n_dof * args.steps / (ms_total * 1e-3)

    # dominant kernel class over the timed region
    classes = L.PROFILE_CLASSES
    k_dom = max(range(6), key=lambda k: ms_c[k])
    peak, peak_kind = peaks()
    per_launch_ms = ms_c[k_dom] / max(cnt[k_dom], 1)
    per_launch_bytes = by_c[k_dom] / max(cnt[k_dom], 1)
    achieved = per_launch_bytes / (per_launch_ms * 1e-3) / 1e9
    # per class: algorithmic GB/s over the class's launches and its fraction
    # of the HBM peak (explicit: the north-star explicit-operator figure;
    # gradient + div_hv: the Helmholtz pair, div_hv incl. its fused dots)
    breakdown = {}
    for k in range(6):
        gbs = (by_c[k] / (ms_c[k] * 1e-3) / 1e9) if ms_c[k] else None
        breakdown[classes[k]] = {"ms": ms_c[k], "launches": int(cnt[k]), "GB_s": gbs,
                                 "frac_hbm": (gbs / peak) if gbs else None,
                                 "ms_per_launch": (ms_c[k] / cnt[k]) if cnt[k] else None}

    # e2e through the public API with host buffers (each rank: its local
    # state copied host->device, the step, the result copied back)
    Uh = torch.empty(U.shape, dtype=torch.float64, pin_memory=True)
    Uh.copy_(U)
    barrier()
    e0 = time.perf_counter()
    ev0.record(stream)
    ne = max(1, min(args.steps, 3))
    for _ in range(ne):
        Ud = Uh.to(dev, non_blocking=True)
        Ud, _ = step(Ud, t)
        Uh.copy_(Ud, non_blocking=True)
        torch.cuda.current_stream().synchronize()
    ev1.record(stream)
    barrier()
    ms_e2e = max_over_ranks(ev0.elapsed_time(ev1) / ne)
    wall_e2e = max_over_ranks((time.perf_counter() - e0) / ne)
    bytes_step = int(max_over_ranks(U.numel() * 8, op="sum"))
    e2e = {"value": n_dof / (ms_e2e * 1e-3), "unit": "DoF/s",
           "h2d_bytes_per_step": bytes_step, "d2h_bytes_per_step": bytes_step,
           "ms_per_step": ms_e2e, "wall_s_per_step": wall_e2e}

    cpu = None
    same = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            from threadpoolctl import threadpool_limits
            _import_reference()
            with threadpool_limits(1):
                res, kind = cpu_sample(args.workload, 1, 1)
            v = res["dof"] * len(res["seconds"]) / sum(res["seconds"])
            cpu = {"value": v, "unit": "DoF/s", "cores": 1, "kind": kind,
                   "sample": res["desc"] + "; 1 ARS(2,2,2) step from the initial state, "
                             "WorkerPool(1), BLAS 1 thread",
                   "seconds_per_step": sum(res["seconds"]) / len(res["seconds"]),
                   "iterations": res["iterations"]}
            same = same_problem(args.workload, dev, cpu)
        except Exception as err:  # pragma: no cover
            cpu = {"error": str(err)}

    if rank == 0:
        line = {
            "metric": "fp64 DoF/s per ARS(2,2,2) IMEX-RK step (all variables)",
            "value": value, "unit": "DoF/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (analytic hydrostatic background flow over the hill, "
                    "seeded recipe of SURVEY.md §8d; no dataset)",
            "config": {"workload": args.workload, "description": DESC[args.workload],
                       "n_el": case.mesh.n_leaves, "degree": case.geometry.basis.degree,
                       "dof_total": n_dof, "dt": case.dt,
                       "solver": {"fp_tol": cfg.fp_tol, "krylov_tol": cfg.krylov_tol,
                                  "restart": cfg.krylov_restart},
                       "parallelism": f"element-block partition x{world}",
                       "l2": "inputs larger than L2 (state 8 B x DoF)",
                       "iterations": kry, "setup_s": setup_s},
            "roofline": {"bound": "hbm", "kernel": classes[k_dom], "achieved": achieved,
                         "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                         "peak_kind": peak_kind,
                         "traffic": traffic(args.workload, classes[k_dom], per_launch_bytes)[0],
                         "traffic_source": traffic(args.workload, classes[k_dom],
                                                   per_launch_bytes)[1],
                         "bytes_per_launch": per_launch_bytes,
                         "ms_per_launch": per_launch_ms,
                         "share_of_step": ms_c[k_dom] / ms_prof_total},
            "kernel_breakdown": breakdown,
            "kernel_breakdown_steps": n_prof,
            "cpu_baseline": cpu,
            "same_problem": same,
            "e2e": e2e,
            "gpu_launches": int(launches),
            "clocks": clocks.summary(),
        }
        print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
