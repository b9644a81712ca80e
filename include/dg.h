/*
 * libdg -- C ABI of the B200-native IMEX-DG hot path (sm_100a, fp64).
 *
 * The reference (orodg, Python/numpy) has no FFI; its hot path sits behind
 * Python objects.  Each entry point below replaces one reference interface,
 * cited as orodg/<file>:<line> (= /root/reference/pkg/src/orodg/...).  The
 * Python drop-in (paper_2408_08129_b200) binds these with ctypes; see
 * INTEGRATION.md for the binding a maintainer adds on the reference side.
 *
 * Conventions
 *   - every array argument is a DEVICE pointer, caller-owned (e.g. a torch
 *     CUDA tensor's data_ptr()), C-contiguous float64 unless noted;
 *   - state arrays have the reference layout (n_el, d+2, (r+1)^d)
 *     (orodg/field.py:12); scalar fields (n_el, (r+1)^d); vector fields
 *     (n_el, d, (r+1)^d);
 *   - calls are stream-ordered on the context's stream and allocate nothing
 *     (the context owns all scratch); only calls returning host scalars
 *     synchronise;
 *   - return value: DG_OK or a DG_ERR_* code, mapped 1:1 by the Python shim
 *     onto the reference exception classes (orodg/errors.py:4-39);
 *     dg_last_error() gives the message (thread-local).
 */
#ifndef DG_H
#define DG_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
  DG_OK = 0,
  DG_ERR_CUDA = 1,        /* CUDA runtime / launch failure        -> DeviceError        */
  DG_ERR_USAGE = 2,       /* bad arguments, shapes, unsupported   -> UsageError         */
  DG_ERR_CONFIG = 3,      /* invalid configuration                 -> ConfigurationError */
  DG_ERR_POSITIVITY = 4,  /* non-positive density/pressure        -> PositivityError    */
  DG_ERR_SOLVER = 5,      /* GMRES stall / fixed point diverged   -> SolverError        */
  DG_ERR_COMM = 6         /* NCCL failure                          -> DeviceError        */
};

typedef struct dg_ctx dg_ctx;

/* Mesh, geometry, boundary and physics description (host pointers; copied).
 * Built by paper_2408_08129_b200.device from ForestMesh/MeshGeometry
 * (orodg/mesh.py:101-242, orodg/geometry.py:167-357, orodg/cases.py:127-174). */
typedef struct dg_ctx_desc {
  int dim;                 /* 2 or 3 */
  int degree;              /* r, 1..6; quadrature n_q = r+1 */
  int n_el;                /* elements owned (processed) by this context */
  int n_tot;               /* owned + ghost elements (== n_el on one rank) */
  double per_root[3];      /* extents[a] / root_counts[a] */
  double z_top;
  int terrain;             /* 0: flat; 1: col table valid */
  int n_col, col_stride;
  const int32_t* elem;     /* (n_tot, 2+dim): level, origin[dim], column id */
  const double* col;       /* (n_col, col_stride) terrain column data */
  const int32_t* nbr;      /* (n_tot, 2*dim) neighbour / boundary row / hanging group */
  const uint8_t* kind;     /* (n_tot, 2*dim) face kind (DG_FACE_*) | subface << 4 */
  const int32_t* hang_children; /* (n_hang_groups, 2^(dim-1)) fine leaves of a coarse face */
  int n_hang_groups;
  int n_bface;             /* far-field boundary face rows */
  const double* ff_U;      /* (n_bface, dim+2, n_q^(dim-1)) far-field conserved traces */
  const double* ff_p;      /* (n_bface, n_q^(dim-1)) far-field pressure traces */
  const double* ff_h;      /* (n_bface, n_q^(dim-1)) far-field enthalpy traces */
  const double* sigma;     /* (n_el, n^d) sponge rate or NULL (orodg/imex.py:155-156) */
  const double* background;/* (n_el, dim+2, n^d) sponge background or NULL */
  double gamma, gravity, inv_mach_sq, kinetic_factor;   /* FlowModel, physics.py:80-100 */
  const double* tabs;      /* 1D basis tables in the Tab<N> layout (dg_common.cuh) */
  int tabs_len;
  int device;              /* CUDA device ordinal */
} dg_ctx_desc;

enum { DG_FACE_WALL = 0, DG_FACE_FARFIELD = 1, DG_FACE_CONF = 2, DG_FACE_FINE = 3,
       DG_FACE_COARSE = 4 };

/* ImplicitSolveConfig (orodg/imex.py:95-114) */
typedef struct dg_solve_cfg {
  double fp_tol;
  int fp_max_iter;
  double krylov_tol;
  int krylov_restart;
  int krylov_max_iter;
  /* preconditioner == 1: block_jacobi with a caller-side cache (imex.py:334-342:
     cfg.preconditioner == "block_jacobi" and precond is not None); the context
     keeps the blocks, their age (solves since the last build) and rebuilds when
     age >= precond_refresh */
  int preconditioner;
  int precond_refresh;
} dg_solve_cfg;

/* KrylovStats (orodg/krylov.py:17-24) */
typedef struct dg_krylov_stats {
  int iterations;
  int restarts;
  int converged;
  int breakdown;
  double residual;
  int n_history;           /* entries written to the caller's history buffer */
} dg_krylov_stats;

#define DG_MAX_SOLVES 256
/* StepStats (orodg/imex.py:117-122) plus failure location */
typedef struct dg_step_stats {
  int n_fp;                          /* implicit stages */
  int fp_iters[8];
  int n_krylov;                      /* linear solves */
  int krylov_iters[DG_MAX_SOLVES];
  double pressure_increments[DG_MAX_SOLVES];
  double mass_rate;
  /* failure info (DG_ERR_POSITIVITY / DG_ERR_SOLVER) */
  int fail_stage;
  int fail_kind;                     /* 0 density, 1 pressure, 2 gmres, 3 fixed point */
  long long fail_element;
  int fail_node;
  double fail_value;
} dg_step_stats;

const char* dg_last_error(void);
int dg_version(void);

/* context (replaces DGOperators.__init__ + SplitOperators.__init__,
   orodg/dgops.py:35-55, orodg/imex.py:133-142) */
int dg_ctx_create(const dg_ctx_desc* desc, dg_ctx** out);
int dg_ctx_destroy(dg_ctx* ctx);
int dg_ctx_set_stream(dg_ctx* ctx, void* cuda_stream);
int dg_ctx_sync(dg_ctx* ctx);
/* per-launch record of the last operator launch: grid, threads, smem bytes */
int dg_ctx_launch_info(dg_ctx* ctx, int* grid, int* threads, long long* smem);

/* ---- weak-form operators returning duals (orodg/dgops.py:285-397) ---- */
int dg_divergence_advective(dg_ctx* ctx, const double* U, double* dual);
int dg_gradient_scalar(dg_ctx* ctx, const double* p, int homogeneous, double* dual);
int dg_divergence_hv(dg_ctx* ctx, const double* V, long long v_estride, const double* h,
                     int homogeneous, double* dual);
/* full Euler flux divergence dual (DGOperators.divergence_full, orodg/dgops.py:298-328);
   flux 1 = 'rusanov' (lambda = max |u.n| + c), 2 = 'centered' */
int dg_divergence_full(dg_ctx* ctx, const double* U, int flux, double* dual);
/* factorised mass inverse (orodg/geometry.py:372-396); ncomp comps per element */
int dg_apply_mass_inverse(dg_ctx* ctx, const double* dual, int ncomp, double* out);

/* ---- explicit residual (orodg/imex.py:144-159); mass_rate: host out or NULL */
int dg_explicit_residual(dg_ctx* ctx, const double* U, double* R, double* mass_rate);

/* ---- implicit-stage pieces (orodg/imex.py:182-242) ---- */
int dg_frozen_coefficients(dg_ctx* ctx, const double* U, double* h, double* K);
/* grad_p(x) = Minv Grad((gamma-1)(x - kf K)) -> (n_el, d, n^d) ; out_estride for
   writing straight into a state's momentum slots */
int dg_grad_p(dg_ctx* ctx, const double* x, const double* K, double* out, long long out_estride,
              const double* base, long long base_estride, double coef);
/* F(x) = e_e - a dt Minv Div_h(m_e - a dt/M^2 grad_p(x)); x may be NULL (F0) */
int dg_energy_F(dg_ctx* ctx, double a_dt, const double* h, const double* K,
                const double* m_e, long long m_estride, const double* e_e, long long e_estride,
                const double* x, double* Fx);
/* homogeneous Helmholtz action y = x - (F(x) - F(0)) (build_helmholtz_action) */
int dg_helmholtz_apply(dg_ctx* ctx, double a_dt, const double* h, const double* x, double* y);
/* prepare_divergence_hv + the action with h frozen (dgops.py:399-479,
   imex.py:221-242): dg_helmholtz_prepare interpolates h to the Gauss points
   (and its face traces) once; dg_helmholtz_apply_prepared then applies the
   homogeneous action without redoing it (re-preparing only when a different
   h was prepared since) -- the operator GMRES applies */
int dg_helmholtz_prepare(dg_ctx* ctx, const double* h);
int dg_helmholtz_apply_prepared(dg_ctx* ctx, double a_dt, const double* h, const double* x,
                                double* y);

/* ---- GMRES on the Helmholtz action (orodg/krylov.py:27-115) ---- */
int dg_gmres_helmholtz(dg_ctx* ctx, double a_dt, const double* h, const double* rhs, double* x,
                       double tol_rel, int restart, int max_iter, dg_krylov_stats* stats,
                       double* history, int history_cap);

/* right-preconditioned variant: precond != 0 applies the context's block-Jacobi
   inverse (dg_bj_build) as M in A M y = rhs, x = M y (krylov.py:27-115) */
int dg_gmres_helmholtz_pc(dg_ctx* ctx, double a_dt, const double* h, const double* rhs, double* x,
                          double tol_rel, int restart, int max_iter, int precond,
                          dg_krylov_stats* stats, double* history, int history_cap);

/* ---- block-Jacobi preconditioner (orodg/krylov.py:118-178) ----
   greedy colouring of the face-adjacency graph given as element pairs
   (element_coloring, krylov.py:118-140); host only, no device needed */
int dg_element_coloring(long long n_el, long long n_pairs, const long long* a, const long long* b,
                        long long* colors, int* n_colors);
/* colours of the owned elements (host array) used to probe the blocks */
int dg_bj_set_coloring(dg_ctx* ctx, const long long* colors, long long n_el);
/* probe + invert the diagonal blocks of the Helmholtz action at (a_dt, h)
   (block_jacobi_preconditioner, krylov.py:143-178); singular blocks become
   the identity (count returned); generation increments per build */
int dg_bj_build(dg_ctx* ctx, double a_dt, const double* h, int* n_singular,
                long long* generation);
/* out = M in (the blockwise inverse, krylov.py:175-176) */
int dg_bj_apply(dg_ctx* ctx, const double* in, double* out);
/* refresh state mirrored to the caller's cache object (_PrecondCache) */
int dg_bj_state(dg_ctx* ctx, int* valid, int* age, long long* generation);
int dg_bj_set_state(dg_ctx* ctx, int valid, int age);

/* ---- one implicit stage and one IMEX step (orodg/imex.py:252-370) ---- */
int dg_solve_implicit_stage(dg_ctx* ctx, const double* acc, const double* guess, double a_dt,
                            const dg_solve_cfg* cfg, double* iterate, dg_step_stats* stats);
int dg_imex_step(dg_ctx* ctx, const double* U, double* U_out, double t, double dt,
                 const dg_solve_cfg* cfg, dg_step_stats* stats);

/* ---- reductions / vector ops ---- */
int dg_integrate_conserved(dg_ctx* ctx, const double* U, double* out_host /* d+2 */);
/* max over the owned nodes of |U[num] / U[den]| (mask: optional uint8 per
   node, n_el x n^d) -- the runner's max |w| diagnostic and its probes
   (orodg/runner.py:247-260: w = data[:, d] / data[:, 0]); max over ranks */
int dg_max_abs_ratio(dg_ctx* ctx, const double* U, int num, int den, const uint8_t* mask,
                     double* out_host);
/* quadrature-weighted inner product of two (n_el, ncomp, n^d) fields
   (DGOperators.global_inner_product, orodg/dgops.py:491-503) */
int dg_global_inner_product(dg_ctx* ctx, const double* a, const double* b, int ncomp,
                            double* out_host);
/* Courant ingredients over the volume quadrature points (courant_numbers,
   orodg/physics.py:255-272): max sound speed, max |u|, min rho, min p */
int dg_courant_ingredients(dg_ctx* ctx, const double* U, double* out4);
int dg_check_positivity(dg_ctx* ctx, const double* U, double* min_rho, long long* at_rho,
                        double* min_p, long long* at_p);
int dg_lincomb(dg_ctx* ctx, long long n, int m, const double* coefs, const double* const* xs,
               double* y);
int dg_dots(dg_ctx* ctx, long long n, int nv, const double* V, long long vstride,
            const double* w, double* out_host /* nv+1: V_i.w, w.w */);
/* Arnoldi update + normalisation dst = (w - sum_i c_i V_i) / na (krylov.py:69-72, 81);
   w may be used as scratch */
int dg_gs_update(dg_ctx* ctx, long long n, int nv, const double* V, long long vstride,
                 const double* coefs_host, double* w, double na, double* dst);
/* DCGS2 Arnoldi update (one pass; the re-orthogonalised form of
   krylov.py:69-81): with Q_i = V + i*vstride, i < nv, and coefs_host =
   [s (nv), g (nv+1), h (nv+1), alpha]:
     q = (u - sum s_i Q_i) / alpha,  w = (z - sum_{i<nv} g_i Q_i - g_nv q) / alpha,
     u_next = w - sum_{i<nv} h_i Q_i - h_nv q;
   u <- q (in place), *norm2_host = |u_next|^2.  0 <= nv <= 31. */
int dg_dcgs2_update(dg_ctx* ctx, long long n, int nv, const double* V, long long vstride,
                    const double* coefs_host, double* u, const double* z, double* u_next,
                    double* norm2_host);

/* DCGS2 dual Gram-Schmidt dots in one streaming pass over V_0..V_{nv-1}, z, u:
   out = (V_i.z, V_i.u) for i < nv, then (z.z, z.u), (u.z, u.u) -- 2 (nv + 2)
   values, summed over ranks.  0 <= nv <= 31. */
int dg_dual_dots(dg_ctx* ctx, long long n, int nv, const double* V, long long vstride,
                 const double* z, const double* u, double* out_host);

/* ---- multi-GPU (one process per GPU) ---- */
int dg_nccl_unique_id(void* out128);
int dg_ctx_set_comm(dg_ctx* ctx, const void* unique_id128, int rank, int nranks,
                    const int32_t* send_counts, const int32_t* send_elems,
                    const int32_t* recv_counts);
/* the same partition plans between nranks contexts of ONE process (one host
   thread per context, e.g. several contexts on one GPU): ghost rows arrive by
   one cudaMemcpyAsync per peer ordered by CUDA events and host barriers, the
   allreduces sum on the host in rank order.  Every rank of `group` must call
   it (concurrently).  The executable stand-in for the NCCL path on a box with
   fewer GPUs than ranks (orodg/parallel.py has no multi-process path). */
int dg_ctx_set_comm_loopback(dg_ctx* ctx, int group, int rank, int nranks,
                             const int32_t* send_counts, const int32_t* send_elems,
                             const int32_t* recv_counts);
int dg_halo_exchange(dg_ctx* ctx, double* field, int ncomp);
/* face-row halo plans of the Helmholtz pair ("halo face-trace
   exchange"; the reference ships whole ghost leaves, orodg/partition.py:68-99
   + parallel.py): per field layout `which` (0 scalar nodal x: (n_tot, n^d),
   1 psi: (n_tot, 2d, n^(d-1)), 2 V traces: (n_tot, 2(d-1)+2d, n^(d-1))) the
   offsets in doubles of the values sent to / received from each peer rank,
   grouped by peer, both sides in the same (element, face, point) order.
   Every rank sets all three (possibly empty) after dg_ctx_set_comm*. */
int dg_ctx_set_halo_rows(dg_ctx* ctx, int which, const int64_t* send_counts /*nranks*/,
                         const int64_t* send_idx, const int64_t* recv_counts /*nranks*/,
                         const int64_t* recv_idx);
/* doubles this rank has sent in halo exchanges since creation / the last reset */
int dg_halo_stats(dg_ctx* ctx, long long* values_sent, int reset);

/* ---- instrumentation (no reference counterpart; orodg/timing.py is host-only) ----
   launches of libdg kernels since load; optional per-class CUDA-event timing
   (classes: 0 explicit, 1 gradient, 2 div(hV), 3 multi-dot, 4 axpy, 5 other) */
long long dg_launch_count(void);
int dg_profile_enable(int on);
int dg_profile_read(double* ms /*6*/, double* bytes /*6*/, long long* count /*6*/);
/* small-problem GMRES (device-resident Arnoldi scalars, the Givens loop of
   orodg/krylov.py:86-96 on the device): host synchronisations taken by the
   Arnoldi cycles so far and Arnoldi steps enqueued past a stopping step */
int dg_arnoldi_stats(dg_ctx* ctx, long long* syncs, long long* wasted_steps);
/* mode: 0 host-driven Arnoldi loop (two synchronisations per step), 1 device
   scalars below 2^24 scalar DoF (default), 2 device scalars always, -1 the
   DG_DEVARN environment default; multi-rank contexts always take mode 0 */
int dg_set_arnoldi_mode(dg_ctx* ctx, int mode);

/* ---- partitioner (orodg/partition.py:45-67): bounds has n_chunks+1 slots ---- */
int dg_split_contiguous(const double* weights, long long n, int n_chunks, long long* bounds);

/* ---- native face-topology builder (host; orodg/mesh.py:178-242, the
   ForestMesh topology): from the Morton-sorted leaves (level, integer origin
   (n, dim)) of a forest over root_counts[dim] the reference's face batches --
   conforming per axis, hanging per (axis, orient) sorted by (coarse,
   subface), boundary per (axis, side).  Returns 0, or non-zero for a mesh the
   reference rejects (tiling gap, 2:1 violation) or outside the key range; the
   Python caller then runs its numpy builder, which raises the reference's
   MeshError.  counts: n_conf[dim], n_hang[2 dim] ((axis, orient) -> 2 axis +
   orient), n_bdry[2 dim]; copy: the batches concatenated in that order. ---- */
typedef struct dg_topo dg_topo;
int dg_topology_build(int dim, const int64_t* root_counts, const uint8_t* periodic, int64_t n,
                      const int64_t* levels, const int64_t* origins, dg_topo** out);
int dg_topology_counts(const dg_topo* t, int64_t* n_conf, int64_t* n_hang, int64_t* n_bdry);
int dg_topology_copy(const dg_topo* t, int64_t* conf_left, int64_t* conf_right,
                     int64_t* hang_coarse, int64_t* hang_fine, int64_t* hang_subface,
                     int64_t* bdry_leaves);
int dg_topology_free(dg_topo* t);

#ifdef __cplusplus
}
#endif
#endif /* DG_H */
