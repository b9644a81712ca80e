// libdg runtime: context, C ABI (include/dg.h), and the native solver loops
// -- restarted GMRES (orodg/krylov.py:27-115), the pressure fixed point
// (orodg/imex.py:302-370) and the ARS(2,2,2) IMEX step (imex.py:252-299) --
// driving the fused element kernels and the streaming vector kernels on one
// CUDA stream.  One context per GPU per process; not re-entrant across host
// threads (same contract as the reference's single driving thread).
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/dg.h"
#include "dg_launch.cuh"
#include "dg_vector.cuh"
#include "dg_comm.h"
#include "dg_prof.h"
#include "dg_precond.cuh"

using namespace dg;

namespace {

thread_local std::string g_err;

int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}

#define CK(call)                                                                   \
  do {                                                                             \
    cudaError_t _e = (call);                                                       \
    if (_e != cudaSuccess)                                                         \
      return fail(DG_ERR_CUDA, std::string(#call) + ": " + cudaGetErrorString(_e)); \
  } while (0)

#define RET(call)                 \
  do {                            \
    int _r = (call);              \
    if (_r != DG_OK) return _r;   \
  } while (0)

template <typename T>
struct DevBuf {
  T* p = nullptr;
  size_t n = 0;
  cudaError_t alloc(size_t count) {
    if (count <= n && p) return cudaSuccess;
    if (p) cudaFree(p);
    p = nullptr;
    n = 0;
    if (count == 0) return cudaSuccess;
    cudaError_t e = cudaMalloc(&p, count * sizeof(T));
    if (e == cudaSuccess) n = count;
    return e;
  }
  cudaError_t upload(const T* h, size_t count) {
    cudaError_t e = alloc(count);
    if (e != cudaSuccess || count == 0) return e;
    return cudaMemcpy(p, h, count * sizeof(T), cudaMemcpyHostToDevice);
  }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    n = 0;
  }
};

}  // namespace

struct dg_ctx {
  int dim = 0, N = 0, NP = 0, V = 0, NQF = 0, S = 0;
  int n_el = 0, n_tot = 0;
  long long n_global = 0;  // global scalar-field length (sum over ranks)
  int device = 0;
  cudaStream_t stream = nullptr;
  MeshDev mesh{};
  GeoConst gc{};
  Model model{};
  std::vector<double> tabs;
  DevBuf<double> tabs_dev;  // device copy of tabs (warp-element kernel staging)
  DevBuf<int> elem, nbr, hang, clist;
  DevBuf<double> cflux;  // coarse-face fluxes (MeshDev::cflux)
  DevBuf<uint8_t> kind;
  DevBuf<double> col, ffU, ffp, ffh, sigma, bg;
  // scratch
  DevBuf<double> mass_partial, partial, redout, coef_dev, gs_part;
  double* pinned = nullptr;  // 2 * pin_half doubles: reads at [0, pin_half), coefs above
  int pin_half = 128;
  int kcap = 31;             // restart length the Krylov scratch is sized for
  int max_grid = 0;
  double* pin_coef() const { return pinned + pin_half; }
  DevBuf<double> sV;         // vector field (n_tot, d, NP)
  DevBuf<double> sh, sK, sx, srhs, spold, sw, sr, sx2, shq;  // scalar fields
  DevBuf<double> basis;      // (m+1) x (n_tot NP)
  DevBuf<double> st[6];      // state fields (n_tot, V, NP)
  // block-Jacobi preconditioner (dg_precond.cu): colouring of the owned
  // elements, inverse blocks (transposed), probe / apply scratch, refresh state
  DevBuf<int> bj_colors, bj_sing;
  int bj_ncolors = 0;
  DevBuf<double> bj_inv, sz, su;
  DevBuf<double> trV, trH;  // trace mode: face traces of V (H1 output) and of h
  DevBuf<double> psi;       // flux-trace mode: 1/2 ws h (V . n+) per face point (H1 output)
  const double* hq_for = nullptr;  // the nodal h that shq / trH were last prepared from
  DevBuf<double> pin;       // ... and the conforming neighbours' values, scattered by H1
  DevBuf<int> frec;         // 64-byte element records of the pipelined pair
  DevBuf<int> pinfix;       // (element, face, ghost) triples: pin rows fed by a ghost
  int n_pinfix = 0;
  int bj_valid = 0, bj_age = 1 << 30;
  long long bj_gen = 0;
  LaunchInfo last{};
  Comm comm;
  // device-resident Arnoldi scalars of the small-problem GMRES path
  // (dcgs2_cycle_dev): state, its pinned read-back copy, and the Krylov
  // counts of the previous time step's solves (the enqueue-ahead depth)
  DevBuf<ArnState> arn;
  ArnState* arn_host = nullptr;
  std::vector<int> arn_pred;
  long long halo_values = 0;  // doubles this rank has sent in halo exchanges
  int arn_ord = 0;
  int arn_mode = -1;  // -1: DG_DEVARN (default 1), 0 host loop, 1 small problems, 2 always
  long long arn_syncs = 0, arn_wasted = 0;
  long long scal() const { return (long long)n_tot * NP; }
  long long stat() const { return (long long)n_tot * V * NP; }
};

namespace {

// ------------------------------------------------------------------ basics
int sync_read(dg_ctx* c, const double* dev, int n, double* host) {
  CK(cudaMemcpyAsync(c->pinned, dev, n * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
  CK(cudaStreamSynchronize(c->stream));
  std::memcpy(host, c->pinned, n * sizeof(double));
  return DG_OK;
}

// a device read of arbitrary length (pageable, synchronous)
int sync_read_n(dg_ctx* c, const double* dev, int n, double* host) {
  CK(cudaMemcpyAsync(host, dev, n * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
  CK(cudaStreamSynchronize(c->stream));
  return DG_OK;
}

// global sums over ranks (in place on the device) then read to host
int reduce_read(dg_ctx* c, double* dev, int n, double* host) {
  if (c->comm.active()) {
    if (!c->comm.allreduce_sum(dev, n, c->stream)) return fail(DG_ERR_COMM, c->comm.error());
  }
  return sync_read(c, dev, n, host);
}

int halo(dg_ctx* c, double* field, int ncomp) {
  if (!c->comm.active()) return DG_OK;
  if (!c->comm.exchange(field, ncomp, c->NP, c->stream)) return fail(DG_ERR_COMM, c->comm.error());
  c->halo_values += c->comm.elem_send_count() * (long long)ncomp * c->NP;
  return DG_OK;
}

OpArgs base_args(dg_ctx* c) {
  OpArgs a;
  std::memset(&a, 0, sizeof(a));
  a.mesh = c->mesh;
  a.gc = c->gc;
  a.model = c->model;
  a.tabs = c->tabs.data();
  a.tabs_dev = c->tabs_dev.p;
  a.alpha = 1.0;
  a.coef = 1.0;
  static const int dbg = getenv("DG_DEBUG_SKIP") ? atoi(getenv("DG_DEBUG_SKIP")) : 0;
  a.dbg = dbg;
  return a;
}

// algorithmic bytes of one element-kernel launch (SURVEY.md §8d / DESIGN.md §3)
double op_bytes(dg_ctx* c, int opk, const OpArgs& a) {
  const double n = (double)c->n_el * c->NP * 8.0;
  const int d = c->dim;
  if (opk == OP_ADV) {
    double b = 2.0 * c->V * n;                                // U in, R out
    if (a.mode == OUT_MINV && a.sigma) b += c->V * n;          // sigma + (V-1) background
    return b;
  }
  if (opk == OP_GRAD) return n * (1 + (a.has_K ? 1 : 0) + d + (a.has_base ? d : 0));
  // V, h in, y out, base; + the basis vectors of fused Gram-Schmidt dots
  return n * (d + 1 + 1 + (a.has_base ? 1 : 0) + (a.gs_part ? a.gs_nv : 0));  // (dual: u = base)
}

int launch(dg_ctx* c, int opk, const OpArgs& a) {
  prof_begin(c->stream);
  cudaError_t e = (c->dim == 2) ? launch_elem_d2(c->N, opk, a, c->stream, &c->last)
                                : launch_elem_d3(c->N, opk, a, c->stream, &c->last);
  prof_end(c->stream, opk == OP_ADV ? P_ADV : (opk == OP_GRAD ? P_GRAD : P_DIVHV),
           op_bytes(c, opk, a), 1);
  if (e != cudaSuccess) return fail(DG_ERR_CUDA, std::string("element kernel: ") + cudaGetErrorString(e));
  return DG_OK;
}

CView cv(const double* p, long long es, long long cs) { return CView{p, es, cs}; }
MView mv(double* p, long long es, long long cs) { return MView{p, es, cs}; }

// ---------------------------------------------------------------- operators
int op_advective(dg_ctx* c, const double* U, double* out, int mode, double* mass_rate_host,
                 int full = 0) {
  OpArgs a = base_args(c);
  a.full = full;
  a.in = cv(U, (long long)c->V * c->NP, c->NP);
  a.out = mv(out, (long long)c->V * c->NP, c->NP);
  a.mode = mode;
  if (mode == OUT_MINV && c->sigma.p) {
    a.sigma = c->sigma.p;
    a.bg = cv(c->bg.p, (long long)c->V * c->NP, c->NP);
  }
  a.mass_partial = mass_rate_host ? c->mass_partial.p : nullptr;
  RET(launch(c, OP_ADV, a));
  if (mass_rate_host) {
    CK(reduce_cols(c->stream, c->mass_partial.p, c->last.grid, 1, c->redout.p));
    double s = 0.0;
    RET(reduce_read(c, c->redout.p, 1, &s));
    *mass_rate_host = -s;  // imex.py:148
  }
  return DG_OK;
}

// V_k = base_k + coef * [Minv] G(alpha (x - beta K))
int op_grad(dg_ctx* c, const double* x, const double* K, double alpha, double beta, int homog,
            int mode, MView out, CView base, int has_base, double coef, int out_quad = 0,
            double* tr_out = nullptr, double* psi_out = nullptr, double* pin_out = nullptr) {
  OpArgs a = base_args(c);
  a.tr_out = tr_out;
  a.psi_out = psi_out;
  a.pin_out = pin_out;
  a.frec = pin_out ? c->frec.p : nullptr;
  if (psi_out) a.trH = c->trH.p;  // psi = 1/2 ws h (V . n+): the own h traces
  a.in = cv(x, c->NP, c->NP);
  if (K) {
    a.inK = cv(K, c->NP, c->NP);
    a.has_K = 1;
  }
  a.alpha = alpha;
  a.beta = beta;
  a.homogeneous = homog;
  a.mode = mode;
  a.out = out;
  a.base = base;
  a.has_base = has_base;
  a.coef = coef;
  a.out_quad = out_quad;
  return launch(c, OP_GRAD, a);
}

// y = base + coef * [Minv] Div(h V)
struct GsFuse {  // fused Gram-Schmidt dots of the div(hV) result (gs_dots)
  const double* V = nullptr;
  long long vs = 0;
  int nv = 0;
  double* part = nullptr;
  int dual = 0;  // DCGS2: also the dots with the action's input (gs_dots)
};

int op_divhv(dg_ctx* c, CView V, const double* h, int homog, int mode, MView out, CView base,
             int has_base, double coef, int in_quad = 0, const GsFuse* gs = nullptr,
             const double* trV = nullptr, const double* trH = nullptr,
             const double* psi = nullptr, const double* pin = nullptr) {
  OpArgs a = base_args(c);
  a.trV = trV;
  a.trH = trH;
  a.psi = psi;
  a.pin = pin;
  a.frec = pin ? c->frec.p : nullptr;
  if (gs) {
    a.gsV = gs->V;
    a.gs_vs = gs->vs;
    a.gs_nv = gs->nv;
    a.gs_part = gs->part;
    a.gs_dual = gs->dual;
  }
  a.in = V;
  a.inH = cv(h, c->NP, c->NP);
  a.homogeneous = homog;
  a.mode = mode;
  a.out = out;
  a.base = base;
  a.has_base = has_base;
  a.coef = coef;
  a.in_quad = in_quad;
  return launch(c, OP_DIVHV, a);
}

// Face-trace mode of the Helmholtz pair: V and h live at the Gauss points,
// H1 writes V's face traces, H2 takes its neighbours' traces from them (no
// nodal interpolation, no tangential face passes for conforming faces)
bool psi_env_ok(dg_ctx* c) {
  static const char* env = getenv("DG_PSI");
  static const bool on = env == nullptr || std::string(env) != "0";
  return on && (c->mesh.n_coarse == 0 || c->cflux.p != nullptr);
}

bool trace_mode(dg_ctx* c) {
  // default on (the nodal path: DG_TRACE=0).  The flux-trace pair needs no
  // asynchronous staging in the general kernel, so it also enables the
  // Gauss-point storage where that kernel could not (3D r = 4)
  static const char* env = getenv("DG_TRACE");
  static const bool on = env == nullptr || std::string(env) != "0";
  return on && ((welem_enabled(c->dim, c->N) && welem_trace_ok(c->dim, c->N)) ||
                (hk_enabled(c->dim, c->N) && psi_env_ok(c)));
}

// Flux-trace (psi) mode of the trace-mode pair (dg_hkernel.cuh): H1 writes
// 1/2 ws h (V . n+) per face point, H2 sums its own and its neighbours'
// values instead of evaluating face traces, metrics and ghosts.  Needs the
// coarse faces in flux mode.  Default on (DG_PSI=0: the trace-mode pair)
bool psi_mode(dg_ctx* c) { return psi_env_ok(c) && trace_mode(c); }

// Pipelined H2 (hdiv2_kernel: persistent warps fed by cp.async.bulk; odd
// n^d blocks copied as their 16-byte aligned superset).  Default on
// (DG_PIPE=0: hdiv)
bool pipe_mode(dg_ctx* c) {
  static const char* env = getenv("DG_PIPE");
  static const bool on = env == nullptr || std::string(env) != "0";
  // small problems are launch-bound: there the non-persistent div(hV) with
  // the fused Gram-Schmidt dots (one launch fewer per Arnoldi step) wins
  static const long long min_dof =
      getenv("DG_PIPE_MIN") ? atoll(getenv("DG_PIPE_MIN")) : (1LL << 20);
  // (one-warp teams only: the stage ring is per warp)
  return on && (long long)c->n_el * c->NP >= min_dof && c->NQF <= 32;
}

// DCGS2 with the pipelined H2: the Gram-Schmidt dots in their own streaming
// pass instead of the div(hV) epilogue (DG_SEPDOTS=0 keeps them fused)
bool sep_dots(dg_ctx* c) {
  static const char* env = getenv("DG_SEPDOTS");
  static const bool on = env == nullptr || std::string(env) != "0";
  // (two-warp teams, 3D r >= 5, have no fused dots)
  return on && trace_mode(c) && psi_mode(c) && (pipe_mode(c) || c->NQF > 32);
}

// the pin buffer (zero: boundary, fine and coarse faces are never written)
// and the 32-byte face records of the pipelined H2
int setup_pin(dg_ctx* c, int psl) {
  CK(c->pin.alloc((size_t)c->n_tot * psl));
  CK(cudaMemsetAsync(c->pin.p, 0, (size_t)c->n_tot * psl * sizeof(double), c->stream));
  CK(c->frec.alloc((size_t)c->n_tot * REC_INTS));
  if (c->dim == 2)
    hk_elem_records<2><<<(c->n_tot + 255) / 256, 256, 0, c->stream>>>(
        c->nbr.p, c->kind.p, c->elem.p, c->n_tot, c->frec.p);
  else
    hk_elem_records<3><<<(c->n_tot + 255) / 256, 256, 0, c->stream>>>(
        c->nbr.p, c->kind.p, c->elem.p, c->n_tot, c->frec.p);
  CK(cudaGetLastError());
  return DG_OK;
}

bool quad_mode(dg_ctx* c) {
  // Gauss-point storage of the Helmholtz intermediate.  DG_QUAD=1 alone
  // keeps the n-deep neighbour gathers of the first version (measured
  // slower); the trace mode is its default form
  static const bool on = getenv("DG_QUAD") != nullptr;
  return (on && welem_enabled(c->dim, c->N)) || trace_mode(c);
}

int halo_elems(dg_ctx* c, double* field, int per_elem) {
  if (!c->comm.active()) return DG_OK;
  if (!c->comm.exchange(field, 1, per_elem, c->stream)) return fail(DG_ERR_COMM, c->comm.error());
  c->halo_values += c->comm.elem_send_count() * (long long)per_elem;
  return DG_OK;
}

// face-row halo of the flux-trace Helmholtz pair (Comm::exchange_rows):
// which = 0 x (nodal face values), 1 psi (face rows), 2 trV (the coarse
// parents' trace slots).  DG_HALO_POISON=1 first fills the ghost rows with
// NaN, so a kernel reading an unshipped ghost value shows up in the tests.
bool lean_halo(dg_ctx* c) {
  static const bool off = getenv("DG_LEAN_HALO") && std::string(getenv("DG_LEAN_HALO")) == "0";
  return !off && c->comm.active() && c->comm.has_rows();
}
int halo_rows(dg_ctx* c, double* field, int which, int per_elem) {
  static const bool poison = getenv("DG_HALO_POISON") && atoi(getenv("DG_HALO_POISON")) != 0;
  if (poison && c->n_tot > c->n_el)
    CK(cudaMemsetAsync(field + (size_t)c->n_el * per_elem, 0xFF,
                       (size_t)(c->n_tot - c->n_el) * per_elem * sizeof(double), c->stream));
  if (!c->comm.exchange_rows(field, which, c->stream)) return fail(DG_ERR_COMM, c->comm.error());
  c->halo_values += c->comm.row_send_values(which);
  return DG_OK;
}

int tr_len(dg_ctx* c) { return (2 * (c->dim - 1) + 2 * c->dim) * c->NQF; }  // V trace slots

// frozen h at the Gauss points (once per fixed-point iterate), + its face
// traces in trace mode
int interp_h(dg_ctx* c, const double* h, double* hq) {
  c->hq_for = (hq == c->shq.p) ? h : nullptr;
  AuxArgs a;
  std::memset(&a, 0, sizeof a);
  a.elem = c->elem.p;
  a.col = c->col.p;
  a.gc = c->gc;
  a.n_el = c->n_el;
  a.ncomp = 1;
  a.in = cv(h, c->NP, c->NP);
  a.out = mv(hq, c->NP, c->NP);
  a.tabs = c->tabs.data();
  const bool tm = trace_mode(c);
  if (tm) {
    CK(c->trH.alloc((size_t)c->n_tot * 2 * c->dim * c->NQF));
    a.tr = c->trH.p;
  }
  int grid = 0;
  prof_begin(c->stream);
  cudaError_t e = c->dim == 2 ? launch_aux_d2(c->N, 2, a, c->stream, &grid)
                              : launch_aux_d3(c->N, 2, a, c->stream, &grid);
  prof_end(c->stream, P_OTHER, 16.0 * c->n_el * c->NP, 1);
  CK(e);
  RET(halo(c, hq, 1));
  if (tm) RET(halo_elems(c, c->trH.p, 2 * c->dim * c->NQF));
  return DG_OK;
}

// homogeneous Helmholtz action y = x + a_dt Minv Div_h(V), V = -(a_dt/M^2)(g-1) Minv G(x).
// With hq (Gauss-point h) the intermediate V stays at the Gauss points.
int helm_apply(dg_ctx* c, double a_dt, const double* h, const double* hq, double* x, double* y,
               const GsFuse* gs = nullptr) {
  const int d = c->dim;
  const double gm1 = c->model.gamma - 1.0;
  const int qd = hq != nullptr;
  const bool tm = qd && trace_mode(c);
  const bool pm = tm && psi_mode(c);
  // flux-trace pair: the ghosts' face rows only (x face nodes, psi rows, the
  // coarse parents' trV slots) instead of whole ghost elements
  const bool lean = pm && lean_halo(c);
  if (lean) RET(halo_rows(c, x, 0, c->NP));
  else RET(halo(c, x, 1));
  if (tm) CK(c->trV.alloc((size_t)c->n_tot * tr_len(c)));
  const int psl = 2 * d * c->NQF;  // psi values per element
  const bool pp = pm && pipe_mode(c);
  if (pm) CK(c->psi.alloc((size_t)c->n_tot * psl));
  if (pp && c->pin.p == nullptr) RET(setup_pin(c, psl));
  RET(op_grad(c, x, nullptr, gm1, 0.0, 1, OUT_MINV, mv(c->sV.p, (long long)d * c->NP, c->NP),
              CView{}, 0, -(a_dt * c->model.inv_mach_sq), qd, tm ? c->trV.p : nullptr,
              pm ? c->psi.p : nullptr, pp ? c->pin.p : nullptr));
  if (lean) RET(halo_rows(c, c->psi.p, 1, psl));
  else if (pm) RET(halo_elems(c, c->psi.p, psl));   // H2 reads its neighbours' psi
  if (pp && c->n_pinfix > 0) {
    const long long nt = (long long)c->n_pinfix * c->NQF;
    hk_pin_fixup<<<(unsigned)((nt + 255) / 256), 256, 0, c->stream>>>(
        c->pinfix.p, c->n_pinfix, c->NQF, 2 * d, c->psi.p, c->pin.p);
    CK(cudaGetLastError());
  }
  if (lean) RET(halo_rows(c, c->trV.p, 2, tr_len(c)));
  else if (tm) RET(halo_elems(c, c->trV.p, tr_len(c)));  // (and the coarse parents' traces)
  else RET(halo(c, c->sV.p, d));
  RET(op_divhv(c, cv(c->sV.p, (long long)d * c->NP, c->NP), qd ? hq : h, 1, OUT_MINV,
               mv(y, c->NP, c->NP), cv(x, c->NP, c->NP), 1, a_dt, qd, gs,
               tm ? c->trV.p : nullptr, tm ? c->trH.p : nullptr, pm ? c->psi.p : nullptr,
               pp ? c->pin.p : nullptr));
  return DG_OK;
}

// the warp-element div(hV) kernel can fuse the Gram-Schmidt dots
bool gs_fusable(dg_ctx* c) {
  static const bool off = getenv("DG_GS_FUSE") && std::string(getenv("DG_GS_FUSE")) == "0";
  return !off && welem_enabled(c->dim, c->N) && (!quad_mode(c) || trace_mode(c));
}

// F(x) = e_e - a_dt Minv Div_h(m_e - a_dt/M^2 Minv G((g-1)(x - kf K)))   (imex.py:190-218)
int energy_F(dg_ctx* c, double a_dt, const double* h, const double* K, CView m_e, CView e_e,
             double* x, double* Fx) {
  const int d = c->dim;
  if (x) RET(halo(c, x, 1));
  const double gm1 = c->model.gamma - 1.0;
  RET(op_grad(c, x, K, gm1, c->model.kinetic_factor, 0, OUT_MINV,
              mv(c->sV.p, (long long)d * c->NP, c->NP), m_e, 1, -(a_dt * c->model.inv_mach_sq)));
  RET(halo(c, c->sV.p, d));
  RET(op_divhv(c, cv(c->sV.p, (long long)d * c->NP, c->NP), h, 0, OUT_MINV,
               mv(Fx, c->NP, c->NP), e_e, 1, -a_dt));
  return DG_OK;
}

// ----------------------------------------------------------------- GMRES
struct Gm {
  int iterations = 0, restarts = 0, converged = 0, breakdown = 0;
  double residual = INFINITY;
  std::vector<double> hist;
};

int norm2(dg_ctx* c, const double* x, double* out) {
  const long long n = (long long)c->n_el * c->NP;
  CK(multidot(c->stream, n, 0, nullptr, 0, x, c->partial.p, c->redout.p));
  double v;
  RET(reduce_read(c, c->redout.p, 1, &v));
  *out = v;
  return DG_OK;
}

int bj_apply_ctx(dg_ctx* c, const double* in, double* out) {
  if (!c->bj_valid) return fail(DG_ERR_USAGE, "block-Jacobi preconditioner not built");
  CK(bj_apply(c->stream, c->n_el, c->NP, c->bj_inv.p, in, out));
  return DG_OK;
}

// Krylov scratch for restart length m: the reduction partials (groups of 8
// dots per pass), the read-back and coefficient slots and the pinned staging
// are sized for m <= 31 at context creation and grown here for longer
// restarts (imex.py:96-114 accepts any krylov_restart >= 1)
int ensure_krylov_cap(dg_ctx* c, int m) {
  if (m <= c->kcap) return DG_OK;
  CK(cudaStreamSynchronize(c->stream));
  const size_t cols = (size_t)2 * (m + 4) + 9 * (size_t)((m + 9) / 8);
  CK(c->partial.alloc((size_t)RED_BLOCKS * cols + (size_t)c->max_grid * 8));
  CK(c->redout.alloc(2 * (size_t)(m + 8)));
  CK(c->coef_dev.alloc(3 * (size_t)(m + 8)));
  const int half = 3 * (m + 8);
  double* pin = nullptr;
  CK(cudaMallocHost(&pin, 2 * (size_t)half * sizeof(double)));
  cudaFreeHost(c->pinned);
  c->pinned = pin;
  c->pin_half = half;
  c->kcap = m;
  return DG_OK;
}

// One restart cycle of GMRES with DCGS2 Arnoldi (classical Gram-Schmidt with
// delayed re-orthogonalisation; Bielich et al. 2022).  Slot j of the basis
// holds the lagged vector u_j (projected once, not yet re-orthogonalised nor
// normalised) until iteration j finalises it.  Iteration j:
//   z = A u_j, and in the epilogue of the kernel producing z the dots
//   t = Q^T z, s = Q^T u_j, z.z, u_j.z, u_j.u_j  (Q = q_0..q_{j-1}, one read);
//   alpha = |u_j - Q s| (Pythagorean: s is a rounding-level correction);
//   column j-1 of Hbar gets += s, Hbar[j][j-1] = alpha (now final);
//   A q_j = (z - Q_{j+1} Hbar s) / alpha (Arnoldi relation), so its
//   projections h = (Q_{j+1}^T z - Hbar s) / alpha need no further pass;
//   ONE update pass writes q_j (in place) and u_{j+1} = A q_j - Q_{j+1} h,
//   with |u_{j+1}| as Hbar[j+1][j].
// The same Krylov space and the same re-orthogonalised basis as CGS2 (and as
// the reference's MGS + re-orthogonalisation, krylov.py:69-79, up to
// rounding); per Arnoldi step the basis is read twice instead of three times.
// Convergence, happy breakdown and max_iter tests as krylov.py:82-103 on the
// running Givens estimate; the least-squares solve at the end of the cycle
// re-factors the corrected Hbar.
int dcgs2_cycle(dg_ctx* c, double a_dt, const double* h, const double* hq, int m, int max_iter,
                double bn, double target, double beta, double* Vb, long long vs, Gm& st, std::vector<double>& g,
                std::vector<double>& y, int& done) {
  const long long n = (long long)c->n_el * c->NP;
  double* coefs = c->pin_coef();
  double* z = c->sw.p;
  std::vector<double> Hb((size_t)(m + 1) * m, 0.0), R((size_t)(m + 1) * m, 0.0);
  std::vector<double> cs(m), sn(m), dots(2 * (m + 2)), sv(m), gv(m + 1), hv(m + 1);
  auto HB = [&](int i, int j) -> double& { return Hb[(size_t)i * m + j]; };
  auto RR = [&](int i, int j) -> double& { return R[(size_t)i * m + j]; };
  done = 0;
  for (int j = 0; j < m; ++j) {
    double* u = Vb + (size_t)j * vs;
    const int nvt = 2 * (j + 2);
    if (sep_dots(c)) {
      // the pipelined div(hV) kernel streams without the dots; one dual-dot
      // pass over Q, z and u follows (dg_vector.cu k_dual_dots)
      RET(helm_apply(c, a_dt, h, hq, u, z));
      int rows = 0;
      CK(dual_dots(c->stream, n, j, Vb, vs, z, u, c->gs_part.p, &rows));
      CK(reduce_rows(c->stream, c->gs_part.p, rows, nvt, c->partial.p, c->redout.p));
    } else {
      GsFuse gs{Vb, vs, j, c->gs_part.p, 1};
      RET(helm_apply(c, a_dt, h, hq, u, z, &gs));
      CK(reduce_rows(c->stream, c->gs_part.p, c->last.grid, nvt, c->partial.p, c->redout.p));
    }
    RET(reduce_read(c, c->redout.p, nvt, dots.data()));
    // dots: (Q_i.z, Q_i.u) pairs, then (z.z, z.u), then (u.z, u.u)
    const double zz = dots[2 * j], uz = dots[2 * j + 1], uu = dots[2 * j + 3];
    double alpha = 1.0, s2 = 0.0, st_ = 0.0;
    for (int i = 0; i < j; ++i) {
      sv[i] = dots[2 * i + 1];
      s2 += sv[i] * sv[i];
      st_ += sv[i] * dots[2 * i];
    }
    if (j > 0) {
      // finalise u_j: q_j = (u_j - Q s) / alpha, and column j-1 of Hbar
      const double a2 = uu - s2;
      for (int i = 0; i < j; ++i) HB(i, j - 1) += sv[i];
      if (!(a2 > 1e-20 * uu) || !std::isfinite(a2)) {
        // u_j lies in span(Q) to rounding (or the dots are not finite): the
        // re-orthogonalised norm is the breakdown of column j-1 -- stop with
        // the j finished columns (krylov.py:82 happy-breakdown rule) instead
        // of dividing by a vanishing alpha
        HB(j, j - 1) = (a2 > 0.0 && std::isfinite(a2)) ? std::sqrt(a2) : 0.0;
        st.breakdown = 1;
        break;
      }
      alpha = std::sqrt(a2);
      HB(j, j - 1) = alpha;
    }
    // g = Hbar[0:j+1, 0:j] s
    for (int i = 0; i <= j; ++i) {
      double t = 0.0;
      for (int k = std::max(0, i - 1); k < j; ++k) t += HB(i, k) * sv[k];
      gv[i] = t;
    }
    // h = (Q_{j+1}^T z - g) / alpha, Q_{j+1}^T z = [t; (u.z - s.t) / alpha]
    for (int i = 0; i < j; ++i) hv[i] = (dots[2 * i] - gv[i]) / alpha;
    hv[j] = ((uz - st_) / alpha - gv[j]) / alpha;
    const double nb = std::sqrt(std::max(zz, 0.0)) / alpha;  // |A q_j| (breakdown scale)
    for (int i = 0; i <= j; ++i) HB(i, j) = hv[i];
    // one pass: q_j in place, u_{j+1}, |u_{j+1}|^2
    for (int i = 0; i < j; ++i) coefs[i] = sv[i];
    for (int i = 0; i <= j; ++i) coefs[j + i] = gv[i];
    for (int i = 0; i <= j; ++i) coefs[2 * j + 1 + i] = hv[i];
    coefs[3 * j + 2] = alpha;
    CK(cudaMemcpyAsync(c->coef_dev.p, coefs, (3 * j + 3) * sizeof(double),
                       cudaMemcpyHostToDevice, c->stream));
    double* un = Vb + (size_t)(j + 1) * vs;
    CK(dcgs2_update(c->stream, n, j, Vb, vs, c->coef_dev.p, u, z, un, c->partial.p,
                    c->redout.p));
    double na2;
    RET(reduce_read(c, c->redout.p, 1, &na2));
    const double na = std::sqrt(na2);
    HB(j + 1, j) = na;
    const bool happy = na <= 1e-14 * std::max(bn, nb);
    st.iterations += 1;
    // running Givens QR of the (provisional) column j
    for (int i = 0; i <= j + 1; ++i) RR(i, j) = HB(i, j);
    for (int i = 0; i < j; ++i) {
      const double t = cs[i] * RR(i, j) + sn[i] * RR(i + 1, j);
      RR(i + 1, j) = -sn[i] * RR(i, j) + cs[i] * RR(i + 1, j);
      RR(i, j) = t;
    }
    const double den = std::hypot(RR(j, j), RR(j + 1, j));
    cs[j] = den != 0.0 ? RR(j, j) / den : 1.0;
    sn[j] = den != 0.0 ? RR(j + 1, j) / den : 0.0;
    RR(j, j) = den;
    RR(j + 1, j) = 0.0;
    g[j + 1] = -sn[j] * g[j];
    g[j] = cs[j] * g[j];
    done = j + 1;
    const double est = std::fabs(g[j + 1]);
    st.hist.push_back(est / bn);
    if (happy) {
      st.breakdown = 1;
      break;
    }
    if (est <= target || st.iterations >= max_iter) break;
  }
  if (!done) return DG_OK;
  // least squares on the corrected Hbar (columns < done - 1 carry their
  // re-orthogonalisation corrections): fresh Givens QR, then back-substitution
  std::vector<double> gg(done + 1, 0.0);
  gg[0] = beta;
  for (int j = 0; j < done; ++j) {
    for (int i = 0; i <= j + 1; ++i) RR(i, j) = HB(i, j);
    for (int i = 0; i < j; ++i) {
      const double t = cs[i] * RR(i, j) + sn[i] * RR(i + 1, j);
      RR(i + 1, j) = -sn[i] * RR(i, j) + cs[i] * RR(i + 1, j);
      RR(i, j) = t;
    }
    const double den = std::hypot(RR(j, j), RR(j + 1, j));
    cs[j] = den != 0.0 ? RR(j, j) / den : 1.0;
    sn[j] = den != 0.0 ? RR(j + 1, j) / den : 0.0;
    RR(j, j) = den;
    RR(j + 1, j) = 0.0;
    gg[j + 1] = -sn[j] * gg[j];
    gg[j] = cs[j] * gg[j];
  }
  for (int i = done - 1; i >= 0; --i) {
    double t = gg[i];
    for (int k = i + 1; k < done; ++k) t -= RR(i, k) * y[k];
    y[i] = t / RR(i, i);
  }
  return DG_OK;
}

// The same cycle with the Arnoldi scalars on the device (k_arn_pre /
// k_arn_post, dg_vector.cu): steps are enqueued `ahead` at a time with ONE
// host synchronisation per chunk instead of two per step.  Steps enqueued
// past the stopping step leave the scalar state untouched (the scalar
// kernels return once `stop` is set) and only write basis slots >= done,
// which the solution update never reads.  `ahead` is the Krylov count of the
// same solve in the previous time step (c->arn_pred), so a steady run
// synchronises about once per solve.
bool devarn_mode(dg_ctx* c) {
  static const int env0 = getenv("DG_DEVARN") ? atoi(getenv("DG_DEVARN")) : 1;
  const int env = c->arn_mode >= 0 ? c->arn_mode : env0;
  // large problems keep the host loop: an Arnoldi step costs milliseconds
  // there and one enqueued past the stop more than the synchronisations
  // saved (cfg3, 4.4 M scalar DoF, 0.5 ms per Arnoldi step: 71.3 -> 68.5 ms
  // per time step with the device scalars; cfg4, 160 M: 13 ms per step)
  return env != 0 && !c->comm.active() &&
         (env == 2 || !sep_dots(c) || c->n_global < (1LL << 24));
}

int dcgs2_cycle_dev(dg_ctx* c, double a_dt, const double* h, const double* hq, int m, int max_iter,
                    double bn, double target, double beta, double* Vb, long long vs, Gm& st,
                    std::vector<double>& y, int& done, int ahead) {
  const long long n = (long long)c->n_el * c->NP;
  double* z = c->sw.p;
  CK(c->arn.alloc(1));
  if (!c->arn_host) CK(cudaMallocHost(&c->arn_host, sizeof(ArnState)));
  ArnState* A = c->arn.p;
  CK(arn_init(c->stream, A, m, bn, target, beta, st.iterations, max_iter));
  const ArnState& H = *c->arn_host;
  int j = 0, chunks = 0;
  done = 0;
  // the steps' kernels are launched as programmatic dependents of one
  // another (dg_pdl.cuh; DG_PDL=0: plain stream order)
  static const bool pdl_env = !(getenv("DG_PDL") && std::string(getenv("DG_PDL")) == "0");
  struct PdlScope {
    PdlScope(bool on) { tl_pdl = on ? 1 : 0; }
    ~PdlScope() { tl_pdl = 0; }
  } pdl_scope(pdl_env && !prof().on && !sep_dots(c));
  // (only where a kernel is a single wave: at cfg3, 4.4 M scalar DoF, the
  // early-resident dependents take SM resources from the kernel still
  // running and the step gets slower, 70.6 vs 68.4 ms)
  while (j < m) {
    int K = std::max(1, std::min(ahead, m - j));
    for (int jj = j; jj < j + K; ++jj) {
      double* u = Vb + (size_t)jj * vs;
      const int nvt = 2 * (jj + 2);
      long long rows = 0;
      if (sep_dots(c)) {
        RET(helm_apply(c, a_dt, h, hq, u, z));
        int r = 0;
        CK(dual_dots(c->stream, n, jj, Vb, vs, z, u, c->gs_part.p, &r));
        rows = r;
      } else {
        GsFuse gs{Vb, vs, jj, c->gs_part.p, 1};
        RET(helm_apply(c, a_dt, h, hq, u, z, &gs));
        rows = c->last.grid;
      }
      // few partial rows: the scalar kernel sums them itself (one launch
      // instead of three)
      if (rows <= 2048) {
        CK(arn_pre(c->stream, A, jj, c->gs_part.p, (int)rows, c->coef_dev.p));
      } else {
        CK(reduce_rows(c->stream, c->gs_part.p, rows, nvt, c->partial.p, c->redout.p));
        CK(arn_pre(c->stream, A, jj, c->redout.p, 0, c->coef_dev.p));
      }
      int nparts = 0;
      CK(dcgs2_update_partials(c->stream, n, jj, Vb, vs, c->coef_dev.p, u, z,
                               Vb + (size_t)(jj + 1) * vs, c->partial.p, &nparts));
      CK(arn_post(c->stream, A, jj, c->partial.p, nparts));
    }
    CK(cudaMemcpyAsync(c->arn_host, A, sizeof(ArnState), cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    c->arn_syncs += 1;
    j += K;
    if (H.stop) {
      c->arn_wasted += j - H.steps_run;
      break;
    }
    // the prediction was short (counts drift by a step or two between time
    // steps): single steps first -- a synchronisation is cheaper than an
    // Arnoldi step enqueued past the stop -- then small chunks
    ahead = ++chunks <= 3 ? 1 : 3;
  }
  done = H.done;
  for (int i = 0; i < H.steps_run; ++i) st.hist.push_back(H.hist[i]);
  st.iterations = H.iterations;
  if (H.breakdown) st.breakdown = 1;
  if (!done) return DG_OK;
  // least squares on the corrected Hbar, as dcgs2_cycle
  std::vector<double> R((size_t)(m + 1) * m, 0.0), cs(m), sn(m), gg(done + 1, 0.0);
  auto HB = [&](int i, int k) -> double { return H.Hb[(size_t)i * m + k]; };
  auto RR = [&](int i, int k) -> double& { return R[(size_t)i * m + k]; };
  gg[0] = beta;
  for (int k = 0; k < done; ++k) {
    for (int i = 0; i <= k + 1; ++i) RR(i, k) = HB(i, k);
    for (int i = 0; i < k; ++i) {
      const double t = cs[i] * RR(i, k) + sn[i] * RR(i + 1, k);
      RR(i + 1, k) = -sn[i] * RR(i, k) + cs[i] * RR(i + 1, k);
      RR(i, k) = t;
    }
    const double den = std::hypot(RR(k, k), RR(k + 1, k));
    cs[k] = den != 0.0 ? RR(k, k) / den : 1.0;
    sn[k] = den != 0.0 ? RR(k + 1, k) / den : 0.0;
    RR(k, k) = den;
    RR(k + 1, k) = 0.0;
    gg[k + 1] = -sn[k] * gg[k];
    gg[k] = cs[k] * gg[k];
  }
  for (int i = done - 1; i >= 0; --i) {
    double t = gg[i];
    for (int k = i + 1; k < done; ++k) t -= RR(i, k) * y[k];
    y[i] = t / RR(i, i);
  }
  return DG_OK;
}

// right-preconditioned (pc: M = block-Jacobi inverse, krylov.py:56-66,105-109)
int gmres(dg_ctx* c, double a_dt, const double* h, const double* hq, const double* rhs, double* x,
          double tol, int restart, int max_iter, Gm& st, bool pc = false) {
  if (!(tol > 0.0 && tol < 1.0)) return fail(DG_ERR_CONFIG, "tol_rel must be in (0,1)");
  const long long ns = c->scal();
  const long long n = (long long)c->n_el * c->NP;
  int m = restart < 1 ? 1 : restart;
  if (m > c->n_global) m = (int)c->n_global;
  if (m < 1) m = 1;
  RET(ensure_krylov_cap(c, m));
  // basis vectors at a padded stride: a power-of-two-rich stride makes the
  // j+1 streams of one Gram-Schmidt pass collide in the same DRAM channels
  const long long vs = ((ns + 31) / 32) * 32 + 32 * 13;
  CK(c->basis.alloc((size_t)(m + 1) * vs));
  double* Vb = c->basis.p;
  // (the fused dots' partial rows hold <= 32 + 2 column pairs: longer
  // restarts take the unfused CGS passes)
  const bool fuse = gs_fusable(c) && m <= 31;
  const bool sep = sep_dots(c) && m <= 31;
  // DCGS2 (delayed re-orthogonalisation) needs the fused dual
  // dots and u = the action's input (no preconditioner); DG_GMRES=cgs2 keeps
  // the CGS + selective re-orthogonalisation path
  static const bool cgs_env = getenv("DG_GMRES") && std::string(getenv("DG_GMRES")) == "cgs2";
  const bool dcgs2 = (fuse || sep) && !pc && !cgs_env;
  const bool devarn = dcgs2 && m <= ARN_M && devarn_mode(c);
  const int ord = c->arn_ord++;
  const int pred = (devarn && ord < (int)c->arn_pred.size()) ? c->arn_pred[ord] : 0;
  struct PredKeep {  // remember this solve's count for the next time step
    dg_ctx* c; int ord; const Gm& st; bool on;
    ~PredKeep() {
      if (!on || ord >= 64) return;
      if ((int)c->arn_pred.size() <= ord) c->arn_pred.resize(ord + 1, 0);
      c->arn_pred[ord] = st.iterations;
    }
  } keep{c, ord, st, devarn};
  if (fuse || sep) {
    // one row of <= m + 1 dot partials per element-kernel warp (>= 1 element
    // each) and per coarse element
    // (or one row per block of the separate dual-dot pass: <= RED_BLOCKS)
    const long long rows =
        std::max((long long)c->n_el + 4 + c->mesh.n_coarse + 1, (long long)RED_BLOCKS);
    CK(c->gs_part.alloc((size_t)rows * 2 * (32 + 2)));
  }
  double* coefs = c->pin_coef();  // pinned staging for the coefficient uploads
  double* w = c->sw.p;
  double* r = c->sr.p;
  double bn2;
  RET(norm2(c, rhs, &bn2));
  const double bn = std::sqrt(bn2);
  if (bn == 0.0) {
    CK(cudaMemsetAsync(x, 0, n * sizeof(double), c->stream));
    st.converged = 1;
    st.residual = 0.0;
    return DG_OK;
  }
  auto residual_into_r = [&]() -> int {
    RET(helm_apply(c, a_dt, h, hq, x, w));
    const double cf[2] = {1.0, -1.0};
    const double* xs[2] = {rhs, w};
    CK(lincomb(c->stream, n, 2, cf, xs, r));
    return DG_OK;
  };
  RET(residual_into_r());
  const double target = tol * bn;
  std::vector<double> H((size_t)(m + 1) * m, 0.0), cs(m), sn(m), g(m + 1), y(m), hc(m + 2);
  auto Hij = [&](int i, int j) -> double& { return H[(size_t)i * m + j]; };
  while (true) {
    double b2;
    RET(norm2(c, r, &b2));
    const double beta = std::sqrt(b2);
    st.residual = beta / bn;
    st.hist.push_back(st.residual);
    if (beta <= target || st.iterations >= max_iter || st.breakdown) break;
    CK(scale(c->stream, n, beta, true, r, Vb));
    std::fill(g.begin(), g.end(), 0.0);
    g[0] = beta;
    int done = 0;
    if (dcgs2 && devarn) {
      // enqueue-ahead depth: what is left of the previous time step's count
      // for this solve (first solves: a short chunk)
      // (one short of the count: the last step is confirmed by a read-back)
      const int ahead = pred > st.iterations + 1 ? pred - st.iterations - 1 : (pred > 0 ? 1 : 4);
      RET(dcgs2_cycle_dev(c, a_dt, h, hq, m, max_iter, bn, target, beta, Vb, vs, st, y, done,
                          ahead));
    } else if (dcgs2) {
      RET(dcgs2_cycle(c, a_dt, h, hq, m, max_iter, bn, target, beta, Vb, vs, st, g, y, done));
    }
    for (int j = 0; j < m && !dcgs2; ++j) {
      // classical Gram-Schmidt: h_i = V_i . w and |w|^2 in one pass,
      // fused into the div(hV) kernel that produces w when it can
      double* src = Vb + (size_t)j * vs;
      if (pc) {
        RET(bj_apply_ctx(c, src, c->sz.p));  // w = A M v_j
        src = c->sz.p;
      }
      if (fuse) {
        GsFuse gs{Vb, vs, j + 1, c->gs_part.p};
        RET(helm_apply(c, a_dt, h, hq, src, w, &gs));
        CK(reduce_rows(c->stream, c->gs_part.p, c->last.grid, j + 2, c->partial.p, c->redout.p));
      } else {
        RET(helm_apply(c, a_dt, h, hq, src, w));
        CK(multidot(c->stream, n, j + 1, Vb, vs, w, c->partial.p, c->redout.p));
      }
      RET(reduce_read(c, c->redout.p, j + 2, hc.data()));
      const double nb2 = hc[j + 1];
      const double nb = std::sqrt(nb2);
      double s2 = 0.0;
      for (int i = 0; i <= j; ++i) {
        Hij(i, j) = hc[i];
        s2 += hc[i] * hc[i];
        coefs[i] = hc[i];
      }
      CK(cudaMemcpyAsync(c->coef_dev.p, coefs, (j + 1) * sizeof(double), cudaMemcpyHostToDevice,
                         c->stream));
      double* dst = Vb + (size_t)(j + 1) * vs;
      // |w - V h|^2 = |w|^2 - |h|^2 for orthonormal V: when no more than half of
      // |w|^2 cancels (the reference's re-orthogonalisation test, krylov.py:76,
      // is then false) update and normalise in one fused pass
      const double na2_est = nb2 - s2;
      double na;
      bool happy;
      if (na2_est > 0.5 * nb2) {
        na = std::sqrt(na2_est);
        happy = na <= 1e-14 * std::max(bn, nb);
        if (!happy) CK(axpy_div(c->stream, n, j + 1, Vb, vs, c->coef_dev.p, w, na, dst));
      } else {
        // update, |w|^2 and the re-orthogonalisation dots V^T w in ONE pass
        // (the dots are only used when the norm test below asks for them)
        CK(axpy_dots(c->stream, n, j + 1, Vb, vs, c->coef_dev.p, w, c->partial.p, c->redout.p));
        RET(reduce_read(c, c->redout.p, j + 2, hc.data()));
        const double na2 = hc[j + 1];
        na = std::sqrt(na2);
        if (na < 0.7071067811865476 * nb) {
          // one re-orthogonalisation pass (krylov.py:73-79)
          double s2r = 0.0;
          for (int i = 0; i <= j; ++i) {
            Hij(i, j) += hc[i];
            coefs[i] = hc[i];
            s2r += hc[i] * hc[i];
          }
          CK(cudaMemcpyAsync(c->coef_dev.p, coefs, (j + 1) * sizeof(double),
                             cudaMemcpyHostToDevice, c->stream));
          const double nr2 = na2 - s2r;  // |w - V h2|^2, Pythagorean (h2 is a small correction)
          if (nr2 > 0.5 * na2) {
            na = std::sqrt(nr2);
            happy = na <= 1e-14 * std::max(bn, nb);
            if (!happy) CK(axpy_div(c->stream, n, j + 1, Vb, vs, c->coef_dev.p, w, na, dst));
          } else {
            double nr2x;
            CK(axpy_multi(c->stream, n, j + 1, Vb, vs, c->coef_dev.p, w, c->partial.p,
                          c->redout.p));
            RET(reduce_read(c, c->redout.p, 1, &nr2x));
            na = std::sqrt(nr2x);
            happy = na <= 1e-14 * std::max(bn, nb);
            if (!happy) CK(scale(c->stream, n, na, true, w, dst));
          }
        } else {
          happy = na <= 1e-14 * std::max(bn, nb);
          if (!happy) CK(scale(c->stream, n, na, true, w, dst));
        }
      }
      Hij(j + 1, j) = na;
      st.iterations += 1;
      for (int i = 0; i < j; ++i) {
        const double t = cs[i] * Hij(i, j) + sn[i] * Hij(i + 1, j);
        Hij(i + 1, j) = -sn[i] * Hij(i, j) + cs[i] * Hij(i + 1, j);
        Hij(i, j) = t;
      }
      const double den = std::hypot(Hij(j, j), Hij(j + 1, j));
      cs[j] = den != 0.0 ? Hij(j, j) / den : 1.0;
      sn[j] = den != 0.0 ? Hij(j + 1, j) / den : 0.0;
      Hij(j, j) = den;
      Hij(j + 1, j) = 0.0;
      g[j + 1] = -sn[j] * g[j];
      g[j] = cs[j] * g[j];
      done = j + 1;
      const double est = std::fabs(g[j + 1]);
      st.hist.push_back(est / bn);
      if (happy) {
        st.breakdown = 1;
        break;
      }
      if (est <= target || st.iterations >= max_iter) break;
    }
    if (done) {
      for (int i = done - 1; i >= 0 && !dcgs2; --i) {  // (dcgs2_cycle solved for y)
        double s = g[i];
        for (int k = i + 1; k < done; ++k) s -= Hij(i, k) * y[k];
        y[i] = s / Hij(i, i);
      }
      // x <- x + V y  ==  x - sum(-y_i) V_i
      for (int i = 0; i < done; ++i) coefs[i] = -y[i];
      CK(cudaMemcpyAsync(c->coef_dev.p, coefs, done * sizeof(double), cudaMemcpyHostToDevice,
                         c->stream));
      if (!pc) {
        CK(axpy_multi(c->stream, n, done, Vb, vs, c->coef_dev.p, x, c->partial.p, nullptr));
      } else {
        // x <- x + M (V y)
        CK(cudaMemsetAsync(c->su.p, 0, n * sizeof(double), c->stream));
        CK(axpy_multi(c->stream, n, done, Vb, vs, c->coef_dev.p, c->su.p, c->partial.p, nullptr));
        RET(bj_apply_ctx(c, c->su.p, c->sz.p));
        const double cf[2] = {1.0, 1.0};
        const double* xs[2] = {x, c->sz.p};
        CK(lincomb(c->stream, n, 2, cf, xs, x));
      }
    }
    RET(residual_into_r());
    st.restarts += 1;
  }
  st.restarts = std::max(0, st.restarts - 1);
  // the final true residual equals the last beta: x is unchanged since r
  st.converged = st.residual <= tol ? 1 : 0;
  return DG_OK;
}

// ------------------------------------------------ block-Jacobi (dg_precond.cu)
// probe the diagonal blocks of the homogeneous Helmholtz action at (a_dt, h)
// colour by colour, node by node (krylov.py:143-160), then invert them
int bj_build(dg_ctx* c, double a_dt, const double* h, const double* hq, int* n_sing) {
  if (c->bj_ncolors <= 0)
    return fail(DG_ERR_USAGE, "block-Jacobi: no element colouring set (dg_bj_set_coloring)");
  const long long ns = c->scal();
  const int NP = c->NP;
  CK(c->bj_inv.alloc((size_t)c->n_el * NP * NP));
  CK(c->sz.alloc(ns));
  CK(c->su.alloc(ns));
  CK(c->bj_sing.alloc(1));
  CK(cudaMemsetAsync(c->bj_sing.p, 0, sizeof(int), c->stream));
  for (int col = 0; col < c->bj_ncolors; ++col)
    for (int node = 0; node < NP; ++node) {
      CK(bj_probe(c->stream, c->n_el, NP, c->bj_colors.p, col, node, c->sz.p));
      RET(helm_apply(c, a_dt, h, hq, c->sz.p, c->su.p));
      CK(bj_scatter(c->stream, c->n_el, NP, c->bj_colors.p, col, node, c->su.p, c->bj_inv.p));
    }
  CK(bj_invert(c->stream, c->n_el, NP, c->bj_inv.p, c->bj_inv.p, c->bj_sing.p));
  int ns_local = 0;
  CK(cudaMemcpyAsync(&ns_local, c->bj_sing.p, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
  CK(cudaStreamSynchronize(c->stream));
  double tot = ns_local;
  if (c->comm.active()) {
    c->pinned[0] = tot;
    CK(cudaMemcpyAsync(c->redout.p, c->pinned, sizeof(double), cudaMemcpyHostToDevice, c->stream));
    RET(reduce_read(c, c->redout.p, 1, &tot));
  }
  if (n_sing) *n_sing = (int)tot;
  c->bj_valid = 1;
  c->bj_gen += 1;
  return DG_OK;
}

// -------------------------------------------------------- implicit stage
int check_positivity(dg_ctx* c, const double* U, dg_step_stats* stats, int stage) {
  const double gm1 = c->model.gamma - 1.0;
  CK(positivity(c->stream, c->n_el, c->NP, c->dim, U, gm1, c->model.kinetic_factor,
                c->partial.p));
  std::vector<double> part(RED_BLOCKS * 4);
  CK(cudaStreamSynchronize(c->stream));
  CK(cudaMemcpy(part.data(), c->partial.p, part.size() * sizeof(double), cudaMemcpyDeviceToHost));
  double mr = INFINITY, mp = INFINITY;
  long long ir = -1, ip = -1;
  for (int b = 0; b < RED_BLOCKS; ++b) {
    const double v = part[b * 4], iv = part[b * 4 + 1];
    if (v < mr || (v == mr && (long long)iv < ir)) { mr = v; ir = (long long)iv; }
    const double p = part[b * 4 + 2], ipv = part[b * 4 + 3];
    if (p < mp || (p == mp && (long long)ipv < ip)) { mp = p; ip = (long long)ipv; }
  }
  if (c->comm.active()) {
    // global minimum with the owning rank's global element id
    double loc[4] = {mr, (double)(ir < 0 ? -1 : c->comm.global_index(ir / c->NP) * c->NP + ir % c->NP),
                     mp, (double)(ip < 0 ? -1 : c->comm.global_index(ip / c->NP) * c->NP + ip % c->NP)};
    if (!c->comm.allreduce_minloc(loc, c->stream)) return fail(DG_ERR_COMM, c->comm.error());
    mr = loc[0]; ir = (long long)loc[1]; mp = loc[2]; ip = (long long)loc[3];
  }
  if (!(mr > 0.0) || !(mp > 0.0)) {
    const bool dens = !(mr > 0.0);
    const long long at = dens ? ir : ip;
    if (stats) {
      stats->fail_stage = stage;
      stats->fail_kind = dens ? 0 : 1;
      stats->fail_element = at / c->NP;
      stats->fail_node = (int)(at % c->NP);
      stats->fail_value = dens ? mr : mp;
    }
    char buf[256];
    std::snprintf(buf, sizeof buf, "non-positive %s (%.6e) at index (%lld, %d) in stage %d",
                  dens ? "density" : "pressure", dens ? mr : mp, at / c->NP, (int)(at % c->NP),
                  stage);
    return fail(DG_ERR_POSITIVITY, buf);
  }
  return DG_OK;
}

int solve_stage(dg_ctx* c, const double* acc, const double* guess, double a_dt,
                const dg_solve_cfg& cfg, double* it, dg_step_stats* stats, int* n_fp) {
  const int d = c->dim, NP = c->NP, V = c->V;
  const long long n = (long long)c->n_el * NP;
  const long long sst = (long long)V * NP;
  const double gm1 = c->model.gamma - 1.0, kf = c->model.kinetic_factor;
  CK(set_iterate(c->stream, c->n_el, NP, V, acc, guess, it));
  CK(state_pressure(c->stream, c->n_el, NP, d, it, gm1, kf, c->spold.p));
  CK(copy_comps(c->stream, c->n_el, NP, 1, it + (long long)(d + 1) * NP, sst, c->sx.p, NP));
  const CView m_e = cv(acc + NP, sst, NP);
  const CView e_e = cv(acc + (long long)(d + 1) * NP, sst, NP);
  double last_dp = INFINITY;
  for (int k = 0; k < cfg.fp_max_iter; ++k) {
    CK(frozen(c->stream, c->n_el, NP, d, it, gm1, kf, c->sh.p, c->sK.p));
    RET(halo(c, c->sh.p, 1));
    RET(halo(c, c->sK.p, 1));
    RET(energy_F(c, a_dt, c->sh.p, c->sK.p, m_e, e_e, nullptr, c->srhs.p));
    const double* hq = nullptr;
    if (quad_mode(c)) {
      RET(interp_h(c, c->sh.p, c->shq.p));
      hq = c->shq.p;
    }
    // block-Jacobi refresh cadence of imex.py:334-342 (age counts solves)
    bool pc = false;
    if (cfg.preconditioner == 1) {
      if (!c->bj_valid || c->bj_age >= cfg.precond_refresh) {
        RET(bj_build(c, a_dt, c->sh.p, hq, nullptr));
        c->bj_age = 0;
      }
      c->bj_age += 1;
      pc = true;
    }
    Gm gs;
    RET(gmres(c, a_dt, c->sh.p, hq, c->srhs.p, c->sx.p, cfg.krylov_tol, cfg.krylov_restart,
              cfg.krylov_max_iter, gs, pc));
    if (stats && stats->n_krylov < DG_MAX_SOLVES) stats->krylov_iters[stats->n_krylov++] = gs.iterations;
    if (!gs.converged) {
      if (stats) {
        stats->fail_kind = 2;
        stats->fail_value = gs.residual;
      }
      char buf[160];
      std::snprintf(buf, sizeof buf, "GMRES stalled: residual %.3e after %d iterations",
                    gs.residual, gs.iterations);
      return fail(DG_ERR_SOLVER, buf);
    }
    double nrm[2];
    CK(pressure_dp(c->stream, n, c->sx.p, c->sK.p, gm1, kf, c->spold.p, c->partial.p, c->redout.p));
    RET(reduce_read(c, c->redout.p, 2, nrm));
    // momentum back-substitution straight into the iterate (imex.py:356-358)
    RET(halo(c, c->sx.p, 1));
    RET(op_grad(c, c->sx.p, c->sK.p, gm1, kf, 0, OUT_MINV, mv(it + NP, sst, NP), m_e, 1,
                -(a_dt * c->model.inv_mach_sq)));
    CK(copy_comps(c->stream, c->n_el, NP, 1, c->sx.p, NP, it + (long long)(d + 1) * NP, sst));
    const double dp = std::sqrt(nrm[0]) / std::max(std::sqrt(nrm[1]), 1e-300);
    if (stats && stats->n_krylov - 1 < DG_MAX_SOLVES)
      stats->pressure_increments[stats->n_krylov - 1] = dp;
    last_dp = dp;
    if (dp <= cfg.fp_tol) {
      *n_fp = k + 1;
      return DG_OK;
    }
  }
  if (stats) {
    stats->fail_kind = 3;
    stats->fail_value = last_dp;
  }
  char buf[200];
  std::snprintf(buf, sizeof buf,
                "pressure fixed point did not converge: last increment %.3e after %d iterations",
                last_dp, cfg.fp_max_iter);
  return fail(DG_ERR_SOLVER, buf);
}

int ensure_work(dg_ctx* c) {
  const long long ns = c->scal();
  for (auto* b : {&c->sh, &c->sK, &c->sx, &c->srhs, &c->spold, &c->sw, &c->sr, &c->sx2, &c->shq})
    CK(b->alloc(ns));
  CK(c->sV.alloc((size_t)ns * c->dim));
  return DG_OK;
}

int ensure_states(dg_ctx* c) {
  for (auto& s : c->st) CK(s.alloc(c->stat()));
  return DG_OK;
}

}  // namespace

// =================================================================== C ABI
extern "C" {

const char* dg_last_error(void) { return g_err.c_str(); }
int dg_version(void) { return 100; }

int dg_ctx_create(const dg_ctx_desc* d, dg_ctx** out) {
  if (!d || !out) return fail(DG_ERR_USAGE, "null argument");
  if (d->dim != 2 && d->dim != 3) return fail(DG_ERR_USAGE, "dim must be 2 or 3");
  if (d->degree < 1 || d->degree > 6) return fail(DG_ERR_USAGE, "degree must be in 1..6 on the device path");
  if (d->n_tot < d->n_el || d->n_el < 0) return fail(DG_ERR_USAGE, "bad element counts");
  CK(cudaSetDevice(d->device));
  dg_ctx* c = new dg_ctx();
  c->device = d->device;
  c->dim = d->dim;
  c->N = d->degree + 1;
  int np = 1, nqf = 1;
  for (int a = 0; a < d->dim; ++a) np *= c->N;
  for (int a = 0; a < d->dim - 1; ++a) nqf *= c->N;
  c->NP = np;
  c->NQF = nqf;
  c->V = d->dim + 2;
  c->S = 1 << (d->dim - 1);
  c->n_el = d->n_el;
  c->n_tot = d->n_tot;
  c->n_global = (long long)d->n_el * np;
  const int N = c->N;
  const int expect_tabs = 3 * N * N + 2 * N + 4 * N * N + 3 * N;
  if (d->tabs_len != expect_tabs) {
    delete c;
    return fail(DG_ERR_USAGE, "basis table length mismatch");
  }
  c->tabs.assign(d->tabs, d->tabs + d->tabs_len);
  if (c->tabs_dev.upload(c->tabs.data(), c->tabs.size()) != cudaSuccess)
    return fail(DG_ERR_CUDA, "tables upload failed");
  auto up = [&](auto& buf, const auto* h, size_t cnt) -> cudaError_t { return buf.upload(h, cnt); };
  const size_t nf = (size_t)d->n_tot * 2 * d->dim;
  cudaError_t e = cudaSuccess;
  if (e == cudaSuccess) e = up(c->elem, d->elem, (size_t)d->n_tot * (2 + d->dim));
  if (e == cudaSuccess) e = up(c->nbr, d->nbr, nf);
  if (e == cudaSuccess) e = up(c->kind, d->kind, nf);
  if (e == cudaSuccess && d->n_hang_groups > 0)
    e = up(c->hang, d->hang_children, (size_t)d->n_hang_groups * c->S);
  if (e == cudaSuccess && d->terrain && d->n_col > 0)
    e = up(c->col, d->col, (size_t)d->n_col * d->col_stride);
  if (e == cudaSuccess && d->n_bface > 0) {
    e = up(c->ffU, d->ff_U, (size_t)d->n_bface * c->V * nqf);
    if (e == cudaSuccess) e = up(c->ffp, d->ff_p, (size_t)d->n_bface * nqf);
    if (e == cudaSuccess) e = up(c->ffh, d->ff_h, (size_t)d->n_bface * nqf);
  }
  if (e == cudaSuccess && d->sigma) {
    e = up(c->sigma, d->sigma, (size_t)d->n_el * np);
    if (e == cudaSuccess) e = up(c->bg, d->background, (size_t)d->n_el * c->V * np);
  }
  // owned elements with a coarse hanging face -> coarse fix-up kernel
  // records (MeshDev::coarse_list): [element, then per face its 2^(d-1)
  // children (fine leaves) or -1] -- the kernel reads one record instead of
  // the dependent kind -> nbr -> hang_children chain
  {
    std::vector<int> cl;
    const int nf = 2 * d->dim, S = c->S;
    int ncoarse = 0;
    for (int e2 = 0; e2 < d->n_el; ++e2) {
      bool has = false;
      for (int f = 0; f < nf; ++f)
        if ((d->kind[(size_t)e2 * nf + f] & 15) == DG_FACE_COARSE) has = true;
      if (!has) continue;
      ++ncoarse;
      cl.push_back(e2);
      for (int f = 0; f < nf; ++f)
        cl.push_back((d->kind[(size_t)e2 * nf + f] & 15) == DG_FACE_COARSE
                         ? d->nbr[(size_t)e2 * nf + f]
                         : -1);
      for (int f = 0; f < nf; ++f)
        for (int sub = 0; sub < S; ++sub)
          cl.push_back((d->kind[(size_t)e2 * nf + f] & 15) == DG_FACE_COARSE
                           ? d->hang_children[(size_t)d->nbr[(size_t)e2 * nf + f] * S + sub]
                           : -1);
    }
    if (e == cudaSuccess && !cl.empty()) e = c->clist.upload(cl.data(), cl.size());
    c->mesh.n_coarse = ncoarse;
    // owned conforming faces whose neighbour is a ghost (partitioned runs):
    // their incoming psi rows come from the halo (hk_pin_fixup)
    std::vector<int> pf;
    for (int e2 = 0; e2 < d->n_el; ++e2)
      for (int f = 0; f < nf; ++f)
        if ((d->kind[(size_t)e2 * nf + f] & 15) == DG_FACE_CONF && d->nbr[(size_t)e2 * nf + f] >= d->n_el) {
          pf.push_back(e2);
          pf.push_back(f);
          pf.push_back(d->nbr[(size_t)e2 * nf + f]);
        }
    if (e == cudaSuccess && !pf.empty()) e = c->pinfix.upload(pf.data(), pf.size());
    c->n_pinfix = (int)(pf.size() / 3);
    // coarse-face flux buffer (flux mode; DG_COARSE_FLUX=0: the coarse side
    // is added afterwards by the fix-up epilogue instead)
    static const bool cf_off =
        getenv("DG_COARSE_FLUX") && std::string(getenv("DG_COARSE_FLUX")) == "0";
    if (e == cudaSuccess && ncoarse > 0 && !cf_off)
      e = c->cflux.alloc((size_t)d->n_hang_groups * c->V * nqf);
  }
  const int max_grid = d->n_el + 1 + c->mesh.n_coarse;
  c->max_grid = max_grid;
  if (e == cudaSuccess) e = c->mass_partial.alloc(max_grid);
  if (e == cudaSuccess) e = c->partial.alloc((size_t)RED_BLOCKS * 72 + (size_t)max_grid * 8);
  if (e == cudaSuccess) e = c->redout.alloc(256);
  if (e == cudaSuccess) e = c->coef_dev.alloc(128);
  if (e == cudaSuccess) e = cudaMallocHost(&c->pinned, 256 * sizeof(double));
  if (e != cudaSuccess) {
    dg_ctx_destroy(c);
    return fail(DG_ERR_CUDA, std::string("context allocation: ") + cudaGetErrorString(e));
  }
  c->mesh.elem = c->elem.p;
  c->mesh.col = c->col.p;
  c->mesh.nbr = c->nbr.p;
  c->mesh.kind = c->kind.p;
  c->mesh.hang_children = c->hang.p;
  c->mesh.ff_U = c->ffU.p;
  c->mesh.ff_p = c->ffp.p;
  c->mesh.ff_h = c->ffh.p;
  c->mesh.n_el = d->n_el;
  c->mesh.coarse_list = c->clist.p;
  c->mesh.cflux = c->cflux.p;
  for (int a = 0; a < 3; ++a) c->gc.per_root[a] = d->per_root[a];
  c->gc.z_top = d->z_top;
  c->gc.inv_ztop = 1.0 / d->z_top;
  c->gc.terrain = d->terrain;
  c->gc.col_stride = d->col_stride;
  c->model = Model{d->gamma, d->gravity, d->inv_mach_sq, d->kinetic_factor};
  *out = c;
  return DG_OK;
}

int dg_ctx_destroy(dg_ctx* c) {
  if (!c) return DG_OK;
  cudaSetDevice(c->device);
  for (auto* b : {&c->col, &c->ffU, &c->ffp, &c->ffh, &c->sigma, &c->bg, &c->mass_partial,
                  &c->partial, &c->redout, &c->coef_dev, &c->gs_part, &c->trV, &c->trH, &c->psi, &c->pin, &c->sV, &c->sh, &c->sK, &c->sx,
                  &c->srhs, &c->spold, &c->sw, &c->sr, &c->sx2, &c->basis})
    b->release();
  for (auto& s : c->st) s.release();
  c->elem.release();
  c->frec.release();
  c->pinfix.release();
  c->clist.release();
  c->cflux.release();
  c->nbr.release();
  c->hang.release();
  c->kind.release();
  if (c->pinned) cudaFreeHost(c->pinned);
  if (c->arn_host) cudaFreeHost(c->arn_host);
  c->comm.shutdown();
  delete c;
  return DG_OK;
}

int dg_ctx_set_stream(dg_ctx* c, void* s) {
  c->stream = (cudaStream_t)s;
  return DG_OK;
}

int dg_ctx_sync(dg_ctx* c) {
  CK(cudaStreamSynchronize(c->stream));
  return DG_OK;
}

int dg_ctx_launch_info(dg_ctx* c, int* grid, int* threads, long long* smem) {
  if (grid) *grid = c->last.grid;
  if (threads) *threads = c->last.threads;
  if (smem) *smem = (long long)c->last.smem;
  return DG_OK;
}

int dg_divergence_advective(dg_ctx* c, const double* U, double* dual) {
  RET(halo(c, const_cast<double*>(U), c->V));
  return op_advective(c, U, dual, OUT_DUAL, nullptr);
}

int dg_divergence_full(dg_ctx* c, const double* U, int flux, double* dual) {
  if (flux != 1 && flux != 2) return fail(DG_ERR_CONFIG, "flux must be 1 (rusanov) or 2 (centered)");
  RET(halo(c, const_cast<double*>(U), c->V));
  return op_advective(c, U, dual, OUT_DUAL, nullptr, flux);
}

int dg_explicit_residual(dg_ctx* c, const double* U, double* R, double* mass_rate) {
  RET(halo(c, const_cast<double*>(U), c->V));
  return op_advective(c, U, R, OUT_MINV, mass_rate);
}

int dg_gradient_scalar(dg_ctx* c, const double* p, int homogeneous, double* dual) {
  RET(halo(c, const_cast<double*>(p), 1));
  return op_grad(c, p, nullptr, 1.0, 0.0, homogeneous, OUT_DUAL,
                 mv(dual, (long long)c->dim * c->NP, c->NP), CView{}, 0, 1.0);
}

int dg_divergence_hv(dg_ctx* c, const double* V, long long v_estride, const double* h,
                     int homogeneous, double* dual) {
  RET(halo(c, const_cast<double*>(h), 1));
  if (c->comm.active() && !c->comm.exchange(const_cast<double*>(V), c->dim, c->NP, c->stream, v_estride))
    return fail(DG_ERR_COMM, c->comm.error());
  return op_divhv(c, cv(V, v_estride, c->NP), h, homogeneous, OUT_DUAL, mv(dual, c->NP, c->NP),
                  CView{}, 0, 1.0);
}

int dg_apply_mass_inverse(dg_ctx* c, const double* dual, int ncomp, double* out) {
  AuxArgs a;
  std::memset(&a, 0, sizeof a);
  a.elem = c->elem.p;
  a.col = c->col.p;
  a.gc = c->gc;
  a.n_el = c->n_el;
  a.ncomp = ncomp;
  a.in = cv(dual, (long long)ncomp * c->NP, c->NP);
  a.out = mv(out, (long long)ncomp * c->NP, c->NP);
  a.tabs = c->tabs.data();
  int grid = 0;
  cudaError_t e = c->dim == 2 ? launch_aux_d2(c->N, 0, a, c->stream, &grid)
                              : launch_aux_d3(c->N, 0, a, c->stream, &grid);
  CK(e);
  return DG_OK;
}

int dg_frozen_coefficients(dg_ctx* c, const double* U, double* h, double* K) {
  CK(frozen(c->stream, c->n_el, c->NP, c->dim, U, c->model.gamma - 1.0, c->model.kinetic_factor,
            h, K));
  return DG_OK;
}

int dg_grad_p(dg_ctx* c, const double* x, const double* K, double* out, long long out_estride,
              const double* base, long long base_estride, double coef) {
  RET(halo(c, const_cast<double*>(x), 1));
  if (K) RET(halo(c, const_cast<double*>(K), 1));
  return op_grad(c, x, K, c->model.gamma - 1.0, c->model.kinetic_factor, 0, OUT_MINV,
                 mv(out, out_estride, c->NP), cv(base, base_estride, c->NP), base ? 1 : 0, coef);
}

int dg_energy_F(dg_ctx* c, double a_dt, const double* h, const double* K, const double* m_e,
                long long m_estride, const double* e_e, long long e_estride, const double* x,
                double* Fx) {
  RET(ensure_work(c));
  RET(halo(c, const_cast<double*>(h), 1));
  RET(halo(c, const_cast<double*>(K), 1));
  return energy_F(c, a_dt, h, K, cv(m_e, m_estride, c->NP), cv(e_e, e_estride, c->NP),
                  const_cast<double*>(x), Fx);
}

int dg_helmholtz_apply(dg_ctx* c, double a_dt, const double* h, const double* x, double* y) {
  RET(ensure_work(c));
  RET(halo(c, const_cast<double*>(h), 1));
  const double* hq = nullptr;
  if (quad_mode(c)) {
    RET(interp_h(c, h, c->shq.p));
    hq = c->shq.p;
  }
  return helm_apply(c, a_dt, h, hq, const_cast<double*>(x), y);
}

// prepare_divergence_hv (dgops.py:399-479): h frozen at the Gauss points
// (and its face traces) once; the prepared apply reuses them
int dg_helmholtz_prepare(dg_ctx* c, const double* h) {
  RET(ensure_work(c));
  RET(halo(c, const_cast<double*>(h), 1));
  if (quad_mode(c)) RET(interp_h(c, h, c->shq.p));
  return DG_OK;
}

int dg_helmholtz_apply_prepared(dg_ctx* c, double a_dt, const double* h, const double* x,
                                double* y) {
  RET(ensure_work(c));
  if (quad_mode(c) && c->hq_for != h) RET(dg_helmholtz_prepare(c, h));
  return helm_apply(c, a_dt, h, quad_mode(c) ? c->shq.p : nullptr, const_cast<double*>(x), y);
}

int dg_gmres_helmholtz(dg_ctx* c, double a_dt, const double* h, const double* rhs, double* x,
                       double tol_rel, int restart, int max_iter, dg_krylov_stats* stats,
                       double* history, int history_cap) {
  return dg_gmres_helmholtz_pc(c, a_dt, h, rhs, x, tol_rel, restart, max_iter, 0, stats, history,
                               history_cap);
}

int dg_gmres_helmholtz_pc(dg_ctx* c, double a_dt, const double* h, const double* rhs, double* x,
                          double tol_rel, int restart, int max_iter, int precond,
                          dg_krylov_stats* stats, double* history, int history_cap) {
  c->arn_ord = 0;
  RET(ensure_work(c));
  RET(halo(c, const_cast<double*>(h), 1));
  const double* hq = nullptr;
  if (quad_mode(c)) {
    RET(interp_h(c, h, c->shq.p));
    hq = c->shq.p;
  }
  Gm gs;
  RET(gmres(c, a_dt, h, hq, rhs, x, tol_rel, restart, max_iter, gs, precond != 0));
  if (stats) {
    stats->iterations = gs.iterations;
    stats->restarts = gs.restarts;
    stats->converged = gs.converged;
    stats->breakdown = gs.breakdown;
    stats->residual = gs.residual;
    const int nh = (int)std::min<size_t>(gs.hist.size(), history_cap > 0 ? history_cap : 0);
    stats->n_history = nh;
    if (history)
      for (int i = 0; i < nh; ++i) history[i] = gs.hist[i];
  }
  return DG_OK;
}

int dg_solve_implicit_stage(dg_ctx* c, const double* acc, const double* guess, double a_dt,
                            const dg_solve_cfg* cfg, double* iterate, dg_step_stats* stats) {
  c->arn_ord = 0;
  RET(ensure_work(c));
  int nfp = 0;
  RET(solve_stage(c, acc, guess, a_dt, *cfg, iterate, stats, &nfp));
  if (stats && stats->n_fp < 8) stats->fp_iters[stats->n_fp++] = nfp;
  return DG_OK;
}

int dg_imex_step(dg_ctx* c, const double* U, double* U_out, double t, double dt,
                 const dg_solve_cfg* cfg, dg_step_stats* stats) {
  (void)t;
  c->arn_ord = 0;
  RET(ensure_work(c));
  RET(ensure_states(c));
  const int d = c->dim, NP = c->NP, V = c->V;
  const long long ns = (long long)c->n_el * V * NP;
  const long long sst = (long long)V * NP;
  double* U0 = c->st[0].p;
  double* KE0 = c->st[1].p;   // later acc2
  double* acc1 = c->st[2].p;  // later KI1
  double* U1 = c->st[3].p;    // later U2
  double* KE1 = c->st[4].p;
  const double g = 1.0 - 1.0 / std::sqrt(2.0);
  const double dl = 1.0 - 1.0 / (2.0 * g);
  dg_step_stats local;
  if (!stats) stats = &local;
  std::memset(stats, 0, sizeof(*stats));
  CK(copy_comps(c->stream, c->n_el, NP, V, U, sst, U0, sst));
  // stage 0 (explicit): U_stage = U
  RET(check_positivity(c, U0, stats, 0));
  double mr = 0.0;
  RET(halo(c, U0, V));
  RET(op_advective(c, U0, KE0, OUT_MINV, &mr));
  stats->mass_rate += dl * mr;
  {
    const double cf[2] = {1.0, dt * g};
    const double* xs[2] = {U0, KE0};
    CK(lincomb(c->stream, ns, 2, cf, xs, acc1));
  }
  // stage 1 (implicit)
  int nfp = 0;
  RET(solve_stage(c, acc1, U0, dt * g, *cfg, U1, stats, &nfp));
  stats->fp_iters[stats->n_fp++] = nfp;
  {
    // KI1 = (U1 - acc1) / (dt g)   (in place over acc1)
    const double cf[2] = {1.0, -1.0};
    const double* xs[2] = {U1, acc1};
    CK(lincomb(c->stream, ns, 2, cf, xs, acc1));
    CK(scale(c->stream, ns, dt * g, true, acc1, acc1));
  }
  RET(check_positivity(c, U1, stats, 1));
  RET(halo(c, U1, V));
  RET(op_advective(c, U1, KE1, OUT_MINV, &mr));
  stats->mass_rate += (1.0 - dl) * mr;
  {
    // acc2 = U + dt dl KE0 + dt (1-dl) KE1 + dt (1-g) KI1   (in place over KE0)
    const double cf[4] = {1.0, dt * dl, dt * (1.0 - dl), dt * (1.0 - g)};
    const double* xs[4] = {U0, KE0, KE1, acc1};
    CK(lincomb(c->stream, ns, 4, cf, xs, KE0));
  }
  // stage 2 (implicit), guess = U1, result in place over U1
  RET(solve_stage(c, KE0, U1, dt * g, *cfg, U1, stats, &nfp));
  stats->fp_iters[stats->n_fp++] = nfp;
  RET(check_positivity(c, U1, stats, 2));
  CK(copy_comps(c->stream, c->n_el, NP, V, U1, sst, U_out, sst));
  return DG_OK;
}

int dg_integrate_conserved(dg_ctx* c, const double* U, double* out_host) {
  AuxArgs a;
  std::memset(&a, 0, sizeof a);
  a.elem = c->elem.p;
  a.col = c->col.p;
  a.gc = c->gc;
  a.n_el = c->n_el;
  a.ncomp = c->V;
  a.in = cv(U, (long long)c->V * c->NP, c->NP);
  a.partial = c->partial.p;
  a.tabs = c->tabs.data();
  int grid = 0;
  cudaError_t e = c->dim == 2 ? launch_aux_d2(c->N, 1, a, c->stream, &grid)
                              : launch_aux_d3(c->N, 1, a, c->stream, &grid);
  CK(e);
  if (grid == 0) {
    for (int v = 0; v < c->V; ++v) out_host[v] = 0.0;
    return DG_OK;
  }
  CK(reduce_cols(c->stream, c->partial.p, grid, c->V, c->redout.p));
  return reduce_read(c, c->redout.p, c->V, out_host);
}

int dg_max_abs_ratio(dg_ctx* c, const double* U, int num, int den, const uint8_t* mask,
                     double* out_host) {
  if (num < 0 || num >= c->V || den < 0 || den >= c->V)
    return fail(DG_ERR_USAGE, "dg_max_abs_ratio: component out of range");
  CK(max_ratio(c->stream, c->n_el, c->V, c->NP, U, num, den, mask, c->partial.p));
  std::vector<double> part(RED_BLOCKS);
  RET(sync_read_n(c, c->partial.p, RED_BLOCKS, part.data()));
  double m = 0.0;
  for (double v : part) m = std::max(m, v);
  if (c->comm.active()) {
    c->pinned[0] = m;
    CK(cudaMemcpyAsync(c->redout.p, c->pinned, sizeof(double), cudaMemcpyHostToDevice, c->stream));
    if (!c->comm.allreduce_max(c->redout.p, 1, c->stream)) return fail(DG_ERR_COMM, c->comm.error());
    RET(sync_read(c, c->redout.p, 1, &m));
  }
  *out_host = m;
  return DG_OK;
}

int dg_global_inner_product(dg_ctx* c, const double* a, const double* b, int ncomp,
                            double* out_host) {
  AuxArgs x;
  std::memset(&x, 0, sizeof x);
  x.elem = c->elem.p;
  x.col = c->col.p;
  x.gc = c->gc;
  x.n_el = c->n_el;
  x.ncomp = ncomp;
  x.in = cv(a, (long long)ncomp * c->NP, c->NP);
  x.in2 = cv(b, (long long)ncomp * c->NP, c->NP);
  x.partial = c->partial.p;
  x.tabs = c->tabs.data();
  int grid = 0;
  cudaError_t e = c->dim == 2 ? launch_aux_d2(c->N, 3, x, c->stream, &grid)
                              : launch_aux_d3(c->N, 3, x, c->stream, &grid);
  CK(e);
  if (grid == 0) CK(cudaMemsetAsync(c->redout.p, 0, sizeof(double), c->stream));
  else CK(reduce_rows(c->stream, c->partial.p, grid, 1, c->partial.p + (size_t)grid, c->redout.p));
  return reduce_read(c, c->redout.p, 1, out_host);  // (summed over ranks)
}

int dg_courant_ingredients(dg_ctx* c, const double* U, double* out4) {
  AuxArgs x;
  std::memset(&x, 0, sizeof x);
  x.elem = c->elem.p;
  x.col = c->col.p;
  x.gc = c->gc;
  x.n_el = c->n_el;
  x.ncomp = c->V;
  x.in = cv(U, (long long)c->V * c->NP, c->NP);
  x.model = c->model;
  x.partial = c->partial.p;
  x.tabs = c->tabs.data();
  int grid = 0;
  cudaError_t e = c->dim == 2 ? launch_aux_d2(c->N, 4, x, c->stream, &grid)
                              : launch_aux_d3(c->N, 4, x, c->stream, &grid);
  CK(e);
  std::vector<double> part((size_t)grid * 4);
  CK(cudaStreamSynchronize(c->stream));
  if (grid) CK(cudaMemcpy(part.data(), c->partial.p, part.size() * sizeof(double),
                          cudaMemcpyDeviceToHost));
  double r[4] = {-INFINITY, -INFINITY, INFINITY, INFINITY};
  for (int b = 0; b < grid; ++b) {
    r[0] = std::max(r[0], part[b * 4 + 0]);
    r[1] = std::max(r[1], part[b * 4 + 1]);
    r[2] = std::min(r[2], part[b * 4 + 2]);
    r[3] = std::min(r[3], part[b * 4 + 3]);
  }
  if (c->comm.active()) {
    // max of (c, |u|, -rho_min, -p_min) over ranks
    double m[4] = {r[0], r[1], -r[2], -r[3]};
    std::memcpy(c->pinned, m, sizeof m);
    CK(cudaMemcpyAsync(c->redout.p, c->pinned, sizeof m, cudaMemcpyHostToDevice, c->stream));
    if (!c->comm.allreduce_max(c->redout.p, 4, c->stream)) return fail(DG_ERR_COMM, c->comm.error());
    RET(sync_read(c, c->redout.p, 4, m));
    r[0] = m[0]; r[1] = m[1]; r[2] = -m[2]; r[3] = -m[3];
  }
  for (int i = 0; i < 4; ++i) out4[i] = r[i];
  return DG_OK;
}

int dg_check_positivity(dg_ctx* c, const double* U, double* min_rho, long long* at_rho,
                        double* min_p, long long* at_p) {
  dg_step_stats s;
  std::memset(&s, 0, sizeof s);
  int r = check_positivity(c, U, &s, -1);
  if (min_rho) *min_rho = s.fail_kind == 0 ? s.fail_value : 0.0;
  if (at_rho) *at_rho = s.fail_element;
  if (min_p) *min_p = s.fail_value;
  if (at_p) *at_p = s.fail_node;
  return r;
}

int dg_lincomb(dg_ctx* c, long long n, int m, const double* coefs, const double* const* xs,
               double* y) {
  if (m < 1 || m > 4) return fail(DG_ERR_USAGE, "lincomb takes 1..4 terms");
  CK(lincomb(c->stream, n, m, coefs, xs, y));
  return DG_OK;
}

int dg_dots(dg_ctx* c, long long n, int nv, const double* V, long long vstride, const double* w,
            double* out_host) {
  if (nv < 0 || nv > 32) return fail(DG_ERR_USAGE, "dg_dots: 0..32 vectors");
  CK(multidot(c->stream, n, nv, V, vstride, w, c->partial.p, c->redout.p));
  return reduce_read(c, c->redout.p, nv + 1, out_host);
}

int dg_gs_update(dg_ctx* c, long long n, int nv, const double* V, long long vstride,
                 const double* coefs_host, double* w, double na, double* dst) {
  if (nv < 1 || nv > 32) return fail(DG_ERR_USAGE, "dg_gs_update: 1..32 vectors");
  if (!(na != 0.0)) return fail(DG_ERR_USAGE, "dg_gs_update: zero norm");
  CK(cudaStreamSynchronize(c->stream));  // the pinned staging slot is free
  std::memcpy(c->pin_coef(), coefs_host, nv * sizeof(double));
  CK(cudaMemcpyAsync(c->coef_dev.p, c->pin_coef(), nv * sizeof(double), cudaMemcpyHostToDevice,
                     c->stream));
  CK(axpy_div(c->stream, n, nv, V, vstride, c->coef_dev.p, w, na, dst));
  return DG_OK;
}

int dg_dcgs2_update(dg_ctx* c, long long n, int nv, const double* V, long long vstride,
                    const double* coefs_host, double* u, const double* z, double* u_next,
                    double* norm2_host) {
  if (nv < 0 || nv > 31) return fail(DG_ERR_USAGE, "dg_dcgs2_update: 0..31 vectors");
  if (!(coefs_host[3 * nv + 2] != 0.0)) return fail(DG_ERR_USAGE, "dg_dcgs2_update: zero alpha");
  CK(cudaStreamSynchronize(c->stream));  // the pinned staging slot is free
  std::memcpy(c->pin_coef(), coefs_host, (3 * nv + 3) * sizeof(double));
  CK(cudaMemcpyAsync(c->coef_dev.p, c->pin_coef(), (3 * nv + 3) * sizeof(double),
                     cudaMemcpyHostToDevice, c->stream));
  CK(dcgs2_update(c->stream, n, nv, V, vstride, c->coef_dev.p, u, z, u_next, c->partial.p,
                  c->redout.p));
  return reduce_read(c, c->redout.p, 1, norm2_host);
}

int dg_nccl_unique_id(void* out128) {
  std::string err;
  if (!Comm::unique_id(out128, &err)) return fail(DG_ERR_COMM, err);
  return DG_OK;
}

int dg_ctx_set_comm(dg_ctx* c, const void* uid, int rank, int nranks, const int32_t* send_counts,
                    const int32_t* send_elems, const int32_t* recv_counts) {
  CK(cudaSetDevice(c->device));
  if (!c->comm.init(uid, rank, nranks, send_counts, send_elems, recv_counts, c->n_el, c->n_tot))
    return fail(DG_ERR_COMM, c->comm.error());
  long long tot = (long long)c->n_el * c->NP;
  double v = (double)tot;
  DevBuf<double> tmp;
  CK(tmp.upload(&v, 1));
  if (!c->comm.allreduce_sum(tmp.p, 1, c->stream)) return fail(DG_ERR_COMM, c->comm.error());
  CK(cudaMemcpy(&v, tmp.p, sizeof(double), cudaMemcpyDeviceToHost));
  tmp.release();
  c->n_global = (long long)v;
  return DG_OK;
}

int dg_ctx_set_comm_loopback(dg_ctx* c, int group, int rank, int nranks,
                             const int32_t* send_counts, const int32_t* send_elems,
                             const int32_t* recv_counts) {
  CK(cudaSetDevice(c->device));
  if (!c->comm.init_loopback(group, rank, nranks, send_counts, send_elems, recv_counts, c->n_el,
                             c->n_tot))
    return fail(DG_ERR_COMM, c->comm.error());
  long long tot = (long long)c->n_el * c->NP;
  double v = (double)tot;
  DevBuf<double> tmp;
  CK(tmp.upload(&v, 1));
  if (!c->comm.allreduce_sum(tmp.p, 1, c->stream)) return fail(DG_ERR_COMM, c->comm.error());
  CK(cudaMemcpy(&v, tmp.p, sizeof(double), cudaMemcpyDeviceToHost));
  tmp.release();
  c->n_global = (long long)v;
  return DG_OK;
}

int dg_ctx_set_halo_rows(dg_ctx* c, int which, const int64_t* send_counts,
                         const int64_t* send_idx, const int64_t* recv_counts,
                         const int64_t* recv_idx) {
  CK(cudaSetDevice(c->device));
  if (!c->comm.set_rows(which, send_counts, send_idx, recv_counts, recv_idx))
    return fail(DG_ERR_COMM, c->comm.error());
  return DG_OK;
}

int dg_halo_stats(dg_ctx* c, long long* values_sent, int reset) {
  if (values_sent) *values_sent = c->halo_values;
  if (reset) c->halo_values = 0;
  return DG_OK;
}

// DCGS2 dual dots (Q_i.z, Q_i.u for i < nv, then z.z, z.u, u.z, u.u) in one
// streaming pass, reduced over ranks: the dots krylov.py:69-72 takes per
// Arnoldi step, in the delayed re-orthogonalisation form
int dg_dual_dots(dg_ctx* c, long long n, int nv, const double* V, long long vstride,
                 const double* z, const double* u, double* out_host) {
  if (nv < 0 || nv > 31) return fail(DG_ERR_USAGE, "dg_dual_dots: 0 <= nv <= 31");
  CK(c->gs_part.alloc((size_t)RED_BLOCKS * 2 * (32 + 2)));
  int rows = 0;
  CK(dual_dots(c->stream, n, nv, V, vstride, z, u, c->gs_part.p, &rows));
  CK(reduce_rows(c->stream, c->gs_part.p, rows, 2 * (nv + 2), c->partial.p, c->redout.p));
  return reduce_read(c, c->redout.p, 2 * (nv + 2), out_host);
}

int dg_halo_exchange(dg_ctx* c, double* field, int ncomp) { return halo(c, field, ncomp); }

long long dg_launch_count(void) { return prof().launches; }

int dg_set_arnoldi_mode(dg_ctx* c, int mode) {
  if (mode < -1 || mode > 2) return fail(DG_ERR_USAGE, "arnoldi mode must be -1, 0, 1 or 2");
  c->arn_mode = mode;
  c->arn_pred.clear();
  return DG_OK;
}

int dg_arnoldi_stats(dg_ctx* c, long long* syncs, long long* wasted_steps) {
  if (syncs) *syncs = c->arn_syncs;
  if (wasted_steps) *wasted_steps = c->arn_wasted;
  return DG_OK;
}

int dg_profile_enable(int on) {
  Profiler& p = prof();
  p.on = on != 0;
  p.used = 0;
  p.cls.clear();
  p.bytes.clear();
  return DG_OK;
}

int dg_profile_read(double* ms, double* bytes, long long* count) {
  Profiler& p = prof();
  for (int k = 0; k < P_NCLS; ++k) {
    ms[k] = 0.0;
    bytes[k] = 0.0;
    count[k] = 0;
  }
  if (p.used) CK(cudaEventSynchronize(p.ev[2 * p.used - 1]));
  for (size_t i = 0; i < p.used; ++i) {
    float t = 0.f;
    CK(cudaEventElapsedTime(&t, p.ev[2 * i], p.ev[2 * i + 1]));
    ms[p.cls[i]] += t;
    bytes[p.cls[i]] += p.bytes[i];
    count[p.cls[i]] += 1;
  }
  return DG_OK;
}

// greedy colouring of the face-adjacency graph (orodg/krylov.py:118-140):
// elements in order, each takes the smallest colour none of its already
// coloured neighbours has; self pairs (periodic wraps) are ignored
int dg_element_coloring(long long n_el, long long n_pairs, const long long* a, const long long* b,
                        long long* colors, int* n_colors) {
  if (n_el < 0 || n_pairs < 0) return fail(DG_ERR_USAGE, "negative sizes");
  std::vector<long long> deg(n_el + 1, 0);
  for (long long k = 0; k < n_pairs; ++k) {
    const long long i = a[k], j = b[k];
    if (i < 0 || j < 0 || i >= n_el || j >= n_el) return fail(DG_ERR_USAGE, "pair out of range");
    if (i == j) continue;
    deg[i + 1] += 1;
    deg[j + 1] += 1;
  }
  for (long long i = 0; i < n_el; ++i) deg[i + 1] += deg[i];
  std::vector<long long> adj(deg[n_el]), fill(deg.begin(), deg.end() - 1);
  for (long long k = 0; k < n_pairs; ++k) {
    const long long i = a[k], j = b[k];
    if (i == j) continue;
    adj[fill[i]++] = j;
    adj[fill[j]++] = i;
  }
  std::vector<long long> stamp;  // stamp[c] == i + 1: colour c used around element i
  long long maxc = -1;
  for (long long i = 0; i < n_el; ++i) colors[i] = -1;
  for (long long i = 0; i < n_el; ++i) {
    for (long long k = deg[i]; k < deg[i + 1]; ++k) {
      const long long cj = colors[adj[k]];
      if (cj >= 0) {
        if ((long long)stamp.size() <= cj) stamp.resize(cj + 1, 0);
        stamp[cj] = i + 1;
      }
    }
    long long col = 0;
    while (col < (long long)stamp.size() && stamp[col] == i + 1) ++col;
    colors[i] = col;
    maxc = std::max(maxc, col);
  }
  if (n_colors) *n_colors = (int)(maxc + 1);
  return DG_OK;
}

int dg_bj_set_coloring(dg_ctx* c, const long long* colors, long long n) {
  if (n != c->n_el) return fail(DG_ERR_USAGE, "colouring must cover the owned elements");
  std::vector<int> h(n);
  int nc = 0;
  for (long long i = 0; i < n; ++i) {
    if (colors[i] < 0) return fail(DG_ERR_USAGE, "negative colour");
    h[i] = (int)colors[i];
    nc = std::max(nc, h[i] + 1);
  }
  if (c->comm.active()) {
    // every rank probes every colour (the action's halo exchanges are collective)
    c->pinned[0] = nc;
    CK(cudaMemcpyAsync(c->redout.p, c->pinned, sizeof(double), cudaMemcpyHostToDevice, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    if (!c->comm.allreduce_max(c->redout.p, 1, c->stream)) return fail(DG_ERR_COMM, c->comm.error());
    double v;
    RET(sync_read(c, c->redout.p, 1, &v));
    nc = (int)v;
  }
  CK(c->bj_colors.upload(h.data(), h.size()));
  c->bj_ncolors = nc;
  c->bj_valid = 0;
  return DG_OK;
}

int dg_bj_build(dg_ctx* c, double a_dt, const double* h, int* n_singular, long long* generation) {
  RET(ensure_work(c));
  RET(halo(c, const_cast<double*>(h), 1));
  const double* hq = nullptr;
  if (quad_mode(c)) {
    RET(interp_h(c, h, c->shq.p));
    hq = c->shq.p;
  }
  RET(bj_build(c, a_dt, h, hq, n_singular));
  if (generation) *generation = c->bj_gen;
  return DG_OK;
}

int dg_bj_apply(dg_ctx* c, const double* in, double* out) { return bj_apply_ctx(c, in, out); }

int dg_bj_state(dg_ctx* c, int* valid, int* age, long long* generation) {
  if (valid) *valid = c->bj_valid;
  if (age) *age = c->bj_age;
  if (generation) *generation = c->bj_gen;
  return DG_OK;
}

int dg_bj_set_state(dg_ctx* c, int valid, int age) {
  c->bj_valid = (valid && c->bj_inv.p) ? 1 : 0;
  c->bj_age = age;
  return DG_OK;
}

int dg_split_contiguous(const double* w, long long n, int n_chunks, long long* bounds) {
  // orodg/partition.py:45-67 : bisection on the capacity + greedy packing
  if (n_chunks < 1) return fail(DG_ERR_CONFIG, "need >= 1 chunk");
  if (n_chunks >= n) {
    for (long long i = 0; i <= n; ++i) bounds[i] = i;
    for (long long i = n + 1; i <= n_chunks; ++i) bounds[i] = n;
    return DG_OK;
  }
  auto pack = [&](double cap, std::vector<long long>& b, long long limit) -> bool {
    b.clear();
    b.push_back(0);
    double acc = 0.0;
    for (long long i = 0; i < n; ++i) {
      if (w[i] > cap) return false;
      if (acc + w[i] > cap) {
        b.push_back(i);
        acc = w[i];
        if ((long long)b.size() - 1 > limit) return true;
      } else {
        acc += w[i];
      }
    }
    b.push_back(n);
    return true;
  };
  double lo = 0.0, hi = 0.0;
  for (long long i = 0; i < n; ++i) {
    lo = std::max(lo, w[i]);
    hi += w[i];
  }
  std::vector<long long> b;
  for (int it = 0; it < 200; ++it) {
    const double mid = 0.5 * (lo + hi);
    const bool ok = pack(mid, b, n_chunks) && (long long)b.size() - 1 <= n_chunks;
    if (ok) hi = mid;
    else lo = mid;
    if (hi - lo <= 1e-12 * std::max(hi, 1.0)) break;
  }
  pack(hi * (1 + 1e-12), b, n);
  while ((long long)b.size() - 1 < n_chunks) b.push_back(n);
  for (int i = 0; i <= n_chunks; ++i) bounds[i] = b[i];
  return DG_OK;
}

}  // extern "C"
