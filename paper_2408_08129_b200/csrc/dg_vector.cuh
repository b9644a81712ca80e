// Host wrappers of the streaming vector kernels (dg_vector.cu).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace dg {

constexpr int RED_THREADS = 256;
constexpr int RED_BLOCKS = 592;  // 4 x 148 SMs; fixed => deterministic reductions

cudaError_t lincomb(cudaStream_t st, long long n, int m, const double* c, const double* const* x,
                    double* y);
cudaError_t multidot(cudaStream_t st, long long n, int nv, const double* V, long long vstride,
                     const double* w, double* partials, double* out);
// w <- w - sum c_i V_i, then out[0..nv-1] = V_i . w, out[nv] = |w|^2 (one pass)
cudaError_t axpy_dots(cudaStream_t st, long long n, int nv, const double* V, long long vstride,
                      const double* coefs_dev, double* w, double* partials, double* out);
cudaError_t axpy_multi(cudaStream_t st, long long n, int nv, const double* V, long long vstride,
                       const double* coefs_dev, double* w, double* partials, double* norm2_out);
cudaError_t axpy_div(cudaStream_t st, long long n, int nv, const double* V, long long vstride,
                     const double* coefs_dev, double* w, double na, double* dst);
// DCGS2 Arnoldi update (see dg_vector.cu): u <- q, unext <- u', out[0] = |u'|^2
cudaError_t dcgs2_update(cudaStream_t st, long long n, int nv, const double* Q, long long vstride,
                         const double* coefs_dev, double* u, const double* z, double* unext,
                         double* partials, double* out);
// DCGS2 dual dots (Q_i.z, Q_i.u, z.z, z.u, u.z, u.u) as per-block rows
cudaError_t dual_dots(cudaStream_t st, long long n, int nv, const double* Q, long long vstride,
                      const double* z, const double* u, double* rows, int* nrows);
// per-block maxima of |U[num] / U[den]| over (masked) nodes
cudaError_t max_ratio(cudaStream_t st, long long n_el, int V, int np, const double* U, int num,
                      int den, const uint8_t* mask, double* partials);
cudaError_t scale(cudaStream_t st, long long n, double a, bool divide, const double* x,
                  double* y);
cudaError_t frozen(cudaStream_t st, long long n_el, int np, int d, const double* U, double gm1,
                   double kf, double* h, double* K);
cudaError_t state_pressure(cudaStream_t st, long long n_el, int np, int d, const double* U,
                           double gm1, double kf, double* p);
cudaError_t pressure_dp(cudaStream_t st, long long n, const double* x, const double* K, double gm1,
                        double kf, double* p_old, double* partials, double* out2);
cudaError_t set_iterate(cudaStream_t st, long long n_el, int np, int V, const double* acc,
                        const double* guess, double* it);
cudaError_t copy_comps(cudaStream_t st, long long n_el, int np, int nc, const double* src,
                       long long s_estride, double* dst, long long d_estride);
cudaError_t positivity(cudaStream_t st, long long n_el, int np, int d, const double* U, double gm1,
                       double kf, double* partials);
cudaError_t reduce_cols(cudaStream_t st, const double* partials, int nblocks, int ncols, double* out);
cudaError_t reduce_rows(cudaStream_t st, const double* partials, long long nrows, int ncols,
                        double* tmp, double* out);

// Device-resident scalar state of one DCGS2 Arnoldi cycle (restart m <= 31):
// the small-problem GMRES path keeps Hbar, the running Givens QR and the
// stopping tests on the device so that several Arnoldi steps are enqueued
// per host synchronisation (dg_runtime.cu dcgs2_cycle_dev; the arithmetic
// and its order are those of the host loop of dcgs2_cycle).
constexpr int ARN_M = 31;
struct ArnState {
  double bn, target, nb;
  double g[ARN_M + 1], cs[ARN_M], sn[ARN_M], hist[ARN_M];
  double Hb[(ARN_M + 1) * ARN_M];
  int m, done, stop, breakdown, iterations, max_iter, steps_run, pad;
};
cudaError_t arn_init(cudaStream_t st, ArnState* a, int m, double bn, double target, double beta,
                     int iterations, int max_iter);
// step j, after the dual dots landed in dots[2 (j + 2)]: alpha, s, g, h ->
// coefs (dcgs2_update layout), Hbar column j (and the correction of j-1)
// (nrows > 0: src = nrows partial rows, summed by the kernel itself)
cudaError_t arn_pre(cudaStream_t st, ArnState* a, int j, const double* src, int nrows,
                    double* coefs);
// step j, after the update: Hbar[j+1][j] = sqrt(|u'|^2), Givens, stop tests
// (nparts > 0: na2 = the update kernel's per-CTA partials)
cudaError_t arn_post(cudaStream_t st, ArnState* a, int j, const double* na2, int nparts);
cudaError_t dcgs2_update_partials(cudaStream_t st, long long n, int nv, const double* Q,
                                  long long vstride, const double* coefs_dev, double* u,
                                  const double* z, double* unext, double* partials, int* nparts);

}  // namespace dg
