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

}  // namespace dg
