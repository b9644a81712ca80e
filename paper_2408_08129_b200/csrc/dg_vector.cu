#include <algorithm>
// Streaming vector kernels of the implicit solver: IMEX stage linear
// combinations (orodg/imex.py:267-298), GMRES Gram-Schmidt dots/updates
// (orodg/krylov.py:69-80, 105-109), pressure fixed-point norms
// (imex.py:355-359), frozen coefficients (imex.py:182-188) and the
// positivity check (physics.py:136-164).
//
// All reductions are deterministic: a fixed grid of RED_BLOCKS CTAs writes
// per-CTA partials in a fixed traversal order, a second kernel combines
// them with a fixed warp tree.  Results are bitwise reproducible run to run.
#include <cstdint>
#include <cstdlib>

#include "dg_vector.cuh"
#include "dg_pdl.cuh"
#include "dg_prof.h"

namespace dg {

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// y = c0 x0 (+ c1 x1 (+ c2 x2 (+ c3 x3))), left to right, unfused like numpy
__global__ void k_lincomb(long long n, int m, double c0, double c1, double c2, double c3,
                          const double* __restrict__ x0, const double* __restrict__ x1,
                          const double* __restrict__ x2, const double* __restrict__ x3,
                          double* __restrict__ y) {
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    double v = (c0 == 1.0) ? x0[i] : __dmul_rn(c0, x0[i]);
    if (m > 1) v = __dadd_rn(v, __dmul_rn(c1, x1[i]));
    if (m > 2) v = __dadd_rn(v, __dmul_rn(c2, x2[i]));
    if (m > 3) v = __dadd_rn(v, __dmul_rn(c3, x3[i]));
    y[i] = v;
  }
}

// partials[b][i] = sum V_i . w  (i < nv),  partials[b][nv] = w . w
template <int MAXV>
__global__ void __launch_bounds__(RED_THREADS)
k_multidot(long long n, int nv, const double* __restrict__ V, long long vstride,
           const double* __restrict__ w, double* __restrict__ partials) {
  double acc[MAXV + 1];
#pragma unroll
  for (int i = 0; i <= MAXV; ++i) acc[i] = 0.0;
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long k = (long long)blockIdx.x * blockDim.x + threadIdx.x; k < n; k += stride) {
    const double wk = w[k];
#pragma unroll
    for (int i = 0; i < MAXV; ++i)
      if (i < nv) acc[i] = fma(V[i * vstride + k], wk, acc[i]);
    acc[MAXV] = fma(wk, wk, acc[MAXV]);
  }
  __shared__ double red[RED_THREADS / 32][MAXV + 1];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
  for (int i = 0; i <= MAXV; ++i) {
    if (i < nv || i == MAXV) {
      const double v = warp_sum(acc[i]);
      if (lane == 0) red[wid][i] = v;
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i <= MAXV; i += blockDim.x) {
    if (i < nv || i == MAXV) {
      double s = 0.0;
      for (int w2 = 0; w2 < RED_THREADS / 32; ++w2) s += red[w2][i];
      partials[(long long)blockIdx.x * (nv + 1) + (i == MAXV ? nv : i)] = s;
    }
  }
}

// partials[b] = partial of w . w (multidot with nv = 0: the residual norms of
// GMRES): 16-byte loads, four k-pairs in flight per thread -- the general
// kernel keeps one 8-byte load in flight and ran at 1.9 TB/s there
__global__ void __launch_bounds__(RED_THREADS)
k_norm2(long long n, const double* __restrict__ w, double* __restrict__ partials) {
  double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
  const long long n2 = n >> 1;
  const long long stride = (long long)gridDim.x * blockDim.x;
  const double2* w2 = reinterpret_cast<const double2*>(w);
  long long k = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  for (; k + 3 * stride < n2; k += 4 * stride) {
    const double2 v0 = w2[k], v1 = w2[k + stride], v2 = w2[k + 2 * stride], v3 = w2[k + 3 * stride];
    a0 = fma(v0.x, v0.x, a0); a0 = fma(v0.y, v0.y, a0);
    a1 = fma(v1.x, v1.x, a1); a1 = fma(v1.y, v1.y, a1);
    a2 = fma(v2.x, v2.x, a2); a2 = fma(v2.y, v2.y, a2);
    a3 = fma(v3.x, v3.x, a3); a3 = fma(v3.y, v3.y, a3);
  }
  for (; k < n2; k += stride) {
    const double2 v0 = w2[k];
    a0 = fma(v0.x, v0.x, a0); a0 = fma(v0.y, v0.y, a0);
  }
  if ((n & 1) && blockIdx.x == 0 && threadIdx.x == 0) a1 = fma(w[n - 1], w[n - 1], a1);
  double acc = (a0 + a1) + (a2 + a3);
  __shared__ double red[RED_THREADS / 32];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  acc = warp_sum(acc);
  if (lane == 0) red[wid] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int i = 0; i < RED_THREADS / 32; ++i) t += red[i];
    partials[blockIdx.x] = t;
  }
}

// w <- w - sum_i c_i V_i ; partial |w|^2.  coefs on the device.
template <int MAXV>
__global__ void __launch_bounds__(RED_THREADS)
k_axpy_multi(long long n, int nv, const double* __restrict__ V, long long vstride,
             const double* __restrict__ coefs, double* __restrict__ w,
             double* __restrict__ partials) {
  __shared__ double c[MAXV];
  for (int i = threadIdx.x; i < MAXV; i += blockDim.x) c[i] = i < nv ? coefs[i] : 0.0;
  __syncthreads();
  double acc = 0.0;
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long k = (long long)blockIdx.x * blockDim.x + threadIdx.x; k < n; k += stride) {
    double t = 0.0;
#pragma unroll
    for (int i = 0; i < MAXV; ++i)
      if (i < nv) t = fma(c[i], V[i * vstride + k], t);
    const double v = w[k] - t;
    w[k] = v;
    acc = fma(v, v, acc);
  }
  __shared__ double red[RED_THREADS / 32];
  acc = warp_sum(acc);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int i = 0; i < RED_THREADS / 32; ++i) s += red[i];
    if (partials) partials[blockIdx.x] = s;
  }
}

// dst <- (w - sum_i c_i V_i) / na : Gram-Schmidt update and normalisation in
// one pass (the norm comes from the Pythagorean identity)
template <int MAXV>
__global__ void __launch_bounds__(RED_THREADS)
k_axpy_div(long long n, int nv, const double* __restrict__ V, long long vstride,
           const double* __restrict__ coefs, const double* __restrict__ w, double na,
           double* __restrict__ dst) {
  __shared__ double c[MAXV];
  for (int i = threadIdx.x; i < MAXV; i += blockDim.x) c[i] = i < nv ? coefs[i] : 0.0;
  __syncthreads();
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long k = (long long)blockIdx.x * blockDim.x + threadIdx.x; k < n; k += stride) {
    double t = 0.0;
#pragma unroll
    for (int i = 0; i < MAXV; ++i)
      if (i < nv) t = fma(c[i], V[i * vstride + k], t);
    dst[k] = (w[k] - t) / na;
  }
}

// out[c] = sum_b partials[b][c]   (one warp per column, fixed order)
__global__ void k_reduce_cols(const double* __restrict__ partials, int nblocks, int ncols,
                              double* __restrict__ out) {
  pdl_trigger();
  pdl_wait();
  const int col = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (col >= ncols) return;
  double s = 0.0;
  for (int b = lane; b < nblocks; b += 32) s += partials[(long long)b * ncols + col];
  s = warp_sum(s);
  if (lane == 0) out[col] = s;
}

__global__ void k_scale(long long n, double a, int divide, const double* __restrict__ x,
                        double* __restrict__ y) {
  // y = x * a, or y = x / a (numpy's r / beta, w / norm)
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride)
    y[i] = divide ? x[i] / a : x[i] * a;
}

// h = e + p/rho, K = rho k at every node (imex.py:182-188)
__global__ void k_frozen(long long n_el, int np, int d, const double* __restrict__ U,
                         double gm1, double kf, double* __restrict__ h, double* __restrict__ K) {
  const long long n = n_el * np;
  const long long stride = (long long)gridDim.x * blockDim.x;
  const int V = d + 2;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    const long long e = i / np;
    const int q = (int)(i - e * np);
    const double* u = U + e * V * np + q;
    const double rho = u[0];
    double k = 0.0;
    for (int a = 0; a < d; ++a) {
      const double v = u[(1 + a) * np] / rho;
      k += v * v;
    }
    k *= 0.5;
    const double p = gm1 * (u[(d + 1) * np] - kf * rho * k);
    h[i] = p / (gm1 * rho) + p / rho;
    K[i] = rho * k;
  }
}

// p from a conserved state (scalar field)
__global__ void k_state_pressure(long long n_el, int np, int d, const double* __restrict__ U,
                                 double gm1, double kf, double* __restrict__ p) {
  const long long n = n_el * np;
  const long long stride = (long long)gridDim.x * blockDim.x;
  const int V = d + 2;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    const long long e = i / np;
    const int q = (int)(i - e * np);
    const double* u = U + e * V * np + q;
    const double rho = u[0];
    double k = 0.0;
    for (int a = 0; a < d; ++a) {
      const double v = u[(1 + a) * np] / rho;
      k += v * v;
    }
    k *= 0.5;
    p[i] = gm1 * (u[(d + 1) * np] - kf * rho * k);
  }
}

// p_new = gm1 (x - kf K);  partials: |p_new - p_old|^2, |p_old|^2; p_old <- p_new
__global__ void __launch_bounds__(RED_THREADS)
k_pressure_dp(long long n, const double* __restrict__ x, const double* __restrict__ K,
              double gm1, double kf, double* __restrict__ p_old, double* __restrict__ partials) {
  double a = 0.0, b = 0.0;
  const long long stride = (long long)gridDim.x * blockDim.x;
  // four elements per trip (fixed order per thread): 12 loads in flight
  for (long long i0 = (long long)blockIdx.x * blockDim.x + threadIdx.x; i0 < n; i0 += 4 * stride) {
    double xv[4], kv[4], pv[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const long long i = i0 + u * stride;
      const bool ok = i < n;
      xv[u] = ok ? x[i] : 0.0;
      kv[u] = ok ? K[i] : 0.0;
      pv[u] = ok ? p_old[i] : 0.0;
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const long long i = i0 + u * stride;
      if (i < n) {
        const double pn = gm1 * (xv[u] - kf * kv[u]);
        const double df = pn - pv[u];
        a = fma(df, df, a);
        b = fma(pv[u], pv[u], b);
        p_old[i] = pn;
      }
    }
  }
  __shared__ double red[2][RED_THREADS / 32];
  a = warp_sum(a);
  b = warp_sum(b);
  if ((threadIdx.x & 31) == 0) {
    red[0][threadIdx.x >> 5] = a;
    red[1][threadIdx.x >> 5] = b;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double sa = 0.0, sb = 0.0;
    for (int i = 0; i < RED_THREADS / 32; ++i) {
      sa += red[0][i];
      sb += red[1][i];
    }
    partials[blockIdx.x * 2] = sa;
    partials[blockIdx.x * 2 + 1] = sb;
  }
}

// iterate = acc with components >= 1 taken from guess (imex.py:315-317)
__global__ void k_set_iterate(long long n_el, int np, int V, const double* __restrict__ acc,
                              const double* __restrict__ guess, double* __restrict__ it) {
  const long long n = n_el * V * np;
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    const int c = (int)((i / np) % V);
    it[i] = c == 0 ? acc[i] : guess[i];
  }
}

// strided component copy: dst(e, c0+c) = src(e, s0+c)
__global__ void k_copy_comps(long long n_el, int np, int nc, const double* __restrict__ src,
                             long long s_estride, double* __restrict__ dst, long long d_estride) {
  const long long n = n_el * nc * np;
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    const long long e = i / (nc * np);
    const long long r = i - e * nc * np;
    dst[e * d_estride + r] = src[e * s_estride + r];
  }
}

// positivity: per-CTA (min rho, idx, min p, idx); first index among ties
struct MinLoc {
  double v;
  long long i;
};
__device__ __forceinline__ MinLoc minloc(MinLoc a, MinLoc b) {
  if (b.v < a.v || (b.v == a.v && b.i < a.i)) return b;
  return a;
}
__global__ void __launch_bounds__(RED_THREADS)
k_positivity(long long n_el, int np, int d, const double* __restrict__ U, double gm1, double kf,
             double* __restrict__ partials) {
  MinLoc r{INFINITY, 0x7fffffffffffffffLL}, p{INFINITY, 0x7fffffffffffffffLL};
  const long long n = n_el * np;
  const long long stride = (long long)gridDim.x * blockDim.x;
  const int V = d + 2;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    const long long e = i / np;
    const int q = (int)(i - e * np);
    const double* u = U + e * V * np + q;
    const double rho = u[0];
    double k = 0.0;
    for (int a = 0; a < d; ++a) {
      const double v = u[(1 + a) * np] / rho;
      k += v * v;
    }
    k *= 0.5;
    const double pr = gm1 * (u[(d + 1) * np] - kf * rho * k);
    r = minloc(r, MinLoc{rho != rho ? -INFINITY : rho, i});
    p = minloc(p, MinLoc{pr != pr ? -INFINITY : pr, i});
  }
  for (int o = 16; o > 0; o >>= 1) {
    MinLoc r2{__shfl_xor_sync(0xffffffffu, r.v, o), __shfl_xor_sync(0xffffffffu, r.i, o)};
    MinLoc p2{__shfl_xor_sync(0xffffffffu, p.v, o), __shfl_xor_sync(0xffffffffu, p.i, o)};
    r = minloc(r, r2);
    p = minloc(p, p2);
  }
  __shared__ MinLoc sr[RED_THREADS / 32], sp[RED_THREADS / 32];
  if ((threadIdx.x & 31) == 0) {
    sr[threadIdx.x >> 5] = r;
    sp[threadIdx.x >> 5] = p;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int i = 1; i < RED_THREADS / 32; ++i) {
      r = minloc(sr[0], sr[i]);
      sr[0] = r;
      p = minloc(sp[0], sp[i]);
      sp[0] = p;
    }
    partials[blockIdx.x * 4 + 0] = sr[0].v;
    partials[blockIdx.x * 4 + 1] = (double)sr[0].i;
    partials[blockIdx.x * 4 + 2] = sp[0].v;
    partials[blockIdx.x * 4 + 3] = (double)sp[0].i;
  }
}

// ------------------------------------------------------------ profiling
Profiler& prof() {
  static Profiler p;
  return p;
}

void prof_begin(cudaStream_t st) {
  Profiler& p = prof();
  if (!p.on) return;
  if (2 * (p.used + 1) > p.ev.size()) {
    for (int i = 0; i < 256; ++i) {
      cudaEvent_t e;
      cudaEventCreate(&e);
      p.ev.push_back(e);
    }
  }
  cudaEventRecord(p.ev[2 * p.used], st);
}

void prof_end(cudaStream_t st, int cls, double bytes, int nlaunch) {
  Profiler& p = prof();
  p.launches += nlaunch;
  if (!p.on) return;
  cudaEventRecord(p.ev[2 * p.used + 1], st);
  p.cls.push_back(cls);
  p.bytes.push_back(bytes);
  p.used += 1;
}

// ------------------------------------------------------------ host wrappers
// streaming kernels (no reduction): enough resident threads per SM to keep
// the loads in flight (a 592-CTA grid leaves them latency-bound)
static int grid_for(long long n) {
  long long g = (n + RED_THREADS - 1) / RED_THREADS;
  if (g > 148 * 32) g = 148 * 32;
  if (g < 1) g = 1;
  return (int)g;
}

cudaError_t lincomb(cudaStream_t st, long long n, int m, const double* c, const double* const* x,
                    double* y) {
  if (n <= 0) return cudaSuccess;
  prof_begin(st);
  k_lincomb<<<grid_for(n), RED_THREADS, 0, st>>>(
      n, m, c[0], m > 1 ? c[1] : 0.0, m > 2 ? c[2] : 0.0, m > 3 ? c[3] : 0.0, x[0],
      m > 1 ? x[1] : nullptr, m > 2 ? x[2] : nullptr, m > 3 ? x[3] : nullptr, y);
  prof_end(st, P_OTHER, 8.0 * n * (m + 1), 1);
  return cudaGetLastError();
}

// Gram-Schmidt passes run in groups of GS = 8 basis vectors: the 8-wide
// kernels stream at the HBM copy rate (tools/vecbench.py), the 16/32-wide
// ones are register-limited to ~40% of it, so w is re-read once per extra
// group instead (+1 vector pass per 8).
constexpr int GS = 8;

// out[c] for grouped multidot partials (one warp per column)
__global__ void k_reduce_groups(const double* __restrict__ partials, int nblocks, int nv,
                                double* __restrict__ out) {
  const int col = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (col > nv) return;
  int g, i, cnt;
  if (col == nv) {
    g = 0;
    cnt = nv < GS ? nv : GS;
    i = cnt;
  } else {
    g = col / GS;
    i = col % GS;
    cnt = (nv - g * GS) < GS ? (nv - g * GS) : GS;
  }
  const double* p = partials + (long long)g * nblocks * (GS + 1);
  double s = 0.0;
  for (int b = lane; b < nblocks; b += 32) s += p[(long long)b * (cnt + 1) + i];
  s = warp_sum(s);
  if (lane == 0) out[col] = s;
}

cudaError_t multidot(cudaStream_t st, long long n, int nv, const double* V, long long vstride,
                     const double* w, double* partials, double* out) {
  // out[0..nv-1] = V_i . w, out[nv] = w . w  (fixed RED_BLOCKS grid)
  if (nv > 32) return cudaErrorInvalidValue;
  prof_begin(st);
  const int ng = nv == 0 ? 1 : (nv + GS - 1) / GS;
  if (nv == 0 && (reinterpret_cast<unsigned long long>(w) & 15) == 0) {
    k_norm2<<<RED_BLOCKS, RED_THREADS, 0, st>>>(n, w, partials);
    k_reduce_groups<<<1, 256, 0, st>>>(partials, RED_BLOCKS, 0, out);
    prof_end(st, P_DOT, 8.0 * n, 2);
    return cudaGetLastError();
  }
  for (int g = 0; g < ng; ++g) {
    const int cnt = nv - g * GS < GS ? nv - g * GS : GS;
    k_multidot<GS><<<RED_BLOCKS, RED_THREADS, 0, st>>>(
        n, cnt, V + (long long)g * GS * vstride, vstride, w,
        partials + (long long)g * RED_BLOCKS * (GS + 1));
  }
  k_reduce_groups<<<(nv + 1 + 7) / 8, 256, 0, st>>>(partials, RED_BLOCKS, nv, out);
  prof_end(st, P_DOT, 8.0 * n * (nv + ng), ng + 1);
  return cudaGetLastError();
}

cudaError_t axpy_multi(cudaStream_t st, long long n, int nv, const double* V, long long vstride,
                       const double* coefs_dev, double* w, double* partials, double* norm2_out) {
  if (nv > 32 || nv < 1) return cudaErrorInvalidValue;
  prof_begin(st);
  const int ng = (nv + GS - 1) / GS;
  for (int g = 0; g < ng; ++g) {
    const int cnt = nv - g * GS < GS ? nv - g * GS : GS;
    k_axpy_multi<GS><<<RED_BLOCKS, RED_THREADS, 0, st>>>(
        n, cnt, V + (long long)g * GS * vstride, vstride, coefs_dev + g * GS, w,
        g == ng - 1 ? partials : nullptr);
  }
  if (norm2_out) k_reduce_cols<<<1, 32, 0, st>>>(partials, RED_BLOCKS, 1, norm2_out);
  prof_end(st, P_AXPY, 8.0 * n * (nv + 2 * ng), ng + (norm2_out ? 1 : 0));
  return cudaGetLastError();
}

// dst <- (w - sum_{i<NV} c_i V_i) / na in ONE pass over all NV <= 32 basis
// vectors (no grouped re-read / re-write of w): NV is a template parameter,
// so all NV + 1 loads of an element are issued back to back
template <int NV>
__global__ void __launch_bounds__(RED_THREADS)
k_axpy_div_all(long long n, const double* __restrict__ V, long long vstride,
               const double* __restrict__ coefs, const double* __restrict__ w, double na,
               double* __restrict__ dst) {
  __shared__ double c[NV];
  for (int i = threadIdx.x; i < NV; i += blockDim.x) c[i] = coefs[i];
  __syncthreads();
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long k = (long long)blockIdx.x * blockDim.x + threadIdx.x; k < n; k += stride) {
    double a[NV];
#pragma unroll
    for (int i = 0; i < NV; ++i) a[i] = V[i * vstride + k];
    const double wk = w[k];
    double t = 0.0;
#pragma unroll
    for (int i = 0; i < NV; ++i) t = fma(c[i], a[i], t);
    dst[k] = (wk - t) / na;
  }
}

template <int NV>
cudaError_t launch_axpy_div_all(cudaStream_t st, long long n, int nv, const double* V,
                                long long vstride, const double* coefs, const double* w,
                                double na, double* dst) {
  if constexpr (NV > 1) {
    if (nv < NV) return launch_axpy_div_all<NV - 1>(st, n, nv, V, vstride, coefs, w, na, dst);
  }
  k_axpy_div_all<NV><<<RED_BLOCKS, RED_THREADS, 0, st>>>(n, V, vstride, coefs, w, na, dst);
  return cudaGetLastError();
}

// Gram-Schmidt update fused with the re-orthogonalisation dots: in one pass
// w <- w - sum_i c_i V_i, then partials of V_i . w (new w) and |w|^2.  The
// second use of V_i[k] re-reads the line the first loop just brought to L1.
template <int NV>
__global__ void __launch_bounds__(RED_THREADS)
k_axpy_dots(long long n, const double* __restrict__ V, long long vstride,
            const double* __restrict__ coefs, double* __restrict__ w,
            double* __restrict__ partials) {
  __shared__ double c[NV];
  for (int i = threadIdx.x; i < NV; i += blockDim.x) c[i] = coefs[i];
  __syncthreads();
  double acc[NV + 1];
#pragma unroll
  for (int i = 0; i <= NV; ++i) acc[i] = 0.0;
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long k = (long long)blockIdx.x * blockDim.x + threadIdx.x; k < n; k += stride) {
    double a[NV];
#pragma unroll
    for (int i = 0; i < NV; ++i) a[i] = V[i * vstride + k];
    double t = 0.0;
#pragma unroll
    for (int i = 0; i < NV; ++i) t = fma(c[i], a[i], t);
    const double wn = w[k] - t;
    w[k] = wn;
#pragma unroll
    for (int i = 0; i < NV; ++i) acc[i] = fma(V[i * vstride + k], wn, acc[i]);
    acc[NV] = fma(wn, wn, acc[NV]);
  }
  __shared__ double red[RED_THREADS / 32][NV + 1];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
  for (int i = 0; i <= NV; ++i) {
    const double v = warp_sum(acc[i]);
    if (lane == 0) red[wid][i] = v;
  }
  __syncthreads();
  for (int i = threadIdx.x; i <= NV; i += blockDim.x) {
    double s = 0.0;
    for (int w2 = 0; w2 < RED_THREADS / 32; ++w2) s += red[w2][i];
    partials[(long long)blockIdx.x * (NV + 1) + i] = s;
  }
}

template <int NV>
cudaError_t launch_axpy_dots(cudaStream_t st, long long n, int nv, const double* V,
                             long long vstride, const double* coefs, double* w,
                             double* partials) {
  if constexpr (NV > 1) {
    if (nv < NV) return launch_axpy_dots<NV - 1>(st, n, nv, V, vstride, coefs, w, partials);
  }
  k_axpy_dots<NV><<<RED_BLOCKS, RED_THREADS, 0, st>>>(n, V, vstride, coefs, w, partials);
  return cudaGetLastError();
}

cudaError_t axpy_dots(cudaStream_t st, long long n, int nv, const double* V, long long vstride,
                      const double* coefs_dev, double* w, double* partials, double* out) {
  if (nv > 32 || nv < 1) return cudaErrorInvalidValue;
  prof_begin(st);
  cudaError_t e = launch_axpy_dots<32>(st, n, nv, V, vstride, coefs_dev, w, partials);
  if (e == cudaSuccess) {
    k_reduce_cols<<<(nv + 1 + 7) / 8, 256, 0, st>>>(partials, RED_BLOCKS, nv + 1, out);
    e = cudaGetLastError();
  }
  prof_end(st, P_AXPY, 8.0 * n * (nv + 2), 2);
  return e;
}

cudaError_t axpy_div(cudaStream_t st, long long n, int nv, const double* V, long long vstride,
                     const double* coefs_dev, double* w, double na, double* dst) {
  // w is scratch: earlier groups update it in place, the last one divides
  if (nv > 32 || nv < 1) return cudaErrorInvalidValue;
  static const bool grouped = getenv("DG_AXPY_GROUPED") != nullptr;
  if (!grouped) {
    prof_begin(st);
    cudaError_t e = launch_axpy_div_all<32>(st, n, nv, V, vstride, coefs_dev, w, na, dst);
    prof_end(st, P_AXPY, 8.0 * n * (nv + 2), 1);
    return e;
  }
  prof_begin(st);
  const int ng = (nv + GS - 1) / GS;
  for (int g = 0; g < ng; ++g) {
    const int cnt = nv - g * GS < GS ? nv - g * GS : GS;
    const double* Vg = V + (long long)g * GS * vstride;
    if (g < ng - 1)
      k_axpy_multi<GS><<<RED_BLOCKS, RED_THREADS, 0, st>>>(n, cnt, Vg, vstride, coefs_dev + g * GS,
                                                           w, nullptr);
    else
      k_axpy_div<GS><<<RED_BLOCKS, RED_THREADS, 0, st>>>(n, cnt, Vg, vstride, coefs_dev + g * GS,
                                                         w, na, dst);
  }
  prof_end(st, P_AXPY, 8.0 * n * (nv + 2 * ng), ng);
  return cudaGetLastError();
}

// DCGS2 Arnoldi update, ONE pass over the NV finalised basis
// vectors Q_i, the lagged vector u (in/out) and z = A u:
//   q  = (u - sum s_i Q_i) / alpha                       (re-orthogonalised u)
//   w  = (z - sum_{i<NV} g_i Q_i - g_NV q) / alpha       (= A q, Arnoldi relation)
//   u' = w - sum_{i<NV} h_i Q_i - h_NV q                 (next lagged vector)
// u <- q, unext <- u', partials of |u'|^2.  coefs = [s (NV), g (NV+1),
// h (NV+1), alpha].
#ifndef DG_DCGS2_MINB
#define DG_DCGS2_MINB 1
#endif
template <int NV>
__global__ void __launch_bounds__(RED_THREADS, DG_DCGS2_MINB)
k_dcgs2_update(long long n, const double* __restrict__ Q, long long vstride,
               const double* __restrict__ coefs, double* __restrict__ u,
               const double* __restrict__ z, double* __restrict__ unext,
               double* __restrict__ partials) {
  // u' = z / alpha - sum_{i<NV} c_i Q_i - c_NV q with c = g / alpha + h: two
  // coefficient sets (s, c) instead of three.  k-pairs with 16-byte loads
  // and stores (twice the bytes in flight per instruction); odd n: the last
  // element by one thread
  __shared__ double cs[NV + 1], cc[NV + 1];
  pdl_trigger();
  pdl_wait();  // (programmatic dependent launch, small problems: dg_common.cuh)
  const double alpha = coefs[3 * NV + 2];
  for (int i = threadIdx.x; i <= NV; i += blockDim.x) {
    cs[i] = i < NV ? coefs[i] : 0.0;
    cc[i] = coefs[NV + i] / alpha + coefs[2 * NV + 1 + i];
  }
  __syncthreads();
  double acc = 0.0;
  const long long n2 = n >> 1;
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long k = (long long)blockIdx.x * blockDim.x + threadIdx.x; k < n2; k += stride) {
    double2 a[NV + 1];
#pragma unroll
    for (int i = 0; i < NV; ++i) a[i] = reinterpret_cast<const double2*>(Q + i * vstride)[k];
    const double2 uk = reinterpret_cast<const double2*>(u)[k];
    const double2 zk = reinterpret_cast<const double2*>(z)[k];
    double t1x = 0.0, t2x = 0.0, t1y = 0.0, t2y = 0.0;
#pragma unroll
    for (int i = 0; i < NV; ++i) {
      t1x = fma(cs[i], a[i].x, t1x);
      t2x = fma(cc[i], a[i].x, t2x);
      t1y = fma(cs[i], a[i].y, t1y);
      t2y = fma(cc[i], a[i].y, t2y);
    }
    double2 q, un;
    q.x = (uk.x - t1x) / alpha;
    q.y = (uk.y - t1y) / alpha;
    un.x = zk.x / alpha - t2x - cc[NV] * q.x;
    un.y = zk.y / alpha - t2y - cc[NV] * q.y;
    reinterpret_cast<double2*>(u)[k] = q;
    reinterpret_cast<double2*>(unext)[k] = un;
    acc = fma(un.x, un.x, acc);
    acc = fma(un.y, un.y, acc);
  }
  if ((n & 1) && blockIdx.x == 0 && threadIdx.x == 0) {
    const long long k = n - 1;
    double t1 = 0.0, t2 = 0.0;
#pragma unroll
    for (int i = 0; i < NV; ++i) {
      const double ai = Q[i * vstride + k];
      t1 = fma(cs[i], ai, t1);
      t2 = fma(cc[i], ai, t2);
    }
    const double q = (u[k] - t1) / alpha;
    const double un = z[k] / alpha - t2 - cc[NV] * q;
    u[k] = q;
    unext[k] = un;
    acc = fma(un, un, acc);
  }
  __shared__ double red[RED_THREADS / 32];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  acc = warp_sum(acc);
  if (lane == 0) red[wid] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int w2 = 0; w2 < RED_THREADS / 32; ++w2) s += red[w2];
    partials[blockIdx.x] = s;
  }
}

template <int NV>
cudaError_t launch_dcgs2(cudaStream_t st, long long n, int nv, const double* Q, long long vstride,
                         const double* coefs, double* u, const double* z, double* unext,
                         double* partials, int* used_grid) {
  if constexpr (NV > 0) {
    if (nv < NV)
      return launch_dcgs2<NV - 1>(st, n, nv, Q, vstride, coefs, u, z, unext, partials, used_grid);
  }
  // one wave: every resident CTA slot once (the register footprint grows
  // with NV; <= RED_BLOCKS partials for the deterministic column reduction)
  static int grid = 0;
  if (grid == 0) {
    int dev = 0, nsm = 0, occ = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_dcgs2_update<NV>, RED_THREADS, 0);
    grid = std::min(RED_BLOCKS, std::max(1, nsm * std::max(occ, 1)));
  }
  *used_grid = grid;
  return launch_k(k_dcgs2_update<NV>, dim3(grid), dim3(RED_THREADS), 0, st, n, Q, vstride, coefs, u,
                  z, unext, partials);
}

// DCGS2 dual Gram-Schmidt dots (the unfused form of the dots the div(hV)
// kernel can fuse, dg_wkernel.cuh gs_dots).  Row b of rows = block b's
// partials of (Q_i.z, Q_i.u) for i < nv, then (z.z, z.u), then (u.z, u.u):
// 2 (nv + 2) columns, summed over the rows by reduce_rows (deterministic).
// The vectors go in groups of at most 8, one launch per group (each its own
// one-wave grid; the last group also takes the z / u products): with all
// 2 nv accumulators in registers the kernel spilled from nv ~ 12 on (1.5
// TB/s at nv = 16).  Each thread handles k-pairs with 16-byte loads so a
// group keeps 2 x (G + 2) loads in flight per thread.
template <int G, bool LAST>
__global__ void __launch_bounds__(RED_THREADS)
k_dual_dots(long long n, int nv, int g0, const double* __restrict__ Q, long long vstride,
            const double* __restrict__ z, const double* __restrict__ u, double* __restrict__ rows) {
  constexpr int GA = G > 0 ? G : 1;
  pdl_trigger();
  pdl_wait();  // (programmatic dependent launch below 2^24 DoF: dg_pdl.cuh)
  double pz[GA], pu[GA];
#pragma unroll
  for (int i = 0; i < GA; ++i) pz[i] = pu[i] = 0.0;
  double zz = 0.0, zu = 0.0, uu = 0.0;
  const long long n2 = n >> 1;
  const long long stride = (long long)gridDim.x * blockDim.x;
  const double* Qg = Q + (long long)g0 * vstride;
  for (long long k = (long long)blockIdx.x * blockDim.x + threadIdx.x; k < n2; k += stride) {
    double2 a[GA];
#pragma unroll
    for (int i = 0; i < G; ++i) a[i] = reinterpret_cast<const double2*>(Qg + i * vstride)[k];
    const double2 zk = reinterpret_cast<const double2*>(z)[k];
    const double2 uk = reinterpret_cast<const double2*>(u)[k];
#pragma unroll
    for (int i = 0; i < G; ++i) {
      pz[i] = fma(a[i].x, zk.x, pz[i]);
      pu[i] = fma(a[i].x, uk.x, pu[i]);
      pz[i] = fma(a[i].y, zk.y, pz[i]);
      pu[i] = fma(a[i].y, uk.y, pu[i]);
    }
    if (LAST) {
      zz = fma(zk.x, zk.x, zz);
      zu = fma(zk.x, uk.x, zu);
      uu = fma(uk.x, uk.x, uu);
      zz = fma(zk.y, zk.y, zz);
      zu = fma(zk.y, uk.y, zu);
      uu = fma(uk.y, uk.y, uu);
    }
  }
  if ((n & 1) && blockIdx.x == 0 && threadIdx.x == 0) {  // odd n: the last element
    const long long k = n - 1;
    const double zk = z[k], uk = u[k];
#pragma unroll
    for (int i = 0; i < G; ++i) {
      const double a = Qg[i * vstride + k];
      pz[i] = fma(a, zk, pz[i]);
      pu[i] = fma(a, uk, pu[i]);
    }
    if (LAST) {
      zz = fma(zk, zk, zz);
      zu = fma(zk, uk, zu);
      uu = fma(uk, uk, uu);
    }
  }
  constexpr int NT = 2 * G + (LAST ? 4 : 0);
  __shared__ double red[RED_THREADS / 32][NT > 0 ? NT : 1];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
  for (int col = 0; col < NT; ++col) {
    double v;
    if (col < 2 * G) v = (col & 1) ? pu[col >> 1] : pz[col >> 1];
    else if (col == 2 * G) v = zz;
    else if (col == 2 * G + 1 || col == 2 * G + 2) v = zu;
    else v = uu;
    v = warp_sum(v);
    if (lane == 0) red[wid][col] = v;
  }
  __syncthreads();
  const int ncols = 2 * (nv + 2);
  for (int col = threadIdx.x; col < NT; col += blockDim.x) {
    double t = 0.0;
    for (int w2 = 0; w2 < RED_THREADS / 32; ++w2) t += red[w2][col];
    const int dst = (col < 2 * G) ? 2 * g0 + col : 2 * nv + (col - 2 * G);
    rows[(long long)blockIdx.x * ncols + dst] = t;
  }
}

// vectors per dual-dot launch (z and u are re-read once per group): 12 (80
// registers) measured best at cfg4 size -- nv = 12 / 24 / 31: 2.74 / 5.54 /
// 7.36 ms against 3.15 / 6.01 / 7.97 with groups of 8 and 2.73 / 6.69 / 7.73
// with groups of 16 (100 registers)
#ifndef DG_DD_GROUP
#define DG_DD_GROUP 12
#endif
template <int G, bool LAST>
int dd_grid() {
  static int grid = 0;
  if (grid == 0) {
    int dev = 0, nsm = 0, per_sm = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_dual_dots<G, LAST>, RED_THREADS, 0);
    grid = std::min(RED_BLOCKS, std::max(1, nsm * std::max(per_sm, 1)));
  }
  return grid;
}

template <int T>
cudaError_t launch_dd_tail(cudaStream_t st, int tail, long long n, int nv, int g0,
                           const double* Q, long long vstride, const double* z, const double* u,
                           double* rows, int* grid) {
  if constexpr (T > 0) {
    if (tail < T) return launch_dd_tail<T - 1>(st, tail, n, nv, g0, Q, vstride, z, u, rows, grid);
  }
  *grid = dd_grid<T, true>();
  launch_k(k_dual_dots<T, true>, dim3(*grid), dim3(RED_THREADS), 0, st, n, nv, g0, Q, vstride, z, u,
           rows);
  return cudaGetLastError();
}

cudaError_t launch_dual_dots(cudaStream_t st, long long n, int nv, const double* Q,
                             long long vstride, const double* z, const double* u, double* rows,
                             int* used_grid) {
  // one one-wave launch per group of DG_DD_GROUP vectors + the tail group
  // (1..DG_DD_GROUP vectors and the u / z products); the row block is zeroed first so the
  // groups' different grids sum exactly in reduce_rows
  constexpr int GF = DG_DD_GROUP;
  const int nfull = nv > 0 ? (nv - 1) / GF : 0;
  const int tail = nv - GF * nfull;
  const int ncols = 2 * (nv + 2);
  cudaError_t e = cudaMemsetAsync(rows, 0, (size_t)RED_BLOCKS * ncols * sizeof(double), st);
  if (e != cudaSuccess) return e;
  int gmax = 1;
  for (int g = 0; g < nfull; ++g) {
    const int grid = dd_grid<GF, false>();
    launch_k(k_dual_dots<GF, false>, dim3(grid), dim3(RED_THREADS), 0, st, n, nv, GF * g, Q,
             vstride, z, u, rows);
    e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    gmax = std::max(gmax, grid);
  }
  int gt = 1;
  e = launch_dd_tail<GF>(st, tail, n, nv, GF * nfull, Q, vstride, z, u, rows, &gt);
  *used_grid = std::max(gmax, gt);
  return e;
}

cudaError_t dual_dots(cudaStream_t st, long long n, int nv, const double* Q, long long vstride,
                      const double* z, const double* u, double* rows, int* nrows) {
  if (nv > 31 || nv < 0) return cudaErrorInvalidValue;
  prof_begin(st);
  cudaError_t e = launch_dual_dots(st, n, nv, Q, vstride, z, u, rows, nrows);
  prof_end(st, P_DOT, 8.0 * n * (nv + 2), 1);
  return e;
}

// max over the nodes of |U[e][num][i] / U[e][den][i]| (optionally only where
// mask[e n^d + i] != 0): the runner's max |w| diagnostic (runner.py:247-260);
// per-block maxima in partials, exact (order-independent)
__global__ void __launch_bounds__(RED_THREADS)
k_max_ratio(long long n_el, int V, int np, const double* __restrict__ U, int num, int den,
            const uint8_t* __restrict__ mask, double* __restrict__ partials) {
  double m = 0.0;
  const long long n = n_el * np;
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long k = (long long)blockIdx.x * blockDim.x + threadIdx.x; k < n; k += stride) {
    if (mask && !mask[k]) continue;
    const long long e = k / np, i = k - e * np;
    const double* u = U + e * V * np;
    m = fmax(m, fabs(u[(long long)num * np + i] / u[(long long)den * np + i]));
  }
  for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
  __shared__ double red[RED_THREADS / 32];
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < RED_THREADS / 32; ++w) t = fmax(t, red[w]);
    partials[blockIdx.x] = t;
  }
}

cudaError_t max_ratio(cudaStream_t st, long long n_el, int V, int np, const double* U, int num,
                      int den, const uint8_t* mask, double* partials) {
  prof_begin(st);
  k_max_ratio<<<RED_BLOCKS, RED_THREADS, 0, st>>>(n_el, V, np, U, num, den, mask, partials);
  prof_end(st, P_OTHER, 8.0 * n_el * np * 2, 1);
  return cudaGetLastError();
}

cudaError_t dcgs2_update(cudaStream_t st, long long n, int nv, const double* Q, long long vstride,
                         const double* coefs_dev, double* u, const double* z, double* unext,
                         double* partials, double* out) {
  if (nv > 31 || nv < 0) return cudaErrorInvalidValue;
  prof_begin(st);
  int grid = RED_BLOCKS;
  cudaError_t e = launch_dcgs2<31>(st, n, nv, Q, vstride, coefs_dev, u, z, unext, partials, &grid);
  if (e == cudaSuccess) {
    k_reduce_cols<<<1, 256, 0, st>>>(partials, grid, 1, out);
    e = cudaGetLastError();
  }
  prof_end(st, P_AXPY, 8.0 * n * (nv + 4), 2);
  return e;
}

cudaError_t scale(cudaStream_t st, long long n, double a, bool divide, const double* x,
                  double* y) {
  prof_begin(st);
  k_scale<<<grid_for(n), RED_THREADS, 0, st>>>(n, a, divide ? 1 : 0, x, y);
  prof_end(st, P_OTHER, 16.0 * n, 1);
  return cudaGetLastError();
}

cudaError_t frozen(cudaStream_t st, long long n_el, int np, int d, const double* U, double gm1,
                   double kf, double* h, double* K) {
  prof_begin(st);
  k_frozen<<<grid_for(n_el * np), RED_THREADS, 0, st>>>(n_el, np, d, U, gm1, kf, h, K);
  prof_end(st, P_OTHER, 8.0 * n_el * np * (d + 4), 1);
  return cudaGetLastError();
}

cudaError_t state_pressure(cudaStream_t st, long long n_el, int np, int d, const double* U,
                           double gm1, double kf, double* p) {
  prof_begin(st);
  k_state_pressure<<<grid_for(n_el * np), RED_THREADS, 0, st>>>(n_el, np, d, U, gm1, kf, p);
  prof_end(st, P_OTHER, 8.0 * n_el * np * (d + 3), 1);
  return cudaGetLastError();
}

cudaError_t pressure_dp(cudaStream_t st, long long n, const double* x, const double* K, double gm1,
                        double kf, double* p_old, double* partials, double* out2) {
  prof_begin(st);
  k_pressure_dp<<<RED_BLOCKS, RED_THREADS, 0, st>>>(n, x, K, gm1, kf, p_old, partials);
  k_reduce_cols<<<1, 64, 0, st>>>(partials, RED_BLOCKS, 2, out2);
  prof_end(st, P_OTHER, 32.0 * n, 2);
  return cudaGetLastError();
}

cudaError_t set_iterate(cudaStream_t st, long long n_el, int np, int V, const double* acc,
                        const double* guess, double* it) {
  prof_begin(st);
  k_set_iterate<<<grid_for(n_el * V * np), RED_THREADS, 0, st>>>(n_el, np, V, acc, guess, it);
  prof_end(st, P_OTHER, 16.0 * n_el * V * np, 1);
  return cudaGetLastError();
}

cudaError_t copy_comps(cudaStream_t st, long long n_el, int np, int nc, const double* src,
                       long long s_estride, double* dst, long long d_estride) {
  prof_begin(st);
  k_copy_comps<<<grid_for(n_el * nc * np), RED_THREADS, 0, st>>>(n_el, np, nc, src, s_estride,
                                                                  dst, d_estride);
  prof_end(st, P_OTHER, 16.0 * n_el * nc * np, 1);
  return cudaGetLastError();
}

cudaError_t positivity(cudaStream_t st, long long n_el, int np, int d, const double* U, double gm1,
                       double kf, double* partials) {
  prof_begin(st);
  k_positivity<<<RED_BLOCKS, RED_THREADS, 0, st>>>(n_el, np, d, U, gm1, kf, partials);
  prof_end(st, P_OTHER, 8.0 * n_el * np * (d + 2), 1);
  return cudaGetLastError();
}

// many rows (e.g. one per element-kernel warp) x ncols (<= 96): RED_BLOCKS
// CTAs each sum a contiguous row range in order, 32 columns at a time, then
// k_reduce_cols (deterministic)
__global__ void __launch_bounds__(RED_THREADS)
k_reduce_rows(const double* __restrict__ partials, long long nrows, int ncols,
              double* __restrict__ out) {
  pdl_trigger();
  pdl_wait();
  const long long per = (nrows + gridDim.x - 1) / gridDim.x;
  const long long r0 = (long long)blockIdx.x * per;
  const long long r1 = r0 + per < nrows ? r0 + per : nrows;
  const int cl = threadIdx.x & 31, grp = threadIdx.x >> 5;  // 8 row groups
  __shared__ double red[RED_THREADS / 32][32];
  for (int c0 = 0; c0 < ncols; c0 += 32) {
    const int col = c0 + cl;
    double s = 0.0;
    if (col < ncols)
      for (long long r = r0 + grp; r < r1; r += RED_THREADS / 32) s += partials[r * ncols + col];
    red[grp][cl] = s;
    __syncthreads();
    if (threadIdx.x < 32 && c0 + threadIdx.x < ncols) {
      double t = 0.0;
      for (int g = 0; g < RED_THREADS / 32; ++g) t += red[g][threadIdx.x];
      out[(long long)blockIdx.x * ncols + c0 + threadIdx.x] = t;
    }
    __syncthreads();
  }
}

cudaError_t reduce_rows(cudaStream_t st, const double* partials, long long nrows, int ncols,
                        double* tmp, double* out) {
  prof_begin(st);
  launch_k(k_reduce_rows, dim3(RED_BLOCKS), dim3(RED_THREADS), 0, st, partials, nrows, ncols, tmp);
  launch_k(k_reduce_cols, dim3((ncols + 7) / 8), dim3(256), 0, st, (const double*)tmp,
           (int)RED_BLOCKS, ncols, out);
  prof_end(st, P_DOT, 8.0 * nrows * ncols, 2);
  return cudaGetLastError();
}

// ---- device-resident DCGS2 Arnoldi scalars (ArnState, dg_vector.cuh) -------
// One warp per kernel; every sum runs in the order of the host loop of
// dcgs2_cycle (dg_runtime.cu), lane i owning row i of the O(j^2) products.
__global__ void k_arn_init(ArnState* a, int m, double bn, double target, double beta,
                           int iterations, int max_iter) {
  const int t = threadIdx.x;
  for (int i = t; i < (ARN_M + 1) * ARN_M; i += blockDim.x) a->Hb[i] = 0.0;
  for (int i = t; i < ARN_M; i += blockDim.x) {
    a->cs[i] = 0.0;
    a->sn[i] = 0.0;
    a->hist[i] = 0.0;
  }
  for (int i = t; i <= ARN_M; i += blockDim.x) a->g[i] = i == 0 ? beta : 0.0;
  if (t == 0) {
    a->bn = bn;
    a->target = target;
    a->nb = 0.0;
    a->m = m;
    a->done = 0;
    a->stop = 0;
    a->breakdown = 0;
    a->iterations = iterations;
    a->max_iter = max_iter;
    a->steps_run = 0;
  }
}

// nrows > 0: `src` holds nrows partial rows of 2 (j + 2) columns (the fused
// dots of the div(hV) kernel / the dual-dot pass); the block (1024 threads)
// first sums them, warp w columns w, w + 32, ... with lane-strided rows and a
// fixed warp tree (deterministic).  nrows == 0: `src` holds the reduced dots.
// Hbar is staged in shared memory by the whole block while the rows are
// summed, so the serial part runs out of shared memory only.
__global__ void k_arn_pre(ArnState* a, int j, const double* __restrict__ src, int nrows,
                          double* __restrict__ coefs) {
  pdl_trigger();
  pdl_wait();
  if (a->stop) return;
  __shared__ double sdots[2 * (ARN_M + 2)];
  __shared__ double sH[(ARN_M + 1) * ARN_M];
  const int m = a->m;
  for (int i = threadIdx.x; i < (j + 1) * m; i += blockDim.x) sH[i] = a->Hb[i];
  const int ncols = 2 * (j + 2);
  if (nrows > 0) {
    const int wl = threadIdx.x & 31, ww = threadIdx.x >> 5, nw = blockDim.x >> 5;
    for (int col = ww; col < ncols; col += nw) {
      double t = 0.0;
      for (int r = wl; r < nrows; r += 32) t += src[(long long)r * ncols + col];
      t = warp_sum(t);
      if (wl == 0) sdots[col] = t;
    }
  } else {
    for (int i = threadIdx.x; i < ncols; i += blockDim.x) sdots[i] = src[i];
  }
  __syncthreads();
  if (threadIdx.x >= 32) return;
  const double* dots = sdots;
  const int lane = threadIdx.x;
  __shared__ double sv[ARN_M + 1], gv[ARN_M + 1];
  __shared__ double sh_alpha, sh_st;
  __shared__ int sh_brk;
  if (lane < j) sv[lane] = dots[2 * lane + 1];
  __syncwarp();
  if (lane == 0) {
    const double uu = dots[2 * j + 3];
    double s2 = 0.0, st_ = 0.0;
    for (int i = 0; i < j; ++i) {
      s2 = __dadd_rn(s2, __dmul_rn(sv[i], sv[i]));  // (unfused, as the host loop rounds)
      st_ = __dadd_rn(st_, __dmul_rn(sv[i], dots[2 * i]));
    }
    double alpha = 1.0;
    int brk = 0;
    if (j > 0) {
      const double a2 = uu - s2;
      double hjj;
      if (!(a2 > 1e-20 * uu) || !isfinite(a2)) {
        hjj = (a2 > 0.0 && isfinite(a2)) ? sqrt(a2) : 0.0;
        brk = 1;
      } else {
        alpha = sqrt(a2);
        hjj = alpha;
      }
      sH[j * m + j - 1] = hjj;
      a->Hb[j * m + j - 1] = hjj;
    }
    sh_alpha = alpha;
    sh_st = st_;
    sh_brk = brk;
  }
  // column j-1 of Hbar takes the re-orthogonalisation correction
  if (j > 0 && lane < j) {
    const double v = sH[lane * m + j - 1] + sv[lane];
    sH[lane * m + j - 1] = v;
    a->Hb[lane * m + j - 1] = v;
  }
  __syncwarp();
  if (sh_brk) {
    if (lane == 0) {
      a->breakdown = 1;
      a->stop = 1;
    }
    return;
  }
  const double alpha = sh_alpha;
  // g = Hbar[0:j+1, 0:j] s
  if (lane <= j) {
    double t = 0.0;
    for (int k = (lane - 1 > 0 ? lane - 1 : 0); k < j; ++k)
      t = __dadd_rn(t, __dmul_rn(sH[lane * m + k], sv[k]));
    gv[lane] = t;
  }
  __syncwarp();
  double hv = 0.0;
  if (lane < j) hv = (dots[2 * lane] - gv[lane]) / alpha;
  if (lane == j) hv = ((dots[2 * j + 1] - sh_st) / alpha - gv[j]) / alpha;
  if (lane <= j) {
    a->Hb[lane * m + j] = hv;
    if (lane < j) coefs[lane] = sv[lane];
    coefs[j + lane] = gv[lane];
    coefs[2 * j + 1 + lane] = hv;
  }
  if (lane == 0) {
    coefs[3 * j + 2] = alpha;
    const double zz = dots[2 * j];
    a->nb = sqrt(fmax(zz, 0.0)) / alpha;
  }
}

// nparts > 0: na2p holds the update kernel's per-CTA partials of |u'|^2
// (summed here as k_reduce_cols would: lane-strided, fixed warp tree).  One
// warp: the lanes stage column j of Hbar and the rotations in shared memory
// (one round trip), lane 0 runs the dependent Givens chain from there.
__global__ void k_arn_post(ArnState* a, int j, const double* __restrict__ na2p, int nparts) {
  pdl_trigger();
  pdl_wait();
  if (a->stop || threadIdx.x >= 32) return;
  const int lane = threadIdx.x;
  const int m = a->m;
  __shared__ double col[ARN_M + 2], cs[ARN_M + 1], sn[ARN_M + 1];
  if (lane <= j) col[lane] = a->Hb[lane * m + j];
  if (lane < j) {
    cs[lane] = a->cs[lane];
    sn[lane] = a->sn[lane];
  }
  const double bn = a->bn, nb = a->nb, target = a->target, gj = a->g[j];
  const int it0 = a->iterations, max_iter = a->max_iter, steps0 = a->steps_run;
  double na2 = 0.0;
  if (nparts > 0) {
    for (int b = lane; b < nparts; b += 32) na2 += na2p[b];
    na2 = warp_sum(na2);
  } else {
    na2 = na2p[0];
  }
  __syncwarp();
  if (lane != 0) return;
  const double na = sqrt(na2);
  a->Hb[(j + 1) * m + j] = na;
  col[j + 1] = na;
  const bool happy = na <= 1e-14 * fmax(bn, nb);
  for (int i = 0; i < j; ++i) {
    const double t = __dadd_rn(__dmul_rn(cs[i], col[i]), __dmul_rn(sn[i], col[i + 1]));
    col[i + 1] = __dadd_rn(__dmul_rn(-sn[i], col[i]), __dmul_rn(cs[i], col[i + 1]));
    col[i] = t;
  }
  const double den = hypot(col[j], col[j + 1]);
  const double c = den != 0.0 ? col[j] / den : 1.0;
  const double sj = den != 0.0 ? col[j + 1] / den : 0.0;
  a->cs[j] = c;
  a->sn[j] = sj;
  const double g1 = -sj * gj;
  a->g[j + 1] = g1;
  a->g[j] = c * gj;
  a->done = j + 1;
  a->iterations = it0 + 1;
  a->steps_run = steps0 + 1;
  const double est = fabs(g1);
  a->hist[j] = est / bn;
  if (happy) a->breakdown = 1;
  if (happy || est <= target || it0 + 1 >= max_iter) a->stop = 1;
}

cudaError_t arn_init(cudaStream_t st, ArnState* a, int m, double bn, double target, double beta,
                     int iterations, int max_iter) {
  if (m < 1 || m > ARN_M) return cudaErrorInvalidValue;
  k_arn_init<<<1, 256, 0, st>>>(a, m, bn, target, beta, iterations, max_iter);
  return cudaGetLastError();
}

cudaError_t arn_pre(cudaStream_t st, ArnState* a, int j, const double* src, int nrows,
                    double* coefs) {
  prof_begin(st);
  launch_k(k_arn_pre, dim3(1), dim3(nrows > 0 ? 1024 : 32), 0, st, a, j, src, nrows, coefs);
  prof_end(st, P_DOT, 8.0 * (nrows > 0 ? nrows : 1) * 2 * (j + 2), 1);
  return cudaGetLastError();
}

cudaError_t arn_post(cudaStream_t st, ArnState* a, int j, const double* na2, int nparts) {
  prof_begin(st);
  launch_k(k_arn_post, dim3(1), dim3(32), 0, st, a, j, na2, nparts);
  prof_end(st, P_AXPY, 8.0 * (nparts > 0 ? nparts : 1), 1);
  return cudaGetLastError();
}

// the update pass without its column reduction (arn_post sums the partials)
cudaError_t dcgs2_update_partials(cudaStream_t st, long long n, int nv, const double* Q,
                                  long long vstride, const double* coefs_dev, double* u,
                                  const double* z, double* unext, double* partials, int* nparts) {
  if (nv > 31 || nv < 0) return cudaErrorInvalidValue;
  prof_begin(st);
  int grid = RED_BLOCKS;
  cudaError_t e = launch_dcgs2<31>(st, n, nv, Q, vstride, coefs_dev, u, z, unext, partials, &grid);
  *nparts = grid;
  prof_end(st, P_AXPY, 8.0 * n * (nv + 4), 1);
  return e;
}

cudaError_t reduce_cols(cudaStream_t st, const double* partials, int nblocks, int ncols, double* out) {
  prof_begin(st);
  k_reduce_cols<<<(ncols + 7) / 8, 256, 0, st>>>(partials, nblocks, ncols, out);
  prof_end(st, P_OTHER, 8.0 * nblocks * ncols, 1);
  return cudaGetLastError();
}

}  // namespace dg
