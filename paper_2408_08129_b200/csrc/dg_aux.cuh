// Auxiliary per-element kernels: standalone factorised mass inverse
// (orodg/geometry.py:372-396) and conserved-variable integrals
// (orodg/dgops.py:505-511).  Same thread-per-point shared-memory passes as
// the fused operator kernel.
#pragma once
#include "dg_operator.cuh"

namespace dg {

template <int N>
struct AuxParams {
  const int* elem;
  const double* col;
  GeoConst gc;
  int n_el;
  int ncomp;
  CView in;          // dual (mass inverse) or state (integrate)
  CView in2;         // inner product: second field
  Model model;       // Courant report
  double* tr;        // interp (trace mode): face traces of component 0, (n_el, 2d, n^(d-1))
  MView out;         // nodal result (mass inverse)
  double* partial;   // integrate: (grid, ncomp)
  Tab<N> tab;
};

template <int D, int N>
struct AuxLayout {
  static constexpr int NP = ipow(N, D);
  static constexpr int KMAX = 5;
  static constexpr int EPB = (256 / NP) > 1 ? (256 / NP) : 1;
  static constexpr int THREADS = ((EPB * NP + 31) / 32) * 32;
  static constexpr int SLOTS = (THREADS + NP - 1) / NP;
  static constexpr int TABD = (int)(sizeof(Tab<N>) / sizeof(double));
  static constexpr size_t SMEM = (size_t)(TABD + 64 + SLOTS * 2 * KMAX * NP) * sizeof(double);
};

template <int D, int N>
__device__ __forceinline__ double wdet_at(const int* elem, const double* col, const GeoConst& gc,
                                          long long e, int q, const Tab<N>& T) {
  constexpr int NQH = ipow(N, D - 1);
  const ElemGeo<D> g = elem_geo<D>(elem, gc, e);
  const int qh = q / N;
  double omh = 1.0;  // 1 - h/z_top (column table)
  if (gc.terrain) omh = col[(long long)g.col * gc.col_stride + qh];
  (void)NQH;
  const double zz = g.s[D - 1] * omh;
  double det = 1.0;
  for (int a = 0; a < D - 1; ++a) det = det * g.s[a];
  det = det * zz;
  double w = 1.0;
  for (int a = 0; a < D; ++a) w *= T.qw[digit<D, N>(q, a)];
  return w * det;
}

// nodal = B^-1 (x) .. diag(1/(w det)) B^-T (x) .. dual
template <int D, int N>
__global__ void __launch_bounds__(AuxLayout<D, N>::THREADS)
minv_kernel(const __grid_constant__ AuxParams<N> P) {
  using L = AuxLayout<D, N>;
  constexpr int NP = L::NP;
  extern __shared__ double smem[];
  double* tb = smem;
  {
    const double* src = reinterpret_cast<const double*>(&P.tab);
    for (int i = threadIdx.x; i < L::TABD; i += blockDim.x) tb[i] = src[i];
    __syncthreads();
  }
  const Tab<N>& T = *reinterpret_cast<const Tab<N>*>(tb);
  const int el = threadIdx.x / NP, q = threadIdx.x - el * NP;
  const long long e = (long long)blockIdx.x * L::EPB + el;
  const bool valid = el < L::EPB && e < P.n_el;
  const long long es = valid ? e : 0;
  double* X = smem + L::TABD + 64 + el * 2 * L::KMAX * NP;
  double* Y = X + L::KMAX * NP;
  for (int c0 = 0; c0 < P.ncomp; c0 += L::KMAX) {
    const int kc = min(L::KMAX, P.ncomp - c0);
    for (int c = 0; c < L::KMAX; ++c) X[c * NP + q] = c < kc ? P.in(es, c0 + c, q) : 0.0;
    __syncthreads();
    // B^-T along every axis
    double* s = X;
    double* d = Y;
    for (int a = D - 1; a >= 0; --a) {
      pass1d<D, N, L::KMAX, true>(&T.Binv[0][0], s, d, q, a, NP);
      __syncthreads();
      double* t = s; s = d; d = t;
    }
    const double inv = 1.0 / wdet_at<D, N>(P.elem, P.col, P.gc, es, q, T);
    for (int c = 0; c < L::KMAX; ++c) s[c * NP + q] *= inv;
    __syncthreads();
    for (int a = D - 1; a >= 0; --a) {
      pass1d<D, N, L::KMAX, false>(&T.Binv[0][0], s, d, q, a, NP);
      __syncthreads();
      double* t = s; s = d; d = t;
    }
    if (valid)
      for (int c = 0; c < kc; ++c)
        P.out.p[e * P.out.estride + (c0 + c) * P.out.cstride + q] = s[c * NP + q];
    __syncthreads();
  }
}

// per-CTA partial integrals sum_q w det (B U)_q for every component
template <int D, int N>
__global__ void __launch_bounds__(AuxLayout<D, N>::THREADS)
integrate_kernel(const __grid_constant__ AuxParams<N> P) {
  using L = AuxLayout<D, N>;
  constexpr int NP = L::NP;
  extern __shared__ double smem[];
  double* tb = smem;
  {
    const double* src = reinterpret_cast<const double*>(&P.tab);
    for (int i = threadIdx.x; i < L::TABD; i += blockDim.x) tb[i] = src[i];
    __syncthreads();
  }
  const Tab<N>& T = *reinterpret_cast<const Tab<N>*>(tb);
  double* red = smem + L::TABD;
  const int el = threadIdx.x / NP, q = threadIdx.x - el * NP;
  const long long e = (long long)blockIdx.x * L::EPB + el;
  const bool valid = el < L::EPB && e < P.n_el;
  const long long es = valid ? e : 0;
  double* X = smem + L::TABD + 64 + el * 2 * L::KMAX * NP;
  double* Y = X + L::KMAX * NP;
  const double wd = wdet_at<D, N>(P.elem, P.col, P.gc, es, q, T);
  for (int c0 = 0; c0 < P.ncomp; c0 += L::KMAX) {
    const int kc = min(L::KMAX, P.ncomp - c0);
    for (int c = 0; c < L::KMAX; ++c) X[c * NP + q] = c < kc ? P.in(es, c0 + c, q) : 0.0;
    __syncthreads();
    double* s = X;
    double* d = Y;
    for (int a = D - 1; a >= 0; --a) {
      pass1d<D, N, L::KMAX, false>(&T.B[0][0], s, d, q, a, NP);
      __syncthreads();
      double* t = s; s = d; d = t;
    }
    for (int c = 0; c < kc; ++c) {
      double v = valid ? s[c * NP + q] * wd : 0.0;
      for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
      if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
      __syncthreads();
      if (threadIdx.x == 0) {
        double acc = 0.0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) acc += red[w];
        P.partial[(long long)blockIdx.x * P.ncomp + c0 + c] = acc;
      }
      __syncthreads();
    }
  }
}

// nodes -> Gauss points for ncomp components (frozen h of the Helmholtz pair,
// evaluated once per pressure fixed-point iterate)
// KC: components per pass round (1 for the frozen h: no idle comps)
template <int D, int N, int KC>
__global__ void __launch_bounds__(AuxLayout<D, N>::THREADS)
interp_kernel(const __grid_constant__ AuxParams<N> P) {
  using L = AuxLayout<D, N>;
  constexpr int NP = L::NP;
  extern __shared__ double smem[];
  {
    const double* src = reinterpret_cast<const double*>(&P.tab);
    for (int i = threadIdx.x; i < L::TABD; i += blockDim.x) smem[i] = src[i];
    __syncthreads();
  }
  const Tab<N>& T = *reinterpret_cast<const Tab<N>*>(smem);
  const int el = threadIdx.x / NP, q = threadIdx.x - el * NP;
  const long long e = (long long)blockIdx.x * L::EPB + el;
  const bool valid = el < L::EPB && e < P.n_el;
  const long long es = valid ? e : 0;
  double* X = smem + L::TABD + 64 + el * 2 * L::KMAX * NP;
  double* Y = X + L::KMAX * NP;
  for (int c0 = 0; c0 < P.ncomp; c0 += KC) {
    const int kc = min(KC, P.ncomp - c0);
    for (int c = 0; c < KC; ++c) X[c * NP + q] = c < kc ? P.in(es, c0 + c, q) : 0.0;
    __syncthreads();
    double* s = X;
    double* d = Y;
    for (int a = D - 1; a >= 0; --a) {
      pass1d<D, N, KC, false>(&T.B[0][0], s, d, q, a, NP);
      __syncthreads();
      double* t = s; s = d; d = t;
    }
    if (valid)
      for (int c = 0; c < kc; ++c)
        P.out.p[e * P.out.estride + (c0 + c) * P.out.cstride + q] = s[c * NP + q];
    if (P.tr != nullptr && c0 == 0 && valid) {
      // trace mode: component 0's traces at the face Gauss points (lift
      // contractions of the Gauss pencils, as the warp-element kernel)
      constexpr int NQF = ipow(N, D - 1);
      for (int it = q; it < 2 * D * NQF; it += NP) {
        const int f = it / NQF, j = it - (it / NQF) * NQF;
        double t = 0.0;
        for (int p = 0; p < N; ++p)
          t = fma(T.lift[f & 1][p], s[nbr_pencil_node<D, N>(f >> 1, p, j)], t);
        P.tr[e * (2 * D * NQF) + it] = t;
      }
    }
    __syncthreads();
  }
}

// nodes -> Gauss points of KC comps staged in X (Y scratch); returns the
// buffer holding the result (d ping-pong passes, CTA-synchronised)
template <int D, int N, int KC>
__device__ __forceinline__ const double* interp_inplace(const Tab<N>& T, double* X, double* Y,
                                                        int q) {
  constexpr int NP = ipow(N, D);
  double* s = X;
  double* d = Y;
  for (int a = D - 1; a >= 0; --a) {
    pass1d<D, N, KC, false>(&T.B[0][0], s, d, q, a, NP);
    __syncthreads();
    double* t = s;
    s = d;
    d = t;
  }
  return s;
}

// per-CTA partial of sum_{k,q} w det (B a)_k (B b)_k  (dgops.py:491-503)
template <int D, int N>
__global__ void __launch_bounds__(AuxLayout<D, N>::THREADS)
inner_kernel(const __grid_constant__ AuxParams<N> P) {
  using L = AuxLayout<D, N>;
  constexpr int NP = L::NP;
  extern __shared__ double smem[];
  {
    const double* src = reinterpret_cast<const double*>(&P.tab);
    for (int i = threadIdx.x; i < L::TABD; i += blockDim.x) smem[i] = src[i];
    __syncthreads();
  }
  const Tab<N>& T = *reinterpret_cast<const Tab<N>*>(smem);
  double* red = smem + L::TABD;
  const int el = threadIdx.x / NP, q = threadIdx.x - el * NP;
  const long long e = (long long)blockIdx.x * L::EPB + el;
  const bool valid = el < L::EPB && e < P.n_el;
  const long long es = valid ? e : 0;
  double* X = smem + L::TABD + 64 + el * 2 * L::KMAX * NP;
  double* Y = X + L::KMAX * NP;
  const double wd = wdet_at<D, N>(P.elem, P.col, P.gc, es, q, T);
  double acc = 0.0;
  for (int c0 = 0; c0 < P.ncomp; c0 += L::KMAX) {
    const int kc = min(L::KMAX, P.ncomp - c0);
    double va[L::KMAX];
    // field a -> Gauss points, kept in registers
    for (int c = 0; c < L::KMAX; ++c) X[c * NP + q] = c < kc ? P.in(es, c0 + c, q) : 0.0;
    __syncthreads();
    const double* ra = interp_inplace<D, N, L::KMAX>(T, X, Y, q);
    for (int c = 0; c < L::KMAX; ++c) va[c] = ra[c * NP + q];
    __syncthreads();
    // field b -> Gauss points, products
    for (int c = 0; c < L::KMAX; ++c) X[c * NP + q] = c < kc ? P.in2(es, c0 + c, q) : 0.0;
    __syncthreads();
    const double* rb = interp_inplace<D, N, L::KMAX>(T, X, Y, q);
    for (int c = 0; c < kc; ++c) acc += va[c] * rb[c * NP + q] * wd;
    __syncthreads();
  }
  double v = valid ? acc : 0.0;
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) s += red[w];
    P.partial[blockIdx.x] = s;
  }
}

// per-CTA (max sound speed, max |u|, min rho, min p) over the volume
// quadrature points (physics.py:255-272)
template <int D, int N>
__global__ void __launch_bounds__(AuxLayout<D, N>::THREADS)
courant_kernel(const __grid_constant__ AuxParams<N> P) {
  using L = AuxLayout<D, N>;
  constexpr int NP = L::NP;
  static_assert(D + 2 <= L::KMAX, "state components");
  extern __shared__ double smem[];
  {
    const double* src = reinterpret_cast<const double*>(&P.tab);
    for (int i = threadIdx.x; i < L::TABD; i += blockDim.x) smem[i] = src[i];
    __syncthreads();
  }
  const Tab<N>& T = *reinterpret_cast<const Tab<N>*>(smem);
  double* red = smem + L::TABD;
  const int el = threadIdx.x / NP, q = threadIdx.x - el * NP;
  const long long e = (long long)blockIdx.x * L::EPB + el;
  const bool valid = el < L::EPB && e < P.n_el;
  const long long es = valid ? e : 0;
  double* X = smem + L::TABD + 64 + el * 2 * L::KMAX * NP;
  double* Y = X + L::KMAX * NP;
  for (int c = 0; c < L::KMAX; ++c) X[c * NP + q] = c < D + 2 ? P.in(es, c, q) : 0.0;
  __syncthreads();
  double* s = X;
  double* d = Y;
  for (int a = D - 1; a >= 0; --a) {
    pass1d<D, N, L::KMAX, false>(&T.B[0][0], s, d, q, a, NP);
    __syncthreads();
    double* t = s; s = d; d = t;
  }
  double cm = -INFINITY, um = -INFINITY, rmin = INFINITY, pmin = INFINITY;
  if (valid) {
    const double rho = s[q];
    double u2 = 0.0;
    for (int a = 0; a < D; ++a) {
      const double ua = s[(1 + a) * NP + q] / rho;
      u2 += ua * ua;
    }
    const double k = 0.5 * u2;
    const Model& md = P.model;
    const double p = (md.gamma - 1.0) * (s[(D + 1) * NP + q] - md.kinetic_factor * rho * k);
    cm = sqrt(md.gamma * md.inv_mach_sq * p / rho);
    um = sqrt(u2);
    rmin = rho;
    pmin = p;
  }
  for (int o = 16; o > 0; o >>= 1) {
    cm = fmax(cm, __shfl_xor_sync(0xffffffffu, cm, o));
    um = fmax(um, __shfl_xor_sync(0xffffffffu, um, o));
    rmin = fmin(rmin, __shfl_xor_sync(0xffffffffu, rmin, o));
    pmin = fmin(pmin, __shfl_xor_sync(0xffffffffu, pmin, o));
  }
  if ((threadIdx.x & 31) == 0) {
    red[(threadIdx.x >> 5) * 4 + 0] = cm;
    red[(threadIdx.x >> 5) * 4 + 1] = um;
    red[(threadIdx.x >> 5) * 4 + 2] = rmin;
    red[(threadIdx.x >> 5) * 4 + 3] = pmin;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double r[4] = {-INFINITY, -INFINITY, INFINITY, INFINITY};
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) {
      r[0] = fmax(r[0], red[w * 4 + 0]);
      r[1] = fmax(r[1], red[w * 4 + 1]);
      r[2] = fmin(r[2], red[w * 4 + 2]);
      r[3] = fmin(r[3], red[w * 4 + 3]);
    }
    for (int i = 0; i < 4; ++i) P.partial[(long long)blockIdx.x * 4 + i] = r[i];
  }
}

template <int D, int N>
cudaError_t launch_aux(int which, const AuxParams<N>& P, cudaStream_t st, int* grid_out) {
  using L = AuxLayout<D, N>;
  const int grid = (P.n_el + L::EPB - 1) / L::EPB;
  if (grid_out) *grid_out = grid;
  if (grid == 0) return cudaSuccess;
  if (which == 0) {
    cudaFuncSetAttribute(minv_kernel<D, N>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)L::SMEM);
    minv_kernel<D, N><<<grid, L::THREADS, L::SMEM, st>>>(P);
  } else if (which == 1) {
    cudaFuncSetAttribute(integrate_kernel<D, N>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)L::SMEM);
    integrate_kernel<D, N><<<grid, L::THREADS, L::SMEM, st>>>(P);
  } else if (which == 2) {
    if (P.ncomp == 1) {
      cudaFuncSetAttribute(interp_kernel<D, N, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)L::SMEM);
      interp_kernel<D, N, 1><<<grid, L::THREADS, L::SMEM, st>>>(P);
    } else {
      cudaFuncSetAttribute(interp_kernel<D, N, L::KMAX>,
                           cudaFuncAttributeMaxDynamicSharedMemorySize, (int)L::SMEM);
      interp_kernel<D, N, L::KMAX><<<grid, L::THREADS, L::SMEM, st>>>(P);
    }
  } else if (which == 3) {
    cudaFuncSetAttribute(inner_kernel<D, N>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)L::SMEM);
    inner_kernel<D, N><<<grid, L::THREADS, L::SMEM, st>>>(P);
  } else {
    cudaFuncSetAttribute(courant_kernel<D, N>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)L::SMEM);
    courant_kernel<D, N><<<grid, L::THREADS, L::SMEM, st>>>(P);
  }
  return cudaGetLastError();
}

}  // namespace dg
