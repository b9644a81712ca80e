// Element-centric, fused, sum-factorised DG operator kernel (fp64, sm_100a).
//
// One kernel launch evaluates a full weak-form operator of the reference's
// engine (orodg/dgops.py:87-230) for a block of elements per CTA, with no
// cross-element scatter and no atomics ("owner computes"):
//
//   1. stage the element's nodal input (KIN comps) in shared memory;
//   2. interpolate to Gauss points with d 1D passes of B;
//   3. volume flux, contravariant metric (rebuilt in registers from the
//      compact element/column tables, geometry.py:204-238) and the weak
//      divergence as d collocation passes of Dhat^T accumulated in Z --
//      Z holds the dual in Gauss-point coordinates, Z = B^-T dual;
//   4. every one of the element's 2d faces, axis by axis: the neighbour's
//      nodal face values are gathered (conforming neighbour, coarse parent
//      through the mortar, or the 2^(d-1) fine children of a hanging face),
//      both traces formed at the face Gauss points, the numerical flux
//      evaluated with the minus-side (conforming) / fine-side (hanging)
//      face metric exactly as the reference batches do, and the lift added
//      to Z as a rank-1 update lift[side] (x) flux*ws (coarse side: through
//      the transposed Gauss-point mortar halfq^T);
//   5. epilogue: either the dual (B^T passes) or the mass-inverted nodal
//      field B^-1 diag(1/(w detJ)) Z -- the factorised inverse of
//      geometry.py:240-251, 372-396 -- fused with the operator's affine
//      combination (explicit residual sources and sponge, Helmholtz
//      base + coef * result).
//
// Both elements of an interior face evaluate flux(minus, plus, n) with the
// same arguments and metric, so conservation holds to rounding.
#pragma once
#include "dg_common.cuh"

namespace dg {

enum OpKind { OP_ADV = 0, OP_GRAD = 1, OP_DIVHV = 2 };
enum OutMode { OUT_DUAL = 0, OUT_MINV = 1 };

template <int N>
struct KParams {
  MeshDev mesh;
  GeoConst gc;
  Model model;
  CView in;        // ADV: state; GRAD: x (scalar); DIVHV: V (d comps)
  CView inK;       // GRAD: K (optional, p = alpha (x - beta K))
  CView inH;       // DIVHV: frozen h (scalar)
  CView base;      // MINV epilogue base (optional)
  CView bg;        // ADV: sponge background (optional)
  const double* sigma;  // ADV: sponge rate (n_el, n^d) or null
  MView out;
  double alpha, beta, coef;
  int has_K, has_base, homogeneous, mode;
  double* mass_partial;  // ADV: per-CTA sum of the density dual (or null)
  Tab<N> tab;
};

template <int D, int OPK> struct OpDims;
template <int D> struct OpDims<D, OP_ADV> { static constexpr int KIN = D + 2, KOUT = D + 2; };
template <int D> struct OpDims<D, OP_GRAD> { static constexpr int KIN = 1, KOUT = D; };
template <int D> struct OpDims<D, OP_DIVHV> { static constexpr int KIN = D + 1, KOUT = 1; };

template <int D, int N, int OPK>
struct Layout {
  static constexpr int NP = ipow(N, D);
  static constexpr int NQF = ipow(N, D - 1);
  static constexpr int S = 1 << (D - 1);
  static constexpr int KIN = OpDims<D, OPK>::KIN;
  static constexpr int KOUT = OpDims<D, OPK>::KOUT;
  static constexpr int KT = KIN > KOUT ? KIN : KOUT;
  // per-element shared memory (doubles)
  static constexpr int OFF_A = 0;
  static constexpr int OFF_Q = OFF_A + KIN * NP;
  static constexpr int OFF_Z = OFF_Q + KIN * NP;
  static constexpr int OFF_T = OFF_Z + KOUT * NP;
  static constexpr int OFF_GN = OFF_T + KT * NP;
  static constexpr int OFF_FW = OFF_GN + 2 * S * KIN * NQF;
  static constexpr int ELEM = OFF_FW + 2 * S * KOUT * NQF;
  static constexpr int TABD = (int)(sizeof(Tab<N>) / sizeof(double));
  static constexpr int EPB_T = (256 / NP) > 1 ? (256 / NP) : 1;
  static constexpr int EPB_S = (12288 - TABD) / ELEM > 1 ? (12288 - TABD) / ELEM : 1;  // <= 96 KB
  static constexpr int EPB = EPB_T < EPB_S ? EPB_T : EPB_S;
  // padded to whole warps; padding threads own a scratch element slot
  static constexpr int THREADS = ((EPB * NP + 31) / 32) * 32;
  static constexpr int SLOTS = (THREADS + NP - 1) / NP;
  static constexpr size_t SMEM = (size_t)(TABD + SLOTS * ELEM + 64) * sizeof(double);
};

// index helpers -------------------------------------------------------------
template <int D, int N>
__device__ __forceinline__ int stride_of(int a) {
  int s = 1;
  for (int b = D - 1; b > a; --b) s *= N;
  return s;
}

template <int D, int N>
__device__ __forceinline__ int digit(int q, int a) {
  return (q / stride_of<D, N>(a)) % N;
}

// tangential axes of face axis a, in increasing order
template <int D>
__device__ __forceinline__ void tangential(int a, int t[2]) {
  int k = 0;
  for (int b = 0; b < D; ++b)
    if (b != a) t[k++] = b;
  if (D == 2) t[1] = -1;
}

// volume node index of face point j (C-order over tangential axes) on face (a, s)
template <int D, int N>
__device__ __forceinline__ int face_to_vol(int a, int s, int j) {
  int t[2];
  tangential<D>(a, t);
  int idx = (s ? N - 1 : 0) * stride_of<D, N>(a);
  if (D == 2) {
    idx += j * stride_of<D, N>(t[0]);
  } else {
    idx += (j / N) * stride_of<D, N>(t[0]) + (j % N) * stride_of<D, N>(t[1]);
  }
  return idx;
}

// shared-memory 1D pass: dst[c][q] = sum_j M(i_a, j) src[c][q(a->j)]
template <int D, int N, int KC, bool TRANS>
__device__ __forceinline__ void pass1d(const double* __restrict__ M, const double* src,
                                       double* dst, int q, int a, int NP) {
  const int st = stride_of<D, N>(a);
  const int ia = (q / st) % N;
  const int q0 = q - ia * st;
#pragma unroll
  for (int c = 0; c < KC; ++c) {
    double acc = 0.0;
#pragma unroll
    for (int j = 0; j < N; ++j) {
      const double m = TRANS ? M[j * N + ia] : M[ia * N + j];
      acc = fma(m, src[c * NP + q0 + j * st], acc);
    }
    dst[c * NP + q] = acc;
  }
}

// face metric (geometry.py:305-357) of the owner's (axis, oside) face at
// face Gauss point qf; returns unit normal (+axis oriented, or outward) and
// the quadrature weight times the surface Jacobian.
template <int D, int N>
__device__ __forceinline__ void face_metric(const GeoConst& gc, const double* __restrict__ col,
                                            const ElemGeo<D>& g, int axis, int oside,
                                            bool outward, int qf, const double* qw,
                                            double n[D], double& ws) {
  constexpr int HD = D - 1;
  constexpr int NQH = ipow(N, HD);
  const double zt = gc.z_top;
  double nt[D];
  double fw;
  if (axis == D - 1) {
    double dh[2] = {0.0, 0.0};
    if (gc.terrain) {
      const double* c = col + (long long)g.col * gc.col_stride;
      for (int a = 0; a < HD; ++a) dh[a] = c[NQH + a * NQH + qf];
    }
    const double decay = 1.0 - (g.lo[D - 1] + g.s[D - 1] * (double)oside) / zt;
    if (D == 2) {
      nt[0] = -dh[0] * g.s[0] * decay;
      nt[1] = g.s[0];
      fw = qw[qf];
    } else {
      nt[0] = -g.s[1] * dh[0] * g.s[0] * decay;
      nt[1] = -g.s[0] * dh[1] * g.s[1] * decay;
      nt[D - 1] = g.s[0] * g.s[1];
      fw = qw[qf / N] * qw[qf % N];
    }
  } else {
    const int qo = (D == 2) ? 0 : qf / N;
    double he = 0.0;
    if (gc.terrain) {
      const double* c = col + (long long)g.col * gc.col_stride;
      constexpr int NE = ipow(N, HD - 1);
      he = c[NQH * (1 + HD) + (axis * 2 + oside) * NE + qo];
    }
    const double zzv = g.s[D - 1] * (1.0 - he / zt);
#pragma unroll
    for (int a = 0; a < D; ++a) nt[a] = 0.0;
    if (D == 2) {
      nt[0] = zzv;
      fw = qw[qf];
    } else {
      nt[axis] = g.s[1 - axis] * zzv;
      fw = qw[qf / N] * qw[qf % N];
    }
  }
  if (outward && oside == 0) {
#pragma unroll
    for (int a = 0; a < D; ++a) nt[a] = -nt[a];
  }
  double m2 = 0.0;
#pragma unroll
  for (int a = 0; a < D; ++a) m2 += nt[a] * nt[a];
  const double mag = sqrt(m2);
#pragma unroll
  for (int a = 0; a < D; ++a) n[a] = nt[a] / mag;
  ws = fw * mag;
}

// ------------------------------------------------------------- the kernel
template <int D, int N, int OPK>
__global__ void __launch_bounds__(Layout<D, N, OPK>::THREADS)
elem_kernel(const __grid_constant__ KParams<N> P) {
  using L = Layout<D, N, OPK>;
  constexpr int NP = L::NP, NQF = L::NQF, S = L::S, KIN = L::KIN, KOUT = L::KOUT;
  constexpr int HD = D - 1;
  constexpr int NQH = ipow(N, HD);
  extern __shared__ double smem[];
  double* tb = smem;  // staged tables (Tab<N> layout)
  {
    const double* src = reinterpret_cast<const double*>(&P.tab);
    for (int i = threadIdx.x; i < L::TABD; i += blockDim.x) tb[i] = src[i];
    __syncthreads();
  }
  const Tab<N>& T = *reinterpret_cast<const Tab<N>*>(tb);
  double* red = smem + L::TABD;  // 64 doubles for block reductions
  double* base = red + 64;

  const int tid = threadIdx.x;
  const int el = tid / NP;
  const int q = tid - el * NP;
  const long long e = (long long)blockIdx.x * L::EPB + el;
  const bool valid = (el < L::EPB) && (e < P.mesh.n_el);
  const long long es = valid ? e : 0;  // safe index for idle threads
  double* A = base + el * L::ELEM + L::OFF_A;
  double* Q = base + el * L::ELEM + L::OFF_Q;
  double* Z = base + el * L::ELEM + L::OFF_Z;
  double* Tm = base + el * L::ELEM + L::OFF_T;
  double* GN = base + el * L::ELEM + L::OFF_GN;
  double* FW = base + el * L::ELEM + L::OFF_FW;
  const MeshDev& mesh = P.mesh;

  // ---- 1. nodal input ----------------------------------------------------
  auto load_in = [&](long long ee, int c, int i) -> double {
    if (OPK == OP_GRAD) {
      const double x = P.in.p ? P.in(ee, 0, i) : 0.0;
      return P.has_K ? P.alpha * (x - P.beta * P.inK(ee, 0, i)) : P.alpha * x;
    } else if (OPK == OP_DIVHV) {
      return c < D ? P.in(ee, c, i) : P.inH(ee, 0, i);
    } else {
      return P.in(ee, c, i);
    }
  };
#pragma unroll
  for (int c = 0; c < KIN; ++c) A[c * NP + q] = load_in(es, c, q);
  __syncthreads();

  // ---- 2. nodes -> Gauss points -----------------------------------------
  if (D == 2) {
    pass1d<D, N, KIN, false>(&T.B[0][0], A, Tm, q, 1, NP);
    __syncthreads();
    pass1d<D, N, KIN, false>(&T.B[0][0], Tm, Q, q, 0, NP);
  } else {
    pass1d<D, N, KIN, false>(&T.B[0][0], A, Q, q, 2, NP);
    __syncthreads();
    pass1d<D, N, KIN, false>(&T.B[0][0], Q, Tm, q, 1, NP);
    __syncthreads();
    pass1d<D, N, KIN, false>(&T.B[0][0], Tm, Q, q, 0, NP);
  }
  __syncthreads();

  // ---- 3. metric + volume flux -------------------------------------------
  const ElemGeo<D> g = elem_geo<D>(mesh.elem, P.gc, es);
  int qi[D];
#pragma unroll
  for (int a = 0; a < D; ++a) qi[a] = digit<D, N>(q, a);
  const int qh = q / N;        // horizontal Gauss index (C-order)
  const int qz = qi[D - 1];
  double hq = 0.0, dhq[2] = {0.0, 0.0};
  if (P.gc.terrain) {
    const double* c = mesh.col + (long long)g.col * P.gc.col_stride;
    hq = c[qh];
    for (int a = 0; a < HD; ++a) dhq[a] = c[NQH + a * NQH + qh];
  }
  const double zt = P.gc.z_top;
  const double zz = g.s[D - 1] * (1.0 - hq / zt);
  double det = 1.0;
#pragma unroll
  for (int a = 0; a < HD; ++a) det = det * g.s[a];
  det = det * zz;
  const double decay = 1.0 - (g.lo[D - 1] + g.s[D - 1] * T.qx[qz]) / zt;
  double ctrv[D][D];
  {
    double zg[2];
    for (int a = 0; a < HD; ++a) zg[a] = dhq[a] * g.s[a] * decay;
#pragma unroll
    for (int b = 0; b < D; ++b)
#pragma unroll
      for (int a = 0; a < D; ++a) ctrv[b][a] = 0.0;
    if (D == 2) {
      ctrv[0][0] = zz;
      ctrv[1][0] = -zg[0];
      ctrv[1][1] = g.s[0];
    } else {
      ctrv[0][0] = g.s[1] * zz;
      ctrv[1][1] = g.s[0] * zz;
      ctrv[D - 1][0] = -g.s[1] * zg[0];
      ctrv[D - 1][1] = -g.s[0] * zg[1];
      ctrv[D - 1][D - 1] = g.s[0] * g.s[1];
    }
  }
  double wq = 1.0;
#pragma unroll
  for (int a = 0; a < D; ++a) wq *= T.qw[qi[a]];

  // physical flux F[ax][k] at this Gauss point
  double F[D][KOUT];
  if (OPK == OP_ADV) {
    const double rho = Q[q];
    double u[D];
    double k = 0.0;
#pragma unroll
    for (int a = 0; a < D; ++a) {
      u[a] = Q[(1 + a) * NP + q] / rho;
      k += u[a] * u[a];
    }
    k *= 0.5;
    const double kf = P.model.kinetic_factor;
#pragma unroll
    for (int a = 0; a < D; ++a) {
      F[a][0] = Q[(1 + a) * NP + q];
#pragma unroll
      for (int b = 0; b < D; ++b) F[a][1 + b] = Q[(1 + b) * NP + q] * u[a];
      F[a][D + 1] = kf * rho * k * u[a];
    }
  } else if (OPK == OP_DIVHV) {
    const double h = Q[D * NP + q];
#pragma unroll
    for (int a = 0; a < D; ++a) F[a][0] = h * Q[a * NP + q];
  } else {  // GRAD: F[a][k] = p delta_ak
    const double p = Q[q];
#pragma unroll
    for (int a = 0; a < D; ++a)
#pragma unroll
      for (int k = 0; k < KOUT; ++k) F[a][k] = (a == k) ? p : 0.0;
  }

#pragma unroll
  for (int k = 0; k < KOUT; ++k) Z[k * NP + q] = 0.0;
  for (int bx = 0; bx < D; ++bx) {
#pragma unroll
    for (int k = 0; k < KOUT; ++k) {
      double acc = 0.0;
#pragma unroll
      for (int a = 0; a < D; ++a) acc += F[a][k] * ctrv[bx][a];
      Tm[k * NP + q] = acc * wq;
    }
    __syncthreads();
    {
      const int st = stride_of<D, N>(bx);
      const int ia = qi[bx];
      const int q0 = q - ia * st;
#pragma unroll
      for (int k = 0; k < KOUT; ++k) {
        double acc = 0.0;
#pragma unroll
        for (int j = 0; j < N; ++j) acc = fma(T.Dhat[j][ia], Tm[k * NP + q0 + j * st], acc);
        Z[k * NP + q] -= acc;
      }
    }
    __syncthreads();
  }

  // ---- 4. faces, one axis at a time ------------------------------------
  const int* nbr_e = mesh.nbr + es * (2 * D);
  const uint8_t* kind_e = mesh.kind + es * (2 * D);
  for (int axis = 0; axis < D; ++axis) {
    int tg[2];
    tangential<D>(axis, tg);
    // 4a. gather neighbour nodal face values (side, sub, comp, node)
    for (int it = q; it < 2 * S * KIN * NQF; it += NP) {
      const int j = it % NQF;
      const int c = (it / NQF) % KIN;
      const int sub = (it / (NQF * KIN)) % S;
      const int side = it / (NQF * KIN * S);
      const uint8_t kd = kind_e[2 * axis + side] & 15;
      long long src = -1;
      if (kd == KIND_CONF || kd == KIND_FINE) {
        if (sub == 0) src = nbr_e[2 * axis + side];
      } else if (kd == KIND_COARSE) {
        src = mesh.hang_children[(long long)nbr_e[2 * axis + side] * S + sub];
      }
      if (valid && src >= 0)
        GN[it] = load_in(src, c, face_to_vol<D, N>(axis, 1 - side, j));
    }
    __syncthreads();
    // 4b. traces + numerical flux at (side, sub, qf)
    for (int it = q; it < 2 * S * NQF; it += NP) {
      const int qf = it % NQF;
      const int sub = (it / NQF) % S;
      const int side = it / (NQF * S);
      const uint8_t kraw = kind_e[2 * axis + side];
      const uint8_t kd = kraw & 15;
      if (!valid || (sub > 0 && kd != KIND_COARSE)) continue;
      const int qt0 = (D == 2) ? qf : qf / N;
      const int qt1 = (D == 2) ? 0 : qf % N;
      double TO[KIN], TN[KIN];
      // own trace
      if (kd == KIND_COARSE) {
        const int b0 = sub & 1, b1 = (sub >> 1) & 1;
#pragma unroll
        for (int c = 0; c < KIN; ++c) {
          double acc = 0.0;
          for (int j = 0; j < NQF; ++j) {
            const int j0 = (D == 2) ? j : j / N;
            const int j1 = (D == 2) ? 0 : j % N;
            double m = T.half[b0][qt0][j0];
            if (D == 3) m *= T.half[b1][qt1][j1];
            acc = fma(m, A[c * NP + face_to_vol<D, N>(axis, side, j)], acc);
          }
          TO[c] = acc;
        }
      } else {
        int qv = 0;
        if (D == 2) qv = qt0 * stride_of<D, N>(tg[0]);
        else qv = qt0 * stride_of<D, N>(tg[0]) + qt1 * stride_of<D, N>(tg[1]);
        const int sa = stride_of<D, N>(axis);
#pragma unroll
        for (int c = 0; c < KIN; ++c) {
          double acc = 0.0;
#pragma unroll
          for (int p = 0; p < N; ++p) acc = fma(T.lift[side][p], Q[c * NP + qv + p * sa], acc);
          TO[c] = acc;
        }
      }
      // neighbour trace / ghost, and the face-metric owner
      ElemGeo<D> og = g;
      int oside = side;
      bool outward = false;
      const double* gnb = GN + (side * S + sub) * KIN * NQF;
      if (kd == KIND_CONF || kd == KIND_COARSE || kd == KIND_FINE) {
        const bool mort = (kd == KIND_FINE);
        const int sf = (kraw >> 4) & 3;
        const int b0 = sf & 1, b1 = (sf >> 1) & 1;
#pragma unroll
        for (int c = 0; c < KIN; ++c) {
          double acc = 0.0;
          for (int j = 0; j < NQF; ++j) {
            const int j0 = (D == 2) ? j : j / N;
            const int j1 = (D == 2) ? 0 : j % N;
            double m = mort ? T.half[b0][qt0][j0] : T.B[qt0][j0];
            if (D == 3) m *= mort ? T.half[b1][qt1][j1] : T.B[qt1][j1];
            acc = fma(m, gnb[c * NQF + j], acc);
          }
          TN[c] = acc;
        }
        if (kd == KIND_CONF && side == 0) {
          og = elem_geo<D>(mesh.elem, P.gc, nbr_e[2 * axis + side]);
          oside = 1;
        } else if (kd == KIND_COARSE) {
          og = elem_geo<D>(mesh.elem, P.gc,
                           mesh.hang_children[(long long)nbr_e[2 * axis + side] * S + sub]);
          oside = 1 - side;
        }
      } else {
        outward = true;
      }
      double n[D], ws;
      face_metric<D, N>(P.gc, mesh.col, og, axis, oside, outward, qf, T.qw, n, ws);
      if (outward) {
        const long long row = nbr_e[2 * axis + side];
        if (OPK == OP_ADV) {
          if (kd == KIND_WALL) {
            double mn = 0.0;
#pragma unroll
            for (int a = 0; a < D; ++a) mn += TO[1 + a] * n[a];
#pragma unroll
            for (int c = 0; c < KIN; ++c) TN[c] = TO[c];
#pragma unroll
            for (int a = 0; a < D; ++a) TN[1 + a] = TO[1 + a] - 2.0 * mn * n[a];
          } else {
#pragma unroll
            for (int c = 0; c < KIN; ++c) TN[c] = mesh.ff_U[(row * KIN + c) * NQF + qf];
          }
        } else if (OPK == OP_GRAD) {
          TN[0] = (kd == KIND_WALL) ? TO[0] : (P.homogeneous ? 0.0 : mesh.ff_p[row * NQF + qf]);
        } else {
          if (kd == KIND_WALL) {
            double vn = 0.0;
#pragma unroll
            for (int a = 0; a < D; ++a) vn += TO[a] * n[a];
#pragma unroll
            for (int a = 0; a < D; ++a) TN[a] = TO[a] - 2.0 * vn * n[a];
            TN[D] = TO[D];
          } else {
#pragma unroll
            for (int a = 0; a < D; ++a)
              TN[a] = P.homogeneous ? 0.0 : mesh.ff_U[(row * (D + 2) + 1 + a) * NQF + qf];
            TN[D] = mesh.ff_h[row * NQF + qf];
          }
        }
      }
      // numerical flux: flux(minus, plus, n); minus side gets +lift
      const bool minus = outward || side == 1;
      const double* TLp = minus ? TO : TN;
      const double* TRp = minus ? TN : TO;
      double fl[KOUT];
      if (OPK == OP_ADV) {
        double mnL = 0.0, mnR = 0.0;
#pragma unroll
        for (int a = 0; a < D; ++a) {
          mnL += TLp[1 + a] * n[a];
          mnR += TRp[1 + a] * n[a];
        }
        const double rL = TLp[0], rR = TRp[0];
        const double uL = mnL / rL, uR = mnR / rR;
        const double lam = fmax(fabs(uL), fabs(uR));
        double kL = 0.0, kR = 0.0;
#pragma unroll
        for (int a = 0; a < D; ++a) {
          const double vl = TLp[1 + a] / rL, vr = TRp[1 + a] / rR;
          kL += vl * vl;
          kR += vr * vr;
        }
        fl[0] = 0.5 * (mnL + mnR);
#pragma unroll
        for (int a = 0; a < D; ++a) fl[1 + a] = 0.5 * (TLp[1 + a] * uL + TRp[1 + a] * uR);
        fl[D + 1] = 0.25 * P.model.kinetic_factor * (rL * kL * uL + rR * kR * uR);
#pragma unroll
        for (int c = 0; c < KOUT; ++c) fl[c] -= 0.5 * lam * (TRp[c] - TLp[c]);
      } else if (OPK == OP_GRAD) {
        const double ph = 0.5 * (TLp[0] + TRp[0]);
#pragma unroll
        for (int a = 0; a < D; ++a) fl[a] = ph * n[a];
      } else {
        double vL = 0.0, vR = 0.0;
#pragma unroll
        for (int a = 0; a < D; ++a) {
          vL += TLp[a] * n[a];
          vR += TRp[a] * n[a];
        }
        fl[0] = 0.5 * (TLp[D] * vL + TRp[D] * vR);
      }
      const double sg = minus ? ws : -ws;
      double* fw = FW + (side * S + sub) * KOUT * NQF;
#pragma unroll
      for (int c = 0; c < KOUT; ++c) fw[c * NQF + qf] = fl[c] * sg;
    }
    __syncthreads();
    // 4c. lift into Z: Z[k][q] += lift[side][q_axis] * L_side[k](q_t)
    if (valid) {
      const int ia = qi[axis];
      const int qt0 = qi[tg[0]];
      const int qt1 = (D == 3) ? qi[tg[1]] : 0;
      const int qf = (D == 2) ? qt0 : qt0 * N + qt1;
      for (int side = 0; side < 2; ++side) {
        const uint8_t kd = kind_e[2 * axis + side] & 15;
        const double lw = T.lift[side][ia];
        if (kd == KIND_COARSE) {
#pragma unroll
          for (int k = 0; k < KOUT; ++k) {
            double acc = 0.0;
            for (int sub = 0; sub < S; ++sub) {
              const int b0 = sub & 1, b1 = (sub >> 1) & 1;
              const double* fw = FW + (side * S + sub) * KOUT * NQF + k * NQF;
              for (int j = 0; j < NQF; ++j) {
                const int j0 = (D == 2) ? j : j / N;
                const int j1 = (D == 2) ? 0 : j % N;
                double m = T.halfq[b0][j0][qt0];
                if (D == 3) m *= T.halfq[b1][j1][qt1];
                acc = fma(m, fw[j], acc);
              }
            }
            Z[k * NP + q] += lw * acc;
          }
        } else {
          const double* fw = FW + side * S * KOUT * NQF;
#pragma unroll
          for (int k = 0; k < KOUT; ++k) Z[k * NP + q] += lw * fw[k * NQF + qf];
        }
      }
    }
    __syncthreads();
  }

  // ---- 5. epilogue ---------------------------------------------------------
  if (OPK == OP_ADV && P.mass_partial != nullptr) {
    // sum of the density dual = sum_q Z[0][q] (rows of B sum to one)
    double v = valid ? Z[q] : 0.0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if ((tid & 31) == 0) red[tid >> 5] = v;
    __syncthreads();
    if (tid == 0) {
      double s = 0.0;
      for (int w = 0; w < (int)((blockDim.x + 31) >> 5); ++w) s += red[w];
      P.mass_partial[blockIdx.x] = s;
    }
  }
  double* res;
  if (P.mode == OUT_MINV) {
    const double inv = 1.0 / (wq * det);
#pragma unroll
    for (int k = 0; k < KOUT; ++k) Z[k * NP + q] *= inv;
    __syncthreads();
    if (D == 2) {
      pass1d<D, N, KOUT, false>(&T.Binv[0][0], Z, Tm, q, 1, NP);
      __syncthreads();
      pass1d<D, N, KOUT, false>(&T.Binv[0][0], Tm, Z, q, 0, NP);
      res = Z;
    } else {
      pass1d<D, N, KOUT, false>(&T.Binv[0][0], Z, Tm, q, 2, NP);
      __syncthreads();
      pass1d<D, N, KOUT, false>(&T.Binv[0][0], Tm, Z, q, 1, NP);
      __syncthreads();
      pass1d<D, N, KOUT, false>(&T.Binv[0][0], Z, Tm, q, 0, NP);
      res = Tm;
    }
  } else {
    if (D == 2) {
      pass1d<D, N, KOUT, true>(&T.B[0][0], Z, Tm, q, 1, NP);
      __syncthreads();
      pass1d<D, N, KOUT, true>(&T.B[0][0], Tm, Z, q, 0, NP);
      res = Z;
    } else {
      pass1d<D, N, KOUT, true>(&T.B[0][0], Z, Tm, q, 2, NP);
      __syncthreads();
      pass1d<D, N, KOUT, true>(&T.B[0][0], Tm, Z, q, 1, NP);
      __syncthreads();
      pass1d<D, N, KOUT, true>(&T.B[0][0], Z, Tm, q, 0, NP);
      res = Tm;
    }
  }
  __syncthreads();
  if (!valid) return;
  double* out = P.out.p + e * P.out.estride + q;
  if (P.mode == OUT_DUAL) {
#pragma unroll
    for (int k = 0; k < KOUT; ++k) out[k * P.out.cstride] = res[k * NP + q];
    return;
  }
  if (OPK == OP_ADV) {
    // R = -Minv dual + gravity source - sigma (U - U_bg)   (imex.py:144-159)
    const double rho = A[q];
    const Model& md = P.model;
    double R[KOUT];
#pragma unroll
    for (int k = 0; k < KOUT; ++k) R[k] = -res[k * NP + q];
    R[D] += -md.gravity * rho;
    R[D + 1] += -md.kinetic_factor * md.gravity * rho * (A[D * NP + q] / rho);
    if (P.sigma != nullptr) {
      const double sg = P.sigma[e * NP + q];
#pragma unroll
      for (int k = 1; k < KOUT; ++k) R[k] -= sg * (A[k * NP + q] - P.bg(e, k, q));
    }
#pragma unroll
    for (int k = 0; k < KOUT; ++k) out[k * P.out.cstride] = R[k];
  } else {
#pragma unroll
    for (int k = 0; k < KOUT; ++k) {
      // unfused like the reference's numpy: base + (coef * result)
      const double r = __dmul_rn(P.coef, res[k * NP + q]);
      out[k * P.out.cstride] = P.has_base ? __dadd_rn(P.base(e, k, q), r) : r;
    }
  }
}

}  // namespace dg
