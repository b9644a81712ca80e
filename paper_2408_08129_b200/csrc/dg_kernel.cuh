// Fused element-centric DG operator kernel, v2 (fp64, sm_100a).
//
// Evaluates one weak-form operator of the reference engine
// (orodg/dgops.py:87-230) for EPB elements per CTA, owner-computes, no
// atomics, and fuses the factorised mass inverse (geometry.py:240-251,
// 372-396) and the operator's affine epilogue:
//
//   1. nodal input -> shared memory (KIN comps per element);
//   2. nodes -> Gauss points: d pencil passes of B;
//   3. volume: flux + contravariant metric (rebuilt in registers from the
//      compact element/column tables, geometry.py:204-238) per point, then
//      per reference direction bx one pencil pass of Dhat^T along bx,
//      accumulated in Z = B^-T dual (Gauss-point coordinates);
//   4. faces, all 2d at once: neighbour nodal face values gathered,
//      tangential pencil passes (B, or the mortar halves for a fine leaf
//      seeing its coarse parent), own trace = lift[side] . Gauss column,
//      numerical flux with the minus-side (conforming) / fine-side (hanging)
//      face metric exactly as the reference batches, then the rank-1 lift
//      Z += lift[side] (x) flux*ws;
//      the coarse side of hanging faces (2^(d-1) subfaces) is added by the
//      small coarse_kernel over the compact list of coarse elements;
//   5. epilogue: dual = B^T (x) Z, or nodal = B^-1 (x) diag(1/(w detJ)) Z
//      fused with base + coef * nodal (explicit: sources and sponge).
//
// Pencil passes take the 1D matrices straight from the kernel-parameter
// constant bank with compile-time indices (DFMA with a constant operand:
// no shared-memory traffic for the matrices); every axis is a template
// parameter so all index arithmetic folds at compile time.
#pragma once
#include "dg_operator.cuh"

namespace dg {

template <int D, int N, int OPK>
struct Layout {
  static constexpr int NP = ipow(N, D);
  static constexpr int NQF = ipow(N, D - 1);
  static constexpr int NF = 2 * D;
  static constexpr int S = 1 << (D - 1);
  static constexpr int KIN = OpDims<D, OPK>::KIN;
  static constexpr int KOUT = OpDims<D, OPK>::KOUT;
  static constexpr int KT = KIN > KOUT ? KIN : KOUT;
  static constexpr int OFF_A = 0;
  static constexpr int OFF_Q = OFF_A + KIN * NP;
  static constexpr int OFF_Z = OFF_Q + KIN * NP;
  static constexpr int OFF_T = OFF_Z + KOUT * NP;
  static constexpr int OFF_G = OFF_T + KT * NP;
  static constexpr int OFF_H = OFF_G + NF * KIN * NQF;
  static constexpr int OFF_L = OFF_H + NF * KIN * NQF;
  static constexpr int KW = (OPK == OP_GRAD) ? 1 : KOUT;  // comps per direction bx < d-1
  static constexpr int OFF_W = OFF_L + NF * KOUT * NQF;
  static constexpr int ELEM = OFF_W + (D - 1) * KW * NP;
  static constexpr int TABD = (int)(sizeof(Tab<N>) / sizeof(double));
  static constexpr int EPB_T = (128 / NP) > 1 ? (128 / NP) : 1;
  static constexpr int EPB_S = (12288 - TABD - 64) / ELEM > 1 ? (12288 - TABD - 64) / ELEM : 1;
  static constexpr int EPB = EPB_T < EPB_S ? EPB_T : EPB_S;
  static constexpr int THREADS = ((EPB * NP + 31) / 32) * 32;
  static constexpr int SLOTS = EPB;  // padding threads shadow slot 0 (elem_kernel)
  static constexpr size_t SMEM = (size_t)(TABD + 64 + SLOTS * ELEM) * sizeof(double);
  static constexpr int REGCAP = (OPK == OP_ADV) ? 128 : 96;
  static constexpr int MINB0 = 65536 / (THREADS * REGCAP);
  static constexpr int MINB = MINB0 < 1 ? 1 : (MINB0 > 8 ? 8 : MINB0);
  // coarse fix-up kernel (one CTA per coarse element)
  static constexpr int CTHREADS = ((NP + 31) / 32) * 32;
  static constexpr int C_A = 0;
  static constexpr int C_FW = C_A + KIN * NP;
  static constexpr int C_Z = C_FW + S * KOUT * NQF;  // one coarse face at a time
  static constexpr int C_T = C_Z + KOUT * NP;
  static constexpr int C_CH = C_T + KOUT * NP;  // children's nodal face values (one face)
  static constexpr int C_GS = C_CH + S * KIN * NQF;  // fused-dot warp sums
  static constexpr int C_OT = C_GS + CTHREADS;       // trace mode: own face traces (one face)
  // flux mode, 3D: the separable mortar passes' partials
  static constexpr int C_SC = C_OT + KIN * NQF;
  static constexpr int SC_A = KIN * 2 * N * N + S * KIN * N * N;
  static constexpr int SC_C = S * KOUT * N * N;
  static constexpr int CELEM = C_SC + (SC_A > SC_C ? SC_A : SC_C);
  static constexpr size_t CSMEM = (size_t)(TABD + 64 + CELEM) * sizeof(double);
};

// ---------------------------------------------------------------- passes
// dst (op)= M along axis AX of a DIM-dim N^DIM tensor, for KC comps of nv
// elements.  M from the parameter constant bank (compile-time indices).
// MODE: 0 dst = M src, 1 dst = -M src, 2 dst -= M src.
// Runs over all EPB element slots of the CTA (compile-time trip count; slots
// past the last valid element compute on their own scratch and are never
// stored to global memory).
template <int DIM, int N, int AX, bool TRANS, int MODE, int KC, int ELEM, int CS, int NE, int TH>
__device__ __forceinline__ void vpass(const double (&M)[N][N], double* base, int soff, int doff) {
  constexpr int NPEN = ipow(N, DIM - 1);
  constexpr int ST = ipow(N, DIM - 1 - AX);
  constexpr int ITEMS = NE * KC * NPEN;
#pragma unroll
  for (int rr = 0; rr < (ITEMS + TH - 1) / TH; ++rr) {
    const int it = rr * TH + (int)threadIdx.x;
    if ((ITEMS % TH) != 0 && it >= ITEMS) break;
    const int p = it % NPEN;
    const int r = it / NPEN;
    const int c = r % KC;
    const int e = r / KC;
    const int b = (p / ST) * (ST * N) + (p % ST);
    const double* s = base + e * ELEM + soff + c * CS + b;
    double* d = base + e * ELEM + doff + c * CS + b;
    double v[N];
#pragma unroll
    for (int j = 0; j < N; ++j) v[j] = s[j * ST];
#pragma unroll
    for (int i = 0; i < N; ++i) {
      double acc = 0.0;
#pragma unroll
      for (int j = 0; j < N; ++j) acc = fma(TRANS ? M[j][i] : M[i][j], v[j], acc);
      if (MODE == 0) d[i * ST] = acc;
      else if (MODE == 1) d[i * ST] = -acc;
      else d[i * ST] -= acc;
    }
  }
}

// nodes -> Gauss points (all axes), src (A) preserved; result at Q
template <int D, int N, int KC, int ELEM, int NP, int NE, int TH>
__device__ __forceinline__ void interp_all(const double (&B)[N][N], double* base, int a_off,
                                           int q_off, int t_off) {
  if constexpr (D == 2) {
    vpass<2, N, 1, false, 0, KC, ELEM, NP, NE, TH>(B, base, a_off, t_off);
    __syncthreads();
    vpass<2, N, 0, false, 0, KC, ELEM, NP, NE, TH>(B, base, t_off, q_off);
  } else {
    vpass<3, N, 2, false, 0, KC, ELEM, NP, NE, TH>(B, base, a_off, q_off);
    __syncthreads();
    vpass<3, N, 1, false, 0, KC, ELEM, NP, NE, TH>(B, base, q_off, t_off);
    __syncthreads();
    vpass<3, N, 0, false, 0, KC, ELEM, NP, NE, TH>(B, base, t_off, q_off);
  }
}

// tangential pass on the gathered face tensors: matrix per face from the
// smem tables (B, or half[bit] for a fine leaf's view of its coarse parent)
template <int D, int N, int TAX, int KC, int ELEM, int NF, int NE, int TH>
__device__ __forceinline__ void fpass(const Tab<N>& TS, const uint8_t* __restrict__ kind,
                                      long long e0, double* base, int soff, int doff, int nv) {
  constexpr int NQF = ipow(N, D - 1);
  constexpr int NPEN = NQF / N;
  constexpr int ST = ipow(N, D - 2 - TAX);
  constexpr int ITEMS = NE * NF * KC * NPEN;
#pragma unroll
  for (int rr = 0; rr < (ITEMS + TH - 1) / TH; ++rr) {
    const int it = rr * TH + (int)threadIdx.x;
    if ((ITEMS % TH) != 0 && it >= ITEMS) break;
    const int p = it % NPEN;
    int r = it / NPEN;
    const int c = r % KC;
    r /= KC;
    const int f = r % NF;
    const int e = r / NF;
    if (e >= nv) continue;
    const uint8_t kraw = kind[(e0 + e) * NF + f];
    const int kd = kraw & 15;
    if (kd != KIND_CONF && kd != KIND_FINE) continue;
    const double* M = (kd == KIND_FINE) ? &TS.half[((kraw >> 4) >> TAX) & 1][0][0] : &TS.B[0][0];
    const int b = (p / ST) * (ST * N) + (p % ST);
    const double* s = base + e * ELEM + soff + (f * KC + c) * NQF + b;
    double* d = base + e * ELEM + doff + (f * KC + c) * NQF + b;
    double v[N];
#pragma unroll
    for (int j = 0; j < N; ++j) v[j] = s[j * ST];
#pragma unroll
    for (int i = 0; i < N; ++i) {
      double acc = 0.0;
#pragma unroll
      for (int j = 0; j < N; ++j) acc = fma(M[i * N + j], v[j], acc);
      d[i * ST] = acc;
    }
  }
}

// Face metric of the owner's (AX, oside) face at face Gauss point qf, the
// geometry.py:305-357 formulas specialised per axis: vertical faces have an
// exact +-e_AX normal (the reference's ntilde/|ntilde| is exactly that), as
// do horizontal faces without terrain, so only terrain z-faces pay the
// sqrt and division.
template <int D, int N, int AX>
__device__ __forceinline__ void face_metric_ax(const GeoConst& gc, const double* __restrict__ col,
                                               const ElemGeo<D>& g, int oside, bool outward,
                                               int qf, const Tab<N>& T, double n[D],
                                               double& ws) {
  constexpr int HD = D - 1;
  constexpr int NQH = ipow(N, HD);
  const double fw = (D == 2) ? T.qw[qf] : T.qw[qf / N] * T.qw[qf % N];
  const double sgn = (outward && oside == 0) ? -1.0 : 1.0;
#pragma unroll
  for (int a = 0; a < D; ++a) n[a] = 0.0;
  if constexpr (AX < D - 1) {
    const int qo = (D == 2) ? 0 : qf / N;
    double omh = 1.0;  // 1 - h_edge/z_top from the column table
    if (gc.terrain) {
      constexpr int NE = ipow(N, HD - 1);
      omh = col[(long long)g.col * gc.col_stride + NQH * (1 + HD) + (AX * 2 + oside) * NE + qo];
    }
    const double zzv = g.s[D - 1] * omh;
    const double mag = (D == 2) ? zzv : g.s[1 - AX] * zzv;
    n[AX] = sgn;
    ws = fw * fabs(mag);
  } else {
    const double top = (D == 2) ? g.s[0] : g.s[0] * g.s[1];
    if (!gc.terrain) {
      n[D - 1] = sgn;
      ws = fw * top;
      return;
    }
    const double* c = col + (long long)g.col * gc.col_stride;
    const double decay = 1.0 - (g.lo[D - 1] + g.s[D - 1] * (double)oside) / gc.z_top;
    double nt[D];
    if constexpr (D == 2) {
      nt[0] = -c[NQH + qf] * g.s[0] * decay;
    } else {
      nt[0] = -g.s[1] * c[NQH + qf] * g.s[0] * decay;
      nt[1] = -g.s[0] * c[2 * NQH + qf] * g.s[1] * decay;
    }
    nt[D - 1] = top;
    double m2 = 0.0;
#pragma unroll
    for (int a = 0; a < D; ++a) m2 += nt[a] * nt[a];
    const double mag = sqrt(m2);
#pragma unroll
    for (int a = 0; a < D; ++a) n[a] = sgn * (nt[a] / mag);
    ws = fw * mag;
  }
}

// -------------------------------------------------------------- physics
// full Euler flux tensor of one state, F[v][a] (physics.py:149-187: the
// primitive variables and inviscid_flux, same operation order)
template <int D>
__device__ __forceinline__ void full_flux(const double* U, const Model& md, double F[][D],
                                          double* un_speed = nullptr, const double* n = nullptr) {
  const double rho = U[0];
  double u[D];
  double k = 0.0;
#pragma unroll
  for (int a = 0; a < D; ++a) {
    u[a] = U[1 + a] / rho;
    k += u[a] * u[a];
  }
  k = 0.5 * k;
  const double gm1 = md.gamma - 1.0;
  const double p = gm1 * (U[D + 1] - md.kinetic_factor * rho * k);
  const double e = p / (gm1 * rho);
  double ru[D];
#pragma unroll
  for (int a = 0; a < D; ++a) ru[a] = rho * u[a];
#pragma unroll
  for (int a = 0; a < D; ++a) F[0][a] = ru[a];
#pragma unroll
  for (int b = 0; b < D; ++b) {
#pragma unroll
    for (int a = 0; a < D; ++a) F[1 + b][a] = ru[b] * u[a];
    F[1 + b][b] += md.inv_mach_sq * p;
  }
  const double enth = rho * e + md.kinetic_factor * rho * k + p;
#pragma unroll
  for (int a = 0; a < D; ++a) F[D + 1][a] = enth * u[a];
  if (un_speed) {
    // |u . n| + c, c = sqrt(gamma / M^2 p / rho) (physics.py:127-129)
    double un = 0.0;
#pragma unroll
    for (int a = 0; a < D; ++a) un += u[a] * n[a];
    *un_speed = fabs(un) + sqrt(md.gamma * md.inv_mach_sq * p / rho);
  }
}

template <int D, int OPK, int KIN, int KOUT>
__device__ __forceinline__ void num_flux(const double* TL, const double* TR, const double* n,
                                         double kf, double* fl, const Model* md = nullptr,
                                         int full = 0) {
  if constexpr (OPK == OP_ADV) {
    if (full) {
      // divergence_full (dgops.py:298-328): centred full flux, Rusanov with
      // lambda = max(|u.n| + c) when full == 1
      double FL[D + 2][D], FR[D + 2][D], sL, sR;
      full_flux<D>(TL, *md, FL, &sL, n);
      full_flux<D>(TR, *md, FR, &sR, n);
      const double lam = fmax(sL, sR);
#pragma unroll
      for (int c = 0; c < KOUT; ++c) {
        double s = 0.0;
#pragma unroll
        for (int a = 0; a < D; ++a) s += (FL[c][a] + FR[c][a]) * n[a];
        fl[c] = 0.5 * s;
        if (full == 1) fl[c] -= 0.5 * lam * (TR[c] - TL[c]);
      }
      return;
    }
    // Rusanov with the flow speed only (orodg/dgops.py:256-283)
    double mnL = 0.0, mnR = 0.0;
#pragma unroll
    for (int a = 0; a < D; ++a) {
      mnL += TL[1 + a] * n[a];
      mnR += TR[1 + a] * n[a];
    }
    const double rL = TL[0], rR = TR[0];
#ifndef DG_ADV_RCP
#define DG_ADV_RCP 1
#endif
    // DG_ADV_RCP: one reciprocal per side instead of d + 1 divisions (a
    // rounding-level change, inside the reference's own 1-ulp sensitivity)
    const double irL = DG_ADV_RCP ? __drcp_rn(rL) : 0.0, irR = DG_ADV_RCP ? __drcp_rn(rR) : 0.0;
    const double uL = DG_ADV_RCP ? mnL * irL : mnL / rL, uR = DG_ADV_RCP ? mnR * irR : mnR / rR;
    const double lam = fmax(fabs(uL), fabs(uR));
    double kL = 0.0, kR = 0.0;
#pragma unroll
    for (int a = 0; a < D; ++a) {
      const double vl = DG_ADV_RCP ? TL[1 + a] * irL : TL[1 + a] / rL;
      const double vr = DG_ADV_RCP ? TR[1 + a] * irR : TR[1 + a] / rR;
      kL += vl * vl;
      kR += vr * vr;
    }
    fl[0] = 0.5 * (mnL + mnR);
#pragma unroll
    for (int a = 0; a < D; ++a) fl[1 + a] = 0.5 * (TL[1 + a] * uL + TR[1 + a] * uR);
    fl[D + 1] = 0.25 * kf * (rL * kL * uL + rR * kR * uR);
#pragma unroll
    for (int c = 0; c < KOUT; ++c) fl[c] -= 0.5 * lam * (TR[c] - TL[c]);
  } else if constexpr (OPK == OP_GRAD) {
    // centred pressure (dgops.py:343-348)
    const double ph = 0.5 * (TL[0] + TR[0]);
#pragma unroll
    for (int a = 0; a < D; ++a) fl[a] = ph * n[a];
  } else {
    // average of products (dgops.py:452-460)
    double vL = 0.0, vR = 0.0;
#pragma unroll
    for (int a = 0; a < D; ++a) {
      vL += TL[a] * n[a];
      vR += TR[a] * n[a];
    }
    fl[0] = 0.5 * (TL[D] * vL + TR[D] * vR);
  }
}

// boundary ghost state (boundary.py:17-84, dgops.py:462-474)
template <int D, int N, int OPK, int KIN>
__device__ __forceinline__ void ghost(const KParams<N>& P, int kd, long long row, int qf,
                                      const double* TO, const double* n, double* TN) {
  constexpr int NQF = ipow(N, D - 1);
  const MeshDev& mesh = P.mesh;
  if constexpr (OPK == OP_ADV) {
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
  } else if constexpr (OPK == OP_GRAD) {
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

template <int D, int N, int OPK>
__device__ __forceinline__ double load_input(const KParams<N>& P, long long ee, int c, int i) {
  if constexpr (OPK == OP_GRAD) {
    const double x = P.in.p ? P.in(ee, 0, i) : 0.0;
    return P.has_K ? P.alpha * (x - P.beta * P.inK(ee, 0, i)) : P.alpha * x;
  } else if constexpr (OPK == OP_DIVHV) {
    return c < D ? P.in(ee, c, i) : P.inH(ee, 0, i);
  } else {
    return P.in(ee, c, i);
  }
}

// Gauss-point metric: det J (z-independent) and the adjugate rows
template <int D, int N>
__device__ __forceinline__ void point_metric(const KParams<N>& P, const ElemGeo<D>& g, int q,
                                             double& det, double ctrv[D][D]) {
  constexpr int HD = D - 1;
  constexpr int NQH = ipow(N, HD);
  const int qh = q / N;
  const int qz = q % N;
#pragma unroll
  for (int b = 0; b < D; ++b)
#pragma unroll
    for (int a = 0; a < D; ++a) ctrv[b][a] = 0.0;
  if (!P.gc.terrain) {
    // flat: zz = s_z exactly, diagonal adjugate (geometry.py:204-231 with h = 0)
    if constexpr (D == 2) {
      det = g.s[0] * g.s[1];
      ctrv[0][0] = g.s[1];
      ctrv[1][1] = g.s[0];
    } else {
      det = g.s[0] * g.s[1] * g.s[2];
      ctrv[0][0] = g.s[1] * g.s[2];
      ctrv[1][1] = g.s[0] * g.s[2];
      ctrv[2][2] = g.s[0] * g.s[1];
    }
    return;
  }
  double omh, dhq[2] = {0.0, 0.0};
  {
    const double* c = P.mesh.col + (long long)g.col * P.gc.col_stride;
    omh = c[qh];  // 1 - h/z_top
#pragma unroll
    for (int a = 0; a < HD; ++a) dhq[a] = c[NQH + a * NQH + qh];
  }
  const double zt = P.gc.z_top;
  const double zz = g.s[D - 1] * omh;
  det = 1.0;
#pragma unroll
  for (int a = 0; a < HD; ++a) det = det * g.s[a];
  det = det * zz;
  const double decay = 1.0 - (g.lo[D - 1] + g.s[D - 1] * P.tab.qx[qz]) / zt;
  double zg[2];
#pragma unroll
  for (int a = 0; a < HD; ++a) zg[a] = dhq[a] * g.s[a] * decay;
#pragma unroll
  for (int b = 0; b < D; ++b)
#pragma unroll
    for (int a = 0; a < D; ++a) ctrv[b][a] = 0.0;
  if constexpr (D == 2) {
    ctrv[0][0] = zz;
    ctrv[1][0] = -zg[0];
    ctrv[1][1] = g.s[0];
  } else {
    ctrv[0][0] = g.s[1] * zz;
    ctrv[1][1] = g.s[0] * zz;
    ctrv[2][0] = -g.s[1] * zg[0];
    ctrv[2][1] = -g.s[0] * zg[1];
    ctrv[2][2] = g.s[0] * g.s[1];
  }
}

template <int D, int N>
__device__ __forceinline__ double point_weight(const Tab<N>& T, int q) {
  double w = 1.0;
#pragma unroll
  for (int a = 0; a < D; ++a) w *= T.qw[digit<D, N>(q, a)];
  return w;
}

// --------------------------------------------------------- face flux phase
// items (e, side, qf) of axis AX; writes L[f][k][qf] = +-flux*ws (0 for coarse)
template <int D, int N, int OPK, int AX>
__device__ __forceinline__ void face_flux_axis(const KParams<N>& P, const Tab<N>& TS, double* base,
                                               long long e0, int nv, int nb_off) {
  using L = Layout<D, N, OPK>;
  constexpr int NQF = L::NQF, NF = L::NF, KIN = L::KIN, KOUT = L::KOUT, NP = L::NP;
  constexpr int T0 = (AX == 0) ? 1 : 0;
  constexpr int T1 = (D == 3) ? ((AX == 2) ? 1 : 2) : -1;
  constexpr int SA = ipow(N, D - 1 - AX);
  constexpr int S0 = ipow(N, D - 1 - T0);
  constexpr int S1 = (D == 3) ? ipow(N, D - 1 - (T1 < 0 ? 0 : T1)) : 0;
  const MeshDev& mesh = P.mesh;
  const int items = nv * 2 * NQF;
  for (int it = threadIdx.x; it < items; it += blockDim.x) {
    const int qf = it % NQF;
    const int side = (it / NQF) & 1;
    const int e = it / (2 * NQF);
    const int f = 2 * AX + side;
    const long long ge = e0 + e;
    const uint8_t kraw = mesh.kind[ge * NF + f];
    const int kd = kraw & 15;
    double* Lf = base + e * L::ELEM + L::OFF_L + f * KOUT * NQF;
    if (kd == KIND_COARSE) {
      // precomputed coarse-face flux (flux mode), else added by coarse_kernel
      const double* cf = mesh.cflux;
      const long long grp = mesh.nbr[ge * NF + f];
#pragma unroll
      for (int k = 0; k < KOUT; ++k)
        Lf[k * NQF + qf] = cf ? cf[(grp * KOUT + k) * NQF + qf] : 0.0;
      continue;
    }
    // own trace: nodal value at the face = lift[side] . Gauss column
    const int qt0 = (D == 2) ? qf : qf / N;
    const int qt1 = (D == 2) ? 0 : qf % N;
    const int qv = qt0 * S0 + qt1 * S1;
    const double* Qe = base + e * L::ELEM + L::OFF_Q;
    double TO[KIN], TN[KIN];
#pragma unroll
    for (int c = 0; c < KIN; ++c) {
      double acc = 0.0;
#pragma unroll
      for (int p = 0; p < N; ++p) acc = fma(TS.lift[side][p], Qe[c * NP + qv + p * SA], acc);
      TO[c] = acc;
    }
    const long long nb = mesh.nbr[ge * NF + f];
    ElemGeo<D> og = elem_geo<D>(mesh.elem, P.gc, (kd == KIND_CONF && side == 0) ? nb : ge);
    const int oside = (kd == KIND_CONF && side == 0) ? 1 : side;
    const bool outward = (kd == KIND_WALL || kd == KIND_FARFIELD);
    double n[D], ws;
    face_metric_ax<D, N, AX>(P.gc, mesh.col, og, oside, outward, qf, TS, n, ws);
    if (outward) {
      ghost<D, N, OPK, KIN>(P, kd, nb, qf, TO, n, TN);
    } else {
      const double* tn = base + e * L::ELEM + nb_off + f * KIN * NQF;
#pragma unroll
      for (int c = 0; c < KIN; ++c) TN[c] = tn[c * NQF + qf];
    }
    const bool minus = outward || side == 1;
    double TLv[KIN], TRv[KIN];
#pragma unroll
    for (int c = 0; c < KIN; ++c) {
      TLv[c] = minus ? TO[c] : TN[c];
      TRv[c] = minus ? TN[c] : TO[c];
    }
    double fl[KOUT];
    num_flux<D, OPK, KIN, KOUT>(TLv, TRv, n, P.model.kinetic_factor, fl, &P.model, P.full);
    const double sg = minus ? ws : -ws;
#pragma unroll
    for (int k = 0; k < KOUT; ++k) Lf[k * NQF + qf] = fl[k] * sg;
  }
}

// ------------------------------------------------------------- the kernel
template <int D, int N, int OPK>
__global__ void __launch_bounds__(Layout<D, N, OPK>::THREADS, Layout<D, N, OPK>::MINB)
elem_kernel(const __grid_constant__ KParams<N> P) {
  using L = Layout<D, N, OPK>;
  constexpr int NP = L::NP, NQF = L::NQF, NF = L::NF, KIN = L::KIN, KOUT = L::KOUT;
  constexpr int E = L::ELEM;
  extern __shared__ double smem[];
  __shared__ short fnode[NF * NQF];  // volume node of face point j on face f
  {
    for (int i = threadIdx.x; i < L::TABD; i += blockDim.x) smem[i] = P.tab_g[i];
    for (int i = threadIdx.x; i < NF * NQF; i += blockDim.x)
      fnode[i] = (short)face_to_vol<D, N>((i / NQF) >> 1, (i / NQF) & 1, i % NQF);
  }
  __syncthreads();
  const Tab<N>& TS = *reinterpret_cast<const Tab<N>*>(smem);
  const Tab<N>& TC = P.tab;
  double* red = smem + L::TABD;
  double* base = red + 64;
  const MeshDev& mesh = P.mesh;
  const int tid = threadIdx.x;
  const long long e0 = (long long)blockIdx.x * L::EPB;
  const int nv = (int)min((long long)L::EPB, (long long)mesh.n_el - e0);
  const int el0 = tid / NP;
  const bool act = el0 < nv;
  // padding threads (EPB * NP not a multiple of 32) shadow slot 0: their
  // per-point writes repeat the owner's identical values inside the same
  // barrier phase, and every accumulation / store is guarded by act
  const int el = el0 < L::EPB ? el0 : 0;
  const int q = el0 < L::EPB ? tid - el0 * NP : (tid - L::EPB * NP) % NP;
  double* A = base + el * E + L::OFF_A;
  double* Q = base + el * E + L::OFF_Q;
  double* Z = base + el * E + L::OFF_Z;
  double* Tm = base + el * E + L::OFF_T;

  // 1. nodal input
  if (act) {
#pragma unroll
    for (int c = 0; c < KIN; ++c) A[c * NP + q] = load_input<D, N, OPK>(P, e0 + el, c, q);
  }
  // 4a (early). gather neighbour nodal face values: overlaps with the volume work
  const bool do_faces = !(P.dbg & 1);
  if (do_faces) {
    const int items = nv * NF * KIN * NQF;
    for (int it = tid; it < items; it += blockDim.x) {
      const int j = it % NQF;
      int r = it / NQF;
      const int c = r % KIN;
      r /= KIN;
      const int f = r % NF;
      const int e = r / NF;
      const long long ge = e0 + e;
      const int kd = mesh.kind[ge * NF + f] & 15;
      if (kd != KIND_CONF && kd != KIND_FINE) continue;
      const long long src = mesh.nbr[ge * NF + f];
      base[e * E + L::OFF_G + (f * KIN + c) * NQF + j] =
          load_input<D, N, OPK>(P, src, c, fnode[(f ^ 1) * NQF + j]);
    }
  }
  __syncthreads();

  // 2. nodes -> Gauss points
  interp_all<D, N, KIN, E, NP, L::EPB, L::THREADS>(TC.B, base, L::OFF_A, L::OFF_Q, L::OFF_T);
  // tangential passes of the gathered faces (independent buffers: no sync)
  if constexpr (D == 2) {
    fpass<D, N, 0, KIN, E, NF, L::EPB, L::THREADS>(TS, mesh.kind, e0, base, L::OFF_G, L::OFF_H, nv);
  } else {
    fpass<D, N, 0, KIN, E, NF, L::EPB, L::THREADS>(TS, mesh.kind, e0, base, L::OFF_G, L::OFF_H, nv);
  }
  __syncthreads();
  if constexpr (D == 3) fpass<D, N, 1, KIN, E, NF, L::EPB, L::THREADS>(TS, mesh.kind, e0, base, L::OFF_H, L::OFF_G, nv);
  constexpr int NB_OFF = (D == 2) ? L::OFF_H : L::OFF_G;  // neighbour traces at Gauss points

  // 3. metric + volume flux at this Gauss point
  const long long es = act ? e0 + el : e0;
  const ElemGeo<D> g = elem_geo<D>(mesh.elem, P.gc, es);
  double det, ctrv[D][D];
  point_metric<D, N>(P, g, q, det, ctrv);
  const double wq = point_weight<D, N>(TC, q);
  double F[D][KOUT];
  if constexpr (OPK == OP_ADV) {
    if (P.full) {
      double Uq[D + 2], Ff[D + 2][D];
#pragma unroll
      for (int c = 0; c < D + 2; ++c) Uq[c] = Q[c * NP + q];
      full_flux<D>(Uq, P.model, Ff);
#pragma unroll
      for (int a = 0; a < D; ++a)
#pragma unroll
        for (int c = 0; c < D + 2; ++c) F[a][c] = Ff[c][a];
    } else {
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
    }
  } else if constexpr (OPK == OP_DIVHV) {
    const double h = Q[D * NP + q];
#pragma unroll
    for (int a = 0; a < D; ++a) F[a][0] = h * Q[a * NP + q];
  } else {
    const double p = Q[q];
#pragma unroll
    for (int a = 0; a < D; ++a)
#pragma unroll
      for (int k = 0; k < KOUT; ++k) F[a][k] = (a == k) ? p : 0.0;
  }
  // Z = -sum_bx Dhat^T_bx G_bx, G_bx = w sum_a ctrv[bx][a] F_a: every
  // direction is written at once (bx < d-1 to W, bx = d-1 to T), passed in
  // place concurrently and summed into Z in the lift phase -- one barrier
  // instead of two per direction
  const bool flat = !P.gc.terrain;
  constexpr int KW = L::KW;
  double* W = base + el * E + L::OFF_W;
  if constexpr (OPK == OP_GRAD) {
    // rows bx < d-1 of the adjugate are structurally diagonal
    // (geometry.py:219-231): only component bx moves in those directions
#pragma unroll
    for (int bx = 0; bx < D - 1; ++bx) W[bx * NP + q] = F[bx][bx] * ctrv[bx][bx] * wq;
#pragma unroll
    for (int k = 0; k < KOUT; ++k) Tm[k * NP + q] = F[k][k] * ctrv[D - 1][k] * wq;
  } else {
#pragma unroll
    for (int bx = 0; bx < D; ++bx) {
      double* dst = (bx < D - 1) ? W + bx * KOUT * NP : Tm;
#pragma unroll
      for (int k = 0; k < KOUT; ++k) {
        double acc;
        if (flat) {
          acc = F[bx][k] * ctrv[bx][bx];
        } else {
          acc = 0.0;
#pragma unroll
          for (int a = 0; a < D; ++a) acc += F[a][k] * ctrv[bx][a];
        }
        dst[k * NP + q] = acc * wq;
      }
    }
  }
  __syncthreads();
  vpass<D, N, 0, true, 1, KW, E, NP, L::EPB, L::THREADS>(TC.Dhat, base, L::OFF_W, L::OFF_W);
  if constexpr (D == 3)
    vpass<D, N, 1, true, 1, KW, E, NP, L::EPB, L::THREADS>(TC.Dhat, base, L::OFF_W + KW * NP,
                                                           L::OFF_W + KW * NP);
  vpass<D, N, D - 1, true, 1, KOUT, E, NP, L::EPB, L::THREADS>(TC.Dhat, base, L::OFF_T, L::OFF_T);

  // 4b. numerical fluxes on all faces (disjoint outputs per axis: no sync)
  if (do_faces) {
    face_flux_axis<D, N, OPK, 0>(P, TS, base, e0, nv, NB_OFF);
    face_flux_axis<D, N, OPK, 1>(P, TS, base, e0, nv, NB_OFF);
    if constexpr (D == 3) face_flux_axis<D, N, OPK, 2>(P, TS, base, e0, nv, NB_OFF);
  }
  __syncthreads();
  // 4c. Z = (volume directions) + lift[side][q_a] * L_{a,side}[k][q_t]
  if (act) {
    double zk[KOUT];
#pragma unroll
    for (int k = 0; k < KOUT; ++k) {
      zk[k] = Tm[k * NP + q];
#pragma unroll
      for (int bx = 0; bx < D - 1; ++bx) {
        if constexpr (OPK == OP_GRAD) {
          if (k == bx) zk[k] += W[bx * NP + q];
        } else {
          zk[k] += W[(bx * KOUT + k) * NP + q];
        }
      }
    }
    if (do_faces) {
      const double* Lb = base + el * E + L::OFF_L;
      int qi[D];
#pragma unroll
      for (int a = 0; a < D; ++a) qi[a] = digit<D, N>(q, a);
#pragma unroll
      for (int a = 0; a < D; ++a) {
        int qf;
        if constexpr (D == 2) qf = qi[1 - a];
        else qf = (a == 0) ? qi[1] * N + qi[2] : (a == 1 ? qi[0] * N + qi[2] : qi[0] * N + qi[1]);
        const double l0 = TS.lift[0][qi[a]], l1 = TS.lift[1][qi[a]];
#pragma unroll
        for (int k = 0; k < KOUT; ++k)
          zk[k] += l0 * Lb[((2 * a) * KOUT + k) * NQF + qf] +
                   l1 * Lb[((2 * a + 1) * KOUT + k) * NQF + qf];
      }
    }
#pragma unroll
    for (int k = 0; k < KOUT; ++k) Z[k * NP + q] = zk[k];
  }

  // 5. epilogue
  if constexpr (OPK == OP_ADV) {
    if (P.mass_partial != nullptr) {
      double v = act ? Z[q] : 0.0;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
      if ((tid & 31) == 0) red[tid >> 5] = v;
    }
  }
  if (P.mode == OUT_MINV && act) {
    const double inv = 1.0 / (wq * det);
#pragma unroll
    for (int k = 0; k < KOUT; ++k) Z[k * NP + q] *= inv;
  }
  __syncthreads();
  if constexpr (OPK == OP_ADV) {
    if (P.mass_partial != nullptr && tid == 0) {
      double s = 0.0;
      for (int w = 0; w < (int)(blockDim.x >> 5); ++w) s += red[w];
      P.mass_partial[blockIdx.x] = s;
    }
  }
  const double* res;
  if (P.mode == OUT_MINV) {
    if constexpr (D == 2) {
      vpass<2, N, 1, false, 0, KOUT, E, NP, L::EPB, L::THREADS>(TC.Binv, base, L::OFF_Z, L::OFF_T);
      __syncthreads();
      vpass<2, N, 0, false, 0, KOUT, E, NP, L::EPB, L::THREADS>(TC.Binv, base, L::OFF_T, L::OFF_Z);
      res = Z;
    } else {
      vpass<3, N, 2, false, 0, KOUT, E, NP, L::EPB, L::THREADS>(TC.Binv, base, L::OFF_Z, L::OFF_T);
      __syncthreads();
      vpass<3, N, 1, false, 0, KOUT, E, NP, L::EPB, L::THREADS>(TC.Binv, base, L::OFF_T, L::OFF_Z);
      __syncthreads();
      vpass<3, N, 0, false, 0, KOUT, E, NP, L::EPB, L::THREADS>(TC.Binv, base, L::OFF_Z, L::OFF_T);
      res = Tm;
    }
  } else {
    if constexpr (D == 2) {
      vpass<2, N, 1, true, 0, KOUT, E, NP, L::EPB, L::THREADS>(TC.B, base, L::OFF_Z, L::OFF_T);
      __syncthreads();
      vpass<2, N, 0, true, 0, KOUT, E, NP, L::EPB, L::THREADS>(TC.B, base, L::OFF_T, L::OFF_Z);
      res = Z;
    } else {
      vpass<3, N, 2, true, 0, KOUT, E, NP, L::EPB, L::THREADS>(TC.B, base, L::OFF_Z, L::OFF_T);
      __syncthreads();
      vpass<3, N, 1, true, 0, KOUT, E, NP, L::EPB, L::THREADS>(TC.B, base, L::OFF_T, L::OFF_Z);
      __syncthreads();
      vpass<3, N, 0, true, 0, KOUT, E, NP, L::EPB, L::THREADS>(TC.B, base, L::OFF_Z, L::OFF_T);
      res = Tm;
    }
  }
  __syncthreads();
  if (!act) return;
  const long long e = e0 + el;
  double* out = P.out.p + e * P.out.estride + q;
  if (P.mode == OUT_DUAL) {
#pragma unroll
    for (int k = 0; k < KOUT; ++k) out[k * P.out.cstride] = res[k * NP + q];
    return;
  }
  if constexpr (OPK == OP_ADV) {
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
      const double r = __dmul_rn(P.coef, res[k * NP + q]);
      out[k * P.out.cstride] = P.has_base ? __dadd_rn(P.base(e, k, q), r) : r;
    }
  }
}

// fused Gram-Schmidt dots of one complete coarse element (CTHREADS threads,
// thread q owns node q with final value yv), row gs_row0 + CTA of gs_part;
// columns as gs_dots (dg_wkernel.cuh): single (V_i.y, y.y) or dual pairs
// (item.y, item.u) over the items V_i, y, u (u = the base)
template <int D, int N, int OPK>
__device__ __forceinline__ void coarse_dots(const KParams<N>& P, long long e, int q, bool act,
                                            double yv, double* wr /* NW x 32 */) {
  using L = Layout<D, N, OPK>;
  constexpr int NP = L::NP;
  if (P.gs_part == nullptr) return;
  const bool dual = P.gs_dual != 0;
  const int nv = P.gs_nv;
  const int nvt = dual ? 2 * (nv + 2) : nv + 1;
  const double uq = (act && dual) ? P.base(e, 0, q) : 0.0;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  constexpr int NW = L::CTHREADS / 32;
  for (int c0 = 0; c0 < nvt; c0 += 32) {
    const int cnt = min(32, nvt - c0);
    for (int cc = 0; cc < cnt; ++cc) {
      const int col = c0 + cc;
      const int item = dual ? col >> 1 : col;
      const double other = (dual && (col & 1)) ? uq : yv;
      double s = 0.0;
      if (act) {
        const double v = item < nv ? P.gsV[(long long)item * P.gs_vs + e * NP + q]
                                   : (item == nv ? yv : uq);
        s = v * other;
      }
      for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
      if (lane == 0) wr[wid * 32 + cc] = s;
    }
    __syncthreads();
    if (threadIdx.x < cnt) {
      double s = 0.0;
      for (int w = 0; w < NW; ++w) s += wr[w * 32 + threadIdx.x];
      P.gs_part[((long long)P.gs_row0 + blockIdx.x) * nvt + c0 + threadIdx.x] = s;
    }
    __syncthreads();
  }
}

// ---------------------------------------------------- coarse-side fix-up
// One CTA per element owning >= 1 coarse hanging face: the coarse side's
// subface fluxes (fine-side metric, mortar traces, dgops.py:159-206) lifted
// through halfq^T, then the same epilogue as the main kernel, ADDED to the
// main kernel's output (linear in the lift).
#ifndef DG_CMINB_GRAD
#define DG_CMINB_GRAD 8
#endif
#ifndef DG_CFLUX_THREADS
#define DG_CFLUX_THREADS 1024
#endif
// FM: flux-mode instantiation (only the coarse faces' fluxes into
// mesh.cflux, no epilogue): capped at 64 registers so DG_CFLUX_THREADS
// threads stay resident per SM -- the kernel is latency-bound (dependent
// record -> children -> data loads)
template <int OPK, bool FM, int CT>
constexpr int coarse_minb() {
  return FM ? (DG_CFLUX_THREADS / CT > 0 ? DG_CFLUX_THREADS / CT : 1)
            : (OPK == OP_GRAD ? DG_CMINB_GRAD : (OPK == OP_DIVHV ? 10 : 6));
}
template <int D, int N, int OPK, bool FM = false>
__global__ void __launch_bounds__(Layout<D, N, OPK>::CTHREADS,
                                  coarse_minb<OPK, FM, Layout<D, N, OPK>::CTHREADS>())
coarse_kernel(const __grid_constant__ KParams<N> P, const int* __restrict__ clist, int ncoarse,
              double* mass_partial) {
  using L = Layout<D, N, OPK>;
  constexpr int NP = L::NP, NQF = L::NQF, NF = L::NF, S = L::S, KIN = L::KIN, KOUT = L::KOUT;
  extern __shared__ double smem[];
  // tables from their global copy (coalesced; the kernel-parameter copy
  // serialises on divergent constant-bank reads)
  pdl_trigger();
  for (int i = threadIdx.x; i < L::TABD; i += blockDim.x) smem[i] = P.tab_g[i];
  pdl_wait();  // (programmatic dependent launch, small problems: dg_common.cuh)
  const Tab<N>& T = *reinterpret_cast<const Tab<N>*>(smem);
  double* red = smem + L::TABD;
  double* A = red + 64 + L::C_A;
  double* FW = red + 64 + L::C_FW;
  double* Z = red + 64 + L::C_Z;
  double* Tm = red + 64 + L::C_T;
  double* OT = red + 64 + L::C_OT;
  const MeshDev& mesh = P.mesh;
  const int* crec = clist + (long long)blockIdx.x * (1 + NF + NF * S);  // coarse record
  const long long e = crec[0];
  // flux mode: only the coarse faces' lifted fluxes, into mesh.cflux (the
  // element kernel lifts them with the rest of its faces)
  const bool fmode = FM || P.mesh.cflux != nullptr;
  const int q = threadIdx.x;
  const bool act = q < NP;
  // the Helmholtz H1 output at this Gauss point (read-modify-written at the
  // end): issued first so the final update does not wait on it
  double out_pre[KOUT];
  if (OPK == OP_GRAD && P.out_quad && act && !fmode)
#pragma unroll
    for (int k = 0; k < KOUT; ++k) out_pre[k] = P.out.p[e * P.out.estride + k * P.out.cstride + q];
  // (trace mode: the own traces come from the trace buffers, no input tile)
  if (act && !(OPK == OP_DIVHV && P.in_quad && P.trV != nullptr))
    for (int c = 0; c < KIN; ++c) A[c * NP + q] = load_input<D, N, OPK>(P, e, c, q);
  __syncthreads();
  __shared__ short cfnode[NF * NQF];
  for (int i = threadIdx.x; i < NF * NQF; i += blockDim.x)
    cfnode[i] = (short)face_to_vol<D, N>((i / NQF) >> 1, (i / NQF) & 1, i % NQF);
  double* CH = red + 64 + L::C_CH;
  // the element's face records and each coarse face's children, loaded once
  __shared__ uint8_t s_kind[NF];
  __shared__ int s_child[NF][S];
  __shared__ int s_grp[NF];
  if (threadIdx.x < NF * S) {
    const int f = threadIdx.x / S, sub = threadIdx.x % S;
    const int ch = crec[1 + NF + threadIdx.x];
    s_child[f][sub] = ch < 0 ? 0 : ch;
    if (sub == 0) {
      s_kind[f] = ch < 0 ? 0 : KIND_COARSE;
      s_grp[f] = crec[1 + f];
    }
  }
  if (act)
#pragma unroll
    for (int k = 0; k < KOUT; ++k) Z[k * NP + q] = 0.0;
  // one coarse face at a time (the face kind is uniform over the CTA): stage
  // the children's nodal face values, subface fluxes, lift into Z
  for (int f = 0; f < NF; ++f) {
    __syncthreads();  // face records staged; previous face's CH / FW consumed
    if (s_kind[f] != KIND_COARSE) continue;
    for (int it = threadIdx.x; it < S * KIN * NQF; it += blockDim.x) {
      const int j = it % NQF;
      int r = it / NQF;
      const int cp = r % KIN;
      const int sub = r / KIN;
      const long long child = s_child[f][sub];
      if (OPK == OP_DIVHV && P.psi != nullptr) {
        // flux-trace mode: the child's psi = 1/2 ws h (V . n+) on its face
        // f ^ 1 at its face Gauss point j (dg_hkernel.cuh)
        constexpr int PSL = NF * NQF;
        CH[it] = (cp == 0) ? P.psi[child * PSL + (f ^ 1) * NQF + j] : 0.0;
      } else if (OPK == OP_DIVHV && P.in_quad && P.trV != nullptr) {
        // trace mode: the child's V / h traces on its face f ^ 1 at its face
        // Gauss point j (vertical faces carry only the normal component)
        const bool vert = (f >> 1) < D - 1;
        constexpr int TSL = tr_slots<D>() * NQF, THL = 2 * D * NQF;
        double t = 0.0;
        if (cp == D) t = P.trH[child * THL + (f ^ 1) * NQF + j];
        else if (!vert || cp == (f >> 1)) t = P.trV[child * TSL + tr_slot<D>(f ^ 1, cp) * NQF + j];
        CH[it] = t;
      } else if (OPK == OP_DIVHV && P.in_quad) {
        // Gauss-point input: the child's trace at its face Gauss point j
        const int ax = f >> 1, cs = 1 - (f & 1);
        const int b = face_to_vol<D, N>(ax, 0, j), st = stride_of<D, N>(ax);
        double t = 0.0;
        for (int p = 0; p < N; ++p)
          t = fma(T.lift[cs][p], load_input<D, N, OPK>(P, child, cp, b + p * st), t);
        CH[it] = t;
      } else {
        // the child's node on the opposite face of the same axis (f ^ 1)
        CH[it] = load_input<D, N, OPK>(P, child, cp, cfnode[(f ^ 1) * NQF + j]);
      }
    }
    if (OPK == OP_DIVHV && P.in_quad && P.trV != nullptr) {
      // trace mode: this element's own traces on face f (the coarse side)
      const bool vert = (f >> 1) < D - 1;
      constexpr int TSL = tr_slots<D>() * NQF, THL = 2 * D * NQF;
      for (int it = threadIdx.x; it < KIN * NQF; it += blockDim.x) {
        const int cp = it / NQF, j = it - (it / NQF) * NQF;
        double t = 0.0;
        if (cp == D) t = P.trH[e * THL + f * NQF + j];
        else if (!vert || cp == (f >> 1)) t = P.trV[e * TSL + tr_slot<D>(f, cp) * NQF + j];
        OT[it] = t;
      }
    }
    __syncthreads();
    // the separable path covers nodal inputs and the flux-trace (psi) mode;
    // the Gauss-point-input variants without psi keep the generic loop
    const bool sep_ok = (OPK != OP_DIVHV) || !P.in_quad || (P.trV != nullptr && P.psi != nullptr);
    if (D == 3 && FM && sep_ok) {
      // Flux mode, 3D: the mortar interpolations factor over the two
      // tangential directions, so each is two 1D passes through a shared
      // scratch instead of an n^2-term sum per point with product
      // coefficients.
      double* SC = red + 64 + L::C_SC;
      // own traces staged (flux-trace mode) or own nodal face values (A)
      const bool TRC = (OPK == OP_DIVHV) && P.in_quad;
      constexpr int NN = N * N;
      double* T1 = SC;                        // [KIN][2][N][N]  own partials
      double* U = SC + KIN * 2 * NN;          // [S][KIN][N][N]  children's partials (nodal)
      const int axis = f >> 1, side = f & 1;
      // A: T1[c][b1][j0][q1] = sum_j1 M_b1[q1][j1] own[c][j0 N + j1]
      for (int it = threadIdx.x; it < KIN * 2 * NN; it += blockDim.x) {
        const int q1 = it % N, j0 = (it / N) % N, b1 = (it / NN) % 2, cc = it / (2 * NN);
        double t = 0.0;
        for (int j1 = 0; j1 < N; ++j1) {
          const int j = j0 * N + j1;
          const double own = TRC ? OT[cc * NQF + j] : A[cc * NP + cfnode[f * NQF + j]];
          const double m = TRC ? T.halfq[b1][q1][j1] : T.half[b1][q1][j1];
          t = fma(m, own, t);
        }
        T1[it] = t;
      }
      // A': U[sub][c][j0][q1] = sum_j1 B[q1][j1] child[sub][c][j0 N + j1]
      if (!TRC) {
        for (int it = threadIdx.x; it < S * KIN * NN; it += blockDim.x) {
          const int q1 = it % N, j0 = (it / N) % N, r = it / NN;  // r = sub * KIN + c
          double t = 0.0;
          for (int j1 = 0; j1 < N; ++j1) t = fma(T.B[q1][j1], CH[r * NQF + j0 * N + j1], t);
          U[it] = t;
        }
      }
      __syncthreads();
      // B: the subface fluxes (fine-side metric) at every fine point
      for (int it = threadIdx.x; it < S * NQF; it += blockDim.x) {
        const int qf = it % NQF, sub = it / NQF;
        const int q0 = qf / N, q1 = qf % N;
        const int b0 = sub & 1, b1 = (sub >> 1) & 1;
        const long long child = s_child[f][sub];
        double TO[KIN], TN[KIN];
#pragma unroll
        for (int cc = 0; cc < KIN; ++cc) {
          double ao = 0.0;
          for (int j0 = 0; j0 < N; ++j0) {
            const double m = TRC ? T.halfq[b0][q0][j0] : T.half[b0][q0][j0];
            ao = fma(m, T1[((cc * 2 + b1) * N + j0) * N + q1], ao);
          }
          TO[cc] = ao;
          if (TRC) {
            TN[cc] = CH[(sub * KIN + cc) * NQF + qf];
          } else {
            double an = 0.0;
            for (int j0 = 0; j0 < N; ++j0)
              an = fma(T.B[q0][j0], U[((sub * KIN + cc) * N + j0) * N + q1], an);
            TN[cc] = an;
          }
        }
        const ElemGeo<D> og = elem_geo<D>(mesh.elem, P.gc, child);
        double n[D], ws;
        if (axis == 0) face_metric_ax<D, N, 0>(P.gc, mesh.col, og, 1 - side, false, qf, T, n, ws);
        else if (axis == 1) face_metric_ax<D, N, 1>(P.gc, mesh.col, og, 1 - side, false, qf, T, n, ws);
        else face_metric_ax<D, N, D - 1>(P.gc, mesh.col, og, 1 - side, false, qf, T, n, ws);
        const bool minus = side == 1;
        double fl[KOUT];
        if (OPK == OP_DIVHV && P.psi != nullptr) {
          double vn = 0.0;
#pragma unroll
          for (int a = 0; a < D; ++a) vn = fma(TO[a], n[a], vn);
          fl[0] = (minus ? 1.0 : -1.0) * (TN[0] + (0.5 * ws) * (TO[D] * vn));
#pragma unroll
          for (int k = 0; k < KOUT; ++k) FW[(sub * KOUT + k) * NQF + qf] = fl[k];
        } else {
          double TLv[KIN], TRv[KIN];
#pragma unroll
          for (int cc = 0; cc < KIN; ++cc) {
            TLv[cc] = minus ? TO[cc] : TN[cc];
            TRv[cc] = minus ? TN[cc] : TO[cc];
          }
          num_flux<D, OPK, KIN, KOUT>(TLv, TRv, n, P.model.kinetic_factor, fl, &P.model, P.full);
          const double sg = minus ? ws : -ws;
#pragma unroll
          for (int k = 0; k < KOUT; ++k) FW[(sub * KOUT + k) * NQF + qf] = fl[k] * sg;
        }
      }
      __syncthreads();
      // C: Pp[sub][k][j0][q1] = sum_j1 halfq[b1][j1][q1] FW[sub][k][j0 N + j1]
      double* Pp = SC;
      for (int it = threadIdx.x; it < S * KOUT * NN; it += blockDim.x) {
        const int q1 = it % N, j0 = (it / N) % N, r = it / NN;  // r = sub * KOUT + k
        const int b1 = ((r / KOUT) >> 1) & 1;
        double t = 0.0;
        for (int j1 = 0; j1 < N; ++j1) t = fma(T.halfq[b1][j1][q1], FW[r * NQF + j0 * N + j1], t);
        Pp[it] = t;
      }
      __syncthreads();
      // C': G[k][q0 N + q1] = sum_sub sum_j0 halfq[b0][j0][q0] Pp[sub][k][j0][q1] -> cflux
      const long long grp = s_grp[f];
      for (int it = threadIdx.x; it < KOUT * NQF; it += blockDim.x) {
        const int k = it / NQF, qt = it % NQF, q0 = qt / N, q1 = qt % N;
        double acc = 0.0;
        for (int sub = 0; sub < S; ++sub) {
          const int b0 = sub & 1;
          for (int j0 = 0; j0 < N; ++j0)
            acc = fma(T.halfq[b0][j0][q0], Pp[((sub * KOUT + k) * N + j0) * N + q1], acc);
        }
        P.mesh.cflux[grp * KOUT * NQF + it] = acc;
      }
      continue;
    }
    // subface fluxes of this coarse face
    for (int it = threadIdx.x; it < S * NQF; it += blockDim.x) {
      const int qf = it % NQF;
      const int sub = it / NQF;
      const int axis = f >> 1, side = f & 1;
      const long long child = s_child[f][sub];
      const int qt0 = (D == 2) ? qf : qf / N;
      const int qt1 = (D == 2) ? 0 : qf % N;
      const int b0 = sub & 1, b1 = (sub >> 1) & 1;
      double TO[KIN], TN[KIN];
      const double* chv = CH + (sub * KIN) * NQF;
      const bool iq = (OPK == OP_DIVHV) && P.in_quad;
#pragma unroll
      for (int c = 0; c < KIN; ++c) {
        double ao = 0.0, an = 0.0;
        if (iq && P.trV != nullptr) {
          // trace mode: own coarse-face Gauss trace (staged from the trace
          // buffers) -> fine Gauss points through halfq (x) halfq
          for (int j = 0; j < NQF; ++j) {
            const int j0 = (D == 2) ? j : j / N;
            const int j1 = (D == 2) ? 0 : j % N;
            double mo = T.halfq[b0][qt0][j0];
            if (D == 3) mo *= T.halfq[b1][qt1][j1];
            ao = fma(mo, OT[c * NQF + j], ao);
          }
          an = chv[c * NQF + qf];
        } else if (iq) {
          // own coarse-face Gauss trace (lift contraction) -> fine Gauss points
          // through halfq (x) halfq; the child's trace was staged at qf
          const int st = stride_of<D, N>(axis);
          for (int j = 0; j < NQF; ++j) {
            const int j0 = (D == 2) ? j : j / N;
            const int j1 = (D == 2) ? 0 : j % N;
            double mo = T.halfq[b0][qt0][j0];
            if (D == 3) mo *= T.halfq[b1][qt1][j1];
            const int bj = face_to_vol<D, N>(axis, 0, j);
            double tg = 0.0;
            for (int p = 0; p < N; ++p) tg = fma(T.lift[side][p], A[c * NP + bj + p * st], tg);
            ao = fma(mo, tg, ao);
          }
          an = chv[c * NQF + qf];
        } else {
          for (int j = 0; j < NQF; ++j) {
            const int j0 = (D == 2) ? j : j / N;
            const int j1 = (D == 2) ? 0 : j % N;
            double mo = T.half[b0][qt0][j0];
            double mb = T.B[qt0][j0];
            if (D == 3) {
              mo *= T.half[b1][qt1][j1];
              mb *= T.B[qt1][j1];
            }
            ao = fma(mo, A[c * NP + cfnode[f * NQF + j]], ao);
            an = fma(mb, chv[c * NQF + j], an);
          }
        }
        TO[c] = ao;
        TN[c] = an;
      }
      const ElemGeo<D> og = elem_geo<D>(mesh.elem, P.gc, child);
      double n[D], ws;
      if (axis == 0) face_metric_ax<D, N, 0>(P.gc, mesh.col, og, 1 - side, false, qf, T, n, ws);
      else if (axis == 1 || D == 2) face_metric_ax<D, N, (D == 2 ? 1 : 1)>(P.gc, mesh.col, og, 1 - side, false, qf, T, n, ws);
      else face_metric_ax<D, N, D - 1>(P.gc, mesh.col, og, 1 - side, false, qf, T, n, ws);
      const bool minus = side == 1;
      double TLv[KIN], TRv[KIN];
#pragma unroll
      for (int c = 0; c < KIN; ++c) {
        TLv[c] = minus ? TO[c] : TN[c];
        TRv[c] = minus ? TN[c] : TO[c];
      }
      double fl[KOUT];
      if (OPK == OP_DIVHV && P.psi != nullptr) {
        // flux-trace mode: the child's half is its psi (fine-side metric,
        // the same n+ and ws as below), the coarse half 1/2 ws h (V . n+)
        // from the mortar-interpolated own traces
        double vn = 0.0;
#pragma unroll
        for (int a = 0; a < D; ++a) vn = fma(TO[a], n[a], vn);
        fl[0] = (minus ? 1.0 : -1.0) * (TN[0] + (0.5 * ws) * (TO[D] * vn));
#pragma unroll
        for (int k = 0; k < KOUT; ++k) FW[(sub * KOUT + k) * NQF + qf] = fl[k];
      } else {
      num_flux<D, OPK, KIN, KOUT>(TLv, TRv, n, P.model.kinetic_factor, fl, &P.model, P.full);
      const double sg = minus ? ws : -ws;
#pragma unroll
      for (int k = 0; k < KOUT; ++k) FW[(sub * KOUT + k) * NQF + qf] = fl[k] * sg;
      }
    }
    __syncthreads();
    // coarse-face flux at the coarse face Gauss points, once per point:
    // G[k][qt] = sum_sub (halfq^T (x) halfq^T) FW[sub][k]  (into the consumed
    // children staging area CH)
    {
      double* G = CH;
      for (int it = threadIdx.x; it < KOUT * NQF; it += blockDim.x) {
        const int k = it / NQF, qt = it - (it / NQF) * NQF;
        const int qt0 = (D == 2) ? qt : qt / N;
        const int qt1 = (D == 2) ? 0 : qt % N;
        double acc = 0.0;
        for (int sub = 0; sub < S; ++sub) {
          const int b0 = sub & 1, b1 = (sub >> 1) & 1;
          const double* fw = FW + (sub * KOUT + k) * NQF;
          for (int j = 0; j < NQF; ++j) {
            const int j0 = (D == 2) ? j : j / N;
            const int j1 = (D == 2) ? 0 : j % N;
            double m = T.halfq[b0][j0][qt0];
            if (D == 3) m *= T.halfq[b1][j1][qt1];
            acc = fma(m, fw[j], acc);
          }
        }
        G[it] = acc;
      }
    }
    __syncthreads();
    if (fmode) {
      // flux mode: hand the coarse face's flux to the element kernel
      const long long grp = s_grp[f];
      for (int it = threadIdx.x; it < KOUT * NQF; it += blockDim.x)
        P.mesh.cflux[grp * KOUT * NQF + it] = CH[it];
      continue;
    }
    // lift: Z += lift[side] (x) G
    if (act) {
      int qi[D];
#pragma unroll
      for (int a = 0; a < D; ++a) qi[a] = digit<D, N>(q, a);
      const int a = f >> 1, side = f & 1;
      int qt0, qt1 = 0;
      if (D == 2) qt0 = qi[1 - a];
      else {
        qt0 = (a == 0) ? qi[1] : qi[0];
        qt1 = (a == 2) ? qi[1] : qi[2];
      }
      const int qt = (D == 2) ? qt0 : qt0 * N + qt1;
      const double lw = T.lift[side][qi[a]];
#pragma unroll
      for (int k = 0; k < KOUT; ++k) Z[k * NP + q] += lw * CH[k * NQF + qt];
    }
  }
  if (fmode) return;
  if constexpr (!FM) {
  double wq = 1.0, det = 1.0;
  if (act) {
    const ElemGeo<D> g = elem_geo<D>(mesh.elem, P.gc, e);
    double ctrv[D][D];
    point_metric<D, N>(P, g, q, det, ctrv);
    wq = point_weight<D, N>(T, q);
  }
  if (OPK == OP_ADV && mass_partial != nullptr) {
    double v = act ? Z[q] : 0.0;
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  }
  __syncthreads();
  if (OPK == OP_ADV && mass_partial != nullptr && threadIdx.x == 0) {
    double s = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) s += red[w];
    mass_partial[blockIdx.x] = s;
  }
  const double* res;
  const int qq = act ? q : 0;
  if (OPK == OP_GRAD && P.out_quad) {
    // Gauss-point output (Helmholtz H1): coef * Z / (w det), no B^-1
    if (act) {
      const double inv = 1.0 / (wq * det);
      for (int k = 0; k < KOUT; ++k) {
        double* o = P.out.p + e * P.out.estride + k * P.out.cstride + q;
        const double v = out_pre[k] + P.coef * (Z[k * NP + q] * inv);
        *o = v;
        Tm[k * NP + q] = v;  // the final V of this coarse element
      }
    }
    if (P.tr_out != nullptr) {
      // trace mode: this element's V changed -- rewrite all its face traces
      // (same lift contractions as the warp-element kernel)
      __syncthreads();
      constexpr int TSL = tr_slots<D>() * NQF;
      for (int it = threadIdx.x; it < TSL; it += blockDim.x) {
        const int slot = it / NQF, j = it - (it / NQF) * NQF;
        int f, comp;
        if (slot < 2 * (D - 1)) {
          f = slot;
          comp = slot >> 1;
        } else {
          f = 2 * (D - 1) + (slot - 2 * (D - 1)) / D;
          comp = (slot - 2 * (D - 1)) % D;
        }
        const int ax = f >> 1, side = f & 1;
        double t = 0.0;
        for (int p = 0; p < N; ++p)
          t = fma(T.lift[side][p], Tm[comp * NP + nbr_pencil_node<D, N>(ax, p, j)], t);
        P.tr_out[e * TSL + it] = t;
      }
    }
    return;
  }
  if (P.mode == OUT_MINV) {
    if (act) {
      const double inv = 1.0 / (wq * det);
      for (int k = 0; k < KOUT; ++k) Z[k * NP + q] *= inv;
    }
    __syncthreads();
    if (D == 2) {
      if (act) pass1d<D, N, KOUT,false>(&T.Binv[0][0], Z, Tm, qq, 1, NP);
      __syncthreads();
      if (act) pass1d<D, N, KOUT,false>(&T.Binv[0][0], Tm, Z, qq, 0, NP);
      res = Z;
    } else {
      if (act) pass1d<D, N, KOUT,false>(&T.Binv[0][0], Z, Tm, qq, 2, NP);
      __syncthreads();
      if (act) pass1d<D, N, KOUT,false>(&T.Binv[0][0], Tm, Z, qq, 1, NP);
      __syncthreads();
      if (act) pass1d<D, N, KOUT,false>(&T.Binv[0][0], Z, Tm, qq, 0, NP);
      res = Tm;
    }
  } else {
    if (D == 2) {
      if (act) pass1d<D, N, KOUT,true>(&T.B[0][0], Z, Tm, qq, 1, NP);
      __syncthreads();
      if (act) pass1d<D, N, KOUT,true>(&T.B[0][0], Tm, Z, qq, 0, NP);
      res = Z;
    } else {
      if (act) pass1d<D, N, KOUT,true>(&T.B[0][0], Z, Tm, qq, 2, NP);
      __syncthreads();
      if (act) pass1d<D, N, KOUT,true>(&T.B[0][0], Tm, Z, qq, 1, NP);
      __syncthreads();
      if (act) pass1d<D, N, KOUT,true>(&T.B[0][0], Z, Tm, qq, 0, NP);
      res = Tm;
    }
  }
  __syncthreads();
  double yv = 0.0;  // final value (KOUT == 1 when the Gram-Schmidt dots are fused)
  if (act) {
    double* out = P.out.p + e * P.out.estride + q;
#pragma unroll
    for (int k = 0; k < KOUT; ++k) {
      const double r = res[k * NP + q];
      double add;
      if (P.mode == OUT_DUAL) add = r;
      else if (OPK == OP_ADV) add = -r;
      else add = __dmul_rn(P.coef, r);
      const double y = out[k * P.out.cstride] + add;
      out[k * P.out.cstride] = y;
      yv = y;
    }
  }
  if constexpr (OPK == OP_DIVHV) coarse_dots<D, N, OPK>(P, e, q, act, yv, red + 64 + L::C_GS);
  }  // !FM
}


}  // namespace dg
