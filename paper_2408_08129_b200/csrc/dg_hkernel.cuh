// Lean warp-element kernels of the homogeneous pressure-Helmholtz action in
// flux-trace mode (fp64, sm_100a): the GMRES hot path.
//
//   H1 (hgrad_kernel):  V = coef diag(1/(w detJ)) G(alpha x)   at the Gauss
//                       points (the weak gradient, dgops.py:332-366, with the
//                       homogeneous ghosts of imex.py:221-242), and for every
//                       face f of the element, at its face Gauss point c,
//                           psi[e][f][c] = 1/2 ws h (V . n+)
//                       with n+ the +axis-oriented unit normal and ws the
//                       face weight of the element's own face metric
//                       (geometry.py:305-357); elements with a coarse hanging
//                       face also write their V face traces (trV) for the
//                       mortar of the fine side.
//   H2 (hdiv_kernel):   y = x + coef Minv Div_h(V)  (dgops.py:368-479).  The
//                       centred face flux 1/2 (h_L V_L.n + h_R V_R.n) ws of a
//                       conforming face is psi_own + psi_neighbour: the
//                       kernel reads two 128-byte rows per face instead of
//                       staging traces, evaluating metrics and ghosts.  Wall:
//                       the mirrored ghost cancels the flux (0); far field
//                       (homogeneous): V ghost 0, flux psi_own; fine side of
//                       a hanging face: the coarse parent's traces through the
//                       Gauss-point mortar (halfq), own metric; coarse side:
//                       precomputed by coarse_kernel (psi mode).
//
// Lane layout as the general warp-element kernel (dg_wkernel.cuh): an element
// is owned by n^(d-1) consecutive lanes, lane c holds z-column c in registers
// and face point c of every face; x / y passes go through a per-element smem
// tile under __syncwarp() only.  The 1D tables are brought into shared memory
// by one bulk copy (cp.async.bulk + mbarrier) per CTA.
#pragma once
#include "dg_wkernel.cuh"

namespace dg {

// DG_HK1_ASYNC=1: H1 stages the neighbours' face nodes and its own h-trace
// rows with cp.async (no register, no scoreboard wait at the staging store)
// and waits for them only after the own-column interpolation passes; the
// vertical faces' terrain scalars are loaded with the column data.  ncu of
// the synchronous version: long_scoreboard 4.7 of ~10.7 stall cycles per
// issue (the staging stores and the late h-trace loads).
#ifndef DG_HK1_ASYNC
#define DG_HK1_ASYNC 1
#endif
#ifndef DG_HK_THREADS
#define DG_HK_THREADS 128  // threads per CTA of the non-persistent pair (a multiple of 64)
#endif
template <int D, int N>
struct HLayout {
  static constexpr int NP = ipow(N, D);
  static constexpr int NC = ipow(N, D - 1);   // lanes per element
  // a "team" owns whole elements: one warp for n^(d-1) <= 32, a pair of
  // warps (named barriers) for 3D r = 5, 6
  static constexpr int TPE = NC <= 32 ? 32 : 64;
  static constexpr int EPW = TPE / NC;        // elements per team
  static constexpr int NSLOT = EPW + ((TPE % NC) ? 1 : 0);
  static constexpr int THREADS = DG_HK_THREADS;
  static constexpr int WPB = THREADS / TPE;   // teams per CTA
  static constexpr int NF = 2 * D;
  static constexpr int TSZ = tile_size<D, N>();
  static constexpr int TABD = (int)(sizeof(Tab<N>) / sizeof(double));
  static constexpr int TABP = (TABD + 1) & ~1;  // element slots 16-byte aligned
  static constexpr int KX = (D - 1) > 1 ? (D - 1) : 1;  // tile comps
  static constexpr int NHW = 2 * (D - 1) + 2 * D;       // 1/2 ws n+ values per face point
  static constexpr int odd(int s) { return (s % 2 == 0) ? s + 1 : s; }
  // H1 slot: tile | neighbour face nodes (NF x NC) | 1/2 ws n+ (NHW x NC)
  // | own h traces (NF x NC, staged by cp.async; DG_HK1_ASYNC)
  static constexpr int GSLOT = odd(KX * TSZ + NF * NC + NHW * NC + (DG_HK1_ASYNC ? NF * NC : 0));
  // H2 slot: tile (the fine-face staging (d+1) x NC and the fused dots'
  // warp totals reuse it)
  static constexpr int DRAW = KX * TSZ > (D + 1) * NC ? KX * TSZ : (D + 1) * NC;
  static constexpr int DSLOT = odd(DRAW > 40 ? DRAW : 40);
  static constexpr size_t GSMEM = (size_t)(TABP + WPB * NSLOT * GSLOT) * sizeof(double);
  static constexpr size_t DSMEM = (size_t)(TABP + WPB * NSLOT * DSLOT) * sizeof(double);
  static constexpr bool OK = NC <= 64;
};

#ifndef DG_HK1_MINB
#define DG_HK1_MINB 5
#endif
#ifndef DG_HK2_MINB
#define DG_HK2_MINB 4
#endif

__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return (unsigned)__cvta_generic_to_shared(p);
}

// the Tab<N> tables (global copy) -> smem by one bulk copy issued by thread 0;
// every thread waits on the mbarrier (phase 0) before its first table read
__device__ __forceinline__ void tab_bulk_issue(double* dst, const double* src, unsigned bytes,
                                               unsigned long long* bar) {
  if (threadIdx.x == 0) {
    const unsigned b = smem_u32(bar);
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(b) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(b), "r"(bytes)
                 : "memory");
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::
            "r"(smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(b)
        : "memory");
  }
}
__device__ __forceinline__ void tab_bulk_wait(unsigned long long* bar) {
  const unsigned b = smem_u32(bar);
  asm volatile(
      "{\n .reg .pred P1;\n"
      "HK_WAIT:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n"
      " @P1 bra HK_DONE;\n"
      " bra HK_WAIT;\n"
      "HK_DONE:\n}\n" ::"r"(b)
      : "memory");
}

// global loads that keep their program order among each other and the
// cp.async staging (volatile asm): the prologue of H1 issues all of its
// first-level loads before anything consumes one
__device__ __forceinline__ double ldg_f64_ordered(const double* p) {
  double v;
  asm volatile("ld.global.f64 %0, [%1];\n" : "=d"(v) : "l"(p));
  return v;
}
__device__ __forceinline__ int ldg_s32_ordered(const int* p) {
  int v;
  asm volatile("ld.global.s32 %0, [%1];\n" : "=r"(v) : "l"(p));
  return v;
}
__device__ __forceinline__ uint8_t ldg_u8_ordered(const uint8_t* p) {
  unsigned v;
  asm volatile("ld.global.u8 %0, [%1];\n" : "=r"(v) : "l"(p));
  return (uint8_t)v;
}

__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, unsigned bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::
          "r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(bar)
      : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned bar, unsigned parity) {
  asm volatile(
      "{\n .reg .pred P1;\n"
      "HK2_WAIT:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      " @P1 bra HK2_DONE;\n"
      " bra HK2_WAIT;\n"
      "HK2_DONE:\n}\n" ::"r"(bar),
      "r"(parity)
      : "memory");
}

// own-geometry face metric at face point c of face (AX, side): the
// +axis-oriented unit normal n+ and the face weight ws (geometry.py:305-357;
// vertical faces have the exact normal e_AX, terrain z faces pay the sqrt)
template <int D, int N, int AX>
__device__ __forceinline__ void face_nplus(const GeoConst& gc, const ElemGeo<D>& g, int side, int c,
                                           const Tab<N>& TS, double omh_edge, const double* dh,
                                           double n[D], double& ws) {
  const double fw = (D == 2) ? TS.qw[c] : TS.qw[c / N] * TS.qw[c % N];
#pragma unroll
  for (int a = 0; a < D; ++a) n[a] = 0.0;
  if constexpr (AX < D - 1) {
    const double zzv = g.s[D - 1] * omh_edge;
    const double mag = (D == 2) ? zzv : g.s[1 - AX] * zzv;
    n[AX] = 1.0;
    ws = fw * fabs(mag);
  } else {
    const double top = (D == 2) ? g.s[0] : g.s[0] * g.s[1];
    if (!gc.terrain) {
      n[D - 1] = 1.0;
      ws = fw * top;
      return;
    }
    const double decay = 1.0 - (g.lo[D - 1] + g.s[D - 1] * (double)side) * gc.inv_ztop;
    double nt[D];
    if constexpr (D == 2) {
      nt[0] = -dh[0] * g.s[0] * decay;
    } else {
      nt[0] = -g.s[1] * dh[0] * g.s[0] * decay;
      nt[1] = -g.s[0] * dh[1] * g.s[1] * decay;
    }
    nt[D - 1] = top;
    double m2 = 0.0;
#pragma unroll
    for (int a = 0; a < D; ++a) m2 += nt[a] * nt[a];
    const double mag = sqrt(m2);
    const double im = 1.0 / mag;
#pragma unroll
    for (int a = 0; a < D; ++a) n[a] = nt[a] * im;
    ws = fw * mag;
  }
}

// 1/2 ws n+ directly: the normal's magnitude cancels in ws n+ = fw |nt| nt/|nt|,
// so the flux-trace pair (which only ever uses the product) needs neither the
// square root nor the division of face_nplus -- a rounding-level change
#ifndef DG_HK_NONORM
#define DG_HK_NONORM 1
#endif
template <int D, int N, int AX>
__device__ __forceinline__ void face_half_wn(const GeoConst& gc, const ElemGeo<D>& g, int side,
                                             double fw, double omh_edge, const double* dh,
                                             double hw[D]) {
#pragma unroll
  for (int a = 0; a < D; ++a) hw[a] = 0.0;
  const double hfw = 0.5 * fw;
  if constexpr (AX < D - 1) {
    const double zzv = g.s[D - 1] * omh_edge;
    const double mag = (D == 2) ? zzv : g.s[1 - AX] * zzv;
    hw[AX] = hfw * fabs(mag);
  } else {
    const double top = (D == 2) ? g.s[0] : g.s[0] * g.s[1];
    hw[D - 1] = hfw * top;
    if (!gc.terrain) return;
    const double decay = 1.0 - (g.lo[D - 1] + g.s[D - 1] * (double)side) * gc.inv_ztop;
    if constexpr (D == 2) {
      hw[0] = hfw * (-dh[0] * g.s[0] * decay);
    } else {
      hw[0] = hfw * (-g.s[1] * dh[0] * g.s[0] * decay);
      hw[1] = hfw * (-g.s[0] * dh[1] * g.s[1] * decay);
    }
  }
}

// the contravariant metric rows of a Gauss point of the lane's column
// (geometry.py:204-238): c[bx][a] = ctrv[bx][a]; det is z-independent
template <int D, int N>
__device__ __forceinline__ void col_metric(const GeoConst& gc, const ElemGeo<D>& g, double omh,
                                           const double* dh, double qxz, double ct[D][D]) {
#pragma unroll
  for (int b = 0; b < D; ++b)
#pragma unroll
    for (int a = 0; a < D; ++a) ct[b][a] = 0.0;
  const double zz = g.s[D - 1] * omh;
  const double decay = 1.0 - (g.lo[D - 1] + g.s[D - 1] * qxz) * gc.inv_ztop;
  if constexpr (D == 2) {
    ct[0][0] = zz;
    ct[1][0] = gc.terrain ? -(dh[0] * g.s[0] * decay) : 0.0;
    ct[1][1] = g.s[0];
  } else {
    ct[0][0] = g.s[1] * zz;
    ct[1][1] = g.s[0] * zz;
    ct[2][0] = gc.terrain ? -g.s[1] * (dh[0] * g.s[0] * decay) : 0.0;
    ct[2][1] = gc.terrain ? -g.s[0] * (dh[1] * g.s[1] * decay) : 0.0;
    ct[2][2] = g.s[0] * g.s[1];
  }
}

template <int D>
__device__ __forceinline__ double col_det(const ElemGeo<D>& g, double omh) {
  double det = 1.0;
#pragma unroll
  for (int a = 0; a < D - 1; ++a) det = det * g.s[a];
  return det * (g.s[D - 1] * omh);
}

// pencil offset of lane c's pencil along axis AX, point k
template <int D, int N, int AX>
__device__ __forceinline__ int poff(int c, int k) {
  if constexpr (AX == D - 1) return coff<D, N>(c, k);
  else if constexpr (AX == 0) return xoff<D, N>(c, k);
  else return yoff<N>(c, k);
}

// the element's terrain scalars at the lane's column / face points
template <int D, int N>
struct ColData {
  double omh;          // 1 - h/z_top at the column's horizontal Gauss point
  double dh[2];        // grad h there (also the z faces' point-c values)
};

template <int D, int N>
__device__ __forceinline__ ColData<D, N> col_data(const GeoConst& gc, const double* col,
                                                  const ElemGeo<D>& g, int c, bool act) {
  ColData<D, N> cd;
  cd.omh = 1.0;
  cd.dh[0] = cd.dh[1] = 0.0;
  if (gc.terrain && act) {
    constexpr int NQH = ipow(N, D - 1);
    const double* colp = col + (long long)g.col * gc.col_stride;
    cd.omh = colp[c];
#pragma unroll
    for (int a = 0; a < D - 1; ++a) cd.dh[a] = colp[NQH * (1 + a) + c];
  }
  return cd;
}

// 1 - h_edge/z_top along vertical face (AX, side) at the lane's point
template <int D, int N>
__device__ __forceinline__ double edge_omh(const GeoConst& gc, const double* col,
                                          const ElemGeo<D>& g, int f, int c, bool act) {
  if (!(gc.terrain && act)) return 1.0;
  constexpr int NQH = ipow(N, D - 1), NE = ipow(N, D - 2);
  return col[(long long)g.col * gc.col_stride + NQH * D + f * NE + ((D == 2) ? 0 : c / N)];
}

// ---------------------------------------------------------------------- H1
// 64-byte element records of the pipelined kernels (hk_elem_records):
// int32 nbr[2d] | uint8 kind[2d] at byte 24 | int32 elem row (level,
// origin[d], column) at byte 32
constexpr int REC_INTS = 16;

// One element's H1 on lane c (see the file comment).  Inputs: the lane's
// nodal x column (xcol[k], k < n), the neighbours' raw face nodes staged at
// FG[f n^(d-1) + c] (0 where there is no interior neighbour), the own h
// traces hf(f) = hrow[f n^(d-1)], the element's face records, geometry and
// column row (terrain).  Writes V, psi (+ pin scatter, + trV for elements
// with a coarse face).
template <int D, int N, bool AS = false>
__device__ __forceinline__ void hgrad_body(const KParams<N>& P, const Tab<N>& TS, int c, bool act,
                                           long long e, const uint8_t (&kf)[2 * D],
                                           const int (&nf)[2 * D], const ElemGeo<D>& g,
                                           const double* colrow, const double* xcol,
                                           const double* hrow, double* X, double* FG, double* HW,
                                           int team, unsigned long long* tbar = nullptr) {
  using HL = HLayout<D, N>;
  constexpr int NC = HL::NC, NF = HL::NF, TSZ = HL::TSZ;
  constexpr int NQH = ipow(N, D - 1), NE = ipow(N, D - 2);
  const Tab<N>& TC = P.tab;
  const MeshDev& mesh = P.mesh;
  ColData<D, N> cd;
  cd.omh = 1.0;
  cd.dh[0] = cd.dh[1] = 0.0;
  if (P.gc.terrain && act) {
    cd.omh = colrow[c];
#pragma unroll
    for (int a = 0; a < D - 1; ++a) cd.dh[a] = colrow[NQH * (1 + a) + c];
  }
  // 1 - h_edge/z_top of the vertical faces, loaded with the column data
  double oedge[2 * (D - 1)];
#pragma unroll
  for (int f = 0; f < 2 * (D - 1); ++f)
    oedge[f] = (P.gc.terrain && act) ? colrow[NQH * D + f * NE + ((D == 2) ? 0 : c / N)] : 1.0;
  auto edge = [&](int f) -> double { return oedge[f < 2 * (D - 1) ? f : 0]; };
  // ---- p = alpha x to the Gauss points (z in registers, y / x via the tile)
  {
    double col[N], q[N];
#pragma unroll
    for (int k = 0; k < N; ++k) col[k] = P.alpha * xcol[k];
    mat_apply<N, false>(TC.B, col, q);
#pragma unroll
    for (int k = 0; k < N; ++k) X[coff<D, N>(c, k)] = q[k];
  }
  esync<HL::TPE>(team);
  if constexpr (D == 3) {
    double v[N], o[N];
#pragma unroll
    for (int jj = 0; jj < N; ++jj) v[jj] = X[yoff<N>(c, jj)];
    mat_apply<N, false>(TC.B, v, o);
#pragma unroll
    for (int jj = 0; jj < N; ++jj) X[yoff<N>(c, jj)] = o[jj];
    esync<HL::TPE>(team);
  }
  {
    double v[N], o[N];
#pragma unroll
    for (int ii = 0; ii < N; ++ii) v[ii] = X[xoff<D, N>(c, ii)];
    mat_apply<N, false>(TC.B, v, o);
#pragma unroll
    for (int ii = 0; ii < N; ++ii) X[xoff<D, N>(c, ii)] = o[ii];
  }
  if constexpr (AS) {
    // the staged face nodes / h traces (cp.async) have landed, for every lane
    asm volatile("cp.async.wait_group 0;\n" ::: "memory");
    esync<HL::TPE>(team);
    // ... and the CTA's 1D tables (first read by the passes below; waiting
    // here instead of before the own-column passes keeps the CTA's warps
    // from meeting at a barrier right after their first-level loads)
    if (tbar != nullptr) tab_bulk_wait(tbar);
  }
  // ---- neighbour traces at face point c: tangential passes over the staged
  // face nodes (B, or the mortar halves for a fine leaf's coarse parent)
  const int fa = (D == 2) ? c : c / N;
  const int fb = (D == 2) ? 0 : c % N;
  double tn[NF];
#pragma unroll
  for (int f = 0; f < NF; ++f) {
    const int kd = kf[f] & 15;
    const int sf = (kf[f] >> 4) & 3;
    const double* M0 = (kd == KIND_FINE) ? &TS.half[sf & 1][0][0] : &TS.B[0][0];
    double t = 0.0;
    if constexpr (D == 2) {
#pragma unroll
      for (int j = 0; j < N; ++j) t = fma(M0[fa * N + j], FG[f * NC + j], t);
    } else {
#pragma unroll
      for (int j = 0; j < N; ++j) t = fma(M0[fa * N + j], FG[f * NC + j * N + fb], t);
    }
    tn[f] = t;
  }
  if constexpr (D == 3) {
    esync<HL::TPE>(team);
#pragma unroll
    for (int f = 0; f < NF; ++f) FG[f * NC + c] = tn[f];
    esync<HL::TPE>(team);
#pragma unroll
    for (int f = 0; f < NF; ++f) {
      const int kd = kf[f] & 15;
      const int sf = (kf[f] >> 4) & 3;
      const double* M1 = (kd == KIND_FINE) ? &TS.half[(sf >> 1) & 1][0][0] : &TS.B[0][0];
      double t = 0.0;
#pragma unroll
      for (int j = 0; j < N; ++j) t = fma(M1[fb * N + j], FG[f * NC + fa * N + j], t);
      tn[f] = t;
    }
  }
  esync<HL::TPE>(team);  // the tile holds p at the Gauss points of every lane
  // ---- face fluxes  sg 1/2 ws n+ (p_own + p_x): p_x = neighbour (interior),
  // p_own (wall), 0 (far field, homogeneous); coarse side precomputed
  double flv[2 * (D - 1)];  // vertical faces: the AX component only
  double flz[2][D];         // z faces
  const double wface = (D == 2) ? TS.qw[c] : TS.qw[c / N] * TS.qw[c % N];  // face point weight
  auto face = [&](auto ax_c, auto side_c) {
    constexpr int AX = decltype(ax_c)::value;
    constexpr int side = decltype(side_c)::value;
    constexpr int f = 2 * AX + side;
    const int kd = kf[f] & 15;
    double to = 0.0;
#pragma unroll
    for (int k = 0; k < N; ++k) to = fma(TC.lift[side][k], X[poff<D, N, AX>(c, k)], to);
    double fl[D];
    double hw[D];
#pragma unroll
    for (int a = 0; a < D; ++a) hw[a] = 0.0;
    if (kd == KIND_COARSE || !act) {
      const bool cf = act && mesh.cflux != nullptr;
#pragma unroll
      for (int a = 0; a < D; ++a) fl[a] = cf ? mesh.cflux[((long long)nf[f] * D + a) * NC + c] : 0.0;
    } else {
#if DG_HK_NONORM
      face_half_wn<D, N, AX>(P.gc, g, side, wface, (AX < D - 1) ? edge(f) : 1.0, cd.dh, hw);
#else
      double n[D], ws;
      face_nplus<D, N, AX>(P.gc, g, side, c, TS, (AX < D - 1) ? edge(f) : 1.0, cd.dh, n, ws);
#pragma unroll
      for (int a = 0; a < D; ++a) hw[a] = (0.5 * ws) * n[a];
#endif
      const double px = (kd == KIND_WALL) ? to : (kd == KIND_FARFIELD ? 0.0 : P.alpha * tn[f]);
      const double ph = to + px;
      const double sg = side ? 1.0 : -1.0;
#pragma unroll
      for (int a = 0; a < D; ++a) fl[a] = sg * (hw[a] * ph);
    }
    // (a wall's mirrored ghost cancels the div(hV) flux: psi = 0 there, so
    // H2 sums psi + pin uniformly over conforming, wall and far-field faces)
    const double keep = (kd == KIND_WALL) ? 0.0 : 1.0;
    if constexpr (AX < D - 1) {
      flv[f] = fl[AX];
      HW[f * NC + c] = keep * hw[AX];
    } else {
#pragma unroll
      for (int a = 0; a < D; ++a) {
        flz[side][a] = fl[a];
        HW[(2 * (D - 1) + side * D + a) * NC + c] = keep * hw[a];
      }
    }
  };
  face(std::integral_constant<int, 0>{}, std::integral_constant<int, 0>{});
  face(std::integral_constant<int, 0>{}, std::integral_constant<int, 1>{});
  if constexpr (D == 3) {
    face(std::integral_constant<int, 1>{}, std::integral_constant<int, 0>{});
    face(std::integral_constant<int, 1>{}, std::integral_constant<int, 1>{});
  }
  face(std::integral_constant<int, D - 1>{}, std::integral_constant<int, 0>{});
  face(std::integral_constant<int, D - 1>{}, std::integral_constant<int, 1>{});

  // ---- volume: G_bx,k = ctrv[bx][k] p wq; bx < d-1 through the tile
  double Zc[D][N];
  const double det = col_det<D>(g, cd.omh);
  const double wcol = wface;
  {
    double Gz[D][N];
#pragma unroll
    for (int kz = 0; kz < N; ++kz) {
      double ct[D][D];
      col_metric<D, N>(P.gc, g, cd.omh, cd.dh, TC.qx[kz], ct);
      const double wq = wcol * TC.qw[kz];
      const double p = X[coff<D, N>(c, kz)];
      X[coff<D, N>(c, kz)] = (p * ct[0][0]) * wq;
      if constexpr (D == 3) X[TSZ + coff<D, N>(c, kz)] = (p * ct[1][1]) * wq;
#pragma unroll
      for (int k = 0; k < D; ++k) Gz[k][kz] = (p * ct[D - 1][k]) * wq;
    }
#pragma unroll
    for (int k = 0; k < D; ++k) {
      mat_apply<N, true>(TC.Dhat, Gz[k], Zc[k]);
#pragma unroll
      for (int kz = 0; kz < N; ++kz)
        Zc[k][kz] = TC.lift[0][kz] * flz[0][k] + TC.lift[1][kz] * flz[1][k] - Zc[k][kz];
    }
  }
  esync<HL::TPE>(team);
  {
    double v[N], o[N];
#pragma unroll
    for (int ii = 0; ii < N; ++ii) v[ii] = X[xoff<D, N>(c, ii)];
    mat_apply<N, true>(TC.Dhat, v, o);
#pragma unroll
    for (int ii = 0; ii < N; ++ii)
      X[xoff<D, N>(c, ii)] = TC.lift[0][ii] * flv[0] + TC.lift[1][ii] * flv[1] - o[ii];
    if constexpr (D == 3) {
#pragma unroll
      for (int jj = 0; jj < N; ++jj) v[jj] = X[TSZ + yoff<N>(c, jj)];
      mat_apply<N, true>(TC.Dhat, v, o);
#pragma unroll
      for (int jj = 0; jj < N; ++jj)
        X[TSZ + yoff<N>(c, jj)] = TC.lift[0][jj] * flv[2] + TC.lift[1][jj] * flv[3] - o[jj];
    }
  }
  esync<HL::TPE>(team);
#pragma unroll
  for (int kz = 0; kz < N; ++kz) {
    Zc[0][kz] += X[coff<D, N>(c, kz)];
    if constexpr (D == 3) Zc[1][kz] += X[TSZ + coff<D, N>(c, kz)];
  }
  // ---- epilogue: V = coef Z / (w det) at the Gauss points
  double iwh = 1.0 / det;
  if constexpr (D == 3) iwh *= TS.iqw[c / N] * TS.iqw[c % N];
  else iwh *= TS.iqw[c];
  double Vg[D][N];
#pragma unroll
  for (int k = 0; k < D; ++k)
#pragma unroll
    for (int kz = 0; kz < N; ++kz) Vg[k][kz] = P.coef * (Zc[k][kz] * (iwh * TC.iqw[kz]));
  if (act) {
#pragma unroll
    for (int k = 0; k < D; ++k) {
      double* out = P.out.p + e * P.out.estride + (long long)k * P.out.cstride + c * N;
#pragma unroll
      for (int kz = 0; kz < N; ++kz) out[kz] = Vg[k][kz];
    }
  }
  // ---- face traces of V and psi = 1/2 ws h (V . n+)
  double tz[2][D];
#pragma unroll
  for (int side = 0; side < 2; ++side)
#pragma unroll
    for (int k = 0; k < D; ++k) {
      double t = 0.0;
#pragma unroll
      for (int kz = 0; kz < N; ++kz) t = fma(TC.lift[side][kz], Vg[k][kz], t);
      tz[side][k] = t;
    }
  esync<HL::TPE>(team);  // every lane is done with the tile
#pragma unroll
  for (int a = 0; a < D - 1; ++a)
#pragma unroll
    for (int kz = 0; kz < N; ++kz) X[a * TSZ + coff<D, N>(c, kz)] = Vg[a][kz];
  esync<HL::TPE>(team);
  double tv[2 * (D - 1)];
#pragma unroll
  for (int a = 0; a < D - 1; ++a)
#pragma unroll
    for (int side = 0; side < 2; ++side) {
      double t = 0.0;
#pragma unroll
      for (int p = 0; p < N; ++p) {
        const int off = (a == 0) ? xoff<D, N>(c, p) : yoff<N>(c, p);
        t = fma(TC.lift[side][p], X[a * TSZ + off], t);
      }
      tv[2 * a + side] = t;
    }
  if (act) {
    double* ps = P.psi_out + e * (NF * NC);
    double pv[NF];
#pragma unroll
    for (int f = 0; f < 2 * (D - 1); ++f) pv[f] = hrow[f * NC] * (HW[f * NC + c] * tv[f]);
#pragma unroll
    for (int side = 0; side < 2; ++side) {
      double vn = 0.0;
#pragma unroll
      for (int a = 0; a < D; ++a) vn = fma(HW[(2 * (D - 1) + side * D + a) * NC + c], tz[side][a], vn);
      pv[2 * (D - 1) + side] = hrow[(2 * (D - 1) + side) * NC] * vn;
    }
#pragma unroll
    for (int f = 0; f < NF; ++f) {
      ps[f * NC + c] = pv[f];
      // the conforming neighbour's incoming slot (its face f ^ 1): H2 then
      // reads only its own contiguous rows (ghost neighbours: hk_pin_fixup
      // after the halo exchange)
      if (P.pin_out != nullptr && (kf[f] & 15) == KIND_CONF && nf[f] < mesh.n_el)
        P.pin_out[(long long)nf[f] * (NF * NC) + (f ^ 1) * NC + c] = pv[f];
    }
    bool coarse = false;
#pragma unroll
    for (int f = 0; f < NF; ++f) coarse |= (kf[f] & 15) == KIND_COARSE;
    if (coarse && P.tr_out != nullptr) {
      // the mortar of the fine neighbours (hdiv) and the coarse-side fluxes
      // (coarse_kernel) read this element's V traces
      constexpr int TSL = tr_slots<D>() * NC;
      double* tr = P.tr_out + e * TSL;
#pragma unroll
      for (int f = 0; f < 2 * (D - 1); ++f) tr[tr_slot<D>(f, f >> 1) * NC + c] = tv[f];
#pragma unroll
      for (int side = 0; side < 2; ++side)
#pragma unroll
        for (int k = 0; k < D; ++k) tr[tr_slot<D>(2 * (D - 1) + side, k) * NC + c] = tz[side][k];
    }
  }
}

template <int D, int N>
__global__ void __launch_bounds__(HLayout<D, N>::THREADS,
                                  HLayout<D, N>::TPE == 32 ? DG_HK1_MINB : 3)
hgrad_kernel(const __grid_constant__ KParams<N> P) {
  using HL = HLayout<D, N>;
  constexpr int NC = HL::NC, EPW = HL::EPW, NF = HL::NF, TSZ = HL::TSZ;
  extern __shared__ __align__(16) double smem[];
  __shared__ unsigned long long tbar;
  tab_bulk_issue(smem, P.tab_g, HL::TABD * 8, &tbar);
  pdl_trigger();
  pdl_wait();  // (programmatic dependent launch, small problems: dg_common.cuh)
#if DG_HK1_ASYNC
  __syncthreads();  // the table barrier is initialised (waited for in hgrad_body)
#endif
  const Tab<N>& TS = *reinterpret_cast<const Tab<N>*>(smem);
  const MeshDev& mesh = P.mesh;
  const int lane = threadIdx.x % HL::TPE, wid = threadIdx.x / HL::TPE;  // team lane, team
  const int eiw = lane / NC, c = lane - eiw * NC;
  const bool slot_ok = eiw < EPW;
  const long long e = ((long long)blockIdx.x * HL::WPB + wid) * EPW + eiw;
  const bool act = slot_ok && e < mesh.n_el;
  const long long es = act ? e : 0;
  double* X = smem + HL::TABP + (wid * HL::NSLOT + (slot_ok ? eiw : EPW)) * HL::GSLOT;
  double* FG = X + HL::KX * TSZ;
  double* HW = FG + NF * NC;
  // Every first-level load (own column, own h traces, element row, face
  // records) is issued -- as volatile asm, in this order -- before the first
  // use of any of them, so the in-order warp waits ONE memory latency.  Left
  // to the scheduler, the face-kind compares were hoisted above the
  // element-row and own-column loads and each chain paid its own latency
  // (ncu, per source line: three long-scoreboard waits of ~8 % of the warp
  // time each).  Inactive lanes load element 0 and discard it.
  uint8_t kf[NF];
  int nf[NF];
  int er[2 + D];
  double xc[N];
#if DG_HK1_ASYNC
  double* HR = HW + HL::NHW * NC;
#pragma unroll
  for (int k = 0; k < N; ++k) xc[k] = ldg_f64_ordered(P.in.p + es * P.in.estride + c * N + k);
#pragma unroll
  for (int f = 0; f < NF; ++f) cp_async8(&HR[f * NC + c], P.trH + es * (NF * NC) + f * NC + c);
#pragma unroll
  for (int k = 0; k < 2 + D; ++k) er[k] = ldg_s32_ordered(mesh.elem + es * (2 + D) + k);
#pragma unroll
  for (int f = 0; f < NF; ++f) nf[f] = ldg_s32_ordered(mesh.nbr + es * NF + f);
#pragma unroll
  for (int f = 0; f < NF; ++f) kf[f] = ldg_u8_ordered(mesh.kind + es * NF + f);
  // (ptxas does not sink loads below a warp barrier: without it the
  // element-row and own-column loads were scheduled after the first wait)
  __syncwarp();
#pragma unroll
  for (int f = 0; f < NF; ++f) {
    if (!act) {
      kf[f] = (uint8_t)KIND_WALL;
      nf[f] = 0;
    }
  }
#pragma unroll
  for (int k = 0; k < N; ++k) xc[k] = act ? xc[k] : 0.0;
#else
#pragma unroll
  for (int f = 0; f < NF; ++f) {
    kf[f] = act ? mesh.kind[es * NF + f] : (uint8_t)KIND_WALL;
    nf[f] = act ? mesh.nbr[es * NF + f] : 0;
  }
#pragma unroll
  for (int k = 0; k < 2 + D; ++k) er[k] = mesh.elem[es * (2 + D) + k];
#pragma unroll
  for (int k = 0; k < N; ++k) xc[k] = act ? P.in.p[es * P.in.estride + c * N + k] : 0.0;
#endif
#if DG_HK1_ASYNC
#pragma unroll
  for (int f = 0; f < NF; ++f) {
    const int kd = kf[f] & 15;
    const bool inter = act && (kd == KIND_CONF || kd == KIND_FINE);
    if (inter)
      cp_async8(&FG[f * NC + c],
                P.in.p + (long long)nf[f] * P.in.estride + nbr_face_node<D, N>(f >> 1, f & 1, c));
    else
      FG[f * NC + c] = 0.0;
  }
  asm volatile("cp.async.commit_group;\n" ::: "memory");
  const double* hrow = HR + c;
#else
#pragma unroll
  for (int f = 0; f < NF; ++f) {
    const int kd = kf[f] & 15;
    const bool inter = act && (kd == KIND_CONF || kd == KIND_FINE);
    FG[f * NC + c] =
        inter ? P.in.p[(long long)nf[f] * P.in.estride + nbr_face_node<D, N>(f >> 1, f & 1, c)]
              : 0.0;
  }
  const double* hrow = P.trH + es * (NF * NC) + c;
#endif
  const ElemGeo<D> g = geo_from_row<D>(er, P.gc);
  const double* colrow = P.gc.terrain ? mesh.col + (long long)g.col * P.gc.col_stride : nullptr;
#if DG_HK1_ASYNC
  hgrad_body<D, N, true>(P, TS, c, act, e, kf, nf, g, colrow, xc, hrow, X, FG, HW, wid, &tbar);
#else
  __syncthreads();  // the table barrier is initialised
  tab_bulk_wait(&tbar);
  hgrad_body<D, N, false>(P, TS, c, act, e, kf, nf, g, colrow, xc, hrow, X, FG, HW, wid);
#endif
}

// H1, pipelined (hgrad2_kernel): persistent warps over strided element
// groups as hdiv2_kernel.  Per group a two-stage ring holds, by
// cp.async.bulk, the nodal x blocks, the own h-trace rows and the 64-byte
// element records; one group AHEAD, as soon as its records have landed, the
// lanes stage the neighbours' face nodes (cp.async, 8 B each) and the first
// lane of each element its column row (cp.async.bulk, terrain) -- so every
// load of a group is in flight while the previous group is computed.
template <int D, int N>
struct H1Pipe {
  using HL = HLayout<D, N>;
  static constexpr int NP = HL::NP, NC = HL::NC, NF = HL::NF, EPW = HL::EPW;
  static constexpr int COLS = 2 * ((ipow(N, D - 1) * D + 2 * (D - 1) * ipow(N, D - 2) + 1) / 2);
  static constexpr bool OK = HL::OK && HL::TPE == 32 && (NP % 2 == 0) && ((NF * NC) % 2 == 0);
  static constexpr int OX = 0;                      // nodal x (bulk)
  static constexpr int OH = OX + EPW * NP;          // own h traces (bulk)
  static constexpr int OR = OH + EPW * NF * NC;     // records (bulk), 8 doubles each
  static constexpr int BULK = OR + EPW * 8;
  static constexpr int OF = BULK;                   // neighbour face nodes (cp.async),
                                                    // one slot per lane group (+ padding)
  static constexpr int OC = OF + HL::NSLOT * NF * NC;  // column rows (bulk, terrain)
  static constexpr int STG = OC + EPW * COLS;
  static constexpr int ESLOT = HL::odd(HL::KX * HL::TSZ + HL::NHW * NC);  // tile + HW
  static constexpr int WREG = ((2 * STG + HL::NSLOT * ESLOT) + 1) & ~1;
  static constexpr int WPB = 4;
  static constexpr size_t SMEM = (size_t)(HL::TABP + WPB * WREG) * sizeof(double);
};

#ifndef DG_HK1P_MINB
#define DG_HK1P_MINB 3
#endif

__device__ __forceinline__ void cp_async8_raw(double* dst, const double* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(smem_u32(dst)), "l"(src)
               : "memory");
}

template <int D, int N>
__global__ void __launch_bounds__(128, DG_HK1P_MINB)
hgrad2_kernel(const __grid_constant__ KParams<N> P) {
  using HL = HLayout<D, N>;
  using PL = H1Pipe<D, N>;
  constexpr int NC = HL::NC, EPW = HL::EPW, NF = HL::NF, TSZ = HL::TSZ, NP = HL::NP;
  extern __shared__ __align__(16) double smem[];
  __shared__ unsigned long long tbar;
  __shared__ unsigned long long sbar[PL::WPB][2], cbar[PL::WPB][2];
  tab_bulk_issue(smem, P.tab_g, HL::TABD * 8, &tbar);
  const Tab<N>& TS = *reinterpret_cast<const Tab<N>*>(smem);
  const MeshDev& mesh = P.mesh;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int eiw = lane / NC, c = lane - eiw * NC;
  const bool slot_ok = eiw < EPW;
  double* W = smem + HL::TABP + wid * PL::WREG;
  double* ES = W + 2 * PL::STG + (slot_ok ? eiw : EPW) * PL::ESLOT;
  double* X = ES;
  double* HW = ES + HL::KX * TSZ;
  const unsigned bar[2] = {smem_u32(&sbar[wid][0]), smem_u32(&sbar[wid][1])};
  const unsigned cb[2] = {smem_u32(&cbar[wid][0]), smem_u32(&cbar[wid][1])};
  const long long ngroups = ((long long)mesh.n_el + EPW - 1) / EPW;
  const long long gw = (long long)blockIdx.x * PL::WPB + wid;
  const long long GW = (long long)gridDim.x * PL::WPB;
  const bool terr = P.gc.terrain != 0;

  auto issue = [&](long long g, int s) {  // lane 0: the bulk part of group g
    const long long e0 = g * EPW;
    const int ne = (int)min((long long)EPW, (long long)mesh.n_el - e0);
    double* st = W + s * PL::STG;
    const unsigned bytes = 8u * ne * (NP + NF * NC + 8);
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(bar[s]),
                 "r"(bytes)
                 : "memory");
    bulk_g2s(st + PL::OX, P.in.p + e0 * P.in.estride, 8u * ne * NP, bar[s]);
    bulk_g2s(st + PL::OH, P.trH + e0 * (NF * NC), 8u * ne * NF * NC, bar[s]);
    bulk_g2s(st + PL::OR, P.frec + e0 * REC_INTS, 64u * ne, bar[s]);
  };
  // all lanes: the lookahead part of group g (its records landed): the
  // neighbours' face nodes and (terrain) the column rows
  auto lookahead = [&](long long g, int s) {
    double* st = W + s * PL::STG;
    const long long e = g * EPW + eiw;
    const bool act = slot_ok && e < mesh.n_el;
    const int esl = act ? eiw : 0;
    const int* rec = reinterpret_cast<const int*>(st + PL::OR) + esl * REC_INTS;
    const uint8_t* rk = reinterpret_cast<const uint8_t*>(rec + 6);
    double* fg = st + PL::OF + (slot_ok ? eiw : EPW) * (NF * NC);
#pragma unroll
    for (int f = 0; f < NF; ++f) {
      const int kd = rk[f] & 15;
      const bool inter = act && (kd == KIND_CONF || kd == KIND_FINE);
      if (inter)
        cp_async8_raw(fg + f * NC + c,
                      P.in.p + (long long)rec[f] * P.in.estride + nbr_face_node<D, N>(f >> 1, f & 1, c));
      else
        fg[f * NC + c] = 0.0;
    }
    asm volatile("cp.async.commit_group;\n" ::: "memory");
    if (terr) {
      // one column row per element, by the element's first lane
      const int ne = (int)min((long long)EPW, (long long)mesh.n_el - g * EPW);
      if (lane == 0) {
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(cb[s]),
                     "r"(8u * ne * PL::COLS)
                     : "memory");
      }
      __syncwarp();
      if (act && c == 0) {
        const int colid = rec[8 + 1 + D];
        bulk_g2s(st + PL::OC + eiw * PL::COLS, mesh.col + (long long)colid * P.gc.col_stride,
                 8u * PL::COLS, cb[s]);
      }
    }
  };

  if (lane == 0) {
    for (int s = 0; s < 2; ++s) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(bar[s]) : "memory");
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(cb[s]) : "memory");
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    if (gw < ngroups) issue(gw, 0);
    if (gw + GW < ngroups) issue(gw + GW, 1);
  }
  __syncthreads();  // barriers initialised
  if (gw < ngroups) {
    mbar_wait(bar[0], 0);
    lookahead(gw, 0);
  }
  tab_bulk_wait(&tbar);

  int k = 0;
  for (long long g = gw; g < ngroups; g += GW, ++k) {
    const int s = k & 1;
    const unsigned par = (unsigned)((k >> 1) & 1);
    mbar_wait(bar[s], par);  // (already complete: waited before the lookahead)
    // this group's lookahead copies, then the next group's lookahead
    asm volatile("cp.async.wait_group 0;\n" ::: "memory");
    if (terr) mbar_wait(cb[s], par);
    __syncwarp();
    if (g + GW < ngroups) {
      const int s1 = s ^ 1;
      mbar_wait(bar[s1], (unsigned)(((k + 1) >> 1) & 1));
      lookahead(g + GW, s1);
    }
    double* st = W + s * PL::STG;
    const long long e = g * EPW + eiw;
    const bool act = slot_ok && e < mesh.n_el;
    const int esl = act ? eiw : 0;
    const int* rec = reinterpret_cast<const int*>(st + PL::OR) + esl * REC_INTS;
    const uint8_t* rk = reinterpret_cast<const uint8_t*>(rec + 6);
    uint8_t kf[NF];
    int nf[NF];
#pragma unroll
    for (int f = 0; f < NF; ++f) {
      kf[f] = act ? rk[f] : (uint8_t)KIND_WALL;
      nf[f] = rec[f];
    }
    const ElemGeo<D> g3 = geo_from_row<D>(rec + 8, P.gc);
    hgrad_body<D, N>(P, TS, c, act, e, kf, nf, g3, st + PL::OC + esl * PL::COLS,
                     st + PL::OX + esl * NP + c * N, st + PL::OH + esl * (NF * NC) + c, X,
                     st + PL::OF + (slot_ok ? eiw : EPW) * (NF * NC), HW, wid);
    __syncwarp();  // every lane is done with this stage
    if (lane == 0 && g + 2 * GW < ngroups) issue(g + 2 * GW, s);
  }
  asm volatile("cp.async.wait_group 0;\n" ::: "memory");
}

// 64-byte element records of the pipelined kernels (see REC_INTS)
template <int D>
__global__ void hk_elem_records(const int* __restrict__ nbr, const uint8_t* __restrict__ kind,
                                const int* __restrict__ elem, int n, int* __restrict__ rec) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= n) return;
  int r[REC_INTS];
  for (int i = 0; i < REC_INTS; ++i) r[i] = 0;
  for (int f = 0; f < 2 * D; ++f) r[f] = nbr[(long long)e * 2 * D + f];
  uint8_t* kb = reinterpret_cast<uint8_t*>(r + 6);
  for (int f = 0; f < 2 * D; ++f) kb[f] = kind[(long long)e * 2 * D + f];
  for (int i = 0; i < 2 + D; ++i) r[8 + i] = elem[(long long)e * (2 + D) + i];
  for (int i = 0; i < REC_INTS; ++i) rec[(long long)e * REC_INTS + i] = r[i];
}

// ---------------------------------------------------------------------- H2
template <int D, int N>
__global__ void __launch_bounds__(HLayout<D, N>::THREADS,
                                  HLayout<D, N>::TPE == 32 ? DG_HK2_MINB : 3)
hdiv_kernel(const __grid_constant__ KParams<N> P) {
  using HL = HLayout<D, N>;
  constexpr int NC = HL::NC, EPW = HL::EPW, NF = HL::NF, TSZ = HL::TSZ;
  extern __shared__ __align__(16) double smem[];
  __shared__ unsigned long long tbar;
  tab_bulk_issue(smem, P.tab_g, HL::TABD * 8, &tbar);
  pdl_trigger();
  pdl_wait();  // (programmatic dependent launch, small problems)
  const Tab<N>& TS = *reinterpret_cast<const Tab<N>*>(smem);
  const Tab<N>& TC = P.tab;
  const MeshDev& mesh = P.mesh;
  const int lane = threadIdx.x % HL::TPE, wid = threadIdx.x / HL::TPE;  // team lane, team
  const int eiw = lane / NC, c = lane - eiw * NC;
  const bool slot_ok = eiw < EPW;
  const long long e = ((long long)blockIdx.x * HL::WPB + wid) * EPW + eiw;
  const bool act = slot_ok && e < mesh.n_el;
  const long long es = act ? e : 0;
  double* X = smem + HL::TABP + (wid * HL::NSLOT + (slot_ok ? eiw : EPW)) * HL::DSLOT;

  uint8_t kf[NF];
  int nf[NF];
#pragma unroll
  for (int f = 0; f < NF; ++f) {
    kf[f] = act ? mesh.kind[es * NF + f] : (uint8_t)KIND_WALL;
    nf[f] = act ? mesh.nbr[es * NF + f] : 0;
  }
  // face fluxes first (their loads are the dependent ones)
  double fl[NF];
  {
    const double* ps = P.psi + es * (NF * NC) + c;
#pragma unroll
    for (int f = 0; f < NF; ++f) {
      const int kd = kf[f] & 15;
      const double po = act ? ps[f * NC] : 0.0;
      const double pn = (act && kd == KIND_CONF)
                            ? P.psi[(long long)nf[f] * (NF * NC) + (f ^ 1) * NC + c] : 0.0;
      const double sg = (f & 1) ? 1.0 : -1.0;
      double v = 0.0;
      if (kd == KIND_CONF) v = sg * (po + pn);
      else if (kd == KIND_FARFIELD || kd == KIND_FINE) v = sg * po;  // (fine: + the mortar part)
      else if (kd == KIND_COARSE && mesh.cflux != nullptr && act)
        v = mesh.cflux[(long long)nf[f] * NC + c];
      fl[f] = act ? v : 0.0;
    }
  }
  double Vq[D][N], hq[N], bv[N];
#pragma unroll
  for (int a = 0; a < D; ++a)
#pragma unroll
    for (int kz = 0; kz < N; ++kz)
      Vq[a][kz] = act ? P.in.p[es * P.in.estride + (long long)a * P.in.cstride + c * N + kz] : 0.0;
#pragma unroll
  for (int kz = 0; kz < N; ++kz) hq[kz] = act ? P.inH.p[es * P.inH.estride + c * N + kz] : 0.0;
#pragma unroll
  for (int ii = 0; ii < N; ++ii) {
    const int node = (D == 3) ? ii * N * N + c : ii * N + c;
    bv[ii] = (act && P.has_base) ? P.base.p[es * P.base.estride + node] : 0.0;
  }
  const ElemGeo<D> g = elem_geo<D>(mesh.elem, P.gc, es);
  const ColData<D, N> cd = col_data<D, N>(P.gc, mesh.col, g, c, act);
  __syncthreads();  // the table barrier is initialised
  tab_bulk_wait(&tbar);

  // ---- fine side of hanging faces: the coarse parent's V / h traces at its
  // face Gauss points through halfq (x) halfq, flux with the own metric
  const int fa = (D == 2) ? c : c / N;
  const int fb = (D == 2) ? 0 : c % N;
  auto fine_face = [&](auto ax_c, auto side_c) {
    constexpr int AX = decltype(ax_c)::value;
    constexpr int side = decltype(side_c)::value;
    constexpr int f = 2 * AX + side;
    const int kd = kf[f] & 15;
    const bool fine = act && kd == KIND_FINE;
    if (!eany<HL::TPE>(fine, wid)) return;
    constexpr int FC = (AX < D - 1) ? 2 : D + 1;  // (V_AX, h) or (V, h)
    constexpr int TSL = tr_slots<D>() * NC, THL = 2 * D * NC;
    const long long pe = nf[f];
#pragma unroll
    for (int r = 0; r < FC; ++r) {
      double v = 0.0;
      if (fine) {
        const bool isv = r < FC - 1;
        const int comp = (AX < D - 1) ? AX : r;
        v = isv ? P.trV[pe * TSL + tr_slot<D>(f ^ 1, comp) * NC + c]
                : P.trH[pe * THL + (f ^ 1) * NC + c];
      }
      X[r * NC + c] = v;
    }
    esync<HL::TPE>(wid);
    const int sf = (kf[f] >> 4) & 3;
    const double* Mq0 = &TS.halfq[sf & 1][0][0];
    const double* Mq1 = &TS.halfq[(sf >> 1) & 1][0][0];
    double tr[FC];
#pragma unroll
    for (int r = 0; r < FC; ++r) {
      double t = 0.0;
      if constexpr (D == 2) {
#pragma unroll
        for (int j = 0; j < N; ++j) t = fma(Mq0[fa * N + j], X[r * NC + j], t);
      } else {
#pragma unroll
        for (int j = 0; j < N; ++j) t = fma(Mq0[fa * N + j], X[r * NC + j * N + fb], t);
      }
      tr[r] = t;
    }
    if constexpr (D == 3) {
      esync<HL::TPE>(wid);
#pragma unroll
      for (int r = 0; r < FC; ++r) X[r * NC + c] = tr[r];
      esync<HL::TPE>(wid);
#pragma unroll
      for (int r = 0; r < FC; ++r) {
        double t = 0.0;
#pragma unroll
        for (int j = 0; j < N; ++j) t = fma(Mq1[fb * N + j], X[r * NC + fa * N + j], t);
        tr[r] = t;
      }
    }
    esync<HL::TPE>(wid);  // the staging area is reused by the next face
    if (fine) {
      double n[D], ws;
      const double oe = (AX < D - 1) ? edge_omh<D, N>(P.gc, mesh.col, g, f, c, act) : 1.0;
      face_nplus<D, N, AX>(P.gc, g, side, c, TS, oe, cd.dh, n, ws);
      double vn;
      if constexpr (AX < D - 1) {
        vn = tr[0] * n[AX];
      } else {
        vn = 0.0;
#pragma unroll
        for (int a = 0; a < D; ++a) vn = fma(tr[a], n[a], vn);
      }
      const double sg = side ? 1.0 : -1.0;
      fl[f] += sg * ((0.5 * ws) * (tr[FC - 1] * vn));
    }
  };
  if (mesh.n_coarse > 0) {
    fine_face(std::integral_constant<int, 0>{}, std::integral_constant<int, 0>{});
    fine_face(std::integral_constant<int, 0>{}, std::integral_constant<int, 1>{});
    if constexpr (D == 3) {
      fine_face(std::integral_constant<int, 1>{}, std::integral_constant<int, 0>{});
      fine_face(std::integral_constant<int, 1>{}, std::integral_constant<int, 1>{});
    }
    fine_face(std::integral_constant<int, D - 1>{}, std::integral_constant<int, 0>{});
    fine_face(std::integral_constant<int, D - 1>{}, std::integral_constant<int, 1>{});
  }

  // ---- volume: G_bx = (sum_a ctrv[bx][a] h V_a) wq; bx < d-1 via the tile
  double Zc[N];
  const double det = col_det<D>(g, cd.omh);
  const double wcol = (D == 3) ? TS.qw[c / N] * TS.qw[c % N] : TS.qw[c];
  {
    double Gz[N];
#pragma unroll
    for (int kz = 0; kz < N; ++kz) {
      double ct[D][D];
      col_metric<D, N>(P.gc, g, cd.omh, cd.dh, TC.qx[kz], ct);
      const double wq = wcol * TC.qw[kz];
      double F[D];
#pragma unroll
      for (int a = 0; a < D; ++a) F[a] = hq[kz] * Vq[a][kz];
      X[coff<D, N>(c, kz)] = (F[0] * ct[0][0]) * wq;
      if constexpr (D == 3) X[TSZ + coff<D, N>(c, kz)] = (F[1] * ct[1][1]) * wq;
      double acc = 0.0;
#pragma unroll
      for (int a = 0; a < D; ++a) acc += F[a] * ct[D - 1][a];
      Gz[kz] = acc * wq;
    }
    mat_apply<N, true>(TC.Dhat, Gz, Zc);
    const int zf = 2 * (D - 1);
#pragma unroll
    for (int kz = 0; kz < N; ++kz)
      Zc[kz] = TC.lift[0][kz] * fl[zf] + TC.lift[1][kz] * fl[zf + 1] - Zc[kz];
  }
  esync<HL::TPE>(wid);
  {
    double v[N], o[N];
#pragma unroll
    for (int ii = 0; ii < N; ++ii) v[ii] = X[xoff<D, N>(c, ii)];
    mat_apply<N, true>(TC.Dhat, v, o);
#pragma unroll
    for (int ii = 0; ii < N; ++ii)
      X[xoff<D, N>(c, ii)] = TC.lift[0][ii] * fl[0] + TC.lift[1][ii] * fl[1] - o[ii];
    if constexpr (D == 3) {
#pragma unroll
      for (int jj = 0; jj < N; ++jj) v[jj] = X[TSZ + yoff<N>(c, jj)];
      mat_apply<N, true>(TC.Dhat, v, o);
#pragma unroll
      for (int jj = 0; jj < N; ++jj)
        X[TSZ + yoff<N>(c, jj)] = TC.lift[0][jj] * fl[2] + TC.lift[1][jj] * fl[3] - o[jj];
    }
  }
  esync<HL::TPE>(wid);
#pragma unroll
  for (int kz = 0; kz < N; ++kz) {
    Zc[kz] += X[coff<D, N>(c, kz)];
    if constexpr (D == 3) Zc[kz] += X[TSZ + coff<D, N>(c, kz)];
  }
  // ---- epilogue: y = base + coef B^-1 diag(1/(w det)) Z, + fused dots
  double iwh = 1.0 / det;
  if constexpr (D == 3) iwh *= TS.iqw[c / N] * TS.iqw[c % N];
  else iwh *= TS.iqw[c];
  {
    double t[N];
#pragma unroll
    for (int kz = 0; kz < N; ++kz) t[kz] = Zc[kz] * (iwh * TC.iqw[kz]);
    mat_apply<N, false>(TC.Binv, t, Zc);
  }
  esync<HL::TPE>(wid);
#pragma unroll
  for (int kz = 0; kz < N; ++kz) X[coff<D, N>(c, kz)] = Zc[kz];
  esync<HL::TPE>(wid);
  if constexpr (D == 3) {
    double v[N], o[N];
#pragma unroll
    for (int jj = 0; jj < N; ++jj) v[jj] = X[yoff<N>(c, jj)];
    mat_apply<N, false>(TC.Binv, v, o);
#pragma unroll
    for (int jj = 0; jj < N; ++jj) X[yoff<N>(c, jj)] = o[jj];
    esync<HL::TPE>(wid);
  }
  double wv[N], uv[N];
  {
    double v[N], o[N];
#pragma unroll
    for (int ii = 0; ii < N; ++ii) v[ii] = X[xoff<D, N>(c, ii)];
    mat_apply<N, false>(TC.Binv, v, o);
#pragma unroll
    for (int ii = 0; ii < N; ++ii) {
      const double r = __dmul_rn(P.coef, o[ii]);
      const double val = P.has_base ? __dadd_rn(bv[ii], r) : r;
      wv[ii] = act ? val : 0.0;
      uv[ii] = act ? bv[ii] : 0.0;
      if (act) {
        const int node = (D == 3) ? ii * N * N + c : ii * N + c;
        P.out.p[e * P.out.estride + node] = val;
      }
    }
  }
  if (HL::TPE == 32 && P.gs_part != nullptr) {
    // fused Gram-Schmidt dots (one-warp teams only; two-warp teams take the
    // separate dual-dot pass) (as gs_dots, dg_wkernel.cuh): every element is
    // complete here (coarse faces in flux mode)
    constexpr int AREA = HL::NSLOT * HL::DSLOT;
    static_assert(AREA >= 2 * (32 + 2), "warp area too small for the fused dots");
    const bool dual = P.gs_dual != 0;
    const int nv = P.gs_nv;
    const int nvt = dual ? 2 * (nv + 2) : nv + 1;
    double* wtot = smem + HL::TABP + wid * AREA;
    esync<HL::TPE>(wid);
    for (int c0 = 0; c0 < nvt; c0 += 16) {
      if (dual) gs_round<D, N, 2>(P, act, e, c, wv, uv, c0, nv, nvt, wtot);
      else gs_round<D, N, 1>(P, act, e, c, wv, uv, c0, nv, nvt, wtot);
    }
    __syncthreads();
    if (wid == 0) {
      const long long row = (long long)P.gs_row0 + blockIdx.x;
      for (int col = lane; col < nvt; col += 32) {
        double t = 0.0;
#pragma unroll
        for (int w = 0; w < HL::WPB; ++w) t += smem[HL::TABP + w * AREA + col];
        P.gs_part[row * nvt + col] = t;
      }
    }
  }
}

// ---------------------------------------------------------------------------
// H2, pipelined (hdiv2_kernel): persistent warps, each owning a strided
// sequence of element groups (the EPW elements of one warp); every group's
// inputs are contiguous per-element blocks -- V and h at the Gauss points,
// the own psi rows and the incoming pin rows written by the neighbours' H1,
// the base (the action's input), the 32-byte face records -- brought into a
// two-stage shared-memory ring by cp.async.bulk (TMA) issued by one lane, so
// the next group's loads are in flight while this one is computed and the
// memory parallelism no longer depends on registers or occupancy.  Same
// arithmetic as hdiv_kernel.  Even n^d only (16-byte aligned element blocks).
// DG_H2_SLIM=1: the base (the action's input) and the column rows are read
// by plain loads instead of being staged -- 4 KB less shared memory per warp,
// which lets a third CTA (12 instead of 8 warps) share an SM
#ifndef DG_H2_SLIM
#define DG_H2_SLIM 0
#endif
#ifndef DG_H2_COLDIRECT
#define DG_H2_COLDIRECT 1  // the column rows by plain loads issued at the top of the iteration
#endif
#ifndef DG_H2_FUSED_DOTS
#define DG_H2_FUSED_DOTS 0
#endif
#ifndef DG_H2_WPB
#define DG_H2_WPB 0   // 0: the most warps per SM that fit (H2Pipe::pick)
#endif
#ifndef DG_HK2P_MINB
#define DG_HK2P_MINB 2  // CTAs per SM when DG_H2_WPB forces the warps per CTA
#endif
template <int D, int N>
struct H2Pipe {
  using HL = HLayout<D, N>;
  static constexpr bool SLIM = DG_H2_SLIM != 0;
  static constexpr int NP = HL::NP, NC = HL::NC, NF = HL::NF, EPW = HL::EPW;
  static constexpr bool OK = HL::OK && HL::TPE == 32;
  static constexpr int ev(int x) { return (x + 1) & ~1; }
  // stage sub-arrays (doubles, all even offsets); the odd-n^d blocks (V, h,
  // base) are copied as their 16-byte aligned superset, shifted by 0 or 1
  static constexpr int OV = 0;
  static constexpr int OH = OV + ev(EPW * D * NP + 2);
  static constexpr int OP = OH + ev(EPW * NP + 2);
  static constexpr int OI = OP + EPW * NF * NC;
  static constexpr int OB = OI + EPW * NF * NC;
  static constexpr int OR = OB + (SLIM ? 0 : ev(EPW * NP + 2));
  static constexpr int OC = OR + EPW * 8;   // + 64-byte records
  static constexpr int COLS = 2 * ((ipow(N, D - 1) * D + 2 * (D - 1) * ipow(N, D - 2) + 1) / 2);
  static constexpr bool COLDIRECT = DG_H2_COLDIRECT != 0;
  static constexpr int STG = OC + ((SLIM || COLDIRECT) ? 0 : EPW * COLS);  // + column rows (lookahead, terrain)
  static constexpr int TSLOT = HL::odd(HL::DRAW);
  // fused Gram-Schmidt dots in this kernel (measured slower than the separate
  // dual-dot pass; DG_H2_FUSED_DOTS=1 keeps the code and its
  // per-warp totals): without them the launcher sends a fused request to the
  // non-pipelined kernel
  static constexpr bool FUSED = DG_H2_FUSED_DOTS != 0;
  static constexpr int WT = FUSED ? 2 * (32 + 2) : 0;
  static constexpr int WREG = ((2 * STG + HL::NSLOT * TSLOT + WT) + 1) & ~1;  // per warp
  // CTAs per SM x warps per CTA: the stage ring's shared memory (21.9 KB per
  // warp at 3D r = 3) limits the resident warps, and H2 is short of warps (2
  // per scheduler at 2 x 4): take the split with the most warps per SM that
  // fits (3D r = 3: 2 x 5, 6.48 -> 6.25 ms per apply; 3 x 3: 6.40)
  static constexpr long SM_BYTES = 228 * 1024, CTA_BYTES = 227 * 1024, CTA_RES = 1024;
  static constexpr bool fits(int ctas, int w) {
    const long per = (long)(HL::TABP + w * WREG) * (long)sizeof(double);
    // (<= 12 warps per SM: the kernel needs up to 168 registers per thread)
    return ctas * w <= 12 && per <= CTA_BYTES && ctas * (per + CTA_RES) <= SM_BYTES;
  }
  static constexpr int pick(bool want_ctas) {
    int bc = 1, bw = 1, best = 0;
    for (int ctas = 3; ctas >= 1; --ctas)
      for (int w = 1; w <= 8; ++w)
        if (fits(ctas, w) && ctas * w > best) {
          best = ctas * w;
          bc = ctas;
          bw = w;
        }
    return want_ctas ? bc : bw;
  }
  static constexpr int WPB = DG_H2_WPB > 0 ? DG_H2_WPB : pick(false);
  static constexpr int CTAS = DG_H2_WPB > 0 ? DG_HK2P_MINB : pick(true);
  static constexpr size_t SMEM = (size_t)(HL::TABP + WPB * WREG) * sizeof(double);
};

// the fused Gram-Schmidt dots accumulated over the groups of a warp
// (gs_round with += into the warp's column totals)
template <int D, int N, int PER>
__device__ __forceinline__ void gs_round_acc(const KParams<N>& P, bool own, long long e, int c,
                                             const double* wv, const double* uv, int c0, int nv,
                                             int nvt, double* wtot) {
  constexpr int NP = ipow(N, D), NI = 16 / PER;
  const int lane = threadIdx.x & 31;
  const int i0 = c0 / PER;
  double sv[16];
#pragma unroll
  for (int t = 0; t < NI; ++t) {
    const int it = i0 + t;
    const bool ld = own && it < nv;
    const double* vp = P.gsV + (long long)it * P.gs_vs + e * NP;
    double v[N];
#pragma unroll
    for (int ii = 0; ii < N; ++ii) {
      const int node = (D == 3) ? ii * N * N + c : ii * N + c;
      v[ii] = ld ? vp[node] : (it == nv ? wv[ii] : uv[ii]);
    }
    double s0 = 0.0, s1 = 0.0;
#pragma unroll
    for (int ii = 0; ii < N; ++ii) {
      s0 = fma(v[ii], wv[ii], s0);
      if (PER == 2) s1 = fma(v[ii], uv[ii], s1);
    }
    sv[t * PER] = own ? s0 : 0.0;
    if (PER == 2) sv[t * PER + 1] = own ? s1 : 0.0;
  }
#pragma unroll
  for (int o = 16, m = 16; o >= 2; o >>= 1, m >>= 1) {
    const bool up = (lane & o) != 0;
#pragma unroll
    for (int k = 0; k < m / 2; ++k) {
      const double send = up ? sv[k] : sv[k + m / 2];
      const double keep = up ? sv[k + m / 2] : sv[k];
      sv[k] = keep + __shfl_xor_sync(0xffffffffu, send, o);
    }
  }
  sv[0] += __shfl_xor_sync(0xffffffffu, sv[0], 1);
  const int col = c0 + ((lane >> 1) & 15);
  if ((lane & 1) == 0 && col < nvt) wtot[col] += sv[0];
}

#ifndef DG_H2_LATE_LA
#define DG_H2_LATE_LA 1
#endif

template <int D, int N, bool LA>
__global__ void __launch_bounds__(32 * H2Pipe<D, N>::WPB, H2Pipe<D, N>::CTAS)
hdiv2_kernel(const __grid_constant__ KParams<N> P) {
  using HL = HLayout<D, N>;
  using PL = H2Pipe<D, N>;
  constexpr int NC = HL::NC, EPW = HL::EPW, NF = HL::NF, TSZ = HL::TSZ, NP = HL::NP;
  extern __shared__ __align__(16) double smem[];
  __shared__ unsigned long long tbar;
  __shared__ unsigned long long sbar[PL::WPB][2], cbar[PL::WPB][2];
  tab_bulk_issue(smem, P.tab_g, HL::TABD * 8, &tbar);
  pdl_trigger();
  pdl_wait();  // (programmatic dependent launch below 2^24 DoF: dg_pdl.cuh)
  const Tab<N>& TS = *reinterpret_cast<const Tab<N>*>(smem);
  const Tab<N>& TC = P.tab;
  const MeshDev& mesh = P.mesh;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int eiw = lane / NC, c = lane - eiw * NC;
  const bool slot_ok = eiw < EPW;
  // LA: geometry from the staged records and the column rows by lookahead
  // bulk copies; else both by (latency-exposed) global loads
  const bool terr = LA && !PL::SLIM && !PL::COLDIRECT && P.gc.terrain != 0;
  const unsigned cb[2] = {smem_u32(&cbar[wid][0]), smem_u32(&cbar[wid][1])};
  double* W = smem + HL::TABP + wid * PL::WREG;
  double* STG0 = W;
  double* X = W + 2 * PL::STG + (slot_ok ? eiw : EPW) * PL::TSLOT;
  double* wtot = W + 2 * PL::STG + HL::NSLOT * PL::TSLOT;
  const unsigned bar0 = smem_u32(&sbar[wid][0]), bar1 = smem_u32(&sbar[wid][1]);
  const long long ngroups = ((long long)mesh.n_el + EPW - 1) / EPW;
  const long long gw = (long long)blockIdx.x * PL::WPB + wid;
  const long long GW = (long long)gridDim.x * PL::WPB;
  const bool dots = PL::FUSED && P.gs_part != nullptr;
  const bool dual = P.gs_dual != 0;
  const int nv = P.gs_nv;
  const int nvt = dual ? 2 * (nv + 2) : nv + 1;
  for (int i = lane; i < PL::WT; i += 32) wtot[i] = 0.0;

  // lane 0: bring group g into stage s
  auto issue = [&](long long g, int s) {
    const long long e0 = g * EPW;
    const int ne = (int)min((long long)EPW, (long long)mesh.n_el - e0);
    double* st = STG0 + s * PL::STG;
    const unsigned b = s ? bar1 : bar0;
    // 16-byte aligned spans covering the element blocks (odd n^d)
    auto span = [](const double* p, int count, unsigned long long& a0) -> unsigned {
      a0 = reinterpret_cast<unsigned long long>(p) & ~15ULL;
      const unsigned long long a1 =
          (reinterpret_cast<unsigned long long>(p + count) + 15ULL) & ~15ULL;
      return (unsigned)(a1 - a0);
    };
    unsigned long long aV, aH, aB = 0;
    const unsigned bV = span(P.in.p + e0 * P.in.estride, ne * D * NP, aV);
    const unsigned bH = span(P.inH.p + e0 * P.inH.estride, ne * NP, aH);
    const unsigned bB = (P.has_base && !PL::SLIM)
                            ? span(P.base.p + e0 * P.base.estride, ne * NP, aB) : 0u;
    const unsigned bytes = bV + bH + bB + 8u * ne * (2 * NF * NC + 8);
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(b), "r"(bytes)
                 : "memory");
    bulk_g2s(st + PL::OV, reinterpret_cast<const void*>(aV), bV, b);
    bulk_g2s(st + PL::OH, reinterpret_cast<const void*>(aH), bH, b);
    bulk_g2s(st + PL::OP, P.psi + e0 * (NF * NC), 8u * ne * NF * NC, b);
    bulk_g2s(st + PL::OI, P.pin + e0 * (NF * NC), 8u * ne * NF * NC, b);
    if (P.has_base && !PL::SLIM) bulk_g2s(st + PL::OB, reinterpret_cast<const void*>(aB), bB, b);
    bulk_g2s(st + PL::OR, P.frec + e0 * REC_INTS, 64u * ne, b);
    if (dots) {
      // the fused dots' basis slices of this group into L2
      for (int i = 0; i < nv; ++i) {
        const double* src = P.gsV + (long long)i * P.gs_vs + e0 * NP;
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;\n" ::"l"(src),
                     "r"(8u * ne * NP)
                     : "memory");
      }
    }
  };
  // all lanes, once group g's records have landed: its column rows (terrain)
  auto lookahead = [&](long long g, int s) {
    if (!terr) return;
    double* st = STG0 + s * PL::STG;
    const int ne = (int)min((long long)EPW, (long long)mesh.n_el - g * EPW);
    if (lane == 0)
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(cb[s]),
                   "r"(8u * ne * PL::COLS)
                   : "memory");
    __syncwarp();
    if (slot_ok && c == 0 && g * EPW + eiw < mesh.n_el) {
      const int* rec = reinterpret_cast<const int*>(st + PL::OR) + eiw * REC_INTS;
      bulk_g2s(st + PL::OC + eiw * PL::COLS, mesh.col + (long long)rec[8 + 1 + D] * P.gc.col_stride,
               8u * PL::COLS, cb[s]);
    }
  };
  if (lane == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(bar0) : "memory");
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(bar1) : "memory");
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(cb[0]) : "memory");
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(cb[1]) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    if (gw < ngroups) issue(gw, 0);
    if (gw + GW < ngroups) issue(gw + GW, 1);
  }
  __syncthreads();  // the table barrier is initialised (and every stage barrier)
  if (gw < ngroups) {
    mbar_wait(bar0, 0);
    lookahead(gw, 0);
  }
  tab_bulk_wait(&tbar);
  const int fa = (D == 2) ? c : c / N;
  const int fb = (D == 2) ? 0 : c % N;
  const double wcol = (D == 3) ? TS.qw[c / N] * TS.qw[c % N] : TS.qw[c];
  double iwq = (D == 3) ? TS.iqw[c / N] * TS.iqw[c % N] : TS.iqw[c];

  int k = 0;
  for (long long g = gw; g < ngroups; g += GW, ++k) {
    const int s = k & 1;
    const unsigned par = (unsigned)((k >> 1) & 1);
    mbar_wait(s ? bar1 : bar0, par);
    if (terr) mbar_wait(cb[s], par);
#if !DG_H2_LATE_LA
    if (g + GW < ngroups) {
      mbar_wait(s ? bar0 : bar1, (unsigned)(((k + 1) >> 1) & 1));
      lookahead(g + GW, s ^ 1);
    }
#endif
    const double* st = STG0 + s * PL::STG;
    const long long e = g * EPW + eiw;
    const bool act = slot_ok && e < mesh.n_el;
    const int esl = act ? eiw : 0;
    const int* rec = reinterpret_cast<const int*>(st + PL::OR) + esl * REC_INTS;
    const uint8_t* rk = reinterpret_cast<const uint8_t*>(rec + 6);
    uint8_t kf[NF];
    int nf[NF];
#pragma unroll
    for (int f = 0; f < NF; ++f) {
      kf[f] = act ? rk[f] : (uint8_t)KIND_WALL;
      nf[f] = rec[f];
    }
    // (the column's terrain scalars first: with DG_H2_COLDIRECT they are
    // plain loads, in flight during the face-flux phase)
    const ElemGeo<D> g3 = LA ? geo_from_row<D>(rec + 8, P.gc) : elem_geo<D>(mesh.elem, P.gc, act ? e : 0);
    const double* colrow = (LA && !PL::SLIM && !PL::COLDIRECT) ? st + PL::OC + esl * PL::COLS
                                             : mesh.col + (long long)g3.col * P.gc.col_stride;
    ColData<D, N> cd;
    cd.omh = 1.0;
    cd.dh[0] = cd.dh[1] = 0.0;
    if (P.gc.terrain && act) {
      constexpr int NQH = ipow(N, D - 1);
      cd.omh = colrow[c];
#pragma unroll
      for (int a = 0; a < D - 1; ++a) cd.dh[a] = colrow[NQH * (1 + a) + c];
    }
    // face fluxes: psi + pin (conforming, wall, far field, fine), coarse side
    // precomputed
    double fl[NF];
    {
      const double* ps = st + PL::OP + esl * (NF * NC) + c;
      const double* pi = st + PL::OI + esl * (NF * NC) + c;
#pragma unroll
      for (int f = 0; f < NF; ++f) {
        const int kd = kf[f] & 15;
        const double sg = (f & 1) ? 1.0 : -1.0;
        double v = sg * (ps[f * NC] + pi[f * NC]);
        if (kd == KIND_COARSE) v = (mesh.cflux != nullptr) ? mesh.cflux[(long long)nf[f] * NC + c] : 0.0;
        fl[f] = act ? v : 0.0;
      }
    }
    // fine side of hanging faces (as hdiv_kernel)
    auto fine_face = [&](auto ax_c, auto side_c) {
      constexpr int AX = decltype(ax_c)::value;
      constexpr int side = decltype(side_c)::value;
      constexpr int f = 2 * AX + side;
      const int kd = kf[f] & 15;
      const bool fine = act && kd == KIND_FINE;
      if (!__any_sync(0xffffffffu, fine)) return;
      constexpr int FC = (AX < D - 1) ? 2 : D + 1;
      constexpr int TSL = tr_slots<D>() * NC, THL = 2 * D * NC;
      const long long pe = nf[f];
#pragma unroll
      for (int r = 0; r < FC; ++r) {
        double v = 0.0;
        if (fine) {
          const bool isv = r < FC - 1;
          const int comp = (AX < D - 1) ? AX : r;
          v = isv ? P.trV[pe * TSL + tr_slot<D>(f ^ 1, comp) * NC + c]
                  : P.trH[pe * THL + (f ^ 1) * NC + c];
        }
        X[r * NC + c] = v;
      }
      __syncwarp();
      const int sf = (kf[f] >> 4) & 3;
      const double* Mq0 = &TS.halfq[sf & 1][0][0];
      const double* Mq1 = &TS.halfq[(sf >> 1) & 1][0][0];
      double tr[FC];
#pragma unroll
      for (int r = 0; r < FC; ++r) {
        double t = 0.0;
        if constexpr (D == 2) {
#pragma unroll
          for (int j = 0; j < N; ++j) t = fma(Mq0[fa * N + j], X[r * NC + j], t);
        } else {
#pragma unroll
          for (int j = 0; j < N; ++j) t = fma(Mq0[fa * N + j], X[r * NC + j * N + fb], t);
        }
        tr[r] = t;
      }
      if constexpr (D == 3) {
        __syncwarp();
#pragma unroll
        for (int r = 0; r < FC; ++r) X[r * NC + c] = tr[r];
        __syncwarp();
#pragma unroll
        for (int r = 0; r < FC; ++r) {
          double t = 0.0;
#pragma unroll
          for (int j = 0; j < N; ++j) t = fma(Mq1[fb * N + j], X[r * NC + fa * N + j], t);
          tr[r] = t;
        }
      }
      __syncwarp();
      if (fine) {
        double n[D], ws;
        constexpr int NQH = ipow(N, D - 1), NE = ipow(N, D - 2);
        const double oe = (AX < D - 1 && P.gc.terrain)
                              ? colrow[NQH * D + f * NE + ((D == 2) ? 0 : c / N)] : 1.0;
        face_nplus<D, N, AX>(P.gc, g3, side, c, TS, oe, cd.dh, n, ws);
        double vn;
        if constexpr (AX < D - 1) {
          vn = tr[0] * n[AX];
        } else {
          vn = 0.0;
#pragma unroll
          for (int a = 0; a < D; ++a) vn = fma(tr[a], n[a], vn);
        }
        const double sg = side ? 1.0 : -1.0;
        fl[f] += sg * ((0.5 * ws) * (tr[FC - 1] * vn));
      }
    };
    // (one vote per group: most warps own no fine side of a hanging face)
    bool has_fine = false;
#pragma unroll
    for (int f = 0; f < NF; ++f) has_fine |= act && (kf[f] & 15) == KIND_FINE;
    if (mesh.n_coarse > 0 && __any_sync(0xffffffffu, has_fine)) {
      fine_face(std::integral_constant<int, 0>{}, std::integral_constant<int, 0>{});
      fine_face(std::integral_constant<int, 0>{}, std::integral_constant<int, 1>{});
      if constexpr (D == 3) {
        fine_face(std::integral_constant<int, 1>{}, std::integral_constant<int, 0>{});
        fine_face(std::integral_constant<int, 1>{}, std::integral_constant<int, 1>{});
      }
      fine_face(std::integral_constant<int, D - 1>{}, std::integral_constant<int, 0>{});
      fine_face(std::integral_constant<int, D - 1>{}, std::integral_constant<int, 1>{});
    }
#if DG_H2_LATE_LA == 2
    if (terr && g + GW < ngroups) {  // (variant: the lookahead before the volume phase)
      mbar_wait(s ? bar0 : bar1, (unsigned)(((k + 1) >> 1) & 1));
      lookahead(g + GW, s ^ 1);
    }
#endif
    // volume
    double Zc[N];
    const double det = col_det<D>(g3, cd.omh);
    {
      const long long e0g = g * EPW;
      const int shV = (int)((reinterpret_cast<unsigned long long>(P.in.p + e0g * P.in.estride) >> 3) & 1);
      const int shH = (int)((reinterpret_cast<unsigned long long>(P.inH.p + e0g * P.inH.estride) >> 3) & 1);
      const double* Vs = st + PL::OV + shV + esl * (D * NP) + c * N;
      const double* Hs = st + PL::OH + shH + esl * NP + c * N;
      double Gz[N];
#pragma unroll
      for (int kz = 0; kz < N; ++kz) {
        double ct[D][D];
        col_metric<D, N>(P.gc, g3, cd.omh, cd.dh, TC.qx[kz], ct);
        const double wq = wcol * TC.qw[kz];
        const double h = Hs[kz];
        double F[D];
#pragma unroll
        for (int a = 0; a < D; ++a) F[a] = h * Vs[a * NP + kz];
        X[coff<D, N>(c, kz)] = (F[0] * ct[0][0]) * wq;
        if constexpr (D == 3) X[TSZ + coff<D, N>(c, kz)] = (F[1] * ct[1][1]) * wq;
        double acc = 0.0;
#pragma unroll
        for (int a = 0; a < D; ++a) acc += F[a] * ct[D - 1][a];
        Gz[kz] = acc * wq;
      }
      mat_apply<N, true>(TC.Dhat, Gz, Zc);
      const int zf = 2 * (D - 1);
#pragma unroll
      for (int kz = 0; kz < N; ++kz)
        Zc[kz] = TC.lift[0][kz] * fl[zf] + TC.lift[1][kz] * fl[zf + 1] - Zc[kz];
    }
    __syncwarp();
#if DG_H2_LATE_LA == 1
    // the next group's column rows: its records were requested at the end of
    // the previous iteration, so by now (half of this group's arithmetic
    // later) they have landed and this wait costs nothing -- at the top of
    // the iteration it exposed a full memory latency per group (ncu: 15 % of
    // the warp time in that wait)
    if (terr && g + GW < ngroups) {
      mbar_wait(s ? bar0 : bar1, (unsigned)(((k + 1) >> 1) & 1));
      lookahead(g + GW, s ^ 1);
    }
#endif
    {
      double v[N], o[N];
#pragma unroll
      for (int ii = 0; ii < N; ++ii) v[ii] = X[xoff<D, N>(c, ii)];
      mat_apply<N, true>(TC.Dhat, v, o);
#pragma unroll
      for (int ii = 0; ii < N; ++ii)
        X[xoff<D, N>(c, ii)] = TC.lift[0][ii] * fl[0] + TC.lift[1][ii] * fl[1] - o[ii];
      if constexpr (D == 3) {
#pragma unroll
        for (int jj = 0; jj < N; ++jj) v[jj] = X[TSZ + yoff<N>(c, jj)];
        mat_apply<N, true>(TC.Dhat, v, o);
#pragma unroll
        for (int jj = 0; jj < N; ++jj)
          X[TSZ + yoff<N>(c, jj)] = TC.lift[0][jj] * fl[2] + TC.lift[1][jj] * fl[3] - o[jj];
      }
    }
    __syncwarp();
#pragma unroll
    for (int kz = 0; kz < N; ++kz) {
      Zc[kz] += X[coff<D, N>(c, kz)];
      if constexpr (D == 3) Zc[kz] += X[TSZ + coff<D, N>(c, kz)];
    }
    // epilogue
    const double iwh = (1.0 / det) * iwq;
    {
      double t[N];
#pragma unroll
      for (int kz = 0; kz < N; ++kz) t[kz] = Zc[kz] * (iwh * TC.iqw[kz]);
      mat_apply<N, false>(TC.Binv, t, Zc);
    }
    __syncwarp();
#pragma unroll
    for (int kz = 0; kz < N; ++kz) X[coff<D, N>(c, kz)] = Zc[kz];
    __syncwarp();
    if constexpr (D == 3) {
      double v[N], o[N];
#pragma unroll
      for (int jj = 0; jj < N; ++jj) v[jj] = X[yoff<N>(c, jj)];
      mat_apply<N, false>(TC.Binv, v, o);
#pragma unroll
      for (int jj = 0; jj < N; ++jj) X[yoff<N>(c, jj)] = o[jj];
      __syncwarp();
    }
    double wv[N], uv[N];
    {
      const int shB = P.has_base
          ? (int)((reinterpret_cast<unsigned long long>(P.base.p + g * EPW * P.base.estride) >> 3) & 1)
          : 0;
      const double* Bs = PL::SLIM ? P.base.p + (act ? e : 0) * P.base.estride
                                  : st + PL::OB + shB + esl * NP;
      double v[N], o[N];
#pragma unroll
      for (int ii = 0; ii < N; ++ii) v[ii] = X[xoff<D, N>(c, ii)];
      mat_apply<N, false>(TC.Binv, v, o);
#pragma unroll
      for (int ii = 0; ii < N; ++ii) {
        const int node = (D == 3) ? ii * N * N + c : ii * N + c;
        const double bv = P.has_base ? Bs[node] : 0.0;
        const double r = __dmul_rn(P.coef, o[ii]);
        const double val = P.has_base ? __dadd_rn(bv, r) : r;
        wv[ii] = act ? val : 0.0;
        uv[ii] = act ? bv : 0.0;
        if (act) P.out.p[e * P.out.estride + node] = val;
      }
    }
    __syncwarp();  // every lane is done with this stage and the tile
    if (lane == 0 && g + 2 * GW < ngroups) issue(g + 2 * GW, s);
    if (dots) {
      for (int c0 = 0; c0 < nvt; c0 += 16) {
        if (dual) gs_round_acc<D, N, 2>(P, act, e, c, wv, uv, c0, nv, nvt, wtot);
        else gs_round_acc<D, N, 1>(P, act, e, c, wv, uv, c0, nv, nvt, wtot);
      }
    }
  }
  if (dots) {
    __syncthreads();
    if (wid == 0) {
      for (int col = lane; col < nvt; col += 32) {
        double t = 0.0;
#pragma unroll
        for (int w = 0; w < PL::WPB; ++w) t += smem[HL::TABP + w * PL::WREG + 2 * PL::STG + HL::NSLOT * PL::TSLOT + col];
        P.gs_part[((long long)P.gs_row0 + blockIdx.x) * nvt + col] = t;
      }
    }
  }
}

// pin rows of owned elements whose conforming neighbour is a ghost (another
// rank's element): copied from the ghost's exchanged psi after the halo
// exchange; fix = (element, face, ghost) triples
static __global__ void hk_pin_fixup(const int* __restrict__ fix, int nfix, int nc, int nf,
                             const double* __restrict__ psi, double* __restrict__ pin) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= (long long)nfix * nc) return;
  const int t = (int)(i / nc), c = (int)(i % nc);
  const int e = fix[3 * t], f = fix[3 * t + 1], gh = fix[3 * t + 2];
  pin[((long long)e * nf + f) * nc + c] = psi[((long long)gh * nf + (f ^ 1)) * nc + c];
}

}  // namespace dg
