// Warp-element DG operator kernel (v3) for the Helmholtz pair
// (gradient H1 and div(hV) H2), fp64, sm_100a.
//
// Each element is owned by NC = n^(d-1) consecutive lanes of ONE warp; lane
// c holds the z-column c of the element (points c*n + k, k = 0..n-1) in
// registers.  Consequently:
//   * z passes (interpolation, Dhat^T, B^-1) are register-only;
//   * x / y passes go through a per-element shared-memory tile with a padded
//     column stride, synchronised by __syncwarp() only -- the kernel has no
//     CTA-wide barrier at all;
//   * lane c also owns face point c of EVERY face, and that face point lies
//     on the lane's pencil along the face normal: own traces are pencil
//     contractions, neighbour traces are one global load per face followed
//     by 2 tangential passes done with warp shuffles, and each face's lift
//     is added straight onto the lane's normal-direction pencil while that
//     direction's volume pass is in registers.
// Same algebra and reference citations as dg_kernel.cuh (weak form
// dgops.py:87-230, centred fluxes dgops.py:343-348 / 452-460, metric
// geometry.py:204-238 / 305-357, factorised mass inverse geometry.py:372-396).
// The coarse side of hanging faces is added afterwards by coarse_kernel.
#pragma once
#include "dg_kernel.cuh"

namespace dg {

// per-element tile layout.  3D point (i, j, k) (z fastest; z-column
// c = i*N + j): columns at a padded stride n+1, except for n = 4, where 16
// lanes per element meet the 16 double-wide smem banks exactly: the
// swizzle 16 k + 4 ((i + j) & 3) + ((j + k) & 3) maps every axis-aligned
// plane (a column access, an x- or a y-pencil access across the element's
// 16 lanes) onto 16 distinct banks, without padding.
template <int D, int N>
__host__ __device__ constexpr int tile_size() {
  return (D == 3 && N == 4) ? 64 : ipow(N, D - 1) * (N + 1);
}
template <int D, int N>
__device__ __forceinline__ int toff3(int i, int j, int k) {
  if constexpr (D == 3 && N == 4) return 16 * k + 4 * ((i + j) & 3) + ((j + k) & 3);
  else return (i * N + j) * (N + 1) + k;
}
template <int D, int N>
__device__ __forceinline__ int coff(int c, int k) {  // own z-column c, point k
  if constexpr (D == 3) return toff3<D, N>(c / N, c % N, k);
  else return c * (N + 1) + k;
}
template <int D, int N>
__device__ __forceinline__ int xoff(int c, int ii) {  // x-pencil of lane c, point ii
  if constexpr (D == 3) return toff3<D, N>(ii, c / N, c % N);
  else return ii * (N + 1) + c;
}
template <int N>
__device__ __forceinline__ int yoff(int c, int jj) {  // 3D y-pencil of lane c, point jj
  return toff3<3, N>(c / N, jj, c % N);
}

template <int D, int N, int OPK>
struct WLayout {
  static constexpr int NP = ipow(N, D);
  static constexpr int NC = ipow(N, D - 1);  // lanes per element
  static constexpr int EPW = 32 / NC;          // elements per warp
  static constexpr int KIN = OpDims<D, OPK>::KIN;
  static constexpr int KOUT = OpDims<D, OPK>::KOUT;
  static constexpr int KW = (OPK == OP_GRAD) ? 1 : KOUT;
  static constexpr int TSZ = tile_size<D, N>();  // one tensor (tile layout: coff)
  static constexpr int KX0 = KIN > KOUT ? KIN : KOUT;
  static constexpr int KX1 = (D - 1) * KW;
  static constexpr int KX = KX0 > KX1 ? KX0 : KX1;
  // raw input components behind one face value (gradient: x and K)
  static constexpr int RAW = (OPK == OP_GRAD) ? 2 : KIN;
  static constexpr int WPB = 4;                // warps per CTA
  static constexpr int THREADS = 32 * WPB;
  static constexpr int TABD = (int)(sizeof(Tab<N>) / sizeof(double));
  // padding lanes (32 % NC != 0) get a private scratch slot
  static constexpr int NSLOT = EPW + ((32 % NC) ? 1 : 0);
  static constexpr int odd(int s) { return (s % 2 == 0) ? s + 1 : s; }  // bank shift
  // async prefetch of the neighbour face nodes into smem, as long as the
  // staging area keeps 4 CTAs (the register-limited occupancy) per SM
  // (+ the lane's terrain scalars: omh, dh at its column and omh at its point
  // of every vertical face; the epilogue's base values reuse the face area)
  static constexpr int GEON = 1 + (D - 1);  // + the compact edge table GEE
  static constexpr int NE = ipow(N, D - 2);  // distinct edge values per vertical face
  static constexpr int GEE = 2 * (D - 1) * NE;
  // staged components per face: a vertical face has the exact normal
  // +-e_AX, so div(hV) needs only (V_AX, h) of the neighbour there
  static constexpr int FCX = (OPK == OP_DIVHV) ? 2 : RAW;
  static constexpr int FCZ = RAW;
  static constexpr int FGA = (2 * (D - 1) * FCX + 2 * FCZ) * NC;
  static constexpr int FGB = (FGA > KOUT * NP ? FGA : KOUT * NP) + GEON * NC + GEE;
  static constexpr bool ASYNC =
      (TABD + WPB * NSLOT * odd(KX * TSZ + FGB)) * 8 <= 54 * 1024;
  static constexpr int FGN = ASYNC ? FGB - GEON * NC - GEE : 0;
  __host__ __device__ static constexpr int fg_off(int f) {  // staged face f
    return (f < 2 * (D - 1)) ? f * FCX * NC : (2 * (D - 1) * FCX + (f - 2 * (D - 1)) * FCZ) * NC;
  }
  __host__ __device__ static constexpr int fg_cnt(int f) { return (f < 2 * (D - 1)) ? FCX : FCZ; }
  static constexpr int SLOT = odd(KX * TSZ + (ASYNC ? FGB : 0));
  static constexpr size_t SMEM = (size_t)(TABD + WPB * NSLOT * SLOT) * sizeof(double);
  static constexpr bool OK = (NC <= 32) && (OPK != OP_ADV);
  // resident CTAs per SM the register allocation is capped for
#ifndef DG_WMINB_GRAD
#define DG_WMINB_GRAD 5
#endif
#ifndef DG_WMINB_DIVHV
#define DG_WMINB_DIVHV 4
#endif
  static constexpr int MINB = (OPK == OP_GRAD) ? DG_WMINB_GRAD : DG_WMINB_DIVHV;
};


// team-wide barrier and vote (a warp, or two warps on named barrier 1 + team)
template <int TPE>
__device__ __forceinline__ void esync(int team) {
  if constexpr (TPE == 32) {
    __syncwarp();
  } else {
    asm volatile("bar.sync %0, %1;\n" ::"r"(1 + team), "r"(TPE) : "memory");
  }
}
template <int TPE>
__device__ __forceinline__ bool eany(bool pred, int team) {
  if constexpr (TPE == 32) {
    return __any_sync(0xffffffffu, pred);
  } else {
    unsigned out;
    asm volatile(
        "{\n .reg .pred p, q;\n setp.ne.u32 q, %1, 0;\n"
        " bar.red.or.pred p, %2, %3, q;\n selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(out)
        : "r"((unsigned)pred), "r"(1 + team), "r"(TPE)
        : "memory");
    return out != 0;
  }
}

__device__ __forceinline__ void cp_async8(void* smem_ptr, const void* gptr) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem_ptr);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(s), "l"(gptr) : "memory");
}

// terrain scalars, staged in smem: GE[i * NC + c] for lane c,
//   i = 0: 1 - h/z_top at the column's horizontal Gauss point
//   i = 1..HD: dh/dx_a there (also the z-face values of face point c)
// followed by the compact edge table GE[GEON * NC + (2 AX + side) * NE + qo]:
// 1 - h_edge/z_top along vertical face (AX, side) (column table order)
template <int D, int N>
__device__ __forceinline__ int geo_src(int i, int c) {
  constexpr int HD = D - 1, NQH = ipow(N, HD);
  return (i == 0) ? c : NQH * i + c;
}

// Gauss-point metric (as point_metric) from the staged terrain scalars
template <int D, int N>
__device__ __forceinline__ void point_metric_ge(const GeoConst& gc, const Tab<N>& T,
                                                const ElemGeo<D>& g, int qz, const double* GE,
                                                int NCs, int c, double& det, double ctrv[D][D]) {
  constexpr int HD = D - 1;
  const double omh = GE[c];
  const double zz = g.s[D - 1] * omh;
  det = 1.0;
#pragma unroll
  for (int a = 0; a < HD; ++a) det = det * g.s[a];
  det = det * zz;
  const double decay = 1.0 - (g.lo[D - 1] + g.s[D - 1] * T.qx[qz]) * gc.inv_ztop;
  double zg[2];
#pragma unroll
  for (int a = 0; a < HD; ++a) zg[a] = GE[(1 + a) * NCs + c] * g.s[a] * decay;
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

// face metric (as face_metric_ax, own geometry) from the staged terrain scalars
template <int D, int N, int AX>
__device__ __forceinline__ void face_metric_ge(const GeoConst& gc, const ElemGeo<D>& g, int side,
                                               bool outward, int qf, const Tab<N>& T,
                                               const double* GE, int NCs, double n[D],
                                               double& ws) {
  constexpr int HD = D - 1;
  const double fw = (D == 2) ? T.qw[qf] : T.qw[qf / N] * T.qw[qf % N];
  const double sgn = (outward && side == 0) ? -1.0 : 1.0;
#pragma unroll
  for (int a = 0; a < D; ++a) n[a] = 0.0;
  if constexpr (AX < D - 1) {
    constexpr int NE = ipow(N, HD - 1);
    const double omh =
        gc.terrain ? GE[(1 + HD) * NCs + (2 * AX + side) * NE + ((D == 2) ? 0 : qf / N)] : 1.0;
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
    const double decay = 1.0 - (g.lo[D - 1] + g.s[D - 1] * (double)side) * gc.inv_ztop;
    double nt[D];
    if constexpr (D == 2) {
      nt[0] = -GE[NCs + qf] * g.s[0] * decay;
    } else {
      nt[0] = -g.s[1] * GE[NCs + qf] * g.s[0] * decay;
      nt[1] = -g.s[0] * GE[2 * NCs + qf] * g.s[1] * decay;
    }
    nt[D - 1] = top;
    double m2 = 0.0;
#pragma unroll
    for (int a = 0; a < D; ++a) m2 += nt[a] * nt[a];
    const double mag = sqrt(m2);
    const double im = sgn / mag;
#pragma unroll
    for (int a = 0; a < D; ++a) n[a] = nt[a] * im;
    ws = fw * mag;
  }
}
__device__ __forceinline__ void cp_async_wait_all() {
  asm volatile("cp.async.commit_group;\n" ::);
  asm volatile("cp.async.wait_group 0;\n" ::: "memory");
}

template <int N, bool TRANS>
__device__ __forceinline__ void mat_apply(const double (&M)[N][N], const double* v, double* o) {
#pragma unroll
  for (int i = 0; i < N; ++i) {
    double acc = 0.0;
#pragma unroll
    for (int j = 0; j < N; ++j) acc = fma(TRANS ? M[j][i] : M[i][j], v[j], acc);
    o[i] = acc;
  }
}

// Fused Gram-Schmidt dots (GMRES, krylov.py:69-72 with the classical
// variant of DESIGN.md §4): the CTA's partial sums of V_i . y (i < nv) and
// y . y over its elements' nodes, written as row (gs_row0 + CTA) of gs_part.
// Dual mode (P.gs_dual, DCGS2): also V_i . u, y . u and u . u, u = the
// action's input (the epilogue's base values uv[]); items i = 0..nv+1 (V_i,
// then y, then u) give the column pairs (item . y, item . u).
// The lane's stored values wv[] are its x-pencil nodes (ii, c).  Elements
// with a coarse-side hanging face are left to coarse_kernel, which adds to
// their result afterwards.  Per round of 16 columns each lane forms its
// partials in registers and a butterfly transpose-reduction over the warp
// (16 double shuffles) leaves one column total per lane pair; the warps'
// totals meet in smem (one CTA barrier at the very end).  Deterministic:
// fixed lane / warp / row order.
template <int D, int N, int PER>
__device__ __forceinline__ void gs_round(const KParams<N>& P, bool own, long long e, int c,
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
  // butterfly: m values -> m/2 at offsets 16, 8, 4, 2; lane keeps the half
  // selected by its offset bit, so column = (lane >> 1) & 15 at the end
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
  if ((lane & 1) == 0 && col < nvt) wtot[col] = sv[0];
}

template <int D, int N, int OPK>
__device__ __forceinline__ void gs_dots(const KParams<N>& P, double* smem, const uint8_t* kf,
                                        bool act, long long e, int c, const double* wv,
                                        const double* uv) {
  using WL = WLayout<D, N, OPK>;
  constexpr int NF = 2 * D;
  constexpr int AREA = WL::NSLOT * WL::SLOT;  // this warp's element slots
  static_assert(AREA >= 2 * (32 + 2), "warp area too small for the fused dots");
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  bool own = act;
  if (P.mesh.cflux == nullptr) {  // (flux mode: coarse elements are complete here)
#pragma unroll
    for (int f = 0; f < NF; ++f)
      if ((kf[f] & 15) == KIND_COARSE) own = false;
  }
  const bool dual = P.gs_dual != 0;
  const int nv = P.gs_nv;
  const int nvt = dual ? 2 * (nv + 2) : nv + 1;  // columns of the row
  double* wtot = smem + WL::TABD + wid * AREA;   // this warp's column totals
  __syncwarp();  // every lane is done with this warp's tiles
  for (int c0 = 0; c0 < nvt; c0 += 16) {
    if (dual) gs_round<D, N, 2>(P, own, e, c, wv, uv, c0, nv, nvt, wtot);
    else gs_round<D, N, 1>(P, own, e, c, wv, uv, c0, nv, nvt, wtot);
  }
  __syncthreads();
  if (wid == 0) {
    const long long row = (long long)P.gs_row0 + blockIdx.x;
    for (int col = lane; col < nvt; col += 32) {
      double t = 0.0;
#pragma unroll
      for (int w = 0; w < WL::WPB; ++w) t += smem[WL::TABD + w * AREA + col];
      P.gs_part[row * nvt + col] = t;
    }
  }
}

// IQ: Gauss-point input (H2 of the Helmholtz pair in quad mode) -- a
// separate instantiation so the nodal path carries none of its registers
template <int D, int N, int OPK, bool IQ = false>
__global__ void __launch_bounds__(WLayout<D, N, OPK>::THREADS, WLayout<D, N, OPK>::MINB)
welem_kernel(const __grid_constant__ KParams<N> P) {
  using WL = WLayout<D, N, OPK>;
  constexpr int NC = WL::NC, EPW = WL::EPW, KIN = WL::KIN, KOUT = WL::KOUT;
  constexpr int KW = WL::KW, TSZ = WL::TSZ, NF = 2 * D;
  extern __shared__ double smem[];
  // tables -> smem from their global copy (asynchronous, coalesced; the
  // kernel-parameter copy would serialise on divergent constant-bank reads)
  for (int i = threadIdx.x; i < WL::TABD; i += blockDim.x) cp_async8(smem + i, P.tab_g + i);
  // (the tables are first read at the face phase: the barrier is placed there)
  const Tab<N>& TS = *reinterpret_cast<const Tab<N>*>(smem);
  const Tab<N>& TC = P.tab;
  const MeshDev& mesh = P.mesh;
  const int lane = threadIdx.x & 31;
  const int wid = threadIdx.x >> 5;
  const int eiw = lane / NC;
  const int c = lane - eiw * NC;
  const bool slot_ok = eiw < EPW;
  const long long e = ((long long)blockIdx.x * WL::WPB + wid) * EPW + eiw;
  const bool act = slot_ok && e < mesh.n_el;
  const long long es = act ? e : 0;
  const int b0 = slot_ok ? eiw * NC : 0;  // first lane of this element
  // padding lanes (32 % NC != 0) scribble on a private scratch slot
  double* X = smem + WL::TABD + (wid * WL::NSLOT + (slot_ok ? eiw : EPW)) * WL::SLOT;
  const bool flat = !P.gc.terrain;

  // ---- 0. face records, and (small KIN) the neighbour face-node values,
  // issued first so their L2 latency overlaps the interpolation work
  const uint8_t* kind_e = mesh.kind + es * NF;
  const int* nbr_e = mesh.nbr + es * NF;
  uint8_t kf[NF];
  int nf[NF];
#pragma unroll
  for (int f = 0; f < NF; ++f) {
    kf[f] = act ? kind_e[f] : (uint8_t)KIND_WALL;
    nf[f] = act ? nbr_e[f] : 0;
  }
  const ElemGeo<D> g = elem_geo<D>(mesh.elem, P.gc, es);
  // the element's own nodal column, raw components (gradient: x and K),
  // issued before anything consumes a load so all of them are in flight
  constexpr int RAW = WL::RAW;
  double a[RAW][N];
#pragma unroll
  for (int r = 0; r < RAW; ++r)
#pragma unroll
    for (int k = 0; k < N; ++k) {
      double v = 0.0;
      if (act) {
        if constexpr (OPK == OP_GRAD) {
          if (r == 0 && P.in.p) v = P.in(es, 0, c * N + k);
          if (r == 1 && P.has_K) v = P.inK(es, 0, c * N + k);
        } else {
          v = load_input<D, N, OPK>(P, es, r, c * N + k);
        }
      }
      a[r][k] = v;
    }
  // neighbour face node c of every face, copied asynchronously (cp.async)
  // into this lane's private smem slots: the L2 gathers run underneath the
  // interpolation work and are waited for only at the face phase
  double* FGs = X + WL::KX * TSZ;
  constexpr bool iq0 = (OPK == OP_DIVHV) && IQ;
  constexpr bool SMP = WL::ASYNC && !iq0;  // tangential passes through smem
  constexpr bool TRM = WL::ASYNC && iq0;   // trace mode: neighbours' face traces staged
  if (WL::ASYNC) {
    constexpr int TSL = tr_slots<D>() * NC, THL = 2 * D * NC;  // trace floats / element
#pragma unroll
    for (int f = 0; f < NF; ++f) {
      const int kd = kf[f] & 15;
      const bool inter = act && (kd == KIND_CONF || kd == KIND_FINE);
      const long long nb = nf[f];
      const int node = nbr_face_node<D, N>(f >> 1, f & 1, c);
#pragma unroll
      for (int r = 0; r < WL::fg_cnt(f); ++r) {
        double* dst = FGs + WL::fg_off(f) + r * NC + c;
        const double* src = nullptr;
        if (inter) {
          if constexpr (OPK == OP_GRAD) {
            if (r == 0 && P.in.p) src = P.in.p + nb * P.in.estride + node;
            if (r == 1 && P.has_K) src = P.inK.p + nb * P.inK.estride + node;
          } else if constexpr (TRM) {
            // the neighbour's traces on its face f ^ 1, at ITS face Gauss
            // point c (the same point for a conforming neighbour)
            const bool vert = (f >> 1) < D - 1;
            const int comp = vert ? (r == 0 ? (f >> 1) : D) : r;
            src = (comp < D) ? P.trV + nb * TSL + tr_slot<D>(f ^ 1, comp) * NC + c
                             : P.trH + nb * THL + (f ^ 1) * NC + c;
          } else {
            // vertical face: (V_AX, h); z face: every component
            const int cin = (WL::fg_cnt(f) == KIN) ? r : (r == 0 ? (f >> 1) : D);
            src = (cin < D) ? P.in.p + nb * P.in.estride + cin * P.in.cstride + node
                            : P.inH.p + nb * P.inH.estride + node;
          }
        }
        if (src) cp_async8(dst, src);
        else *dst = 0.0;
      }
    }
  }
  double* GEs = FGs + WL::FGN;  // [GEON][NC] terrain scalars (ASYNC only)
  if (WL::ASYNC && P.gc.terrain && act) {
    const double* colp = mesh.col + (long long)g.col * P.gc.col_stride;
#pragma unroll
    for (int i = 0; i < WL::GEON; ++i) cp_async8(GEs + i * NC + c, colp + geo_src<D, N>(i, c));
    constexpr int NQH = ipow(N, D - 1);
    for (int i = c; i < WL::GEE; i += NC)
      cp_async8(GEs + WL::GEON * NC + i, colp + NQH * D + i);
  }
  if constexpr (OPK == OP_DIVHV) {
    // fused Gram-Schmidt dots: pull this element's slice of every basis
    // vector into L2 now (one bulk TMA prefetch of n^d doubles per vector,
    // spread over the element's lanes) so the epilogue's dot loads hit L2
#ifndef DG_GS_PREFETCH
#define DG_GS_PREFETCH 1
#endif
    if (DG_GS_PREFETCH && P.gs_part != nullptr && act) {
      for (int i = c; i < P.gs_nv; i += NC) {
        const double* src = P.gsV + (long long)i * P.gs_vs + e * WL::NP;
        // 16-byte aligned span covering the slice (odd n^d: 8-byte aligned)
        const unsigned long long a0 = reinterpret_cast<unsigned long long>(src) & ~15ULL;
        const unsigned long long a1 =
            (reinterpret_cast<unsigned long long>(src + WL::NP) + 15ULL) & ~15ULL;
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;\n" ::"l"(a0),
                     "r"((unsigned)(a1 - a0))
                     : "memory");
      }
    }
  }
  // ---- 1. nodal column, z interpolation in registers -------------------
  // in_quad (H2 of the Helmholtz pair): inputs are already Gauss values
  constexpr bool iq = iq0;
  double q[KIN][N];
#pragma unroll
  for (int cp = 0; cp < KIN; ++cp) {
    double col[N];
#pragma unroll
    for (int k = 0; k < N; ++k) {
      if constexpr (OPK == OP_GRAD)
        col[k] = P.has_K ? P.alpha * (a[0][k] - P.beta * a[1][k]) : P.alpha * a[0][k];
      else
        col[k] = a[cp][k];
    }
    if (iq) {
#pragma unroll
      for (int k = 0; k < N; ++k) q[cp][k] = col[k];
    } else {
      mat_apply<N, false>(TC.B, col, q[cp]);
    }
  }
  // ---- 2. x (and y) interpolation through the tile ------------------------
#pragma unroll
  for (int cp = 0; cp < KIN; ++cp)
#pragma unroll
    for (int k = 0; k < N; ++k) X[cp * TSZ + coff<D, N>(c, k)] = q[cp][k];
  __syncwarp();
  if constexpr (D == 3) {
    if (!iq) {
#pragma unroll
      for (int cp = 0; cp < KIN; ++cp) {
        double v[N], o[N];
#pragma unroll
        for (int jj = 0; jj < N; ++jj) v[jj] = X[cp * TSZ + yoff<N>(c, jj)];
        mat_apply<N, false>(TC.B, v, o);
#pragma unroll
        for (int jj = 0; jj < N; ++jj) X[cp * TSZ + yoff<N>(c, jj)] = o[jj];
      }
      __syncwarp();
    }
  }
  // x pass: the tile now holds the element's Gauss-point values, kept intact
  // through the face phase (own traces are pencil contractions read from it)
  if (!iq) {
#pragma unroll
    for (int cp = 0; cp < KIN; ++cp) {
      double v[N], o[N];
#pragma unroll
      for (int ii = 0; ii < N; ++ii) v[ii] = X[cp * TSZ + xoff<D, N>(c, ii)];
      mat_apply<N, false>(TC.B, v, o);
#pragma unroll
      for (int ii = 0; ii < N; ++ii) X[cp * TSZ + xoff<D, N>(c, ii)] = o[ii];
    }
  }
  __syncwarp();
  // ---- 3. faces: flux at face point c of every face --------------------
  // fl_l[f][k]: lifted flux*ws (with sign) at face point c of face f
  double fl[NF][KOUT];
  auto face = [&](auto ax_c, int side) {
    constexpr int AX = decltype(ax_c)::value;
    const int f = 2 * AX + side;
    const uint8_t kraw = kf[f];
    const int kd = kraw & 15;
    const bool inter = (kd == KIND_CONF || kd == KIND_FINE);
    const long long nb = nf[f];
    // neighbour trace at face point c: gather node c of the neighbour's
    // opposite face, then tangential passes across the element's lanes
    double TN[KIN], TO[KIN];
    const int fa = (D == 2) ? c : c / N;   // tangential index t0
    const int fb = (D == 2) ? 0 : c % N;   // tangential index t1
    const int sf = (kraw >> 4) & 3;
    const double* M0 = (kd == KIND_FINE) ? &TS.half[sf & 1][0][0] : &TS.B[0][0];
    const double* M1 = (kd == KIND_FINE) ? &TS.half[(sf >> 1) & 1][0][0] : &TS.B[0][0];
    bool need_pass = true;
    if (iq) {
      // Gauss-point input: the neighbour's trace at its own face Gauss point
      // (fa, fb) is a lift contraction of its normal pencil; conforming faces
      // need no tangential transform, a fine leaf applies halfq (x) halfq
      need_pass = __any_sync(0xffffffffu, act && kd == KIND_FINE);
    }
    const double* Mq0 = &TS.halfq[sf & 1][0][0];
    const double* Mq1 = &TS.halfq[(sf >> 1) & 1][0][0];
    if constexpr (SMP) {
      // the element's staged neighbour face nodes are read straight from
      // smem by the first tangential pass, whose results replace them in
      // place for the second pass
      // (vertical faces of div(hV): only V_AX and h are staged and needed --
      // the other components meet an exact zero normal component)
      double* G0 = FGs + WL::fg_off(f);
      constexpr int FC = (OPK == OP_DIVHV && AX < D - 1) ? 2 : KIN;  // passed comps
      auto slot_comp = [&](int r) { return (FC == KIN) ? r : (r == 0 ? AX : D); };
#pragma unroll
      for (int cp = 0; cp < KIN; ++cp) TN[cp] = 0.0;
      double t1[FC];
#pragma unroll
      for (int r = 0; r < FC; ++r) {
        double t1v = 0.0;
        if constexpr (D == 2) {
#pragma unroll
          for (int j = 0; j < N; ++j) t1v = fma(M0[fa * N + j], G0[r * NC + j], t1v);
          TN[slot_comp(r)] = t1v;
        } else {
#pragma unroll
          for (int j = 0; j < N; ++j) t1v = fma(M0[fa * N + j], G0[r * NC + j * N + fb], t1v);
          t1[r] = t1v;
        }
      }
      if constexpr (D == 3) {
        double* S = G0;
        __syncwarp();
#pragma unroll
        for (int r = 0; r < FC; ++r) S[r * NC + c] = t1[r];
        __syncwarp();
#pragma unroll
        for (int r = 0; r < FC; ++r) {
          double t2v = 0.0;
#pragma unroll
          for (int j = 0; j < N; ++j) t2v = fma(M1[fb * N + j], S[r * NC + fa * N + j], t2v);
          TN[slot_comp(r)] = t2v;
        }
      }
    }
    if constexpr (TRM) {
      // trace mode: the neighbour's V / h traces at its face Gauss points
      // are staged; a conforming neighbour's points coincide with ours, a
      // fine leaf maps its coarse parent's through halfq (x) halfq in place
      double* G0 = FGs + WL::fg_off(f);
      constexpr int FC = (AX < D - 1) ? 2 : KIN;
      auto slot_comp = [&](int r) { return (FC == KIN) ? r : (r == 0 ? AX : D); };
#pragma unroll
      for (int cp = 0; cp < KIN; ++cp) TN[cp] = 0.0;
      if (!need_pass) {
#pragma unroll
        for (int r = 0; r < FC; ++r) TN[slot_comp(r)] = G0[r * NC + c];
      } else {
        const bool fine = kd == KIND_FINE;
        double t1[FC];
#pragma unroll
        for (int r = 0; r < FC; ++r) {
          double t1v = 0.0;
          if constexpr (D == 2) {
#pragma unroll
            for (int j = 0; j < N; ++j) t1v = fma(Mq0[fa * N + j], G0[r * NC + j], t1v);
            TN[slot_comp(r)] = fine ? t1v : G0[r * NC + c];
          } else {
#pragma unroll
            for (int j = 0; j < N; ++j) t1v = fma(Mq0[fa * N + j], G0[r * NC + j * N + fb], t1v);
            t1[r] = fine ? t1v : G0[r * NC + c];
          }
        }
        if constexpr (D == 3) {
          double* S = G0;
          __syncwarp();
#pragma unroll
          for (int r = 0; r < FC; ++r) S[r * NC + c] = t1[r];
          __syncwarp();
#pragma unroll
          for (int r = 0; r < FC; ++r) {
            double t2v = 0.0;
#pragma unroll
            for (int j = 0; j < N; ++j) t2v = fma(Mq1[fb * N + j], S[r * NC + fa * N + j], t2v);
            TN[slot_comp(r)] = fine ? t2v : S[r * NC + c];
          }
        }
      }
    }
#pragma unroll
    for (int cp = 0; cp < KIN; ++cp) {
      double gval = 0.0;
      if constexpr (iq && !TRM) {
        if (act && inter) {
          double t = 0.0;
#pragma unroll
          for (int p = 0; p < N; ++p)
            t = fma(TC.lift[1 - side][p],
                    load_input<D, N, OPK>(P, nb, cp, nbr_pencil_node<D, N>(AX, p, c)), t);
          gval = t;
        }
        if (!need_pass) {
          TN[cp] = gval;
        } else {
          const bool fine = kd == KIND_FINE;
          double t1v = 0.0;
          if constexpr (D == 2) {
#pragma unroll
            for (int j = 0; j < N; ++j)
              t1v = fma(Mq0[fa * N + j], __shfl_sync(0xffffffffu, gval, b0 + j), t1v);
            TN[cp] = fine ? t1v : gval;
          } else {
#pragma unroll
            for (int j = 0; j < N; ++j)
              t1v = fma(Mq0[fa * N + j], __shfl_sync(0xffffffffu, gval, b0 + j * N + fb), t1v);
            double t2v = 0.0;
#pragma unroll
            for (int j = 0; j < N; ++j)
              t2v = fma(Mq1[fb * N + j], __shfl_sync(0xffffffffu, t1v, b0 + fa * N + j), t2v);
            TN[cp] = fine ? t2v : gval;
          }
        }
      } else if constexpr (!SMP && !TRM) {
      if (act && inter) {
        gval = load_input<D, N, OPK>(P, nb, cp, nbr_face_node<D, N>(AX, side, c));
      }
      double t1v = 0.0;
      if constexpr (D == 2) {
#pragma unroll
        for (int j = 0; j < N; ++j)
          t1v = fma(M0[fa * N + j], __shfl_sync(0xffffffffu, gval, b0 + j), t1v);
        TN[cp] = t1v;
      } else {
#pragma unroll
        for (int j = 0; j < N; ++j)
          t1v = fma(M0[fa * N + j], __shfl_sync(0xffffffffu, gval, b0 + j * N + fb), t1v);
        double t2v = 0.0;
#pragma unroll
        for (int j = 0; j < N; ++j)
          t2v = fma(M1[fb * N + j], __shfl_sync(0xffffffffu, t1v, b0 + fa * N + j), t2v);
        TN[cp] = t2v;
      }
      }  // nodal input
      // own trace: lift contraction of the lane's pencil along AX (vertical
      // faces of div(hV): only V_AX and h meet a non-zero normal component)
      if (OPK == OP_DIVHV && AX < D - 1 && cp != AX && cp != D) {
        TO[cp] = 0.0;
      } else {
        double t = 0.0;
#pragma unroll
        for (int k = 0; k < N; ++k) {
          const int off = (AX == D - 1) ? coff<D, N>(c, k)
                        : (AX == 0)     ? xoff<D, N>(c, k)
                                        : yoff<N>(c, k);
          t = fma(TC.lift[side][k], X[cp * TSZ + off], t);
        }
        TO[cp] = t;
      }
    }
    if (kd == KIND_COARSE || !act) {
      // coarse side of a hanging face: its lifted flux was precomputed by
      // coarse_kernel (flux mode, mesh.cflux), else added afterwards
      const bool cf = act && kd == KIND_COARSE && mesh.cflux != nullptr;
#pragma unroll
      for (int k = 0; k < KOUT; ++k)
        fl[f][k] = cf ? mesh.cflux[(nb * KOUT + k) * NC + c] : 0.0;
      return;
    }
    const bool outward = (kd == KIND_WALL || kd == KIND_FARFIELD);
    // the face metric from this element's own geometry: a conforming
    // neighbour shares the face, so its (minus-side) metric is the same
    // values up to rounding in the corner coordinates
    double n[D], ws;
    if constexpr (WL::ASYNC)
      face_metric_ge<D, N, AX>(P.gc, g, side, outward, c, TS, GEs, NC, n, ws);
    else
      face_metric_ax<D, N, AX>(P.gc, mesh.col, g, side, outward, c, TS, n, ws);
    if (outward) ghost<D, N, OPK, KIN>(P, kd, nb, c, TO, n, TN);
    const bool minus = outward || side == 1;
    double TLv[KIN], TRv[KIN];
#pragma unroll
    for (int cp = 0; cp < KIN; ++cp) {
      TLv[cp] = minus ? TO[cp] : TN[cp];
      TRv[cp] = minus ? TN[cp] : TO[cp];
    }
    double fv[KOUT];
    num_flux<D, OPK, KIN, KOUT>(TLv, TRv, n, P.model.kinetic_factor, fv);
    const double sg = minus ? ws : -ws;
#pragma unroll
    for (int k = 0; k < KOUT; ++k) fl[f][k] = fv[k] * sg;
  };
  // each lane reads back only the face slots it issued itself
  cp_async_wait_all();  // this thread's staged copies (tables, face nodes) landed
  __syncthreads();      // ... and every thread's: the tables are visible CTA-wide
  if constexpr (SMP) {
    if constexpr (OPK == OP_GRAD) {
      // p = alpha (x - beta K) at the staged nodes, in place (own slots)
#pragma unroll
      for (int f = 0; f < NF; ++f) {
        const double xv = FGs[WL::fg_off(f) + c];
        FGs[WL::fg_off(f) + c] =
            P.has_K ? P.alpha * (xv - P.beta * FGs[WL::fg_off(f) + NC + c]) : P.alpha * xv;
      }
    }
    __syncwarp();  // staged nodes visible warp-wide; the tile is free
  }
  face(std::integral_constant<int, 0>{}, 0);
  face(std::integral_constant<int, 0>{}, 1);
  face(std::integral_constant<int, 1>{}, 0);
  face(std::integral_constant<int, 1>{}, 1);
  if constexpr (D == 3) {
    face(std::integral_constant<int, 2>{}, 0);
    face(std::integral_constant<int, 2>{}, 1);
  }
  // the epilogue's base values (the x-pencil nodes this lane stores) are
  // copied into the face-node area, now consumed, under the volume work
  const bool pre_base = WL::ASYNC && act && P.mode == OUT_MINV && P.has_base && !P.out_quad;
  double* BSs = FGs;
  if (pre_base) {
#pragma unroll
    for (int k = 0; k < KOUT; ++k)
#pragma unroll
      for (int ii = 0; ii < N; ++ii) {
        const int node = (D == 3) ? ii * N * N + c : ii * N + c;
        cp_async8(BSs + (k * N + ii) * NC + c, P.base.p + es * P.base.estride +
                                                   (long long)k * P.base.cstride + node);
      }
  }

  // ---- 4. volume: metric + flux per column point -------------------------
  __syncwarp();  // every lane is done reading Q from the tile
  double Zc[KOUT][N];
  double det_c = 1.0;  // det J is z-independent: one value per column
  // the column's horizontal quadrature weight, from the smem tables (a
  // lane-dependent index into the parameter bank would serialise the warp)
  const double wcol = (D == 3) ? TS.qw[c / N] * TS.qw[c % N] : TS.qw[c];
  {
    double Gz[KOUT][N];
#pragma unroll
    for (int kz = 0; kz < N; ++kz) {
      const int qp = c * N + kz;
      double det, ctrv[D][D];
      if (WL::ASYNC && !flat)
        point_metric_ge<D, N>(P.gc, TC, g, kz, GEs, NC, c, det, ctrv);
      else
        point_metric<D, N>(P, g, qp, det, ctrv);
      const double wq = wcol * TC.qw[kz];  // = point_weight(qp), same product order
      double F[D][KOUT];
      if constexpr (OPK == OP_DIVHV) {
        // own column of the Gauss-point tile (read before G overwrites it)
        const double h = X[D * TSZ + coff<D, N>(c, kz)];
#pragma unroll
        for (int a = 0; a < D; ++a) F[a][0] = h * X[a * TSZ + coff<D, N>(c, kz)];
      } else {
        const double p = X[coff<D, N>(c, kz)];
#pragma unroll
        for (int a = 0; a < D; ++a)
#pragma unroll
          for (int k = 0; k < KOUT; ++k) F[a][k] = (a == k) ? p : 0.0;
      }
#pragma unroll
      for (int bx = 0; bx < D; ++bx) {
#pragma unroll
        for (int k = 0; k < KOUT; ++k) {
          double acc;
          if (OPK == OP_GRAD) {
            acc = F[k][k] * ctrv[bx][k];
          } else if (flat) {
            acc = F[bx][k] * ctrv[bx][bx];
          } else {
            acc = 0.0;
#pragma unroll
            for (int a = 0; a < D; ++a) acc += F[a][k] * ctrv[bx][a];
          }
          acc *= wq;
          if (bx == D - 1) {
            Gz[k][kz] = acc;
          } else if (OPK == OP_GRAD) {
            if (k == bx) X[(bx * KW) * TSZ + coff<D, N>(c, kz)] = acc;
          } else {
            X[(bx * KW + k) * TSZ + coff<D, N>(c, kz)] = acc;
          }
        }
      }
      det_c = det;
    }
    // z direction in registers: Zc = -Dhat^T Gz + z-face lifts
#pragma unroll
    for (int k = 0; k < KOUT; ++k) {
      mat_apply<N, true>(TC.Dhat, Gz[k], Zc[k]);
#pragma unroll
      for (int kz = 0; kz < N; ++kz)
        Zc[k][kz] = TC.lift[0][kz] * fl[2 * (D - 1)][k] + TC.lift[1][kz] * fl[2 * (D - 1) + 1][k] -
                    Zc[k][kz];
    }
  }
  __syncwarp();
  // x (and y) directions on the lane's pencils, with that direction's lifts
#pragma unroll
  for (int k = 0; k < KW; ++k) {
    const int kx = (OPK == OP_GRAD) ? 0 : k;
    double* T0 = X + (0 * KW + k) * TSZ;
    double v[N], o[N];
#pragma unroll
    for (int ii = 0; ii < N; ++ii) v[ii] = T0[xoff<D, N>(c, ii)];
    mat_apply<N, true>(TC.Dhat, v, o);
#pragma unroll
    for (int ii = 0; ii < N; ++ii)
      T0[xoff<D, N>(c, ii)] = TC.lift[0][ii] * fl[0][kx] + TC.lift[1][ii] * fl[1][kx] - o[ii];
    if constexpr (D == 3) {
      const int ky = (OPK == OP_GRAD) ? 1 : k;
      double* T1 = X + (1 * KW + k) * TSZ;
#pragma unroll
      for (int jj = 0; jj < N; ++jj) v[jj] = T1[yoff<N>(c, jj)];
      mat_apply<N, true>(TC.Dhat, v, o);
#pragma unroll
      for (int jj = 0; jj < N; ++jj)
        T1[yoff<N>(c, jj)] = TC.lift[0][jj] * fl[2][ky] + TC.lift[1][jj] * fl[3][ky] - o[jj];
    }
  }
  __syncwarp();
#pragma unroll
  for (int kz = 0; kz < N; ++kz) {
    if constexpr (OPK == OP_GRAD) {
      Zc[0][kz] += X[0 * TSZ + coff<D, N>(c, kz)];
      if constexpr (D == 3) Zc[1][kz] += X[1 * TSZ + coff<D, N>(c, kz)];
    } else {
#pragma unroll
      for (int k = 0; k < KOUT; ++k) {
        Zc[k][kz] += X[(0 * KW + k) * TSZ + coff<D, N>(c, kz)];
        if constexpr (D == 3) Zc[k][kz] += X[(1 * KW + k) * TSZ + coff<D, N>(c, kz)];
      }
    }
  }
  // ---- 5. epilogue: B^-1 diag(1/(w det)) (MINV) or B^T (DUAL) -----------
  const bool minv = (P.mode == OUT_MINV);
  // 1/(w det): det is z-independent, 1/w a product of 1D reciprocals
  double iwh = 1.0 / det_c;
  if constexpr (D == 3) iwh *= TS.iqw[c / N] * TS.iqw[c % N];
  else iwh *= TS.iqw[c];
  if (OPK == OP_GRAD && P.out_quad) {
    // H1 of the Helmholtz pair: V = coef * diag(1/(w det)) Z at the Gauss
    // points -- the B^-1 transform and H2's B interpolation cancel exactly
    double Vg[KOUT][N];
#pragma unroll
    for (int k = 0; k < KOUT; ++k)
#pragma unroll
      for (int kz = 0; kz < N; ++kz) Vg[k][kz] = P.coef * (Zc[k][kz] * (iwh * TC.iqw[kz]));
    if (act) {
#pragma unroll
      for (int k = 0; k < KOUT; ++k) {
        double* out = P.out.p + e * P.out.estride + (long long)k * P.out.cstride + c * N;
#pragma unroll
        for (int kz = 0; kz < N; ++kz) out[kz] = Vg[k][kz];
      }
    }
    if (P.tr_out != nullptr) {
      // trace mode: V's traces at the face Gauss points (lift contractions of
      // the Gauss pencils): every component on the z faces from the lane's
      // column, the normal component on the vertical faces through the tile
      constexpr int TSL = tr_slots<D>() * NC;
      double* tr = P.tr_out + es * TSL;
#pragma unroll
      for (int side = 0; side < 2; ++side)
#pragma unroll
        for (int k = 0; k < D; ++k) {
          double t = 0.0;
#pragma unroll
          for (int kz = 0; kz < N; ++kz) t = fma(TC.lift[side][kz], Vg[k][kz], t);
          if (act) tr[tr_slot<D>(2 * (D - 1) + side, k) * NC + c] = t;
        }
      __syncwarp();  // every lane is done with the tile
#pragma unroll
      for (int a = 0; a < D - 1; ++a)
#pragma unroll
        for (int kz = 0; kz < N; ++kz) X[a * TSZ + coff<D, N>(c, kz)] = Vg[a][kz];
      __syncwarp();
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
          if (act) tr[tr_slot<D>(2 * a + side, a) * NC + c] = t;
        }
    }
    return;
  }
#pragma unroll
  for (int k = 0; k < KOUT; ++k) {
    double t[N];
    if (minv) {
#pragma unroll
      for (int kz = 0; kz < N; ++kz) t[kz] = Zc[k][kz] * (iwh * TC.iqw[kz]);
      mat_apply<N, false>(TC.Binv, t, Zc[k]);
    } else {
#pragma unroll
      for (int kz = 0; kz < N; ++kz) t[kz] = Zc[k][kz];
      mat_apply<N, true>(TC.B, t, Zc[k]);
    }
  }
  __syncwarp();
#pragma unroll
  for (int k = 0; k < KOUT; ++k)
#pragma unroll
    for (int kz = 0; kz < N; ++kz) X[k * TSZ + coff<D, N>(c, kz)] = Zc[k][kz];
  __syncwarp();
  if constexpr (D == 3) {
#pragma unroll
    for (int k = 0; k < KOUT; ++k) {
      double v[N], o[N];
#pragma unroll
      for (int jj = 0; jj < N; ++jj) v[jj] = X[k * TSZ + yoff<N>(c, jj)];
      if (minv) mat_apply<N, false>(TC.Binv, v, o);
      else mat_apply<N, true>(TC.B, v, o);
#pragma unroll
      for (int jj = 0; jj < N; ++jj) X[k * TSZ + yoff<N>(c, jj)] = o[jj];
    }
    __syncwarp();
  }
  if (pre_base) cp_async_wait_all();
  // x pass and store from the x-pencil: points (ii, [j,] k) of lane c
  double wv[N];  // the stored values (KOUT == 1 when the dots are fused)
  double uv[N];  // their base values (the Helmholtz action's input u)
#pragma unroll
  for (int ii = 0; ii < N; ++ii) wv[ii] = uv[ii] = 0.0;
  if (act) {
#pragma unroll
    for (int k = 0; k < KOUT; ++k) {
      double v[N], o[N];
#pragma unroll
      for (int ii = 0; ii < N; ++ii) v[ii] = X[k * TSZ + xoff<D, N>(c, ii)];
      if (minv) mat_apply<N, false>(TC.Binv, v, o);
      else mat_apply<N, true>(TC.B, v, o);
#pragma unroll
      for (int ii = 0; ii < N; ++ii) {
        const int node = (D == 3) ? ii * N * N + c : ii * N + c;
        double* out = P.out.p + e * P.out.estride + (long long)k * P.out.cstride + node;
        double val;
        if (!minv) {
          val = o[ii];
        } else {
          const double r = __dmul_rn(P.coef, o[ii]);
          const double bv = pre_base ? BSs[(k * N + ii) * NC + c]
                                     : (P.has_base ? P.base(e, k, node) : 0.0);
          val = (pre_base || P.has_base) ? __dadd_rn(bv, r) : r;
          uv[ii] = bv;
        }
        *out = val;
        wv[ii] = val;
      }
    }
  }
  if constexpr (OPK == OP_DIVHV) {
    if (P.gs_part != nullptr) gs_dots<D, N, OPK>(P, smem, kf, act, e, c, wv, uv);
  }
}

}  // namespace dg
