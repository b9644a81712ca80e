// Warp-element kernel for the explicit (advective) operator, fp64, sm_100a:
// SplitOperators.explicit_residual (imex.py:144-159) = -M^-1 weak_form with
// the split advective volume flux (dgops.py:234-254), Rusanov faces with the
// flow speed (dgops.py:256-283), mortar traces on the fine side of hanging
// faces (dgops.py:159-206), wall / far-field ghosts (boundary.py:17-84),
// gravity (physics.py:207-216) and the Rayleigh sponge, plus the full-flux
// divergence of dgops.py:298-328 (P.full) and the plain dual (OUT_DUAL).
//
// Same decomposition as the Helmholtz pair's welem_kernel (dg_wkernel.cuh):
// NC = n^(d-1) consecutive lanes of one warp own an element, lane c holds
// z-column c in registers and face point c of every face.  With d+2
// conserved variables the per-element working set is larger, so each
// element slot carries three smem areas:
//   X   (V x TSZ)  Gauss-point values Q, then the x-direction volume terms;
//   GY  (V x TSZ)  y-direction volume terms (3D);
//   FG  (2d x V x NC)  the neighbours' nodal face values (cp.async, issued
//       with the own-column loads), replaced face by face by the lane's
//       numerical flux * ws once that face is done;
//   GE  terrain scalars of the column (as welem_kernel).
// z-face fluxes and the z direction stay in registers; x / y directions go
// through the tile with __syncwarp() only.  The coarse side of hanging faces
// is added afterwards by coarse_kernel (dg_kernel.cuh), unchanged.
#pragma once
#include "dg_wkernel.cuh"

namespace dg {

// Gauss-point metric (as point_metric_ge) from the column's terrain scalars
// held in registers (omh = 1 - h/z_top, dh = grad h at the column)
template <int D, int N>
__device__ __forceinline__ void point_metric_reg(const GeoConst& gc, const Tab<N>& T,
                                                 const ElemGeo<D>& g, int qz, double omh,
                                                 const double* dh, double& det,
                                                 double ctrv[D][D]) {
  constexpr int HD = D - 1;
  const double zz = g.s[D - 1] * omh;
  det = 1.0;
#pragma unroll
  for (int a = 0; a < HD; ++a) det = det * g.s[a];
  det = det * zz;
  const double decay = 1.0 - (g.lo[D - 1] + g.s[D - 1] * T.qx[qz]) * gc.inv_ztop;
  double zg[2];
#pragma unroll
  for (int a = 0; a < HD; ++a) zg[a] = dh[a] * g.s[a] * decay;
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

// smem-only component loops are kept rolled (instruction-cache footprint of
// the d+2-variable kernel); DG_XUNROLL=1 unrolls them
#if defined(DG_XUNROLL) && DG_XUNROLL == 1
#define XROLL _Pragma("unroll")
#elif defined(DG_XUNROLL) && DG_XUNROLL == 2
#define XROLL _Pragma("unroll 2")
#elif defined(DG_XUNROLL) && DG_XUNROLL == 3
#define XROLL _Pragma("unroll 3")
#else
#define XROLL _Pragma("unroll 1")
#endif

// staging area of face f's neighbour nodes (see XLayout::NFG)
template <int D, int V, int NC>
__device__ __forceinline__ double* fstage(double* FG, double* GY, int f) {
  if (D == 3 && f >= 2 * (D - 1)) return GY + (f - 2 * (D - 1)) * V * NC;
  return FG + f * V * NC;
}

template <int D, int N>
struct XLayout {
  static constexpr int V = D + 2;
  static constexpr int NP = ipow(N, D);
  static constexpr int NC = ipow(N, D - 1);  // lanes per element
  // a team owns whole elements: one warp for n^(d-1) <= 32, two warps on a
  // named barrier for 3D r = 5, 6 (dg_hkernel.cuh esync)
  static constexpr int TPE = NC <= 32 ? 32 : 64;
  static constexpr int EPW = TPE / NC;         // elements per team
  static constexpr int TSZ = tile_size<D, N>();  // one tensor (tile layout: coff)
#ifndef DG_XWPB
#define DG_XWPB 1
#endif
  static constexpr int TEAMS = DG_XWPB;        // teams per CTA
  static constexpr int WPB = TEAMS * TPE / 32;  // warps per CTA (mass-rate partial rows)
  static constexpr int THREADS = 32 * WPB;
  static constexpr int TABD = (int)(sizeof(Tab<N>) / sizeof(double));
  static constexpr int NSLOT = EPW + ((TPE % NC) ? 1 : 0);
  static constexpr int GEON = 1 + (D - 1);
  static constexpr int NE = ipow(N, D - 2);
  static constexpr int GEE = 2 * (D - 1) * NE;
  static constexpr int OFF_X = 0;
  static constexpr int OFF_GY = OFF_X + V * TSZ;
  static constexpr int OFF_FG = OFF_GY + (D == 3 ? V * TSZ : 0);
  // 3D: the z faces' staged nodes live in the GY tile, free until the
  // volume phase (FG keeps the x / y faces, later their fluxes)
  static constexpr int NFG = (D == 3) ? 2 * (D - 1) : 2 * D;
  static constexpr int OFF_GE = OFF_FG + NFG * V * NC;
  static constexpr int SLOT0 = OFF_GE + GEON * NC + GEE;
  static constexpr int SLOT = (SLOT0 % 2 == 0) ? SLOT0 + 1 : SLOT0;  // bank shift
  static constexpr size_t SMEM = (size_t)(TABD + WPB * NSLOT * SLOT) * sizeof(double);
  // two-warp teams (r = 5, 6) compile but measured slower than the CTA
  // kernel (255 registers: cfg5 r=5 5.9 vs 5.0 ms, r=6 12.2 vs 7.5 ms), so
  // the explicit operator keeps one-warp teams
  static constexpr bool OK = (NC <= 32) && (SMEM <= 200 * 1024);
#ifndef DG_XMINB
#define DG_XMINB 11
#endif
  static constexpr int MINB = TPE == 32 ? DG_XMINB : 4;
};

// FULL: divergence_full (P.full != 0) -- a separate instantiation keeps the
// full Euler flux out of the explicit residual's code
template <int D, int N, bool FULL>
__global__ void __launch_bounds__(XLayout<D, N>::THREADS, XLayout<D, N>::MINB)
xelem_kernel(const __grid_constant__ KParams<N> P) {
  using XL = XLayout<D, N>;
  constexpr int NC = XL::NC, EPW = XL::EPW, V = XL::V, TSZ = XL::TSZ, NF = 2 * D;
  constexpr int NP = XL::NP;
  extern __shared__ double smem[];
  for (int i = threadIdx.x; i < XL::TABD; i += blockDim.x) cp_async8(smem + i, P.tab_g + i);
  const Tab<N>& TS = *reinterpret_cast<const Tab<N>*>(smem);
  const Tab<N>& TC = P.tab;
  const MeshDev& mesh = P.mesh;
  const Model& md = P.model;
  const int lane = threadIdx.x % XL::TPE;  // lane in the team
  const int wid = threadIdx.x / XL::TPE;   // team
  const int eiw = lane / NC;
  const int c = lane - eiw * NC;
  const bool slot_ok = eiw < EPW;
  const long long e = ((long long)blockIdx.x * XL::TEAMS + wid) * EPW + eiw;
  const bool act = slot_ok && e < mesh.n_el;
  const long long es = act ? e : 0;
  double* S = smem + XL::TABD + (wid * XL::NSLOT + (slot_ok ? eiw : EPW)) * XL::SLOT;
  double* X = S + XL::OFF_X;
  double* GY = S + XL::OFF_GY;
  double* FG = S + XL::OFF_FG;
  double* GE = S + XL::OFF_GE;
  const bool flat = !P.gc.terrain;

  // ---- 0. records, own column, neighbour face nodes (async) -------------
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
  double q[V][N];
#pragma unroll
  for (int r = 0; r < V; ++r)
#pragma unroll
    for (int k = 0; k < N; ++k) q[r][k] = act ? P.in(es, r, c * N + k) : 0.0;
#pragma unroll
  for (int f = 0; f < NF; ++f) {
    const int kd = kf[f] & 15;
    const bool inter = act && (kd == KIND_CONF || kd == KIND_FINE);
    const long long nb = nf[f];
    const int node = nbr_face_node<D, N>(f >> 1, f & 1, c);
#pragma unroll
    for (int r = 0; r < V; ++r) {
      double* dst = fstage<D, V, NC>(FG, GY, f) + r * NC + c;
      if (inter) cp_async8(dst, P.in.p + nb * P.in.estride + r * P.in.cstride + node);
      else *dst = 0.0;
    }
  }
  if (!flat && act) {
    const double* colp = mesh.col + (long long)g.col * P.gc.col_stride;
#pragma unroll
    for (int i = 0; i < XL::GEON; ++i) cp_async8(GE + i * NC + c, colp + geo_src<D, N>(i, c));
    constexpr int NQH = ipow(N, D - 1);
    for (int i = c; i < XL::GEE; i += NC) cp_async8(GE + XL::GEON * NC + i, colp + NQH * D + i);
  }

  // ---- 1. nodes -> Gauss points: z in registers, y / x through the tile --
#pragma unroll
  for (int r = 0; r < V; ++r) {
    double o[N];
    mat_apply<N, false>(TC.B, q[r], o);
#pragma unroll
    for (int k = 0; k < N; ++k) X[r * TSZ + coff<D, N>(c, k)] = o[k];
  }
  esync<XL::TPE>(wid);
  if constexpr (D == 3) {
XROLL
    for (int r = 0; r < V; ++r) {
      double v[N], o[N];
#pragma unroll
      for (int jj = 0; jj < N; ++jj) v[jj] = X[r * TSZ + yoff<N>(c, jj)];
      mat_apply<N, false>(TC.B, v, o);
#pragma unroll
      for (int jj = 0; jj < N; ++jj) X[r * TSZ + yoff<N>(c, jj)] = o[jj];
    }
    esync<XL::TPE>(wid);
  }
XROLL
  for (int r = 0; r < V; ++r) {
    double v[N], o[N];
#pragma unroll
    for (int ii = 0; ii < N; ++ii) v[ii] = X[r * TSZ + xoff<D, N>(c, ii)];
    mat_apply<N, false>(TC.B, v, o);
#pragma unroll
    for (int ii = 0; ii < N; ++ii) X[r * TSZ + xoff<D, N>(c, ii)] = o[ii];
  }
  cp_async_wait_all();  // this thread's staged copies (tables, face nodes, terrain)
  __syncthreads();      // ... and every thread's (the tables are CTA-wide)

  // ---- 2. faces: Rusanov flux at face point c of every face --------------
  double flz[2][V];  // z faces: flux * (+-ws), kept for the z lift
  auto face = [&](auto ax_c, int side) {
    constexpr int AX = decltype(ax_c)::value;
    const int f = 2 * AX + side;
    const uint8_t kraw = kf[f];
    const int kd = kraw & 15;
    const int fa = (D == 2) ? c : c / N;
    const int fb = (D == 2) ? 0 : c % N;
    const int sf = (kraw >> 4) & 3;
    const double* M0 = (kd == KIND_FINE) ? &TS.half[sf & 1][0][0] : &TS.B[0][0];
    const double* M1 = (kd == KIND_FINE) ? &TS.half[(sf >> 1) & 1][0][0] : &TS.B[0][0];
    double* G0 = fstage<D, V, NC>(FG, GY, f);
    double TN[V], TO[V];
    // neighbour trace: tangential passes straight from the staged nodes
    double t1[V];
#pragma unroll
    for (int r = 0; r < V; ++r) {
      double t = 0.0;
      if constexpr (D == 2) {
#pragma unroll
        for (int j = 0; j < N; ++j) t = fma(M0[fa * N + j], G0[r * NC + j], t);
        TN[r] = t;
      } else {
#pragma unroll
        for (int j = 0; j < N; ++j) t = fma(M0[fa * N + j], G0[r * NC + j * N + fb], t);
        t1[r] = t;
      }
    }
    if constexpr (D == 3) {
      esync<XL::TPE>(wid);
#pragma unroll
      for (int r = 0; r < V; ++r) G0[r * NC + c] = t1[r];
      esync<XL::TPE>(wid);
#pragma unroll
      for (int r = 0; r < V; ++r) {
        double t = 0.0;
#pragma unroll
        for (int j = 0; j < N; ++j) t = fma(M1[fb * N + j], G0[r * NC + fa * N + j], t);
        TN[r] = t;
      }
    }
    // own trace: lift contraction of the lane's Gauss pencil along AX
#pragma unroll
    for (int r = 0; r < V; ++r) {
      double t = 0.0;
#pragma unroll
      for (int k = 0; k < N; ++k) {
        const int off = (AX == D - 1) ? coff<D, N>(c, k) : (AX == 0) ? xoff<D, N>(c, k) : yoff<N>(c, k);
        t = fma(TC.lift[side][k], X[r * TSZ + off], t);
      }
      TO[r] = t;
    }
    double fv[V];
    if (kd == KIND_COARSE || !act) {
      // coarse side of a hanging face: precomputed by coarse_kernel (flux mode)
      const bool cf = act && kd == KIND_COARSE && mesh.cflux != nullptr;
#pragma unroll
      for (int k = 0; k < V; ++k)
        fv[k] = cf ? mesh.cflux[((long long)nf[f] * V + k) * NC + c] : 0.0;
    } else {
      const bool outward = (kd == KIND_WALL || kd == KIND_FARFIELD);
      double n[D], ws;
      face_metric_ge<D, N, AX>(P.gc, g, side, outward, c, TS, GE, NC, n, ws);
      if (outward) ghost<D, N, OP_ADV, V>(P, kd, nf[f], c, TO, n, TN);
      const bool minus = outward || side == 1;
      double TL[V], TR[V];
#pragma unroll
      for (int k = 0; k < V; ++k) {
        TL[k] = minus ? TO[k] : TN[k];
        TR[k] = minus ? TN[k] : TO[k];
      }
      num_flux<D, OP_ADV, V, V>(TL, TR, n, md.kinetic_factor, fv, &md, FULL ? P.full : 0);
      const double sg = minus ? ws : -ws;
#pragma unroll
      for (int k = 0; k < V; ++k) fv[k] *= sg;
    }
    if constexpr (AX == D - 1) {
#pragma unroll
      for (int k = 0; k < V; ++k) {
        if (side == 0) flz[0][k] = fv[k];
        else flz[1][k] = fv[k];
      }
    } else {
      esync<XL::TPE>(wid);  // every lane is done reading this face's staged nodes
#pragma unroll
      for (int k = 0; k < V; ++k) G0[k * NC + c] = fv[k];
    }
  };
  // both sides unrolled (DG_XSIDEUNROLL=0: one code copy per axis, measured slower)
#if !defined(DG_XSIDEUNROLL) || DG_XSIDEUNROLL
#pragma unroll
#else
#pragma unroll 1
#endif
  for (int side = 0; side < 2; ++side) face(std::integral_constant<int, 0>{}, side);
  if constexpr (D == 3) {
#if !defined(DG_XSIDEUNROLL) || DG_XSIDEUNROLL
#pragma unroll
#else
#pragma unroll 1
#endif
    for (int side = 0; side < 2; ++side) face(std::integral_constant<int, 1>{}, side);
  }
#if !defined(DG_XSIDEUNROLL) || DG_XSIDEUNROLL
#pragma unroll
#else
#pragma unroll 1
#endif
  for (int side = 0; side < 2; ++side) face(std::integral_constant<int, D - 1>{}, side);
  esync<XL::TPE>(wid);  // every lane is done reading the Gauss tile's pencils

  // ---- 3. volume: flux + metric per column point ------------------------
  double omh_c = 1.0, dh_c[D - 1];
#pragma unroll
  for (int a = 0; a < D - 1; ++a) dh_c[a] = 0.0;
  if (!flat) {
    omh_c = GE[c];
#pragma unroll
    for (int a = 0; a < D - 1; ++a) dh_c[a] = GE[(1 + a) * NC + c];
  }
  double Zc[V][N];
  double det_c = 1.0;
  {
    double Gz[V][N];
#pragma unroll
    for (int kz = 0; kz < N; ++kz) {
      double det, ctrv[D][D];
      if (!flat) {
        point_metric_reg<D, N>(P.gc, TC, g, kz, omh_c, dh_c, det, ctrv);
      } else {
#pragma unroll
        for (int b = 0; b < D; ++b)
#pragma unroll
          for (int a = 0; a < D; ++a) ctrv[b][a] = 0.0;
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
      }
      det_c = det;
      double wq = TC.qw[kz];
      if constexpr (D == 3) wq *= TS.qw[c / N] * TS.qw[c % N];  // smem: lane-dependent index
      else wq *= TS.qw[c];
      double Uq[V];
#pragma unroll
      for (int r = 0; r < V; ++r) Uq[r] = X[r * TSZ + coff<D, N>(c, kz)];
      double F[D][V];
      if (FULL) {
        double Ff[V][D];
        full_flux<D>(Uq, md, Ff);
#pragma unroll
        for (int a = 0; a < D; ++a)
#pragma unroll
          for (int r = 0; r < V; ++r) F[a][r] = Ff[r][a];
      } else {
        // split advective flux (dgops.py:234-254)
        const double rho = Uq[0];
        const double irho = DG_ADV_RCP ? __drcp_rn(rho) : 0.0;
        double u[D];
        double k = 0.0;
#pragma unroll
        for (int a = 0; a < D; ++a) {
          u[a] = DG_ADV_RCP ? Uq[1 + a] * irho : Uq[1 + a] / rho;
          k += u[a] * u[a];
        }
        k *= 0.5;
#pragma unroll
        for (int a = 0; a < D; ++a) {
          F[a][0] = Uq[1 + a];
#pragma unroll
          for (int b = 0; b < D; ++b) F[a][1 + b] = Uq[1 + b] * u[a];
          F[a][D + 1] = md.kinetic_factor * rho * k * u[a];
        }
      }
#pragma unroll
      for (int bx = 0; bx < D; ++bx) {
#pragma unroll
        for (int r = 0; r < V; ++r) {
          double acc;
          if (flat) {
            acc = F[bx][r] * ctrv[bx][bx];
          } else {
            acc = 0.0;
#pragma unroll
            for (int a = 0; a < D; ++a) acc += F[a][r] * ctrv[bx][a];
          }
          acc *= wq;
          if (bx == D - 1) Gz[r][kz] = acc;
          else if (bx == 0) X[r * TSZ + coff<D, N>(c, kz)] = acc;  // own column, in place
          else GY[r * TSZ + coff<D, N>(c, kz)] = acc;
        }
      }
    }
    // z direction in registers: Zc = lifts(z faces) - Dhat^T Gz
#pragma unroll
    for (int r = 0; r < V; ++r) {
      mat_apply<N, true>(TC.Dhat, Gz[r], Zc[r]);
#pragma unroll
      for (int kz = 0; kz < N; ++kz)
        Zc[r][kz] = TC.lift[0][kz] * flz[0][r] + TC.lift[1][kz] * flz[1][r] - Zc[r][kz];
    }
  }
  esync<XL::TPE>(wid);
  // x (and y) directions on the lane's pencils, with that direction's lifts
XROLL
  for (int r = 0; r < V; ++r) {
    double v[N], o[N];
    const double f0 = FG[(0 * V + r) * NC + c], f1 = FG[(1 * V + r) * NC + c];
#pragma unroll
    for (int ii = 0; ii < N; ++ii) v[ii] = X[r * TSZ + xoff<D, N>(c, ii)];
    mat_apply<N, true>(TC.Dhat, v, o);
#pragma unroll
    for (int ii = 0; ii < N; ++ii)
      X[r * TSZ + xoff<D, N>(c, ii)] = TC.lift[0][ii] * f0 + TC.lift[1][ii] * f1 - o[ii];
    if constexpr (D == 3) {
      const double f2 = FG[(2 * V + r) * NC + c], f3 = FG[(3 * V + r) * NC + c];
#pragma unroll
      for (int jj = 0; jj < N; ++jj) v[jj] = GY[r * TSZ + yoff<N>(c, jj)];
      mat_apply<N, true>(TC.Dhat, v, o);
#pragma unroll
      for (int jj = 0; jj < N; ++jj)
        GY[r * TSZ + yoff<N>(c, jj)] = TC.lift[0][jj] * f2 + TC.lift[1][jj] * f3 - o[jj];
    }
  }
  esync<XL::TPE>(wid);
#pragma unroll
  for (int r = 0; r < V; ++r)
#pragma unroll
    for (int kz = 0; kz < N; ++kz) {
      Zc[r][kz] += X[r * TSZ + coff<D, N>(c, kz)];
      if constexpr (D == 3) Zc[r][kz] += GY[r * TSZ + coff<D, N>(c, kz)];
    }

  // mass rate: per-warp partial of the density dual (imex.py:148; the dual's
  // node sum equals its Gauss-coordinate sum, rows of B sum to one)
  if (P.mass_partial != nullptr) {
    double v = 0.0;
    if (act) {
#pragma unroll
      for (int kz = 0; kz < N; ++kz) v += Zc[0][kz];
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if ((threadIdx.x & 31) == 0)  // one row per warp
      P.mass_partial[(long long)blockIdx.x * XL::WPB + (threadIdx.x >> 5)] = v;
  }

  // ---- 4. epilogue: B^-1 diag(1/(w det)) (MINV) or B^T (DUAL) -----------
  const bool minv = (P.mode == OUT_MINV);
  // the source terms' inputs at the lane's output nodes, loaded now so their
  // latency hides under the B^-1 passes
  double uin[V][N], bgv[V][N], sgm[N];
  const bool src = act && minv;
  const bool spg = src && P.sigma != nullptr;
#pragma unroll
  for (int ii = 0; ii < N; ++ii) {
    const int node = (D == 3) ? ii * N * N + c : ii * N + c;
#pragma unroll
    for (int r = 0; r < V; ++r) {
      uin[r][ii] = (src && (r == 0 || r == D || spg)) ? P.in(e, r, node) : 0.0;
      bgv[r][ii] = (spg && r > 0) ? P.bg(e, r, node) : 0.0;
    }
    sgm[ii] = spg ? P.sigma[e * NP + node] : 0.0;
  }
  double iwh = 1.0 / det_c;
  if constexpr (D == 3) iwh *= TS.iqw[c / N] * TS.iqw[c % N];
  else iwh *= TS.iqw[c];
#pragma unroll
  for (int r = 0; r < V; ++r) {
    double t[N];
    if (minv) {
#pragma unroll
      for (int kz = 0; kz < N; ++kz) t[kz] = Zc[r][kz] * (iwh * TC.iqw[kz]);
      mat_apply<N, false>(TC.Binv, t, Zc[r]);
    } else {
#pragma unroll
      for (int kz = 0; kz < N; ++kz) t[kz] = Zc[r][kz];
      mat_apply<N, true>(TC.B, t, Zc[r]);
    }
  }
  esync<XL::TPE>(wid);
#pragma unroll
  for (int r = 0; r < V; ++r)
#pragma unroll
    for (int kz = 0; kz < N; ++kz) X[r * TSZ + coff<D, N>(c, kz)] = Zc[r][kz];
  esync<XL::TPE>(wid);
  if constexpr (D == 3) {
XROLL
    for (int r = 0; r < V; ++r) {
      double v[N], o[N];
#pragma unroll
      for (int jj = 0; jj < N; ++jj) v[jj] = X[r * TSZ + yoff<N>(c, jj)];
      if (minv) mat_apply<N, false>(TC.Binv, v, o);
      else mat_apply<N, true>(TC.B, v, o);
#pragma unroll
      for (int jj = 0; jj < N; ++jj) X[r * TSZ + yoff<N>(c, jj)] = o[jj];
    }
    esync<XL::TPE>(wid);
  }
  if (!act) return;
  // x pass and store from the x-pencil: nodes (ii, [j,] k) of lane c
  double res[V][N];
#pragma unroll
  for (int r = 0; r < V; ++r) {
    double v[N];
#pragma unroll
    for (int ii = 0; ii < N; ++ii) v[ii] = X[r * TSZ + xoff<D, N>(c, ii)];
    if (minv) mat_apply<N, false>(TC.Binv, v, res[r]);
    else mat_apply<N, true>(TC.B, v, res[r]);
  }
#pragma unroll
  for (int ii = 0; ii < N; ++ii) {
    const int node = (D == 3) ? ii * N * N + c : ii * N + c;
    double* out = P.out.p + e * P.out.estride + node;
    if (!minv) {
#pragma unroll
      for (int r = 0; r < V; ++r) out[r * P.out.cstride] = res[r][ii];
      continue;
    }
    // R = -Minv dual + gravity source - sigma (U - U_bg)   (imex.py:144-159)
    double R[V];
#pragma unroll
    for (int r = 0; r < V; ++r) R[r] = -res[r][ii];
    const double rho = uin[0][ii];
    R[D] += -md.gravity * rho;
    R[D + 1] += -md.kinetic_factor * md.gravity * rho * (uin[D][ii] * __drcp_rn(rho));
    if (spg) {
#pragma unroll
      for (int r = 1; r < V; ++r) R[r] -= sgm[ii] * (uin[r][ii] - bgv[r][ii]);
    }
#pragma unroll
    for (int r = 0; r < V; ++r) out[r * P.out.cstride] = R[r];
  }
}

}  // namespace dg
