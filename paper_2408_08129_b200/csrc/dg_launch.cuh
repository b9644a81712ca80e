// Host-side launcher for the templated element kernels (one translation
// unit per dimension instantiates N = 2..7 and the three operator kinds).
#pragma once
#include <algorithm>
#include <cstring>
#include <cstdlib>
#include <string>
#include <type_traits>
#include "dg_xkernel.cuh"
#include "dg_hkernel.cuh"

namespace dg {

// N-independent operator arguments; the launcher copies the 1D tables
// (flat, Tab<N> layout) into the kernel parameter block.
struct OpArgs {
  MeshDev mesh;
  GeoConst gc;
  Model model;
  CView in, inK, inH, base, bg;
  const double* sigma;
  MView out;
  double alpha, beta, coef;
  int has_K, has_base, homogeneous, mode;
  int dbg;  // phase-skip flags for profiling experiments only (0 in production)
  int in_quad, out_quad;
  double* tr_out;      // trace mode (see KParams)
  const double* trV;
  const double* trH;
  double* psi_out;     // flux-trace mode (see KParams)
  const double* psi;
  double* pin_out;
  const double* pin;
  const int* frec;
  int full;  // ADV: divergence_full flux (see KParams)
  double* mass_partial;
  const double* gsV;  // fused Gram-Schmidt dots (see KParams)
  long long gs_vs;
  int gs_nv, gs_dual;
  double* gs_part;
  const double* tabs;  // host pointer, Tab<N> layout
  const double* tabs_dev;  // the same tables in device memory
};

struct LaunchInfo {
  int epb;
  int threads;
  size_t smem;
  int grid;
};

template <int D, int N, int OPK>
cudaError_t launch_elem(const OpArgs& a, cudaStream_t st, LaunchInfo* info) {
  using L = Layout<D, N, OPK>;
  KParams<N> P;
  P.mesh = a.mesh;
  P.gc = a.gc;
  P.model = a.model;
  P.in = a.in;
  P.inK = a.inK;
  P.inH = a.inH;
  P.base = a.base;
  P.bg = a.bg;
  P.sigma = a.sigma;
  P.out = a.out;
  P.alpha = a.alpha;
  P.beta = a.beta;
  P.coef = a.coef;
  P.has_K = a.has_K;
  P.has_base = a.has_base;
  P.homogeneous = a.homogeneous;
  P.mode = a.mode;
  P.dbg = a.dbg;
  P.in_quad = a.in_quad;
  P.out_quad = a.out_quad;
  P.mass_partial = a.mass_partial;
  P.full = a.full;
  P.tr_out = a.tr_out;
  P.trV = a.trV;
  P.trH = a.trH;
  P.psi_out = a.psi_out;
  P.psi = a.psi;
  P.pin_out = a.pin_out;
  P.pin = a.pin;
  P.frec = a.frec;
  P.gsV = a.gsV;
  P.gs_vs = a.gs_vs;
  P.gs_nv = a.gs_nv;
  P.gs_part = a.gs_part;
  P.gs_dual = a.gs_dual;
  P.gs_row0 = 0;
  P.tab_g = a.tabs_dev;
  std::memcpy(&P.tab, a.tabs, sizeof(Tab<N>));
  using HL = HLayout<D, N>;
  if constexpr (HL::OK && OPK != OP_ADV) {
    // flux-trace mode of the Helmholtz pair (dg_hkernel.cuh)
    const bool hk = (OPK == OP_GRAD) ? a.psi_out != nullptr : a.psi != nullptr;
    if (hk) {
      constexpr int EPC = HL::EPW * HL::WPB;
      const int hgrid = (a.mesh.n_el + EPC - 1) / EPC;
      const size_t hsm = (OPK == OP_GRAD) ? HL::GSMEM : HL::DSMEM;
      if (info) {
        info->epb = EPC;
        info->threads = HL::THREADS;
        info->smem = hsm;
        info->grid = hgrid;
      }
      if (hgrid == 0) return cudaSuccess;
      static bool hconf = false;
      if (!hconf) {
        cudaError_t e = (OPK == OP_GRAD)
            ? cudaFuncSetAttribute(hgrad_kernel<D, N>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   (int)HL::GSMEM)
            : cudaFuncSetAttribute(hdiv_kernel<D, N>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   (int)HL::DSMEM);
        if (e != cudaSuccess) return e;
        e = cudaFuncSetAttribute(coarse_kernel<D, N, OPK, true>,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, (int)L::CSMEM);
        if (e == cudaSuccess) e = cudaFuncSetAttribute(coarse_kernel<D, N, OPK>,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, (int)L::CSMEM);
        if (e != cudaSuccess) return e;
        hconf = true;
      }
      if (a.mesh.n_coarse > 0) {
        if (a.mesh.cflux == nullptr) return cudaErrorInvalidValue;  // flux mode required
        cudaError_t e = launch_k(coarse_kernel<D, N, OPK, true>, dim3(a.mesh.n_coarse),
                                 dim3(L::CTHREADS), L::CSMEM, st, P, a.mesh.coarse_list,
                                 (int)a.mesh.n_coarse, (double*)nullptr);
        if (e != cudaSuccess) return e;
      }
      if constexpr (OPK == OP_GRAD) {
        using PL = H1Pipe<D, N>;
        static const bool pipe1 = getenv("DG_PIPE1") && std::string(getenv("DG_PIPE1")) == "1";
        if constexpr (PL::OK) {
          if (pipe1 && a.pin_out != nullptr && a.frec != nullptr) {
            static int pgrid = 0;
            if (pgrid == 0) {
              cudaError_t e = cudaFuncSetAttribute(
                  hgrad2_kernel<D, N>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)PL::SMEM);
              if (e != cudaSuccess) return e;
              int dev = 0, sms = 0, occ = 0;
              cudaGetDevice(&dev);
              cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
              e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, hgrad2_kernel<D, N>, 128,
                                                                PL::SMEM);
              if (e != cudaSuccess) return e;
              pgrid = sms * (occ > 0 ? occ : 1);
            }
            const long long groups = (a.mesh.n_el + HL::EPW - 1) / HL::EPW;
            const int g = (int)std::min<long long>(pgrid, (groups + PL::WPB - 1) / PL::WPB);
            if (info) {
              info->threads = 128;
              info->smem = PL::SMEM;
              info->grid = g;
            }
            hgrad2_kernel<D, N><<<g, 128, PL::SMEM, st>>>(P);
            return cudaGetLastError();
          }
        }
        return launch_k(hgrad_kernel<D, N>, dim3(hgrid), dim3(HL::THREADS), HL::GSMEM, st, P);
      } else {
        using PL = H2Pipe<D, N>;
        if constexpr (PL::OK) {
          if (a.pin != nullptr && a.frec != nullptr && (a.gs_part == nullptr || PL::FUSED)) {
            // persistent pipelined H2: every SM's resident CTAs, the groups
            // strided over the warps (DG_H2LA=1: records / column rows staged)
            static const bool la = !(getenv("DG_H2LA") && std::string(getenv("DG_H2LA")) == "0");
            auto kfn = la ? hdiv2_kernel<D, N, true> : hdiv2_kernel<D, N, false>;
            static int pgrid = 0;
            if (pgrid == 0) {
              cudaError_t e = cudaFuncSetAttribute(
                  kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)PL::SMEM);
              if (e != cudaSuccess) return e;
              int dev = 0, sms = 0, occ = 0;
              cudaGetDevice(&dev);
              cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
              e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kfn, 32 * PL::WPB, PL::SMEM);
              if (e != cudaSuccess) return e;
              pgrid = sms * (occ > 0 ? occ : 1);
            }
            const long long groups = (a.mesh.n_el + HL::EPW - 1) / HL::EPW;
            const int g = (int)std::min<long long>(pgrid, (groups + PL::WPB - 1) / PL::WPB);
            if (info) {
              info->threads = 32 * PL::WPB;
              info->smem = PL::SMEM;
              info->grid = g;  // one dot-partial row per CTA
            }
            return launch_k(kfn, dim3(g), dim3(32 * PL::WPB), PL::SMEM, st, P);
          }
        }
        return launch_k(hdiv_kernel<D, N>, dim3(hgrid), dim3(HL::THREADS), HL::DSMEM, st, P);
      }
      return cudaGetLastError();
    }
  }
  using WL = WLayout<D, N, OPK>;
  if constexpr (WL::OK) {
    // warp-element kernel (v3) for the Helmholtz pair unless DG_KERNEL=v2
    static const bool use_w = !(getenv("DG_KERNEL") && std::string(getenv("DG_KERNEL")) == "v2");
    if (use_w) {
      constexpr int EPC = WL::EPW * WL::WPB;
      const int wgrid = (a.mesh.n_el + EPC - 1) / EPC;
      if (info) {
        info->epb = EPC;
        info->threads = WL::THREADS;
        info->smem = WL::SMEM;
        info->grid = wgrid;
      }
      if (wgrid == 0) return cudaSuccess;
      static bool wconf = false;
      if (!wconf) {
        for (auto kfn : {welem_kernel<D, N, OPK, false>, welem_kernel<D, N, OPK, OPK == OP_DIVHV>}) {
          cudaError_t e = cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                               (int)WL::SMEM);
          if (e != cudaSuccess) return e;
          e = cudaFuncSetAttribute(kfn, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
          if (e != cudaSuccess) return e;
        }
        cudaError_t e = cudaFuncSetAttribute(coarse_kernel<D, N, OPK, true>,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, (int)L::CSMEM);
        if (e == cudaSuccess) e = cudaFuncSetAttribute(coarse_kernel<D, N, OPK>,
                                             cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)L::CSMEM);
        if (e != cudaSuccess) return e;
        wconf = true;
      }
      const bool fmode = a.mesh.n_coarse > 0 && a.mesh.cflux != nullptr;
      if (fmode) {
        // the coarse faces' fluxes first; the element kernel lifts them
        coarse_kernel<D, N, OPK, true><<<a.mesh.n_coarse, L::CTHREADS, L::CSMEM, st>>>(
            P, a.mesh.coarse_list, a.mesh.n_coarse, nullptr);
        cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) return e;
      }
      if (OPK == OP_DIVHV && a.in_quad)
        welem_kernel<D, N, OPK, OPK == OP_DIVHV><<<wgrid, WL::THREADS, WL::SMEM, st>>>(P);
      else
        welem_kernel<D, N, OPK, false><<<wgrid, WL::THREADS, WL::SMEM, st>>>(P);
      cudaError_t e = cudaGetLastError();
      if (e != cudaSuccess) return e;
      if (a.mesh.n_coarse > 0 && !fmode) {
        P.gs_row0 = wgrid;  // coarse elements' dot partials follow the CTA rows
        coarse_kernel<D, N, OPK><<<a.mesh.n_coarse, L::CTHREADS, L::CSMEM, st>>>(
            P, a.mesh.coarse_list, a.mesh.n_coarse, nullptr);
        e = cudaGetLastError();
      }
      // dot partial rows written
      if (info) info->grid = wgrid + (fmode ? 0 : a.mesh.n_coarse);
      return e;
    }
  }
  if constexpr (OPK == OP_ADV && XLayout<D, N>::OK) {
    // warp-element explicit kernel (dg_xkernel.cuh) unless DG_KERNEL=v2
    using XL = XLayout<D, N>;
    static const bool use_x = !(getenv("DG_KERNEL") && std::string(getenv("DG_KERNEL")) == "v2");
    if (use_x) {
      constexpr int EPC = XL::EPW * XL::TEAMS;
      const int xgrid = (a.mesh.n_el + EPC - 1) / EPC;
      if (info) {
        info->epb = EPC;
        info->threads = XL::THREADS;
        info->smem = XL::SMEM;
        info->grid = xgrid * XL::WPB;
      }
      if (xgrid == 0) return cudaSuccess;
      static bool xconf = false;
      if (!xconf) {
        for (auto kfn : {xelem_kernel<D, N, false>, xelem_kernel<D, N, true>}) {
          cudaError_t e = cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                               (int)XL::SMEM);
          if (e != cudaSuccess) return e;
          e = cudaFuncSetAttribute(kfn, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
          if (e != cudaSuccess) return e;
        }
        cudaError_t e = cudaFuncSetAttribute(coarse_kernel<D, N, OPK, true>,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, (int)L::CSMEM);
        if (e == cudaSuccess) e = cudaFuncSetAttribute(coarse_kernel<D, N, OPK>,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, (int)L::CSMEM);
        if (e != cudaSuccess) return e;
        xconf = true;
      }
      const bool fmode = a.mesh.n_coarse > 0 && a.mesh.cflux != nullptr;
      if (fmode) {
        coarse_kernel<D, N, OPK, true><<<a.mesh.n_coarse, L::CTHREADS, L::CSMEM, st>>>(
            P, a.mesh.coarse_list, a.mesh.n_coarse, nullptr);
        cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) return e;
      }
      if (a.full) xelem_kernel<D, N, true><<<xgrid, XL::THREADS, XL::SMEM, st>>>(P);
      else xelem_kernel<D, N, false><<<xgrid, XL::THREADS, XL::SMEM, st>>>(P);
      cudaError_t e = cudaGetLastError();
      if (e != cudaSuccess) return e;
      const int rows = xgrid * XL::WPB;  // mass-rate partials: one per warp
      if (fmode) {
        if (info) info->grid = rows;
        return e;
      }
      if (a.mesh.n_coarse > 0) {
        coarse_kernel<D, N, OPK><<<a.mesh.n_coarse, L::CTHREADS, L::CSMEM, st>>>(
            P, a.mesh.coarse_list, a.mesh.n_coarse,
            a.mass_partial ? a.mass_partial + rows : nullptr);
        e = cudaGetLastError();
      }
      if (info) info->grid = rows + a.mesh.n_coarse;  // partial slots written
      return e;
    }
  }
  const int grid = (a.mesh.n_el + L::EPB - 1) / L::EPB;
  if (info) {
    info->epb = L::EPB;
    info->threads = L::THREADS;
    info->smem = L::SMEM;
    info->grid = grid;
  }
  if (grid == 0) return cudaSuccess;
  static bool configured = false;
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(elem_kernel<D, N, OPK>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)L::SMEM);
    if (e != cudaSuccess) return e;
    e = cudaFuncSetAttribute(elem_kernel<D, N, OPK>,
                             cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    if (e != cudaSuccess) return e;
    e = cudaFuncSetAttribute(coarse_kernel<D, N, OPK, true>,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, (int)L::CSMEM);
        if (e == cudaSuccess) e = cudaFuncSetAttribute(coarse_kernel<D, N, OPK>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize, (int)L::CSMEM);
    if (e != cudaSuccess) return e;
    configured = true;
  }
  const bool fmode = a.mesh.n_coarse > 0 && a.mesh.cflux != nullptr;
  if (fmode) {
    coarse_kernel<D, N, OPK, true><<<a.mesh.n_coarse, L::CTHREADS, L::CSMEM, st>>>(
        P, a.mesh.coarse_list, a.mesh.n_coarse, nullptr);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
  }
  elem_kernel<D, N, OPK><<<grid, L::THREADS, L::SMEM, st>>>(P);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  if (fmode) {
    if (info) info->grid = grid;
    return e;
  }
  if (a.mesh.n_coarse > 0) {
    coarse_kernel<D, N, OPK><<<a.mesh.n_coarse, L::CTHREADS, L::CSMEM, st>>>(
        P, a.mesh.coarse_list, a.mesh.n_coarse,
        a.mass_partial ? a.mass_partial + grid : nullptr);
    e = cudaGetLastError();
  }
  if (info) info->grid = grid + a.mesh.n_coarse;  // partial slots written
  return e;
}

// is the warp-element kernel (and with it Gauss-point storage of the
// Helmholtz intermediate and the fused Gram-Schmidt dots) used for this (dim, n)?
inline bool welem_enabled(int D, int N) {
  int nc = 1;
  for (int a = 0; a < D - 1; ++a) nc *= N;
  static const bool v2 = getenv("DG_KERNEL") && std::string(getenv("DG_KERNEL")) == "v2";
  return nc <= 32 && !v2;
}

// the flux-trace Helmholtz kernels (dg_hkernel.cuh): one- or two-warp teams
inline bool hk_enabled(int D, int N) {
  int nc = 1;
  for (int a = 0; a < D - 1; ++a) nc *= N;
  static const bool v2 = getenv("DG_KERNEL") && std::string(getenv("DG_KERNEL")) == "v2";
  return nc <= 64 && !v2;
}

// can the warp-element div(hV) kernel stage face data asynchronously (and
// with it run the face-trace mode) for this (dim, n)?
template <int D>
inline bool welem_async_divhv(int N) {
  switch (N) {
    case 2: return WLayout<D, 2, OP_DIVHV>::ASYNC;
    case 3: return WLayout<D, 3, OP_DIVHV>::ASYNC;
    case 4: return WLayout<D, 4, OP_DIVHV>::ASYNC;
    case 5: return WLayout<D, 5, OP_DIVHV>::ASYNC;
    case 6: return WLayout<D, 6, OP_DIVHV>::ASYNC;
    case 7: return WLayout<D, 7, OP_DIVHV>::ASYNC;
  }
  return false;
}
inline bool welem_trace_ok(int D, int N) {
  return D == 2 ? welem_async_divhv<2>(N) : welem_async_divhv<3>(N);
}

// grid size only (for sizing the per-CTA partial buffers)
template <int D, int N, int OPK>
int elem_grid(int n_el) {
  using L = Layout<D, N, OPK>;
  return (n_el + L::EPB - 1) / L::EPB;
}

cudaError_t launch_elem_d2(int N, int opk, const OpArgs& a, cudaStream_t st, LaunchInfo* info);
cudaError_t launch_elem_d3(int N, int opk, const OpArgs& a, cudaStream_t st, LaunchInfo* info);

}  // namespace dg

namespace dg {

struct AuxArgs {
  const int* elem;
  const double* col;
  GeoConst gc;
  int n_el;
  int ncomp;
  CView in;
  CView in2;    // inner product: second field
  Model model;  // Courant report
  double* tr;   // interp: face traces (trace mode)
  MView out;
  double* partial;
  const double* tabs;
};

cudaError_t launch_aux_d2(int N, int which, const AuxArgs& a, cudaStream_t st, int* grid);
cudaError_t launch_aux_d3(int N, int which, const AuxArgs& a, cudaStream_t st, int* grid);

}  // namespace dg
