// Shared device-side types of libdg (B200 / sm_100a, fp64).
//
// Layout contract:
//   state        (n_el, V, n^d)     element-major, identical to the reference
//                                   StateField (orodg/field.py:12)
//   scalar field (n_el, n^d)        Krylov vectors, h, K, p
//   elem table   (n_el_total, 2+d)  int32 level, origin[d], column id
//   col table    (n_col, stride)    float64 terrain data per leaf footprint
//   face table   nbr (n_el_total, 2d) int32 + kind (n_el_total, 2d) uint8
#pragma once
#include "dg_pdl.cuh"
#include <cstdint>
#include <cuda_runtime.h>

namespace dg {

__host__ __device__ constexpr int ipow(int b, int e) { return e == 0 ? 1 : b * ipow(b, e - 1); }

// face kinds (low nibble) -- subface index in bits 4..5 for KIND_FINE
enum FaceKind : uint8_t {
  KIND_WALL = 0,      // boundary, slip wall
  KIND_FARFIELD = 1,  // boundary, prescribed far-field traces (row = nbr)
  KIND_CONF = 2,      // same-level neighbour nbr (incl. periodic wraps)
  KIND_FINE = 3,      // I am the fine side; nbr = coarse leaf; my subface in bits 4-5
  KIND_COARSE = 4,    // I am the coarse side; nbr = row of hang_children
};

// 1D basis tables, passed by value in the kernel parameter space (constant
// bank) and staged to shared memory by each CTA.
template <int N>
struct Tab {
  double B[N][N];      // B[q][j] = l_j(x_q): nodes -> Gauss points
  double Binv[N][N];   // B^-1
  double Dhat[N][N];   // D B^-1: collocation derivative at Gauss points
  double lift[2][N];   // lift[s][q] = Binv[end_s][q]
  double half[2][N][N];   // half[s][q][j] = l_j((x_q + s)/2)  (mortar, nodal)
  double halfq[2][N][N];  // half[s] B^-1 (mortar acting on Gauss traces)
  double qw[N];
  double qx[N];
  double iqw[N];       // 1 / qw (mass-inverse epilogue without divisions)
};

struct Model {
  double gamma, gravity, inv_mach_sq, kinetic_factor;
};

// Mesh-wide geometry scalars
struct GeoConst {
  double per_root[3];  // extents[a] / root_counts[a]
  double z_top;
  double inv_ztop;     // 1 / z_top (warp-element kernel: multiply, no division)
  int terrain;         // 0: flat, column table unused
  int col_stride;
};

// Element-centric mesh data (device pointers)
struct MeshDev {
  const int* elem;          // (n_tot, 2 + d)
  const double* col;        // (n_col, col_stride)
  const int* nbr;           // (n_tot, 2d)
  const uint8_t* kind;      // (n_tot, 2d)
  const int* hang_children; // (n_groups, 2^(d-1))
  const double* ff_U;       // (n_bface, V, nqf) far-field conserved traces
  const double* ff_p;       // (n_bface, nqf)
  const double* ff_h;       // (n_bface, nqf)
  int n_el;                 // owned elements processed by the kernels
  const int* coarse_list;   // per owned element with >= 1 coarse hanging face:
                            // [element, (2d) hanging groups or -1,
                            //  (2d) x 2^(d-1) children or -1]
  int n_coarse;
  // coarse-face fluxes (flux mode): the coarse side's lifted numerical flux
  // at the coarse face's Gauss points, (n_groups, KOUT, n^(d-1)) per hanging
  // group, written by coarse_kernel before the element kernel reads them
  double* cflux;
};

// Strided component view: comp c of element e at p + e*estride + c*cstride
struct CView {
  const double* p;
  long long estride;
  long long cstride;
  __device__ __forceinline__ double operator()(long long e, int c, int i) const {
    return p[e * estride + c * cstride + i];
  }
};
struct MView {
  double* p;
  long long estride;
  long long cstride;
};

template <int D>
struct ElemGeo {
  double s[D];   // box edge lengths
  double lo[D];  // lower corner
  int col;
};

template <int D>
__device__ __forceinline__ ElemGeo<D> elem_geo(const int* elem, const GeoConst& gc, long long e) {
  ElemGeo<D> g;
  const int* r = elem + e * (2 + D);
  const int level = r[0];
  // (extents/root) / 2^level is an exact power-of-two scaling
  // (geometry.py:195-197): multiply by 2^-level instead of dividing
  const double scale = __longlong_as_double((long long)(1023 - level) << 52);
#pragma unroll
  for (int a = 0; a < D; ++a) {
    g.s[a] = gc.per_root[a] * scale;
    g.lo[a] = g.s[a] * (double)r[1 + a];
  }
  g.col = r[1 + D];
  return g;
}

// the same from an element row already in registers / shared memory
// (level, integer origin[d], column)
template <int D>
__device__ __forceinline__ ElemGeo<D> geo_from_row(const int* r, const GeoConst& gc) {
  ElemGeo<D> g;
  const double scale = __longlong_as_double((long long)(1023 - r[0]) << 52);
#pragma unroll
  for (int a = 0; a < D; ++a) {
    g.s[a] = gc.per_root[a] * scale;
    g.lo[a] = g.s[a] * (double)r[1 + a];
  }
  g.col = r[1 + D];
  return g;
}


}  // namespace dg
