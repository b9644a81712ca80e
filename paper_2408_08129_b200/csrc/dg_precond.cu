// Block-Jacobi preconditioner of the Helmholtz action on the device
// (orodg/krylov.py:143-178; used by imex.py:334-342).
//
// The per-element diagonal blocks are probed exactly as the reference
// does -- for every colour of the greedy face-adjacency colouring
// (krylov.py:118-140) and every node i, the action is applied to the probe
// e_i on all elements of that colour and column i of each such element's
// block is read off its own rows (the 1-hop colouring lets 2-hop
// neighbours contaminate a block, as in the reference) --
// then inverted in place, one CTA per element (Gauss-Jordan with partial
// pivoting; an exactly singular block becomes the identity, as the
// reference's LinAlgError fallback).  The inverse is stored transposed so
// the blockwise apply streams it coalesced (warp per element): the apply
// is HBM-bound at 8 NP^2 bytes per element.
#include <cstdint>

#include "dg_precond.cuh"
#include "dg_prof.h"

namespace dg {

namespace {

__global__ void k_bj_probe(long long n_el, int np, const int* __restrict__ colors, int col,
                           int node, double* __restrict__ x) {
  const long long n = n_el * np;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    const long long e = i / np;
    const int q = (int)(i - e * np);
    x[i] = (q == node && colors[e] == col) ? 1.0 : 0.0;
  }
}

// column `node` of the blocks of colour `col`: blocks[e][r][node] = y[e][r]
__global__ void k_bj_scatter(long long n_el, int np, const int* __restrict__ colors, int col,
                             int node, const double* __restrict__ y, double* __restrict__ blocks) {
  const long long n = n_el * np;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    const long long e = i / np;
    if (colors[e] != col) continue;
    const int r = (int)(i - e * np);
    blocks[(e * np + r) * np + node] = y[i];
  }
}

constexpr int INV_THREADS = 256;

// in-place Gauss-Jordan inverse of one np x np block per CTA; the result is
// written transposed into invT (may alias blocks: each CTA owns its block)
template <bool SMEM>
__global__ void __launch_bounds__(INV_THREADS)
k_bj_invert(int np, double* blocks, double* invT, int* singular) {
  extern __shared__ double sm[];
  const long long e = blockIdx.x;
  double* A = SMEM ? sm : blocks + e * np * np;
  int* perm = reinterpret_cast<int*>(SMEM ? sm + np * np : sm);
  double* colk = SMEM ? sm + np * np + (np + 1) / 2 + 1 : sm + (np + 1) / 2 + 1;
  __shared__ int s_piv, s_sing;
  const int nn = np * np;
  if (SMEM)
    for (int i = threadIdx.x; i < nn; i += blockDim.x) A[i] = blocks[e * nn + i];
  if (threadIdx.x == 0) s_sing = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  for (int k = 0; k < np; ++k) {
    if (wid == 0) {
      // partial pivot: largest |A[i][k]|, i >= k (first index on ties)
      double bv = -1.0;
      int bi = np;
      for (int i = k + lane; i < np; i += 32) {
        const double v = fabs(A[i * np + k]);
        if (v > bv) { bv = v; bi = i; }
      }
      for (int o = 16; o > 0; o >>= 1) {
        const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
        const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
        if (ov > bv || (ov == bv && oi < bi)) { bv = ov; bi = oi; }
      }
      if (lane == 0) {
        s_piv = bi;
        perm[k] = bi;
        if (!(bv > 0.0)) s_sing = 1;
      }
    }
    __syncthreads();
    if (s_sing) break;
    const int p = s_piv;
    if (p != k)
      for (int j = threadIdx.x; j < np; j += blockDim.x) {
        const double t = A[k * np + j];
        A[k * np + j] = A[p * np + j];
        A[p * np + j] = t;
      }
    __syncthreads();
    const double piv = A[k * np + k];
    __syncthreads();
    for (int j = threadIdx.x; j < np; j += blockDim.x)
      A[k * np + j] = (j == k) ? 1.0 / piv : A[k * np + j] / piv;
    for (int i = threadIdx.x; i < np; i += blockDim.x) colk[i] = A[i * np + k];
    __syncthreads();
    for (int t = threadIdx.x; t < nn; t += blockDim.x) {
      const int i = t / np, j = t - (t / np) * np;
      if (i == k) continue;
      const double base = (j == k) ? 0.0 : A[t];
      A[t] = base - colk[i] * A[k * np + j];
    }
    __syncthreads();
  }
  if (s_sing) {
    if (threadIdx.x == 0) atomicAdd(singular, 1);
    for (int t = threadIdx.x; t < nn; t += blockDim.x) {
      const int i = t / np, j = t - (t / np) * np;
      invT[e * nn + t] = (i == j) ? 1.0 : 0.0;
    }
    return;
  }
  // undo the row pivoting: swap columns in reverse order
  for (int k = np - 1; k >= 0; --k) {
    const int p = perm[k];
    if (p != k)
      for (int i = threadIdx.x; i < np; i += blockDim.x) {
        const double t = A[i * np + k];
        A[i * np + k] = A[i * np + p];
        A[i * np + p] = t;
      }
    __syncthreads();
  }
  if (SMEM) {
    for (int t = threadIdx.x; t < nn; t += blockDim.x) {
      const int i = t / np, j = t - (t / np) * np;
      invT[e * nn + j * np + i] = A[t];
    }
  } else {
    // in place (A aliases invT): transpose through the pairs above the diagonal
    for (int t = threadIdx.x; t < nn; t += blockDim.x) {
      const int i = t / np, j = t - (t / np) * np;
      if (j > i) {
        const double a = A[i * np + j], b = A[j * np + i];
        A[i * np + j] = b;
        A[j * np + i] = a;
      }
    }
  }
}

constexpr int APPLY_WARPS = 8;
constexpr int MAXT = 11;  // rows per lane: np <= 352 (n = 7 in 3D)

// out_e = inv_e in_e, warp per element, inverse stored transposed; T rows per lane
template <int T>
__global__ void __launch_bounds__(APPLY_WARPS * 32)
k_bj_apply(long long n_el, int np, const double* __restrict__ invT, const double* __restrict__ in,
           double* __restrict__ out) {
  extern __shared__ double sv[];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  double* v = sv + wid * np;
  for (long long e = (long long)blockIdx.x * APPLY_WARPS + wid; e < n_el;
       e += (long long)gridDim.x * APPLY_WARPS) {
    for (int j = lane; j < np; j += 32) v[j] = in[e * np + j];
    __syncwarp();
    double acc[T];
#pragma unroll
    for (int t = 0; t < T; ++t) acc[t] = 0.0;
    const double* M = invT + e * np * np;
    for (int j = 0; j < np; ++j) {
      const double vj = v[j];
#pragma unroll
      for (int t = 0; t < T; ++t) {
        const int r = lane + 32 * t;
        if (r < np) acc[t] = fma(M[(long long)j * np + r], vj, acc[t]);
      }
    }
#pragma unroll
    for (int t = 0; t < T; ++t) {
      const int r = lane + 32 * t;
      if (r < np) out[e * np + r] = acc[t];
    }
    __syncwarp();
  }
}

int grid_for(long long n) {
  long long g = (n + 255) / 256;
  return (int)(g > 148 * 16 ? 148 * 16 : (g < 1 ? 1 : g));
}

}  // namespace

cudaError_t bj_probe(cudaStream_t st, long long n_el, int np, const int* colors, int col, int node,
                     double* x) {
  prof_begin(st);
  k_bj_probe<<<grid_for(n_el * np), 256, 0, st>>>(n_el, np, colors, col, node, x);
  prof_end(st, P_OTHER, 8.0 * n_el * np, 1);
  return cudaGetLastError();
}

cudaError_t bj_scatter(cudaStream_t st, long long n_el, int np, const int* colors, int col,
                       int node, const double* y, double* blocks) {
  prof_begin(st);
  k_bj_scatter<<<grid_for(n_el * np), 256, 0, st>>>(n_el, np, colors, col, node, y, blocks);
  prof_end(st, P_OTHER, 8.0 * n_el * np, 1);
  return cudaGetLastError();
}

cudaError_t bj_invert(cudaStream_t st, long long n_el, int np, double* blocks, double* invT,
                      int* singular) {
  if (n_el == 0) return cudaSuccess;
  const size_t extra = ((size_t)(np + 1) / 2 + 1 + np) * sizeof(double);
  const size_t sm = (size_t)np * np * sizeof(double) + extra;
  prof_begin(st);
  if (sm <= 200 * 1024) {
    cudaFuncSetAttribute(k_bj_invert<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    k_bj_invert<true><<<(unsigned)n_el, INV_THREADS, sm, st>>>(np, blocks, invT, singular);
  } else {
    // block in global memory, inverted in place (invT must alias blocks)
    k_bj_invert<false><<<(unsigned)n_el, INV_THREADS, extra, st>>>(np, blocks, blocks, singular);
  }
  prof_end(st, P_OTHER, 16.0 * n_el * np * np, 1);
  return cudaGetLastError();
}

cudaError_t bj_apply(cudaStream_t st, long long n_el, int np, const double* invT, const double* in,
                     double* out) {
  if (np > 32 * MAXT) return cudaErrorInvalidValue;
  long long g = (n_el + APPLY_WARPS - 1) / APPLY_WARPS;
  if (g > 148 * 32) g = 148 * 32;
  if (g < 1) g = 1;
  prof_begin(st);
  const size_t sm = APPLY_WARPS * np * sizeof(double);
  switch ((np + 31) / 32) {
#define DG_BJ_CASE(T) \
  case T: k_bj_apply<T><<<(unsigned)g, APPLY_WARPS * 32, sm, st>>>(n_el, np, invT, in, out); break;
    DG_BJ_CASE(1) DG_BJ_CASE(2) DG_BJ_CASE(3) DG_BJ_CASE(4) DG_BJ_CASE(5) DG_BJ_CASE(6)
    DG_BJ_CASE(7) DG_BJ_CASE(8) DG_BJ_CASE(9) DG_BJ_CASE(10) DG_BJ_CASE(11)
#undef DG_BJ_CASE
    default: return cudaErrorInvalidValue;
  }
  prof_end(st, P_OTHER, 8.0 * n_el * np * (np + 2), 1);
  return cudaGetLastError();
}

}  // namespace dg
