// Block-Jacobi preconditioner kernels (dg_precond.cu; orodg/krylov.py:143-178)
#pragma once
#include <cuda_runtime.h>

namespace dg {

// x = e_node on every element of colour col, 0 elsewhere (owned elements)
cudaError_t bj_probe(cudaStream_t st, long long n_el, int np, const int* colors, int col, int node,
                     double* x);
// blocks[e][:, node] = y[e] for the elements of colour col
cudaError_t bj_scatter(cudaStream_t st, long long n_el, int np, const int* colors, int col,
                       int node, const double* y, double* blocks);
// in-place inverse of every block, stored transposed in invT (may alias blocks);
// singular blocks become the identity and are counted in *singular (device)
cudaError_t bj_invert(cudaStream_t st, long long n_el, int np, double* blocks, double* invT,
                      int* singular);
// out_e = inv_e in_e
cudaError_t bj_apply(cudaStream_t st, long long n_el, int np, const double* invT, const double* in,
                     double* out);

}  // namespace dg
