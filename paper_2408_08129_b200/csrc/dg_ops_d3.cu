// Element-kernel instantiations for d = 3, N = r+1 = 2..7.
#include "dg_launch.cuh"

namespace dg {

template <int N>
static cudaError_t by_op(int opk, const OpArgs& a, cudaStream_t st, LaunchInfo* info) {
  switch (opk) {
    case OP_ADV: return launch_elem<3, N, OP_ADV>(a, st, info);
    case OP_GRAD: return launch_elem<3, N, OP_GRAD>(a, st, info);
    case OP_DIVHV: return launch_elem<3, N, OP_DIVHV>(a, st, info);
  }
  return cudaErrorInvalidValue;
}

cudaError_t launch_elem_d3(int N, int opk, const OpArgs& a, cudaStream_t st, LaunchInfo* info) {
  switch (N) {
    case 2: return by_op<2>(opk, a, st, info);
    case 3: return by_op<3>(opk, a, st, info);
    case 4: return by_op<4>(opk, a, st, info);
    case 5: return by_op<5>(opk, a, st, info);
    case 6: return by_op<6>(opk, a, st, info);
    case 7: return by_op<7>(opk, a, st, info);
  }
  return cudaErrorInvalidValue;
}

}  // namespace dg

#include "dg_aux.cuh"

namespace dg {

template <int N>
static cudaError_t aux_n(int which, const AuxArgs& a, cudaStream_t st, int* grid) {
  AuxParams<N> P;
  P.elem = a.elem;
  P.col = a.col;
  P.gc = a.gc;
  P.n_el = a.n_el;
  P.ncomp = a.ncomp;
  P.in = a.in;
  P.in2 = a.in2;
  P.model = a.model;
  P.tr = a.tr;
  P.out = a.out;
  P.partial = a.partial;
  std::memcpy(&P.tab, a.tabs, sizeof(Tab<N>));
  return launch_aux<3, N>(which, P, st, grid);
}

cudaError_t launch_aux_d3(int N, int which, const AuxArgs& a, cudaStream_t st, int* grid) {
  switch (N) {
    case 2: return aux_n<2>(which, a, st, grid);
    case 3: return aux_n<3>(which, a, st, grid);
    case 4: return aux_n<4>(which, a, st, grid);
    case 5: return aux_n<5>(which, a, st, grid);
    case 6: return aux_n<6>(which, a, st, grid);
    case 7: return aux_n<7>(which, a, st, grid);
  }
  return cudaErrorInvalidValue;
}

}  // namespace dg
