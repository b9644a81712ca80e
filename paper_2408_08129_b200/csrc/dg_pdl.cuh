// Programmatic dependent launch helpers shared by the element and vector
// kernels of the small-problem GMRES path.
#pragma once
#include <cuda_runtime.h>

namespace dg {

// ---- programmatic dependent launch (small problems, dcgs2_cycle_dev) --------
// The Arnoldi step of a small problem is a chain of ~7 dependent kernels of a
// few microseconds each: launched with the programmatic-stream-serialization
// attribute, a kernel's CTAs become resident while its predecessor drains
// and wait in griddepcontrol.wait (which returns once the predecessor grid
// has completed and its writes are visible) instead of paying the launch
// latency after it.  Every kernel of the chain triggers its dependents first
// and waits before its first read of predecessor data; launched normally,
// both instructions are no-ops.
__device__ __forceinline__ void pdl_trigger() {
  asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
}
__device__ __forceinline__ void pdl_wait() {
  asm volatile("griddepcontrol.wait;\n" ::: "memory");
}
// (host) set by dcgs2_cycle_dev around the steps it enqueues
inline thread_local int tl_pdl = 0;
template <typename... KArgs, typename... Args>
inline cudaError_t launch_k(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem,
                            cudaStream_t st, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = tl_pdl ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kern, KArgs(args)...);
}


}  // namespace dg
