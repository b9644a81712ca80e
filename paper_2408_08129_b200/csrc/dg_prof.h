// Launch accounting and optional per-kernel-class CUDA-event timing.
// Every host wrapper that launches kernels reports (class, algorithmic
// bytes, launches); with profiling enabled each report is bracketed by
// events on the launching stream, so bench.py can compute the achieved
// bandwidth of the dominant kernel class over its own timed region.
#pragma once
#include <cuda_runtime.h>
#include <vector>

namespace dg {

enum ProfCls { P_ADV = 0, P_GRAD, P_DIVHV, P_DOT, P_AXPY, P_OTHER, P_NCLS };

struct Profiler {
  bool on = false;
  std::vector<cudaEvent_t> ev;   // pairs
  size_t used = 0;               // pairs in use
  std::vector<int> cls;
  std::vector<double> bytes;
  long long launches = 0;
};

Profiler& prof();
void prof_begin(cudaStream_t st);
void prof_end(cudaStream_t st, int cls, double bytes, int nlaunch);

}  // namespace dg
