// fp64 FMA throughput of this B200 (the fp64 roofline denominator of
// SURVEY.md §8d): every thread runs 8 independent DFMA chains; grid = 8 CTAs
// of 1024 threads per SM.  Timed with CUDA events after a warm-up.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/dfma_peak tools/dfma_peak.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_dfma(double* out, int iters, double a, double b) {
  double x[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) x[i] = threadIdx.x * 1e-3 + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int r = 0; r < 16; ++r)
#pragma unroll
      for (int i = 0; i < 8; ++i) x[i] = fma(x[i], a, b);
  }
  double s = 0.0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += x[i];
  if (s == 12345.678) out[0] = s;  // keep the chains alive
}

int main() {
  int dev = 0, nsm = 0;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  double* out;
  cudaMalloc(&out, sizeof(double));
  const int threads = 1024, blocks = nsm * 2, iters = 4000;
  k_dfma<<<blocks, threads>>>(out, 100, 0.999999, 1e-7);
  cudaDeviceSynchronize();
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float best = 1e30f;
  for (int rep = 0; rep < 5; ++rep) {
    cudaEventRecord(e0);
    k_dfma<<<blocks, threads>>>(out, iters, 0.999999, 1e-7);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  const double flops = 2.0 * 8 * 16 * (double)iters * threads * blocks;
  printf("{\"dfma_tflops\": %.3f, \"sms\": %d, \"ms\": %.3f}\n", flops / (best * 1e-3) / 1e12, nsm,
         best);
  return 0;
}
