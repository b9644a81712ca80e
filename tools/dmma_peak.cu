// fp64 tensor-core (DMMA m8n8k4) throughput of this B200, next to the DFMA
// peak of tools/dfma_peak.cu: decides whether the 1D contractions of the
// element kernels should move onto DMMA fragments.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/dmma_peak tools/dmma_peak.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_dmma(double* out, int iters) {
  // 4 independent accumulator fragments per warp (ILP), A / B fragments fixed
  double a = 1.0 + threadIdx.x * 1e-6, b = 0.5 - threadIdx.x * 1e-6;
  double c[4][2];
#pragma unroll
  for (int i = 0; i < 4; ++i) c[i][0] = c[i][1] = 0.0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int r = 0; r < 8; ++r)
#pragma unroll
      for (int i = 0; i < 4; ++i)
        asm volatile(
            "mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};\n"
            : "+d"(c[i][0]), "+d"(c[i][1])
            : "d"(a), "d"(b));
  }
  double s = 0.0;
#pragma unroll
  for (int i = 0; i < 4; ++i) s += c[i][0] + c[i][1];
  if (s == 12345.678) out[0] = s;
}

int main() {
  int nsm = 0;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  double* out;
  cudaMalloc(&out, sizeof(double));
  const int threads = 512, blocks = nsm * 4, iters = 2000;
  k_dmma<<<blocks, threads>>>(out, 50);
  cudaDeviceSynchronize();
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float best = 1e30f;
  for (int rep = 0; rep < 5; ++rep) {
    cudaEventRecord(e0);
    k_dmma<<<blocks, threads>>>(out, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  // per warp-MMA: 8 x 8 x 4 FMA = 512 flops
  const double mmas = (double)iters * 8 * 4 * (threads / 32) * blocks;
  printf("{\"dmma_tflops\": %.3f, \"ms\": %.3f, \"err\": \"%s\"}\n", mmas * 512.0 / (best * 1e-3) / 1e12,
         best, cudaGetErrorString(cudaGetLastError()));
  return 0;
}
