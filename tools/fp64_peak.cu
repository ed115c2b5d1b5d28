// fp64_peak.cu — measured fp64 FMA throughput of this B200 (the roofline denominator for the
// fp64-bound ISM kernels; MEASURED_PEAKS.json has no fp64 entry).  Prints one JSON line.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void dfma_loop(double* out, int iters, double a, double b) {
  double x0 = threadIdx.x * 1e-9, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int r = 0; r < 16; ++r) {
      x0 = fma(x0, a, b); x1 = fma(x1, a, b); x2 = fma(x2, a, b); x3 = fma(x3, a, b);
      x4 = fma(x4, a, b); x5 = fma(x5, a, b); x6 = fma(x6, a, b); x7 = fma(x7, a, b);
    }
  }
  if (x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7 == 42.0) out[0] = x0;
}

int main() {
  cudaDeviceProp prop;
  cudaGetDeviceProperties(&prop, 0);
  double* out;
  cudaMalloc(&out, 8);
  const int blocks = prop.multiProcessorCount * 8, threads = 256, iters = 4096;
  dfma_loop<<<blocks, threads>>>(out, 16, 0.999999, 1e-7);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  float best = 1e30f;
  for (int rep = 0; rep < 5; ++rep) {
    cudaEventRecord(a);
    dfma_loop<<<blocks, threads>>>(out, iters, 0.999999, 1e-7);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    if (ms < best) best = ms;
  }
  const double flops = 2.0 * 8 * 16 * (double)iters * blocks * threads;
  int clk = 0;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  printf("{\"fp64_fma_tflops\": %.3f, \"sms\": %d, \"ms\": %.3f, \"max_clock_mhz\": %.0f, \"how\": \"%d CTAs x %d threads, 8 independent DFMA chains, best of 5, CUDA events\"}\n",
         flops / (best * 1e-3) / 1e12, prop.multiProcessorCount, best, clk / 1e3, blocks, threads);
  return 0;
}
