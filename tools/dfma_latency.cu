// Dependent-chain latency of DFMA / FFMA / LDS on one warp (clock64 bracket).
#include <cstdio>
__global__ void lat(double* out, long long* cyc, double a, double b, int n) {
  double x = a;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) x = fma(x, b, a);
  long long t1 = clock64();
  float y = (float)a;
  for (int i = 0; i < n; ++i) y = fmaf(y, (float)b, (float)a);
  long long t2 = clock64();
  double z = a;
  for (int i = 0; i < n; ++i) z = 1.0 / (z + b);
  long long t3 = clock64();
  if (threadIdx.x == 0) {
    out[0] = x + y + z;
    cyc[0] = t1 - t0;
    cyc[1] = t2 - t1;
    cyc[2] = t3 - t2;
  }
}
int main() {
  double* o;
  long long* c;
  cudaMalloc(&o, 8);
  cudaMalloc(&c, 24);
  const int n = 4096;
  lat<<<1, 32>>>(o, c, 0.5, 0.999, n);
  lat<<<1, 32>>>(o, c, 0.5, 0.999, n);
  long long h[3];
  cudaMemcpy(h, c, 24, cudaMemcpyDeviceToHost);
  printf("{\"dfma_latency_cycles\": %.2f, \"ffma_latency_cycles\": %.2f, \"drcp_div_latency_cycles\": %.2f}\n",
         (double)h[0] / n, (double)h[1] / n, (double)h[2] / n);
  return 0;
}
