// asm_probe.cu — A/B probe of one propagator-assembly sweep for the batched dense kind
// (BASELINE config 5: 4096 problems x 128 subintervals x 16 steps, d = 16, C = 1).
//
// Each variant computes, per task, P_{j+1} = C_j P_j with C_j = 2 B_j^-1 - I,
// B_j = I + i dt/2 (H0 + u_j Hc) (propagation.cpp:14-16,236-249), storing every P_{j+1} to the
// cache (optional) and the final P to `out`.  Outputs are compared against variant V0.
//   V0  row per lane, 16 lanes per task: in-register Gauss-Jordan inverse + DFMA matmul
//       (the round-1 dense_pc_assemble<16> algorithm, pivot-free path)
//   V4  32 lanes per task: Gauss-Jordan on the augmented system [B_j | P_j] (no explicit
//       inverse, no matmul): X = B_j^-1 P_j, P_{j+1} = 2X - P_j
//   V3  32 lanes per task: Gauss-Jordan inverse, then the 16x16 complex product on the fp64
//       tensor cores (mma.sync m8n8k4 f64, four real products)
#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "../paper_1603_01237_b200/csrc/dense.cuh"

using namespace qoc;

constexpr int D = 16;

__device__ __forceinline__ double2 cfma_(double2 a, double2 b, double2 c) { return cfma(a, b, c); }

// ---------------------------------------------------------------- V0
template <bool STORE>
__global__ void __launch_bounds__(128) v0_kernel(const double2* H0, const double2* Hc, const double* u, double2* cache,
                                                 double2* out, int L, int len, int K, double half) {
  using Cfg = DenseCfg<D, 1>;
  __shared__ double2 ops[2 * D * D];
  constexpr int GB = sizeof(double2) * (Cfg::PIV + Cfg::VEC + 2 * Cfg::MAT) + 2 * D * 4;
  extern __shared__ __align__(16) unsigned char scratch_raw[];
  const int b = blockIdx.y;
  for (int e = threadIdx.x; e < 2 * D * D; e += blockDim.x) ops[e] = e < D * D ? H0[b * D * D + e] : Hc[b * D * D + e - D * D];
  __syncthreads();
  const int warp = threadIdx.x >> 5, l32 = threadIdx.x & 31, gid = warp * 2 + l32 / 16, lane = l32 % 16;
  const int n = blockIdx.x * 8 + gid;
  if (n >= L) return;
  DenseScratch<D, 1> S;
  S.piv = reinterpret_cast<double2*>(scratch_raw + GB * gid);
  S.vec = S.piv + Cfg::PIV;
  S.matW = S.vec + Cfg::VEC;
  S.matP = S.matW + Cfg::MAT;
  S.perm = reinterpret_cast<int*>(S.matP + Cfg::MAT);
  DenseLane<D, 1> Ln;
  Ln.row = lane;
  Ln.g = 0;
  double2 W[D], Pm[D];
#pragma unroll
  for (int t = 0; t < D; ++t) Pm[t] = cx(lane == t ? 1.0 : 0.0, 0.0);
  const size_t task = (size_t)b * L + n;
  for (int j = 0; j < len; ++j) {
    const double uj = u[(size_t)b * K + n * len + j];
    Ln.build(W, ops, 1, 0, &uj, half, false);
    Ln.invert_fast(W, S.piv);
    Ln.cayley_matmul(W, Pm, S, true);
    if (STORE) {
      double2* dst = cache + (task * len + j) * D * D + lane * D;
#pragma unroll
      for (int t = 0; t < D; ++t) dst[t] = Pm[t];
    }
  }
#pragma unroll
  for (int t = 0; t < D; ++t) out[task * D * D + lane * D + t] = Pm[t];
}

// ---------------------------------------------------------------- shared 32-lane helpers
// lane (row = l & 15, g = l >> 4) holds columns 2t + g, t = 0..7 of its row
__device__ __forceinline__ void build32(double2 (&Bm)[8], const double2* ops, double uj, double half, int row, int g) {
#pragma unroll
  for (int t = 0; t < 8; ++t) {
    const int col = 2 * t + g;
    const double2 h0 = ops[row * D + col], hc = ops[D * D + row * D + col];
    const double hr = fma(uj, hc.x, h0.x), hi = fma(uj, hc.y, h0.y);
    Bm[t] = cx((row == col ? 1.0 : 0.0) - half * hi, half * hr);
  }
}

// ---------------------------------------------------------------- V4: augmented Gauss-Jordan
template <bool STORE>
__global__ void __launch_bounds__(256, 2) v4_kernel(const double2* H0, const double2* Hc, const double* u, double2* cache,
                                                 double2* out, int L, int len, int K, double half) {
  __shared__ double2 ops[2 * D * D];
  __shared__ double2 rowbuf[8][2][2 * D];
  __shared__ double2 pold[8][D * D];
  const int b = blockIdx.y;
  for (int e = threadIdx.x; e < 2 * D * D; e += blockDim.x) ops[e] = e < D * D ? H0[b * D * D + e] : Hc[b * D * D + e - D * D];
  __syncthreads();
  const int warp = threadIdx.x >> 5, l = threadIdx.x & 31, row = l & 15, g = l >> 4;
  const int n = blockIdx.x * 8 + warp;
  if (n >= L) return;
  const size_t task = (size_t)b * L + n;
  double2 X[8];
#pragma unroll
  for (int t = 0; t < 8; ++t) X[t] = cx(row == 2 * t + g ? 1.0 : 0.0, 0.0);
  for (int j = 0; j < len; ++j) {
    const double uj = u[(size_t)b * K + n * len + j];
    double2 Bm[8];
    build32(Bm, ops, uj, half, row, g);
    double2* Po = pold[warp] + row * D + g;
#pragma unroll
    for (int t = 0; t < 8; ++t) Po[2 * t] = X[t];
#pragma unroll
    for (int k = 0; k < D; ++k) {
      const int kt = k >> 1, kg = k & 1;
      double2* rb = rowbuf[warp][k & 1];
      const bool is_k = row == k;
      if (is_k) {
#pragma unroll
        for (int t = kt; t < 8; ++t) rb[2 * t + g] = Bm[t];
#pragma unroll
        for (int t = 0; t < 8; ++t) rb[D + 2 * t + g] = X[t];
      }
      const double2 f = shfl(Bm[kt], row + 16 * kg);
      const double2 p = shfl(Bm[kt], k + 16 * kg);
      __syncwarp();
      const double2 pinv = crcp(p);
      const double2 fp = cmul(f, pinv);
      const double2 bb = is_k ? pinv : cneg(fp);
#pragma unroll
      for (int t = kt; t < 8; ++t) {
        if (2 * t + g > k) {
          const double2 x = is_k ? Bm[t] : rb[2 * t + g];
          const double2 a = is_k ? cx(0.0, 0.0) : Bm[t];
          Bm[t] = cfma(bb, x, a);
        }
      }
#pragma unroll
      for (int t = 0; t < 8; ++t) {
        const double2 x = is_k ? X[t] : rb[D + 2 * t + g];
        const double2 a = is_k ? cx(0.0, 0.0) : X[t];
        X[t] = cfma(bb, x, a);
      }
    }
#pragma unroll
    for (int t = 0; t < 8; ++t) X[t] = cx(2.0 * X[t].x - Po[2 * t].x, 2.0 * X[t].y - Po[2 * t].y);
    if (STORE) {
      double2* dst = cache + (task * len + j) * D * D + row * D + g;
#pragma unroll
      for (int t = 0; t < 8; ++t) dst[2 * t] = X[t];
    }
  }
  double2* dst = out + task * D * D + row * D + g;
#pragma unroll
  for (int t = 0; t < 8; ++t) dst[2 * t] = X[t];
}

// ---------------------------------------------------------------- V3: GJ inverse + DMMA
__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

template <bool STORE>
__global__ void __launch_bounds__(256, 2) v3_kernel(const double2* H0, const double2* Hc, const double* u, double2* cache,
                                                 double2* out, int L, int len, int K, double half) {
  __shared__ double2 ops[2 * D * D];
  __shared__ double2 rowbuf[8][2][D];
  extern __shared__ __align__(16) double2 dyn[];
  const int b = blockIdx.y;
  for (int e = threadIdx.x; e < 2 * D * D; e += blockDim.x) ops[e] = e < D * D ? H0[b * D * D + e] : Hc[b * D * D + e - D * D];
  __syncthreads();
  const int warp = threadIdx.x >> 5, l = threadIdx.x & 31, row = l & 15, g = l >> 4, q = l >> 2, r = l & 3;
  const int n = blockIdx.x * 8 + warp;
  if (n >= L) return;
  const size_t task = (size_t)b * L + n;
  double2* W_ = dyn + (size_t)warp * 2 * D * D;
  double2* P_ = W_ + D * D;
  for (int e = l; e < D * D; e += 32) P_[e] = cx((e / D) == (e % D) ? 1.0 : 0.0, 0.0);
  __syncwarp();
  for (int j = 0; j < len; ++j) {
    const double uj = u[(size_t)b * K + n * len + j];
    double2 Bm[8];
    build32(Bm, ops, uj, half, row, g);
#pragma unroll
    for (int k = 0; k < D; ++k) {
      const int kt = k >> 1, kg = k & 1;
      double2* rb = rowbuf[warp][k & 1];
      const bool is_k = row == k;
      if (is_k) {
#pragma unroll
        for (int t = 0; t < 8; ++t) rb[2 * t + g] = Bm[t];
      }
      const double2 f = shfl(Bm[kt], row + 16 * kg);
      const double2 p = shfl(Bm[kt], k + 16 * kg);
      __syncwarp();
      const double2 pinv = crcp(p);
      const double2 fp = cmul(f, pinv);
      const double2 bb = is_k ? pinv : cneg(fp);
#pragma unroll
      for (int t = 0; t < 8; ++t) {
        const int col = 2 * t + g;
        const bool ck = col == k;
        const double2 x = ck ? cx(1.0, 0.0) : (is_k ? Bm[t] : rb[col]);
        const double2 a = (is_k || ck) ? cx(0.0, 0.0) : Bm[t];
        Bm[t] = cfma(bb, x, a);
      }
    }
#pragma unroll
    for (int t = 0; t < 8; ++t) W_[row * D + 2 * t + g] = Bm[t];
    __syncwarp();
    double2 af[2][4], bf[4][2];
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
      for (int kk = 0; kk < 4; ++kk) af[i][kk] = W_[(8 * i + q) * D + 4 * kk + r];
#pragma unroll
    for (int kk = 0; kk < 4; ++kk)
#pragma unroll
      for (int jn = 0; jn < 2; ++jn) bf[kk][jn] = P_[(4 * kk + r) * D + 8 * jn + q];
    double cr[2][2][2], ci[2][2][2];
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
      for (int jn = 0; jn < 2; ++jn) {
        cr[i][jn][0] = cr[i][jn][1] = ci[i][jn][0] = ci[i][jn][1] = 0.0;
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) {
          dmma(cr[i][jn][0], cr[i][jn][1], af[i][kk].x, bf[kk][jn].x);
          dmma(cr[i][jn][0], cr[i][jn][1], -af[i][kk].y, bf[kk][jn].y);
          dmma(ci[i][jn][0], ci[i][jn][1], af[i][kk].x, bf[kk][jn].y);
          dmma(ci[i][jn][0], ci[i][jn][1], af[i][kk].y, bf[kk][jn].x);
        }
      }
    __syncwarp();
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
      for (int jn = 0; jn < 2; ++jn)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int idx = (8 * i + q) * D + 8 * jn + 2 * r + e;
          const double2 po = P_[idx];
          const double2 pn = cx(2.0 * cr[i][jn][e] - po.x, 2.0 * ci[i][jn][e] - po.y);
          P_[idx] = pn;
          if (STORE) cache[(task * len + j) * D * D + idx] = pn;
        }
    __syncwarp();
  }
  for (int e = l; e < D * D; e += 32) out[task * D * D + e] = P_[e];
}

// ---------------------------------------------------------------- host
static double herm_rand(std::vector<double2>& m, int b, unsigned& s, double scale) {
  auto rnd = [&]() {
    s = s * 1664525u + 1013904223u;
    return ((s >> 8) / 16777216.0) * 2.0 - 1.0;
  };
  for (int i = 0; i < D; ++i)
    for (int j = i; j < D; ++j) {
      double re = rnd() * scale, im = (i == j) ? 0.0 : rnd() * scale;
      m[(size_t)b * D * D + i * D + j] = make_double2(re, im);
      m[(size_t)b * D * D + j * D + i] = make_double2(re, -im);
    }
  return 0.0;
}

#define CK(x)                                                                 \
  do {                                                                        \
    cudaError_t e_ = (x);                                                     \
    if (e_ != cudaSuccess) {                                                  \
      fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_)); \
      exit(1);                                                                \
    }                                                                         \
  } while (0)

int main(int argc, char** argv) {
  const int B = argc > 1 ? atoi(argv[1]) : 4096, L = 128, len = 16, K = L * len;
  const double half = 0.5 * 10.0 / 2000.0;
  std::vector<double2> h0((size_t)B * D * D), hc((size_t)B * D * D);
  std::vector<double> uu((size_t)B * K);
  unsigned s = 12345u;
  for (int b = 0; b < B; ++b) {
    herm_rand(h0, b, s, 0.35);
    herm_rand(hc, b, s, 0.35);
  }
  for (auto& x : uu) {
    s = s * 1664525u + 1013904223u;
    x = 0.1 + 0.5 * (((s >> 8) / 16777216.0) - 0.5);
  }
  double2 *dH0, *dHc, *dcache, *dout[3];
  double* du;
  const size_t tasks = (size_t)B * L;
  CK(cudaMalloc(&dH0, h0.size() * 16));
  CK(cudaMalloc(&dHc, hc.size() * 16));
  CK(cudaMalloc(&du, uu.size() * 8));
  CK(cudaMalloc(&dcache, tasks * len * D * D * 16));
  for (auto& o : dout) CK(cudaMalloc(&o, tasks * D * D * 16));
  CK(cudaMemcpy(dH0, h0.data(), h0.size() * 16, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dHc, hc.data(), hc.size() * 16, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(du, uu.data(), uu.size() * 8, cudaMemcpyHostToDevice));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  auto timeit = [&](const char* name, auto launch, int oi) {
    launch();
    CK(cudaDeviceSynchronize());
    float best = 1e30f;
    for (int rep = 0; rep < 3; ++rep) {
      cudaEventRecord(e0);
      launch();
      cudaEventRecord(e1);
      CK(cudaEventSynchronize(e1));
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      best = ms < best ? ms : best;
    }
    double diff = 0.0;
    if (oi > 0) {
      std::vector<double2> a(tasks * D * D), c(tasks * D * D);
      CK(cudaMemcpy(a.data(), dout[0], a.size() * 16, cudaMemcpyDeviceToHost));
      CK(cudaMemcpy(c.data(), dout[oi], c.size() * 16, cudaMemcpyDeviceToHost));
      for (size_t i = 0; i < a.size(); ++i) diff = fmax(diff, fmax(fabs(a[i].x - c[i].x), fabs(a[i].y - c[i].y)));
    }
    const double steps = (double)tasks * len;
    printf("{\"variant\": \"%s\", \"ms\": %.3f, \"ns_per_task_step\": %.4f, \"max_abs_diff_vs_v0\": %.3e}\n", name, best,
           best * 1e6 / steps, diff);
    fflush(stdout);
  };
  const dim3 g0((L + 7) / 8, B), g4((L + 7) / 8, B);
  using Cfg = DenseCfg<D, 1>;
  const int s0 = 8 * (sizeof(double2) * (Cfg::PIV + Cfg::VEC + 2 * Cfg::MAT) + 2 * D * 4), s3 = 8 * 2 * D * D * 16;
  CK(cudaFuncSetAttribute(v0_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, s0));
  CK(cudaFuncSetAttribute(v0_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, s0));
  CK(cudaFuncSetAttribute(v3_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, s3));
  CK(cudaFuncSetAttribute(v3_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, s3));
  timeit("v0_store", [&] { v0_kernel<true><<<g0, 128, s0>>>(dH0, dHc, du, dcache, dout[0], L, len, K, half); }, 0);
  timeit("v0_nostore", [&] { v0_kernel<false><<<g0, 128, s0>>>(dH0, dHc, du, dcache, dout[0], L, len, K, half); }, 0);
  timeit("v4_store", [&] { v4_kernel<true><<<g4, 256>>>(dH0, dHc, du, dcache, dout[1], L, len, K, half); }, 1);
  timeit("v4_nostore", [&] { v4_kernel<false><<<g4, 256>>>(dH0, dHc, du, dcache, dout[1], L, len, K, half); }, 1);
  timeit("v3_store", [&] { v3_kernel<true><<<g4, 256, s3>>>(dH0, dHc, du, dcache, dout[2], L, len, K, half); }, 2);
  timeit("v3_nostore", [&] { v3_kernel<false><<<g4, 256, s3>>>(dH0, dHc, du, dcache, dout[2], L, len, K, half); }, 2);
  return 0;
}
