// bitflip_cluster.cu — the full-horizon node sweeps of the spin-register kind (node_sweeps,
// ism.cpp:35-84, and the exact payoff, objective.cpp:93-100) on a thread-block CLUSTER, sm_100a.
//
// The direct plan's node sweeps are the serial critical path of BASELINE config 3: K = 4000
// dependent Cayley steps per direction, each ~7 Jacobi sweeps of the bit-flip fixed point
//     z <- (1 + sD)^-1 (x - s V z),   x' = 2z - x          (bitflip_kernels.cu, oracle BitM::cayley)
// over d = 2^n amplitudes.  On one SM a sweep of d = 1024 costs ~1,570 cycles; here
// CL = 2^LOG2CL CTAs of one cluster split the amplitudes: CTA `rank` owns s = rank * Dl + t + e*T.
// A flip of bit b pairs
//   b < LOG2T                      -> thread t ^ 2^b of the same CTA   (shared memory)
//   LOG2T <= b < LOG2T + LOG2E     -> register slot e ^ 2^(b - LOG2T)   (same thread)
//   b >= LOG2T + LOG2E             -> CTA rank ^ 2^(b - LOG2T - LOG2E)  (distributed shared memory)
// and one cluster barrier per sweep orders every exchange (the double-buffered publish makes a
// second barrier unnecessary).  Arithmetic, coefficient signs and the a-priori sweep count are
// those of the single-CTA kernel, so results are identical to rounding order.
#include <cooperative_groups.h>
#include <cstdlib>

#include "kernels.h"

namespace cg = cooperative_groups;

namespace qoc {

namespace {

__device__ __forceinline__ double2 flip_coef(double2 ab, int one) { return cx(ab.x, one ? ab.y : -ab.y); }

template <int LOG2E, int LOG2T, int LOG2CL, int MODE>
__global__ void __launch_bounds__(1 << LOG2T) bitflip_horizon_cluster_kernel(DevProblem P, DevRun R, int which, int k,
                                                                             SweepRange SR) {
  constexpr bool PUSH = MODE >= 1, ASYNC = MODE == 2;
  constexpr int E = 1 << LOG2E, T = 1 << LOG2T, CL = 1 << LOG2CL, Dl = E * T, N = LOG2E + LOG2T + LOG2CL;
  if (R.kdev) k = *R.kdev;
  cg::cluster_group cluster = cg::this_cluster();
  const int rank = (int)cluster.block_rank();
  const int nl = SR.nloc > 0 ? SR.nloc : 1;
  const int b = blockIdx.y / nl, g = SR.g0 + (int)(blockIdx.y % nl), dir = blockIdx.z;
  if (R.done[b] || R.status[b]) return;  // uniform over the cluster (same problem)
  if (which == 1 && dir == 1) return;
  __shared__ __align__(16) double2 buf[2][Dl];
  // PUSH: partner rb's amplitudes of the current sweep, written by the partner (remote stores
  // before the barrier, local loads after it) instead of loaded remotely after the barrier
  __shared__ __align__(16) double2 inbox[PUSH ? 2 : 1][PUSH ? (LOG2CL > 0 ? LOG2CL : 1) : 1][PUSH ? Dl : 1];
  __shared__ __align__(8) unsigned long long mbar[2];  // ASYNC: inbox arrival per buffer parity
  __shared__ double2 sa[2][N];
  __shared__ int ssw[2];
  __shared__ double red[T / 32 + 1];
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5, d = P.d, C = P.C;
  const double half = 0.5 * P.dt;
  const double* u = R.u + (size_t)b * P.K * C;
  const double* coef = P.bf_coef + (size_t)b * C * P.nspins;
  const size_t nb = (size_t)b * (P.L + 1) * d;
  const int base = rank * Dl + t;  // amplitude of slot e: base + e * T
  double dg[E];
#pragma unroll
  for (int e = 0; e < E; ++e) dg[e] = P.bf_diag[(size_t)b * d + base + e * T];
  // partner CTAs' exchange buffers (distributed shared memory)
  const double2* rem[LOG2CL > 0 ? LOG2CL : 1];
  double2* outbox[LOG2CL > 0 ? LOG2CL : 1];  // PUSH: my slot rb in partner rank ^ 2^rb's inbox
#pragma unroll
  for (int rb = 0; rb < LOG2CL; ++rb) {
    rem[rb] = cluster.map_shared_rank(&buf[0][0], rank ^ (1 << rb));
    if constexpr (PUSH) outbox[rb] = cluster.map_shared_rank(&inbox[0][rb][0], rank ^ (1 << rb));
  }
  // ASYNC: shared::cluster addresses of my slot in each partner's inbox and of its barriers
  unsigned r_inbox[LOG2CL > 0 ? LOG2CL : 1], r_bar[LOG2CL > 0 ? LOG2CL : 1][2];
  if constexpr (ASYNC) {
    if (t == 0) {
      mbar_init(&mbar[0], 1);
      mbar_init(&mbar[1], 1);
      mbar_init_fence();
    }
#pragma unroll
    for (int rb = 0; rb < LOG2CL; ++rb) {
      const unsigned peer = (unsigned)(rank ^ (1 << rb));
      asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r_inbox[rb]) : "r"(smem_addr(&inbox[0][rb][0])), "r"(peer));
      asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r_bar[rb][0]) : "r"(smem_addr(&mbar[0])), "r"(peer));
      asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r_bar[rb][1]) : "r"(smem_addr(&mbar[1])), "r"(peer));
    }
    cluster.sync();  // every barrier is initialised before any peer signals it
  }
  unsigned phase[2] = {0u, 0u};
  double2 cl[LOG2T > 0 ? LOG2T : 1], ch[LOG2E > 0 ? LOG2E : 1], cr[LOG2CL > 0 ? LOG2CL : 1];
  int par = 0, spar = 0;
  bool ok = true;
  double2 x[E];

  auto begin_step = [&](const double* uj) -> int {
    spar ^= 1;
    if (warp == 0) {
      double nrm = 0.0;
      if (lane < N) {
        double ax = 0.0, ay = 0.0;
        for (int c = 0; c < C; ++c) {
          const double g = uj[c] * coef[c * N + lane];
          if (P.bf_axis[c] == 0) ax += g;
          else ay += g;
        }
        sa[spar][lane] = cx(ax, ay);
        nrm = sqrt(ax * ax + ay * ay);
      }
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) nrm += __shfl_xor_sync(0xffffffffu, nrm, off);
      if (lane == 0) {
        const double q = half * nrm;
        ssw[spar] = !(q < 0.5) ? -1 : (q <= 0.0 ? 0 : (int)ceil(54.0 * 0.6931471805599453 / -log(q)));
      }
    }
    __syncthreads();
#pragma unroll
    for (int bb = 0; bb < LOG2T; ++bb) cl[bb] = flip_coef(sa[spar][N - 1 - bb], (t >> bb) & 1);
#pragma unroll
    for (int hb = 0; hb < LOG2E; ++hb) ch[hb] = sa[spar][N - 1 - (LOG2T + hb)];
#pragma unroll
    for (int rb = 0; rb < LOG2CL; ++rb) cr[rb] = flip_coef(sa[spar][N - 1 - (LOG2T + LOG2E + rb)], (rank >> rb) & 1);
    return ssw[spar];
  };

  auto cayley = [&](double sh, int sweeps) {
    double2 z[E], vv[E], inv[E];
#pragma unroll
    for (int e = 0; e < E; ++e) {
      const double a = sh * dg[e];
      const double den = 1.0 / fma(a, a, 1.0);
      inv[e] = cx(den, -a * den);
      z[e] = cmul(x[e], inv[e]);
    }
    for (int it = 0; it < sweeps; ++it) {
      par ^= 1;
#pragma unroll
      for (int e = 0; e < E; ++e) buf[par][t + e * T] = z[e];
      if constexpr (ASYNC) {
        // asynchronous remote stores that complete on the partner's barrier: no cluster-wide
        // release fence (a GPU-scope MEMBAR per sweep with the cluster barrier)
#pragma unroll
        for (int rb = 0; rb < LOG2CL; ++rb)
#pragma unroll
          for (int e = 0; e < E; ++e) {
            const unsigned dst = r_inbox[rb] + (unsigned)sizeof(double2) * (unsigned)(par * LOG2CL * Dl + t + e * T);
            asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.f64 [%0], {%1, %2}, [%3];" ::"r"(dst),
                         "d"(z[e].x), "d"(z[e].y), "r"(r_bar[rb][par])
                         : "memory");
          }
        if (t == 0) mbar_expect_tx(&mbar[par], (unsigned)(LOG2CL * Dl * sizeof(double2)));
        __syncthreads();  // the CTA-local publish
      } else if constexpr (PUSH) {
#pragma unroll
        for (int rb = 0; rb < LOG2CL; ++rb)
#pragma unroll
          for (int e = 0; e < E; ++e) outbox[rb][par * LOG2CL * Dl + t + e * T] = z[e];
        cluster.sync();  // every CTA's publish of this sweep is visible cluster-wide
      } else {
        cluster.sync();
      }
#pragma unroll
      for (int e = 0; e < E; ++e) vv[e] = cx(0.0, 0.0);
      if constexpr (!ASYNC) {
#pragma unroll
        for (int rb = 0; rb < LOG2CL; ++rb) {
          const double2* rbuf = PUSH ? &inbox[par][rb][0] : rem[rb] + par * Dl;
#pragma unroll
          for (int e = 0; e < E; ++e) vv[e] = cfma(cr[rb], rbuf[t + e * T], vv[e]);
        }
      }
#pragma unroll
      for (int hb = 0; hb < LOG2E; ++hb)
#pragma unroll
        for (int e = 0; e < E; ++e) vv[e] = cfma(flip_coef(ch[hb], (e >> hb) & 1), z[e ^ (1 << hb)], vv[e]);
#pragma unroll
      for (int bb = 0; bb < LOG2T; ++bb)
#pragma unroll
        for (int e = 0; e < E; ++e) vv[e] = cfma(cl[bb], buf[par][(t ^ (1 << bb)) + e * T], vv[e]);
      if constexpr (ASYNC) {  // the partners' amplitudes of this sweep have landed
        mbar_wait(&mbar[par], phase[par]);
        phase[par] ^= 1u;
#pragma unroll
        for (int rb = 0; rb < LOG2CL; ++rb)
#pragma unroll
          for (int e = 0; e < E; ++e) vv[e] = cfma(cr[rb], inbox[par][rb][t + e * T], vv[e]);
      }
#pragma unroll
      for (int e = 0; e < E; ++e) {
        const double2 tt = cx(x[e].x + sh * vv[e].y, x[e].y - sh * vv[e].x);  // x - s V z
        z[e] = cmul(tt, inv[e]);
      }
    }
#pragma unroll
    for (int e = 0; e < E; ++e) x[e] = cx(fma(2.0, z[e].x, -x[e].x), fma(2.0, z[e].y, -x[e].y));
  };
  auto load = [&](const double2* src) {
#pragma unroll
    for (int e = 0; e < E; ++e) x[e] = src[base + e * T];
  };
  auto store = [&](double2* dst) {
#pragma unroll
    for (int e = 0; e < E; ++e) dst[base + e * T] = x[e];
  };
  auto step = [&](const double* uj, double sh) {
    const int sweeps = begin_step(uj);
    ok &= sweeps >= 0;
    cayley(sh, sweeps < 0 ? 0 : sweeps);
  };

  // node range [na, nz] of this sweep (SweepRange, common.cuh); the full horizon also writes
  // its two end nodes, a block of the blocked plan only its interior nodes
  const bool full = SR.nloc == 0;
  const int na = full ? 0 : SR.bnode[g], nz = full ? P.L : SR.bnode[g + 1];
  if (dir == 0) {
    load(full ? P.init + (size_t)b * d : R.psi_nodes + nb + (size_t)na * d);
    if (which == 0 && full) store(R.psi_nodes + nb);
    int nxt = na + 1;
    const int last = full ? nz : nz - 1;
    for (int j = P.node[na]; j < P.node[nz]; ++j) {
      step(u + (size_t)j * C, half);
      if (which == 0 && nxt <= last && P.node[nxt] == j + 1) {
        store(R.psi_nodes + nb + (size_t)nxt * d);
        ++nxt;
      }
    }
    if (which == 1) {  // Re<target, psi(T)> over the cluster, fixed rank order
      double s = 0.0;
#pragma unroll
      for (int e = 0; e < E; ++e) s += cconjmul(P.targ[(size_t)b * d + base + e * T], x[e]).x;
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
      if (lane == 0) red[warp] = s;
      __syncthreads();
      if (t == 0) {
        double a = 0.0;
        for (int w = 0; w < T / 32; ++w) a += red[w];
        red[T / 32] = a;
      }
      cluster.sync();
      if (rank == 0 && t == 0) {
        double tot = 0.0;
        for (int r = 0; r < CL; ++r) tot += cluster.map_shared_rank(red, r)[T / 32];
        double pen = 0.0;
        for (int n = 0; n < P.L; ++n) pen += R.pen[(size_t)b * P.L + n];
        R.rec_exact[(size_t)b * R.cap + k] = P.ip_w * tot - 0.5 * P.dt * pen;
      }
    }
  } else {
    load(full ? P.targ + (size_t)b * d : R.chi_nodes + nb + (size_t)nz * d);
    if (full) store(R.chi_nodes + nb + (size_t)P.L * d);
    int prev = nz - 1;
    const int first = full ? na : na + 1;
    for (int j = P.node[nz] - 1; j >= P.node[na]; --j) {
      step(u + (size_t)j * C, -half);
      if (prev >= first && P.node[prev] == j) {
        store(R.chi_nodes + nb + (size_t)prev * d);
        --prev;
      }
    }
  }
  if (!ok && t == 0 && rank == 0 && R.err_flags) atomicOr(R.err_flags, 2);
  cluster.sync();  // no CTA leaves while a peer may still read its shared memory
}

template <int LOG2E, int LOG2T, int LOG2CL, int MODE = 0>
cudaError_t launch_cluster(const DevProblem& P, const DevRun& R, int which, int k, const SweepRange& SR,
                           cudaStream_t st) {
  auto kern = bitflip_horizon_cluster_kernel<LOG2E, LOG2T, LOG2CL, MODE>;
  constexpr int CL = 1 << LOG2CL;
  if (CL > 8) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    if (e != cudaSuccess) return e;
  }
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(CL, P.B * (SR.nloc > 0 ? SR.nloc : 1), 2);
  cfg.blockDim = dim3(1 << LOG2T, 1, 1);
  cfg.dynamicSmemBytes = 0;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = CL;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, P, R, which, k, SR);
}

}  // namespace

// QOC_BF_CLUSTER selects the cluster shape for d = 1024 node sweeps ("0" keeps the single-CTA
// kernel).  "16a" (default; 8a where 16-CTA clusters cannot launch): 16 CTAs x 64 threads x 1
// amplitude; "8a": 8 CTAs x 128 threads x 1 amplitude, partner amplitudes pushed with
// st.async onto the partner's mbarrier (no cluster barrier, so no GPU-scope MEMBAR per sweep);
// "4a" / "2a" / "8b" / "16a": 4 x 128 x 2, 2 x 128 x 4, 8 x 64 x 2, 16 x 64 x 1 of the same.
// Barrier-synchronised variants: "8x1" pull, "8p" push (8 x 128 x 1), "8q" / "4p" / "2p" push
// with 2 / 2 / 4 amplitudes, "8x2", "16x1".  Measured per config-3 outer iteration (node
// sweeps): single CTA 22.8 ms; barrier variants 20.0-21.2 ms (MEMBAR.ALL.GPU per cluster
// barrier); 16a 13.1 ms, 8a 13.8, 2a 16.4, 8b 19.4, 4a 19.7.
cudaError_t bitflip_horizon_cluster(const DevProblem& P, const DevRun& R, int which, int k, const SweepRange& SR,
                                    cudaStream_t st, bool* used) {
  *used = false;
  if (P.nspins != 10 || P.C > 4) return cudaSuccess;
  const char* e = std::getenv("QOC_BF_CLUSTER");
  const char* shape = e ? e : "16a";
  if (shape[0] == '0') return cudaSuccess;
  cudaError_t r;
  if (shape[0] == '1' && shape[1] == '6' && shape[2] != 'a') r = launch_cluster<0, 6, 4>(P, R, which, k, SR, st);
  else if (shape[2] == '2') r = launch_cluster<1, 6, 3>(P, R, which, k, SR, st);
  else if (shape[0] == '8' && shape[1] == 'a') r = launch_cluster<0, 7, 3, 2>(P, R, which, k, SR, st);
  else if (shape[0] == '1' && shape[1] == '6' && shape[2] == 'a') r = launch_cluster<0, 6, 4, 2>(P, R, which, k, SR, st);
  else if (shape[0] == '4' && shape[1] == 'a') r = launch_cluster<1, 7, 2, 2>(P, R, which, k, SR, st);
  else if (shape[0] == '2' && shape[1] == 'a') r = launch_cluster<2, 7, 1, 2>(P, R, which, k, SR, st);
  else if (shape[0] == '8' && shape[1] == 'b') r = launch_cluster<1, 6, 3, 2>(P, R, which, k, SR, st);
  else if (shape[1] == 'p') r = launch_cluster<0, 7, 3, 1>(P, R, which, k, SR, st);
  else if (shape[1] == 'q') r = launch_cluster<1, 6, 3, 1>(P, R, which, k, SR, st);
  else if (shape[0] == '4') r = launch_cluster<1, 7, 2, 1>(P, R, which, k, SR, st);
  else if (shape[0] == '2') r = launch_cluster<2, 7, 1, 1>(P, R, which, k, SR, st);
  else r = launch_cluster<0, 7, 3>(P, R, which, k, SR, st);
  if (r != cudaSuccess && !e) {  // 16-CTA clusters are non-portable: fall back to 8
    cudaGetLastError();
    r = launch_cluster<0, 7, 3, 2>(P, R, which, k, SR, st);
  }
  *used = r == cudaSuccess;
  if (r != cudaSuccess) cudaGetLastError();  // e.g. no cluster support: the single-CTA kernel
  return cudaSuccess;
}

}  // namespace qoc
