// glue.cu — kind-independent ISM coordinator kernels (sm_100a).
//
// These replace the serial coordinator of run_ism (ism.cpp:481-591): the deterministic
// index-order merge of task results, the abort checks, the propagator chain
// (compose_from_propagators, ism.cpp:298-312), the split-variant node refresh
// (ism.cpp:546-552), the boundary objective (ism.cpp:285-296) and the waypoint rebuild
// (interpolated_waypoints + make_subproblems, ism.cpp:100-159).  Every reduction runs in a
// fixed order, so results do not depend on scheduling.
#include <cuda_pipeline.h>
#include <math.h>

#include "kernels.h"

namespace qoc {

namespace {

__device__ __forceinline__ double qnan() { return __longlong_as_double(0x7ff8000000000000ULL); }

template <int NT>
__device__ double block_sum(double v, double* sh) {
  sh[threadIdx.x] = v;
  __syncthreads();
#pragma unroll
  for (int s = NT / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s) sh[threadIdx.x] += sh[threadIdx.x + s];
    __syncthreads();
  }
  const double r = sh[0];
  __syncthreads();
  return r;
}

// sum_j alpha_j |u_j|^2 over each task window (weighted_l2_penalty, controls.cpp:174-181)
// and the finite-control flag (ism.cpp:527-539).
__global__ void penalty_kernel(DevProblem P, DevRun R, int ignore_done) {
  const int n = blockIdx.x, b = blockIdx.y;
  if (ignore_done ? R.status[b] : (R.done[b] | R.status[b])) return;
  const int j0 = P.node[n], j1 = P.node[n + 1];
  const double* u = R.u + (size_t)b * P.K * P.C;
  double acc = 0.0;
  int bad = 0;
  for (int j = j0 + (int)threadIdx.x; j < j1; j += 32) {
    double sq = 0.0;
    for (int c = 0; c < P.C; ++c) {
      const double v = u[(size_t)j * P.C + c];
      sq += v * v;
      bad |= !isfinite(v);
    }
    acc += P.alpha[j] * sq;
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
  bad = __any_sync(0xffffffffu, bad);
  if (threadIdx.x == 0) {
    R.pen[(size_t)b * P.L + n] = acc;
    R.bad_u[(size_t)b * P.L + n] = bad;
  }
}

// Index-order merge of task results (ism.cpp:481-539).
// One block per problem: the L task results are reduced in a fixed tree order (deterministic).
__global__ void __launch_bounds__(128) merge_kernel(DevProblem P, DevRun R, int k) {
  if (R.kdev) k = *R.kdev;  // graph replay: the iteration index lives on the device
  __shared__ double sh[128];
  __shared__ int bad_sh;
  const int b = blockIdx.x;
  if (R.done[b] || R.status[b]) return;
  if (threadIdx.x == 0) bad_sh = 0;
  double tot = 0.0, esum = 0.0;
  int bad = 0;
  double* tv = R.rec_tv + ((size_t)b * R.cap + (k - 1)) * P.L;
  for (int n = threadIdx.x; n < P.L; n += 128) {
    const double e = R.entry[(size_t)b * P.L + n];
    tv[n] = e;
    esum += e;
    tot += R.err[(size_t)b * P.L + n];
    bad |= R.bad_u[(size_t)b * P.L + n];
  }
  __syncthreads();
  if (bad) atomicOr(&bad_sh, 1);
  tot = block_sum<128>(tot, sh);
  if (P.L == 1) esum = block_sum<128>(esum, sh);
  if (threadIdx.x != 0) return;
  if (P.L == 1) R.rec_obj[(size_t)b * R.cap + (k - 1)] = esum;
  R.tot_err[b] = tot;
  if (bad_sh) {
    R.status[b] = 1;
    R.abort_iter[b] = k;
    R.rec_obj[(size_t)b * R.cap + k] = qnan();
    R.rec_flags[(size_t)b * R.cap + k] = 0;
    R.n_recs[b] = k + 1;
  }
}

// one-pass iteration: the update of the previous evaluation pass (R.gpend) lands first
__global__ void apply_pending_kernel(DevProblem P, DevRun R, double rho) {
  const int b = blockIdx.y;
  if (R.done[b] || R.status[b]) return;
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < P.K; j += gridDim.x * blockDim.x) {
    const size_t i = (size_t)b * P.K + j;
    R.u[i] = __fma_rn(rho, R.gpend[i], R.u[i]);
  }
}

__global__ void save_tasks_kernel(DevProblem P, DevRun R) {
  const int b = blockIdx.y;
  if (R.done[b] || R.status[b]) return;
  const size_t n = (size_t)P.L * P.d;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    R.old_init[(size_t)b * n + i] = R.task_init[(size_t)b * n + i];
    R.old_targ[(size_t)b * n + i] = R.task_targ[(size_t)b * n + i];
  }
}

// the residual total the merge would have formed (same index-order block reduction)
__global__ void __launch_bounds__(128) total_error_kernel(DevProblem P, DevRun R) {
  __shared__ double sh[128];
  const int b = blockIdx.x;
  if (R.done[b] || R.status[b]) return;
  double tot = 0.0;
  for (int n = threadIdx.x; n < P.L; n += 128) tot += R.err[(size_t)b * P.L + n];
  tot = block_sum<128>(tot, sh);
  if (threadIdx.x == 0) R.tot_err[b] = tot;
}

// compose_from_propagators for d <= 1024 held row-major: psi_{n+1} = M_n psi_n,
// chi_n = M_n^dagger chi_{n+1}.  One CTA per problem, rows over threads.
__global__ void chain_kernel(DevProblem P, DevRun R) {
  extern __shared__ double2 vsh[];
  const int b = blockIdx.x;
  if (R.done[b] || R.status[b]) return;
  const int d = P.d, L = P.L;
  double2* psi = R.psi_nodes + (size_t)b * (L + 1) * d;
  double2* chi = R.chi_nodes + (size_t)b * (L + 1) * d;
  for (int i = threadIdx.x; i < d; i += blockDim.x) {
    psi[i] = P.init[(size_t)b * d + i];
    chi[(size_t)L * d + i] = P.targ[(size_t)b * d + i];
  }
  __syncthreads();
  for (int n = 0; n < L; ++n) {
    const double2* M = R.prop + ((size_t)b * L + n) * (size_t)d * d;
    for (int i = threadIdx.x; i < d; i += blockDim.x) vsh[i] = psi[(size_t)n * d + i];
    __syncthreads();
    for (int i = threadIdx.x; i < d; i += blockDim.x) {
      double2 acc = cx(0.0, 0.0);
      for (int kk = 0; kk < d; ++kk) acc = cfma(M[(size_t)i * d + kk], vsh[kk], acc);
      psi[(size_t)(n + 1) * d + i] = acc;
    }
    __syncthreads();
  }
  for (int n = L - 1; n >= 0; --n) {
    const double2* M = R.prop + ((size_t)b * L + n) * (size_t)d * d;
    for (int i = threadIdx.x; i < d; i += blockDim.x) vsh[i] = chi[(size_t)(n + 1) * d + i];
    __syncthreads();
    for (int i = threadIdx.x; i < d; i += blockDim.x) {
      double2 acc = cx(0.0, 0.0);
      for (int kk = 0; kk < d; ++kk) acc = cfmaconj(M[(size_t)kk * d + i], vsh[kk], acc);
      chi[(size_t)n * d + i] = acc;
    }
    __syncthreads();
  }
}

// compose_from_propagators for d <= 32: one warp per (problem, direction) -- blockIdx.y = 0
// runs psi_{n+1} = M_n psi_n upward, 1 runs chi_n = M_n^dag chi_{n+1} downward; the two chains
// are independent.  The chain is bound by instruction latency on one warp, so each step is
// kept to a minimum of instructions: the matrices stream into an S-deep shared-memory ring
// by TMA bulk copies (one instruction per matrix, issued S-1 steps ahead, completing on
// per-slot mbarriers) and the state vector is broadcast through shared memory (one LDS.128
// per element instead of four SHFL).
template <int TD, int S, int DIM = 0>
__global__ void __launch_bounds__(32) chain_small_kernel(DevProblem P, DevRun R) {
  extern __shared__ __align__(128) unsigned char chain_smem[];
  const int b = blockIdx.x, dir = blockIdx.y, lane = threadIdx.x;
  if (R.done[b] || R.status[b]) return;
  // DIM > 0: dimension fixed at compile time (the rotor, d = 21): no guards in the dot products
  const int d = DIM > 0 ? DIM : P.d, L = P.L, dd = d * d;
  const unsigned mbytes = (unsigned)(sizeof(double2) * dd);
  const unsigned slot = (mbytes + 127u) & ~127u;
  unsigned long long* bars = reinterpret_cast<unsigned long long*>(chain_smem);
  double2* vsh = reinterpret_cast<double2*>(chain_smem + 128);
  unsigned char* ring = chain_smem + 128 + 16 * 32;
  double2* psi = R.psi_nodes + (size_t)b * (L + 1) * d;
  double2* chi = R.chi_nodes + (size_t)b * (L + 1) * d;
  const double2* base = R.prop + (size_t)b * L * dd;
  const bool act = lane < d;
  const int li = act ? lane : 0;
  auto idx = [&](int q) { return dir == 0 ? q : L - 1 - q; };
  if (lane == 0) {
    for (int k = 0; k < S; ++k) mbar_init(&bars[k], 1);
    mbar_init_fence();
  }
  __syncwarp();
  auto issue = [&](int q) {
    if (lane == 0 && q < L) {
      unsigned long long* bar = &bars[q % S];
      mbar_expect_tx(bar, mbytes);
      bulk_g2s(ring + (size_t)(q % S) * slot, base + (size_t)idx(q) * dd, mbytes, bar);
    }
  };
  double2 v = cx(0.0, 0.0);
  if (dir == 0) {
    if (act) v = P.init[(size_t)b * d + lane];
    if (act) psi[lane] = v;
  } else {
    if (act) v = P.targ[(size_t)b * d + lane];
    if (act) chi[(size_t)L * d + lane] = v;
  }
  for (int q = 0; q < S - 1; ++q) issue(q);
  for (int q = 0; q < L; ++q) {
    issue(q + S - 1);
    vsh[lane] = v;
    mbar_wait(&bars[q % S], (unsigned)((q / S) & 1));
    __syncwarp();
    const double2* M = reinterpret_cast<const double2*>(ring + (size_t)(q % S) * slot);
    double2 acc[4] = {cx(0.0, 0.0), cx(0.0, 0.0), cx(0.0, 0.0), cx(0.0, 0.0)};
    if (dir == 0) {
#pragma unroll
      for (int k = 0; k < TD; ++k)
        if (k < d) acc[k & 3] = cfma(M[li * d + k], vsh[k], acc[k & 3]);
    } else {
#pragma unroll
      for (int k = 0; k < TD; ++k)
        if (k < d) acc[k & 3] = cfmaconj(M[k * d + li], vsh[k], acc[k & 3]);
    }
    v = cadd(cadd(acc[0], acc[1]), cadd(acc[2], acc[3]));
    const int n = idx(q);
    if (act) {
      if (dir == 0) psi[(size_t)(n + 1) * d + lane] = v;
      else chi[(size_t)n * d + lane] = v;
    }
    __syncwarp();  // slot q % S and vsh are rewritten next iteration
  }
}

// Split variant, assembled plan: lagged endpoint states become the new nodes (ism.cpp:546-552).
__global__ void split_nodes_kernel(DevProblem P, DevRun R) {
  const int b = blockIdx.x;
  if (R.done[b] || R.status[b]) return;
  const int d = P.d, L = P.L;
  double2* psi = R.psi_nodes + (size_t)b * (L + 1) * d;
  double2* chi = R.chi_nodes + (size_t)b * (L + 1) * d;
  for (int e = threadIdx.x; e < L * d; e += blockDim.x) {
    const int n = e / d, i = e % d;
    psi[(size_t)(n + 1) * d + i] = R.psi_end[((size_t)b * L + n) * d + i];
    chi[(size_t)n * d + i] = R.chi_start[((size_t)b * L + n) * d + i];
  }
  for (int i = threadIdx.x; i < d; i += blockDim.x) {
    psi[i] = P.init[(size_t)b * d + i];
    chi[(size_t)L * d + i] = P.targ[(size_t)b * d + i];
  }
}

// Finite checks of the nodes, boundary objective, task rebuild.
template <int NT>
__global__ void __launch_bounds__(NT) boundary_kernel(DevProblem P, DevRun R, int k, int split, int boot) {
  if (R.kdev) k = *R.kdev;  // graph replay: the iteration index lives on the device
  __shared__ double sh[NT];
  __shared__ int bad_sh;
  const int b = blockIdx.x;
  if (R.done[b] || R.status[b]) return;
  const int d = P.d, L = P.L;
  const double2* psi = R.psi_nodes + (size_t)b * (L + 1) * d;
  const double2* chi = R.chi_nodes + (size_t)b * (L + 1) * d;
  if (threadIdx.x == 0) bad_sh = 0;
  __syncthreads();
  int bad = 0;
  for (int e = threadIdx.x; e < (L + 1) * d; e += NT) bad |= !cfinite(psi[e]) | !cfinite(chi[e]);
  if (bad) atomicOr(&bad_sh, 1);
  __syncthreads();
  if (bad_sh) {
    if (threadIdx.x == 0) {
      R.status[b] = boot ? 3 : 2;
      R.abort_iter[b] = k;
      R.rec_obj[(size_t)b * R.cap + k] = qnan();
      R.rec_flags[(size_t)b * R.cap + k] = 0;
      R.n_recs[b] = k + 1;
    }
    return;
  }
  // boundary_objective (ism.cpp:285-296)
  const double2* last = psi + (size_t)L * d;
  const double2* tg = P.targ + (size_t)b * d;
  double part = 0.0;
  for (int i = threadIdx.x; i < d; i += NT) {
    if (split) part += cconjmul(tg[i], last[i]).x;
    else part += cabs2(csub(last[i], tg[i]));
  }
  const double s = block_sum<NT>(part, sh);
  double penp = 0.0;
  for (int n = threadIdx.x; n < L; n += NT) penp += R.pen[(size_t)b * L + n];
  const double pen = block_sum<NT>(penp, sh);
  if (threadIdx.x == 0) {
    double fid;
    if (split) {
      fid = P.ip_w * s;
    } else {
      const double dist = sqrt(fmax(0.0, P.ip_w * s));
      fid = -0.5 * dist * dist;
    }
    R.rec_obj[(size_t)b * R.cap + k] = fid - 0.5 * P.dt * pen;
  }
  // rebuild_tasks (ism.cpp:260-280)
  const double total = (double)P.K;
  for (int e = threadIdx.x; e < L * d; e += NT) {
    const int n = e / d, i = e % d;
    double2 in, tgv;
    if (split) {
      in = psi[(size_t)n * d + i];
      tgv = chi[(size_t)(n + 1) * d + i];
    } else {
      const int j0 = P.node[n], j1 = P.node[n + 1];
      const double a0 = (total - j0) / total, b0 = j0 / total;
      const double a1 = (total - j1) / total, b1 = j1 / total;
      const double2 p0 = psi[(size_t)n * d + i], c0 = chi[(size_t)n * d + i];
      const double2 p1 = psi[(size_t)(n + 1) * d + i], c1 = chi[(size_t)(n + 1) * d + i];
      in = cx(a0 * p0.x + b0 * c0.x, a0 * p0.y + b0 * c0.y);
      tgv = cx(a1 * p1.x + b1 * c1.x, a1 * p1.y + b1 * c1.y);
    }
    R.task_init[((size_t)b * L + n) * d + i] = in;
    R.task_targ[((size_t)b * L + n) * d + i] = tgv;
  }
}

__global__ void single_tasks_kernel(DevProblem P, DevRun R) {
  const int b = blockIdx.x;
  for (int i = threadIdx.x; i < P.d; i += blockDim.x) {
    R.task_init[(size_t)b * P.d + i] = P.init[(size_t)b * P.d + i];
    R.task_targ[(size_t)b * P.d + i] = P.targ[(size_t)b * P.d + i];
  }
}

// Record the residual, stop on eta (ism.cpp:586-591).
__global__ void finish_kernel(DevProblem P, DevRun R, int k, int compute_error, double eta, int log_exact) {
  if (R.kdev) k = *R.kdev;  // graph replay: the iteration index lives on the device
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= P.B || R.done[b] || R.status[b]) return;
  const size_t r = (size_t)b * R.cap + k;
  if (P.L == 1) R.rec_obj[r] = qnan();
  R.rec_err[r] = compute_error ? R.tot_err[b] : qnan();
  R.rec_flags[r] = (compute_error ? 1 : 0) | (log_exact ? 2 : 0);
  R.n_recs[b] = k + 1;
  if (compute_error && R.tot_err[b] <= eta) R.done[b] = 1;
}

// Trailing evaluation (ism.cpp:594-609).
__global__ void trailing_kernel(DevProblem P, DevRun R) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= P.B || R.status[b]) return;
  const int last = R.n_recs[b] - 1;
  double* tv = R.rec_tv + ((size_t)b * R.cap + last) * P.L;
  for (int n = 0; n < P.L; ++n) tv[n] = R.entry[(size_t)b * P.L + n];
  if (P.L == 1) R.rec_obj[(size_t)b * R.cap + last] = R.entry[b];
}

}  // namespace

cudaError_t penalty_partials(const DevProblem& P, const DevRun& R, int ignore_done, cudaStream_t st) {
  penalty_kernel<<<dim3(P.L, P.B), 32, 0, st>>>(P, R, ignore_done);
  return cudaGetLastError();
}
cudaError_t merge_iteration(const DevProblem& P, const DevRun& R, int k, double*, cudaStream_t st) {
  merge_kernel<<<P.B, 128, 0, st>>>(P, R, k);
  return cudaGetLastError();
}
cudaError_t chain_propagators(const DevProblem& P, const DevRun& R, cudaStream_t st) {
  if (P.kind == 4 /* QOC_KIND_DENSITY */) return density_chain(P, R, st);
  const size_t slot = (sizeof(double2) * P.d * P.d + 127) & ~(size_t)127;
  auto go = [&](auto kern, int S) -> cudaError_t {
    const size_t smem = 128 + 16 * 32 + S * slot;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    kern<<<dim3(P.B, 2), 32, smem, st>>>(P, R);
    return cudaGetLastError();
  };
  if (P.d <= 8) {
    return go(chain_small_kernel<8, 8>, 8);
  } else if (P.d <= 16) {
    return go(chain_small_kernel<16, 8>, 8);
  } else if (P.d == 21) {
    return go(chain_small_kernel<21, 8, 21>, 8);
  } else if (P.d <= 24) {
    return go(chain_small_kernel<24, 8>, 8);
  } else if (P.d <= 32) {
    return go(chain_small_kernel<32, 4>, 4);
  } else {
    const int nt = P.d >= 256 ? 1024 : 256;
    chain_kernel<<<P.B, nt, sizeof(double2) * P.d, st>>>(P, R);
  }
  return cudaGetLastError();
}
cudaError_t split_nodes(const DevProblem& P, const DevRun& R, cudaStream_t st) {
  split_nodes_kernel<<<P.B, 256, 0, st>>>(P, R);
  return cudaGetLastError();
}
cudaError_t boundary_update(const DevProblem& P, const DevRun& R, int k, int split, int boot, cudaStream_t st) {
  if (P.B <= 64 && P.L * P.d >= 1024)  // few problems, many nodes: wider blocks hide the L2 latency
    boundary_kernel<512><<<P.B, 512, 0, st>>>(P, R, k, split, boot);
  else
    boundary_kernel<128><<<P.B, 128, 0, st>>>(P, R, k, split, boot);
  return cudaGetLastError();
}
cudaError_t set_single_tasks(const DevProblem& P, const DevRun& R, cudaStream_t st) {
  single_tasks_kernel<<<P.B, 128, 0, st>>>(P, R);
  return cudaGetLastError();
}
cudaError_t finish_iteration(const DevProblem& P, const DevRun& R, int k, const double*, int compute_error,
                             double eta, cudaStream_t st) {
  finish_kernel<<<(P.B + 127) / 128, 128, 0, st>>>(P, R, k, compute_error, eta, 0);
  return cudaGetLastError();
}
cudaError_t finish_iteration_ex(const DevProblem& P, const DevRun& R, int k, int compute_error, double eta,
                                int log_exact, cudaStream_t st) {
  finish_kernel<<<(P.B + 127) / 128, 128, 0, st>>>(P, R, k, compute_error, eta, log_exact);
  return cudaGetLastError();
}
cudaError_t apply_pending(const DevProblem& P, const DevRun& R, double rho, cudaStream_t st) {
  apply_pending_kernel<<<dim3((P.K + 255) / 256, P.B), 256, 0, st>>>(P, R, rho);
  return cudaGetLastError();
}
cudaError_t save_tasks(const DevProblem& P, const DevRun& R, cudaStream_t st) {
  save_tasks_kernel<<<dim3((P.L * P.d + 255) / 256, P.B), 256, 0, st>>>(P, R);
  return cudaGetLastError();
}
cudaError_t total_error(const DevProblem& P, const DevRun& R, cudaStream_t st) {
  total_error_kernel<<<P.B, 128, 0, st>>>(P, R);
  return cudaGetLastError();
}
cudaError_t trailing_values(const DevProblem& P, const DevRun& R, cudaStream_t st) {
  trailing_kernel<<<(P.B + 127) / 128, 128, 0, st>>>(P, R);
  return cudaGetLastError();
}

}  // namespace qoc
