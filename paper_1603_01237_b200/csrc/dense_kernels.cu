// dense_kernels.cu — task and horizon kernels for QOC_KIND_DENSE (sm_100a).
//
// Task kernel = one ISM subinterval task of ism.cpp:401-479, fused:
//   phase 1 (control u):      forward sweep with trajectory (entry value, sub_functional,
//                             objective.cpp:131-134) + adjoint sweep with the gradient
//                             (gradient_sweep cn_dense, objective.cpp:48-60) and the in-place
//                             ascent update u += rho * w g (optimizers.cpp:102-107).
//   phase 2 (updated control): one forward sweep that carries the residual state, the lagged
//                             split state and the propagator product together (one inverse
//                             per step), then one adjoint sweep that carries the residual
//                             adjoint (error_norm, objective.cpp:152-160) and the lagged
//                             adjoint (ism.cpp:424-459).
#include "dense.cuh"
#include "kernels.h"

namespace qoc {

template <int D, int G>
struct DenseKernel {
  using Cfg = DenseCfg<D, G>;
  using Lane = DenseLane<D, G>;
  static constexpr int NL = Cfg::NL, COLS = Cfg::COLS, TPW = Cfg::TPW;

  __host__ __device__ static size_t group_bytes() {
    return sizeof(double2) * (Cfg::PIV + Cfg::VEC + 2 * Cfg::MAT) + sizeof(int) * 2 * D;
  }
  __host__ __device__ static size_t ops_bytes(int C, int has_quad) {
    return sizeof(double2) * (size_t)(1 + C + (has_quad ? C : 0)) * D * D;
  }
};

template <int D, int G>
__device__ __forceinline__ DenseScratch<D, G> group_scratch(unsigned char* base, int gid) {
  using Cfg = DenseCfg<D, G>;
  const size_t bytes = sizeof(double2) * (Cfg::PIV + Cfg::VEC + 2 * Cfg::MAT) + sizeof(int) * 2 * D;
  unsigned char* p = base + bytes * gid;
  DenseScratch<D, G> s;
  s.piv = reinterpret_cast<double2*>(p);
  s.vec = s.piv + Cfg::PIV;
  s.matW = s.vec + Cfg::VEC;
  s.matP = s.matW + Cfg::MAT;
  s.perm = reinterpret_cast<int*>(s.matP + Cfg::MAT);
  return s;
}

__device__ __forceinline__ void load_ops(double2* ops, const DevProblem& P, int b, int D) {
  const int nops = 1 + P.C + (P.has_quad ? P.C : 0);
  const int d = P.d;
  for (int e = threadIdx.x; e < nops * D * D; e += blockDim.x) {
    const int o = e / (D * D), r = (e / D) % D, c = e % D;
    double2 v = cx(0.0, 0.0);
    if (r < d && c < d) {
      const size_t dd = (size_t)d * d;
      if (o == 0) v = P.h0[(size_t)b * dd + r * d + c];
      else if (o <= P.C) v = P.lin[((size_t)b * P.C + (o - 1)) * dd + r * d + c];
      else v = P.quad[((size_t)b * P.C + (o - 1 - P.C)) * dd + r * d + c];
    }
    ops[e] = v;
  }
}

// Pivot-free Gauss-Jordan is exact partial pivoting while dt/2 ||H(u)||_1 < 1.
__device__ __forceinline__ bool needs_pivoting(const DevProblem& P, int b, const double* u, double half) {
  const double* nrm = P.norm1 + (size_t)b * (1 + 2 * P.C);
  double bound = nrm[0];
  for (int c = 0; c < P.C; ++c) {
    bound += fabs(u[c]) * nrm[1 + c];
    if (P.has_quad) bound += 0.5 * u[c] * u[c] * nrm[1 + P.C + c];
  }
  return !(half * bound < 1.0);
}

template <int D, int G>
__device__ __forceinline__ void step_inverse(const Lane_t<D, G>& L, double2 (&W)[D / G], const double2* ops,
                                             const DevProblem& P, int b, const double* uj, double half,
                                             bool adj, const DenseScratch<D, G>& s, int lane) {
  L.build(W, ops, P.C, P.has_quad, uj, half, adj);
  if (__any_sync(0xffffffffu, needs_pivoting(P, b, uj, half)))
    L.invert_pivot(W, s, lane);
  else
    L.invert_fast(W, s.piv);
}

template <int D, int G>
__global__ void __launch_bounds__(256) dense_task_kernel(DevProblem P, DevRun R, TaskArgs A, int tasks_per_cta,
                                                         int ignore_done) {
  using K_ = DenseKernel<D, G>;
  constexpr int NL = K_::NL, COLS = K_::COLS, TPW = K_::TPW;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double2* ops = reinterpret_cast<double2*>(smem_raw);
  const int b = blockIdx.y;
  const bool skip = ignore_done ? (R.status[b] != 0) : ((R.done[b] | R.status[b]) != 0);
  if (skip) return;  // uniform over the CTA
  load_ops(ops, P, b, D);
  __syncthreads();

  const int warp = threadIdx.x >> 5, l32 = threadIdx.x & 31;
  const int gid = warp * TPW + l32 / NL;
  const int lane = l32 % NL;
  const int n_raw = blockIdx.x * tasks_per_cta + gid;
  const bool live_task = n_raw < P.L;
  if (!__any_sync(0xffffffffu, live_task)) return;
  const int n = live_task ? n_raw : P.L - 1;
  unsigned char* scratch_base = smem_raw + K_::ops_bytes(P.C, P.has_quad);
  const DenseScratch<D, G> S = group_scratch<D, G>(scratch_base, gid);
  Lane_t<D, G> L;
  L.row = lane % D;
  L.g = lane / D;
  const int row = L.row, g = L.g, d = P.d, C = P.C;

  const int node0 = P.node[n];
  const int len = P.node[n + 1] - node0;
  int lenmax = len;
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) lenmax = max(lenmax, __shfl_xor_sync(0xffffffffu, lenmax, off));
  const double Kd = (double)P.K;
  const double weight = A.weighted ? Kd / (double)len : 1.0;
  const double scale = (double)len / Kd;
  const double half = 0.5 * P.dt, dt = P.dt, w = P.ip_w;
  double* u = R.u + ((size_t)b * P.K + node0) * C;
  double2* traj = R.traj + ((size_t)b * P.L + n) * (size_t)R.traj_len * D;
  const size_t tix = ((size_t)b * P.L + n) * d;
  const double2 zero = cx(0.0, 0.0);
  const double2 init = row < d ? R.task_init[tix + row] : zero;
  const double2 targ = row < d ? R.task_targ[tix + row] : zero;
  const bool writer = live_task && g == 0 && row < d;
  const bool lead = live_task && lane == 0;
  const int mode = A.mode;

  double2 W[COLS];

  // ---------------- phase 1: sweeps at the current control -------------------------
  if (mode & (M_ENTRY | M_UPDATE | M_FINAL | M_GRAD)) {
    const bool need_traj = (mode & (M_UPDATE | M_GRAD)) != 0;
    const int iters = (mode & M_UPDATE) ? A.inner : 1;
    for (int it = 0; it < iters; ++it) {
      double2 x = init;
      double pen = 0.0;
      if (need_traj && g == 0 && live_task) traj[row] = x;
      for (int j = 0; j < lenmax; ++j) {
        const bool live = j < len;
        const double* uj = u + (size_t)min(j, len - 1) * C;
        step_inverse<D, G>(L, W, ops, P, b, uj, half, false, S, lane);
        const double2 xn = L.cayley_apply(W, x, S.vec);
        if (live) {
          x = xn;
          if (need_traj && g == 0 && live_task) traj[(size_t)(j + 1) * D + row] = x;
          double sq = 0.0;
          for (int c = 0; c < C; ++c) sq += uj[c] * uj[c];
          pen += (P.alpha[node0 + j] * scale) * sq;
        }
      }
      if (it == 0 && (mode & M_ENTRY)) {
        double2 t;
        if (A.form == 0) {
          t = row < d ? cconjmul(targ, x) : zero;
        } else {
          const double2 df = csub(x, targ);
          t = cx(row < d ? cabs2(df) : 0.0, 0.0);
        }
        const double2 s = L.row_sum(t);
        const double payoff = A.form == 0 ? (w * s.x) : (-0.5 * (w * s.x));
        if (lead) R.entry[(size_t)b * P.L + n] = weight * (payoff - 0.5 * dt * pen);
      }
      if (it == 0 && (mode & M_FINAL) && writer) R.psi_end[tix + row] = x;
      if (mode & (M_UPDATE | M_GRAD)) {
        double2 chi = A.form == 0 ? targ : csub(targ, x);
        __syncwarp();
        for (int j = lenmax - 1; j >= 0; --j) {
          const bool live = j < len;
          const int jj = min(j, len - 1);
          const double* uj = u + (size_t)jj * C;
          step_inverse<D, G>(L, W, ops, P, b, uj, half, true, S, lane);
          const double2 cn = L.cayley_apply(W, chi, S.vec);
          const double2 ps = cadd(traj[(size_t)jj * D + row], traj[(size_t)(jj + 1) * D + row]);
          const double2 cs = cadd(cn, chi);
          const double aj = P.alpha[node0 + jj] * scale;
          for (int c = 0; c < C; ++c) {
            const double uc = uj[c];  // channel c is written only after its own gradient
            const double im = L.grad_term(ops, C, P.has_quad, c, uc, ps, cs, S.vec);
            const double gc = -aj * dt * uc + 0.25 * dt * (w * im);
            if (live && lead) {
              if (mode & M_GRAD) R.grad[((size_t)b * P.K + node0 + jj) * C + c] = gc;
              if (mode & M_UPDATE) u[(size_t)jj * C + c] = uc + A.rho * (weight * gc);
            }
          }
          if (live) chi = cn;
          __syncwarp();
        }
      }
      __syncwarp();
    }
  }

  // ---------------- phase 2: sweeps at the updated control -------------------------
  const bool do_err = (mode & M_ERROR) != 0, do_asm = (mode & M_ASSEMBLE) != 0,
             do_lag = (mode & M_LAGGED) != 0;
  if (do_err || do_asm || do_lag) {
    double2 xe = init;
    double2 xl = (do_lag && row < d) ? R.psi_nodes[((size_t)b * (P.L + 1) + n) * d + row] : zero;
    double2 Pm[COLS];
#pragma unroll
    for (int t = 0; t < COLS; ++t) Pm[t] = cx(row == L.col(t, g) ? 1.0 : 0.0, 0.0);
    if (do_err && g == 0 && live_task) traj[row] = xe;
    for (int j = 0; j < lenmax; ++j) {
      const bool live = j < len;
      const double* uj = u + (size_t)min(j, len - 1) * C;
      step_inverse<D, G>(L, W, ops, P, b, uj, half, false, S, lane);
      double2 a = xe, c2 = xl;
      if (do_err && do_lag) L.cayley_apply2(W, a, c2, S.vec);
      else if (do_err) a = L.cayley_apply(W, a, S.vec);
      else if (do_lag) c2 = L.cayley_apply(W, c2, S.vec);
      if (do_asm) {
        double2 Q[COLS];
#pragma unroll
        for (int t = 0; t < COLS; ++t) Q[t] = Pm[t];
        L.cayley_matmul(W, Q, S);
        if (live) {
#pragma unroll
          for (int t = 0; t < COLS; ++t) Pm[t] = Q[t];
        }
      }
      if (live) {
        xe = a;
        xl = c2;
        if (do_err && g == 0 && live_task) traj[(size_t)(j + 1) * D + row] = xe;
      }
    }
    if (do_asm && live_task && row < d) {
      double2* M = R.prop + ((size_t)b * P.L + n) * (size_t)d * d;
#pragma unroll
      for (int t = 0; t < COLS; ++t) {
        const int jc = L.col(t, g);
        if (jc < d) M[(size_t)row * d + jc] = Pm[t];
      }
    }
    if (do_lag && writer) R.psi_end[tix + row] = xl;
    if (do_err || do_lag) {
      double2 ce = A.form == 0 ? targ : csub(targ, xe);
      double2 cl = (do_lag && row < d) ? R.chi_nodes[((size_t)b * (P.L + 1) + n + 1) * d + row] : zero;
      double err = 0.0;
      __syncwarp();
      for (int j = lenmax - 1; j >= 0; --j) {
        const bool live = j < len;
        const int jj = min(j, len - 1);
        const double* uj = u + (size_t)jj * C;
        step_inverse<D, G>(L, W, ops, P, b, uj, half, true, S, lane);
        double2 a = ce, c2 = cl;
        if (do_err && do_lag) L.cayley_apply2(W, a, c2, S.vec);
        else if (do_err) a = L.cayley_apply(W, a, S.vec);
        else c2 = L.cayley_apply(W, c2, S.vec);
        if (do_err) {
          const double2 ps = cadd(traj[(size_t)jj * D + row], traj[(size_t)(jj + 1) * D + row]);
          const double2 cs = cadd(a, ce);
          const double aj = P.alpha[node0 + jj] * scale;
          double sq = 0.0;
          for (int c = 0; c < C; ++c) {
            const double uc = uj[c];
            const double im = L.grad_term(ops, C, P.has_quad, c, uc, ps, cs, S.vec);
            const double gc = -aj * dt * uc + 0.25 * dt * (w * im);
            sq += gc * gc;
          }
          if (live) err += sqrt(sq);
        }
        if (live) {
          ce = a;
          cl = c2;
        }
      }
      if (do_err && lead) R.err[(size_t)b * P.L + n] = err;
      if (do_lag && writer) R.chi_start[tix + row] = cl;
    }
  }
}

// Serial full-horizon sweeps on one lane group per problem (node_sweeps, ism.cpp:35-84, and
// the exact payoff instrumentation, ism.cpp:580-584 / objective.cpp:93-100).
//   which = 0: forward nodes psi_n + adjoint nodes chi_n (seeded with the target, ism.cpp:72)
//   which = 1: overlap payoff of the full propagation minus the full penalty -> rec_exact[k]
template <int D, int G>
__global__ void __launch_bounds__(32) dense_horizon_kernel(DevProblem P, DevRun R, int which, int k) {
  if (R.kdev) k = *R.kdev;
  using K_ = DenseKernel<D, G>;
  constexpr int NL = K_::NL, COLS = K_::COLS;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double2* ops = reinterpret_cast<double2*>(smem_raw);
  const int b = blockIdx.x;
  if (R.done[b] || R.status[b]) return;
  load_ops(ops, P, b, D);
  __syncthreads();
  const int lane32 = threadIdx.x & 31;
  const bool live_lane = lane32 < NL;  // groups beyond the first only mirror group 0
  const int lane = lane32 % NL;
  const DenseScratch<D, G> S = group_scratch<D, G>(smem_raw + K_::ops_bytes(P.C, P.has_quad), lane32 / NL);
  Lane_t<D, G> L;
  L.row = lane % D;
  L.g = lane / D;
  const int row = L.row, g = L.g, d = P.d, C = P.C;
  const double half = 0.5 * P.dt;
  const double* u = R.u + (size_t)b * P.K * C;
  const double2 zero = cx(0.0, 0.0);
  double2 W[COLS];
  double2 x = row < d ? P.init[(size_t)b * d + row] : zero;
  const size_t nb = (size_t)b * (P.L + 1) * d;
  int nxt = 1;
  if (which == 0 && live_lane && g == 0 && row < d) R.psi_nodes[nb + row] = x;
  for (int j = 0; j < P.K; ++j) {
    step_inverse<D, G>(L, W, ops, P, b, u + (size_t)j * C, half, false, S, lane);
    x = L.cayley_apply(W, x, S.vec);
    if (which == 0 && nxt <= P.L && P.node[nxt] == j + 1) {
      if (live_lane && g == 0 && row < d) R.psi_nodes[nb + (size_t)nxt * d + row] = x;
      ++nxt;
    }
  }
  if (which == 1) {
    const double2 t = row < d ? cconjmul(P.targ[(size_t)b * d + row], x) : zero;
    const double s = L.row_sum(t).x;
    if (lane32 == 0) {
      double pen = 0.0;
      for (int n = 0; n < P.L; ++n) pen += R.pen[(size_t)b * P.L + n];
      R.rec_exact[(size_t)b * R.cap + k] = P.ip_w * s - 0.5 * P.dt * pen;
    }
    return;
  }
  double2 chi = row < d ? P.targ[(size_t)b * d + row] : zero;
  if (live_lane && g == 0 && row < d) R.chi_nodes[nb + (size_t)P.L * d + row] = chi;
  int prev = P.L - 1;
  for (int j = P.K - 1; j >= 0; --j) {
    step_inverse<D, G>(L, W, ops, P, b, u + (size_t)j * C, half, true, S, lane);
    chi = L.cayley_apply(W, chi, S.vec);
    if (prev >= 0 && P.node[prev] == j) {
      if (live_lane && g == 0 && row < d) R.chi_nodes[nb + (size_t)prev * d + row] = chi;
      --prev;
    }
  }
}

// ---- launchers ------------------------------------------------------------------------
template <int D, int G>
static cudaError_t launch_dense_task(const DevProblem& P, const DevRun& R, const TaskArgs& A, int ignore_done,
                                     cudaStream_t st) {
  using K_ = DenseKernel<D, G>;
  constexpr int TPW = K_::TPW;
  int warps = (P.L + TPW - 1) / TPW;
  if (warps > 8) warps = 8;
  const int tpc = warps * TPW;
  const size_t smem = K_::ops_bytes(P.C, P.has_quad) + K_::group_bytes() * tpc;
  auto kern = dense_task_kernel<D, G>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  dim3 grid((P.L + tpc - 1) / tpc, P.B);
  kern<<<grid, warps * 32, smem, st>>>(P, R, A, tpc, ignore_done);
  return cudaGetLastError();
}

template <int D, int G>
static cudaError_t launch_dense_horizon(const DevProblem& P, const DevRun& R, int which, int k, cudaStream_t st) {
  using K_ = DenseKernel<D, G>;
  const size_t smem = K_::ops_bytes(P.C, P.has_quad) + K_::group_bytes() * K_::TPW;
  auto kern = dense_horizon_kernel<D, G>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  kern<<<P.B, 32, smem, st>>>(P, R, which, k);
  return cudaGetLastError();
}

int dense_pad(int d) {
  if (d <= 2) return 2;
  if (d <= 4) return 4;
  if (d <= 8) return 8;
  if (d <= 16) return 16;
  if (d <= 32) return 32;
  return -1;
}

cudaError_t dense_task(const DevProblem& P, const DevRun& R, const TaskArgs& A, int ignore_done, cudaStream_t st) {
  switch (dense_pad(P.d)) {
    case 2: return launch_dense_task<2, 1>(P, R, A, ignore_done, st);
    case 4: return launch_dense_task<4, 1>(P, R, A, ignore_done, st);
    case 8: return launch_dense_task<8, 1>(P, R, A, ignore_done, st);
    case 16: return launch_dense_task<16, 2>(P, R, A, ignore_done, st);
    case 32: return launch_dense_task<32, 1>(P, R, A, ignore_done, st);
  }
  return cudaErrorInvalidValue;
}

cudaError_t dense_horizon(const DevProblem& P, const DevRun& R, int which, int k, cudaStream_t st) {
  switch (dense_pad(P.d)) {
    case 2: return launch_dense_horizon<2, 1>(P, R, which, k, st);
    case 4: return launch_dense_horizon<4, 1>(P, R, which, k, st);
    case 8: return launch_dense_horizon<8, 1>(P, R, which, k, st);
    case 16: return launch_dense_horizon<16, 2>(P, R, which, k, st);
    case 32: return launch_dense_horizon<32, 1>(P, R, which, k, st);
  }
  return cudaErrorInvalidValue;
}

}  // namespace qoc
