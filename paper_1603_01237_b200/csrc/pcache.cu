// pcache.cu — propagator-cache engine for the linear kinds (DENSE, TRIDIAG; d <= 32), sm_100a.
//
// The reference evaluates each subinterval task with step-by-step sweeps: a forward sweep, an
// adjoint sweep with the gradient (objective.cpp:38-89), a residual forward/adjoint pair and a
// d-column assembly sweep (ism.cpp:401-479).  Every one of them is a dependent chain of len
// Cayley steps.  This engine keeps, per task, the partial products of the one-step maps
//     P_0 = I,  P_{j+1} = C_j P_j,   C_j = (I + L_j)^-1 (I - L_j)     (propagation.cpp:236-249)
// and uses two exact identities of the discrete scheme:
//   forward states   psi_j = P_j phi                                   (propagate, 184-192)
//   adjoint states   chi_j = C_j^dag ... C_{len-1}^dag seed = P_j chi_0,  chi_0 = P_len^dag seed
// (C_j is unitary because H(u_j) is Hermitian, so C_j^-dag = C_j).  Given the cache, the
// entry value, gradient, residual and lagged endpoints are matvecs that are independent
// across j; the only sequential chain per outer iteration is one assembly sweep at the
// updated control, which the assembled plan needs for M_n = P_len anyway.
//
//   pc_eval_kernel      warp per (task, j-chunk): entry payoff, gradient + in-place ascent
//                       update (optimizers.cpp:102-107), residual norm partials, lagged
//                       endpoints, final state / raw gradient for the helper API.
//   pc_finalize_kernel  index-order reduction of the chunk partials.
//   dense_pc_assemble   lane group per task: in-register Gauss-Jordan inverse of B_j, then
//                       P_{j+1} = 2 B_j^-1 P_j - P_j.
//   tri_pc_assemble     warp per task, lane per column: Thomas elimination per column.
#include "dense.cuh"
#include "kernels.h"
#include "qoc_gpu.h"

namespace qoc {

namespace {

constexpr int PC_ENTRY = 1, PC_GRAD = 2, PC_ERR = 4, PC_LAG = 8, PC_FINAL = 16, PC_RAWGRAD = 32;

template <int D>
struct PcSmem {
  double2 phi[D];
  double2 chi0[D];
  double2 vec[D];
  double red[32];
};

// (dH/du_c ps)_i for this lane's row i, dense operators (row-major, global / L1); the row is
// loaded with all loads in flight (DM-wide unrolled) before the dot product.
template <int DM>
__device__ __forceinline__ double2 dense_dH_row(const DevProblem& P, int b, int c, double uc, int i,
                                                const double2* ps_sh) {
  const int d = P.d;
  const double2* a = P.lin + (((size_t)b * P.C + c) * d + i) * d;
  const double2* q = P.has_quad ? P.quad + (((size_t)b * P.C + c) * d + i) * d : nullptr;
  double2 m[DM];
#pragma unroll
  for (int k = 0; k < DM; ++k) m[k] = k < d ? __ldg(a + k) : cx(0.0, 0.0);
  if (q) {
#pragma unroll
    for (int k = 0; k < DM; ++k)
      if (k < d) {
        const double2 qq = __ldg(q + k);
        m[k] = cx(fma(uc, qq.x, m[k].x), fma(uc, qq.y, m[k].y));
      }
  }
  double2 acc0 = cx(0.0, 0.0), acc1 = cx(0.0, 0.0);
#pragma unroll
  for (int k = 0; k < DM; k += 2) {
    if (k < d) acc0 = cfma(m[k], ps_sh[k], acc0);
    if (k + 1 < d) acc1 = cfma(m[k + 1], ps_sh[k + 1], acc1);
  }
  return cadd(acc0, acc1);
}

// Tridiagonal (dH/du_c ps)_i with neighbours by shuffle.
__device__ __forceinline__ double2 tri_dH_row(const DevProblem& P, int b, int c, double uc, int i, double2 ps) {
  const int d = P.d, C = P.C;
  const int nops = 1 + C + (P.has_quad ? C : 0);
  const double* dg = P.tri_diag + (size_t)b * nops * d;
  const double2* sb = P.tri_sub + (size_t)b * nops * (d - 1);
  const double2 up = shfl(ps, (i + 31) & 31);   // ps_{i-1}
  const double2 dn = shfl(ps, (i + 1) & 31);    // ps_{i+1}
  if (i >= d) return cx(0.0, 0.0);
  double g = dg[(1 + c) * d + i];
  if (P.has_quad) g = fma(uc, dg[(1 + C + c) * d + i], g);
  double2 h = cx(g * ps.x, g * ps.y);
  if (i > 0) {
    double2 s = sb[(size_t)(1 + c) * (d - 1) + i - 1];
    if (P.has_quad) {
      const double2 qq = sb[(size_t)(1 + C + c) * (d - 1) + i - 1];
      s = cx(fma(uc, qq.x, s.x), fma(uc, qq.y, s.y));
    }
    h = cfma(s, up, h);
  }
  if (i + 1 < d) {
    double2 s = sb[(size_t)(1 + c) * (d - 1) + i];
    if (P.has_quad) {
      const double2 qq = sb[(size_t)(1 + C + c) * (d - 1) + i];
      s = cx(fma(uc, qq.x, s.x), fma(uc, qq.y, s.y));
    }
    h = cfmaconj(s, dn, h);
  }
  return h;
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
  return v;
}
template <int NL>
__device__ __forceinline__ double group_sum(double v) {  // sum over aligned groups of NL lanes
#pragma unroll
  for (int off = NL / 2; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
  return v;
}

// y_i = sum_k M[i][k] v_k (M row-major d x d, v in smem); lanes >= d return 0.  The row is
// loaded with every load in flight at once (these reads are HBM-latency-bound).
template <int DM>
__device__ __forceinline__ double2 matvec_row(const double2* M, int d, int i, const double2* v) {
  double2 r[DM];
  const double2* row = M + (size_t)(i < d ? i : 0) * d;
#pragma unroll
  for (int k = 0; k < DM; ++k) r[k] = k < d ? row[k] : cx(0.0, 0.0);
  double2 a = cx(0.0, 0.0), b = cx(0.0, 0.0);
#pragma unroll
  for (int k = 0; k < DM; k += 2) {
    if (k < d) a = cfma(r[k], v[k], a);
    if (k + 1 < d) b = cfma(r[k + 1], v[k + 1], b);
  }
  return i < d ? cadd(a, b) : cx(0.0, 0.0);
}
// Both y1 = M v1 and y2 = M v2 for this lane's row, the row loaded once with all its loads
// in flight together (the step loop is HBM-latency-bound, so the loads must not serialise).
template <int DM>
__device__ __forceinline__ void matvec_row2(const double2* M, int d, int i, const double2* v1,
                                            const double2* v2, double2& y1, double2& y2) {
  double2 r[DM];
  const double2* row = M + (size_t)(i < d ? i : 0) * d;
#pragma unroll
  for (int k = 0; k < DM; ++k) r[k] = k < d ? __ldcs(row + k) : cx(0.0, 0.0);
  double2 a0 = cx(0.0, 0.0), a1 = cx(0.0, 0.0), b0 = cx(0.0, 0.0), b1 = cx(0.0, 0.0);
#pragma unroll
  for (int k = 0; k < DM; k += 2) {
    if (k < d) {
      a0 = cfma(r[k], v1[k], a0);
      b0 = cfma(r[k], v2[k], b0);
    }
    if (k + 1 < d) {
      a1 = cfma(r[k + 1], v1[k + 1], a1);
      b1 = cfma(r[k + 1], v2[k + 1], b1);
    }
  }
  y1 = i < d ? cadd(a0, a1) : cx(0.0, 0.0);
  y2 = i < d ? cadd(b0, b1) : cx(0.0, 0.0);
}
template <int DM>
__device__ __forceinline__ void load_row(const double2* M, int d, int i, double2 (&r)[DM]) {
  const double2* row = M + (size_t)(i < d ? i : 0) * d;
#pragma unroll
  for (int k = 0; k < DM; ++k) r[k] = k < d ? __ldcs(row + k) : cx(0.0, 0.0);
}
template <int DM>
__device__ __forceinline__ void rows_dot2(const double2 (&r)[DM], int d, int i, const double2* v1,
                                          const double2* v2, double2& y1, double2& y2) {
  double2 a0 = cx(0.0, 0.0), a1 = cx(0.0, 0.0), b0 = cx(0.0, 0.0), b1 = cx(0.0, 0.0);
#pragma unroll
  for (int k = 0; k < DM; k += 2) {
    if (k < d) {
      a0 = cfma(r[k], v1[k], a0);
      b0 = cfma(r[k], v2[k], b0);
    }
    if (k + 1 < d) {
      a1 = cfma(r[k + 1], v1[k + 1], a1);
      b1 = cfma(r[k + 1], v2[k + 1], b1);
    }
  }
  y1 = i < d ? cadd(a0, a1) : cx(0.0, 0.0);
  y2 = i < d ? cadd(b0, b1) : cx(0.0, 0.0);
}
// y_i = sum_k conj(M[k][i]) v_k
template <int DM>
__device__ __forceinline__ double2 matvec_adj_row(const double2* M, int d, int i, const double2* v) {
  double2 c[DM];
  const int ii = i < d ? i : 0;
#pragma unroll
  for (int k = 0; k < DM; ++k) c[k] = k < d ? M[(size_t)k * d + ii] : cx(0.0, 0.0);
  double2 a = cx(0.0, 0.0), b = cx(0.0, 0.0);
#pragma unroll
  for (int k = 0; k < DM; k += 2) {
    if (k < d) a = cfmaconj(c[k], v[k], a);
    if (k + 1 < d) b = cfmaconj(c[k + 1], v[k + 1], b);
  }
  return i < d ? cadd(a, b) : cx(0.0, 0.0);
}

// NLT lanes per (task, chunk) item: 32, or 16 for d <= 16 (two items per warp; dense kinds
// with one chunk per task -- every group of a warp then runs the same control flow).
template <bool TRI, int DM, int DIM = 0, int NLT = 32>
__global__ void __launch_bounds__(128) pc_eval_kernel(DevProblem P, DevRun R, TaskArgs A, int chunk, int nchunk,
                                                      int ignore_done) {
  constexpr int GPW = 32 / NLT;
  __shared__ PcSmem<32> sm_all[4 * GPW];
  const int b = blockIdx.y;
  if (ignore_done ? R.status[b] : (R.done[b] | R.status[b])) return;
  const int warp = threadIdx.x >> 5, i = threadIdx.x & (NLT - 1), gid = (threadIdx.x & 31) / NLT;
  const int item_raw = (blockIdx.x * 4 + warp) * GPW + gid;
  const bool live = item_raw < P.L * nchunk;
  if (!__any_sync(0xffffffffu, live)) return;
  const int item = live ? item_raw : P.L * nchunk - 1;
  PcSmem<32>& S = sm_all[warp * GPW + gid];
  const int n = item / nchunk, ch = item % nchunk;
  const int d = DIM > 0 ? DIM : P.d, C = P.C, mode = A.mode;  // DIM: compile-time dimension
  const int node0 = P.node[n], len = P.node[n + 1] - node0;
  const int j0 = ch * chunk;
  const int j1 = min(len, j0 + chunk);
  int jmax = j1;  // uniform trip count over the warp's groups
#pragma unroll
  for (int off = 16; off >= NLT; off >>= 1) jmax = max(jmax, __shfl_xor_sync(0xffffffffu, jmax, off));
  const double Kd = (double)P.K;
  const double weight = A.weighted ? Kd / (double)len : 1.0;
  const double scale = (double)len / Kd;
  const double dt = P.dt, w = P.ip_w;
  double* u = R.u + ((size_t)b * P.K + node0) * C;
  const size_t dd = (size_t)d * d;
  const double2* Pc = R.pc + ((size_t)b * P.L + n) * (size_t)R.traj_len * dd;
  const size_t tix = ((size_t)b * P.L + n) * d;
  const size_t cix = ((size_t)b * P.L + n) * nchunk + ch;
  const double2 zero = cx(0.0, 0.0);
  const double2 phi = i < d ? R.task_init[tix + i] : zero;
  const double2 targ = i < d ? R.task_targ[tix + i] : zero;
  S.phi[i] = phi;
  __syncwarp();
  const double2* PL = Pc + (size_t)len * dd;
  const double2 psiL = matvec_row<DM>(PL, d, i, S.phi);

  if (mode & (PC_GRAD | PC_ERR | PC_RAWGRAD)) {
    // chi_0 = P_len^dag seed (objective.cpp:31-34 seed)
    S.vec[i] = A.form == 0 ? targ : csub(targ, psiL);
    __syncwarp();
    S.chi0[i] = matvec_adj_row<DM>(PL, d, i, S.vec);
    __syncwarp();
  }
  if (ch == 0) {
    if (mode & PC_ENTRY) {  // payoff of the task (objective.cpp:22-29)
      double t = 0.0;
      if (i < d) t = A.form == 0 ? cconjmul(targ, psiL).x : cabs2(csub(psiL, targ));
      const double s = group_sum<NLT>(t);
      if (i == 0 && live) R.entry_pay[(size_t)b * P.L + n] = A.form == 0 ? (w * s) : (-0.5 * (w * s));
    }
    if ((mode & PC_FINAL) && i < d && live) R.psi_end[tix + i] = psiL;
    if (mode & PC_LAG) {  // ism.cpp:424-459 through the cached product
      S.vec[i] = i < d ? R.psi_nodes[((size_t)b * (P.L + 1) + n) * d + i] : zero;
      __syncwarp();
      const double2 pe = matvec_row<DM>(PL, d, i, S.vec);
      __syncwarp();
      S.vec[i] = i < d ? R.chi_nodes[((size_t)b * (P.L + 1) + n + 1) * d + i] : zero;
      __syncwarp();
      const double2 cs = matvec_adj_row<DM>(PL, d, i, S.vec);
      if (i < d && live) {
        R.psi_end[tix + i] = pe;
        R.chi_start[tix + i] = cs;
      }
      __syncwarp();
    }
  }
  // penalty of the task window at the current control (before any update of this chunk)
  double pen = 0.0;
  for (int j = j0 + i; j < j1; j += NLT) {
    double sq = 0.0;
    for (int c = 0; c < C; ++c) sq += u[(size_t)j * C + c] * u[(size_t)j * C + c];
    pen += (P.alpha[node0 + j] * scale) * sq;
  }
  pen = group_sum<NLT>(pen);

  double err = 0.0;
  if (mode & (PC_GRAD | PC_ERR | PC_RAWGRAD)) {
    double2 psa, cha;
    matvec_row2<DM>(Pc + (size_t)j0 * dd, d, i, S.phi, S.chi0, psa, cha);
    // compile-time dimension: software pipeline, the row of P_{j+2} is in flight while step j
    // computes with P_{j+1} (the registers it costs only pay off when d is fixed)
    constexpr int DP = DIM > 0 ? DM : 1;
    double2 rcur[DP], rnext[DP];
    if constexpr (DIM > 0) load_row<DP>(Pc + (size_t)(j0 + 1) * dd, d, i, rcur);
    for (int jj = j0; jj < jmax; ++jj) {
      const bool act = jj < j1;
      const int j = act ? jj : j1 - 1;
      double2 psb, chb;
      if constexpr (DIM > 0) {
        if (j + 2 <= j1) load_row<DP>(Pc + (size_t)(j + 2) * dd, d, i, rnext);
        rows_dot2<DP>(rcur, d, i, S.phi, S.chi0, psb, chb);
#pragma unroll
        for (int k = 0; k < DP; ++k) rcur[k] = rnext[k];
      } else {
        matvec_row2<DM>(Pc + (size_t)(j + 1) * dd, d, i, S.phi, S.chi0, psb, chb);
      }
      const double2 ps = cadd(psa, psb), cs = cadd(cha, chb);
      const double* uj = u + (size_t)j * C;
      const double aj = P.alpha[node0 + j] * scale;
      double g[MAXC];
      double sq = 0.0;
#pragma unroll 1
      for (int c = 0; c < C; ++c) {
        const double uc = uj[c];
        double2 h;
        if (TRI) {
          h = tri_dH_row(P, b, c, uc, i, ps);
        } else {
          S.vec[i] = ps;
          __syncwarp();
          h = i < d ? dense_dH_row<DM>(P, b, c, uc, i, S.vec) : zero;
          __syncwarp();
        }
        const double im = group_sum<NLT>(i < d ? cconjmul(cs, h).y : 0.0);
        g[c] = -aj * dt * uc + 0.25 * dt * (w * im);  // gradient_sweep, objective.cpp:55-57
        sq += g[c] * g[c];
      }
      if (i == 0 && act && live) {
        for (int c = 0; c < C; ++c) {
          if (mode & PC_RAWGRAD) R.grad[((size_t)b * P.K + node0 + j) * C + c] = g[c];
          if (mode & PC_GRAD) u[(size_t)j * C + c] = uj[c] + A.rho * (weight * g[c]);
        }
      }
      if (act) err += sqrt(sq);
      psa = psb;
      cha = chb;
    }
  }
  if (i == 0 && live) {
    R.chunk_pen[cix] = pen;
    R.chunk_err[cix] = err;
  }
}

// entry value = weight * (payoff - penalty), residual = sum of chunk partials (index order)
__global__ void pc_finalize_kernel(DevProblem P, DevRun R, TaskArgs A, int nchunk, int ignore_done) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= P.B * P.L) return;
  const int b = t / P.L, n = t % P.L;
  if (ignore_done ? R.status[b] : (R.done[b] | R.status[b])) return;
  const int len = P.node[n + 1] - P.node[n];
  const double weight = A.weighted ? (double)P.K / (double)len : 1.0;
  double pen = 0.0, err = 0.0;
  for (int c = 0; c < nchunk; ++c) {
    pen += R.chunk_pen[(size_t)t * nchunk + c];
    err += R.chunk_err[(size_t)t * nchunk + c];
  }
  if (A.mode & PC_ENTRY) R.entry[t] = weight * (R.entry_pay[t] - 0.5 * P.dt * pen);
  if (A.mode & PC_ERR) R.err[t] = err;
}

// ---- dense assembly sweep: lane group of D lanes per task (row per lane) ------------------
template <int D>
__global__ void __launch_bounds__(128) dense_pc_assemble_kernel(DevProblem P, DevRun R, int tasks_per_cta,
                                                                int ignore_done) {
  using Cfg = DenseCfg<D, 1>;
  constexpr int NL = Cfg::NL, COLS = Cfg::COLS, TPW = Cfg::TPW;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double2* ops = reinterpret_cast<double2*>(smem_raw);
  const int b = blockIdx.y;
  if (ignore_done ? R.status[b] : (R.done[b] | R.status[b])) return;
  // after the Neumann kernel (dense_nm.cu) only the tasks it handed off run here
  auto handed_off = [&](int n) { return !R.nm_fallback || R.nm_fallback[(size_t)b * P.L + n] != 0; };
  if (R.nm_fallback) {
    if (*R.nm_count == 0) return;  // nothing was handed off (the common case)
    const int t0 = blockIdx.x * tasks_per_cta;
    const int mine = (int)threadIdx.x < tasks_per_cta && t0 + (int)threadIdx.x < P.L && handed_off(t0 + threadIdx.x);
    if (!__syncthreads_or(mine)) return;
  }
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
  __syncthreads();
  const int warp = threadIdx.x >> 5, l32 = threadIdx.x & 31;
  const int gid = warp * TPW + l32 / NL, lane = l32 % NL;
  const int n_raw = blockIdx.x * tasks_per_cta + gid;
  const bool live_task = n_raw < P.L && handed_off(n_raw);
  if (!__any_sync(0xffffffffu, live_task)) return;
  const int n = live_task ? n_raw : P.L - 1;
  const size_t gbytes = sizeof(double2) * (Cfg::PIV + Cfg::VEC + 2 * Cfg::MAT) + sizeof(int) * 2 * D;
  unsigned char* sp = smem_raw + sizeof(double2) * (size_t)nops * D * D + gbytes * gid;
  DenseScratch<D, 1> S;
  S.piv = reinterpret_cast<double2*>(sp);
  S.vec = S.piv + Cfg::PIV;
  S.matW = S.vec + Cfg::VEC;
  S.matP = S.matW + Cfg::MAT;
  S.perm = reinterpret_cast<int*>(S.matP + Cfg::MAT);
  DenseLane<D, 1> Ln;
  Ln.row = lane;
  Ln.g = 0;
  const int row = lane, C = P.C;
  const int node0 = P.node[n], len = P.node[n + 1] - node0;
  int lenmax = len;
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) lenmax = max(lenmax, __shfl_xor_sync(0xffffffffu, lenmax, off));
  const double half = 0.5 * P.dt;
  const double* u = R.u + ((size_t)b * P.K + node0) * C;
  const size_t dd = (size_t)d * d;
  double2* Pc = R.pc + ((size_t)b * P.L + n) * (size_t)R.traj_len * dd;
  double2 W[COLS], Pm[COLS];
#pragma unroll
  for (int t = 0; t < COLS; ++t) Pm[t] = cx(row == t ? 1.0 : 0.0, 0.0);
  // the Neumann path's cache is column-major (dense_nm.cu): its hand-offs store transposed
  const bool colmajor = R.nm_fallback != nullptr;
  auto at = [&](int i, int c) { return colmajor ? (size_t)c * d + i : (size_t)i * d + c; };
  if (live_task && row < d)
#pragma unroll
    for (int t = 0; t < COLS; ++t)
      if (t < d) Pc[at(row, t)] = Pm[t];
  const double* nrm = P.norm1 + (size_t)b * (1 + 2 * C);
  for (int j = 0; j < lenmax; ++j) {
    const bool live = j < len;
    const double* uj = u + (size_t)min(j, len - 1) * C;
    Ln.build(W, ops, C, P.has_quad, uj, half, false);
    double bound = nrm[0];
    for (int c = 0; c < C; ++c) {
      bound += fabs(uj[c]) * nrm[1 + c];
      if (P.has_quad) bound += 0.5 * uj[c] * uj[c] * nrm[1 + C + c];
    }
    if (__any_sync(0xffffffffu, !(half * bound < 1.0)))
      Ln.invert_pivot(W, S, lane);
    else
      Ln.invert_fast(W, S.piv);
    Ln.cayley_matmul(W, Pm, S, live);  // P_{j+1} = 2 B_j^-1 P_j - P_j (kept when past len)
    if (live) {
      if (live_task && row < d) {
        double2* dst = Pc + (size_t)(j + 1) * dd;
#pragma unroll
        for (int t = 0; t < COLS; ++t)
          if (t < d) dst[at(row, t)] = Pm[t];
      }
    }
  }
  if (live_task && row < d && R.prop) {
    double2* M = R.prop + ((size_t)b * P.L + n) * dd + (size_t)row * d;
#pragma unroll
    for (int t = 0; t < COLS; ++t)
      if (t < d) M[t] = Pm[t];
  }
}

}  // namespace

// ---- dense split assembly (few tasks): (1) every one-step Cayley matrix C_j = 2 B_j^-1 - I,
// j < K, in parallel (one lane group per step); (2) per task the sequential product
// P_{j+1} = C_j P_j, a pure matmul chain with the next C_j row prefetched into registers.
template <int D>
__global__ void __launch_bounds__(128) dense_cayley_kernel(DevProblem P, DevRun R, int steps_per_cta,
                                                           int ignore_done) {
  using Cfg = DenseCfg<D, 1>;
  constexpr int NL = Cfg::NL, COLS = Cfg::COLS, TPW = Cfg::TPW;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double2* ops = reinterpret_cast<double2*>(smem_raw);
  const int b = blockIdx.y;
  if (ignore_done ? R.status[b] : (R.done[b] | R.status[b])) return;
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
  __syncthreads();
  const int warp = threadIdx.x >> 5, l32 = threadIdx.x & 31;
  const int gid = warp * TPW + l32 / NL, lane = l32 % NL;
  const int j_raw = blockIdx.x * steps_per_cta + gid;
  if (!__any_sync(0xffffffffu, j_raw < P.K)) return;
  const int j = j_raw < P.K ? j_raw : P.K - 1;
  const size_t gbytes = sizeof(double2) * (Cfg::PIV + Cfg::VEC + 2 * Cfg::MAT) + sizeof(int) * 2 * D;
  unsigned char* sp = smem_raw + sizeof(double2) * (size_t)nops * D * D + gbytes * gid;
  DenseScratch<D, 1> S;
  S.piv = reinterpret_cast<double2*>(sp);
  S.vec = S.piv + Cfg::PIV;
  S.matW = S.vec + Cfg::VEC;
  S.matP = S.matW + Cfg::MAT;
  S.perm = reinterpret_cast<int*>(S.matP + Cfg::MAT);
  DenseLane<D, 1> Ln;
  Ln.row = lane;
  Ln.g = 0;
  const int C = P.C;
  const double half = 0.5 * P.dt;
  const double* uj = R.u + ((size_t)b * P.K + j) * C;
  double2 W[COLS];
  Ln.build(W, ops, C, P.has_quad, uj, half, false);
  const double* nrm = P.norm1 + (size_t)b * (1 + 2 * C);
  double bound = nrm[0];
  for (int c = 0; c < C; ++c) {
    bound += fabs(uj[c]) * nrm[1 + c];
    if (P.has_quad) bound += 0.5 * uj[c] * uj[c] * nrm[1 + C + c];
  }
  if (__any_sync(0xffffffffu, !(half * bound < 1.0)))
    Ln.invert_pivot(W, S, lane);
  else
    Ln.invert_fast(W, S.piv);
  if (j_raw < P.K && lane < d) {
    double2* dst = R.cay + ((size_t)b * P.K + j) * (size_t)d * d + (size_t)lane * d;
#pragma unroll
    for (int t = 0; t < COLS; ++t)
      if (t < d) dst[t] = cx(2.0 * W[t].x - (t == lane ? 1.0 : 0.0), 2.0 * W[t].y);
  }
}

template <int D>
__global__ void __launch_bounds__(128) dense_pc_chain_kernel(DevProblem P, DevRun R, int tasks_per_cta,
                                                             int ignore_done) {
  constexpr int NL = D, TPW = 32 / D;
  __shared__ __align__(16) double2 matP_all[(128 / 32) * TPW][D * D];
  const int b = blockIdx.y;
  if (ignore_done ? R.status[b] : (R.done[b] | R.status[b])) return;
  const int warp = threadIdx.x >> 5, l32 = threadIdx.x & 31;
  const int gid = warp * TPW + l32 / NL, row = l32 % NL;
  const int n_raw = blockIdx.x * tasks_per_cta + gid;
  const bool live_task = n_raw < P.L;
  if (!__any_sync(0xffffffffu, live_task)) return;
  const int n = live_task ? n_raw : P.L - 1;
  const int d = P.d;
  double2* matP = matP_all[gid];
  const int node0 = P.node[n], len = P.node[n + 1] - node0;
  int lenmax = len;
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) lenmax = max(lenmax, __shfl_xor_sync(0xffffffffu, lenmax, off));
  const size_t dd = (size_t)d * d;
  double2* Pc = R.pc + ((size_t)b * P.L + n) * (size_t)R.traj_len * dd;
  const double2* Cb = R.cay + ((size_t)b * P.K + node0) * dd;
  const bool wr = live_task && row < d;
  double2 Pm[D], cr[D], cn[D];
#pragma unroll
  for (int t = 0; t < D; ++t) Pm[t] = cx(row == t ? 1.0 : 0.0, 0.0);
  if (wr)
#pragma unroll
    for (int t = 0; t < D; ++t)
      if (t < d) Pc[(size_t)row * d + t] = Pm[t];
  auto load_row = [&](int j, double2 (&r)[D]) {
    const double2* src = Cb + (size_t)min(j, len - 1) * dd + (size_t)(row < d ? row : 0) * d;
#pragma unroll
    for (int t = 0; t < D; ++t) r[t] = t < d ? src[t] : cx(0.0, 0.0);
  };
  load_row(0, cr);
  for (int j = 0; j < lenmax; ++j) {
    if (j + 1 < lenmax) load_row(j + 1, cn);
    const bool live = j < len;
#pragma unroll
    for (int t = 0; t < D; ++t) matP[row * D + t] = Pm[t];
    __syncwarp();
    double2 acc[D];
#pragma unroll
    for (int t = 0; t < D; ++t) acc[t] = cx(0.0, 0.0);
#pragma unroll
    for (int k = 0; k < D; ++k) {
#pragma unroll
      for (int t = 0; t < D; ++t) acc[t] = cfma(cr[k], matP[k * D + t], acc[t]);
    }
    __syncwarp();
    if (live) {
#pragma unroll
      for (int t = 0; t < D; ++t) Pm[t] = acc[t];
      if (wr) {
        double2* dst = Pc + (size_t)(j + 1) * dd + (size_t)row * d;
#pragma unroll
        for (int t = 0; t < D; ++t)
          if (t < d) dst[t] = Pm[t];
      }
    }
#pragma unroll
    for (int t = 0; t < D; ++t) cr[t] = cn[t];
  }
  if (wr && R.prop) {
    double2* M = R.prop + ((size_t)b * P.L + n) * dd + (size_t)row * d;
#pragma unroll
    for (int t = 0; t < D; ++t)
      if (t < d) M[t] = Pm[t];
  }
}

template <int D>
static cudaError_t launch_dense_split(const DevProblem& P, const DevRun& R, int ignore_done, cudaStream_t st) {
  using Cfg = DenseCfg<D, 1>;
  constexpr int TPW = Cfg::TPW;
  const int nops = 1 + P.C + (P.has_quad ? P.C : 0);
  const size_t gbytes = sizeof(double2) * (Cfg::PIV + Cfg::VEC + 2 * Cfg::MAT) + sizeof(int) * 2 * D;
  const int spc = 4 * TPW;  // steps per CTA (4 warps)
  const size_t smem = sizeof(double2) * (size_t)nops * D * D + gbytes * spc;
  auto kc = dense_cayley_kernel<D>;
  cudaError_t e = cudaFuncSetAttribute(kc, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  kc<<<dim3((P.K + spc - 1) / spc, P.B), 128, smem, st>>>(P, R, spc, ignore_done);
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  const int tpc = 4 * TPW;
  dense_pc_chain_kernel<D><<<dim3((P.L + tpc - 1) / tpc, P.B), 128, 0, st>>>(P, R, tpc, ignore_done);
  return cudaGetLastError();
}

// ---- tridiagonal assembly sweep (defined in tridiag_kernels.cu) ---------------------------
cudaError_t tri_pc_assemble(const DevProblem& P, const DevRun& R, int ignore_done, cudaStream_t st);

int pc_chunk(const DevProblem& P, const DevRun& R) {
  // steps per warp: whole short tasks; otherwise enough chunks for ~16 warps per SM
  const int maxlen = R.traj_len - 1;
  if (maxlen <= 32) return maxlen;
  const long long want = 148LL * 16;
  const long long tasks = (long long)P.L * P.B;
  int chunk = (int)((tasks * maxlen + want - 1) / want);
  return chunk < 4 ? 4 : (chunk > 16 ? 16 : chunk);
}

cudaError_t pc_eval(const DevProblem& P, const DevRun& R, const TaskArgs& A, int ignore_done, cudaStream_t st) {
  const int chunk = pc_chunk(P, R);
  const int nchunk = (R.traj_len - 1 + chunk - 1) / chunk;
  if (dense_pc_eval16_applicable(P, R, A.mode, nchunk)) {  // dense d = 16, one control (dense_nm.cu)
    cudaError_t e = dense_pc_eval16(P, R, A, ignore_done, st);
    if (e != cudaSuccess) return e;
    pc_finalize_kernel<<<(P.B * P.L + 127) / 128, 128, 0, st>>>(P, R, A, nchunk, ignore_done);
    return cudaGetLastError();
  }
  if (R.nm) return cudaErrorNotSupported;  // the Neumann path's column-major cache has no other reader
  dim3 grid((P.L * nchunk + 3) / 4, P.B);
  const bool small = P.d <= 16;  // narrower register arrays -> higher occupancy
  if (P.kind == QOC_KIND_TRIDIAG) {
    if (P.d == 21) pc_eval_kernel<true, 24, 21><<<grid, 128, 0, st>>>(P, R, A, chunk, nchunk, ignore_done);
    else if (small) pc_eval_kernel<true, 16><<<grid, 128, 0, st>>>(P, R, A, chunk, nchunk, ignore_done);
    else pc_eval_kernel<true, 32><<<grid, 128, 0, st>>>(P, R, A, chunk, nchunk, ignore_done);
  } else {
    if (small && nchunk == 1) {  // two tasks per warp
      const dim3 g2((P.L * nchunk + 7) / 8, P.B);
      pc_eval_kernel<false, 16, 0, 16><<<g2, 128, 0, st>>>(P, R, A, chunk, nchunk, ignore_done);
    } else if (small) {
      pc_eval_kernel<false, 16><<<grid, 128, 0, st>>>(P, R, A, chunk, nchunk, ignore_done);
    } else {
      pc_eval_kernel<false, 32><<<grid, 128, 0, st>>>(P, R, A, chunk, nchunk, ignore_done);
    }
  }
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  pc_finalize_kernel<<<(P.B * P.L + 127) / 128, 128, 0, st>>>(P, R, A, nchunk, ignore_done);
  return cudaGetLastError();
}

cudaError_t pc_eval_dual(const DevProblem& P, const DevRun& R, int form, int weighted, double rho, int dual,
                         cudaStream_t st) {
  if (!dense_pc_eval16_applicable(P, R, PCM_ENTRY | PCM_GRAD | PCM_ERR, 1)) return cudaErrorNotSupported;
  const TaskArgs A{dual == 1 ? (PCM_ENTRY | PCM_ERR) : PCM_ENTRY, form, weighted, 1, rho};
  cudaError_t e = dense_pc_eval16(P, R, A, 0, st, 0, dual);
  if (e != cudaSuccess) return e;
  pc_finalize_kernel<<<(P.B * P.L + 127) / 128, 128, 0, st>>>(P, R, A, 1, 0);
  return cudaGetLastError();
}

template <int D>
static cudaError_t launch_dense_pc(const DevProblem& P, const DevRun& R, int ignore_done, cudaStream_t st) {
  using Cfg = DenseCfg<D, 1>;
  constexpr int TPW = Cfg::TPW;
  int warps = (P.L + TPW - 1) / TPW;
  if (warps > 4) warps = 4;
  const int tpc = warps * TPW;
  const int nops = 1 + P.C + (P.has_quad ? P.C : 0);
  const size_t gbytes = sizeof(double2) * (Cfg::PIV + Cfg::VEC + 2 * Cfg::MAT) + sizeof(int) * 2 * D;
  const size_t smem = sizeof(double2) * (size_t)nops * D * D + gbytes * tpc;
  auto kern = dense_pc_assemble_kernel<D>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  kern<<<dim3((P.L + tpc - 1) / tpc, P.B), warps * 32, smem, st>>>(P, R, tpc, ignore_done);
  return cudaGetLastError();
}

bool dense_nm_fuse_residual();
bool pc_fuses_residual(const DevProblem& P, const DevRun& R) {
  return R.nm != nullptr && R.nm_v != nullptr && dense_nm_fuse_residual();
}

cudaError_t pc_assemble(const DevProblem& P, const DevRun& R, int ignore_done, cudaStream_t st, int residual_form) {
  if (P.kind == QOC_KIND_TRIDIAG) return tri_pc_assemble(P, R, ignore_done, st);
  if (R.nm) {  // Neumann + tensor-core sweep; out-of-range tasks continue in Gauss-Jordan below
    const int fused = residual_form >= 0 && pc_fuses_residual(P, R);
    if (fused && residual_form != QOC_FORM_TRACKING) return cudaErrorNotSupported;  // interpolated runs only
    cudaError_t e = cudaMemsetAsync(R.nm_count, 0, sizeof(int), st);
    if (e != cudaSuccess) return e;
    e = dense_nm_assemble(P, R, ignore_done, fused, st);
    if (e != cudaSuccess) return e;
    if ((e = launch_dense_pc<16>(P, R, ignore_done, st)) != cudaSuccess) return e;
    if (fused) {  // residual of the handed-off tasks through the cache
      const TaskArgs E{PCM_ERR, residual_form, 1, 1, 0.0};
      return dense_pc_eval16(P, R, E, ignore_done, st, 1);
    }
    return cudaSuccess;
  }
  if (R.cay) {
    switch (dense_pad(P.d)) {
      case 2: return launch_dense_split<2>(P, R, ignore_done, st);
      case 4: return launch_dense_split<4>(P, R, ignore_done, st);
      case 8: return launch_dense_split<8>(P, R, ignore_done, st);
      case 16: return launch_dense_split<16>(P, R, ignore_done, st);
      default: break;
    }
  }
  switch (dense_pad(P.d)) {
    case 2: return launch_dense_pc<2>(P, R, ignore_done, st);
    case 4: return launch_dense_pc<4>(P, R, ignore_done, st);
    case 8: return launch_dense_pc<8>(P, R, ignore_done, st);
    case 16: return launch_dense_pc<16>(P, R, ignore_done, st);
    case 32: return launch_dense_pc<32>(P, R, ignore_done, st);
  }
  return cudaErrorInvalidValue;
}

int pc_nchunk(const DevProblem& P, const DevRun& R) {
  const int chunk = pc_chunk(P, R);
  return (R.traj_len - 1 + chunk - 1) / chunk;
}

}  // namespace qoc
