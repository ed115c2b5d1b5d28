// bitflip_kernels.cu — ISM task/horizon kernels for spin registers in bit-flip form
// (QOC_KIND_BITFLIP, d = 2^n, 5 <= n <= 12; BASELINE config 3, the n = 10 Ising chain).
//
// H(u) = diag(h0) + V(u),  V(u) = sum_i (ax_i sigma^x_i + ay_i sigma^y_i),
// ax_i = sum_{c: axis x} u_c coef[c][i],  ay_i = sum_{c: axis y} u_c coef[c][i].
// The matrix is never formed: V y is n bit-flip gathers per element.  The Cayley step of the
// reference (propagation.cpp:85-106, (I + sH) y = (I - sH) x, s = +-i dt/2) is solved by the
// Jacobi-preconditioned fixed point the oracle restates (oracle.cpp BitM::cayley)
//     y <- (1 + sD)^-1 (r - s V y),    r = x - s H x,
// i.e. the Neumann series of (I + sH)^-1 around its diagonal.  |1 + sD_i| >= 1, so the
// iteration contracts by q = dt/2 * sum_i sqrt(ax_i^2 + ay_i^2) per sweep; the sweep count
// is fixed per step from that a-priori bound (q^(k+1) <= 2^-54, as y = 2z - x doubles the error of z) instead of a data-dependent
// stopping test, so every thread agrees without a reduction.
//
// Layout: one CTA of T = min(d, 512) threads per (problem, subinterval) task (the d = 1024
// node sweeps use T = 128, E = 8, see bitflip_horizon); thread t
// holds the E = d/T amplitudes s = t + e*T (all compile-time: one instantiation per n).  A flip of bit b pairs
//   b < log2 T         -> thread t ^ 2^b      (shared memory, double buffer; one LDS.128 per
//                                               partner -- cheaper than 4 SHFL for a double2)
//   b >= log2 T        -> register slot e ^ 2^(b - log2 T)     (same thread)
// so one fixed-point sweep costs one __syncthreads.  d = 1024 runs two amplitudes per
// thread on 16 warps (98 registers, no spills); the per-spin coefficients of a step live in
// registers across all its sweeps, so a sweep is n LDS.128 + n complex FMAs per amplitude.  Spin i <-> bit n-1-i (spin_operator,
// models.cpp:296-318).  The forward trajectory of a task (len+1 states, 16 KB each at
// d = 1024) lives in HBM/L2 (R.traj); the adjoint sweep reads it back for the gradient.
#include <cstdlib>

#include "kernels.h"

namespace qoc {

namespace {

constexpr int BF_MAXN = 12;
constexpr int BF_T = 512;

// <s| (a sigma^x + b sigma^y) |s ^ m> = a + (bit(s) ? +i : -i) b   (oracle.cpp BitM::offdiag)
__device__ __forceinline__ double2 flip_coef(double2 ab, int one) { return cx(ab.x, one ? ab.y : -ab.y); }

struct BfOps {
  const double* diag;  // [d]
  const double* coef;  // [C][n]
  const int* axis;     // [C]
  int C, n;
};

// Everything about the register layout is compile-time: N = log2 d spins, T = 2^LOG2T threads,
// E = 2^LOG2E amplitudes per thread, so every flip loop unrolls, partner addresses are
// constant offsets and the per-spin coefficients sit in registers for the whole step.
template <int LOG2E, int LOG2T>
struct Bf {
  static constexpr int E = 1 << LOG2E, T = 1 << LOG2T, N = LOG2E + LOG2T, D = E * T;
  int t, lane, warp;
  double dg[E];       // diagonal of H at this thread's amplitudes
  double2 cl[LOG2T];  // low spins (bit b < LOG2T): coefficient signed for this thread's bit
  double2 ch[LOG2E > 0 ? LOG2E : 1];  // high spins: raw (ax, ay); the sign is a compile-time function of e
  double2* buf;       // smem [2][D] exchange
  double2* sa;        // smem [2][N] per-step channel sums (by step parity)
  int* ssw;           // smem [2] per-step sweep count
  double* red;        // smem [T / 32][4] reduction scratch
  int par = 0, spar = 0;

  __device__ void publish(const double2 (&v)[E]) {
    par ^= 1;
    double2* b = buf + par * D;
#pragma unroll
    for (int e = 0; e < E; ++e) b[t + e * T] = v[e];
  }
  __device__ const double2* cur() const { return buf + par * D; }

  // V v (after publish(v) + __syncthreads)
  __device__ void apply_V(const double2 (&v)[E], double2 (&out)[E]) const {
    const double2* c = cur();
#pragma unroll
    for (int e = 0; e < E; ++e) out[e] = cx(0.0, 0.0);
#pragma unroll
    for (int hb = 0; hb < LOG2E; ++hb)
#pragma unroll
      for (int e = 0; e < E; ++e) out[e] = cfma(flip_coef(ch[hb], (e >> hb) & 1), v[e ^ (1 << hb)], out[e]);
#pragma unroll
    for (int b = 0; b < LOG2T; ++b)
#pragma unroll
      for (int e = 0; e < E; ++e) out[e] = cfma(cl[b], c[(t ^ (1 << b)) + e * T], out[e]);
  }

  // Step setup: warp 0 forms the channel sums of u_j and the sweep count (q^(k+1) <= 2^-54,
  // q = dt/2 sum_i |(ax_i, ay_i)|; -1 if the series would not contract); after the barrier
  // every thread pulls its signed coefficients into registers.  Returns the sweep count.
  __device__ int begin_step(const BfOps& O, const double* uj, double half) {
    spar ^= 1;
    double2* sa_w = sa + spar * N;
    if (warp == 0) {
      double nrm = 0.0;
      if (lane < N) {
        double ax = 0.0, ay = 0.0;
        for (int c = 0; c < O.C; ++c) {
          const double g = uj[c] * O.coef[c * N + lane];
          if (O.axis[c] == 0) ax += g;
          else ay += g;
        }
        sa_w[lane] = cx(ax, ay);
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
    for (int b = 0; b < LOG2T; ++b) cl[b] = flip_coef(sa_w[N - 1 - b], (t >> b) & 1);
#pragma unroll
    for (int hb = 0; hb < LOG2E; ++hb) ch[hb] = sa_w[N - 1 - (LOG2T + hb)];
    return ssw[spar];
  }

  // x <- (I + sH)^-1 (I - sH) x = 2 z - x with (I + sH) z = x, s = (0, sh): the Jacobi
  // sweeps z <- (1 + sD)^-1 (x - s V z) start from z = (1 + sD)^-1 x, so no V x product is
  // needed for the right-hand side.
  __device__ void cayley(double2 (&x)[E], double sh, int sweeps) {
    double2 z[E], vv[E], inv[E];
#pragma unroll
    for (int e = 0; e < E; ++e) {
      const double a = sh * dg[e];
      const double den = 1.0 / fma(a, a, 1.0);
      inv[e] = cx(den, -a * den);  // (1 + s D)^-1
      z[e] = cmul(x[e], inv[e]);
    }
    for (int k = 0; k < sweeps; ++k) {
      publish(z);
      __syncthreads();
      apply_V(z, vv);
#pragma unroll
      for (int e = 0; e < E; ++e) {
        const double2 tt = cx(x[e].x + sh * vv[e].y, x[e].y - sh * vv[e].x);  // x - s V z
        z[e] = cmul(tt, inv[e]);
      }
    }
#pragma unroll
    for (int e = 0; e < E; ++e) x[e] = cx(fma(2.0, z[e].x, -x[e].x), fma(2.0, z[e].y, -x[e].y));
  }

  // Deterministic block sum of up to 4 values (fixed warp order).
  __device__ void block_sum(double (&v)[4], int nv) {
    for (int q = 0; q < nv; ++q) {
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) v[q] += __shfl_xor_sync(0xffffffffu, v[q], off);
    }
    __syncthreads();
    if (lane == 0)
      for (int q = 0; q < nv; ++q) red[warp * 4 + q] = v[q];
    __syncthreads();
    for (int q = 0; q < nv; ++q) {
      double s = 0.0;
      for (int w = 0; w < T / 32; ++w) s += red[w * 4 + q];
      v[q] = s;
    }
  }

  // Im <cs, A_c ps> for every channel (A_c = sum_i coef[c][i] sigma^{axis_c}_i), block-summed.
  // ps must be published (and synced) by the caller.
  __device__ void grad_terms(const BfOps& O, const double2 (&cs)[E], const double2 (&ps)[E], double (&out)[4]) {
    double2 acc[4] = {cx(0.0, 0.0), cx(0.0, 0.0), cx(0.0, 0.0), cx(0.0, 0.0)};
    const double2* c = cur();
    auto add = [&](int e, int spin, int one, double2 pv) {
      for (int ch_ = 0; ch_ < O.C && ch_ < 4; ++ch_) {
        const double g = O.coef[ch_ * N + spin];
        const double2 a = O.axis[ch_] == 0 ? cx(g, 0.0) : flip_coef(cx(0.0, g), one);
        acc[ch_] = cfmaconj(cs[e], cmul(a, pv), acc[ch_]);
      }
    };
#pragma unroll
    for (int hb = 0; hb < LOG2E; ++hb)
#pragma unroll
      for (int e = 0; e < E; ++e) add(e, N - 1 - (LOG2T + hb), (e >> hb) & 1, ps[e ^ (1 << hb)]);
#pragma unroll
    for (int b = 0; b < LOG2T; ++b)
#pragma unroll
      for (int e = 0; e < E; ++e) add(e, N - 1 - b, (t >> b) & 1, c[(t ^ (1 << b)) + e * T]);
    for (int q = 0; q < 4; ++q) out[q] = acc[q].y;
    block_sum(out, O.C < 4 ? O.C : 4);
  }
};

template <int LOG2E, int LOG2T>
__device__ __forceinline__ Bf<LOG2E, LOG2T> make_bf(const DevProblem& P, int b, unsigned char* smem) {
  using F_ = Bf<LOG2E, LOG2T>;
  F_ F;
  F.t = threadIdx.x;
  F.lane = threadIdx.x & 31;
  F.warp = threadIdx.x >> 5;
  F.buf = reinterpret_cast<double2*>(smem);
  F.sa = F.buf + 2 * F_::D;
  F.red = reinterpret_cast<double*>(F.sa + 2 * F_::N);
  F.ssw = reinterpret_cast<int*>(F.red + (F_::T / 32) * 4);
#pragma unroll
  for (int e = 0; e < F_::E; ++e) F.dg[e] = P.bf_diag[(size_t)b * P.d + F.t + e * F_::T];
  return F;
}

__host__ __device__ constexpr size_t bf_smem(int d) {
  return sizeof(double2) * (2 * (size_t)d + 2 * BF_MAXN) + sizeof(double) * (BF_T / 32) * 4 + 2 * sizeof(int);
}

template <int E>
__device__ __forceinline__ void load_state(double2 (&x)[E], const double2* src, int t, int T) {
#pragma unroll
  for (int e = 0; e < E; ++e) x[e] = src[t + e * T];
}
template <int E>
__device__ __forceinline__ void store_state(const double2 (&x)[E], double2* dst, int t, int T) {
#pragma unroll
  for (int e = 0; e < E; ++e) dst[t + e * T] = x[e];
}

template <int LOG2E, int LOG2T>
__global__ void __launch_bounds__(1 << LOG2T) bitflip_task_kernel(DevProblem P, DevRun R, TaskArgs A, int ignore_done) {
  using F_ = Bf<LOG2E, LOG2T>;
  constexpr int E = 1 << LOG2E, T = 1 << LOG2T;
  using Vec = double2[1 << LOG2E];
  const int n = A.n_lo + blockIdx.x, b = blockIdx.y;
  if (ignore_done ? R.status[b] : (R.done[b] | R.status[b])) return;
  extern __shared__ __align__(16) unsigned char smem[];
  F_ F = make_bf<LOG2E, LOG2T>(P, b, smem);
  const int d = P.d, C = P.C, t = F.t;
  const BfOps O{P.bf_diag + (size_t)b * d, P.bf_coef + (size_t)b * C * P.nspins, P.bf_axis, C, P.nspins};
  const int node0 = P.node[n], len = P.node[n + 1] - node0;
  const double Kd = (double)P.K;
  const double weight = A.weighted ? Kd / (double)len : 1.0;
  const double scale = (double)len / Kd;
  const double half = 0.5 * P.dt, dt = P.dt, w = P.ip_w;
  double* u = R.u + ((size_t)b * P.K + node0) * C;
  double2* traj = R.traj + ((size_t)b * P.L + n) * (size_t)R.traj_len * d;
  const size_t tix = ((size_t)b * P.L + n) * d;
  const int mode = A.mode;
  bool ok = true;
  double2 x[E], chi[E], cn[E], ps[E], tg[E];
  load_state<E>(tg, R.task_targ + tix, t, T);

  auto step = [&](Vec& v, const double* uj, double sh) {
    const int sweeps = F.begin_step(O, uj, half);
    ok &= sweeps >= 0;
    F.cayley(v, sh, sweeps < 0 ? 0 : sweeps);
  };
  // forward sweep from `init`, optionally recording the trajectory
  auto forward = [&](Vec& v, bool rec, double* pen) {
    if (rec) store_state<E>(v, traj, t, T);
    for (int j = 0; j < len; ++j) {
      const double* uj = u + (size_t)j * C;
      step(v, uj, half);
      if (rec) store_state<E>(v, traj + (size_t)(j + 1) * d, t, T);
      if (pen) {
        double sq = 0.0;
        for (int c = 0; c < C; ++c) sq += uj[c] * uj[c];
        *pen += (P.alpha[node0 + j] * scale) * sq;
      }
    }
  };
  // adjoint sweep with the gradient of objective.cpp:48-60 at every step; `act(j, g)`
  auto adjoint = [&](Vec& c0, auto&& act) {
    for (int j = len - 1; j >= 0; --j) {
      const double* uj = u + (size_t)j * C;
      double uold[4];
      for (int c = 0; c < C && c < 4; ++c) uold[c] = uj[c];
#pragma unroll
      for (int e = 0; e < E; ++e) cn[e] = c0[e];
      step(cn, uj, -half);
      double2 cs[E];
#pragma unroll
      for (int e = 0; e < E; ++e) {
        const double2 a = traj[(size_t)j * d + t + e * T], bb = traj[(size_t)(j + 1) * d + t + e * T];
        ps[e] = cadd(a, bb);
        cs[e] = cadd(cn[e], c0[e]);
      }
      F.publish(ps);
      __syncthreads();
      double im[4];
      F.grad_terms(O, cs, ps, im);
      const double aj = P.alpha[node0 + j] * scale;
      double g[4];
      for (int c = 0; c < C && c < 4; ++c) g[c] = -aj * dt * uold[c] + 0.25 * dt * (w * im[c]);
      act(j, uold, g);
#pragma unroll
      for (int e = 0; e < E; ++e) c0[e] = cn[e];
    }
  };

  // ---------------- phase 1: sweeps at the current control -------------------------
  if (mode & (M_ENTRY | M_UPDATE | M_FINAL | M_GRAD)) {
    const bool need_traj = (mode & (M_UPDATE | M_GRAD)) != 0;
    const int iters = (mode & M_UPDATE) ? A.inner : 1;
    for (int it = 0; it < iters; ++it) {
      load_state<E>(x, R.task_init + tix, t, T);
      double pen = 0.0;
      forward(x, need_traj, &pen);
      if (it == 0 && (mode & M_ENTRY)) {
        double s[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
        for (int e = 0; e < E; ++e) s[0] += A.form == 0 ? cconjmul(tg[e], x[e]).x : cabs2(csub(x[e], tg[e]));
        F.block_sum(s, 1);
        const double payoff = A.form == 0 ? (w * s[0]) : (-0.5 * (w * s[0]));
        if (t == 0) R.entry[(size_t)b * P.L + n] = weight * (payoff - 0.5 * dt * pen);
      }
      if (it == 0 && (mode & M_FINAL)) store_state<E>(x, R.psi_end + tix, t, T);
      if (mode & (M_UPDATE | M_GRAD)) {
#pragma unroll
        for (int e = 0; e < E; ++e) chi[e] = A.form == 0 ? tg[e] : csub(tg[e], x[e]);  // objective.cpp:31-34
        adjoint(chi, [&](int j, const double* uold, const double* g) {
          if (t == 0) {
            for (int c = 0; c < C && c < 4; ++c) {
              if (mode & M_GRAD) R.grad[((size_t)b * P.K + node0 + j) * C + c] = g[c];
              if (mode & M_UPDATE) u[(size_t)j * C + c] = uold[c] + A.rho * (weight * g[c]);
            }
          }
          __syncthreads();  // the updated u_j is read by every thread at the next sweep
        });
      }
    }
  }

  // ---------------- phase 2: sweeps at the updated control -------------------------
  if (mode & M_ERROR) {
    load_state<E>(x, R.task_init + tix, t, T);
    forward(x, true, nullptr);
#pragma unroll
    for (int e = 0; e < E; ++e) chi[e] = A.form == 0 ? tg[e] : csub(tg[e], x[e]);
    double err = 0.0;
    adjoint(chi, [&](int, const double*, const double* g) {
      double sq = 0.0;
      for (int c = 0; c < C && c < 4; ++c) sq += g[c] * g[c];
      err += sqrt(sq);
    });
    if (t == 0) R.err[(size_t)b * P.L + n] = err;
  }
  if (mode & M_LAGGED) {  // ism.cpp:424-459
    load_state<E>(x, R.psi_nodes + ((size_t)b * (P.L + 1) + n) * d, t, T);
    forward(x, false, nullptr);
    store_state<E>(x, R.psi_end + tix, t, T);
    load_state<E>(chi, R.chi_nodes + ((size_t)b * (P.L + 1) + n + 1) * d, t, T);
    for (int j = len - 1; j >= 0; --j) step(chi, u + (size_t)j * C, -half);
    store_state<E>(chi, R.chi_start + tix, t, T);
  }
  if (!ok && t == 0 && R.err_flags) atomicOr(R.err_flags, 2);
}

// node_sweeps (ism.cpp:35-84) / exact payoff (objective.cpp:93-100) over the full horizon.
// blockIdx.y = 0: forward nodes psi_n (which = 0) or the exact payoff (which = 1);
// blockIdx.y = 1: adjoint nodes chi_n seeded with the target (ism.cpp:72), which = 0 only.
// SR.nloc > 0: the interior nodes of blocks [SR.g0, SR.g0 + SR.nloc) of the blocked plan, each
// seeded from its chain-formed end nodes (blockIdx.x = b * nloc + local block).
template <int LOG2E, int LOG2T>
__global__ void __launch_bounds__(1 << LOG2T) bitflip_horizon_kernel(DevProblem P, DevRun R, int which, int k,
                                                                     SweepRange SR) {
  if (R.kdev) k = *R.kdev;
  using F_ = Bf<LOG2E, LOG2T>;
  constexpr int E = 1 << LOG2E, T = 1 << LOG2T;
  const int nl = SR.nloc > 0 ? SR.nloc : 1;
  const int b = blockIdx.x / nl, g = SR.g0 + (int)(blockIdx.x % nl), dir = blockIdx.y;
  if (R.done[b] || R.status[b]) return;
  if (which == 1 && dir == 1) return;
  extern __shared__ __align__(16) unsigned char smem[];
  F_ F = make_bf<LOG2E, LOG2T>(P, b, smem);
  const int d = P.d, C = P.C, t = F.t;
  const BfOps O{P.bf_diag + (size_t)b * d, P.bf_coef + (size_t)b * C * P.nspins, P.bf_axis, C, P.nspins};
  const double half = 0.5 * P.dt;
  const double* u = R.u + (size_t)b * P.K * C;
  const size_t nb = (size_t)b * (P.L + 1) * d;
  // node range [na, nz] of this sweep; the full horizon also writes its two end nodes
  const bool full = SR.nloc == 0;
  const int na = full ? 0 : SR.bnode[g], nz = full ? P.L : SR.bnode[g + 1];
  bool ok = true;
  double2 x[E];
  auto step = [&](const double* uj, double sh) {
    const int sweeps = F.begin_step(O, uj, half);
    ok &= sweeps >= 0;
    F.cayley(x, sh, sweeps < 0 ? 0 : sweeps);
  };
  if (dir == 0) {
    load_state<E>(x, full ? P.init + (size_t)b * d : R.psi_nodes + nb + (size_t)na * d, t, T);
    if (which == 0 && full) store_state<E>(x, R.psi_nodes + nb, t, T);
    int nxt = na + 1;
    const int last = full ? nz : nz - 1;  // highest node this sweep writes
    for (int j = P.node[na]; j < P.node[nz]; ++j) {
      step(u + (size_t)j * C, half);
      if (which == 0 && nxt <= last && P.node[nxt] == j + 1) {
        store_state<E>(x, R.psi_nodes + nb + (size_t)nxt * d, t, T);
        ++nxt;
      }
    }
    if (which == 1) {
      double s[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
      for (int e = 0; e < E; ++e) s[0] += cconjmul(P.targ[(size_t)b * d + t + e * T], x[e]).x;
      F.block_sum(s, 1);
      if (t == 0) {
        double pen = 0.0;
        for (int n = 0; n < P.L; ++n) pen += R.pen[(size_t)b * P.L + n];
        R.rec_exact[(size_t)b * R.cap + k] = P.ip_w * s[0] - 0.5 * P.dt * pen;
      }
    }
  } else {
    load_state<E>(x, full ? P.targ + (size_t)b * d : R.chi_nodes + nb + (size_t)nz * d, t, T);
    if (full) store_state<E>(x, R.chi_nodes + nb + (size_t)P.L * d, t, T);
    int prev = nz - 1;
    const int first = full ? na : na + 1;  // lowest node this sweep writes
    for (int j = P.node[nz] - 1; j >= P.node[na]; --j) {
      step(u + (size_t)j * C, -half);
      if (prev >= first && P.node[prev] == j) {
        store_state<E>(x, R.chi_nodes + nb + (size_t)prev * d, t, T);
        --prev;
      }
    }
  }
  if (!ok && t == 0 && R.err_flags) atomicOr(R.err_flags, 2);
}

// Block products of the blocked plan: P_g = A_{j1-1} ... A_{j0} over the steps of block g,
// column c = the basis state e_c carried through the block's Cayley steps (the propagator
// assembly of propagation.cpp:236-249 on the bit-flip operator: d independent column sweeps
// instead of one dense LU per step).  blockIdx.x = column, blockIdx.y = local block,
// blockIdx.z = problem (B = 1 on this path).  Writes column-major into the rank's slab.
template <int LOG2E, int LOG2T, int MINB>
__global__ void __launch_bounds__(1 << LOG2T, MINB) bitflip_block_kernel(DevProblem P, DevRun R, DevBlocks BK, int g0) {
  using F_ = Bf<LOG2E, LOG2T>;
  constexpr int E = 1 << LOG2E, T = 1 << LOG2T;
  const int col = blockIdx.x, g = g0 + blockIdx.y, b = blockIdx.z;
  if (R.done[b] || R.status[b]) return;
  extern __shared__ __align__(16) unsigned char smem[];
  F_ F = make_bf<LOG2E, LOG2T>(P, b, smem);
  const int d = P.d, C = P.C, t = F.t;
  const BfOps O{P.bf_diag + (size_t)b * d, P.bf_coef + (size_t)b * C * P.nspins, P.bf_axis, C, P.nspins};
  const double half = 0.5 * P.dt;
  const double* u = R.u + (size_t)b * P.K * C;
  bool ok = true;
  double2 x[E];
#pragma unroll
  for (int e = 0; e < E; ++e) x[e] = cx(t + e * T == col ? 1.0 : 0.0, 0.0);
  const int j0 = P.node[BK.bnode[g]], j1 = P.node[BK.bnode[g + 1]];
  for (int j = j0; j < j1; ++j) {
    const int sweeps = F.begin_step(O, u + (size_t)j * C, half);
    ok &= sweeps >= 0;
    F.cayley(x, half, sweeps < 0 ? 0 : sweeps);
  }
  store_state<E>(x, BK.block(g, d) + (size_t)col * d, t, T);
  if (!ok && t == 0 && R.err_flags) atomicOr(R.err_flags, 2);
}

template <int LOG2E, int LOG2T>
cudaError_t launch_task(const DevProblem& P, const DevRun& R, const TaskArgs& A, int ignore_done, cudaStream_t st) {
  const size_t smem = bf_smem(P.d);
  auto kern = bitflip_task_kernel<LOG2E, LOG2T>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  kern<<<dim3(A.n_cnt > 0 ? A.n_cnt : P.L, P.B), 1 << LOG2T, smem, st>>>(P, R, A, ignore_done);
  return cudaGetLastError();
}

template <int LOG2E, int LOG2T>
cudaError_t launch_horizon(const DevProblem& P, const DevRun& R, int which, int k, const SweepRange& SR,
                           cudaStream_t st) {
  const size_t smem = bf_smem(P.d);
  auto kern = bitflip_horizon_kernel<LOG2E, LOG2T>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  kern<<<dim3(P.B * (SR.nloc > 0 ? SR.nloc : 1), 2), 1 << LOG2T, smem, st>>>(P, R, which, k, SR);
  return cudaGetLastError();
}

template <int LOG2E, int LOG2T, int MINB = 1>
cudaError_t launch_blocks(const DevProblem& P, const DevRun& R, const DevBlocks& BK, int g0, int nloc,
                          cudaStream_t st) {
  const size_t smem = bf_smem(P.d);
  auto kern = bitflip_block_kernel<LOG2E, LOG2T, MINB>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  kern<<<dim3(P.d, nloc, P.B), 1 << LOG2T, smem, st>>>(P, R, BK, g0);
  return cudaGetLastError();
}

}  // namespace

// d = 2^n: T = min(d, 512) threads, E = d / T amplitudes per thread.
cudaError_t bitflip_task(const DevProblem& P, const DevRun& R, const TaskArgs& A, int ignore_done, cudaStream_t st) {
  if (A.mode & M_ASSEMBLE) return cudaErrorNotSupported;  // the driver runs the direct plan
  if (P.C > 4) return cudaErrorNotSupported;
  switch (P.nspins) {
    case 5: return launch_task<0, 5>(P, R, A, ignore_done, st);
    case 6: return launch_task<0, 6>(P, R, A, ignore_done, st);
    case 7: return launch_task<0, 7>(P, R, A, ignore_done, st);
    case 8: return launch_task<0, 8>(P, R, A, ignore_done, st);
    case 9: return launch_task<0, 9>(P, R, A, ignore_done, st);
    case 10: return launch_task<1, 9>(P, R, A, ignore_done, st);
    case 11: return launch_task<2, 9>(P, R, A, ignore_done, st);
    case 12: return launch_task<3, 9>(P, R, A, ignore_done, st);
  }
  return cudaErrorNotSupported;
}

cudaError_t bitflip_horizon_cluster(const DevProblem& P, const DevRun& R, int which, int k, const SweepRange& SR,
                                    cudaStream_t st, bool* used);

cudaError_t bitflip_horizon_range(const DevProblem& P, const DevRun& R, int which, int k, const SweepRange& SR,
                                  cudaStream_t st) {
  if (P.C > 4) return cudaErrorNotSupported;
  {  // d = 1024: the node sweeps split over a thread-block cluster (bitflip_cluster.cu)
    bool used = false;
    cudaError_t e = bitflip_horizon_cluster(P, R, which, k, SR, st, &used);
    if (e != cudaSuccess || used) return e;
  }
  switch (P.nspins) {
    case 5: return launch_horizon<0, 5>(P, R, which, k, SR, st);
    case 6: return launch_horizon<0, 6>(P, R, which, k, SR, st);
    case 7: return launch_horizon<0, 7>(P, R, which, k, SR, st);
    case 8: return launch_horizon<0, 8>(P, R, which, k, SR, st);
    case 9: return launch_horizon<0, 9>(P, R, which, k, SR, st);
    // node sweeps at d = 1024: 128 threads x 8 amplitudes (measured per outer iteration of
    // config 3: 24.3 ms, vs 25.2 / 25.9 / 36.3 ms at 256 / 512 / 1024 threads)
    case 10: return launch_horizon<3, 7>(P, R, which, k, SR, st);
    case 11: return launch_horizon<2, 9>(P, R, which, k, SR, st);
    case 12: return launch_horizon<3, 9>(P, R, which, k, SR, st);
  }
  return cudaErrorNotSupported;
}

cudaError_t bitflip_horizon(const DevProblem& P, const DevRun& R, int which, int k, cudaStream_t st) {
  return bitflip_horizon_range(P, R, which, k, SweepRange{nullptr, 0, 0}, st);
}

// d = 1024: 128 threads x 8 amplitudes capped at 128 registers (4 CTAs per SM) measured fastest
// per outer iteration of config 3 with 8 blocks: 119.4 ms, vs 123.2 (3 CTAs per SM), 127.0
// (uncapped, 208 registers) and 162.5 / 172.0 for 256 threads x 4 amplitudes (gpurun ab_blocks).
// QOC_BF_BLOCK_SHAPE = 1 | 3 | 8 | 9 selects the other shapes for A/B runs (tools/ab_blocks.sh).
cudaError_t bitflip_block_products(const DevProblem& P, const DevRun& R, const DevBlocks& BK, int g0, int nloc,
                                   cudaStream_t st) {
  if (P.C > 4) return cudaErrorNotSupported;
  if (nloc <= 0) return cudaSuccess;
  switch (P.nspins) {
    case 5: return launch_blocks<0, 5>(P, R, BK, g0, nloc, st);
    case 6: return launch_blocks<0, 6>(P, R, BK, g0, nloc, st);
    case 7: return launch_blocks<0, 7>(P, R, BK, g0, nloc, st);
    case 8: return launch_blocks<0, 8>(P, R, BK, g0, nloc, st);
    case 9: return launch_blocks<1, 8>(P, R, BK, g0, nloc, st);
    case 10: {
      const char* e = std::getenv("QOC_BF_BLOCK_SHAPE");
      if (e && e[0] == '8') return launch_blocks<2, 8>(P, R, BK, g0, nloc, st);
      if (e && e[0] == '9') return launch_blocks<2, 8, 3>(P, R, BK, g0, nloc, st);
      if (e && e[0] == '3') return launch_blocks<3, 7, 3>(P, R, BK, g0, nloc, st);
      if (e && e[0] == '1') return launch_blocks<3, 7, 1>(P, R, BK, g0, nloc, st);
      return launch_blocks<3, 7, 4>(P, R, BK, g0, nloc, st);
    }
    case 11: return launch_blocks<3, 8>(P, R, BK, g0, nloc, st);
    case 12: return launch_blocks<3, 9>(P, R, BK, g0, nloc, st);
  }
  return cudaErrorNotSupported;
}

}  // namespace qoc
