// solvers.cu — the Newton inner solver on the device (sm_100a).
//
// Reference: newton_step / newton_direction / gmres (optimizers.cpp:21-98,215-259).  Per task
// (problem b, subinterval n) the update solves (Hessian) d = -g0 by restarted GMRES, where the
// Hessian-vector product is the central finite difference of the weighted task gradient
//     A v = (grad(u + h v) - grad(u - h v)) / (2 h),   h = hvp_scale * (1 + ||u||) / ||v||,
// and applies u + d, or the plain gradient step rho * g0 when d is not an ascent direction.
//
// B200 shape of it: the expensive part of a GMRES iteration is the pair of gradient sweeps, and
// those already exist as throughput kernels for every propagator kind (task kernels, M_GRAD).  So
// all B x L tasks iterate in lockstep rounds: one advance kernel (a CTA per task) runs each
// task's GMRES state machine on the result of the previous product and writes the next pair of
// perturbed controls into its window of two control-grid buffers; two launches of the kind's own
// task kernel then evaluate every task's gradients at once.  Tasks that converged idle (their
// windows keep valid controls); the host polls one counter per round.  All reductions run in a
// fixed order (thread-strided partials, then a shared-memory tree), so runs are bitwise repeatable.
#include "common.cuh"
#include "kernels.h"

namespace qoc {

namespace {

constexpr int NT = 128;
enum Phase : int { PH_RESID = 0, PH_ARNOLDI = 1, PH_CHECK = 2 };
enum St : int { S_PHASE = 0, S_I = 1, S_USED = 2, S_SPANNED = 3, S_ZERO = 4, S_DONE = 5, S_M = 6 };
enum Sc : int { C_BNORM = 0, C_REL = 1, C_H = 2, C_USCALE = 3 };

__device__ double block_sum(double v, double* red) {
  red[threadIdx.x] = v;
  __syncthreads();
  for (int s = NT / 2; s > 0; s >>= 1) {
    if ((int)threadIdx.x < s) red[threadIdx.x] += red[threadIdx.x + s];
    __syncthreads();
  }
  const double r = red[0];
  __syncthreads();
  return r;
}

struct TaskView {
  int n, b, nel;       // nel = C * len elements of the task's window
  size_t off;          // window offset on the control grid
  double weight;
  double *Hm, *gv, *cs, *sn, *sc;
  int* st;
};

__device__ TaskView view(const DevProblem& P, const DevNewton& N, int n, int b) {
  TaskView T;
  T.n = n;
  T.b = b;
  const int node0 = P.node[n], len = P.node[n + 1] - node0;
  T.nel = P.C * len;
  T.off = ((size_t)b * P.K + node0) * P.C;
  T.weight = N.weighted ? (double)P.K / (double)len : 1.0;
  const size_t t = (size_t)b * P.L + n;
  T.Hm = N.Hm + t * (size_t)(N.restart + 1) * N.restart;
  T.gv = N.gv + t * (N.restart + 1);
  T.cs = N.cs + t * N.restart;
  T.sn = N.sn + t * N.restart;
  T.sc = N.sc + t * 4;
  T.st = N.st + t * 8;
  return T;
}

// Writes the next product's operand: v = x (RESID / CHECK) or V[i] (ARNOLDI); the perturbed
// controls u +- h v, or the zero flag when v = 0 (hessian_apply returns 0 without a gradient).
__device__ void prepare(const DevRun& R, const DevNewton& N, const TaskView& T, double* red) {
  const int phase = T.st[S_PHASE];
  const double* v = phase == PH_ARNOLDI ? N.V + (size_t)T.st[S_I] * N.vstride + T.off : N.x + T.off;
  double s = 0.0;
  for (int e = threadIdx.x; e < T.nel; e += NT) s += v[e] * v[e];
  const double vn = sqrt(block_sum(s, red));
  const double* u = R.u + T.off;
  if (vn == 0.0) {
    if (threadIdx.x == 0) T.st[S_ZERO] = 1;
  } else {
    const double h = N.hvp_scale * T.sc[C_USCALE] / vn;
    for (int e = threadIdx.x; e < T.nel; e += NT) {
      N.up[T.off + e] = u[e] + h * v[e];
      N.um[T.off + e] = u[e] - h * v[e];
    }
    if (threadIdx.x == 0) {
      T.st[S_ZERO] = 0;
      T.sc[C_H] = h;
    }
  }
  __syncthreads();
}

// One transition of the GMRES state machine given w = A v in N.gp (already scaled).
// Returns with st[S_DONE] set, or with the next phase (and Arnoldi index) stored.
__device__ void transition(const DevNewton& N, const TaskView& T, double* red, double* ysm) {
  const int m = T.st[S_M], RS = N.restart;
  const double bnorm = T.sc[C_BNORM];
  double* w = N.gp + T.off;
  const double* g0 = N.g0 + T.off;
  int phase = T.st[S_PHASE], i = T.st[S_I], used = T.st[S_USED], spanned = T.st[S_SPANNED];
  double rel = T.sc[C_REL];
  bool done = false, end_inner = false;
  __syncthreads();
  if (phase == PH_RESID) {
    // r = b - A x with b = -weight g0 (optimizers.cpp:36-41)
    double* v0 = N.V + T.off;
    double s = 0.0;
    for (int e = threadIdx.x; e < T.nel; e += NT) {
      const double r = -T.weight * g0[e] - w[e];
      v0[e] = r;
      s += r * r;
    }
    const double beta = sqrt(block_sum(s, red));
    ++used;
    rel = beta / bnorm;
    if (rel <= N.tol) {
      done = true;
    } else {
      for (int e = threadIdx.x; e < T.nel; e += NT) v0[e] /= beta;
      if (threadIdx.x == 0) {
        for (int r = 0; r <= RS; ++r) T.gv[r] = 0.0;
        T.gv[0] = beta;
        for (int e = 0; e < (RS + 1) * RS; ++e) T.Hm[e] = 0.0;
        for (int c = 0; c < RS; ++c) {
          T.cs[c] = 1.0;
          T.sn[c] = 0.0;
        }
      }
      spanned = 0;
      i = 0;
      if (m > 0 && used < N.max_iter) phase = PH_ARNOLDI;
      else end_inner = true;
    }
    __syncthreads();
  } else if (phase == PH_ARNOLDI) {
    ++used;
    for (int k = 0; k <= i; ++k) {  // modified Gram-Schmidt (optimizers.cpp:56-59)
      const double* vk = N.V + (size_t)k * N.vstride + T.off;
      double s = 0.0;
      for (int e = threadIdx.x; e < T.nel; e += NT) s += vk[e] * w[e];
      const double hk = block_sum(s, red);
      for (int e = threadIdx.x; e < T.nel; e += NT) w[e] -= hk * vk[e];
      if (threadIdx.x == 0) T.Hm[k * RS + i] = hk;
      __syncthreads();
    }
    double s = 0.0;
    for (int e = threadIdx.x; e < T.nel; e += NT) s += w[e] * w[e];
    const double hn = sqrt(block_sum(s, red));
    const bool breakdown = hn <= 1e-14 * bnorm;
    if (!breakdown) {
      double* vn = N.V + (size_t)(i + 1) * N.vstride + T.off;
      for (int e = threadIdx.x; e < T.nel; e += NT) vn[e] = w[e] / hn;
    }
    if (threadIdx.x == 0) {  // Givens rotations (optimizers.cpp:64-76)
      double* H = T.Hm;
      H[(i + 1) * RS + i] = hn;
      for (int k = 0; k < i; ++k) {
        const double t = T.cs[k] * H[k * RS + i] + T.sn[k] * H[(k + 1) * RS + i];
        H[(k + 1) * RS + i] = -T.sn[k] * H[k * RS + i] + T.cs[k] * H[(k + 1) * RS + i];
        H[k * RS + i] = t;
      }
      const double denom = hypot(H[i * RS + i], H[(i + 1) * RS + i]);
      T.cs[i] = denom == 0.0 ? 1.0 : H[i * RS + i] / denom;
      T.sn[i] = denom == 0.0 ? 0.0 : H[(i + 1) * RS + i] / denom;
      H[i * RS + i] = denom;
      H[(i + 1) * RS + i] = 0.0;
      T.gv[i + 1] = -T.sn[i] * T.gv[i];
      T.gv[i] = T.cs[i] * T.gv[i];
      red[0] = fabs(T.gv[i + 1]) / bnorm;
    }
    __syncthreads();
    rel = red[0];
    __syncthreads();
    spanned = i + 1;
    if (rel <= N.tol || breakdown) {
      end_inner = true;
    } else {
      ++i;
      if (!(i < m && used < N.max_iter)) end_inner = true;
    }
  } else {  // PH_CHECK (optimizers.cpp:87-92)
    double s = 0.0;
    for (int e = threadIdx.x; e < T.nel; e += NT) {
      const double r = -T.weight * g0[e] - w[e];
      s += r * r;
    }
    ++used;
    rel = sqrt(block_sum(s, red)) / bnorm;
    if (rel <= N.tol) done = true;
    else if (used < N.max_iter) phase = PH_RESID;
    else done = true;
  }
  if (end_inner) {
    if (spanned > 0) {  // x += V y, y from the rotated upper-triangular block (optimizers.cpp:80-85)
      if (threadIdx.x == 0) {
        for (int r = spanned - 1; r >= 0; --r) {
          double acc = T.gv[r];
          for (int c = r + 1; c < spanned; ++c) acc -= T.Hm[r * RS + c] * ysm[c];
          ysm[r] = acc / T.Hm[r * RS + r];
        }
      }
      __syncthreads();
      double* x = N.x + T.off;
      for (int e = threadIdx.x; e < T.nel; e += NT) {
        double acc = x[e];
        for (int c = 0; c < spanned; ++c) acc += N.V[(size_t)c * N.vstride + T.off + e] * ysm[c];
        x[e] = acc;
      }
      __syncthreads();
    }
    if (rel <= N.tol) phase = PH_CHECK;
    else if (used < N.max_iter) phase = PH_RESID;
    else done = true;
  }
  if (threadIdx.x == 0) {
    T.st[S_PHASE] = phase;
    T.st[S_I] = i;
    T.st[S_USED] = used;
    T.st[S_SPANNED] = spanned;
    T.st[S_DONE] = done ? 1 : 0;
    T.sc[C_REL] = rel;
  }
  __syncthreads();
}

// Advance until a product that needs gradients is pending, or the solve is over.
__device__ void run_until_product(const DevRun& R, const DevNewton& N, const TaskView& T, double* red, double* ysm) {
  for (;;) {
    if (T.st[S_DONE]) return;
    prepare(R, N, T, red);
    if (!T.st[S_ZERO]) return;
    // A 0 = 0: no gradient evaluation (optimizers.cpp:223)
    for (int e = threadIdx.x; e < T.nel; e += NT) N.gp[T.off + e] = 0.0;
    __syncthreads();
    transition(N, T, red, ysm);
  }
}

__global__ void __launch_bounds__(NT) newton_begin_kernel(DevProblem P, DevRun R, DevNewton N) {
  __shared__ double red[NT];
  extern __shared__ double ysm[];
  const int n = blockIdx.x, b = blockIdx.y;
  const TaskView T = view(P, N, n, b);
  if (R.done[b] | R.status[b]) {
    if (threadIdx.x == 0) T.st[S_DONE] = 1;
    return;
  }
  const double* u = R.u + T.off;
  const double* g0 = N.g0 + T.off;
  double su = 0.0;
  for (int e = threadIdx.x; e < T.nel; e += NT) {
    su += u[e] * u[e];
    N.x[T.off + e] = 0.0;
    N.up[T.off + e] = u[e];  // valid controls for the lockstep gradient launches of idle tasks
    N.um[T.off + e] = u[e];
  }
  const double un = sqrt(block_sum(su, red));
  // ||b|| = ||-(weight g0)||: scale every element first, as the reference's sub_gradient does
  double sb = 0.0;
  for (int e = threadIdx.x; e < T.nel; e += NT) {
    const double be = T.weight * g0[e];
    sb += be * be;
  }
  const double bnorm = sqrt(block_sum(sb, red));
  if (threadIdx.x == 0) {
    T.sc[C_BNORM] = bnorm;
    T.sc[C_REL] = 0.0;
    T.sc[C_USCALE] = 1.0 + un;
    T.st[S_PHASE] = PH_RESID;
    T.st[S_I] = 0;
    T.st[S_USED] = 0;
    T.st[S_SPANNED] = 0;
    T.st[S_ZERO] = 0;
    T.st[S_DONE] = bnorm == 0.0 ? 1 : 0;  // optimizers.cpp:31-35
    T.st[S_M] = min(N.restart, T.nel);
  }
  __syncthreads();
  if (!(N.max_iter > 0)) {
    if (threadIdx.x == 0) T.st[S_DONE] = 1;
    __syncthreads();
  }
  run_until_product(R, N, T, red, ysm);
  if (threadIdx.x == 0 && !T.st[S_DONE]) atomicAdd(N.active, 1);
}

__global__ void __launch_bounds__(NT) newton_advance_kernel(DevProblem P, DevRun R, DevNewton N, int round) {
  __shared__ double red[NT];
  extern __shared__ double ysm[];
  const int n = blockIdx.x, b = blockIdx.y;
  const TaskView T = view(P, N, n, b);
  if (T.st[S_DONE]) return;
  // w = A v = weight (grad(u + h v) - grad(u - h v)) / (2 h)   (optimizers.cpp:224-228)
  const double h = T.sc[C_H];
  for (int e = threadIdx.x; e < T.nel; e += NT) {
    const double gp = T.weight * N.gp[T.off + e], gm = T.weight * N.gm[T.off + e];
    N.gp[T.off + e] = (gp - gm) / (2.0 * h);
  }
  __syncthreads();
  transition(N, T, red, ysm);
  run_until_product(R, N, T, red, ysm);
  if (threadIdx.x == 0 && !T.st[S_DONE]) atomicAdd(N.active + round, 1);
}

// newton_step's tail (optimizers.cpp:246-257): u += d, or the gradient fallback.
__global__ void __launch_bounds__(NT) newton_apply_kernel(DevProblem P, DevRun R, DevNewton N) {
  __shared__ double red[NT];
  const int n = blockIdx.x, b = blockIdx.y;
  if (R.done[b] | R.status[b]) return;
  const TaskView T = view(P, N, n, b);
  const double* g0 = N.g0 + T.off;
  const double* x = N.x + T.off;
  double s = 0.0;
  for (int e = threadIdx.x; e < T.nel; e += NT) s += x[e] * (T.weight * g0[e]);
  const double dot = block_sum(s, red);
  const bool fallback = !(dot > 0.0);
  double* u = R.u + T.off;
  for (int e = threadIdx.x; e < T.nel; e += NT) {
    const double d = fallback ? N.step_size * (T.weight * g0[e]) : x[e];
    u[e] = u[e] + d;
  }
  if (threadIdx.x == 0) {
    int* stats = N.stats + ((size_t)b * P.L + n) * 3;
    if (fallback) stats[1] += 1;
    stats[2] += T.st[S_USED];
  }
}

}  // namespace

cudaError_t newton_begin(const DevProblem& P, const DevRun& R, const DevNewton& N, cudaStream_t st) {
  newton_begin_kernel<<<dim3(P.L, P.B), NT, sizeof(double) * (N.restart + 1), st>>>(P, R, N);
  return cudaGetLastError();
}
cudaError_t newton_advance(const DevProblem& P, const DevRun& R, const DevNewton& N, int round, cudaStream_t st) {
  newton_advance_kernel<<<dim3(P.L, P.B), NT, sizeof(double) * (N.restart + 1), st>>>(P, R, N, round);
  return cudaGetLastError();
}
cudaError_t newton_apply(const DevProblem& P, const DevRun& R, const DevNewton& N, cudaStream_t st) {
  newton_apply_kernel<<<dim3(P.L, P.B), NT, 0, st>>>(P, R, N);
  return cudaGetLastError();
}

}  // namespace qoc
