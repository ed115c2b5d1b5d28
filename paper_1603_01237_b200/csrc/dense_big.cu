// dense_big.cu — QOC_KIND_DENSE task and horizon kernels for 32 < d <= 64 (sm_100a).
//
// The reference's DenseModel takes any d (models.cpp:45-75) and its micro-benchmarks time a
// d = 64 Crank-Nicolson step (benchmarks.cpp:76).  Above the warp-resident sizes of
// dense_kernels.cu a task owns a CTA: the step matrix B_j = I + i dt/2 H(u_j) (models.cpp:57-68,
// propagation.cpp:14-16) is built in shared memory, inverted in place by Gauss-Jordan with
// partial pivoting (largest |.| in the column, first row on ties, then the column unscramble --
// the pivot order of Eigen's PartialPivLU, propagation.cpp:85-90), and every sweep applies
//     C_j = 2 B_j^-1 - I          forward          (cn_step, propagation.cpp:85-90)
//     C_j^dag = 2 B_j^-dag - I     adjoint          (cn_adjoint_step, propagation.cpp:101-106)
// as matvecs (threads over rows), and P <- 2 B_j^-1 P - P for the assembled propagator
// (propagation.cpp:236-249).  The task body is the same as dense_task_kernel's (ism.cpp:401-479):
// entry value, gradient sweep with the fused update (objective.cpp:48-60, optimizers.cpp:102-107),
// residual sweep (error_norm), assembly and the split-variant lagged refresh.
#include <cstdlib>
#include <cstring>

#include "common.cuh"
#include "kernels.h"
#include "qoc_gpu.h"

namespace qoc {

namespace {

constexpr int BT = 256;     // threads per task CTA
constexpr int BIG_MAX = 64;  // three d x d complex buffers (assembly) within 227 KB

struct BigSmem {
  double2* W;     // [d][d] row-major: B_j, then its inverse
  double2* Pm;    // [d][d] assembly product (M_ASSEMBLE only)
  double2* T;     // [d][d] matmul scratch (M_ASSEMBLE only)
  double2* x;     // [d] state vectors
  double2* y;
  double2* z;
  double2* v;
  double2* prow;  // [d] pivot row
  double2* colk;  // [d] pivot column (read before the elimination writes it)
  double* red;    // [BT] reduction scratch
  int* perm;      // [d]
  int* piv;       // [2]
};

__device__ double block_sum(double v, double* red) {
  red[threadIdx.x] = v;
  __syncthreads();
  for (int s = BT / 2; s > 0; s >>= 1) {
    if ((int)threadIdx.x < s) red[threadIdx.x] += red[threadIdx.x + s];
    __syncthreads();
  }
  const double r = red[0];
  __syncthreads();
  return r;
}

// B = I + s i H(u), s = +half (forward) -- H(u) = H0 + sum u_c A_c + sum (u_c^2/2) B_c
__device__ void build(const DevProblem& P, int b, const double* u, double half, double2* W, int dmat = 0) {
  const int d = dmat ? dmat : P.d, C = P.C;
  const size_t dd = (size_t)d * d;
  for (int e = threadIdx.x; e < d * d; e += BT) {
    double2 h = P.h0[(size_t)b * dd + e];
    for (int c = 0; c < C; ++c) {
      const double2 a = P.lin[((size_t)b * C + c) * dd + e];
      h = cx(fma(u[c], a.x, h.x), fma(u[c], a.y, h.y));
      if (P.has_quad) {
        const double2 q = P.quad[((size_t)b * C + c) * dd + e];
        const double s = 0.5 * u[c] * u[c];
        h = cx(fma(s, q.x, h.x), fma(s, q.y, h.y));
      }
    }
    const int i = e / d, j = e % d;
    W[e] = cx((i == j ? 1.0 : 0.0) - half * h.y, half * h.x);
  }
  __syncthreads();
}

// In-place Gauss-Jordan inverse with partial pivoting and the column unscramble.
__device__ void invert(int d, const BigSmem& S) {
  double2* W = S.W;
  for (int k = 0; k < d; ++k) {
    // pivot: first row of largest |W[i][k]|, i >= k
    double best = -1.0;
    int bi = d;
    for (int i = k + threadIdx.x; i < d; i += BT) {
      const double v = cabs2(W[i * d + k]);
      if (v > best) {
        best = v;
        bi = i;
      }
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
      const double ob = __shfl_xor_sync(0xffffffffu, best, off);
      const int oi = __shfl_xor_sync(0xffffffffu, bi, off);
      if (ob > best || (ob == best && oi < bi)) {
        best = ob;
        bi = oi;
      }
    }
    if ((threadIdx.x & 31) == 0) {
      S.red[threadIdx.x >> 5] = best;
      S.perm[d + (threadIdx.x >> 5)] = bi;  // scratch after perm[0..d)
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      double bb = S.red[0];
      int ii = S.perm[d];
      for (int w = 1; w < BT / 32; ++w) {
        const double ob = S.red[w];
        const int oi = S.perm[d + w];
        if (ob > bb || (ob == bb && oi < ii)) {
          bb = ob;
          ii = oi;
        }
      }
      S.piv[0] = ii;
      S.perm[k] = ii;
    }
    __syncthreads();
    const int p = S.piv[0];
    if (p != k)
      for (int j = threadIdx.x; j < d; j += BT) {
        const double2 t = W[k * d + j];
        W[k * d + j] = W[p * d + j];
        W[p * d + j] = t;
      }
    __syncthreads();
    const double2 pinv = crcp(W[k * d + k]);
    for (int j = threadIdx.x; j < d; j += BT) {
      S.prow[j] = (j == k) ? pinv : cmul(W[k * d + j], pinv);
      S.colk[j] = W[j * d + k];
    }
    __syncthreads();
    for (int e = threadIdx.x; e < d * d; e += BT) {
      const int i = e / d, j = e % d;
      if (i == k) continue;
      const double2 f = S.colk[i];
      W[e] = (j == k) ? cneg(cmul(f, pinv)) : cfms(f, S.prow[j], W[e]);
    }
    __syncthreads();
    for (int j = threadIdx.x; j < d; j += BT) W[k * d + j] = S.prow[j];
    __syncthreads();
  }
  // undo the row interchanges on the columns of the inverse (reverse order)
  for (int k = d - 1; k >= 0; --k) {
    const int p = S.perm[k];
    if (p != k)
      for (int i = threadIdx.x; i < d; i += BT) {
        const double2 t = W[i * d + k];
        W[i * d + k] = W[i * d + p];
        W[i * d + p] = t;
      }
    __syncthreads();
  }
}

// y = 2 W x - x (adj: 2 W^dag x - x); rows over threads, x in smem; y may not alias x
__device__ void cayley(int d, const double2* W, const double2* x, double2* y, bool adj) {
  for (int i = threadIdx.x; i < d; i += BT) {
    double2 acc = cx(0.0, 0.0);
    if (adj)
      for (int k = 0; k < d; ++k) acc = cfmaconj(W[k * d + i], x[k], acc);
    else
      for (int k = 0; k < d; ++k) acc = cfma(W[i * d + k], x[k], acc);
    y[i] = cx(2.0 * acc.x - x[i].x, 2.0 * acc.y - x[i].y);
  }
  __syncthreads();
}

__device__ void copy_vec(int d, const double2* src, double2* dst) {
  for (int i = threadIdx.x; i < d; i += BT) dst[i] = src[i];
  __syncthreads();
}

// Im <cs, dH/du_c(u_c) ps>, dH/du_c = A_c + u_c B_c (models.cpp:70-75)
__device__ double grad_im(const DevProblem& P, int b, int c, double uc, const double2* ps, const double2* cs,
                          double* red) {
  const int d = P.d;
  const size_t dd = (size_t)d * d;
  double im = 0.0;
  for (int i = threadIdx.x; i < d; i += BT) {
    double2 acc = cx(0.0, 0.0);
    for (int k = 0; k < d; ++k) {
      double2 a = P.lin[((size_t)b * P.C + c) * dd + (size_t)i * d + k];
      if (P.has_quad) {
        const double2 q = P.quad[((size_t)b * P.C + c) * dd + (size_t)i * d + k];
        a = cx(fma(uc, q.x, a.x), fma(uc, q.y, a.y));
      }
      acc = cfma(a, ps[k], acc);
    }
    im += cconjmul(cs[i], acc).y;
  }
  return block_sum(im, red);
}

__device__ BigSmem carve(unsigned char* raw, int d, bool with_asm) {
  BigSmem S;
  double2* p = reinterpret_cast<double2*>(raw);
  S.W = p;
  p += (size_t)d * d;
  S.Pm = with_asm ? p : nullptr;
  if (with_asm) p += (size_t)d * d;
  S.T = with_asm ? p : nullptr;
  if (with_asm) p += (size_t)d * d;
  S.x = p;
  S.y = p + d;
  S.z = p + 2 * d;
  S.v = p + 3 * d;
  S.prow = p + 4 * d;
  S.colk = p + 5 * d;
  p += 6 * d;
  S.red = reinterpret_cast<double*>(p);
  S.perm = reinterpret_cast<int*>(S.red + BT);
  S.piv = S.perm + d + BT / 32;
  return S;
}

size_t big_smem(int d, bool with_asm) {
  return sizeof(double2) * ((size_t)d * d * (with_asm ? 3 : 1) + 6 * (size_t)d) + sizeof(double) * BT +
         sizeof(int) * (d + BT / 32 + 2);
}

__global__ void __launch_bounds__(BT) dense_big_task_kernel(DevProblem P, DevRun R, TaskArgs A, int ignore_done) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int n = blockIdx.x, b = blockIdx.y;
  if (ignore_done ? R.status[b] : (R.done[b] | R.status[b])) return;
  const int mode = A.mode;
  const bool do_asm = (mode & M_ASSEMBLE) != 0;
  const BigSmem S = carve(smem_raw, P.d, do_asm);
  const int d = P.d, C = P.C;
  const int node0 = P.node[n], len = P.node[n + 1] - node0;
  const double Kd = (double)P.K, weight = A.weighted ? Kd / (double)len : 1.0, scale = (double)len / Kd;
  const double half = 0.5 * P.dt, dt = P.dt, w = P.ip_w;
  double* u = R.u + ((size_t)b * P.K + node0) * C;
  double2* traj = R.traj + ((size_t)b * P.L + n) * (size_t)R.traj_len * d;
  const size_t tix = ((size_t)b * P.L + n) * d;
  const double2* init = R.task_init + tix;
  const double2* targ = R.task_targ + tix;

  // ---- phase 1: sweeps at the current control
  if (mode & (M_ENTRY | M_UPDATE | M_FINAL | M_GRAD)) {
    const bool need_traj = (mode & (M_UPDATE | M_GRAD)) != 0;
    const int iters = (mode & M_UPDATE) ? A.inner : 1;
    for (int it = 0; it < iters; ++it) {
      copy_vec(d, init, S.x);
      if (need_traj) copy_vec(d, S.x, traj);
      double pen = 0.0;
      for (int j = 0; j < len; ++j) {
        const double* uj = u + (size_t)j * C;
        build(P, b, uj, half, S.W);
        invert(d, S);
        cayley(d, S.W, S.x, S.y, false);
        copy_vec(d, S.y, S.x);
        if (need_traj) copy_vec(d, S.x, traj + (size_t)(j + 1) * d);
        double sq = 0.0;
        for (int c = 0; c < C; ++c) sq += uj[c] * uj[c];
        pen += (P.alpha[node0 + j] * scale) * sq;
      }
      if (it == 0 && (mode & M_ENTRY)) {  // sub_functional (objective.cpp:131-134)
        double t = 0.0;
        for (int i = threadIdx.x; i < d; i += BT)
          t += A.form == 0 ? cconjmul(targ[i], S.x[i]).x : cabs2(csub(S.x[i], targ[i]));
        t = block_sum(t, S.red);
        const double payoff = A.form == 0 ? (w * t) : (-0.5 * (w * t));
        if (threadIdx.x == 0) R.entry[(size_t)b * P.L + n] = weight * (payoff - 0.5 * dt * pen);
      }
      if (it == 0 && (mode & M_FINAL)) copy_vec(d, S.x, R.psi_end + tix);
      if (mode & (M_UPDATE | M_GRAD)) {
        for (int i = threadIdx.x; i < d; i += BT) S.z[i] = A.form == 0 ? targ[i] : csub(targ[i], S.x[i]);
        __syncthreads();
        for (int j = len - 1; j >= 0; --j) {
          const double* uj = u + (size_t)j * C;
          build(P, b, uj, half, S.W);
          invert(d, S);
          cayley(d, S.W, S.z, S.y, true);  // chi_j
          for (int i = threadIdx.x; i < d; i += BT) {
            S.v[i] = cadd(traj[(size_t)j * d + i], traj[(size_t)(j + 1) * d + i]);  // psi sum
            S.prow[i] = cadd(S.y[i], S.z[i]);                                     // chi sum
          }
          __syncthreads();
          const double aj = P.alpha[node0 + j] * scale;
          for (int c = 0; c < C; ++c) {
            const double uc = uj[c];
            const double im = grad_im(P, b, c, uc, S.v, S.prow, S.red);
            const double gc = -aj * dt * uc + 0.25 * dt * (w * im);
            if (threadIdx.x == 0) {
              if (mode & M_GRAD) R.grad[((size_t)b * P.K + node0 + j) * C + c] = gc;
              if (mode & M_UPDATE) u[(size_t)j * C + c] = uc + A.rho * (weight * gc);
            }
            __syncthreads();
          }
          copy_vec(d, S.y, S.z);
        }
      }
    }
  }

  // ---- phase 2: sweeps at the updated control
  const bool do_err = (mode & M_ERROR) != 0, do_lag = (mode & M_LAGGED) != 0;
  if (do_err || do_asm || do_lag) {
    copy_vec(d, init, S.x);
    if (do_lag) copy_vec(d, R.psi_nodes + ((size_t)b * (P.L + 1) + n) * d, S.z);
    if (do_err) copy_vec(d, S.x, traj);
    if (do_asm)
      for (int e = threadIdx.x; e < d * d; e += BT) S.Pm[e] = cx((e / d) == (e % d) ? 1.0 : 0.0, 0.0);
    __syncthreads();
    for (int j = 0; j < len; ++j) {
      build(P, b, u + (size_t)j * C, half, S.W);
      invert(d, S);
      if (do_err) {
        cayley(d, S.W, S.x, S.y, false);
        copy_vec(d, S.y, S.x);
        copy_vec(d, S.x, traj + (size_t)(j + 1) * d);
      }
      if (do_lag) {
        cayley(d, S.W, S.z, S.y, false);
        copy_vec(d, S.y, S.z);
      }
      if (do_asm) {  // P <- 2 W P - P
        for (int e = threadIdx.x; e < d * d; e += BT) {
          const int i = e / d, c = e % d;
          double2 acc = cx(0.0, 0.0);
          for (int k = 0; k < d; ++k) acc = cfma(S.W[i * d + k], S.Pm[k * d + c], acc);
          S.T[e] = cx(2.0 * acc.x - S.Pm[e].x, 2.0 * acc.y - S.Pm[e].y);
        }
        __syncthreads();
        for (int e = threadIdx.x; e < d * d; e += BT) S.Pm[e] = S.T[e];
        __syncthreads();
      }
    }
    if (do_asm)
      for (int e = threadIdx.x; e < d * d; e += BT) R.prop[((size_t)b * P.L + n) * (size_t)d * d + e] = S.Pm[e];
    if (do_lag) copy_vec(d, S.z, R.psi_end + tix);
    if (do_err || do_lag) {
      // residual adjoint (error_norm) seeded from the residual forward state; lagged adjoint from chi_{n+1}
      for (int i = threadIdx.x; i < d; i += BT) S.v[i] = A.form == 0 ? targ[i] : csub(targ[i], S.x[i]);
      if (do_lag) copy_vec(d, R.chi_nodes + ((size_t)b * (P.L + 1) + n + 1) * d, S.z);
      __syncthreads();
      double err = 0.0;
      for (int j = len - 1; j >= 0; --j) {
        const double* uj = u + (size_t)j * C;
        build(P, b, uj, half, S.W);
        invert(d, S);
        if (do_lag) {
          cayley(d, S.W, S.z, S.y, true);
          copy_vec(d, S.y, S.z);
        }
        if (do_err) {
          cayley(d, S.W, S.v, S.y, true);  // chi_j
          double2* ps = S.Pm ? S.T : S.prow;   // scratch vectors (T is free after the assembly)
          double2* cs = S.x;
          for (int i = threadIdx.x; i < d; i += BT) {
            ps[i] = cadd(traj[(size_t)j * d + i], traj[(size_t)(j + 1) * d + i]);
            cs[i] = cadd(S.y[i], S.v[i]);
          }
          __syncthreads();
          const double aj = P.alpha[node0 + j] * scale;
          double sq = 0.0;
          for (int c = 0; c < C; ++c) {
            const double uc = uj[c];
            const double im = grad_im(P, b, c, uc, ps, cs, S.red);
            const double gc = -aj * dt * uc + 0.25 * dt * (w * im);
            sq += gc * gc;
          }
          err += sqrt(sq);
          copy_vec(d, S.y, S.v);
        }
      }
      if (do_err && threadIdx.x == 0) R.err[(size_t)b * P.L + n] = err;
      if (do_lag) copy_vec(d, S.z, R.chi_start + tix);
    }
  }
}

// node_sweeps (ism.cpp:35-84) / exact payoff (which = 1), one CTA per problem
__global__ void __launch_bounds__(BT) dense_big_horizon_kernel(DevProblem P, DevRun R, int which, int k) {
  if (R.kdev) k = *R.kdev;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int b = blockIdx.x;
  if (R.done[b] || R.status[b]) return;
  const BigSmem S = carve(smem_raw, P.d, false);
  const int d = P.d, C = P.C;
  const double half = 0.5 * P.dt;
  const double* u = R.u + (size_t)b * P.K * C;
  const size_t nb = (size_t)b * (P.L + 1) * d;
  copy_vec(d, P.init + (size_t)b * d, S.x);
  if (which == 0) copy_vec(d, S.x, R.psi_nodes + nb);
  int nxt = 1;
  for (int j = 0; j < P.K; ++j) {
    build(P, b, u + (size_t)j * C, half, S.W);
    invert(d, S);
    cayley(d, S.W, S.x, S.y, false);
    copy_vec(d, S.y, S.x);
    if (which == 0 && nxt <= P.L && P.node[nxt] == j + 1) {
      copy_vec(d, S.x, R.psi_nodes + nb + (size_t)nxt * d);
      ++nxt;
    }
  }
  if (which == 1) {
    double t = 0.0;
    for (int i = threadIdx.x; i < d; i += BT) t += cconjmul(P.targ[(size_t)b * d + i], S.x[i]).x;
    t = block_sum(t, S.red);
    if (threadIdx.x == 0) {
      double pen = 0.0;
      for (int n = 0; n < P.L; ++n) pen += R.pen[(size_t)b * P.L + n];
      R.rec_exact[(size_t)b * R.cap + k] = P.ip_w * t - 0.5 * P.dt * pen;
    }
    return;
  }
  copy_vec(d, P.targ + (size_t)b * d, S.x);
  copy_vec(d, S.x, R.chi_nodes + nb + (size_t)P.L * d);
  int prev = P.L - 1;
  for (int j = P.K - 1; j >= 0; --j) {
    build(P, b, u + (size_t)j * C, half, S.W);
    invert(d, S);
    cayley(d, S.W, S.x, S.y, true);
    copy_vec(d, S.y, S.x);
    if (prev >= 0 && P.node[prev] == j) {
      copy_vec(d, S.x, R.chi_nodes + nb + (size_t)prev * d);
      --prev;
    }
  }
}

// ---- density-matrix (conjugation) kind: CTA per task --------------------------------------
// States are dm x dm matrices held column-major (the packed ABI layout, state length P.d = dm^2);
// W = B_j^-1 is row-major (build + invert above).  With A = 2W - I (propagation.cpp:92-129):
//   forward   rho' = A rho A^dag : G = 2 W rho - rho,  rho' = 2 G W^dag - G
//   adjoint   X'   = A^dag X A   : b = 2 W^dag X - X,  X'   = 2 b W - b
//   gradient  g_c  = -alpha dt u_c + 2 dt Im tr(r1^dag dH_c r2),  r1 = W^dag X_{j+1},
//             r2 = W^dag rho_{j+1}  (cn_conjugation_backward_stage + objective.cpp:61-71), and
//             b = 2 r1 - X_{j+1}.
constexpr int DENS_MAX = 32;

// C = op(A) op(B), dm x dm; A/B/C accessors select layout and conjugate-transpose
enum MOp { ROW = 0, ROW_H = 1, COL = 2, COL_H = 3 };
__device__ __forceinline__ double2 at(const double2* M, int dm, int i, int j, MOp op) {
  switch (op) {
    case ROW: return M[i * dm + j];
    case ROW_H: return cconj(M[j * dm + i]);
    case COL: return M[i + j * dm];
    default: return cconj(M[j + i * dm]);
  }
}
// fp64 tensor-core form of mm for dm = 32 (the 5-spin density matrices): the complex product as
// four real m8n8k4 products per 8 x 8 output tile and k-chunk.  Warp w of the CTA's eight owns the
// 8 x 16 strip of tile row w / 2, tile columns 2 (w % 2) and 2 (w % 2) + 1, so one A fragment
// feeds two tiles.  Fragments (PTX m8n8k4 f64): lane l holds A[l / 4][l % 4], B[l % 4][l / 4]
// and C[l / 4][2 (l % 4) + {0, 1}]; operands are read straight from their row- / column-major,
// plain / conjugate-transposed buffers through at().  1 = on (QOC_DISABLE=densmma switches off).
__constant__ int c_dens_dmma = 1;

__device__ __forceinline__ void dmma884(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

__device__ void mm_dmma32(const double2* A, MOp oa, const double2* Bm, MOp ob, double alpha, const double2* Cin,
                          double beta, double2* out) {
  constexpr int dm = 32;
  const int warp = threadIdx.x >> 5, l = threadIdx.x & 31;
  const int q = l >> 2, r = l & 3;
  const int i = 8 * (warp >> 1) + q;  // A row of this lane's fragment element
  const int tc0 = 2 * (warp & 1);
  double cr[2][2] = {{0.0, 0.0}, {0.0, 0.0}}, ci[2][2] = {{0.0, 0.0}, {0.0, 0.0}};
#pragma unroll
  for (int kc = 0; kc < dm / 4; ++kc) {
    const int k = 4 * kc + r;
    const double2 a = at(A, dm, i, k, oa);
#pragma unroll
    for (int t = 0; t < 2; ++t) {
      const double2 b = at(Bm, dm, k, 8 * (tc0 + t) + q, ob);
      dmma884(cr[t][0], cr[t][1], a.x, b.x);
      dmma884(cr[t][0], cr[t][1], -a.y, b.y);
      dmma884(ci[t][0], ci[t][1], a.x, b.y);
      dmma884(ci[t][0], ci[t][1], a.y, b.x);
    }
  }
#pragma unroll
  for (int t = 0; t < 2; ++t)
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int j = 8 * (tc0 + t) + 2 * r + h, e = i + j * dm;
      double2 v = cx(alpha * cr[t][h], alpha * ci[t][h]);
      if (beta != 0.0) v = cx(fma(beta, Cin[e].x, v.x), fma(beta, Cin[e].y, v.y));
      out[e] = v;
    }
  __syncthreads();
}

// out (column-major) = alpha * op(A) op(B) + beta * Cin (column-major, may alias out only if beta == 0)
__device__ void mm(int dm, const double2* A, MOp oa, const double2* Bm, MOp ob, double alpha, const double2* Cin,
                   double beta, double2* out) {
  if (dm == 32 && c_dens_dmma) {
    mm_dmma32(A, oa, Bm, ob, alpha, Cin, beta, out);
    return;
  }
  for (int e = threadIdx.x; e < dm * dm; e += BT) {
    const int i = e % dm, j = e / dm;
    double2 acc = cx(0.0, 0.0);
    for (int k = 0; k < dm; ++k) acc = cfma(at(A, dm, i, k, oa), at(Bm, dm, k, j, ob), acc);
    double2 r = cx(alpha * acc.x, alpha * acc.y);
    if (beta != 0.0) r = cx(fma(beta, Cin[e].x, r.x), fma(beta, Cin[e].y, r.y));
    out[e] = r;
  }
  __syncthreads();
}

struct DensSmem {
  double2 *W, *S, *G, *T, *X;  // W row-major; states column-major
  BigSmem lin;                 // vectors / reduction scratch of invert
};

__device__ DensSmem carve_dens(unsigned char* raw, int dm) {
  DensSmem D;
  double2* p = reinterpret_cast<double2*>(raw);
  const size_t mm2 = (size_t)dm * dm;
  D.W = p;
  D.S = p + mm2;
  D.G = p + 2 * mm2;
  D.T = p + 3 * mm2;
  D.X = p + 4 * mm2;
  BigSmem& S = D.lin;
  S.W = D.W;
  S.Pm = S.T = nullptr;
  double2* v = p + 5 * mm2;
  S.x = v;
  S.y = v + dm;
  S.z = v + 2 * dm;
  S.v = v + 3 * dm;
  S.prow = v + 4 * dm;
  S.colk = v + 5 * dm;
  S.red = reinterpret_cast<double*>(v + 6 * dm);
  S.perm = reinterpret_cast<int*>(S.red + BT);
  S.piv = S.perm + dm + BT / 32;
  return D;
}

size_t dens_smem(int dm) {
  return sizeof(double2) * (5 * (size_t)dm * dm + 6 * (size_t)dm) + sizeof(double) * BT +
         sizeof(int) * (dm + BT / 32 + 2);
}

// Gauss-Jordan inverse without row interchanges: two barriers per pivot instead of the pivot
// search, swap and unscramble of invert().  Valid when B = I + i dt/2 H(u) is strictly column
// diagonally dominant, where partial pivoting never swaps (the same test as dense.cuh).
__device__ void invert_nopivot(int d, const BigSmem& S) {
  double2* W = S.W;
  for (int k = 0; k < d; ++k) {
    const double2 pinv = crcp(W[k * d + k]);
    for (int j = threadIdx.x; j < d; j += BT) {
      S.prow[j] = (j == k) ? pinv : cmul(W[k * d + j], pinv);
      S.colk[j] = W[j * d + k];
    }
    __syncthreads();
    for (int e = threadIdx.x; e < d * d; e += BT) {
      const int i = e / d, j = e % d;
      if (i == k) {
        W[e] = S.prow[j];
      } else {
        const double2 f = S.colk[i];
        W[e] = (j == k) ? cneg(cmul(f, pinv)) : cfms(f, S.prow[j], W[e]);
      }
    }
    __syncthreads();
  }
}

// W = B_j^-1 at control uj
__device__ void dens_inverse(const DevProblem& P, int b, const double* uj, DensSmem& D) {
  build(P, b, uj, 0.5 * P.dt, D.W, P.dm);
  // dt/2 ||H(u_j)||_1 < 1 (column sums bounded through the operators' 1-norms)
  const double* nb = P.norm1 + (size_t)b * (1 + 2 * P.C);
  double bound = nb[0];
  for (int c = 0; c < P.C; ++c) {
    bound += fabs(uj[c]) * nb[1 + c];
    if (P.has_quad) bound += 0.5 * uj[c] * uj[c] * nb[1 + P.C + c];
  }
  if (0.5 * P.dt * bound < 1.0) invert_nopivot(P.dm, D.lin);
  else invert(P.dm, D.lin);
}
// rho (column-major in/out) <- A rho A^dag ; uses G
__device__ void dens_forward(int dm, DensSmem& D, double2* rho) {
  mm(dm, D.W, ROW, rho, COL, 2.0, rho, -1.0, D.G);     // G = 2 W rho - rho
  mm(dm, D.G, COL, D.W, ROW_H, 2.0, D.G, -1.0, rho);   // rho' = 2 G W^dag - G
}
// X (column-major in/out) <- A^dag X A ; uses G
__device__ void dens_adjoint(int dm, DensSmem& D, double2* X) {
  mm(dm, D.W, ROW_H, X, COL, 2.0, X, -1.0, D.G);       // b = 2 W^dag X - X
  mm(dm, D.G, COL, D.W, ROW, 2.0, D.G, -1.0, X);       // X' = 2 b W - b
}
__device__ void dens_copy(int n, const double2* src, double2* dst) {
  for (int i = threadIdx.x; i < n; i += BT) dst[i] = src[i];
  __syncthreads();
}
// All channels' Im tr(r1^dag dH_c r2) at once: tr(r1^dag dH_c r2) = tr(dH_c M) with
// M = r2 r1^dag (one dm^3 product, column-major in Mx), so each channel is a dm^2 contraction
// sum_{i,k} dH_c[i][k] M[k][i] instead of its own dm^3 product.  out[c] for c < C (all threads).
constexpr int TRC = 8;  // channels per pass over M
__device__ void dens_traces(const DevProblem& P, int b, const double* uj, const double2* Mx, double* red,
                            double* out) {
  const int dm = P.dm, C = P.C;
  const size_t dd = (size_t)dm * dm;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int c0 = 0; c0 < C; c0 += TRC) {
    double im[TRC];
#pragma unroll
    for (int q = 0; q < TRC; ++q) im[q] = 0.0;
    for (int e = threadIdx.x; e < dm * dm; e += BT) {
      const int i = e / dm, k = e % dm;       // dH_c[i][k] (row-major) with M[k][i]
      const double2 m = Mx[k + i * dm];
#pragma unroll
      for (int q = 0; q < TRC; ++q) {
        const int c = c0 + q;
        if (c < C) {
          double2 a = P.lin[((size_t)b * C + c) * dd + e];
          if (P.has_quad) {
            const double2 qd = P.quad[((size_t)b * C + c) * dd + e];
            a = cx(fma(uj[c], qd.x, a.x), fma(uj[c], qd.y, a.y));
          }
          im[q] += a.x * m.y + a.y * m.x;  // Im(a m)
        }
      }
    }
#pragma unroll
    for (int q = 0; q < TRC; ++q)
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) im[q] += __shfl_xor_sync(0xffffffffu, im[q], off);
    __syncthreads();
    if (lane == 0)
#pragma unroll
      for (int q = 0; q < TRC; ++q) red[warp * TRC + q] = im[q];
    __syncthreads();
#pragma unroll
    for (int q = 0; q < TRC; ++q) {
      double sacc = 0.0;
      for (int w2 = 0; w2 < BT / 32; ++w2) sacc += red[w2 * TRC + q];
      if (c0 + q < C) out[c0 + q] = sacc;
    }
    __syncthreads();
  }
}

__global__ void __launch_bounds__(BT) density_task_kernel(DevProblem P, DevRun R, TaskArgs A, int ignore_done) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int n = blockIdx.x, b = blockIdx.y;
  if (ignore_done ? R.status[b] : (R.done[b] | R.status[b])) return;
  DensSmem D = carve_dens(smem_raw, P.dm);
  const int dm = P.dm, sl = P.d, C = P.C, mode = A.mode;
  const int node0 = P.node[n], len = P.node[n + 1] - node0;
  const double Kd = (double)P.K, weight = A.weighted ? Kd / (double)len : 1.0, scale = (double)len / Kd;
  const double dt = P.dt, w = P.ip_w;
  double* u = R.u + ((size_t)b * P.K + node0) * C;
  double2* traj = R.traj + ((size_t)b * P.L + n) * (size_t)R.traj_len * sl;
  // the forward sweep's inverses W_j, re-read by the adjoint sweep over the same controls
  double2* winv = R.winv ? R.winv + ((size_t)b * P.L + n) * (size_t)(R.traj_len - 1) * dm * dm : nullptr;
  const size_t tix = ((size_t)b * P.L + n) * sl;
  const double2* init = R.task_init + tix;
  const double2* targ = R.task_targ + tix;
  double* red = D.lin.red;

  if (mode & (M_ENTRY | M_UPDATE | M_FINAL | M_GRAD)) {
    const bool need_traj = (mode & (M_UPDATE | M_GRAD)) != 0;
    const int iters = (mode & M_UPDATE) ? A.inner : 1;
    for (int it = 0; it < iters; ++it) {
      dens_copy(sl, init, D.S);
      if (need_traj) dens_copy(sl, D.S, traj);
      double pen = 0.0;
      for (int j = 0; j < len; ++j) {
        const double* uj = u + (size_t)j * C;
        dens_inverse(P, b, uj, D);
        if (need_traj && winv) dens_copy(dm * dm, D.W, winv + (size_t)j * dm * dm);
        dens_forward(dm, D, D.S);
        if (need_traj) dens_copy(sl, D.S, traj + (size_t)(j + 1) * sl);
        double sq = 0.0;
        for (int c = 0; c < C; ++c) sq += uj[c] * uj[c];
        pen += (P.alpha[node0 + j] * scale) * sq;
      }
      if (it == 0 && (mode & M_ENTRY)) {
        double t = 0.0;
        for (int i = threadIdx.x; i < sl; i += BT)
          t += A.form == 0 ? cconjmul(targ[i], D.S[i]).x : cabs2(csub(D.S[i], targ[i]));
        t = block_sum(t, red);
        const double payoff = A.form == 0 ? (w * t) : (-0.5 * (w * t));
        if (threadIdx.x == 0) R.entry[(size_t)b * P.L + n] = weight * (payoff - 0.5 * dt * pen);
      }
      if (it == 0 && (mode & M_FINAL)) dens_copy(sl, D.S, R.psi_end + tix);
      if (mode & (M_UPDATE | M_GRAD)) {
        for (int i = threadIdx.x; i < sl; i += BT) D.X[i] = A.form == 0 ? targ[i] : csub(targ[i], D.S[i]);
        __syncthreads();
        for (int j = len - 1; j >= 0; --j) {
          const double* uj = u + (size_t)j * C;
          if (winv) dens_copy(dm * dm, winv + (size_t)j * dm * dm, D.W);
          else dens_inverse(P, b, uj, D);
          mm(dm, D.W, ROW_H, D.X, COL, 1.0, nullptr, 0.0, D.T);                          // r1 = W^dag X
          mm(dm, D.W, ROW_H, traj + (size_t)(j + 1) * sl, COL, 1.0, nullptr, 0.0, D.S);  // r2 = W^dag rho_{j+1}
          const double aj = P.alpha[node0 + j] * scale;
          mm(dm, D.S, COL, D.T, COL_H, 1.0, nullptr, 0.0, D.G);  // M = r2 r1^dag
          double tr[QOC_MAX_DENSITY_CHANNELS];
          dens_traces(P, b, uj, D.G, red, tr);
          if (threadIdx.x == 0)
            for (int c = 0; c < C; ++c) {
              const double uc = uj[c];
              const double gc = -aj * dt * uc + 2.0 * dt * tr[c];
              if (mode & M_GRAD) R.grad[((size_t)b * P.K + node0 + j) * C + c] = gc;
              if (mode & M_UPDATE) u[(size_t)j * C + c] = uc + A.rho * (weight * gc);
            }
          __syncthreads();
          for (int i = threadIdx.x; i < sl; i += BT)  // b = 2 r1 - X
            D.G[i] = cx(2.0 * D.T[i].x - D.X[i].x, 2.0 * D.T[i].y - D.X[i].y);
          __syncthreads();
          mm(dm, D.G, COL, D.W, ROW, 2.0, D.G, -1.0, D.X);  // X_j = 2 b W - b
        }
      }
    }
  }

  const bool do_err = (mode & M_ERROR) != 0, do_asm = (mode & M_ASSEMBLE) != 0, do_lag = (mode & M_LAGGED) != 0;
  // product of the one-step A's (row-major dm x dm; assemble_propagator, 236-249): rides on the
  // residual's forward sweep when both run (same controls, same inverses), else its own sweep
  const bool fuse_asm = do_asm && do_err;
  if (do_asm && !fuse_asm) {
    for (int e = threadIdx.x; e < dm * dm; e += BT) D.S[e] = cx((e / dm) == (e % dm) ? 1.0 : 0.0, 0.0);
    __syncthreads();
    for (int j = 0; j < len; ++j) {
      dens_inverse(P, b, u + (size_t)j * C, D);
      // S (row-major) <- 2 W S - S  : via column-major views of the transposes
      mm(dm, D.S, COL, D.W, COL, 2.0, D.S, -1.0, D.T);  // (2 W S - S)^T = 2 S^T W^T - S^T as column-major
      dens_copy(dm * dm, D.T, D.S);
    }
    for (int e = threadIdx.x; e < dm * dm; e += BT) R.prop[((size_t)b * P.L + n) * (size_t)dm * dm + e] = D.S[e];
  }
  if (do_err || do_lag) {
    // residual: forward at the updated control (trajectory), then the adjoint with its gradient
    if (do_err) {
      dens_copy(sl, init, D.S);
      dens_copy(sl, D.S, traj);
      if (fuse_asm) {  // the product lives in X (free until the adjoint seed), T is its scratch
        for (int e = threadIdx.x; e < dm * dm; e += BT) D.X[e] = cx((e / dm) == (e % dm) ? 1.0 : 0.0, 0.0);
        __syncthreads();
      }
      for (int j = 0; j < len; ++j) {
        dens_inverse(P, b, u + (size_t)j * C, D);
        if (winv) dens_copy(dm * dm, D.W, winv + (size_t)j * dm * dm);
        dens_forward(dm, D, D.S);
        dens_copy(sl, D.S, traj + (size_t)(j + 1) * sl);
        if (fuse_asm) {
          mm(dm, D.X, COL, D.W, COL, 2.0, D.X, -1.0, D.T);  // (2 W Pm - Pm)^T as column-major
          dens_copy(dm * dm, D.T, D.X);
        }
      }
      if (fuse_asm) {
        for (int e = threadIdx.x; e < dm * dm; e += BT) R.prop[((size_t)b * P.L + n) * (size_t)dm * dm + e] = D.X[e];
        __syncthreads();
      }
      for (int i = threadIdx.x; i < sl; i += BT) D.X[i] = A.form == 0 ? targ[i] : csub(targ[i], D.S[i]);
      __syncthreads();
      double err = 0.0;
      for (int j = len - 1; j >= 0; --j) {
        const double* uj = u + (size_t)j * C;
        if (winv) dens_copy(dm * dm, winv + (size_t)j * dm * dm, D.W);
        else dens_inverse(P, b, uj, D);
        mm(dm, D.W, ROW_H, D.X, COL, 1.0, nullptr, 0.0, D.T);
        mm(dm, D.W, ROW_H, traj + (size_t)(j + 1) * sl, COL, 1.0, nullptr, 0.0, D.S);
        const double aj = P.alpha[node0 + j] * scale;
        double sq = 0.0;
        mm(dm, D.S, COL, D.T, COL_H, 1.0, nullptr, 0.0, D.G);  // M = r2 r1^dag
        double tr[QOC_MAX_DENSITY_CHANNELS];
        dens_traces(P, b, uj, D.G, red, tr);
        for (int c = 0; c < C; ++c) {
          const double gc = -aj * dt * uj[c] + 2.0 * dt * tr[c];
          sq += gc * gc;
        }
        err += sqrt(sq);
        for (int i = threadIdx.x; i < sl; i += BT) D.G[i] = cx(2.0 * D.T[i].x - D.X[i].x, 2.0 * D.T[i].y - D.X[i].y);
        __syncthreads();
        mm(dm, D.G, COL, D.W, ROW, 2.0, D.G, -1.0, D.X);
      }
      if (threadIdx.x == 0) R.err[(size_t)b * P.L + n] = err;
    }
    if (do_lag) {  // lagged boundary refresh (ism.cpp:424-459)
      dens_copy(sl, R.psi_nodes + ((size_t)b * (P.L + 1) + n) * sl, D.S);
      for (int j = 0; j < len; ++j) {
        dens_inverse(P, b, u + (size_t)j * C, D);
        dens_forward(dm, D, D.S);
      }
      dens_copy(sl, D.S, R.psi_end + tix);
      dens_copy(sl, R.chi_nodes + ((size_t)b * (P.L + 1) + n + 1) * sl, D.X);
      for (int j = len - 1; j >= 0; --j) {
        dens_inverse(P, b, u + (size_t)j * C, D);
        dens_adjoint(dm, D, D.X);
      }
      dens_copy(sl, D.X, R.chi_start + tix);
    }
  }
}

__global__ void __launch_bounds__(BT) density_horizon_kernel(DevProblem P, DevRun R, int which, int k) {
  if (R.kdev) k = *R.kdev;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int b = blockIdx.x;
  if (R.done[b] || R.status[b]) return;
  DensSmem D = carve_dens(smem_raw, P.dm);
  const int dm = P.dm, sl = P.d, C = P.C;
  const double* u = R.u + (size_t)b * P.K * C;
  const size_t nb = (size_t)b * (P.L + 1) * sl;
  dens_copy(sl, P.init + (size_t)b * sl, D.S);
  if (which == 0) dens_copy(sl, D.S, R.psi_nodes + nb);
  int nxt = 1;
  for (int j = 0; j < P.K; ++j) {
    dens_inverse(P, b, u + (size_t)j * C, D);
    dens_forward(dm, D, D.S);
    if (which == 0 && nxt <= P.L && P.node[nxt] == j + 1) {
      dens_copy(sl, D.S, R.psi_nodes + nb + (size_t)nxt * sl);
      ++nxt;
    }
  }
  if (which == 1) {
    double t = 0.0;
    for (int i = threadIdx.x; i < sl; i += BT) t += cconjmul(P.targ[(size_t)b * sl + i], D.S[i]).x;
    t = block_sum(t, D.lin.red);
    if (threadIdx.x == 0) {
      double pen = 0.0;
      for (int n = 0; n < P.L; ++n) pen += R.pen[(size_t)b * P.L + n];
      R.rec_exact[(size_t)b * R.cap + k] = P.ip_w * t - 0.5 * P.dt * pen;
    }
    return;
  }
  dens_copy(sl, P.targ + (size_t)b * sl, D.X);
  dens_copy(sl, D.X, R.chi_nodes + nb + (size_t)P.L * sl);
  int prev = P.L - 1;
  for (int j = P.K - 1; j >= 0; --j) {
    dens_inverse(P, b, u + (size_t)j * C, D);
    dens_adjoint(dm, D, D.X);
    if (prev >= 0 && P.node[prev] == j) {
      dens_copy(sl, D.X, R.chi_nodes + nb + (size_t)prev * sl);
      --prev;
    }
  }
}


// Boundary chain of the density kind's assembled plan (compose_from_propagators with
// apply_propagator = prop * state * prop^dag, ism.cpp:298-312, propagation.cpp:251-261): the
// tasks' dm x dm products P_n (row-major in R.prop) carry the matrix states across the nodes,
//   rho_{n+1} = P_n rho_n P_n^dag   (blockIdx.y = 0),     X_n = P_n^dag X_{n+1} P_n   (blockIdx.y = 1).
__global__ void __launch_bounds__(BT) density_chain_kernel(DevProblem P, DevRun R) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int b = blockIdx.x;
  if (R.done[b] || R.status[b]) return;
  DensSmem D = carve_dens(smem_raw, P.dm);
  const int dm = P.dm, sl = P.d, L = P.L;
  const size_t nb = (size_t)b * (L + 1) * sl;
  const double2* props = R.prop + (size_t)b * L * (size_t)dm * dm;
  if (blockIdx.y == 0) {
    dens_copy(sl, P.init + (size_t)b * sl, D.S);
    dens_copy(sl, D.S, R.psi_nodes + nb);
    for (int n = 0; n < L; ++n) {
      dens_copy(dm * dm, props + (size_t)n * dm * dm, D.W);
      mm(dm, D.W, ROW, D.S, COL, 1.0, nullptr, 0.0, D.G);    // G = P rho
      mm(dm, D.G, COL, D.W, ROW_H, 1.0, nullptr, 0.0, D.S);  // rho' = G P^dag
      dens_copy(sl, D.S, R.psi_nodes + nb + (size_t)(n + 1) * sl);
    }
  } else {
    dens_copy(sl, P.targ + (size_t)b * sl, D.X);
    dens_copy(sl, D.X, R.chi_nodes + nb + (size_t)L * sl);
    for (int n = L - 1; n >= 0; --n) {
      dens_copy(dm * dm, props + (size_t)n * dm * dm, D.W);
      mm(dm, D.W, ROW_H, D.X, COL, 1.0, nullptr, 0.0, D.G);  // G = P^dag X
      mm(dm, D.G, COL, D.W, ROW, 1.0, nullptr, 0.0, D.X);    // X' = G P
      dens_copy(sl, D.X, R.chi_nodes + nb + (size_t)n * sl);
    }
  }
}

// ---- monotonic slice-rebuilding sweep (monotonic_step, optimizers.cpp:109-213) ----------------
// A CTA per task.  The adjoint nodes chi_j along the previous control go to the task's
// trajectory workspace; the forward sweep then rebuilds the control slice by slice: with
// psi~ = (I + L(u_j))^-1 psi_j and chi~(v) = (I - L(v))^-1 chi_{j+1}, L(v) = i dt/2 H(v), the
// implicit update v (alpha_j - m_pol(v)) = m_mu(v), m_X = Im <chi~| X |psi~>, dH/dv = M + v P, is
// solved by fixed point; a slice whose exact payoff increment comes out negative (or whose
// fixed point is unusable) keeps its previous value and counts as a guard rejection.
// y = W x (plain matvec through the inverse)
__device__ void solve_apply(int d, const double2* W, const double2* x, double2* y) {
  for (int i = threadIdx.x; i < d; i += BT) {
    double2 acc = cx(0.0, 0.0);
    for (int k = 0; k < d; ++k) acc = cfma(W[i * d + k], x[k], acc);
    y[i] = acc;
  }
  __syncthreads();
}

// B = I + s i H(v) inverted in place: pivot-free when dt/2 ||H(v)||_1 < 1 (strict column diagonal
// dominance, where partial pivoting never swaps), else the pivoting path.  One channel.
__device__ void mono_inverse(const DevProblem& P, int b, double v, double shalf, const BigSmem& S) {
  build(P, b, &v, shalf, S.W);
  const double* nb = P.norm1 + (size_t)b * 3;  // ||H0||_1, ||A_0||_1, ||B_0||_1
  double bound = nb[0] + fabs(v) * nb[1];
  if (P.has_quad) bound += 0.5 * v * v * nb[2];
  if (0.5 * P.dt * bound < 1.0) invert_nopivot(P.d, S);
  else invert(P.d, S);
}

__global__ void __launch_bounds__(BT) monotonic_kernel(DevProblem P, DevRun R, int weighted, double fp_tol,
                                                        int fp_max_iter, int* stats) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int n = blockIdx.x, b = blockIdx.y;
  if (R.done[b] | R.status[b]) return;
  (void)weighted;  // the task weight scales the functional, not the slice update
  const BigSmem S = carve(smem_raw, P.d, true);
  const int d = P.d;
  const size_t dd = (size_t)d * d;
  const int node0 = P.node[n], len = P.node[n + 1] - node0;
  const double scale = (double)len / (double)P.K, half = 0.5 * P.dt, dt = P.dt;
  double* u = R.u + (size_t)b * P.K + node0;
  double2* chi = R.traj + ((size_t)b * P.L + n) * (size_t)R.traj_len * d;
  const size_t tix = ((size_t)b * P.L + n) * d;
  const double2* mu_op = P.lin + (size_t)b * dd;                     // M = A_0
  const double2* pol_op = P.has_quad ? P.quad + (size_t)b * dd : nullptr;  // P = B_0
  double2* chin = S.Pm;         // chi_{j+1}
  double2* chit = S.Pm + d;     // chi~(v)
  double2* amu = S.T;           // M psi~
  double2* apol = S.T + d;      // P psi~

  // adjoint nodes along the previous control (optimizers.cpp:145-150)
  copy_vec(d, R.task_targ + tix, S.x);
  for (int i = threadIdx.x; i < d; i += BT) chi[(size_t)len * d + i] = S.x[i];
  for (int j = len - 1; j >= 0; --j) {
    mono_inverse(P, b, u[j], half, S);
    cayley(d, S.W, S.x, S.y, true);
    copy_vec(d, S.y, S.x);
    for (int i = threadIdx.x; i < d; i += BT) chi[(size_t)j * d + i] = S.x[i];
  }
  __syncthreads();

  copy_vec(d, R.task_init + tix, S.x);  // psi_j
  int rejected = 0;
  for (int j = 0; j < len; ++j) {
    const double uj = u[j], aj = P.alpha[node0 + j] * scale;
    mono_inverse(P, b, uj, half, S);
    solve_apply(d, S.W, S.x, S.y);  // psi~
    for (int i = threadIdx.x; i < d; i += BT) {
      double2 a = cx(0.0, 0.0), q = cx(0.0, 0.0);
      for (int k = 0; k < d; ++k) {
        a = cfma(mu_op[(size_t)i * d + k], S.y[k], a);
        if (pol_op) q = cfma(pol_op[(size_t)i * d + k], S.y[k], q);
      }
      amu[i] = a;
      apol[i] = q;
      chin[i] = chi[(size_t)(j + 1) * d + i];
    }
    __syncthreads();
    double m_mu = 0.0, m_pol = 0.0;
    auto pairings_at = [&](double v) {
      mono_inverse(P, b, v, -half, S);  // I - L(v)
      solve_apply(d, S.W, chin, chit);
      double sm = 0.0, sp = 0.0;
      for (int i = threadIdx.x; i < d; i += BT) {
        sm += cconjmul(chit[i], amu[i]).y;
        sp += cconjmul(chit[i], apol[i]).y;
      }
      m_mu = block_sum(sm, S.red);
      m_pol = block_sum(sp, S.red);
    };
    double v = uj;
    bool usable = true;
    for (int it = 0; it < fp_max_iter; ++it) {
      pairings_at(v);
      const double denom = aj - m_pol;
      if (!(fabs(denom) > 1e-14 * (1.0 + aj))) {
        usable = false;
        break;
      }
      const double next = m_mu / denom;
      const bool settled = fabs(next - v) <= fp_tol * (1.0 + fabs(v));
      v = next;
      if (settled) break;
    }
    if (usable && isfinite(v)) {
      pairings_at(v);
      const double gain = dt * (v - uj) * (m_mu + 0.5 * (v + uj) * (m_pol - aj));
      if (!(gain >= 0.0)) usable = false;
    } else {
      usable = false;
    }
    if (!usable) {
      v = uj;
      ++rejected;
    }
    __syncthreads();
    if (threadIdx.x == 0) u[j] = v;
    mono_inverse(P, b, v, half, S);
    cayley(d, S.W, S.x, S.y, false);
    copy_vec(d, S.y, S.x);
  }
  if (threadIdx.x == 0) stats[((size_t)b * P.L + n) * 3] += rejected;
}

}  // namespace

bool dense_big_supported(int d) { return d > 32 && d <= BIG_MAX; }

cudaError_t dense_big_task(const DevProblem& P, const DevRun& R, const TaskArgs& A, int ignore_done, cudaStream_t st) {
  const size_t smem = big_smem(P.d, (A.mode & M_ASSEMBLE) != 0);
  cudaError_t e = cudaFuncSetAttribute(dense_big_task_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  dense_big_task_kernel<<<dim3(P.L, P.B), BT, smem, st>>>(P, R, A, ignore_done);
  return cudaGetLastError();
}

cudaError_t dense_big_horizon(const DevProblem& P, const DevRun& R, int which, int k, cudaStream_t st) {
  const size_t smem = big_smem(P.d, false);
  cudaError_t e =
      cudaFuncSetAttribute(dense_big_horizon_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  dense_big_horizon_kernel<<<P.B, BT, smem, st>>>(P, R, which, k);
  return cudaGetLastError();
}


bool monotonic_supported(const DevProblem& P) { return P.kind == QOC_KIND_DENSE && P.d <= BIG_MAX && P.C == 1; }

cudaError_t monotonic_sweep(const DevProblem& P, const DevRun& R, int weighted, double fp_tol, int fp_max_iter,
                            int* stats, cudaStream_t st) {
  const size_t smem = big_smem(P.d, true);
  cudaError_t e = cudaFuncSetAttribute(monotonic_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  monotonic_kernel<<<dim3(P.L, P.B), BT, smem, st>>>(P, R, weighted, fp_tol, fp_max_iter, stats);
  return cudaGetLastError();
}
}  // namespace qoc

namespace qoc {

bool density_supported(int dm) { return dm >= 1 && dm <= DENS_MAX; }

// QOC_DISABLE=densmma keeps the CUDA-core products (A/B of the tensor-core path)
static cudaError_t dens_mma_switch() {
  static int done = 0;
  if (done) return cudaSuccess;
  done = 1;
  const char* e = std::getenv("QOC_DISABLE");
  const int on = !(e && std::strstr(e, "densmma"));
  return cudaMemcpyToSymbol(c_dens_dmma, &on, sizeof(int));
}

cudaError_t density_task(const DevProblem& P, const DevRun& R, const TaskArgs& A, int ignore_done, cudaStream_t st) {
  if (cudaError_t e0 = dens_mma_switch(); e0 != cudaSuccess) return e0;
  const size_t smem = dens_smem(P.dm);
  cudaError_t e = cudaFuncSetAttribute(density_task_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  density_task_kernel<<<dim3(P.L, P.B), BT, smem, st>>>(P, R, A, ignore_done);
  return cudaGetLastError();
}

cudaError_t density_horizon(const DevProblem& P, const DevRun& R, int which, int k, cudaStream_t st) {
  if (cudaError_t e0 = dens_mma_switch(); e0 != cudaSuccess) return e0;
  const size_t smem = dens_smem(P.dm);
  cudaError_t e =
      cudaFuncSetAttribute(density_horizon_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  density_horizon_kernel<<<P.B, BT, smem, st>>>(P, R, which, k);
  return cudaGetLastError();
}

cudaError_t density_chain(const DevProblem& P, const DevRun& R, cudaStream_t st) {
  if (cudaError_t e0 = dens_mma_switch(); e0 != cudaSuccess) return e0;
  const size_t smem = dens_smem(P.dm);
  cudaError_t e = cudaFuncSetAttribute(density_chain_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  density_chain_kernel<<<dim3(P.B, 2), BT, smem, st>>>(P, R);
  return cudaGetLastError();
}

}  // namespace qoc
