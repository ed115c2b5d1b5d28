// dense.cuh — dense-operator ISM task kernels (QOC_KIND_DENSE, d <= 32), sm_100a.
//
// One lane group of NL = D*G lanes owns one (problem, subinterval) task.  Lane (row, g)
// keeps row `row` of every d x d working matrix in registers, columns j = t*G + g.
// Each grid step forms the Cayley matrix of the reference's Crank-Nicolson step
//     C_j = (I + L_j)^-1 (I - L_j) = 2 B_j^-1 - I,  B_j = I + i dt/2 H(u_j)
// (propagation.cpp:14-16,85-90) by an in-register Gauss-Jordan inversion of B_j, and the
// exact adjoint C_j^dagger = 2 (B_j^dagger)^-1 - I (propagation.cpp:101-106) by inverting
// B_j^dagger.  Every sweep is then a matvec (forward, adjoint) or a matmul (propagator
// assembly, propagation.cpp:236-249) against the inverse -- rectangular work with no
// triangular-solve chains.  Partial pivoting: when dt/2 * ||H(u_j)||_1 < 1, B_j is strictly
// column diagonally dominant and partial pivoting provably never swaps, so the
// pivot-free path is exactly the pivoted algorithm; otherwise the pivoting path runs.
#pragma once

#include "common.cuh"

namespace qoc {

template <int D, int G>
struct DenseCfg {
  static constexpr int NL = D * G;        // lanes per task
  static constexpr int COLS = D / G;      // matrix columns per lane
  static constexpr int TPW = 32 / NL;     // tasks per warp
  // per-task shared memory (double2 units unless noted)
  static constexpr int PIV = 2 * D;       // double-buffered pivot row
  static constexpr int VEC = 2 * D;       // vector broadcast (two vectors)
  static constexpr int MAT = D * D;       // matrix staging (assembly / unscramble)
};

// Per-group view of the shared-memory scratch.
template <int D, int G>
struct DenseScratch {
  double2* piv;   // [2][D]
  double2* vec;   // [2][D]
  double2* matW;  // [D][D]
  double2* matP;  // [D][D]
  int* perm;      // [2][D]
};

template <int D, int G>
struct DenseLane {
  using Cfg = DenseCfg<D, G>;
  static constexpr int NL = Cfg::NL, COLS = Cfg::COLS;
  int row, g;

  __device__ __forceinline__ static int col(int t, int g) { return t * G + g; }

  // B = I + s H(u) (s = +i dt/2 forward, -i dt/2 adjoint) for this lane's row slots.
  // H(u) = H0 + sum u_c A_c + sum (u_c^2/2) B_c  (models.cpp:57-68); operators in smem,
  // zero-padded to D x D, so rows >= d are identity rows.
  __device__ __forceinline__ void build(double2 (&W)[COLS], const double2* ops, int C, int has_quad,
                                        const double* u, double half, bool adj) const {
    const double sh = adj ? -half : half;
#pragma unroll
    for (int t = 0; t < COLS; ++t) {
      const int j = col(t, g);
      double2 h = ops[row * D + j];
      for (int c = 0; c < C; ++c) {
        const double2 a = ops[(1 + c) * D * D + row * D + j];
        h = cx(fma(u[c], a.x, h.x), fma(u[c], a.y, h.y));
      }
      if (has_quad) {
        for (int c = 0; c < C; ++c) {
          const double2 q = ops[(1 + C + c) * D * D + row * D + j];
          const double s = 0.5 * u[c] * u[c];
          h = cx(fma(s, q.x, h.x), fma(s, q.y, h.y));
        }
      }
      // (0 + i sh)(hr + i hi) = (-sh hi, sh hr)
      W[t] = cx((row == j ? 1.0 : 0.0) - sh * h.y, sh * h.x);
    }
  }

  // In-place Gauss-Jordan inversion without row interchanges.
  __device__ __forceinline__ void invert_fast(double2 (&W)[COLS], double2* piv) const {
#pragma unroll
    for (int k = 0; k < D; ++k) {
      const int gk = k % G, tk = k / G;
      const double2 p = shfl(W[tk], k + gk * D, NL);        // pivot W[k][k]
      const double2 f = shfl(W[tk], row + gk * D, NL);      // W[row][k]
      const double2 pinv = crcp(p);
      double2* buf = piv + (k & 1) * D;
      if (row == k) {
#pragma unroll
        for (int t = 0; t < COLS; ++t) {
          const int j = col(t, g);
          buf[j] = (j == k) ? pinv : cmul(W[t], pinv);
        }
      }
      __syncwarp();
#pragma unroll
      for (int t = 0; t < COLS; ++t) {
        const int j = col(t, g);
        const double2 r = buf[j];
        if (row == k) {
          W[t] = r;
        } else if (j == k) {
          W[t] = cneg(cmul(f, r));
        } else {
          W[t] = cfms(f, r, W[t]);
        }
      }
    }
  }

  // Gauss-Jordan with partial pivoting (largest |.| in the column, first row on ties),
  // then the column unscramble of the row interchanges.  Must be called warp-uniformly.
  __device__ void invert_pivot(double2 (&W)[COLS], const DenseScratch<D, G>& s, int lane) const {
    bool any_swap = false;
#pragma unroll 1
    for (int k = 0; k < D; ++k) {
      const int gk = k % G;
      // dynamic slot k / G: extract through a small unrolled select (no local memory)
      double2 wk = W[0];
#pragma unroll
      for (int t = 0; t < COLS; ++t)
        if (t == k / G) wk = W[t];
      double sc = (row >= k) ? cabs2(wk) : -1.0;
      int idx = row;
#pragma unroll
      for (int off = D / 2; off > 0; off >>= 1) {
        const double os = __shfl_xor_sync(0xffffffffu, sc, off, NL);
        const int oi = __shfl_xor_sync(0xffffffffu, idx, off, NL);
        if (os > sc || (os == sc && oi < idx)) {
          sc = os;
          idx = oi;
        }
      }
      const int p = __shfl_sync(0xffffffffu, idx, gk * D, NL);
      if (__any_sync(0xffffffffu, p != k)) {
        any_swap = true;
        const int src = (row == k) ? p : ((row == p) ? k : row);
#pragma unroll
        for (int t = 0; t < COLS; ++t) W[t] = shfl(W[t], src + g * D, NL);
      }
      if (lane == 0) s.perm[k] = p;
      // standard round on the (possibly swapped) rows
      double2 wk2 = W[0];
#pragma unroll
      for (int t = 0; t < COLS; ++t)
        if (t == k / G) wk2 = W[t];
      const double2 pv = shfl(wk2, k + gk * D, NL);
      const double2 f = shfl(wk2, row + gk * D, NL);
      const double2 pinv = crcp(pv);
      double2* buf = s.piv + (k & 1) * D;
      if (row == k) {
#pragma unroll
        for (int t = 0; t < COLS; ++t) {
          const int j = col(t, g);
          buf[j] = (j == k) ? pinv : cmul(W[t], pinv);
        }
      }
      __syncwarp();
#pragma unroll
      for (int t = 0; t < COLS; ++t) {
        const int j = col(t, g);
        const double2 r = buf[j];
        if (row == k) {
          W[t] = r;
        } else if (j == k) {
          W[t] = cneg(cmul(f, r));
        } else {
          W[t] = cfms(f, r, W[t]);
        }
      }
    }
    if (__any_sync(0xffffffffu, any_swap)) {
      __syncwarp();
#pragma unroll
      for (int t = 0; t < COLS; ++t) s.matW[row * D + col(t, g)] = W[t];
      int* sigma = s.perm + D;
      if (lane == 0) {
        for (int j = 0; j < D; ++j) sigma[j] = j;
        for (int k = D - 1; k >= 0; --k) {
          const int q = s.perm[k];
          const int tmp = sigma[k];
          sigma[k] = sigma[q];
          sigma[q] = tmp;
        }
      }
      __syncwarp();
#pragma unroll
      for (int t = 0; t < COLS; ++t) W[t] = s.matW[row * D + sigma[col(t, g)]];
      __syncwarp();
    }
  }

  // y = 2 W x - x  (Cayley step through the inverse); x, y replicated over the g lanes of a row.
  __device__ __forceinline__ double2 cayley_apply(const double2 (&W)[COLS], double2 x, double2* vec) const {
    if (g == 0) vec[row] = x;
    __syncwarp();
    double2 acc = cx(0.0, 0.0);
#pragma unroll
    for (int t = 0; t < COLS; ++t) acc = cfma(W[t], vec[col(t, g)], acc);
    if (G > 1) acc = cadd(acc, shfl_xor(acc, D, NL));
    __syncwarp();
    return cx(2.0 * acc.x - x.x, 2.0 * acc.y - x.y);
  }

  // Two vectors through the same inverse.
  __device__ __forceinline__ void cayley_apply2(const double2 (&W)[COLS], double2& x, double2& y,
                                                double2* vec) const {
    if (g == 0) {
      vec[row] = x;
      vec[D + row] = y;
    }
    __syncwarp();
    double2 a = cx(0.0, 0.0), b = cx(0.0, 0.0);
#pragma unroll
    for (int t = 0; t < COLS; ++t) {
      a = cfma(W[t], vec[col(t, g)], a);
      b = cfma(W[t], vec[D + col(t, g)], b);
    }
    if (G > 1) {
      a = cadd(a, shfl_xor(a, D, NL));
      b = cadd(b, shfl_xor(b, D, NL));
    }
    __syncwarp();
    x = cx(2.0 * a.x - x.x, 2.0 * a.y - x.y);
    y = cx(2.0 * b.x - y.x, 2.0 * b.y - y.y);
  }

  // P <- 2 W P - P  (one step of assemble_propagator)
  __device__ __forceinline__ void cayley_matmul(const double2 (&W)[COLS], double2 (&P)[COLS],
                                                const DenseScratch<D, G>& s, bool live = true) const {
#pragma unroll
    for (int t = 0; t < COLS; ++t) {
      if (G > 1) s.matW[row * D + col(t, g)] = W[t];
      s.matP[row * D + col(t, g)] = P[t];
    }
    __syncwarp();
    double2 acc[COLS];
#pragma unroll
    for (int t = 0; t < COLS; ++t) acc[t] = cx(0.0, 0.0);
    if constexpr (G == 1) {  // the lane's row of the inverse is already in registers
#pragma unroll
      for (int k = 0; k < D; ++k) {
#pragma unroll
        for (int t = 0; t < COLS; ++t) acc[t] = cfma(W[k], s.matP[k * D + t], acc[t]);
      }
    } else {
#pragma unroll 4
      for (int k = 0; k < D; ++k) {
        const double2 w = s.matW[row * D + k];
#pragma unroll
        for (int t = 0; t < COLS; ++t) acc[t] = cfma(w, s.matP[k * D + col(t, g)], acc[t]);
      }
    }
    __syncwarp();
#pragma unroll
    for (int t = 0; t < COLS; ++t)
      if (live) P[t] = cx(2.0 * acc[t].x - P[t].x, 2.0 * acc[t].y - P[t].y);
  }

  // Sum over the D rows of a per-row value (each g block reduces independently).
  __device__ __forceinline__ double2 row_sum(double2 v) const {
#pragma unroll
    for (int off = D / 2; off > 0; off >>= 1) v = cadd(v, shfl_xor(v, off, NL));
    return v;
  }
  __device__ __forceinline__ double row_sum(double v) const {
#pragma unroll
    for (int off = D / 2; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off, NL);
    return v;
  }

  // Im <chi_sum, dH/du_c(u) psi_sum> (unweighted) for channel c; operators in smem.
  __device__ __forceinline__ double grad_term(const double2* ops, int C, int has_quad, int c, double uc,
                                              double2 psi_sum, double2 chi_sum, double2* vec) const {
    if (g == 0) vec[row] = psi_sum;
    __syncwarp();
    double2 acc = cx(0.0, 0.0);
#pragma unroll
    for (int t = 0; t < COLS; ++t) {
      const int j = col(t, g);
      double2 a = ops[(1 + c) * D * D + row * D + j];
      if (has_quad) {
        const double2 q = ops[(1 + C + c) * D * D + row * D + j];
        a = cx(fma(uc, q.x, a.x), fma(uc, q.y, a.y));
      }
      acc = cfma(a, vec[j], acc);
    }
    if (G > 1) acc = cadd(acc, shfl_xor(acc, D, NL));
    __syncwarp();
    const double2 term = cconjmul(chi_sum, acc);
    return row_sum(term).y;
  }
};

template <int D, int G>
using Lane_t = DenseLane<D, G>;

}  // namespace qoc
