// oracle.cpp — CPU restatement of the reference ISM hot path (TEST INFRASTRUCTURE ONLY).
//
// Every function cites the reference file:line whose behaviour it restates.  The reference
// itself cannot be built here (Eigen3 absent), so this is the checker the
// device path is compared against; it is pinned by tests/test_oracle_kats.py.
//
// Deliberate generalisations:
//   F4  the decomposition may be non-uniform (balanced or explicit node indices); with L | K
//       the balanced partition is the reference's Decomposition::uniform.
//   F6  operator classes beyond the reference's dense/condensate models (tridiagonal,
//       bit-flip spin register, cos^2 lattice) plug in behind the same model contract.
#include "oracle.h"

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <complex>
#include <condition_variable>
#include <cstdio>
#include <cstring>
#include <functional>
#include <limits>
#include <memory>
#include <mutex>
#include <numbers>
#include <optional>
#include <random>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

namespace orc {

using cd = std::complex<double>;
using CV = std::vector<cd>;
using RV = std::vector<double>;
constexpr double kNaN = std::numeric_limits<double>::quiet_NaN();

struct InvalidArg : std::invalid_argument {
  using std::invalid_argument::invalid_argument;
};
struct LogicErr : std::logic_error {
  using std::logic_error::logic_error;
};
struct RuntimeErr : std::runtime_error {
  using std::runtime_error::runtime_error;
};

// ---------------------------------------------------------------------------------------
// linalg.cpp:15-63,99-100 — unitary DFT: radix-2 iterative transform for powers of two
// (twiddles from std::polar inside the butterfly loop), direct O(n^2) sum otherwise.
// ---------------------------------------------------------------------------------------
static bool pow2(size_t n) { return n > 0 && (n & (n - 1)) == 0; }

static void fft_inplace(CV& a, int sign) {
  const size_t n = a.size();
  size_t j = 0;
  for (size_t i = 1; i < n; ++i) {  // bit-reversal permutation
    size_t bit = n >> 1;
    while (j & bit) {
      j ^= bit;
      bit >>= 1;
    }
    j ^= bit;
    if (i < j) std::swap(a[i], a[j]);
  }
  for (size_t len = 2; len <= n; len <<= 1) {
    const double ang = sign * 2.0 * std::numbers::pi / static_cast<double>(len);
    const size_t half = len / 2;
    for (size_t base = 0; base < n; base += len) {
      for (size_t k = 0; k < half; ++k) {
        const cd w = std::polar(1.0, ang * static_cast<double>(k));
        const cd lo = a[base + k];
        const cd hi = w * a[base + k + half];
        a[base + k] = lo + hi;
        a[base + k + half] = lo - hi;
      }
    }
  }
}

static CV dft_sum(const CV& x, int sign) {
  const size_t n = x.size();
  CV out(n);
  for (size_t k = 0; k < n; ++k) {
    cd acc = 0.0;
    for (size_t m = 0; m < n; ++m) {
      const long long r = (static_cast<long long>(m) * static_cast<long long>(k)) %
                          static_cast<long long>(n);
      acc += x[m] * std::polar(1.0, sign * 2.0 * std::numbers::pi * static_cast<double>(r) /
                                        static_cast<double>(n));
    }
    out[k] = acc;
  }
  return out;
}

static CV unitary_dft(const CV& x, int sign) {
  if (x.empty()) throw InvalidArg("dft: empty input");
  CV out;
  if (pow2(x.size())) {
    out = x;
    fft_inplace(out, sign);
  } else {
    out = dft_sum(x, sign);
  }
  const double s = std::sqrt(static_cast<double>(x.size()));
  for (cd& v : out) v /= s;
  return out;
}
static CV dft(const CV& x) { return unitary_dft(x, -1); }
static CV idft(const CV& x) { return unitary_dft(x, +1); }

// ---------------------------------------------------------------------------------------
// Dense complex matrices (column-major, like Eigen::MatrixXcd) and a partial-pivot LU with
// Eigen::PartialPivLU semantics: pivot = first row of largest |a_ik| in the column.
// Used for every Cayley solve of the reference arithmetic (propagation.cpp:85-106,236-249).
// ---------------------------------------------------------------------------------------
struct CMat {
  int rows = 0, cols = 0;
  CV v;
  CMat() = default;
  CMat(int r, int c) : rows(r), cols(c), v(static_cast<size_t>(r) * c) {}
  cd& operator()(int i, int j) { return v[static_cast<size_t>(i) + static_cast<size_t>(j) * rows]; }
  const cd& operator()(int i, int j) const {
    return v[static_cast<size_t>(i) + static_cast<size_t>(j) * rows];
  }
  static CMat identity(int n) {
    CMat m(n, n);
    for (int i = 0; i < n; ++i) m(i, i) = 1.0;
    return m;
  }
};

static CMat matmul(const CMat& a, const CMat& b) {
  CMat out(a.rows, b.cols);
  for (int j = 0; j < b.cols; ++j)
    for (int k = 0; k < a.cols; ++k) {
      const cd bk = b(k, j);
      for (int i = 0; i < a.rows; ++i) out(i, j) += a(i, k) * bk;
    }
  return out;
}

static CMat adjoint(const CMat& a) {
  CMat out(a.cols, a.rows);
  for (int j = 0; j < a.cols; ++j)
    for (int i = 0; i < a.rows; ++i) out(j, i) = std::conj(a(i, j));
  return out;
}

struct PivLU {
  int n = 0;
  CMat lu;
  std::vector<int> perm;  // row transpositions, Eigen style
  explicit PivLU(const CMat& a) : n(a.rows), lu(a), perm(static_cast<size_t>(a.rows)) {
    for (int k = 0; k < n; ++k) {
      int p = k;
      double best = std::abs(lu(k, k));
      for (int i = k + 1; i < n; ++i) {
        const double s = std::abs(lu(i, k));
        if (s > best) {
          best = s;
          p = i;
        }
      }
      perm[static_cast<size_t>(k)] = p;
      if (p != k)
        for (int j = 0; j < n; ++j) std::swap(lu(k, j), lu(p, j));
      const cd piv = lu(k, k);
      if (piv == cd(0.0, 0.0)) continue;  // Eigen leaves the column; solve yields inf/nan
      for (int i = k + 1; i < n; ++i) lu(i, k) /= piv;
      for (int j = k + 1; j < n; ++j) {
        const cd ukj = lu(k, j);
        for (int i = k + 1; i < n; ++i) lu(i, j) -= lu(i, k) * ukj;
      }
    }
  }
  void solve_inplace(CMat& b) const {
    for (int k = 0; k < n; ++k) {
      const int p = perm[static_cast<size_t>(k)];
      if (p != k)
        for (int j = 0; j < b.cols; ++j) std::swap(b(k, j), b(p, j));
    }
    for (int j = 0; j < b.cols; ++j) {
      for (int k = 0; k < n; ++k) {
        const cd y = b(k, j);
        for (int i = k + 1; i < n; ++i) b(i, j) -= lu(i, k) * y;
      }
      for (int k = n - 1; k >= 0; --k) {
        b(k, j) /= lu(k, k);
        const cd x = b(k, j);
        for (int i = 0; i < k; ++i) b(i, j) -= lu(i, k) * x;
      }
    }
  }
};

// ---------------------------------------------------------------------------------------
// Models: the HamiltonianModel plugin contract (propagation.hpp:20-38).
// ---------------------------------------------------------------------------------------
struct Model {
  int kind = 0, d = 0, C = 0;
  double w = 1.0;  // ip_weight
  virtual ~Model() = default;
  virtual bool linear() const { return true; }
  // Cayley step on the m columns of X (d x m): forward (I+L)X' = (I-L)X, or the exact
  // adjoint (I-L)X' = (I+L)X, with L = i dt/2 H(u) (propagation.cpp:85-90,101-106,236-249).
  virtual void cayley(const double* u, double dt, CMat& X, bool adjoint) const = 0;
  // y = dH/du_c (u) x  (models.cpp:70-75 and analogues)
  virtual void dH(int c, const double* u, const cd* x, cd* y) const = 0;
};

// DenseModel (models.cpp:45-75) with reference arithmetic: H(u) rebuilt densely every call,
// one partial-pivot LU per step.
struct DenseM : Model {
  CMat h0;
  std::vector<CMat> lin, quad;
  CMat hamiltonian(const double* u) const {  // models.cpp:57-68
    CMat h = h0;
    for (int c = 0; c < C; ++c)
      for (size_t e = 0; e < h.v.size(); ++e) h.v[e] += u[c] * lin[static_cast<size_t>(c)].v[e];
    for (size_t c = 0; c < quad.size(); ++c) {
      const double uc = u[c];
      const double s = 0.5 * uc * uc;
      for (size_t e = 0; e < h.v.size(); ++e) h.v[e] += s * quad[c].v[e];
    }
    return h;
  }
  void cayley(const double* u, double dt, CMat& X, bool adj) const override {
    const CMat h = hamiltonian(u);
    const cd half(0.0, 0.5 * dt);  // half_step_matrix, propagation.cpp:14-16
    CMat plus = CMat::identity(d), minus = CMat::identity(d);
    for (size_t e = 0; e < h.v.size(); ++e) {
      const cd l = half * h.v[e];
      plus.v[e] += l;
      minus.v[e] -= l;
    }
    // forward: solve plus X' = minus X ; adjoint: solve minus X' = plus X
    CMat rhs = matmul(adj ? plus : minus, X);
    PivLU lu(adj ? minus : plus);
    lu.solve_inplace(rhs);
    X = std::move(rhs);
  }
  void dH(int c, const double* u, const cd* x, cd* y) const override {
    const CMat& a = lin[static_cast<size_t>(c)];
    for (int i = 0; i < d; ++i) y[i] = 0.0;
    for (int k = 0; k < d; ++k)
      for (int i = 0; i < d; ++i) {
        cd m = a(i, k);
        if (!quad.empty()) m += u[c] * quad[static_cast<size_t>(c)](i, k);
        y[i] += m * x[k];
      }
  }
};

// Density-matrix kind: DenseModel with PropagatorKind::cn_conjugation (models.cpp:45-75,
// propagation.cpp:92-129).  A state is a dm x dm matrix held as a dm^2 column-major vector
// (Model::d = dm^2), stepped rho' = A rho A^dag with A = (I+L)^-1 (I-L); the adjoint is
// X' = A^dag X A.  The same LU solves, in the same order, as the reference.
struct ConjM : Model {
  int dm = 0;
  CMat h0;
  std::vector<CMat> lin, quad;
  CMat hamiltonian(const double* u) const {  // models.cpp:57-68
    CMat h = h0;
    for (int c = 0; c < C; ++c)
      for (size_t e = 0; e < h.v.size(); ++e) h.v[e] += u[c] * lin[static_cast<size_t>(c)].v[e];
    for (size_t c = 0; c < quad.size(); ++c) {
      const double s = 0.5 * u[c] * u[c];
      for (size_t e = 0; e < h.v.size(); ++e) h.v[e] += s * quad[c].v[e];
    }
    return h;
  }
  CMat derivative(int c, const double* u) const {  // models.cpp:70-75
    CMat a = lin[static_cast<size_t>(c)];
    if (!quad.empty())
      for (size_t e = 0; e < a.v.size(); ++e) a.v[e] += u[c] * quad[static_cast<size_t>(c)].v[e];
    return a;
  }
  void plus_minus(const double* u, double dt, CMat& plus, CMat& minus) const {
    const CMat h = hamiltonian(u);
    const cd half(0.0, 0.5 * dt);  // half_step_matrix, propagation.cpp:14-16
    plus = CMat::identity(dm);
    minus = CMat::identity(dm);
    for (size_t e = 0; e < h.v.size(); ++e) {
      plus.v[e] += half * h.v[e];
      minus.v[e] -= half * h.v[e];
    }
  }
  static CMat mat_of(const cd* x, int n) {
    CMat r(n, n);
    for (size_t e = 0; e < r.v.size(); ++e) r.v[e] = x[e];
    return r;
  }
  void cayley(const double* u, double dt, CMat& X, bool adj) const override {
    CMat plus, minus;
    plus_minus(u, dt, plus, minus);
    const PivLU lu(adj ? minus : plus);
    for (int col = 0; col < X.cols; ++col) {
      cd* x = &X(0, col);
      const CMat r = mat_of(x, dm);
      CMat out;
      if (!adj) {  // cn_conjugation_step (92-99): g = A rho, out = (A g^dag)^dag
        CMat g = matmul(minus, r);
        lu.solve_inplace(g);
        CMat t = matmul(minus, adjoint(g));
        lu.solve_inplace(t);
        out = adjoint(t);
      } else {  // cn_conjugation_adjoint_step (108-115): b = A^dag X, out = (A^dag b^dag)^dag
        CMat s0 = r;
        lu.solve_inplace(s0);
        const CMat b = matmul(plus, s0);
        CMat t = adjoint(b);
        lu.solve_inplace(t);
        out = adjoint(matmul(plus, t));
      }
      for (size_t e = 0; e < out.v.size(); ++e) x[e] = out.v[e];
    }
  }
  // cn_conjugation_backward_stage (117-129) and the gradient row of objective.cpp:61-71:
  // chi <- X_j; g[c] = 2 dt Im tr(r1^dag dH_c r2), r1 = (I-L)^-1 X_{j+1}, r2 = (I-L)^-1 rho_{j+1}
  void backward(const double* u, double dt, CV& chi, const CV& rho_next, double* trace_im) const {
    CMat plus, minus;
    plus_minus(u, dt, plus, minus);
    const PivLU lm(minus);
    CMat r1 = mat_of(chi.data(), dm), r2 = mat_of(rho_next.data(), dm);
    lm.solve_inplace(r1);
    lm.solve_inplace(r2);
    const CMat b = matmul(plus, r1);
    CMat t = adjoint(b);
    lm.solve_inplace(t);
    const CMat xj = adjoint(matmul(plus, t));
    chi = xj.v;
    const CMat r1h = adjoint(r1);
    for (int c = 0; c < C; ++c) {
      const CMat m = matmul(matmul(r1h, derivative(c, u)), r2);
      cd tr = 0.0;
      for (int i = 0; i < dm; ++i) tr += m(i, i);
      trace_im[c] = tr.imag();
    }
  }
  CMat assemble_dm(const double* u, int len, double dt) const {  // propagation.cpp:236-249
    CMat prod = CMat::identity(dm);
    for (int j = 0; j < len; ++j) {
      CMat plus, minus;
      plus_minus(u + static_cast<size_t>(j) * C, dt, plus, minus);
      CMat rhs = matmul(minus, prod);
      PivLU(plus).solve_inplace(rhs);
      prod = std::move(rhs);
    }
    return prod;
  }
  void dH(int, const double*, const cd*, cd*) const override {
    throw LogicErr("the conjugation kind has its own gradient row");
  }
};

// Hermitian tridiagonal operators, Thomas elimination.  I + i dt/2 H is strictly diagonally
// dominant for the rotor (|diag| >= 1 > off-diagonal), so Eigen's partial pivoting never
// swaps and the LU it forms is exactly this elimination; a swap is detected and refused.
struct TriM : Model {
  // op 0 = H0, 1..C = A_c, C+1..2C = B_c; diag real, sub = entry (j+1, j)
  std::vector<RV> diag;
  std::vector<CV> sub;
  bool has_quad = false;
  void bands(const double* u, RV& dg, CV& sb) const {
    dg = diag[0];
    sb = sub[0];
    for (int c = 0; c < C; ++c) {
      for (int i = 0; i < d; ++i) dg[static_cast<size_t>(i)] += u[c] * diag[1 + c][i];
      for (int i = 0; i + 1 < d; ++i) sb[static_cast<size_t>(i)] += u[c] * sub[1 + c][i];
    }
    if (has_quad)
      for (int c = 0; c < C; ++c) {
        const double s = 0.5 * u[c] * u[c];
        for (int i = 0; i < d; ++i) dg[static_cast<size_t>(i)] += s * diag[1 + C + c][i];
        for (int i = 0; i + 1 < d; ++i) sb[static_cast<size_t>(i)] += s * sub[1 + C + c][i];
      }
  }
  void cayley(const double* u, double dt, CMat& X, bool adj) const override {
    RV dg;
    CV sb;
    bands(u, dg, sb);
    const double h = 0.5 * dt;
    const cd s = adj ? cd(0.0, -h) : cd(0.0, h);  // solve matrix  I + s H ; rhs matrix I - s H
    // matrix entries: a_i (sub, row i col i-1) = s*sb[i-1]; b_i = 1 + s*dg[i]; c_i (super,
    // row i col i+1) = s*conj(sb[i])
    CV a(static_cast<size_t>(d)), b(static_cast<size_t>(d)), c(static_cast<size_t>(d));
    CV ra(static_cast<size_t>(d)), rb(static_cast<size_t>(d)), rc(static_cast<size_t>(d));
    for (int i = 0; i < d; ++i) {
      const cd hd = dg[static_cast<size_t>(i)];
      b[i] = 1.0 + s * hd;
      rb[i] = 1.0 - s * hd;
      if (i > 0) {
        a[i] = s * sb[i - 1];
        ra[i] = -(s * sb[i - 1]);
      }
      if (i + 1 < d) {
        c[i] = s * std::conj(sb[i]);
        rc[i] = -(s * std::conj(sb[i]));
      }
    }
    // LU (no pivot): u_0 = b_0; l_i = a_i / u_{i-1}; u_i = b_i - l_i c_{i-1}
    CV uu(static_cast<size_t>(d)), ll(static_cast<size_t>(d));
    uu[0] = b[0];
    for (int i = 1; i < d; ++i) {
      if (std::abs(a[i]) > std::abs(uu[i - 1]))
        throw RuntimeErr("tridiagonal solve would pivot; use the reference arithmetic");
      ll[i] = a[i] / uu[i - 1];
      uu[i] = b[i] - ll[i] * c[i - 1];
    }
    for (int col = 0; col < X.cols; ++col) {
      CV r(static_cast<size_t>(d));
      for (int i = 0; i < d; ++i) {
        cd acc = 0.0;
        if (i > 0) acc += ra[i] * X(i - 1, col);
        acc += rb[i] * X(i, col);
        if (i + 1 < d) acc += rc[i] * X(i + 1, col);
        r[i] = acc;
      }
      for (int i = 1; i < d; ++i) r[i] -= ll[i] * r[i - 1];
      for (int i = d - 1; i >= 0; --i) {
        r[i] /= uu[i];
        if (i > 0) r[i - 1] -= c[i - 1] * r[i];
      }
      for (int i = 0; i < d; ++i) X(i, col) = r[i];
    }
  }
  void dH(int c, const double* u, const cd* x, cd* y) const override {
    for (int i = 0; i < d; ++i) {
      double dg = diag[1 + c][i];
      if (has_quad) dg += u[c] * diag[1 + C + c][i];
      cd acc = dg * x[i];
      if (i > 0) {
        cd s = sub[1 + c][i - 1];
        if (has_quad) s += u[c] * sub[1 + C + c][i - 1];
        acc += s * x[i - 1];
      }
      if (i + 1 < d) {
        cd s = sub[1 + c][i];
        if (has_quad) s += u[c] * sub[1 + C + c][i];
        acc += std::conj(s) * x[i + 1];
      }
      y[i] = acc;
    }
  }
};

// Bit-flip spin register: H(u) = diag(h0) + sum_c u_c sum_i coef[c][i] sigma^{axis_c}_i.
// Structured Cayley solve: Jacobi-preconditioned fixed point
//   y <- (1 + s D)^-1 (r - s V(u) y),  s = +-i dt/2,
// iterated until the update is below 2^-53 of |y| (the Neumann series of (I + iA)^-1).
struct BitM : Model {
  int nspins = 0;
  RV diagH;
  std::vector<int> axis;
  std::vector<RV> coef;
  void offdiag(const double* u, const cd* x, cd* y) const {  // y = V(u) x
    for (int s = 0; s < d; ++s) y[s] = 0.0;
    for (int c = 0; c < C; ++c) {
      for (int i = 0; i < nspins; ++i) {
        const double g = u[c] * coef[static_cast<size_t>(c)][static_cast<size_t>(i)];
        const int mask = 1 << (nspins - 1 - i);
        for (int s = 0; s < d; ++s) {
          const cd v = x[s ^ mask];
          if (axis[static_cast<size_t>(c)] == 0) {
            y[s] += g * v;
          } else {  // sigma_y: <s|sy|s^m> = +i if bit of s is 1, -i if 0
            const bool one = (s & mask) != 0;
            y[s] += g * (one ? cd(-v.imag(), v.real()) : cd(v.imag(), -v.real()));
          }
        }
      }
    }
  }
  void cayley(const double* u, double dt, CMat& X, bool adj) const override {
    const double h = 0.5 * dt;
    const cd s = adj ? cd(0.0, -h) : cd(0.0, h);
    CV Vx(static_cast<size_t>(d)), r(static_cast<size_t>(d)), y(static_cast<size_t>(d)),
        yn(static_cast<size_t>(d)), Vy(static_cast<size_t>(d));
    for (int col = 0; col < X.cols; ++col) {
      cd* x = &X(0, col);
      offdiag(u, x, Vx.data());
      for (int i = 0; i < d; ++i) r[i] = x[i] - s * (diagH[i] * x[i] + Vx[i]);
      for (int i = 0; i < d; ++i) y[i] = r[i] / (1.0 + s * diagH[i]);
      for (int it = 0; it < 200; ++it) {
        offdiag(u, y.data(), Vy.data());
        double dmax = 0.0, ymax = 0.0;
        for (int i = 0; i < d; ++i) {
          yn[i] = (r[i] - s * Vy[i]) / (1.0 + s * diagH[i]);
          dmax = std::max(dmax, std::abs(yn[i] - y[i]));
          ymax = std::max(ymax, std::abs(yn[i]));
        }
        y.swap(yn);
        if (dmax <= 0x1p-53 * ymax) break;
        if (it == 199) throw RuntimeErr("bit-flip Cayley solve did not converge");
      }
      for (int i = 0; i < d; ++i) x[i] = y[i];
    }
  }
  void dH(int c, const double*, const cd* x, cd* y) const override {
    RV unit(static_cast<size_t>(C), 0.0);  // H is affine in u: dH/du_c = channel operator
    unit[static_cast<size_t>(c)] = 1.0;
    offdiag(unit.data(), x, y);
  }
  DenseM densify() const {  // reference arithmetic: the same operators as dense matrices
    DenseM m;
    m.kind = kind;
    m.d = d;
    m.C = C;
    m.w = w;
    m.h0 = CMat(d, d);
    for (int i = 0; i < d; ++i) m.h0(i, i) = diagH[i];
    for (int c = 0; c < C; ++c) {
      CMat a(d, d);
      RV uu(static_cast<size_t>(C), 0.0);
      uu[static_cast<size_t>(c)] = 1.0;
      CV e(static_cast<size_t>(d)), col(static_cast<size_t>(d));
      for (int k = 0; k < d; ++k) {
        std::fill(e.begin(), e.end(), cd(0.0));
        e[k] = 1.0;
        offdiag(uu.data(), e.data(), col.data());
        for (int i = 0; i < d; ++i) a(i, k) = col[i];
      }
      m.lin.push_back(a);
    }
    return m;
  }
};

// Split-step condensate (propagation.cpp:27-53,131-170; models.cpp:77-127).
struct StrangM : Model {
  RV kin, x;
  int pot = 0;
  double pp[4] = {0, 0, 0, 0};
  double kappa = 0.0;
  // QOC_POT_BASIS: V = sum_m a_m(x) f_m(u) -- a caller-supplied potential()/potential_derivative()
  // of the HamiltonianModel plugin (propagation.hpp:35-36) in separable form
  std::vector<RV> basis;
  std::vector<int> term_type;
  RV term_param;
  double term_value(size_t m2, double u0, bool deriv) const {
    const double q = term_param[m2];
    if (term_type[m2] == QOC_TERM_POWER) {
      const int k = static_cast<int>(q);
      if (deriv) return k > 0 ? k * std::pow(u0, k - 1) : 0.0;
      return std::pow(u0, k);
    }
    if (term_type[m2] == QOC_TERM_COS) return deriv ? -q * std::sin(q * u0) : std::cos(q * u0);
    return deriv ? q * std::cos(q * u0) : std::sin(q * u0);
  }
  RV basis_sum(double u0, bool deriv) const {
    RV v(static_cast<size_t>(d), 0.0);
    for (size_t m2 = 0; m2 < basis.size(); ++m2) {
      const double f = term_value(m2, u0, deriv);
      for (int i = 0; i < d; ++i) v[i] += basis[m2][i] * f;
    }
    return v;
  }
  bool linear() const override { return false; }
  void cayley(const double*, double, CMat&, bool) const override {
    throw LogicErr("no dense one-step matrices to assemble for this propagator kind");
  }
  void dH(int, const double*, const cd*, cd*) const override {
    throw LogicErr("model does not provide dense control derivatives");
  }
  RV potential(const double* u) const {
    if (pot == QOC_POT_BASIS) return basis_sum(u[0], false);
    RV v(static_cast<size_t>(d));
    if (pot == QOC_POT_TRAP) {  // models.cpp:95-110
      const double ld = u[0] * pp[0];
      for (int i = 0; i < d; ++i) {
        const double ax = std::abs(x[i]);
        if (ax > 0.25 * ld) {
          const double r = ax - 0.5 * ld;
          v[i] = 0.5 * r * r;
        } else {
          v[i] = 0.5 * (0.125 * ld * ld - x[i] * x[i]);
        }
      }
    } else {  // cos^2 lattice + harmonic trap (BASELINE config 4)
      for (int i = 0; i < d; ++i) {
        const double cs = std::cos(pp[2] * (x[i] - u[0]));
        v[i] = 0.5 * pp[0] * x[i] * x[i] + pp[1] * cs * cs;
      }
    }
    return v;
  }
  RV potential_derivative(const double* u) const {
    if (pot == QOC_POT_BASIS) return basis_sum(u[0], true);
    RV dv(static_cast<size_t>(d));
    if (pot == QOC_POT_TRAP) {  // models.cpp:112-127
      const double l = u[0], dd = pp[0], ld = l * dd;
      for (int i = 0; i < d; ++i) {
        const double ax = std::abs(x[i]);
        dv[i] = (ax > 0.25 * ld) ? -0.5 * dd * (ax - 0.5 * ld) : 0.125 * l * dd * dd;
      }
    } else {
      for (int i = 0; i < d; ++i) dv[i] = pp[1] * pp[2] * std::sin(2.0 * pp[2] * (x[i] - u[0]));
    }
    return dv;
  }
  CV half_phase(double dt, bool adj) const {  // kinetic_half_phase, propagation.cpp:33-40
    CV ph(static_cast<size_t>(d));
    const double sign = adj ? 1.0 : -1.0;
    for (int i = 0; i < d; ++i) ph[i] = std::polar(1.0, sign * 0.5 * dt * kin[i]);
    return ph;
  }
  static CV spectral(const CV& psi, const CV& ph) {  // apply_spectral_phase, 27-31
    CV hat = dft(psi);
    for (size_t i = 0; i < hat.size(); ++i) hat[i] *= ph[i];
    return idft(hat);
  }
  void midpoint(const double* u, double dt, const CV& psi, CV& psi_a, RV& wv) const {
    psi_a = spectral(psi, half_phase(dt, false));  // strang_midpoint, 47-53
    wv = potential(u);
    for (int i = 0; i < d; ++i) wv[i] += kappa * std::norm(psi_a[i]);
  }
  CV step(const double* u, double dt, const CV& psi) const {  // strang_step, 131-139
    CV pa;
    RV wv;
    midpoint(u, dt, psi, pa, wv);
    CV pb(static_cast<size_t>(d));
    for (int i = 0; i < d; ++i) pb[i] = std::polar(1.0, -dt * wv[i]) * pa[i];
    return spectral(pb, half_phase(dt, false));
  }
  // strang_backward_stage, 146-170
  void backward(const double* u, double dt, const CV& psi_j, const CV& chi_next, bool naive,
                CV& chi_j, CV& psi_b, CV& chi_b) const {
    CV pa;
    RV wv;
    midpoint(u, dt, psi_j, pa, wv);
    const CV adj = half_phase(dt, true);
    psi_b.assign(static_cast<size_t>(d), cd(0.0));
    chi_b = spectral(chi_next, adj);
    CV chi_a(static_cast<size_t>(d));
    for (int i = 0; i < d; ++i) {
      const cd flow = std::polar(1.0, -dt * wv[i]);
      psi_b[i] = flow * pa[i];
      if (naive) {
        chi_a[i] = std::conj(flow) * chi_b[i];
      } else {
        const double dens = std::norm(pa[i]);
        const cd p = flow * (1.0 - cd(0.0, dt * kappa) * dens);
        const cd q = -cd(0.0, dt * kappa) * flow * pa[i] * pa[i];
        chi_a[i] = std::conj(p) * chi_b[i] + q * std::conj(chi_b[i]);
      }
    }
    chi_j = spectral(chi_a, adj);
  }
};

// ---------------------------------------------------------------------------------------
// Problem view of one batch member.
// ---------------------------------------------------------------------------------------
struct Prob {
  std::shared_ptr<Model> m;
  int d = 0, C = 0, K = 0;
  double t0 = 0.0, dt = 0.0;
  CV init, targ;
  RV alpha;
};

static CV load_cvec(const double* p, size_t n) {
  CV v(n);
  for (size_t i = 0; i < n; ++i) v[i] = cd(p[2 * i], p[2 * i + 1]);
  return v;
}
static CMat load_cmat(const double* p, int n) {
  CMat m(n, n);
  for (size_t e = 0; e < m.v.size(); ++e) m.v[e] = cd(p[2 * e], p[2 * e + 1]);
  return m;
}

static void validate(const qoc_problem_v1* p) {
  if (!p) throw InvalidArg("problem has no model");
  if (p->abi_version != QOC_ABI_VERSION) throw InvalidArg("problem ABI version mismatch");
  if (p->dim < 1 || p->channels < 1 || p->steps < 1 || p->batch < 1)
    throw InvalidArg("dim, channels, steps and batch must be positive");
  if (!(p->dt > 0.0)) throw InvalidArg("TimeGrid: dt must be positive");
  if (!p->initial || !p->target) throw InvalidArg("initial and target states are required");
}

static Prob make_prob(const qoc_problem_v1* p, int b, int arith) {
  validate(p);
  Prob P;
  const int d = p->dim, C = p->channels;
  const int slen = p->kind == QOC_KIND_DENSITY ? d * d : d;  // state length
  P.d = slen;
  P.C = C;
  P.K = p->steps;
  P.t0 = p->t_start;
  P.dt = p->dt;
  const size_t dd = static_cast<size_t>(d) * d;
  switch (p->kind) {
    case QOC_KIND_DENSE: {
      if (!p->h0 || !p->linear) throw InvalidArg("dense model needs h0 and linear operators");
      auto m = std::make_shared<DenseM>();
      m->h0 = load_cmat(p->h0 + 2 * dd * b, d);
      auto hermitian = [&](const CMat& a, const char* what) {  // models.cpp:20-25
        double scale = 1.0, defect = 0.0;
        for (int j = 0; j < d; ++j)
          for (int i = 0; i < d; ++i) {
            scale = std::max(scale, std::abs(a(i, j)));
            defect = std::max(defect, std::abs(a(i, j) - std::conj(a(j, i))));
          }
        if (defect > 1e-10 * scale) throw InvalidArg(std::string(what) + " must be Hermitian");
      };
      for (int c = 0; c < C; ++c) m->lin.push_back(load_cmat(p->linear + 2 * dd * (static_cast<size_t>(b) * C + c), d));
      if (p->quadratic)
        for (int c = 0; c < C; ++c)
          m->quad.push_back(load_cmat(p->quadratic + 2 * dd * (static_cast<size_t>(b) * C + c), d));
      hermitian(m->h0, "free Hamiltonian");
      for (const CMat& a : m->lin) hermitian(a, "control operator");
      for (const CMat& a : m->quad) hermitian(a, "quadratic operator");
      P.m = m;
      break;
    }
    case QOC_KIND_DENSITY: {
      if (!p->h0 || !p->linear) throw InvalidArg("density model needs h0 and linear operators");
      auto m = std::make_shared<ConjM>();
      m->dm = d;
      m->h0 = load_cmat(p->h0 + 2 * dd * b, d);
      for (int c = 0; c < C; ++c) m->lin.push_back(load_cmat(p->linear + 2 * dd * (static_cast<size_t>(b) * C + c), d));
      if (p->quadratic)
        for (int c = 0; c < C; ++c)
          m->quad.push_back(load_cmat(p->quadratic + 2 * dd * (static_cast<size_t>(b) * C + c), d));
      P.m = m;
      break;
    }
    case QOC_KIND_TRIDIAG: {
      if (!p->tri_diag || !p->tri_sub) throw InvalidArg("tridiagonal model needs bands");
      const int nops = 1 + C + (p->tri_has_quadratic ? C : 0);
      auto t = std::make_shared<TriM>();
      t->has_quad = p->tri_has_quadratic != 0;
      for (int o = 0; o < nops; ++o) {
        const double* dg = p->tri_diag + (static_cast<size_t>(b) * nops + o) * d;
        const double* sb = p->tri_sub + 2 * (static_cast<size_t>(b) * nops + o) * (d - 1);
        t->diag.emplace_back(dg, dg + d);
        t->sub.push_back(load_cvec(sb, static_cast<size_t>(d - 1)));
      }
      t->kind = p->kind;
      t->d = d;
      t->C = C;
      if (arith == ORACLE_ARITH_STRUCTURED) {
        P.m = t;
      } else {  // densify: DenseModel over the same matrices
        auto m = std::make_shared<DenseM>();
        auto dense = [&](int o) {
          CMat a(d, d);
          for (int i = 0; i < d; ++i) a(i, i) = t->diag[static_cast<size_t>(o)][static_cast<size_t>(i)];
          for (int i = 0; i + 1 < d; ++i) {
            a(i + 1, i) = t->sub[static_cast<size_t>(o)][static_cast<size_t>(i)];
            a(i, i + 1) = std::conj(t->sub[static_cast<size_t>(o)][static_cast<size_t>(i)]);
          }
          return a;
        };
        m->h0 = dense(0);
        for (int c = 0; c < C; ++c) m->lin.push_back(dense(1 + c));
        if (t->has_quad)
          for (int c = 0; c < C; ++c) m->quad.push_back(dense(1 + C + c));
        P.m = m;
      }
      break;
    }
    case QOC_KIND_BITFLIP: {
      if (!p->h0 || !p->bf_axis || !p->bf_coef) throw InvalidArg("bit-flip model needs h0/axis/coef");
      if (p->nspins < 1 || (1 << p->nspins) != d) throw InvalidArg("bit-flip dim must be 2^nspins");
      auto bm = std::make_shared<BitM>();
      bm->kind = p->kind;
      bm->d = d;
      bm->C = C;
      bm->nspins = p->nspins;
      bm->diagH.assign(p->h0 + static_cast<size_t>(b) * d, p->h0 + static_cast<size_t>(b + 1) * d);
      for (int c = 0; c < C; ++c) {
        bm->axis.push_back(p->bf_axis[c]);
        const double* cf = p->bf_coef + (static_cast<size_t>(b) * C + c) * p->nspins;
        bm->coef.emplace_back(cf, cf + p->nspins);
      }
      if (arith == ORACLE_ARITH_STRUCTURED) {
        P.m = bm;
      } else {
        if (d > 512) throw InvalidArg("reference (dense LU) arithmetic limited to d <= 512");
        P.m = std::make_shared<DenseM>(bm->densify());
      }
      break;
    }
    case QOC_KIND_STRANG: {
      if (!p->kinetic || !p->grid_x) throw InvalidArg("condensate model needs kinetic/grid");
      if (C != 1) throw InvalidArg("single control channel expected");
      auto s = std::make_shared<StrangM>();
      s->kin.assign(p->kinetic, p->kinetic + d);
      s->x.assign(p->grid_x, p->grid_x + d);
      s->pot = p->potential;
      for (int i = 0; i < 4; ++i) s->pp[i] = p->pot_params[i];
      s->kappa = p->kappa;
      if (p->potential == QOC_POT_BASIS) {
        if (p->pot_terms < 1 || p->pot_terms > QOC_MAX_POT_TERMS || !p->pot_term_type || !p->pot_term_param ||
            !p->pot_basis)
          throw InvalidArg("basis potential needs 1..QOC_MAX_POT_TERMS terms with type, parameter and profile arrays");
        for (int m2 = 0; m2 < p->pot_terms; ++m2) {
          s->term_type.push_back(p->pot_term_type[m2]);
          s->term_param.push_back(p->pot_term_param[m2]);
          s->basis.emplace_back(p->pot_basis + static_cast<size_t>(m2) * p->dim,
                                p->pot_basis + static_cast<size_t>(m2 + 1) * p->dim);
        }
      }
      P.m = s;
      break;
    }
    default:
      throw InvalidArg("unknown model kind");
  }
  P.m->kind = p->kind;
  P.m->d = slen;
  P.m->C = C;
  P.m->w = p->ip_weight;
  P.init = load_cvec(p->initial + 2 * static_cast<size_t>(b) * slen, static_cast<size_t>(slen));
  P.targ = load_cvec(p->target + 2 * static_cast<size_t>(b) * slen, static_cast<size_t>(slen));
  P.alpha.assign(static_cast<size_t>(P.K), 0.0);
  if (p->penalty) P.alpha.assign(p->penalty, p->penalty + P.K);
  return P;
}

// ---------------------------------------------------------------------------------------
// propagation.cpp:77-83 state_dot / state_norm; 172-234 propagate / checkpointed trajectory.
// Controls are column-major C x len: sample (c, j) at u[c + j*C].
// ---------------------------------------------------------------------------------------
static cd sdot(const Model& m, const CV& a, const CV& b) {
  cd acc = 0.0;
  for (size_t i = 0; i < a.size(); ++i) acc += std::conj(a[i]) * b[i];
  return m.w * acc;
}
static double snorm(const Model& m, const CV& a) {
  return std::sqrt(std::max(0.0, sdot(m, a, a).real()));
}

static CV step_fwd(const Model& m, const double* uj, double dt, const CV& s) {
  if (m.kind == QOC_KIND_STRANG) return static_cast<const StrangM&>(m).step(uj, dt, s);
  CMat X(static_cast<int>(s.size()), 1);
  X.v = s;
  m.cayley(uj, dt, X, false);
  return X.v;
}
static CV step_adj_linear(const Model& m, const double* uj, double dt, const CV& s) {
  CMat X(static_cast<int>(s.size()), 1);
  X.v = s;
  m.cayley(uj, dt, X, true);
  return X.v;
}
static CV step_adj(const Model& m, const double* uj, double dt, const CV& chi, const CV* psi_j,
                   bool naive) {
  if (m.kind == QOC_KIND_STRANG) {
    CV cj, pb, cb;
    static_cast<const StrangM&>(m).backward(uj, dt, *psi_j, chi, naive, cj, pb, cb);
    return cj;
  }
  return step_adj_linear(m, uj, dt, chi);
}

static std::vector<CV> propagate(const Model& m, const double* u, int len, double dt, const CV& init) {
  std::vector<CV> traj;
  traj.reserve(static_cast<size_t>(len) + 1);
  traj.push_back(init);
  for (int j = 0; j < len; ++j) traj.push_back(step_fwd(m, u + static_cast<size_t>(j) * m.C, dt, traj.back()));
  return traj;
}
static CV propagate_final(const Model& m, const double* u, int len, double dt, const CV& init) {
  CV s = init;
  for (int j = 0; j < len; ++j) s = step_fwd(m, u + static_cast<size_t>(j) * m.C, dt, s);
  return s;
}

// CheckpointedTrajectory (propagation.cpp:202-234): snapshots at stride multiples, windows
// recomputed on demand; states are bit-identical to dense storage.
struct Checkpointed {
  const Model& m;
  const double* u;
  int len, stride;
  double dt;
  std::vector<CV> snaps;
  mutable int base = -1;
  mutable std::vector<CV> window;
  Checkpointed(const Model& mm, const double* uu, int n, double dtt, const CV& init, int s)
      : m(mm), u(uu), len(n), stride(s), dt(dtt) {
    if (stride <= 0) throw InvalidArg("checkpoint stride must be positive");
    CV st = init;
    snaps.push_back(st);
    for (int j = 0; j < len; ++j) {
      st = step_fwd(m, u + static_cast<size_t>(j) * m.C, dt, st);
      if ((j + 1) % stride == 0) snaps.push_back(st);
    }
  }
  const CV& state(int j) const {
    const int b = (j / stride) * stride;
    if (b != base) {
      const int n = std::min(stride, len - b);
      window.assign(1, snaps[static_cast<size_t>(b / stride)]);
      for (int i = 0; i < n; ++i)
        window.push_back(step_fwd(m, u + static_cast<size_t>(b + i) * m.C, dt, window.back()));
      base = b;
    }
    return window[static_cast<size_t>(j - b)];
  }
};

// ---------------------------------------------------------------------------------------
// objective.cpp:22-160.
// ---------------------------------------------------------------------------------------
static double penalty(const double* u, int C, int len, double dt, const double* alpha) {
  double acc = 0.0;  // weighted_l2_penalty, controls.cpp:174-181
  for (int j = 0; j < len; ++j) {
    double sq = 0.0;
    for (int c = 0; c < C; ++c) sq += u[c + static_cast<size_t>(j) * C] * u[c + static_cast<size_t>(j) * C];
    acc += alpha[j] * sq;
  }
  return 0.5 * dt * acc;
}

static double payoff(const Model& m, const CV& fin, const CV& targ, int form) {  // 22-29
  if (form == QOC_FORM_OVERLAP) return sdot(m, targ, fin).real();
  CV diff(fin.size());
  for (size_t i = 0; i < fin.size(); ++i) diff[i] = fin[i] - targ[i];
  return -0.5 * sdot(m, diff, diff).real();
}

static CV seed_of(const CV& fin, const CV& targ, int form) {  // 31-34
  if (form == QOC_FORM_OVERLAP) return targ;
  CV s(fin.size());
  for (size_t i = 0; i < fin.size(); ++i) s[i] = targ[i] - fin[i];
  return s;
}

static double evaluate(const Model& m, const double* u, int len, double dt, const CV& init,
                       const CV& targ, const double* alpha, int form) {  // 93-100
  const CV fin = propagate_final(m, u, len, dt, init);
  return payoff(m, fin, targ, form) - penalty(u, m.C, len, dt, alpha);
}

// gradient_sweep (38-89); state_at(j) gives the forward state at node j
static RV sweep(const Model& m, const double* u, int len, double dt,
                const std::function<const CV&(int)>& state_at, const CV& seed,
                const double* alpha, bool naive) {
  const int C = m.C;
  RV g(static_cast<size_t>(C) * len);
  CV chi = seed;
  CV tmp(static_cast<size_t>(m.d));
  for (int j = len - 1; j >= 0; --j) {
    const double* uj = u + static_cast<size_t>(j) * C;
    if (m.kind == QOC_KIND_DENSITY) {  // objective.cpp:61-71
      double tr[64];
      static_cast<const ConjM&>(m).backward(uj, dt, chi, state_at(j + 1), tr);
      for (int c = 0; c < C; ++c) g[c + static_cast<size_t>(j) * C] = -alpha[j] * dt * uj[c] + 2.0 * dt * tr[c];
    } else if (m.kind == QOC_KIND_STRANG) {
      CV cj, pb, cb;
      const auto& sm = static_cast<const StrangM&>(m);
      sm.backward(uj, dt, state_at(j), chi, naive, cj, pb, cb);
      chi = std::move(cj);
      const RV dv = sm.potential_derivative(uj);
      for (int c = 0; c < C; ++c) {
        cd ip(0.0, 0.0);
        for (int i = 0; i < m.d; ++i) ip += std::conj(cb[i]) * dv[i] * pb[i];
        g[c + static_cast<size_t>(j) * C] = -alpha[j] * dt * uj[c] + dt * m.w * ip.imag();
      }
    } else {
      const CV chi_next = chi;
      chi = step_adj_linear(m, uj, dt, chi_next);
      CV cs(chi.size()), ps(chi.size());
      const CV& pj = state_at(j);
      const CV& pj1 = state_at(j + 1);
      for (size_t i = 0; i < chi.size(); ++i) {
        cs[i] = chi[i] + chi_next[i];
        ps[i] = pj[i] + pj1[i];
      }
      for (int c = 0; c < C; ++c) {
        m.dH(c, uj, ps.data(), tmp.data());
        g[c + static_cast<size_t>(j) * C] =
            -alpha[j] * dt * uj[c] + 0.25 * dt * sdot(m, cs, tmp).imag();
      }
    }
  }
  return g;
}

static RV gradient(const Model& m, const double* u, int len, double dt, const CV& init,
                   const CV& targ, const double* alpha, int form, bool naive, int stride) {
  if (stride > 0) {  // 113-119
    Checkpointed tr(m, u, len, dt, init, stride);
    const CV seed = seed_of(tr.state(len), targ, form);
    return sweep(m, u, len, dt, [&tr](int j) -> const CV& { return tr.state(j); }, seed, alpha, naive);
  }
  const std::vector<CV> tr = propagate(m, u, len, dt, init);
  const CV seed = seed_of(tr.back(), targ, form);
  return sweep(m, u, len, dt, [&tr](int j) -> const CV& { return tr[static_cast<size_t>(j)]; }, seed,
               alpha, naive);
}

static CMat assemble(const Model& m, const double* u, int len, double dt) {  // 236-249
  if (!m.linear()) throw LogicErr("no dense one-step matrices to assemble for this propagator kind");
  if (m.kind == QOC_KIND_DENSITY) return static_cast<const ConjM&>(m).assemble_dm(u, len, dt);
  CMat prod = CMat::identity(m.d);
  for (int j = 0; j < len; ++j) m.cayley(u + static_cast<size_t>(j) * m.C, dt, prod, false);
  return prod;
}

static double error_norm(const RV& g, int C) {  // 152-160
  double acc = 0.0;
  const size_t cols = g.size() / static_cast<size_t>(C);
  for (size_t j = 0; j < cols; ++j) {
    double sq = 0.0;
    for (int c = 0; c < C; ++c) sq += g[c + j * C] * g[c + j * C];
    acc += std::sqrt(sq);
  }
  return acc;
}

// ---------------------------------------------------------------------------------------
// runtime.cpp:16-90 — fixed thread pool with an atomic ticket; results merged by index.
// ---------------------------------------------------------------------------------------
class Pool {
 public:
  explicit Pool(int n) : n_(std::max(1, n)) {
    if (n_ > 1)
      for (int i = 0; i < n_; ++i) threads_.emplace_back([this] { loop(); });
  }
  ~Pool() {
    if (!threads_.empty()) {
      {
        std::lock_guard<std::mutex> g(mu_);
        stop_ = true;
      }
      wake_.notify_all();
      for (auto& t : threads_) t.join();
    }
  }
  void run(int count, const std::function<void(int)>& fn) {
    if (count <= 0) return;
    if (threads_.empty()) {
      for (int i = 0; i < count; ++i) fn(i);
      return;
    }
    {
      std::lock_guard<std::mutex> g(mu_);
      fn_ = &fn;
      count_ = count;
      next_.store(0);
      pending_ = static_cast<int>(threads_.size());
      err_ = nullptr;
      ++gen_;
    }
    wake_.notify_all();
    std::unique_lock<std::mutex> lk(mu_);
    done_.wait(lk, [&] { return pending_ == 0; });
    fn_ = nullptr;
    if (err_) std::rethrow_exception(err_);
  }

 private:
  void loop() {
    uint64_t seen = 0;
    for (;;) {
      {
        std::unique_lock<std::mutex> lk(mu_);
        wake_.wait(lk, [&] { return stop_ || gen_ != seen; });
        if (stop_) return;
        seen = gen_;
      }
      for (;;) {
        const int i = next_.fetch_add(1);
        if (i >= count_) break;
        try {
          (*fn_)(i);
        } catch (...) {
          std::lock_guard<std::mutex> g(mu_);
          if (!err_) err_ = std::current_exception();
        }
      }
      std::lock_guard<std::mutex> g(mu_);
      if (--pending_ == 0) done_.notify_all();
    }
  }
  int n_;
  std::vector<std::thread> threads_;
  std::mutex mu_;
  std::condition_variable wake_, done_;
  const std::function<void(int)>* fn_ = nullptr;
  std::atomic<int> next_{0};
  int count_ = 0, pending_ = 0;
  uint64_t gen_ = 0;
  bool stop_ = false;
  std::exception_ptr err_;
};

// ---------------------------------------------------------------------------------------
// Decomposition (controls.cpp:110-140), generalised per SURVEY F4.
// ---------------------------------------------------------------------------------------
static std::vector<int> decomposition(int K, int L, int mode, const int32_t* explicit_nodes) {
  if (L < 1) throw RuntimeErr("Decomposition: parts must be positive");
  std::vector<int> node;
  if (mode == QOC_PARTITION_EXPLICIT) {
    if (!explicit_nodes) throw InvalidArg("explicit partition needs node_index");
    for (int n = 0; n <= L; ++n) node.push_back(explicit_nodes[n]);
    if (node.front() != 0 || node.back() != K)
      throw RuntimeErr("Decomposition: boundaries must span the full grid");
    for (int n = 0; n < L; ++n)
      if (node[n + 1] <= node[n]) throw RuntimeErr("Decomposition: boundary times must strictly increase");
    return node;
  }
  if (mode == QOC_PARTITION_UNIFORM && K % L != 0)
    throw RuntimeErr("Decomposition: step count " + std::to_string(K) + " is not divisible into " +
                     std::to_string(L) + " equal parts");
  if (L > K) throw RuntimeErr("Decomposition: more parts than steps");
  const int base = K / L, extra = K % L;
  int pos = 0;
  node.push_back(0);
  for (int n = 0; n < L; ++n) {
    pos += base + (n < extra ? 1 : 0);
    node.push_back(pos);
  }
  return node;
}

// ---------------------------------------------------------------------------------------
// ism.cpp — node_sweeps (35-84), waypoints (100-120), subproblems (131-159), run_ism (211-612).
// ---------------------------------------------------------------------------------------
struct Task {
  int b = 0, len = 0;
  CV init, targ;
  RV alpha;  // scaled by len/total
  double weight = 1.0;
  int form = QOC_FORM_TRACKING;
};

static void node_sweeps(const Prob& P, const double* u, const std::vector<int>& node, bool naive,
                        std::vector<CV>& psi, std::vector<CV>& chi) {
  const Model& m = *P.m;
  const int parts = static_cast<int>(node.size()) - 1, K = P.K;
  psi.assign(static_cast<size_t>(parts) + 1, CV());
  chi.assign(static_cast<size_t>(parts) + 1, CV());
  CV st = P.init;
  psi[0] = st;
  int nxt = 1;
  for (int j = 0; j < K; ++j) {
    st = step_fwd(m, u + static_cast<size_t>(j) * m.C, P.dt, st);
    if (nxt <= parts && node[nxt] == j + 1) psi[nxt++] = st;
  }
  const bool need_fwd = m.kind == QOC_KIND_STRANG;
  const int stride = (need_fwd && K > 4096) ? static_cast<int>(std::lround(std::sqrt(static_cast<double>(K)))) : 0;
  std::vector<CV> full;
  std::optional<Checkpointed> win;
  if (need_fwd) {
    if (stride > 0)
      win.emplace(m, u, K, P.dt, P.init, stride);
    else
      full = propagate(m, u, K, P.dt, P.init);
  }
  CV c = P.targ;
  chi[static_cast<size_t>(parts)] = c;
  int prev = parts - 1;
  for (int j = K - 1; j >= 0; --j) {
    const CV* pj = need_fwd ? (win ? &win->state(j) : &full[static_cast<size_t>(j)]) : nullptr;
    c = step_adj(m, u + static_cast<size_t>(j) * m.C, P.dt, c, pj, naive);
    if (prev >= 0 && node[prev] == j) chi[static_cast<size_t>(prev--)] = c;
  }
}

static std::vector<CV> waypoints(const std::vector<CV>& psi, const std::vector<CV>& chi,
                                 const std::vector<int>& node) {
  const int parts = static_cast<int>(node.size()) - 1;
  const int total = node.back();
  std::vector<CV> phi(static_cast<size_t>(parts) + 1);
  for (int n = 0; n <= parts; ++n) {
    const int j = node[n];
    const double a = static_cast<double>(total - j) / static_cast<double>(total);
    const double b = static_cast<double>(j) / static_cast<double>(total);
    CV v(psi[n].size());
    for (size_t i = 0; i < v.size(); ++i) v[i] = a * psi[n][i] + b * chi[n][i];
    phi[n] = std::move(v);
  }
  return phi;
}

static std::vector<Task> subproblems(const Prob& P, const std::vector<int>& node,
                                     const std::vector<CV>& inits, const std::vector<CV>& targs,
                                     bool weighted, int form) {
  const int parts = static_cast<int>(node.size()) - 1;
  const double total = static_cast<double>(P.K);
  std::vector<Task> tasks(static_cast<size_t>(parts));
  for (int n = 0; n < parts; ++n) {
    Task& t = tasks[static_cast<size_t>(n)];
    t.b = node[n];
    t.len = node[n + 1] - node[n];
    t.init = inits[static_cast<size_t>(n)];
    t.targ = targs[static_cast<size_t>(n)];
    t.alpha.assign(P.alpha.begin() + t.b, P.alpha.begin() + t.b + t.len);
    const double scale = static_cast<double>(t.len) / total;
    for (double& a : t.alpha) a *= scale;
    t.weight = weighted ? total / static_cast<double>(t.len) : 1.0;
    t.form = form;
  }
  return tasks;
}

static bool finite_vec(const CV& v) {
  for (const cd& x : v)
    if (!std::isfinite(x.real()) || !std::isfinite(x.imag())) return false;
  return true;
}

// ---------------------------------------------------------------------------------------
// optimizers.cpp — the two other inner solvers (the gradient update is inline in run_ism).
// ---------------------------------------------------------------------------------------
struct InnerOut {
  int guard_rejections = 0, newton_fallbacks = 0, gmres_iterations = 0;
};

static double vnorm(const RV& v) {
  double s = 0.0;
  for (double x : v) s += x * x;
  return std::sqrt(s);
}
static double vdot(const RV& a, const RV& b) {
  double s = 0.0;
  for (size_t i = 0; i < a.size(); ++i) s += a[i] * b[i];
  return s;
}

// Restarted GMRES on v -> A v (optimizers.cpp:21-98).
static RV gmres(const std::function<RV(const RV&)>& apply, const RV& b, int restart, int max_iter,
                double tol, int* iterations, double* relative_residual) {
  const size_t n = b.size();
  RV x(n, 0.0);
  const double bnorm = vnorm(b);
  int used = 0;
  double rel = 0.0;
  if (bnorm == 0.0) {
    *iterations = 0;
    *relative_residual = 0.0;
    return x;
  }
  while (used < max_iter) {
    RV r = apply(x);
    for (size_t e = 0; e < n; ++e) r[e] = b[e] - r[e];
    ++used;
    const double beta = vnorm(r);
    rel = beta / bnorm;
    if (rel <= tol) break;
    const int m = std::min(restart, static_cast<int>(n));
    std::vector<RV> v(static_cast<size_t>(m) + 1, RV(n, 0.0));
    std::vector<RV> h(static_cast<size_t>(m) + 1, RV(static_cast<size_t>(std::max(m, 1)), 0.0));  // h[row][col]
    RV g(static_cast<size_t>(m) + 1, 0.0), cs(static_cast<size_t>(std::max(m, 1)), 1.0),
        sn(static_cast<size_t>(std::max(m, 1)), 0.0);
    for (size_t e = 0; e < n; ++e) v[0][e] = r[e] / beta;
    g[0] = beta;
    int spanned = 0;
    for (int i = 0; i < m && used < max_iter; ++i) {
      RV w = apply(v[static_cast<size_t>(i)]);
      ++used;
      for (int k = 0; k <= i; ++k) {  // modified Gram-Schmidt
        const double hk = vdot(v[static_cast<size_t>(k)], w);
        h[k][i] = hk;
        for (size_t e = 0; e < n; ++e) w[e] -= hk * v[static_cast<size_t>(k)][e];
      }
      h[i + 1][i] = vnorm(w);
      const bool breakdown = h[i + 1][i] <= 1e-14 * bnorm;
      if (!breakdown)
        for (size_t e = 0; e < n; ++e) v[static_cast<size_t>(i) + 1][e] = w[e] / h[i + 1][i];
      for (int k = 0; k < i; ++k) {  // earlier Givens rotations on the new column
        const double t = cs[k] * h[k][i] + sn[k] * h[k + 1][i];
        h[k + 1][i] = -sn[k] * h[k][i] + cs[k] * h[k + 1][i];
        h[k][i] = t;
      }
      const double denom = std::hypot(h[i][i], h[i + 1][i]);
      cs[i] = denom == 0.0 ? 1.0 : h[i][i] / denom;
      sn[i] = denom == 0.0 ? 0.0 : h[i + 1][i] / denom;
      h[i][i] = denom;
      h[i + 1][i] = 0.0;
      g[i + 1] = -sn[i] * g[i];
      g[i] = cs[i] * g[i];
      spanned = i + 1;
      rel = std::abs(g[i + 1]) / bnorm;
      if (rel <= tol || breakdown) break;
    }
    if (spanned > 0) {  // back substitution on the rotated Hessenberg block
      RV y(static_cast<size_t>(spanned));
      for (int r2 = spanned - 1; r2 >= 0; --r2) {
        double acc = g[r2];
        for (int c2 = r2 + 1; c2 < spanned; ++c2) acc -= h[r2][c2] * y[c2];
        y[r2] = acc / h[r2][r2];
      }
      for (int c2 = 0; c2 < spanned; ++c2)
        for (size_t e = 0; e < n; ++e) x[e] += v[static_cast<size_t>(c2)][e] * y[c2];
    }
    if (rel <= tol) {
      RV check = apply(x);
      for (size_t e = 0; e < n; ++e) check[e] = b[e] - check[e];
      ++used;
      rel = vnorm(check) / bnorm;
      if (rel <= tol) break;
    }
  }
  *iterations = used;
  *relative_residual = rel;
  return x;
}

// newton_direction + newton_step (optimizers.cpp:215-259): (Hessian) d = -g0 with central
// finite-difference Hessian-vector products of the weighted task gradient.
static void newton_step(const Model& m, RV& u, const Task& t, double dt, const qoc_solver_v1& sv,
                        bool naive, int stride, InnerOut& out) {
  auto grad = [&](const RV& samples) {
    RV g = gradient(m, samples.data(), t.len, dt, t.init, t.targ, t.alpha.data(), t.form, naive, stride);
    for (double& x : g) x *= t.weight;
    return g;
  };
  const RV g0 = grad(u);
  const double u_scale = 1.0 + vnorm(u);
  auto hessian_apply = [&](const RV& v) {
    const double vn = vnorm(v);
    if (vn == 0.0) return RV(v.size(), 0.0);
    const double h = sv.hvp_scale * u_scale / vn;
    RV up(u), um(u);
    for (size_t e = 0; e < u.size(); ++e) {
      up[e] = u[e] + h * v[e];
      um[e] = u[e] - h * v[e];
    }
    RV gp = grad(up);
    const RV gm = grad(um);
    for (size_t e = 0; e < gp.size(); ++e) gp[e] = (gp[e] - gm[e]) / (2.0 * h);
    return gp;
  };
  RV rhs(g0.size());
  for (size_t e = 0; e < g0.size(); ++e) rhs[e] = -g0[e];
  int iters = 0;
  double rel = 0.0;
  RV d = gmres(hessian_apply, rhs, sv.gmres_restart, sv.gmres_max_iter, sv.gmres_tol, &iters, &rel);
  out.gmres_iterations += iters;
  if (!(vdot(d, g0) > 0.0)) {  // not an ascent direction: plain gradient step
    for (size_t e = 0; e < d.size(); ++e) d[e] = sv.step_size * g0[e];
    ++out.newton_fallbacks;
  }
  for (size_t e = 0; e < u.size(); ++e) u[e] += d[e];
}

// monotonic_step (optimizers.cpp:109-213): forward sweep that rebuilds the control slice by
// slice against the adjoint nodes of the previous control.
static void monotonic_step(const Model& m, RV& u, const Task& t, double dt, const qoc_solver_v1& sv,
                           InnerOut& out) {
  const DenseM* dm = m.kind == QOC_KIND_DENSITY ? nullptr : dynamic_cast<const DenseM*>(&m);
  if (!dm)
    throw LogicErr("the monotonic sweep requires column states with the one-step rational scheme");
  if (m.C != 1) throw LogicErr("the monotonic sweep handles a single control channel");
  for (int j = 0; j < t.len; ++j)
    if (t.alpha[static_cast<size_t>(j)] <= 0.0)
      throw LogicErr("the monotonic sweep requires strictly positive penalty weights");
  const int d = m.d, steps = t.len;
  // dH/dv = M + v P (DenseModel: M = A_0, P = B_0; models.cpp:70-75)
  const CMat& mu_op = dm->lin[0];
  CMat pol_op(d, d);
  if (!dm->quad.empty()) pol_op = dm->quad[0];
  const cd half(0.0, 0.5 * dt);
  auto shifted = [&](double v, double sign) {  // I + sign * (i dt/2) H(v)
    const CMat h = dm->hamiltonian(&v);
    CMat a = CMat::identity(d);
    for (size_t e = 0; e < h.v.size(); ++e) a.v[e] += sign * (half * h.v[e]);
    return a;
  };
  auto col = [&](const CV& s) {
    CMat c(d, 1);
    c.v = s;
    return c;
  };
  std::vector<CV> chi(static_cast<size_t>(steps) + 1);
  chi[static_cast<size_t>(steps)] = t.targ;
  for (int j = steps - 1; j >= 0; --j)
    chi[static_cast<size_t>(j)] = step_adj_linear(m, &u[static_cast<size_t>(j)], dt, chi[static_cast<size_t>(j) + 1]);
  CV psi = t.init;
  for (int j = 0; j < steps; ++j) {
    const double uj = u[static_cast<size_t>(j)], aj = t.alpha[static_cast<size_t>(j)];
    CMat psi_tilde = col(psi);
    PivLU(shifted(uj, +1.0)).solve_inplace(psi_tilde);
    double m_mu = 0.0, m_pol = 0.0;
    auto pairings_at = [&](double v) {
      CMat chi_tilde = col(chi[static_cast<size_t>(j) + 1]);
      PivLU(shifted(v, -1.0)).solve_inplace(chi_tilde);
      const CMat a = matmul(mu_op, psi_tilde), b2 = matmul(pol_op, psi_tilde);
      cd sm(0.0, 0.0), sp(0.0, 0.0);
      for (int i = 0; i < d; ++i) {
        sm += std::conj(chi_tilde.v[i]) * a.v[i];
        sp += std::conj(chi_tilde.v[i]) * b2.v[i];
      }
      m_mu = sm.imag();
      m_pol = sp.imag();
    };
    double v = uj;
    bool usable = true;
    for (int it = 0; it < sv.fixed_point_max_iter; ++it) {  // v (alpha - m_pol(v)) = m_mu(v)
      pairings_at(v);
      const double denom = aj - m_pol;
      if (!(std::abs(denom) > 1e-14 * (1.0 + aj))) {
        usable = false;
        break;
      }
      const double next = m_mu / denom;
      const bool settled = std::abs(next - v) <= sv.fixed_point_tol * (1.0 + std::abs(v));
      v = next;
      if (settled) break;
    }
    if (usable && std::isfinite(v)) {
      pairings_at(v);
      const double gain = dt * (v - uj) * (m_mu + 0.5 * (v + uj) * (m_pol - aj));
      if (!(gain >= 0.0)) usable = false;
    } else {
      usable = false;
    }
    if (!usable) {
      v = uj;
      ++out.guard_rejections;
    }
    u[static_cast<size_t>(j)] = v;
    psi = step_fwd(m, &v, dt, psi);
  }
}

struct IterRec {
  int iteration = 0;
  double objective = 0.0;
  std::optional<double> exact, error;
  RV task_values;
  double wall = 0.0;
  std::vector<InnerOut> inner;  // per task (ism.cpp:409-411)
};

struct RunOut {
  RV u;
  std::vector<IterRec> its;
  bool aborted = false;
  std::string reason;
};

static double now() {
  using clk = std::chrono::steady_clock;
  return std::chrono::duration<double>(clk::now().time_since_epoch()).count();
}

static RunOut run_ism(const Prob& P, const double* u0, const qoc_ism_config_v1& cfg,
                      const qoc_solver_v1& sv, Pool& pool) {
  const Model& m = *P.m;
  const bool lin = m.linear();
  if (cfg.subintervals < 1 || cfg.workers < 1 || cfg.max_outer < 0 || cfg.eta < 0.0)
    throw InvalidArg("subintervals and workers must be >= 1, max_outer and eta >= 0");
  const bool split = cfg.variant == QOC_VARIANT_SPLIT;
  if (!split && !lin)
    throw InvalidArg(
        "interpolated waypoints require linear one-step flows; use the split variant for "
        "split-step states");
  if (sv.kind < QOC_SOLVER_GRADIENT || sv.kind > QOC_SOLVER_NEWTON) throw InvalidArg("unknown solver kind");
  const int parts = cfg.subintervals;
  const std::vector<int> node = decomposition(P.K, parts, cfg.partition, cfg.node_index);
  const bool direct = cfg.plan == QOC_PLAN_DIRECT;
  const int stride = cfg.checkpoint_stride > 0 ? cfg.checkpoint_stride : sv.checkpoint_stride;
  const bool naive = sv.naive_nonlinear_adjoint != 0;
  const int C = P.C;
  const double dt = P.dt;

  RunOut out;
  out.u.assign(u0, u0 + static_cast<size_t>(C) * P.K);
  auto upart = [&](int n) { return out.u.data() + static_cast<size_t>(node[n]) * C; };

  std::vector<CV> psi, chi;
  std::vector<Task> tasks;
  auto rebuild = [&]() {  // ism.cpp:260-280
    if (parts == 1) {
      tasks = subproblems(P, node, {P.init}, {P.targ}, !split, split ? QOC_FORM_OVERLAP : QOC_FORM_TRACKING);
      return;
    }
    if (split) {
      std::vector<CV> in(psi.begin(), psi.end() - 1), tg(chi.begin() + 1, chi.end());
      tasks = subproblems(P, node, in, tg, false, QOC_FORM_OVERLAP);
    } else {
      const std::vector<CV> phi = waypoints(psi, chi, node);
      std::vector<CV> in(phi.begin(), phi.end() - 1), tg(phi.begin() + 1, phi.end());
      tasks = subproblems(P, node, in, tg, true, QOC_FORM_TRACKING);
    }
  };
  auto boundary_objective = [&]() {  // ism.cpp:285-296
    const CV& fin = psi[static_cast<size_t>(parts)];
    double fid;
    if (split) {
      fid = sdot(m, P.targ, fin).real();
    } else {
      CV diff(fin.size());
      for (size_t i = 0; i < fin.size(); ++i) diff[i] = fin[i] - P.targ[i];
      const double dist = snorm(m, diff);
      fid = -0.5 * dist * dist;
    }
    return fid - penalty(out.u.data(), C, P.K, dt, P.alpha.data());
  };
  std::vector<CMat> props(static_cast<size_t>(parts));
  auto compose = [&]() {  // ism.cpp:298-312
    psi.assign(static_cast<size_t>(parts) + 1, CV());
    chi.assign(static_cast<size_t>(parts) + 1, CV());
    // apply_propagator (propagation.cpp:251-261): prop * state for column states,
    // prop * state * prop^dag for the density kind's dm x dm matrix states
    auto apply = [&](const CMat& prop, const CV& state) {
      if (m.kind == QOC_KIND_DENSITY) {
        const int dm = prop.rows;
        CMat s(dm, dm);
        s.v = state;
        return matmul(matmul(prop, s), adjoint(prop)).v;
      }
      CMat s(m.d, 1);
      s.v = state;
      return matmul(prop, s).v;
    };
    psi[0] = P.init;
    for (int n = 0; n < parts; ++n) psi[n + 1] = apply(props[n], psi[n]);
    chi[static_cast<size_t>(parts)] = P.targ;
    for (int n = parts - 1; n >= 0; --n) chi[n] = apply(adjoint(props[n]), chi[n + 1]);
  };
  auto finite_controls = [&]() {
    for (double v : out.u)
      if (!std::isfinite(v)) return false;
    return true;
  };
  auto finite_nodes = [&]() {
    if (parts == 1) return true;
    for (const CV& s : psi)
      if (!finite_vec(s)) return false;
    for (const CV& s : chi)
      if (!finite_vec(s)) return false;
    return true;
  };

  {  // bootstrap, ism.cpp:344-393
    IterRec boot;
    const double w0 = now();
    if (parts > 1) {
      if (!split && !direct) {
        pool.run(parts, [&](int n) { props[n] = assemble(m, upart(n), node[n + 1] - node[n], dt); });
        compose();
      } else {
        node_sweeps(P, out.u.data(), node, naive, psi, chi);
      }
      boot.objective = boundary_objective();
    } else {
      boot.objective = kNaN;
    }
    rebuild();
    boot.wall = now() - w0;
    if (!finite_nodes()) {
      out.aborted = true;
      out.reason = "non-finite boundary state during bootstrap";
      out.its.push_back(boot);
      return out;
    }
    out.its.push_back(boot);
  }

  struct Slot {
    double entry = 0.0, error = 0.0;
    RV unew;
    InnerOut inner;
    CV psi_end, chi_start;
  };
  std::vector<Slot> slots(static_cast<size_t>(parts));
  bool aborted = false;
  for (int k = 1; k <= cfg.max_outer && !aborted; ++k) {
    IterRec it;
    it.iteration = k;
    const double w0 = now();
    pool.run(parts, [&](int n) {  // ism.cpp:401-479
      Slot& r = slots[static_cast<size_t>(n)];
      const Task& t = tasks[static_cast<size_t>(n)];
      const double* un = upart(n);
      r.entry = t.weight * evaluate(m, un, t.len, dt, t.init, t.targ, t.alpha.data(), t.form);
      r.unew.assign(un, un + static_cast<size_t>(C) * t.len);
      r.inner = InnerOut{};
      for (int inner = 0; inner < sv.inner_iterations; ++inner) {  // run_inner, optimizers.cpp:261-285
        if (sv.kind == QOC_SOLVER_MONOTONIC) {
          monotonic_step(m, r.unew, t, dt, sv, r.inner);
        } else if (sv.kind == QOC_SOLVER_NEWTON) {
          newton_step(m, r.unew, t, dt, sv, naive, stride, r.inner);
        } else {  // gradient_step
          RV g = gradient(m, r.unew.data(), t.len, dt, t.init, t.targ, t.alpha.data(), t.form, naive, stride);
          for (size_t e = 0; e < g.size(); ++e) r.unew[e] += sv.step_size * (t.weight * g[e]);
        }
      }
      if (cfg.compute_error) {
        const RV g = gradient(m, r.unew.data(), t.len, dt, t.init, t.targ, t.alpha.data(), t.form, naive, stride);
        r.error = error_norm(g, C);
      } else {
        r.error = 0.0;
      }
      if (parts > 1 && !split && !direct) props[n] = assemble(m, r.unew.data(), t.len, dt);
      if (parts > 1 && split && !direct) {  // lagged boundary refresh, ism.cpp:424-459
        const CV& start = psi[static_cast<size_t>(n)];
        if (!lin) {
          std::vector<CV> tr = propagate(m, r.unew.data(), t.len, dt, start);
          r.psi_end = tr.back();
          CV c = chi[static_cast<size_t>(n) + 1];
          for (int j = t.len - 1; j >= 0; --j)
            c = step_adj(m, r.unew.data() + static_cast<size_t>(j) * C, dt, c, &tr[static_cast<size_t>(j)], naive);
          r.chi_start = c;
        } else {
          r.psi_end = propagate_final(m, r.unew.data(), t.len, dt, start);
          CV c = chi[static_cast<size_t>(n) + 1];
          for (int j = t.len - 1; j >= 0; --j)
            c = step_adj(m, r.unew.data() + static_cast<size_t>(j) * C, dt, c, nullptr, naive);
          r.chi_start = c;
        }
      }
    });
    double total_error = 0.0;
    for (int n = 0; n < parts; ++n) {
      std::copy(slots[n].unew.begin(), slots[n].unew.end(), upart(n));
      total_error += slots[n].error;
      it.inner.push_back(slots[n].inner);
    }
    IterRec& prev = out.its.back();
    prev.task_values.assign(static_cast<size_t>(parts), 0.0);
    double esum = 0.0;
    for (int n = 0; n < parts; ++n) {
      prev.task_values[static_cast<size_t>(n)] = slots[n].entry;
      esum += slots[n].entry;
    }
    if (parts == 1) prev.objective = esum;

    if (!finite_controls()) {
      out.aborted = true;
      out.reason = "non-finite control after the task updates of iteration " + std::to_string(k);
      it.objective = kNaN;
      it.wall = now() - w0;
      out.its.push_back(it);
      aborted = true;
      break;
    }
    if (parts > 1) {
      if (direct) {
        node_sweeps(P, out.u.data(), node, naive, psi, chi);
      } else if (split) {
        for (int n = 0; n < parts; ++n) {
          psi[static_cast<size_t>(n) + 1] = slots[n].psi_end;
          chi[static_cast<size_t>(n)] = slots[n].chi_start;
        }
        psi[0] = P.init;
        chi[static_cast<size_t>(parts)] = P.targ;
      } else {
        compose();
      }
      if (!finite_nodes()) {
        out.aborted = true;
        out.reason = "non-finite boundary state at iteration " + std::to_string(k);
        it.objective = kNaN;
        it.wall = now() - w0;
        out.its.push_back(it);
        aborted = true;
        break;
      }
      it.objective = boundary_objective();
      rebuild();
    } else {
      it.objective = kNaN;
    }
    if (cfg.compute_error) it.error = total_error;
    if (cfg.log_exact_objective)
      it.exact = evaluate(m, out.u.data(), P.K, dt, P.init, P.targ, P.alpha.data(), QOC_FORM_OVERLAP);
    it.wall = now() - w0;
    out.its.push_back(it);
    if (cfg.compute_error && total_error <= cfg.eta) break;
  }
  if (!aborted) {  // trailing evaluation, ism.cpp:594-609
    RV fin(static_cast<size_t>(parts), 0.0);
    pool.run(parts, [&](int n) {
      const Task& t = tasks[static_cast<size_t>(n)];
      fin[static_cast<size_t>(n)] = t.weight * evaluate(m, upart(n), t.len, dt, t.init, t.targ, t.alpha.data(), t.form);
    });
    IterRec& last = out.its.back();
    last.task_values = fin;
    if (parts == 1) last.objective = fin[0];
  }
  return out;
}

// Fixture generators, tests/support/fixtures.hpp (same <random> calls, same order).
static CMat random_hermitian(std::mt19937& rng, int dim, double scale) {
  std::normal_distribution<double> g(0.0, scale);
  CMat a(dim, dim);
  for (int j = 0; j < dim; ++j)
    for (int i = 0; i < dim; ++i) a(i, j) = cd(g(rng), g(rng));
  CMat h(dim, dim);
  for (int j = 0; j < dim; ++j)
    for (int i = 0; i < dim; ++i) h(i, j) = 0.5 * (a(i, j) + std::conj(a(j, i)));
  return h;
}
static CV random_state(std::mt19937& rng, int dim) {
  std::normal_distribution<double> g(0.0, 1.0);
  CV v(static_cast<size_t>(dim));
  for (int i = 0; i < dim; ++i) v[i] = cd(g(rng), g(rng));
  double nrm = 0.0;
  for (const cd& x : v) nrm += std::norm(x);
  nrm = std::sqrt(nrm);
  for (cd& x : v) x /= nrm;
  return v;
}
static CV random_cvec(std::mt19937& rng, int n) {
  std::normal_distribution<double> g(0.0, 1.0);
  CV v(static_cast<size_t>(n));
  for (int i = 0; i < n; ++i) v[i] = cd(g(rng), g(rng));
  return v;
}

static void store(const CV& v, double* out) {
  for (size_t i = 0; i < v.size(); ++i) {
    out[2 * i] = v[i].real();
    out[2 * i + 1] = v[i].imag();
  }
}

}  // namespace orc

// ========================================================================================
// C API
// ========================================================================================
using namespace orc;

static int32_t fail(int32_t code, const char* msg, char* err, size_t errlen) {
  if (err && errlen) {
    std::snprintf(err, errlen, "%s", msg);
  }
  return code;
}

template <class F>
static int32_t guarded(char* err, size_t errlen, F&& f) {
  try {
    f();
    if (err && errlen) err[0] = 0;
    return QOC_OK;
  } catch (const InvalidArg& e) {
    return fail(QOC_EINVAL, e.what(), err, errlen);
  } catch (const LogicErr& e) {
    return fail(QOC_ELOGIC, e.what(), err, errlen);
  } catch (const RuntimeErr& e) {
    return fail(QOC_ERUNTIME, e.what(), err, errlen);
  } catch (const std::exception& e) {
    return fail(QOC_ERUNTIME, e.what(), err, errlen);
  }
}

// per-task inner-solver counters of the last oracle_ism_run: [b][k][n]
static std::vector<std::vector<std::vector<InnerOut>>> g_inner_stats;

extern "C" int32_t oracle_solver_stats(int32_t b, int32_t iteration, int32_t subintervals, int32_t* out) {
  if (b < 0 || b >= static_cast<int>(g_inner_stats.size()) || iteration < 0 ||
      iteration >= static_cast<int>(g_inner_stats[static_cast<size_t>(b)].size()) || !out)
    return QOC_EINVAL;
  const auto& row = g_inner_stats[static_cast<size_t>(b)][static_cast<size_t>(iteration)];
  for (int n = 0; n < subintervals; ++n) {
    const InnerOut z = n < static_cast<int>(row.size()) ? row[static_cast<size_t>(n)] : InnerOut{};
    out[n] = z.guard_rejections;
    out[subintervals + n] = z.newton_fallbacks;
    out[2 * subintervals + n] = z.gmres_iterations;
  }
  return QOC_OK;
}

extern "C" int32_t oracle_ism_run(const qoc_problem_v1* p, const qoc_ism_config_v1* cfg,
                                  const qoc_solver_v1* solver, const double* u0, double* u_out,
                                  qoc_iter_record_v1* recs, int32_t rec_cap, double* task_values,
                                  qoc_run_status_v1* status, int32_t arith, int32_t threads,
                                  char* err, size_t errlen) {
  return guarded(err, errlen, [&] {
    validate(p);
    if (!cfg || !solver || !u0 || !u_out || !recs || !status) throw InvalidArg("null argument");
    if (rec_cap < cfg->max_outer + 1) throw InvalidArg("rec_cap must be >= max_outer + 1");
    const int B = p->batch, L = cfg->subintervals;
    const size_t CK = static_cast<size_t>(p->channels) * p->steps;
    std::vector<Prob> probs;
    for (int b = 0; b < B; ++b) probs.push_back(make_prob(p, b, arith));
    g_inner_stats.assign(static_cast<size_t>(B), {});
    auto one = [&](int b, Pool& pool) {
      RunOut r = run_ism(probs[static_cast<size_t>(b)], u0 + CK * b, *cfg, *solver, pool);
      for (const IterRec& it : r.its) g_inner_stats[static_cast<size_t>(b)].push_back(it.inner);
      std::copy(r.u.begin(), r.u.end(), u_out + CK * b);
      qoc_run_status_v1& st = status[b];
      std::memset(&st, 0, sizeof(st));
      st.aborted = r.aborted;
      st.iterations_recorded = static_cast<int32_t>(r.its.size());
      std::snprintf(st.abort_reason, sizeof(st.abort_reason), "%s", r.reason.c_str());
      for (size_t k = 0; k < r.its.size(); ++k) {
        qoc_iter_record_v1& o = recs[static_cast<size_t>(b) * rec_cap + k];
        const IterRec& it = r.its[k];
        o.iteration = it.iteration;
        o.objective = it.objective;
        o.has_error = it.error.has_value();
        o.error = it.error.value_or(kNaN);
        o.has_exact_objective = it.exact.has_value();
        o.exact_objective = it.exact.value_or(kNaN);
        o.device_seconds = it.wall;
        o.reserved = 0;
        if (task_values) {
          double* tv = task_values + (static_cast<size_t>(b) * rec_cap + k) * L;
          for (int n = 0; n < L; ++n)
            tv[n] = n < static_cast<int>(it.task_values.size()) ? it.task_values[static_cast<size_t>(n)] : kNaN;
        }
      }
    };
    const int W = std::max(1, threads);
    if (B == 1) {
      Pool pool(std::min(W, L));
      one(0, pool);
    } else {  // independent problems: spread problems over threads, tasks serial
      Pool outer(W);
      outer.run(B, [&](int b) {
        Pool serial(1);
        one(b, serial);
      });
    }
  });
}

extern "C" int32_t oracle_propagate_final(const qoc_problem_v1* p, const double* u,
                                          double* states_out, int32_t arith, char* err,
                                          size_t errlen) {
  return guarded(err, errlen, [&] {
    validate(p);
    const size_t CK = static_cast<size_t>(p->channels) * p->steps;
    for (int b = 0; b < p->batch; ++b) {
      const Prob P = make_prob(p, b, arith);
      store(propagate_final(*P.m, u + CK * b, P.K, P.dt, P.init), states_out + 2 * static_cast<size_t>(b) * P.d);
    }
  });
}

extern "C" int32_t oracle_propagate(const qoc_problem_v1* p, const double* u, double* traj_out,
                                    int32_t arith, char* err, size_t errlen) {
  return guarded(err, errlen, [&] {
    validate(p);
    const size_t CK = static_cast<size_t>(p->channels) * p->steps;
    for (int b = 0; b < p->batch; ++b) {
      const Prob P = make_prob(p, b, arith);
      const std::vector<CV> tr = propagate(*P.m, u + CK * b, P.K, P.dt, P.init);
      for (size_t j = 0; j < tr.size(); ++j)
        store(tr[j], traj_out + 2 * ((static_cast<size_t>(b) * (P.K + 1) + j) * P.d));
    }
  });
}

extern "C" int32_t oracle_objective_gradient(const qoc_problem_v1* p, const double* u,
                                             int32_t form, int32_t naive, int32_t stride,
                                             double* value_out, double* grad_out, int32_t arith,
                                             char* err, size_t errlen) {
  return guarded(err, errlen, [&] {
    validate(p);
    const size_t CK = static_cast<size_t>(p->channels) * p->steps;
    for (int b = 0; b < p->batch; ++b) {
      const Prob P = make_prob(p, b, arith);
      if (value_out)
        value_out[b] = evaluate(*P.m, u + CK * b, P.K, P.dt, P.init, P.targ, P.alpha.data(), form);
      if (grad_out) {
        const RV g = gradient(*P.m, u + CK * b, P.K, P.dt, P.init, P.targ, P.alpha.data(), form, naive != 0, stride);
        std::copy(g.begin(), g.end(), grad_out + CK * b);
      }
    }
  });
}

extern "C" int32_t oracle_assemble_propagator(const qoc_problem_v1* p, const double* u,
                                              double* prop_out, int32_t arith, char* err,
                                              size_t errlen) {
  return guarded(err, errlen, [&] {
    validate(p);
    const size_t CK = static_cast<size_t>(p->channels) * p->steps;
    for (int b = 0; b < p->batch; ++b) {
      const Prob P = make_prob(p, b, arith);
      const CMat M = assemble(*P.m, u + CK * b, P.K, P.dt);
      store(M.v, prop_out + 2 * static_cast<size_t>(b) * p->dim * p->dim);
    }
  });
}

extern "C" int32_t oracle_step(const qoc_problem_v1* p, const double* u_col, double dt,
                               const double* in, const double* psi_j, int32_t mode, int32_t naive,
                               double* out, int32_t arith, char* err, size_t errlen) {
  return guarded(err, errlen, [&] {
    const Prob P = make_prob(p, 0, arith);
    const CV s = load_cvec(in, static_cast<size_t>(P.d));
    CV r;
    if (mode == 0) {
      r = step_fwd(*P.m, u_col, dt, s);
    } else {
      CV pj;
      if (psi_j) pj = load_cvec(psi_j, static_cast<size_t>(P.d));
      r = step_adj(*P.m, u_col, dt, s, psi_j ? &pj : nullptr, naive != 0);
    }
    store(r, out);
  });
}

extern "C" int32_t oracle_dft(int32_t n, const double* in, double* out, int32_t inverse) {
  char e[8];
  return guarded(e, sizeof(e), [&] {
    const CV x = load_cvec(in, static_cast<size_t>(n));
    store(inverse ? idft(x) : dft(x), out);
  });
}

extern "C" int32_t oracle_boundary_sweep(const qoc_problem_v1* p, const double* u, int32_t parts,
                                         const int32_t* node_index, double* psi_nodes,
                                         double* chi_nodes, int32_t arith, char* err,
                                         size_t errlen) {
  return guarded(err, errlen, [&] {
    const Prob P = make_prob(p, 0, arith);
    const std::vector<int> node = decomposition(P.K, parts, QOC_PARTITION_EXPLICIT, node_index);
    std::vector<CV> ps, cs;
    node_sweeps(P, u, node, false, ps, cs);
    for (int n = 0; n <= parts; ++n) {
      store(ps[n], psi_nodes + 2 * static_cast<size_t>(n) * P.d);
      store(cs[n], chi_nodes + 2 * static_cast<size_t>(n) * P.d);
    }
  });
}

// verify_decomposition, ism.cpp:161-191
extern "C" int32_t oracle_verify_decomposition(const qoc_problem_v1* p, const double* u,
                                               int32_t parts, double* fmis, double* gmis,
                                               int32_t arith, char* err, size_t errlen) {
  return guarded(err, errlen, [&] {
    const Prob P = make_prob(p, 0, arith);
    const Model& m = *P.m;
    const std::vector<int> node = decomposition(P.K, parts, QOC_PARTITION_UNIFORM, nullptr);
    std::vector<CV> ps, cs;
    node_sweeps(P, u, node, false, ps, cs);
    const std::vector<CV> phi = waypoints(ps, cs, node);
    std::vector<CV> in(phi.begin(), phi.end() - 1), tg(phi.begin() + 1, phi.end());
    const std::vector<Task> tasks = subproblems(P, node, in, tg, true, QOC_FORM_TRACKING);
    double summed = 0.0;
    for (int n = 0; n < parts; ++n) {
      const Task& t = tasks[static_cast<size_t>(n)];
      summed += t.weight * evaluate(m, u + static_cast<size_t>(t.b) * P.C, t.len, P.dt, t.init, t.targ, t.alpha.data(), t.form);
    }
    const double global = evaluate(m, u, P.K, P.dt, P.init, P.targ, P.alpha.data(), QOC_FORM_TRACKING);
    *fmis = std::abs(summed - global);
    const RV gg = gradient(m, u, P.K, P.dt, P.init, P.targ, P.alpha.data(), QOC_FORM_TRACKING, false, 0);
    double worst = 0.0;
    for (int n = 0; n < parts; ++n) {
      const Task& t = tasks[static_cast<size_t>(n)];
      const RV g = gradient(m, u + static_cast<size_t>(t.b) * P.C, t.len, P.dt, t.init, t.targ, t.alpha.data(), t.form, false, 0);
      for (size_t e = 0; e < g.size(); ++e)
        worst = std::max(worst, std::abs(t.weight * g[e] - gg[static_cast<size_t>(t.b) * P.C + e]));
    }
    *gmis = worst;
  });
}

extern "C" int32_t oracle_dense_fixture(uint32_t seed, int32_t dim, int32_t steps,
                                        int32_t channels, int32_t quadratic, double alpha,
                                        int32_t random_penalty, double control_amplitude,
                                        double* h0, double* linear, double* quadratic_out,
                                        double* initial, double* target, double* penalty_out,
                                        double* control) {
  std::mt19937 rng(seed);  // fixtures.hpp:66-112 (vector kind)
  store(random_hermitian(rng, dim, 1.0).v, h0);
  const size_t dd = static_cast<size_t>(dim) * dim;
  for (int c = 0; c < channels; ++c) store(random_hermitian(rng, dim, 1.0).v, linear + 2 * dd * c);
  if (quadratic)
    for (int c = 0; c < channels; ++c) store(random_hermitian(rng, dim, 0.5).v, quadratic_out + 2 * dd * c);
  store(random_state(rng, dim), initial);
  store(random_state(rng, dim), target);
  if (random_penalty) {
    std::uniform_real_distribution<double> a(0.0, alpha);
    for (int j = 0; j < steps; ++j) penalty_out[j] = a(rng);
  } else {
    for (int j = 0; j < steps; ++j) penalty_out[j] = alpha;
  }
  std::uniform_real_distribution<double> uc(-control_amplitude, control_amplitude);
  for (int c = 0; c < channels; ++c)
    for (int j = 0; j < steps; ++j) control[c + static_cast<size_t>(j) * channels] = uc(rng);
  return QOC_OK;
}

extern "C" int32_t oracle_strang_fixture(uint32_t seed, int32_t points, double x_min, double x_max,
                                         int32_t steps, double control_amplitude, double* initial,
                                         double* target, double* control) {
  std::mt19937 rng(seed);  // fixtures.hpp:208-234
  const double dx = (x_max - x_min) / points;
  CV a = random_state(rng, points);
  CV b = random_state(rng, points);
  const double s = std::sqrt(dx);
  for (cd& v : a) v /= s;
  for (cd& v : b) v /= s;
  store(a, initial);
  store(b, target);
  std::uniform_real_distribution<double> uc(-control_amplitude, control_amplitude);
  for (int j = 0; j < steps; ++j) control[j] = uc(rng);
  return QOC_OK;
}

extern "C" int32_t oracle_rng(void* state, int32_t init, uint32_t seed, int32_t what, int32_t n,
                              double scale, double* out) {
  static_assert(sizeof(std::mt19937) <= 5000, "rng state buffer too small");
  auto* rng = static_cast<std::mt19937*>(state);
  if (init) new (rng) std::mt19937(seed);
  if (what == 0) store(random_cvec(*rng, n), out);
  else if (what == 1) store(random_state(*rng, n), out);
  else if (what == 2) store(random_hermitian(*rng, n, scale).v, out);
  return QOC_OK;
}
