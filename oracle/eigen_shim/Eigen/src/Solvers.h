// Eigen-subset shim (test infrastructure): the two decompositions the reference calls.
#pragma once

namespace Eigen {

// PartialPivLU: LU with row partial pivoting, PA = LU, L unit lower triangular -- the unblocked
// form of Eigen's partial_lu_impl: per column the pivot is the first row of largest |a_ik|
// among i >= k, rows are swapped whole, the column below the pivot is divided by it, and the
// trailing block takes the rank-1 update.
template <class M>
class PartialPivLU {
  using S = typename M::Scalar;

 public:
  PartialPivLU() = default;
  explicit PartialPivLU(const M& a) { compute(a); }
  PartialPivLU& compute(const M& a) {
    if (a.rows() != a.cols()) throw std::invalid_argument("PartialPivLU: matrix not square");
    lu_ = a;
    const Index n = a.rows();
    perm_.resize(static_cast<size_t>(n));
    for (Index i = 0; i < n; ++i) perm_[static_cast<size_t>(i)] = i;
    for (Index k = 0; k < n; ++k) {
      Index p = k;
      double best = std::abs(lu_(k, k));
      for (Index i = k + 1; i < n; ++i) {
        const double v = std::abs(lu_(i, k));
        if (v > best) {
          best = v;
          p = i;
        }
      }
      if (p != k) {
        for (Index j = 0; j < n; ++j) std::swap(lu_(k, j), lu_(p, j));
        std::swap(perm_[static_cast<size_t>(k)], perm_[static_cast<size_t>(p)]);
      }
      const S piv = lu_(k, k);
      if (piv != S(0))
        for (Index i = k + 1; i < n; ++i) lu_(i, k) /= piv;
      for (Index j = k + 1; j < n; ++j) {
        const S ukj = lu_(k, j);
        for (Index i = k + 1; i < n; ++i) lu_(i, j) -= lu_(i, k) * ukj;
      }
    }
    return *this;
  }
  const M& matrixLU() const { return lu_; }
  template <int C2, int D2>
  Matrix<S, C2> solve(const Matrix<S, C2, D2>& b) const {
    const Index n = lu_.rows();
    if (b.rows() != n) throw std::invalid_argument("PartialPivLU::solve: rhs dimension mismatch");
    Matrix<S, C2> x(n, b.cols());
    for (Index j = 0; j < b.cols(); ++j) {
      for (Index i = 0; i < n; ++i) x(i, j) = b(perm_[static_cast<size_t>(i)], j);
      for (Index i = 0; i < n; ++i) {  // L y = P b
        S acc = x(i, j);
        for (Index k = 0; k < i; ++k) acc -= lu_(i, k) * x(k, j);
        x(i, j) = acc;
      }
      for (Index i = n - 1; i >= 0; --i) {  // U x = y
        S acc = x(i, j);
        for (Index k = i + 1; k < n; ++k) acc -= lu_(i, k) * x(k, j);
        x(i, j) = acc / lu_(i, i);
      }
    }
    return x;
  }

 private:
  M lu_;
  std::vector<Index> perm_;
};

// SelfAdjointEigenSolver: cyclic complex Jacobi rotations to full convergence, eigenvalues
// ascending, eigenvectors as columns (unit norm; their phase is whatever the rotations give --
// the reference fixes phases itself where it matters, models.cpp:265-272).
template <class M>
class SelfAdjointEigenSolver {
  using S = typename M::Scalar;

 public:
  explicit SelfAdjointEigenSolver(const M& a) {
    const Index n = a.rows();
    M A = a;
    M V = M::Identity(n, n);
    for (int sweep = 0; sweep < 100; ++sweep) {
      double off = 0.0, tot = 0.0;
      for (Index j = 0; j < n; ++j)
        for (Index i = 0; i < n; ++i) {
          const double v = internal::abs2_(A(i, j));
          tot += v;
          if (i != j) off += v;
        }
      if (off <= 1e-32 * tot || off == 0.0) break;
      for (Index p = 0; p < n; ++p)
        for (Index q = p + 1; q < n; ++q) {
          const S apq = A(p, q);
          const double mag = std::abs(apq);
          if (mag == 0.0) continue;
          const double app = std::real(A(p, p)), aqq = std::real(A(q, q));
          // Hermitian 2x2 [[app, apq], [conj(apq), aqq]] -> real symmetric via phase e^{i phi}
          const S ph = apq / mag;
          const double theta = 0.5 * std::atan2(2.0 * mag, aqq - app);
          const double c = std::cos(theta), s = std::sin(theta);
          // rotation G on columns p, q: [c, s*ph; -s*conj(ph), c] (unitary)
          for (Index k = 0; k < n; ++k) {  // A <- A G
            const S akp = A(k, p), akq = A(k, q);
            A(k, p) = c * akp - s * internal::conj_(ph) * akq;
            A(k, q) = s * ph * akp + c * akq;
          }
          for (Index k = 0; k < n; ++k) {  // A <- G^dag A
            const S apk = A(p, k), aqk = A(q, k);
            A(p, k) = c * apk - s * ph * aqk;
            A(q, k) = s * internal::conj_(ph) * apk + c * aqk;
          }
          A(p, q) = S(0);
          A(q, p) = S(0);
          for (Index k = 0; k < n; ++k) {  // V <- V G
            const S vkp = V(k, p), vkq = V(k, q);
            V(k, p) = c * vkp - s * internal::conj_(ph) * vkq;
            V(k, q) = s * ph * vkp + c * vkq;
          }
        }
    }
    std::vector<Index> order(static_cast<size_t>(n));
    for (Index i = 0; i < n; ++i) order[static_cast<size_t>(i)] = i;
    std::stable_sort(order.begin(), order.end(),
                     [&](Index x, Index y) { return std::real(A(x, x)) < std::real(A(y, y)); });
    values_ = VectorXd(n);
    vectors_ = M(n, n);
    for (Index k = 0; k < n; ++k) {
      const Index src = order[static_cast<size_t>(k)];
      values_[k] = std::real(A(src, src));
      for (Index i = 0; i < n; ++i) vectors_(i, k) = V(i, src);
    }
  }
  ComputationInfo info() const { return Success; }
  const VectorXd& eigenvalues() const { return values_; }
  const M& eigenvectors() const { return vectors_; }

 private:
  VectorXd values_;
  M vectors_;
};

}  // namespace Eigen
