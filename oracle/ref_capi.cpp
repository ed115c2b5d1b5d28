// ref_capi.cpp -- TEST INFRASTRUCTURE: a C entry point onto the REFERENCE's own run_ism.
//
// oracle/Makefile (target `ref`) compiles the reference sources where they lie
// (/root/reference/proj/core/src/{linalg,controls,propagation,objective,optimizers,ism,models,
// runtime}.cpp, unmodified) against the Eigen-subset shim in oracle/eigen_shim, plus this file,
// into oracle/_ref/libqocref.so.  The tests drive it with the same packed qoc_problem_v1 the
// device library and the restated oracle take, to pin the restatement (oracle/oracle.cpp) to
// the reference itself ("pin the oracle to the reference").
//
//   qoc::run_ism   ism.hpp:80-81 / ism.cpp:211-612   -- called as-is, one problem at a time
//   DenseModel     models.hpp:15-31                  -- DENSE; TRIDIAG and BITFLIP expanded to dense
//   TrappedCondensateModel models.hpp:40-64          -- STRANG with the trap potential
//   LatticeCondensate (below)                        -- STRANG with the BASELINE config-4 lattice
//                                                       potential, a new model behind the
//                                                       reference's HamiltonianModel plugin
//                                                       interface (propagation.hpp:20-38)
// The reference's Decomposition::uniform is kept: K % L == 0 is required here (ism.cpp:234).
#include <cmath>
#include <cstdio>
#include <cstring>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "qoc/ism.hpp"
#include "qoc/models.hpp"
#include "qoc_gpu.h"

namespace {

using qoc::CMat;
using qoc::Complex;
using qoc::RVec;

CMat load_cmat(const double* p, int d) {  // interleaved complex, column-major (the ABI layout)
  CMat m(d, d);
  for (int j = 0; j < d; ++j)
    for (int i = 0; i < d; ++i) m(i, j) = Complex(p[2 * (i + j * d)], p[2 * (i + j * d) + 1]);
  return m;
}

CMat load_state(const double* p, int d) {
  CMat m(d, 1);
  for (int i = 0; i < d; ++i) m(i, 0) = Complex(p[2 * i], p[2 * i + 1]);
  return m;
}

// V(x, u) = 0.5 w2 x^2 + v0 cos^2(k (x - u)), dV/du = v0 k sin(2 k (x - u))  (qoc_gpu.h LATTICE)
class LatticeCondensate : public qoc::HamiltonianModel {
 public:
  LatticeCondensate(const double* x, const double* kin, int n, double w2, double v0, double k, double kappa)
      : x_(n), kin_(n), w2_(w2), v0_(v0), k_(k), kappa_(kappa) {
    for (int i = 0; i < n; ++i) {
      x_[i] = x[i];
      kin_[i] = kin[i];
    }
    dx_ = n > 1 ? x[1] - x[0] : 1.0;
  }
  qoc::PropagatorKind kind() const override { return qoc::PropagatorKind::strang; }
  int state_dim() const override { return static_cast<int>(x_.size()); }
  int channels() const override { return 1; }
  double ip_weight() const override { return dx_; }
  const RVec& kinetic_spectrum() const override { return kin_; }
  RVec potential(const RVec& u) const override {
    RVec v(x_.size());
    for (Eigen::Index i = 0; i < x_.size(); ++i) {
      const double c = std::cos(k_ * (x_[i] - u[0]));
      v[i] = 0.5 * w2_ * x_[i] * x_[i] + v0_ * c * c;
    }
    return v;
  }
  RVec potential_derivative(int, const RVec& u) const override {
    RVec v(x_.size());
    for (Eigen::Index i = 0; i < x_.size(); ++i) v[i] = v0_ * k_ * std::sin(2.0 * k_ * (x_[i] - u[0]));
    return v;
  }
  double nonlinearity() const override { return kappa_; }

 private:
  RVec x_, kin_;
  double dx_, w2_, v0_, k_, kappa_;
};

// A user plugin of the reference's HamiltonianModel contract whose potential has the separable
// form V(x_i, u) = sum_m a_m[i] f_m(u) (qoc_gpu.h QOC_POT_BASIS): run by the REFERENCE's own
// strang path through its virtual potential() / potential_derivative().
class BasisCondensate : public qoc::HamiltonianModel {
 public:
  explicit BasisCondensate(const qoc_problem_v1* p) : x_(p->dim), kin_(p->dim), kappa_(p->kappa) {
    const int n = p->dim;
    for (int i = 0; i < n; ++i) {
      x_[i] = p->grid_x[i];
      kin_[i] = p->kinetic[i];
    }
    dx_ = n > 1 ? x_[1] - x_[0] : 1.0;
    for (int m = 0; m < p->pot_terms; ++m) {
      type_.push_back(p->pot_term_type[m]);
      param_.push_back(p->pot_term_param[m]);
      RVec a(n);
      for (int i = 0; i < n; ++i) a[i] = p->pot_basis[(size_t)m * n + i];
      basis_.push_back(a);
    }
  }
  qoc::PropagatorKind kind() const override { return qoc::PropagatorKind::strang; }
  int state_dim() const override { return static_cast<int>(x_.size()); }
  int channels() const override { return 1; }
  double ip_weight() const override { return dx_; }
  const RVec& kinetic_spectrum() const override { return kin_; }
  RVec potential(const RVec& u) const override { return sum(u[0], false); }
  RVec potential_derivative(int, const RVec& u) const override { return sum(u[0], true); }
  double nonlinearity() const override { return kappa_; }

 private:
  RVec sum(double u, bool deriv) const {
    RVec v = RVec::Zero(x_.size());
    for (size_t m = 0; m < basis_.size(); ++m) {
      const double q = param_[m];
      double f;
      if (type_[m] == QOC_TERM_POWER) {
        const int k = static_cast<int>(q);
        f = deriv ? (k > 0 ? k * std::pow(u, k - 1) : 0.0) : std::pow(u, k);
      } else if (type_[m] == QOC_TERM_COS) {
        f = deriv ? -q * std::sin(q * u) : std::cos(q * u);
      } else {
        f = deriv ? q * std::cos(q * u) : std::sin(q * u);
      }
      for (Eigen::Index i = 0; i < v.size(); ++i) v[i] += basis_[m][i] * f;
    }
    return v;
  }
  RVec x_, kin_;
  double dx_, kappa_;
  std::vector<int> type_;
  std::vector<double> param_;
  std::vector<RVec> basis_;
};

std::shared_ptr<const qoc::HamiltonianModel> make_model(const qoc_problem_v1* p, int b) {
  const int d = p->dim, C = p->channels;
  const size_t dd = static_cast<size_t>(d) * d;
  switch (p->kind) {
    case QOC_KIND_DENSE: {
      CMat h0 = load_cmat(p->h0 + 2 * dd * b, d);
      std::vector<CMat> lin, quad;
      for (int c = 0; c < C; ++c) lin.push_back(load_cmat(p->linear + 2 * dd * ((size_t)b * C + c), d));
      if (p->quadratic)
        for (int c = 0; c < C; ++c) quad.push_back(load_cmat(p->quadratic + 2 * dd * ((size_t)b * C + c), d));
      return std::make_shared<qoc::DenseModel>(qoc::PropagatorKind::cn_dense, h0, lin, quad);
    }
    case QOC_KIND_DENSITY: {  // the same payload, PropagatorKind::cn_conjugation (propagation.cpp:92-129)
      CMat h0 = load_cmat(p->h0 + 2 * dd * b, d);
      std::vector<CMat> lin, quad;
      for (int c = 0; c < C; ++c) lin.push_back(load_cmat(p->linear + 2 * dd * ((size_t)b * C + c), d));
      if (p->quadratic)
        for (int c = 0; c < C; ++c) quad.push_back(load_cmat(p->quadratic + 2 * dd * ((size_t)b * C + c), d));
      return std::make_shared<qoc::DenseModel>(qoc::PropagatorKind::cn_conjugation, h0, lin, quad);
    }
    case QOC_KIND_TRIDIAG: {
      const int nops = 1 + C + (p->tri_has_quadratic ? C : 0);
      std::vector<CMat> ops;
      for (int o = 0; o < nops; ++o) {
        CMat m = CMat::Zero(d, d);
        const double* dg = p->tri_diag + ((size_t)b * nops + o) * d;
        const double* sb = p->tri_sub + 2 * ((size_t)b * nops + o) * (d - 1);
        for (int j = 0; j < d; ++j) m(j, j) = dg[j];
        for (int j = 0; j + 1 < d; ++j) {
          m(j + 1, j) = Complex(sb[2 * j], sb[2 * j + 1]);
          m(j, j + 1) = std::conj(m(j + 1, j));
        }
        ops.push_back(m);
      }
      std::vector<CMat> lin(ops.begin() + 1, ops.begin() + 1 + C), quad;
      if (p->tri_has_quadratic) quad.assign(ops.begin() + 1 + C, ops.end());
      return std::make_shared<qoc::DenseModel>(qoc::PropagatorKind::cn_dense, ops[0], lin, quad);
    }
    case QOC_KIND_BITFLIP: {  // diag(h0) + sum_c sum_i coef[c][i] sigma^{axis_c}_i, spin i <-> bit n-1-i
      const int n = p->nspins;
      CMat h0 = CMat::Zero(d, d);
      for (int s = 0; s < d; ++s) h0(s, s) = p->h0[(size_t)b * d + s];
      std::vector<CMat> lin;
      for (int c = 0; c < C; ++c) {
        CMat m = CMat::Zero(d, d);
        for (int i = 0; i < n; ++i) {
          const double a = p->bf_coef[((size_t)b * C + c) * n + i];
          const int bit = n - 1 - i;
          for (int s = 0; s < d; ++s) {
            const int t = s ^ (1 << bit);
            const bool up = ((s >> bit) & 1) == 0;  // |0> = spin up
            // <t| sigma |s>: sigma_x -> 1; sigma_y -> +i if s is down (|1> -> i|0>... ) :
            // sigma_y |0> = i|1>, sigma_y |1> = -i|0>
            const Complex e = p->bf_axis[c] == 0 ? Complex(1.0, 0.0) : (up ? Complex(0.0, 1.0) : Complex(0.0, -1.0));
            m(t, s) += a * e;
          }
        }
        lin.push_back(m);
      }
      return std::make_shared<qoc::DenseModel>(qoc::PropagatorKind::cn_dense, h0, lin);
    }
    case QOC_KIND_STRANG: {
      const double x0 = p->grid_x[0], dx = p->grid_x[1] - p->grid_x[0];
      if (p->potential == QOC_POT_TRAP)
        return std::make_shared<qoc::TrappedCondensateModel>(d, x0, x0 + d * dx, p->pot_params[0], p->kappa);
      if (p->potential == QOC_POT_BASIS) return std::make_shared<BasisCondensate>(p);
      return std::make_shared<LatticeCondensate>(p->grid_x, p->kinetic, d, p->pot_params[0], p->pot_params[1],
                                                 p->pot_params[2], p->kappa);
    }
  }
  throw std::invalid_argument("unknown model kind");
}

}  // namespace

// IterationStat::events of the last ref_ism_run, newline-joined: [b][k]
static thread_local std::vector<std::vector<std::string>> g_events;

extern "C" int32_t ref_iteration_events(int32_t b, int32_t k, char* out, size_t len) {
  if (b < 0 || b >= static_cast<int>(g_events.size()) || k < 0 ||
      k >= static_cast<int>(g_events[static_cast<size_t>(b)].size()) || !out || !len)
    return QOC_EINVAL;
  std::snprintf(out, len, "%s", g_events[static_cast<size_t>(b)][static_cast<size_t>(k)].c_str());
  return QOC_OK;
}

// The reference's own ground_state (models.cpp:129-294) on a TrappedCondensateModel.
extern "C" int32_t ref_ground_state(int32_t points, double x_min, double x_max, double distance, double kappa,
                                    double u_frozen, double imaginary_dt, double energy_tol, int32_t max_iterations,
                                    double* psi_out, double* scalars_out /* energy, mu, residual, iterations */) {
  try {
    const qoc::TrappedCondensateModel m(points, x_min, x_max, distance, kappa);
    RVec u(1);
    u << u_frozen;
    const qoc::StationaryState s = qoc::ground_state(m, u, imaginary_dt, energy_tol, max_iterations);
    for (int i = 0; i < points; ++i) {
      psi_out[2 * i] = s.psi[i].real();
      psi_out[2 * i + 1] = s.psi[i].imag();
    }
    scalars_out[0] = s.energy;
    scalars_out[1] = s.chemical_potential;
    scalars_out[2] = s.residual;
    scalars_out[3] = s.iterations;
    return QOC_OK;
  } catch (const std::exception&) {
    return QOC_ERUNTIME;
  }
}

extern "C" int32_t ref_ism_run(const qoc_problem_v1* p, const qoc_ism_config_v1* cfg, const qoc_solver_v1* sv,
                               const double* u0, double* u_out, qoc_iter_record_v1* recs, int32_t rec_cap,
                               double* task_values, qoc_run_status_v1* status, char* err, size_t errlen) {
  try {
    const int d = p->dim, C = p->channels, K = p->steps, L = cfg->subintervals;
    for (int b = 0; b < p->batch; ++b) {
      qoc::ControlProblem prob;
      prob.model = make_model(p, b);
      prob.grid = qoc::TimeGrid{p->t_start, p->dt, K};
      if (p->kind == QOC_KIND_DENSITY) {  // d x d matrix states, column-major
        prob.initial = load_cmat(p->initial + 2 * (size_t)d * d * b, d);
        prob.target = load_cmat(p->target + 2 * (size_t)d * d * b, d);
      } else {
        prob.initial = load_state(p->initial + 2 * (size_t)d * b, d);
        prob.target = load_state(p->target + 2 * (size_t)d * b, d);
      }
      prob.penalty.values.assign(K, 0.0);
      if (p->penalty) prob.penalty.values.assign(p->penalty, p->penalty + K);
      qoc::RMat samples(C, K);
      for (int j = 0; j < K; ++j)
        for (int c = 0; c < C; ++c) samples(c, j) = u0[(size_t)b * K * C + (size_t)j * C + c];
      qoc::IsmConfig ic;
      ic.subintervals = L;
      ic.workers = cfg->workers;
      ic.eta = cfg->eta;
      ic.max_outer = cfg->max_outer;
      ic.variant = cfg->variant == QOC_VARIANT_SPLIT ? qoc::IsmConfig::Variant::split
                                                      : qoc::IsmConfig::Variant::interpolated;
      ic.plan = cfg->plan == QOC_PLAN_DIRECT ? qoc::IsmConfig::BoundaryPlan::direct
                                             : qoc::IsmConfig::BoundaryPlan::assembled;
      ic.compute_error = cfg->compute_error != 0;
      ic.log_exact_objective = cfg->log_exact_objective != 0;
      ic.checkpoint_stride = cfg->checkpoint_stride;
      qoc::SolverSpec spec;
      spec.kind = sv->kind == QOC_SOLVER_MONOTONIC ? qoc::SolverSpec::Kind::monotonic
                  : sv->kind == QOC_SOLVER_NEWTON  ? qoc::SolverSpec::Kind::newton
                                                   : qoc::SolverSpec::Kind::gradient;
      spec.fixed_point_tol = sv->fixed_point_tol;
      spec.fixed_point_max_iter = sv->fixed_point_max_iter;
      spec.gmres_restart = sv->gmres_restart;
      spec.gmres_max_iter = sv->gmres_max_iter;
      spec.gmres_tol = sv->gmres_tol;
      spec.hvp_scale = sv->hvp_scale;
      spec.step_size = sv->step_size;
      spec.inner_iterations = sv->inner_iterations;
      spec.gradient.naive_nonlinear_adjoint = sv->naive_nonlinear_adjoint != 0;
      spec.gradient.checkpoint_stride = sv->checkpoint_stride;
      const qoc::IsmRun run = qoc::run_ism(prob, qoc::ControlField(prob.grid, samples), ic, spec);
      for (int j = 0; j < K; ++j)
        for (int c = 0; c < C; ++c) u_out[(size_t)b * K * C + (size_t)j * C + c] = run.control(c, j);
      qoc_run_status_v1& st = status[b];
      std::memset(&st, 0, sizeof(st));
      st.aborted = run.record.aborted ? 1 : 0;
      std::snprintf(st.abort_reason, sizeof(st.abort_reason), "%s", run.record.abort_reason.c_str());
      if (b == 0) g_events.clear();
      g_events.emplace_back();
      for (const qoc::IterationStat& it : run.record.iterations) {
        std::string joined;
        for (const std::string& e : it.events) joined += e + "\n";
        g_events.back().push_back(joined);
      }
      const int n = std::min<int>(rec_cap, static_cast<int>(run.record.iterations.size()));
      st.iterations_recorded = n;
      for (int k = 0; k < n; ++k) {
        const qoc::IterationStat& it = run.record.iterations[static_cast<size_t>(k)];
        qoc_iter_record_v1& o = recs[(size_t)b * rec_cap + k];
        std::memset(&o, 0, sizeof(o));
        o.iteration = it.iteration;
        o.objective = it.objective;
        o.has_error = it.error.has_value();
        o.error = it.error.value_or(0.0);
        o.has_exact_objective = it.exact_objective.has_value();
        o.exact_objective = it.exact_objective.value_or(0.0);
        o.device_seconds = it.wall_seconds;  // measured wall time of the iteration (runtime.hpp:61)
        double* tv = task_values + ((size_t)b * rec_cap + k) * L;
        for (int m = 0; m < L; ++m) tv[m] = m < static_cast<int>(it.task_values.size()) ? it.task_values[m] : NAN;
      }
    }
    return QOC_OK;
  } catch (const std::invalid_argument& e) {
    std::snprintf(err, errlen, "%s", e.what());
    return QOC_EINVAL;
  } catch (const std::logic_error& e) {
    std::snprintf(err, errlen, "%s", e.what());
    return QOC_ELOGIC;
  } catch (const std::exception& e) {
    std::snprintf(err, errlen, "%s", e.what());
    return QOC_ERUNTIME;
  }
}
