// dropin_check.cpp -- the drop-in exercised end to end, in one process: the reference's own
// problem builders and run_ism (compiled from /root/reference by oracle/Makefile `ref`) against
// run_ism_gpu (ism_gpu.cpp -> libqoc_b200.so) on the same inputs.  Prints one JSON line per case
// and exits non-zero on any mismatch.  Built here (integration/Makefile); run on the GPU box by
// tests/test_gpu_dropin.py.
#include <cmath>
#include <cstdio>
#include <functional>
#include <stdexcept>
#include <string>

#include "ism_gpu.hpp"
#include "qoc/models.hpp"

using namespace qoc;

static bool compare(const char* name, const IsmRun& ref, const IsmRun& gpu, double ctl_tol, double obj_tol) {
  const RMat& a = ref.control.samples();
  const RMat& b = gpu.control.samples();
  double du = 0.0, scale = 1e-300, dobj = 0.0, dex = 0.0;
  for (Eigen::Index i = 0; i < a.size(); ++i) {
    du = std::max(du, std::abs(a.data()[i] - b.data()[i]));
    scale = std::max(scale, std::abs(a.data()[i]));
  }
  const size_t n = std::min(ref.record.iterations.size(), gpu.record.iterations.size());
  for (size_t k = 0; k < n; ++k) {
    const auto& x = ref.record.iterations[k];
    const auto& y = gpu.record.iterations[k];
    // absolute for O(1) payoffs, relative once the penalty term dominates
    if (std::isfinite(x.objective))
      dobj = std::max(dobj, std::abs(x.objective - y.objective) / std::max(1.0, std::abs(x.objective)));
    if (x.exact_objective && y.exact_objective)
      dex = std::max(dex, std::abs(*x.exact_objective - *y.exact_objective) / std::max(1.0, std::abs(*x.exact_objective)));
  }
  const bool same_len = ref.record.iterations.size() == gpu.record.iterations.size();
  const bool meta = ref.record.solver == gpu.record.solver && ref.record.variant == gpu.record.variant &&
                    ref.record.plan == gpu.record.plan && ref.record.subintervals == gpu.record.subintervals;
  const bool ok = same_len && meta && du / scale <= ctl_tol && dobj <= obj_tol && dex <= obj_tol;
  std::printf("{\"case\": \"%s\", \"iterations\": %zu, \"control_rel\": %.3e, \"objective_abs\": %.3e, "
              "\"exact_abs\": %.3e, \"record_metadata_equal\": %s, \"ok\": %s}\n",
              name, ref.record.iterations.size(), du / scale, dobj, dex, meta ? "true" : "false", ok ? "true" : "false");
  return ok;
}

template <class F>
static bool throws_logic(const char* name, F&& f) {
  bool ok = false;
  std::string what;
  try {
    f();
  } catch (const std::logic_error& e) {
    ok = dynamic_cast<const std::invalid_argument*>(&e) == nullptr;
    what = e.what();
  } catch (const std::exception& e) {
    what = e.what();
  }
  std::printf("{\"case\": \"%s\", \"throws\": \"std::logic_error\", \"what\": \"%s\", \"ok\": %s}\n", name,
              what.c_str(), ok ? "true" : "false");
  return ok;
}

// A user plugin: a condensate in a tilted, breathing trap.  The reference steps it through its
// virtual potential()/potential_derivative(); the device reads the separable form.
class TiltedTrap : public HamiltonianModel, public DevicePotentialBasis {
 public:
  TiltedTrap(int n, double x_min, double x_max, double kappa) : x_(n), kin_(n), kappa_(kappa) {
    const double len = x_max - x_min;
    dx_ = len / n;
    const double pi = std::acos(-1.0);
    for (int i = 0; i < n; ++i) {
      x_[i] = x_min + i * dx_;
      const int f = i <= n / 2 ? i : i - n;
      const double k = 2.0 * pi * f / len;
      kin_[i] = 0.5 * k * k;
    }
  }
  PropagatorKind kind() const override { return PropagatorKind::strang; }
  int state_dim() const override { return static_cast<int>(x_.size()); }
  int channels() const override { return 1; }
  double ip_weight() const override { return dx_; }
  const RVec& kinetic_spectrum() const override { return kin_; }
  double nonlinearity() const override { return kappa_; }
  RVec potential(const RVec& u) const override {  // x^2/2 + 0.3 x u + 0.05 x^2 u^2 + 0.4 sin(1.3 u) cos(x)
    RVec v(x_.size());
    for (Eigen::Index i = 0; i < x_.size(); ++i)
      v[i] = 0.5 * x_[i] * x_[i] + 0.3 * x_[i] * u[0] + 0.05 * x_[i] * x_[i] * u[0] * u[0] +
             0.4 * std::sin(1.3 * u[0]) * std::cos(x_[i]);
    return v;
  }
  RVec potential_derivative(int, const RVec& u) const override {
    RVec v(x_.size());
    for (Eigen::Index i = 0; i < x_.size(); ++i)
      v[i] = 0.3 * x_[i] + 0.1 * x_[i] * x_[i] * u[0] + 0.4 * 1.3 * std::cos(1.3 * u[0]) * std::cos(x_[i]);
    return v;
  }
  std::vector<PotentialTerm> potential_terms() const override {
    const Eigen::Index n = x_.size();
    RVec a(n), b(n), c(n), e(n);
    for (Eigen::Index i = 0; i < n; ++i) {
      a[i] = 0.5 * x_[i] * x_[i];
      b[i] = 0.3 * x_[i];
      c[i] = 0.05 * x_[i] * x_[i];
      e[i] = 0.4 * std::cos(x_[i]);
    }
    return {{a, PotentialTerm::Kind::power, 0.0}, {b, PotentialTerm::Kind::power, 1.0},
            {c, PotentialTerm::Kind::power, 2.0}, {e, PotentialTerm::Kind::sine, 1.3}};
  }
  const RVec& potential_grid() const override { return x_; }

 private:
  RVec x_, kin_;
  double dx_ = 1.0, kappa_;
};

int main() {
  bool all = true;
  {  // BASELINE config 1 physics from the reference's spin operators (sigma/2): two spins
    ControlProblem p;
    const CMat h0 = 2.0 * std::acos(-1.0) * (spin_operator(2, 0, 'z') * spin_operator(2, 1, 'z'));
    const CMat hc = spin_operator(2, 0, 'x') + spin_operator(2, 1, 'x');
    p.model = std::make_shared<DenseModel>(PropagatorKind::cn_dense, h0, std::vector<CMat>{hc});
    p.grid = TimeGrid::over(0.0, 10.0, 1000);
    p.initial = CMat::Zero(4, 1);
    p.initial(0, 0) = 1.0;
    p.target = CMat::Zero(4, 1);
    p.target(3, 0) = 1.0;
    p.penalty = PenaltySchedule::constant(0.0, 1000);
    const ControlField u0 = random_control(p.grid, 1, 7u, 0.3);
    IsmConfig cfg;
    cfg.subintervals = 8;
    cfg.max_outer = 200;
    cfg.eta = 0.0;
    SolverSpec sv;
    sv.step_size = 10.0;
    all &= compare("spin2_config1_200it", run_ism(p, u0, cfg, sv), run_ism_gpu(p, u0, cfg, sv), 1e-9, 1e-10);
    cfg.plan = IsmConfig::BoundaryPlan::direct;
    cfg.max_outer = 20;
    all &= compare("spin2_direct_plan", run_ism(p, u0, cfg, sv), run_ism_gpu(p, u0, cfg, sv), 1e-9, 1e-10);
    SolverSpec mono = sv;
    mono.kind = SolverSpec::Kind::monotonic;
    // zero penalty: the monotonic sweep's precondition fails on both sides (optimizers.cpp:118-122)
    all &= throws_logic("monotonic_solver_rejected", [&] { run_ism_gpu(p, u0, cfg, mono); });
    all &= throws_logic("monotonic_solver_rejected_reference", [&] { run_ism(p, u0, cfg, mono); });
    // with a positive penalty both run the slice-rebuilding sweep; events (guard rejections) included
    p.penalty = PenaltySchedule::constant(0.05, 1000);
    cfg.plan = IsmConfig::BoundaryPlan::assembled;
    cfg.max_outer = 6;
    {
      const IsmRun a = run_ism(p, u0, cfg, mono), b = run_ism_gpu(p, u0, cfg, mono);
      bool ev = a.record.iterations.size() == b.record.iterations.size();
      for (size_t k = 0; ev && k < a.record.iterations.size(); ++k)
        ev = a.record.iterations[k].events == b.record.iterations[k].events;
      all &= compare("spin2_monotonic", a, b, 1e-9, 1e-10) && ev;
      std::printf("{\"case\": \"spin2_monotonic_events\", \"ok\": %s}\n", ev ? "true" : "false");
    }
    SolverSpec nw = sv;
    nw.kind = SolverSpec::Kind::newton;
    nw.step_size = 0.5;
    cfg.max_outer = 4;
    {
      // finite-difference Hessian products amplify rounding by ~1/hvp_scale: 1e-6 / 1e-8 bounds
      const IsmRun a = run_ism(p, u0, cfg, nw), b = run_ism_gpu(p, u0, cfg, nw);
      all &= compare("spin2_newton", a, b, 1e-6, 1e-8);
    }
  }
  {  // the reference's HCN-style rotor preset: dense, quadratic polarizability, t-dependent penalty
    ControlProblem p = rotor_problem(20, 1.0, 1.0, 0.5, 0.3, 5.0, 1024, 100.0, 1e-3);
    const ControlField u0 = random_control(p.grid, 1, 11u, 0.5);
    IsmConfig cfg;
    cfg.subintervals = 8;
    cfg.max_outer = 20;
    cfg.eta = 0.0;
    SolverSpec sv;
    sv.step_size = 0.5;
    all &= compare("rotor_preset_quadratic", run_ism(p, u0, cfg, sv), run_ism_gpu(p, u0, cfg, sv), 1e-9, 1e-10);
  }
  {  // the reference's condensate preset (KAT-8 configuration): split variant, exact payoff logged
    ControlProblem p = condensate_problem(50, -10.0, 10.0, 6.0, 1.0, 8.0, 512);
    const ControlField u0 = ramp_control(p.grid, 1.0, 0.0);
    IsmConfig cfg;
    cfg.subintervals = 4;
    cfg.max_outer = 10;
    cfg.eta = 0.0;
    cfg.variant = IsmConfig::Variant::split;
    cfg.log_exact_objective = true;
    SolverSpec sv;
    sv.step_size = 0.1;
    all &= compare("condensate_preset_kat8", run_ism(p, u0, cfg, sv), run_ism_gpu(p, u0, cfg, sv), 1e-9, 1e-10);
    sv.gradient.naive_nonlinear_adjoint = true;
    all &= compare("condensate_naive_adjoint", run_ism(p, u0, cfg, sv), run_ism_gpu(p, u0, cfg, sv), 1e-9, 1e-10);
  }
  {  // a user-defined split-step model (virtual potential on the reference side, basis form on the device)
    ControlProblem p = condensate_problem(50, -10.0, 10.0, 6.0, 1.0, 8.0, 256);  // grid, states, penalty
    p.model = std::make_shared<TiltedTrap>(50, -10.0, 10.0, 1.0);
    const ControlField u0 = ramp_control(p.grid, 1.0, 0.0);
    IsmConfig cfg;
    cfg.subintervals = 4;
    cfg.max_outer = 6;
    cfg.eta = 0.0;
    cfg.variant = IsmConfig::Variant::split;
    cfg.log_exact_objective = true;
    SolverSpec sv;
    sv.step_size = 0.1;
    all &= compare("user_potential_plugin", run_ism(p, u0, cfg, sv), run_ism_gpu(p, u0, cfg, sv), 1e-9, 1e-10);
  }
  {  // the density-matrix spin chain (cn_conjugation, the reference's `spins` preset builder)
    ControlProblem p = spin_chain_problem(3, {{1, 2}, {2, 3}}, 1.0, 1.0, 64, 0.0);
    const ControlField u0 = random_control(p.grid, p.model->channels(), 3u, 0.2);
    IsmConfig cfg;
    cfg.subintervals = 2;
    cfg.max_outer = 5;
    cfg.eta = 0.0;
    cfg.plan = IsmConfig::BoundaryPlan::direct;
    SolverSpec sv;
    sv.step_size = 0.5;
    all &= compare("density_matrix_spin_chain", run_ism(p, u0, cfg, sv), run_ism_gpu(p, u0, cfg, sv), 1e-9, 1e-10);
  }
  std::printf("{\"all_ok\": %s}\n", all ? "true" : "false");
  return all ? 0 : 1;
}
