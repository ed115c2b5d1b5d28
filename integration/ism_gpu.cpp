// ism_gpu.cpp -- the reference-side drop-in: qoc::run_ism_gpu has run_ism's
// signature (/root/reference/proj/core/include/qoc/ism.hpp:80-81) and runs the ISM outer
// iteration on the B200 through include/qoc_gpu.h.  A maintainer adds this translation unit to
// core/ and links libqoc_b200.so; run_ism dispatches to it under a build option.  It compiles
// against the reference headers unchanged (here: with the Eigen-subset shim, oracle/eigen_shim).
#include "ism_gpu.hpp"

#include <stdexcept>
#include <string>
#include <vector>

#include "qoc/models.hpp"
#include "qoc_gpu.h"

namespace qoc {
namespace {

qoc_ctx* device_context() {  // one context per host thread: contexts are not thread-safe,
  thread_local qoc_ctx* ctx = nullptr;  // distinct contexts are independent (no globals)
  if (!ctx && qoc_ctx_create(nullptr, &ctx) != QOC_OK) throw std::runtime_error("no sm_100 device for the ISM path");
  return ctx;
}

void rethrow(int32_t code, qoc_ctx* ctx) {  // ism.cpp:213-231, controls.cpp:16-18
  const std::string msg = qoc_ctx_last_error(ctx);
  switch (code) {
    case QOC_OK: return;
    case QOC_EINVAL: throw std::invalid_argument(msg);
    case QOC_ELOGIC: throw std::logic_error(msg);
    default: throw std::runtime_error(msg);
  }
}

int32_t solver_kind(SolverSpec::Kind k) {  // all three inner solvers run on the device
  switch (k) {
    case SolverSpec::Kind::gradient: return QOC_SOLVER_GRADIENT;
    case SolverSpec::Kind::monotonic: return QOC_SOLVER_MONOTONIC;
    case SolverSpec::Kind::newton: return QOC_SOLVER_NEWTON;
  }
  return -1;
}

const char* solver_name(SolverSpec::Kind k) {  // ism.cpp:86-97
  switch (k) {
    case SolverSpec::Kind::gradient: return "gradient";
    case SolverSpec::Kind::monotonic: return "monotonic";
    case SolverSpec::Kind::newton: return "newton";
  }
  return "unknown";
}

}  // namespace

IsmRun run_ism_gpu(const ControlProblem& p, const ControlField& u0, const IsmConfig& cfg, const SolverSpec& solver) {
  if (!p.model) throw std::invalid_argument("problem has no model");  // ism.cpp:213
  const HamiltonianModel& m = *p.model;
  const int d = m.state_dim(), C = m.channels(), K = p.grid.steps;
  qoc_problem_v1 q{};
  q.abi_version = QOC_ABI_VERSION;
  q.dim = d;
  q.channels = C;
  q.steps = K;
  q.batch = 1;
  q.t_start = p.grid.t_start;
  q.dt = p.grid.dt;
  q.ip_weight = m.ip_weight();
  // keep-alive buffers of the operator payload
  CMat h0;
  std::vector<Complex> lin, quad;
  std::vector<double> grid_x, pot_basis, pot_param;
  std::vector<int32_t> pot_type;
  switch (m.kind()) {
    case PropagatorKind::cn_dense:
    case PropagatorKind::cn_conjugation: {  // same DenseModel payload; states are d x d matrices
      // DenseModel members are private (models.hpp:26-30): H0 = H(0), A_c = dH/du_c(0),
      // B_c = dH/du_c(e_c) - A_c, the extraction optimizers.cpp:124-138 already uses
      const RVec zero = RVec::Zero(C);
      h0 = m.hamiltonian(zero);
      lin.resize(size_t(C) * d * d);
      quad.resize(size_t(C) * d * d);
      bool any_quad = false;
      for (int c = 0; c < C; ++c) {
        RVec e = RVec::Zero(C);
        e[c] = 1.0;
        const CMat a = m.control_derivative(c, zero);
        const CMat b = m.control_derivative(c, e) - a;
        std::copy(a.data(), a.data() + size_t(d) * d, lin.begin() + size_t(c) * d * d);
        std::copy(b.data(), b.data() + size_t(d) * d, quad.begin() + size_t(c) * d * d);
        for (Eigen::Index i = 0; i < b.size(); ++i) any_quad = any_quad || b.data()[i] != Complex(0.0, 0.0);
      }
      q.kind = m.kind() == PropagatorKind::cn_conjugation ? QOC_KIND_DENSITY : QOC_KIND_DENSE;
      q.h0 = reinterpret_cast<const double*>(h0.data());
      q.linear = reinterpret_cast<const double*>(lin.data());
      q.quadratic = any_quad ? reinterpret_cast<const double*>(quad.data()) : nullptr;
      break;
    }
    case PropagatorKind::strang: {
      q.kind = QOC_KIND_STRANG;
      q.kinetic = m.kinetic_spectrum().data();
      q.kappa = m.nonlinearity();
      if (const auto* tc = dynamic_cast<const TrappedCondensateModel*>(&m)) {
        q.grid_x = tc->grid_points().data();
        q.potential = QOC_POT_TRAP;
        q.pot_params[0] = tc->trap_distance();
      } else if (const auto* pb = dynamic_cast<const DevicePotentialBasis*>(&m)) {
        // a user-defined potential in separable form (ism_gpu.hpp)
        const std::vector<PotentialTerm> terms = pb->potential_terms();
        if (terms.empty() || terms.size() > QOC_MAX_POT_TERMS)
          throw std::logic_error("between 1 and QOC_MAX_POT_TERMS potential terms are supported");
        pot_basis.resize(terms.size() * size_t(d));
        for (size_t t = 0; t < terms.size(); ++t) {
          if (terms[t].profile.size() != d) throw std::invalid_argument("potential profile length != grid size");
          std::copy(terms[t].profile.data(), terms[t].profile.data() + d, pot_basis.begin() + t * size_t(d));
          pot_type.push_back(static_cast<int32_t>(terms[t].kind));
          pot_param.push_back(terms[t].parameter);
        }
        q.grid_x = pb->potential_grid().data();
        q.potential = QOC_POT_BASIS;
        q.pot_terms = static_cast<int32_t>(terms.size());
        q.pot_term_type = pot_type.data();
        q.pot_term_param = pot_param.data();
        q.pot_basis = pot_basis.data();
      } else {
        throw std::logic_error("split-step model without a device potential payload: derive from "
                               "qoc::DevicePotentialBasis (integration/ism_gpu.hpp)");
      }
      break;
    }
  }
  q.initial = reinterpret_cast<const double*>(p.initial.data());
  q.target = reinterpret_cast<const double*>(p.target.data());
  q.penalty = p.penalty.values.empty() ? nullptr : p.penalty.values.data();

  qoc_ism_config_v1 c{};
  c.subintervals = cfg.subintervals;
  c.workers = cfg.workers;
  c.max_outer = cfg.max_outer;
  c.variant = cfg.variant == IsmConfig::Variant::split ? QOC_VARIANT_SPLIT : QOC_VARIANT_INTERPOLATED;
  c.plan = cfg.plan == IsmConfig::BoundaryPlan::direct ? QOC_PLAN_DIRECT : QOC_PLAN_ASSEMBLED;
  c.compute_error = cfg.compute_error;
  c.log_exact_objective = cfg.log_exact_objective;
  c.checkpoint_stride = cfg.checkpoint_stride;
  c.eta = cfg.eta;
  c.partition = QOC_PARTITION_UNIFORM;  // Decomposition::uniform (ism.cpp:234)

  qoc_solver_v1 s{};
  s.kind = solver_kind(solver.kind);
  s.inner_iterations = solver.inner_iterations;
  s.naive_nonlinear_adjoint = solver.gradient.naive_nonlinear_adjoint;
  s.checkpoint_stride = solver.gradient.checkpoint_stride;
  s.step_size = solver.step_size;
  s.fixed_point_tol = solver.fixed_point_tol;
  s.fixed_point_max_iter = solver.fixed_point_max_iter;
  s.gmres_restart = solver.gmres_restart;
  s.gmres_max_iter = solver.gmres_max_iter;
  s.gmres_tol = solver.gmres_tol;
  s.hvp_scale = solver.hvp_scale;

  if (u0.channels() != C || u0.steps() != K)
    throw std::invalid_argument("initial control grid/channel count does not match the problem");
  ControlField out = u0;
  const int cap = std::max(cfg.max_outer, 0) + 1;
  std::vector<qoc_iter_record_v1> recs(static_cast<size_t>(cap));
  std::vector<double> tv(size_t(cap) * std::max(cfg.subintervals, 1));
  qoc_run_status_v1 st{};
  qoc_ctx* ctx = device_context();
  rethrow(qoc_ism_run(ctx, &q, &c, &s, u0.samples().data(), out.samples().data(), recs.data(), cap, tv.data(), &st),
          ctx);

  IsmRun run{out, {}};
  run.record.subintervals = cfg.subintervals;  // ism.cpp:245-249
  run.record.workers = cfg.workers;
  run.record.solver = solver_name(solver.kind);
  run.record.variant = cfg.variant == IsmConfig::Variant::split ? "split" : "interpolated";
  run.record.plan = cfg.plan == IsmConfig::BoundaryPlan::direct ? "direct" : "assembled";
  for (int k = 0; k < st.iterations_recorded; ++k) {  // RunRecord (runtime.hpp:44-75)
    IterationStat it;
    it.iteration = recs[k].iteration;
    it.objective = recs[k].objective;
    if (recs[k].has_error) it.error = recs[k].error;
    if (recs[k].has_exact_objective) it.exact_objective = recs[k].exact_objective;
    it.task_values.assign(tv.begin() + size_t(k) * cfg.subintervals, tv.begin() + size_t(k + 1) * cfg.subintervals);
    it.critical_path_seconds = recs[k].device_seconds;  // device time of the iteration
    it.wall_seconds = recs[k].device_seconds;
    // inner-solver events of the iteration's tasks (ism.cpp:503-511)
    std::vector<int32_t> counters(size_t(3) * std::max(cfg.subintervals, 1));
    if (k > 0 && qoc_ctx_solver_stats(ctx, 0, k, cfg.subintervals, counters.data()) == QOC_OK) {
      const int L = cfg.subintervals;
      for (int n = 0; n < L; ++n) {
        if (counters[n] > 0)
          it.events.push_back("task " + std::to_string(n) + ": kept " + std::to_string(counters[n]) +
                              " slices at previous values");
        if (counters[L + n] > 0)
          it.events.push_back("task " + std::to_string(n) + ": " + std::to_string(counters[L + n]) +
                              " Newton directions replaced by gradient steps");
      }
    }
    run.record.iterations.push_back(std::move(it));
  }
  run.record.aborted = st.aborted != 0;
  run.record.abort_reason = st.abort_reason;
  return run;
}

}  // namespace qoc
