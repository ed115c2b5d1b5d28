// ism_gpu.hpp -- run_ism on the B200 with the reference's signature (ism.hpp:80-81).
#pragma once
#include <vector>

#include "qoc/ism.hpp"

namespace qoc {
IsmRun run_ism_gpu(const ControlProblem& p, const ControlField& u0, const IsmConfig& cfg, const SolverSpec& solver);

// The device cannot call a model's virtual potential(u) / potential_derivative(c, u)
// (propagation.hpp:35-36) once per grid step.  A user-defined split-step model runs on the device
// by also deriving from this interface and naming its potential in the separable form
//   V(x_i, u) = sum_m profile_m[i] * f_m(u),  f_m in {u^k, cos(w u), sin(w u)}
// (qoc_gpu.h QOC_POT_BASIS).  TrappedCondensateModel needs nothing: it maps to QOC_POT_TRAP.
struct PotentialTerm {
  enum class Kind { power = 0, cosine = 1, sine = 2 };
  RVec profile;  // sampled on the model's grid
  Kind kind = Kind::power;
  double parameter = 0.0;  // exponent k, or angular frequency w
};
class DevicePotentialBasis {
 public:
  virtual ~DevicePotentialBasis() = default;
  virtual std::vector<PotentialTerm> potential_terms() const = 0;
  virtual const RVec& potential_grid() const = 0;
};
}  // namespace qoc
