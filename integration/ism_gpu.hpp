// ism_gpu.hpp -- run_ism on the B200 with the reference's signature (ism.hpp:80-81).
#pragma once
#include "qoc/ism.hpp"

namespace qoc {
IsmRun run_ism_gpu(const ControlProblem& p, const ControlField& u0, const IsmConfig& cfg, const SolverSpec& solver);
}  // namespace qoc
