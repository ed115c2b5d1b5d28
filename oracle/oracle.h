/*
 * oracle.h — CPU restatement of the reference ISM hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Nothing in the product (paper_1603_01237_b200/) links,
 * loads or calls this library; only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference leg use it, and only as the checker or the timed
 * CPU baseline.  It follows /root/reference/proj/core/src/{ism,objective,optimizers,
 * propagation,controls,linalg,models,runtime}.cpp (cited per function in oracle.cpp)
 * and takes the same qoc_problem_v1 / qoc_ism_config_v1 / qoc_solver_v1 structs as the
 * device library, so both sides read identical inputs.
 *
 * Parity pins (tests/test_oracle_kats.py): KAT-1..8 and the Theorem/N-invariance/
 * finite-difference/adjointness properties of SURVEY.md §8(c), plus the reference's own
 * seeded test fixtures regenerated with the same std::mt19937 draws (fixtures.hpp).
 */
#ifndef QOC_ORACLE_H_
#define QOC_ORACLE_H_

#include "qoc_gpu.h"

#ifdef __cplusplus
extern "C" {
#endif

/* Arithmetic of the linear one-step solve.
 *   REFERENCE : dense partial-pivot LU of (I + i dt/2 H) every step, like Eigen::PartialPivLU
 *               in propagation.cpp:85-106,236-249 (all linear kinds; BITFLIP only for d <= 512).
 *   STRUCTURED: same Cayley map, structured solve - Thomas for TRIDIAG (no pivot is ever
 *               taken; asserted), Jacobi-preconditioned fixed point to fp64 convergence for
 *               BITFLIP (the "Taylor"/Neumann series of (I + iA)^-1).  DENSE stays LU. */
enum oracle_arith { ORACLE_ARITH_REFERENCE = 0, ORACLE_ARITH_STRUCTURED = 1 };

int32_t oracle_ism_run(const qoc_problem_v1* p, const qoc_ism_config_v1* cfg,
                       const qoc_solver_v1* solver, const double* u0, double* u_out,
                       qoc_iter_record_v1* recs, int32_t rec_cap, double* task_values,
                       qoc_run_status_v1* status, int32_t arith, int32_t threads, char* err,
                       size_t errlen);

/* Per-task InnerResult counters of the last oracle_ism_run (ism.cpp:409-411): out[3][L] =
 * guard_rejections, newton_fallbacks, gmres_iterations of batch member b, record k. */
int32_t oracle_solver_stats(int32_t b, int32_t iteration, int32_t subintervals, int32_t* out);

int32_t oracle_propagate_final(const qoc_problem_v1* p, const double* u, double* states_out,
                               int32_t arith, char* err, size_t errlen);
/* traj_out [B][K+1][d] */
int32_t oracle_propagate(const qoc_problem_v1* p, const double* u, double* traj_out,
                         int32_t arith, char* err, size_t errlen);
int32_t oracle_objective_gradient(const qoc_problem_v1* p, const double* u, int32_t form,
                                  int32_t naive, int32_t checkpoint_stride, double* value_out,
                                  double* grad_out, int32_t arith, char* err, size_t errlen);
int32_t oracle_assemble_propagator(const qoc_problem_v1* p, const double* u, double* prop_out,
                                   int32_t arith, char* err, size_t errlen);
/* One step of batch member 0 on one column state (u_col = C control values).
 * mode 0: cn_step / strang_step;  mode 1: cn_adjoint_step / strang_adjoint_step
 * (psi_j = forward state at the node for STRANG). */
int32_t oracle_step(const qoc_problem_v1* p, const double* u_col, double dt, const double* in,
                    const double* psi_j, int32_t mode, int32_t naive, double* out, int32_t arith,
                    char* err, size_t errlen);
/* Unitary DFT (linalg.cpp:15-63,99-100): inverse = 0 forward, 1 inverse. */
int32_t oracle_dft(int32_t n, const double* in, double* out, int32_t inverse);
/* verify_decomposition (ism.cpp:161-191) with the uniform decomposition of `parts`. */
int32_t oracle_verify_decomposition(const qoc_problem_v1* p, const double* u, int32_t parts,
                                    double* functional_mismatch, double* gradient_mismatch,
                                    int32_t arith, char* err, size_t errlen);
/* boundary_sweep (ism.cpp:122-129): psi_nodes, chi_nodes [L+1][d] for batch member 0,
 * decomposition given as node_index [L+1]. */
int32_t oracle_boundary_sweep(const qoc_problem_v1* p, const double* u, int32_t parts,
                              const int32_t* node_index, double* psi_nodes, double* chi_nodes,
                              int32_t arith, char* err, size_t errlen);

/* The reference test fixtures (tests/support/fixtures.hpp:19-112,208-234), regenerated with
 * the same std::mt19937 / <random> distribution calls so the draws match the reference
 * suite built with this toolchain.  Vector kind only (conjugation is out of scope).
 * Output buffers sized by the caller from the options:
 *   h0 [d*d], linear [C][d*d], quadratic [C][d*d] (if quadratic), initial [d], target [d],
 *   penalty [steps], control [C*steps]. */
int32_t oracle_dense_fixture(uint32_t seed, int32_t dim, int32_t steps, int32_t channels,
                             int32_t quadratic, double alpha, int32_t random_penalty,
                             double control_amplitude, double* h0, double* linear,
                             double* quadratic_out, double* initial, double* target,
                             double* penalty, double* control);
/* strang_fixture: initial, target [points] (unit grid norm), control [steps]. */
int32_t oracle_strang_fixture(uint32_t seed, int32_t points, double x_min, double x_max,
                              int32_t steps, double control_amplitude, double* initial,
                              double* target, double* control);
/* Random std::mt19937 draws used by individual reference tests (random_cvec / random_state /
 * random_hermitian of fixtures.hpp and propagation_test.cpp:19-25), in call order.
 * what: 0 random_cvec(n), 1 random_state(n), 2 random_hermitian(n, scale).  The rng state is
 * carried in `state` (an opaque 5000-byte buffer; call with init=1 first). */
int32_t oracle_rng(void* state, int32_t init, uint32_t seed, int32_t what, int32_t n,
                   double scale, double* out);

#ifdef __cplusplus
}
#endif

#endif /* QOC_ORACLE_H_ */
