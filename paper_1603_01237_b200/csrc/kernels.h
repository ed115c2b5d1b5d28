// kernels.h — launchers exported by the kernel translation units to the host driver.
#pragma once

#include "common.cuh"

namespace qoc {

// dense (d <= 32)
int dense_pad(int d);
cudaError_t dense_task(const DevProblem& P, const DevRun& R, const TaskArgs& A, int ignore_done, cudaStream_t st);
cudaError_t dense_horizon(const DevProblem& P, const DevRun& R, int which, int k, cudaStream_t st);

// dense 32 < d <= 64 (CTA per task, dense_big.cu)
bool dense_big_supported(int d);
cudaError_t dense_big_task(const DevProblem& P, const DevRun& R, const TaskArgs& A, int ignore_done, cudaStream_t st);
cudaError_t dense_big_horizon(const DevProblem& P, const DevRun& R, int which, int k, cudaStream_t st);

// density-matrix conjugation kind, dm <= 32 (CTA per task, dense_big.cu)
bool density_supported(int dm);
cudaError_t density_task(const DevProblem& P, const DevRun& R, const TaskArgs& A, int ignore_done, cudaStream_t st);
cudaError_t density_horizon(const DevProblem& P, const DevRun& R, int which, int k, cudaStream_t st);
// boundary chain of the assembled plan: rho_{n+1} = P_n rho_n P_n^dag, X_n = P_n^dag X_{n+1} P_n
cudaError_t density_chain(const DevProblem& P, const DevRun& R, cudaStream_t st);

// tridiagonal (d <= 32)
cudaError_t tridiag_task(const DevProblem& P, const DevRun& R, const TaskArgs& A, int ignore_done, cudaStream_t st);
cudaError_t tridiag_horizon(const DevProblem& P, const DevRun& R, int which, int k, cudaStream_t st);

// bit-flip spin register (d = 2^n, n <= 12)
cudaError_t bitflip_task(const DevProblem& P, const DevRun& R, const TaskArgs& A, int ignore_done, cudaStream_t st);
cudaError_t bitflip_horizon(const DevProblem& P, const DevRun& R, int which, int k, cudaStream_t st);
// node sweeps over the interior of blocks [SR.g0, SR.g0 + SR.nloc) of the blocked plan
cudaError_t bitflip_horizon_range(const DevProblem& P, const DevRun& R, int which, int k, const SweepRange& SR,
                                  cudaStream_t st);
// block products P_g, g in [g0, g0 + nloc), into the exchange slab (column-major)
cudaError_t bitflip_block_products(const DevProblem& P, const DevRun& R, const DevBlocks& BK, int g0, int nloc,
                                   cudaStream_t st);

// blocked plan glue (blocks.cu)
cudaError_t block_chain(const DevProblem& P, const DevRun& R, const DevBlocks& BK, cudaStream_t st);
cudaError_t slab_pack(const DevProblem& P, const DevRun& R, const DevBlocks& BK, int with_controls, cudaStream_t st);
cudaError_t slab_unpack(const DevProblem& P, const DevRun& R, const DevBlocks& BK, int with_controls,
                        cudaStream_t st);
cudaError_t exact_from_nodes(const DevProblem& P, const DevRun& R, int k, cudaStream_t st);

// split-step condensate
cudaError_t strang_task(const DevProblem& P, const DevRun& R, const TaskArgs& A, int ignore_done, cudaStream_t st);
cudaError_t strang_horizon(const DevProblem& P, const DevRun& R, int which, int k, cudaStream_t st);

// stationary states of the condensate by imaginary-time splitting (models.cpp:146-182), one CTA
// per state; psi_io [states][d], lower [states][nlower][d]
cudaError_t strang_imaginary_time(const DevProblem& P, int states, const double* u_frozen, double tau, double tol,
                                  int max_iter, int nlower, const double2* lower, const double* kin,
                                  const double2* half_kin, double2* psi_io, double* energy_out, int* iter_out,
                                  cudaStream_t st);

// propagator-cache engine for the linear kinds (d <= 32)
int pc_nchunk(const DevProblem& P, const DevRun& R);
cudaError_t pc_eval(const DevProblem& P, const DevRun& R, const TaskArgs& A, int ignore_done, cudaStream_t st);
// residual_form >= 0: the assembly sweep also writes the tasks' residual err[b][n] at the new
// control (objective form residual_form) when the path fuses it; pc_fuses_residual tells the
// driver to skip its separate residual evaluation
cudaError_t pc_assemble(const DevProblem& P, const DevRun& R, int ignore_done, cudaStream_t st,
                        int residual_form = -1);
bool pc_fuses_residual(const DevProblem& P, const DevRun& R);
constexpr int PCM_ENTRY = 1, PCM_GRAD = 2, PCM_ERR = 4, PCM_LAG = 8, PCM_FINAL = 16, PCM_RAWGRAD = 32;

// Neumann-in-the-control assembly for dense d = 16, C = 1, linear control (dense_nm.cu)
constexpr int NM_TERMS = 16;
bool dense_nm_applicable(const DevProblem& P);
cudaError_t dense_nm_setup(const DevProblem& P, const DevRun& R, cudaStream_t st);
cudaError_t dense_nm_assemble(const DevProblem& P, const DevRun& R, int ignore_done, int residual, cudaStream_t st);
bool dense_pc_eval16_applicable(const DevProblem& P, const DevRun& R, int mode, int nchunk);
cudaError_t dense_pc_eval16(const DevProblem& P, const DevRun& R, const TaskArgs& A, int ignore_done, cudaStream_t st,
                            int handed_off_only = 0, int dual = 0);
// One-pass iteration (dense_nm.cu): dual = 1 evaluates the residual of the saved tasks and the
// entry value + pending update of the current tasks in one cache pass; dual = 2 only the latter.
cudaError_t pc_eval_dual(const DevProblem& P, const DevRun& R, int form, int weighted, double rho, int dual,
                         cudaStream_t st);

// inner solvers other than the gradient update (solvers.cu, dense_big.cu)
//   Newton (every kind): begin after a raw-gradient launch into N.g0, then rounds of
//   [task(M_GRAD) at N.up -> N.gp, task(M_GRAD) at N.um -> N.gm, newton_advance]; N.active[round]
//   counts the tasks still iterating; newton_apply writes u += d (or the gradient fallback).
cudaError_t newton_begin(const DevProblem& P, const DevRun& R, const DevNewton& N, cudaStream_t st);
cudaError_t newton_advance(const DevProblem& P, const DevRun& R, const DevNewton& N, int round, cudaStream_t st);
cudaError_t newton_apply(const DevProblem& P, const DevRun& R, const DevNewton& N, cudaStream_t st);
//   Monotonic slice-rebuilding sweep (optimizers.cpp:109-213): DENSE kind, d <= 64, one channel;
//   stats[b][n][0] += guard rejections
bool monotonic_supported(const DevProblem& P);
cudaError_t monotonic_sweep(const DevProblem& P, const DevRun& R, int weighted, double fp_tol, int fp_max_iter,
                            int* stats, cudaStream_t st);

// glue (kind independent)
cudaError_t penalty_partials(const DevProblem& P, const DevRun& R, int ignore_done, cudaStream_t st);
cudaError_t merge_iteration(const DevProblem& P, const DevRun& R, int k, double* tot_err, cudaStream_t st);
cudaError_t chain_propagators(const DevProblem& P, const DevRun& R, cudaStream_t st);
cudaError_t split_nodes(const DevProblem& P, const DevRun& R, cudaStream_t st);
cudaError_t boundary_update(const DevProblem& P, const DevRun& R, int k, int split, int boot, cudaStream_t st);
cudaError_t set_single_tasks(const DevProblem& P, const DevRun& R, cudaStream_t st);
cudaError_t finish_iteration(const DevProblem& P, const DevRun& R, int k, const double* tot_err, int compute_error,
                             double eta, cudaStream_t st);
cudaError_t finish_iteration_ex(const DevProblem& P, const DevRun& R, int k, int compute_error, double eta,
                                int log_exact, cudaStream_t st);
// one-pass iteration glue: u += rho R.gpend, the task backup S_k -> R.old_*, and R.tot_err
cudaError_t apply_pending(const DevProblem& P, const DevRun& R, double rho, cudaStream_t st);
cudaError_t save_tasks(const DevProblem& P, const DevRun& R, cudaStream_t st);
cudaError_t total_error(const DevProblem& P, const DevRun& R, cudaStream_t st);
cudaError_t trailing_values(const DevProblem& P, const DevRun& R, cudaStream_t st);

}  // namespace qoc
