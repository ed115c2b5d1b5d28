/*
 * qoc_gpu.h — C ABI of the B200-native ISM (Intermediate State Method) hot path.
 *
 * This is the drop-in boundary for the reference solver entry
 *
 *     IsmRun qoc::run_ism(const ControlProblem&, const ControlField& u0,
 *                         const IsmConfig&, const SolverSpec&)
 *       -- /root/reference/proj/core/include/qoc/ism.hpp:80-81, core/src/ism.cpp:211-612
 *
 * and for the helper entry points the reference exposes on the same path:
 *
 *     propagate_final        propagation.hpp:88 / propagation.cpp:194-200
 *     evaluate_objective     objective.hpp:37-40 / objective.cpp:93-105
 *     objective_gradient     objective.hpp:46-51 / objective.cpp:107-129
 *     assemble_propagator    propagation.hpp:112 / propagation.cpp:236-249
 *
 * Plain C: pointers and sizes only, caller-owned host buffers, library-owned
 * device state.  Complex arrays are interleaved (re, im) doubles in Eigen's
 * column-major order, i.e. exactly the bytes of an Eigen::MatrixXcd / VectorXcd
 * (`.data()`), so a reference-side shim passes Eigen buffers through unchanged.
 * Controls are channels x steps, column-major: sample (c, j) at c + j*C
 * (controls.hpp:54), again the bytes of the reference's RMat.
 *
 * Error behaviour mirrors the reference (ism.cpp:213-231, controls.cpp:16-18):
 *   QOC_EINVAL   <-> std::invalid_argument   (bad shapes, L < 1, eta < 0, ...)
 *   QOC_ERUNTIME <-> std::runtime_error      (decomposition errors)
 *   QOC_ELOGIC   <-> std::logic_error        (unsupported kind/plan combination)
 *   QOC_ECUDA / QOC_ENCCL                    (device / collective failures)
 * Numerical aborts are NOT errors: they return QOC_OK with status.aborted = 1
 * and the reference's reason text (ism.cpp:387,529-530,558).
 *
 * A context is bound to one device and is not thread-safe; distinct contexts
 * are independent (no globals), matching the reference's re-entrancy.
 */
#ifndef QOC_GPU_H_
#define QOC_GPU_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define QOC_ABI_VERSION 2

/* Largest control-channel count C the device kernels carry (DENSE, TRIDIAG, STRANG; the BITFLIP
 * kind takes C <= 4).  Larger C is rejected with QOC_ELOGIC before any work runs. */
#define QOC_MAX_CHANNELS 8

enum qoc_status_code {
  QOC_OK = 0,
  QOC_EINVAL = 1,
  QOC_ELOGIC = 2,
  QOC_ECUDA = 3,
  QOC_ENCCL = 4,
  QOC_ERUNTIME = 5
};

/* Operator classes.  All four implement the reference's HamiltonianModel
 * plugin contract (propagation.hpp:20-38):
 *   DENSE   - DenseModel (models.hpp:15-31): H(u) = H0 + sum u_c A_c + sum (u_c^2/2) B_c,
 *             one-step map = Cayley / Crank-Nicolson (propagation.cpp:85-90).
 *   TRIDIAG - the same model with Hermitian tridiagonal H0, A_c, B_c (rotor, models.cpp:349-359).
 *   BITFLIP - spin register: diagonal H0 plus channels sum_i coef[c][i] sigma^{axis_c}_i
 *             (Pauli matrices; spin i <-> bit (nspins-1-i) of the basis index, spin 0 most
 *             significant as in spin_operator, models.cpp:296-318).
 *   STRANG  - periodic-grid condensate, split-step Fourier (propagation.cpp:131-170),
 *             TrappedCondensateModel-style potentials (models.cpp:77-127). */
enum qoc_kind { QOC_KIND_DENSE = 0, QOC_KIND_TRIDIAG = 1, QOC_KIND_BITFLIP = 2, QOC_KIND_STRANG = 3,
                QOC_KIND_DENSITY = 4 };
/* QOC_KIND_DENSITY - DenseModel with PropagatorKind::cn_conjugation (propagation.cpp:92-129):
 *             the same H0 / A_c / B_c payload as DENSE (dim = d <= 32), but every state is a
 *             d x d matrix rho (initial / target: [B][d*d] complex, column-major) stepped as
 *             rho' = A rho A^dag, A = (I + L)^-1 (I - L); channel count up to QOC_MAX_DENSITY_CHANNELS.
 *             The boundary refresh always runs as direct node sweeps (assembled and direct agree
 *             to rounding, ism_test.cpp:248-265). */
#define QOC_MAX_DENSITY_CHANNELS 32

/* Potentials of QOC_KIND_STRANG: the device side of the reference's virtual
 * potential(u) / potential_derivative(c, u) plugin (propagation.hpp:35-36).
 *   TRAP    : models.cpp:95-127, pot_params = {trap_distance}
 *   LATTICE : V(x,u) = 0.5*w2*x^2 + v0*cos^2(k (x - u)),  dV/du = v0*k*sin(2 k (x - u)),
 *             pot_params = {w2, v0, k}  (BASELINE config 4)
 *   BASIS   : any model of the separable form V(x_i, u) = sum_m a_m[i] f_m(u),
 *             dV/du = sum_m a_m[i] f_m'(u), with pot_terms <= QOC_MAX_POT_TERMS sampled profiles
 *             pot_basis[m][i] and f_m named by pot_term_type[m] / pot_term_param[m]:
 *               QOC_TERM_POWER  f = u^k,       param = k (integer >= 0; k = 0 is the static part)
 *               QOC_TERM_COS    f = cos(w u),  param = w
 *               QOC_TERM_SIN    f = sin(w u),  param = w
 *             (shifted or modulated lattices, tilted / breathing traps, polynomial couplings). */
enum qoc_potential { QOC_POT_TRAP = 0, QOC_POT_LATTICE = 1, QOC_POT_BASIS = 2 };
enum qoc_pot_term { QOC_TERM_POWER = 0, QOC_TERM_COS = 1, QOC_TERM_SIN = 2 };
#define QOC_MAX_POT_TERMS 8

typedef struct qoc_problem_v1 {
  int32_t abi_version; /* QOC_ABI_VERSION */
  int32_t kind;        /* enum qoc_kind */
  int32_t dim;         /* state length d */
  int32_t channels;    /* C */
  int32_t steps;       /* K (TimeGrid::steps) */
  int32_t batch;       /* B independent problems sharing kind, d, C and the grid */
  double t_start;      /* TimeGrid::t_start */
  double dt;           /* TimeGrid::dt */
  double ip_weight;    /* HamiltonianModel::ip_weight(): dx for STRANG, 1 otherwise */

  /* DENSE:  h0 [B][d*d], linear [B][C][d*d], quadratic [B][C][d*d] or NULL (complex).
   * BITFLIP: h0 [B][d] REAL diagonal. */
  const double* h0;
  const double* linear;
  const double* quadratic;

  /* TRIDIAG: nops = 1 + C (+ C when tri_has_quadratic), order H0, A_0.., B_0..
   * tri_diag [B][nops][d] real diagonal; tri_sub [B][nops][d-1] complex entry (j+1, j);
   * entry (j, j+1) is its conjugate. */
  const double* tri_diag;
  const double* tri_sub;
  int32_t tri_has_quadratic;

  /* BITFLIP channels. */
  int32_t nspins;
  const int32_t* bf_axis; /* [C]: 0 = sigma_x, 1 = sigma_y */
  const double* bf_coef;  /* [B][C][nspins] */

  /* STRANG. */
  const double* kinetic; /* [d] kinetic spectrum, dft mode order (models.cpp:87-92) */
  const double* grid_x;  /* [d] grid points */
  int32_t potential;     /* enum qoc_potential */
  double pot_params[4];
  double kappa;          /* nonlinearity() */
  int32_t pot_terms;             /* QOC_POT_BASIS: number of terms M */
  int32_t pot_reserved;
  const int32_t* pot_term_type;  /* [M] enum qoc_pot_term */
  const double* pot_term_param;  /* [M] */
  const double* pot_basis;       /* [M][d] sampled profiles a_m(x_i) */

  /* States and penalty (ControlProblem, objective.hpp:18-24). */
  const double* initial; /* [B][d] complex */
  const double* target;  /* [B][d] complex */
  const double* penalty; /* [K] per-step alpha_j (shared by the batch), or NULL = 0 */
} qoc_problem_v1;

enum qoc_variant { QOC_VARIANT_INTERPOLATED = 0, QOC_VARIANT_SPLIT = 1 };
enum qoc_plan { QOC_PLAN_ASSEMBLED = 0, QOC_PLAN_DIRECT = 1 };
/* Decomposition of the K steps into L subintervals.  UNIFORM is the reference's
 * Decomposition::uniform (controls.cpp:110-120; fails with QOC_ERUNTIME when L does not
 * divide K).  BALANCED gives the first K mod L parts ceil(K/L) steps and the rest
 * floor(K/L) (identical to UNIFORM when L | K).  EXPLICIT takes node_index. */
enum qoc_partition { QOC_PARTITION_BALANCED = 0, QOC_PARTITION_UNIFORM = 1, QOC_PARTITION_EXPLICIT = 2 };

/* IsmConfig (ism.hpp:12-39). */
typedef struct qoc_ism_config_v1 {
  int32_t subintervals;        /* L */
  int32_t workers;             /* accepted for API parity; the device schedules tasks */
  int32_t max_outer;
  int32_t variant;             /* enum qoc_variant */
  int32_t plan;                /* enum qoc_plan */
  int32_t compute_error;
  int32_t log_exact_objective;
  int32_t checkpoint_stride;   /* forwarded to gradient sweeps; results are bit-identical */
  int32_t partition;           /* enum qoc_partition */
  int32_t blocks;              /* BITFLIP + ASSEMBLED: contiguous subinterval blocks G of the
                                  blocked boundary refresh (1 <= G <= L; G = L is the reference's
                                  per-subinterval chain, ism.cpp:298-312).  0 = direct node sweeps
                                  on one GPU, G = world size under a communicator.  Ignored by the
                                  other kinds. */
  double eta;
  const int32_t* node_index;   /* [L+1] for QOC_PARTITION_EXPLICIT */
} qoc_ism_config_v1;

enum qoc_solver_kind { QOC_SOLVER_GRADIENT = 0, QOC_SOLVER_MONOTONIC = 1, QOC_SOLVER_NEWTON = 2 };

/* SolverSpec (optimizers.hpp:9-30).  All three inner solvers run on the device: the
 * constant-step gradient update (optimizers.cpp:102-107), the monotonic slice-rebuilding sweep
 * (optimizers.cpp:109-213; DENSE kind, one channel, positive penalty, at most quadratic
 * control — anything else returns QOC_ELOGIC as the reference throws std::logic_error) and the
 * Newton update by restarted GMRES on finite-difference Hessian-vector products
 * (optimizers.cpp:21-98,215-259; every kind).  The fields after step_size carry the reference's
 * SolverSpec values literally (its defaults: 1e-12, 50, 30, 200, 1e-6, 1e-5). */
typedef struct qoc_solver_v1 {
  int32_t kind;                    /* enum qoc_solver_kind */
  int32_t inner_iterations;
  int32_t naive_nonlinear_adjoint; /* GradientOptions::naive_nonlinear_adjoint */
  int32_t checkpoint_stride;       /* GradientOptions::checkpoint_stride */
  double step_size;                /* rho */
  double fixed_point_tol;          /* monotonic: per-slice fixed point */
  int32_t fixed_point_max_iter;
  int32_t gmres_restart;           /* newton */
  int32_t gmres_max_iter;
  int32_t reserved;
  double gmres_tol;
  double hvp_scale;
} qoc_solver_v1;

/* IterationStat (runtime.hpp:44-63), one per recorded iteration (entry 0 = bootstrap). */
typedef struct qoc_iter_record_v1 {
  int32_t iteration;
  int32_t has_error;
  int32_t has_exact_objective;
  int32_t reserved;
  double objective;        /* NaN where the reference records NaN */
  double exact_objective;
  double error;
  double device_seconds;   /* CUDA-event time of this iteration's device work */
} qoc_iter_record_v1;

/* RunRecord abort state (runtime.hpp:65-75), per batch member. */
typedef struct qoc_run_status_v1 {
  int32_t aborted;
  int32_t iterations_recorded;
  char abort_reason[240];
} qoc_run_status_v1;

typedef struct qoc_ctx qoc_ctx;

typedef struct qoc_ctx_opts_v1 {
  int32_t abi_version;
  int32_t device;   /* CUDA ordinal, -1 = current */
  int32_t reserved[6];
} qoc_ctx_opts_v1;

int32_t qoc_abi_version(void);
int32_t qoc_ctx_create(const qoc_ctx_opts_v1* opts, qoc_ctx** out);
void qoc_ctx_destroy(qoc_ctx* ctx);
/* Text of the last error raised on this context (empty when none). */
const char* qoc_ctx_last_error(const qoc_ctx* ctx);

/* run_ism over a batch of B independent problems.
 *   u0, u_out     [B][C*K]
 *   recs          [B][rec_cap]   (rec_cap >= max_outer + 1)
 *   task_values   [B][rec_cap][L] or NULL  (IterationStat::task_values)
 *   status        [B]
 * Returns an enum qoc_status_code; the message is in qoc_ctx_last_error. */
int32_t qoc_ism_run(qoc_ctx* ctx, const qoc_problem_v1* problem, const qoc_ism_config_v1* cfg,
                    const qoc_solver_v1* solver, const double* u0, double* u_out,
                    qoc_iter_record_v1* recs, int32_t rec_cap, double* task_values,
                    qoc_run_status_v1* status);

/* Per-task inner-solver counters of the last qoc_ism_run on this context (InnerResult,
 * optimizers.hpp:32-37, as merged per task at ism.cpp:409-411,503-511): for batch member b and
 * outer iteration k (1-based), out[3][L] = guard_rejections, newton_fallbacks, gmres_iterations
 * per subinterval.  All zero for the gradient solver.  QOC_EINVAL when (b, k) was not run. */
int32_t qoc_ctx_solver_stats(const qoc_ctx* ctx, int32_t b, int32_t iteration, int32_t subintervals,
                             int32_t* out);

/* Objective forms (objective.hpp:16). */
enum qoc_form { QOC_FORM_OVERLAP = 0, QOC_FORM_TRACKING = 1 };

/* propagate_final for every batch member: states_out [B][d] complex. */
int32_t qoc_propagate_final(qoc_ctx* ctx, const qoc_problem_v1* problem, const double* u,
                            double* states_out);
/* evaluate_objective + objective_gradient: value_out [B], grad_out [B][C*K] (either may be NULL). */
int32_t qoc_objective_gradient(qoc_ctx* ctx, const qoc_problem_v1* problem, const double* u,
                               int32_t form, int32_t naive_nonlinear_adjoint, double* value_out,
                               double* grad_out);
/* assemble_propagator: prop_out [B][d*d] complex, column-major (linear kinds only). */
int32_t qoc_assemble_propagator(qoc_ctx* ctx, const qoc_problem_v1* problem, const double* u,
                                double* prop_out);

/* Stationary states of a QOC_KIND_STRANG model by normalized imaginary-time splitting -- the first
 * stage of ground_state (models.cpp:129-182) -- for `states` frozen controls at once (one CTA
 * each).  psi_io [states][d] complex holds the starting guesses and returns the states
 * (normalised to dx sum |psi|^2 = 1); with n_lower > 0 every iteration first projects out
 * lower [states][n_lower][d] (Gram-Schmidt in the dx-weighted inner product; excited states).
 * Stops when the discrete energy moves by less than energy_tol between iterations or after
 * max_iterations; energy_out [states], iterations_out [states].  The problem's grid, kinetic
 * spectrum, potential payload, kappa and ip_weight (= dx) are used; steps / states / penalty are
 * ignored.  The residual polish of models.cpp:184-262 (gradient flow, dense self-consistent
 * diagonalisation) stays with the caller. */
int32_t qoc_imaginary_time(qoc_ctx* ctx, const qoc_problem_v1* problem, int32_t states, const double* u_frozen,
                           double imaginary_dt, double energy_tol, int32_t max_iterations, int32_t n_lower,
                           const double* lower, double* psi_io, double* energy_out, int32_t* iterations_out);

/* Multi-GPU: one process and one context per GPU.  Rank 0 draws the NCCL unique
 * id (QOC_COMM_ID_BYTES bytes), the host side broadcasts it, and every rank binds its context
 * with qoc_ctx_init_comm.  A bit-flip run with plan ASSEMBLED then shards its subinterval blocks
 * over the world (blocks = 0 -> one block per rank): rank r owns blocks [r G/W, (r+1) G/W),
 * computes their tasks and block products, and ONE in-place ncclAllGather per outer iteration
 * exchanges block products, entry values, residuals and controls.  Every rank returns the same
 * controls and records.  world = 1 with id = NULL releases the communicator (with an id it
 * builds a one-rank communicator: the exchange path runs, trivially).  NCCL is loaded at run time
 * (dlopen "libnccl.so.2"; QOC_NCCL_LIBRARY overrides); failures return QOC_ENCCL.  Other kinds
 * run as independent replicas under a communicator (config 5 shards problems on the host). */
#define QOC_COMM_ID_BYTES 128
int32_t qoc_comm_unique_id(void* id_out, size_t len);
int32_t qoc_ctx_init_comm(qoc_ctx* ctx, int32_t rank, int32_t world, const void* id, size_t len);

/* Kernel-launch counter of this context (for the bench's gpu_launches claim). */
int64_t qoc_ctx_launch_count(const qoc_ctx* ctx);

/* Context options.
 *   QOC_OPT_PROFILE        1 = bracket every kernel launch of qoc_ism_run with CUDA events on
 *                          the launching stream and accumulate them into qoc_profile_v1.
 *   QOC_OPT_FLUSH_L2_BYTES >0 = overwrite that many bytes of scratch between outer iterations
 *                          (outside the per-iteration event brackets) so every iteration
 *                          starts with a cold L2. */
enum qoc_ctx_option { QOC_OPT_PROFILE = 1, QOC_OPT_FLUSH_L2_BYTES = 2 };
int32_t qoc_ctx_set_option(qoc_ctx* ctx, int32_t option, int64_t value);

/* Device-time totals since the last reset (CUDA events on the context stream). */
typedef struct qoc_profile_v1 {
  int64_t task_launches;   /* per-subinterval task kernels (the dominant kernel) */
  double task_ms;
  int64_t other_launches;  /* coordinator kernels (merge, chain, boundary, ...) */
  double other_ms;
  int64_t iterations;      /* outer iterations run */
  double iteration_ms;     /* summed per-iteration device time (L2 flush excluded) */
  int64_t iteration_launches; /* kernel launches inside the outer iterations */
} qoc_profile_v1;
int32_t qoc_ctx_profile(qoc_ctx* ctx, qoc_profile_v1* out, int32_t reset);
/* Per-launch-site device time of the profiled launches since the last reset (QOC_OPT_PROFILE):
 * entry `index` (0-based, first-seen order) -> its label ("assembly", "gradient", "residual",
 * "node sweeps", "task", "merge", ...), summed ms and launch count.  QOC_EINVAL past the end. */
int32_t qoc_ctx_kernel_profile(const qoc_ctx* ctx, int32_t index, char* name, size_t name_len, double* ms,
                               int64_t* launches);

#ifdef __cplusplus
}
#endif

#endif /* QOC_GPU_H_ */
