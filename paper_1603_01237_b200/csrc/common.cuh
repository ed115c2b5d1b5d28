// common.cuh — device-side types shared by the ISM kernels (sm_100a).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace qoc {

// Control channels the device kernels carry per grid step (per-step register arrays).  The
// driver rejects larger C with QOC_ELOGIC before anything runs (qoc_gpu.h QOC_MAX_CHANNELS).
constexpr int MAXC = 8;

// ---- complex128 as double2 ------------------------------------------------------------
__host__ __device__ __forceinline__ double2 cx(double r, double i) { return make_double2(r, i); }
__host__ __device__ __forceinline__ double2 cadd(double2 a, double2 b) { return cx(a.x + b.x, a.y + b.y); }
__host__ __device__ __forceinline__ double2 csub(double2 a, double2 b) { return cx(a.x - b.x, a.y - b.y); }
__host__ __device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return cx(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
// a * conj(b)
__host__ __device__ __forceinline__ double2 cmulc(double2 a, double2 b) {
  return cx(a.x * b.x + a.y * b.y, a.y * b.x - a.x * b.y);
}
// conj(a) * b
__host__ __device__ __forceinline__ double2 cconjmul(double2 a, double2 b) {
  return cx(a.x * b.x + a.y * b.y, a.x * b.y - a.y * b.x);
}
__host__ __device__ __forceinline__ double2 cscale(double2 a, double s) { return cx(a.x * s, a.y * s); }
__host__ __device__ __forceinline__ double2 cconj(double2 a) { return cx(a.x, -a.y); }
__host__ __device__ __forceinline__ double2 cneg(double2 a) { return cx(-a.x, -a.y); }
__host__ __device__ __forceinline__ double cabs2(double2 a) { return a.x * a.x + a.y * a.y; }
// acc + a*b
__host__ __device__ __forceinline__ double2 cfma(double2 a, double2 b, double2 acc) {
  return cx(fma(a.x, b.x, fma(-a.y, b.y, acc.x)), fma(a.x, b.y, fma(a.y, b.x, acc.y)));
}
// acc - a*b
__host__ __device__ __forceinline__ double2 cfms(double2 a, double2 b, double2 acc) {
  return cx(fma(-a.x, b.x, fma(a.y, b.y, acc.x)), fma(-a.x, b.y, fma(-a.y, b.x, acc.y)));
}
// acc + conj(a)*b
__host__ __device__ __forceinline__ double2 cfmaconj(double2 a, double2 b, double2 acc) {
  return cx(fma(a.x, b.x, fma(a.y, b.y, acc.x)), fma(a.x, b.y, fma(-a.y, b.x, acc.y)));
}
__host__ __device__ __forceinline__ double2 cdiv(double2 a, double2 b) {
  const double den = b.x * b.x + b.y * b.y;
  const double inv = 1.0 / den;
  return cx((a.x * b.x + a.y * b.y) * inv, (a.y * b.x - a.x * b.y) * inv);
}
__host__ __device__ __forceinline__ double2 crcp(double2 b) {
  const double inv = 1.0 / (b.x * b.x + b.y * b.y);
  return cx(b.x * inv, -b.y * inv);
}
__device__ __forceinline__ bool cfinite(double2 a) { return isfinite(a.x) && isfinite(a.y); }

__device__ __forceinline__ double2 shfl(double2 v, int src, int width = 32) {
  return cx(__shfl_sync(0xffffffffu, v.x, src, width), __shfl_sync(0xffffffffu, v.y, src, width));
}
__device__ __forceinline__ double2 shfl_xor(double2 v, int m, int width = 32) {
  return cx(__shfl_xor_sync(0xffffffffu, v.x, m, width), __shfl_xor_sync(0xffffffffu, v.y, m, width));
}

// ---- TMA bulk copies (cp.async.bulk) completing on a shared-memory mbarrier ---------------
__device__ __forceinline__ unsigned smem_addr(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_init_fence() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
// arrive (count 1) announcing `bytes` of incoming async transactions
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)), "r"(bytes)
               : "memory");
}
// plain arrive (count 1, release semantics)
__device__ __forceinline__ void mbar_arrive(unsigned long long* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_addr(bar)) : "memory");
}
// global -> shared bulk copy (bytes % 16 == 0, both addresses 16-byte aligned)
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, unsigned long long* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_addr(dst)),
      "l"(src), "r"(bytes), "r"(smem_addr(bar))
      : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned parity) {
  asm volatile(
      "{\n .reg .pred p;\n WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra WAIT_%=;\n}" ::"r"(
          smem_addr(bar)),
      "r"(parity)
      : "memory");
}

// ---- run modes of the task kernels -----------------------------------------------------
enum TaskMode : int {
  M_ENTRY = 1,      // entry value of the task at the current control -> entry[b][n]
  M_UPDATE = 2,     // inner gradient steps, controls updated in place
  M_ERROR = 4,      // residual sweep at the updated control -> err[b][n]
  M_ASSEMBLE = 8,   // propagator product at the updated control -> prop[b][n]
  M_LAGGED = 16,    // split refresh: psi_end / chi_start at the updated control
  M_FINAL = 32,     // store the final state of the first forward sweep -> psi_end[b][n]
  M_GRAD = 64,      // store the raw gradient (weight 1, no update) -> grad[b][K][C]
};

// ---- problem + run state as seen by kernels ------------------------------------------
struct DevProblem {
  int kind, d, C, K, B, L;
  int dm;  // matrix edge of the density kind (its states are dm x dm, d = dm^2); = d otherwise
  int has_quad;
  double dt, ip_w;
  // DENSE: row-major [B][d][d]; quad may be null.  Column 1-norms for the pivot bound.
  const double2* h0;
  const double2* lin;   // [B][C][d][d]
  const double2* quad;  // [B][C][d][d]
  const double* norm1;  // [B][1 + 2C] : ||H0||_1, ||A_c||_1, ||B_c||_1 (max column sums)
  // TRIDIAG: [B][nops][d] real diag, [B][nops][d-1] complex sub
  const double* tri_diag;
  const double2* tri_sub;
  // BITFLIP
  int nspins;
  const double* bf_diag;  // [B][d]
  const int* bf_axis;     // [C]
  const double* bf_coef;  // [B][C][nspins]
  // STRANG
  const double2* kin_fwd;  // [d] exp(-i dt/2 k)   (kinetic_half_phase, forward)
  const double2* kin_adj;  // [d] exp(+i dt/2 k)
  const double2* kin_fwd2;  // [d] exp(-i dt k): two consecutive kinetic half steps merged (strang sweeps)
  const double2* kin_adj2;  // [d] exp(+i dt k)
  int merge_kinetic;        // 1: sweeps merge the half steps between grid steps (QOC_DISABLE=strangmerge: 0)
  const double2* twiddle;  // FFT twiddles / DFT matrix
  const double* grid_x;
  int potential;
  double pp[4];
  double kappa;
  int pot_terms;               // QOC_POT_BASIS: V = sum_m pot_basis[m][i] f_m(u)
  int pot_type[8];
  double pot_param[8];
  const double* pot_basis;     // [pot_terms][d]
  int naive;  // GradientOptions::naive_nonlinear_adjoint (split-step adjoints, propagation.cpp:159-166)
  // states and penalty
  const double2* init;  // [B][d]
  const double2* targ;  // [B][d]
  const double* alpha;  // [K]
  const int* node;      // [L+1]
};

struct DevRun {
  double* u;            // [B][K][C] (column-major C x K per problem)
  double* grad;         // [B][K][C] (M_GRAD)
  double2* task_init;   // [B][L][d]
  double2* task_targ;   // [B][L][d]
  double2* psi_nodes;   // [B][L+1][d]
  double2* chi_nodes;   // [B][L+1][d]
  double2* prop;        // [B][L][d][d] row-major
  double2* psi_end;     // [B][L][d]
  double2* chi_start;   // [B][L][d]
  double2* traj;        // workspace [B*L][traj_len][d]
  int traj_len;         // >= max len + 1
  double2* winv;        // density kind: per-task one-step inverses W_j [B*L][traj_len - 1][dm*dm] kept by
                        // a forward sweep for the adjoint sweep that follows it (or null: recompute)
  double* entry;        // [B][L]
  double* err;          // [B][L]
  double* pen;          // [B][L] sum_j alpha_j |u_j|^2 over the task window (updated control)
  int* bad_u;           // [B][L]
  int* done;            // [B]
  int* status;          // [B] abort kind: 0 none, 1 controls, 2 boundary, 3 bootstrap
  int* abort_iter;      // [B]
  int* n_recs;          // [B]
  double* rec_obj;      // [B][cap]
  double* rec_err;      // [B][cap]
  double* rec_exact;    // [B][cap]
  double* rec_tv;       // [B][cap][L]
  int* rec_flags;       // [B][cap] bit 1 = has error, bit 2 = has exact objective
  double* tot_err;      // [B] summed task residual of the current iteration
  int* err_flags;       // [1] bit 1: a structured solve would have needed pivoting
  // propagator-cache engine (pcache.cu)
  const int* kdev;      // outer-iteration index read on the device (CUDA-graph replays), or null
  double2* pc;          // [B][L][traj_len][d][d] partial products P_j (row-major)
  double2* cay;         // [B][K][d][d] one-step Cayley matrices C_j (split dense assembly), or null
  double* chunk_pen;    // [B][L][nchunk]
  double* chunk_err;    // [B][L][nchunk]
  double* entry_pay;    // [B][L]
  // Neumann-in-the-control assembly (dense_nm.cu): per-problem coefficient matrices in MMA
  // fragment order [B][NM_TERMS][8][32], and the per-task hand-off flag to Gauss-Jordan
  double2* nm;
  int* nm_fallback;     // [B][L]
  double2* nm_v;        // [B][L][traj_len - 1][d] fused-residual vectors v_j
  int* nm_count;        // [1] tasks handed to Gauss-Jordan by the last Neumann sweep
  // one-pass iteration (dense_nm.cu dual evaluation): the update computed at the end of an
  // iteration and applied at the start of the next, and the previous iteration's tasks
  double* gpend;        // [B][K] weight * g_j
  double2* old_init;    // [B][L][d]
  double2* old_targ;    // [B][L][d]
  int cap;
};

struct TaskArgs {
  int mode;
  int form;      // 0 overlap, 1 tracking
  int weighted;  // task weight K/len
  int inner;     // inner gradient iterations
  double rho;
  int n_lo = 0;   // first subinterval of this launch (blocked plan: this rank's subintervals)
  int n_cnt = 0;  // subintervals in this launch (0 = all L)
};

// Blocked boundary refresh (bit-flip kind; SURVEY §8(e) option A).  The L subintervals form G
// contiguous blocks, block g = subintervals [bnode[g], bnode[g+1]); rank r of W owns blocks
// [r*bpr, (r+1)*bpr), bpr = G / W.  Each rank's exchange slab holds its block products
// P_g = A_{last} ... A_{first} (d x d, column-major: column c = the propagated basis state e_c),
// then its subintervals' entry values and residuals, then its steps' controls; one in-place
// all-gather of the slabs per outer iteration is the only collective.
struct DevBlocks {
  int G, bpr, W, rank;
  const int* bnode;   // [G+1] block boundaries as subinterval indices
  double2* slab;      // [W][slab_elems] (double2 units)
  size_t slab_elems;  // per rank
  int lmax, kmax;     // padded subinterval / step counts per rank
  __host__ __device__ double2* block(int g, int d) const {
    return slab + (size_t)(g / bpr) * slab_elems + (size_t)(g % bpr) * d * d;
  }
  __host__ __device__ double* scalars(int r, int d) const {  // [2][lmax]: entry, err
    return reinterpret_cast<double*>(slab + (size_t)r * slab_elems + (size_t)bpr * d * d);
  }
  __host__ __device__ double* controls(int r, int d) const {  // [kmax][C]
    return scalars(r, d) + 2 * (size_t)lmax;
  }
};

// Node sweeps over part of the horizon: the blocks [g0, g0 + nloc) of a DevBlocks split, each
// seeded from its chain-formed end nodes (psi at bnode[g], chi at bnode[g+1]) and writing only
// its interior nodes.  nloc = 0: the full horizon (node_sweeps, ism.cpp:35-84).
struct SweepRange {
  const int* bnode;
  int g0, nloc;
};

// Inner-solver workspace of the Newton update (optimizers.cpp:21-98,215-259; solvers.cu): one
// restarted GMRES per (problem, subinterval) task, all tasks advanced in lockstep rounds -- a
// round is two gradient launches of the kind's own task kernel at u +- h v (the central
// finite-difference Hessian-vector product) and one advance kernel that runs every task's
// GMRES state machine.  Vectors live on the control grid [B][K][C]; a task owns its window.
struct DevNewton {
  int restart, max_iter;  // SolverSpec::gmres_restart / gmres_max_iter
  double tol, hvp_scale, step_size;
  int weighted;           // task weight K/len (interpolated variant)
  double* g0;             // raw gradient at u (weight applied on use)
  double* x;              // GMRES iterate
  double* V;              // [restart + 1] Krylov basis vectors
  double *up, *um;        // perturbed controls u + h v, u - h v
  double *gp, *gm;        // raw gradients there; gp is reused for w = A v
  double* Hm;             // [B][L][(restart + 1) * restart] Hessenberg columns, h(row, col) at row * restart + col
  double* gv;             // [B][L][restart + 1] rotated right-hand side
  double *cs, *sn;        // [B][L][restart] Givens rotations
  double* sc;             // [B][L][4]: bnorm, rel, h, u_scale
  int* st;                // [B][L][8]: phase, i, used, spanned, zero, done, m
  int* active;            // [rounds] tasks still iterating after each round
  int* stats;             // [B][L][3] guard_rejections, newton_fallbacks, gmres_iterations (this outer iteration)
  size_t vstride;         // elements between basis vectors (= B * K * C)
};

}  // namespace qoc
