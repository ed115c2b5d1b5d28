// blocks.cu — the blocked boundary refresh of the bit-flip kind (SURVEY §8(e) option A):
// the block-product chain that forms the block-boundary nodes, the exchange-slab packing around
// the one all-gather per outer iteration, and the exact payoff from the chained final node.
//
// The chain is compose_from_propagators (ism.cpp:298-312) over the G block products instead
// of the L subinterval propagators:
//     psi_{bnode[g+1]} = P_g psi_{bnode[g]},      chi_{bnode[g]} = P_g^dag chi_{bnode[g+1]},
// seeded with psi_0 = initial and chi_L = target.  With G = L this is exactly the reference's
// assembled plan; with G < L the nodes inside a block come from node sweeps seeded at the
// block's chain-formed ends (bitflip horizon kernels with a SweepRange).  Each chain step is a
// d x d complex matvec over a column-major block product (16 MB at d = 1024), read once from
// L2/HBM by the whole grid: HBM-bound, ~2.6 us per step at the measured 6.55 TB/s.
#include "kernels.h"

namespace qoc {

namespace {

constexpr int CH_T = 256;   // threads per chain CTA
constexpr int CH_ROWS = 8;  // forward matvec: rows per CTA (8 rows x 32 column phases)

// psi_0 = initial, chi_L = target
__global__ void chain_seed_kernel(DevProblem P, DevRun R) {
  if (R.done[0] || R.status[0]) return;
  const int d = P.d, L = P.L;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < d; i += gridDim.x * blockDim.x) {
    R.psi_nodes[i] = P.init[i];
    R.chi_nodes[(size_t)L * d + i] = P.targ[i];
  }
}

// One chain step s: blockIdx.y = 0 forms psi at bnode[s+1] from psi at bnode[s] with P_s;
// blockIdx.y = 1 forms chi at bnode[G-1-s] from chi at bnode[G-s] with P_{G-1-s}^dag.
// Fixed-order reductions (deterministic).
__global__ void __launch_bounds__(CH_T) chain_step_kernel(DevProblem P, DevRun R, DevBlocks BK, int s) {
  if (R.done[0] || R.status[0]) return;
  __shared__ double2 red[CH_T];
  const int d = P.d, t = threadIdx.x;
  if (blockIdx.y == 0) {
    const int g = s;
    const double2* M = BK.block(g, d);
    const double2* x = R.psi_nodes + (size_t)BK.bnode[g] * d;
    double2* y = R.psi_nodes + (size_t)BK.bnode[g + 1] * d;
    // y_i = sum_c M[i + c d] x_c: thread (r, q) takes row row0 + r, columns c = q mod 32
    const int r = t % CH_ROWS, q = t / CH_ROWS;
    for (int row0 = blockIdx.x * CH_ROWS; row0 < d; row0 += gridDim.x * CH_ROWS) {
      double2 acc = cx(0.0, 0.0);
      if (row0 + r < d)
        for (int c = q; c < d; c += CH_T / CH_ROWS) acc = cfma(M[(size_t)c * d + row0 + r], x[c], acc);
      red[t] = acc;
      __syncthreads();
      if (t < CH_ROWS && row0 + t < d) {
        double2 a = cx(0.0, 0.0);
        for (int qq = 0; qq < CH_T / CH_ROWS; ++qq) a = cadd(a, red[qq * CH_ROWS + t]);
        y[row0 + t] = a;
      }
      __syncthreads();
    }
  } else {
    const int g = BK.G - 1 - s;
    const double2* M = BK.block(g, d);
    const double2* x = R.chi_nodes + (size_t)BK.bnode[g + 1] * d;
    double2* y = R.chi_nodes + (size_t)BK.bnode[g] * d;
    // y_c = sum_i conj(M[i + c d]) x_i: one warp per column, coalesced down the column
    const int lane = t & 31, w = t >> 5;
    for (int c = blockIdx.x * (CH_T / 32) + w; c < d; c += gridDim.x * (CH_T / 32)) {
      double2 acc = cx(0.0, 0.0);
      for (int i = lane; i < d; i += 32) acc = cfmaconj(M[(size_t)c * d + i], x[i], acc);
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) {
        acc.x += __shfl_xor_sync(0xffffffffu, acc.x, off);
        acc.y += __shfl_xor_sync(0xffffffffu, acc.y, off);
      }
      if (lane == 0) y[c] = acc;
    }
  }
}

// subinterval / step ranges of rank r
__device__ __forceinline__ void rank_range(const DevProblem& P, const DevBlocks& BK, int r, int& n0, int& n1, int& j0,
                                           int& j1) {
  n0 = BK.bnode[r * BK.bpr];
  n1 = BK.bnode[(r + 1) * BK.bpr];
  j0 = P.node[n0];
  j1 = P.node[n1];
}

// this rank's entry values, residuals and controls -> its slab (before the all-gather)
__global__ void slab_pack_kernel(DevProblem P, DevRun R, DevBlocks BK, int with_controls) {
  int n0, n1, j0, j1;
  rank_range(P, BK, BK.rank, n0, n1, j0, j1);
  double* sc = BK.scalars(BK.rank, P.d);
  double* ct = BK.controls(BK.rank, P.d);
  const int tid = blockIdx.x * blockDim.x + threadIdx.x, nt = gridDim.x * blockDim.x;
  for (int n = n0 + tid; n < n1; n += nt) {
    sc[n - n0] = R.entry[n];
    sc[BK.lmax + n - n0] = R.err[n];
  }
  if (with_controls)
    for (int i = tid; i < (j1 - j0) * P.C; i += nt) ct[i] = R.u[(size_t)j0 * P.C + i];
}

// every other rank's slab -> R.entry / R.err / R.u (after the all-gather)
__global__ void slab_unpack_kernel(DevProblem P, DevRun R, DevBlocks BK, int with_controls) {
  const int r = blockIdx.y;
  if (r == BK.rank) return;
  int n0, n1, j0, j1;
  rank_range(P, BK, r, n0, n1, j0, j1);
  const double* sc = BK.scalars(r, P.d);
  const double* ct = BK.controls(r, P.d);
  const int tid = blockIdx.x * blockDim.x + threadIdx.x, nt = gridDim.x * blockDim.x;
  for (int n = n0 + tid; n < n1; n += nt) {
    R.entry[n] = sc[n - n0];
    R.err[n] = sc[BK.lmax + n - n0];
  }
  if (with_controls)
    for (int i = tid; i < (j1 - j0) * P.C; i += nt) R.u[(size_t)j0 * P.C + i] = ct[i];
}

// exact payoff of objective.cpp:93-100 from the chained final node psi_L (which the direct
// plan gets from a full-horizon forward sweep at the same control)
__global__ void __launch_bounds__(256) exact_from_nodes_kernel(DevProblem P, DevRun R, int k) {
  if (R.kdev) k = *R.kdev;
  if (R.done[0] || R.status[0]) return;
  __shared__ double sh[256];
  const int d = P.d, t = threadIdx.x;
  const double2* last = R.psi_nodes + (size_t)P.L * d;
  double s = 0.0;
  for (int i = t; i < d; i += 256) s += cconjmul(P.targ[i], last[i]).x;
  sh[t] = s;
  __syncthreads();
  for (int w = 128; w > 0; w >>= 1) {
    if (t < w) sh[t] += sh[t + w];
    __syncthreads();
  }
  if (t == 0) {
    double pen = 0.0;
    for (int n = 0; n < P.L; ++n) pen += R.pen[n];
    R.rec_exact[k] = P.ip_w * sh[0] - 0.5 * P.dt * pen;
  }
}

}  // namespace

cudaError_t block_chain(const DevProblem& P, const DevRun& R, const DevBlocks& BK, cudaStream_t st) {
  chain_seed_kernel<<<(P.d + 255) / 256, 256, 0, st>>>(P, R);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  // enough CTAs to stream a 16 MB block at full bandwidth: d / 8 rows (forward) and d / 8
  // columns (adjoint) per grid
  const int gx = (P.d + CH_ROWS - 1) / CH_ROWS;
  for (int s = 0; s < BK.G; ++s) {
    chain_step_kernel<<<dim3(gx, 2), CH_T, 0, st>>>(P, R, BK, s);
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
  }
  return cudaSuccess;
}

cudaError_t slab_pack(const DevProblem& P, const DevRun& R, const DevBlocks& BK, int with_controls, cudaStream_t st) {
  slab_pack_kernel<<<8, 256, 0, st>>>(P, R, BK, with_controls);
  return cudaGetLastError();
}

cudaError_t slab_unpack(const DevProblem& P, const DevRun& R, const DevBlocks& BK, int with_controls,
                        cudaStream_t st) {
  slab_unpack_kernel<<<dim3(8, BK.W), 256, 0, st>>>(P, R, BK, with_controls);
  return cudaGetLastError();
}

cudaError_t exact_from_nodes(const DevProblem& P, const DevRun& R, int k, cudaStream_t st) {
  exact_from_nodes_kernel<<<1, 256, 0, st>>>(P, R, k);
  return cudaGetLastError();
}

}  // namespace qoc
