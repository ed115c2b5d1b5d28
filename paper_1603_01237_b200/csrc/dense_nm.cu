// dense_nm.cu — propagator assembly for batched dense single-control problems (BASELINE
// config 5: d = 16, C = 1, H(u) = H0 + u Hc), sm_100a.
//
// The reference forms every one-step map by an LU solve of B(u_j) = I + i(dt/2)H(u_j)
// (propagation.cpp:14-16,85-90) and assembles M = prod_j C_j (propagation.cpp:236-249).  For a
// single linear control the step matrix factors as
//     B(u) = B0 (I + u G),   B0 = I + i a H0,   G = B0^-1 (i a Hc),   a = dt/2,
// so its inverse is the Neumann series of (I + uG)^-1 -- the "Taylor expansion of
// (I + iA)^-1 truncated at fp64 precision" of SURVEY F3 -- and the Cayley matrix is a
// polynomial in the control with per-problem matrix coefficients:
//     C(u) = 2 B(u)^-1 - I = sum_{m>=0} u^m N_m,
//     N_0 = 2 B0^-1 - I,   N_m = 2 (-G)^m B0^-1  (m >= 1).
// ||B0^-1||_2 <= 1 (B0 is normal with |eigenvalues| >= 1) and ||G||_2 <= a ||Hc||_1, so with
// x = |u| a ||Hc||_1 the truncation after M terms is bounded by 2 x^(M+1) / (1 - x); every step
// uses the smallest M that puts this below 2^-54 (the certified fp64 evaluation of the same
// discrete map; the reference's LU solve differs from it at rounding level, like the
// Gauss-Jordan path it replaces).
//
//   dense_nm_setup_kernel     warp per problem: B0^-1 by pivoted Gauss-Jordan, then the
//                             coefficient chain N_m, stored in MMA-fragment order.
//   dense_nm_assemble_kernel  warp per task: per grid step, Horner in u_j over the N_m
//                             staged in shared memory (TMA bulk copy), elementwise in
//                             registers; then P_{j+1}^T = P_j^T C_j^T on the fp64 tensor
//                             cores (mma.sync m8n8k4 f64, four real products) and the cache
//                             store (column-major P_j: the evaluation kernel below reads each
//                             matrix as 512-byte runs).  A task whose control leaves the certified range is
//                             flagged and handed to the Gauss-Jordan kernel (pcache.cu),
//                             which keeps the partial-pivoting path.
#include <cstdlib>
#include <cstring>
#include <type_traits>

#include "dense.cuh"
#include "kernels.h"
#include "qoc_gpu.h"

namespace qoc {

namespace {

constexpr int ND = 16;                 // matrix dimension of this path
constexpr int SLOTS = 8;               // complex fragment slots per lane (256 / 32)
constexpr int NM_WARPS = 8;            // tasks (warps) per CTA
constexpr int XS = ND + 1;             // padded row stride of the layout-exchange scratch

// Fragment order: slot s = jn*4 + kk of lane (q = l >> 2, r = l & 3) holds element
// (8 jn + q, 4 kk + r) of a 16 x 16 matrix -- the B operand of m8n8k4 for its transpose.

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

// ---- setup: one warp per problem ------------------------------------------------------
__global__ void __launch_bounds__(32) dense_nm_setup_kernel(DevProblem P, DevRun R) {
  using Cfg = DenseCfg<ND, 1>;
  __shared__ __align__(16) double2 ops[ND * ND];   // H0 (row-major), then i a Hc
  __shared__ __align__(16) double2 hc[ND * ND];
  __shared__ __align__(16) double2 T[ND * ND];
  __shared__ __align__(16) unsigned char scratch[sizeof(double2) * (Cfg::PIV + Cfg::VEC + 2 * Cfg::MAT) + 2 * ND * 4];
  const int b = blockIdx.x, lane = threadIdx.x, row = lane & 15;
  const double a = 0.5 * P.dt;
  for (int e = lane; e < ND * ND; e += 32) {
    ops[e] = P.h0[(size_t)b * ND * ND + e];
    const double2 h = P.lin[(size_t)b * ND * ND + e];
    hc[e] = cx(-a * h.y, a * h.x);  // i a Hc
  }
  __syncwarp();
  DenseScratch<ND, 1> S;
  S.piv = reinterpret_cast<double2*>(scratch);
  S.vec = S.piv + Cfg::PIV;
  S.matW = S.vec + Cfg::VEC;
  S.matP = S.matW + Cfg::MAT;
  S.perm = reinterpret_cast<int*>(S.matP + Cfg::MAT);
  DenseLane<ND, 1> Ln;
  Ln.row = row;
  Ln.g = 0;
  double2 W[ND];
  const double u0 = 0.0;
  Ln.build(W, ops, 0, 0, &u0, a, false);  // B0 = I + i a H0
  // both half-warps run the same 16-lane Gauss-Jordan (partial pivoting: setup, once per run)
  Ln.invert_pivot(W, S, row);            // W = B0^-1, row `row`
  double2 G[ND];
#pragma unroll
  for (int c = 0; c < ND; ++c) {
    double2 acc = cx(0.0, 0.0);
#pragma unroll
    for (int k = 0; k < ND; ++k) acc = cfma(W[k], hc[k * ND + c], acc);
    G[c] = cneg(acc);  // -G
  }
  double2* nm = R.nm + (size_t)b * NM_TERMS * SLOTS * 32;
  auto store_term = [&](int m, const double2 (&Trow)[ND]) {
    if (lane < 16) {
#pragma unroll
      for (int c = 0; c < ND; ++c) {
        const int s = (row >> 3) * 4 + (c >> 2), l = (row & 7) * 4 + (c & 3);
        nm[((size_t)m * SLOTS + s) * 32 + l] = Trow[c];
      }
    }
  };
  double2 Tr[ND];
#pragma unroll
  for (int c = 0; c < ND; ++c) Tr[c] = cx(2.0 * W[c].x, 2.0 * W[c].y);  // T_0 = 2 B0^-1
  {
    double2 N0[ND];
#pragma unroll
    for (int c = 0; c < ND; ++c) N0[c] = cx(Tr[c].x - (c == row ? 1.0 : 0.0), Tr[c].y);
    store_term(0, N0);
  }
  for (int m = 1; m < NM_TERMS; ++m) {  // T_m = (-G) T_{m-1} = N_m
    __syncwarp();
    if (lane < 16)
#pragma unroll
      for (int c = 0; c < ND; ++c) T[row * ND + c] = Tr[c];
    __syncwarp();
#pragma unroll
    for (int c = 0; c < ND; ++c) {
      double2 acc = cx(0.0, 0.0);
#pragma unroll
      for (int k = 0; k < ND; ++k) acc = cfma(G[k], T[k * ND + c], acc);
      Tr[c] = acc;
    }
    store_term(m, Tr);
  }
}

// smallest M with 2 x^(M+1) / (1 - x) <= 2^-54, or -1 past the staged terms
__device__ __forceinline__ int neumann_terms(double x) {
  if (!(x < 0.5)) return -1;
  const double lim = 0x1p-54 * (1.0 - x) * 0.5;
  double p = x;
  int M = 0;
  while (p > lim) {
    p *= x;
    if (++M >= NM_TERMS) return -1;
  }
  return M;
}

// ---- assembly: one warp per task ----------------------------------------------------------
// residual != 0 also evaluates the task's residual (error_norm of the weight-1 gradient at the
// control just assembled, ism.cpp:413-419) in the same sweep, through
//     Im<chi_j + chi_{j+1}, Hc (psi_j + psi_{j+1})> = Im( y^dag v_j ),
//     v_j = (P_j + P_{j+1})^dag Hc (psi_j + psi_{j+1}),   y = P_len^dag seed,
// (chi_j = P_j y by unitarity, as in pcache.cu): v_j is formed on the way (psi_{j+1} = C_j psi_j
// from the Horner output), parked in `R.nm_v`, and contracted with y once P_len exists.
template <bool GAUSS3, bool RESIDUAL, int HB>
__global__ void __launch_bounds__(NM_WARPS * 32, 2) dense_nm_assemble_kernel(DevProblem P, DevRun R, int ignore_done) {
  constexpr bool residual = RESIDUAL;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  double2* nm_s = reinterpret_cast<double2*>(smem_raw);                       // [NM_TERMS][SLOTS][32]
  double2* xch_all = nm_s + NM_TERMS * SLOTS * 32;                            // [NM_WARPS][ND][XS]
  double2* hc_s = xch_all + NM_WARPS * ND * XS;                               // [SLOTS][32] (residual)
  __shared__ __align__(8) unsigned long long bar;
  const int b = blockIdx.y;
  if (ignore_done ? R.status[b] : (R.done[b] | R.status[b])) return;
  const int tid = threadIdx.x, warp = tid >> 5, l = tid & 31, q = l >> 2, r = l & 3;
  // stage the problem's coefficient matrices once per CTA (TMA bulk copy, 4 x 16 KB)
  constexpr unsigned kBytes = NM_TERMS * SLOTS * 32 * sizeof(double2);
  constexpr unsigned kChunk = 16384;
  if (tid == 0) {
    mbar_init(&bar, 1);
    mbar_init_fence();
  }
  __syncthreads();
  if (tid == 0) {
    mbar_expect_tx(&bar, kBytes);
    const char* src = reinterpret_cast<const char*>(R.nm + (size_t)b * NM_TERMS * SLOTS * 32);
    for (unsigned off = 0; off < kBytes; off += kChunk)
      bulk_g2s(reinterpret_cast<char*>(nm_s) + off, src + off, kChunk < kBytes - off ? kChunk : kBytes - off, &bar);
  }
  const size_t dd = (size_t)ND * ND;
  if (residual)  // Hc in fragment order: slot s = jn*4 + kk of lane (q, r) = Hc[8 jn + q][4 kk + r]
    for (int e = tid; e < SLOTS * 32; e += blockDim.x) {
      const int s = e >> 5, ll = e & 31;
      hc_s[e] = P.lin[(size_t)b * dd + (8 * (s >> 2) + (ll >> 2)) * ND + 4 * (s & 3) + (ll & 3)];
    }
  const double gam = 0.5 * P.dt * P.norm1[(size_t)b * (1 + 2 * P.C) + 1];  // a ||Hc||_1 >= ||G||_2
  double2* xch = xch_all + warp * ND * XS;

  const int nr = blockIdx.x * NM_WARPS + warp;
  bool live = nr < P.L;
  const int n = live ? nr : P.L - 1;
  const int node0 = P.node[n], len = P.node[n + 1] - node0;
  const double* u = R.u + (size_t)b * P.K + node0;
  // certified range check over the task's steps (warp-uniform); out-of-range tasks are handed
  // to the Gauss-Jordan kernel
  // (len <= 32: lane j holds step j's control and certified term count, computed once here
  // instead of as a dependent multiply chain in front of every step's Horner evaluation)
  const double u_l = l < len ? u[l] : 0.0;
  const int M_l = neumann_terms(fabs(u_l) * gam);  // NaN controls give -1
  {
    const bool ok = __all_sync(0xffffffffu, M_l >= 0);
    if (l == 0 && live) {
      R.nm_fallback[(size_t)b * P.L + n] = ok ? 0 : 1;
      if (!ok) atomicAdd(R.nm_count, 1);
    }
    if (!ok) live = false;
  }
  const size_t task = (size_t)b * P.L + n;
  double2* Pc = R.pc + task * (size_t)R.traj_len * dd;
  // P^T in A-fragment layout: Pa[i][kk] = P[4kk + r][8i + q]
  double2 Pa[2][4];
#pragma unroll
  for (int i = 0; i < 2; ++i)
#pragma unroll
    for (int kk = 0; kk < 4; ++kk) Pa[i][kk] = cx((4 * kk + r) == (8 * i + q) ? 1.0 : 0.0, 0.0);
  if (live)  // P_0 = I into the cache (column-major)
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
      for (int kk = 0; kk < 4; ++kk) Pc[(8 * i + q) * ND + 4 * kk + r] = Pa[i][kk];
  // residual state: psi_j at columns 4kk + r ("column layout")
  double2 psc[4];
  if (residual)
#pragma unroll
    for (int kk = 0; kk < 4; ++kk) psc[kk] = R.task_init[task * ND + 4 * kk + r];
  double2* vj = R.nm_v + task * (size_t)(R.traj_len - 1) * ND;
  auto quad_sum = [](double2 v) {
    v = cadd(v, shfl_xor(v, 1));
    return cadd(v, shfl_xor(v, 2));
  };
  mbar_wait(&bar, 0);
  if (residual) __syncthreads();  // hc_s visible

  // Horner for HB consecutive steps at once: every coefficient fragment read from shared memory
  // (the kernel's bound: (M + 1) x 4 KB per step) serves HB controls.  The batch uses the largest
  // certified term count of its steps (extra terms only shrink the truncation error).
  for (int j0 = 0; j0 < len; j0 += HB) {
    double uh[HB];
    int M = 0;
#pragma unroll
    for (int h = 0; h < HB; ++h) {
      uh[h] = __shfl_sync(0xffffffffu, u_l, (j0 + h) & 31);  // 0 past len
      M = max(M, __shfl_sync(0xffffffffu, M_l, (j0 + h) & 31));
    }
    if (!live) M = 0;
    // Horner: Y = N_M; Y = N_m + u Y (m = M-1 .. 0); Y[s] = C(u)[8 jn + q][4 kk + r]
    double2 YH[HB][SLOTS];
#pragma unroll
    for (int s = 0; s < SLOTS; ++s) {
      const double2 nv = nm_s[(M * SLOTS + s) * 32 + l];
#pragma unroll
      for (int h = 0; h < HB; ++h) YH[h][s] = nv;
    }
    for (int m = M - 1; m >= 0; --m) {
#pragma unroll
      for (int s = 0; s < SLOTS; ++s) {
        const double2 nv = nm_s[(m * SLOTS + s) * 32 + l];
#pragma unroll
        for (int h = 0; h < HB; ++h) YH[h][s] = cx(fma(uh[h], YH[h][s].x, nv.x), fma(uh[h], YH[h][s].y, nv.y));
      }
    }
#pragma unroll
    for (int h = 0; h < HB; ++h) {
    const int j = j0 + h;
    if (j < len) {
    const double2* Y = YH[h];
    double2 bc[4], vp[2];
    if (residual) {
      // psi_{j+1} = C_j psi_j: rows 8 jn + q, reduced over the quad's columns
      double2 pn[2];
#pragma unroll
      for (int jn = 0; jn < 2; ++jn) {
        double2 acc = cx(0.0, 0.0);
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) acc = cfma(Y[jn * 4 + kk], psc[kk], acc);
        pn[jn] = quad_sum(acc);
      }
      // to column layout: psi_{j+1}[4kk + r] lives in quad 4(kk & 1) + r, slot kk >> 1; ps = psi_j + psi_{j+1}
      double2 ps[4];
#pragma unroll
      for (int kk = 0; kk < 4; ++kk) {
        const double2 v = shfl(pn[kk >> 1], 4 * (4 * (kk & 1) + r));
        ps[kk] = cadd(psc[kk], v);
        psc[kk] = v;
      }
      // b = Hc ps (rows 8 jn + q), back to column layout
      double2 br[2];
#pragma unroll
      for (int jn = 0; jn < 2; ++jn) {
        double2 acc = cx(0.0, 0.0);
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) acc = cfma(hc_s[(jn * 4 + kk) * 32 + l], ps[kk], acc);
        br[jn] = quad_sum(acc);
      }
#pragma unroll
      for (int kk = 0; kk < 4; ++kk) bc[kk] = shfl(br[kk >> 1], 4 * (4 * (kk & 1) + r));
      // v partial with P_j: v[8i + q] += sum conj(P_j[4kk + r][8i + q]) b[4kk + r]
#pragma unroll
      for (int i = 0; i < 2; ++i) {
        double2 acc = cx(0.0, 0.0);
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) acc = cfmaconj(Pa[i][kk], bc[kk], acc);
        vp[i] = acc;
      }
    }
    // P_{j+1}^T = P_j^T C_j^T: A = P^T (Pa), B = C^T (Y: B[4kk + r][8jn + q] = C[8jn + q][4kk + r])
    double cr[2][2][2], ci[2][2][2];
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
      for (int jn = 0; jn < 2; ++jn) {
        cr[i][jn][0] = cr[i][jn][1] = ci[i][jn][0] = ci[i][jn][1] = 0.0;
        if constexpr (GAUSS3) {  // three real products: re = ArBr - AiBi, im = (Ar+Ai)(Br+Bi) - ArBr - AiBi
          double t2[2] = {0.0, 0.0};
#pragma unroll
          for (int kk = 0; kk < 4; ++kk) {
            const double2 av = Pa[i][kk], bv = Y[jn * 4 + kk];
            dmma(cr[i][jn][0], cr[i][jn][1], av.x, bv.x);
            dmma(t2[0], t2[1], av.y, bv.y);
            dmma(ci[i][jn][0], ci[i][jn][1], av.x + av.y, bv.x + bv.y);
          }
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            ci[i][jn][e] = ci[i][jn][e] - cr[i][jn][e] - t2[e];
            cr[i][jn][e] = cr[i][jn][e] - t2[e];
          }
        } else {
#pragma unroll
          for (int kk = 0; kk < 4; ++kk) {
            const double2 av = Pa[i][kk], bv = Y[jn * 4 + kk];
            dmma(cr[i][jn][0], cr[i][jn][1], av.x, bv.x);
            dmma(cr[i][jn][0], cr[i][jn][1], -av.y, bv.y);
            dmma(ci[i][jn][0], ci[i][jn][1], av.x, bv.y);
            dmma(ci[i][jn][0], ci[i][jn][1], av.y, bv.x);
          }
        }
      }
    // lane holds P_{j+1}[8 jn + 2r + e][8 i + q]; C-fragment -> A-fragment layout through the
    // warp's scratch, then the cache store (column-major: 64-byte runs of a column per lane quad)
    __syncwarp();
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
      for (int jn = 0; jn < 2; ++jn)
#pragma unroll
        for (int e = 0; e < 2; ++e) xch[(8 * jn + 2 * r + e) * XS + 8 * i + q] = cx(cr[i][jn][e], ci[i][jn][e]);
    __syncwarp();
    double2* dst = Pc + (size_t)(j + 1) * dd;
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
      for (int kk = 0; kk < 4; ++kk) {
        Pa[i][kk] = xch[(4 * kk + r) * XS + 8 * i + q];
        if (live) __stcs(dst + (8 * i + q) * ND + 4 * kk + r, Pa[i][kk]);
      }
    if (residual) {  // v partial with P_{j+1}; park v_j
#pragma unroll
      for (int i = 0; i < 2; ++i) {
        double2 acc = vp[i];
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) acc = cfmaconj(Pa[i][kk], bc[kk], acc);
        acc = quad_sum(acc);
        if (r == 0 && live) vj[(size_t)j * ND + 8 * i + q] = acc;
      }
    }
    }
    }
  }
  // M_n = P_len for the boundary chain (row-major)
  if (R.prop && live) {
    double2* Mn = R.prop + task * dd;
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
      for (int kk = 0; kk < 4; ++kk) Mn[(4 * kk + r) * ND + 8 * i + q] = Pa[i][kk];
  }
  if (residual) {
    // seed = targ - psi_len (tracking form, interpolated variant); y = P_len^dag seed
    double2 sc[4];
#pragma unroll
    for (int kk = 0; kk < 4; ++kk) sc[kk] = csub(R.task_targ[task * ND + 4 * kk + r], psc[kk]);
    double2 yr[2];
#pragma unroll
    for (int i = 0; i < 2; ++i) {
      double2 acc = cx(0.0, 0.0);
#pragma unroll
      for (int kk = 0; kk < 4; ++kk) acc = cfmaconj(Pa[i][kk], sc[kk], acc);
      yr[i] = quad_sum(acc);  // y[8i + q]
    }
    __syncwarp();
    // g_j = -alpha_j dt u_j + dt/4 w Im(y^dag v_j): lane (j = l & 15, half h = l >> 4) takes 8 of
    // the 16 components, y from the quads through the scratch
    if (r == 0) {
      xch[8 * 0 + q] = yr[0];
      xch[8 + q] = yr[1];
    }
    __syncwarp();
    const int jl = l & 15, h = l >> 4;
    double im = 0.0;
    if (jl < len) {
      double2 acc = cx(0.0, 0.0);
#pragma unroll
      for (int c = 0; c < 8; ++c) acc = cfmaconj(xch[8 * h + c], vj[(size_t)jl * ND + 8 * h + c], acc);
      im = acc.y;
    }
    im += __shfl_xor_sync(0xffffffffu, im, 16);
    const double Kd = (double)P.K, scale = (double)len / Kd, dt = P.dt, w = P.ip_w;
    double err = 0.0;
    if (jl < len && h == 0) {
      const double gj = -(P.alpha[node0 + jl] * scale) * dt * u[jl] + 0.25 * dt * (w * im);
      err = fabs(gj);
    }
#pragma unroll
    for (int off = 1; off < 16; off <<= 1) err += __shfl_xor_sync(0xffffffffu, err, off);
    if (l == 0 && live) R.err[task] = err;
  }
}

// ---- gradient / residual evaluation through the cache: one warp per task ----------------
// Streams P_1..P_len (4 KB each, coalesced 512-byte rows of lanes) once with two steps in
// flight and evaluates, exactly as pc_eval_kernel (pcache.cu) does,
//   psi_j = P_j phi,  chi_j = P_j chi_0,  chi_0 = P_len^dag seed       (objective.cpp:31-34)
//   g_j = -alpha_j dt u_j + dt/4 w Im<chi_j + chi_{j+1}, Hc (psi_j + psi_{j+1})>  (objective.cpp:55-57)
// Lane (row = l & 15, g = l >> 4) holds columns 2t + g of its row of every matrix.
//
// dual = 1 is the one-pass iteration: the two warps of a pair read the same P_j (the second
// read hits L1/L2, so the 36 GB cache leaves HBM once) and evaluate
//   warp 0: the residual of iteration k with its tasks S_k (R.old_*) at the updated control;
//   warp 1: the entry value and gradient of iteration k + 1 with the refreshed tasks S_{k+1},
//           whose weighted gradient w g_j goes to R.gpend (applied by the next iteration's first kernel).
// dual = 2 is warp-1 work only (bootstrap).
//
// RING (dual = 1 only): a pair shares one stream, which halves the loads a warp keeps in flight;
// the pair's matrices instead arrive by TMA bulk copies (4 KB each) into a DS-stage shared
// ring per task, issued by lane 0 of the pair's second warp, so DS matrices per task are in
// flight regardless of registers.  Consumption order c = 0..len reads P_len, P_1, ..., P_len.
// Each warp marks a stage consumed on its `empty` barrier without waiting; the producer refills
// the stage one step late (so it rarely waits for the slower warp of the pair).
constexpr int DT = 4, DS = 5;  // tasks per CTA, ring stages per task
template <bool RING>
__global__ void __launch_bounds__(256, 2) dense_pc_eval16_kernel(DevProblem P, DevRun R, TaskArgs A, int ignore_done,
                                                                  int handed_off_only, int dual) {
  constexpr int PE_ENTRY = 1, PE_GRAD = 2, PE_ERR = 4;
  __shared__ double2 hcs[ND * ND];  // Hc column-major: lane (row, g) reads 512-byte runs
  __shared__ double2 xs[8][ND];
  __shared__ double2 pss[8][ND];       // psi_j + psi_{j+1} by row, read back as broadcasts
  __shared__ double ush[8][32], ash[8][32];  // the task's controls and penalty weights (len <= 32)
  extern __shared__ __align__(128) unsigned char ring_raw[];  // RING: [DT][DS][256] double2 + barriers
  double2* ring = reinterpret_cast<double2*>(ring_raw);
  unsigned long long* full = reinterpret_cast<unsigned long long*>(ring + DT * DS * ND * ND);
  unsigned long long* empty = full + DT * DS;
  const int b = blockIdx.y;
  if (handed_off_only && *R.nm_count == 0) return;  // nothing was handed off (the common case)
  if (ignore_done ? R.status[b] : (R.done[b] | R.status[b])) return;
  const size_t dd = (size_t)ND * ND;
  for (int e = threadIdx.x; e < ND * ND; e += blockDim.x) hcs[(e & 15) * ND + (e >> 4)] = P.lin[(size_t)b * dd + e];
  const int warp = threadIdx.x >> 5, l = threadIdx.x & 31, row = l & 15, g = l >> 4;
  const int n = dual == 1 ? blockIdx.x * 4 + (warp >> 1) : blockIdx.x * 8 + warp;
  const int role = dual == 1 ? (warp & 1) : 1;  // 0: residual of S_k, 1: entry + gradient
  const int tl = warp >> 1;                     // RING: task slot of the pair
  const bool producer = RING && role == 1 && l == 0 && n < P.L;
  const int plen = n < P.L ? P.node[n + 1] - P.node[n] : 0;
  const double2* Pg = R.pc + ((size_t)b * P.L + n) * (size_t)R.traj_len * dd;
  auto issue = [&](int c) {  // producer: matrix of consumption step c into its stage
    const int st = c % DS;
    mbar_expect_tx(&full[tl * DS + st], (unsigned)(dd * sizeof(double2)));
    bulk_g2s(ring + (size_t)(tl * DS + st) * dd, Pg + (size_t)(c ? c : plen) * dd, (unsigned)(dd * sizeof(double2)),
             &full[tl * DS + st]);
  };
  if (RING) {
    if (threadIdx.x == 0) {
      for (int i = 0; i < DT * DS; ++i) {
        mbar_init(&full[i], 1);
        mbar_init(&empty[i], 2);
      }
      mbar_init_fence();
    }
    __syncthreads();
    if (producer)
      for (int c = 0; c < DS && c <= plen; ++c) issue(c);
  } else {
    __syncthreads();
  }
  if (n >= P.L) return;
  // residual of the tasks the Neumann sweep handed to Gauss-Jordan (its fused residual covers the rest)
  if (handed_off_only && R.nm_fallback[(size_t)b * P.L + n] == 0) return;
  const int mode = dual ? (role ? (PE_ENTRY | PE_GRAD) : PE_ERR) : A.mode;
  const double2* t_init = (dual && !role) ? R.old_init : R.task_init;
  const double2* t_targ = (dual && !role) ? R.old_targ : R.task_targ;
  const int node0 = P.node[n], len = P.node[n + 1] - node0;
  const double Kd = (double)P.K, weight = A.weighted ? Kd / (double)len : 1.0, scale = (double)len / Kd;
  const double dt = P.dt, w = P.ip_w;
  const size_t tix = ((size_t)b * P.L + n) * ND;
  // column-major cache: P_j[row][2t + g] at (2t + g) * 16 + row = l + 32 t
  const double2* Pc = R.pc + ((size_t)b * P.L + n) * (size_t)R.traj_len * dd + l;
  double* u = R.u + (size_t)b * P.K + node0;
  double2 phi[8];
#pragma unroll
  for (int t = 0; t < 8; ++t) phi[t] = t_init[tix + 2 * t + g];
  auto half_sum = [&](double2 v) { return cadd(v, shfl_xor(v, 16)); };
  auto row_sum = [&](double v) {
#pragma unroll
    for (int off = 1; off < 16; off <<= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
    return v;
  };
  // matrix of consumption step c (P_len for c = 0, else P_c) into m
  auto fetch = [&](int c, double2* m) {
    if (RING) {
      const int st = c % DS;
      mbar_wait(&full[tl * DS + st], (unsigned)((c / DS) & 1));
      const double2* src = ring + (size_t)(tl * DS + st) * dd + l;
#pragma unroll
      for (int t = 0; t < 8; ++t) m[t] = src[32 * t];
    } else {
      const double2* src = Pc + (size_t)(c ? c : len) * dd;
#pragma unroll
      for (int t = 0; t < 8; ++t) m[t] = __ldcs(src + 32 * t);
    }
  };
  // this warp is done with step c's stage; the producer refills step c - 1's stage (both
  // warps done with it) with step c - 1 + DS
  auto release = [&](int c) {
    if (RING) {
      __syncwarp();
      if (l == 0) mbar_arrive(&empty[tl * DS + c % DS]);
      if (producer && c >= 1 && c - 1 + DS <= len) {
        mbar_wait(&empty[tl * DS + (c - 1) % DS], (unsigned)(((c - 1) / DS) & 1));
        issue(c - 1 + DS);
      }
    }
  };
  double2 m[8];
  fetch(0, m);  // P_len
  double2 acc = cx(0.0, 0.0);
#pragma unroll
  for (int t = 0; t < 8; ++t) acc = cfma(m[t], phi[t], acc);
  const double2 psiL = half_sum(acc);  // row `row` of P_len phi
  const double2 targ = t_targ[tix + row];
  if (mode & PE_ENTRY) {
    const double tv = A.form == 0 ? cconjmul(targ, psiL).x : cabs2(csub(psiL, targ));
    const double s = row_sum(g == 0 ? tv : 0.0);
    if (l == 0) R.entry_pay[(size_t)b * P.L + n] = A.form == 0 ? (w * s) : (-0.5 * (w * s));
  }
  double pen = 0.0;
  for (int j = l; j < len; j += 32) pen += (P.alpha[node0 + j] * scale) * (u[j] * u[j]);
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) pen += __shfl_xor_sync(0xffffffffu, pen, off);
  double err = 0.0;
  if (mode & (PE_GRAD | PE_ERR)) {
    // chi_0[c] = sum_r conj(P_len[r][c]) seed[r]: lane keeps columns 2t + g
    const double2 seed = A.form == 0 ? targ : csub(targ, psiL);
    double2 chi0[8];
#pragma unroll
    for (int t = 0; t < 8; ++t) {
      double2 v = cconjmul(m[t], seed);
#pragma unroll
      for (int off = 1; off < 16; off <<= 1) v = cadd(v, shfl_xor(v, off));
      chi0[t] = v;
    }
    release(0);
    // row-distributed psi_0 = phi and chi_0 (column slots -> rows through shared memory)
    if (row == 0)
#pragma unroll
      for (int t = 0; t < 8; ++t) xs[warp][2 * t + g] = chi0[t];
    __syncwarp();
    double2 psi_prev = t_init[tix + row], chi_prev = xs[warp][row];
    if (l < len) {
      ush[warp][l] = u[l];
      ash[warp][l] = P.alpha[node0 + l];
    }
    __syncwarp();
    for (int j = 0; j < len; ++j) {
      fetch(j + 1, m);
      // two accumulators per product (even / odd column slots) halve the dependent fma chains
      double2 a0 = cx(0.0, 0.0), a1 = cx(0.0, 0.0), c0 = cx(0.0, 0.0), c1 = cx(0.0, 0.0);
#pragma unroll
      for (int t = 0; t < 8; t += 2) {
        a0 = cfma(m[t], phi[t], a0);
        c0 = cfma(m[t], chi0[t], c0);
        a1 = cfma(m[t + 1], phi[t + 1], a1);
        c1 = cfma(m[t + 1], chi0[t + 1], c1);
      }
      const double2 psi_n = half_sum(cadd(a0, a1)), chi_n = half_sum(cadd(c0, c1));
      release(j + 1);
      const double2 ps = cadd(psi_prev, psi_n), cs = cadd(chi_prev, chi_n);
      // (Hc ps)[row]: ps of column 2t + g read back from shared memory (broadcast)
      __syncwarp();
      if (g == 0) pss[warp][row] = ps;
      __syncwarp();
      double2 h0 = cx(0.0, 0.0), h1 = cx(0.0, 0.0);
#pragma unroll
      for (int t = 0; t < 8; t += 2) {
        h0 = cfma(hcs[(2 * t + g) * ND + row], pss[warp][2 * t + g], h0);
        h1 = cfma(hcs[(2 * t + 2 + g) * ND + row], pss[warp][2 * t + 2 + g], h1);
      }
      // Im <cs, Hc ps> = sum over all 32 lanes of Im(conj(cs_row) (this half's part of (Hc ps)_row))
      double im = cconjmul(cs, cadd(h0, h1)).y;
#pragma unroll
      for (int off = 1; off < 32; off <<= 1) im += __shfl_xor_sync(0xffffffffu, im, off);
      const double uj = ush[warp][j];
      const double gj = -(ash[warp][j] * scale) * dt * uj + 0.25 * dt * (w * im);
      if (l == 0 && (mode & PE_GRAD)) {
        // u + rho (w g) as one explicit fma in both orders (apply_pending_kernel repeats it)
        if (dual) R.gpend[(size_t)b * P.K + node0 + j] = weight * gj;
        else u[j] = __fma_rn(A.rho, weight * gj, uj);
      }
      err += fabs(gj);  // C = 1: ||g_j||_2 = |g_j| (error_norm, objective.cpp:152-160)
      psi_prev = psi_n;
      chi_prev = chi_n;
    }
  }
  if (l == 0) {
    if (handed_off_only) {
      R.err[(size_t)b * P.L + n] = err;
    } else if (dual) {
      if (role) R.chunk_pen[(size_t)b * P.L + n] = pen;
      else R.chunk_err[(size_t)b * P.L + n] = err;
    } else {
      R.chunk_pen[(size_t)b * P.L + n] = pen;
      R.chunk_err[(size_t)b * P.L + n] = err;
    }
  }
}

}  // namespace

// QOC_DISABLE="nm,eval16" switches either path off (A/B and bisection on the GPU box)
static bool disabled(const char* what) {
  const char* e = std::getenv("QOC_DISABLE");
  return e && std::strstr(e, what) != nullptr;
}

// The fused residual (RESIDUAL kernels) measured even with the separate streaming evaluation
// (28.9 vs 28.8 ms per config-5 iteration: +7 ms in the sweep vs one more 36 GB cache pass); it
// stays available behind QOC_ENABLE=fuse.
bool dense_nm_fuse_residual() {
  const char* e = std::getenv("QOC_ENABLE");
  return e && std::strstr(e, "fuse") != nullptr;
}

bool dense_nm_applicable(const DevProblem& P) {
  return P.kind == QOC_KIND_DENSE && P.d == ND && P.C == 1 && !P.has_quad && !disabled("nm");
}

cudaError_t dense_nm_setup(const DevProblem& P, const DevRun& R, cudaStream_t st) {
  dense_nm_setup_kernel<<<P.B, 32, 0, st>>>(P, R);
  return cudaGetLastError();
}

// pc_eval for the same problems when the evaluation needs only ENTRY / GRAD / ERR and the task
// is a single chunk (pc_finalize_kernel then reduces exactly as for pc_eval_kernel)
bool dense_pc_eval16_applicable(const DevProblem& P, const DevRun& R, int mode, int nchunk) {
  return R.nm && !disabled("eval16") && nchunk == 1 && (mode & ~7) == 0 && R.traj_len - 1 <= 32;
}

cudaError_t dense_pc_eval16(const DevProblem& P, const DevRun& R, const TaskArgs& A, int ignore_done, cudaStream_t st,
                            int handed_off_only, int dual) {
  if (dual == 1 && !disabled("ring")) {
    const size_t smem = sizeof(double2) * DT * DS * ND * ND + 2 * sizeof(unsigned long long) * DT * DS;
    cudaError_t e = cudaFuncSetAttribute(dense_pc_eval16_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem);
    if (e != cudaSuccess) return e;
    dense_pc_eval16_kernel<true><<<dim3((P.L + DT - 1) / DT, P.B), 256, smem, st>>>(P, R, A, ignore_done, 0, 1);
    return cudaGetLastError();
  }
  const int per = dual == 1 ? 4 : 8;
  dense_pc_eval16_kernel<false><<<dim3((P.L + per - 1) / per, P.B), 256, 0, st>>>(P, R, A, ignore_done, handed_off_only, dual);
  return cudaGetLastError();
}

size_t dense_nm_smem() {
  return sizeof(double2) * ((size_t)NM_TERMS * SLOTS * 32 + (size_t)NM_WARPS * ND * XS + SLOTS * 32);
}

// The complex product as three real tensor-core products (Gauss) instead of four: 48 instead of
// 64 DMMA per grid step (12.8 vs 13.4 ms per config-5 sweep); QOC_NM_GAUSS3=0 selects four.
static bool nm_gauss3() {
  const char* e = std::getenv("QOC_NM_GAUSS3");
  return !(e && e[0] == '0');
}

cudaError_t dense_nm_assemble(const DevProblem& P, const DevRun& R, int ignore_done, int residual, cudaStream_t st) {
  // QOC_NM_HB: steps per Horner batch (1, 2 or 4; default 2)
  const char* hbe = std::getenv("QOC_NM_HB");
  const int hb = hbe ? std::atoi(hbe) : 2;
  auto pick = [&](auto g3) {
    constexpr bool G = decltype(g3)::value;
    if (residual) return dense_nm_assemble_kernel<G, true, 1>;
    return hb == 4 ? dense_nm_assemble_kernel<G, false, 4>
                   : hb == 1 ? dense_nm_assemble_kernel<G, false, 1> : dense_nm_assemble_kernel<G, false, 2>;
  };
  auto kern = nm_gauss3() ? pick(std::true_type{}) : pick(std::false_type{});
  const size_t smem = dense_nm_smem();
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  kern<<<dim3((P.L + NM_WARPS - 1) / NM_WARPS, P.B), NM_WARPS * 32, smem, st>>>(P, R, ignore_done);
  return cudaGetLastError();
}

}  // namespace qoc
