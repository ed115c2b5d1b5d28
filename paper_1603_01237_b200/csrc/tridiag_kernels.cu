// tridiag_kernels.cu — ISM task/horizon kernels for Hermitian tridiagonal operators
// (QOC_KIND_TRIDIAG, d <= 30; BASELINE config 2, the rigid rotor of models.cpp:349-359).
//
// One warp per (problem, subinterval) task, one lane per right-hand-side column.  Each lane
// runs the Thomas elimination of B = I + s H(u_j) (s = +-i dt/2) on its own column: the
// elimination coefficients are recomputed redundantly by every lane (no communication), and
// equal the partial-pivot LU the reference forms with Eigen (propagation.cpp:85-106) because
// B is strictly diagonally dominant -- a row interchange would be required only if
// |a_i| > |u_{i-1}|, which is detected and reported (QOC_ERUNTIME).
//   phase 1 (control u):  lane-redundant single-vector forward sweep (trajectory to global),
//                         adjoint sweep with the fused gradient + in-place update.
//   phase 2 (updated u):  lanes 0..d-1 carry the identity columns (propagator assembly,
//                         propagation.cpp:236-249), lane d the residual state, lane d+1 the
//                         lagged split state; then lane 0 the residual adjoint and lane 1 the
//                         lagged adjoint.
#include "kernels.h"

namespace qoc {

namespace {

struct TriView {
  const double* diag;   // [nops][d]
  const double2* sub;   // [nops][d-1]
  int d, C, has_quad;
};

// Bands of H(u) = H0 + sum u_c A_c + sum (u_c^2/2) B_c at row i: the real diagonal entry and
// the sub-diagonal entry (i, i-1) (zero for i = 0 or i >= d).
__device__ __forceinline__ void bands_at(const TriView& T, const double* u, int i, double& dg, double2& sb) {
  dg = 0.0;
  sb = cx(0.0, 0.0);
  if (i >= T.d) return;
  dg = T.diag[i];
  if (i > 0) sb = T.sub[i - 1];
  for (int c = 0; c < T.C; ++c) {
    dg = fma(u[c], T.diag[(1 + c) * T.d + i], dg);
    if (i > 0) {
      const double2 a = T.sub[(size_t)(1 + c) * (T.d - 1) + i - 1];
      sb = cx(fma(u[c], a.x, sb.x), fma(u[c], a.y, sb.y));
    }
  }
  if (T.has_quad) {
    for (int c = 0; c < T.C; ++c) {
      const double s = 0.5 * u[c] * u[c];
      dg = fma(s, T.diag[(1 + T.C + c) * T.d + i], dg);
      if (i > 0) {
        const double2 a = T.sub[(size_t)(1 + T.C + c) * (T.d - 1) + i - 1];
        sb = cx(fma(s, a.x, sb.x), fma(s, a.y, sb.y));
      }
    }
  }
}

// x <- (I + sH)^-1 (I - sH) x,  s = (0, sh); x holds d <= TD entries.
// Returns false when partial pivoting would have interchanged rows.
template <int TD>
__device__ __forceinline__ bool cayley_tri_inl(const TriView& T, const double* u, double sh, double2 (&x)[TD]) {
  const int d = T.d;
  double2 uinv[TD];
  bool ok = true;
  double dg_i, dg_n;
  double2 sb_i, sb_n;
  bands_at(T, u, 0, dg_i, sb_i);
  double2 xo_prev = cx(0.0, 0.0);  // original x_{i-1}
  double2 c_prev = cx(0.0, 0.0);   // c_{i-1} = s conj(sb_i)
#pragma unroll
  for (int i = 0; i < TD; ++i) {
    if (i < d) {
      bands_at(T, u, i + 1, dg_n, sb_n);
      const double2 xo = x[i];
      // h = (H x)_i = sb_i x_{i-1} + dg_i x_i + conj(sb_{i+1}) x_{i+1}
      double2 h = cx(dg_i * xo.x, dg_i * xo.y);
      if (i > 0) h = cfma(sb_i, xo_prev, h);
      if (i + 1 < d) h = cfmaconj(sb_n, x[i + 1], h);
      // r = x - s h,  s h = (-sh hi, sh hr)
      double2 r = cx(xo.x + sh * h.y, xo.y - sh * h.x);
      double2 ui = cx(1.0, sh * dg_i);
      if (i > 0) {
        const double2 a = cx(-sh * sb_i.y, sh * sb_i.x);  // s sb_i
        ok = ok && !(cabs2(a) * cabs2(uinv[i - 1]) > 1.0);  // |a_i| > |u_{i-1}| would pivot
        const double2 l = cmul(a, uinv[i - 1]);
        ui = cfms(l, c_prev, ui);
        r = cfms(l, x[i - 1], r);
      }
      uinv[i] = crcp(ui);
      c_prev = cx(sh * sb_n.y, sh * sb_n.x);  // s conj(sb_{i+1})
      xo_prev = xo;
      x[i] = r;
      dg_i = dg_n;
      sb_i = sb_n;
    }
  }
#pragma unroll
  for (int i = TD - 1; i >= 0; --i) {
    if (i < d) {
      double2 v = x[i];
      if (i + 1 < d) {
        double dg;
        double2 sb;
        bands_at(T, u, i + 1, dg, sb);
        v = cfms(cx(sh * sb.y, sh * sb.x), x[i + 1], v);
      }
      x[i] = cmul(v, uinv[i]);
    }
  }
  return ok;
}

// Out-of-line copy for the multi-sweep task/horizon kernels: inlining the unrolled solve at
// every call site made ptxas time explode; the state round-trips through local memory
// (L1-resident) there, while the hot assembly sweep below keeps the inlined form.
template <int TD>
__device__ __noinline__ bool cayley_tri(const TriView& T, const double* u, double sh, double2 (&x)[TD]) {
  return cayley_tri_inl<TD>(T, u, sh, x);
}

// Im sum_i conj(cs_i) (dH/du_c ps)_i with ps_i = p0[i] + p1[i] read from the trajectory.
template <int TD>
__device__ __forceinline__ double grad_im(const TriView& T, int c, double uc, const double2 (&ca)[TD],
                                          const double2 (&cb)[TD], const double2* p0, const double2* p1) {
  const int d = T.d;
  double2 acc = cx(0.0, 0.0);
  double2 ps_prev = cx(0.0, 0.0);
  double2 ps_i = cadd(p0[0], p1[0]);
#pragma unroll
  for (int i = 0; i < TD; ++i) {
    if (i < d) {
      const double2 ps_n = (i + 1 < d) ? cadd(p0[i + 1], p1[i + 1]) : cx(0.0, 0.0);
      double dg = T.diag[(1 + c) * d + i];
      if (T.has_quad) dg = fma(uc, T.diag[(1 + T.C + c) * d + i], dg);
      double2 h = cx(dg * ps_i.x, dg * ps_i.y);
      if (i > 0) {
        double2 s = T.sub[(size_t)(1 + c) * (d - 1) + i - 1];
        if (T.has_quad) {
          const double2 q = T.sub[(size_t)(1 + T.C + c) * (d - 1) + i - 1];
          s = cx(fma(uc, q.x, s.x), fma(uc, q.y, s.y));
        }
        h = cfma(s, ps_prev, h);
      }
      if (i + 1 < d) {
        double2 s = T.sub[(size_t)(1 + c) * (d - 1) + i];
        if (T.has_quad) {
          const double2 q = T.sub[(size_t)(1 + T.C + c) * (d - 1) + i];
          s = cx(fma(uc, q.x, s.x), fma(uc, q.y, s.y));
        }
        h = cfmaconj(s, ps_n, h);
      }
      acc = cfmaconj(cadd(ca[i], cb[i]), h, acc);
      ps_prev = ps_i;
      ps_i = ps_n;
    }
  }
  return acc.y;
}

template <int TD>
__global__ void __launch_bounds__(32) tridiag_task_kernel(DevProblem P, DevRun R, TaskArgs A, int ignore_done) {
  const int n = blockIdx.x, b = blockIdx.y, lane = threadIdx.x;
  if (ignore_done ? R.status[b] : (R.done[b] | R.status[b])) return;
  const int d = P.d, C = P.C;
  const int nops = 1 + C + (P.has_quad ? C : 0);
  const TriView T{P.tri_diag + (size_t)b * nops * d, P.tri_sub + (size_t)b * nops * (d - 1), d, C, P.has_quad};
  const int node0 = P.node[n], len = P.node[n + 1] - node0;
  const double Kd = (double)P.K;
  const double weight = A.weighted ? Kd / (double)len : 1.0;
  const double scale = (double)len / Kd;
  const double half = 0.5 * P.dt, dt = P.dt, w = P.ip_w;
  double* u = R.u + ((size_t)b * P.K + node0) * C;
  double2* traj = R.traj + ((size_t)b * P.L + n) * (size_t)R.traj_len * d;
  const size_t tix = ((size_t)b * P.L + n) * d;
  const double2 zero = cx(0.0, 0.0);
  const int mode = A.mode;
  bool ok = true;
  double2 x[TD], y[TD];

  if (mode & (M_ENTRY | M_UPDATE | M_FINAL | M_GRAD)) {
    const bool need_traj = (mode & (M_UPDATE | M_GRAD)) != 0;
    const int iters = (mode & M_UPDATE) ? A.inner : 1;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int i = 0; i < TD; ++i) x[i] = i < d ? R.task_init[tix + i] : zero;
      double pen = 0.0;
      if (need_traj && lane == 0)
        for (int i = 0; i < TD; ++i) if (i < d) traj[i] = x[i];
      for (int j = 0; j < len; ++j) {
        const double* uj = u + (size_t)j * C;
        ok &= cayley_tri<TD>(T, uj, half, x);
        if (need_traj && lane == 0)
          for (int i = 0; i < TD; ++i) if (i < d) traj[(size_t)(j + 1) * d + i] = x[i];
        double sq = 0.0;
        for (int c = 0; c < C; ++c) sq += uj[c] * uj[c];
        pen += (P.alpha[node0 + j] * scale) * sq;
      }
      if (it == 0 && (mode & M_ENTRY) && lane == 0) {
        double s = 0.0;
#pragma unroll
        for (int i = 0; i < TD; ++i) {
          if (i < d) {
            const double2 t = R.task_targ[tix + i];
            s += A.form == 0 ? cconjmul(t, x[i]).x : cabs2(csub(x[i], t));
          }
        }
        const double payoff = A.form == 0 ? (w * s) : (-0.5 * (w * s));
        R.entry[(size_t)b * P.L + n] = weight * (payoff - 0.5 * dt * pen);
      }
      if (it == 0 && (mode & M_FINAL) && lane == 0)
        for (int i = 0; i < TD; ++i) if (i < d) R.psi_end[tix + i] = x[i];
      if (mode & (M_UPDATE | M_GRAD)) {
#pragma unroll
        for (int i = 0; i < TD; ++i) {
          const double2 t = i < d ? R.task_targ[tix + i] : zero;
          y[i] = A.form == 0 ? t : csub(t, x[i]);  // adjoint seed (objective.cpp:31-34)
        }
        __syncwarp();
        for (int j = len - 1; j >= 0; --j) {
          const double* uj = u + (size_t)j * C;
#pragma unroll
          for (int i = 0; i < TD; ++i) x[i] = y[i];
          ok &= cayley_tri<TD>(T, uj, -half, x);  // x = chi_j, y = chi_{j+1}
          const double aj = P.alpha[node0 + j] * scale;
          double gcs[MAXC];
          for (int c = 0; c < C; ++c) {
            const double uc = uj[c];
            const double im = grad_im<TD>(T, c, uc, x, y, traj + (size_t)j * d, traj + (size_t)(j + 1) * d);
            gcs[c] = -aj * dt * uc + 0.25 * dt * (w * im);
          }
          __syncwarp();
          if (lane == 0) {
            for (int c = 0; c < C; ++c) {
              if (mode & M_GRAD) R.grad[((size_t)b * P.K + node0 + j) * C + c] = gcs[c];
              if (mode & M_UPDATE) u[(size_t)j * C + c] = uj[c] + A.rho * (weight * gcs[c]);
            }
          }
          __syncwarp();
#pragma unroll
          for (int i = 0; i < TD; ++i) y[i] = x[i];
        }
      }
      __syncwarp();
    }
  }

  const bool do_err = (mode & M_ERROR) != 0, do_asm = (mode & M_ASSEMBLE) != 0, do_lag = (mode & M_LAGGED) != 0;
  if (do_err || do_asm || do_lag) {
    const bool role_asm = do_asm && lane < d;
    const bool role_err = do_err && lane == d;
    const bool role_lag = do_lag && lane == d + 1;
    const double2* src = role_err ? R.task_init + tix
                                  : (role_lag ? R.psi_nodes + ((size_t)b * (P.L + 1) + n) * d : nullptr);
#pragma unroll
    for (int i = 0; i < TD; ++i) x[i] = src ? (i < d ? src[i] : zero) : cx(i == lane ? 1.0 : 0.0, 0.0);
    if (role_err)
      for (int i = 0; i < TD; ++i) if (i < d) traj[i] = x[i];
    for (int j = 0; j < len; ++j) {
      ok &= cayley_tri<TD>(T, u + (size_t)j * C, half, x);
      if (role_err)
        for (int i = 0; i < TD; ++i) if (i < d) traj[(size_t)(j + 1) * d + i] = x[i];
    }
    if (role_asm) {
      double2* M = R.prop + ((size_t)b * P.L + n) * (size_t)d * d;
#pragma unroll
      for (int i = 0; i < TD; ++i)
        if (i < d) M[(size_t)i * d + lane] = x[i];
    }
    if (role_lag)
      for (int i = 0; i < TD; ++i) if (i < d) R.psi_end[tix + i] = x[i];
    __syncwarp();
    if (do_err || do_lag) {
      const bool adj_err = do_err && lane == 0;
      const bool adj_lag = do_lag && lane == 1;
      // residual seed from the final residual state (written to traj[len] by lane d)
#pragma unroll
      for (int i = 0; i < TD; ++i) {
        double2 v = zero;
        if (i < d) {
          if (adj_lag) {
            v = R.chi_nodes[((size_t)b * (P.L + 1) + n + 1) * d + i];
          } else if (do_err) {
            const double2 t = R.task_targ[tix + i];
            v = A.form == 0 ? t : csub(t, traj[(size_t)len * d + i]);
          }
        }
        y[i] = v;
      }
      double err = 0.0;
      for (int j = len - 1; j >= 0; --j) {
        const double* uj = u + (size_t)j * C;
#pragma unroll
        for (int i = 0; i < TD; ++i) x[i] = y[i];
        ok &= cayley_tri<TD>(T, uj, -half, x);
        if (adj_err) {
          const double aj = P.alpha[node0 + j] * scale;
          double sq = 0.0;
          for (int c = 0; c < C; ++c) {
            const double uc = uj[c];
            const double im = grad_im<TD>(T, c, uc, x, y, traj + (size_t)j * d, traj + (size_t)(j + 1) * d);
            const double gc = -aj * dt * uc + 0.25 * dt * (w * im);
            sq += gc * gc;
          }
          err += sqrt(sq);
        }
#pragma unroll
        for (int i = 0; i < TD; ++i) y[i] = x[i];
      }
      if (adj_err) R.err[(size_t)b * P.L + n] = err;
      if (adj_lag)
        for (int i = 0; i < TD; ++i) if (i < d) R.chi_start[tix + i] = y[i];
    }
  }
  if (!ok && R.err_flags) atomicOr(R.err_flags, 1);
}

template <int TD>
__global__ void __launch_bounds__(32) tridiag_horizon_kernel(DevProblem P, DevRun R, int which, int k) {
  if (R.kdev) k = *R.kdev;
  const int b = blockIdx.x, lane = threadIdx.x;
  if (R.done[b] || R.status[b] || lane != 0) return;
  const int d = P.d, C = P.C;
  const int nops = 1 + C + (P.has_quad ? C : 0);
  const TriView T{P.tri_diag + (size_t)b * nops * d, P.tri_sub + (size_t)b * nops * (d - 1), d, C, P.has_quad};
  const double half = 0.5 * P.dt;
  const double* u = R.u + (size_t)b * P.K * C;
  const size_t nb = (size_t)b * (P.L + 1) * d;
  bool ok = true;
  double2 x[TD];
#pragma unroll
  for (int i = 0; i < TD; ++i) x[i] = i < d ? P.init[(size_t)b * d + i] : cx(0.0, 0.0);
  if (which == 0)
    for (int i = 0; i < TD; ++i) if (i < d) R.psi_nodes[nb + i] = x[i];
  int nxt = 1;
  for (int j = 0; j < P.K; ++j) {
    ok &= cayley_tri<TD>(T, u + (size_t)j * C, half, x);
    if (which == 0 && nxt <= P.L && P.node[nxt] == j + 1) {
      for (int i = 0; i < TD; ++i) if (i < d) R.psi_nodes[nb + (size_t)nxt * d + i] = x[i];
      ++nxt;
    }
  }
  if (which == 1) {
    double s = 0.0;
    for (int i = 0; i < TD; ++i) if (i < d) s += cconjmul(P.targ[(size_t)b * d + i], x[i]).x;
    double pen = 0.0;
    for (int n = 0; n < P.L; ++n) pen += R.pen[(size_t)b * P.L + n];
    R.rec_exact[(size_t)b * R.cap + k] = P.ip_w * s - 0.5 * P.dt * pen;
  } else {
#pragma unroll
    for (int i = 0; i < TD; ++i) x[i] = i < d ? P.targ[(size_t)b * d + i] : cx(0.0, 0.0);
    for (int i = 0; i < TD; ++i) if (i < d) R.chi_nodes[nb + (size_t)P.L * d + i] = x[i];
    int prev = P.L - 1;
    for (int j = P.K - 1; j >= 0; --j) {
      ok &= cayley_tri<TD>(T, u + (size_t)j * C, -half, x);
      if (prev >= 0 && P.node[prev] == j) {
        for (int i = 0; i < TD; ++i) if (i < d) R.chi_nodes[nb + (size_t)prev * d + i] = x[i];
        --prev;
      }
    }
  }
  if (!ok && R.err_flags) atomicOr(R.err_flags, 1);
}

// Assembly sweep of the propagator cache (pcache.cu): P_{j+1} = C_j P_j, lane k carries
// column k of P_j.  The LU factors of B_j = I + s H(u_j) depend on u_j only, so they are
// computed step-parallel (lane q factors step j0 + q of a 32-step chunk, into shared memory)
// and the sequential sweep over j only applies the factored solve: per step and column one
// tridiagonal matvec (I - sH) x, one forward and one backward substitution -- no band
// recomputation and no global loads on the dependent chain.
constexpr int TRI_CHUNK = 32;

template <int TD>
struct TriFactors {
  double2 lf[TRI_CHUNK][TD];  // elimination multipliers l_i = a_i / u_{i-1}
  double2 cs[TRI_CHUNK][TD];  // super-diagonal c_i = s conj(sb_{i+1})
  double2 ui[TRI_CHUNK][TD];  // 1 / u_i
};

template <int TD>
__global__ void __launch_bounds__(32) tri_pc_assemble_kernel(DevProblem P, DevRun R, int ignore_done) {
  const int n = blockIdx.x, b = blockIdx.y, lane = threadIdx.x;
  if (ignore_done ? R.status[b] : (R.done[b] | R.status[b])) return;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  TriFactors<TD>& F = *reinterpret_cast<TriFactors<TD>*>(smem_raw);
  const int d = P.d, C = P.C;
  const int nops = 1 + C + (P.has_quad ? C : 0);
  const TriView T{P.tri_diag + (size_t)b * nops * d, P.tri_sub + (size_t)b * nops * (d - 1), d, C, P.has_quad};
  const int node0 = P.node[n], len = P.node[n + 1] - node0;
  const double half = 0.5 * P.dt;
  const double* u = R.u + ((size_t)b * P.K + node0) * C;
  const size_t dd = (size_t)d * d;
  double2* Pc = R.pc + ((size_t)b * P.L + n) * (size_t)R.traj_len * dd;
  const bool col = lane < d;
  bool ok = true;
  double2 x[TD];
#pragma unroll
  for (int i = 0; i < TD; ++i) x[i] = cx(i == lane ? 1.0 : 0.0, 0.0);
  if (col)
#pragma unroll
    for (int i = 0; i < TD; ++i)
      if (i < d) Pc[(size_t)i * d + lane] = x[i];
  for (int j0 = 0; j0 < len; j0 += TRI_CHUNK) {
    const int cnt = min(TRI_CHUNK, len - j0);
    __syncwarp();
    if (lane < cnt) {  // factor B_j = I + sH(u_j), s = i*half (oracle.cpp TriM::cayley)
      const double* uj = u + (size_t)(j0 + lane) * C;
      double2 uinv_prev = cx(0.0, 0.0);
      double dg;
      double2 sb;
      bands_at(T, uj, 0, dg, sb);
      for (int i = 0; i < d; ++i) {
        double dgn;
        double2 sbn;
        bands_at(T, uj, i + 1, dgn, sbn);  // zero beyond the last row
        double2 ui = cx(1.0, half * dg);
        double2 lf = cx(0.0, 0.0);
        if (i > 0) {
          const double2 a = cx(-half * sb.y, half * sb.x);      // s sb_i
          ok = ok && !(cabs2(a) * cabs2(uinv_prev) > 1.0);     // |a_i| > |u_{i-1}| would pivot
          lf = cmul(a, uinv_prev);
          ui = cfms(lf, cx(half * sb.y, half * sb.x), ui);     // - l_i * s conj(sb_i)
        }
        uinv_prev = crcp(ui);
        F.lf[lane][i] = lf;
        F.ui[lane][i] = uinv_prev;
        F.cs[lane][i] = cx(half * sbn.y, half * sbn.x);         // s conj(sb_{i+1})
        dg = dgn;
        sb = sbn;
      }
    }
    __syncwarp();
    // C_j x = (I + sH)^-1 (I - sH) x = 2 z - x with (I + sH) z = x: one forward and one
    // backward substitution per column, no right-hand-side matvec.
    for (int q = 0; q < cnt; ++q) {
      const double2* flf = F.lf[q];
      const double2* fcs = F.cs[q];
      const double2* fui = F.ui[q];
      double2 z[TD];
#pragma unroll
      for (int i = 0; i < TD; ++i)
        if (i < d) z[i] = i > 0 ? cfms(flf[i], z[i - 1], x[i]) : x[i];
#pragma unroll
      for (int i = TD - 1; i >= 0; --i) {
        if (i < d) {
          const double2 v = (i + 1 < d) ? cfms(fcs[i], z[i + 1], z[i]) : z[i];
          z[i] = cmul(v, fui[i]);
          x[i] = cx(fma(2.0, z[i].x, -x[i].x), fma(2.0, z[i].y, -x[i].y));
        }
      }
      if (col) {
        double2* dst = Pc + (size_t)(j0 + q + 1) * dd;
#pragma unroll
        for (int i = 0; i < TD; ++i)
          if (i < d) dst[(size_t)i * d + lane] = x[i];
      }
    }
  }
  if (col && R.prop) {
    double2* M = R.prop + ((size_t)b * P.L + n) * dd;
#pragma unroll
    for (int i = 0; i < TD; ++i)
      if (i < d) M[(size_t)i * d + lane] = x[i];
  }
  ok = __all_sync(0xffffffffu, ok);
  if (!ok && lane == 0 && R.err_flags) atomicOr(R.err_flags, 1);
}

// Twisted ("burn at both ends") variant of the cache sweep: two warps per task, compiled for
// an exact dimension (the BASELINE rotor, d = 21) so each warp's row loops cover only its half.  Warp 0
// eliminates rows 0..m-1 top-down (LU), warp 1 rows d-1..m+1 bottom-up (UL), they meet at the
// middle row m = d/2 through shared memory, then substitute outward concurrently.  The serial
// dependent chain per step -- the bound of the one-warp kernel -- is halved.  Factors are
// again computed step-parallel per 32-step chunk (warp 0 the LU side and the reference's
// pivot check, warp 1 the UL side).  Same Cayley map; rounding differs from the LU sweep at
// the 1e-16 level (diagonally dominant B, no pivoting on either side).
template <int TD>
struct TwistFactors {
  double2 lf[TRI_CHUNK][TD];   // top: l_i = a_i / u_{i-1} (i = 1..m)
  double2 ui[TRI_CHUNK][TD];   // top: 1 / u_i (i = 0..m-1)
  double2 cs[TRI_CHUNK][TD];   // c_i = s conj(sb_{i+1}) (super)
  double2 as[TRI_CHUNK][TD];   // a_i = s sb_i (sub)
  double2 kf[TRI_CHUNK][TD];   // bottom: k_i = c_i / w_{i+1} (i = m..d-2)
  double2 wi[TRI_CHUNK][TD];   // bottom: 1 / w_i (i = m+1..d-1)
  double2 cu[TRI_CHUNK][TD];   // top: c_i / u_i  (back substitution z_i = z'_i/u_i - (c_i/u_i) z_{i+1})
  double2 au[TRI_CHUNK][TD];   // bottom: a_i / w_i
  double2 gm[TRI_CHUNK];       // 1 / gamma_m
  double2 bm[TRI_CHUNK];       // b_m (middle diagonal)
  double2 zt[2][32];           // z'_{m-1} per column (top -> middle), double-buffered by step
  double2 zb[2][32];           // z''_{m+1} per column (bottom -> middle)
};

template <int TD, int DIM>
__global__ void __launch_bounds__(64) tri_pc_assemble2_kernel(DevProblem P, DevRun R, int ignore_done) {
  const int n = blockIdx.x, b = blockIdx.y, lane = threadIdx.x & 31, side = threadIdx.x >> 5;
  if (ignore_done ? R.status[b] : (R.done[b] | R.status[b])) return;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  TwistFactors<TD>& F = *reinterpret_cast<TwistFactors<TD>*>(smem_raw);
  constexpr int d = DIM, m = DIM / 2;  // compile-time: every row loop unrolls to its own half
  const int C = P.C;
  const int nops = 1 + C + (P.has_quad ? C : 0);
  const TriView T{P.tri_diag + (size_t)b * nops * d, P.tri_sub + (size_t)b * nops * (d - 1), d, C, P.has_quad};
  const int node0 = P.node[n], len = P.node[n + 1] - node0;
  const double half = 0.5 * P.dt;
  const double* u = R.u + ((size_t)b * P.K + node0) * C;
  const size_t dd = (size_t)d * d;
  double2* Pc = R.pc + ((size_t)b * P.L + n) * (size_t)R.traj_len * dd;
  const bool col = lane < d;
  bool ok = true;
  // rows owned: top [0, m], bottom [m, d-1] (the middle row in both)
  const int r0 = side == 0 ? 0 : m, r1 = side == 0 ? m : d - 1;
  double2 x[TD];
#pragma unroll
  for (int i = 0; i < TD; ++i) x[i] = cx(i == lane ? 1.0 : 0.0, 0.0);
  if (col)
#pragma unroll
    for (int i = 0; i < TD; ++i)
      if (i < d && i >= r0 && i <= r1 && (side == 0 || i > m)) Pc[(size_t)i * d + lane] = x[i];
  auto sband = [&](const double* uj, int i, double& dg, double2& sb) { bands_at(T, uj, i, dg, sb); };
  for (int j0 = 0; j0 < len; j0 += TRI_CHUNK) {
    const int cnt = min(TRI_CHUNK, len - j0);
    __syncthreads();
    if (lane < cnt) {
      const double* uj = u + (size_t)(j0 + lane) * C;
      if (side == 0) {
        // LU top-down over rows 0..m (and the full-LU pivot check of the reference solve)
        double2 uinv_prev = cx(0.0, 0.0);
        double dg;
        double2 sb;
        sband(uj, 0, dg, sb);
        for (int i = 0; i < d; ++i) {
          double dgn;
          double2 sbn;
          sband(uj, i + 1, dgn, sbn);
          const double2 bi = cx(1.0, half * dg);
          const double2 ci = cx(half * sbn.y, half * sbn.x);  // s conj(sb_{i+1})
          double2 ui = bi, lf = cx(0.0, 0.0);
          if (i > 0) {
            const double2 a = cx(-half * sb.y, half * sb.x);  // s sb_i
            ok = ok && !(cabs2(a) * cabs2(uinv_prev) > 1.0);
            lf = cmul(a, uinv_prev);
            ui = cfms(lf, cx(half * sb.y, half * sb.x), ui);
          }
          uinv_prev = crcp(ui);
          if (i <= m) {
            F.lf[lane][i] = lf;
            F.cs[lane][i] = ci;
            if (i < m) {
              F.ui[lane][i] = uinv_prev;
              F.cu[lane][i] = cmul(ci, uinv_prev);
            }
            if (i == m) F.bm[lane] = bi;
          }
          dg = dgn;
          sb = sbn;
        }
      } else {
        // UL bottom-up over rows d-1..m
        double2 winv_next = cx(0.0, 0.0);
        for (int i = d - 1; i >= m; --i) {
          double dg, dgn;
          double2 sb, sbn;
          sband(uj, i, dg, sb);
          sband(uj, i + 1, dgn, sbn);
          const double2 ci = cx(half * sbn.y, half * sbn.x);  // c_i = s conj(sb_{i+1})
          const double2 ai = cx(-half * sb.y, half * sb.x);   // a_i = s sb_i
          F.as[lane][i] = ai;
          double2 kf = cx(0.0, 0.0), wi = cx(1.0, half * dg);
          if (i + 1 < d) {
            kf = cmul(ci, winv_next);
            wi = cfms(kf, F.as[lane][i + 1], wi);  // b_i - k_i a_{i+1}
          }
          F.kf[lane][i] = kf;
          if (i > m) {
            winv_next = crcp(wi);
            F.wi[lane][i] = winv_next;
            F.au[lane][i] = cmul(ai, winv_next);
          }
        }
      }
    }
    __syncthreads();
    if (side == 0 && lane < cnt) {  // gamma_m = b_m - l_m c_{m-1} - k_m a_{m+1}
      double2 g = F.bm[lane];
      if (m > 0) g = cfms(F.lf[lane][m], F.cs[lane][m - 1], g);
      if (m + 1 < d) g = cfms(F.kf[lane][m], F.as[lane][m + 1], g);
      F.gm[lane] = crcp(g);
    }
    __syncthreads();
    for (int q = 0; q < cnt; ++q) {
      const int par = q & 1;
      double2 z[TD];
      if (side == 0) {
#pragma unroll
        for (int i = 0; i < TD; ++i)
          if (i < m) z[i] = i > 0 ? cfms(F.lf[q][i], z[i - 1], x[i]) : x[i];
#pragma unroll
        for (int i = 0; i < TD; ++i)
          if (i + 1 == m) F.zt[par][lane] = z[i];  // static register index
#pragma unroll
        for (int i = 0; i < TD; ++i)
          if (i < m) z[i] = cmul(z[i], F.ui[q][i]);  // z'_i / u_i, off the back-substitution chain
      } else {
#pragma unroll
        for (int i = TD - 1; i >= 0; --i)
          if (i < d && i > m) z[i] = (i + 1 < d) ? cfms(F.kf[q][i], z[i + 1], x[i]) : x[i];
#pragma unroll
        for (int i = 0; i < TD; ++i)
          if (i == m + 1 && i < d) F.zb[par][lane] = z[i];
#pragma unroll
        for (int i = 0; i < TD; ++i)
          if (i < d && i > m) z[i] = cmul(z[i], F.wi[q][i]);
      }
      __syncthreads();
      // middle row (both warps, identical arithmetic)
      double2 xm = x[0];
#pragma unroll
      for (int i = 0; i < TD; ++i)
        if (i == m) xm = x[i];
      double2 zm = xm;
      if (m > 0) zm = cfms(F.lf[q][m], F.zt[par][lane], zm);
      if (m + 1 < d) zm = cfms(F.kf[q][m], F.zb[par][lane], zm);
      zm = cmul(zm, F.gm[q]);
      double2* dst = Pc + (size_t)(j0 + q + 1) * dd;
      if (side == 0) {
        double2 zn = zm;
#pragma unroll
        for (int i = TD - 1; i >= 0; --i) {
          if (i < m) {
            zn = cfms(F.cu[q][i], zn, z[i]);  // one complex FMA per row on the chain
            x[i] = cx(fma(2.0, zn.x, -x[i].x), fma(2.0, zn.y, -x[i].y));
            if (col) dst[(size_t)i * d + lane] = x[i];
          }
        }
      } else {
        double2 zp = zm;
#pragma unroll
        for (int i = 0; i < TD; ++i) {
          if (i < d && i > m) {
            zp = cfms(F.au[q][i], zp, z[i]);
            x[i] = cx(fma(2.0, zp.x, -x[i].x), fma(2.0, zp.y, -x[i].y));
            if (col) dst[(size_t)i * d + lane] = x[i];
          }
        }
      }
      xm = cx(fma(2.0, zm.x, -xm.x), fma(2.0, zm.y, -xm.y));
#pragma unroll
      for (int i = 0; i < TD; ++i)
        if (i == m) x[i] = xm;
      if (side == 0 && col) dst[(size_t)m * d + lane] = xm;
    }
  }
  if (col && R.prop) {
    double2* M = R.prop + ((size_t)b * P.L + n) * dd;
#pragma unroll
    for (int i = 0; i < TD; ++i)
      if (i < d && ((side == 0 && i <= m) || (side == 1 && i > m))) M[(size_t)i * d + lane] = x[i];
  }
  ok = __all_sync(0xffffffffu, ok);
  if (!ok && lane == 0 && side == 0 && R.err_flags) atomicOr(R.err_flags, 1);
}

}  // namespace

cudaError_t tri_pc_assemble(const DevProblem& P, const DevRun& R, int ignore_done, cudaStream_t st) {
  if (P.d > 30) return cudaErrorNotSupported;
  if (P.d == 21) {
    auto k = tri_pc_assemble2_kernel<24, 21>;
    const int smem = (int)sizeof(TwistFactors<24>);
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    k<<<dim3(P.L, P.B), 64, smem, st>>>(P, R, ignore_done);
    return cudaGetLastError();
  }
  if (P.d <= 24) {
    auto k = tri_pc_assemble_kernel<24>;
    const int smem = (int)sizeof(TriFactors<24>);
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    k<<<dim3(P.L, P.B), 32, smem, st>>>(P, R, ignore_done);
  } else {
    auto k = tri_pc_assemble_kernel<32>;
    const int smem = (int)sizeof(TriFactors<32>);
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    k<<<dim3(P.L, P.B), 32, smem, st>>>(P, R, ignore_done);
  }
  return cudaGetLastError();
}

cudaError_t tridiag_task(const DevProblem& P, const DevRun& R, const TaskArgs& A, int ignore_done, cudaStream_t st) {
  if (P.d > 30) return cudaErrorNotSupported;
  if (P.d <= 24)
    tridiag_task_kernel<24><<<dim3(P.L, P.B), 32, 0, st>>>(P, R, A, ignore_done);
  else
    tridiag_task_kernel<32><<<dim3(P.L, P.B), 32, 0, st>>>(P, R, A, ignore_done);
  return cudaGetLastError();
}

cudaError_t tridiag_horizon(const DevProblem& P, const DevRun& R, int which, int k, cudaStream_t st) {
  if (P.d > 30) return cudaErrorNotSupported;
  if (P.d <= 24)
    tridiag_horizon_kernel<24><<<P.B, 32, 0, st>>>(P, R, which, k);
  else
    tridiag_horizon_kernel<32><<<P.B, 32, 0, st>>>(P, R, which, k);
  return cudaGetLastError();
}

}  // namespace qoc
