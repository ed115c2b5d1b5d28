// strang_kernels.cu — split-step (Strang) condensate kernels (QOC_KIND_STRANG; BASELINE
// config 4, the 1024-point Gross-Pitaevskii lattice, and the reference's 50-point trap preset).
//
// One CTA of 256 threads per (problem, subinterval) task.  The state and three work vectors
// live in shared memory; every kinetic half step is
//     spectral(psi, phase) = idft(phase . dft(psi))          (propagation.cpp:27-31)
// evaluated as two unnormalised transforms with the 1/n of the two unitary 1/sqrt(n) factors
// folded into the phase multiply.  Powers of two use a Stockham radix-4 autosort FFT in
// shared memory (phase multiply fused into the first stage, twiddles staged once per CTA);
// other sizes (<= 256 points, e.g. the reference's 50-point preset) use the
// direct O(n^2) sum of linalg.cpp:37-50 against a precomputed DFT matrix.  (The transform is
// a Stockham radix-4 FFT; `src` is used as scratch and is clobbered.)
//
// Forward step (strang_step, propagation.cpp:131-139): kinetic half phase, potential +
// kappa |psi_a|^2 phase, kinetic half phase.  Backward stage (strang_backward_stage,
// propagation.cpp:146-170): recompute the midpoint from the stored forward state psi_j,
// chi_b = kinetic-adjoint(chi_{j+1}), the real-linear transpose
//     chi_a = conj(p) chi_b + q conj(chi_b),  p = flow (1 - i dt kappa |psi_a|^2),
//     q = -i dt kappa flow psi_a^2
// (or conj(flow) chi_b for the naive adjoint), chi_j = kinetic-adjoint(chi_a), and the
// gradient dt dx Im sum conj(chi_b) dV/du psi_b (objective.cpp:72-84).  The forward
// trajectory of a task lives in HBM (R.traj); node sweeps over the whole horizon reuse the
// problem's trajectory workspace (L * traj_len >= K + 1 states).
#include <math.h>

#include "../../include/qoc_gpu.h"
#include "kernels.h"

namespace qoc {

namespace {

constexpr int ST_T = 256;
constexpr int ST_MAXD = 2048;
constexpr int ST_STAGE_MAXD = 1024;  // kinetic phase tables staged in shared memory up to this size

struct StrangCtx {
  int d, log2d;
  bool pow2;
  double inv_n;
  const double2* tw;     // smem [d/2] (pow2) -- exp(-2 pi i k / d)
  const double2* dftm;   // global [d][d] (direct DFT)
  double2 *A, *B, *S, *Q;  // smem work vectors [d]
  double* red;           // smem [ST_T / 32]
  double2* kx;           // smem [d] (cos k x_i, sin k x_i) of the lattice potential
  double* pf;            // smem [2][QOC_MAX_POT_TERMS]: f_m(u), f_m'(u) of the basis potential (per step)
  // kinetic phases staged in shared memory (they multiply the first stage's loads of half the
  // transforms): half step forward / adjoint and the merged full steps
  const double2 *kf, *ka, *kf2, *ka2;
};

// V(x_i, u) and dV/du for grid point i.  The cos^2 lattice uses cos/sin(k(x_i - u)) by angle
// addition from the per-point table and one sincos(k u) per step (cs = (cos k u, sin k u)).
struct PotStep {
  double2 cs;
};
__device__ __forceinline__ PotStep pot_step(const StrangCtx& X, const DevProblem& P, double u) {
  PotStep S{cx(1.0, 0.0)};
  if (P.potential == QOC_POT_LATTICE) {
    double sn, cn;
    sincos(P.pp[2] * u, &sn, &cn);
    S.cs = cx(cn, sn);
  } else if (P.potential == QOC_POT_BASIS) {
    // the terms' control factors once per step (block-uniform call sites)
    __syncthreads();
    const int m = threadIdx.x;
    if (m < P.pot_terms) {
      const double q = P.pot_param[m];
      double f, df;
      if (P.pot_type[m] == QOC_TERM_POWER) {
        const int k = (int)q;
        f = pow(u, (double)k);
        df = k > 0 ? k * pow(u, (double)(k - 1)) : 0.0;
      } else {
        double sn, cn;
        sincos(q * u, &sn, &cn);
        f = P.pot_type[m] == QOC_TERM_COS ? cn : sn;
        df = P.pot_type[m] == QOC_TERM_COS ? -q * sn : q * cn;
      }
      X.pf[m] = f;
      X.pf[QOC_MAX_POT_TERMS + m] = df;
    }
    __syncthreads();
  }
  return S;
}
__device__ __forceinline__ double basis_sum(const StrangCtx& X, const DevProblem& P, int i, int deriv) {
  double v = 0.0;
  for (int m = 0; m < P.pot_terms; ++m) v = fma(P.pot_basis[(size_t)m * X.d + i], X.pf[deriv * QOC_MAX_POT_TERMS + m], v);
  return v;
}

// dst = DFT_sign(pre . src) unnormalised (sign -1 forward, +1 inverse); pre may be null.
// src and dst are distinct shared-memory vectors.  Ends with a __syncthreads.
// Power-of-two sizes known at compile time: the same radix-4 Stockham stages with every stride,
// twiddle shift and trip count folded to constants and the stage loop unrolled.
// The out-of-line wrapper below serves the sizes other than 1024 (every size inlined at ~20 call
// sites costs minutes of compile time); the work
// vectors and the twiddle table are passed as offsets into the dynamic shared memory so that the
// stage loads and stores stay shared-memory instructions across the call.
template <int LOG2D, int SIGN, bool PRE>
__device__ __forceinline__ void transform_pow2_core(int src_off, int dst_off, int tw_off, const double2* pre, double scale) {
  extern __shared__ __align__(16) unsigned char fft_smem[];
  constexpr int d = 1 << LOG2D, NS4 = LOG2D / 2, NST = NS4 + (LOG2D & 1);
  const int t = threadIdx.x;
  double2* const base = reinterpret_cast<double2*>(fft_smem);
  const double2* const twv = base + tw_off;
  double2* const dst = base + dst_off;
  double2* in = base + src_off;
  double2* out = dst;
#pragma unroll
  for (int s = 0; s < NST; ++s) {
    const int lNs = 2 * s, Ns = 1 << lNs;
    const bool r4 = s < NS4;
    const int lR = r4 ? 2 : 1, R = 1 << lR;
    const int nb = d >> lR;
    const int tws = LOG2D - lNs - lR;
    for (int j = t; j < nb; j += ST_T) {
      const int jm = j & (Ns - 1);
      double2 v[4];
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        if (r < R) {
          double2 x = in[j + r * nb];
          if (PRE && s == 0) {  // PRE = false: plain transform (no pre-multiply, scale 1)
            if (pre) x = cmul(x, pre[j + r * nb]);
            if (scale != 1.0) x = cscale(x, scale);
          }
          if (r > 0 && s > 0) {  // twiddle exp(SIGN 2 pi i jm r / (Ns R)); jm = 0 gives 1
            const int k = (jm * r) << tws;
            double2 w = twv[k & (d / 2 - 1)];
            if (k >= d / 2) w = cx(-w.x, -w.y);
            if (SIGN > 0) w.y = -w.y;
            x = cmul(x, w);
          }
          v[r] = x;
        }
      }
      const int idxD = ((j >> lNs) << (lNs + lR)) + jm;
      if (r4) {
        const double2 a0 = cadd(v[0], v[2]), a1 = csub(v[0], v[2]), a2 = cadd(v[1], v[3]);
        const double2 dd = csub(v[1], v[3]);
        const double2 a3 = SIGN < 0 ? cx(dd.y, -dd.x) : cx(-dd.y, dd.x);
        out[idxD] = cadd(a0, a2);
        out[idxD + Ns] = cadd(a1, a3);
        out[idxD + 2 * Ns] = csub(a0, a2);
        out[idxD + 3 * Ns] = csub(a1, a3);
      } else {
        out[idxD] = cadd(v[0], v[1]);
        out[idxD + Ns] = csub(v[0], v[1]);
      }
    }
    __syncthreads();
    double2* tmp = in;
    in = out;
    out = tmp;
  }
  if (NST % 2 == 0) {  // even number of stages: the result sits in src
    for (int i = t; i < d; i += ST_T) dst[i] = in[i];
    __syncthreads();
  }
}

template <int LOG2D, int SIGN, bool PRE>
__device__ __noinline__ void transform_pow2(int src_off, int dst_off, int tw_off, const double2* pre, double scale) {
  transform_pow2_core<LOG2D, SIGN, PRE>(src_off, dst_off, tw_off, pre, scale);
}

__device__ __noinline__ void transform_other(const StrangCtx& X, const double2* src, double2* dst, int sign,
                                             const double2* pre, double scale) {
  const int d = X.d, t = threadIdx.x;
  if (X.pow2 && X.log2d >= 8 && X.log2d <= 11) {
    // every work vector and the twiddle table are carved from the dynamic shared memory whose
    // first vector is X.A (make_ctx)
    const int so = (int)(src - X.A), dof = (int)(dst - X.A), to = (int)(X.tw - X.A);
    const bool plain = pre == nullptr && scale == 1.0;
#define QOC_FFT_CASE(LG, SG)                                                   \
  if (plain) transform_pow2<LG, SG, false>(so, dof, to, pre, scale);           \
  else transform_pow2<LG, SG, true>(so, dof, to, pre, scale);                  \
  return;
    switch (X.log2d * 2 + (sign > 0)) {
      case 16: QOC_FFT_CASE(8, -1)
      case 17: QOC_FFT_CASE(8, +1)
      case 18: QOC_FFT_CASE(9, -1)
      case 19: QOC_FFT_CASE(9, +1)
      case 20: QOC_FFT_CASE(10, -1)
      case 21: QOC_FFT_CASE(10, +1)
      case 22: QOC_FFT_CASE(11, -1)
      default: QOC_FFT_CASE(11, +1)
    }
#undef QOC_FFT_CASE
  }
  if (X.pow2) {
    // Stockham autosort, radix 4 (plus one radix-2 stage when log2 d is odd): no bit-reversal
    // pass and half the barriers of radix 2.  Ping-pongs between dst and src (src is scratch
    // afterwards); the pre-multiply and scale are fused into the first stage's loads.
    double2* in = const_cast<double2*>(src);
    double2* out = dst;
    bool first = true;
    for (int Ns = 1, lNs = 0; Ns < d;) {
      const int R = (Ns * 4 <= d) ? 4 : 2, lR = R == 4 ? 2 : 1;
      const int nb = d >> lR;
      const int tws = X.log2d - lNs - lR;  // twiddle index = jm * r << tws  (d / (Ns R) = 2^tws)
      for (int j = t; j < nb; j += ST_T) {
        const int jm = j & (Ns - 1);  // j % Ns
        double2 v[4];
#pragma unroll
        for (int r = 0; r < 4; ++r) {
          if (r < R) {
            double2 x = in[j + r * nb];
            if (first) {
              if (pre) x = cmul(x, pre[j + r * nb]);
              if (scale != 1.0) x = cscale(x, scale);
            }
            if (r > 0 && jm != 0) {  // twiddle exp(sign 2 pi i jm r / (Ns R))
              const int k = (jm * r) << tws;
              double2 w;
              if (k < d / 2) {
                w = X.tw[k];
              } else {
                w = X.tw[k - d / 2];
                w = cx(-w.x, -w.y);
              }
              if (sign > 0) w.y = -w.y;
              x = cmul(x, w);
            }
            v[r] = x;
          }
        }
        const int idxD = ((j >> lNs) << (lNs + lR)) + jm;
        if (R == 4) {
          const double2 a0 = cadd(v[0], v[2]), a1 = csub(v[0], v[2]), a2 = cadd(v[1], v[3]);
          const double2 dd = csub(v[1], v[3]);
          const double2 a3 = sign < 0 ? cx(dd.y, -dd.x) : cx(-dd.y, dd.x);  // -+i (v1 - v3)
          out[idxD] = cadd(a0, a2);
          out[idxD + Ns] = cadd(a1, a3);
          out[idxD + 2 * Ns] = csub(a0, a2);
          out[idxD + 3 * Ns] = csub(a1, a3);
        } else {
          out[idxD] = cadd(v[0], v[1]);
          out[idxD + Ns] = csub(v[0], v[1]);
        }
      }
      __syncthreads();
      first = false;
      Ns <<= lR;
      lNs += lR;
      double2* tmp = in;
      in = out;
      out = tmp;
    }
    if (in != dst) {  // even number of stages: the result sits in src
      for (int i = t; i < d; i += ST_T) dst[i] = in[i];
      __syncthreads();
    }
    if (d == 1 && (pre || scale != 1.0)) {  // no stages ran
      for (int i = t; i < d; i += ST_T) {
        double2 x = src[i];
        if (pre) x = cmul(x, pre[i]);
        dst[i] = cscale(x, scale);
      }
      __syncthreads();
    }
  } else {
    for (int k = t; k < d; k += ST_T) {
      double2 acc = cx(0.0, 0.0);
      const double2* row = X.dftm + (size_t)k * d;
      for (int m = 0; m < d; ++m) {
        double2 v = src[m];
        if (pre) v = cmul(v, pre[m]);
        double2 w = row[m];
        if (sign > 0) w.y = -w.y;
        acc = cfma(v, w, acc);
      }
      dst[k] = scale != 1.0 ? cscale(acc, scale) : acc;
    }
    __syncthreads();
  }
}

// dst = DFT_sign(pre . src) unnormalised; 1024 points (BASELINE config 4) run the compile-time
// stages inlined at the call site, every other size goes through one out-of-line function.
__device__ __forceinline__ void transform(const StrangCtx& X, const double2* src, double2* dst, int sign,
                                          const double2* pre, double scale) {
  if (X.log2d == 10 && X.pow2) {
    const int so = (int)(src - X.A), dof = (int)(dst - X.A), to = (int)(X.tw - X.A);
    const bool plain = pre == nullptr && scale == 1.0;
    if (sign < 0) {
      if (plain) transform_pow2_core<10, -1, false>(so, dof, to, pre, scale);
      else transform_pow2_core<10, -1, true>(so, dof, to, pre, scale);
    } else {
      if (plain) transform_pow2_core<10, +1, false>(so, dof, to, pre, scale);
      else transform_pow2_core<10, +1, true>(so, dof, to, pre, scale);
    }
    return;
  }
  transform_other(X, src, dst, sign, pre, scale);
}

__device__ __forceinline__ double block_sum(const StrangCtx& X, double v) {
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  __syncthreads();
  if (lane == 0) X.red[warp] = v;
  __syncthreads();
  double s = 0.0;
  for (int w = 0; w < ST_T / 32; ++w) s += X.red[w];
  return s;
}

// V(x_i, u) and dV/du (models.cpp:95-127; cos^2 lattice of BASELINE config 4)
__device__ __forceinline__ double potential(const DevProblem& P, double x, double u) {
  if (P.potential == QOC_POT_TRAP) {
    const double ld = u * P.pp[0];
    const double ax = fabs(x);
    if (ax > 0.25 * ld) {
      const double r = ax - 0.5 * ld;
      return 0.5 * r * r;
    }
    return 0.5 * (0.125 * ld * ld - x * x);
  }
  const double cs = cos(P.pp[2] * (x - u));
  return 0.5 * P.pp[0] * x * x + P.pp[1] * cs * cs;
}
__device__ __forceinline__ double potential_du(const DevProblem& P, double x, double u) {
  if (P.potential == QOC_POT_TRAP) {
    const double dd = P.pp[0], ld = u * dd;
    const double ax = fabs(x);
    return (ax > 0.25 * ld) ? -0.5 * dd * (ax - 0.5 * ld) : 0.125 * u * dd * dd;
  }
  return P.pp[1] * P.pp[2] * sin(2.0 * P.pp[2] * (x - u));
}

__device__ __forceinline__ double potential_at(const StrangCtx& X, const DevProblem& P, int i, double u,
                                               const PotStep& S) {
  if (P.potential == QOC_POT_BASIS) return basis_sum(X, P, i, 0);
  const double x = P.grid_x[i];
  if (P.potential == QOC_POT_TRAP) return potential(P, x, u);
  const double2 k = X.kx[i];
  const double c = fma(k.x, S.cs.x, k.y * S.cs.y);  // cos(k(x - u))
  return 0.5 * P.pp[0] * x * x + P.pp[1] * c * c;
}
__device__ __forceinline__ double potential_du_at(const StrangCtx& X, const DevProblem& P, int i, double u,
                                                  const PotStep& S) {
  if (P.potential == QOC_POT_BASIS) return basis_sum(X, P, i, 1);
  if (P.potential == QOC_POT_TRAP) return potential_du(P, P.grid_x[i], u);
  const double2 k = X.kx[i];
  const double c = fma(k.x, S.cs.x, k.y * S.cs.y);   // cos(k(x - u))
  const double sn = fma(k.y, S.cs.x, -k.x * S.cs.y);  // sin(k(x - u))
  return 2.0 * P.pp[1] * P.pp[2] * sn * c;           // v0 k sin(2k(x - u))
}

// psi (in X.A) -> strang_step(psi); uses B, S.
__device__ void strang_forward(const StrangCtx& X, const DevProblem& P, double u, double dt) {
  transform(X, X.A, X.B, -1, nullptr, 1.0);
  transform(X, X.B, X.S, +1, X.kf, X.inv_n);  // psi_a
  const PotStep ps = pot_step(X, P, u);
  for (int i = threadIdx.x; i < X.d; i += ST_T) {
    const double2 pa = X.S[i];
    const double w = potential_at(X, P, i, u, ps) + P.kappa * cabs2(pa);
    double s, c;
    sincos(-dt * w, &s, &c);
    X.S[i] = cmul(cx(c, s), pa);  // psi_b
  }
  __syncthreads();
  transform(X, X.S, X.B, -1, nullptr, 1.0);
  transform(X, X.B, X.A, +1, X.kf, X.inv_n);
}

// chi_{j+1} (in X.A), psi_j (in X.Q) -> chi_j (in X.A); returns Im sum conj(chi_b) dV psi_b.
__device__ double strang_backward(const StrangCtx& X, const DevProblem& P, double u, double dt, bool naive,
                                  bool want_grad) {
  const int d = X.d;
  transform(X, X.Q, X.B, -1, nullptr, 1.0);
  transform(X, X.B, X.S, +1, X.kf, X.inv_n);  // psi_a in S
  transform(X, X.A, X.B, -1, nullptr, 1.0);
  transform(X, X.B, X.A, +1, X.ka, X.inv_n);  // chi_b in A
  double g = 0.0;
  const PotStep pst = pot_step(X, P, u);
  for (int i = threadIdx.x; i < d; i += ST_T) {
    const double2 pa = X.S[i], cb = X.A[i];
    const double dens = cabs2(pa);
    const double w = potential_at(X, P, i, u, pst) + P.kappa * dens;
    double s, c;
    sincos(-dt * w, &s, &c);
    const double2 flow = cx(c, s);
    const double2 pb = cmul(flow, pa);
    if (want_grad) g += potential_du_at(X, P, i, u, pst) * cconjmul(cb, pb).y;
    double2 ca;
    if (naive) {
      ca = cconjmul(flow, cb);
    } else {
      const double kd = dt * P.kappa;
      const double2 p = cmul(flow, cx(1.0, -kd * dens));           // flow (1 - i dt kappa dens)
      const double2 q = cmul(cx(0.0, -kd), cmul(flow, cmul(pa, pa)));  // -i dt kappa flow pa^2
      ca = cadd(cconjmul(p, cb), cmul(q, cconj(cb)));
    }
    X.B[i] = ca;
  }
  __syncthreads();
  transform(X, X.B, X.S, -1, nullptr, 1.0);
  transform(X, X.S, X.A, +1, X.ka, X.inv_n);
  return want_grad ? block_sum(X, g) : 0.0;
}

__device__ __forceinline__ StrangCtx make_ctx(const DevProblem& P, unsigned char* smem) {
  StrangCtx X;
  const int d = P.d;
  X.d = d;
  X.pow2 = (d & (d - 1)) == 0;
  X.log2d = X.pow2 ? __ffs(d) - 1 : 0;
  X.inv_n = 1.0 / (double)d;
  double2* base = reinterpret_cast<double2*>(smem);
  X.A = base;
  X.B = base + d;
  X.S = base + 2 * d;
  X.Q = base + 3 * d;
  double2* tw = base + 4 * d;
  X.dftm = P.twiddle;
  if (X.pow2) {
    for (int k = threadIdx.x; k < d / 2; k += ST_T) tw[k] = P.twiddle[k];
    X.tw = tw;
    X.red = reinterpret_cast<double*>(tw + (d / 2 > 0 ? d / 2 : 1));
  } else {
    X.tw = nullptr;
    X.red = reinterpret_cast<double*>(tw);
  }
  X.kx = reinterpret_cast<double2*>(X.red + ST_T / 32);
  X.pf = reinterpret_cast<double*>(X.kx + d);
  if (d > ST_STAGE_MAXD) {  // 2048 points: the tables stay in global memory (L2)
    X.kf = P.kin_fwd;
    X.ka = P.kin_adj;
    X.kf2 = P.kin_fwd2;
    X.ka2 = P.kin_adj2;
  } else {
    double2* ph = reinterpret_cast<double2*>(X.pf + 2 * QOC_MAX_POT_TERMS);
    for (int i = threadIdx.x; i < d; i += ST_T) {
      ph[i] = P.kin_fwd[i];
      ph[d + i] = P.kin_adj[i];
      ph[2 * d + i] = P.kin_fwd2[i];
      ph[3 * d + i] = P.kin_adj2[i];
    }
    X.kf = ph;
    X.ka = ph + d;
    X.kf2 = ph + 2 * d;
    X.ka2 = ph + 3 * d;
  }
  for (int i = threadIdx.x; i < d; i += ST_T) {
    double sn, cn;
    sincos(P.pp[2] * P.grid_x[i], &sn, &cn);
    X.kx[i] = cx(cn, sn);
  }
  __syncthreads();
  return X;
}

size_t strang_smem(int d) {
  const bool pow2 = (d & (d - 1)) == 0;
  return sizeof(double2) * (4 * (size_t)d + (pow2 ? (d / 2 > 0 ? d / 2 : 1) : 0)) + sizeof(double) * (ST_T / 32) +
         sizeof(double2) * (size_t)d + sizeof(double) * 2 * QOC_MAX_POT_TERMS + (d > ST_STAGE_MAXD ? 0 : sizeof(double2) * 4 * (size_t)d);
}

__device__ __forceinline__ void load_vec(double2* dst, const double2* src, int d) {
  for (int i = threadIdx.x; i < d; i += ST_T) dst[i] = src[i];
  __syncthreads();
}
__device__ __forceinline__ void store_vec(double2* dst, const double2* src, int d) {
  for (int i = threadIdx.x; i < d; i += ST_T) dst[i] = src[i];
}

// ---- sweeps with the kinetic half steps between grid steps merged -------------------------------
// Consecutive split steps meet in two kinetic half steps, K_h K_h = one spectral multiply by
// exp(-i dt k): a forward sweep then costs two transforms per grid step instead of four, and an
// adjoint sweep two instead of six, because the forward sweep keeps psi_a(j) = K_h psi_j (the
// state the potential/nonlinear phase acts on, which the backward stage of the reference
// recomputes from psi_j, propagation.cpp:146-170) instead of psi_j.  Same map as strang_step /
// strang_backward_stage applied step by step, up to the rounding of the skipped
// inverse-then-forward transform pair.
//
// psi (in X.A) -> psi_a(0) = K_h psi (in X.S)
__device__ void merged_begin_forward(const StrangCtx& X, const DevProblem& P) {
  transform(X, X.A, X.B, -1, nullptr, 1.0);
  transform(X, X.B, X.S, +1, X.kf, X.inv_n);
}
// psi_a(j) in X.S -> potential + nonlinear phase, then either psi_a(j+1) in X.S (last = false)
// or the step's end state psi_{j+1} in X.A (last = true).  node_out != null also writes
// psi_{j+1} there when last = false (node sweeps; uses Q).
__device__ void merged_forward_step(const StrangCtx& X, const DevProblem& P, double u, double dt, bool last,
                                    double2* node_out) {
  const PotStep ps = pot_step(X, P, u);
  for (int i = threadIdx.x; i < X.d; i += ST_T) {
    const double2 pa = X.S[i];
    const double w = potential_at(X, P, i, u, ps) + P.kappa * cabs2(pa);
    double s, c;
    sincos(-dt * w, &s, &c);
    X.S[i] = cmul(cx(c, s), pa);  // psi_b
  }
  __syncthreads();
  transform(X, X.S, X.B, -1, nullptr, 1.0);  // spectrum of psi_b
  if (last) {
    transform(X, X.B, X.A, +1, X.kf, X.inv_n);
    return;
  }
  if (node_out) {
    for (int i = threadIdx.x; i < X.d; i += ST_T) X.Q[i] = X.B[i];
    __syncthreads();
    transform(X, X.Q, X.A, +1, X.kf, X.inv_n);  // psi_{j+1}
    for (int i = threadIdx.x; i < X.d; i += ST_T) node_out[i] = X.A[i];
    __syncthreads();
  }
  transform(X, X.B, X.S, +1, X.kf2, X.inv_n);  // psi_a(j+1) = K_h K_h psi_b
}
// chi_len (in X.A) -> chi_b(len-1) = K_h^dag chi_len (in X.A)
__device__ void merged_begin_adjoint(const StrangCtx& X, const DevProblem& P) {
  transform(X, X.A, X.B, -1, nullptr, 1.0);
  transform(X, X.B, X.A, +1, X.ka, X.inv_n);
}
// chi_b(j) in X.A, psi_a(j) at pa_g (global) -> chi_b(j-1) in X.A (first = false) or chi_j in X.A
// (first = true, the sweep's last stage); returns Im sum conj(chi_b) dV psi_b.  node_out != null
// also writes chi_j there when first = false.
__device__ double merged_adjoint_step(const StrangCtx& X, const DevProblem& P, double u, double dt, bool naive,
                                      bool want_grad, const double2* pa_g, bool first, double2* node_out) {
  const int d = X.d;
  double g = 0.0;
  const PotStep pst = pot_step(X, P, u);
  for (int i = threadIdx.x; i < d; i += ST_T) {
    const double2 pa = pa_g[i], cb = X.A[i];
    const double dens = cabs2(pa);
    const double w = potential_at(X, P, i, u, pst) + P.kappa * dens;
    double s, c;
    sincos(-dt * w, &s, &c);
    const double2 flow = cx(c, s);
    const double2 pb = cmul(flow, pa);
    if (want_grad) g += potential_du_at(X, P, i, u, pst) * cconjmul(cb, pb).y;
    double2 ca;
    if (naive) {
      ca = cconjmul(flow, cb);
    } else {
      const double kd = dt * P.kappa;
      const double2 p = cmul(flow, cx(1.0, -kd * dens));
      const double2 q = cmul(cx(0.0, -kd), cmul(flow, cmul(pa, pa)));
      ca = cadd(cconjmul(p, cb), cmul(q, cconj(cb)));
    }
    X.B[i] = ca;
  }
  __syncthreads();
  transform(X, X.B, X.S, -1, nullptr, 1.0);  // spectrum of chi_a
  if (first) {
    transform(X, X.S, X.A, +1, X.ka, X.inv_n);
  } else {
    if (node_out) {
      for (int i = threadIdx.x; i < d; i += ST_T) X.Q[i] = X.S[i];
      __syncthreads();
      transform(X, X.Q, X.A, +1, X.ka, X.inv_n);  // chi_j
      for (int i = threadIdx.x; i < d; i += ST_T) node_out[i] = X.A[i];
      __syncthreads();
    }
    transform(X, X.S, X.A, +1, X.ka2, X.inv_n);  // chi_b(j-1) = K_h^dag K_h^dag chi_a
  }
  return want_grad ? block_sum(X, g) : 0.0;
}

__global__ void __launch_bounds__(ST_T, 1) strang_task_kernel(DevProblem P, DevRun R, TaskArgs A, int ignore_done) {
  const int n = blockIdx.x, b = blockIdx.y;
  if (ignore_done ? R.status[b] : (R.done[b] | R.status[b])) return;
  extern __shared__ __align__(16) unsigned char smem[];
  const StrangCtx X = make_ctx(P, smem);
  const int d = P.d, t = threadIdx.x;
  const int node0 = P.node[n], len = P.node[n + 1] - node0;
  const double Kd = (double)P.K;
  const double weight = A.weighted ? Kd / (double)len : 1.0;
  const double scale = (double)len / Kd;
  const double dt = P.dt, w = P.ip_w;
  const bool naive = (A.mode & (1 << 10)) != 0 || P.naive != 0;
  double* u = R.u + ((size_t)b * P.K + node0);  // C == 1
  int mode = A.mode;
  // phase-2 roles in separate CTAs (blockIdx.z): 0 = residual sweep, 1 = lagged refresh with
  // the second trajectory workspace
  size_t toff = 0;
  if (gridDim.z == 2) {
    if (blockIdx.z == 0) {
      mode &= ~M_LAGGED;
    } else {
      mode &= ~M_ERROR;
      toff = (size_t)P.B * P.L * R.traj_len * d;
    }
  }
  double2* traj = R.traj + toff + ((size_t)b * P.L + n) * (size_t)R.traj_len * d;
  const size_t tix = ((size_t)b * P.L + n) * d;

  auto forward = [&](bool rec, double* pen) {  // state in X.A
    if (P.merge_kinetic) {  // trajectory = psi_a(j), j = 0..len-1
      merged_begin_forward(X, P);
      for (int j = 0; j < len; ++j) {
        if (rec) store_vec(traj + (size_t)j * d, X.S, d);
        merged_forward_step(X, P, u[j], dt, j == len - 1, nullptr);
        if (pen) *pen += (P.alpha[node0 + j] * scale) * (u[j] * u[j]);
      }
      return;
    }
    if (rec) store_vec(traj, X.A, d);
    for (int j = 0; j < len; ++j) {
      strang_forward(X, P, u[j], dt);
      if (rec) store_vec(traj + (size_t)(j + 1) * d, X.A, d);
      if (pen) *pen += (P.alpha[node0 + j] * scale) * (u[j] * u[j]);
    }
  };
  // adjoint from the seed in X.A along the stored trajectory; act(j, uold, g)
  auto adjoint = [&](bool grad, auto&& act) {
    if (P.merge_kinetic) {
      __syncthreads();
      merged_begin_adjoint(X, P);
      for (int j = len - 1; j >= 0; --j) {
        const double uold = u[j];
        const double im = merged_adjoint_step(X, P, uold, dt, naive, grad, traj + (size_t)j * d, j == 0, nullptr);
        const double g = -(P.alpha[node0 + j] * scale) * dt * uold + dt * (w * im);
        act(j, uold, g);
      }
      return;
    }
    for (int j = len - 1; j >= 0; --j) {
      const double uold = u[j];
      __syncthreads();
      for (int i = t; i < d; i += ST_T) X.Q[i] = traj[(size_t)j * d + i];
      __syncthreads();
      const double im = strang_backward(X, P, uold, dt, naive, grad);
      const double g = -(P.alpha[node0 + j] * scale) * dt * uold + dt * (w * im);
      act(j, uold, g);
    }
  };
  auto seed = [&](int form) {  // adjoint_seed (objective.cpp:31-34), from the final state in A
    for (int i = t; i < d; i += ST_T) {
      const double2 tg = R.task_targ[tix + i];
      X.A[i] = form == 0 ? tg : csub(tg, X.A[i]);
    }
    __syncthreads();
  };

  if (mode & (M_ENTRY | M_UPDATE | M_FINAL | M_GRAD)) {
    const bool need_traj = (mode & (M_UPDATE | M_GRAD)) != 0;
    const int iters = (mode & M_UPDATE) ? A.inner : 1;
    for (int it = 0; it < iters; ++it) {
      load_vec(X.A, R.task_init + tix, d);
      double pen = 0.0;
      forward(need_traj, &pen);
      if (it == 0 && (mode & M_ENTRY)) {
        double s = 0.0;
        for (int i = t; i < d; i += ST_T) {
          const double2 tg = R.task_targ[tix + i];
          s += A.form == 0 ? cconjmul(tg, X.A[i]).x : cabs2(csub(X.A[i], tg));
        }
        s = block_sum(X, s);
        const double payoff = A.form == 0 ? (w * s) : (-0.5 * (w * s));
        if (t == 0) R.entry[(size_t)b * P.L + n] = weight * (payoff - 0.5 * dt * pen);
      }
      if (it == 0 && (mode & M_FINAL)) store_vec(R.psi_end + tix, X.A, d);
      if (mode & (M_UPDATE | M_GRAD)) {
        __syncthreads();
        seed(A.form);
        adjoint(true, [&](int j, double uold, double g) {
          if (t == 0) {
            if (mode & M_GRAD) R.grad[(size_t)b * P.K + node0 + j] = g;
            if (mode & M_UPDATE) u[j] = uold + A.rho * (weight * g);
          }
          __syncthreads();
        });
      }
    }
  }
  if (mode & M_ERROR) {
    __syncthreads();
    load_vec(X.A, R.task_init + tix, d);
    forward(true, nullptr);
    __syncthreads();
    seed(A.form);
    double err = 0.0;
    adjoint(true, [&](int, double, double g) { err += fabs(g); });
    if (t == 0) R.err[(size_t)b * P.L + n] = err;
  }
  if (mode & M_LAGGED) {  // ism.cpp:424-459 (strang branch): trajectory from psi_nodes[n]
    __syncthreads();
    load_vec(X.A, R.psi_nodes + ((size_t)b * (P.L + 1) + n) * d, d);
    forward(true, nullptr);
    __syncthreads();
    store_vec(R.psi_end + tix, X.A, d);
    __syncthreads();
    load_vec(X.A, R.chi_nodes + ((size_t)b * (P.L + 1) + n + 1) * d, d);
    adjoint(false, [&](int, double, double) {});
    __syncthreads();
    store_vec(R.chi_start + tix, X.A, d);
  }
}

// node_sweeps (ism.cpp:35-84; strang: forward trajectory kept for the nonlinear adjoint) and
// the exact payoff (which = 1).  One CTA per problem; the trajectory uses the problem's task
// workspace (L * traj_len >= K + 1 states).
__global__ void __launch_bounds__(ST_T, 1) strang_horizon_kernel(DevProblem P, DevRun R, int which, int k) {
  if (R.kdev) k = *R.kdev;
  const int b = blockIdx.x;
  if (R.done[b] || R.status[b]) return;
  extern __shared__ __align__(16) unsigned char smem[];
  const StrangCtx X = make_ctx(P, smem);
  const int d = P.d, t = threadIdx.x;
  const double dt = P.dt;
  const double* u = R.u + (size_t)b * P.K;
  double2* traj = R.traj + (size_t)b * P.L * R.traj_len * d;
  const size_t nb = (size_t)b * (P.L + 1) * d;
  load_vec(X.A, P.init + (size_t)b * d, d);
  if (which == 0) {
    store_vec(R.psi_nodes + nb, X.A, d);
    store_vec(traj, X.A, d);
  }
  int nxt = 1;
  if (P.merge_kinetic) {
    merged_begin_forward(X, P);
    for (int j = 0; j < P.K; ++j) {
      if (which == 0) store_vec(traj + (size_t)j * d, X.S, d);  // psi_a(j)
      const bool last = j == P.K - 1;
      const bool at_node = which == 0 && nxt <= P.L && P.node[nxt] == j + 1;
      merged_forward_step(X, P, u[j], dt, last,
                          (at_node && !last) ? R.psi_nodes + nb + (size_t)nxt * d : nullptr);
      if (at_node) {
        if (last) store_vec(R.psi_nodes + nb + (size_t)nxt * d, X.A, d);
        ++nxt;
      }
    }
  }
  for (int j = 0; j < (P.merge_kinetic ? 0 : P.K); ++j) {
    strang_forward(X, P, u[j], dt);
    if (which == 0) {
      store_vec(traj + (size_t)(j + 1) * d, X.A, d);
      if (nxt <= P.L && P.node[nxt] == j + 1) {
        store_vec(R.psi_nodes + nb + (size_t)nxt * d, X.A, d);
        ++nxt;
      }
    }
  }
  if (which == 1) {
    double s = 0.0;
    for (int i = t; i < d; i += ST_T) s += cconjmul(P.targ[(size_t)b * d + i], X.A[i]).x;
    s = block_sum(X, s);
    if (t == 0) {
      double pen = 0.0;
      for (int n = 0; n < P.L; ++n) pen += R.pen[(size_t)b * P.L + n];
      R.rec_exact[(size_t)b * R.cap + k] = P.ip_w * s - 0.5 * P.dt * pen;
    }
    return;
  }
  __syncthreads();
  load_vec(X.A, P.targ + (size_t)b * d, d);
  store_vec(R.chi_nodes + nb + (size_t)P.L * d, X.A, d);
  int prev = P.L - 1;
  if (P.merge_kinetic) {
    __syncthreads();
    merged_begin_adjoint(X, P);
    for (int j = P.K - 1; j >= 0; --j) {
      const bool first = j == 0;
      const bool at_node = prev >= 0 && P.node[prev] == j;
      merged_adjoint_step(X, P, u[j], dt, P.naive != 0, false, traj + (size_t)j * d, first,
                          (at_node && !first) ? R.chi_nodes + nb + (size_t)prev * d : nullptr);
      if (at_node) {
        if (first) store_vec(R.chi_nodes + nb + (size_t)prev * d, X.A, d);
        --prev;
      }
    }
    return;
  }
  for (int j = P.K - 1; j >= 0; --j) {
    __syncthreads();
    for (int i = t; i < d; i += ST_T) X.Q[i] = traj[(size_t)j * d + i];
    __syncthreads();
    strang_backward(X, P, u[j], dt, P.naive != 0, false);  // node_sweeps(.., naive), ism.cpp:373,543
    if (prev >= 0 && P.node[prev] == j) {
      store_vec(R.chi_nodes + nb + (size_t)prev * d, X.A, d);
      --prev;
    }
  }
}


// ---- stationary states by imaginary-time splitting (ground_state, models.cpp:146-182) ----------
// One CTA per state (blockIdx.x): psi <- normalise(K_h exp(-tau (V + kappa |psi_a|^2)) K_h psi),
// K_h = idft(exp(-tau/2 k) dft(.)), optionally Gram-Schmidt-orthogonalised against `nlower` fixed
// states first (excited states; BASELINE config 4's target), until the discrete energy
//   E = dx (sum k |hat|^2 + sum V |psi|^2 + kappa/2 sum |psi|^4)           (models.cpp:152-163)
// moves by less than `tol` between iterations, or max_iter iterations.  The spectrum of the new
// state from the energy evaluation is the first transform of the next iteration.
__global__ void __launch_bounds__(ST_T, 1) imag_time_kernel(DevProblem P, const double* u_frozen, double tau, double tol,
                                                            int max_iter, int nlower, const double2* lower,
                                                            const double* kin, const double2* half_kin, double2* psi_io,
                                                            double* energy_out, int* iter_out) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const StrangCtx X = make_ctx(P, smem_raw);
  const int d = X.d, s = blockIdx.x;
  const double u = u_frozen[s], dx = P.ip_w, kappa = P.kappa;
  double2* psi_g = psi_io + (size_t)s * d;
  const double2* low = lower + (size_t)s * nlower * d;
  load_vec(X.A, psi_g, d);
  const PotStep ps = pot_step(X, P, u);
  // V(x_i, u) is fixed: keep it in the Q vector's real parts
  for (int i = threadIdx.x; i < d; i += ST_T) X.Q[i] = cx(potential_at(X, P, i, u, ps), 0.0);
  __syncthreads();
  auto normalise = [&]() {  // psi (in A) <- orth(psi) / (sqrt(dx) ||psi||)
    for (int q = 0; q < nlower; ++q) {
      double re = 0.0, im = 0.0;
      for (int i = threadIdx.x; i < d; i += ST_T) {
        const double2 t = cconjmul(low[(size_t)q * d + i], X.A[i]);
        re += t.x;
        im += t.y;
      }
      const double2 ov = cx(dx * block_sum(X, re), dx * block_sum(X, im));
      for (int i = threadIdx.x; i < d; i += ST_T) X.A[i] = csub(X.A[i], cmul(ov, low[(size_t)q * d + i]));
      __syncthreads();
    }
    double nn = 0.0;
    for (int i = threadIdx.x; i < d; i += ST_T) nn += cabs2(X.A[i]);
    const double inv = 1.0 / (sqrt(dx) * sqrt(block_sum(X, nn)));
    for (int i = threadIdx.x; i < d; i += ST_T) X.A[i] = cscale(X.A[i], inv);
    __syncthreads();
  };
  // energy of psi (in A); leaves the unnormalised spectrum of psi in B and psi untouched in A
  auto energy = [&]() {
    double pe = 0.0, ie = 0.0;
    for (int i = threadIdx.x; i < d; i += ST_T) {
      const double den = cabs2(X.A[i]);
      pe += X.Q[i].x * den;
      ie += den * den;
      X.S[i] = X.A[i];
    }
    __syncthreads();
    transform(X, X.S, X.B, -1, nullptr, 1.0);
    double ke = 0.0;
    for (int i = threadIdx.x; i < d; i += ST_T) ke += kin[i] * cabs2(X.B[i]);
    ke = block_sum(X, ke) * X.inv_n;  // unitary dft: |hat|^2 / n
    pe = block_sum(X, pe);
    ie = block_sum(X, ie);
    return dx * (ke + pe + 0.5 * kappa * ie);
  };
  normalise();
  double e = energy();
  int k = 0;
  for (; k < max_iter; ++k) {
    transform(X, X.B, X.S, +1, half_kin, X.inv_n);  // psi_a = K_h psi (B holds dft(psi))
    for (int i = threadIdx.x; i < d; i += ST_T) {
      const double2 pa = X.S[i];
      X.S[i] = cscale(pa, exp(-tau * (X.Q[i].x + kappa * cabs2(pa))));
    }
    __syncthreads();
    transform(X, X.S, X.B, -1, nullptr, 1.0);
    transform(X, X.B, X.A, +1, half_kin, X.inv_n);
    normalise();
    const double next = energy();
    const bool done = fabs(next - e) < tol;
    e = next;
    if (done) {
      ++k;
      break;
    }
  }
  for (int i = threadIdx.x; i < d; i += ST_T) psi_g[i] = X.A[i];
  if (threadIdx.x == 0) {
    energy_out[s] = e;
    iter_out[s] = k;
  }
}

}  // namespace

cudaError_t strang_task(const DevProblem& P, const DevRun& R, const TaskArgs& A, int ignore_done, cudaStream_t st) {
  if (A.mode & M_ASSEMBLE) return cudaErrorNotSupported;
  if (P.C != 1 || P.d > ST_MAXD) return cudaErrorNotSupported;
  const size_t smem = strang_smem(P.d);
  cudaError_t e = cudaFuncSetAttribute(strang_task_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  // phase 1 (entry value, gradient sweep + update) then phase 2 (residual sweep and lagged
  // refresh at the updated control, independent of each other: concurrent CTAs)
  const int p1 = A.mode & (M_ENTRY | M_UPDATE | M_FINAL | M_GRAD), p2 = A.mode & (M_ERROR | M_LAGGED);
  if (p1) {
    TaskArgs A1 = A;
    A1.mode = A.mode & ~(M_ERROR | M_LAGGED);
    strang_task_kernel<<<dim3(P.L, P.B, 1), ST_T, smem, st>>>(P, R, A1, ignore_done);
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
  }
  if (p2) {
    TaskArgs A2 = A;
    A2.mode = p2 | (A.mode & (1 << 10));
    const int roles = (p2 & M_ERROR) && (p2 & M_LAGGED) ? 2 : 1;
    strang_task_kernel<<<dim3(P.L, P.B, roles), ST_T, smem, st>>>(P, R, A2, ignore_done);
  }
  return cudaGetLastError();
}

cudaError_t strang_horizon(const DevProblem& P, const DevRun& R, int which, int k, cudaStream_t st) {
  if (P.C != 1 || P.d > ST_MAXD) return cudaErrorNotSupported;
  const size_t smem = strang_smem(P.d);
  cudaError_t e = cudaFuncSetAttribute(strang_horizon_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  strang_horizon_kernel<<<P.B, ST_T, smem, st>>>(P, R, which, k);
  return cudaGetLastError();
}

cudaError_t strang_imaginary_time(const DevProblem& P, int states, const double* u_frozen, double tau, double tol,
                                  int max_iter, int nlower, const double2* lower, const double* kin,
                                  const double2* half_kin, double2* psi_io, double* energy_out, int* iter_out,
                                  cudaStream_t st) {
  if (P.d > ST_MAXD) return cudaErrorNotSupported;
  const size_t smem = strang_smem(P.d);
  cudaError_t e = cudaFuncSetAttribute(imag_time_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  imag_time_kernel<<<states, ST_T, smem, st>>>(P, u_frozen, tau, tol, max_iter, nlower, lower, kin, half_kin, psi_io,
                                               energy_out, iter_out);
  return cudaGetLastError();
}

}  // namespace qoc
