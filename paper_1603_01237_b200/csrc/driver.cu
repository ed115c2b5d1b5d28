// driver.cu — host driver of the B200 ISM path behind the C ABI of include/qoc_gpu.h.
//
// qoc_ism_run restates the control flow of run_ism (ism.cpp:211-612) as a sequence of
// device kernels on one stream: bootstrap, then per outer iteration
//   task kernel (entry value + gradient update + residual + assembly / lagged refresh)
//   -> penalty partials -> index-order merge -> boundary refresh (chain / lagged / direct)
//   -> boundary objective + waypoint rebuild -> [exact payoff] -> record + eta stop,
// then the trailing task-value evaluation.  Per-problem stop and abort state lives on the
// device, so a batch of independent problems runs in one launch sequence with no host
// round trip per iteration.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>  // types only: the library is resolved at run time (dlopen), see nccl_api()

#include <algorithm>
#include <chrono>
#include <exception>
#include <mutex>
#include <thread>
#include <cstdlib>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <stdexcept>
#include <string>
#include <tuple>
#include <vector>

#include "../../include/qoc_gpu.h"
#include "kernels.h"

static_assert(qoc::MAXC == QOC_MAX_CHANNELS, "device channel arrays must match the ABI bound");

using namespace qoc;

struct qoc_ctx {
  // InnerResult counters of the last qoc_ism_run: [iterations + 1][B][L][3]
  std::vector<int> solver_stats;
  int solver_stats_dims[3] = {0, 0, 0};
  int device = 0;
  cudaStream_t stream = nullptr;
  cudaStream_t aux = nullptr;          // side stream: boundary chain overlapped with the residual
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  std::string last_error;
  int64_t launches = 0;
  bool profile = false;
  int64_t flush_bytes = 0;
  void* flush_buf = nullptr;
  qoc_profile_v1 prof{};
  // event pairs of the current run: (start, stop, is_task, label)
  std::vector<std::tuple<cudaEvent_t, cudaEvent_t, bool, const char*>> marks;
  // per-label device time of profiled launches: label -> (ms, launches), first-seen order
  std::vector<std::pair<std::string, std::pair<double, int64_t>>> by_label;
  int* khost = nullptr;        // pinned iteration indices for graph replays
  void* stage = nullptr;       // pinned staging buffer for large device -> host results
  size_t stage_bytes = 0;
  cudaGraphExec_t gcache = nullptr;  // last instantiated iteration graph and its parameter key
  std::vector<unsigned char> gkey;
  int64_t gcache_launches = 0;
  size_t khost_n = 0;
  void* prob_slots = nullptr;  // Slots* (driver.cu anonymous namespace)
  void* run_slots = nullptr;
  // multi-GPU (qoc_ctx_init_comm): rank of world; the NCCL communicator when world > 1
  int rank = 0, world = 1;
  ncclComm_t comm = nullptr;
};

namespace {

struct Fail {
  int32_t code;
  std::string msg;
};

[[noreturn]] void fail(int32_t code, const std::string& msg) { throw Fail{code, msg}; }

void ck(cudaError_t e, const char* what) {
  if (e != cudaSuccess) fail(QOC_ECUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

// RAII device allocation
struct DBuf {
  void* p = nullptr;
  size_t bytes = 0;
  DBuf() = default;
  explicit DBuf(size_t n) : bytes(n) {
    if (n) ck(cudaMalloc(&p, n), "cudaMalloc");
  }
  DBuf(const DBuf&) = delete;
  DBuf& operator=(const DBuf&) = delete;
  DBuf(DBuf&& o) noexcept : p(o.p), bytes(o.bytes) { o.p = nullptr; }
  DBuf& operator=(DBuf&& o) noexcept {
    std::swap(p, o.p);
    std::swap(bytes, o.bytes);
    return *this;
  }
  ~DBuf() {
    if (p) cudaFree(p);
  }
  template <class T>
  T* as() const {
    return static_cast<T*>(p);
  }
};

// Grow-only device buffers owned by a context: the i-th request of a call reuses slot i when
// it is large enough, so repeated solves on one context make no cudaMalloc/cudaFree calls.
struct Slots {
  std::vector<DBuf> bufs;
  size_t next = 0;
  void reset() { next = 0; }
  void* get(size_t bytes) {
    bytes = std::max<size_t>(bytes, 1);
    if (next < bufs.size()) {
      if (bufs[next].bytes < bytes) bufs[next] = DBuf(bytes);
    } else {
      bufs.emplace_back(bytes);
    }
    return bufs[next++].p;
  }
};

template <class T>
DBuf upload(const T* host, size_t n, cudaStream_t st) {
  DBuf b(sizeof(T) * n);
  if (n) ck(cudaMemcpyAsync(b.p, host, sizeof(T) * n, cudaMemcpyHostToDevice, st), "upload");
  return b;
}

template <class T>
DBuf filled(size_t n, T value, cudaStream_t st) {
  std::vector<T> h(n, value);
  DBuf b = upload(h.data(), n, st);
  ck(cudaStreamSynchronize(st), "sync");
  return b;
}

std::vector<int> decomposition(int K, int L, int mode, const int32_t* explicit_nodes) {
  // Decomposition::uniform / from_times (controls.cpp:110-140), generalised
  if (L < 1) fail(QOC_ERUNTIME, "Decomposition: parts must be positive");
  std::vector<int> node;
  if (mode == QOC_PARTITION_EXPLICIT) {
    if (!explicit_nodes) fail(QOC_EINVAL, "explicit partition needs node_index");
    for (int n = 0; n <= L; ++n) node.push_back(explicit_nodes[n]);
    if (node.front() != 0 || node.back() != K)
      fail(QOC_ERUNTIME, "Decomposition: boundaries must span the full grid");
    for (int n = 0; n < L; ++n)
      if (node[n + 1] <= node[n]) fail(QOC_ERUNTIME, "Decomposition: boundary times must strictly increase");
    return node;
  }
  if (mode == QOC_PARTITION_UNIFORM && K % L != 0)
    fail(QOC_ERUNTIME, "Decomposition: step count " + std::to_string(K) + " is not divisible into " +
                           std::to_string(L) + " equal parts");
  if (L > K) fail(QOC_ERUNTIME, "Decomposition: more parts than steps");
  const int base = K / L, extra = K % L;
  node.push_back(0);
  for (int n = 0; n < L; ++n) node.push_back(node.back() + base + (n < extra ? 1 : 0));
  return node;
}

// Device copy of a problem (operators converted to the kernels' layouts).
struct DeviceProblem {
  DevProblem P{};
  Slots* slots = nullptr;
  cudaStream_t st = nullptr;
  int stride = 0;  // state stride of the kind's trajectory workspace

  // device copy of n host elements, returned as the kernels' element type T
  template <class T, class H>
  const T* put(const H* host, size_t n) {
    void* d = slots->get(sizeof(H) * n);
    if (n) ck(cudaMemcpyAsync(d, host, sizeof(H) * n, cudaMemcpyHostToDevice, st), "upload");
    return static_cast<const T*>(d);
  }
};

void validate_problem(const qoc_problem_v1* p) {
  if (!p) fail(QOC_EINVAL, "problem has no model");
  if (p->abi_version != QOC_ABI_VERSION) fail(QOC_EINVAL, "problem ABI version mismatch");
  if (p->dim < 1 || p->channels < 1 || p->steps < 1 || p->batch < 1)
    fail(QOC_EINVAL, "dim, channels, steps and batch must be positive");
  if (!(p->dt > 0.0)) fail(QOC_EINVAL, "TimeGrid: dt must be positive");
  const int cmax = p->kind == QOC_KIND_DENSITY ? QOC_MAX_DENSITY_CHANNELS
                                                 : (p->kind == QOC_KIND_BITFLIP ? 4 : QOC_MAX_CHANNELS);
  if (p->channels > cmax)
    fail(QOC_ELOGIC, "control channel count above what the device kernels carry (QOC_MAX_CHANNELS; 4 for the "
                     "bit-flip kind, QOC_MAX_DENSITY_CHANNELS for the density kind)");
  if (!p->initial || !p->target) fail(QOC_EINVAL, "initial and target states are required");
}

// Host-side per-problem packing of large batches on the host threads (the batch's operator
// conversion is the bulk of the e2e upload); the first exception is rethrown on the caller.
template <class F>
void parallel_for(int n, F&& f) {
  const int hw = static_cast<int>(std::thread::hardware_concurrency());
  const int nt = std::max(1, std::min({hw, 16, n / 64}));
  if (nt <= 1) {
    for (int i = 0; i < n; ++i) f(i);
    return;
  }
  std::exception_ptr err;
  std::mutex mu;
  std::vector<std::thread> pool;
  for (int t = 0; t < nt; ++t)
    pool.emplace_back([&, t] {
      try {
        for (int i = t; i < n; i += nt) f(i);
      } catch (...) {
        std::lock_guard<std::mutex> g(mu);
        if (!err) err = std::current_exception();
      }
    });
  for (auto& th : pool) th.join();
  if (err) std::rethrow_exception(err);
}

// Device -> pageable host copy of a large result through the context's pinned staging buffer:
// the DMA runs at full rate into pinned memory in 32 MiB pieces while the host threads move the
// previous piece to the caller's buffer (a plain cudaMemcpy to pageable memory measured 4 GB/s
// on the config-5 results: 36 ms for 150 MB).
void download_large(qoc_ctx* ctx, void* dst, const void* src, size_t bytes, const char* what) {
  constexpr size_t PIECE = (size_t)32 << 20;
  if (bytes < ((size_t)8 << 20)) {
    ck(cudaMemcpy(dst, src, bytes, cudaMemcpyDeviceToHost), what);
    return;
  }
  if (ctx->stage_bytes < 2 * PIECE) {
    if (ctx->stage) cudaFreeHost(ctx->stage);
    ctx->stage = nullptr;
    ctx->stage_bytes = 0;
    if (cudaHostAlloc(&ctx->stage, 2 * PIECE, cudaHostAllocDefault) != cudaSuccess) {
      cudaGetLastError();
      ck(cudaMemcpy(dst, src, bytes, cudaMemcpyDeviceToHost), what);
      return;
    }
    ctx->stage_bytes = 2 * PIECE;
  }
  cudaStream_t st = ctx->stream;
  char* out = static_cast<char*>(dst);
  const char* in = static_cast<const char*>(src);
  char* buf[2] = {static_cast<char*>(ctx->stage), static_cast<char*>(ctx->stage) + PIECE};
  const size_t n = (bytes + PIECE - 1) / PIECE;
  auto len = [&](size_t i) { return std::min(PIECE, bytes - i * PIECE); };
  ck(cudaMemcpyAsync(buf[0], in, len(0), cudaMemcpyDeviceToHost, st), what);
  for (size_t i = 0; i < n; ++i) {
    ck(cudaStreamSynchronize(st), what);
    if (i + 1 < n) ck(cudaMemcpyAsync(buf[(i + 1) & 1], in + (i + 1) * PIECE, len(i + 1), cudaMemcpyDeviceToHost, st), what);
    const size_t L = len(i);
    const char* from = buf[i & 1];
    char* to = out + i * PIECE;
    std::vector<std::thread> pool;
    const int hw = std::max(1, std::min(8, (int)std::thread::hardware_concurrency()));
    const size_t chunk = (L + hw - 1) / hw;
    for (int t = 0; t < hw; ++t) {
      const size_t a = std::min(L, (size_t)t * chunk), z = std::min(L, a + chunk);
      if (z > a) pool.emplace_back([=] { std::memcpy(to + a, from + a, z - a); });
    }
    for (auto& th : pool) th.join();
  }
}

void hermitian_check(const double* m, int d, const char* what) {  // models.cpp:20-25
  double scale2 = 1.0, defect2 = 0.0;  // squared moduli: no hypot in the per-element loop
  for (int j = 0; j < d; ++j)
    for (int i = 0; i <= j; ++i) {
      const double ar = m[2 * (i + (size_t)j * d)], ai = m[2 * (i + (size_t)j * d) + 1];
      const double br = m[2 * (j + (size_t)i * d)], bi = m[2 * (j + (size_t)i * d) + 1];
      scale2 = std::max(scale2, std::max(ar * ar + ai * ai, br * br + bi * bi));
      defect2 = std::max(defect2, (ar - br) * (ar - br) + (ai + bi) * (ai + bi));
    }
  if (!(defect2 <= 1e-20 * scale2)) fail(QOC_EINVAL, std::string(what) + " must be Hermitian");
}

bool disabled_path(const char* what);

void upload_problem(const qoc_problem_v1* p, const std::vector<int>& node, cudaStream_t st, DeviceProblem& out) {
  out.st = st;
  validate_problem(p);
  DevProblem& P = out.P;
  const int d = p->dim, C = p->channels, B = p->batch, K = p->steps;
  P.kind = p->kind;
  P.d = d;
  P.C = C;
  P.K = K;
  P.B = B;
  P.L = static_cast<int>(node.size()) - 1;
  P.dt = p->dt;
  P.ip_w = p->ip_weight;
  P.dm = d;
  out.stride = d;
  switch (p->kind) {
    case QOC_KIND_DENSITY:
    case QOC_KIND_DENSE: {
      if (!p->h0 || !p->linear) fail(QOC_EINVAL, "dense model needs h0 and linear operators");
      if (p->kind == QOC_KIND_DENSITY) {
        if (!density_supported(d)) fail(QOC_ELOGIC, "density-matrix device kernels support d <= 32");
        P.d = d * d;  // the state is the d x d matrix (column-major)
        out.stride = d * d;
      } else {
        if (dense_pad(d) < 0 && !dense_big_supported(d))
          fail(QOC_ELOGIC, "dense device kernels support d <= 64; use a structured kind");
        out.stride = dense_pad(d) > 0 ? dense_pad(d) : d;
      }
      const size_t dd = (size_t)d * d;
      P.has_quad = p->quadratic != nullptr;
      const int nq = P.has_quad ? C : 0;
      std::vector<double> h0((size_t)2 * B * dd), lin((size_t)2 * B * C * dd), quad((size_t)2 * B * nq * dd);
      std::vector<double> norms((size_t)B * (1 + 2 * C), 0.0);
      auto convert = [&](const double* src, double* dst, double* norm, const char* what) {
        hermitian_check(src, d, what);
        double best = 0.0;
        for (int j = 0; j < d; ++j) {
          double colsum = 0.0;
          for (int i = 0; i < d; ++i) {
            const double re = src[2 * (i + (size_t)j * d)], im = src[2 * (i + (size_t)j * d) + 1];
            dst[2 * ((size_t)i * d + j)] = re;  // column-major -> row-major
            dst[2 * ((size_t)i * d + j) + 1] = im;
            colsum += std::sqrt(re * re + im * im);
          }
          best = std::max(best, colsum);
        }
        *norm = best * (1.0 + 1e-12);
      };
      parallel_for(B, [&](int b) {
        double* nb = norms.data() + (size_t)b * (1 + 2 * C);
        convert(p->h0 + 2 * dd * b, h0.data() + 2 * dd * b, nb, "free Hamiltonian");
        for (int c = 0; c < C; ++c)
          convert(p->linear + 2 * dd * ((size_t)b * C + c), lin.data() + 2 * dd * ((size_t)b * C + c), nb + 1 + c,
                  "control operator");
        for (int c = 0; c < nq; ++c)
          convert(p->quadratic + 2 * dd * ((size_t)b * C + c), quad.data() + 2 * dd * ((size_t)b * C + c),
                  nb + 1 + C + c, "quadratic operator");
      });
      P.h0 = out.put<double2>(h0.data(), h0.size());
      P.lin = out.put<double2>(lin.data(), lin.size());
      P.quad = nq ? out.put<double2>(quad.data(), quad.size()) : nullptr;
      P.norm1 = out.put<double>(norms.data(), norms.size());
      break;
    }
    case QOC_KIND_TRIDIAG: {
      if (!p->tri_diag || !p->tri_sub) fail(QOC_EINVAL, "tridiagonal model needs bands");
      if (d > 32) fail(QOC_ELOGIC, "tridiagonal device kernels support d <= 32");
      P.has_quad = p->tri_has_quadratic != 0;
      const int nops = 1 + C + (P.has_quad ? C : 0);
      P.tri_diag = out.put<double>(p->tri_diag, (size_t)B * nops * d);
      P.tri_sub = out.put<double2>(reinterpret_cast<const double2*>(p->tri_sub), (size_t)B * nops * (d - 1));
      break;
    }
    case QOC_KIND_BITFLIP: {
      if (!p->h0 || !p->bf_axis || !p->bf_coef) fail(QOC_EINVAL, "bit-flip model needs h0/axis/coef");
      if (p->nspins < 5 || p->nspins > 12 || (1 << p->nspins) != d)
        fail(QOC_EINVAL, "bit-flip dim must be 2^nspins (5 <= nspins <= 12)");
      P.nspins = p->nspins;
      P.bf_diag = out.put<double>(p->h0, (size_t)B * d);
      P.bf_axis = out.put<int>(p->bf_axis, (size_t)C);
      P.bf_coef = out.put<double>(p->bf_coef, (size_t)B * C * p->nspins);
      break;
    }
    case QOC_KIND_STRANG: {
      if (!p->kinetic || !p->grid_x) fail(QOC_EINVAL, "condensate model needs kinetic/grid");
      if (C != 1) fail(QOC_EINVAL, "single control channel expected");
      if (d > 2048) fail(QOC_ELOGIC, "split-step device kernels support d <= 2048");
      const bool pow2 = (d & (d - 1)) == 0;
      if (!pow2 && d > 256) fail(QOC_ELOGIC, "split-step device kernels need a power-of-two grid above 256 points");
      // kinetic_half_phase (propagation.cpp:33-40): polar(1, sign * 0.5 * dt * k)
      std::vector<double> kf(2 * (size_t)d), ka(2 * (size_t)d);
      for (int i = 0; i < d; ++i) {
        const double af = -1.0 * 0.5 * p->dt * p->kinetic[i];
        const double aa = 1.0 * 0.5 * p->dt * p->kinetic[i];
        kf[2 * i] = std::cos(af);
        kf[2 * i + 1] = std::sin(af);
        ka[2 * i] = std::cos(aa);
        ka[2 * i + 1] = std::sin(aa);
      }
      P.kin_fwd = out.put<double2>(reinterpret_cast<const double2*>(kf.data()), (size_t)d);
      P.kin_adj = out.put<double2>(reinterpret_cast<const double2*>(ka.data()), (size_t)d);
      // two consecutive half steps as one spectral multiply: the product of the two half phases
      // (the same two roundings the separate multiplies apply)
      std::vector<double> kf2(2 * (size_t)d), ka2(2 * (size_t)d);
      for (int i = 0; i < d; ++i) {
        kf2[2 * i] = kf[2 * i] * kf[2 * i] - kf[2 * i + 1] * kf[2 * i + 1];
        kf2[2 * i + 1] = 2.0 * kf[2 * i] * kf[2 * i + 1];
        ka2[2 * i] = ka[2 * i] * ka[2 * i] - ka[2 * i + 1] * ka[2 * i + 1];
        ka2[2 * i + 1] = 2.0 * ka[2 * i] * ka[2 * i + 1];
      }
      P.kin_fwd2 = out.put<double2>(reinterpret_cast<const double2*>(kf2.data()), (size_t)d);
      P.kin_adj2 = out.put<double2>(reinterpret_cast<const double2*>(ka2.data()), (size_t)d);
      P.merge_kinetic = disabled_path("strangmerge") ? 0 : 1;
      // twiddles of linalg.cpp:26-27 (polar(1, ang * k), ang = -2 pi / n; the inverse
      // transform conjugates) or the direct DFT kernel of linalg.cpp:37-50
      std::vector<double> tw;
      if (pow2) {
        tw.resize(2 * (size_t)(d / 2 > 0 ? d / 2 : 1));
        const double ang = -1.0 * 2.0 * M_PI / static_cast<double>(d);
        for (int k = 0; k < d / 2; ++k) {
          tw[2 * k] = std::cos(ang * k);
          tw[2 * k + 1] = std::sin(ang * k);
        }
      } else {
        tw.resize(2 * (size_t)d * d);
        for (int k = 0; k < d; ++k)
          for (int m = 0; m < d; ++m) {
            const long long r = (static_cast<long long>(m) * k) % d;
            const double a = -1.0 * 2.0 * M_PI * static_cast<double>(r) / static_cast<double>(d);
            tw[2 * ((size_t)k * d + m)] = std::cos(a);
            tw[2 * ((size_t)k * d + m) + 1] = std::sin(a);
          }
      }
      P.twiddle = out.put<double2>(reinterpret_cast<const double2*>(tw.data()), tw.size() / 2);
      P.grid_x = out.put<double>(p->grid_x, (size_t)d);
      P.potential = p->potential;
      for (int i = 0; i < 4; ++i) P.pp[i] = p->pot_params[i];
      P.kappa = p->kappa;
      if (p->potential < QOC_POT_TRAP || p->potential > QOC_POT_BASIS) fail(QOC_EINVAL, "unknown potential kind");
      if (p->potential == QOC_POT_BASIS) {  // caller-supplied potential()/potential_derivative(), separable form
        if (p->pot_terms < 1 || p->pot_terms > QOC_MAX_POT_TERMS || !p->pot_term_type || !p->pot_term_param ||
            !p->pot_basis)
          fail(QOC_EINVAL, "basis potential needs 1..QOC_MAX_POT_TERMS terms with type, parameter and profile arrays");
        P.pot_terms = p->pot_terms;
        for (int m = 0; m < p->pot_terms; ++m) {
          const int ty = p->pot_term_type[m];
          const double q = p->pot_term_param[m];
          if (ty < QOC_TERM_POWER || ty > QOC_TERM_SIN) fail(QOC_EINVAL, "unknown potential term type");
          if (ty == QOC_TERM_POWER && (q < 0.0 || q != std::floor(q)))
            fail(QOC_EINVAL, "power terms take a non-negative integer exponent");
          P.pot_type[m] = ty;
          P.pot_param[m] = q;
        }
        P.pot_basis = out.put<double>(p->pot_basis, (size_t)p->pot_terms * d);
      }
      break;
    }
    default:
      fail(QOC_EINVAL, "unknown model kind");
  }
  P.init = out.put<double2>(reinterpret_cast<const double2*>(p->initial), (size_t)B * P.d);  // state length
  P.targ = out.put<double2>(reinterpret_cast<const double2*>(p->target), (size_t)B * P.d);
  std::vector<double> alpha(K, 0.0);
  if (p->penalty) alpha.assign(p->penalty, p->penalty + K);
  P.alpha = out.put<double>(alpha.data(), alpha.size());
  P.node = out.put<int>(node.data(), node.size());
}

Slots* fresh_slots(void*& handle) {
  if (!handle) handle = new Slots;
  Slots* sl = static_cast<Slots*>(handle);
  sl->reset();
  return sl;
}

struct DeviceRun {
  DevRun R{};
  Slots* slots = nullptr;
  template <class T>
  T* alloc(size_t n) {
    return static_cast<T*>(slots->get(sizeof(T) * std::max<size_t>(n, 1)));
  }
};

// Bytes of the propagator cache (pcache.cu) for a run, or 0 when the engine does not apply.
size_t pc_bytes(const DevProblem& P, const std::vector<int>& node) {
  if (!(P.kind == QOC_KIND_DENSE || (P.kind == QOC_KIND_TRIDIAG && P.d <= 30)) || P.d > 32) return 0;
  int maxlen = 0;
  for (size_t n = 0; n + 1 < node.size(); ++n) maxlen = std::max(maxlen, node[n + 1] - node[n]);
  return sizeof(double2) * (size_t)P.B * P.L * (maxlen + 1) * P.d * P.d;
}

bool use_pcache(const DevProblem& P, const std::vector<int>& node) {
  const size_t need = pc_bytes(P, node);
  if (!need) return false;
  size_t freeb = 0, total = 0;
  if (cudaMemGetInfo(&freeb, &total) != cudaSuccess) return false;
  return need < freeb / 10 * 7;
}

void alloc_run(const DeviceProblem& dp, int cap, const std::vector<int>& node, bool need_prop, bool need_grad,
               cudaStream_t st, DeviceRun& out, bool with_pc = false, bool split = false) {
  const DevProblem& P = dp.P;
  DevRun& R = out.R;
  const size_t B = P.B, L = P.L, d = P.d, K = P.K, C = P.C;
  int maxlen = 0;
  for (size_t n = 0; n < L; ++n) maxlen = std::max(maxlen, node[n + 1] - node[n]);
  R.cap = cap;
  R.traj_len = maxlen + 1;
  R.u = out.alloc<double>(B * K * C);
  R.grad = need_grad ? out.alloc<double>(B * K * C) : nullptr;
  R.task_init = out.alloc<double2>(B * L * d);
  R.task_targ = out.alloc<double2>(B * L * d);
  R.psi_nodes = out.alloc<double2>(B * (L + 1) * d);
  R.chi_nodes = out.alloc<double2>(B * (L + 1) * d);
  // task propagators: d x d, or dm x dm for the density kind (its states are dm x dm matrices)
  const size_t pe = P.kind == QOC_KIND_DENSITY ? (size_t)P.dm * P.dm : d * d;
  R.prop = need_prop ? out.alloc<double2>(B * L * pe) : nullptr;
  R.psi_end = out.alloc<double2>(B * L * d);
  R.chi_start = out.alloc<double2>(B * L * d);
  // the split-step kind runs its residual and lagged sweeps as concurrent CTAs, each with its
  // own trajectory: two workspaces
  R.traj = out.alloc<double2>(B * L * (size_t)R.traj_len * dp.stride * (P.kind == QOC_KIND_STRANG ? 2 : 1));
  R.winv = nullptr;
  if (P.kind == QOC_KIND_DENSITY && R.traj_len > 1) {
    const size_t need = sizeof(double2) * B * L * (size_t)(R.traj_len - 1) * P.dm * P.dm;
    size_t freeb = 0, total = 0;
    if (cudaMemGetInfo(&freeb, &total) == cudaSuccess && need < freeb / 2) R.winv = out.alloc<double2>(need / sizeof(double2));
  }
  R.entry = out.alloc<double>(B * L);
  R.err = out.alloc<double>(B * L);
  R.pen = out.alloc<double>(B * L);
  R.bad_u = out.alloc<int>(B * L);
  R.done = out.alloc<int>(B);
  R.status = out.alloc<int>(B);
  R.abort_iter = out.alloc<int>(B);
  R.n_recs = out.alloc<int>(B);
  R.tot_err = out.alloc<double>(B);
  R.rec_obj = out.alloc<double>(B * cap);
  R.rec_err = out.alloc<double>(B * cap);
  R.rec_exact = out.alloc<double>(B * cap);
  R.rec_tv = out.alloc<double>(B * cap * L);
  R.rec_flags = out.alloc<int>(B * cap);
  R.err_flags = out.alloc<int>(1);
  if (with_pc) {
    R.pc = out.alloc<double2>(pc_bytes(P, node) / sizeof(double2));
    R.cay = nullptr;
    // Few dense tasks (one lane group each would leave the GPU idle through a long dependent
    // sweep): form every step's Cayley matrix in parallel first, then run the per-task matmul
    // chain.  Many tasks (the batch) keep the fused sweep, which measured faster there.
    const bool nm = dense_nm_applicable(P) && !split && R.traj_len - 1 <= 32;  // one chunk per task
    if (P.kind == QOC_KIND_DENSE && P.d <= 16 && B * L <= 1024 && !nm) {
      const size_t cb = sizeof(double2) * B * K * d * d;
      size_t freeb = 0, total = 0;
      if (cudaMemGetInfo(&freeb, &total) == cudaSuccess && cb < freeb / 10 * 6)
        R.cay = out.alloc<double2>(cb / sizeof(double2));
    }
    // the Neumann path keeps a column-major cache that only the interpolated-variant
    // evaluations read (dense_nm.cu); split runs keep the Gauss-Jordan sweep
    if (nm) {
      R.nm = out.alloc<double2>(B * NM_TERMS * 256);
      R.nm_fallback = out.alloc<int>(B * L);
      R.nm_v = out.alloc<double2>(B * L * (R.traj_len - 1) * d);
      R.nm_count = out.alloc<int>(1);
      R.gpend = out.alloc<double>(B * K);
      R.old_init = out.alloc<double2>(B * L * d);
      R.old_targ = out.alloc<double2>(B * L * d);
      ck(cudaMemsetAsync(R.nm_fallback, 0, sizeof(int) * B * L, st), "memset");
    }
    const int nchunk = pc_nchunk(P, R);
    R.chunk_pen = out.alloc<double>(B * L * nchunk);
    R.chunk_err = out.alloc<double>(B * L * nchunk);
    R.entry_pay = out.alloc<double>(B * L);
  }
  ck(cudaMemsetAsync(R.err_flags, 0, sizeof(int), st), "memset");
  ck(cudaMemsetAsync(R.done, 0, sizeof(int) * B, st), "memset");
  ck(cudaMemsetAsync(R.status, 0, sizeof(int) * B, st), "memset");
  ck(cudaMemsetAsync(R.abort_iter, 0, sizeof(int) * B, st), "memset");
  ck(cudaMemsetAsync(R.err, 0, sizeof(double) * B * L, st), "memset");
  ck(cudaMemsetAsync(R.rec_flags, 0, sizeof(int) * B * cap, st), "memset");
  ck(cudaMemsetAsync(R.bad_u, 0, sizeof(int) * B * L, st), "memset");
  // NaN fill (0xff bytes is a NaN pattern for doubles)
  ck(cudaMemsetAsync(R.rec_obj, 0xff, sizeof(double) * B * cap, st), "memset");
  ck(cudaMemsetAsync(R.rec_err, 0xff, sizeof(double) * B * cap, st), "memset");
  ck(cudaMemsetAsync(R.rec_exact, 0xff, sizeof(double) * B * cap, st), "memset");
  ck(cudaMemsetAsync(R.rec_tv, 0xff, sizeof(double) * B * cap * L, st), "memset");
  std::vector<int> ones(B, 1);
  ck(cudaMemcpyAsync(R.n_recs, ones.data(), sizeof(int) * B, cudaMemcpyHostToDevice, st), "n_recs");
  ck(cudaStreamSynchronize(st), "sync");
}

// Kind dispatch ------------------------------------------------------------------------
cudaError_t task(const DevProblem& P, const DevRun& R, const TaskArgs& A, int ignore_done, cudaStream_t st) {
  switch (P.kind) {
    case QOC_KIND_DENSE:
      return P.d > 32 ? dense_big_task(P, R, A, ignore_done, st) : dense_task(P, R, A, ignore_done, st);
    case QOC_KIND_TRIDIAG: return tridiag_task(P, R, A, ignore_done, st);
    case QOC_KIND_BITFLIP: return bitflip_task(P, R, A, ignore_done, st);
    case QOC_KIND_STRANG: return strang_task(P, R, A, ignore_done, st);
    case QOC_KIND_DENSITY: return density_task(P, R, A, ignore_done, st);
  }
  return cudaErrorInvalidValue;
}
cudaError_t horizon(const DevProblem& P, const DevRun& R, int which, int k, cudaStream_t st) {
  switch (P.kind) {
    case QOC_KIND_DENSE:
      return P.d > 32 ? dense_big_horizon(P, R, which, k, st) : dense_horizon(P, R, which, k, st);
    case QOC_KIND_TRIDIAG: return tridiag_horizon(P, R, which, k, st);
    case QOC_KIND_BITFLIP: return bitflip_horizon(P, R, which, k, st);
    case QOC_KIND_STRANG: return strang_horizon(P, R, which, k, st);
    case QOC_KIND_DENSITY: return density_horizon(P, R, which, k, st);
  }
  return cudaErrorInvalidValue;
}

void check_flags(const DevRun& R) {
  int flags = 0;
  ck(cudaMemcpy(&flags, R.err_flags, sizeof(int), cudaMemcpyDeviceToHost), "flags");
  if (flags & 1)
    fail(QOC_ERUNTIME, "tridiagonal Cayley solve would need a row interchange (dt/2 |H| too large for the "
                       "structured kind); use QOC_KIND_DENSE");
  if (flags & 2)
    fail(QOC_ERUNTIME, "bit-flip Cayley solve would not converge (dt/2 sum_i |V_i(u)| >= 1/2)");
}

// Launch wrapper: counts launches and, when profiling, brackets each launch with events.
struct Launcher {
  qoc_ctx* ctx;
  bool in_iteration = false;
  template <class F>
  void run(F&& f, const char* what, bool is_task = false) {
    cudaEvent_t a = nullptr, b = nullptr;
    if (ctx->profile) {
      ck(cudaEventCreate(&a), "event");
      ck(cudaEventCreate(&b), "event");
      ck(cudaEventRecord(a, ctx->stream), "event");
    }
    const cudaError_t e = f();
    ++ctx->launches;
    if (in_iteration) ++ctx->prof.iteration_launches;
    if (ctx->profile) {
      ck(cudaEventRecord(b, ctx->stream), "event");
      ctx->marks.emplace_back(a, b, is_task, what);
    }
    if (e == cudaErrorNotSupported) fail(QOC_ELOGIC, std::string(what) + ": not supported for this model kind");
    ck(e, what);
  }
  void extra(int64_t n) {  // launch sites that issue more than one kernel
    ctx->launches += n;
    if (in_iteration) ctx->prof.iteration_launches += n;
  }
  void operator()(cudaError_t e, const char* what) {  // already-launched form (no timing)
    ++ctx->launches;
    if (e == cudaErrorNotSupported) fail(QOC_ELOGIC, std::string(what) + ": not supported for this model kind");
    ck(e, what);
  }
};

void harvest_marks(qoc_ctx* ctx) {
  for (auto& [a, b, is_task, what] : ctx->marks) {
    float ms = 0.f;
    if (cudaEventElapsedTime(&ms, a, b) == cudaSuccess) {
      auto it = std::find_if(ctx->by_label.begin(), ctx->by_label.end(),
                             [&](const auto& e) { return e.first == what; });
      if (it == ctx->by_label.end()) {
        ctx->by_label.push_back({std::string(what), {0.0, 0}});
        it = ctx->by_label.end() - 1;
      }
      it->second.first += ms;
      it->second.second += 1;
      if (is_task) {
        ctx->prof.task_ms += ms;
        ++ctx->prof.task_launches;
      } else {
        ctx->prof.other_ms += ms;
        ++ctx->prof.other_launches;
      }
    }
    cudaEventDestroy(a);
    cudaEventDestroy(b);
  }
  ctx->marks.clear();
}

// QOC_TRACE_HOST=1: wall-clock phases of qoc_ism_run on stderr (host-side e2e breakdown)
struct HostTrace {
  bool on = std::getenv("QOC_TRACE_HOST") != nullptr;
  std::chrono::steady_clock::time_point t0 = std::chrono::steady_clock::now(), last = t0;
  void mark(const char* what, cudaStream_t st = nullptr) {
    if (!on) return;
    if (st) cudaStreamSynchronize(st);
    const auto now = std::chrono::steady_clock::now();
    std::fprintf(stderr, "[qoc host] %-22s %9.3f ms\n", what, std::chrono::duration<double, std::milli>(now - last).count());
    last = now;
  }
};

template <class F>
int32_t guarded(qoc_ctx* ctx, F&& f) {
  if (!ctx) return QOC_EINVAL;
  try {
    ck(cudaSetDevice(ctx->device), "cudaSetDevice");
    f();
    ctx->last_error.clear();
    return QOC_OK;
  } catch (const Fail& e) {
    ctx->last_error = e.msg;
    if (e.code == QOC_ECUDA) cudaGetLastError();
    return e.code;
  } catch (const std::exception& e) {
    ctx->last_error = e.what();
    return QOC_ERUNTIME;
  }
}

// QOC_DISABLE="onepass" restores the two-pass iteration order (A/B on the GPU box)
bool disabled_path(const char* what) {
  const char* e = std::getenv("QOC_DISABLE");
  return e && std::strstr(e, what) != nullptr;
}

// NCCL entry points resolved at run time: libqoc_b200.so links no NCCL, so single-GPU use
// needs none; in a PyTorch process dlopen("libnccl.so.2") returns the NCCL torch already
// loaded (one NCCL per process), elsewhere the system one.
struct NcclApi {
  ncclResult_t (*get_unique_id)(ncclUniqueId*) = nullptr;
  ncclResult_t (*comm_init_rank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
  ncclResult_t (*all_gather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  const char* (*error_string)(ncclResult_t) = nullptr;
  std::string why;
  bool ok() const { return get_unique_id && comm_init_rank && comm_destroy && all_gather && error_string; }
};

const NcclApi& nccl_api() {
  static NcclApi api = [] {
    NcclApi a;
    void* h = nullptr;
    const char* env = std::getenv("QOC_NCCL_LIBRARY");
    for (const char* name : {env, "libnccl.so.2", "libnccl.so"}) {
      if (name && (h = dlopen(name, RTLD_NOW | RTLD_GLOBAL))) break;
    }
    if (!h) {
      a.why = std::string("cannot load libnccl.so.2: ") + (dlerror() ? dlerror() : "not found");
      return a;
    }
    a.get_unique_id = reinterpret_cast<decltype(a.get_unique_id)>(dlsym(h, "ncclGetUniqueId"));
    a.comm_init_rank = reinterpret_cast<decltype(a.comm_init_rank)>(dlsym(h, "ncclCommInitRank"));
    a.comm_destroy = reinterpret_cast<decltype(a.comm_destroy)>(dlsym(h, "ncclCommDestroy"));
    a.all_gather = reinterpret_cast<decltype(a.all_gather)>(dlsym(h, "ncclAllGather"));
    a.error_string = reinterpret_cast<decltype(a.error_string)>(dlsym(h, "ncclGetErrorString"));
    if (!a.ok()) a.why = "libnccl.so.2 lacks an expected entry point";
    return a;
  }();
  return api;
}

void nccl_ck(ncclResult_t r, const char* what) {
  if (r != ncclSuccess) fail(QOC_ENCCL, std::string(what) + ": " + nccl_api().error_string(r));
}

// Balanced contiguous split of L subintervals into G blocks (the first L mod G blocks get one
// more), as subinterval boundary indices [G+1].
std::vector<int> block_nodes(int L, int G) {
  std::vector<int> b{0};
  for (int g = 0; g < G; ++g) b.push_back(b.back() + L / G + (g < L % G ? 1 : 0));
  return b;
}

}  // namespace

extern "C" {

int32_t qoc_abi_version(void) { return QOC_ABI_VERSION; }

int32_t qoc_ctx_create(const qoc_ctx_opts_v1* opts, qoc_ctx** out) {
  if (!out) return QOC_EINVAL;
  *out = nullptr;
  if (opts && opts->abi_version != QOC_ABI_VERSION) return QOC_EINVAL;
  int dev = opts ? opts->device : -1;
  if (dev < 0 && cudaGetDevice(&dev) != cudaSuccess) return QOC_ECUDA;
  if (cudaSetDevice(dev) != cudaSuccess) return QOC_ECUDA;
  cudaDeviceProp prop{};
  if (cudaGetDeviceProperties(&prop, dev) != cudaSuccess) return QOC_ECUDA;
  if (prop.major < 10) return QOC_ECUDA;  // built for sm_100a only
  auto* c = new qoc_ctx;
  c->device = dev;
  if (cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking) != cudaSuccess ||
      cudaStreamCreateWithFlags(&c->aux, cudaStreamNonBlocking) != cudaSuccess ||
      cudaEventCreateWithFlags(&c->ev_fork, cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&c->ev_join, cudaEventDisableTiming) != cudaSuccess) {
    delete c;
    return QOC_ECUDA;
  }
  *out = c;
  return QOC_OK;
}

void qoc_ctx_destroy(qoc_ctx* ctx) {
  if (!ctx) return;
  cudaSetDevice(ctx->device);
  if (ctx->stream) cudaStreamDestroy(ctx->stream);
  if (ctx->aux) cudaStreamDestroy(ctx->aux);
  if (ctx->ev_fork) cudaEventDestroy(ctx->ev_fork);
  if (ctx->ev_join) cudaEventDestroy(ctx->ev_join);
  if (ctx->flush_buf) cudaFree(ctx->flush_buf);
  if (ctx->khost) cudaFreeHost(ctx->khost);
  if (ctx->stage) cudaFreeHost(ctx->stage);
  if (ctx->gcache) cudaGraphExecDestroy(ctx->gcache);
  if (ctx->comm && nccl_api().ok()) nccl_api().comm_destroy(ctx->comm);
  delete static_cast<Slots*>(ctx->prob_slots);
  delete static_cast<Slots*>(ctx->run_slots);
  delete ctx;
}

int32_t qoc_ctx_set_option(qoc_ctx* ctx, int32_t option, int64_t value) {
  if (!ctx) return QOC_EINVAL;
  cudaSetDevice(ctx->device);
  if (option == QOC_OPT_PROFILE) {
    ctx->profile = value != 0;
    return QOC_OK;
  }
  if (option == QOC_OPT_FLUSH_L2_BYTES) {
    if (ctx->flush_buf) cudaFree(ctx->flush_buf);
    ctx->flush_buf = nullptr;
    ctx->flush_bytes = 0;
    if (value > 0) {
      if (cudaMalloc(&ctx->flush_buf, (size_t)value) != cudaSuccess) return QOC_ECUDA;
      ctx->flush_bytes = value;
    }
    return QOC_OK;
  }
  return QOC_EINVAL;
}

int32_t qoc_ctx_solver_stats(const qoc_ctx* ctx, int32_t b, int32_t iteration, int32_t subintervals, int32_t* out) {
  if (!ctx || !out) return QOC_EINVAL;
  const int* dm = ctx->solver_stats_dims;
  if (iteration < 1 || iteration >= dm[0] || b < 0 || b >= dm[1] || subintervals != dm[2]) return QOC_EINVAL;
  const int L = dm[2];
  const int* row = ctx->solver_stats.data() + ((size_t)iteration * dm[1] + b) * L * 3;
  for (int n = 0; n < L; ++n)
    for (int q = 0; q < 3; ++q) out[q * L + n] = row[n * 3 + q];
  return QOC_OK;
}

int32_t qoc_ctx_profile(qoc_ctx* ctx, qoc_profile_v1* out, int32_t reset) {
  if (!ctx) return QOC_EINVAL;
  if (out) *out = ctx->prof;
  if (reset) {
    ctx->prof = qoc_profile_v1{};
    ctx->by_label.clear();
  }
  return QOC_OK;
}

int32_t qoc_ctx_kernel_profile(const qoc_ctx* ctx, int32_t index, char* name, size_t name_len, double* ms,
                               int64_t* launches) {
  if (!ctx || index < 0) return QOC_EINVAL;
  if ((size_t)index >= ctx->by_label.size()) return QOC_EINVAL;
  const auto& e = ctx->by_label[(size_t)index];
  if (name && name_len) std::snprintf(name, name_len, "%s", e.first.c_str());
  if (ms) *ms = e.second.first;
  if (launches) *launches = e.second.second;
  return QOC_OK;
}

const char* qoc_ctx_last_error(const qoc_ctx* ctx) { return ctx ? ctx->last_error.c_str() : "null context"; }

int64_t qoc_ctx_launch_count(const qoc_ctx* ctx) { return ctx ? ctx->launches : 0; }

int32_t qoc_comm_unique_id(void* out, size_t len) {
  if (!out || len < NCCL_UNIQUE_ID_BYTES) return QOC_EINVAL;
  const NcclApi& a = nccl_api();
  if (!a.ok()) return QOC_ENCCL;
  ncclUniqueId id;
  if (a.get_unique_id(&id) != ncclSuccess) return QOC_ENCCL;
  std::memcpy(out, &id, sizeof id);
  return QOC_OK;
}

int32_t qoc_ctx_init_comm(qoc_ctx* ctx, int32_t rank, int32_t world, const void* id, size_t len) {
  return guarded(ctx, [&] {
    if (world < 1 || rank < 0 || rank >= world) fail(QOC_EINVAL, "rank must lie in [0, world)");
    if (ctx->comm) {
      nccl_api().comm_destroy(ctx->comm);
      ctx->comm = nullptr;
    }
    ctx->rank = 0;
    ctx->world = 1;
    // world = 1 with an id: a one-rank communicator (the exchange path runs, trivially)
    if (world > 1 || id) {
      if (!id || len < NCCL_UNIQUE_ID_BYTES) fail(QOC_EINVAL, "a communicator of world > 1 needs the 128-byte NCCL unique id");
      const NcclApi& a = nccl_api();
      if (!a.ok()) fail(QOC_ENCCL, a.why);
      ncclUniqueId uid;
      std::memcpy(&uid, id, sizeof uid);
      nccl_ck(a.comm_init_rank(&ctx->comm, world, uid, rank), "ncclCommInitRank");
    }
    ctx->rank = rank;
    ctx->world = world;
  });
}

int32_t qoc_ism_run(qoc_ctx* ctx, const qoc_problem_v1* p, const qoc_ism_config_v1* cfg,
                    const qoc_solver_v1* solver, const double* u0, double* u_out, qoc_iter_record_v1* recs,
                    int32_t rec_cap, double* task_values, qoc_run_status_v1* status) {
  return guarded(ctx, [&] {
    HostTrace trace;
    validate_problem(p);
    if (!cfg || !solver || !u0 || !u_out || !recs || !status) fail(QOC_EINVAL, "null argument");
    // ism.cpp:213-231
    if (cfg->subintervals < 1 || cfg->workers < 1 || cfg->max_outer < 0 || cfg->eta < 0.0)
      fail(QOC_EINVAL, "subintervals and workers must be >= 1, max_outer and eta >= 0");
    const bool split = cfg->variant == QOC_VARIANT_SPLIT;
    if (!split && p->kind == QOC_KIND_STRANG)
      fail(QOC_EINVAL,
           "interpolated waypoints require linear one-step flows; use the split variant for split-step states");
    if (solver->kind < QOC_SOLVER_GRADIENT || solver->kind > QOC_SOLVER_NEWTON) fail(QOC_EINVAL, "unknown solver kind");
    // run_inner dispatches per inner iteration (optimizers.cpp:261-285): a run that never calls the
    // solver never sees its preconditions
    const bool alt_solver = solver->kind != QOC_SOLVER_GRADIENT;
    const bool monotonic = solver->kind == QOC_SOLVER_MONOTONIC, newton = solver->kind == QOC_SOLVER_NEWTON;
    if (monotonic && cfg->max_outer > 0 && solver->inner_iterations > 0) {  // optimizers.cpp:110-122
      if (p->kind == QOC_KIND_DENSITY || p->kind == QOC_KIND_STRANG)
        fail(QOC_ELOGIC, "the monotonic sweep requires column states with the one-step rational scheme");
      if (p->kind == QOC_KIND_BITFLIP)
        fail(QOC_ELOGIC, "the monotonic sweep on the device takes the operators as matrices; repack the spin "
                         "register as QOC_KIND_DENSE (d <= 64)");
      if (p->channels != 1) fail(QOC_ELOGIC, "the monotonic sweep handles a single control channel");
      for (int j = 0; j < p->steps; ++j)
        if (!p->penalty || p->penalty[j] <= 0.0)
          fail(QOC_ELOGIC, "the monotonic sweep requires strictly positive penalty weights");
      if (p->dim < 2 || p->dim > 64) fail(QOC_ELOGIC, "the monotonic sweep on the device takes 2 <= d <= 64");
    }
    if (rec_cap < cfg->max_outer + 1) fail(QOC_EINVAL, "rec_cap must be >= max_outer + 1");
    const std::vector<int> node = decomposition(p->steps, cfg->subintervals, cfg->partition, cfg->node_index);
    const int L = cfg->subintervals, B = p->batch, C = p->channels, K = p->steps;
    // Blocked boundary refresh (bit-flip kind, assembled plan, SURVEY §8(e) option A): G
    // contiguous blocks of subintervals; each rank forms its blocks' d x d products, one
    // all-gather exchanges them, every rank chains the G products into the block-boundary
    // nodes and sweeps its blocks' interiors.  G = L is the reference's assembled plan
    // (ism.cpp:298-312); blocks = 0 on one GPU keeps the direct node sweeps, which agree with
    // the assembled chain to rounding (ism_test.cpp:248-265); on W GPUs it means G = W.
    if (cfg->blocks < 0) fail(QOC_EINVAL, "blocks must be >= 0");
    const int G = (p->kind == QOC_KIND_BITFLIP && !split && L > 1 && cfg->plan == QOC_PLAN_ASSEMBLED)
                      ? (cfg->blocks > 0 ? cfg->blocks : (ctx->world > 1 ? ctx->world : 0))
                      : 0;
    const bool blocked = G > 0;
    if (blocked && alt_solver) fail(QOC_ELOGIC, "the blocked plan runs the gradient solver");
    if (blocked) {
      if (G > L) fail(QOC_EINVAL, "blocks must not exceed subintervals");
      if (G % ctx->world != 0) fail(QOC_EINVAL, "blocks must be a multiple of the communicator size");
      if (B != 1) fail(QOC_ELOGIC, "the blocked plan runs one problem per call (batch = 1)");
    }
    // the density kind's assembled plan chains the tasks' dm x dm products as prop * rho * prop^dag
    // (apply_propagator, propagation.cpp:251-261); QOC_DISABLE=denschain keeps the serial node sweeps
    const bool direct = !blocked && (cfg->plan == QOC_PLAN_DIRECT || p->kind == QOC_KIND_BITFLIP ||
                                     (p->kind == QOC_KIND_DENSITY && disabled_path("denschain")));
    const bool assembled_interp = L > 1 && !split && !direct && !blocked;
    cudaStream_t st = ctx->stream;
    Launcher launch{ctx};

    // The monotonic sweep needs dH/dv as matrices: a tridiagonal model (the reference's rotor is a
    // DenseModel, models.cpp:349-380) is expanded to the dense payload for that solver.
    qoc_problem_v1 dense_view;
    std::vector<double> tri_h0, tri_lin, tri_quad;
    if (monotonic && p->kind == QOC_KIND_TRIDIAG && cfg->max_outer > 0 && solver->inner_iterations > 0) {
      const int d = p->dim;
      const size_t dd = (size_t)d * d;
      const int nq = p->tri_has_quadratic ? C : 0, nops = 1 + C + nq;
      tri_h0.assign(2 * dd * B, 0.0);
      tri_lin.assign(2 * dd * B * C, 0.0);
      tri_quad.assign(2 * dd * B * std::max(nq, 1), 0.0);
      for (int b = 0; b < B; ++b)
        for (int o = 0; o < nops; ++o) {
          double* dst = o == 0 ? tri_h0.data() + 2 * dd * b
                               : (o <= C ? tri_lin.data() + 2 * dd * ((size_t)b * C + o - 1)
                                         : tri_quad.data() + 2 * dd * ((size_t)b * C + o - 1 - C));
          const double* dg = p->tri_diag + ((size_t)b * nops + o) * d;
          const double* sb = p->tri_sub + 2 * ((size_t)b * nops + o) * (d - 1);
          for (int j = 0; j < d; ++j) dst[2 * (j + (size_t)j * d)] = dg[j];
          for (int j = 0; j + 1 < d; ++j) {  // column-major: entry (j+1, j) and its conjugate at (j, j+1)
            dst[2 * ((j + 1) + (size_t)j * d)] = sb[2 * j];
            dst[2 * ((j + 1) + (size_t)j * d) + 1] = sb[2 * j + 1];
            dst[2 * (j + (size_t)(j + 1) * d)] = sb[2 * j];
            dst[2 * (j + (size_t)(j + 1) * d) + 1] = -sb[2 * j + 1];
          }
        }
      dense_view = *p;
      dense_view.kind = QOC_KIND_DENSE;
      dense_view.h0 = tri_h0.data();
      dense_view.linear = tri_lin.data();
      dense_view.quadratic = nq ? tri_quad.data() : nullptr;
      p = &dense_view;
    }
    DeviceProblem dp;
    dp.slots = fresh_slots(ctx->prob_slots);
    upload_problem(p, node, st, dp);
    trace.mark("upload problem", st);
    // gradient options of the task sweeps, lagged refresh and node sweeps (ism.cpp:373,437,446,543)
    dp.P.naive = (solver->naive_nonlinear_adjoint && p->kind == QOC_KIND_STRANG) ? 1 : 0;
    const DevProblem& P = dp.P;
    DeviceRun dr;
    dr.slots = fresh_slots(ctx->run_slots);
    // the monotonic and Newton solvers run on the kinds' own task kernels (no propagator cache)
    const bool pcache = !alt_solver && use_pcache(P, node);
    alloc_run(dp, rec_cap, node, assembled_interp, false, st, dr, pcache, split);
    const DevRun& R = dr.R;
    ck(cudaMemcpyAsync(R.u, u0, sizeof(double) * B * K * C, cudaMemcpyHostToDevice, st), "u0");
    // inner-solver workspace and per-task counters (InnerResult, optimizers.hpp:32-37)
    DevNewton NW{};
    int* sstats = nullptr;       // [B][L][3] of the running outer iteration
    int* sstats_hist = nullptr;  // [max_outer + 1][B][L][3]
    const size_t nstat = (size_t)B * L * 3;
    if (alt_solver) {
      sstats = dr.alloc<int>(nstat);
      sstats_hist = dr.alloc<int>(nstat * (cfg->max_outer + 1));
      ck(cudaMemsetAsync(sstats_hist, 0, sizeof(int) * nstat * (cfg->max_outer + 1), st), "memset");
    }
    if (newton) {
      const size_t grid = (size_t)B * K * C, T = (size_t)B * L;
      const int RS = std::max(1, solver->gmres_restart);
      NW.restart = RS;
      NW.max_iter = solver->gmres_max_iter;
      NW.tol = solver->gmres_tol;
      NW.hvp_scale = solver->hvp_scale;
      NW.step_size = solver->step_size;
      NW.weighted = split ? 0 : 1;
      NW.vstride = grid;
      NW.g0 = dr.alloc<double>(grid);
      NW.x = dr.alloc<double>(grid);
      NW.V = dr.alloc<double>(grid * (RS + 1));
      NW.up = dr.alloc<double>(grid);
      NW.um = dr.alloc<double>(grid);
      NW.gp = dr.alloc<double>(grid);
      NW.gm = dr.alloc<double>(grid);
      NW.Hm = dr.alloc<double>(T * (RS + 1) * RS);
      NW.gv = dr.alloc<double>(T * (RS + 1));
      NW.cs = dr.alloc<double>(T * RS);
      NW.sn = dr.alloc<double>(T * RS);
      NW.sc = dr.alloc<double>(T * 4);
      NW.st = dr.alloc<int>(T * 8);
      NW.active = dr.alloc<int>(std::max(0, NW.max_iter) + 4);
      NW.stats = sstats;
      if (solver->gmres_restart < 1) fail(QOC_EINVAL, "gmres_restart must be >= 1");
    }
    // blocked plan: the exchange slabs and this rank's blocks / subintervals
    DevBlocks BK{};
    int g_lo = 0, n_lo = 0, n_cnt = 0;
    bool interior = false;
    if (blocked) {
      const std::vector<int> bn = block_nodes(L, G);
      BK.G = G;
      BK.W = ctx->world;
      BK.rank = ctx->rank;
      BK.bpr = G / BK.W;
      for (int r = 0; r < BK.W; ++r) {
        const int a = bn[r * BK.bpr], z = bn[(r + 1) * BK.bpr];
        BK.lmax = std::max(BK.lmax, z - a);
        BK.kmax = std::max(BK.kmax, node[z] - node[a]);
      }
      for (int g = 0; g < G; ++g) interior = interior || bn[g + 1] - bn[g] > 1;
      const size_t dd = (size_t)P.d * P.d, scal = 2 * (size_t)BK.lmax + (size_t)BK.kmax * C;
      BK.slab_elems = (size_t)BK.bpr * dd + (scal + 1) / 2;
      BK.slab = dr.alloc<double2>((size_t)BK.W * BK.slab_elems);
      int* bnd = dr.alloc<int>(G + 1);
      ck(cudaMemcpyAsync(bnd, bn.data(), sizeof(int) * (G + 1), cudaMemcpyHostToDevice, st), "block nodes");
      BK.bnode = bnd;
      g_lo = ctx->rank * BK.bpr;
      n_lo = bn[g_lo];
      n_cnt = bn[g_lo + BK.bpr] - n_lo;
      // other ranks' interior nodes stay zero here (finite for the boundary check)
      ck(cudaMemsetAsync(R.psi_nodes, 0, sizeof(double2) * (L + 1) * P.d, st), "memset");
      ck(cudaMemsetAsync(R.chi_nodes, 0, sizeof(double2) * (L + 1) * P.d, st), "memset");
    }
    const SweepRange SR{BK.bnode, g_lo, BK.bpr};
    // the one collective per outer iteration: every rank's slab (block products, entry values,
    // residuals, controls) to every rank, in place, on the compute stream
    auto exchange = [&](Launcher& ln) {
      if (!blocked || !ctx->comm) return;
      ln.run([&] { return slab_pack(P, R, BK, 1, st); }, "pack");
      const size_t bytes = sizeof(double2) * BK.slab_elems;
      nccl_ck(nccl_api().all_gather(BK.slab + (size_t)BK.rank * BK.slab_elems, BK.slab, bytes, ncclUint8, ctx->comm, st),
              "ncclAllGather");
      ln.run([&] { return slab_unpack(P, R, BK, 1, st); }, "unpack");
    };
    auto blocked_refresh = [&](Launcher& ln, const DevRun& RR, int k) {
      ln.run([&] { return bitflip_block_products(P, RR, BK, g_lo, BK.bpr, st); }, "block products", true);
      exchange(ln);
      ln.run([&] { return block_chain(P, RR, BK, st); }, "chain");
      ln.extra(G);  // the chain issues G + 1 kernels
      if (interior) ln.run([&] { return bitflip_horizon_range(P, RR, 0, k, SR, st); }, "node sweeps", true);
    };
    trace.mark("alloc + u0", st);

    const int max_outer = cfg->max_outer;
    std::vector<cudaEvent_t> ev(max_outer + 2);
    for (auto& e : ev) ck(cudaEventCreate(&e), "event");
    auto destroy_events = [&] {
      for (auto& e : ev) cudaEventDestroy(e);
    };
    const int form = split ? QOC_FORM_OVERLAP : QOC_FORM_TRACKING;
    // run_inner (optimizers.cpp:261-285): inner_iterations <= 0 makes no update but the entry
    // value is still evaluated (ism.cpp:407)
    const int inner = std::max(0, solver->inner_iterations);
    // One cache pass per iteration instead of two (Neumann path, one inner update, residual
    // logged): the pass after the boundary refresh evaluates the residual of iteration k with
    // the saved tasks S_k and the entry value + update of iteration k + 1 with S_{k+1}, both at
    // the control u_{k+1} the cache was assembled for; the update lands at the start of k + 1.
    // Same arithmetic as the gradient -> assembly -> residual order, reordered.
    const bool onepass = pcache && R.nm && !split && inner == 1 && cfg->compute_error &&
                         dense_pc_eval16_applicable(P, R, PCM_ENTRY | PCM_GRAD | PCM_ERR, 1) && !disabled_path("onepass");
    try {
      ck(cudaEventRecord(ev[0], st), "event");
      // ---- bootstrap (ism.cpp:344-393)
      if (R.nm) launch(dense_nm_setup(P, R, st), "neumann coefficients");
      if (pcache) launch(pc_assemble(P, R, 0, st), "propagator cache");
      if (L > 1) {
        if (blocked) {
          blocked_refresh(launch, R, 0);
        } else if (assembled_interp) {
          if (!pcache) {
            TaskArgs A{M_ASSEMBLE, QOC_FORM_TRACKING, 1, 1, 0.0};
            launch(task(P, R, A, 0, st), "assemble");
          }
          launch(chain_propagators(P, R, st), "chain");
        } else {
          launch(horizon(P, R, 0, 0, st), "node sweeps");
        }
        launch(penalty_partials(P, R, 0, st), "penalty");
        launch(boundary_update(P, R, 0, split, 1, st), "boundary");
      } else {
        launch(set_single_tasks(P, R, st), "tasks");
      }
      // one-pass iteration: the first entry value and update come from the bootstrap cache
      if (onepass) launch(pc_eval_dual(P, R, form, split ? 0 : 1, solver->step_size, 2, st), "gradient");
      ck(cudaEventRecord(ev[1], st), "event");
      trace.mark("bootstrap", st);

      int mode = M_ENTRY | (inner > 0 ? M_UPDATE : 0);
      if (cfg->compute_error) mode |= M_ERROR;
      if (assembled_interp) mode |= M_ASSEMBLE;
      if (L > 1 && split && !direct) mode |= M_LAGGED;
      TaskArgs A{mode, form, split ? 0 : 1, inner, solver->step_size};
      if (blocked) {  // this rank's subintervals only
        A.n_lo = n_lo;
        A.n_cnt = n_cnt;
      }
      std::vector<int> h_done(B), h_status(B);
      std::vector<cudaEvent_t> ev_end(max_outer + 2);
      for (auto& e : ev_end) ck(cudaEventCreate(&e), "event");
      int ran = 0;
      launch.in_iteration = true;
      // One outer iteration (ism.cpp:396-592) as a launch sequence on `st` (+ the side stream).
      auto body = [&](const DevRun& RR, int k) {
        if (blocked) {
          launch.run([&] { return task(P, RR, A, 0, st); }, "task", true);
          blocked_refresh(launch, RR, k);  // block products at the updated control + exchange
          launch.run([&] { return penalty_partials(P, RR, 0, st); }, "penalty");
          launch.run([&] { return merge_iteration(P, RR, k, nullptr, st); }, "merge");
          launch.run([&] { return boundary_update(P, RR, k, 0, 0, st); }, "boundary");
          if (cfg->log_exact_objective) launch.run([&] { return exact_from_nodes(P, RR, k, st); }, "exact objective");
          launch.run([&] { return finish_iteration_ex(P, RR, k, cfg->compute_error, cfg->eta,
                                                      cfg->log_exact_objective, st); }, "finish");
          return;
        }
        if (onepass) {
          launch.run([&] { return apply_pending(P, RR, solver->step_size, st); }, "update");
          launch.run([&] { return penalty_partials(P, RR, 0, st); }, "penalty");
          launch.run([&] { return merge_iteration(P, RR, k, nullptr, st); }, "merge");
          launch.run([&] { return pc_assemble(P, RR, 0, st); }, "assembly", true);
          launch.run([&] { return save_tasks(P, RR, st); }, "save tasks");
          if (L > 1) {
            if (direct) launch.run([&] { return horizon(P, RR, 0, k, st); }, "node sweeps", true);
            else launch.run([&] { return chain_propagators(P, RR, st); }, "chain");
            launch.run([&] { return boundary_update(P, RR, k, split, 0, st); }, "boundary");
          }
          if (cfg->log_exact_objective) launch.run([&] { return horizon(P, RR, 1, k, st); }, "exact objective", true);
          launch.run([&] { return pc_eval_dual(P, RR, form, 1, solver->step_size, 1, st); }, "evaluation", true);
          launch.run([&] { return total_error(P, RR, st); }, "error total");
          launch.run([&] { return finish_iteration_ex(P, RR, k, cfg->compute_error, cfg->eta,
                                                      cfg->log_exact_objective, st); }, "finish");
          return;
        }
        if (pcache) {
          // gradient + update through the cache, then the assembly sweep at the new control,
          // then residual / lagged endpoints through the new cache
          const TaskArgs G{PCM_ENTRY | (inner > 0 ? PCM_GRAD : 0), form, split ? 0 : 1, 1, solver->step_size};
          launch.run([&] { return pc_eval(P, RR, G, 0, st); }, "gradient", true);
          for (int it = 1; it < inner; ++it) {
            launch.run([&] { return pc_assemble(P, RR, 0, st); }, "assembly", true);
            const TaskArgs G2{PCM_GRAD, form, split ? 0 : 1, 1, solver->step_size};
            launch.run([&] { return pc_eval(P, RR, G2, 0, st); }, "gradient", true);
          }
          // no update (inner = 0): the cache and the propagators already belong to this control.
          // Where the assembly sweep fuses the residual (dense_nm.cu), it is evaluated there.
          const bool fuse_err = cfg->compute_error && inner > 0 && !(L > 1 && split && !direct) &&
                                pc_fuses_residual(P, RR);
          if (inner > 0)
            launch.run([&] { return pc_assemble(P, RR, 0, st, fuse_err ? form : -1); }, "assembly", true);
          if (assembled_interp) {
            // the boundary chain needs only the new propagators: run it on the side stream,
            // concurrently with the residual sweep, penalty and merge (joined before boundary)
            ck(cudaEventRecord(ctx->ev_fork, st), "fork");
            ck(cudaStreamWaitEvent(ctx->aux, ctx->ev_fork, 0), "fork");
            launch(chain_propagators(P, RR, ctx->aux), "chain");
            ck(cudaEventRecord(ctx->ev_join, ctx->aux), "join");
          }
          const int em = ((cfg->compute_error && !fuse_err) ? PCM_ERR : 0) | ((L > 1 && split && !direct) ? PCM_LAG : 0);
          if (em) {
            const TaskArgs E{em, form, split ? 0 : 1, 1, 0.0};
            launch.run([&] { return pc_eval(P, RR, E, 0, st); }, "residual", true);
          }
        } else if (alt_solver) {
          // entry value, then run_inner with the monotonic / Newton solver, then the sweeps at the
          // updated control (ism.cpp:407-459)
          const TaskArgs E{M_ENTRY, form, split ? 0 : 1, 1, 0.0};
          launch.run([&] { return task(P, RR, E, 0, st); }, "task", true);
          ck(cudaMemsetAsync(sstats, 0, sizeof(int) * nstat, st), "memset");
          for (int it = 0; it < inner; ++it) {
            if (monotonic) {
              launch.run([&] { return monotonic_sweep(P, RR, split ? 0 : 1, solver->fixed_point_tol,
                                                      solver->fixed_point_max_iter, sstats, st); }, "monotonic sweep", true);
              continue;
            }
            const TaskArgs Gm{M_GRAD, form, 0, 1, 0.0};
            DevRun RG0 = RR, RGp = RR, RGm = RR;
            RG0.grad = NW.g0;
            RGp.u = NW.up;
            RGp.grad = NW.gp;
            RGm.u = NW.um;
            RGm.grad = NW.gm;
            launch.run([&] { return task(P, RG0, Gm, 0, st); }, "newton gradient", true);
            ck(cudaMemsetAsync(NW.active, 0, sizeof(int) * (std::max(0, NW.max_iter) + 4), st), "memset");
            launch.run([&] { return newton_begin(P, RR, NW, st); }, "gmres");
            for (int round = 1; round <= std::max(0, NW.max_iter) + 3; ++round) {
              int act = 0;  // tasks with a Hessian-vector product pending
              ck(cudaMemcpyAsync(&act, NW.active + round - 1, sizeof(int), cudaMemcpyDeviceToHost, st), "poll");
              ck(cudaStreamSynchronize(st), "poll");
              if (act == 0) break;
              launch.run([&] { return task(P, RGp, Gm, 0, st); }, "newton gradient", true);
              launch.run([&] { return task(P, RGm, Gm, 0, st); }, "newton gradient", true);
              launch.run([&] { return newton_advance(P, RR, NW, round, st); }, "gmres");
            }
            launch.run([&] { return newton_apply(P, RR, NW, st); }, "newton update");
          }
          const int rest = mode & (M_ERROR | M_ASSEMBLE | M_LAGGED);
          if (rest) {
            const TaskArgs Rm{rest, form, split ? 0 : 1, 1, 0.0};
            launch.run([&] { return task(P, RR, Rm, 0, st); }, "task", true);
          }
          ck(cudaMemcpyAsync(sstats_hist + nstat * k, sstats, sizeof(int) * nstat, cudaMemcpyDeviceToDevice, st),
             "solver counters");
        } else {
          launch.run([&] { return task(P, RR, A, 0, st); }, "task", true);
        }
        launch.run([&] { return penalty_partials(P, RR, 0, st); }, "penalty");
        launch.run([&] { return merge_iteration(P, RR, k, nullptr, st); }, "merge");
        if (L > 1) {
          if (direct) launch.run([&] { return horizon(P, RR, 0, k, st); }, "node sweeps", true);
          else if (split) launch.run([&] { return split_nodes(P, RR, st); }, "split nodes");
          else if (pcache) ck(cudaStreamWaitEvent(st, ctx->ev_join, 0), "join");
          else launch.run([&] { return chain_propagators(P, RR, st); }, "chain");
          launch.run([&] { return boundary_update(P, RR, k, split, 0, st); }, "boundary");
        }
        if (cfg->log_exact_objective) launch.run([&] { return horizon(P, RR, 1, k, st); }, "exact objective", true);
        launch.run([&] { return finish_iteration_ex(P, RR, k, cfg->compute_error, cfg->eta,
                                                    cfg->log_exact_objective, st); }, "finish");
      };
      // Long runs replay the iteration as one CUDA graph (captured once; the iteration index
      // is read from device memory), which removes the per-kernel launch gaps of the small
      // latency-bound configs.  Profiling mode keeps direct launches (per-launch events).
      bool use_graph = !ctx->profile && max_outer >= 8 && !(blocked && ctx->comm) && !alt_solver;
      cudaGraphExec_t gexec = nullptr;
      int* kdev = nullptr;
      int64_t launches_per_body = 0;
      DevRun RG = R;
      if (use_graph) {
        kdev = dr.alloc<int>(1);
        RG.kdev = kdev;
        if ((int)ctx->khost_n < max_outer + 2) {
          if (ctx->khost) cudaFreeHost(ctx->khost);
          ctx->khost = nullptr;
          ctx->khost_n = 0;
          ck(cudaHostAlloc(reinterpret_cast<void**>(&ctx->khost), sizeof(int) * (max_outer + 2), cudaHostAllocDefault),
             "pinned iteration index");
          ctx->khost_n = max_outer + 2;
        }
        for (int k = 0; k < max_outer + 2; ++k) ctx->khost[k] = k;
      }
      // The instantiated graph is cached on the context and reused by the next call when every
      // launch parameter is byte-identical (same problem/run structs -- the workspace slots keep
      // the device pointers stable -- and the same loop configuration).
      std::vector<unsigned char> gkey;
      if (use_graph) {
        auto put = [&](const void* p, size_t n) {
          const unsigned char* c = static_cast<const unsigned char*>(p);
          gkey.insert(gkey.end(), c, c + n);
        };
        put(&P, sizeof(P));
        put(&RG, sizeof(RG));
        const int cfgv[] = {form, (int)split, (int)direct, (int)pcache, (int)assembled_interp, L,
                            cfg->compute_error, cfg->log_exact_objective, solver->inner_iterations, (int)onepass, G};
        put(&BK, sizeof(BK));
        put(cfgv, sizeof(cfgv));
        const double cfgd[] = {solver->step_size, cfg->eta};
        put(cfgd, sizeof(cfgd));
        if (ctx->gcache && ctx->gkey == gkey) {
          gexec = ctx->gcache;
          launches_per_body = ctx->gcache_launches;
        }
      }
      auto destroy_graph = [&] {
        if (gexec && gexec != ctx->gcache) cudaGraphExecDestroy(gexec);
        gexec = nullptr;
      };
      try {
        for (int k = 1; k <= max_outer; ++k) {
          if (ctx->flush_bytes > 0) {  // cold L2 for every iteration, outside the brackets
            ck(cudaMemsetAsync(ctx->flush_buf, k & 0xff, (size_t)ctx->flush_bytes, st), "flush");
            ck(cudaEventRecord(ev[k], st), "event");
          }
          if (use_graph) {
            ck(cudaMemcpyAsync(kdev, ctx->khost + k, sizeof(int), cudaMemcpyHostToDevice, st), "iteration index");
            if (!gexec) {
              const int64_t l0 = ctx->launches, i0 = ctx->prof.iteration_launches;
              cudaGraph_t graph = nullptr;
              bool ok = cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal) == cudaSuccess;
              if (ok) {
                try {
                  body(RG, k);
                } catch (...) {
                  ok = false;
                }
                ok = (cudaStreamEndCapture(st, &graph) == cudaSuccess) && ok && graph;
                if (ok) ok = cudaGraphInstantiate(&gexec, graph, 0) == cudaSuccess;
              }
              launches_per_body = ctx->launches - l0;  // counted during capture, added per replay
              if (ok) {  // exact kernel count of one replay: the graph's kernel nodes
                size_t nn = 0;
                if (cudaGraphGetNodes(graph, nullptr, &nn) == cudaSuccess && nn) {
                  std::vector<cudaGraphNode_t> nodes(nn);
                  if (cudaGraphGetNodes(graph, nodes.data(), &nn) == cudaSuccess) {
                    int64_t kn = 0;
                    for (auto nd : nodes) {
                      cudaGraphNodeType ty;
                      if (cudaGraphNodeGetType(nd, &ty) == cudaSuccess && ty == cudaGraphNodeTypeKernel) ++kn;
                    }
                    launches_per_body = kn;
                  }
                }
              }
              if (graph) cudaGraphDestroy(graph);
              ctx->launches = l0;
              ctx->prof.iteration_launches = i0;
              if (!ok) {  // capture unsupported here: fall back to direct launches
                cudaGetLastError();
                gexec = nullptr;
                use_graph = false;
                body(R, k);
              } else {
                if (ctx->gcache) cudaGraphExecDestroy(ctx->gcache);
                ctx->gcache = gexec;
                ctx->gkey = gkey;
                ctx->gcache_launches = launches_per_body;
              }
            }
            if (use_graph) {
              ck(cudaGraphLaunch(gexec, st), "graph launch");
              ctx->launches += launches_per_body;
              ctx->prof.iteration_launches += launches_per_body;
            }
          } else {
            body(R, k);
          }
          ck(cudaEventRecord(ev_end[k + 1], st), "event");
          if (ctx->flush_bytes <= 0) ck(cudaEventRecord(ev[k + 1], st), "event");
          ran = k;
          if (k % 8 == 0 || k == max_outer) {  // early exit once every problem stopped
            ck(cudaMemcpyAsync(h_done.data(), R.done, sizeof(int) * B, cudaMemcpyDeviceToHost, st), "poll");
            ck(cudaMemcpyAsync(h_status.data(), R.status, sizeof(int) * B, cudaMemcpyDeviceToHost, st), "poll");
            ck(cudaStreamSynchronize(st), "poll");
            bool all = true;
            for (int b = 0; b < B; ++b) all = all && (h_done[b] || h_status[b]);
            if (all) break;
          }
        }
      } catch (...) {
        destroy_graph();
        throw;
      }
      destroy_graph();
      launch.in_iteration = false;
      trace.mark("outer iterations", st);
      // ---- trailing evaluation (ism.cpp:594-609)
      {
        if (onepass) {
          // the last evaluation pass already left every problem's final entry values
        } else if (pcache) {
          const TaskArgs T{PCM_ENTRY, form, split ? 0 : 1, 1, 0.0};
          launch(pc_eval(P, R, T, 1, st), "trailing task");
        } else {
          TaskArgs T{M_ENTRY, form, split ? 0 : 1, 1, 0.0};
          if (blocked) {
            T.n_lo = n_lo;
            T.n_cnt = n_cnt;
          }
          launch(task(P, R, T, 1, st), "trailing task");
          exchange(launch);  // every rank's final entry values
        }
        launch(trailing_values(P, R, st), "trailing");
      }
      ck(cudaStreamSynchronize(st), "run");
      check_flags(R);
      trace.mark("trailing evaluation");

      // ---- download
      std::vector<int> n_recs(B), stat(B), abort_iter(B), flags((size_t)B * rec_cap);
      std::vector<double> obj((size_t)B * rec_cap), err((size_t)B * rec_cap), exact((size_t)B * rec_cap);
      download_large(ctx, u_out, R.u, sizeof(double) * B * K * C, "u_out");
      ck(cudaMemcpy(n_recs.data(), R.n_recs, sizeof(int) * B, cudaMemcpyDeviceToHost), "n_recs");
      ck(cudaMemcpy(stat.data(), R.status, sizeof(int) * B, cudaMemcpyDeviceToHost), "status");
      ck(cudaMemcpy(abort_iter.data(), R.abort_iter, sizeof(int) * B, cudaMemcpyDeviceToHost), "abort");
      ck(cudaMemcpy(flags.data(), R.rec_flags, sizeof(int) * flags.size(), cudaMemcpyDeviceToHost), "flags");
      ck(cudaMemcpy(obj.data(), R.rec_obj, sizeof(double) * obj.size(), cudaMemcpyDeviceToHost), "obj");
      ck(cudaMemcpy(err.data(), R.rec_err, sizeof(double) * err.size(), cudaMemcpyDeviceToHost), "err");
      ck(cudaMemcpy(exact.data(), R.rec_exact, sizeof(double) * exact.size(), cudaMemcpyDeviceToHost), "exact");
      if (task_values)
        download_large(ctx, task_values, R.rec_tv, sizeof(double) * (size_t)B * rec_cap * L, "task values");
      ctx->solver_stats.clear();
      ctx->solver_stats_dims[0] = ctx->solver_stats_dims[1] = ctx->solver_stats_dims[2] = 0;
      if (alt_solver) {  // per-task counters of iterations 1..ran
        ctx->solver_stats.resize(nstat * (ran + 1));
        ck(cudaMemcpy(ctx->solver_stats.data(), sstats_hist, sizeof(int) * nstat * (ran + 1), cudaMemcpyDeviceToHost),
           "solver counters");
        ctx->solver_stats_dims[0] = ran + 1;
        ctx->solver_stats_dims[1] = B;
        ctx->solver_stats_dims[2] = L;
      }
      std::vector<float> secs(ran + 1, 0.f);
      ck(cudaEventElapsedTime(&secs[0], ev[0], ev[1]), "elapsed");
      for (int k = 1; k <= ran; ++k) {
        // iteration k spans [ev[k], ev_end[k+1]] (the L2 flush, if any, precedes ev[k])
        ck(cudaEventElapsedTime(&secs[k], ev[k], ev_end[k + 1]), "elapsed");
        ctx->prof.iteration_ms += secs[k];
      }
      ctx->prof.iterations += ran;
      trace.mark("download");
      harvest_marks(ctx);
      for (auto& e : ev_end) cudaEventDestroy(e);
      for (int b = 0; b < B; ++b) {
        qoc_run_status_v1& s = status[b];
        std::memset(&s, 0, sizeof(s));
        s.aborted = stat[b] != 0;
        s.iterations_recorded = n_recs[b];
        if (stat[b] == 1)
          std::snprintf(s.abort_reason, sizeof(s.abort_reason),
                        "non-finite control after the task updates of iteration %d", abort_iter[b]);
        else if (stat[b] == 2)
          std::snprintf(s.abort_reason, sizeof(s.abort_reason), "non-finite boundary state at iteration %d",
                        abort_iter[b]);
        else if (stat[b] == 3)
          std::snprintf(s.abort_reason, sizeof(s.abort_reason), "non-finite boundary state during bootstrap");
        for (int k = 0; k < n_recs[b]; ++k) {
          const size_t r = (size_t)b * rec_cap + k;
          qoc_iter_record_v1& o = recs[r];
          o.iteration = k;
          o.objective = obj[r];
          o.has_error = (flags[r] & 1) != 0;
          o.error = err[r];
          o.has_exact_objective = (flags[r] & 2) != 0;
          o.exact_objective = exact[r];
          o.device_seconds = k <= ran ? 1e-3 * secs[k] : 0.0;
          o.reserved = 0;
        }
      }
    } catch (...) {
      cudaStreamSynchronize(st);
      harvest_marks(ctx);
      destroy_events();
      throw;
    }
    destroy_events();
  });
}

namespace {
// Single-task helper runs for the reference's helper entry points (L = 1 over the horizon).
void single_run(qoc_ctx* ctx, const qoc_problem_v1* p, const double* u, int mode, int form, bool need_prop,
                bool need_grad, DeviceProblem& dp, DeviceRun& dr) {
  const std::vector<int> node{0, p->steps};
  cudaStream_t st = ctx->stream;
  upload_problem(p, node, st, dp);
  alloc_run(dp, 1, node, need_prop, need_grad, st, dr);
  ck(cudaMemcpyAsync(dr.R.u, u, sizeof(double) * p->batch * p->steps * p->channels, cudaMemcpyHostToDevice, st),
     "u");
  Launcher launch{ctx};
  launch(set_single_tasks(dp.P, dr.R, st), "tasks");
  TaskArgs A{mode, form, 0, 1, 0.0};
  launch(task(dp.P, dr.R, A, 0, st), "task");
  ck(cudaStreamSynchronize(st), "run");
  check_flags(dr.R);
}
}  // namespace

int32_t qoc_propagate_final(qoc_ctx* ctx, const qoc_problem_v1* p, const double* u, double* states_out) {
  return guarded(ctx, [&] {
    validate_problem(p);
    if (!u || !states_out) fail(QOC_EINVAL, "null argument");
    DeviceProblem dp;
    dp.slots = fresh_slots(ctx->prob_slots);
    DeviceRun dr;
    dr.slots = fresh_slots(ctx->run_slots);
    single_run(ctx, p, u, M_FINAL, QOC_FORM_OVERLAP, false, false, dp, dr);
    ck(cudaMemcpy(states_out, dr.R.psi_end, sizeof(double2) * p->batch * dp.P.d, cudaMemcpyDeviceToHost), "out");
  });
}

int32_t qoc_objective_gradient(qoc_ctx* ctx, const qoc_problem_v1* p, const double* u, int32_t form,
                               int32_t naive, double* value_out, double* grad_out) {
  return guarded(ctx, [&] {
    validate_problem(p);
    if (!u) fail(QOC_EINVAL, "null argument");
    if (naive && p->kind != QOC_KIND_STRANG) naive = 0;
    DeviceProblem dp;
    dp.slots = fresh_slots(ctx->prob_slots);
    DeviceRun dr;
    dr.slots = fresh_slots(ctx->run_slots);
    int mode = M_ENTRY | (grad_out ? M_GRAD : 0) | (naive ? (1 << 10) : 0);
    single_run(ctx, p, u, mode, form, false, grad_out != nullptr, dp, dr);
    if (value_out) ck(cudaMemcpy(value_out, dr.R.entry, sizeof(double) * p->batch, cudaMemcpyDeviceToHost), "value");
    if (grad_out)
      ck(cudaMemcpy(grad_out, dr.R.grad, sizeof(double) * p->batch * p->steps * p->channels,
                    cudaMemcpyDeviceToHost),
         "grad");
  });
}

int32_t qoc_imaginary_time(qoc_ctx* ctx, const qoc_problem_v1* p, int32_t states, const double* u_frozen, double tau,
                           double tol, int32_t max_iter, int32_t n_lower, const double* lower, double* psi_io,
                           double* energy_out, int32_t* iterations_out) {
  return guarded(ctx, [&] {
    validate_problem(p);
    if (p->kind != QOC_KIND_STRANG) fail(QOC_ELOGIC, "imaginary-time stationary states need the split-step kind");
    if (states < 1 || !u_frozen || !psi_io || !energy_out || !iterations_out || n_lower < 0 || (n_lower && !lower))
      fail(QOC_EINVAL, "null or empty argument");
    if (!(tau > 0.0) || tol < 0.0 || max_iter < 0) fail(QOC_EINVAL, "imaginary_dt > 0, energy_tol >= 0, max_iterations >= 0");
    cudaStream_t st = ctx->stream;
    DeviceProblem dp;
    dp.slots = fresh_slots(ctx->prob_slots);
    qoc_problem_v1 q = *p;
    q.batch = 1;
    upload_problem(&q, std::vector<int>{0, q.steps}, st, dp);
    DeviceRun dr;
    dr.slots = fresh_slots(ctx->run_slots);
    const int d = p->dim;
    std::vector<double> hk(2 * (size_t)d);
    for (int i = 0; i < d; ++i) {
      hk[2 * i] = std::exp(-0.5 * tau * p->kinetic[i]);  // models.cpp:138-139
      hk[2 * i + 1] = 0.0;
    }
    double* kin = dr.alloc<double>(d);
    double2* half_kin = dr.alloc<double2>(d);
    double* uf = dr.alloc<double>(states);
    double2* psi = dr.alloc<double2>((size_t)states * d);
    double2* low = dr.alloc<double2>((size_t)states * std::max(1, n_lower) * d);
    double* en = dr.alloc<double>(states);
    int* it = dr.alloc<int>(states);
    ck(cudaMemcpyAsync(kin, p->kinetic, sizeof(double) * d, cudaMemcpyHostToDevice, st), "kinetic");
    ck(cudaMemcpyAsync(half_kin, hk.data(), sizeof(double2) * d, cudaMemcpyHostToDevice, st), "half kinetic");
    ck(cudaMemcpyAsync(uf, u_frozen, sizeof(double) * states, cudaMemcpyHostToDevice, st), "controls");
    ck(cudaMemcpyAsync(psi, psi_io, sizeof(double2) * states * d, cudaMemcpyHostToDevice, st), "states");
    if (n_lower)
      ck(cudaMemcpyAsync(low, lower, sizeof(double2) * states * n_lower * d, cudaMemcpyHostToDevice, st), "lower states");
    Launcher launch{ctx};
    launch(strang_imaginary_time(dp.P, states, uf, tau, tol, max_iter, n_lower, low, kin, half_kin, psi, en, it, st),
           "imaginary time");
    ck(cudaMemcpyAsync(psi_io, psi, sizeof(double2) * states * d, cudaMemcpyDeviceToHost, st), "states");
    ck(cudaMemcpyAsync(energy_out, en, sizeof(double) * states, cudaMemcpyDeviceToHost, st), "energy");
    ck(cudaMemcpyAsync(iterations_out, it, sizeof(int) * states, cudaMemcpyDeviceToHost, st), "iterations");
    ck(cudaStreamSynchronize(st), "imaginary time");
  });
}

int32_t qoc_assemble_propagator(qoc_ctx* ctx, const qoc_problem_v1* p, const double* u, double* prop_out) {
  return guarded(ctx, [&] {
    validate_problem(p);
    if (!u || !prop_out) fail(QOC_EINVAL, "null argument");
    if (p->kind == QOC_KIND_STRANG)
      fail(QOC_ELOGIC, "no dense one-step matrices to assemble for this propagator kind");
    if (p->kind == QOC_KIND_BITFLIP)
      fail(QOC_ELOGIC, "the bit-flip kind does not assemble d x d propagators; use QOC_KIND_DENSE");
    DeviceProblem dp;
    dp.slots = fresh_slots(ctx->prob_slots);
    DeviceRun dr;
    dr.slots = fresh_slots(ctx->run_slots);
    single_run(ctx, p, u, M_ASSEMBLE, QOC_FORM_TRACKING, true, false, dp, dr);
    const size_t B = p->batch, d = p->dim;
    std::vector<double2> rm(B * d * d);
    ck(cudaMemcpy(rm.data(), dr.R.prop, sizeof(double2) * rm.size(), cudaMemcpyDeviceToHost), "prop");
    for (size_t b = 0; b < B; ++b)  // row-major -> column-major (Eigen layout)
      for (size_t i = 0; i < d; ++i)
        for (size_t j = 0; j < d; ++j) {
          const double2 v = rm[b * d * d + i * d + j];
          prop_out[2 * (b * d * d + i + j * d)] = v.x;
          prop_out[2 * (b * d * d + i + j * d) + 1] = v.y;
        }
  });
}

}  // extern "C"
