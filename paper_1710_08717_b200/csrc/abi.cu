// extern "C" operator entry points (include/dla.h): host-side validation that
// mirrors the reference's ShapeError / alias sites, then stream-ordered
// launches.  Backward ops follow the reference's closed-form compositions
// (dl/adjoints.hpp) on the batched device kernels.
//
// Boundary contract:
//   * ownership -- every entry point takes (ws, ws_bytes): the caller's device
//     workspace, sized by dla_workspace_bytes(); all internal scratch is
//     carved from it (Arena, common.cuh).  No entry point allocates.
//   * threading -- no process-global mutable state on the compute path: the
//     SM count and kernel attributes are per device; the fork/join side
//     streams and events are per (device, caller stream) and locked for the
//     enqueue (fork_res).
#include <algorithm>
#include <atomic>
#include <map>
#include <memory>
#include <mutex>
#include <tuple>
#include <vector>

#include "common.cuh"
#include "ops.cuh"

namespace dlab {

// ------------------------------------------------------------ device state
namespace {
constexpr int kMaxDev = 64;
std::atomic<int> g_sms[kMaxDev];
}  // namespace

Ctx make_ctx(void* stream, int32_t* info, Arena* arena) {
  int dev = 0;
  cudaGetDevice(&dev);
  int sms = (dev >= 0 && dev < kMaxDev) ? g_sms[dev].load(std::memory_order_relaxed) : 0;
  if (sms == 0) {
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (dev >= 0 && dev < kMaxDev) g_sms[dev].store(sms, std::memory_order_relaxed);
  }
  Ctx c{reinterpret_cast<cudaStream_t>(stream), sms, info};
  c.arena = arena;
  return c;
}

void smem_opt_in(const void* func, size_t bytes) {
  static std::mutex mu;
  static std::map<std::pair<int, const void*>, size_t> done;
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lk(mu);
  size_t& cur = done[{dev, func}];
  if (bytes > cur) {
    cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
    cur = bytes;
  }
}

void ForkRes::grow(int64_t steps) {
  while ((int64_t)panel.size() < steps) {
    cudaEvent_t a, b;
    cudaEventCreateWithFlags(&a, cudaEventDisableTiming);
    cudaEventCreateWithFlags(&b, cudaEventDisableTiming);
    panel.push_back(a);
    done.push_back(b);
  }
}

ForkRes& fork_res(ForkKind kind, cudaStream_t caller) {
  static std::mutex mu;
  static std::map<std::tuple<int, int, cudaStream_t>, std::unique_ptr<ForkRes>> sets;
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lk(mu);
  auto& slot = sets[std::make_tuple(dev, (int)kind, caller)];
  if (!slot) {
    slot.reset(new ForkRes());
    ForkRes& f = *slot;
    // the critical chain gets the highest stream priority so that freed SMs
    // go to its panel CTAs before the bulk update's next tiles
    int lo = 0, hi = 0;
    cudaDeviceGetStreamPriorityRange(&lo, &hi);
    cudaStreamCreateWithPriority(&f.side, cudaStreamNonBlocking, lo);
    cudaStreamCreateWithPriority(&f.crit, cudaStreamNonBlocking, hi);
    f.prio_hi = hi;
    for (auto& e : f.ev) cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
  }
  return *slot;
}

// ------------------------------------------------------- instrumentation
static std::atomic<long long> g_launches{0};
static std::atomic<bool> g_prof{false};
static std::mutex g_prof_mu;
struct ProfRec {
  cudaEvent_t a, b;
  double flops;
};
static std::vector<ProfRec> g_prof_recs;
static std::vector<cudaEvent_t> g_event_pool;
static thread_local cudaEvent_t t_pending = nullptr;

void note_launch(int k) { g_launches.fetch_add(k, std::memory_order_relaxed); }
bool gemm_prof_on() { return g_prof.load(std::memory_order_relaxed); }

static cudaEvent_t take_event() {
  std::lock_guard<std::mutex> lk(g_prof_mu);
  if (!g_event_pool.empty()) {
    cudaEvent_t e = g_event_pool.back();
    g_event_pool.pop_back();
    return e;
  }
  cudaEvent_t e;
  cudaEventCreate(&e);
  return e;
}

void gemm_prof_begin(cudaStream_t s) {
  t_pending = take_event();
  cudaEventRecord(t_pending, s);
}

void gemm_prof_cancel() {  // a begin whose launch did not happen
  if (!t_pending) return;
  std::lock_guard<std::mutex> lk(g_prof_mu);
  g_event_pool.push_back(t_pending);
  t_pending = nullptr;
}

void gemm_prof_end(cudaStream_t s, double flops) {
  cudaEvent_t e = take_event();
  cudaEventRecord(e, s);
  std::lock_guard<std::mutex> lk(g_prof_mu);
  g_prof_recs.push_back(ProfRec{t_pending, e, flops});
}

namespace {

bool overlap(const void* a, size_t abytes, const void* b, size_t bbytes) {
  if (!a || !b || abytes == 0 || bbytes == 0) return false;
  const char* pa = static_cast<const char*>(a);
  const char* pb = static_cast<const char*>(b);
  return pa < pb + bbytes && pb < pa + abytes;
}

template <typename T>
size_t bytes(int64_t batch, int64_t r, int64_t c) {
  return sizeof(T) * (size_t)batch * (size_t)r * (size_t)c;
}

dla_status reset_info(const Ctx& c, int64_t batch) {
  if (c.info && batch > 0)
    if (cudaMemsetAsync(c.info, 0, sizeof(int32_t) * batch, c.stream) != cudaSuccess) return DLA_ERR_CUDA;
  return DLA_OK;
}

bool bad_dims(int64_t batch, int64_t a, int64_t b = 0, int64_t c = 0) {
  return batch < 0 || a < 0 || b < 0 || c < 0 || a > 0xFFFFFF || b > 0x7FFFFFFF;
}

template <typename T>
MatB<const T> cpk(const T* p, int64_t r, int64_t c) {
  return MatB<const T>{p, c, r * c};
}
template <typename T>
MatB<T> pk(T* p, int64_t r, int64_t c) {
  return MatB<T>{p, c, r * c};
}
template <typename T>
MatB<const T> C_(MatB<T> m) {
  return MatB<const T>{m.p, m.ld, m.bs};
}

// =================================================================== ops
// Each op: validation (host, synchronous), then `<op>_run(cx, ...)` on a Ctx
// whose arena is the caller's workspace; `ws_<op>` is the workspace mirror
// of the same run (dla_workspace_bytes).

// ------------------------------------------------------------------- gemm
template <typename T>
dla_status gemm_run(const Ctx& cx, int64_t batch, int64_t m, int64_t n, int64_t k, T* c, const T* a, const T* b,
                    int ta, int tb, T alpha, T beta) {
  if (beta == T(0)) {  // the reference zero-fills C (gemm_accum accumulate=false)
    if (k == 0 || alpha == T(0)) {
      return cudaMemsetAsync(c, 0, bytes<T>(batch, m, n), cx.stream) == cudaSuccess ? DLA_OK : DLA_ERR_CUDA;
    }
  }
  return gemm<T>(cx, batch, m, n, k, alpha, cpk(a, ta ? k : m, ta ? m : k), ta, cpk(b, tb ? n : k, tb ? k : n),
                 tb, beta, pk(c, m, n));
}

template <typename T>
dla_status gemm_fwd(const Ctx& cx, int64_t batch, int64_t m, int64_t n, int64_t k, T* c, const T* a, const T* b,
                    int ta, int tb, T alpha, T beta) {
  if (batch < 0 || m < 0 || n < 0 || k < 0) return DLA_ERR_SHAPE;
  if (overlap(c, bytes<T>(batch, m, n), a, bytes<T>(batch, m, k)) ||
      overlap(c, bytes<T>(batch, m, n), b, bytes<T>(batch, k, n)))
    return DLA_ERR_ALIAS;
  return gemm_run<T>(cx, batch, m, n, k, c, a, b, ta, tb, alpha, beta);
}

template <typename T>
size_t ws_gemm_bwd(int64_t batch, int64_t m, int64_t n, int64_t k, int ta, int tb) {
  size_t w = !ta ? ws_gemm<T>(batch, m, k, n) : ws_gemm<T>(batch, k, m, n);
  w += !tb ? ws_gemm<T>(batch, k, n, m) : ws_gemm<T>(batch, n, k, m);
  return w;
}

template <typename T>
dla_status gemm_bwd(const Ctx& cx, int64_t batch, int64_t m, int64_t n, int64_t k, T* abar, T* bbar, T* cbar_io,
                    const T* a, const T* b, int ta, int tb, T alpha, T beta, bool has_c) {
  if (batch < 0 || m < 0 || n < 0 || k < 0) return DLA_ERR_SHAPE;
  const size_t asz = bytes<T>(batch, m, k), bsz = bytes<T>(batch, k, n), csz = bytes<T>(batch, m, n);
  if (overlap(abar, asz, cbar_io, csz) || overlap(abar, asz, b, bsz) || overlap(bbar, bsz, cbar_io, csz) ||
      overlap(bbar, bsz, a, asz) || overlap(abar, asz, bbar, bsz))
    return DLA_ERR_ALIAS;
  // dl/adjoints.hpp:39-48
  if (!ta) DLAB_TRY(gemm_run<T>(cx, batch, m, k, n, abar, cbar_io, b, 0, !tb, alpha, T(0)));
  else DLAB_TRY(gemm_run<T>(cx, batch, k, m, n, abar, b, cbar_io, tb, 1, alpha, T(0)));
  if (!tb) DLAB_TRY(gemm_run<T>(cx, batch, k, n, m, bbar, a, cbar_io, !ta, 0, alpha, T(0)));
  else DLAB_TRY(gemm_run<T>(cx, batch, n, k, m, bbar, cbar_io, a, 1, ta, alpha, T(0)));
  if (has_c) {
    if (beta == T(0))
      return cudaMemsetAsync(cbar_io, 0, csz, cx.stream) == cudaSuccess ? DLA_OK : DLA_ERR_CUDA;
    return ew_scale<T>(cx, batch, m, n, pk(cbar_io, m, n), beta);
  }
  return DLA_OK;
}

// ------------------------------------------------------------------- syrk
template <typename T>
size_t ws_syrk_bwd(int64_t batch, int64_t n, int64_t k, int ta) {
  return 2 * (!ta ? ws_gemm<T>(batch, n, k, n) : ws_gemm<T>(batch, k, n, n));
}

template <typename T>
dla_status syrk_fwd(const Ctx& cx, int64_t batch, int64_t n, int64_t k, T* bo, const T* a, int ta, T alpha) {
  if (batch < 0 || n < 0 || k < 0) return DLA_ERR_SHAPE;
  if (overlap(bo, bytes<T>(batch, n, n), a, bytes<T>(batch, n, k))) return DLA_ERR_ALIAS;
  if (batch * n == 0) return DLA_OK;
  if (k == 0 || alpha == T(0))
    return cudaMemsetAsync(bo, 0, bytes<T>(batch, n, n), cx.stream) == cudaSuccess ? DLA_OK : DLA_ERR_CUDA;
  MatB<const T> av = cpk(a, ta ? k : n, ta ? n : k);
  bool tma = false;
  if constexpr (sizeof(T) == 8) {  // A A^T (f64): the TMA-fed persistent update kernel (syrk_tma.cu)
    MatB<const double> ad{reinterpret_cast<const double*>(av.p), av.ld, av.bs};
    MatB<double> bd{reinterpret_cast<double*>(bo), n, n * n};
    if (!ta && syrk_tma_eligible(n, k, ad, bd, batch)) {
      DLAB_TRY(syrk_tma(cx, batch, n, k, (double)alpha, ad, 0.0, bd, 0));
      tma = true;
    }
  }
  if (!tma) DLAB_TRY(gemm<T>(cx, batch, n, n, k, alpha, av, ta, av, !ta, T(0), pk(bo, n, n), MASK_LOWER));
  return ew_square<T>(cx, batch, n, pk(bo, n, n), /*copyltu*/ 2);
}

template <typename T>
dla_status syrk_bwd(const Ctx& cx, int64_t batch, int64_t n, int64_t k, T* abar, const T* bbar, const T* a, int ta,
                    T alpha) {
  if (batch < 0 || n < 0 || k < 0) return DLA_ERR_SHAPE;
  const size_t asz = bytes<T>(batch, n, k);
  if (overlap(abar, asz, bbar, bytes<T>(batch, n, n)) || overlap(abar, asz, a, asz)) return DLA_ERR_ALIAS;
  // dl/adjoints.hpp:71-77
  if (!ta) {
    DLAB_TRY(gemm_run<T>(cx, batch, n, k, n, abar, bbar, a, 0, 0, alpha, T(0)));
    DLAB_TRY(gemm_run<T>(cx, batch, n, k, n, abar, bbar, a, 1, 0, alpha, T(1)));
  } else {
    DLAB_TRY(gemm_run<T>(cx, batch, k, n, n, abar, a, bbar, 0, 0, alpha, T(0)));
    DLAB_TRY(gemm_run<T>(cx, batch, k, n, n, abar, a, bbar, 0, 1, alpha, T(1)));
  }
  return DLA_OK;
}

// ------------------------------------------------------------ trmm / trsm
template <typename T>
dla_status trmm_fwd(const Ctx& cx, int64_t batch, int64_t m, int64_t n, const T* t, T* x, int right, int trans,
                    int lower, T alpha) {
  if (bad_dims(batch, m, n)) return DLA_ERR_SHAPE;
  const int64_t nt = right ? n : m;
  if (overlap(x, bytes<T>(batch, m, n), t, bytes<T>(batch, nt, nt))) return DLA_ERR_ALIAS;
  return trmm<T>(cx, batch, m, n, cpk(t, nt, nt), pk(x, m, n), right, trans, lower, alpha);
}

// Out-of-place trmm: y = alpha op(T) x / alpha x op(T), x and t unchanged (the
// reference's functional trmm, dl/blas.hpp:202-291).  For nt >= 128 one
// triangular GEMM from x into y (no copy, no in-place tile constraint);
// otherwise a copy and the in-place operator.
template <typename T>
dla_status trmm_into(const Ctx& cx, int64_t batch, int64_t m, int64_t n, const T* t, const T* x, T* y, int right,
                     int trans, int lower, T alpha) {
  if (bad_dims(batch, m, n)) return DLA_ERR_SHAPE;
  const int64_t nt = right ? n : m;
  const size_t ysz = bytes<T>(batch, m, n);
  if (overlap(y, ysz, t, bytes<T>(batch, nt, nt)) || overlap(y, ysz, x, ysz)) return DLA_ERR_ALIAS;
  if (batch * m * n == 0) return DLA_OK;
  if (nt >= 128) {
    const int tri = (lower != trans) ? TRI_LOWER : TRI_UPPER;  // of op(T)
    if (!right)
      return gemm<T>(cx, batch, m, n, m, alpha, cpk(t, nt, nt), trans != 0, cpk(x, m, n), false, T(0), pk(y, m, n),
                     MASK_FULL, nullptr, tri, TRI_NONE);
    return gemm<T>(cx, batch, m, n, n, alpha, cpk(x, m, n), false, cpk(t, nt, nt), trans != 0, T(0), pk(y, m, n),
                   MASK_FULL, nullptr, TRI_NONE, tri);
  }
  DLAB_TRY(ew_copy<T>(cx, batch, m, n, cpk(x, m, n), pk(y, m, n)));
  return trmm<T>(cx, batch, m, n, cpk(t, nt, nt), pk(y, m, n), right, trans, lower, alpha);
}

template <typename T>
dla_status trsm_fwd(const Ctx& cx, int64_t batch, int64_t m, int64_t n, const T* t, T* x, int right, int trans,
                    int lower, T alpha) {
  if (bad_dims(batch, m, n)) return DLA_ERR_SHAPE;
  const int64_t nt = right ? n : m;
  if (overlap(x, bytes<T>(batch, m, n), t, bytes<T>(batch, nt, nt))) return DLA_ERR_ALIAS;
  DLAB_TRY(reset_info(cx, batch));
  return trsm<T>(cx, batch, m, n, cpk(t, nt, nt), pk(x, m, n), right, trans, lower, alpha, /*check_diag*/ true);
}

template <typename T>
size_t ws_trmm_bwd(int64_t batch, int64_t m, int64_t n, int right) {
  return (right ? ws_gemm<T>(batch, n, n, m) : ws_gemm<T>(batch, m, m, n)) + ws_trmm<T>(batch, m, n, right);
}

template <typename T>
dla_status trmm_bwd(const Ctx& cx, int64_t batch, int64_t m, int64_t n, T* abar, T* tbar, const T* bbar,
                    const T* t, const T* a, int right, int trans, int lower, T alpha) {
  if (bad_dims(batch, m, n)) return DLA_ERR_SHAPE;
  const int64_t nt = right ? n : m;
  const size_t xsz = bytes<T>(batch, m, n), tsz = bytes<T>(batch, nt, nt);
  if (overlap(tbar, tsz, bbar, xsz) || overlap(tbar, tsz, a, xsz) || overlap(abar, xsz, t, tsz) ||
      overlap(abar, xsz, tbar, tsz) || (abar != bbar && overlap(abar, xsz, bbar, xsz)))
    return DLA_ERR_ALIAS;
  if (batch * m * n == 0) {
    if (batch * nt > 0 && cudaMemsetAsync(tbar, 0, tsz, cx.stream) != cudaSuccess) return DLA_ERR_CUDA;
    return DLA_OK;
  }
  MatB<T> tb = pk(tbar, nt, nt);
  const int mask = lower ? MASK_LOWER : MASK_UPPER;
  auto X = [&](const T* p) { return cpk(p, m, n); };
  // dl/adjoints.hpp:98-107, computed on the kept triangle only
  if (!right && !trans) DLAB_TRY(gemm<T>(cx, batch, m, m, n, alpha, X(bbar), false, X(a), true, T(0), tb, mask));
  else if (!right && trans) DLAB_TRY(gemm<T>(cx, batch, m, m, n, alpha, X(a), false, X(bbar), true, T(0), tb, mask));
  else if (right && !trans) DLAB_TRY(gemm<T>(cx, batch, n, n, m, alpha, X(a), true, X(bbar), false, T(0), tb, mask));
  else DLAB_TRY(gemm<T>(cx, batch, n, n, m, alpha, X(bbar), true, X(a), false, T(0), tb, mask));
  DLAB_TRY(ew_square<T>(cx, batch, nt, tb, lower ? 0 : 1));
  if (abar != bbar && nt >= 128) {
    // Abar = alpha op(T)^T Bbar (or Bbar op(T)^T) as ONE triangular GEMM from
    // Bbar into Abar: no copy pass, no in-place tile constraint
    const int tri = (lower != !trans) ? TRI_LOWER : TRI_UPPER;  // of op(T) with trans flipped
    if (!right)
      return gemm<T>(cx, batch, m, n, m, alpha, cpk(t, nt, nt), !trans, X(bbar), false, T(0), pk(abar, m, n),
                     MASK_FULL, cx.info, tri, TRI_NONE);
    return gemm<T>(cx, batch, m, n, n, alpha, X(bbar), false, cpk(t, nt, nt), !trans, T(0), pk(abar, m, n), MASK_FULL,
                   cx.info, TRI_NONE, tri);
  }
  DLAB_TRY(ew_copy<T>(cx, batch, m, n, cpk(bbar, m, n), pk(abar, m, n)));
  return trmm<T>(cx, batch, m, n, cpk(t, nt, nt), pk(abar, m, n), right, !trans, lower, alpha);
}

template <typename T>
size_t ws_trsm_bwd(int64_t batch, int64_t m, int64_t n, int right) {
  return ws_trsm<T>(batch, m, n, right) + (right ? ws_gemm<T>(batch, n, n, m) : ws_gemm<T>(batch, m, m, n));
}

template <typename T>
dla_status trsm_bwd(const Ctx& cx, int64_t batch, int64_t m, int64_t n, T* abar, T* tbar, const T* bbar,
                    const T* t, const T* b, int right, int trans, int lower, T alpha) {
  if (bad_dims(batch, m, n)) return DLA_ERR_SHAPE;
  const int64_t nt = right ? n : m;
  const size_t xsz = bytes<T>(batch, m, n), tsz = bytes<T>(batch, nt, nt);
  if (overlap(tbar, tsz, bbar, xsz) || overlap(tbar, tsz, b, xsz) || overlap(abar, xsz, t, tsz) ||
      overlap(abar, xsz, tbar, tsz) || overlap(abar, xsz, b, xsz) ||
      (abar != bbar && overlap(abar, xsz, bbar, xsz)))
    return DLA_ERR_ALIAS;
  if (batch * m * n == 0) {
    if (batch * nt > 0 && cudaMemsetAsync(tbar, 0, tsz, cx.stream) != cudaSuccess) return DLA_ERR_CUDA;
    return DLA_OK;
  }
  // dl/adjoints.hpp:136-152: S = op(T)^{-T} Bbar in abar, then Tbar, then alpha.
  DLAB_TRY(ew_copy<T>(cx, batch, m, n, cpk(bbar, m, n), pk(abar, m, n)));
  DLAB_TRY(trsm<T>(cx, batch, m, n, cpk(t, nt, nt), pk(abar, m, n), right, !trans, lower, T(1)));
  MatB<T> tb = pk(tbar, nt, nt);
  const int mask = lower ? MASK_LOWER : MASK_UPPER;
  auto X = [&](const T* p) { return cpk(p, m, n); };
  const T* s = abar;
  {  // rank <= 8 (narrow solves): Tbar written whole, zeros outside the mask, in one pass
    dla_status st = DLA_OK;
    bool done = false;
    if (!right) {
      done = !trans ? outer_tri<T>(cx, batch, m, m, n, T(-1), X(s), false, X(b), true, tb, mask, nullptr, &st)
                    : outer_tri<T>(cx, batch, m, m, n, T(-1), X(b), false, X(s), true, tb, mask, nullptr, &st);
    } else {
      done = !trans ? outer_tri<T>(cx, batch, n, n, m, T(-1), X(b), true, X(s), false, tb, mask, nullptr, &st)
                    : outer_tri<T>(cx, batch, n, n, m, T(-1), X(s), true, X(b), false, tb, mask, nullptr, &st);
    }
    if (done) {
      if (st != DLA_OK) return st;
      return ew_scale<T>(cx, batch, m, n, pk(abar, m, n), alpha);
    }
  }
  if (!right) {
    if (!trans) DLAB_TRY(gemm<T>(cx, batch, m, m, n, T(-1), X(s), false, X(b), true, T(0), tb, mask));
    else DLAB_TRY(gemm<T>(cx, batch, m, m, n, T(-1), X(b), false, X(s), true, T(0), tb, mask));
  } else {
    if (!trans) DLAB_TRY(gemm<T>(cx, batch, n, n, m, T(-1), X(b), true, X(s), false, T(0), tb, mask));
    else DLAB_TRY(gemm<T>(cx, batch, n, n, m, T(-1), X(s), true, X(b), false, T(0), tb, mask));
  }
  DLAB_TRY(ew_square<T>(cx, batch, nt, tb, lower ? 0 : 1));
  return ew_scale<T>(cx, batch, m, n, pk(abar, m, n), alpha);
}

// ------------------------------------------------------------ potrf / potri
template <typename T>
size_t ws_potrf_fwd(int64_t batch, int64_t n) {
  return potrf_fwd_small_eligible<T>(n) ? 0 : ws_check_symmetric(batch) + ws_potrf_lower<T>(batch, n);
}

template <typename T>
dla_status potrf_fwd(const Ctx& cx, int64_t batch, int64_t n, T* a, int lower) {
  if (bad_dims(batch, n)) return DLA_ERR_SHAPE;
  DLAB_TRY(reset_info(cx, batch));
  if (batch * n == 0) return DLA_OK;
  if (potrf_fwd_small_eligible<T>(n)) return potrf_small<T>(cx, batch, n, pk(a, n, n), lower);
  DLAB_TRY(check_symmetric<T>(cx, batch, n, cpk(a, n, n), cx.info));
  DLAB_TRY(potrf_lower<T>(cx, batch, n, pk(a, n, n)));
  if (!lower) DLAB_TRY(ew_square<T>(cx, batch, n, pk(a, n, n), /*transpose*/ 5, T(1), cx.info));
  return DLA_OK;
}

template <typename T>
size_t ws_potrf_bwd(int64_t batch, int64_t n) {
  if (batch * n == 0 || potrf_small_eligible<T>(n)) return 0;
  if (inv_pad<T>(n)) return ws_potrf_bwd_inv<T>(batch, n);
  return ws_trmm<T>(batch, n, n, false) + ws_trsm<T>(batch, n, n, false) + ws_trsm<T>(batch, n, n, true);
}

template <typename T>
dla_status potrf_bwd(const Ctx& cx, int64_t batch, int64_t n, T* abar, const T* lbar, const T* l, int lower) {
  if (bad_dims(batch, n)) return DLA_ERR_SHAPE;
  const size_t sz = bytes<T>(batch, n, n);
  if (overlap(abar, sz, l, sz) || (abar != lbar && overlap(abar, sz, lbar, sz))) return DLA_ERR_ALIAS;
  if (batch * n == 0) return DLA_OK;
  if (potrf_small_eligible<T>(n)) return potrf_bwd_small<T>(cx, batch, n, pk(abar, n, n), cpk(lbar, n, n),
                                                            cpk(l, n, n), lower);
  if (inv_pad<T>(n)) return potrf_bwd_inv<T>(cx, batch, n, pk(abar, n, n), cpk(lbar, n, n), cpk(l, n, n), lower);
  MatB<T> ab = pk(abar, n, n);
  MatB<const T> lv = cpk(l, n, n);
  DLAB_TRY(ew_copy<T>(cx, batch, n, n, cpk(lbar, n, n), ab));
  if (lower) {  // dl/adjoints.hpp:179-182
    DLAB_TRY(trmm<T>(cx, batch, n, n, lv, ab, false, true, true, T(1)));
    DLAB_TRY(ew_square<T>(cx, batch, n, ab, /*copyltu*/ 2));
    DLAB_TRY(trsm<T>(cx, batch, n, n, lv, ab, false, true, true, T(1)));
    DLAB_TRY(trsm<T>(cx, batch, n, n, lv, ab, true, false, true, T(1)));
  } else {      // dl/adjoints.hpp:184-187
    DLAB_TRY(trmm<T>(cx, batch, n, n, lv, ab, true, true, false, T(1)));
    DLAB_TRY(ew_square<T>(cx, batch, n, ab, /*copyutl*/ 3));
    DLAB_TRY(trsm<T>(cx, batch, n, n, lv, ab, false, false, false, T(1)));
    DLAB_TRY(trsm<T>(cx, batch, n, n, lv, ab, true, true, false, T(1)));
  }
  return ew_square<T>(cx, batch, n, ab, /*scaled sym*/ 6, T(0.5));
}

template <typename T>
dla_status potri_fwd(const Ctx& cx, int64_t batch, int64_t n, T* a, int lower) {
  if (bad_dims(batch, n)) return DLA_ERR_SHAPE;
  DLAB_TRY(reset_info(cx, batch));
  if (batch * n == 0) return DLA_OK;
  MatB<T> av = pk(a, n, n);
  if (!lower) DLAB_TRY(ew_square<T>(cx, batch, n, av, /*transpose*/ 5));
  DLAB_TRY(check_zero_diag<T>(cx, batch, n, C_(av), cx.info));
  return potri_lower<T>(cx, batch, n, av);
}

// Out-of-place potri: b = (L L^T)^{-1} from the factor l (unchanged), the
// reference's functional potri (dl/cholesky.hpp:141-147).  fp64
// 64 < n <= 128: one fused launch reading l and writing b (k_trtri128);
// otherwise a copy and the in-place operator.
template <typename T>
dla_status potri_into(const Ctx& cx, int64_t batch, int64_t n, const T* l, T* b, int lower) {
  if (bad_dims(batch, n)) return DLA_ERR_SHAPE;
  const size_t sz = bytes<T>(batch, n, n);
  if (overlap(l, sz, b, sz)) return DLA_ERR_ALIAS;
  if constexpr (sizeof(T) == 8) {
    if (potri_fused_eligible<T>(n)) {
      DLAB_TRY(reset_info(cx, batch));
      if (batch * n == 0) return DLA_OK;
      DLAB_TRY(check_zero_diag<T>(cx, batch, n, cpk(l, n, n), cx.info));
      return potri128_into(cx, batch, n, cpk(l, n, n), lower == 0, pk(b, n, n));
    }
  }
  if (batch * n > 0) DLAB_TRY(ew_copy<T>(cx, batch, n, n, cpk(l, n, n), pk(b, n, n)));
  return potri_fwd<T>(cx, batch, n, b, lower);
}

template <typename T>
size_t ws_potri_bwd(int64_t batch, int64_t n, int lower) {
  if (lower && inv_eligible<T>(n))
    return 2 * carve_bound(bytes<T>(batch, n, n)) + ws_gemm<T>(batch, n, n, n) + ws_trsm_inv_from<T>(batch, n, n, true);
  return carve_bound(bytes<T>(batch, n, n)) + ws_gemm<T>(batch, n, n, n) + ws_trsm<T>(batch, n, n, lower != 0);
}

template <typename T>
dla_status potri_bwd(const Ctx& cx, int64_t batch, int64_t n, T* lbar, const T* bbar, const T* l, const T* b,
                     int lower) {
  if (bad_dims(batch, n)) return DLA_ERR_SHAPE;
  const size_t sz = bytes<T>(batch, n, n);
  if (overlap(lbar, sz, bbar, sz) || overlap(lbar, sz, l, sz) || overlap(lbar, sz, b, sz)) return DLA_ERR_ALIAS;
  if (batch * n == 0) return DLA_OK;
  MatB<T> lb = pk(lbar, n, n);
  MatB<const T> bv = cpk(b, n, n), bb = cpk(bbar, n, n), lv = cpk(l, n, n);
  // The reference forms B Bbar + B Bbar^T as two accumulated products
  // (dl/adjoints.hpp:211-212); here Bbar + Bbar^T is formed once (one n^2
  // pass) and multiplied once: half the O(n^3) work, same value.
  DLAB_SCRATCH(ws, cx, bytes<T>(batch, n, n));
  MatB<T> sb = pk(ws.as<T>(), n, n);
  DLAB_TRY(ew_add_transpose<T>(cx, batch, n, bb, sb));
  if (lower && inv_eligible<T>(n)) {
    // the right solve by the explicit inverse straight from P = B (Bbar +
    // Bbar^T) into Lbar: P in scratch, one GEMM, no copy back
    DLAB_SCRATCH(ps, cx, bytes<T>(batch, n, n));
    MatB<T> pb = pk(ps.as<T>(), n, n);
    DLAB_TRY(gemm<T>(cx, batch, n, n, n, T(1), bv, false, C_(sb), false, T(0), pb));
    DLAB_TRY(trsm_inv_from<T>(cx, batch, n, n, lv, C_(pb), lb, true, true, true, T(-1)));
    return ew_square<T>(cx, batch, n, lb, /*tril*/ 0);
  }
  if (lower) {  // dl/adjoints.hpp:211-215
    DLAB_TRY(gemm<T>(cx, batch, n, n, n, T(1), bv, false, C_(sb), false, T(0), lb));
    DLAB_TRY(trsm<T>(cx, batch, n, n, lv, lb, true, true, true, T(-1)));
    return ew_square<T>(cx, batch, n, lb, /*tril*/ 0);
  }
  // dl/adjoints.hpp:217-221
  DLAB_TRY(gemm<T>(cx, batch, n, n, n, T(1), C_(sb), false, bv, false, T(0), lb));
  DLAB_TRY(trsm<T>(cx, batch, n, n, lv, lb, false, true, false, T(-1)));
  return ew_square<T>(cx, batch, n, lb, /*triu*/ 1);
}

// ------------------------------------------------------------- sumlogdiag
template <typename T>
dla_status sld_fwd(const Ctx& cx, int64_t batch, int64_t n, T* out, const T* a) {
  if (bad_dims(batch, n)) return DLA_ERR_SHAPE;
  return sumlogdiag_fwd<T>(cx, batch, n, out, cpk(a, n, n));
}

template <typename T>
dla_status sld_bwd(const Ctx& cx, int64_t batch, int64_t n, T* abar, const T* g, const T* a, int accumulate) {
  if (bad_dims(batch, n)) return DLA_ERR_SHAPE;
  const size_t sz = bytes<T>(batch, n, n);
  if (overlap(abar, sz, a, sz)) return DLA_ERR_ALIAS;
  return sumlogdiag_bwd<T>(cx, batch, n, pk(abar, n, n), g, cpk(a, n, n), accumulate != 0);
}

// --------------------------------------------------------------- gelqf
template <typename T>
size_t ws_gelqf_fwd(int64_t batch, int64_t m, int64_t n) {
  if (sizeof(T) == 8 && gelqf_cqr_eligible(m, n)) return ws_gelqf_cqr(batch, m, n);
  // the panel GEMMs of gelqf_blocked have N or K = 32: never on the carving route
  return carve_bound(gelqf_ws_bytes<T>(batch, m, n, false));
}

template <typename T>
dla_status gelqf_fwd_abi(const Ctx& cx, int64_t batch, int64_t m, int64_t n, T* q, T* l) {
  if (bad_dims(batch, m, n) || m > n) return DLA_ERR_SHAPE;
  if (overlap(q, bytes<T>(batch, m, n), l, bytes<T>(batch, m, m))) return DLA_ERR_ALIAS;
  DLAB_TRY(reset_info(cx, batch));
  if (batch * m == 0) return DLA_OK;
  if constexpr (sizeof(T) == 8) {
    if (gelqf_cqr_eligible(m, n))
      return gelqf_cqr(cx, batch, m, n, reinterpret_cast<double*>(q), reinterpret_cast<double*>(l));
  }
  DLAB_SCRATCH(ws, cx, gelqf_ws_bytes<T>(batch, m, n, false));
  return gelqf_fwd<T>(cx, batch, m, n, q, l, ws.p);
}

template <typename T>
size_t ws_gelqf_bwd(int64_t batch, int64_t m, int64_t n) {
  return carve_bound(gelqf_ws_bytes<T>(batch, m, n, true)) + ws_trmm<T>(batch, m, m, false) +
         ws_gemm<T>(batch, m, m, n) + ws_gemm<T>(batch, m, n, m) + ws_trsm<T>(batch, m, n, false);
}

template <typename T>
dla_status gelqf_bwd_abi(const Ctx& cx, int64_t batch, int64_t m, int64_t n, T* abar, const T* qbar, const T* lbar,
                         const T* q, const T* l) {
  if (bad_dims(batch, m, n) || m > n) return DLA_ERR_SHAPE;
  const size_t asz = bytes<T>(batch, m, n);
  if (overlap(abar, asz, q, asz) || overlap(abar, asz, l, bytes<T>(batch, m, m)) ||
      overlap(abar, asz, lbar, bytes<T>(batch, m, m)) || (abar != qbar && overlap(abar, asz, qbar, asz)))
    return DLA_ERR_ALIAS;
  if (batch * m == 0) return DLA_OK;
  DLAB_SCRATCH(ws, cx, gelqf_ws_bytes<T>(batch, m, n, true));
  MatB<T> wv = pk(ws.as<T>(), m, m);
  MatB<const T> lv = cpk(l, m, m), qv = cpk(q, m, n);
  // dl/adjoints.hpp:243-251
  DLAB_TRY(ew_copy<T>(cx, batch, m, m, cpk(lbar, m, m), wv));
  DLAB_TRY(trmm<T>(cx, batch, m, m, lv, wv, false, true, true, T(1)));
  DLAB_TRY(gemm<T>(cx, batch, m, m, n, T(-1), cpk(qbar, m, n), false, qv, true, T(1), wv));
  DLAB_TRY(ew_square<T>(cx, batch, m, wv, /*copyltu*/ 2));
  DLAB_TRY(ew_copy<T>(cx, batch, m, n, cpk(qbar, m, n), pk(abar, m, n)));
  DLAB_TRY(gemm<T>(cx, batch, m, n, m, T(1), C_(wv), false, qv, false, T(1), pk(abar, m, n)));
  return trsm<T>(cx, batch, m, n, lv, pk(abar, m, n), false, true, true, T(1));
}

// --------------------------------------------------------------- syevd
template <typename T>
dla_status syevd_fwd_abi(const Ctx& cx, int64_t batch, int64_t n, T* u, T* lambda) {
  if (bad_dims(batch, n)) return DLA_ERR_SHAPE;
  if (overlap(u, bytes<T>(batch, n, n), lambda, bytes<T>(batch, n, 1))) return DLA_ERR_ALIAS;
  DLAB_TRY(reset_info(cx, batch));
  if (batch * n == 0) return DLA_OK;
  DLAB_SCRATCH(ws, cx, syevd_ws_bytes<T>(batch, n, false));
  return syevd_fwd<T>(cx, batch, n, u, lambda, ws.p);
}

template <typename T>
size_t ws_syevd_bwd(int64_t batch, int64_t n) {
  return carve_bound(syevd_ws_bytes<T>(batch, n, true)) + 3 * ws_gemm<T>(batch, n, n, n);
}

template <typename T>
dla_status syevd_bwd_abi(const Ctx& cx, int64_t batch, int64_t n, T* abar, const T* ubar, const T* lambdabar,
                         const T* u, const T* lambda, T eps_gap) {
  if (bad_dims(batch, n)) return DLA_ERR_SHAPE;
  const size_t sz = bytes<T>(batch, n, n);
  if (overlap(abar, sz, ubar, sz) || overlap(abar, sz, u, sz)) return DLA_ERR_ALIAS;
  if (!(eps_gap > T(0))) return DLA_ERR_INVALID;
  if (batch * n == 0) return DLA_OK;
  DLAB_SCRATCH(ws, cx, syevd_ws_bytes<T>(batch, n, true));
  MatB<T> w = pk(ws.as<T>(), n, n);
  MatB<const T> uv = cpk(u, n, n);
  // dl/adjoints.hpp:277-294
  DLAB_TRY(gemm<T>(cx, batch, n, n, n, T(1), cpk(ubar, n, n), false, uv, true, T(0), w));
  DLAB_TRY(syevd_gap_kernel<T>(cx, batch, n, w, lambdabar, lambda, eps_gap));
  DLAB_TRY(gemm<T>(cx, batch, n, n, n, T(1), uv, true, C_(w), false, T(0), pk(abar, n, n)));
  DLAB_TRY(gemm<T>(cx, batch, n, n, n, T(1), cpk(abar, n, n), false, uv, false, T(0), w));
  return ew_sym_into<T>(cx, batch, n, C_(w), pk(abar, n, n));
}

// --------------------------------------------------------------- gesvd
template <typename T>
dla_status gesvd_fwd_abi(const Ctx& cx, int64_t batch, int64_t m, int64_t n, T* v, T* u, T* lambda) {
  if (bad_dims(batch, m, n) || m > n) return DLA_ERR_SHAPE;
  const size_t vsz = bytes<T>(batch, m, n), usz = bytes<T>(batch, m, m), lsz = bytes<T>(batch, m, 1);
  if (overlap(v, vsz, u, usz) || overlap(v, vsz, lambda, lsz) || overlap(u, usz, lambda, lsz)) return DLA_ERR_ALIAS;
  DLAB_TRY(reset_info(cx, batch));
  if (batch * m == 0) return DLA_OK;
  return gesvd_fwd<T>(cx, batch, m, n, v, u, lambda);
}

template <typename T>
dla_status gesvd_bwd_abi(const Ctx& cx, int64_t batch, int64_t m, int64_t n, T* abar, const T* ubar,
                         const T* lambdabar, const T* vbar, const T* u, const T* lambda, const T* v, T eps_gap) {
  if (bad_dims(batch, m, n) || m > n) return DLA_ERR_SHAPE;
  const size_t asz = bytes<T>(batch, m, n), usz = bytes<T>(batch, m, m), lsz = bytes<T>(batch, m, 1);
  if (overlap(abar, asz, ubar, usz) || overlap(abar, asz, lambdabar, lsz) || overlap(abar, asz, u, usz) ||
      overlap(abar, asz, lambda, lsz) || overlap(abar, asz, v, asz) || (abar != vbar && overlap(abar, asz, vbar, asz)))
    return DLA_ERR_ALIAS;
  if (!(eps_gap > T(0))) return DLA_ERR_INVALID;
  DLAB_TRY(reset_info(cx, batch));
  if (batch * m == 0) return DLA_OK;
  return gesvd_bwd<T>(cx, batch, m, n, abar, ubar, lambdabar, vbar, u, lambda, v, eps_gap);
}

// ------------------------------------------------- fused C1 chain (GP NLL)
__global__ void k_fill_ones(int64_t n, double* pd, float* pf) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    if (pd) pd[i] = 1.0;
    if (pf) pf[i] = 1.0f;
  }
}

template <typename T>
size_t ws_chol_chain(int64_t batch, int64_t n) {
  if (n <= 32) return 0;
  return carve_bound(bytes<T>(batch, n, n) + bytes<T>(batch, n, 1) + bytes<T>(batch, 1, 1)) +
         ws_potrf_fwd<T>(batch, n) + ws_trsm<T>(batch, n, 1, false) + ws_gemm<T>(batch, 1, 1, n) +
         ws_trsm_bwd<T>(batch, n, 1, 0) + ws_potrf_bwd<T>(batch, n);
}

// phi = 1/2 |L^-1 y|^2 + sumlogdiag(L), L = potrf(A); ybar, Abar at phibar = 1.
// n <= 32: one fused warp-per-matrix launch (small.cu); otherwise the
// operator chain (the reference's own composition) on workspace scratch.
template <typename T>
dla_status chol_chain_abi(const Ctx& cx, int64_t batch, int64_t n, const T* a, const T* y, T* phi, T* abar,
                          T* ybar) {
  if (bad_dims(batch, n)) return DLA_ERR_SHAPE;
  const size_t asz = bytes<T>(batch, n, n), ysz = bytes<T>(batch, n, 1), psz = bytes<T>(batch, 1, 1);
  if (overlap(abar, asz, a, asz) || overlap(abar, asz, y, ysz) || overlap(ybar, ysz, a, asz) ||
      overlap(ybar, ysz, y, ysz) || overlap(phi, psz, a, asz) || overlap(phi, psz, y, ysz) ||
      overlap(abar, asz, ybar, ysz) || overlap(phi, psz, abar, asz) || overlap(phi, psz, ybar, ysz))
    return DLA_ERR_ALIAS;
  DLAB_TRY(reset_info(cx, batch));
  if (batch == 0) return DLA_OK;
  if (n == 0) return cudaMemsetAsync(phi, 0, psz, cx.stream) == cudaSuccess ? DLA_OK : DLA_ERR_CUDA;
  if (n <= 32) return chol_chain_small<T>(cx, batch, n, cpk(a, n, n), y, phi, pk(abar, n, n), ybar);
  DLAB_SCRATCH(ws, cx, asz + ysz + psz);
  T* l = ws.as<T>();
  T* z = l + batch * n * n;
  T* ones = z + batch * n;
  k_fill_ones<<<blocks_for(batch, 256), 256, 0, cx.stream>>>(batch, sizeof(T) == 8 ? (double*)ones : nullptr,
                                                             sizeof(T) == 4 ? (float*)ones : nullptr);
  DLAB_LAUNCH_CHECK();
  if (cudaMemcpyAsync(l, a, asz, cudaMemcpyDeviceToDevice, cx.stream) != cudaSuccess ||
      cudaMemcpyAsync(z, y, ysz, cudaMemcpyDeviceToDevice, cx.stream) != cudaSuccess)
    return DLA_ERR_CUDA;
  DLAB_TRY(potrf_fwd<T>(cx, batch, n, l, 1));
  // later ops skip failed slices through info (dl/matrix.hpp:232-239 semantics)
  DLAB_TRY(trsm<T>(cx, batch, n, 1, cpk(l, n, n), pk(z, n, 1), false, false, true, T(1)));
  DLAB_TRY(sumlogdiag_fwd<T>(cx, batch, n, phi, cpk(l, n, n)));
  DLAB_TRY(gemm<T>(cx, batch, 1, 1, n, T(0.5), cpk(z, n, 1), true, cpk(z, n, 1), false, T(1), pk(phi, 1, 1)));
  Ctx nx = cx;
  nx.info = nullptr;  // the pullbacks do not report (the reference's backward never throws here)
  DLAB_TRY(trsm_bwd<T>(nx, batch, n, 1, ybar, abar, z, l, z, 0, 0, 1, T(1)));
  DLAB_TRY(sumlogdiag_bwd<T>(nx, batch, n, pk(abar, n, n), ones, cpk(l, n, n), true));
  return potrf_bwd<T>(nx, batch, n, abar, abar, l, 1);
}

// ------------------------------------------- split potrf pullback (drivers)
// L^{-1} for the inverse-based potrf pullback computed on a side stream
// forked from the caller's stream (fork_res(FORK_INV, stream)), so a driver
// can overlap it with work that only needs L (the GP driver's solves).  One
// begin/end pair in flight per (device, caller stream); both halves are
// stream-ordered and graph-capturable.  Events: ev[0] fork, ev[1] done,
// ev[2] mid (early-inverse hook), ev[3] fin.
//
// Workspace layout (the same in every call of the pair): the explicit
// inverse region is the FIRST carve of a fresh arena, then the call's own
// nested scratch.
template <typename T>
size_t potrf_inv_ws(int64_t batch, int64_t n) {
  // wi (n^2) | tt (n^2) | tmp (trtri_levels_tmp(n) bytes) | tmp2 (trtri_levels_tmp(n / 2) bytes)
  return sizeof(T) * (size_t)batch * 2 * (size_t)n * n + (size_t)batch * trtri_levels_tmp<T>(n) +
         (size_t)batch * trtri_levels_tmp<T>(n / 2);
}

template <typename T>
size_t ws_potrf_split(int64_t batch, int64_t n) {
  if (batch * n == 0) return 0;
  if (!inv_eligible<T>(n)) return std::max(ws_potrf_fwd<T>(batch, n), ws_potrf_bwd<T>(batch, n));
  const int64_t h = n / 2;
  const size_t gp = ws_check_symmetric(batch) + ws_potrf_lower<T>(batch, n) + ws_trtri_levels<T>(batch, h) * 2 +
                    2 * ws_gemm<T>(batch, h, h, h);
  const size_t begin = ws_potrf_inv_prepare<T>(batch, n);
  const size_t end = ws_potrf_bwd_tail<T>(batch, n);
  return carve_bound(potrf_inv_ws<T>(batch, n)) + std::max(gp, std::max(begin, end));
}

template <typename T>
dla_status potrf_bwd_begin(const Ctx& cx, int64_t batch, int64_t n, const T* l, int lower) {
  if (bad_dims(batch, n)) return DLA_ERR_SHAPE;
  if (batch * n == 0 || !inv_eligible<T>(n)) return DLA_OK;  // end() takes the direct path
  DLAB_SCRATCH(inv, cx, potrf_inv_ws<T>(batch, n));
  ForkRes& f = fork_res(FORK_INV, cx.stream);
  std::lock_guard<std::mutex> lk(f.mu);
  Ctx side = cx;
  side.stream = f.side;
  cudaEventRecord(f.ev[0], cx.stream);
  cudaStreamWaitEvent(f.side, f.ev[0], 0);
  T* wp = inv.as<T>();
  const dla_status st =
      potrf_inv_prepare<T>(side, batch, n, cpk(l, n, n), lower != 0, pk(wp, n, n), wp + 2 * batch * n * n);
  cudaEventRecord(f.ev[1], f.side);
  return st;
}

template <typename T>
dla_status potrf_bwd_end(const Ctx& cx, int64_t batch, int64_t n, T* abar, const T* lbar, const T* l, int lower) {
  if (bad_dims(batch, n)) return DLA_ERR_SHAPE;
  if (batch * n == 0 || !inv_eligible<T>(n)) return potrf_bwd<T>(cx, batch, n, abar, lbar, l, lower);
  const size_t sz = bytes<T>(batch, n, n);
  if (overlap(abar, sz, l, sz) || (abar != lbar && overlap(abar, sz, lbar, sz))) return DLA_ERR_ALIAS;
  DLAB_SCRATCH(inv, cx, potrf_inv_ws<T>(batch, n));
  T* wp = inv.as<T>();
  MatB<T> tt = pk(wp + batch * n * n, n, n);
  // P' needs only L and Lbar: it overlaps the inverse still running on the side stream
  const dla_status st = potrf_bwd_phi<T>(cx, batch, n, cpk(lbar, n, n), cpk(l, n, n), lower != 0, tt);
  ForkRes& f = fork_res(FORK_INV, cx.stream);
  {
    std::lock_guard<std::mutex> lk(f.mu);
    cudaStreamWaitEvent(cx.stream, f.ev[1], 0);
  }
  if (st != DLA_OK) return st;
  return potrf_bwd_finish<T>(cx, batch, n, pk(abar, n, n), cpk(wp, n, n), tt);
}

// The GP step's pullback tail in one call: potrf_bwd_end up to Z (no Abar
// pass) and the symmetric RBF pullback reading Z directly (gp.cu
// k_rbf_bwd_sym).  lbar is clobbered (W scratch).  Falls back to
// potrf_bwd_end + the row-wise RBF pullback where the inverse path or the
// feature count does not apply.
dla_status gp_pullback(const Ctx& cx, int64_t batch, int64_t n, int64_t d, const double* x, double sigma2,
                       double ell2, double lam, double* lbar, const double* l, double* xbar, double* grads, void* rws,
                       size_t rws_bytes) {
  if (bad_dims(batch, n) || d < 1) return DLA_ERR_SHAPE;
  if (batch * n == 0) return DLA_OK;
  if (!inv_eligible<double>(n) || !gp_rbf_sym_ok(d)) {
    DLAB_TRY(potrf_bwd_end<double>(cx, batch, n, lbar, lbar, l, 1));
    return dla_gp_rbf_bwd_f64(batch, n, d, x, sigma2, ell2, lam, lbar, xbar, grads, rws, rws_bytes, cx.stream);
  }
  DLAB_SCRATCH(inv, cx, potrf_inv_ws<double>(batch, n));
  double* wp = inv.as<double>();
  MatB<double> tt = pk(wp + batch * n * n, n, n);
  const dla_status st = potrf_bwd_phi<double>(cx, batch, n, cpk(lbar, n, n), cpk(l, n, n), true, tt);
  ForkRes& f = fork_res(FORK_INV, cx.stream);
  {
    std::lock_guard<std::mutex> lk(f.mu);
    cudaStreamWaitEvent(cx.stream, f.ev[1], 0);
  }
  if (st != DLA_OK) return st;
  DLAB_TRY(potrf_bwd_finish_z<double>(cx, batch, n, pk(lbar, n, n), cpk(wp, n, n), tt));
  return gp_rbf_bwd_sym(batch, n, d, x, sigma2, ell2, lam, tt.p, xbar, grads, rws, rws_bytes, cx.stream);
}

// Factorization + early inverse for drivers (the GP step): the blocked
// Cholesky signals once block columns [0, n/2) are final; from then on the
// side stream forms L11^{-1} and T1 = L21 L11^{-1} (half of the inverse's
// flops) while the factorization's chain-bound second half runs; after it,
// L22^{-1} and W21 = -L22^{-1} T1 complete L^{-1} into the workspace that
// dla_potrf_bwd_end_f64 consumes.  Same operations as trtri_levels on the
// whole matrix (its top level is exactly T1 and W21).
template <typename T>
struct EarlyInv {
  int64_t batch, n;
  const T* l;
  T* wp;
  Ctx side;
  cudaEvent_t ev;
  bool fired;
  dla_status st;
};

template <typename T>
void early_inv_first(void* user, cudaStream_t crit) {
  EarlyInv<T>& e = *static_cast<EarlyInv<T>*>(user);
  e.fired = true;
  const int64_t n = e.n, h = n / 2, B = e.batch;
  cudaEventRecord(e.ev, crit);
  cudaStreamWaitEvent(e.side.stream, e.ev, 0);
  const Ctx& sc = e.side;
  MatB<T> wi{e.wp, n, n * n};
  T* tmp = e.wp + 2 * B * n * n;
  MatB<const T> lv{e.l, n, n * n};
  // W11 = L11^{-1} read straight from the factor (no copy pass); T1 = L21 W11
  // into tmp, L21 again read from the factor
  T* tmp2 = tmp + B * (trtri_levels_tmp<T>(n) / sizeof(T));
  dla_status st = trtri_levels<T>(sc, B, h, wi, tmp2, &lv, false);
  MatB<T> t1{tmp, h, h * h};
  // T1 runs beside the factorization's chain-bound second half: a grid of
  // long-K tiles on every SM keeps the look-ahead updates and panel launches
  // waiting for SMs (measured: a 100 us stall of the chain when T1 filled the
  // GPU).  DLA_GP_EARLY_CTAS (tuning switch; 0 = unbounded) caps its
  // persistent grid; the per-tile arithmetic is unchanged (bitwise the same).
  static const int early_ctas = [] {
    const char* v = getenv("DLA_GP_EARLY_CTAS");
    return v ? atoi(v) : 0;
  }();
  Ctx tc = sc;
  tc.gemm_ctas = early_ctas;
  if (st == DLA_OK)
    st = gemm<T>(tc, B, h, h, h, T(1), MatB<const T>{e.l + h * n, n, n * n}, false, MatB<const T>{wi.p, n, n * n},
                 false, T(0), t1, MASK_FULL, nullptr, TRI_NONE, TRI_LOWER);
  e.st = st;
}

template <typename T>
dla_status gp_potrf_inv(const Ctx& cx, int64_t batch, int64_t n, T* a) {
  if (bad_dims(batch, n)) return DLA_ERR_SHAPE;
  if (!inv_eligible<T>(n) || batch * n == 0) {  // no early path: factorization, then the plain begin
    DLAB_TRY(potrf_fwd<T>(cx, batch, n, a, 1));
    return potrf_bwd_begin<T>(cx, batch, n, a, 1);
  }
  DLAB_SCRATCH(inv, cx, potrf_inv_ws<T>(batch, n));
  DLAB_TRY(reset_info(cx, batch));
  DLAB_TRY(check_symmetric<T>(cx, batch, n, cpk(a, n, n), cx.info));
  ForkRes& f = fork_res(FORK_INV, cx.stream);
  std::lock_guard<std::mutex> lk(f.mu);
  Ctx sc = cx;
  sc.stream = f.side;
  sc.info = nullptr;
  EarlyInv<T> e{batch, n, a, inv.as<T>(), sc, f.ev[2], false, DLA_OK};
  PotrfHook hook{n / 2, early_inv_first<T>, &e, a, n};
  Ctx hc = cx;
  hc.potrf_hook = &hook;
  bool zeroed = false;  // the blocked factorization zeroes the strict upper triangle as it goes
  const dla_status sf = potrf_lower<T>(hc, batch, n, pk(a, n, n), /*zero_upper*/ false, &zeroed);
  if (!e.fired) early_inv_first<T>(&e, cx.stream);  // a schedule without the hook point (tuning modes)
  const int64_t h = n / 2;
  T* wp = inv.as<T>();
  MatB<T> wi{wp, n, n * n};
  T* tmp = wp + 2 * batch * n * n;
  T* tmp2 = tmp + batch * (trtri_levels_tmp<T>(n) / sizeof(T));
  cudaEventRecord(f.ev[3], cx.stream);
  cudaStreamWaitEvent(f.side, f.ev[3], 0);
  dla_status st = e.st;
  // DLA_GP_SIDE_CTAS (tuning switch, > 0): cap the side stream's GEMM grid
  // from here on, so critical-path kernels find room on every SM.  Measured:
  // the capped inverse and the pullback's first product then share the SMs
  // and both slow down (C2 7.02 vs 6.81 ms), so the default is unbounded.
  static const int side_ctas = [] {
    const char* e = getenv("DLA_GP_SIDE_CTAS");
    return e ? atoi(e) : 0;
  }();
  sc.gemm_ctas = side_ctas;
  // W22 = L22^{-1} (read straight from the factor); W21 = -W22 T1
  const MatB<const T> l22{a + h * n + h, n, n * n};
  if (st == DLA_OK) st = trtri_levels<T>(sc, batch, h, wi.sub(h, h), tmp2, &l22, false);
  if (st == DLA_OK)
    st = gemm<T>(sc, batch, h, h, h, T(-1), MatB<const T>{wi.p + h * n + h, n, n * n}, false,
                 MatB<const T>{tmp, h, h * h}, false, T(0), wi.sub(h, 0), MASK_FULL, nullptr, TRI_LOWER, TRI_NONE);
  // L's strict upper triangle (the potrf contract) is zeroed here, on the side
  // stream: no kernel of the step reads it, so it stays off the critical path.
  // It is complete once dla_potrf_bwd_end_f64 (or dla_potrf_inv_join_f64)
  // has been enqueued on the caller's stream.
  if (st == DLA_OK && !zeroed) {
    Ctx zc = sc;
    zc.info = cx.info;
    st = ew_square<T>(zc, batch, n, pk(a, n, n), /*tril*/ 0, T(1), cx.info);
  }
  cudaEventRecord(f.ev[1], f.side);
  return sf != DLA_OK ? sf : st;
}

// ------------------------------------------------------ workspace query
template <typename T>
size_t ws_query(dla_op op, int64_t batch, int64_t m, int64_t n, int64_t k, int phase) {
  const bool bwd = (phase & DLA_WS_BACKWARD) != 0, right = (phase & DLA_WS_RIGHTSIDE) != 0;
  switch (op) {
    case DLA_OP_GEMM:
    case DLA_OP_GEMM2: {
      if (!bwd) return ws_gemm<T>(batch, m, n, k);
      size_t w = 0;  // the operand transposes are not part of the query: the largest of the four
      for (int ta = 0; ta < 2; ++ta)
        for (int tb = 0; tb < 2; ++tb) w = std::max(w, ws_gemm_bwd<T>(batch, m, n, k, ta, tb));
      return w;
    }
    case DLA_OP_SYRK:
      return !bwd ? ws_gemm<T>(batch, n, n, k) : std::max(ws_syrk_bwd<T>(batch, n, k, 0), ws_syrk_bwd<T>(batch, n, k, 1));
    case DLA_OP_TRMM:
      return !bwd ? ws_trmm<T>(batch, m, n, right) : ws_trmm_bwd<T>(batch, m, n, right);
    case DLA_OP_TRSM:
      return !bwd ? ws_trsm<T>(batch, m, n, right) : ws_trsm_bwd<T>(batch, m, n, right);
    case DLA_OP_POTRF:
      return !bwd ? ws_potrf_fwd<T>(batch, n) : ws_potrf_bwd<T>(batch, n);
    case DLA_OP_POTRI:
      return !bwd ? ws_potri_lower<T>(batch, n) : std::max(ws_potri_bwd<T>(batch, n, 1), ws_potri_bwd<T>(batch, n, 0));
    case DLA_OP_SUMLOGDIAG:
      return 0;
    case DLA_OP_GELQF:
      if (m > n) return 0;  // ShapeError (the op reports it)
      return !bwd ? ws_gelqf_fwd<T>(batch, m, n) : ws_gelqf_bwd<T>(batch, m, n);
    case DLA_OP_SYEVD:
      return !bwd ? carve_bound(syevd_ws_bytes<T>(batch, n, false)) : ws_syevd_bwd<T>(batch, n);
    case DLA_OP_CHOL_CHAIN:
      return ws_chol_chain<T>(batch, n);
    case DLA_OP_GESVD:
      if (m > n) return 0;
      return !bwd ? ws_gesvd_fwd<T>(batch, m, n) : ws_gesvd_bwd<T>(batch, m, n);
  }
  return 0;
}

}  // namespace
}  // namespace dlab

using namespace dlab;

extern "C" {

const char* dla_status_string(dla_status s) {
  switch (s) {
    case DLA_OK: return "ok";
    case DLA_ERR_SHAPE: return "shape error";
    case DLA_ERR_NOT_SPD: return "matrix is not positive definite";
    case DLA_ERR_SINGULAR: return "singular";
    case DLA_ERR_CONVERGENCE: return "did not converge";
    case DLA_ERR_ALIAS: return "output must not alias this input";
    case DLA_ERR_ASYMMETRIC: return "input is not symmetric";
    case DLA_ERR_CUDA: return "CUDA error";
    case DLA_ERR_WORKSPACE: return "workspace missing or too small";
    case DLA_ERR_INVALID: return "invalid argument";
  }
  return "unknown";
}

const char* dla_version(void) { return "dla_b200 0.1 (sm_100a)"; }

long long dla_launch_count(void) { return g_launches.load(); }

void dla_prof_enable(int on) {
  std::lock_guard<std::mutex> lk(g_prof_mu);
  for (auto& r : g_prof_recs) {
    g_event_pool.push_back(r.a);
    g_event_pool.push_back(r.b);
  }
  g_prof_recs.clear();
  g_prof.store(on != 0);
}

// Synchronises the recorded events; returns the number of GEMM launches and
// their summed device time (ms) and algorithmic flops.
long long dla_prof_read(double* ms, double* flops) {
  std::lock_guard<std::mutex> lk(g_prof_mu);
  double t = 0, f = 0;
  for (auto& r : g_prof_recs) {
    cudaEventSynchronize(r.b);
    float x = 0;
    cudaEventElapsedTime(&x, r.a, r.b);
    t += x;
    f += r.flops;
  }
  if (ms) *ms = t;
  if (flops) *flops = f;
  return (long long)g_prof_recs.size();
}

long long dla_prof_read_max(double* ms, double* flops) {
  // the GEMM launch(es) with the largest flop count (ties averaged)
  std::lock_guard<std::mutex> lk(g_prof_mu);
  double fmaxv = 0;
  for (auto& r : g_prof_recs) fmaxv = r.flops > fmaxv ? r.flops : fmaxv;
  double t = 0;
  long long cnt = 0;
  for (auto& r : g_prof_recs) {
    if (r.flops < fmaxv) continue;
    cudaEventSynchronize(r.b);
    float x = 0;
    cudaEventElapsedTime(&x, r.a, r.b);
    t += x;
    ++cnt;
  }
  if (ms) *ms = cnt ? t / cnt : 0;
  if (flops) *flops = fmaxv;
  return cnt;
}

size_t dla_workspace_bytes(dla_op op, dla_dtype dtype, int64_t batch, int64_t m, int64_t n, int64_t k, int phase) {
  if (batch < 0 || m < 0 || n < 0 || k < 0) return 0;
  return dtype == DLA_F64 ? ws_query<double>(op, batch, m, n, k, phase) : ws_query<float>(op, batch, m, n, k, phase);
}

dla_status dla_info_check(const int32_t* info, int64_t batch, void* stream, int64_t* first_bad, int64_t* index) {
  if (first_bad) *first_bad = -1;
  if (index) *index = -1;
  if (!info || batch <= 0) return DLA_OK;
  std::vector<int32_t> h((size_t)batch);
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  if (cudaMemcpyAsync(h.data(), info, sizeof(int32_t) * batch, cudaMemcpyDeviceToHost, s) != cudaSuccess)
    return DLA_ERR_CUDA;
  if (cudaStreamSynchronize(s) != cudaSuccess) return DLA_ERR_CUDA;
  for (int64_t b = 0; b < batch; ++b)
    if (h[(size_t)b] != 0) {
      if (first_bad) *first_bad = b;
      if (index) *index = DLA_INFO_INDEX(h[(size_t)b]);
      return (dla_status)DLA_INFO_CODE(h[(size_t)b]);
    }
  return DLA_OK;
}

#define DLA_ARENA(ws, wsb, stream, info) \
  Arena arena_(ws, wsb);                  \
  const Ctx cx = make_ctx(stream, info, &arena_)

// A short workspace is refused before any launch (outputs untouched); a
// negative dimension skips the check so the op reports DLA_ERR_SHAPE.
#define DLA_NEED(T, op, batch, m, n, k, phase)                                                        \
  do {                                                                                                \
    if ((batch) >= 0 && (m) >= 0 && (n) >= 0 && (k) >= 0 &&                                          \
        (ws == nullptr ? (size_t)0 : wsb) < ws_query<T>(op, batch, m, n, k, phase))                  \
      return DLA_ERR_WORKSPACE;                                                                       \
  } while (0)

#define DLA_DEFINE(T, S)                                                                                          \
  dla_status dla_gemm2_fwd_##S(int64_t batch, int64_t m, int64_t n, int64_t k, T* c, const T* a, const T* b,      \
                               int ta, int tb, T alpha, void* ws, size_t wsb, void* stream) {                    \
    DLA_NEED(T, DLA_OP_GEMM, batch, m, n, k, 0);                                                                  \
    DLA_ARENA(ws, wsb, stream, nullptr);                                                                          \
    return gemm_fwd<T>(cx, batch, m, n, k, c, a, b, ta, tb, alpha, T(0));                                        \
  }                                                                                                               \
  dla_status dla_gemm_fwd_##S(int64_t batch, int64_t m, int64_t n, int64_t k, T* c, const T* a, const T* b,       \
                              int ta, int tb, T alpha, T beta, void* ws, size_t wsb, void* stream) {             \
    DLA_NEED(T, DLA_OP_GEMM, batch, m, n, k, 0);                                                                  \
    DLA_ARENA(ws, wsb, stream, nullptr);                                                                          \
    return gemm_fwd<T>(cx, batch, m, n, k, c, a, b, ta, tb, alpha, beta);                                        \
  }                                                                                                               \
  dla_status dla_gemm2_bwd_##S(int64_t batch, int64_t m, int64_t n, int64_t k, T* abar, T* bbar, const T* cbar,   \
                               const T* a, const T* b, int ta, int tb, T alpha, void* ws, size_t wsb,            \
                               void* stream) {                                                                    \
    DLA_NEED(T, DLA_OP_GEMM, batch, m, n, k, DLA_WS_BACKWARD);                                                    \
    DLA_ARENA(ws, wsb, stream, nullptr);                                                                          \
    return gemm_bwd<T>(cx, batch, m, n, k, abar, bbar, const_cast<T*>(cbar), a, b, ta, tb, alpha, T(0), false);  \
  }                                                                                                               \
  dla_status dla_gemm_bwd_##S(int64_t batch, int64_t m, int64_t n, int64_t k, T* abar, T* bbar, T* cbar_io,       \
                              const T* a, const T* b, int ta, int tb, T alpha, T beta, void* ws, size_t wsb,     \
                              void* stream) {                                                                     \
    DLA_NEED(T, DLA_OP_GEMM, batch, m, n, k, DLA_WS_BACKWARD);                                                    \
    DLA_ARENA(ws, wsb, stream, nullptr);                                                                          \
    return gemm_bwd<T>(cx, batch, m, n, k, abar, bbar, cbar_io, a, b, ta, tb, alpha, beta, true);                \
  }                                                                                                               \
  dla_status dla_syrk_fwd_##S(int64_t batch, int64_t n, int64_t k, T* b, const T* a, int ta, T alpha, void* ws,   \
                              size_t wsb, void* stream) {                                                         \
    DLA_NEED(T, DLA_OP_SYRK, batch, 0, n, k, 0);                                                                  \
    DLA_ARENA(ws, wsb, stream, nullptr);                                                                          \
    return syrk_fwd<T>(cx, batch, n, k, b, a, ta, alpha);                                                         \
  }                                                                                                               \
  dla_status dla_syrk_bwd_##S(int64_t batch, int64_t n, int64_t k, T* abar, const T* bbar, const T* a, int ta,    \
                              T alpha, void* ws, size_t wsb, void* stream) {                                      \
    DLA_NEED(T, DLA_OP_SYRK, batch, 0, n, k, DLA_WS_BACKWARD);                                                    \
    DLA_ARENA(ws, wsb, stream, nullptr);                                                                          \
    return syrk_bwd<T>(cx, batch, n, k, abar, bbar, a, ta, alpha);                                                \
  }                                                                                                               \
  dla_status dla_trmm_fwd_##S(int64_t batch, int64_t m, int64_t n, const T* t, T* x, int r, int tr, int lo,       \
                              T alpha, void* ws, size_t wsb, void* stream) {                                      \
    DLA_NEED(T, DLA_OP_TRMM, batch, m, n, 0, r ? DLA_WS_RIGHTSIDE : 0);                                           \
    DLA_ARENA(ws, wsb, stream, nullptr);                                                                          \
    return trmm_fwd<T>(cx, batch, m, n, t, x, r, tr, lo, alpha);                                                  \
  }                                                                                                               \
  dla_status dla_trmm_into_##S(int64_t batch, int64_t m, int64_t n, const T* t, const T* x, T* y, int r, int tr,   \
                               int lo, T alpha, void* ws, size_t wsb, void* stream) {                            \
    DLA_NEED(T, DLA_OP_TRMM, batch, m, n, 0, r ? DLA_WS_RIGHTSIDE : 0);                                           \
    DLA_ARENA(ws, wsb, stream, nullptr);                                                                          \
    return trmm_into<T>(cx, batch, m, n, t, x, y, r, tr, lo, alpha);                                              \
  }                                                                                                               \
  dla_status dla_trmm_bwd_##S(int64_t batch, int64_t m, int64_t n, T* abar, T* tbar, const T* bbar, const T* t,   \
                              const T* a, int r, int tr, int lo, T alpha, void* ws, size_t wsb, void* stream) {  \
    DLA_NEED(T, DLA_OP_TRMM, batch, m, n, 0, DLA_WS_BACKWARD | (r ? DLA_WS_RIGHTSIDE : 0));                       \
    DLA_ARENA(ws, wsb, stream, nullptr);                                                                          \
    return trmm_bwd<T>(cx, batch, m, n, abar, tbar, bbar, t, a, r, tr, lo, alpha);                                \
  }                                                                                                               \
  dla_status dla_trsm_fwd_##S(int64_t batch, int64_t m, int64_t n, const T* t, T* x, int r, int tr, int lo,       \
                              T alpha, int32_t* info, void* ws, size_t wsb, void* stream) {                       \
    DLA_NEED(T, DLA_OP_TRSM, batch, m, n, 0, r ? DLA_WS_RIGHTSIDE : 0);                                           \
    DLA_ARENA(ws, wsb, stream, info);                                                                             \
    return trsm_fwd<T>(cx, batch, m, n, t, x, r, tr, lo, alpha);                                                  \
  }                                                                                                               \
  dla_status dla_trsm_bwd_##S(int64_t batch, int64_t m, int64_t n, T* abar, T* tbar, const T* bbar, const T* t,   \
                              const T* b, int r, int tr, int lo, T alpha, void* ws, size_t wsb, void* stream) {  \
    DLA_NEED(T, DLA_OP_TRSM, batch, m, n, 0, DLA_WS_BACKWARD | (r ? DLA_WS_RIGHTSIDE : 0));                       \
    DLA_ARENA(ws, wsb, stream, nullptr);                                                                          \
    return trsm_bwd<T>(cx, batch, m, n, abar, tbar, bbar, t, b, r, tr, lo, alpha);                                \
  }                                                                                                               \
  dla_status dla_potrf_fwd_##S(int64_t batch, int64_t n, T* a, int lower, int32_t* info, void* ws, size_t wsb,    \
                               void* stream) {                                                                    \
    DLA_NEED(T, DLA_OP_POTRF, batch, n, n, 0, 0);                                                                 \
    DLA_ARENA(ws, wsb, stream, info);                                                                             \
    return potrf_fwd<T>(cx, batch, n, a, lower);                                                                  \
  }                                                                                                               \
  dla_status dla_potrf_bwd_##S(int64_t batch, int64_t n, T* abar, const T* lbar, const T* l, int lower,           \
                               void* ws, size_t wsb, void* stream) {                                              \
    DLA_NEED(T, DLA_OP_POTRF, batch, n, n, 0, DLA_WS_BACKWARD);                                                   \
    DLA_ARENA(ws, wsb, stream, nullptr);                                                                          \
    return potrf_bwd<T>(cx, batch, n, abar, lbar, l, lower);                                                      \
  }                                                                                                               \
  dla_status dla_potri_fwd_##S(int64_t batch, int64_t n, T* a, int lower, int32_t* info, void* ws, size_t wsb,    \
                               void* stream) {                                                                    \
    DLA_NEED(T, DLA_OP_POTRI, batch, n, n, 0, 0);                                                                 \
    DLA_ARENA(ws, wsb, stream, info);                                                                             \
    return potri_fwd<T>(cx, batch, n, a, lower);                                                                  \
  }                                                                                                               \
  dla_status dla_potri_into_##S(int64_t batch, int64_t n, const T* l, T* b, int lower, int32_t* info, void* ws,  \
                                size_t wsb, void* stream) {                                                       \
    DLA_NEED(T, DLA_OP_POTRI, batch, n, n, 0, 0);                                                                 \
    DLA_ARENA(ws, wsb, stream, info);                                                                             \
    return potri_into<T>(cx, batch, n, l, b, lower);                                                              \
  }                                                                                                               \
  dla_status dla_potri_bwd_##S(int64_t batch, int64_t n, T* lbar, const T* bbar, const T* l, const T* b,          \
                               int lower, void* ws, size_t wsb, void* stream) {                                   \
    DLA_NEED(T, DLA_OP_POTRI, batch, n, n, 0, DLA_WS_BACKWARD);                                                   \
    DLA_ARENA(ws, wsb, stream, nullptr);                                                                          \
    return potri_bwd<T>(cx, batch, n, lbar, bbar, l, b, lower);                                                   \
  }                                                                                                               \
  dla_status dla_sumlogdiag_fwd_##S(int64_t batch, int64_t n, T* out, const T* a, void* ws, size_t wsb,           \
                                    void* stream) {                                                               \
    DLA_ARENA(ws, wsb, stream, nullptr);                                                                          \
    return sld_fwd<T>(cx, batch, n, out, a);                                                                      \
  }                                                                                                               \
  dla_status dla_sumlogdiag_bwd_##S(int64_t batch, int64_t n, T* abar, const T* gbar, const T* a,                 \
                                    int accumulate, void* ws, size_t wsb, void* stream) {                         \
    DLA_ARENA(ws, wsb, stream, nullptr);                                                                          \
    return sld_bwd<T>(cx, batch, n, abar, gbar, a, accumulate);                                                   \
  }                                                                                                               \
  dla_status dla_gelqf_fwd_##S(int64_t batch, int64_t m, int64_t n, T* q, T* l, int32_t* info, void* ws,         \
                               size_t wsb, void* stream) {                                                        \
    DLA_NEED(T, DLA_OP_GELQF, batch, m, n, 0, 0);                                                                 \
    DLA_ARENA(ws, wsb, stream, info);                                                                             \
    return gelqf_fwd_abi<T>(cx, batch, m, n, q, l);                                                               \
  }                                                                                                               \
  dla_status dla_gelqf_bwd_##S(int64_t batch, int64_t m, int64_t n, T* abar, const T* qbar, const T* lbar,        \
                               const T* q, const T* l, void* ws, size_t wsb, void* stream) {                      \
    DLA_NEED(T, DLA_OP_GELQF, batch, m, n, 0, DLA_WS_BACKWARD);                                                   \
    DLA_ARENA(ws, wsb, stream, nullptr);                                                                          \
    return gelqf_bwd_abi<T>(cx, batch, m, n, abar, qbar, lbar, q, l);                                             \
  }                                                                                                               \
  dla_status dla_syevd_fwd_##S(int64_t batch, int64_t n, T* u, T* lambda, int32_t* info, void* ws,               \
                               size_t wsb, void* stream) {                                                        \
    DLA_NEED(T, DLA_OP_SYEVD, batch, n, n, 0, 0);                                                                 \
    DLA_ARENA(ws, wsb, stream, info);                                                                             \
    return syevd_fwd_abi<T>(cx, batch, n, u, lambda);                                                             \
  }                                                                                                               \
  dla_status dla_syevd_bwd_##S(int64_t batch, int64_t n, T* abar, const T* ubar, const T* lambdabar, const T* u,  \
                               const T* lambda, T eps_gap, void* ws, size_t wsb, void* stream) {                  \
    DLA_NEED(T, DLA_OP_SYEVD, batch, n, n, 0, DLA_WS_BACKWARD);                                                   \
    DLA_ARENA(ws, wsb, stream, nullptr);                                                                          \
    return syevd_bwd_abi<T>(cx, batch, n, abar, ubar, lambdabar, u, lambda, eps_gap);                             \
  }                                                                                                               \
  dla_status dla_gesvd_fwd_##S(int64_t batch, int64_t m, int64_t n, T* v, T* u, T* lambda, int32_t* info,        \
                               void* ws, size_t wsb, void* stream) {                                              \
    DLA_NEED(T, DLA_OP_GESVD, batch, m, n, 0, 0);                                                                 \
    DLA_ARENA(ws, wsb, stream, info);                                                                             \
    return gesvd_fwd_abi<T>(cx, batch, m, n, v, u, lambda);                                                       \
  }                                                                                                               \
  dla_status dla_gesvd_bwd_##S(int64_t batch, int64_t m, int64_t n, T* abar, const T* ubar, const T* lambdabar,   \
                               const T* vbar, const T* u, const T* lambda, const T* v, T eps_gap, int32_t* info,  \
                               void* ws, size_t wsb, void* stream) {                                              \
    DLA_NEED(T, DLA_OP_GESVD, batch, m, n, 0, DLA_WS_BACKWARD);                                                   \
    DLA_ARENA(ws, wsb, stream, info);                                                                             \
    return gesvd_bwd_abi<T>(cx, batch, m, n, abar, ubar, lambdabar, vbar, u, lambda, v, eps_gap);                 \
  }                                                                                                               \
  dla_status dla_chol_chain_fwdbwd_##S(int64_t batch, int64_t n, const T* a, const T* y, T* phi, T* abar,         \
                                       T* ybar, int32_t* info, void* ws, size_t wsb, void* stream) {              \
    DLA_NEED(T, DLA_OP_CHOL_CHAIN, batch, n, n, 0, 0);                                                            \
    DLA_ARENA(ws, wsb, stream, info);                                                                             \
    return chol_chain_abi<T>(cx, batch, n, a, y, phi, abar, ybar);                                                \
  }

DLA_DEFINE(float, f32)
DLA_DEFINE(double, f64)

size_t dla_potrf_bwd_ws_bytes_f64(int64_t batch, int64_t n) {
  if (batch < 0 || n < 0) return 0;
  return ws_potrf_split<double>(batch, n);
}
dla_status dla_gp_potrf_inv_f64(int64_t batch, int64_t n, double* a, int32_t* info, void* ws, size_t ws_bytes,
                                void* stream) {
  if (batch >= 0 && n >= 0 && (ws ? ws_bytes : 0) < ws_potrf_split<double>(batch, n)) return DLA_ERR_WORKSPACE;
  DLA_ARENA(ws, ws_bytes, stream, info);
  return gp_potrf_inv<double>(cx, batch, n, a);
}
dla_status dla_potrf_bwd_begin_f64(int64_t batch, int64_t n, const double* l, int lower, void* ws, size_t ws_bytes,
                                   void* stream) {
  if (batch >= 0 && n >= 0 && (ws ? ws_bytes : 0) < ws_potrf_split<double>(batch, n)) return DLA_ERR_WORKSPACE;
  DLA_ARENA(ws, ws_bytes, stream, nullptr);
  return potrf_bwd_begin<double>(cx, batch, n, l, lower);
}
dla_status dla_potrf_bwd_end_f64(int64_t batch, int64_t n, double* abar, const double* lbar, const double* l,
                                 int lower, void* ws, size_t ws_bytes, void* stream) {
  if (batch >= 0 && n >= 0 && (ws ? ws_bytes : 0) < ws_potrf_split<double>(batch, n)) return DLA_ERR_WORKSPACE;
  DLA_ARENA(ws, ws_bytes, stream, nullptr);
  return potrf_bwd_end<double>(cx, batch, n, abar, lbar, l, lower);
}
size_t dla_gp_pullback_ws_bytes(int64_t batch, int64_t n, int64_t d) {
  if (batch < 0 || n < 0 || d < 0) return 0;
  return std::max(dla_gp_rbf_ws_bytes(batch, n, d), dla_gp_rbf_bwd_sym_ws_bytes(batch, n, d));
}
dla_status dla_gp_pullback_f64(int64_t batch, int64_t n, int64_t d, const double* x, double sigma2, double ell2,
                               double lam, double* lbar, const double* l, double* xbar, double* grads, void* iws,
                               size_t iws_bytes, void* rws, size_t rws_bytes, void* stream) {
  if (batch >= 0 && n >= 0 && (iws ? iws_bytes : 0) < ws_potrf_split<double>(batch, n)) return DLA_ERR_WORKSPACE;
  if (batch >= 0 && n >= 0 && d >= 0 && (rws ? rws_bytes : 0) < dla_gp_pullback_ws_bytes(batch, n, d))
    return DLA_ERR_WORKSPACE;
  DLA_ARENA(iws, iws_bytes, stream, nullptr);
  return gp_pullback(cx, batch, n, d, x, sigma2, ell2, lam, lbar, l, xbar, grads, rws, rws_bytes);
}
dla_status dla_potrf_inv_join_f64(void* stream) {
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  ForkRes& f = fork_res(FORK_INV, s);
  std::lock_guard<std::mutex> lk(f.mu);
  return cudaStreamWaitEvent(s, f.ev[1], 0) == cudaSuccess ? DLA_OK : DLA_ERR_CUDA;
}

}  // extern "C"
