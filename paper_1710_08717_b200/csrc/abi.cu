// extern "C" operator entry points (include/dla.h): host-side validation that
// mirrors the reference's ShapeError / alias sites, then stream-ordered
// launches.  Backward ops follow the reference's closed-form compositions
// (dl/adjoints.hpp) on the batched device kernels.
#include <atomic>
#include <mutex>
#include <vector>

#include "common.cuh"
#include "ops.cuh"

namespace dlab {

Ctx make_ctx(void* stream, int32_t* info) {
  static int sms = 0;
  static std::once_flag flag;
  std::call_once(flag, [] {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
      uint64_t thr = UINT64_MAX;  // keep scratch in the pool: no steady-state cudaMalloc
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    }
  });
  return Ctx{reinterpret_cast<cudaStream_t>(stream), sms, info};
}

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

// ------------------------------------------------------------------- gemm
template <typename T>
dla_status gemm_fwd(int64_t batch, int64_t m, int64_t n, int64_t k, T* c, const T* a, const T* b, int ta, int tb,
                    T alpha, T beta, void* stream) {
  if (batch < 0 || m < 0 || n < 0 || k < 0) return DLA_ERR_SHAPE;
  if (overlap(c, bytes<T>(batch, m, n), a, bytes<T>(batch, m, k)) ||
      overlap(c, bytes<T>(batch, m, n), b, bytes<T>(batch, k, n)))
    return DLA_ERR_ALIAS;
  Ctx cx = make_ctx(stream, nullptr);
  if (beta == T(0)) {  // the reference zero-fills C (gemm_accum accumulate=false)
    if (k == 0 || alpha == T(0)) {
      return cudaMemsetAsync(c, 0, bytes<T>(batch, m, n), cx.stream) == cudaSuccess ? DLA_OK : DLA_ERR_CUDA;
    }
  }
  return gemm<T>(cx, batch, m, n, k, alpha, cpk(a, ta ? k : m, ta ? m : k), ta, cpk(b, tb ? n : k, tb ? k : n),
                 tb, beta, pk(c, m, n));
}

template <typename T>
dla_status gemm_bwd(int64_t batch, int64_t m, int64_t n, int64_t k, T* abar, T* bbar, T* cbar_io, const T* a,
                    const T* b, int ta, int tb, T alpha, T beta, bool has_c, void* stream) {
  if (batch < 0 || m < 0 || n < 0 || k < 0) return DLA_ERR_SHAPE;
  const size_t asz = bytes<T>(batch, m, k), bsz = bytes<T>(batch, k, n), csz = bytes<T>(batch, m, n);
  if (overlap(abar, asz, cbar_io, csz) || overlap(abar, asz, b, bsz) || overlap(bbar, bsz, cbar_io, csz) ||
      overlap(bbar, bsz, a, asz) || overlap(abar, asz, bbar, bsz))
    return DLA_ERR_ALIAS;
  // dl/adjoints.hpp:39-48
  if (!ta) DLAB_TRY(gemm_fwd<T>(batch, m, k, n, abar, cbar_io, b, 0, !tb, alpha, T(0), stream));
  else DLAB_TRY(gemm_fwd<T>(batch, k, m, n, abar, b, cbar_io, tb, 1, alpha, T(0), stream));
  if (!tb) DLAB_TRY(gemm_fwd<T>(batch, k, n, m, bbar, a, cbar_io, !ta, 0, alpha, T(0), stream));
  else DLAB_TRY(gemm_fwd<T>(batch, n, k, m, bbar, cbar_io, a, 1, ta, alpha, T(0), stream));
  if (has_c) {
    Ctx cx = make_ctx(stream, nullptr);
    if (beta == T(0))
      return cudaMemsetAsync(cbar_io, 0, csz, cx.stream) == cudaSuccess ? DLA_OK : DLA_ERR_CUDA;
    return ew_scale<T>(cx, batch, m, n, pk(cbar_io, m, n), beta);
  }
  return DLA_OK;
}

// ------------------------------------------------------------------- syrk
template <typename T>
dla_status syrk_fwd(int64_t batch, int64_t n, int64_t k, T* bo, const T* a, int ta, T alpha, void* stream) {
  if (batch < 0 || n < 0 || k < 0) return DLA_ERR_SHAPE;
  if (overlap(bo, bytes<T>(batch, n, n), a, bytes<T>(batch, n, k))) return DLA_ERR_ALIAS;
  Ctx cx = make_ctx(stream, nullptr);
  if (batch * n == 0) return DLA_OK;
  if (k == 0 || alpha == T(0))
    return cudaMemsetAsync(bo, 0, bytes<T>(batch, n, n), cx.stream) == cudaSuccess ? DLA_OK : DLA_ERR_CUDA;
  MatB<const T> av = cpk(a, ta ? k : n, ta ? n : k);
  DLAB_TRY(gemm<T>(cx, batch, n, n, k, alpha, av, ta, av, !ta, T(0), pk(bo, n, n), MASK_LOWER));
  return ew_square<T>(cx, batch, n, pk(bo, n, n), /*copyltu*/ 2);
}

template <typename T>
dla_status syrk_bwd(int64_t batch, int64_t n, int64_t k, T* abar, const T* bbar, const T* a, int ta, T alpha,
                    void* stream) {
  if (batch < 0 || n < 0 || k < 0) return DLA_ERR_SHAPE;
  const size_t asz = bytes<T>(batch, n, k);
  if (overlap(abar, asz, bbar, bytes<T>(batch, n, n)) || overlap(abar, asz, a, asz)) return DLA_ERR_ALIAS;
  // dl/adjoints.hpp:71-77
  if (!ta) {
    DLAB_TRY(gemm_fwd<T>(batch, n, k, n, abar, bbar, a, 0, 0, alpha, T(0), stream));
    DLAB_TRY(gemm_fwd<T>(batch, n, k, n, abar, bbar, a, 1, 0, alpha, T(1), stream));
  } else {
    DLAB_TRY(gemm_fwd<T>(batch, k, n, n, abar, a, bbar, 0, 0, alpha, T(0), stream));
    DLAB_TRY(gemm_fwd<T>(batch, k, n, n, abar, a, bbar, 0, 1, alpha, T(1), stream));
  }
  return DLA_OK;
}

// ------------------------------------------------------------ trmm / trsm
template <typename T>
dla_status trmm_fwd(int64_t batch, int64_t m, int64_t n, const T* t, T* x, int right, int trans, int lower,
                    T alpha, void* stream) {
  if (bad_dims(batch, m, n)) return DLA_ERR_SHAPE;
  const int64_t nt = right ? n : m;
  if (overlap(x, bytes<T>(batch, m, n), t, bytes<T>(batch, nt, nt))) return DLA_ERR_ALIAS;
  Ctx cx = make_ctx(stream, nullptr);
  return trmm<T>(cx, batch, m, n, cpk(t, nt, nt), pk(x, m, n), right, trans, lower, alpha);
}

template <typename T>
dla_status trsm_fwd(int64_t batch, int64_t m, int64_t n, const T* t, T* x, int right, int trans, int lower,
                    T alpha, int32_t* info, void* stream) {
  if (bad_dims(batch, m, n)) return DLA_ERR_SHAPE;
  const int64_t nt = right ? n : m;
  if (overlap(x, bytes<T>(batch, m, n), t, bytes<T>(batch, nt, nt))) return DLA_ERR_ALIAS;
  Ctx cx = make_ctx(stream, info);
  DLAB_TRY(reset_info(cx, batch));
  return trsm<T>(cx, batch, m, n, cpk(t, nt, nt), pk(x, m, n), right, trans, lower, alpha, /*check_diag*/ true);
}

template <typename T>
dla_status trmm_bwd(int64_t batch, int64_t m, int64_t n, T* abar, T* tbar, const T* bbar, const T* t, const T* a,
                    int right, int trans, int lower, T alpha, void* stream) {
  if (bad_dims(batch, m, n)) return DLA_ERR_SHAPE;
  const int64_t nt = right ? n : m;
  const size_t xsz = bytes<T>(batch, m, n), tsz = bytes<T>(batch, nt, nt);
  if (overlap(tbar, tsz, bbar, xsz) || overlap(tbar, tsz, a, xsz) || overlap(abar, xsz, t, tsz) ||
      overlap(abar, xsz, tbar, tsz) || (abar != bbar && overlap(abar, xsz, bbar, xsz)))
    return DLA_ERR_ALIAS;
  Ctx cx = make_ctx(stream, nullptr);
  if (batch * m * n == 0) {
    if (batch * nt > 0) cudaMemsetAsync(tbar, 0, tsz, cx.stream);
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
  DLAB_TRY(ew_copy<T>(cx, batch, m, n, cpk(bbar, m, n), pk(abar, m, n)));
  return trmm<T>(cx, batch, m, n, cpk(t, nt, nt), pk(abar, m, n), right, !trans, lower, alpha);
}

template <typename T>
dla_status trsm_bwd(int64_t batch, int64_t m, int64_t n, T* abar, T* tbar, const T* bbar, const T* t, const T* b,
                    int right, int trans, int lower, T alpha, void* stream) {
  if (bad_dims(batch, m, n)) return DLA_ERR_SHAPE;
  const int64_t nt = right ? n : m;
  const size_t xsz = bytes<T>(batch, m, n), tsz = bytes<T>(batch, nt, nt);
  if (overlap(tbar, tsz, bbar, xsz) || overlap(tbar, tsz, b, xsz) || overlap(abar, xsz, t, tsz) ||
      overlap(abar, xsz, tbar, tsz) || overlap(abar, xsz, b, xsz) ||
      (abar != bbar && overlap(abar, xsz, bbar, xsz)))
    return DLA_ERR_ALIAS;
  Ctx cx = make_ctx(stream, nullptr);
  if (batch * m * n == 0) {
    if (batch * nt > 0) cudaMemsetAsync(tbar, 0, tsz, cx.stream);
    return DLA_OK;
  }
  // dl/adjoints.hpp:136-152: S = op(T)^{-T} Bbar in abar, then Tbar, then alpha.
  DLAB_TRY(ew_copy<T>(cx, batch, m, n, cpk(bbar, m, n), pk(abar, m, n)));
  DLAB_TRY(trsm<T>(cx, batch, m, n, cpk(t, nt, nt), pk(abar, m, n), right, !trans, lower, T(1)));
  MatB<T> tb = pk(tbar, nt, nt);
  const int mask = lower ? MASK_LOWER : MASK_UPPER;
  auto X = [&](const T* p) { return cpk(p, m, n); };
  const T* s = abar;
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
dla_status potrf_fwd(int64_t batch, int64_t n, T* a, int lower, int32_t* info, void* stream) {
  if (bad_dims(batch, n)) return DLA_ERR_SHAPE;
  Ctx cx = make_ctx(stream, info);
  DLAB_TRY(reset_info(cx, batch));
  if (batch * n == 0) return DLA_OK;
  if (potrf_small_eligible<T>(n)) return potrf_small<T>(cx, batch, n, pk(a, n, n), lower);
  DLAB_TRY(check_symmetric<T>(cx, batch, n, cpk(a, n, n), info));
  DLAB_TRY(potrf_lower<T>(cx, batch, n, pk(a, n, n)));
  if (!lower) DLAB_TRY(ew_square<T>(cx, batch, n, pk(a, n, n), /*transpose*/ 5, T(1), info));
  return DLA_OK;
}

template <typename T>
dla_status potrf_bwd(int64_t batch, int64_t n, T* abar, const T* lbar, const T* l, int lower, void* stream) {
  if (bad_dims(batch, n)) return DLA_ERR_SHAPE;
  const size_t sz = bytes<T>(batch, n, n);
  if (overlap(abar, sz, l, sz) || (abar != lbar && overlap(abar, sz, lbar, sz))) return DLA_ERR_ALIAS;
  Ctx cx = make_ctx(stream, nullptr);
  if (batch * n == 0) return DLA_OK;
  if (potrf_small_eligible<T>(n)) return potrf_bwd_small<T>(cx, batch, n, pk(abar, n, n), cpk(lbar, n, n),
                                                            cpk(l, n, n), lower);
  if (inv_eligible<T>(n)) return potrf_bwd_inv<T>(cx, batch, n, pk(abar, n, n), cpk(lbar, n, n), cpk(l, n, n), lower);
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
dla_status potri_fwd(int64_t batch, int64_t n, T* a, int lower, int32_t* info, void* stream) {
  if (bad_dims(batch, n)) return DLA_ERR_SHAPE;
  Ctx cx = make_ctx(stream, info);
  DLAB_TRY(reset_info(cx, batch));
  if (batch * n == 0) return DLA_OK;
  MatB<T> av = pk(a, n, n);
  if (!lower) DLAB_TRY(ew_square<T>(cx, batch, n, av, /*transpose*/ 5));
  DLAB_TRY(check_zero_diag<T>(cx, batch, n, C_(av), info));
  return potri_lower<T>(cx, batch, n, av);
}

template <typename T>
dla_status potri_bwd(int64_t batch, int64_t n, T* lbar, const T* bbar, const T* l, const T* b, int lower,
                     void* stream) {
  if (bad_dims(batch, n)) return DLA_ERR_SHAPE;
  const size_t sz = bytes<T>(batch, n, n);
  if (overlap(lbar, sz, bbar, sz) || overlap(lbar, sz, l, sz) || overlap(lbar, sz, b, sz)) return DLA_ERR_ALIAS;
  Ctx cx = make_ctx(stream, nullptr);
  if (batch * n == 0) return DLA_OK;
  MatB<T> lb = pk(lbar, n, n);
  MatB<const T> bv = cpk(b, n, n), bb = cpk(bbar, n, n), lv = cpk(l, n, n);
  // The reference forms B Bbar + B Bbar^T as two accumulated products
  // (dl/adjoints.hpp:211-212); here Bbar + Bbar^T is formed once (one n^2
  // pass) and multiplied once: half the O(n^3) work, same value.
  Scratch ws(bytes<T>(batch, n, n), cx.stream);
  if (!ws.p) return DLA_ERR_CUDA;
  MatB<T> sb = pk(ws.as<T>(), n, n);
  DLAB_TRY(ew_add_transpose<T>(cx, batch, n, bb, sb));
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
dla_status sld_fwd(int64_t batch, int64_t n, T* out, const T* a, void* stream) {
  if (bad_dims(batch, n)) return DLA_ERR_SHAPE;
  Ctx cx = make_ctx(stream, nullptr);
  return sumlogdiag_fwd<T>(cx, batch, n, out, cpk(a, n, n));
}

template <typename T>
dla_status sld_bwd(int64_t batch, int64_t n, T* abar, const T* g, const T* a, int accumulate, void* stream) {
  if (bad_dims(batch, n)) return DLA_ERR_SHAPE;
  const size_t sz = bytes<T>(batch, n, n);
  if (overlap(abar, sz, a, sz)) return DLA_ERR_ALIAS;
  Ctx cx = make_ctx(stream, nullptr);
  return sumlogdiag_bwd<T>(cx, batch, n, pk(abar, n, n), g, cpk(a, n, n), accumulate != 0);
}

// --------------------------------------------------------------- gelqf
template <typename T>
dla_status gelqf_fwd_abi(int64_t batch, int64_t m, int64_t n, T* q, T* l, int32_t* info, void* ws, size_t wsb,
                         void* stream) {
  if (bad_dims(batch, m, n) || m > n) return DLA_ERR_SHAPE;
  if (overlap(q, bytes<T>(batch, m, n), l, bytes<T>(batch, m, m))) return DLA_ERR_ALIAS;
  Ctx cx = make_ctx(stream, info);
  DLAB_TRY(reset_info(cx, batch));
  if (batch * m == 0) return DLA_OK;
  if (wsb < gelqf_ws_bytes<T>(batch, m, n, false)) return DLA_ERR_WORKSPACE;
  return gelqf_fwd<T>(cx, batch, m, n, q, l, ws);
}

template <typename T>
dla_status gelqf_bwd_abi(int64_t batch, int64_t m, int64_t n, T* abar, const T* qbar, const T* lbar, const T* q,
                         const T* l, void* ws, size_t wsb, void* stream) {
  if (bad_dims(batch, m, n) || m > n) return DLA_ERR_SHAPE;
  const size_t asz = bytes<T>(batch, m, n);
  if (overlap(abar, asz, q, asz) || overlap(abar, asz, l, bytes<T>(batch, m, m)) ||
      overlap(abar, asz, lbar, bytes<T>(batch, m, m)) || (abar != qbar && overlap(abar, asz, qbar, asz)))
    return DLA_ERR_ALIAS;
  Ctx cx = make_ctx(stream, nullptr);
  if (batch * m == 0) return DLA_OK;
  if (wsb < gelqf_ws_bytes<T>(batch, m, n, true) || !ws) return DLA_ERR_WORKSPACE;
  T* w = static_cast<T*>(ws);
  MatB<T> wv = pk(w, m, m);
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
dla_status syevd_fwd_abi(int64_t batch, int64_t n, T* u, T* lambda, int32_t* info, void* ws, size_t wsb,
                         void* stream) {
  if (bad_dims(batch, n)) return DLA_ERR_SHAPE;
  if (overlap(u, bytes<T>(batch, n, n), lambda, bytes<T>(batch, n, 1))) return DLA_ERR_ALIAS;
  Ctx cx = make_ctx(stream, info);
  DLAB_TRY(reset_info(cx, batch));
  if (batch * n == 0) return DLA_OK;
  if (wsb < syevd_ws_bytes<T>(batch, n, false)) return DLA_ERR_WORKSPACE;
  return syevd_fwd<T>(cx, batch, n, u, lambda, ws);
}

template <typename T>
dla_status syevd_bwd_abi(int64_t batch, int64_t n, T* abar, const T* ubar, const T* lambdabar, const T* u,
                         const T* lambda, T eps_gap, void* ws, size_t wsb, void* stream) {
  if (bad_dims(batch, n)) return DLA_ERR_SHAPE;
  const size_t sz = bytes<T>(batch, n, n);
  if (overlap(abar, sz, ubar, sz) || overlap(abar, sz, u, sz)) return DLA_ERR_ALIAS;
  if (!(eps_gap > T(0))) return DLA_ERR_INVALID;
  Ctx cx = make_ctx(stream, nullptr);
  if (batch * n == 0) return DLA_OK;
  if (wsb < syevd_ws_bytes<T>(batch, n, true) || !ws) return DLA_ERR_WORKSPACE;
  MatB<T> w = pk(static_cast<T*>(ws), n, n);
  MatB<const T> uv = cpk(u, n, n);
  // dl/adjoints.hpp:277-294
  DLAB_TRY(gemm<T>(cx, batch, n, n, n, T(1), cpk(ubar, n, n), false, uv, true, T(0), w));
  DLAB_TRY(syevd_gap_kernel<T>(cx, batch, n, w, lambdabar, lambda, eps_gap));
  DLAB_TRY(gemm<T>(cx, batch, n, n, n, T(1), uv, true, C_(w), false, T(0), pk(abar, n, n)));
  DLAB_TRY(gemm<T>(cx, batch, n, n, n, T(1), cpk(abar, n, n), false, uv, false, T(0), w));
  return ew_sym_into<T>(cx, batch, n, C_(w), pk(abar, n, n));
}

}  // namespace
}  // namespace dlab

using namespace dlab;

// ------------------------------------------------- fused C1 chain (GP NLL)
__global__ void k_fill_ones(int64_t n, double* pd, float* pf) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    if (pd) pd[i] = 1.0;
    if (pf) pf[i] = 1.0f;
  }
}

// phi = 1/2 |L^-1 y|^2 + sumlogdiag(L), L = potrf(A); ybar, Abar at phibar = 1.
// n <= 32: one fused warp-per-matrix launch (small.cu); otherwise the
// operator chain (the reference's own composition) on stream-ordered scratch.
template <typename T>
dla_status chol_chain_abi(int64_t batch, int64_t n, const T* a, const T* y, T* phi, T* abar, T* ybar,
                          int32_t* info, void* stream) {
  if (bad_dims(batch, n)) return DLA_ERR_SHAPE;
  const size_t asz = bytes<T>(batch, n, n), ysz = bytes<T>(batch, n, 1), psz = bytes<T>(batch, 1, 1);
  if (overlap(abar, asz, a, asz) || overlap(abar, asz, y, ysz) || overlap(ybar, ysz, a, asz) ||
      overlap(ybar, ysz, y, ysz) || overlap(phi, psz, a, asz) || overlap(phi, psz, y, ysz) ||
      overlap(abar, asz, ybar, ysz) || overlap(phi, psz, abar, asz) || overlap(phi, psz, ybar, ysz))
    return DLA_ERR_ALIAS;
  Ctx cx = make_ctx(stream, info);
  DLAB_TRY(reset_info(cx, batch));
  if (batch == 0) return DLA_OK;
  if (n == 0) return cudaMemsetAsync(phi, 0, psz, cx.stream) == cudaSuccess ? DLA_OK : DLA_ERR_CUDA;
  if (n <= 32) return chol_chain_small<T>(cx, batch, n, cpk(a, n, n), y, phi, pk(abar, n, n), ybar);
  Scratch ws(asz + ysz + psz, cx.stream);
  if (!ws.p) return DLA_ERR_CUDA;
  T* l = ws.as<T>();
  T* z = l + batch * n * n;
  T* ones = z + batch * n;
  k_fill_ones<<<blocks_for(batch, 256), 256, 0, cx.stream>>>(batch, sizeof(T) == 8 ? (double*)ones : nullptr,
                                                             sizeof(T) == 4 ? (float*)ones : nullptr);
  DLAB_LAUNCH_CHECK();
  if (cudaMemcpyAsync(l, a, asz, cudaMemcpyDeviceToDevice, cx.stream) != cudaSuccess ||
      cudaMemcpyAsync(z, y, ysz, cudaMemcpyDeviceToDevice, cx.stream) != cudaSuccess)
    return DLA_ERR_CUDA;
  DLAB_TRY(potrf_fwd<T>(batch, n, l, 1, info, stream));
  // later ops skip failed slices through info (dl/matrix.hpp:232-239 semantics)
  DLAB_TRY(trsm<T>(cx, batch, n, 1, cpk(l, n, n), pk(z, n, 1), false, false, true, T(1)));
  DLAB_TRY(sumlogdiag_fwd<T>(cx, batch, n, phi, cpk(l, n, n)));
  DLAB_TRY(gemm<T>(cx, batch, 1, 1, n, T(0.5), cpk(z, n, 1), true, cpk(z, n, 1), false, T(1), pk(phi, 1, 1)));
  DLAB_TRY(trsm_bwd<T>(batch, n, 1, ybar, abar, z, l, z, 0, 0, 1, T(1), stream));
  DLAB_TRY(sumlogdiag_bwd<T>(cx, batch, n, pk(abar, n, n), ones, cpk(l, n, n), true));
  return potrf_bwd<T>(batch, n, abar, abar, l, 1, stream);
}

// ------------------------------------------- split potrf pullback (drivers)
// L^{-1} for the inverse-based potrf pullback computed on a side stream
// forked from the caller's stream, so a driver can overlap it with work
// that only needs L (the GP driver's solves).  One begin/end pair in flight
// per process; both halves are stream-ordered and graph-capturable.
struct InvFork {
  cudaStream_t side = nullptr;
  cudaEvent_t fork = nullptr, done = nullptr;
  static InvFork& get() {
    static InvFork f;
    static std::once_flag once;
    std::call_once(once, [] {
      int lo = 0, hi = 0;
      cudaDeviceGetStreamPriorityRange(&lo, &hi);
      cudaStreamCreateWithPriority(&f.side, cudaStreamNonBlocking, lo);
      cudaEventCreateWithFlags(&f.fork, cudaEventDisableTiming);
      cudaEventCreateWithFlags(&f.done, cudaEventDisableTiming);
    });
    return f;
  }
};

template <typename T>
size_t potrf_inv_ws(int64_t batch, int64_t n) {
  // wi (n^2) | tt (n^2) | tmp (trtri_levels_tmp(n) bytes) | tmp2 (trtri_levels_tmp(n / 2) bytes)
  return sizeof(T) * (size_t)batch * 2 * (size_t)n * n + (size_t)batch * trtri_levels_tmp<T>(n) +
         (size_t)batch * trtri_levels_tmp<T>(n / 2);
}

template <typename T>
dla_status potrf_bwd_begin(int64_t batch, int64_t n, const T* l, int lower, void* ws, size_t wsb, void* stream) {
  if (bad_dims(batch, n)) return DLA_ERR_SHAPE;
  if (batch * n == 0 || !inv_eligible<T>(n)) return DLA_OK;  // end() takes the direct path
  if (!ws || wsb < potrf_inv_ws<T>(batch, n)) return DLA_ERR_WORKSPACE;
  Ctx cx = make_ctx(stream, nullptr);
  InvFork& f = InvFork::get();
  Ctx side = cx;
  side.stream = f.side;
  cudaEventRecord(f.fork, cx.stream);
  cudaStreamWaitEvent(f.side, f.fork, 0);
  T* wp = static_cast<T*>(ws);
  DLAB_TRY(potrf_inv_prepare<T>(side, batch, n, cpk(l, n, n), lower != 0, pk(wp, n, n), wp + 2 * batch * n * n));
  cudaEventRecord(f.done, f.side);
  return DLA_OK;
}

template <typename T>
dla_status potrf_bwd_end(int64_t batch, int64_t n, T* abar, const T* lbar, const T* l, int lower, void* ws,
                         size_t wsb, void* stream) {
  if (bad_dims(batch, n)) return DLA_ERR_SHAPE;
  if (batch * n == 0 || !inv_eligible<T>(n)) return potrf_bwd<T>(batch, n, abar, lbar, l, lower, stream);
  const size_t sz = bytes<T>(batch, n, n);
  if (overlap(abar, sz, l, sz) || (abar != lbar && overlap(abar, sz, lbar, sz))) return DLA_ERR_ALIAS;
  if (!ws || wsb < potrf_inv_ws<T>(batch, n)) return DLA_ERR_WORKSPACE;
  Ctx cx = make_ctx(stream, nullptr);
  T* wp = static_cast<T*>(ws);
  MatB<T> tt = pk(wp + batch * n * n, n, n);
  // P' needs only L and Lbar: it overlaps the inverse still running on the side stream
  DLAB_TRY(potrf_bwd_phi<T>(cx, batch, n, cpk(lbar, n, n), cpk(l, n, n), lower != 0, tt));
  cudaStreamWaitEvent(cx.stream, InvFork::get().done, 0);
  return potrf_bwd_finish<T>(cx, batch, n, pk(abar, n, n), cpk(wp, n, n), tt);
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
  cudaStream_t side;
  cudaEvent_t ev;
  bool fired;
};

template <typename T>
void early_inv_first(void* user, cudaStream_t crit) {
  EarlyInv<T>& e = *static_cast<EarlyInv<T>*>(user);
  e.fired = true;
  const int64_t n = e.n, h = n / 2, B = e.batch;
  cudaEventRecord(e.ev, crit);
  cudaStreamWaitEvent(e.side, e.ev, 0);
  Ctx sc = make_ctx(e.side, nullptr);
  MatB<T> wi{e.wp, n, n * n};
  T* tmp = e.wp + 2 * B * n * n;
  MatB<const T> lv{e.l, n, n * n};
  // W11 = tril(L11), W21 = L21; L11^{-1} in place; T1 = W21 W11^{-1} into tmp
  if (ew_tri_copy<T>(sc, B, h, lv, wi, false) != DLA_OK) return;
  if (ew_copy<T>(sc, B, h, h, MatB<const T>{e.l + h * n, n, n * n}, wi.sub(h, 0)) != DLA_OK) return;
  T* tmp2 = tmp + B * (trtri_levels_tmp<T>(n) / sizeof(T));
  if (trtri_levels<T>(sc, B, h, wi, tmp2) != DLA_OK) return;
  MatB<T> t1{tmp, h, h * h};
  gemm<T>(sc, B, h, h, h, T(1), MatB<const T>{wi.p + h * n, n, n * n}, false, MatB<const T>{wi.p, n, n * n}, false,
          T(0), t1, MASK_FULL, nullptr, TRI_NONE, TRI_LOWER);
}

template <typename T>
dla_status gp_potrf_inv(int64_t batch, int64_t n, T* a, int32_t* info, void* ws, size_t wsb, void* stream) {
  if (bad_dims(batch, n)) return DLA_ERR_SHAPE;
  if (!inv_eligible<T>(n) || batch * n == 0) {  // no early path: factorization, then the plain begin
    DLAB_TRY(potrf_fwd<T>(batch, n, a, 1, info, stream));
    return potrf_bwd_begin<T>(batch, n, a, 1, ws, wsb, stream);
  }
  if (!ws || wsb < potrf_inv_ws<T>(batch, n)) return DLA_ERR_WORKSPACE;
  Ctx cx = make_ctx(stream, info);
  DLAB_TRY(reset_info(cx, batch));
  DLAB_TRY(check_symmetric<T>(cx, batch, n, cpk(a, n, n), info));
  InvFork& f = InvFork::get();
  static cudaEvent_t mid = nullptr, fin = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    cudaEventCreateWithFlags(&mid, cudaEventDisableTiming);
    cudaEventCreateWithFlags(&fin, cudaEventDisableTiming);
  });
  EarlyInv<T> e{batch, n, a, static_cast<T*>(ws), f.side, mid, false};
  PotrfHook hook{n / 2, early_inv_first<T>, &e, a, n};
  Ctx hc = cx;
  hc.potrf_hook = &hook;
  DLAB_TRY(potrf_lower<T>(hc, batch, n, pk(a, n, n), /*zero_upper*/ false));
  if (!e.fired) early_inv_first<T>(&e, cx.stream);  // a schedule without the hook point (tuning modes)
  const int64_t h = n / 2;
  T* wp = static_cast<T*>(ws);
  MatB<T> wi{wp, n, n * n};
  T* tmp = wp + 2 * batch * n * n;
  T* tmp2 = tmp + batch * (trtri_levels_tmp<T>(n) / sizeof(T));
  cudaEventRecord(fin, cx.stream);
  cudaStreamWaitEvent(f.side, fin, 0);
  Ctx sc = make_ctx(f.side, nullptr);
  // W22 = tril(L22); L22^{-1} in place; W21 = -W22^{-1} T1
  DLAB_TRY(ew_tri_copy<T>(sc, batch, h, MatB<const T>{a + h * n + h, n, n * n}, wi.sub(h, h), false));
  DLAB_TRY(trtri_levels<T>(sc, batch, h, wi.sub(h, h), tmp2));
  DLAB_TRY(gemm<T>(sc, batch, h, h, h, T(-1), MatB<const T>{wi.p + h * n + h, n, n * n}, false,
                   MatB<const T>{tmp, h, h * h}, false, T(0), wi.sub(h, 0), MASK_FULL, nullptr, TRI_LOWER,
                   TRI_NONE));
  // L's strict upper triangle (the potrf contract) is zeroed here, on the side
  // stream: no kernel of the step reads it, so it stays off the critical path
  // and is complete once dla_potrf_bwd_end_f64 has joined `done`
  DLAB_TRY(ew_square<T>(sc, batch, n, pk(a, n, n), /*tril*/ 0, T(1), info));
  cudaEventRecord(f.done, f.side);
  return DLA_OK;
}



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
  (void)k;
  const bool bwd = (phase & DLA_WS_BACKWARD) != 0;
  if (op == DLA_OP_GELQF)
    return dtype == DLA_F64 ? gelqf_ws_bytes<double>(batch, m, n, bwd) : gelqf_ws_bytes<float>(batch, m, n, bwd);
  if (op == DLA_OP_SYEVD)
    return dtype == DLA_F64 ? syevd_ws_bytes<double>(batch, n, bwd) : syevd_ws_bytes<float>(batch, n, bwd);
  return 0;
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

#define DLA_DEFINE(T, S)                                                                                          \
  dla_status dla_gemm2_fwd_##S(int64_t batch, int64_t m, int64_t n, int64_t k, T* c, const T* a, const T* b,      \
                               int ta, int tb, T alpha, void* stream) {                                          \
    return gemm_fwd<T>(batch, m, n, k, c, a, b, ta, tb, alpha, T(0), stream);                                    \
  }                                                                                                               \
  dla_status dla_gemm_fwd_##S(int64_t batch, int64_t m, int64_t n, int64_t k, T* c, const T* a, const T* b,       \
                              int ta, int tb, T alpha, T beta, void* stream) {                                   \
    return gemm_fwd<T>(batch, m, n, k, c, a, b, ta, tb, alpha, beta, stream);                                    \
  }                                                                                                               \
  dla_status dla_gemm2_bwd_##S(int64_t batch, int64_t m, int64_t n, int64_t k, T* abar, T* bbar, const T* cbar,   \
                               const T* a, const T* b, int ta, int tb, T alpha, void* stream) {                  \
    return gemm_bwd<T>(batch, m, n, k, abar, bbar, const_cast<T*>(cbar), a, b, ta, tb, alpha, T(0), false,       \
                       stream);                                                                                   \
  }                                                                                                               \
  dla_status dla_gemm_bwd_##S(int64_t batch, int64_t m, int64_t n, int64_t k, T* abar, T* bbar, T* cbar_io,       \
                              const T* a, const T* b, int ta, int tb, T alpha, T beta, void* stream) {           \
    return gemm_bwd<T>(batch, m, n, k, abar, bbar, cbar_io, a, b, ta, tb, alpha, beta, true, stream);            \
  }                                                                                                               \
  dla_status dla_syrk_fwd_##S(int64_t batch, int64_t n, int64_t k, T* b, const T* a, int ta, T alpha,             \
                              void* stream) {                                                                     \
    return syrk_fwd<T>(batch, n, k, b, a, ta, alpha, stream);                                                     \
  }                                                                                                               \
  dla_status dla_syrk_bwd_##S(int64_t batch, int64_t n, int64_t k, T* abar, const T* bbar, const T* a, int ta,    \
                              T alpha, void* stream) {                                                            \
    return syrk_bwd<T>(batch, n, k, abar, bbar, a, ta, alpha, stream);                                            \
  }                                                                                                               \
  dla_status dla_trmm_fwd_##S(int64_t batch, int64_t m, int64_t n, const T* t, T* x, int r, int tr, int lo,       \
                              T alpha, void* stream) {                                                            \
    return trmm_fwd<T>(batch, m, n, t, x, r, tr, lo, alpha, stream);                                              \
  }                                                                                                               \
  dla_status dla_trmm_bwd_##S(int64_t batch, int64_t m, int64_t n, T* abar, T* tbar, const T* bbar, const T* t,   \
                              const T* a, int r, int tr, int lo, T alpha, void* stream) {                        \
    return trmm_bwd<T>(batch, m, n, abar, tbar, bbar, t, a, r, tr, lo, alpha, stream);                            \
  }                                                                                                               \
  dla_status dla_trsm_fwd_##S(int64_t batch, int64_t m, int64_t n, const T* t, T* x, int r, int tr, int lo,       \
                              T alpha, int32_t* info, void* stream) {                                             \
    return trsm_fwd<T>(batch, m, n, t, x, r, tr, lo, alpha, info, stream);                                        \
  }                                                                                                               \
  dla_status dla_trsm_bwd_##S(int64_t batch, int64_t m, int64_t n, T* abar, T* tbar, const T* bbar, const T* t,   \
                              const T* b, int r, int tr, int lo, T alpha, void* stream) {                        \
    return trsm_bwd<T>(batch, m, n, abar, tbar, bbar, t, b, r, tr, lo, alpha, stream);                            \
  }                                                                                                               \
  dla_status dla_potrf_fwd_##S(int64_t batch, int64_t n, T* a, int lower, int32_t* info, void* stream) {         \
    return potrf_fwd<T>(batch, n, a, lower, info, stream);                                                        \
  }                                                                                                               \
  dla_status dla_potrf_bwd_##S(int64_t batch, int64_t n, T* abar, const T* lbar, const T* l, int lower,           \
                               void* stream) {                                                                    \
    return potrf_bwd<T>(batch, n, abar, lbar, l, lower, stream);                                                  \
  }                                                                                                               \
  dla_status dla_potri_fwd_##S(int64_t batch, int64_t n, T* a, int lower, int32_t* info, void* stream) {         \
    return potri_fwd<T>(batch, n, a, lower, info, stream);                                                        \
  }                                                                                                               \
  dla_status dla_potri_bwd_##S(int64_t batch, int64_t n, T* lbar, const T* bbar, const T* l, const T* b,          \
                               int lower, void* stream) {                                                         \
    return potri_bwd<T>(batch, n, lbar, bbar, l, b, lower, stream);                                              \
  }                                                                                                               \
  dla_status dla_sumlogdiag_fwd_##S(int64_t batch, int64_t n, T* out, const T* a, void* stream) {                \
    return sld_fwd<T>(batch, n, out, a, stream);                                                                  \
  }                                                                                                               \
  dla_status dla_sumlogdiag_bwd_##S(int64_t batch, int64_t n, T* abar, const T* gbar, const T* a,                 \
                                    int accumulate, void* stream) {                                               \
    return sld_bwd<T>(batch, n, abar, gbar, a, accumulate, stream);                                               \
  }                                                                                                               \
  dla_status dla_gelqf_fwd_##S(int64_t batch, int64_t m, int64_t n, T* q, T* l, int32_t* info, void* ws,         \
                               size_t ws_bytes, void* stream) {                                                   \
    return gelqf_fwd_abi<T>(batch, m, n, q, l, info, ws, ws_bytes, stream);                                       \
  }                                                                                                               \
  dla_status dla_gelqf_bwd_##S(int64_t batch, int64_t m, int64_t n, T* abar, const T* qbar, const T* lbar,        \
                               const T* q, const T* l, void* ws, size_t ws_bytes, void* stream) {                \
    return gelqf_bwd_abi<T>(batch, m, n, abar, qbar, lbar, q, l, ws, ws_bytes, stream);                           \
  }                                                                                                               \
  dla_status dla_syevd_fwd_##S(int64_t batch, int64_t n, T* u, T* lambda, int32_t* info, void* ws,               \
                               size_t ws_bytes, void* stream) {                                                   \
    return syevd_fwd_abi<T>(batch, n, u, lambda, info, ws, ws_bytes, stream);                                     \
  }                                                                                                               \
  dla_status dla_syevd_bwd_##S(int64_t batch, int64_t n, T* abar, const T* ubar, const T* lambdabar, const T* u,  \
                               const T* lambda, T eps_gap, void* ws, size_t ws_bytes, void* stream) {            \
    return syevd_bwd_abi<T>(batch, n, abar, ubar, lambdabar, u, lambda, eps_gap, ws, ws_bytes, stream);           \
  }

DLA_DEFINE(float, f32)
DLA_DEFINE(double, f64)

size_t dla_potrf_bwd_ws_bytes_f64(int64_t batch, int64_t n) {
  return inv_eligible<double>(n) ? potrf_inv_ws<double>(batch, n) : 0;
}
dla_status dla_gp_potrf_inv_f64(int64_t batch, int64_t n, double* a, int32_t* info, void* ws, size_t ws_bytes,
                                void* stream) {
  return gp_potrf_inv<double>(batch, n, a, info, ws, ws_bytes, stream);
}
dla_status dla_potrf_bwd_begin_f64(int64_t batch, int64_t n, const double* l, int lower, void* ws, size_t ws_bytes,
                                   void* stream) {
  return potrf_bwd_begin<double>(batch, n, l, lower, ws, ws_bytes, stream);
}
dla_status dla_potrf_bwd_end_f64(int64_t batch, int64_t n, double* abar, const double* lbar, const double* l,
                                 int lower, void* ws, size_t ws_bytes, void* stream) {
  return potrf_bwd_end<double>(batch, n, abar, lbar, l, lower, ws, ws_bytes, stream);
}

dla_status dla_chol_chain_fwdbwd_f64(int64_t batch, int64_t n, const double* a, const double* y, double* phi,
                                     double* abar, double* ybar, int32_t* info, void* stream) {
  return chol_chain_abi<double>(batch, n, a, y, phi, abar, ybar, info, stream);
}
dla_status dla_chol_chain_fwdbwd_f32(int64_t batch, int64_t n, const float* a, const float* y, float* phi,
                                     float* abar, float* ybar, int32_t* info, void* stream) {
  return chol_chain_abi<float>(batch, n, a, y, phi, abar, ybar, info, stream);
}

}  // extern "C"
