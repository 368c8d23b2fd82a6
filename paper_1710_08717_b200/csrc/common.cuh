// Shared device/host plumbing for libdla_b200.so (sm_100a only).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdio>
#include <mutex>
#include <vector>

#include "../../include/dla.h"

#if defined(__CUDA_ARCH__) && (__CUDA_ARCH__ < 1000)
#error "libdla_b200 is built for sm_100a only"
#endif

namespace dlab {

// Batched strided matrix view: element (b, i, j) at p[b*bs + i*ld + j].
// Row-major like the reference's MatrixView (dl/matrix.hpp:64-89), with an
// explicit leading dimension so blocked algorithms address sub-blocks
// in place.
// `bsi` is an optional inner batch stride (GEMM only): the level-batched
// triangular inverse addresses all diagonal blocks of one matrix as an inner
// batch.
template <typename T>
struct MatB {
  T* p;
  int64_t ld;
  int64_t bs;
  int64_t bsi = 0;
  __host__ __device__ T* at(int64_t b, int64_t i, int64_t j) const {
    return p + b * bs + i * ld + j;
  }
  __host__ __device__ MatB sub(int64_t i, int64_t j) const { return MatB{p + i * ld + j, ld, bs, bsi}; }
};

// Triangular-operand flags for gemm(): op(A) / op(B) is lower / upper
// triangular (the other triangle is ignored, whatever memory holds there).
enum Tri : int { TRI_NONE = 0, TRI_LOWER = 1, TRI_UPPER = 2 };

template <typename T>
inline MatB<T> packed(T* p, int64_t rows, int64_t cols) {
  (void)rows;
  return MatB<T>{p, cols, rows * cols};
}

// Optional hook into the blocked Cholesky: fn(user, crit) is called once,
// right after the panel launch that completes block columns [0, col), with
// the critical stream (so `user` can order work after that point).
struct PotrfHook {
  int64_t col;
  void (*fn)(void* user, cudaStream_t crit);
  void* user;
  const void* a;  // the factorization it belongs to: fires only in the blocked loop over this
  int64_t n;      // whole matrix (a recursive schedule's sub-blocks are not final at `col`)
};

// Caller-owned device workspace (include/dla.h: "no entry point allocates
// device memory").  One top-level C-ABI call carves it monotonically -- no
// region is reused within the call, so scratch handed to work on a forked
// side stream stays valid until the call joins that stream back.  The bytes
// a call needs are computed host-side by the ws_* mirrors (ws.cu) of the same
// dispatch; carve_bound() is the per-carve bound they use (size rounded up
// to the 256-byte carve alignment plus the worst-case alignment skip).
constexpr size_t kCarveAlign = 256;
constexpr size_t carve_bound(size_t bytes) {
  return bytes ? (bytes + kCarveAlign - 1) / kCarveAlign * kCarveAlign + kCarveAlign : 0;
}

struct Arena {
  char* base = nullptr;
  size_t cap = 0;
  size_t off = 0;
  Arena() = default;
  Arena(void* p, size_t bytes) : base(static_cast<char*>(p)), cap(p ? bytes : 0) {}
  void* take(size_t bytes) {
    if (!bytes) return nullptr;
    const uintptr_t cur = reinterpret_cast<uintptr_t>(base) + off;
    const uintptr_t al = (cur + kCarveAlign - 1) / kCarveAlign * kCarveAlign;
    const size_t need = (size_t)(al - reinterpret_cast<uintptr_t>(base)) + bytes;
    if (!base || need > cap) return nullptr;
    off = need;
    return reinterpret_cast<void*>(al);
  }
};

// Launch context: stream + device properties + optional per-slice info +
// the call's workspace arena.
struct Ctx {
  cudaStream_t stream;
  int sms;
  int32_t* info;       // nullable: device int32[batch]
  int gemm_ctas = 0;   // > 0: DMMA GEMMs run persistent on at most this many CTAs
  int gemm_rowtile = 0;  // 1: (f64, m <= 128) one 128-row tile per column block, so C may alias op(B)
  const PotrfHook* potrf_hook = nullptr;
  Arena* arena = nullptr;  // the call's workspace (shared by every copy of this Ctx)
};

// SM count of the CURRENT device (cached per device, read-only after first use).
Ctx make_ctx(void* stream, int32_t* info, Arena* arena = nullptr);

// Dynamic shared-memory opt-in of a kernel on the current device: thread-safe,
// set once per (device, kernel) and raised if a larger size is requested.
void smem_opt_in(const void* func, size_t bytes);
template <typename K>
inline void ensure_smem_attr(K* kernel, size_t bytes) {
  smem_opt_in(reinterpret_cast<const void*>(kernel), bytes);
}

// Side streams + events for the fork/join schedules, one set per (device,
// caller stream, user): concurrent calls on different streams (or devices)
// never share an event, and a caller holds `mu` for its whole enqueue, so
// two host threads on one stream serialise instead of re-recording each
// other's events.  Created on first use, owned by the library, read-only
// thereafter except for the lock.
enum ForkKind : int { FORK_LOOKAHEAD = 0, FORK_INV = 1, FORK_BWDINV = 2 };
struct ForkRes {
  std::mutex mu;
  cudaStream_t side = nullptr;  // lowest priority
  cudaStream_t crit = nullptr;  // highest priority (the potrf panel chain)
  int prio_hi = 0;
  cudaEvent_t ev[6] = {};
  std::vector<cudaEvent_t> panel, done;  // per look-ahead step (grown under mu)
  void grow(int64_t steps);
};
ForkRes& fork_res(ForkKind kind, cudaStream_t caller);

// Host-side count of kernels this library launched (bench.py's gpu_launches
// claim) and optional CUDA-event timing of every GEMM launch (roofline).
void note_launch(int k = 1);
bool gemm_prof_on();
void gemm_prof_begin(cudaStream_t s);
void gemm_prof_end(cudaStream_t s, double flops);
void gemm_prof_cancel();

// Scratch carved from the call's workspace arena; `ok` is false when the
// caller's workspace is missing or too small (the op returns
// DLA_ERR_WORKSPACE -- there is no hidden allocation behind it).
struct Scratch {
  void* p = nullptr;
  bool ok = true;
  Scratch(const Ctx& c, size_t bytes) {
    if (!bytes) return;
    p = c.arena ? c.arena->take(bytes) : nullptr;
    ok = p != nullptr;
  }
  Scratch(const Scratch&) = delete;
  Scratch& operator=(const Scratch&) = delete;
  template <typename T>
  T* as() const {
    return static_cast<T*>(p);
  }
};

#define DLAB_SCRATCH(name, ctx, bytes) \
  Scratch name((ctx), (bytes));        \
  if (!name.ok) return DLA_ERR_WORKSPACE

inline unsigned blocks_for(int64_t work, int threads, int64_t cap = 148 * 32) {
  int64_t b = (work + threads - 1) / threads;
  if (b < 1) b = 1;
  if (b > cap) b = cap;
  return (unsigned)b;
}

// Skip rule shared by every kernel: a slice whose info is already set is
// left untouched (the reference throws before writing, dl/blas.hpp:310-314).
__device__ __forceinline__ bool slice_failed(const int32_t* info, int64_t b) {
  return info != nullptr && info[b] != 0;
}

// First-failure-wins recording (serial block order => lowest index wins).
__device__ __forceinline__ void record_failure(int32_t* info, int64_t b, int code, int64_t index) {
  if (info != nullptr) atomicCAS(info + b, 0, DLA_INFO(code, index));
}

template <typename T>
struct Num;
template <>
struct Num<double> {
  __device__ static double sqrt_(double x) { return sqrt(x); }
  __device__ static double log_(double x) { return log(x); }
  // Branch-free 1/sqrt: MUFU.RSQ64H seed + two Newton steps (<= ~1 ulp for
  // normal positive x).  The library rsqrt() carries a special-case slow path
  // whose call/reconvergence code wraps every warp shuffle of the Cholesky
  // pivot chain; non-positive / NaN pivots still yield NaN here and are
  // caught by the callers' !(d > 0) test.
  __device__ static double rsqrt_(double x) {
    double y;
    asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
    double e = fma(-x, y * y, 1.0);
    y = fma(0.5 * y, e, y);
    e = fma(-x, y * y, 1.0);
    return fma(0.5 * y, e, y);
  }
  // Branch-free 1/x: MUFU.RCP64H seed + two Newton steps (finite nonzero x)
  __device__ static double rcp_(double x) {
    double y;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
    double e = fma(-x, y, 1.0);
    y = fma(y, e, y);
    e = fma(-x, y, 1.0);
    return fma(y, e, y);
  }
  static constexpr double sym_rtol = 1e-10;
  static constexpr double rank_rtol = 1e-12;
};
template <>
struct Num<float> {
  __device__ static float sqrt_(float x) { return sqrtf(x); }
  __device__ static float log_(float x) { return logf(x); }
  __device__ static float rsqrt_(float x) {  // MUFU seed + one Newton step, branch-free
    const float y = rsqrtf(x);
    return fmaf(0.5f * y, fmaf(-x, y * y, 1.0f), y);
  }
  __device__ static float rcp_(float x) { return 1.0f / x; }
  static constexpr float sym_rtol = 1e-4f;
  static constexpr float rank_rtol = 1e-5f;
};

#define DLAB_LAUNCH_CHECK()                                  \
  do {                                                       \
    cudaError_t e_ = cudaGetLastError();                     \
    if (e_ != cudaSuccess) {                                 \
      fprintf(stderr, "dla_b200: %s (%s:%d)\n", cudaGetErrorString(e_), __FILE__, __LINE__); \
      return DLA_ERR_CUDA;                                   \
    }                                                        \
    note_launch(1);                                          \
  } while (0)

// Status of the kernel launch just issued (counts it on success).
inline dla_status launch_status() {
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    fprintf(stderr, "dla_b200: %s\n", cudaGetErrorString(e));
    return DLA_ERR_CUDA;
  }
  note_launch(1);
  return DLA_OK;
}

#define DLAB_TRY(expr)              \
  do {                              \
    dla_status s_ = (expr);         \
    if (s_ != DLA_OK) return s_;    \
  } while (0)

// Triangle masks for the GEMM epilogue / elementwise kernels.
enum Mask : int { MASK_FULL = 0, MASK_LOWER = 1, MASK_UPPER = 2 };

// ----------------------------------------------------------------- kernels
// gemm.cu: C = alpha op(A) op(B) + beta C over a batch (beta == 0 => C is
// not read).  mask restricts writes to the lower/upper triangle of C
// (global (i,j) of this C view); masked-out tiles do no math.
// tri_a / tri_b: op(A) / op(B) triangular (K range restricted per tile, the
// ignored triangle masked to zero).  inner > 1: each of the `batch` slices is
// itself an inner batch of `inner` problems at the operands' bsi strides.
template <typename T>
dla_status gemm(const Ctx& c, int64_t batch, int64_t m, int64_t n, int64_t k, T alpha, MatB<const T> a,
                bool ta, MatB<const T> b, bool tb, T beta, MatB<T> cm, int mask = MASK_FULL,
                const int32_t* skip = nullptr, int tri_a = TRI_NONE, int tri_b = TRI_NONE, int64_t inner = 1);

// gemm_tc.cu: fp32 on tcgen05 (3xTF32); false = not handled
bool sgemm_tc(const Ctx& c, int64_t batch, int64_t m, int64_t n, int64_t k, float alpha, MatB<const float> a, bool ta,
              MatB<const float> b, bool tb, float beta, MatB<float> cm, int mask, const int32_t* skip, int tri_a,
              int tri_b, int64_t inner, dla_status* st);

// skinny.cu: n <= 8, m <= 8 or k <= 8 without triangular operands; returns
// false when the shape is not skinny (the caller runs the tiled GEMM).
template <typename T>
bool gemm_skinny(const Ctx& c, int64_t batch, int64_t m, int64_t n, int64_t k, T alpha, MatB<const T> a, bool ta,
                 MatB<const T> b, bool tb, T beta, MatB<T> cm, int mask, const int32_t* skip, dla_status* st);

// C (m x n) = alpha * mask(op(A) op(B)) with exact zeros outside the mask,
// k <= 8, one pass (false: not applicable).
template <typename T>
bool outer_tri(const Ctx& c, int64_t batch, int64_t m, int64_t n, int64_t k, T alpha, MatB<const T> a, bool ta,
               MatB<const T> b, bool tb, MatB<T> cm, int mask, const int32_t* skip, dla_status* st);

// Workspace mirrors: the bytes (carve_bound per carve, summed over the call
// tree) each routine takes from its Ctx's arena, computed host-side from the
// same shapes and eligibility tests as the dispatch (no device needed).
template <typename T>
size_t ws_gemm(int64_t batch, int64_t m, int64_t n, int64_t k, int64_t inner = 1);
size_t sgemm_tc_ws_bytes(int64_t batch, int64_t m, int64_t n, int64_t k);
template <typename T>
size_t ws_trsm(int64_t batch, int64_t m, int64_t n, bool right);
template <typename T>
size_t ws_trmm(int64_t batch, int64_t m, int64_t n, bool right);
template <typename T>
size_t ws_potrf_lower(int64_t batch, int64_t n);
template <typename T>
size_t ws_potri_lower(int64_t batch, int64_t n);

// elementwise.cu
template <typename T>
dla_status ew_copy(const Ctx& c, int64_t batch, int64_t m, int64_t n, MatB<const T> src, MatB<T> dst,
                   const int32_t* skip = nullptr);
template <typename T>
dla_status ew_scale(const Ctx& c, int64_t batch, int64_t m, int64_t n, MatB<T> x, T alpha,
                    const int32_t* skip = nullptr);
// op: 0 tril, 1 triu, 2 copyltu, 3 copyutl, 4 sym, 5 transpose, 6 scaled sym (x*alpha then sym)
template <typename T>
dla_status ew_square(const Ctx& c, int64_t batch, int64_t n, MatB<T> x, int op, T alpha = T(1),
                     const int32_t* skip = nullptr);
// dst = lower-triangular form of src's selected triangle (from_upper: dst(i,j)
// = src(j,i) for j <= i), strict upper of dst zeroed.
template <typename T>
dla_status ew_tri_copy(const Ctx& c, int64_t batch, int64_t n, MatB<const T> src, MatB<T> dst, bool from_upper);
// dst(i,j) = dst(j,i) = alpha * src(max(i,j), min(i,j))  (bit-symmetric)
template <typename T>
dla_status ew_sym_lower_into(const Ctx& c, int64_t batch, int64_t n, MatB<const T> src, MatB<T> dst, T alpha);
// dst = src + src^T
template <typename T>
dla_status ew_add_transpose(const Ctx& c, int64_t batch, int64_t n, MatB<const T> src, MatB<T> dst, T alpha = T(1));
// x(i,i) *= alpha
template <typename T>
dla_status ew_scale_diag(const Ctx& c, int64_t batch, int64_t n, MatB<T> x, T alpha);
template <typename T>
dla_status check_symmetric(const Ctx& c, int64_t batch, int64_t n, MatB<const T> a, int32_t* info);
// its (max |a_ij - a_ji|, max |a_ij|) reduction slots, carved from the workspace
inline size_t ws_check_symmetric(int64_t batch) { return carve_bound(2 * sizeof(unsigned long long) * (size_t)batch); }
template <typename T>
dla_status check_zero_diag(const Ctx& c, int64_t batch, int64_t n, MatB<const T> t, int32_t* info);
template <typename T>
dla_status sumlogdiag_fwd(const Ctx& c, int64_t batch, int64_t n, T* out, MatB<const T> a);
template <typename T>
dla_status sumlogdiag_bwd(const Ctx& c, int64_t batch, int64_t n, MatB<T> abar, const T* g,
                          MatB<const T> a, bool accumulate);

// tri.cu: blocked triangular algorithms (any n), in place.
template <typename T>
dla_status trsm(const Ctx& c, int64_t batch, int64_t m, int64_t n, MatB<const T> t, MatB<T> x,
                bool right, bool trans, bool lower, T alpha, bool check_diag = false);
template <typename T>
dla_status trmm(const Ctx& c, int64_t batch, int64_t m, int64_t n, MatB<const T> t, MatB<T> x,
                bool right, bool trans, bool lower, T alpha);
template <typename T>
dla_status potrf_lower(const Ctx& c, int64_t batch, int64_t n, MatB<T> a, bool zero_upper = true,
                       bool* upper_zeroed = nullptr);
template <typename T>
dla_status potri_lower(const Ctx& c, int64_t batch, int64_t n, MatB<T> a);

}  // namespace dlab
