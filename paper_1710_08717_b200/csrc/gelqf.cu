// Batched LQ factorization (m <= n): A = L Q, Q with orthonormal rows,
// diag(L) > 0.  Reference: dl/lq.hpp:24-106 (row Householder reflectors
// H_k = I - tau v v^T, L extraction + rank check, in-place back-to-front Q
// formation, sign normalization).
//
// One CTA per matrix (512 threads, a warp per row in the reflector
// applications); rows are contiguous so every sweep is coalesced, and the
// per-slice working set (128 x 512 f64 = 512 KiB) stays L2-resident.  tau
// lives in the caller's workspace (m reals per slice, the reference's
// documented budget, dl/lq.hpp:39-40).
#include "common.cuh"
#include "ops.cuh"

namespace dlab {
namespace {

constexpr int GT = 512;

template <typename T>
__device__ T block_sum(T v, T* red) {
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) red[w] = v;
  __syncthreads();
  T r = T(0);
  for (int k = 0; k < GT / 32; ++k) r += red[k];
  return r;
}

template <typename T>
__device__ T block_maxabs(T v, T* red) {
  for (int o = 16; o; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) red[w] = v;
  __syncthreads();
  T r = T(0);
  for (int k = 0; k < GT / 32; ++k) r = fmax(r, red[k]);
  return r;
}

// Apply H_k (vector v = [1, tail of row k]) to rows i in (k, m) of x.
template <typename T>
__device__ void apply_reflector(T* x, int64_t m, int64_t n, int64_t k, const T* vk, T tk) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int64_t i = k + 1 + warp; i < m; i += GT / 32) {
    T* xi = x + i * n;
    const T xik = xi[k];
    T w = T(0);
    for (int64_t j = k + 1 + lane; j < n; j += 32) w += xi[j] * vk[j];
    for (int o = 16; o; o >>= 1) w += __shfl_xor_sync(0xffffffffu, w, o);
    w = (w + xik) * tk;
    __syncwarp();
    if (lane == 0) xi[k] = xik - w;
    for (int64_t j = k + 1 + lane; j < n; j += 32) xi[j] -= w * vk[j];
  }
}

template <typename T>
__global__ void __launch_bounds__(GT) k_gelqf(int64_t m, int64_t n, T* qall, T* lall, T* tauall, int32_t* info,
                                              bool rank_check) {
  __shared__ T red[GT / 32];
  __shared__ int fail_row;
  const int64_t b = blockIdx.x;
  T* q = qall + b * m * n;
  T* l = lall + b * m * m;
  T* tau = tauall + b * m;

  T mx = T(0);
  for (int64_t e = threadIdx.x; e < m * n; e += GT) mx = fmax(mx, fabs(q[e]));
  const T norm_a = block_maxabs(mx, red);
  if (norm_a == T(0) && rank_check) {
    if (threadIdx.x == 0) record_failure(info, b, DLA_ERR_SINGULAR, 0);
    return;
  }
  // reduce: annihilate row k's tail
  for (int64_t k = 0; k < m; ++k) {
    T* xk = q + k * n;
    T s = T(0);
    for (int64_t j = k + 1 + threadIdx.x; j < n; j += GT) s += xk[j] * xk[j];
    const T sigma = block_sum(s, red);
    const T alpha = xk[k];
    if (sigma == T(0)) {
      if (threadIdx.x == 0) tau[k] = T(0);
      __syncthreads();
      continue;
    }
    const T nrm = Num<T>::sqrt_(alpha * alpha + sigma);
    const T beta = alpha >= T(0) ? -nrm : nrm;
    const T tk = (beta - alpha) / beta;
    const T sc = T(1) / (alpha - beta);
    __syncthreads();  // everyone has read alpha
    for (int64_t j = k + 1 + threadIdx.x; j < n; j += GT) xk[j] *= sc;
    if (threadIdx.x == 0) {
      xk[k] = beta;
      tau[k] = tk;
    }
    __syncthreads();
    apply_reflector(q, m, n, k, xk, tk);
    __syncthreads();
  }
  // L extraction and rank check (before the factor storage is consumed)
  const T rank_tol = Num<T>::rank_rtol * norm_a;
  if (threadIdx.x == 0) fail_row = -1;
  __syncthreads();
  for (int64_t e = threadIdx.x; e < m * m; e += GT) {
    const int64_t i = e / m, j = e % m;
    l[e] = j <= i ? q[i * n + j] : T(0);
  }
  __syncthreads();
  if (threadIdx.x == 0 && rank_check) {
    for (int64_t i = 0; i < m; ++i)
      if (fabs(l[i * m + i]) < rank_tol) {
        fail_row = (int)i;
        break;
      }
  }
  __syncthreads();
  if (fail_row >= 0) {
    if (threadIdx.x == 0) record_failure(info, b, DLA_ERR_SINGULAR, fail_row);
    return;
  }
  // form Q in place, back to front
  for (int64_t k = m - 1; k >= 0; --k) {
    T* xk = q + k * n;
    const T tk = tau[k];
    apply_reflector(q, m, n, k, xk, tk);
    __syncthreads();
    for (int64_t j = threadIdx.x; j < n; j += GT) {
      if (j < k) xk[j] = T(0);
      else if (j > k) xk[j] = -tk * xk[j];
    }
    if (threadIdx.x == 0) xk[k] = T(1) - tk;
    __syncthreads();
  }
  // sign normalization: diag(L) > 0 (flip L's column k and Q's row k)
  for (int64_t k = 0; k < m; ++k) {
    const bool flip = l[k * m + k] < T(0);
    __syncthreads();
    if (flip) {
      for (int64_t i = k + threadIdx.x; i < m; i += GT) l[i * m + k] = -l[i * m + k];
      for (int64_t j = threadIdx.x; j < n; j += GT) q[k * n + j] = -q[k * n + j];
    }
    __syncthreads();
  }
}

}  // namespace

template <typename T>
size_t gelqf_ws_bytes(int64_t batch, int64_t m, int64_t n, bool backward) {
  if (backward) return sizeof(T) * (size_t)(batch * m * m);
  if (gelqf_blocked_eligible<T>(m, n)) return gelqf_blocked_ws_bytes<T>(batch, m, n);
  return sizeof(T) * (size_t)(batch * m);
}

template <typename T>
dla_status gelqf_fwd(const Ctx& c, int64_t batch, int64_t m, int64_t n, T* q, T* l, void* ws, bool rank_check) {
  if (!ws) return DLA_ERR_WORKSPACE;
  if (gelqf_blocked_eligible<T>(m, n)) return gelqf_blocked<T>(c, batch, m, n, q, l, ws, rank_check);
  k_gelqf<T><<<(unsigned)batch, GT, 0, c.stream>>>(m, n, q, l, static_cast<T*>(ws), c.info, rank_check);
  DLAB_LAUNCH_CHECK();
  return DLA_OK;
}

template size_t gelqf_ws_bytes<double>(int64_t, int64_t, int64_t, bool);
template size_t gelqf_ws_bytes<float>(int64_t, int64_t, int64_t, bool);
template dla_status gelqf_fwd<double>(const Ctx&, int64_t, int64_t, int64_t, double*, double*, void*, bool);
template dla_status gelqf_fwd<float>(const Ctx&, int64_t, int64_t, int64_t, float*, float*, void*, bool);

}  // namespace dlab
