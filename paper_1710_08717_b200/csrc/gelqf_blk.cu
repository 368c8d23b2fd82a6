// Blocked Householder LQ (compact WY) for the batched gelqf forward,
// dl/lq.hpp:24-106 reorganised for B200.  The unblocked reference streams the
// whole trailing matrix once per reflector (256 passes over 512 KiB for a
// 128 x 512 slice: HBM-bound once the batch exceeds L2).  Here reflectors
// are taken BP = 32 rows at a time:
//
//   reduce, panel j (rows k0 .. k0+BP-1):
//     k_lq_panel   one CTA per slice: the panel rows in shared memory, the
//                  reference's row-by-row reduction restricted to the panel,
//                  then Yc (rows = v_k, unit at k, zeros before), the
//                  forward T of H_k0 ... H_k0+BP-1 = I - Yc^T T Yc and
//                  Z = T Yc into the workspace
//     trailing rows R (rows >= k0+BP, columns >= k0):
//                  W = R Yc^T, R -= W Z      (two batched DMMA / FFMA GEMMs)
//   L extraction + rank check (dl/lq.hpp:70-77)
//   form Q, panels last to first (the reference's back-to-front order):
//     k_lq_form    panel rows emitted in shared memory exactly as
//                  dl/lq.hpp:81-96 does, restricted to the panel's reflectors;
//                  Zq = T^T Yc into the workspace
//     R (rows >= k0+BP) <- R H_k0+BP-1 ... H_k0:  W = R Yc^T, R -= W Zq
//   sign normalisation (dl/lq.hpp:98-105)
//
// The reference's per-element arithmetic of the reflector construction
// (beta, tau, the 1/(alpha - beta) scaling, sigma == 0 => tau = 0) is kept;
// sums are parallel reductions, so results agree to rounding.
#include "common.cuh"
#include "ops.cuh"

#ifndef DLAB_LQ_BP
#define DLAB_LQ_BP 32
#endif

namespace dlab {
namespace {

constexpr int BP = DLAB_LQ_BP;  // reflectors per panel
constexpr int LT = 512;   // threads per CTA (16 warps: one SM's worth of latency hiding)

template <typename T>
__device__ T lq_block_sum(T v, T* red) {
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) red[w] = v;
  __syncthreads();
  T r = T(0);
#pragma unroll
  for (int k = 0; k < LT / 32; ++k) r += red[k];
  return r;
}

template <typename T>
__device__ T lq_block_max(T v, T* red) {
  for (int o = 16; o; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) red[w] = v;
  __syncthreads();
  T r = T(0);
#pragma unroll
  for (int k = 0; k < LT / 32; ++k) r = fmax(r, red[k]);
  return r;
}

// sum_{c = c0 + lane, step 32, c < N} x[c] y[c] with four independent
// accumulators (the panel sweeps are latency-bound: one CTA per SM)
template <typename T>
__device__ __forceinline__ T lane_dot(const T* x, const T* y, int c0, int N) {
  T a0 = T(0), a1 = T(0), a2 = T(0), a3 = T(0);
  int c = c0;
  for (; c + 96 < N; c += 128) {
    a0 += x[c] * y[c];
    a1 += x[c + 32] * y[c + 32];
    a2 += x[c + 64] * y[c + 64];
    a3 += x[c + 96] * y[c + 96];
  }
  for (; c < N; c += 32) a0 += x[c] * y[c];
  return (a0 + a1) + (a2 + a3);
}

template <typename T>
__device__ __forceinline__ void lane_axpy(T* x, const T* y, T w, int c0, int N) {
  int c = c0;
  for (; c + 96 < N; c += 128) {
    const T y0 = y[c], y1 = y[c + 32], y2 = y[c + 64], y3 = y[c + 96];
    x[c] -= w * y0;
    x[c + 32] -= w * y1;
    x[c + 64] -= w * y2;
    x[c + 96] -= w * y3;
  }
  for (; c < N; c += 32) x[c] -= w * y[c];
}

// Workspace per slice (elements of T): Yc [m x n], Z [m x n], T [m x BP],
// W [m x BP], tau [m], norm [1].
template <typename T>
struct LqWs {
  T *yc, *z, *t, *w, *tau, *nrm;
  int64_t per;
  __host__ __device__ static int64_t per_slice(int64_t m, int64_t n) { return 2 * m * n + 2 * m * BP + m + 1; }
  __host__ __device__ LqWs(T* base, int64_t m, int64_t n, int64_t b) {
    per = per_slice(m, n);
    T* p = base + b * per;
    yc = p;
    z = yc + m * n;
    t = z + m * n;
    w = t + m * BP;
    tau = w + m * BP;
    nrm = tau + m;
  }
};

// max|A| per slice; all-zero => SINGULAR(0) (dl/lq.hpp:33-36)
template <typename T>
__global__ void __launch_bounds__(LT) k_lq_norm(int64_t m, int64_t n, const T* a, T* ws, int32_t* info,
                                                bool rank_check) {
  __shared__ T red[LT / 32];
  const int64_t b = blockIdx.x;
  const T* ab = a + b * m * n;
  T mx = T(0);
  for (int64_t e = threadIdx.x; e < m * n; e += LT) mx = fmax(mx, fabs(ab[e]));
  mx = lq_block_max(mx, red);
  if (threadIdx.x == 0) {
    LqWs<T>(ws, m, n, b).nrm[0] = mx;
    if (mx == T(0) && rank_check) record_failure(info, b, DLA_ERR_SINGULAR, 0);
  }
}

// Reduce the panel rows k0 .. k0+bp-1 (columns k0 .. n-1) and build Yc, T, Z.
template <typename T>
__global__ void __launch_bounds__(LT) k_lq_panel(int64_t m, int64_t n, int64_t k0, int bp, T* a, T* ws,
                                                 const int32_t* info) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int64_t b = blockIdx.x;
  if (slice_failed(info, b)) return;
  const int N = (int)(n - k0);
  const int PL = N + 1;  // odd row stride: warp-per-row sweeps stay conflict-free
  T* P = reinterpret_cast<T*>(smem_raw);  // [bp][PL]
  T* G = P + BP * PL;                      // [BP][BP + 1] Gram Yc Yc^T
  T* Ts = G + BP * (BP + 1);               // [BP][BP + 1]
  T* tau = Ts + BP * (BP + 1);             // [BP]
  __shared__ T red[LT / 32];
  LqWs<T> W(ws, m, n, b);
  T* ab = a + b * m * n;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  for (int e = tid; e < bp * N; e += LT) {
    const int r = e / N, c = e % N;
    P[r * PL + c] = ab[(k0 + r) * n + k0 + c];
  }
  __syncthreads();
  for (int j = 0; j < bp; ++j) {
    T* xk = P + j * PL;
    T s = T(0);
    for (int c = j + 1 + tid; c < N; c += LT) s += xk[c] * xk[c];
    const T sigma = lq_block_sum(s, red);
    const T alpha = xk[j];
    if (sigma == T(0)) {
      if (tid == 0) tau[j] = T(0);
      __syncthreads();
      continue;
    }
    const T nrm = Num<T>::sqrt_(alpha * alpha + sigma);
    const T beta = alpha >= T(0) ? -nrm : nrm;
    const T tk = (beta - alpha) / beta;
    const T sc = T(1) / (alpha - beta);
    __syncthreads();  // every thread has read alpha
    for (int c = j + 1 + tid; c < N; c += LT) xk[c] *= sc;
    if (tid == 0) {
      xk[j] = beta;
      tau[j] = tk;
    }
    __syncthreads();
    for (int i = j + 1 + warp; i < bp; i += LT / 32) {  // H_k on the panel rows below
      T* xi = P + i * PL;
      T w = lane_dot(xi, xk, j + 1 + lane, N);
      for (int o = 16; o; o >>= 1) w += __shfl_xor_sync(0xffffffffu, w, o);
      w = (w + xi[j]) * tk;
      __syncwarp();
      if (lane == 0) xi[j] -= w;
      lane_axpy(xi, xk, w, j + 1 + lane, N);
    }
    __syncthreads();
  }
  // factored rows back (beta on the diagonal, v tails), Yc, tau
  for (int e = tid; e < bp * N; e += LT) {
    const int r = e / N, c = e % N;
    const T v = P[r * PL + c];
    ab[(k0 + r) * n + k0 + c] = v;
    W.yc[(k0 + r) * n + k0 + c] = c < r ? T(0) : (c == r ? T(1) : v);
  }
  if (tid < bp) W.tau[k0 + tid] = tau[tid];
  // Yc in shared memory (unit diagonal, zeros before it) for G and Z
  for (int e = tid; e < bp * N; e += LT) {
    const int r = e / N, c = e % N;
    if (c <= r) P[r * PL + c] = c == r ? T(1) : T(0);
  }
  __syncthreads();
  // Gram G = Yc Yc^T (upper part): warp per (i, k) pair
  for (int pr = warp; pr < bp * bp; pr += LT / 32) {
    const int i = pr / bp, k = pr % bp;
    if (k <= i) continue;
    T g = lane_dot(P + i * PL, P + k * PL, k + lane, N);
    for (int o = 16; o; o >>= 1) g += __shfl_xor_sync(0xffffffffu, g, o);
    if (lane == 0) G[i * (BP + 1) + k] = g;
  }
  __syncthreads();
  // forward T (H_0 ... H_{bp-1} = I - Yc^T T Yc):
  // T(j,j) = tau_j, T(0:j, j) = -tau_j T(0:j, 0:j) G(0:j, j)
  for (int j = 0; j < bp; ++j) {
    if (tid < j) {
      T acc = T(0);
      for (int l = tid; l < j; ++l) acc += Ts[tid * (BP + 1) + l] * G[l * (BP + 1) + j];
      Ts[tid * (BP + 1) + j] = -tau[j] * acc;
    }
    if (tid == 0) Ts[j * (BP + 1) + j] = tau[j];
    if (tid >= j && tid < bp && tid != j) Ts[tid * (BP + 1) + j] = T(0);
    __syncthreads();
  }
  for (int e = tid; e < bp * bp; e += LT) W.t[(k0 + e / bp) * BP + e % bp] = Ts[(e / bp) * (BP + 1) + e % bp];
  // Z = T Yc  (rows k0.., columns k0..)
  for (int e = tid; e < bp * N; e += LT) {
    const int i = e / N, c = e % N;
    T acc = T(0);
    for (int l = i; l < bp; ++l) acc += Ts[i * (BP + 1) + l] * P[l * PL + c];
    W.z[(k0 + i) * n + k0 + c] = acc;
  }
}

// L = tril(A[:, :m]) and the rank check (dl/lq.hpp:70-77)
template <typename T>
__global__ void __launch_bounds__(LT) k_lq_extract(int64_t m, int64_t n, const T* a, T* l, T* ws, int32_t* info,
                                                   bool rank_check) {
  const int64_t b = blockIdx.x;
  if (slice_failed(info, b)) return;
  const T* ab = a + b * m * n;
  T* lb = l + b * m * m;
  for (int64_t e = threadIdx.x; e < m * m; e += LT) {
    const int64_t i = e / m, j = e % m;
    lb[e] = j <= i ? ab[i * n + j] : T(0);
  }
  if (threadIdx.x == 0 && rank_check) {
    const T tol = Num<T>::rank_rtol * LqWs<T>(ws, m, n, b).nrm[0];
    for (int64_t i = 0; i < m; ++i)
      if (fabs(ab[i * n + i]) < tol) {
        record_failure(info, b, DLA_ERR_SINGULAR, i);
        break;
      }
  }
}

// Emit Q rows k0 .. k0+bp-1 (dl/lq.hpp:81-96 restricted to the panel's
// reflectors) and Zq = T^T Yc for the block update of the rows below.
template <typename T>
__global__ void __launch_bounds__(LT) k_lq_form(int64_t m, int64_t n, int64_t k0, int bp, T* a, T* ws,
                                                const int32_t* info) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int64_t b = blockIdx.x;
  if (slice_failed(info, b)) return;
  const int N = (int)(n - k0);
  const int PL = N + 1;
  // [bp][PL]: row k holds v_k until reflector k is consumed, then Q row k
  // (rows > k are already emitted when H_k is applied to them)
  T* Y = reinterpret_cast<T*>(smem_raw);
  T* Q = Y;
  __shared__ T Ts[BP][BP + 1];
  __shared__ T tau[BP];
  LqWs<T> W(ws, m, n, b);
  T* ab = a + b * m * n;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  for (int e = tid; e < bp * N; e += LT) {
    const int r = e / N, c = e % N;
    Y[r * PL + c] = W.yc[(k0 + r) * n + k0 + c];
  }
  for (int e = tid; e < bp * bp; e += LT) Ts[e / bp][e % bp] = W.t[(k0 + e / bp) * BP + e % bp];
  if (tid < bp) tau[tid] = W.tau[k0 + tid];
  __syncthreads();
  // Zq = T^T Yc
  for (int e = tid; e < bp * N; e += LT) {
    const int i = e / N, c = e % N;
    T acc = T(0);
    for (int l = 0; l <= i; ++l) acc += Ts[l][i] * Y[l * PL + c];
    W.z[(k0 + i) * n + k0 + c] = acc;
  }
  __syncthreads();  // Yc is overwritten in place below
  // back to front over the panel's reflectors
  for (int k = bp - 1; k >= 0; --k) {
    const T tk = tau[k];
    const T* vk = Y + k * PL;
    for (int i = k + 1 + warp; i < bp; i += LT / 32) {
      T* xi = Q + i * PL;
      T w = lane_dot(xi, vk, k + 1 + lane, N);
      for (int o = 16; o; o >>= 1) w += __shfl_xor_sync(0xffffffffu, w, o);
      w = (w + xi[k]) * tk;
      __syncwarp();
      if (lane == 0) xi[k] -= w;
      lane_axpy(xi, vk, w, k + 1 + lane, N);
    }
    __syncthreads();  // row k (v_k) is read by the sweep above
    T* xk = Q + k * PL;
    for (int c = tid; c < N; c += LT) xk[c] = c < k ? T(0) : (c == k ? T(1) - tk : -tk * xk[c]);
    __syncthreads();
  }
  for (int e = tid; e < bp * (int)n; e += LT) {
    const int r = e / (int)n, c = e % (int)n;
    ab[(k0 + r) * n + c] = c < k0 ? T(0) : Q[r * PL + (c - k0)];
  }
}

// diag(L) > 0: flip L's column k and Q's row k together (dl/lq.hpp:98-105)
constexpr int LQ_MMAX = 2048;
template <typename T>
__global__ void __launch_bounds__(LT) k_lq_sign(int64_t m, int64_t n, T* q, T* l, const int32_t* info) {
  __shared__ unsigned char flip[LQ_MMAX];
  const int64_t b = blockIdx.x;
  if (slice_failed(info, b)) return;
  T* qb = q + b * m * n;
  T* lb = l + b * m * m;
  for (int64_t k = threadIdx.x; k < m; k += LT) flip[k] = lb[k * m + k] < T(0);
  __syncthreads();
  for (int64_t e = threadIdx.x; e < m * n; e += LT)
    if (flip[e / n]) qb[e] = -qb[e];
  for (int64_t e = threadIdx.x; e < m * m; e += LT) {
    const int64_t i = e / m, k = e % m;
    if (k <= i && flip[k]) lb[e] = -lb[e];
  }
}

template <typename T>
size_t panel_smem(int64_t n) {
  const size_t pl = (size_t)n + 1;
  return sizeof(T) * (BP * pl + 2 * BP * (BP + 1) + BP);
}

}  // namespace

template <typename T>
bool gelqf_blocked_eligible(int64_t m, int64_t n) {
  return m >= 2 * BP && m <= LQ_MMAX && panel_smem<T>(n) <= 200 * 1024;
}

template <typename T>
size_t gelqf_blocked_ws_bytes(int64_t batch, int64_t m, int64_t n) {
  return sizeof(T) * (size_t)(batch * LqWs<T>::per_slice(m, n));
}

template <typename T>
dla_status gelqf_blocked(const Ctx& c, int64_t batch, int64_t m, int64_t n, T* q, T* l, void* wsv, bool rank_check) {
  T* ws = static_cast<T*>(wsv);
  const int64_t per = LqWs<T>::per_slice(m, n);
  const size_t sm_panel = panel_smem<T>(n);
  const size_t sm_form = panel_smem<T>(n);
  ensure_smem_attr(k_lq_panel<T>, sm_panel);
  ensure_smem_attr(k_lq_form<T>, sm_form);
  const unsigned grid = (unsigned)batch;
  k_lq_norm<T><<<grid, LT, 0, c.stream>>>(m, n, q, ws, c.info, rank_check);
  DLAB_LAUNCH_CHECK();
  // views: A rows / columns from k0; Yc, Z rows k0.. (same geometry); W [m x BP]
  auto av = [&](int64_t r0, int64_t c0) { return MatB<T>{q + r0 * n + c0, n, m * n}; };
  auto wv = [&](T* base, int64_t r0, int64_t c0) { return MatB<T>{base + r0 * n + c0, n, per}; };
  LqWs<T> w0(ws, m, n, 0);
  const int64_t npan = (m + BP - 1) / BP;
  for (int64_t pj = 0; pj < npan; ++pj) {
    const int64_t k0 = pj * BP;
    const int bp = (int)std::min<int64_t>(BP, m - k0);
    k_lq_panel<T><<<grid, LT, sm_panel, c.stream>>>(m, n, k0, bp, q, ws, c.info);
    DLAB_LAUNCH_CHECK();
    const int64_t rm = m - k0 - bp, nc = n - k0;
    if (rm <= 0) continue;
    MatB<T> wm{w0.w, BP, per};
    // W = R Yc^T ; R -= W Z
    DLAB_TRY(gemm<T>(c, batch, rm, bp, nc, T(1), MatB<const T>{q + (k0 + bp) * n + k0, n, m * n}, false,
                     MatB<const T>{w0.yc + k0 * n + k0, n, per}, true, T(0), wm, MASK_FULL, c.info));
    DLAB_TRY(gemm<T>(c, batch, rm, nc, bp, T(-1), MatB<const T>{wm.p, wm.ld, wm.bs}, false,
                     MatB<const T>{w0.z + k0 * n + k0, n, per}, false, T(1), av(k0 + bp, k0), MASK_FULL, c.info));
  }
  k_lq_extract<T><<<grid, LT, 0, c.stream>>>(m, n, q, l, ws, c.info, rank_check);
  DLAB_LAUNCH_CHECK();
  for (int64_t pj = npan - 1; pj >= 0; --pj) {
    const int64_t k0 = pj * BP;
    const int bp = (int)std::min<int64_t>(BP, m - k0);
    k_lq_form<T><<<grid, LT, sm_form, c.stream>>>(m, n, k0, bp, q, ws, c.info);
    DLAB_LAUNCH_CHECK();
    const int64_t rm = m - k0 - bp, nc = n - k0;
    if (rm <= 0) continue;
    MatB<T> wm{w0.w, BP, per};
    // R <- R H_{k0+bp-1} ... H_{k0} = R - (R Yc^T) (T^T Yc)
    DLAB_TRY(gemm<T>(c, batch, rm, bp, nc, T(1), MatB<const T>{q + (k0 + bp) * n + k0, n, m * n}, false,
                     MatB<const T>{w0.yc + k0 * n + k0, n, per}, true, T(0), wm, MASK_FULL, c.info));
    DLAB_TRY(gemm<T>(c, batch, rm, nc, bp, T(-1), MatB<const T>{wm.p, wm.ld, wm.bs}, false,
                     MatB<const T>{w0.z + k0 * n + k0, n, per}, false, T(1), av(k0 + bp, k0), MASK_FULL, c.info));
  }
  (void)wv;
  k_lq_sign<T><<<grid, LT, 0, c.stream>>>(m, n, q, l, c.info);
  DLAB_LAUNCH_CHECK();
  return DLA_OK;
}

#define INST(T)                                                                  \
  template bool gelqf_blocked_eligible<T>(int64_t, int64_t);                     \
  template size_t gelqf_blocked_ws_bytes<T>(int64_t, int64_t, int64_t);          \
  template dla_status gelqf_blocked<T>(const Ctx&, int64_t, int64_t, int64_t, T*, T*, void*, bool);
INST(double)
INST(float)

}  // namespace dlab
