// gesvd: thin SVD of a wide matrix (m <= n), A = U^T diag(lambda) V with
// U m x m and V m x n (ROWS are the singular vectors), lambda ascending and
// nonnegative, the reference's sign rule on U's rows with V flipped in
// lockstep (dl/svd.hpp:229-284), and its pullback (dl/adjoints.hpp:303-382).
//
// B200 design (not the reference's Golub-Kahan-Reinsch chain of scalar
// recurrences):
//   1. LQ-precondition: A = L Q with the blocked compact-WY gelqf (DMMA
//      trailing updates), rank check off -- a rank-deficient A is a valid
//      SVD input (zero singular values).
//   2. one-sided (Hestenes) Jacobi on the ROWS of the small square L, one
//      CTA per matrix: J L = B with mutually orthogonal rows (round-robin
//      pairs, a warp per pair, rows in shared memory for m <= 64), so
//      lambda_i = |B_i|, W_i = B_i / lambda_i and U = J.  Jacobi on the
//      preconditioned L keeps high relative accuracy in every singular value.
//   3. V = W Q: one batched GEMM.
// Sorting (ascending, stable by index) and the sign rule run inside the
// Jacobi kernel before W is stored, so the GEMM emits V already permuted.
//
// Pullback (dl/adjoints.hpp:315-382), as five batched kernels / GEMMs:
//   abar = Lambda^-1 Vbar;  work = abar V^T (diag kept);  work = work Lambda
//   + Ubar U^T;  work = diag(lambdabar) + 2 sym(work . E) Lambda - diag(d)
//   (gap-guarded);  abar += work V;  abar = U^T abar.
#include <cfloat>

#include "common.cuh"
#include "ops.cuh"

namespace dlab {
namespace {

constexpr int JT = 512;   // Jacobi CTA: 16 warps
constexpr int JSM = 64;   // rows held in shared memory up to this m
constexpr int JSWEEPS = 60;

template <typename T>
struct JTol;
template <>
struct JTol<double> {
  static constexpr double tol = 2.0 * DBL_EPSILON;
};
template <>
struct JTol<float> {
  static constexpr float tol = 2.0f * FLT_EPSILON;
};

template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// One CTA per slice.  B (rows being orthogonalised, starts as L) and U (the
// accumulated rotations, starts as I) live in shared memory (m <= JSM) or in
// the workspace (larger m); outputs: u (m x m), lambda (m), w (m x m).
template <typename T>
__global__ void __launch_bounds__(JT) k_svd_jacobi(int m, const T* lall, T* uall, T* lamall, T* wall, T* gws,
                                                   int32_t* info) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ int rotated;
  __shared__ int order[1024];
  const int64_t b = blockIdx.x;
  if (slice_failed(info, b)) return;
  const bool in_smem = m <= JSM;
  const int ld = in_smem ? m + 1 : m;
  T* B = in_smem ? reinterpret_cast<T*>(smem_raw) : gws + b * 2 * (int64_t)m * m;
  T* U = B + (int64_t)m * ld;
  T* nrm = in_smem ? U + m * ld : reinterpret_cast<T*>(smem_raw);  // lambda_i (unsorted)
  const T* L = lall + b * (int64_t)m * m;
  for (int64_t e = threadIdx.x; e < (int64_t)m * m; e += JT) {
    const int i = (int)(e / m), j = (int)(e % m);
    B[(int64_t)i * ld + j] = j <= i ? L[e] : T(0);
    U[(int64_t)i * ld + j] = i == j ? T(1) : T(0);
  }
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = JT / 32;
  const int mm = (m + 1) & ~1;  // players (one dummy when m is odd)
  int sweep = 0;
  for (; sweep < JSWEEPS; ++sweep) {
    if (threadIdx.x == 0) rotated = 0;
    __syncthreads();
    for (int r = 0; r < mm - 1; ++r) {
      for (int k = warp; k < mm / 2; k += nw) {
        const int a0 = k == 0 ? 0 : (k - 1 + r) % (mm - 1) + 1;
        const int k2 = mm - 1 - k;
        const int a1 = (k2 - 1 + r) % (mm - 1) + 1;
        const int p = min(a0, a1), q = max(a0, a1);
        if (q >= m) continue;  // the dummy player
        T* bp = B + (int64_t)p * ld;
        T* bq = B + (int64_t)q * ld;
        T al = T(0), be = T(0), ga = T(0);
        for (int j = lane; j < m; j += 32) {
          const T x = bp[j], y = bq[j];
          al = fma(x, x, al);
          be = fma(y, y, be);
          ga = fma(x, y, ga);
        }
        al = warp_sum(al);
        be = warp_sum(be);
        ga = warp_sum(ga);
        if (ga == T(0) || !(fabs(ga) > JTol<T>::tol * sqrt(al * be))) continue;
        // rows p' = c p - s q, q' = s p + c q with <p', q'> = 0:
        // t^2 + 2 zeta t - 1 = 0, zeta = (be - al) / (2 ga), smaller root
        const T zeta = (be - al) / (T(2) * ga);
        const T t = (zeta >= T(0) ? T(1) : T(-1)) / (fabs(zeta) + sqrt(T(1) + zeta * zeta));
        const T c = T(1) / sqrt(T(1) + t * t), s = c * t;
        for (int j = lane; j < m; j += 32) {
          const T x = bp[j], y = bq[j];
          bp[j] = c * x - s * y;
          bq[j] = s * x + c * y;
        }
        T* up = U + (int64_t)p * ld;
        T* uq = U + (int64_t)q * ld;
        for (int j = lane; j < m; j += 32) {
          const T x = up[j], y = uq[j];
          up[j] = c * x - s * y;
          uq[j] = s * x + c * y;
        }
        if (lane == 0) rotated = 1;
      }
      __syncthreads();
    }
    if (!rotated) break;
    __syncthreads();
  }
  if (sweep == JSWEEPS) {
    if (threadIdx.x == 0) record_failure(info, b, DLA_ERR_CONVERGENCE, sweep);
    return;
  }
  // lambda_i = |B_i|
  for (int i = warp; i < m; i += nw) {
    T s2 = T(0);
    for (int j = lane; j < m; j += 32) s2 = fma(B[(int64_t)i * ld + j], B[(int64_t)i * ld + j], s2);
    s2 = warp_sum(s2);
    if (lane == 0) nrm[i] = sqrt(s2);
  }
  __syncthreads();
  // ascending, ties by index (stable); sign rule on U's rows: flip when the
  // largest-magnitude entry (smallest index on ties) is negative
  for (int i = threadIdx.x; i < m; i += JT) {
    const T li = nrm[i];
    int rank = 0;
    for (int j = 0; j < m; ++j) rank += (nrm[j] < li) || (nrm[j] == li && j < i);
    order[rank] = i;
  }
  __syncthreads();
  T* uo = uall + b * (int64_t)m * m;
  T* wo = wall + b * (int64_t)m * m;
  T* lo = lamall + b * (int64_t)m;
  for (int r = warp; r < m; r += nw) {
    const int i = order[r];
    const T* ui = U + (int64_t)i * ld;
    // arg max |u_ij|, smallest j on ties
    T best = T(-1);
    int kb = 0;
    for (int j = lane; j < m; j += 32) {
      const T v = fabs(ui[j]);
      if (v > best) {
        best = v;
        kb = j;
      }
    }
    for (int o = 16; o; o >>= 1) {
      const T ob = __shfl_xor_sync(0xffffffffu, best, o);
      const int ok = __shfl_xor_sync(0xffffffffu, kb, o);
      if (ob > best || (ob == best && ok < kb)) {
        best = ob;
        kb = ok;
      }
    }
    const T sg = ui[kb] < T(0) ? T(-1) : T(1);
    const T li = nrm[i];
    const T inv = li > T(0) ? sg / li : T(0);
    for (int j = lane; j < m; j += 32) {
      uo[(int64_t)r * m + j] = sg * ui[j];
      wo[(int64_t)r * m + j] = inv * B[(int64_t)i * ld + j];
    }
    if (lane == 0) lo[r] = li;
  }
}

// ---- pullback pieces (dl/adjoints.hpp:315-382)
// first non-positive-enough lambda (ascending scan: the reference's throw site)
template <typename T>
__global__ void k_svd_bwd_check(int64_t batch, int m, const T* lam, T eps_gap, int32_t* info) {
  const int64_t b = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (b >= batch || slice_failed(info, b)) return;
  for (int i = 0; i < m; ++i)
    if (!(lam[b * m + i] > eps_gap)) {
      record_failure(info, b, DLA_ERR_SINGULAR, i);
      return;
    }
}

// abar = Lambda^-1 Vbar
template <typename T>
__global__ void k_svd_bwd_scale(int64_t batch, int m, int64_t n, const T* vbar, const T* lam, T* abar,
                                const int32_t* info) {
  const int64_t tot = batch * m * n;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < tot; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t b = e / (m * n), i = (e / n) % m;
    if (slice_failed(info, b)) continue;
    abar[e] = vbar[e] / lam[b * m + i];
  }
}

// d_i = work_ii; work_ij *= lambda_j
template <typename T>
__global__ void k_svd_bwd_mid(int64_t batch, int m, T* work, T* d, const T* lam, const int32_t* info) {
  const int64_t tot = batch * m * m;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < tot; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t b = e / ((int64_t)m * m), i = (e / m) % m, j = e % m;
    if (slice_failed(info, b)) continue;
    if (i == j) d[b * m + i] = work[e];
    work[e] *= lam[b * m + j];
  }
}

// work <- diag(lambdabar) + the gap-guarded antisymmetric part times Lambda
// (each thread owns one (i > j) pair and both of its entries, or a diagonal)
template <typename T>
__global__ void k_svd_bwd_gap(int64_t batch, int m, T* work, const T* d, const T* lam, const T* lambdabar, T eps_gap,
                              const int32_t* info) {
  const int64_t tot = batch * m * m;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < tot; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t b = e / ((int64_t)m * m), i = (e / m) % m, j = e % m;
    if (j > i || slice_failed(info, b)) continue;
    T* w = work + b * (int64_t)m * m;
    const T* l = lam + b * m;
    if (i == j) {
      w[i * m + i] = lambdabar[b * m + i] - d[b * m + i];
      continue;
    }
    const T hd = fmax(l[i] - l[j], eps_gap);
    const T hs = fmax(l[i] + l[j], eps_gap);
    const T y = (w[i * m + j] - w[j * m + i]) / (hd * hs);
    w[i * m + j] = y * l[j];
    w[j * m + i] = y * l[i];
  }
}

template <typename T>
MatB<const T> C_(MatB<T> x) {
  return MatB<const T>{x.p, x.ld, x.bs};
}

}  // namespace

template <typename T>
size_t gesvd_fwd_scratch(int64_t batch, int64_t m, int64_t n) {
  // Qs (m x n) | L (m x m) | W (m x m) | Jacobi rows B, U (2 m^2, m > JSM)
  const size_t per = (size_t)m * n + 2 * (size_t)m * m + (m > JSM ? 2 * (size_t)m * m : 0);
  return sizeof(T) * per * (size_t)batch;
}

template <typename T>
size_t ws_gesvd_fwd(int64_t batch, int64_t m, int64_t n) {
  return carve_bound(gesvd_fwd_scratch<T>(batch, m, n)) + carve_bound(gelqf_ws_bytes<T>(batch, m, n, false)) +
         ws_gemm<T>(batch, m, n, m);
}

template <typename T>
dla_status gesvd_fwd(const Ctx& c, int64_t batch, int64_t m, int64_t n, T* v, T* u, T* lambda) {
  if (m > 1024) return DLA_ERR_SHAPE;  // Jacobi ordering buffer (shared) bound
  DLAB_SCRATCH(sc, c, gesvd_fwd_scratch<T>(batch, m, n));
  DLAB_SCRATCH(lq, c, gelqf_ws_bytes<T>(batch, m, n, false));
  T* qs = sc.as<T>();
  T* ls = qs + batch * m * n;
  T* ws = ls + batch * m * m;
  T* gj = ws + batch * m * m;
  if (cudaMemcpyAsync(qs, v, sizeof(T) * (size_t)(batch * m * n), cudaMemcpyDeviceToDevice, c.stream) != cudaSuccess)
    return DLA_ERR_CUDA;
  DLAB_TRY(gelqf_fwd<T>(c, batch, m, n, qs, ls, lq.p, /*rank_check*/ false));
  const size_t smem = m <= JSM ? sizeof(T) * (size_t)(2 * m * (m + 1) + m) : sizeof(T) * (size_t)m;
  ensure_smem_attr(k_svd_jacobi<T>, smem);
  k_svd_jacobi<T><<<(unsigned)batch, JT, smem, c.stream>>>((int)m, ls, u, lambda, ws, gj, c.info);
  DLAB_LAUNCH_CHECK();
  // V = W Q (rows already in ascending-lambda order, signs applied)
  return gemm<T>(c, batch, m, n, m, T(1), MatB<const T>{ws, m, m * m}, false, MatB<const T>{qs, n, m * n}, false,
                 T(0), MatB<T>{v, n, m * n}, MASK_FULL, c.info);
}

template <typename T>
size_t gesvd_bwd_scratch(int64_t batch, int64_t m, int64_t n) {
  return sizeof(T) * (size_t)batch * ((size_t)m * m + (size_t)m + (size_t)m * n);  // work | d | tmp
}

template <typename T>
size_t ws_gesvd_bwd(int64_t batch, int64_t m, int64_t n) {
  return carve_bound(gesvd_bwd_scratch<T>(batch, m, n)) + ws_gemm<T>(batch, m, m, n) + ws_gemm<T>(batch, m, m, m) +
         2 * ws_gemm<T>(batch, m, n, m);
}

template <typename T>
dla_status gesvd_bwd(const Ctx& c, int64_t batch, int64_t m, int64_t n, T* abar, const T* ubar, const T* lambdabar,
                     const T* vbar, const T* u, const T* lambda, const T* v, T eps_gap) {
  DLAB_SCRATCH(sc, c, gesvd_bwd_scratch<T>(batch, m, n));
  T* work = sc.as<T>();
  T* d = work + batch * m * m;
  T* tmp = d + batch * m;
  const int32_t* skip = c.info;
  if (c.info) {
    k_svd_bwd_check<T><<<blocks_for(batch, 128), 128, 0, c.stream>>>(batch, (int)m, lambda, eps_gap, c.info);
    DLAB_LAUNCH_CHECK();
  }
  k_svd_bwd_scale<T><<<blocks_for(batch * m * n, 256), 256, 0, c.stream>>>(batch, (int)m, n, vbar, lambda, abar, skip);
  DLAB_LAUNCH_CHECK();
  MatB<T> wv{work, m, m * m};
  MatB<const T> vv{v, n, m * n}, uv{u, m, m * m};
  DLAB_TRY(gemm<T>(c, batch, m, m, n, T(1), MatB<const T>{abar, n, m * n}, false, vv, true, T(0), wv, MASK_FULL, skip));
  k_svd_bwd_mid<T><<<blocks_for(batch * m * m, 256), 256, 0, c.stream>>>(batch, (int)m, work, d, lambda, skip);
  DLAB_LAUNCH_CHECK();
  DLAB_TRY(gemm<T>(c, batch, m, m, m, T(1), MatB<const T>{ubar, m, m * m}, false, uv, true, T(1), wv, MASK_FULL, skip));
  k_svd_bwd_gap<T><<<blocks_for(batch * m * m, 256), 256, 0, c.stream>>>(batch, (int)m, work, d, lambda, lambdabar,
                                                                         eps_gap, skip);
  DLAB_LAUNCH_CHECK();
  DLAB_TRY(gemm<T>(c, batch, m, n, m, T(1), C_(wv), false, vv, false, T(1), MatB<T>{abar, n, m * n}, MASK_FULL, skip));
  DLAB_TRY(ew_copy<T>(c, batch, m, n, MatB<const T>{abar, n, m * n}, MatB<T>{tmp, n, m * n}, skip));
  return gemm<T>(c, batch, m, n, m, T(1), uv, true, MatB<const T>{tmp, n, m * n}, false, T(0), MatB<T>{abar, n, m * n},
                 MASK_FULL, skip);
}

#define INST(T)                                                                                                 \
  template size_t ws_gesvd_fwd<T>(int64_t, int64_t, int64_t);                                                   \
  template size_t ws_gesvd_bwd<T>(int64_t, int64_t, int64_t);                                                   \
  template dla_status gesvd_fwd<T>(const Ctx&, int64_t, int64_t, int64_t, T*, T*, T*);                          \
  template dla_status gesvd_bwd<T>(const Ctx&, int64_t, int64_t, int64_t, T*, const T*, const T*, const T*,     \
                                   const T*, const T*, const T*, T);
INST(double)
INST(float)

}  // namespace dlab
