#include <algorithm>
// Recursive (divide-and-conquer) triangular algorithms over a batch:
// trsm, trmm, potrf (lower), potri (trtri + lauum, lower), all in place.
//
// Every level splits the triangle at a multiple of NB; the off-diagonal work
// is one batched GEMM (gemm.cu, FP64 DMMA / FP32 FFMA) with K = n/2 at the
// top level, so large problems (n = 1024 .. 4096) are tensor-core bound
// rather than bandwidth bound.  Leaves (n <= NB = 64) are shared-memory
// kernels: one CTA per (slice, vector chunk), a warp per vector with
// shuffle-broadcast pivots.
//
// Reference algorithms these replace (same results up to rounding order):
//   trsm  dl/blas.hpp:307-395     trmm dl/blas.hpp:202-291
//   potrf dl/cholesky.hpp:35-88   potri dl/cholesky.hpp:105-147
#include <mutex>
#include <vector>

#include "chol64.cuh"
#include "common.cuh"
#include "ops.cuh"

namespace dlab {
namespace {

constexpr int NB = 64;        // leaf size
constexpr int LEAF_VEC = 32;  // vectors per CTA in the trmm leaf
constexpr int LDS = NB + 1;   // smem row stride (conflict-free column reads)

template <typename T>
MatB<const T> C_(MatB<T> m) {
  return MatB<const T>{m.p, m.ld, m.bs};
}

int64_t split_point(int64_t n) {
  int64_t h = (n / 2 + NB - 1) / NB * NB;
  return h >= n ? n - NB : h;
}

// Effective triangle S (nb x nb) of a leaf solve/multiply, in smem:
//   left : S = op(T_kk)          (vectors are columns of the X block)
//   right: S = op(T_kk)^T        (vectors are rows of the X block)
// `slower` says whether S is lower triangular.
template <typename T>
__device__ void load_effective(T* S, MatB<const T> t, int64_t b, int nb, bool s_from_transpose_of_t,
                               bool slower) {
  for (int e = threadIdx.x; e < nb * nb; e += blockDim.x) {
    const int i = e / nb, j = e % nb;
    T v = s_from_transpose_of_t ? *t.at(b, j, i) : *t.at(b, i, j);
    if (slower ? (j > i) : (j < i)) v = T(0);
    S[i * LDS + j] = v;
  }
}

// Blocked leaf trsm (the hot one): 64 vectors per CTA, the effective
// triangle S re-indexed to lower form (an upper S is solved in reversed
// order), forward substitution in 8-row blocks: each 8 x 8 diagonal block is
// solved per vector with precomputed reciprocal pivots (as the reference's
// left solve multiplies by 1/t_ii, dl/blas.hpp:353-354), then the rows below
// are updated by an (rows x 8) x (8 x 64) FP64 DMMA product in shared memory.
// alpha is applied on load; with `check` the CTA first tests the diagonal for
// an exact zero (SINGULAR, slice left untouched, dl/blas.hpp:310-314).
constexpr int BV = 64;  // vectors per CTA

template <typename T>
__device__ __forceinline__ void mma884(T& c0, T& c1, T a, T b);
template <>
__device__ __forceinline__ void mma884<double>(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

template <typename T>
__global__ void __launch_bounds__(128) k_trsm_leaf_blk(int nb, int64_t nvec, MatB<const T> t, MatB<T> x, bool right,
                                                       bool s_tt, bool slower, T alpha, bool check,
                                                       int32_t* info) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T* S = reinterpret_cast<T*>(smem_raw);  // [64][LDS], lower form
  T* V = S + NB * LDS;                    // [BV][LDS], vector-major
  T* rd = V + BV * LDS;                   // [64] reciprocal pivots
  __shared__ int zero_at;
  const int64_t chunks = (nvec + BV - 1) / BV;
  const int64_t b = blockIdx.x / chunks, v0 = (blockIdx.x % chunks) * BV;
  if (slice_failed(info, b)) return;
  const int nv = (int)min((int64_t)BV, nvec - v0);
  const int tid = threadIdx.x;
  // S' (lower): S'[i][j] = S[nb-1-i][nb-1-j] when S is upper; zero padded to 64.
  // Loads are issued 8 per thread before any shared store (memory-level
  // parallelism: the leaf is latency bound otherwise).
  for (int e0 = tid; e0 < NB * NB; e0 += 8 * 128) {
    T v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int e = e0 + u * 128, i = e / NB, j = e % NB;
      v[u] = T(0);
      if (i < nb && j < nb && j <= i) {
        const int si = slower ? i : nb - 1 - i, sj = slower ? j : nb - 1 - j;
        v[u] = s_tt ? *t.at(b, sj, si) : *t.at(b, si, sj);
      }
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int e = e0 + u * 128;
      S[(e / NB) * LDS + e % NB] = v[u];
    }
  }
  for (int e0 = tid; e0 < BV * NB; e0 += 8 * 128) {
    T val[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int e = e0 + u * 128;
      int v, i;
      if (right) { v = e / NB; i = e % NB; } else { i = e / BV; v = e % BV; }
      val[u] = T(0);
      if (v < nv && i < nb) {
        const int si = slower ? i : nb - 1 - i;
        val[u] = alpha * (right ? *x.at(b, v0 + v, si) : *x.at(b, si, v0 + v));
      }
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int e = e0 + u * 128;
      int v, i;
      if (right) { v = e / NB; i = e % NB; } else { i = e / BV; v = e % BV; }
      V[v * LDS + i] = val[u];
    }
  }
  if (tid == 0) zero_at = -1;
  __syncthreads();
  if (tid < NB) {
    const T d = tid < nb ? S[tid * LDS + tid] : T(1);
    rd[tid] = T(1) / d;
    if (check && tid < nb && d == T(0)) atomicMax(&zero_at, 0);
  }
  __syncthreads();
  if (check && zero_at >= 0) {
    if (tid == 0) {
      int first = -1;
      for (int k = 0; k < nb && first < 0; ++k)
        if (*t.at(b, k, k) == T(0)) first = k;
      record_failure(info, b, DLA_ERR_SINGULAR, first);
    }
    return;
  }
  const int warp = tid >> 5, lane = tid & 31, fr = lane >> 2, fc = lane & 3;
  for (int c0 = 0; c0 < nb; c0 += 8) {
    // 1) 8 x 8 diagonal block, one thread per vector
    if (tid < nv) {
      T* xv = V + tid * LDS;
      for (int i = c0; i < c0 + 8 && i < nb; ++i) {
        T acc = xv[i];
        for (int p = c0; p < i; ++p) acc -= S[i * LDS + p] * xv[p];
        xv[i] = acc * rd[i];
      }
    }
    __syncthreads();
    // 2) rows below: V[:, r] -= S'[r, c0:c0+8] V[:, c0:c0+8]  (DMMA, K = 8)
    const int r0 = c0 + 8;
    const int rtiles = (nb - r0 + 7) / 8;
    const int ntiles = rtiles * (BV / 8);
    if constexpr (sizeof(T) == 8) {
      for (int tile = warp; tile < ntiles; tile += 4) {
        const int rt = r0 + (tile / (BV / 8)) * 8, nt = (tile % (BV / 8)) * 8;
        T acc0 = T(0), acc1 = T(0);
#pragma unroll
        for (int kk = 0; kk < 8; kk += 4) {
          const T af = S[(rt + fr) * LDS + c0 + kk + fc];
          const T bf = V[(nt + fr) * LDS + c0 + kk + fc];
          mma884<T>(acc0, acc1, af, bf);
        }
        // accumulator (row fr, vectors 2fc, 2fc+1)
        V[(nt + 2 * fc) * LDS + rt + fr] -= acc0;
        V[(nt + 2 * fc + 1) * LDS + rt + fr] -= acc1;
      }
    } else {
      for (int e = tid; e < rtiles * 8 * BV; e += blockDim.x) {
        const int r = r0 + e / BV, v = e % BV;
        T acc = T(0);
#pragma unroll
        for (int p = 0; p < 8; ++p) acc += S[r * LDS + c0 + p] * V[v * LDS + c0 + p];
        V[v * LDS + r] -= acc;
      }
    }
    __syncthreads();
  }
  for (int e = tid; e < BV * NB; e += blockDim.x) {
    int v, i;
    if (right) { v = e / NB; i = e % NB; } else { i = e / BV; v = e % BV; }
    if (v < nv && i < nb) {
      const int si = slower ? i : nb - 1 - i;
      T* dst = right ? x.at(b, v0 + v, si) : x.at(b, si, v0 + v);
      *dst = V[v * LDS + i];
    }
  }
}

// Leaf trmm: y = alpha S x per vector (in place in X).
template <typename T>
__global__ void __launch_bounds__(256) k_trmm_leaf(int nb, int64_t nvec, MatB<const T> t, MatB<T> x, bool right,
                                                   bool s_from_tt, bool slower, T alpha, const int32_t* skip) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T* S = reinterpret_cast<T*>(smem_raw);
  T* V = S + NB * LDS;
  const int64_t chunks = (nvec + LEAF_VEC - 1) / LEAF_VEC;
  const int64_t b = blockIdx.x / chunks, v0 = (blockIdx.x % chunks) * LEAF_VEC;
  if (slice_failed(skip, b)) return;
  const int nv = (int)min((int64_t)LEAF_VEC, nvec - v0);
  load_effective(S, t, b, nb, s_from_tt, slower);
  for (int e = threadIdx.x; e < nv * nb; e += blockDim.x) {
    int v, i;
    if (right) { v = e / nb; i = e % nb; } else { i = e / nv; v = e % nv; }
    V[v * LDS + i] = right ? *x.at(b, v0 + v, i) : *x.at(b, i, v0 + v);
  }
  __syncthreads();
  for (int e = threadIdx.x; e < nv * nb; e += blockDim.x) {
    int v, i;
    if (right) { v = e / nb; i = e % nb; } else { i = e / nv; v = e % nv; }
    const T* xv = V + v * LDS;
    const T* srow = S + i * LDS;
    T acc = T(0);
    const int p0 = slower ? 0 : i, p1 = slower ? i + 1 : nb;
    for (int p = p0; p < p1; ++p) acc += srow[p] * xv[p];
    T* dst = right ? x.at(b, v0 + v, i) : x.at(b, i, v0 + v);
    *dst = alpha * acc;
  }
}

// Leaf Cholesky of a diagonal block (lower triangle read; strict upper of the
// block zeroed).  Right-looking, one column per step.  `k0` is the block's
// global offset for the NOT_SPD step index (dl/cholesky.hpp:49-53).
template <typename T>
__global__ void __launch_bounds__(256) k_potrf_leaf(int nb, int64_t k0, MatB<T> a, int32_t* info) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T* S = reinterpret_cast<T*>(smem_raw);
  __shared__ int flag;
  const int64_t b = blockIdx.x;
  if (slice_failed(info, b)) return;
  T* base = a.at(b, 0, 0);
  for (int e0 = threadIdx.x; e0 < nb * nb; e0 += 8 * 256) {  // 8 loads in flight per thread
    T v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int e = e0 + u * 256, i = e / nb, j = e % nb;
      v[u] = (e < nb * nb && j <= i) ? base[i * a.ld + j] : T(0);
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int e = e0 + u * 256;
      if (e < nb * nb) S[(e / nb) * CH_LD + e % nb] = v[u];
    }
  }
  __syncthreads();
  const int failed = chol_smem64<T>(S, nb, &flag);
  if (failed >= 0) {
    if (threadIdx.x == 0) record_failure(info, b, DLA_ERR_NOT_SPD, k0 + failed);
    return;
  }
  for (int e = threadIdx.x; e < nb * nb; e += 256) {
    const int i = e / nb, j = e % nb;
    base[i * a.ld + j] = j <= i ? S[i * CH_LD + j] : T(0);
  }
}

// Leaf lower-triangular inverse (in place): column j of W^{-1} solves
// L x = e_j by forward substitution; one thread per column.
template <typename T>
__global__ void __launch_bounds__(128) k_trtri_leaf(int nb, MatB<T> a, const int32_t* skip) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T* S = reinterpret_cast<T*>(smem_raw);
  T* W = S + NB * LDS;
  const int64_t b = blockIdx.x;
  if (slice_failed(skip, b)) return;
  for (int e = threadIdx.x; e < nb * nb; e += blockDim.x) {
    const int i = e / nb, j = e % nb;
    S[i * LDS + j] = j <= i ? *a.at(b, i, j) : T(0);
  }
  __syncthreads();
  for (int j = threadIdx.x; j < nb; j += blockDim.x) {
    for (int i = 0; i < j; ++i) W[i * LDS + j] = T(0);
    for (int i = j; i < nb; ++i) {
      T acc = (i == j) ? T(1) : T(0);
      for (int k = j; k < i; ++k) acc -= S[i * LDS + k] * W[k * LDS + j];
      W[i * LDS + j] = acc / S[i * LDS + i];
    }
  }
  __syncthreads();
  for (int e = threadIdx.x; e < nb * nb; e += blockDim.x) {
    const int i = e / nb, j = e % nb;
    if (j <= i) *a.at(b, i, j) = W[i * LDS + j];
  }
}

// Leaf lauum (lower): B = W^T W on the lower triangle, in place.
template <typename T>
__global__ void __launch_bounds__(256) k_lauum_leaf(int nb, MatB<T> a, const int32_t* skip) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T* S = reinterpret_cast<T*>(smem_raw);
  const int64_t b = blockIdx.x;
  if (slice_failed(skip, b)) return;
  for (int e = threadIdx.x; e < nb * nb; e += blockDim.x) {
    const int i = e / nb, j = e % nb;
    S[i * LDS + j] = j <= i ? *a.at(b, i, j) : T(0);
  }
  __syncthreads();
  for (int e = threadIdx.x; e < nb * nb; e += blockDim.x) {
    const int i = e / nb, j = e % nb;
    if (j > i) continue;
    T acc = T(0);
    for (int k = i; k < nb; ++k) acc += S[k * LDS + i] * S[k * LDS + j];
    *a.at(b, i, j) = acc;
  }
}

template <typename T>
size_t leaf_smem(int vecs) {
  return sizeof(T) * (size_t)(NB * LDS + vecs * LDS);
}

// ---------------------------------------------------------------- drivers
// trsm on the triangle of size nt (the X extent along the triangle is nt,
// the other extent nother).  Assumes alpha already applied.
template <typename T>
dla_status trsm_core(const Ctx& c, int64_t batch, int64_t nt, int64_t nother, MatB<const T> t, MatB<T> x,
                     bool right, bool trans, bool lower, T alpha = T(1), bool check = false) {
  const bool op_lower = (lower != trans);
  if (nt <= NB) {
    // left: S = op(T); right: S = op(T)^T.  S(i,j) = T(j,i) when
    // (left && trans) || (right && !trans).
    const bool s_tt = right ? !trans : trans;
    const bool slower = right ? !op_lower : op_lower;
    const int64_t chunks = (nother + BV - 1) / BV;
    const size_t sm = sizeof(T) * (size_t)(NB * LDS + BV * LDS + NB);
    ensure_smem_attr(k_trsm_leaf_blk<T>, sm);
    k_trsm_leaf_blk<T><<<(unsigned)(batch * chunks), 128, sm, c.stream>>>((int)nt, nother, t, x, right, s_tt, slower,
                                                                          alpha, check, c.info);
    DLAB_LAUNCH_CHECK();
    return DLA_OK;
  }
  const int64_t n1 = split_point(nt), n2 = nt - n1;
  MatB<const T> t11 = t, t22 = t.sub(n1, n1);
  MatB<const T> t21 = t.sub(n1, 0), t12 = t.sub(0, n1);
  if (!right) {
    MatB<T> x1 = x, x2 = x.sub(n1, 0);
    if (op_lower) {
      DLAB_TRY(trsm_core<T>(c, batch, n1, nother, t11, x1, right, trans, lower));
      // X2 -= op(T)21 X1, op(T)21 = trans ? T12^T : T21
      DLAB_TRY(gemm<T>(c, batch, n2, nother, n1, T(-1), trans ? t12 : t21, trans, C_(x1), false, T(1), x2,
                       MASK_FULL, c.info));
      DLAB_TRY(trsm_core<T>(c, batch, n2, nother, t22, x2, right, trans, lower));
    } else {
      DLAB_TRY(trsm_core<T>(c, batch, n2, nother, t22, x2, right, trans, lower));
      // X1 -= op(T)12 X2, op(T)12 = trans ? T21^T : T12
      DLAB_TRY(gemm<T>(c, batch, n1, nother, n2, T(-1), trans ? t21 : t12, trans, C_(x2), false, T(1), x1,
                       MASK_FULL, c.info));
      DLAB_TRY(trsm_core<T>(c, batch, n1, nother, t11, x1, right, trans, lower));
    }
  } else {
    MatB<T> x1 = x, x2 = x.sub(0, n1);
    if (op_lower) {  // Y op(T) = X with op(T) lower: Y2 first
      DLAB_TRY(trsm_core<T>(c, batch, n2, nother, t22, x2, right, trans, lower));
      // X1 -= Y2 op(T)21
      DLAB_TRY(gemm<T>(c, batch, nother, n1, n2, T(-1), C_(x2), false, trans ? t12 : t21, trans, T(1), x1,
                       MASK_FULL, c.info));
      DLAB_TRY(trsm_core<T>(c, batch, n1, nother, t11, x1, right, trans, lower));
    } else {
      DLAB_TRY(trsm_core<T>(c, batch, n1, nother, t11, x1, right, trans, lower));
      // X2 -= Y1 op(T)12
      DLAB_TRY(gemm<T>(c, batch, nother, n2, n1, T(-1), C_(x1), false, trans ? t21 : t12, trans, T(1), x2,
                       MASK_FULL, c.info));
      DLAB_TRY(trsm_core<T>(c, batch, n2, nother, t22, x2, right, trans, lower));
    }
  }
  return DLA_OK;
}

template <typename T>
dla_status trmm_core(const Ctx& c, int64_t batch, int64_t nt, int64_t nother, MatB<const T> t, MatB<T> x,
                     bool right, bool trans, bool lower, T alpha) {
  const bool op_lower = (lower != trans);
  if (nt <= NB) {
    const bool s_tt = right ? !trans : trans;
    const bool slower = right ? !op_lower : op_lower;
    const int64_t chunks = (nother + LEAF_VEC - 1) / LEAF_VEC;
    const size_t sm = leaf_smem<T>(LEAF_VEC);
    ensure_smem_attr(k_trmm_leaf<T>, sm);
    k_trmm_leaf<T><<<(unsigned)(batch * chunks), 256, sm, c.stream>>>((int)nt, nother, t, x, right, s_tt, slower,
                                                                       alpha, c.info);
    DLAB_LAUNCH_CHECK();
    return DLA_OK;
  }
  const int64_t n1 = split_point(nt), n2 = nt - n1;
  MatB<const T> t11 = t, t22 = t.sub(n1, n1), t21 = t.sub(n1, 0), t12 = t.sub(0, n1);
  if (!right) {
    MatB<T> x1 = x, x2 = x.sub(n1, 0);
    if (op_lower) {  // Y2 = a(O21 X1 + O22 X2) first, then Y1 = a O11 X1
      DLAB_TRY(trmm_core<T>(c, batch, n2, nother, t22, x2, right, trans, lower, alpha));
      DLAB_TRY(gemm<T>(c, batch, n2, nother, n1, alpha, trans ? t12 : t21, trans, C_(x1), false, T(1), x2,
                       MASK_FULL, c.info));
      DLAB_TRY(trmm_core<T>(c, batch, n1, nother, t11, x1, right, trans, lower, alpha));
    } else {  // Y1 = a(O11 X1 + O12 X2) first
      DLAB_TRY(trmm_core<T>(c, batch, n1, nother, t11, x1, right, trans, lower, alpha));
      DLAB_TRY(gemm<T>(c, batch, n1, nother, n2, alpha, trans ? t21 : t12, trans, C_(x2), false, T(1), x1,
                       MASK_FULL, c.info));
      DLAB_TRY(trmm_core<T>(c, batch, n2, nother, t22, x2, right, trans, lower, alpha));
    }
  } else {
    MatB<T> x1 = x, x2 = x.sub(0, n1);
    if (op_lower) {  // Y1 = a(X1 O11 + X2 O21) first
      DLAB_TRY(trmm_core<T>(c, batch, n1, nother, t11, x1, right, trans, lower, alpha));
      DLAB_TRY(gemm<T>(c, batch, nother, n1, n2, alpha, C_(x2), false, trans ? t12 : t21, trans, T(1), x1,
                       MASK_FULL, c.info));
      DLAB_TRY(trmm_core<T>(c, batch, n2, nother, t22, x2, right, trans, lower, alpha));
    } else {  // Y2 = a(X1 O12 + X2 O22) first
      DLAB_TRY(trmm_core<T>(c, batch, n2, nother, t22, x2, right, trans, lower, alpha));
      DLAB_TRY(gemm<T>(c, batch, nother, n2, n1, alpha, C_(x1), false, trans ? t21 : t12, trans, T(1), x2,
                       MASK_FULL, c.info));
      DLAB_TRY(trmm_core<T>(c, batch, n1, nother, t11, x1, right, trans, lower, alpha));
    }
  }
  return DLA_OK;
}

template <typename T>
dla_status potrf_blocked(const Ctx& c, int64_t batch, int64_t n, MatB<T> a, int64_t kbase, bool* upper_zeroed = nullptr);

// L11^{-1} buffer of the blocked Cholesky's throughput path (large batches of
// multi-chunk panels); sms < 0 gives the bound the workspace query uses.
template <typename T, int NBP>
size_t potrf_linv_bytes(int64_t batch, int64_t n, int sms) {
  if (NBP != 64 || n <= 2 * NBP) return 0;
  if (sms >= 0 && batch * ((n + 63) / 64) <= sms) return 0;
  return sizeof(T) * (size_t)batch * 64 * 64;
}

// DLA_POTRF_MODE (tuning switch): 0 auto (blocked look-ahead), 1 recursive,
// 2 blocked, 3 persistent tile dataflow (f64)
int potrf_mode() {
  static const int mode = [] {
    const char* e = getenv("DLA_POTRF_MODE");
    return e ? atoi(e) : 0;
  }();
  return mode;
}
int potrf_nb() {
  static const int nbp = [] {
    const char* e = getenv("DLA_POTRF_NB");  // tuning switch: 128-wide panels
    return e ? atoi(e) : 0;
  }();
  return nbp == 128 ? 128 : 64;
}

template <typename T>
dla_status potrf_rec(const Ctx& c, int64_t batch, int64_t n, int64_t k0, MatB<T> a) {
  // Bottom of the recursion: blocked right-looking with the fused panel
  // kernel (rank-64 updates are fine at this size; above it, the recursive
  // split keeps the SYRK/trsm GEMMs at K = n/2).
  if (n > NB && n <= 512 && batch <= 64) return potrf_blocked<T>(c, batch, n, a, k0);
  if (n <= NB) {
    const size_t sm = sizeof(T) * NB * LDS;
    (void)sm;
    k_potrf_leaf<T><<<(unsigned)batch, 256, sizeof(T) * NB * CH_LD, c.stream>>>((int)n, k0, a, c.info);
    DLAB_LAUNCH_CHECK();
    return DLA_OK;
  }
  const int64_t n1 = split_point(n), n2 = n - n1;
  DLAB_TRY(potrf_rec<T>(c, batch, n1, k0, a));
  MatB<T> a21 = a.sub(n1, 0), a22 = a.sub(n1, n1);
  // A21 <- A21 L11^{-T}
  if (inv_eligible<T>(n1) && n2 >= 128)  // one triangular GEMM with L11^{-1}
    DLAB_TRY(trsm_inv<T>(c, batch, n2, n1, C_(a), a21, true, true, true, T(1)));
  else
    DLAB_TRY(trsm_core<T>(c, batch, n1, n2, C_(a), a21, true, true, true));
  // A22 -= A21 A21^T (lower triangle only)
  DLAB_TRY(gemm<T>(c, batch, n2, n2, n1, T(-1), C_(a21), false, C_(a21), true, T(1), a22, MASK_LOWER, c.info));
  return potrf_rec<T>(c, batch, n2, k0 + n1, a22);
}

// k-column of DMMA k-step s for fragment column fc (see k_potrf_panel)
__device__ __forceinline__ int kcol(int s, int fc) { return ((s & ~3) << 2) + 4 * fc + (s & 3); }

// 8-byte cp.async global -> shared, zero-filled when !pred
__device__ __forceinline__ void st_async8(void* smem, const void* gmem, bool pred) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(sa), "l"(gmem), "r"(pred ? 8 : 0));
}

#ifndef DLAB_PANEL_TALL
#define DLAB_PANEL_TALL 1  // fp64 panel: chunk solve interleaved with the factorization
#endif

#ifdef DLAB_PANEL_PROF
// tuning build only: %globaltimer stamps of CTA 0's phases per panel step
__device__ unsigned long long g_pprof[128][8];
#define PSTAMP(i)                                                   \
  do {                                                              \
    if (blockIdx.x == 0 && threadIdx.x == 0) {                      \
      unsigned long long t_;                                        \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));        \
      g_pprof[(k0 / 64) & 127][i] = t_;                             \
      g_prof_row = (int)(k0 / 64);                                  \
    }                                                               \
  } while (0)
#else
#define PSTAMP(i)
#endif

// One block column of the right-looking Cholesky in ONE launch: every CTA
// factors the NBP x NBP diagonal block (redundantly — it is latency, not
// work), CTA 0 stores L11, and each CTA solves its own 64 rows of the panel
// A21 <- A21 L11^{-T} in shared memory (blocked substitution + DMMA).
template <typename T, int NBP>
__global__ void __launch_bounds__(256, 1) k_potrf_panel(int nb, int64_t rest, int64_t k0, MatB<T> akk, MatB<T> a21,
                                                     int32_t* info, int* arrive, MatB<const T> lp, int kp) {
  // Row stride 65: row-per-lane accesses are conflict-free.  The DMMA
  // fragments (8 rows x 4 k) of the fp64 path take k-column 4 fc + s within
  // each 16-column group (kcol) instead of fc + 4 s: with stride 65 the
  // fr + fc pattern is a 4-way bank conflict, fr + 4 fc a 2-wavefront load.
  constexpr int LD = NBP + 1;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T* S = reinterpret_cast<T*>(smem_raw);
  T* V = S + NBP * LD;
  T* rd = V + 64 * LD;
  T* P = rd + NBP;  // kp > 0: the previous panel's columns at this block's diagonal rows (64 x kp)
  __shared__ int flag;
  const int64_t chunks = rest > 0 ? (rest + 63) / 64 : 1;
  const int64_t b = blockIdx.x / chunks, cid = blockIdx.x % chunks;
  if (slice_failed(info, b)) return;
  const int tid = threadIdx.x;
  PSTAMP(0);
  T* base = akk.at(b, 0, 0);
  constexpr bool tall = NBP == 64 && sizeof(T) == 8 && DLAB_PANEL_TALL;
  const int64_t r0 = cid * 64;
  const int nv = rest > 0 ? (int)min((int64_t)64, rest - r0) : 0;
  T* pan = a21.at(b, r0, 0);
  T* PC = P + 64 * LD;  // tall: the previous panel's columns at the chunk rows (nv x kp)
  if constexpr (tall) {
    // every operand of the step in flight at once: A11 (lower), the chunk
    // rows, and the previous panel's rows Pd (diagonal) and Pc (chunk)
    const T* gp = lp.at(b, 0, 0);
#pragma unroll 4
    for (int u = 0; u < 16; ++u) {
      const int e = tid + u * 256, i = e / 64, j = e % 64;
      st_async8(S + i * LD + j, base + (i < nb && j <= i ? i * akk.ld + j : 0), i < nb && j <= i);
      st_async8(V + i * LD + j, pan + (i < nv && j < nb ? i * a21.ld + j : 0), i < nv && j < nb);
      if (kp > 0) {
        st_async8(P + i * LD + j, gp + (i < nb && j < kp ? i * lp.ld + j : 0), i < nb && j < kp);
        st_async8(PC + i * LD + j, gp + (i < nv && j < kp ? (nb + r0 + i) * lp.ld + j : 0), i < nv && j < kp);
      }
    }
    asm volatile("cp.async.wait_all;\n" ::: "memory");
    __syncthreads();
  }
  for (int e0 = tid; !tall && e0 < NBP * NBP; e0 += 8 * 256) {
    T v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int e = e0 + u * 256, i = e / NBP, j = e % NBP;
      v[u] = (i < nb && j <= i) ? base[i * akk.ld + j] : T(0);
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int e = e0 + u * 256;
      S[(e / NBP) * LD + e % NBP] = v[u];
    }
  }
  for (int e0 = tid; !tall && e0 < 64 * NBP; e0 += 8 * 256) {  // panel rows, loads in flight during the factorization
    T v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int e = e0 + u * 256, vv = e / NBP, i = e % NBP;
      v[u] = (vv < nv && i < nb) ? pan[vv * a21.ld + i] : T(0);
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int e = e0 + u * 256;
      V[(e / NBP) * LD + e % NBP] = v[u];
    }
  }
  PSTAMP(1);
  if constexpr (NBP == 64) {
    if (kp > 0) {
      // Fused look-ahead column update: this block column still lacks the
      // previous panel's rank-kp update, A11 -= Pd Pd^T (lower) and
      // A21 -= Pc Pd^T, applied here on FP64 DMMA instead of by a separate
      // GEMM launch on the critical chain.  Pd is staged in shared memory;
      // each warp streams its 8 Pc rows' fragments from L2 once per k-step
      // and reuses them across all 8 column tiles.
      const T* gp = lp.at(b, 0, 0);
      if constexpr (!tall) {  // all 16 loads of a thread in flight before the stores
        T v[16];
#pragma unroll
        for (int u = 0; u < 16; ++u) {
          const int e = tid + u * 256, i = e / 64, k = e % 64;
          v[u] = (i < nb && k < kp) ? gp[i * lp.ld + k] : T(0);
        }
#pragma unroll
        for (int u = 0; u < 16; ++u) {
          const int e = tid + u * 256;
          P[(e / 64) * LD + e % 64] = v[u];
        }
      }
      __syncthreads();
      const int warp = tid >> 5, lane = tid & 31, fr = lane >> 2, fc = lane & 3;
      if constexpr (sizeof(T) == 8) {
        // A11 lower tiles of row tile `warp` first (the factorization needs them)
        double acc[8][2];
#pragma unroll
        for (int t = 0; t < 8; ++t) acc[t][0] = acc[t][1] = 0.0;
        for (int kk = 0; kk < kp; kk += 4) {
          const int kc = tall ? kcol(kk >> 2, fc) : kk + fc;
          const double af = P[(8 * warp + fr) * LD + kc];
#pragma unroll
          for (int t = 0; t < 8; ++t) {
            if (t > warp) break;
            const double bf = P[(8 * t + fr) * LD + kc];
            asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                         : "+d"(acc[t][0]), "+d"(acc[t][1])
                         : "d"(af), "d"(bf));
          }
        }
#pragma unroll
        for (int t = 0; t < 8; ++t) {
          if (t > warp) break;
          S[(8 * warp + fr) * LD + 8 * t + 2 * fc] -= acc[t][0];  // entries above the diagonal are scratch
          S[(8 * warp + fr) * LD + 8 * t + 2 * fc + 1] -= acc[t][1];
        }
      } else {
        for (int e = tid; e < 64 * 64; e += 256) {
          const int i = e / 64, j = e % 64;
          if (j > i) continue;
          T acc = T(0);
          for (int k = 0; k < kp; ++k) acc += P[i * LD + k] * P[j * LD + k];
          S[i * LD + j] -= acc;
        }
      }
    }
  }
  __syncthreads();
  PSTAMP(2);
  // A21 -= Pc Pd^T (the chunk rows) runs on warps 1-7 while warp 0 factors
  // the first 16 columns of A11 (chol_smem's side task)
  auto v_update = [&](int warp) {
    if constexpr (NBP == 64 && sizeof(T) == 8) {
      if (kp == 0) return;
      const int lane = tid & 31, fr = lane >> 2, fc = lane & 3;
      const T* gp = lp.at(b, 0, 0);
      for (int rt = warp - 1; rt < 8; rt += 7) {  // warp 1: row tiles 0, 7; warps 2..7: 1..6
        double acc[8][2];
#pragma unroll
        for (int t = 0; t < 8; ++t) acc[t][0] = acc[t][1] = 0.0;
        const int vr = 8 * rt + fr;
        const T* arow = gp + (int64_t)(nb + r0 + vr) * lp.ld;
        const bool okr = vr < nv;
        double afv[16];
#pragma unroll
        for (int q = 0; q < 16; ++q)
          afv[q] = tall ? PC[vr * LD + kcol(q, fc)] : (okr && 4 * q < kp) ? arow[4 * q + fc] : 0.0;
#pragma unroll
        for (int q = 0; q < 16; ++q) {
          const double af = afv[q];
#pragma unroll
          for (int t = 0; t < 8; ++t) {
            const double bf = P[(8 * t + fr) * LD + (tall ? kcol(q, fc) : 4 * q + fc)];
            asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                         : "+d"(acc[t][0]), "+d"(acc[t][1])
                         : "d"(af), "d"(bf));
          }
        }
#pragma unroll
        for (int t = 0; t < 8; ++t) {
          V[vr * LD + 8 * t + 2 * fc] -= acc[t][0];
          V[vr * LD + 8 * t + 2 * fc + 1] -= acc[t][1];
        }
      }
    } else {
      if (kp == 0 || warp != 1) return;
      const T* gp = lp.at(b, 0, 0);
      for (int e = tid - 32; e < 64 * 64; e += 32) {
        const int vv = e / 64, j = e % 64;
        if (vv >= nv) continue;
        const T* ga = gp + (int64_t)(nb + r0 + vv) * lp.ld;
        T acc = T(0);
        for (int k = 0; k < kp; ++k) acc += ga[k] * P[j * LD + k];
        V[vv * LD + j] -= acc;
      }
    }
  };
  // Every CTA reads A11 from global memory; the CTA that arrives LAST (all
  // others have their copy in shared memory by then) writes L11 back over it
  // and re-arms the slice's counter for the next panel launch.
  __shared__ int last;
  int failed;
  if constexpr (tall) {
    // factor + chunk solve interleaved (V holds L21's rows after).  The
    // arrival (after the barrier above: this CTA's A11 copy is complete) is
    // issued now and its result consumed only after the factorization.
    int my = 0;
    if (tid == 0) my = atomicAdd(arrive + b, 1);
    failed = chol_tall64<LD>(reinterpret_cast<double*>(S), reinterpret_cast<double*>(V), nb, nv, &flag, v_update);
    if (tid == 0) last = my == (int)chunks - 1;
    __syncthreads();
  } else {
    if (tid == 0) last = atomicAdd(arrive + b, 1) == (int)chunks - 1;
    failed = chol_smem<T, NBP>(S, nb, &flag, v_update);  // (its first barrier publishes `last`)
  }
  PSTAMP(3);
  if (failed >= 0) {
    if (cid == 0 && tid == 0) record_failure(info, b, DLA_ERR_NOT_SPD, k0 + failed);
    return;
  }
  if (last) {
    if (tid == 0) arrive[b] = 0;
    for (int e = tid; e < nb * nb; e += 256) {
      const int i = e / nb, j = e % nb;
      base[i * akk.ld + j] = j <= i ? S[i * LD + j] : T(0);
    }
  }
  if (nv == 0) return;
  if constexpr (!tall) {
    for (int i = tid; i < NBP; i += 256) rd[i] = i < nb ? T(1) / S[i * LD + i] : T(1);
    __syncthreads();
    PSTAMP(4);
    blocked_fwd_subst<T, LD>(S, V, rd, nb, nv);  // row v: L11 x = a  <=>  x^T L11^T = a^T
    PSTAMP(5);
  }
  for (int e = tid; e < nv * nb; e += 256) {
    const int vv = e / nb, i = e % nb;
    pan[vv * a21.ld + i] = V[vv * LD + i];
  }
  PSTAMP(6);
}

// Throughput variant of the panel step for large batches (batch x chunks
// above the SM count, where the panel kernel's redundant per-CTA A11
// factorization would cost real throughput): ONE CTA per slice factors A11,
// writes L11 and L11^{-1} (into linv), and the panel solve becomes the
// batched DMMA GEMM A21 <- A21 L11^{-T} (in place: N = nb fits one tile).
template <typename T>
__global__ void __launch_bounds__(256) k_potrf_diag_inv(int nb, int64_t k0, MatB<T> akk, T* linv, int32_t* info) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T* S = reinterpret_cast<T*>(smem_raw);
  T* X = S + 64 * CH_LD;  // vector-major: X[v * CH_LD + i] = L11^{-1}(i, v)
  T* rd = X + 64 * CH_LD;
  __shared__ int flag;
  const int64_t b = blockIdx.x;
  if (slice_failed(info, b)) return;
  T* base = akk.at(b, 0, 0);
  for (int e = threadIdx.x; e < 64 * 64; e += 256) {
    const int i = e / 64, j = e % 64;
    S[i * CH_LD + j] = (i < nb && j <= i) ? base[i * akk.ld + j] : T(0);
    X[i * CH_LD + j] = (i == j) ? T(1) : T(0);
  }
  __syncthreads();
  const int failed = chol_smem64<T>(S, nb, &flag);
  if (failed >= 0) {
    if (threadIdx.x == 0) record_failure(info, b, DLA_ERR_NOT_SPD, k0 + failed);
    return;
  }
  for (int e = threadIdx.x; e < nb * nb; e += 256) {
    const int i = e / nb, j = e % nb;
    base[i * akk.ld + j] = j <= i ? S[i * CH_LD + j] : T(0);
  }
  for (int i = threadIdx.x; i < 64; i += 256) rd[i] = i < nb ? T(1) / S[i * CH_LD + i] : T(1);
  __syncthreads();
  blocked_fwd_subst<T>(S, X, rd, nb, nb);  // X rows v: L11 x = e_v
  T* out = linv + b * 64 * 64;
  for (int e = threadIdx.x; e < 64 * 64; e += 256) {
    const int i = e / 64, j = e % 64;
    out[e] = (i < nb && j < nb && j <= i) ? X[j * CH_LD + i] : T(0);  // L11^{-1}(i, j), lower
  }
}

// Right-looking blocked Cholesky (the reference's own loop structure,
// dl/cholesky.hpp:43-70, with nb = NBP): per block column one warp-panel leaf
// factorization and blocked DMMA panel solve (one launch, all rows of the
// panel in parallel, 64 per CTA) and masked DMMA SYRK updates of the
// trailing matrix.  Used for large single matrices where the recursive
// variant's deep chain of tiny GEMMs dominates.
// Persistent-grid cap of the TMA trailing update (DLA_SYRK_CAP: 0 = leave the
// concurrent panel its SMs, -1 = every SM, > 0 = that many CTAs; tuning switch).
inline int syrk_cap(int leave_panel, int sms) {
  static const int env = [] {
    const char* e = getenv("DLA_SYRK_CAP");
    return e ? atoi(e) : 0;
  }();
  if (env < 0) return sms;
  if (env > 0) return env;
  return leave_panel;
}

// *upper_zeroed (optional): when given, the strict upper triangle is zeroed
// here too, on the side stream once the bulk updates have slack (no kernel of
// the factorization reads it), instead of after the last panel.
template <typename T, int NBP>
dla_status potrf_blocked_nb(const Ctx& c, int64_t batch, int64_t n, MatB<T> a, int64_t kbase,
                            bool* upper_zeroed = nullptr) {
  const size_t sm = sizeof(T) * ((NBP + 64) * (NBP + 1) + NBP + (NBP == 64 ? 2 * 64 * (NBP + 1) : 0));
  ensure_smem_attr(k_potrf_panel<T, NBP>, sm);
  // Look-ahead on two streams: the main stream runs the critical chain
  // (panel k, then the update of block column k+1 only), the side stream the
  // bulk trailing update of step k, which overlaps panel k+1.  The side
  // update of step k-1 also writes block column k+1, so the main stream waits
  // for it before its own column update of step k (panel k itself only needs
  // side updates <= k-2, already ordered).  Fork/join by events: stream-
  // ordered w.r.t. the caller and capturable into a CUDA graph.
  const int64_t steps = (n + NBP - 1) / NBP;
  DLAB_SCRATCH(arrive, c, sizeof(int) * (size_t)batch);
  DLAB_SCRATCH(linv, c, (potrf_linv_bytes<T, NBP>(batch, n, c.sms)));
  if (cudaMemsetAsync(arrive.p, 0, sizeof(int) * (size_t)batch, c.stream) != cudaSuccess) return DLA_ERR_CUDA;
  // side / critical streams and events of THIS (device, caller stream),
  // held for the whole enqueue (include/dla.h: thread-safe across streams)
  ForkRes& la = fork_res(FORK_LOOKAHEAD, c.stream);
  std::lock_guard<std::mutex> la_lock(la.mu);
  la.grow(steps);
  static const bool prio = [] {
    const char* e = getenv("DLA_POTRF_PRIO");  // tuning switch: 0 keeps the chain on the caller's stream
    return e ? atoi(e) != 0 : true;
  }();
  Ctx side = c, cc = c;
  side.stream = la.side;
  // The bulk update runs persistent on sms - reserve CTAs: a 128 x 128 GEMM
  // CTA (212 KB smem) cannot share an SM with a panel CTA, so without a
  // reserve every panel launch of the critical chain first waits for update
  // tiles to drain.  Measured: the bulk update is the scarcer resource, so
  // the default reserve is 0; DLA_POTRF_RESERVE sets one (tuning switch).
  static const int reserve_env = [] {
    const char* e = getenv("DLA_POTRF_RESERVE");
    return e ? atoi(e) : -1;
  }();
  {
    const int64_t chunks0 = batch * ((n - NBP + 63) / 64);
    const int reserve = reserve_env > 0 ? (int)std::min<int64_t>(reserve_env, chunks0) : 0;
    if (reserve > 0 && reserve < c.sms) side.gemm_ctas = c.sms - reserve;
  }
  if (prio) cc.stream = la.crit;
  cudaEventRecord(la.ev[0], c.stream);
  cudaStreamWaitEvent(la.side, la.ev[0], 0);
  if (prio) cudaStreamWaitEvent(cc.stream, la.ev[0], 0);
  // Look-ahead with (optionally) grouped trailing updates.  Panels are taken in
  // groups of G.  After the last panel of group g the side stream applies
  // the whole group to every column >= (g+2) G NBP in ONE masked SYRK with
  // K = G NBP (a rank-64 update re-reads and re-writes the trailing triangle
  // for only 64 flops per element; grouping amortises that C traffic G-fold).
  // Before panel p (group g) the critical stream brings block column p up to
  // date with the panels the side updates have not covered — group g-1 and
  // the earlier panels of group g, contiguous in L, K <= (2G-1) NBP — after
  // waiting for side update g-2, the last one that writes column p.
  // Measured on B200 (tools/timeline.py): G = 1 is fastest at n = 1024 and
  // 4096 — the longer critical-path GEMM of G > 1 costs what the cheaper
  // bulk updates save — so DLA_POTRF_GROUP defaults to 1.
  static const int group = [] {
    const char* e = getenv("DLA_POTRF_GROUP");  // tuning switch
    const int gsz = e ? atoi(e) : 1;
    return gsz < 1 ? 1 : gsz;
  }();
  const int64_t G = group;
  const int64_t ngroups = (steps + G - 1) / G;
  // Step p's panel either runs the fused panel kernel (which, for NBP = 64,
  // also applies panel p-1's update to its own block column) or, for large
  // batches of multi-chunk panels, the per-slice factorization + batched
  // GEMM solve (then panel p-1's column update is a separate GEMM).
  auto chunks_of = [&](int64_t p) {
    const int64_t r = n - p * NBP - min((int64_t)NBP, n - p * NBP);
    return r > 0 ? (r + 63) / 64 : (int64_t)1;
  };
  auto throughput = [&](int64_t p) { return NBP == 64 && chunks_of(p) > 1 && batch * chunks_of(p) > c.sms; };
  auto fused = [&](int64_t p) { return NBP == 64 && G == 1 && p >= 1 && !throughput(p); };
  bool hook_fired = false;
  bool zeroed = false;
  dla_status st = DLA_OK;
  // every launch failure leaves the loop through the join below: work already
  // forked onto the side / critical streams is joined back to the caller's
  // stream before the scratch (carved from the caller's workspace) is released
#define LA_TRY(expr)          \
  if ((st = (expr)) != DLA_OK) \
    break
  for (int64_t p = 0; p < steps; ++p) {
    const int64_t k0 = p * NBP;
    const int64_t kb = min((int64_t)NBP, n - k0);
    const int64_t rest = n - k0 - kb;
    const int64_t g = p / G;
    if (p > 0 && !fused(p)) {  // column p: panels [max(0, (g-1) G), p)
      if (g >= 2) cudaStreamWaitEvent(cc.stream, la.done[g - 2], 0);
      const int64_t kk0 = std::max<int64_t>(0, (g - 1) * G) * NBP;
      MatB<T> lrows = a.sub(k0, kk0);
      LA_TRY(gemm<T>(cc, batch, n - k0, kb, k0 - kk0, T(-1), C_(lrows), false, C_(lrows), true, T(1), a.sub(k0, k0),
                       MASK_LOWER, c.info));
    } else if (p >= 2) {
      cudaStreamWaitEvent(cc.stream, la.done[p - 2], 0);  // the last side update that wrote column p
    }
    const int64_t chunks = chunks_of(p);
    if (throughput(p) && rest > 0) {
      // throughput path: one diagonal factorization per slice + a batched GEMM solve
      const size_t smd = sizeof(T) * (2 * 64 * CH_LD + 64);
      ensure_smem_attr(k_potrf_diag_inv<T>, smd);
      k_potrf_diag_inv<T><<<(unsigned)batch, 256, smd, cc.stream>>>((int)kb, kbase + k0, a.sub(k0, k0), linv.as<T>(),
                                                                     c.info);
      LA_TRY(launch_status());
      MatB<T> a21 = a.sub(k0 + kb, k0);
      LA_TRY(gemm<T>(cc, batch, rest, kb, kb, T(1), C_(a21), false, MatB<const T>{linv.as<T>(), 64, 64 * 64}, true,
                       T(0), a21, MASK_FULL, c.info, TRI_NONE, TRI_UPPER));
    } else {
      const int kp = fused(p) ? (int)NBP : 0;
      MatB<const T> lp = C_(p >= 1 ? a.sub(k0, k0 - NBP) : a);
      // the chain's priority as a launch attribute too: a CUDA graph captured
      // from these streams then carries it on the node itself
      cudaLaunchConfig_t cfg{};
      cfg.gridDim = dim3((unsigned)(batch * chunks));
      cfg.blockDim = dim3(256);
      cfg.dynamicSmemBytes = sm;
      cfg.stream = cc.stream;
      cudaLaunchAttribute attr[1];
      attr[0].id = cudaLaunchAttributePriority;
      attr[0].val.priority = la.prio_hi;
      cfg.attrs = attr;
      cfg.numAttrs = prio ? 1 : 0;
      if (cudaLaunchKernelEx(&cfg, k_potrf_panel<T, NBP>, (int)kb, rest, kbase + k0, a.sub(k0, k0),
                             a.sub(k0 + kb, k0), c.info, arrive.as<int>(), lp, kp) != cudaSuccess) {
        st = DLA_ERR_CUDA;
        break;
      }
      LA_TRY(launch_status());
    }
    if (c.potrf_hook && !hook_fired && kbase == 0 && c.potrf_hook->n == n &&
        c.potrf_hook->a == static_cast<const void*>(a.p) && k0 + kb >= c.potrf_hook->col) {
      c.potrf_hook->fn(c.potrf_hook->user, cc.stream);  // block columns [0, col) are final from here on
      hook_fired = true;
    }
    if (rest == 0) break;
    if (p % G == G - 1 || p == steps - 1) {  // last panel of group g: side update U(g)
      const int64_t c0 = (g + 2) * G * NBP;
      if (c0 < n) {
        cudaEventRecord(la.panel[g], cc.stream);
        cudaStreamWaitEvent(la.side, la.panel[g], 0);
        const int64_t gk0 = g * G * NBP;
        MatB<T> p2 = a.sub(c0, gk0);
        bool done_tma = false;
        if constexpr (sizeof(T) == 8) {
          MatB<const double> pd{reinterpret_cast<const double*>(p2.p), p2.ld, p2.bs};
          MatB<double> cd{reinterpret_cast<double*>(a.sub(c0, c0).p), a.ld, a.bs};
          static const bool la_tma = [] {
            // tuning switch: the TMA update kernel inside the look-ahead (measured
            // on par with the two-CTA/SM DMMA GEMM there, so off by default)
            const char* e = getenv("DLA_POTRF_SYRK_TMA");
            return e && atoi(e) != 0;
          }();
          if (la_tma && syrk_tma_eligible(n - c0, k0 + kb - gk0, pd, cd, batch)) {
            // the panel kernel of step p + 1 runs concurrently: leave it its SMs
            const int64_t pc = p + 1 < steps ? batch * chunks_of(p + 1) : 0;
            const int cap = (int)std::max<int64_t>(c.sms / 2, c.sms - pc);
            LA_TRY(syrk_tma(side, batch, n - c0, k0 + kb - gk0, -1.0, pd, 1.0, cd, syrk_cap(cap, c.sms)));
            done_tma = true;
          }
        }
        if (!done_tma)
          LA_TRY(gemm<T>(side, batch, n - c0, n - c0, k0 + kb - gk0, T(-1), C_(p2), false, C_(p2), true, T(1),
                         a.sub(c0, c0), MASK_LOWER, c.info));
      }
      cudaEventRecord(la.done[g], la.side);
    }
    // late in the factorization the side stream's updates are shorter than
    // the panel chain: the strict upper triangle is zeroed in that slack
    // (DLA_POTRF_ZERO_AT: the step, in % of the steps; tuning switch)
    static const int zero_at = [] {
      const char* e = getenv("DLA_POTRF_ZERO_AT");
      return e ? atoi(e) : 75;
    }();
    if (upper_zeroed && !zeroed && 100 * (p + 1) >= zero_at * steps) {
      LA_TRY(ew_square<T>(side, batch, n, a, /*tril*/ 0, T(1), c.info));
      zeroed = true;
    }
  }
#undef LA_TRY
  (void)ngroups;
  if (upper_zeroed) *upper_zeroed = zeroed && st == DLA_OK;
  cudaEventRecord(la.ev[1], la.side);
  cudaStreamWaitEvent(c.stream, la.ev[1], 0);
  if (prio) {
    cudaEventRecord(la.ev[2], cc.stream);
    cudaStreamWaitEvent(c.stream, la.ev[2], 0);
  }
  return st;
}

// Panel width: 128 halves the serial panel chain of a large matrix (each step
// costs one launch + one column update regardless of width); 64 keeps more
// CTAs busy for small n.  DLA_POTRF_NB overrides (tuning switch).
template <typename T>
dla_status potrf_blocked(const Ctx& c, int64_t batch, int64_t n, MatB<T> a, int64_t kbase, bool* upper_zeroed) {
  const bool wide = potrf_nb() == 128;
  return wide ? potrf_blocked_nb<T, 128>(c, batch, n, a, kbase, upper_zeroed)
              : potrf_blocked_nb<T, 64>(c, batch, n, a, kbase, upper_zeroed);
}

template <typename T>
dla_status trtri_rec(const Ctx& c, int64_t batch, int64_t n, MatB<T> a) {
  if (n <= NB) {
    const size_t sm = sizeof(T) * 2 * NB * LDS;
    ensure_smem_attr(k_trtri_leaf<T>, sm);
    k_trtri_leaf<T><<<(unsigned)batch, 128, sm, c.stream>>>((int)n, a, c.info);
    DLAB_LAUNCH_CHECK();
    return DLA_OK;
  }
  const int64_t n1 = split_point(n), n2 = n - n1;
  MatB<T> a21 = a.sub(n1, 0), a22 = a.sub(n1, n1);
  DLAB_TRY(trtri_rec<T>(c, batch, n1, a));
  // W21 <- W21 W11^{-1}   (right trmm with the already inverted W11)
  DLAB_TRY(trmm_core<T>(c, batch, n1, n2, C_(a), a21, true, false, true, T(1)));
  // W21 <- -W22^{-1} W21  (left solve with the not-yet-inverted W22)
  DLAB_TRY(ew_scale<T>(c, batch, n2, n1, a21, T(-1), c.info));
  DLAB_TRY(trsm_core<T>(c, batch, n2, n1, C_(a22), a21, false, false, true));
  return trtri_rec<T>(c, batch, n2, a22);
}

template <typename T>
dla_status lauum_rec(const Ctx& c, int64_t batch, int64_t n, MatB<T> a) {
  if (n <= NB) {
    const size_t sm = sizeof(T) * NB * LDS;
    k_lauum_leaf<T><<<(unsigned)batch, 256, sm, c.stream>>>((int)n, a, c.info);
    DLAB_LAUNCH_CHECK();
    return DLA_OK;
  }
  const int64_t n1 = split_point(n), n2 = n - n1;
  MatB<T> a21 = a.sub(n1, 0), a22 = a.sub(n1, n1);
  DLAB_TRY(lauum_rec<T>(c, batch, n1, a));
  // B11 += W21^T W21 (lower)
  DLAB_TRY(gemm<T>(c, batch, n1, n1, n2, T(1), C_(a21), true, C_(a21), false, T(1), a, MASK_LOWER, c.info));
  // B21 = W22^T W21
  DLAB_TRY(trmm_core<T>(c, batch, n2, n1, C_(a22), a21, false, true, true, T(1)));
  return lauum_rec<T>(c, batch, n2, a22);
}

}  // namespace

template <typename T>
dla_status trsm(const Ctx& c, int64_t batch, int64_t m, int64_t n, MatB<const T> t, MatB<T> x, bool right,
                bool trans, bool lower, T alpha, bool check_diag) {
  if (batch == 0 || m == 0 || n == 0) return DLA_OK;
  const int64_t nt = right ? n : m, no = right ? m : n;
  if (nt <= NB)  // one leaf: alpha and the zero-diagonal test fused into it
    return trsm_core<T>(c, batch, nt, no, t, x, right, trans, lower, alpha, check_diag && c.info);
  if (check_diag) DLAB_TRY(check_zero_diag<T>(c, batch, nt, t, c.info));
  if (trsv_eligible<T>(nt, no)) return trsv<T>(c, batch, m, n, t, x, right, trans, lower, alpha);
  if (inv_eligible<T>(nt) && no >= 128) return trsm_inv<T>(c, batch, m, n, t, x, right, trans, lower, alpha);
  DLAB_TRY(ew_scale<T>(c, batch, m, n, x, alpha, c.info));
  return trsm_core<T>(c, batch, nt, no, t, x, right, trans, lower);
}

template <typename T>
dla_status trmm(const Ctx& c, int64_t batch, int64_t m, int64_t n, MatB<const T> t, MatB<T> x, bool right,
                bool trans, bool lower, T alpha) {
  if (batch == 0 || m == 0 || n == 0) return DLA_OK;
  const int64_t nt = right ? n : m;
  if (nt >= 128) return trmm_gemm<T>(c, batch, m, n, t, x, right, trans, lower, alpha);
  return right ? trmm_core<T>(c, batch, n, m, t, x, right, trans, lower, alpha)
               : trmm_core<T>(c, batch, m, n, t, x, right, trans, lower, alpha);
}

template <typename T>
dla_status potrf_lower(const Ctx& c, int64_t batch, int64_t n, MatB<T> a, bool zero_upper, bool* upper_zeroed) {
  if (upper_zeroed) *upper_zeroed = false;
  if (batch == 0 || n == 0) return DLA_OK;
  ensure_smem_attr(k_potrf_leaf<T>, sizeof(T) * NB * CH_LD);
  ensure_smem_attr(k_lauum_leaf<T>, sizeof(T) * NB * LDS);
  const int mode = potrf_mode();
  if constexpr (sizeof(T) == 8) {  // 64 < n <= 128: the one-launch CTA-per-matrix kernel (small.cu)
    if (mode == 0 && n > 64 && n <= 128 && potrf_fwd_small_eligible<T>(n)) return potrf_small<T>(c, batch, n, a, true, /*check_sym*/ false);
  }
  // default: blocked right-looking with look-ahead (measured faster than the
  // recursive split at every n > 64 on B200, and still ~3% ahead of the
  // persistent tile-dataflow kernel at n = 1024 / 4096, whose per-column
  // chain is the same chol64 + tile solve).  Modes: 1 recursive, 2 blocked,
  // 3 tile dataflow (f64).
  bool tiles = false;
  if constexpr (sizeof(T) == 8) {
    MatB<double> ad{reinterpret_cast<double*>(a.p), a.ld, a.bs};
    tiles = mode == 3 && potrf_tiles_eligible(batch, n, ad);
    if (tiles) DLAB_TRY(potrf_tiles(c, batch, n, ad, 0));
  }
  const bool blocked = mode != 1 && n > NB;
  bool zeroed = false;  // the blocked schedule zeroes the strict upper triangle as it goes
  if (tiles) {
  } else if (blocked) DLAB_TRY(potrf_blocked<T>(c, batch, n, a, 0, &zeroed));
  else DLAB_TRY(potrf_rec<T>(c, batch, n, 0, a));
  if (upper_zeroed) *upper_zeroed = zeroed;
  if (!zero_upper || zeroed) return DLA_OK;  // else the caller zeroes it itself (off its critical path)
  return ew_square<T>(c, batch, n, a, /*tril*/ 0, T(1), c.info);
}

template <typename T>
dla_status potri_lower(const Ctx& c, int64_t batch, int64_t n, MatB<T> a) {
  if (batch == 0 || n == 0) return DLA_OK;
  ensure_smem_attr(k_potrf_leaf<T>, sizeof(T) * NB * CH_LD);
  ensure_smem_attr(k_lauum_leaf<T>, sizeof(T) * NB * LDS);
  if (inv_eligible<T>(n) || potri_fused_eligible<T>(n)) return potri_inv<T>(c, batch, n, a);
  DLAB_TRY(trtri_rec<T>(c, batch, n, a));
  DLAB_TRY(lauum_rec<T>(c, batch, n, a));
  return ew_square<T>(c, batch, n, a, /*copyltu*/ 2, T(1), c.info);
}

// ------------------------------------------------------- workspace mirrors
// Each mirrors the dispatch above call for call (same split points, same
// eligibility tests); gemm carves only on the fp32 tcgen05 route.
namespace {

template <typename T>
size_t ws_trsm_core(int64_t batch, int64_t nt, int64_t no, bool right) {
  if (nt <= NB) return 0;
  const int64_t n1 = split_point(nt), n2 = nt - n1, big = std::max(n1, n2);
  const size_t g = right ? ws_gemm<T>(batch, no, big, big) : ws_gemm<T>(batch, big, no, big);
  return g + ws_trsm_core<T>(batch, n1, no, right) + ws_trsm_core<T>(batch, n2, no, right);
}

template <typename T>
size_t ws_trmm_core(int64_t batch, int64_t nt, int64_t no, bool right) {
  if (nt <= NB) return 0;
  const int64_t n1 = split_point(nt), n2 = nt - n1, big = std::max(n1, n2);
  const size_t g = right ? ws_gemm<T>(batch, no, big, big) : ws_gemm<T>(batch, big, no, big);
  return g + ws_trmm_core<T>(batch, n1, no, right) + ws_trmm_core<T>(batch, n2, no, right);
}

template <typename T, int NBP>
size_t ws_potrf_blocked_nb(int64_t batch, int64_t n) {
  size_t w = carve_bound(sizeof(int) * (size_t)batch) + carve_bound(potrf_linv_bytes<T, NBP>(batch, n, -1));
  const int64_t steps = (n + NBP - 1) / NBP;
  for (int64_t p = 0; p < steps; ++p) {  // column update, throughput solve, side update
    const int64_t k0 = p * NBP, kb = std::min((int64_t)NBP, n - k0), rest = n - k0 - kb;
    w += ws_gemm<T>(batch, n - k0, kb, std::min<int64_t>(k0, NBP));
    w += ws_gemm<T>(batch, rest, kb, kb);
    const int64_t c0 = (p + 2) * NBP;
    if (c0 < n) w += ws_gemm<T>(batch, n - c0, n - c0, k0 + kb - p * NBP);
  }
  return w;
}

template <typename T>
size_t ws_potrf_blocked(int64_t batch, int64_t n) {
  return potrf_nb() == 128 ? ws_potrf_blocked_nb<T, 128>(batch, n) : ws_potrf_blocked_nb<T, 64>(batch, n);
}

template <typename T>
size_t ws_potrf_rec(int64_t batch, int64_t n) {
  if (n > NB && n <= 512 && batch <= 64) return ws_potrf_blocked<T>(batch, n);
  if (n <= NB) return 0;
  const int64_t n1 = split_point(n), n2 = n - n1;
  size_t w = ws_potrf_rec<T>(batch, n1) + ws_potrf_rec<T>(batch, n2) + ws_gemm<T>(batch, n2, n2, n1);
  if (inv_eligible<T>(n1) && n2 >= 128) w += ws_trsm_inv<T>(batch, n2, n1, true);
  else w += ws_trsm_core<T>(batch, n1, n2, true);
  return w;
}

template <typename T>
size_t ws_trtri_rec(int64_t batch, int64_t n) {
  if (n <= NB) return 0;
  const int64_t n1 = split_point(n), n2 = n - n1;
  return ws_trtri_rec<T>(batch, n1) + ws_trtri_rec<T>(batch, n2) + ws_trmm_core<T>(batch, n1, n2, true) +
         ws_trsm_core<T>(batch, n2, n1, false);
}

template <typename T>
size_t ws_lauum_rec(int64_t batch, int64_t n) {
  if (n <= NB) return 0;
  const int64_t n1 = split_point(n), n2 = n - n1;
  return ws_lauum_rec<T>(batch, n1) + ws_lauum_rec<T>(batch, n2) + ws_gemm<T>(batch, n1, n1, n2) +
         ws_trmm_core<T>(batch, n2, n1, false);
}

}  // namespace

template <typename T>
size_t ws_trsm(int64_t batch, int64_t m, int64_t n, bool right) {
  if (batch == 0 || m == 0 || n == 0) return 0;
  const int64_t nt = right ? n : m, no = right ? m : n;
  if (nt <= NB) return 0;
  if (trsv_eligible<T>(nt, no)) return ws_trsv<T>(batch, m, n, right);
  if (inv_eligible<T>(nt) && no >= 128) return ws_trsm_inv<T>(batch, m, n, right);
  return ws_trsm_core<T>(batch, nt, no, right);
}

template <typename T>
size_t ws_trmm(int64_t batch, int64_t m, int64_t n, bool right) {
  if (batch == 0 || m == 0 || n == 0) return 0;
  const int64_t nt = right ? n : m, no = right ? m : n;
  if (nt >= 128) return ws_trmm_gemm<T>(batch, m, n, right);
  return ws_trmm_core<T>(batch, nt, no, right);
}

template <typename T>
size_t ws_potrf_lower(int64_t batch, int64_t n) {
  if (batch == 0 || n == 0) return 0;
  const int mode = potrf_mode();
  if (sizeof(T) == 8 && mode == 3) return ws_potrf_tiles(batch, n) + ws_potrf_blocked<T>(batch, n);  // either route
  if (mode != 1 && n > NB) return ws_potrf_blocked<T>(batch, n);
  return ws_potrf_rec<T>(batch, n);
}

template <typename T>
size_t ws_potri_lower(int64_t batch, int64_t n) {
  if (batch == 0 || n == 0) return 0;
  if (inv_eligible<T>(n)) return ws_potri_inv<T>(batch, n);
  if (potri_fused_eligible<T>(n)) return 0;  // the fused one-launch potri (inv.cu)
  return ws_trtri_rec<T>(batch, n) + ws_lauum_rec<T>(batch, n);
}

#define INST(T)                                                                                             \
  template size_t ws_trsm<T>(int64_t, int64_t, int64_t, bool);                                              \
  template size_t ws_trmm<T>(int64_t, int64_t, int64_t, bool);                                              \
  template size_t ws_potrf_lower<T>(int64_t, int64_t);                                                      \
  template size_t ws_potri_lower<T>(int64_t, int64_t);                                                      \
  template dla_status trsm<T>(const Ctx&, int64_t, int64_t, int64_t, MatB<const T>, MatB<T>, bool, bool, bool, \
                              T, bool);                                                                     \
  template dla_status trmm<T>(const Ctx&, int64_t, int64_t, int64_t, MatB<const T>, MatB<T>, bool, bool, bool, \
                              T);                                                                           \
  template dla_status potrf_lower<T>(const Ctx&, int64_t, int64_t, MatB<T>, bool, bool*);                                \
  template dla_status potri_lower<T>(const Ctx&, int64_t, int64_t, MatB<T>);
INST(double)
INST(float)

}  // namespace dlab

#ifdef DLAB_PANEL_PROF
extern "C" int dla_panel_prof_read(unsigned long long* host) {
  return cudaMemcpyFromSymbol(host, dlab::g_pprof, sizeof(dlab::g_pprof)) == cudaSuccess ? 0 : 1;
}
extern "C" int dla_chol_prof_read(unsigned long long* host) {
  return cudaMemcpyFromSymbol(host, dlab::g_cprof, sizeof(dlab::g_cprof)) == cudaSuccess ? 0 : 1;
}
#endif
