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
#include "common.cuh"

namespace dlab {
namespace {

constexpr int NB = 64;        // leaf size
constexpr int LEAF_VEC = 32;  // vectors per CTA in trsm/trmm leaves
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

// Leaf trsm: solve S y = x for LEAF_VEC vectors per CTA (in place in X).
//   left : X block is nb x nvec (rows k0.., vectors = columns)
//   right: X block is nvec x nb (vectors = rows)
template <typename T>
__global__ void __launch_bounds__(256) k_trsm_leaf(int nb, int64_t nvec, MatB<const T> t, MatB<T> x, bool right,
                                                   bool s_from_tt, bool slower, const int32_t* skip) {
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
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  for (int v = warp; v < nv; v += nw) {
    T* xv = V + v * LDS;
    T r0 = lane < nb ? xv[lane] : T(0);
    T r1 = lane + 32 < nb ? xv[lane + 32] : T(0);
    for (int s = 0; s < nb; ++s) {
      const int i = slower ? s : nb - 1 - s;
      const int owner = i & 31;
      T xi = (i < 32) ? r0 : r1;
      xi = __shfl_sync(0xffffffffu, xi, owner) / S[i * LDS + i];
      if (lane == owner) {
        if (i < 32) r0 = xi; else r1 = xi;
      }
      // update the rows still to be solved
      if (slower) {
        if (lane > i && lane < nb) r0 -= S[lane * LDS + i] * xi;
        if (lane + 32 > i && lane + 32 < nb) r1 -= S[(lane + 32) * LDS + i] * xi;
      } else {
        if (lane < i) r0 -= S[lane * LDS + i] * xi;
        if (lane + 32 < i) r1 -= S[(lane + 32) * LDS + i] * xi;
      }
    }
    if (lane < nb) xv[lane] = r0;
    if (lane + 32 < nb) xv[lane + 32] = r1;
  }
  __syncthreads();
  for (int e = threadIdx.x; e < nv * nb; e += blockDim.x) {
    int v, i;
    if (right) { v = e / nb; i = e % nb; } else { i = e / nv; v = e % nv; }
    T* dst = right ? x.at(b, v0 + v, i) : x.at(b, i, v0 + v);
    *dst = V[v * LDS + i];
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
  const int64_t b = blockIdx.x;
  if (slice_failed(info, b)) return;
  for (int e = threadIdx.x; e < nb * nb; e += blockDim.x) {
    const int i = e / nb, j = e % nb;
    if (j <= i) S[i * LDS + j] = *a.at(b, i, j);
  }
  __syncthreads();
  int failed = -1;
  for (int j = 0; j < nb; ++j) {
    const T d = S[j * LDS + j];
    if (!(d > T(0))) {
      failed = j;
      break;
    }
    const T r = Num<T>::sqrt_(d);
    const T inv = T(1) / r;
    __syncthreads();  // everyone has read d
    if (threadIdx.x == 0) S[j * LDS + j] = r;
    for (int i = j + 1 + threadIdx.x; i < nb; i += blockDim.x) S[i * LDS + j] *= inv;
    __syncthreads();
    // trailing update of the lower triangle
    const int m = nb - j - 1;
    for (int e = threadIdx.x; e < m * m; e += blockDim.x) {
      const int ii = j + 1 + e / m, jj = j + 1 + e % m;
      if (jj <= ii) S[ii * LDS + jj] -= S[ii * LDS + j] * S[jj * LDS + j];
    }
    __syncthreads();
  }
  if (failed >= 0) {
    if (threadIdx.x == 0) record_failure(info, b, DLA_ERR_NOT_SPD, k0 + failed);
    return;
  }
  for (int e = threadIdx.x; e < nb * nb; e += blockDim.x) {
    const int i = e / nb, j = e % nb;
    *a.at(b, i, j) = j <= i ? S[i * LDS + j] : T(0);
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

template <typename K>
void set_smem(K kernel, size_t bytes) {
  cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
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
                     bool right, bool trans, bool lower) {
  const bool op_lower = (lower != trans);
  if (nt <= NB) {
    // left: S = op(T); right: S = op(T)^T.  S(i,j) = T(j,i) when
    // (left && trans) || (right && !trans).
    const bool s_tt = right ? !trans : trans;
    const bool slower = right ? !op_lower : op_lower;
    const int64_t chunks = (nother + LEAF_VEC - 1) / LEAF_VEC;
    const size_t sm = leaf_smem<T>(LEAF_VEC);
    static bool once = false;
    if (!once) {
      set_smem(k_trsm_leaf<T>, sm);
      once = true;
    }
    k_trsm_leaf<T><<<(unsigned)(batch * chunks), 256, sm, c.stream>>>((int)nt, nother, t, x, right, s_tt, slower,
                                                                       c.info);
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
    static bool once = false;
    if (!once) {
      set_smem(k_trmm_leaf<T>, sm);
      once = true;
    }
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
dla_status potrf_rec(const Ctx& c, int64_t batch, int64_t n, int64_t k0, MatB<T> a) {
  if (n <= NB) {
    const size_t sm = sizeof(T) * NB * LDS;
    k_potrf_leaf<T><<<(unsigned)batch, 256, sm, c.stream>>>((int)n, k0, a, c.info);
    DLAB_LAUNCH_CHECK();
    return DLA_OK;
  }
  const int64_t n1 = split_point(n), n2 = n - n1;
  DLAB_TRY(potrf_rec<T>(c, batch, n1, k0, a));
  MatB<T> a21 = a.sub(n1, 0), a22 = a.sub(n1, n1);
  // A21 <- A21 L11^{-T}
  DLAB_TRY(trsm_core<T>(c, batch, n1, n2, C_(a), a21, true, true, true));
  // A22 -= A21 A21^T (lower triangle only)
  DLAB_TRY(gemm<T>(c, batch, n2, n2, n1, T(-1), C_(a21), false, C_(a21), true, T(1), a22, MASK_LOWER, c.info));
  return potrf_rec<T>(c, batch, n2, k0 + n1, a22);
}

template <typename T>
dla_status trtri_rec(const Ctx& c, int64_t batch, int64_t n, MatB<T> a) {
  if (n <= NB) {
    const size_t sm = sizeof(T) * 2 * NB * LDS;
    static bool once = false;
    if (!once) {
      set_smem(k_trtri_leaf<T>, sm);
      once = true;
    }
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
                bool trans, bool lower, T alpha) {
  if (batch == 0 || m == 0 || n == 0) return DLA_OK;
  DLAB_TRY(ew_scale<T>(c, batch, m, n, x, alpha, c.info));
  return right ? trsm_core<T>(c, batch, n, m, t, x, right, trans, lower)
               : trsm_core<T>(c, batch, m, n, t, x, right, trans, lower);
}

template <typename T>
dla_status trmm(const Ctx& c, int64_t batch, int64_t m, int64_t n, MatB<const T> t, MatB<T> x, bool right,
                bool trans, bool lower, T alpha) {
  if (batch == 0 || m == 0 || n == 0) return DLA_OK;
  return right ? trmm_core<T>(c, batch, n, m, t, x, right, trans, lower, alpha)
               : trmm_core<T>(c, batch, m, n, t, x, right, trans, lower, alpha);
}

template <typename T>
dla_status potrf_lower(const Ctx& c, int64_t batch, int64_t n, MatB<T> a) {
  if (batch == 0 || n == 0) return DLA_OK;
  static bool once = false;
  if (!once) {
    set_smem(k_potrf_leaf<T>, sizeof(T) * NB * LDS);
    set_smem(k_lauum_leaf<T>, sizeof(T) * NB * LDS);
    once = true;
  }
  DLAB_TRY(potrf_rec<T>(c, batch, n, 0, a));
  return ew_square<T>(c, batch, n, a, /*tril*/ 0, T(1), c.info);
}

template <typename T>
dla_status potri_lower(const Ctx& c, int64_t batch, int64_t n, MatB<T> a) {
  if (batch == 0 || n == 0) return DLA_OK;
  static bool once = false;
  if (!once) {
    set_smem(k_potrf_leaf<T>, sizeof(T) * NB * LDS);
    set_smem(k_lauum_leaf<T>, sizeof(T) * NB * LDS);
    once = true;
  }
  DLAB_TRY(trtri_rec<T>(c, batch, n, a));
  DLAB_TRY(lauum_rec<T>(c, batch, n, a));
  return ew_square<T>(c, batch, n, a, /*copyltu*/ 2, T(1), c.info);
}

#define INST(T)                                                                                             \
  template dla_status trsm<T>(const Ctx&, int64_t, int64_t, int64_t, MatB<const T>, MatB<T>, bool, bool, bool, \
                              T);                                                                           \
  template dla_status trmm<T>(const Ctx&, int64_t, int64_t, int64_t, MatB<const T>, MatB<T>, bool, bool, bool, \
                              T);                                                                           \
  template dla_status potrf_lower<T>(const Ctx&, int64_t, int64_t, MatB<T>);                                \
  template dla_status potri_lower<T>(const Ctx&, int64_t, int64_t, MatB<T>);
INST(double)
INST(float)

}  // namespace dlab
