// Skinny batched GEMMs: matrix-vector and outer-product shapes.
//
// The reference's GP / marginal-likelihood chains apply gemm2 to n x 1
// vectors (v = G y, the quadratic form v^T v, and their pullbacks
// cbar y^T / G^T cbar, dl/adjoints.hpp:36-49).  On a 128 x 128 DMMA tile
// these waste 127/128 of the tensor-core work and still pay the tile
// pipeline; they are HBM-bound by nature (every A element is used once), so
// they run here as streaming kernels that read each operand once, coalesced:
//
//   N-skinny (n <= 8, k >= 16): P = op(A) op(B) with few columns.
//     !TA: one warp per output row, lanes stride the contiguous k of A's row,
//          warp-shuffle reduction;
//     TA : one thread per output row (= column of A), rows of A are swept in
//          k order, so a warp reads 32 consecutive elements per step.
//   M-skinny (m <= 8) is the N-skinny kernel on the transposed problem
//   (C^T = op(B)^T op(A)^T, written through a transposed store).
//   K-skinny (k <= 8): rank-k outer products, one thread per output
//   element along the contiguous dimension of C (write-bound).
//
// Semantics are gemm()'s: C = alpha P + beta C (beta == 0 => C not read),
// optional lower/upper write mask for the K-skinny case.
#include "common.cuh"

namespace dlab {
namespace {

constexpr int SK_NMAX = 8;

template <typename T>
struct SkinnyArgs {
  int64_t m, n, k;  // product P is m x n
  T alpha, beta;
  MatB<const T> a, b;
  MatB<T> c;
  bool ta, tb, tc;  // tc: C holds P^T (element (i, j) of P at c(j, i))
  int mask;
  const int32_t* skip;
};

template <typename T>
__device__ __forceinline__ T opa(const SkinnyArgs<T>& g, const T* A, int64_t i, int64_t k) {
  return g.ta ? A[k * g.a.ld + i] : A[i * g.a.ld + k];
}
template <typename T>
__device__ __forceinline__ T opb(const SkinnyArgs<T>& g, const T* B, int64_t k, int64_t j) {
  return g.tb ? B[j * g.b.ld + k] : B[k * g.b.ld + j];
}
template <typename T>
__device__ __forceinline__ void put(const SkinnyArgs<T>& g, T* C, int64_t i, int64_t j, T v) {
  T* p = g.tc ? C + j * g.c.ld + i : C + i * g.c.ld + j;
  T r = g.alpha * v;
  if (g.beta != T(0)) r += g.beta * *p;
  *p = r;
}

// !TA: warp per output row.  grid.x = batch * ceil(m / 8), 8 warps per CTA.
template <typename T>
__global__ void __launch_bounds__(256) k_nskinny_rows(SkinnyArgs<T> g, int64_t row_blocks) {
  const int64_t b = blockIdx.x / row_blocks, rb = blockIdx.x % row_blocks;
  if (slice_failed(g.skip, b)) return;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t i = rb * 8 + warp;
  if (i >= g.m) return;
  const T* A = g.a.p + b * g.a.bs;
  const T* B = g.b.p + b * g.b.bs;
  const T* arow = A + i * g.a.ld;
  T acc[SK_NMAX];
#pragma unroll
  for (int j = 0; j < SK_NMAX; ++j) acc[j] = T(0);
#pragma unroll 4
  for (int64_t k = lane; k < g.k; k += 32) {
    const T av = arow[k];
#pragma unroll
    for (int j = 0; j < SK_NMAX; ++j)
      if (j < g.n) acc[j] += av * opb(g, B, k, j);
  }
#pragma unroll
  for (int j = 0; j < SK_NMAX; ++j) {
    if (j < g.n) {  // warp-uniform
      T v = acc[j];
#pragma unroll
      for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
      if (lane == 0) put(g, g.c.p + b * g.c.bs, i, j, v);
    }
  }
}

// TA: thread per output row.  grid.x = batch * ceil(m / 128), 128 threads.
template <typename T>
__global__ void __launch_bounds__(128) k_nskinny_cols(SkinnyArgs<T> g, int64_t row_blocks) {
  const int64_t b = blockIdx.x / row_blocks, rb = blockIdx.x % row_blocks;
  if (slice_failed(g.skip, b)) return;
  const int64_t i = rb * 128 + threadIdx.x;
  const T* A = g.a.p + b * g.a.bs;
  const T* B = g.b.p + b * g.b.bs;
  T acc[SK_NMAX];
#pragma unroll
  for (int j = 0; j < SK_NMAX; ++j) acc[j] = T(0);
  if (i < g.m) {
    const T* acol = A + i;
#pragma unroll 4
    for (int64_t k = 0; k < g.k; ++k) {
      const T av = acol[k * g.a.ld];
#pragma unroll
      for (int j = 0; j < SK_NMAX; ++j)
        if (j < g.n) acc[j] += av * opb(g, B, k, j);
    }
#pragma unroll
    for (int j = 0; j < SK_NMAX; ++j)
      if (j < g.n) put(g, g.c.p + b * g.c.bs, i, j, acc[j]);
  }
}

// TA with a tiny product (m * n <= 16, e.g. the quadratic form v^T v): one
// CTA per slice splits k over its 256 threads (rows of A are contiguous),
// then a warp-shuffle + shared-memory reduction.
constexpr int KS_MN = 16;
template <typename T>
__global__ void __launch_bounds__(256) k_nskinny_ksplit(SkinnyArgs<T> g) {
  __shared__ T red[8][KS_MN];
  const int64_t b = blockIdx.x;
  if (slice_failed(g.skip, b)) return;
  const T* A = g.a.p + b * g.a.bs;
  const T* B = g.b.p + b * g.b.bs;
  const int mn = (int)(g.m * g.n);
  T acc[KS_MN];
#pragma unroll
  for (int e = 0; e < KS_MN; ++e) acc[e] = T(0);
  for (int64_t k = threadIdx.x; k < g.k; k += 256) {
#pragma unroll
    for (int e = 0; e < KS_MN; ++e)
      if (e < mn) {
        const int64_t i = e / g.n, j = e % g.n;
        acc[e] += A[k * g.a.ld + i] * opb(g, B, k, j);
      }
  }
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
#pragma unroll
  for (int e = 0; e < KS_MN; ++e) {
    if (e < mn) {
      T v = acc[e];
#pragma unroll
      for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
      if (lane == 0) red[warp][e] = v;
    }
  }
  __syncthreads();
  if (threadIdx.x < mn) {
    T v = T(0);
#pragma unroll
    for (int w = 0; w < 8; ++w) v += red[w][threadIdx.x];
    put(g, g.c.p + b * g.c.bs, threadIdx.x / g.n, threadIdx.x % g.n, v);
  }
}

// K-skinny: one CTA row-sweep per row of C's storage (grid-stride over
// batch x rows), threads along the contiguous columns: no per-element 64-bit
// index division, coalesced stores.
template <typename T>
__global__ void __launch_bounds__(128) k_kskinny(SkinnyArgs<T> g, int64_t batch) {
  const int64_t rows = g.tc ? g.n : g.m, cols = g.tc ? g.m : g.n;
  const int64_t total = batch * rows;
  for (int64_t t = blockIdx.x; t < total; t += gridDim.x) {
    const int64_t b = t / rows, r = t - b * rows;
    if (slice_failed(g.skip, b)) continue;
    const T* A = g.a.p + b * g.a.bs;
    const T* B = g.b.p + b * g.b.bs;
    T* C = g.c.p + b * g.c.bs;
    for (int64_t s = threadIdx.x; s < cols; s += blockDim.x) {
      const int64_t i = g.tc ? s : r, j = g.tc ? r : s;
      if (g.mask == MASK_LOWER && j > i) continue;
      if (g.mask == MASK_UPPER && j < i) continue;
      T acc = T(0);
      for (int64_t k = 0; k < g.k; ++k) acc += opa(g, A, i, k) * opb(g, B, k, j);
      put(g, C, i, j, acc);
    }
  }
}

// Full-square rank-k outer product with a triangle mask and beta == 0:
// C = alpha P inside the mask, exact zeros outside (trsm pullback's
// Tbar = -mask(S B^T), dl/adjoints.hpp:138-151, written in ONE pass instead of
// a masked product + a zeroing sweep).  Thread per pair of columns, 16-byte
// stores when rows are 16-byte aligned.
template <typename T, int K>
__global__ void __launch_bounds__(256) k_outer_tri(SkinnyArgs<T> g, int64_t batch, bool vec) {
  const int64_t pairs = (g.n + 1) / 2, per = g.m * pairs;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < batch * per; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t b = t / per, r = t - b * per;
    const int64_t i = r / pairs, j = 2 * (r - i * pairs);
    if (slice_failed(g.skip, b)) continue;
    const T* A = g.a.p + b * g.a.bs;
    const T* B = g.b.p + b * g.b.bs;
    T* C = g.c.p + b * g.c.bs + i * g.c.ld + j;
    T v[2];
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const int64_t jj = j + u;
      const bool in = g.mask == MASK_LOWER ? jj <= i : (g.mask == MASK_UPPER ? jj >= i : true);
      T acc = T(0);
      if (in && jj < g.n) {
#pragma unroll
        for (int k = 0; k < K; ++k)
          if (k < g.k) acc += opa(g, A, i, k) * opb(g, B, k, jj);
      }
      v[u] = in ? g.alpha * acc : T(0);
    }
    if (vec && j + 1 < g.n) {
      if constexpr (sizeof(T) == 8)
        *reinterpret_cast<double2*>(C) = make_double2(v[0], v[1]);
      else
        *reinterpret_cast<float2*>(C) = make_float2(v[0], v[1]);
    } else {
      C[0] = v[0];
      if (j + 1 < g.n) C[1] = v[1];
    }
  }
}

}  // namespace

// C (m x n, full) = alpha * mask(op(A) op(B)) with zeros outside the mask, k <= 8.
template <typename T>
bool outer_tri(const Ctx& c, int64_t batch, int64_t m, int64_t n, int64_t k, T alpha, MatB<const T> a, bool ta,
               MatB<const T> b, bool tb, MatB<T> cm, int mask, const int32_t* skip, dla_status* st) {
  if (k > SK_NMAX || k < 1) return false;
  SkinnyArgs<T> g{m, n, k, alpha, T(0), a, b, cm, ta, tb, false, mask, skip};
  const bool vec = (cm.ld % 2 == 0) && (cm.bs % 2 == 0) && (reinterpret_cast<uintptr_t>(cm.p) % (2 * sizeof(T)) == 0);
  const unsigned grid = blocks_for(batch * m * ((n + 1) / 2), 256, 148 * 16);
  if (k == 1)
    k_outer_tri<T, 1><<<grid, 256, 0, c.stream>>>(g, batch, vec);
  else
    k_outer_tri<T, SK_NMAX><<<grid, 256, 0, c.stream>>>(g, batch, vec);
  *st = cudaGetLastError() == cudaSuccess ? DLA_OK : DLA_ERR_CUDA;
  note_launch(1);
  return true;
}
template bool outer_tri<double>(const Ctx&, int64_t, int64_t, int64_t, int64_t, double, MatB<const double>, bool,
                                MatB<const double>, bool, MatB<double>, int, const int32_t*, dla_status*);
template bool outer_tri<float>(const Ctx&, int64_t, int64_t, int64_t, int64_t, float, MatB<const float>, bool,
                               MatB<const float>, bool, MatB<float>, int, const int32_t*, dla_status*);

// Returns true (and launches) when the shape is skinny; false leaves the
// problem to the tiled DMMA / FFMA GEMM.
template <typename T>
bool gemm_skinny(const Ctx& c, int64_t batch, int64_t m, int64_t n, int64_t k, T alpha, MatB<const T> a, bool ta,
                 MatB<const T> b, bool tb, T beta, MatB<T> cm, int mask, const int32_t* skip, dla_status* st) {
  SkinnyArgs<T> g{m, n, k, alpha, beta, a, b, cm, ta, tb, false, mask, skip};
  *st = DLA_OK;
  if (k <= SK_NMAX) {
    k_kskinny<T><<<blocks_for(batch * m, 1, 148 * 64), 128, 0, c.stream>>>(g, batch);
  } else if (mask != MASK_FULL) {
    return false;
  } else if (n <= SK_NMAX || m <= SK_NMAX) {
    if (n > SK_NMAX) {  // C^T = op(B)^T op(A)^T
      g.m = n;
      g.n = m;
      g.a = b;
      g.ta = !tb;
      g.b = a;
      g.tb = !ta;
      g.tc = true;
    }
    if (!g.ta) {
      const int64_t rb = (g.m + 7) / 8;
      k_nskinny_rows<T><<<(unsigned)(batch * rb), 256, 0, c.stream>>>(g, rb);
    } else if (g.m >= 64) {
      const int64_t rb = (g.m + 127) / 128;
      k_nskinny_cols<T><<<(unsigned)(batch * rb), 128, 0, c.stream>>>(g, rb);
    } else if (g.m * g.n <= KS_MN) {
      k_nskinny_ksplit<T><<<(unsigned)batch, 256, 0, c.stream>>>(g);
    } else {
      return false;  // transposed, mid-sized: the tiled GEMM
    }
  } else {
    return false;
  }
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    fprintf(stderr, "dla_b200 skinny gemm: %s\n", cudaGetErrorString(e));
    *st = DLA_ERR_CUDA;
    return true;
  }
  note_launch(1);
  return true;
}

template bool gemm_skinny<double>(const Ctx&, int64_t, int64_t, int64_t, int64_t, double, MatB<const double>, bool,
                                  MatB<const double>, bool, double, MatB<double>, int, const int32_t*, dla_status*);
template bool gemm_skinny<float>(const Ctx&, int64_t, int64_t, int64_t, int64_t, float, MatB<const float>, bool,
                                 MatB<const float>, bool, float, MatB<float>, int, const int32_t*, dla_status*);

}  // namespace dlab
