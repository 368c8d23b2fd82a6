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
// a masked product + a zeroing sweep).  A warp per row (slice and row from one
// division per row, not per element), lanes over column pairs with 16-byte
// stores when rows are 16-byte aligned; the row's k multipliers are loaded once.
template <typename T, int K>
__global__ void __launch_bounds__(256) k_outer_tri(SkinnyArgs<T> g, int64_t batch, bool vec) {
  const int lane = threadIdx.x & 31;
  const int64_t rows = batch * g.m, pairs = (g.n + 1) / 2;
  const int64_t w0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t ws = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t row = w0; row < rows; row += ws) {
    const int64_t b = row / g.m, i = row - b * g.m;
    if (slice_failed(g.skip, b)) continue;
    const T* A = g.a.p + b * g.a.bs;
    const T* B = g.b.p + b * g.b.bs;
    T* Crow = g.c.p + b * g.c.bs + i * g.c.ld;
    T av[K];
#pragma unroll
    for (int k = 0; k < K; ++k) av[k] = k < g.k ? opa(g, A, i, k) : T(0);
    for (int64_t p = lane; p < pairs; p += 32) {
      const int64_t j = 2 * p;
      T v[2];
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        const int64_t jj = j + u;
        const bool in = g.mask == MASK_LOWER ? jj <= i : (g.mask == MASK_UPPER ? jj >= i : true);
        T acc = T(0);
        if (in && jj < g.n) {
#pragma unroll
          for (int k = 0; k < K; ++k)
            if (k < g.k) acc += av[k] * opb(g, B, k, jj);
        }
        v[u] = in ? g.alpha * acc : T(0);
      }
      T* C = Crow + j;
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
}

// ---- single-vector fast paths (n == 1, 16-byte aligned, contiguous vector):
// the GP / marginal-likelihood chains' v = G y, G^T v and v y^T at batch x
// 128 shapes.  Every thread keeps several 16-byte loads or stores in flight
// and walks (slice, row) with incremental counters (no per-element 64-bit
// division): these shapes are HBM streams, not tiles.
//
// y = alpha A x (+ beta y): a warp per 4 rows, lanes over double2 columns.
template <typename T>
__global__ void __launch_bounds__(256) k_matvec_rows(int64_t batch, int64_t m, int64_t k, T alpha, T beta,
                                                     MatB<const T> a, MatB<const T> x, MatB<T> y,
                                                     const int32_t* skip) {
  using V2 = typename std::conditional<sizeof(T) == 8, double2, float2>::type;
  constexpr int R = 4;
  const int lane = threadIdx.x & 31;
  const int64_t groups_per = (m + R - 1) / R, total = batch * groups_per;
  const int64_t w0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t ws = ((int64_t)gridDim.x * blockDim.x) >> 5;
  int64_t b = w0 / groups_per, gi = w0 - b * groups_per;
  const int64_t db = ws / groups_per, dg = ws - db * groups_per;
  for (int64_t t = w0; t < total; t += ws) {
    if (!slice_failed(skip, b)) {
      const T* A = a.p + b * a.bs + gi * R * a.ld;
      const T* X = x.p + b * x.bs;
      T acc[R];
#pragma unroll
      for (int r = 0; r < R; ++r) acc[r] = T(0);
      for (int64_t c = 2 * lane; c < k; c += 64) {
        const V2 xv = *reinterpret_cast<const V2*>(X + c);
        V2 av[R];
#pragma unroll
        for (int r = 0; r < R; ++r)
          if (gi * R + r < m) av[r] = *reinterpret_cast<const V2*>(A + r * a.ld + c);
#pragma unroll
        for (int r = 0; r < R; ++r)
          if (gi * R + r < m) acc[r] += av[r].x * xv.x + av[r].y * xv.y;
      }
#pragma unroll
      for (int r = 0; r < R; ++r) {
#pragma unroll
        for (int o = 16; o; o >>= 1) acc[r] += __shfl_xor_sync(0xffffffffu, acc[r], o);
      }
      if (lane < R && gi * R + lane < m) {
        T v = acc[0];
#pragma unroll
        for (int r = 1; r < R; ++r)
          if (lane == r) v = acc[r];
        T* py = y.p + b * y.bs + (gi * R + lane) * y.ld;
        T o = alpha * v;
        if (beta != T(0)) o += beta * *py;
        *py = o;
      }
    }
    gi += dg;
    b += db;
    if (gi >= groups_per) {
      gi -= groups_per;
      ++b;
    }
  }
}

// y = alpha A^T x (+ beta y), m = columns of A (<= 256 per CTA): a CTA per
// (slice, 256-column block), 64 column-pair lanes x 4 k-groups, shared-memory
// reduction across the k-groups.
template <typename T>
__global__ void __launch_bounds__(256) k_matvec_cols(int64_t batch, int64_t m, int64_t k, T alpha, T beta,
                                                     MatB<const T> a, MatB<const T> x, MatB<T> y,
                                                     const int32_t* skip, int64_t cblocks) {
  using V2 = typename std::conditional<sizeof(T) == 8, double2, float2>::type;
  __shared__ T red[4][2 * 64 * 2];
  const int64_t b = blockIdx.x / cblocks, cb = blockIdx.x % cblocks;
  if (slice_failed(skip, b)) return;
  const int cp = threadIdx.x & 63, kg = threadIdx.x >> 6;
  const T* A = a.p + b * a.bs;
  const T* X = x.p + b * x.bs;
  T acc[2][2] = {{T(0), T(0)}, {T(0), T(0)}};  // two column pairs per lane: cols c0, c0 + 128
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int64_t c0 = cb * 256 + h * 128 + 2 * cp;
    if (c0 < m) {
#pragma unroll 8
      for (int64_t r = kg; r < k; r += 4) {
        const V2 av = *reinterpret_cast<const V2*>(A + r * a.ld + c0);
        const T xv = X[r * x.ld];
        acc[h][0] += av.x * xv;
        acc[h][1] += av.y * xv;
      }
    }
  }
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    red[kg][h * 128 + 2 * cp] = acc[h][0];
    red[kg][h * 128 + 2 * cp + 1] = acc[h][1];
  }
  __syncthreads();
  const int64_t col = cb * 256 + threadIdx.x;
  if (col < m) {
    const T v = ((red[0][threadIdx.x] + red[1][threadIdx.x]) + red[2][threadIdx.x]) + red[3][threadIdx.x];
    T* py = y.p + b * y.bs + col * y.ld;
    T o = alpha * v;
    if (beta != T(0)) o += beta * *py;
    *py = o;
  }
}

// C(i, j) = alpha a_i b_j (+ beta C), rank-1 outer product into a row-major C
// with even columns; mask: entries outside are left untouched.  Thread per
// column pair, rows walked with incremental counters.
template <typename T>
__global__ void __launch_bounds__(256) k_outer1(int64_t batch, int64_t m, int64_t n, T alpha, T beta,
                                                MatB<const T> a, int64_t sa, MatB<const T> bv, int64_t sb,
                                                MatB<T> c, int mask, const int32_t* skip) {
  using V2 = typename std::conditional<sizeof(T) == 8, double2, float2>::type;
  const int64_t pairs = n / 2, rows = batch * m;
  const int64_t ty = blockDim.x / 64 > 0 ? blockDim.x / 64 : 1;
  const int p = threadIdx.x % 64;
  const int64_t r0 = blockIdx.x * ty + threadIdx.x / 64, rs = (int64_t)gridDim.x * ty;
  int64_t b = r0 / m, i = r0 - b * m;
  const int64_t db = rs / m, di = rs - db * m;
  for (int64_t r = r0; r < rows; r += rs) {
    if (!slice_failed(skip, b)) {
      const T ai = a.p[b * a.bs + i * sa];
      const T* B = bv.p + b * bv.bs;
      T* C = c.p + b * c.bs + i * c.ld;
      for (int64_t q = p; q < pairs; q += 64) {
        const int64_t j = 2 * q;
        V2 o;  // alpha (a_i b_j): gemm()'s rounding order
        o.x = alpha * (ai * B[j * sb]);
        o.y = alpha * (ai * B[(j + 1) * sb]);
        const bool in0 = mask == MASK_LOWER ? j <= i : (mask == MASK_UPPER ? j >= i : true);
        const bool in1 = mask == MASK_LOWER ? j + 1 <= i : (mask == MASK_UPPER ? j + 1 >= i : true);
        if (in0 && in1) {
          if (beta != T(0)) {
            const V2 old = *reinterpret_cast<const V2*>(C + j);
            o.x += beta * old.x;
            o.y += beta * old.y;
          }
          *reinterpret_cast<V2*>(C + j) = o;
        } else {
          if (in0) C[j] = beta != T(0) ? o.x + beta * C[j] : o.x;
          if (in1) C[j + 1] = beta != T(0) ? o.y + beta * C[j + 1] : o.y;
        }
      }
    }
    i += di;
    b += db;
    if (i >= m) {
      i -= m;
      ++b;
    }
  }
}

template <typename T>
bool aligned2(const T* p, int64_t ld, int64_t bs) {
  return reinterpret_cast<uintptr_t>(p) % (2 * sizeof(T)) == 0 && ld % 2 == 0 && bs % 2 == 0;
}

}  // namespace

// C (m x n, full) = alpha * mask(op(A) op(B)) with zeros outside the mask, k <= 8.
template <typename T>
bool outer_tri(const Ctx& c, int64_t batch, int64_t m, int64_t n, int64_t k, T alpha, MatB<const T> a, bool ta,
               MatB<const T> b, bool tb, MatB<T> cm, int mask, const int32_t* skip, dla_status* st) {
  if (k > SK_NMAX || k < 1) return false;
  SkinnyArgs<T> g{m, n, k, alpha, T(0), a, b, cm, ta, tb, false, mask, skip};
  const bool vec = (cm.ld % 2 == 0) && (cm.bs % 2 == 0) && (reinterpret_cast<uintptr_t>(cm.p) % (2 * sizeof(T)) == 0);
  const unsigned grid = blocks_for(batch * m * 32, 256, 148 * 16);  // a warp per row
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
  if (k == 1 && n >= 2 && n % 2 == 0 && aligned2<T>(cm.p, cm.ld, cm.bs)) {
    // rank-1 outer product: column of op(A) times row of op(B)
    const int64_t sa = ta ? 1 : a.ld;  // op(A)(i, 0)
    const int64_t sb = tb ? b.ld : 1;  // op(B)(0, j)
    const unsigned grid = blocks_for(batch * m, 4, 148 * 16);
    k_outer1<T><<<grid, 256, 0, c.stream>>>(batch, m, n, alpha, beta, a, sa, b, sb, cm, mask, skip);
  } else if (k <= SK_NMAX) {
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
    // single vector, contiguous, 16-byte aligned rows: the streaming matvecs
    const bool vec1 = g.n == 1 && !g.tc && g.k % 2 == 0 && aligned2<T>(g.a.p, g.a.ld, g.a.bs);
    const bool xcontig = g.tb ? true : g.b.ld == 1;
    if (vec1 && !g.ta && xcontig && reinterpret_cast<uintptr_t>(g.b.p) % (2 * sizeof(T)) == 0 &&
        (batch == 1 || g.b.bs % 2 == 0)) {
      const unsigned grid = blocks_for(batch * ((g.m + 3) / 4), 8, 148 * 8);
      MatB<const T> xv{g.b.p, 1, g.b.bs};
      k_matvec_rows<T><<<grid, 256, 0, c.stream>>>(batch, g.m, g.k, g.alpha, g.beta, g.a, xv, g.c, skip);
    } else if (vec1 && g.ta && g.m % 2 == 0) {
      const int64_t cbk = (g.m + 255) / 256;
      MatB<const T> xv{g.b.p, g.tb ? 1 : g.b.ld, g.b.bs};
      k_matvec_cols<T><<<(unsigned)(batch * cbk), 256, 0, c.stream>>>(batch, g.m, g.k, g.alpha, g.beta, g.a, xv,
                                                                        g.c, skip, cbk);
    } else if (!g.ta) {
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
