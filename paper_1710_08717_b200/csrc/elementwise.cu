// Structural / elementwise kernels: the reference's dl/transforms.hpp helpers
// (tril/triu/copyltu/copyutl/sym/scale, :18-130), the symmetry precheck
// (dl/cholesky.hpp:19-25), the zero-diagonal precheck (dl/blas.hpp:310-314,
// dl/cholesky.hpp:108-110) and the sumlogdiag op (tape chain
// ExtractDiag -> Log -> Sum, dl/tape.hpp:789-795, :714, :747-755, pullbacks
// :1038-1045, :969-975, :1080-1086).  All HBM-bound; grid-stride loops over
// (batch x elements) sized to the SM count.
#include <type_traits>

#include "common.cuh"

namespace dlab {
namespace {

template <typename T>
__global__ void k_copy(int64_t batch, int64_t m, int64_t n, MatB<const T> src, MatB<T> dst, const int32_t* skip) {
  const int64_t total = batch * m * n;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t b = t / (m * n), r = t % (m * n), i = r / n, j = r % n;
    if (slice_failed(skip, b)) continue;
    *dst.at(b, i, j) = *src.at(b, i, j);
  }
}

// Packed (contiguous) copy: 16-byte vectors when both ends are aligned, no
// per-element index arithmetic (the generic k_copy's four 64-bit div/mods per
// element made it ALU-bound).
template <typename T>
__global__ void k_copy_flat(int64_t count, const T* __restrict__ src, T* __restrict__ dst, bool vec) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x, t0 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (vec) {
    constexpr int V = 16 / sizeof(T);
    using V4 = typename std::conditional<sizeof(T) == 8, double2, float4>::type;
    const int64_t nv = count / V;
    for (int64_t t = t0; t < nv; t += stride)
      reinterpret_cast<V4*>(dst)[t] = reinterpret_cast<const V4*>(src)[t];
    for (int64_t t = nv * V + t0; t < count; t += stride) dst[t] = src[t];
  } else {
    for (int64_t t = t0; t < count; t += stride) dst[t] = src[t];
  }
}

// packed per-slice copy honouring the skip array (grid.y = slice)
template <typename T>
__global__ void k_copy_slices(int64_t per, const T* __restrict__ src, T* __restrict__ dst, const int32_t* skip,
                              bool vec) {
  const int64_t b = blockIdx.y;
  if (slice_failed(skip, b)) return;
  const T* s = src + b * per;
  T* d = dst + b * per;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x, t0 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (vec) {
    using V4 = typename std::conditional<sizeof(T) == 8, double2, float4>::type;
    const int64_t nv = per / (16 / sizeof(T));
    for (int64_t t = t0; t < nv; t += stride) reinterpret_cast<V4*>(d)[t] = reinterpret_cast<const V4*>(s)[t];
  } else {
    for (int64_t t = t0; t < per; t += stride) d[t] = s[t];
  }
}

template <typename T>
__global__ void k_scale(int64_t batch, int64_t m, int64_t n, MatB<T> x, T alpha, const int32_t* skip) {
  const int64_t total = batch * m * n;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t b = t / (m * n), r = t % (m * n), i = r / n, j = r % n;
    if (slice_failed(skip, b)) continue;
    *x.at(b, i, j) *= alpha;
  }
}

// Square structural ops over (b, i, j).
// Row-mapped square kernels: blockIdx.y walks the batch * n rows, blockIdx.x
// and the threads the columns -- one division per row instead of four 64-bit
// div/mods per element (which made these HBM-trivial kernels ALU-bound).
#define DLAB_ROWS_BEGIN(batch, n)                                                   \
  for (int64_t row_ = blockIdx.y; row_ < (batch) * (n); row_ += gridDim.y) {       \
    const int64_t b = row_ / (n), i = row_ - b * (n);                               \
    for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < (n); j += (int64_t)gridDim.x * blockDim.x) {
#define DLAB_ROWS_END \
  }                   \
  }

inline dim3 row_grid(int64_t batch, int64_t n) {
  // ~32 CTAs per SM in total (the rows loop covers the rest): one CTA per
  // row-segment would be CTA-launch bound
  const int64_t rows = batch * n, gx = (n + 255) / 256;
  int64_t gy = std::max<int64_t>(1, (148 * 32) / gx);
  gy = std::min<int64_t>(std::min<int64_t>(gy, std::max<int64_t>(rows, 1)), 65535);
  return dim3((unsigned)gx, (unsigned)gy);
}

template <typename T>
__global__ void k_square(int64_t batch, int64_t n, MatB<T> x, int op, T alpha, const int32_t* skip) {
  DLAB_ROWS_BEGIN(batch, n)
    if (slice_failed(skip, b)) continue;
    T* xij = x.at(b, i, j);
    switch (op) {
      case 0:  // tril: zero strict upper
        if (j > i) *xij = T(0);
        break;
      case 1:  // triu: zero strict lower
        if (j < i) *xij = T(0);
        break;
      case 2:  // copyltu: x(i,j) = x(j,i) for j > i
        if (j > i) *xij = *x.at(b, j, i);
        break;
      case 3:  // copyutl: x(i,j) = x(j,i) for j < i
        if (j < i) *xij = *x.at(b, j, i);
        break;
      case 4:    // sym: (x + x^T) / 2, exactly idempotent (dl/transforms.hpp:78-87)
      case 6: {  // scaled sym: x <- alpha x, then sym
        if (j < i) {
          T* xji = x.at(b, j, i);
          T u = *xij, v = *xji;
          if (op == 6) {
            u *= alpha;
            v *= alpha;
          }
          const T s = (v + u) / T(2);  // (x(i',j') + x(j',i'))/2 with i' < j' as the reference
          *xij = s;
          *xji = s;
        } else if (j == i && op == 6) {
          *xij *= alpha;
        }
        break;
      }
      case 5:  // in-place transpose
        if (j < i) {
          T* xji = x.at(b, j, i);
          T u = *xij;
          *xij = *xji;
          *xji = u;
        }
        break;
    }
  DLAB_ROWS_END
}

// tril(src) -> dst (full square, zeros above), row-mapped, two columns per
// thread with 16-byte loads / stores.
template <typename T>
__global__ void k_tri_copy_vec(int64_t batch, int64_t n, MatB<const T> src, MatB<T> dst) {
  // block (tx, ty): ty rows at a time, tx lanes over a row's column pairs
  // (a 128-wide row is 64 pairs: four rows per 256-thread block, no idle lanes)
  using V2 = typename std::conditional<sizeof(T) == 8, double2, float2>::type;
  const int64_t pairs = (n + 1) / 2;
  const int64_t r0 = blockIdx.y * (int64_t)blockDim.y + threadIdx.y, rs = (int64_t)gridDim.y * blockDim.y;
  const int64_t db = rs / n, di = rs - db * n;  // (slice, row) advance incrementally: no division per row
  int64_t b = r0 / n, i = r0 - b * n;
  for (int64_t row = r0; row < batch * n; row += rs, b += db, i += di) {
    if (i >= n) {
      i -= n;
      ++b;
    }
    const T* sr = src.at(b, i, 0);
    T* dr = dst.at(b, i, 0);
    for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < pairs; p += (int64_t)gridDim.x * blockDim.x) {
      const int64_t j = 2 * p;
      if (j + 1 < n) {
        V2 v;
        if (j + 1 <= i) {
          v = *reinterpret_cast<const V2*>(sr + j);
        } else {
          v.x = j <= i ? sr[j] : T(0);
          v.y = T(0);
        }
        *reinterpret_cast<V2*>(dr + j) = v;
      } else {
        dr[j] = j <= i ? sr[j] : T(0);
      }
    }
  }
}

template <typename T>
__global__ void k_tri_copy(int64_t batch, int64_t n, MatB<const T> src, MatB<T> dst, bool from_upper) {
  DLAB_ROWS_BEGIN(batch, n)
    T v = T(0);
    if (j <= i) v = from_upper ? *src.at(b, j, i) : *src.at(b, i, j);
    *dst.at(b, i, j) = v;
  DLAB_ROWS_END
}

// Lower-triangle tile pair p -> (I, J), I >= J (p = I (I + 1) / 2 + J).
__device__ __forceinline__ void tile_pair(int64_t p, int64_t& I, int64_t& J) {
  I = (int64_t)((sqrt(8.0 * (double)p + 1.0) - 1.0) * 0.5);
  while (I * (I + 1) / 2 > p) --I;
  while ((I + 1) * (I + 2) / 2 <= p) ++I;
  J = p - I * (I + 1) / 2;
}

// dst = alpha (src + src^T) by 32 x 32 tile PAIRS: the block of tile (I, J),
// I >= J, reads tiles (I, J) and (J, I) with coalesced rows, writes both
// (in-place safe: no other block touches them).  IEEE addition commutes, so
// the two mirrored sums are the same bits: bit-symmetric output.  grid.x
// enumerates only the T (T + 1) / 2 lower pairs; grid.y strides the batch.
template <typename T>
__global__ void __launch_bounds__(256) k_add_transpose(int64_t batch, int64_t n, MatB<const T> src, MatB<T> dst,
                                                       T alpha) {
  __shared__ T ta[32][33], tb[32][33];
  int64_t I, J;
  tile_pair(blockIdx.x, I, J);
  const int tx = threadIdx.x, ty = threadIdx.y;
  for (int64_t b = blockIdx.y; b < batch; b += gridDim.y) {
#pragma unroll
    for (int r = ty; r < 32; r += 8) {
      const int64_t i = I * 32 + r, j = J * 32 + tx, i2 = J * 32 + r, j2 = I * 32 + tx;
      ta[r][tx] = (i < n && j < n) ? *src.at(b, i, j) : T(0);
      tb[r][tx] = (i2 < n && j2 < n) ? *src.at(b, i2, j2) : T(0);
    }
    __syncthreads();
#pragma unroll
    for (int r = ty; r < 32; r += 8) {
      const int64_t i = I * 32 + r, j = J * 32 + tx, i2 = J * 32 + r, j2 = I * 32 + tx;
      if (i < n && j < n) *dst.at(b, i, j) = alpha * (ta[r][tx] + tb[tx][r]);
      if (I != J && i2 < n && j2 < n) *dst.at(b, i2, j2) = alpha * (tb[r][tx] + ta[tx][r]);
    }
    __syncthreads();
  }
}

// dst(i, j) = dst(j, i) = alpha src(max(i, j), min(i, j)): tile pairs again,
// only the lower tiles of src are read.
template <typename T>
__global__ void __launch_bounds__(256) k_sym_lower_tiles(int64_t batch, int64_t n, MatB<const T> src, MatB<T> dst,
                                                         T alpha) {
  __shared__ T ta[32][33];
  int64_t I, J;
  tile_pair(blockIdx.x, I, J);
  const int tx = threadIdx.x, ty = threadIdx.y;
  for (int64_t b = blockIdx.y; b < batch; b += gridDim.y) {
#pragma unroll
    for (int r = ty; r < 32; r += 8) {
      const int64_t i = I * 32 + r, j = J * 32 + tx;
      ta[r][tx] = (i < n && j < n && (I != J || tx <= r)) ? *src.at(b, i, j) : T(0);
    }
    __syncthreads();
#pragma unroll
    for (int r = ty; r < 32; r += 8) {
      const int64_t i = I * 32 + r, j = J * 32 + tx, i2 = J * 32 + r, j2 = I * 32 + tx;
      if (I != J) {
        if (i < n && j < n) *dst.at(b, i, j) = alpha * ta[r][tx];
        if (i2 < n && j2 < n) *dst.at(b, i2, j2) = alpha * ta[tx][r];
      } else if (i < n && j < n) {
        *dst.at(b, i, j) = alpha * (tx <= r ? ta[r][tx] : ta[tx][r]);
      }
    }
    __syncthreads();
  }
}

inline dim3 pair_grid(int64_t batch, int64_t n) {
  const int64_t t = (n + 31) / 32, pairs = t * (t + 1) / 2;
  const int64_t gy = std::min<int64_t>(std::max<int64_t>(1, batch), std::max<int64_t>(1, (148 * 8) / pairs));
  return dim3((unsigned)pairs, (unsigned)std::min<int64_t>(gy, 65535));
}

template <typename T>
__global__ void k_scale_diag(int64_t batch, int64_t n, MatB<T> x, T alpha) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < batch * n; t += (int64_t)gridDim.x * blockDim.x)
    *x.at(t / n, t % n, t % n) *= alpha;
}

// Symmetry precheck, pass 1: per-slice max|a| and max|a_ij - a_ji| as
// monotone bit patterns (non-negative IEEE values order as unsigned).
template <typename T>
__device__ __forceinline__ unsigned long long ord_bits(T v) {
  if (!(v == v)) return 0ull;  // NaN ignored, like std::max in max_abs
  if constexpr (sizeof(T) == 8) return (unsigned long long)__double_as_longlong((double)v);
  else return (unsigned long long)__float_as_uint((float)v);
}
template <typename T>
__device__ __forceinline__ T from_bits(unsigned long long u) {
  if constexpr (sizeof(T) == 8) return __longlong_as_double((long long)u);
  else return __uint_as_float((unsigned)u);
}

template <typename T>
__global__ void __launch_bounds__(256) k_symcheck_reduce(int64_t batch, int64_t n, MatB<const T> a,
                                                         unsigned long long* red) {
  // one CTA per (slice, 32 x 32 tile pair (ti, tj), ti >= tj): both tiles are
  // read with coalesced row sweeps and compared through shared memory
  __shared__ T t1[32][33], t2[32][33];
  const int64_t nt = (n + 31) / 32, pairs = nt * (nt + 1) / 2;
  const int64_t b = blockIdx.x / pairs;
  int64_t p = blockIdx.x % pairs;
  int64_t ti = (int64_t)((sqrt(8.0 * (double)p + 1.0) - 1.0) * 0.5);
  while (ti * (ti + 1) / 2 > p) --ti;
  while ((ti + 1) * (ti + 2) / 2 <= p) ++ti;
  const int64_t tj = p - ti * (ti + 1) / 2;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  T mabs = T(0), masym = T(0);
#pragma unroll
  for (int r = ty; r < 32; r += 8) {
    const int64_t i1 = ti * 32 + r, j1 = tj * 32 + tx;  // tile (ti, tj)
    const int64_t i2 = tj * 32 + r, j2 = ti * 32 + tx;  // tile (tj, ti)
    const T v1 = (i1 < n && j1 < n) ? *a.at(b, i1, j1) : T(0);
    const T v2 = (i2 < n && j2 < n) ? *a.at(b, i2, j2) : T(0);
    t1[r][tx] = v1;
    t2[r][tx] = v2;
  }
  __syncthreads();
#pragma unroll
  for (int r = ty; r < 32; r += 8) {
    const int64_t i = ti * 32 + r, j = tj * 32 + tx;
    if (i < n && j < n) {
      const T v = t1[r][tx];
      if (fabs(v) > mabs) mabs = fabs(v);
      if (ti != tj) {
        const T w = t2[r][tx];  // element (tj*32 + r, ti*32 + tx): the other triangle
        if (fabs(w) > mabs) mabs = fabs(w);
        const T d = fabs(v - t2[tx][r]);  // a(i, j) vs a(j, i)
        if (d > masym) masym = d;
      } else if (tx > r) {
        const T d = fabs(v - t1[tx][r]);
        if (d > masym) masym = d;
      }
    }
  }
  __shared__ unsigned long long s0[8], s1[8];
  unsigned long long u0 = ord_bits(mabs), u1 = ord_bits(masym);
  for (int o = 16; o; o >>= 1) {
    u0 = max(u0, __shfl_xor_sync(0xffffffffu, u0, o));
    u1 = max(u1, __shfl_xor_sync(0xffffffffu, u1, o));
  }
  if (tx == 0) {
    s0[ty] = u0;
    s1[ty] = u1;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int k = 1; k < 8; ++k) {
      u0 = max(u0, s0[k]);
      u1 = max(u1, s1[k]);
    }
    atomicMax(red + 2 * b, u0);
    atomicMax(red + 2 * b + 1, u1);
  }
}

template <typename T>
__global__ void k_symcheck_decide(int64_t batch, const unsigned long long* red, int32_t* info) {
  for (int64_t b = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; b < batch; b += (int64_t)gridDim.x * blockDim.x) {
    const T scale = from_bits<T>(red[2 * b]);
    const T asym = from_bits<T>(red[2 * b + 1]);
    if (asym > Num<T>::sym_rtol * (scale > T(0) ? scale : T(1))) record_failure(info, b, DLA_ERR_ASYMMETRIC, 0);
  }
}

// Exact-zero diagonal => SINGULAR(first k); checked before any write.
// One CTA per slice; the smallest zero index wins.
template <typename T>
__global__ void k_zero_diag(int64_t batch, int64_t n, MatB<const T> t, int32_t* info) {
  __shared__ int first;
  const int64_t b = blockIdx.x;
  if (threadIdx.x == 0) first = 0x7fffffff;
  __syncthreads();
  if (info[b] != 0) return;
  for (int64_t k = threadIdx.x; k < n; k += blockDim.x)
    if (*t.at(b, k, k) == T(0)) atomicMin(&first, (int)k);
  __syncthreads();
  if (threadIdx.x == 0 && first != 0x7fffffff) info[b] = DLA_INFO(DLA_ERR_SINGULAR, first);
}

// sumlogdiag forward: logs in parallel, sum strictly in i = 0..n-1 order.
template <typename T>
__global__ void k_sumlogdiag(int64_t n, T* out, MatB<const T> a) {
  // per-thread strided partial sums, then a fixed-order tree: deterministic
  // (a sequential sum by one thread was a ~50 us serial chain at n = 4096)
  __shared__ T part[256];
  const int64_t b = blockIdx.x;
  T acc = T(0);
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) acc += Num<T>::log_(*a.at(b, i, i));
  part[threadIdx.x] = acc;
  __syncthreads();
  for (int st = blockDim.x / 2; st; st >>= 1) {
    if ((int)threadIdx.x < st) part[threadIdx.x] += part[threadIdx.x + st];
    __syncthreads();
  }
  if (threadIdx.x == 0) out[b] = part[0];
}

template <typename T>
__global__ void k_sumlogdiag_bwd(int64_t batch, int64_t n, MatB<T> abar, const T* g, MatB<const T> a, int accumulate) {
  const int64_t total = batch * n * n;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t b = t / (n * n), r = t % (n * n), i = r / n, j = r % n;
    T* p = abar.at(b, i, j);
    if (i == j) {
      const T v = g[b] / *a.at(b, i, i);
      *p = accumulate ? *p + v : v;
    } else if (!accumulate) {
      *p = T(0);
    }
  }
}

// accumulate: only the diagonal is touched (batch * n threads, no n^2 sweep)
template <typename T>
__global__ void k_sumlogdiag_bwd_diag(int64_t batch, int64_t n, MatB<T> abar, const T* g, MatB<const T> a) {
  const int64_t total = batch * n;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t b = t / n, i = t - b * n;
    T* p = abar.at(b, i, i);
    *p += g[b] / *a.at(b, i, i);
  }
}

}  // namespace

template <typename T>
dla_status ew_copy(const Ctx& c, int64_t batch, int64_t m, int64_t n, MatB<const T> src, MatB<T> dst,
                   const int32_t* skip) {
  if (batch * m * n == 0 || src.p == dst.p) return DLA_OK;
  const bool packed = src.ld == n && dst.ld == n && (batch == 1 || (src.bs == m * n && dst.bs == m * n));
  if (packed && skip != nullptr && batch <= 65535) {  // per-slice skip: one slice per grid row
    const bool vec = (reinterpret_cast<uintptr_t>(src.p) % 16 == 0) && (reinterpret_cast<uintptr_t>(dst.p) % 16 == 0) &&
                     (m * n) % (16 / sizeof(T)) == 0;
    const int64_t per = m * n;
    const unsigned gx = blocks_for(per / (vec ? 16 / sizeof(T) : 1), 256, std::max<int64_t>(1, 148 * 16 / batch));
    k_copy_slices<T><<<dim3(gx, (unsigned)batch), 256, 0, c.stream>>>(per, src.p, dst.p, skip, vec);
    DLAB_LAUNCH_CHECK();
    return DLA_OK;
  }
  if (packed && skip == nullptr) {
    const int64_t count = batch * m * n;
    const bool vec = (reinterpret_cast<uintptr_t>(src.p) % 16 == 0) && (reinterpret_cast<uintptr_t>(dst.p) % 16 == 0);
    k_copy_flat<T><<<blocks_for(count / (vec ? 16 / sizeof(T) : 1), 256, 148 * 16), 256, 0, c.stream>>>(count, src.p,
                                                                                                        dst.p, vec);
    DLAB_LAUNCH_CHECK();
    return DLA_OK;
  }
  k_copy<T><<<blocks_for(batch * m * n, 256), 256, 0, c.stream>>>(batch, m, n, src, dst, skip);
  DLAB_LAUNCH_CHECK();
  return DLA_OK;
}

template <typename T>
dla_status ew_scale(const Ctx& c, int64_t batch, int64_t m, int64_t n, MatB<T> x, T alpha, const int32_t* skip) {
  if (batch * m * n == 0 || alpha == T(1)) return DLA_OK;
  k_scale<T><<<blocks_for(batch * m * n, 256), 256, 0, c.stream>>>(batch, m, n, x, alpha, skip);
  DLAB_LAUNCH_CHECK();
  return DLA_OK;
}

// tril / triu zeroing (k_square ops 0 / 1): each row visits only its strict
// upper (lower) part, two columns per thread with 16-byte stores.
template <typename T, bool UPPER>
__global__ void k_zero_tri(int64_t batch, int64_t n, MatB<T> x, const int32_t* skip, bool vec) {
  const int64_t r0 = blockIdx.y * (int64_t)blockDim.y + threadIdx.y, rs = (int64_t)gridDim.y * blockDim.y;
  const int64_t db = rs / n, di = rs - db * n;  // (slice, row) advance incrementally: no division per row
  int64_t b = r0 / n, i = r0 - b * n;
  for (int64_t row = r0; row < batch * n; row += rs, b += db, i += di) {
    if (i >= n) {
      i -= n;
      ++b;
    }
    if (slice_failed(skip, b)) continue;
    const int64_t j0 = UPPER ? i + 1 : 0, j1 = UPPER ? n : i;  // zero columns [j0, j1)
    if (j0 >= j1) continue;
    T* xr = x.at(b, i, 0);
    const int64_t p0 = j0 / 2, p1 = (j1 + 1) / 2;
    for (int64_t p = p0 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < p1; p += (int64_t)gridDim.x * blockDim.x) {
      const int64_t j = 2 * p;
      if (vec && j >= j0 && j + 1 < j1) {
        if constexpr (sizeof(T) == 8)
          *reinterpret_cast<double2*>(xr + j) = make_double2(0.0, 0.0);
        else
          *reinterpret_cast<float2*>(xr + j) = make_float2(0.f, 0.f);
      } else {
        if (j >= j0 && j < j1) xr[j] = T(0);
        if (j + 1 >= j0 && j + 1 < j1) xr[j + 1] = T(0);
      }
    }
  }
}

// Launch shape of the row-pair kernels: 256-thread blocks of (tx lanes over a
// row's column pairs) x (ty rows), 16 resident blocks per SM's worth of grid.
inline void row_pair_grid(int64_t batch, int64_t n, dim3& grid, dim3& block) {
  const int64_t pairs = std::max<int64_t>(1, (n + 1) / 2);
  const int tx = (int)std::min<int64_t>(256, (pairs + 31) / 32 * 32);
  const int ty = 256 / tx;
  const int64_t gx = (pairs + tx - 1) / tx;
  int64_t gy = std::max<int64_t>(1, (148 * 16) / gx);
  gy = std::min<int64_t>(std::min<int64_t>(gy, (batch * n + ty - 1) / ty), 65535);
  grid = dim3((unsigned)gx, (unsigned)gy);
  block = dim3((unsigned)tx, (unsigned)ty);
}

template <typename T>
dla_status ew_square(const Ctx& c, int64_t batch, int64_t n, MatB<T> x, int op, T alpha, const int32_t* skip) {
  if (batch * n == 0) return DLA_OK;
  if (op == 0 || op == 1) {
    const bool vec = (x.ld % 2 == 0) && (x.bs % 2 == 0) && (reinterpret_cast<uintptr_t>(x.p) % (2 * sizeof(T)) == 0);
    dim3 grid, block;
    row_pair_grid(batch, n, grid, block);
    if (op == 0)
      k_zero_tri<T, true><<<grid, block, 0, c.stream>>>(batch, n, x, skip, vec);
    else
      k_zero_tri<T, false><<<grid, block, 0, c.stream>>>(batch, n, x, skip, vec);
    DLAB_LAUNCH_CHECK();
    return DLA_OK;
  }
  k_square<T><<<row_grid(batch, n), 256, 0, c.stream>>>(batch, n, x, op, alpha, skip);
  DLAB_LAUNCH_CHECK();
  return DLA_OK;
}

template <typename T>
dla_status ew_tri_copy(const Ctx& c, int64_t batch, int64_t n, MatB<const T> src, MatB<T> dst, bool from_upper) {
  if (batch * n == 0) return DLA_OK;
  const bool vec = !from_upper && src.ld % 2 == 0 && dst.ld % 2 == 0 && (batch == 1 || (src.bs % 2 == 0 && dst.bs % 2 == 0)) &&
                   reinterpret_cast<uintptr_t>(src.p) % (2 * sizeof(T)) == 0 &&
                   reinterpret_cast<uintptr_t>(dst.p) % (2 * sizeof(T)) == 0;
  if (vec) {
    dim3 grid, block;
    row_pair_grid(batch, n, grid, block);
    k_tri_copy_vec<T><<<grid, block, 0, c.stream>>>(batch, n, src, dst);
    DLAB_LAUNCH_CHECK();
    return DLA_OK;
  }
  k_tri_copy<T><<<row_grid(batch, n), 256, 0, c.stream>>>(batch, n, src, dst, from_upper);
  DLAB_LAUNCH_CHECK();
  return DLA_OK;
}

template <typename T>
dla_status ew_add_transpose(const Ctx& c, int64_t batch, int64_t n, MatB<const T> src, MatB<T> dst, T alpha) {
  if (batch * n == 0) return DLA_OK;
  k_add_transpose<T><<<pair_grid(batch, n), dim3(32, 8), 0, c.stream>>>(batch, n, src, dst, alpha);
  DLAB_LAUNCH_CHECK();
  return DLA_OK;
}

template <typename T>
dla_status ew_scale_diag(const Ctx& c, int64_t batch, int64_t n, MatB<T> x, T alpha) {
  if (batch * n == 0) return DLA_OK;
  k_scale_diag<T><<<blocks_for(batch * n, 256), 256, 0, c.stream>>>(batch, n, x, alpha);
  DLAB_LAUNCH_CHECK();
  return DLA_OK;
}

template <typename T>
dla_status ew_sym_lower_into(const Ctx& c, int64_t batch, int64_t n, MatB<const T> src, MatB<T> dst, T alpha) {
  if (batch * n == 0) return DLA_OK;
  // in-place safe: a block reads only its own lower tile (I, J) before it
  // writes (I, J) and the upper tile (J, I), which no block reads
  k_sym_lower_tiles<T><<<pair_grid(batch, n), dim3(32, 8), 0, c.stream>>>(batch, n, src, dst, alpha);
  DLAB_LAUNCH_CHECK();
  return DLA_OK;
}

template <typename T>
dla_status check_symmetric(const Ctx& c, int64_t batch, int64_t n, MatB<const T> a, int32_t* info) {
  if (info == nullptr || batch * n == 0) return DLA_OK;
  DLAB_SCRATCH(red_s, c, ws_check_symmetric(batch));  // from the caller's workspace (no hidden allocation)
  unsigned long long* red = red_s.as<unsigned long long>();
  if (cudaMemsetAsync(red, 0, sizeof(unsigned long long) * 2 * batch, c.stream) != cudaSuccess) return DLA_ERR_CUDA;
  const int64_t nt = (n + 31) / 32;
  k_symcheck_reduce<T><<<(unsigned)(batch * (nt * (nt + 1) / 2)), 256, 0, c.stream>>>(batch, n, a, red);
  k_symcheck_decide<T><<<blocks_for(batch, 256), 256, 0, c.stream>>>(batch, red, info);
  note_launch(1);
  DLAB_LAUNCH_CHECK();
  return DLA_OK;
}

template <typename T>
dla_status check_zero_diag(const Ctx& c, int64_t batch, int64_t n, MatB<const T> t, int32_t* info) {
  if (info == nullptr || batch * n == 0) return DLA_OK;
  k_zero_diag<T><<<(unsigned)batch, 256, 0, c.stream>>>(batch, n, t, info);
  DLAB_LAUNCH_CHECK();
  return DLA_OK;
}

template <typename T>
dla_status sumlogdiag_fwd(const Ctx& c, int64_t batch, int64_t n, T* out, MatB<const T> a) {
  if (batch == 0) return DLA_OK;
  if (n == 0) return cudaMemsetAsync(out, 0, sizeof(T) * batch, c.stream) == cudaSuccess ? DLA_OK : DLA_ERR_CUDA;
  k_sumlogdiag<T><<<(unsigned)batch, n >= 2048 ? 256 : 128, 0, c.stream>>>(n, out, a);
  DLAB_LAUNCH_CHECK();
  return DLA_OK;
}

template <typename T>
dla_status sumlogdiag_bwd(const Ctx& c, int64_t batch, int64_t n, MatB<T> abar, const T* g, MatB<const T> a,
                          bool accumulate) {
  if (batch * n == 0) return DLA_OK;
  if (accumulate) {  // only the diagonal is touched
    k_sumlogdiag_bwd_diag<T><<<blocks_for(batch * n, 256), 256, 0, c.stream>>>(batch, n, abar, g, a);
  } else {
    k_sumlogdiag_bwd<T><<<blocks_for(batch * n * n, 256), 256, 0, c.stream>>>(batch, n, abar, g, a, 0);
  }
  DLAB_LAUNCH_CHECK();
  return DLA_OK;
}

#define INST(T)                                                                                          \
  template dla_status ew_copy<T>(const Ctx&, int64_t, int64_t, int64_t, MatB<const T>, MatB<T>,         \
                                 const int32_t*);                                                       \
  template dla_status ew_scale<T>(const Ctx&, int64_t, int64_t, int64_t, MatB<T>, T, const int32_t*);   \
  template dla_status ew_square<T>(const Ctx&, int64_t, int64_t, MatB<T>, int, T, const int32_t*);      \
  template dla_status check_symmetric<T>(const Ctx&, int64_t, int64_t, MatB<const T>, int32_t*);        \
  template dla_status ew_tri_copy<T>(const Ctx&, int64_t, int64_t, MatB<const T>, MatB<T>, bool);       \
  template dla_status ew_sym_lower_into<T>(const Ctx&, int64_t, int64_t, MatB<const T>, MatB<T>, T);    \
  template dla_status ew_add_transpose<T>(const Ctx&, int64_t, int64_t, MatB<const T>, MatB<T>, T);     \
  template dla_status ew_scale_diag<T>(const Ctx&, int64_t, int64_t, MatB<T>, T);                       \
  template dla_status check_zero_diag<T>(const Ctx&, int64_t, int64_t, MatB<const T>, int32_t*);        \
  template dla_status sumlogdiag_fwd<T>(const Ctx&, int64_t, int64_t, T*, MatB<const T>);               \
  template dla_status sumlogdiag_bwd<T>(const Ctx&, int64_t, int64_t, MatB<T>, const T*, MatB<const T>, \
                                        bool);
INST(double)
INST(float)

}  // namespace dlab
