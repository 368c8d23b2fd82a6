// Inverse-based large-n paths: every triangular solve becomes a triangular
// GEMM on FP64 DMMA instead of a chain of n/64 dependent leaf solves.
//
//   trtri_levels : W <- W^{-1} for lower-triangular W, n = 64 * 2^k.  All
//                  64x64 diagonal blocks are inverted by ONE launch; then for
//                  s = 64, 128, ..., n/2 every pair [A 0; B C] of the level is
//                  finished at once:  B <- -C^{-1} (B A^{-1})  (two batched
//                  triangular GEMMs over the level's n/2s blocks).
//                  2 log2(n/64) + 1 launches for any n (13 at n = 4096).
//   trsm_inv     : X <- alpha op(T)^{-1} X = one triangular GEMM with the
//                  inverse (dl/blas.hpp:307-395 semantics; the reference's
//                  substitution order is replaced, results agree to rounding).
//   potrf_bwd_inv: Abar = 1/2 sym(L^-T copyltu(L^T Lbar) L^-1)
//                  (dl/adjoints.hpp:175-191) as trtri + three triangular
//                  GEMMs: 2 n^3 flops, all DMMA, vs the composed 3 n^3 of
//                  trmm + 2 trsm.
// Scratch (n^2 per slice) is carved from the caller's workspace (ws_* mirrors).
#include <mutex>

#include "chol64.cuh"
#include "common.cuh"
#include "ops.cuh"

namespace dlab {
namespace {

constexpr int IB = 64;
constexpr int ILD = IB + 1;
static_assert(ILD == CH_LD, "shared layout shared with chol64.cuh");

template <typename T>
MatB<const T> C_(MatB<T> m) {
  return MatB<const T>{m.p, m.ld, m.bs, m.bsi};
}

// Invert every 64x64 lower diagonal block of w (slice b, block k) in place:
// L X = I for all 64 columns at once with the blocked substitution (8x8
// diagonal solves + DMMA updates in shared memory, chol64.cuh).
template <typename T>
__global__ void __launch_bounds__(128) k_trtri_blocks(int64_t nblk, MatB<T> w) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T* S = reinterpret_cast<T*>(smem_raw);
  T* X = S + IB * ILD;  // vector-major: X[v * ILD + i] = Linv(i, v)
  T* rd = X + IB * ILD;
  const int64_t b = blockIdx.x / nblk, k = blockIdx.x % nblk;
  T* base = w.p + b * w.bs + k * IB * (w.ld + 1);
  for (int e0 = threadIdx.x; e0 < IB * IB; e0 += 8 * 128) {
    T v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int e = e0 + u * 128, i = e / IB, j = e % IB;
      v[u] = j <= i ? base[i * w.ld + j] : T(0);
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int e = e0 + u * 128, i = e / IB, j = e % IB;
      S[i * ILD + j] = v[u];
      X[i * ILD + j] = (i == j) ? T(1) : T(0);
    }
  }
  __syncthreads();
  if (threadIdx.x < IB) rd[threadIdx.x] = T(1) / S[threadIdx.x * ILD + threadIdx.x];
  __syncthreads();
  blocked_fwd_subst<T>(S, X, rd, IB, IB);
  for (int e = threadIdx.x; e < IB * IB; e += blockDim.x) {
    const int i = e / IB, j = e % IB;
    base[i * w.ld + j] = j <= i ? X[j * ILD + i] : T(0);
  }
}

// fp64: the same inverse by level doubling inside shared memory.  The eight
// 8x8 diagonal blocks are inverted by 64 threads (one column each, a serial
// chain of 8), then for s = 8, 16, 32 every pair [A 0; B C] of the level is
// finished with two triangular DMMA products, B <- -C^{-1} (B A^{-1}) — the
// in-smem analogue of trtri_levels' launches.  ~86k MACs per block on DMMA
// instead of 64 substitution phases: the kernel is bound by its HBM pass.
constexpr int TLD8 = 33;  // T1 scratch row stride (32 x 32 at most)

__device__ __forceinline__ void dmma884(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

// src: the factor (its lower triangle, or with from_upper its upper triangle
// transposed); the inverted diagonal blocks go to w (may be src itself).
__global__ void __launch_bounds__(128) k_trtri64_dmma(int64_t nblk, MatB<const double> src, bool from_upper,
                                                      MatB<double> w) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double* S = reinterpret_cast<double*>(smem_raw);  // [64][ILD]
  double* Tt = S + IB * ILD;                         // [32][TLD8]
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, fr = lane >> 2, fc = lane & 3;
  const int64_t b = blockIdx.x / nblk, k = blockIdx.x % nblk;
  double* base = w.p + b * w.bs + k * IB * (w.ld + 1);
  const double* sb = src.p + b * src.bs + k * IB * (src.ld + 1);
  {
    double v[32];
#pragma unroll
    for (int u = 0; u < 32; ++u) {
      const int e = tid + u * 128, i = e >> 6, j = e & 63;
      v[u] = j <= i ? (from_upper ? sb[j * src.ld + i] : sb[i * src.ld + j]) : 0.0;
    }
#pragma unroll
    for (int u = 0; u < 32; ++u) {
      const int e = tid + u * 128, i = e >> 6, j = e & 63;
      S[i * ILD + j] = v[u];
    }
  }
  __syncthreads();
  // 8x8 diagonal blocks: thread (d, c) solves L_d x = e_c
  {
    const int o = ((tid >> 3) & 7) * 8, c = tid & 7;
    double x[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      double acc = i == c ? 1.0 : 0.0;
#pragma unroll
      for (int q = 0; q < i; ++q)
        if (q >= c) acc -= S[(o + i) * ILD + o + q] * x[q];
      x[i] = i >= c ? acc / S[(o + i) * ILD + o + i] : 0.0;
    }
    __syncthreads();
    if (tid < 64) {
#pragma unroll
      for (int i = 0; i < 8; ++i)
        if (i >= c) S[(o + i) * ILD + o + c] = x[i];
    }
  }
  __syncthreads();
#pragma unroll
  for (int s = 8; s < IB; s *= 2) {
    const int pairs = IB / (2 * s), tps = (s / 8) * (s / 8), tiles = pairs * tps;
    // T1 = B A^{-1}: tile (rt, nt) of pair p, k >= nt (A^{-1} lower)
    for (int t = warp; t < tiles; t += 4) {
      const int p = t / tps, r = t % tps, rt = (r / (s / 8)) * 8, nt = (r % (s / 8)) * 8, o = 2 * s * p;
      double d0 = 0.0, d1 = 0.0;
      for (int kk = nt; kk < s; kk += 4) {
        const double af = S[(o + s + rt + fr) * ILD + o + kk + fc];
        const double bf = S[(o + kk + fc) * ILD + o + nt + fr];
        dmma884(d0, d1, af, bf);
      }
      Tt[(p * s + rt + fr) * TLD8 + nt + 2 * fc] = d0;
      Tt[(p * s + rt + fr) * TLD8 + nt + 2 * fc + 1] = d1;
    }
    __syncthreads();
    // B = -C^{-1} T1: k <= rt + 7 (C^{-1} lower)
    for (int t = warp; t < tiles; t += 4) {
      const int p = t / tps, r = t % tps, rt = (r / (s / 8)) * 8, nt = (r % (s / 8)) * 8, o = 2 * s * p;
      double d0 = 0.0, d1 = 0.0;
      for (int kk = 0; kk < rt + 8; kk += 4) {
        const double af = S[(o + s + rt + fr) * ILD + o + s + kk + fc];
        const double bf = Tt[(p * s + kk + fc) * TLD8 + nt + fr];
        dmma884(d0, d1, af, bf);
      }
      S[(o + s + rt + fr) * ILD + o + nt + 2 * fc] = -d0;
      S[(o + s + rt + fr) * ILD + o + nt + 2 * fc + 1] = -d1;
    }
    __syncthreads();
  }
#pragma unroll 8
  for (int u = 0; u < 32; ++u) {
    const int e = tid + u * 128, i = e >> 6, j = e & 63;
    base[i * w.ld + j] = j <= i ? S[i * ILD + j] : 0.0;
  }
}

// ---------------------------------------------------- n <= 128, fp64, fused
// W = inv([L 0; 0 I]) of one matrix per CTA in ONE launch (256 threads, two
// CTAs per SM): L's lower triangle as three 64 x 64 shared blocks
// (A11, A21, A22; row stride 68 = 4 mod 16, so DMMA fragments load
// conflict-free in both orientations); the 16 diagonal 8 x 8 inverses (one
// column per thread), the s = 8, 16, 32 doubling levels of both diagonal
// blocks together (T1 scratch in each block's unused upper-right quadrant),
// then the top level A21 <- -A22^{-1} (A21 A11^{-1}) by row strips.  Replaces
// tri_copy + k_trtri64_dmma + two level GEMMs (three HBM passes, three
// launches) wherever a 128-wide level-batched inverse was formed.
// LAUUM: instead of W, write B = W^T W (potri, dl/cholesky.hpp:141-147):
// its lower tiles on DMMA, each value stored at (i, j) and (j, i) (exactly
// symmetric).  FROM_UPPER: L(i, j) = src(j, i) (upper-stored factors).
constexpr int TLD = 68;
constexpr int TBLK = 64 * TLD;

__device__ __forceinline__ double* t128(double* S, int i, int j) {
  return i < 64 ? S + i * TLD + j : (j < 64 ? S + TBLK + (i - 64) * TLD + j : S + 2 * TBLK + (i - 64) * TLD + (j - 64));
}

template <bool FROM_UPPER, bool LAUUM>
__global__ void __launch_bounds__(256, 2) k_trtri128(int n, int nout, MatB<const double> src, MatB<double> dst) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double* S = reinterpret_cast<double*>(smem_raw);
  double* S1 = S + TBLK;
  double* S2 = S + 2 * TBLK;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, fr = lane >> 2, fc = lane & 3;
  const int64_t b = blockIdx.x;
  const double* g = src.p + b * src.bs;
  const int64_t lds = src.ld;
  // (1) load: row pairs, one column per thread; identity beyond n; the strict
  // upper of the diagonal blocks zeroed (diagonal DMMA tiles read it)
  {
    const int j = tid & 127;
#pragma unroll 4
    for (int u0 = 0; u0 < 64; u0 += 16) {
      double v[16];
#pragma unroll
      for (int q = 0; q < 16; ++q) {
        const int i = 2 * (u0 + q) + (tid >> 7);
        const bool in = i < n && j < n && (FROM_UPPER ? j >= i : j <= i);
        v[q] = in ? g[i * lds + j] : 0.0;
      }
#pragma unroll
      for (int q = 0; q < 16; ++q) {
        const int i = 2 * (u0 + q) + (tid >> 7);
        const double pad = (i == j && i >= n) ? 1.0 : 0.0;
        if (FROM_UPPER) {
          if (j >= i) *t128(S, j, i) = (i < n && j < n) ? v[q] : pad;  // L(j, i) = src(i, j)
          if (j > i && (i < 64) == (j < 64)) *t128(S, i, j) = 0.0;
        } else {
          if (j <= i) *t128(S, i, j) = (i < n && j < n) ? v[q] : pad;
          else if ((i < 64) == (j < 64)) *t128(S, i, j) = 0.0;
        }
      }
    }
  }
  __syncthreads();
  // (2) 8 x 8 diagonal inverses: thread (block, column)
  {
    const int o8 = (tid >> 3) * 8, c = tid & 7;  // tid < 128
    double x[8];
    if (tid < 128) {
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        double acc = i == c ? 1.0 : 0.0;
#pragma unroll
        for (int q = 0; q < i; ++q)
          if (q >= c) acc -= *t128(S, o8 + i, o8 + q) * x[q];
        x[i] = i >= c ? acc / *t128(S, o8 + i, o8 + i) : 0.0;
      }
    }
    __syncthreads();
    if (tid < 128) {
#pragma unroll
      for (int i = 0; i < 8; ++i)
        if (i >= c) *t128(S, o8 + i, o8 + c) = x[i];
    }
  }
  __syncthreads();
  // (3) doubling levels inside both diagonal blocks
#pragma unroll
  for (int s = 8; s < 64; s *= 2) {
    const int pairs = 64 / (2 * s), tps = (s / 8) * (s / 8), per = pairs * tps;
    for (int t = warp; t < 2 * per; t += 8) {  // T1 = B A^{-1}: k >= nt
      double* blk = t < per ? S : S2;
      const int tt = t % per, pr = tt / tps, r = tt % tps, rt = (r / (s / 8)) * 8, nt = (r % (s / 8)) * 8;
      const int o = 2 * s * pr;
      double d0 = 0.0, d1 = 0.0;
      for (int kk = nt; kk < s; kk += 4)
        dmma884(d0, d1, blk[(o + s + rt + fr) * TLD + o + kk + fc], blk[(o + kk + fc) * TLD + o + nt + fr]);
      double* t1 = blk + (pr * s + rt + fr) * TLD + 32 + pr * s + nt + 2 * fc;
      t1[0] = d0;
      t1[1] = d1;
    }
    __syncthreads();
    for (int t = warp; t < 2 * per; t += 8) {  // B = -C^{-1} T1: k <= rt + 7
      double* blk = t < per ? S : S2;
      const int tt = t % per, pr = tt / tps, r = tt % tps, rt = (r / (s / 8)) * 8, nt = (r % (s / 8)) * 8;
      const int o = 2 * s * pr;
      double d0 = 0.0, d1 = 0.0;
      for (int kk = 0; kk < rt + 8; kk += 4)
        dmma884(d0, d1, blk[(o + s + rt + fr) * TLD + o + s + kk + fc],
                blk[(pr * s + kk + fc) * TLD + 32 + pr * s + nt + fr]);
      double* bo = blk + (o + s + rt + fr) * TLD + o + nt + 2 * fc;
      bo[0] = -d0;
      bo[1] = -d1;
    }
    __syncthreads();
  }
  // (4) top level: A21 <- -A22^{-1} (A21 A11^{-1}); row strip 8 warp .. + 7 per warp
  {
    double acc[8][2];
#pragma unroll
    for (int t = 0; t < 8; ++t) acc[t][0] = acc[t][1] = 0.0;
#pragma unroll 4
    for (int kk = 0; kk < 64; kk += 4) {  // T1 = A21 A11^{-1}: column tile nt needs k >= nt
      const double af = S1[(8 * warp + fr) * TLD + kk + fc];
#pragma unroll
      for (int t = 0; t < 8; ++t)
        if (8 * t <= kk) dmma884(acc[t][0], acc[t][1], af, S[(kk + fc) * TLD + 8 * t + fr]);
    }
    __syncwarp();
#pragma unroll
    for (int t = 0; t < 8; ++t) {  // in place: this strip of A21 is read by this warp only
      S1[(8 * warp + fr) * TLD + 8 * t + 2 * fc] = acc[t][0];
      S1[(8 * warp + fr) * TLD + 8 * t + 2 * fc + 1] = acc[t][1];
      acc[t][0] = acc[t][1] = 0.0;
    }
    __syncthreads();
    for (int kk = 0; kk < 8 * warp + 8; kk += 4) {  // -A22^{-1} T1: k <= row
      const double af = S2[(8 * warp + fr) * TLD + kk + fc];
#pragma unroll
      for (int t = 0; t < 8; ++t) dmma884(acc[t][0], acc[t][1], af, S1[(kk + fc) * TLD + 8 * t + fr]);
    }
    __syncthreads();  // every strip of T1 has been read
#pragma unroll
    for (int t = 0; t < 8; ++t) {
      S1[(8 * warp + fr) * TLD + 8 * t + 2 * fc] = -acc[t][0];
      S1[(8 * warp + fr) * TLD + 8 * t + 2 * fc + 1] = -acc[t][1];
    }
  }
  __syncthreads();
  double* o = dst.p + b * dst.bs;
  const int64_t ldo = dst.ld;
  if constexpr (!LAUUM) {
    const int j = tid & 127;
    if (j < nout) {
#pragma unroll 8
      for (int u = 0; u < 64; ++u) {
        const int i = 2 * u + (tid >> 7);
        if (i < nout) o[i * ldo + j] = j <= i ? *t128(S, i, j) : 0.0;
      }
    }
  } else {
    // (5) B = W^T W: lower 8 x 8 tiles (I >= J), k >= 8 I; stored mirrored
    for (int t = warp; t < 136; t += 8) {
      int I = 0;
      while ((I + 1) * (I + 2) / 2 <= t) ++I;
      const int J = t - I * (I + 1) / 2;
      double d0 = 0.0, d1 = 0.0;
      for (int kk = 8 * I; kk < 128; kk += 4)
        dmma884(d0, d1, *t128(S, kk + fc, 8 * I + fr), *t128(S, kk + fc, 8 * J + fr));
      const int i = 8 * I + fr;
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int j = 8 * J + 2 * fc + e;
        const double v = e ? d1 : d0;
        if (i >= j && i < nout && j < nout) {
          o[i * ldo + j] = v;
          o[j * ldo + i] = v;
        }
      }
    }
  }
}

// The padding of the inverse's operand (see inv_pad): rows < n get zeros in
// columns [n, N), rows >= n the identity row.
template <typename T>
__global__ void k_pad_eye(int64_t batch, int64_t n, int64_t N, MatB<T> w) {
  for (int64_t row = blockIdx.y; row < batch * N; row += gridDim.y) {
    const int64_t b = row / N, i = row - b * N;
    T* wr = w.p + b * w.bs + i * w.ld;
    const int64_t j0 = i < n ? n : 0;
    for (int64_t j = j0 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < N; j += (int64_t)gridDim.x * blockDim.x)
      wr[j] = (i == j) ? T(1) : T(0);
  }
}

}  // namespace

template <typename T>
size_t trtri_levels_tmp(int64_t n) {
  return sizeof(T) * (size_t)(n / 2) * (size_t)(n / 2);
}

template <typename T>
bool inv_eligible(int64_t n) {
  if (n < 2 * IB || n % IB) return false;
  const int64_t q = n / IB;
  return (q & (q - 1)) == 0;
}

// Order of the padded inverse for the potrf pullback at other n: L^{-1} is
// the leading n x n block of inv([L 0; 0 I]) at the next N = 64 * 2^k (block
// algebra: the zero off-diagonal block stays exactly zero), so the inverse
// runs level-batched at N while the three products stay at n.  Taken while the
// N^3 / 3 inverse is at most ~1.1 n^3 (N <= 1.5 n) or N <= 256; 0 = not used.
template <typename T>
int64_t inv_pad(int64_t n) {
  if (inv_eligible<T>(n)) return n;
  if (n <= IB) return 0;
  int64_t N = 2 * IB;
  while (N < n) N *= 2;
  return (N <= 4 * IB || 2 * N <= 3 * n) ? N : 0;
}


template <typename T>
size_t trsm_inv_scratch(int64_t batch, int64_t m, int64_t n, int64_t nt) {
  return sizeof(T) * (size_t)batch * ((size_t)nt * nt + (size_t)m * n) + (size_t)batch * trtri_levels_tmp<T>(nt);
}
template <typename T>
size_t potrf_bwd_inv_scratch(int64_t batch, int64_t n) {
  const int64_t N = inv_pad<T>(n);
  return sizeof(T) * (size_t)batch * ((size_t)N * N + (size_t)n * n) + (size_t)batch * trtri_levels_tmp<T>(N);
}
template <typename T>
size_t potri_inv_scratch(int64_t batch, int64_t n) {
  return sizeof(T) * (size_t)batch * (size_t)n * n + (size_t)batch * trtri_levels_tmp<T>(n);
}

// ---- workspace mirrors (common.cuh): the carves of each routine's call tree
template <typename T>
size_t ws_trtri_levels(int64_t batch, int64_t n) {
  size_t w = 0;
  for (int64_t s = IB; s < n; s *= 2)
    if (n / (2 * s) == 1) w += 2 * ws_gemm<T>(batch, s, s, s, 1);  // inner > 1 levels never carve
  return w;
}
template <typename T>
size_t ws_trsm_inv(int64_t batch, int64_t m, int64_t n, bool right) {
  const int64_t nt = right ? n : m;
  return carve_bound(trsm_inv_scratch<T>(batch, m, n, nt)) + ws_trtri_levels<T>(batch, nt) +
         ws_gemm<T>(batch, m, n, nt);
}
template <typename T>
size_t ws_potrf_inv_prepare(int64_t batch, int64_t n) {
  return ws_trtri_levels<T>(batch, n);
}
template <typename T>
size_t ws_potrf_bwd_tail(int64_t batch, int64_t n) {  // potrf_bwd_phi + potrf_bwd_finish
  return 3 * ws_gemm<T>(batch, n, n, n);
}
template <typename T>
size_t ws_potrf_bwd_inv(int64_t batch, int64_t n) {
  return carve_bound(potrf_bwd_inv_scratch<T>(batch, n)) + ws_potrf_inv_prepare<T>(batch, inv_pad<T>(n)) +
         ws_potrf_bwd_tail<T>(batch, n);
}
template <typename T>
size_t ws_trmm_gemm(int64_t batch, int64_t m, int64_t n, bool right) {
  const int64_t nt = right ? n : m;
  if (sizeof(T) == 8 && !right && m <= 128) return ws_gemm<T>(batch, m, n, m);
  return carve_bound(sizeof(T) * (size_t)batch * (size_t)m * n) + ws_gemm<T>(batch, m, n, nt);
}
template <typename T>
size_t ws_potri_inv(int64_t batch, int64_t n) {
  return carve_bound(potri_inv_scratch<T>(batch, n)) + ws_trtri_levels<T>(batch, n) + ws_gemm<T>(batch, n, n, n);
}

template <typename T>
MatB<const double> as_d(MatB<const T> m) {
  return MatB<const double>{reinterpret_cast<const double*>(m.p), m.ld, m.bs, m.bsi};
}
template <typename T>
MatB<double> as_d(MatB<T> m) {
  return MatB<double>{reinterpret_cast<double*>(m.p), m.ld, m.bs, m.bsi};
}

// Level-batched inverse W = L^{-1}.  src == nullptr: in place, W lower
// triangular on entry (strict upper zero; stays zero).  Otherwise (fp64) L is
// read straight from src's lower triangle (from_upper: its upper triangle,
// transposed) -- the diagonal blocks by the block-inverse kernel, the
// off-diagonal blocks by each level's first product -- so no tri_copy pass
// precedes it; W's strict upper BLOCKS are then left unwritten, and every
// consumer reads W through a triangular operand flag (masked by the GEMM).
// tmp: >= trtri_levels_tmp(n) elements... bytes per slice, batch slices.
template <typename T>
dla_status trtri_levels(const Ctx& c, int64_t batch, int64_t n, MatB<T> w, T* tmp, const MatB<const T>* src,
                        bool from_upper) {
  const int64_t nblk = n / IB;
  if constexpr (sizeof(T) == 8) {
    const size_t sm = sizeof(double) * (IB * ILD + 32 * TLD8);
    ensure_smem_attr(k_trtri64_dmma, sm);
    MatB<double> wd{reinterpret_cast<double*>(w.p), w.ld, w.bs, w.bsi};
    const MatB<const double> sd = src ? as_d(*src) : MatB<const double>{wd.p, wd.ld, wd.bs, wd.bsi};
    k_trtri64_dmma<<<(unsigned)(batch * nblk), 128, sm, c.stream>>>(nblk, sd, src && from_upper, wd);
  } else {
    if (src) {  // fp32: the copy, then in place
      DLAB_TRY(ew_tri_copy<T>(c, batch, n, *src, w, from_upper));
      return trtri_levels<T>(c, batch, n, w, tmp);
    }
    const size_t sm = sizeof(T) * (2 * IB * ILD + IB);
    ensure_smem_attr(k_trtri_blocks<T>, sm);
    k_trtri_blocks<T><<<(unsigned)(batch * nblk), 128, sm, c.stream>>>(nblk, w);
  }
  DLAB_LAUNCH_CHECK();
  for (int64_t s = IB; s < n; s *= 2) {
    const int64_t pairs = n / (2 * s);
    const int64_t stride = 2 * s * (w.ld + 1);
    MatB<T> wa{w.p, w.ld, w.bs, stride};
    MatB<T> wb = wa.sub(s, 0), wc = wa.sub(s, s);
    MatB<T> t1{tmp, s, pairs * s * s, s * s};
    // T1 = B A^{-1}   (A^{-1} lower; B = L's block, from src when given)
    if (src && sizeof(T) == 8) {
      const int64_t sstride = 2 * s * (src->ld + 1);
      const MatB<const T> sa{src->p, src->ld, src->bs, sstride};
      const MatB<const T> bsrc = from_upper ? sa.sub(0, s) : sa.sub(s, 0);  // upper: B = (src block)^T
      DLAB_TRY(gemm<T>(c, batch, s, s, s, T(1), bsrc, from_upper, C_(wa), false, T(0), t1, MASK_FULL, nullptr,
                       TRI_NONE, TRI_LOWER, pairs));
    } else {
      DLAB_TRY(gemm<T>(c, batch, s, s, s, T(1), C_(wb), false, C_(wa), false, T(0), t1, MASK_FULL, nullptr, TRI_NONE,
                       TRI_LOWER, pairs));
    }
    // B = -C^{-1} T1  (C^{-1} lower)
    DLAB_TRY(gemm<T>(c, batch, s, s, s, T(-1), C_(wc), false, C_(t1), false, T(0), wb, MASK_FULL, nullptr,
                     TRI_LOWER, TRI_NONE, pairs));
  }
  return DLA_OK;
}

// fp64 128-wide inverse (or potri) in one launch: dst = lower-form
// inv([L 0; 0 I]) over nout x nout, L read from src's lower (or, from_upper,
// transposed upper) triangle, n <= 128.
inline dla_status trtri128(const Ctx& c, int64_t batch, int n, int nout, MatB<const double> src, bool from_upper,
                           MatB<double> dst, bool lauum) {
  const size_t sm = sizeof(double) * 3 * TBLK;
  auto go = [&](auto kern) {
    ensure_smem_attr(kern, sm);
    kern<<<(unsigned)batch, 256, sm, c.stream>>>(n, nout, src, dst);
  };
  if (lauum)
    from_upper ? go(k_trtri128<true, true>) : go(k_trtri128<false, true>);
  else
    from_upper ? go(k_trtri128<true, false>) : go(k_trtri128<false, false>);
  DLAB_LAUNCH_CHECK();
  return DLA_OK;
}
// The 128 fused path applies (fp64, batched slices of 128 x 128).
template <typename T>
bool use_trtri128(int64_t n) {
  static const bool on = [] {
    const char* e = getenv("DLA_TRTRI128");  // tuning switch: 0 = tri_copy + level-batched launches
    return e ? atoi(e) != 0 : true;
  }();
  return sizeof(T) == 8 && n == 128 && on;
}

template <typename T>
dla_status trsm_inv(const Ctx& c, int64_t batch, int64_t m, int64_t n, MatB<const T> t, MatB<T> x, bool right,
                    bool trans, bool lower, T alpha) {
  const int64_t nt = right ? n : m;
  DLAB_SCRATCH(ws, c, trsm_inv_scratch<T>(batch, m, n, nt));
  T* wp = ws.as<T>();
  MatB<T> w{wp, nt, nt * nt};
  MatB<T> y{wp + batch * nt * nt, n, m * n};
  T* tmp = wp + batch * (nt * nt + m * n);
  // lower-form W: inv(T) for lower T, inv(T^T) = T^{-T} for upper T
  if (use_trtri128<T>(nt)) {
    DLAB_TRY(trtri128(c, batch, 128, 128, as_d(t), !lower, as_d(w), false));
  } else {
    DLAB_TRY(trtri_levels<T>(c, batch, nt, w, tmp, &t, !lower));
  }
  const bool eff = (lower != trans);  // op(T)^{-1} = eff ? W : W^T
  const int tri = eff ? TRI_LOWER : TRI_UPPER;
  if (sizeof(T) == 8 && !right && m <= 128) {
    // X <- op(T)^{-1} X in place: one 128-row tile per column block reads all
    // of its X columns (the K range) before writing them (as trmm_gemm)
    Ctx cr = c;
    cr.gemm_rowtile = 1;
    return gemm<T>(cr, batch, m, n, m, alpha, C_(w), !eff, C_(x), false, T(0), x, MASK_FULL, c.info, tri, TRI_NONE);
  }
  if (!right)
    DLAB_TRY(gemm<T>(c, batch, m, n, m, alpha, C_(w), !eff, C_(x), false, T(0), y, MASK_FULL, c.info, tri, TRI_NONE));
  else
    DLAB_TRY(gemm<T>(c, batch, m, n, n, alpha, C_(x), false, C_(w), !eff, T(0), y, MASK_FULL, c.info, TRI_NONE, tri));
  return ew_copy<T>(c, batch, m, n, C_(y), x, c.info);
}

// Out-of-place trsm_inv: X = alpha op(T)^{-1} S (left) or alpha S op(T)^{-1}
// (right) as one triangular GEMM from S into X (S != X): no y scratch, no
// copy back.
template <typename T>
size_t ws_trsm_inv_from(int64_t batch, int64_t m, int64_t n, bool right) {
  const int64_t nt = right ? n : m;
  return carve_bound(sizeof(T) * (size_t)batch * (size_t)nt * nt + (size_t)batch * trtri_levels_tmp<T>(nt)) +
         ws_trtri_levels<T>(batch, nt) + ws_gemm<T>(batch, m, n, nt);
}
template <typename T>
dla_status trsm_inv_from(const Ctx& c, int64_t batch, int64_t m, int64_t n, MatB<const T> t, MatB<const T> src,
                         MatB<T> x, bool right, bool trans, bool lower, T alpha) {
  const int64_t nt = right ? n : m;
  DLAB_SCRATCH(ws, c, sizeof(T) * (size_t)batch * (size_t)nt * nt + (size_t)batch * trtri_levels_tmp<T>(nt));
  T* wp = ws.as<T>();
  MatB<T> w{wp, nt, nt * nt};
  T* tmp = wp + batch * nt * nt;
  if (use_trtri128<T>(nt)) {
    DLAB_TRY(trtri128(c, batch, 128, 128, as_d(t), !lower, as_d(w), false));
  } else {
    DLAB_TRY(trtri_levels<T>(c, batch, nt, w, tmp, &t, !lower));
  }
  const bool eff = (lower != trans);
  const int tri = eff ? TRI_LOWER : TRI_UPPER;
  if (!right)
    return gemm<T>(c, batch, m, n, m, alpha, C_(w), !eff, src, false, T(0), x, MASK_FULL, c.info, tri, TRI_NONE);
  return gemm<T>(c, batch, m, n, n, alpha, src, false, C_(w), !eff, T(0), x, MASK_FULL, c.info, TRI_NONE, tri);
}

// L^{-1} (lower form) of the factor into wi, with tmp >= trtri_levels_tmp(n)
// per slice: the first half of potrf_bwd_inv, callable ahead of time.
template <typename T>
dla_status potrf_inv_prepare(const Ctx& c, int64_t batch, int64_t n, MatB<const T> l, bool lower, MatB<T> wi, T* tmp) {
  if (use_trtri128<T>(n)) return trtri128(c, batch, 128, 128, as_d(l), !lower, as_d(wi), false);
  return trtri_levels<T>(c, batch, n, wi, tmp, &l, !lower);
}

// The second half: Abar from Lbar, L and the prepared wi = L^{-1}; tt is n^2
// scratch per slice.
// P' = tril(L^T Lbar) with a halved diagonal into tt (needs L and Lbar only).
template <typename T>
dla_status potrf_bwd_phi(const Ctx& c, int64_t batch, int64_t n, MatB<const T> lbar, MatB<const T> l, bool lower,
                         MatB<T> tt) {
  // Upper variant: L = R^T, Lbar = Rbar^T (dl/adjoints.hpp:183-188 is the
  // transposed composition); the result is symmetric, so no final transpose.
  // P = tril(L^T Lbar): op(A) = L^T (upper), op(B) = tril(Lbar); then halve
  // its diagonal so that Phi = copyltu(P) = P' + P'^T exactly.
  DLAB_TRY(gemm<T>(c, batch, n, n, n, T(1), l, lower, lbar, !lower, T(0), tt, MASK_LOWER, nullptr, TRI_UPPER,
                   TRI_LOWER));
  return ew_scale_diag<T>(c, batch, n, tt, T(0.5));
}

// The rest once wi = L^{-1} is ready: tt holds P' on entry.
template <typename T>
dla_status potrf_bwd_finish(const Ctx& c, int64_t batch, int64_t n, MatB<T> abar, MatB<const T> wi, MatB<T> tt) {
  // W = P' L^{-1}: lower x lower = lower  (into abar; lbar is no longer read,
  // so abar may alias it)
  DLAB_TRY(gemm<T>(c, batch, n, n, n, T(1), C_(tt), false, wi, false, T(0), abar, MASK_LOWER, nullptr, TRI_LOWER,
                   TRI_LOWER));
  // Z = L^{-T} W  (upper x lower, full);  L^-T Phi L^-1 = Z + Z^T
  DLAB_TRY(gemm<T>(c, batch, n, n, n, T(1), wi, true, C_(abar), false, T(0), tt, MASK_FULL, nullptr, TRI_UPPER,
                   TRI_LOWER));
  // Abar = 1/2 (Z + Z^T), bit-symmetric
  return ew_add_transpose<T>(c, batch, n, C_(tt), abar, T(0.5));
}

// potrf_bwd_finish without the final symmetrization: Z = L^-T P' L^-1 stays
// in tt (Abar = 1/2 (Z + Z^T) is formed by the caller's consumer; abar is
// clobbered as scratch for W).
template <typename T>
dla_status potrf_bwd_finish_z(const Ctx& c, int64_t batch, int64_t n, MatB<T> abar, MatB<const T> wi, MatB<T> tt) {
  DLAB_TRY(gemm<T>(c, batch, n, n, n, T(1), C_(tt), false, wi, false, T(0), abar, MASK_LOWER, nullptr, TRI_LOWER,
                   TRI_LOWER));
  return gemm<T>(c, batch, n, n, n, T(1), wi, true, C_(abar), false, T(0), tt, MASK_FULL, nullptr, TRI_UPPER,
                 TRI_LOWER);
}

template <typename T>
dla_status potrf_bwd_from_inv(const Ctx& c, int64_t batch, int64_t n, MatB<T> abar, MatB<const T> lbar, MatB<const T> l,
                              bool lower, MatB<const T> wi, MatB<T> tt) {
  DLAB_TRY(potrf_bwd_phi<T>(c, batch, n, lbar, l, lower, tt));
  return potrf_bwd_finish<T>(c, batch, n, abar, wi, tt);
}

template <typename T>
dla_status potrf_bwd_inv(const Ctx& c, int64_t batch, int64_t n, MatB<T> abar, MatB<const T> lbar, MatB<const T> l,
                         bool lower) {
  const int64_t N = inv_pad<T>(n);  // == n unless the inverse is padded
  DLAB_SCRATCH(ws, c, potrf_bwd_inv_scratch<T>(batch, n));
  T* wp = ws.as<T>();
  MatB<T> wi{wp, N, N * N};                  // L^{-1} (lower; the leading n x n block when padded)
  MatB<T> tt{wp + batch * N * N, n, n * n};  // Phi, then the lower half of L^-T Phi L^-1
  T* tmp = wp + batch * (N * N + n * n);
  // L^-1 (trtri) and P' = tril(L^T Lbar) are independent: the inverse runs
  // on a side stream (event fork/join: stream-ordered, graph-capturable)
  // while P' runs on the caller's stream.  The side stream and events belong
  // to this (device, caller stream); the join runs even when a launch fails.
  ForkRes& fr = fork_res(FORK_BWDINV, c.stream);
  std::lock_guard<std::mutex> lk(fr.mu);
  // the inverse is the longer, latency-bound branch (a chain of level
  // launches) and gates W: its stream gets the high priority so P' fills in
  // around it (DLA_BWDINV_PRIO=0: the low-priority side stream)
  static const bool hi = [] {
    const char* e = getenv("DLA_BWDINV_PRIO");
    return e ? atoi(e) != 0 : true;
  }();
  cudaStream_t inv_stream = hi ? fr.crit : fr.side;
  Ctx sc = c;
  sc.stream = inv_stream;
  cudaEventRecord(fr.ev[0], c.stream);
  cudaStreamWaitEvent(inv_stream, fr.ev[0], 0);
  dla_status s1;
  if (N == n) {
    s1 = potrf_inv_prepare<T>(sc, batch, n, l, lower, wi, tmp);
  } else if (use_trtri128<T>(N)) {  // 64 < n < 128: the padded inverse in one launch
    s1 = trtri128(sc, batch, (int)n, 128, as_d(l), !lower, as_d(wi), false);
  } else {
    s1 = ew_tri_copy<T>(sc, batch, n, l, wi, !lower);
    if (s1 == DLA_OK) {
      const unsigned gx = (unsigned)((N + 255) / 256);
      const unsigned gy = (unsigned)std::min<int64_t>(std::max<int64_t>(1, (148 * 16) / gx), batch * N);
      k_pad_eye<T><<<dim3(gx, gy), 256, 0, sc.stream>>>(batch, n, N, wi);
      s1 = cudaGetLastError() == cudaSuccess ? DLA_OK : DLA_ERR_CUDA;
    }
    if (s1 == DLA_OK) s1 = trtri_levels<T>(sc, batch, N, wi, tmp);
  }
  cudaEventRecord(fr.ev[1], inv_stream);
  const dla_status s2 = potrf_bwd_phi<T>(c, batch, n, lbar, l, lower, tt);
  cudaStreamWaitEvent(c.stream, fr.ev[1], 0);
  if (s1 != DLA_OK) return s1;
  if (s2 != DLA_OK) return s2;
  return potrf_bwd_finish<T>(c, batch, n, abar, C_(wi), tt);
}

// X <- alpha op(T) X / alpha X op(T) as ONE triangular GEMM into scratch plus
// a copy back (dl/blas.hpp:202-291 semantics; only the `lower`-selected
// triangle of T is read).
template <typename T>
dla_status trmm_gemm(const Ctx& c, int64_t batch, int64_t m, int64_t n, MatB<const T> t, MatB<T> x, bool right,
                     bool trans, bool lower, T alpha) {
  if (sizeof(T) == 8 && !right && m <= 128) {
    // X <- op(T) X in place: with one 128-row tile per column block every CTA
    // reads the whole of its X columns (the K range) before writing them, and
    // no other CTA reads those columns -- no scratch copy back
    Ctx cr = c;
    cr.gemm_rowtile = 1;
    const int tri = (lower != trans) ? TRI_LOWER : TRI_UPPER;
    return gemm<T>(cr, batch, m, n, m, alpha, t, trans, C_(x), false, T(0), x, MASK_FULL, c.info, tri, TRI_NONE);
  }
  DLAB_SCRATCH(ws, c, sizeof(T) * (size_t)batch * (size_t)m * n);
  MatB<T> y{ws.as<T>(), n, m * n};
  const int tri = (lower != trans) ? TRI_LOWER : TRI_UPPER;  // op(T)
  if (!right)
    DLAB_TRY(gemm<T>(c, batch, m, n, m, alpha, t, trans, C_(x), false, T(0), y, MASK_FULL, c.info, tri, TRI_NONE));
  else
    DLAB_TRY(gemm<T>(c, batch, m, n, n, alpha, C_(x), false, t, trans, T(0), y, MASK_FULL, c.info, TRI_NONE, tri));
  return ew_copy<T>(c, batch, m, n, C_(y), x, c.info);
}

// out-of-place fused potri (64 < n <= 128, fp64): b = inv(L L^T) from l
dla_status potri128_into(const Ctx& c, int64_t batch, int64_t n, MatB<const double> l, bool from_upper,
                         MatB<double> b) {
  return trtri128(c, batch, (int)n, (int)n, l, from_upper, b, true);
}

// potri of 64 < n <= 128 (fp64) as one fused launch (k_trtri128<., LAUUM>)
template <typename T>
bool potri_fused_eligible(int64_t n) {
  return n > 64 && n <= 128 && use_trtri128<T>(128);
}

// potri (lower) via the level-batched inverse: W = L^{-1}, B = W^T W on the
// lower triangle, mirrored exactly (dl/cholesky.hpp:141-147).  The caller has
// checked the diagonal for exact zeros.
template <typename T>
dla_status potri_inv(const Ctx& c, int64_t batch, int64_t n, MatB<T> a) {
  if (potri_fused_eligible<T>(n))  // one launch, in place
    return trtri128(c, batch, (int)n, (int)n, as_d(MatB<const T>{a.p, a.ld, a.bs, a.bsi}), false, as_d(a), true);
  DLAB_SCRATCH(ws, c, potri_inv_scratch<T>(batch, n));
  MatB<T> b{ws.as<T>(), n, n * n};
  T* tmp = ws.as<T>() + batch * n * n;
  DLAB_TRY(ew_square<T>(c, batch, n, a, /*tril*/ 0, T(1), c.info));  // the ignored triangle may hold anything
  DLAB_TRY(trtri_levels<T>(c, batch, n, a, tmp));
  DLAB_TRY(gemm<T>(c, batch, n, n, n, T(1), C_(a), true, C_(a), false, T(0), b, MASK_LOWER, c.info, TRI_UPPER,
                   TRI_LOWER));
  return ew_sym_lower_into<T>(c, batch, n, C_(b), a, T(1));
}

#define INST(T)                                                                                              \
  template dla_status trmm_gemm<T>(const Ctx&, int64_t, int64_t, int64_t, MatB<const T>, MatB<T>, bool, bool, \
                                   bool, T);                                                                 \
  template dla_status potri_inv<T>(const Ctx&, int64_t, int64_t, MatB<T>);                                   \
  template size_t ws_trsm_inv_from<T>(int64_t, int64_t, int64_t, bool);                                      \
  template dla_status trsm_inv_from<T>(const Ctx&, int64_t, int64_t, int64_t, MatB<const T>, MatB<const T>,  \
                                       MatB<T>, bool, bool, bool, T);                                        \
  template bool potri_fused_eligible<T>(int64_t);                                                            \
  template bool inv_eligible<T>(int64_t);                                                                    \
  template int64_t inv_pad<T>(int64_t);                                                                      \
  template size_t trtri_levels_tmp<T>(int64_t);                                                              \
  template size_t ws_trtri_levels<T>(int64_t, int64_t);                                                      \
  template size_t ws_trsm_inv<T>(int64_t, int64_t, int64_t, bool);                                           \
  template size_t ws_potrf_inv_prepare<T>(int64_t, int64_t);                                                 \
  template size_t ws_potrf_bwd_tail<T>(int64_t, int64_t);                                                    \
  template size_t ws_potrf_bwd_inv<T>(int64_t, int64_t);                                                     \
  template size_t ws_trmm_gemm<T>(int64_t, int64_t, int64_t, bool);                                          \
  template size_t ws_potri_inv<T>(int64_t, int64_t);                                                         \
  template dla_status trtri_levels<T>(const Ctx&, int64_t, int64_t, MatB<T>, T*, const MatB<const T>*, bool);                            \
  template dla_status trsm_inv<T>(const Ctx&, int64_t, int64_t, int64_t, MatB<const T>, MatB<T>, bool, bool, \
                                  bool, T);                                                                  \
  template dla_status potrf_bwd_inv<T>(const Ctx&, int64_t, int64_t, MatB<T>, MatB<const T>, MatB<const T>, bool); \
  template dla_status potrf_inv_prepare<T>(const Ctx&, int64_t, int64_t, MatB<const T>, bool, MatB<T>, T*);      \
  template dla_status potrf_bwd_from_inv<T>(const Ctx&, int64_t, int64_t, MatB<T>, MatB<const T>, MatB<const T>, \
                                            bool, MatB<const T>, MatB<T>);                                         \
  template dla_status potrf_bwd_phi<T>(const Ctx&, int64_t, int64_t, MatB<const T>, MatB<const T>, bool, MatB<T>); \
  template dla_status potrf_bwd_finish<T>(const Ctx&, int64_t, int64_t, MatB<T>, MatB<const T>, MatB<T>);        \
  template dla_status potrf_bwd_finish_z<T>(const Ctx&, int64_t, int64_t, MatB<T>, MatB<const T>, MatB<T>);
INST(double)
INST(float)

}  // namespace dlab
