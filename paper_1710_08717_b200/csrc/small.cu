// Fused small-matrix kernels (n <= 64): one warp (n <= 32) or one CTA per
// matrix, the whole
// operator chain in shared memory, one HBM read of each input and one write
// of each output.  This is the batched small-n regime of the north star
// (C1: batch 64 x 32^2; any batch x n <= 64).
//
//   potrf fwd : symmetry precheck (dl/cholesky.hpp:19-25) + Cholesky
//               (dl/cholesky.hpp:35-72) + tril / transpose (:71, :85-86).
//   potrf bwd : Abar = 1/2 sym(L^-T copyltu(L^T Lbar) L^-1)
//               (dl/adjoints.hpp:175-191), upper variant by transposition.
#include "chol64.cuh"
#include "common.cuh"
#include "ops.cuh"

namespace dlab {
namespace {

constexpr int SN = 64;
constexpr int SLD = SN + 1;

template <typename T>
__device__ T block_max(T v, T* red) {
  for (int o = 16; o; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) red[w] = v;
  __syncthreads();
  T r = red[0];
  for (int k = 1; k < (int)(blockDim.x >> 5); ++k) r = fmax(r, red[k]);
  return r;
}

template <typename T>
__global__ void __launch_bounds__(256) k_potrf_small(int n, MatB<T> a, bool lower, int32_t* info) {
  __shared__ T S[SN * SLD];
  __shared__ T red[8];
  __shared__ int flag;
  static_assert(SLD == CH_LD, "shared layout");
  const int64_t b = blockIdx.x;
  for (int e = threadIdx.x; e < n * n; e += blockDim.x) S[(e / n) * SLD + e % n] = *a.at(b, e / n, e % n);
  __syncthreads();
  // symmetry precheck: max|a_ij - a_ji| <= rtol * max|a|  (NaN ignored as in max_abs)
  T mabs = T(0), masym = T(0);
  for (int e = threadIdx.x; e < n * n; e += blockDim.x) {
    const int i = e / n, j = e % n;
    const T v = S[i * SLD + j];
    if (fabs(v) > mabs) mabs = fabs(v);
    if (j > i) {
      const T d = fabs(v - S[j * SLD + i]);
      if (d > masym) masym = d;
    }
  }
  mabs = block_max(mabs, red);
  masym = block_max(masym, red);
  if (masym > Num<T>::sym_rtol * (mabs > T(0) ? mabs : T(1))) {
    if (threadIdx.x == 0) record_failure(info, b, DLA_ERR_ASYMMETRIC, 0);
    return;
  }
  const int failed = chol_smem64<T>(S, n, &flag);
  if (failed >= 0) {
    if (threadIdx.x == 0) record_failure(info, b, DLA_ERR_NOT_SPD, failed);
    return;
  }
  for (int e = threadIdx.x; e < n * n; e += blockDim.x) {
    const int i = e / n, j = e % n;
    T v;
    if (lower) v = j <= i ? S[i * SLD + j] : T(0);
    else v = i <= j ? S[j * SLD + i] : T(0);
    *a.at(b, i, j) = v;
  }
}

template <typename T>
__global__ void __launch_bounds__(256) k_potrf_bwd_small(int n, MatB<T> abar, MatB<const T> lbar, MatB<const T> l,
                                                         bool lower) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T* L = reinterpret_cast<T*>(smem_raw);
  T* G = L + SN * SLD;  // Lbar (lower view)
  T* W = G + SN * SLD;
  const int64_t b = blockIdx.x;
  // Upper variant: L = R^T, Lbar = Rbar^T (dl/adjoints.hpp:183-188 is the
  // transpose of the lower composition).
  for (int e = threadIdx.x; e < n * n; e += blockDim.x) {
    const int i = e / n, j = e % n;
    T lv = lower ? *l.at(b, i, j) : *l.at(b, j, i);
    T gv = lower ? *lbar.at(b, i, j) : *lbar.at(b, j, i);
    L[i * SLD + j] = j <= i ? lv : T(0);
    G[i * SLD + j] = gv;
  }
  __syncthreads();
  // Phi = copyltu(L^T Lbar): Phi_ij (i >= j) = sum_{k >= i} L_ki Lbar_kj
  for (int e = threadIdx.x; e < n * n; e += blockDim.x) {
    const int i = e / n, j = e % n;
    if (j > i) continue;
    T acc = T(0);
    for (int k = i; k < n; ++k) acc += L[k * SLD + i] * G[k * SLD + j];
    W[i * SLD + j] = acc;
    W[j * SLD + i] = acc;
  }
  __syncthreads();
  // X = L^{-T} Phi: back substitution per column
  for (int j = threadIdx.x; j < n; j += blockDim.x) {
    for (int i = n - 1; i >= 0; --i) {
      T acc = W[i * SLD + j];
      for (int k = i + 1; k < n; ++k) acc -= L[k * SLD + i] * W[k * SLD + j];
      W[i * SLD + j] = acc / L[i * SLD + i];
    }
  }
  __syncthreads();
  // Y = X L^{-1}: per row, y_k = (x_k - sum_{j>k} y_j L_jk) / L_kk, k descending
  for (int r = threadIdx.x; r < n; r += blockDim.x) {
    T* wr = W + r * SLD;
    for (int k = n - 1; k >= 0; --k) {
      T acc = wr[k];
      for (int j = k + 1; j < n; ++j) acc -= wr[j] * L[j * SLD + k];
      wr[k] = acc / L[k * SLD + k];
    }
  }
  __syncthreads();
  // Abar = sym(Y / 2), exactly symmetric
  for (int e = threadIdx.x; e < n * n; e += blockDim.x) {
    const int i = e / n, j = e % n;
    const T hi = W[i * SLD + j] * T(0.5), hj = W[j * SLD + i] * T(0.5);
    *abar.at(b, i, j) = (i == j) ? hi : (hi + hj) / T(2);
  }
}

// ----------------------------------------------------------- n <= 32: a warp
// per matrix.  4-8 matrices per CTA, no block barriers: each warp loads its
// matrix with coalesced 32-lane sweeps into a private shared tile and holds
// one row (forward) or one column (backward) per lane in registers.  Values
// every lane needs (a column's multipliers, rows of L) are broadcast from
// shared memory with 16-byte loads: at 65536 matrices the kernels are bound
// by shared-memory instruction issue, and one LDS.128 carries 2 doubles where
// a 64-bit shuffle costs two SHFLs per value.
constexpr int WN = 32;
constexpr int WLD = WN + 1;  // column-per-lane tiles: conflict-free rows and columns

// warps (matrices) per CTA: keeps the per-CTA tile within 70 KB
template <typename T>
constexpr int wpc_fwd() { return 8; }
template <typename T>
constexpr int wpc_bwd() { return sizeof(T) == 8 ? 4 : 8; }

template <typename T>
__device__ __forceinline__ T warp_max(T v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// NFIX = 32: n is the compile-time constant 32 (every `i < n` guard of the
// unrolled register code folds away: ~1/3 fewer instructions); 0: runtime n.
template <typename T, int MINB, int NFIX>
__global__ void __launch_bounds__(256, MINB) k_potrf_warp(int n_, int64_t batch, MatB<T> a, bool lower,
                                                          int32_t* info) {
  const int n = NFIX > 0 ? NFIX : n_;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t b = (int64_t)blockIdx.x * wpc_fwd<T>() + warp;
  if (b >= batch) return;
  T* S = reinterpret_cast<T*>(smem_raw) + warp * (WN * WLD + 2 * WN + 4);
  T* buf = S + WN * WLD;  // 16-byte aligned: (WN * WLD) and the per-warp stride are multiples of 16 bytes
  const T* g = a.at(b, 0, 0);
  const int ld = (int)a.ld;  // 32-bit in-matrix offsets (64-bit only for the slice base)
  {
    T v[WN];  // all rows in flight at once, one coalesced row per load
#pragma unroll
    for (int i = 0; i < WN; ++i) v[i] = (i < n && lane < n) ? g[i * ld + lane] : T(0);
#pragma unroll
    for (int i = 0; i < WN; ++i)
      if (i < n) S[i * WLD + lane] = v[i];
  }
  __syncwarp();
  // symmetry precheck (same rule as k_potrf_small): row `lane` against column `lane`
  T mabs = T(0), masym = T(0);
  if (lane < n)
    for (int j = 0; j < n; ++j) {
      const T v = S[lane * WLD + j];
      if (fabs(v) > mabs) mabs = fabs(v);
      if (j > lane) {
        const T d = fabs(v - S[j * WLD + lane]);
        if (d > masym) masym = d;
      }
    }
  mabs = warp_max(mabs);
  masym = warp_max(masym);
  if (masym > Num<T>::sym_rtol * (mabs > T(0) ? mabs : T(1))) {
    if (lane == 0) record_failure(info, b, DLA_ERR_ASYMMETRIC, 0);
    return;
  }
  // row `lane` of the lower triangle; rows >= n factor an identity block
  T r[WN];
#pragma unroll
  for (int c = 0; c < WN; ++c) r[c] = (lane < n && c <= lane) ? S[lane * WLD + c] : (c == lane ? T(1) : T(0));
  int failed = -1;
  // L's row `lane` lands in S's row `lane` column by column (no other lane
  // reads S until the __syncwarp below)
  wchol_col<T, 0>(r, lane, n, buf, failed, r[0], S + lane * WLD);
  if (failed >= 0) {
    if (lane == 0) record_failure(info, b, DLA_ERR_NOT_SPD, failed);
    return;
  }
  T* o = a.at(b, 0, 0);
  // opaque copies of the slice base and row stride: otherwise the compiler
  // keeps the 32 row offsets of the initial load sweep alive (spilled) for
  // these stores
  asm volatile("mov.b64 %0, %0;" : "+l"(o));
  int ldo = ld;
  asm volatile("mov.b32 %0, %0;" : "+r"(ldo));
  if (!lower) {  // R(i, lane) = L(lane, i): this lane's own row of S
#pragma unroll
    for (int i = 0; i < WN; ++i)
      if (i < n && lane < n) o[i * ldo + lane] = i <= lane ? S[lane * WLD + i] : T(0);
    return;
  }
  __syncwarp();
#pragma unroll
  for (int i = 0; i < WN; ++i)
    if (i < n && lane < n) o[i * ldo + lane] = lane <= i ? S[i * WLD + lane] : T(0);
}

// Column `lane` of L^{-T} M held in registers, in unit-diagonal form: the
// caller has already scaled x by D^{-1} (x_i = m_i / L_ii, off the chain) and
// Ls holds L with every column divided by its diagonal, so
// x_m -= Ls(i, m) x_i for m < i, rows i descending, is the whole back
// substitution — one FMA per row on the serial chain, and row i of Ls is one
// broadcast sweep.
template <typename T>
__device__ __forceinline__ void warp_ltinv_col(const T* Ls, T (&x)[WN], int n) {
  constexpr int VN = Bc<T>::N, LLD = Bc<T>::LLD;
#pragma unroll
  for (int i = WN - 1; i >= 1; --i) {
    if (i < n) {
      const T xi = x[i];
#pragma unroll
      for (int m0 = 0; m0 < i; m0 += VN) {
        T v[VN];
        Bc<T>::ld(Ls + i * LLD + m0, v);
#pragma unroll
        for (int u = 0; u < VN; ++u)
          if (m0 + u < i) x[m0 + u] -= v[u] * xi;
      }
    }
  }
}

// Murray backward of one n <= 32 factor held by a warp, from shared memory:
// L = unit-diagonal L D^{-1} (LLD rows), dg / rd = D / D^{-1}, W = Lbar
// (column `lane` per lane; only its lower triangle is used).  Writes
// Abar = 1/2 sym(L^-T copyltu(L^T Lbar) L^-1) to o (dl/adjoints.hpp:175-191).
template <typename T>
__device__ __forceinline__ void warp_potrf_bwd_core(int n, int lane, const T* L, T* W, const T* dg, const T* rd, T* o,
                                                    int ldo, bool store = true) {
  constexpr int VN = Bc<T>::N, LLD = Bc<T>::LLD;
  // Phi = copyltu(L^T Lbar), lower part of column `lane`: Phi_ij = sum_{k>=i} L_ki Lbar_kj
  // (i >= j = lane) = L_ii (Lbar_ij + sum_{k>i} Ls_ki Lbar_kj), accumulated row by row of Ls
  T acc[WN];
#pragma unroll
  for (int i = 0; i < WN; ++i) acc[i] = T(0);
#pragma unroll
  for (int k = 0; k < WN; ++k) {
    if (k < n) {
      const T xk = lane < n ? W[k * WLD + lane] : T(0);
      acc[k] += xk;  // unit diagonal
#pragma unroll
      for (int i0 = 0; i0 < k; i0 += VN) {
        T v[VN];
        Bc<T>::ld(L + k * LLD + i0, v);
#pragma unroll
        for (int u = 0; u < VN; ++u)
          if (i0 + u < k) acc[i0 + u] += v[u] * xk;
      }
    }
  }
  __syncwarp();
  // mirror into W: W(i, j) = W(j, i) = Phi_ij
#pragma unroll
  for (int i = 0; i < WN; ++i)
    if (i < n && lane < n && i >= lane) {
      const T p = acc[i] * dg[i];
      W[i * WLD + lane] = p;
      W[lane * WLD + i] = p;
    }
  __syncwarp();
  T x[WN];
#pragma unroll
  for (int i = 0; i < WN; ++i) x[i] = (i < n && lane < n) ? W[i * WLD + lane] * rd[i] : T(0);
  // X = L^{-T} Phi (column `lane`), then through shared memory X^T = Phi L^{-1}
  warp_ltinv_col<T>(L, x, n);
  __syncwarp();
#pragma unroll
  for (int i = 0; i < WN; ++i)
    if (i < n && lane < n) W[i * WLD + lane] = x[i];
  __syncwarp();
#pragma unroll
  for (int i = 0; i < WN; ++i) x[i] = (i < n && lane < n) ? W[lane * WLD + i] * rd[i] : T(0);
  // Y = L^{-T} (Phi L^{-1}) = L^{-T} Phi L^{-1}; column `lane`
  warp_ltinv_col<T>(L, x, n);
  __syncwarp();
#pragma unroll
  for (int i = 0; i < WN; ++i)
    if (i < n && lane < n) W[i * WLD + lane] = x[i];
  __syncwarp();
  // Abar = sym(Y / 2), exactly symmetric: element (i, lane) pairs this lane's
  // Y(i, lane) with Y(lane, i) from shared memory
#pragma unroll
  for (int i = 0; i < WN; ++i)
    if (i < n && lane < n) {
      const T hi = x[i] * T(0.5), hj = W[lane * WLD + i] * T(0.5);
      if (store) o[i * ldo + lane] = (i == lane) ? hi : (hi + hj) * T(0.5);  // == (hi + hj) / 2 exactly
    }
}

template <typename T, int NFIX>
__global__ void __launch_bounds__(wpc_bwd<T>() * 32, sizeof(T) == 8 ? 3 : 2) k_potrf_bwd_warp(int n_, int64_t batch,
                                                                                      MatB<T> abar,
                                                                                      MatB<const T> lbar,
                                                                                      MatB<const T> l, bool lower) {
  const int n = NFIX > 0 ? NFIX : n_;
  constexpr int VN = Bc<T>::N, LLD = Bc<T>::LLD;
  constexpr int per_warp = WN * LLD + WN * WLD + 2 * WN + 4;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t b = (int64_t)blockIdx.x * wpc_bwd<T>() + warp;
  if (b >= batch) return;
  T* L = reinterpret_cast<T*>(smem_raw) + warp * per_warp;  // 16-byte aligned (per_warp * sizeof(T) % 16 == 0)
  T* W = L + WN * LLD;
  T* rd = W + WN * WLD;
  // lower views: L = R^T, Lbar = Rbar^T for the upper variant (dl/adjoints.hpp:183-188)
  const T* gl = l.at(b, 0, 0);
  const T* gg = lbar.at(b, 0, 0);
  const int ldl = (int)l.ld, ldg = (int)lbar.ld, ldo = (int)abar.ld;  // 32-bit in-matrix offsets
  // Unit-diagonal form: Ls = L D^{-1} (column j divided by L_jj, unit
  // diagonal), scaled on the way into shared memory; dg / rd keep D and D^{-1}.
  T* dg = rd + WN;
  {
    const T d = lane < n ? gl[lane * ldl + lane] : T(1);
    dg[lane] = d;
    rd[lane] = T(1) / d;
  }
  __syncwarp();
  const T r_own = rd[lane];
#pragma unroll
  for (int i0 = 0; i0 < WN; i0 += 16) {  // 32 coalesced row loads in flight per lane
    T lv[16], gv[16];
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      const int i = i0 + u;
      lv[u] = (i < n && lane < n) ? gl[i * ldl + lane] : T(0);
      gv[u] = (i < n && lane < n) ? gg[i * ldg + lane] : T(0);
    }
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      const int i = i0 + u;
      if (i < n) {
        if (lower) {  // element (i, lane) of L, column `lane`
          L[i * LLD + lane] = lane < i ? lv[u] * r_own : (lane == i ? T(1) : T(0));
          W[i * WLD + lane] = gv[u];
        } else {  // element (lane, i) of the lower view, column i
          L[lane * LLD + i] = i < lane ? lv[u] * rd[i] : (i == lane ? T(1) : T(0));
          W[lane * WLD + i] = gv[u];
        }
      }
    }
  }
  __syncwarp();
  warp_potrf_bwd_core<T>(n, lane, L, W, dg, rd, abar.at(b, 0, 0), ldo);
}


// ---------------------------------------------- n <= 32, fp64, on FP64 DMMA
// The same pullback as warp_potrf_bwd_core, Abar = 1/2 sym(L^-T Phi L^-1),
// Phi = copyltu(L^T Lbar) (dl/adjoints.hpp:175-191), with every product a
// warp-level m8n8k4 DMMA over 8 x 8 tiles and L^-1 formed explicitly (8 x 8
// diagonal inverses, one column per lane, then two doubling levels):
//   P = tril(L^T Lbar) (10 lower tiles), Phi -> G;  Linv -> Lm (in place);
//   X = Linv^T Phi;  Y = X Linv -> G;  Abar = 1/2 sym(Y).
// ~240 DMMAs replace ~3000 FMA / broadcast-load instructions of the
// substitution form: the batched n = 32 pullback is issue-bound, not
// FP64-bound.  Row stride DLD = 36 (= 4 mod 16): both fragment orientations
// (k along rows and k along columns) load conflict-free.
constexpr int DLD = 36;
constexpr int DBUF = WN * DLD;  // one 32 x 32 buffer
constexpr int TLD = 20;         // the doubling levels' T1 scratch (16 x 16 at most; = 4 mod 16)
constexpr int TBUF = 16 * TLD;

__device__ __forceinline__ void dmma8(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

// Lm: L (lower, strict upper zero, identity beyond n); G: tril(Lbar) (zero
// beyond n), reused for Phi, X and Y; X: TBUF scratch for the doubling
// levels.  Writes Abar's n x n block to o (row stride ldo).
__device__ __forceinline__ void warp_potrf_bwd_dmma(int n, int lane, double* Lm, double* G, double* X, double* o,
                                                    int ldo, bool store) {
  const int fr = lane >> 2, fc = lane & 3;
  // (1) P = tril(L^T Lbar): tile (I, J), I >= J, k >= 8 I
  {
    double p[10][2];
#pragma unroll
    for (int t = 0; t < 10; ++t) p[t][0] = p[t][1] = 0.0;
#pragma unroll
    for (int s = 0; s < 8; ++s) {
      double bf[4];
#pragma unroll
      for (int J = 0; J < 4; ++J) bf[J] = G[(4 * s + fc) * DLD + 8 * J + fr];
#pragma unroll
      for (int I = 0; I < 4; ++I) {
        if (2 * I > s) continue;  // k = 4 s .. 4 s + 3 >= 8 I
        const double af = Lm[(4 * s + fc) * DLD + 8 * I + fr];  // (L^T)(8I + fr, k) = L(k, 8I + fr)
#pragma unroll
        for (int J = 0; J <= I; ++J) dmma8(p[I * (I + 1) / 2 + J][0], p[I * (I + 1) / 2 + J][1], af, bf[J]);
      }
    }
    __syncwarp();
    // Phi = copyltu(P) into G (mirrored)
#pragma unroll
    for (int I = 0; I < 4; ++I)
#pragma unroll
      for (int J = 0; J <= I; ++J)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int i = 8 * I + fr, j = 8 * J + 2 * fc + e;
          if (i >= j) {
            G[i * DLD + j] = p[I * (I + 1) / 2 + J][e];
            G[j * DLD + i] = p[I * (I + 1) / 2 + J][e];
          }
        }
  }
  // (2) Linv in place of L: 8 x 8 diagonal blocks (lane = block, column) ...
  {
    const int o8 = (lane >> 3) * 8, c = lane & 7;
    double x[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      double acc = i == c ? 1.0 : 0.0;
#pragma unroll
      for (int q = 0; q < i; ++q)
        if (q >= c) acc -= Lm[(o8 + i) * DLD + o8 + q] * x[q];
      x[i] = i >= c ? acc / Lm[(o8 + i) * DLD + o8 + i] : 0.0;
    }
    __syncwarp();
#pragma unroll
    for (int i = 0; i < 8; ++i)
      if (i >= c) Lm[(o8 + i) * DLD + o8 + c] = x[i];
    __syncwarp();
  }
  // ... then [A 0; B C] -> B = -C^{-1} (B A^{-1}) for s = 8 (two pairs), 16
#pragma unroll
  for (int s = 8; s < WN; s *= 2) {
    const int pairs = WN / (2 * s), tps = (s / 8) * (s / 8);
    double t1[4][2];
#pragma unroll
    for (int t = 0; t < 4; ++t) t1[t][0] = t1[t][1] = 0.0;
#pragma unroll
    for (int t = 0; t < pairs * tps; ++t) {  // T1 = B A^{-1}: k >= nt
      const int pr = t / tps, r = t % tps, rt = (r / (s / 8)) * 8, nt = (r % (s / 8)) * 8, o = 2 * s * pr;
#pragma unroll
      for (int kk = 0; kk < s; kk += 4) {
        if (kk < nt) continue;
        dmma8(t1[t][0], t1[t][1], Lm[(o + s + rt + fr) * DLD + o + kk + fc], Lm[(o + kk + fc) * DLD + o + nt + fr]);
      }
    }
#pragma unroll
    for (int t = 0; t < pairs * tps; ++t) {
      const int pr = t / tps, r = t % tps, rt = (r / (s / 8)) * 8, nt = (r % (s / 8)) * 8;
      X[(pr * s + rt + fr) * TLD + nt + 2 * fc] = t1[t][0];
      X[(pr * s + rt + fr) * TLD + nt + 2 * fc + 1] = t1[t][1];
    }
    __syncwarp();
    double bn[4][2];
#pragma unroll
    for (int t = 0; t < 4; ++t) bn[t][0] = bn[t][1] = 0.0;
#pragma unroll
    for (int t = 0; t < pairs * tps; ++t) {  // B = -C^{-1} T1: k <= rt + 7
      const int pr = t / tps, r = t % tps, rt = (r / (s / 8)) * 8, nt = (r % (s / 8)) * 8, o = 2 * s * pr;
#pragma unroll
      for (int kk = 0; kk < s; kk += 4) {
        if (kk >= rt + 8) continue;
        dmma8(bn[t][0], bn[t][1], Lm[(o + s + rt + fr) * DLD + o + s + kk + fc], X[(pr * s + kk + fc) * TLD + nt + fr]);
      }
    }
    __syncwarp();
#pragma unroll
    for (int t = 0; t < pairs * tps; ++t) {
      const int pr = t / tps, r = t % tps, rt = (r / (s / 8)) * 8, nt = (r % (s / 8)) * 8, o = 2 * s * pr;
      Lm[(o + s + rt + fr) * DLD + o + nt + 2 * fc] = -bn[t][0];
      Lm[(o + s + rt + fr) * DLD + o + nt + 2 * fc + 1] = -bn[t][1];
    }
    __syncwarp();
  }
  // (3) X = Linv^T Phi: k >= 8 I
  {
    double x[16][2];
#pragma unroll
    for (int t = 0; t < 16; ++t) x[t][0] = x[t][1] = 0.0;
#pragma unroll
    for (int s = 0; s < 8; ++s) {
      double bf[4];
#pragma unroll
      for (int J = 0; J < 4; ++J) bf[J] = G[(4 * s + fc) * DLD + 8 * J + fr];
#pragma unroll
      for (int I = 0; I < 4; ++I) {
        if (2 * I > s) continue;
        const double af = Lm[(4 * s + fc) * DLD + 8 * I + fr];  // Linv(k, 8I + fr)
#pragma unroll
        for (int J = 0; J < 4; ++J) dmma8(x[4 * I + J][0], x[4 * I + J][1], af, bf[J]);
      }
    }
    __syncwarp();  // Phi is dead: X replaces it in G
#pragma unroll
    for (int t = 0; t < 16; ++t) {
      const int i = 8 * (t / 4) + fr, j = 8 * (t % 4) + 2 * fc;
      G[i * DLD + j] = x[t][0];
      G[i * DLD + j + 1] = x[t][1];
    }
  }
  __syncwarp();
  // (4) Y = X Linv: k >= 8 J; Y replaces X in G
  {
    double y[16][2];
#pragma unroll
    for (int t = 0; t < 16; ++t) y[t][0] = y[t][1] = 0.0;
#pragma unroll
    for (int s = 0; s < 8; ++s) {
      double af[4];
#pragma unroll
      for (int I = 0; I < 4; ++I) af[I] = G[(8 * I + fr) * DLD + 4 * s + fc];
#pragma unroll
      for (int J = 0; J < 4; ++J) {
        if (2 * J > s) continue;
        const double bf = Lm[(4 * s + fc) * DLD + 8 * J + fr];
#pragma unroll
        for (int I = 0; I < 4; ++I) dmma8(y[4 * I + J][0], y[4 * I + J][1], af[I], bf);
      }
    }
    __syncwarp();
    // Y into G and Y^T into Lm (L^-1 is dead): the symmetrisation below then
    // reads rows of both (a column read of Y would be a 4-way bank conflict)
#pragma unroll
    for (int t = 0; t < 16; ++t) {
      const int i = 8 * (t / 4) + fr, j = 8 * (t % 4) + 2 * fc;
      G[i * DLD + j] = y[t][0];
      G[i * DLD + j + 1] = y[t][1];
      Lm[j * DLD + i] = y[t][0];
      Lm[(j + 1) * DLD + i] = y[t][1];
    }
  }
  __syncwarp();
  // (5) Abar = 1/2 sym(Y), exactly symmetric; column `lane`, coalesced rows
  if (store && lane < n) {
#pragma unroll 8
    for (int i = 0; i < WN; ++i) {
      if (i < n) {
        const double hi = G[i * DLD + lane] * 0.5, hj = Lm[i * DLD + lane] * 0.5;
        o[i * ldo + lane] = (i == lane) ? hi : (hi + hj) * 0.5;
      }
    }
  }
}

// Warp per matrix (BDW per CTA), fp64 n <= 32: loads L and tril(Lbar) (lower
// views of the upper variant), pads to 32, runs warp_potrf_bwd_dmma.  (A
// persistent variant prefetching the next matrix into registers measured
// slower: 234 registers, and the kernel is not HBM-latency bound.)
constexpr int BDW = 2;  // warps per CTA (42 KB): five CTAs per SM
template <bool LOWER, int NFIX>
__global__ void __launch_bounds__(BDW * 32) k_potrf_bwd_dmma(int n_, int64_t batch, MatB<double> abar,
                                                        MatB<const double> lbar, MatB<const double> l) {
  constexpr bool lower = LOWER;
  const int n = NFIX > 0 ? NFIX : n_;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t b = (int64_t)blockIdx.x * BDW + warp;
  if (b >= batch) return;
  double* Lm = reinterpret_cast<double*>(smem_raw) + warp * (2 * DBUF + TBUF);
  double* G = Lm + DBUF;
  double* X = G + DBUF;
  const double* gl = l.at(b, 0, 0);
  const double* gg = lbar.at(b, 0, 0);
  const int ldl = (int)l.ld, ldg = (int)lbar.ld;
#pragma unroll
  for (int i0 = 0; i0 < WN; i0 += 16) {
    double lv[16], gv[16];
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      const int i = i0 + u;
      lv[u] = (i < n && lane < n) ? gl[i * ldl + lane] : 0.0;
      gv[u] = (i < n && lane < n) ? gg[i * ldg + lane] : 0.0;
    }
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      const int i = i0 + u;
      if (lower) {  // element (i, lane)
        Lm[i * DLD + lane] = lane <= i ? (i < n ? lv[u] : (lane == i ? 1.0 : 0.0)) : 0.0;
        G[i * DLD + lane] = lane <= i ? gv[u] : 0.0;
      } else {      // R(i, lane) = L(lane, i), Rbar(i, lane) = Lbar(lane, i)
        Lm[lane * DLD + i] = i <= lane ? (lane < n ? lv[u] : (lane == i ? 1.0 : 0.0)) : 0.0;
        G[lane * DLD + i] = i <= lane ? gv[u] : 0.0;
      }
    }
  }
  __syncwarp();
  warp_potrf_bwd_dmma(n, lane, Lm, G, X, abar.at(b, 0, 0), (int)abar.ld, true);
}

// Fused Gaussian log-likelihood chain, one warp per matrix (n <= 32), the
// whole of BASELINE config C1 in one launch (dl/models.hpp:99-103 given A):
//   L = potrf(A) (dl/cholesky.hpp:35-72), z = L^-1 y (dl/blas.hpp:307-395),
//   phi = 1/2 z^T z + sum_i log L_ii (dl/tape.hpp:789-795)
// and its pullback at phibar = 1: zbar = z; S = L^-T zbar = ybar;
// Lbar = -tril(S z^T) + diag(1 / L_ii) (dl/adjoints.hpp:136-152,
// dl/tape.hpp:1038-1045); Abar = potrf pullback (warp_potrf_bwd_core).
// A and y are read once, Abar / ybar / phi written once.
template <typename T, int NFIX>
__global__ void __launch_bounds__(wpc_bwd<T>() * 32) k_chol_chain_warp(int n_, int64_t batch, MatB<const T> a,
                                                                       const T* y, T* phi, MatB<T> abar, T* ybar,
                                                                       int32_t* info) {
  const int n = NFIX > 0 ? NFIX : n_;
  constexpr int LLD = Bc<T>::LLD;
  constexpr int per_warp = WN * LLD + WN * WLD + 6 * WN;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // The warps of a CTA walk the chain's phases in lockstep (a barrier between
  // phases), so the SM fetches one code region at a time for all of them: the
  // chain is ~14 k straight-line instructions and independent warps each
  // streamed their own region through the instruction cache (ncu: stall
  // no_instruction).  Inactive / failed warps keep computing on a clamped
  // slice and only suppress their stores.
  const int64_t bw = (int64_t)blockIdx.x * wpc_bwd<T>() + warp;
  bool ok = bw < batch;
  const int64_t b = ok ? bw : batch - 1;
  T* L = reinterpret_cast<T*>(smem_raw) + warp * per_warp;  // unit-diagonal L D^-1 (LLD rows)
  T* W = L + WN * LLD;                                       // A, then L (rows), then Lbar (columns)
  T* buf = W + WN * WLD;
  T* dg = buf + 2 * WN;
  T* rd = dg + WN;
  T* sv = rd + WN;
  T* lg = sv + WN;
  const T* ga = a.at(b, 0, 0);
  const int ld = (int)a.ld;
  {
    T v[WN];
#pragma unroll
    for (int i = 0; i < WN; ++i) v[i] = (i < n && lane < n) ? ga[i * ld + lane] : T(0);
#pragma unroll
    for (int i = 0; i < WN; ++i)
      if (i < n) W[i * WLD + lane] = v[i];
  }
  T yv = lane < n ? y[b * n + lane] : T(0);
  __syncwarp();
  // symmetry precheck (dl/cholesky.hpp:19-25), as k_potrf_warp
  T mabs = T(0), masym = T(0);
  if (lane < n)
    for (int j = 0; j < n; ++j) {
      const T v = W[lane * WLD + j];
      if (fabs(v) > mabs) mabs = fabs(v);
      if (j > lane) {
        const T d = fabs(v - W[j * WLD + lane]);
        if (d > masym) masym = d;
      }
    }
  mabs = warp_max(mabs);
  masym = warp_max(masym);
  if (masym > Num<T>::sym_rtol * (mabs > T(0) ? mabs : T(1))) {
    if (lane == 0 && ok) record_failure(info, b, DLA_ERR_ASYMMETRIC, 0);
    ok = false;
  }
  __syncthreads();
  T r[WN];
#pragma unroll
  for (int c = 0; c < WN; ++c) r[c] = (lane < n && c <= lane) ? W[lane * WLD + c] : (c == lane ? T(1) : T(0));
  int failed = -1;
  wchol_col<T, 0>(r, lane, n, buf, failed, r[0]);
  if (failed >= 0) {
    if (lane == 0 && ok) record_failure(info, b, DLA_ERR_NOT_SPD, failed);
    ok = false;
  }
  __syncthreads();
#pragma unroll
  for (int c = 0; c < WN; ++c)
    if (c < n && lane < n) W[lane * WLD + c] = c <= lane ? r[c] : T(0);
  __syncwarp();
  const T d = lane < n ? W[lane * WLD + lane] : T(1);
  const T rinv = T(1) / d;
  dg[lane] = d;
  rd[lane] = rinv;
#pragma unroll
  for (int i = 0; i < WN; ++i)
    if (i < n) L[i * LLD + lane] = lane < i ? (lane < n ? W[i * WLD + lane] * rinv : T(0)) : (lane == i ? T(1) : T(0));
  // z = L^-1 y, column-oriented: z_j = y_j / L_jj moves by one shuffle
  T z = T(0);
#pragma unroll
  for (int j = 0; j < WN; ++j) {
    if (j < n) {
      const T zj = __shfl_sync(0xffffffffu, yv * rinv, j);
      if (lane == j) z = zj;
      if (lane > j) yv -= r[j] * zj;
    }
  }
  sv[lane] = lane < n ? z : T(0);
  lg[lane] = lane < n ? Num<T>::log_(d) : T(0);
  __syncwarp();
  if (lane == 0 && ok) {  // sequential i order, as the tape's Sum node
    T q = T(0), ldt = T(0);
    for (int i = 0; i < n; ++i) q += sv[i] * sv[i];
    for (int i = 0; i < n; ++i) ldt += lg[i];
    phi[b] = T(0.5) * q + ldt;
  }
  // S = L^-T z (zbar = z), row k of L read from W
  T zb = z, s_own = T(0);
#pragma unroll
  for (int k = WN - 1; k >= 0; --k) {
    if (k < n) {
      const T sk = __shfl_sync(0xffffffffu, zb * rinv, k);
      if (lane == k) s_own = sk;
      if (lane < k) zb -= W[k * WLD + lane] * sk;
    }
  }
  if (lane < n && ok) ybar[b * n + lane] = s_own;
  __syncthreads();
  sv[lane] = lane < n ? s_own : T(0);
  __syncwarp();
  // Lbar, column `lane`: -s_i z_lane (i >= lane) + 1 / L_ii on the diagonal
#pragma unroll
  for (int i = 0; i < WN; ++i)
    if (i < n) W[i * WLD + lane] = (i >= lane && lane < n) ? -sv[i] * z + (i == lane ? rinv : T(0)) : T(0);
  __syncthreads();
  warp_potrf_bwd_core<T>(n, lane, L, W, dg, rd, abar.at(b, 0, 0), (int)abar.ld, ok);
}
// fp64 C1 chain with the pullback on DMMA (warp_potrf_bwd_dmma): the
// forward (symmetry check, register Cholesky, z = L^-1 y, phi) and the
// vector pullbacks (S = L^-T z, Lbar = -tril(S z^T) + diag(1 / L_ii)) as in
// k_chol_chain_warp; then the potrf pullback on 8 x 8 DMMA tiles.  Two warps
// per CTA (2 x 9 KB buffers + 2.5 KB per warp), phases in lockstep as there.
constexpr int CDW = 2;  // warps per CTA
template <int NFIX>
__global__ void __launch_bounds__(CDW * 32) k_chol_chain_dmma(int n_, int64_t batch, MatB<const double> a,
                                                             const double* y, double* phi, MatB<double> abar,
                                                             double* ybar, int32_t* info) {
  using T = double;
  const int n = NFIX > 0 ? NFIX : n_;
  constexpr int per_warp = 2 * DBUF + TBUF + 6 * WN;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t bw = (int64_t)blockIdx.x * CDW + warp;
  bool ok = bw < batch;
  const int64_t b = ok ? bw : batch - 1;
  T* Lm = reinterpret_cast<T*>(smem_raw) + warp * per_warp;  // L (true), then L^-1
  T* G = Lm + DBUF;                                          // A, then Lbar / Phi / Y
  T* X = G + DBUF;
  T* buf = X + TBUF;
  T* rd = buf + 2 * WN;
  T* sv = rd + WN;
  T* lg = sv + WN;
  const T* ga = a.at(b, 0, 0);
  const int ld = (int)a.ld;
  {
    T v[WN];
#pragma unroll
    for (int i = 0; i < WN; ++i) v[i] = (i < n && lane < n) ? ga[i * ld + lane] : T(0);
#pragma unroll
    for (int i = 0; i < WN; ++i)
      if (i < n) G[i * DLD + lane] = v[i];
  }
  T yv = lane < n ? y[b * n + lane] : T(0);
  __syncwarp();
  // symmetry precheck (dl/cholesky.hpp:19-25), as k_potrf_warp
  T mabs = T(0), masym = T(0);
  if (lane < n)
    for (int j = 0; j < n; ++j) {
      const T v = G[lane * DLD + j];
      if (fabs(v) > mabs) mabs = fabs(v);
      if (j > lane) {
        const T d = fabs(v - G[j * DLD + lane]);
        if (d > masym) masym = d;
      }
    }
  mabs = warp_max(mabs);
  masym = warp_max(masym);
  if (masym > Num<T>::sym_rtol * (mabs > T(0) ? mabs : T(1))) {
    if (lane == 0 && ok) record_failure(info, b, DLA_ERR_ASYMMETRIC, 0);
    ok = false;
  }
  __syncthreads();
  T r[WN];
#pragma unroll
  for (int c = 0; c < WN; ++c) r[c] = (lane < n && c <= lane) ? G[lane * DLD + c] : (c == lane ? T(1) : T(0));
  int failed = -1;
  wchol_col<T, 0>(r, lane, n, buf, failed, r[0]);
  if (failed >= 0) {
    if (lane == 0 && ok) record_failure(info, b, DLA_ERR_NOT_SPD, failed);
    ok = false;
  }
  __syncthreads();
  // L (true, zero strict upper, identity beyond n) into Lm, row `lane`
#pragma unroll
  for (int c = 0; c < WN; ++c) Lm[lane * DLD + c] = c <= lane ? (lane < n ? r[c] : (c == lane ? T(1) : T(0))) : T(0);
  __syncwarp();
  const T d = Lm[lane * DLD + lane];  // (1 beyond n)
  const T rinv = T(1) / d;
  rd[lane] = rinv;
  // z = L^-1 y, column-oriented: z_j = y_j / L_jj moves by one shuffle
  T z = T(0);
#pragma unroll
  for (int j = 0; j < WN; ++j) {
    if (j < n) {
      const T zj = __shfl_sync(0xffffffffu, yv * rinv, j);
      if (lane == j) z = zj;
      if (lane > j) yv -= r[j] * zj;
    }
  }
  sv[lane] = lane < n ? z : T(0);
  lg[lane] = lane < n ? Num<T>::log_(d) : T(0);
  __syncwarp();
  if (lane == 0 && ok) {  // sequential i order, as the tape's Sum node
    T q = T(0), ldt = T(0);
    for (int i = 0; i < n; ++i) q += sv[i] * sv[i];
    for (int i = 0; i < n; ++i) ldt += lg[i];
    phi[b] = T(0.5) * q + ldt;
  }
  // S = L^-T z (zbar = z), row k of L from Lm
  T zb = z, s_own = T(0);
#pragma unroll
  for (int k = WN - 1; k >= 0; --k) {
    if (k < n) {
      const T sk = __shfl_sync(0xffffffffu, zb * rinv, k);
      if (lane == k) s_own = sk;
      if (lane < k) zb -= Lm[k * DLD + lane] * sk;
    }
  }
  if (lane < n && ok) ybar[b * n + lane] = s_own;
  __syncthreads();
  sv[lane] = lane < n ? s_own : T(0);
  __syncwarp();
  // Lbar, column `lane`: -s_i z_lane (i >= lane) + 1 / L_ii on the diagonal; zero beyond n
#pragma unroll
  for (int i = 0; i < WN; ++i)
    G[i * DLD + lane] = (i < n && i >= lane && lane < n) ? -sv[i] * z + (i == lane ? rinv : T(0)) : T(0);
  __syncthreads();
  warp_potrf_bwd_dmma(n, lane, Lm, G, X, abar.at(b, 0, 0), (int)abar.ld, ok);
}

// ------------------------------------------- 64 < n <= 128 (fp64): CTA per matrix
// The whole factorization of one matrix in ONE launch with its lower
// triangle in shared memory as three 64 x 64 blocks (A11, A21, A22: 100 KB,
// two CTAs per SM): symmetry precheck from the same read, A11 factored with
// the A21 solve interleaved (chol_tall64, the blocked panel kernel's leaf),
// A22 -= L21 L21^T on DMMA, A22 factored (chol_smem), L written once with its
// zero triangle.  Replaces check_symmetric's pass, two panel launches and
// the zeroing pass of the blocked path at these sizes.
constexpr int P2 = 128;
constexpr int P2LD = 65;
__device__ __forceinline__ int kcol16(int s, int fc) { return ((s & ~3) << 2) + 4 * fc + (s & 3); }
template <int MINB>
__global__ void __launch_bounds__(256, MINB) k_potrf128(int n, MatB<double> a, bool lower, int32_t* info,
                                                        bool check_sym) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double* S11 = reinterpret_cast<double*>(smem_raw);
  double* V = S11 + 64 * P2LD;
  double* S22 = V + 64 * P2LD;
  __shared__ double red[8];
  __shared__ int flag;
  const int64_t b = blockIdx.x;
  const int tid = threadIdx.x, nv = n - 64;
  double* g = a.at(b, 0, 0);
  const int64_t ld = a.ld;
  auto sm = [&](int i, int j) -> double* {
    return i < 64 ? S11 + i * P2LD + j : (j < 64 ? V + (i - 64) * P2LD + j : S22 + (i - 64) * P2LD + (j - 64));
  };
  // One read of A, bottom row pairs first, 16 loads in flight per thread:
  // the lower triangle goes to shared memory and each chunk's upper entries
  // are checked against their mirrors, which sit in rows already stored (the
  // symmetry precheck of dl/cholesky.hpp:19-25, as k_potrf_small).
  double mabs = 0.0, masym = 0.0;
  const int j = tid & 127;
  for (int c = P2 * P2 / 256 / 16 - 1; c >= 0; --c) {
    double v[16];
#pragma unroll
    for (int q = 0; q < 16; ++q) {
      const int i = 2 * (16 * c + q) + (tid >> 7);
      v[q] = (i < n && j < n && (check_sym || j <= i)) ? g[i * ld + j] : 0.0;
    }
#pragma unroll
    for (int q = 0; q < 16; ++q) {
      const int i = 2 * (16 * c + q) + (tid >> 7);
      if (j <= i) *sm(i, j) = v[q];
      if (fabs(v[q]) > mabs) mabs = fabs(v[q]);
    }
    __syncthreads();
#pragma unroll
    for (int q = 0; q < 16; ++q) {
      const int i = 2 * (16 * c + q) + (tid >> 7);
      if (check_sym && j > i && j < n) {
        const double d = fabs(v[q] - *sm(j, i));
        if (d > masym) masym = d;
      }
    }
  }
  mabs = block_max(mabs, red);
  masym = block_max(masym, red);
  if (masym > Num<double>::sym_rtol * (mabs > 0.0 ? mabs : 1.0)) {
    if (tid == 0) record_failure(info, b, DLA_ERR_ASYMMETRIC, 0);
    return;
  }
  // L11 and L21
  int failed = chol_tall64<P2LD>(S11, V, 64, nv, &flag, [](int) {});
  if (failed >= 0) {
    if (tid == 0) record_failure(info, b, DLA_ERR_NOT_SPD, failed);
    return;
  }
  // A22 -= L21 L21^T (lower 8 x 8 tiles, K = 64 on DMMA)
  {
    const int warp = tid >> 5, lane = tid & 31, fr = lane >> 2, fc = lane & 3;
    const int mt = (nv + 7) / 8, ntiles = mt * (mt + 1) / 2;
    for (int tile = warp; tile < ntiles; tile += 8) {
      int ta = 0;
      while ((ta + 1) * (ta + 2) / 2 <= tile) ++ta;
      const int tb = tile - ta * (ta + 1) / 2;
      double c0 = 0.0, c1 = 0.0;
#pragma unroll
      for (int q = 0; q < 16; ++q) {
        const int kc = kcol16(q, fc);
        const double af = V[(8 * ta + fr) * P2LD + kc];
        const double bf = V[(8 * tb + fr) * P2LD + kc];
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                     : "+d"(c0), "+d"(c1)
                     : "d"(af), "d"(bf));
      }
      double* crow = S22 + (8 * ta + fr) * P2LD + 8 * tb + 2 * fc;  // above-diagonal entries are scratch
      crow[0] -= c0;
      crow[1] -= c1;
    }
  }
  __syncthreads();
  failed = chol_smem<double, 64>(S22, nv, &flag);
  if (failed >= 0) {
    if (tid == 0) record_failure(info, b, DLA_ERR_NOT_SPD, 64 + failed);
    return;
  }
  // L (or R = L^T) with its zero triangle, coalesced rows
  if (j < n) {
#pragma unroll 8
    for (int u = 0; u < P2 * P2 / 256; ++u) {
      const int i = 2 * u + (tid >> 7);
      if (i < n) {
        double v;
        if (lower) v = j <= i ? *sm(i, j) : 0.0;
        else v = i <= j ? *sm(j, i) : 0.0;
        g[i * ld + j] = v;
      }
    }
  }
}
}  // namespace

template <typename T>
bool potrf_small_eligible(int64_t n) {
  return n >= 1 && n <= SN;
}
// the forward alone also has the one-launch fp64 kernel up to n = 128
template <typename T>
bool potrf_fwd_small_eligible(int64_t n) {
  return n >= 1 && (n <= SN || (sizeof(T) == 8 && n <= P2));
}

template <typename T>
dla_status potrf_small(const Ctx& c, int64_t batch, int64_t n, MatB<T> a, bool lower, bool check_sym) {
  if (n <= WN) {
    constexpr int wpc = wpc_fwd<T>();
    const size_t sm = sizeof(T) * wpc * (WN * WLD + 2 * WN + 4);
    static const int minb = [] {
      const char* e = getenv("DLA_WARP_MINB");  // tuning switch: 1 = no register cap
      return e ? atoi(e) : 2;
    }();
    const unsigned grid = (unsigned)((batch + wpc - 1) / wpc);
    auto go = [&](auto kern) {
      ensure_smem_attr(kern, sm);
      kern<<<grid, wpc * 32, sm, c.stream>>>((int)n, batch, a, lower, c.info);
    };
    if (n == WN)
      minb == 1 ? go(k_potrf_warp<T, 1, WN>) : go(k_potrf_warp<T, 2, WN>);
    else
      minb == 1 ? go(k_potrf_warp<T, 1, 0>) : go(k_potrf_warp<T, 2, 0>);
    DLAB_LAUNCH_CHECK();
    return DLA_OK;
  }
  if (n > SN) {
    if constexpr (sizeof(T) == 8) {
      const size_t sm = sizeof(double) * 3 * 64 * P2LD;
      static const int minb = [] {
        const char* e = getenv("DLA_P128_MINB");  // tuning switch: 1 = no register cap (one CTA per SM)
        return e ? atoi(e) : 2;
      }();
      MatB<double> ad{reinterpret_cast<double*>(a.p), a.ld, a.bs, a.bsi};
      if (minb == 1) {
        ensure_smem_attr(k_potrf128<1>, sm);
        k_potrf128<1><<<(unsigned)batch, 256, sm, c.stream>>>((int)n, ad, lower, c.info, check_sym);
      } else {
        ensure_smem_attr(k_potrf128<2>, sm);
        k_potrf128<2><<<(unsigned)batch, 256, sm, c.stream>>>((int)n, ad, lower, c.info, check_sym);
      }
      DLAB_LAUNCH_CHECK();
    }
    return DLA_OK;
  }
  k_potrf_small<T><<<(unsigned)batch, 256, 0, c.stream>>>((int)n, a, lower, c.info);
  DLAB_LAUNCH_CHECK();
  return DLA_OK;
}

template <typename T>
dla_status potrf_bwd_small(const Ctx& c, int64_t batch, int64_t n, MatB<T> abar, MatB<const T> lbar,
                           MatB<const T> l, bool lower) {
  if (n <= WN) {
    if constexpr (sizeof(T) == 8) {
      static const bool dmma = [] {
        const char* e = getenv("DLA_SMALL_BWD_DMMA");  // tuning switch: 0 = the substitution kernel
        return e ? atoi(e) != 0 : true;
      }();
      if (dmma) {
        const size_t sm = sizeof(double) * BDW * (2 * DBUF + TBUF);
        MatB<double> ab{reinterpret_cast<double*>(abar.p), abar.ld, abar.bs, abar.bsi};
        MatB<const double> lb{reinterpret_cast<const double*>(lbar.p), lbar.ld, lbar.bs, lbar.bsi};
        MatB<const double> lv{reinterpret_cast<const double*>(l.p), l.ld, l.bs, l.bsi};
        auto go = [&](auto kern) {
          ensure_smem_attr(kern, sm);
          kern<<<(unsigned)((batch + BDW - 1) / BDW), BDW * 32, sm, c.stream>>>((int)n, batch, ab, lb, lv);
        };
        if (lower)
          n == WN ? go(k_potrf_bwd_dmma<true, WN>) : go(k_potrf_bwd_dmma<true, 0>);
        else
          n == WN ? go(k_potrf_bwd_dmma<false, WN>) : go(k_potrf_bwd_dmma<false, 0>);
        DLAB_LAUNCH_CHECK();
        return DLA_OK;
      }
    }
    constexpr int wpc = wpc_bwd<T>();
    const size_t sm = sizeof(T) * wpc * (WN * Bc<T>::LLD + WN * WLD + 2 * WN + 4);
    auto go = [&](auto kern) {
      ensure_smem_attr(kern, sm);
      kern<<<(unsigned)((batch + wpc - 1) / wpc), wpc * 32, sm, c.stream>>>((int)n, batch, abar, lbar, l, lower);
    };
    n == WN ? go(k_potrf_bwd_warp<T, WN>) : go(k_potrf_bwd_warp<T, 0>);
    DLAB_LAUNCH_CHECK();
    return DLA_OK;
  }
  const size_t sm = sizeof(T) * 3 * SN * SLD;
  ensure_smem_attr(k_potrf_bwd_small<T>, sm);
  k_potrf_bwd_small<T><<<(unsigned)batch, 256, sm, c.stream>>>((int)n, abar, lbar, l, lower);
  DLAB_LAUNCH_CHECK();
  return DLA_OK;
}


template <typename T>
dla_status chol_chain_small(const Ctx& c, int64_t batch, int64_t n, MatB<const T> a, const T* y, T* phi, MatB<T> abar,
                            T* ybar) {
  if constexpr (sizeof(T) == 8) {
    static const bool dmma = [] {
      const char* e = getenv("DLA_SMALL_BWD_DMMA");  // tuning switch: 0 = the substitution pullback
      return e ? atoi(e) != 0 : true;
    }();
    if (dmma) {
      const size_t sm = sizeof(double) * CDW * (2 * DBUF + TBUF + 6 * WN);
      MatB<const double> ad{reinterpret_cast<const double*>(a.p), a.ld, a.bs, a.bsi};
      MatB<double> abd{reinterpret_cast<double*>(abar.p), abar.ld, abar.bs, abar.bsi};
      auto go = [&](auto kern) {
        ensure_smem_attr(kern, sm);
        kern<<<(unsigned)((batch + CDW - 1) / CDW), CDW * 32, sm, c.stream>>>(
            (int)n, batch, ad, reinterpret_cast<const double*>(y), reinterpret_cast<double*>(phi), abd,
            reinterpret_cast<double*>(ybar), c.info);
      };
      n == WN ? go(k_chol_chain_dmma<WN>) : go(k_chol_chain_dmma<0>);
      DLAB_LAUNCH_CHECK();
      return DLA_OK;
    }
  }
  constexpr int wpc = wpc_bwd<T>();
  const size_t sm = sizeof(T) * wpc * (WN * Bc<T>::LLD + WN * WLD + 6 * WN);
  auto go = [&](auto kern) {
    ensure_smem_attr(kern, sm);
    kern<<<(unsigned)((batch + wpc - 1) / wpc), wpc * 32, sm, c.stream>>>((int)n, batch, a, y, phi, abar, ybar,
                                                                         c.info);
  };
  n == WN ? go(k_chol_chain_warp<T, WN>) : go(k_chol_chain_warp<T, 0>);
  DLAB_LAUNCH_CHECK();
  return DLA_OK;
}

#define INST(T)                                                                                     \
  template bool potrf_small_eligible<T>(int64_t);                                                   \
  template bool potrf_fwd_small_eligible<T>(int64_t);                                               \
  template dla_status potrf_small<T>(const Ctx&, int64_t, int64_t, MatB<T>, bool, bool);            \
  template dla_status potrf_bwd_small<T>(const Ctx&, int64_t, int64_t, MatB<T>, MatB<const T>, MatB<const T>, bool); \
  template dla_status chol_chain_small<T>(const Ctx&, int64_t, int64_t, MatB<const T>, const T*, T*, MatB<T>, T*);
INST(double)
INST(float)

}  // namespace dlab
