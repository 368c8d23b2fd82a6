// Batched strided GEMM for the blocked factorizations and the backward
// compositions:  C = alpha op(A) op(B) + beta C  (beta == 0 => C not read),
// with
//   * an optional lower/upper write mask (SYRK-style updates skip the tiles
//     above/below the diagonal entirely),
//   * optional triangular operands (trmm / inverse-based trsm as one GEMM:
//     the K loop of each tile is restricted to the triangle's nonzero range
//     and the ignored triangle inside boundary k-blocks is zeroed in shared
//     memory, so whatever the caller's memory holds there is never used —
//     the reference reads only the `lower`-selected triangle, dl/blas.hpp:182),
//   * a two-level batch (outer slices x inner blocks) for the level-batched
//     triangular inverse.
//
// f64: FP64 tensor cores.  Each warp owns a WM x WN output tile built from
//      `mma.sync.m8n8k4.f64` (SASS DMMA.8x8x4); tcgen05 has no f64 kind, and
//      the measured DMMA ceiling on B200 is 37.1 TFLOP/s
//      (profiles/peaks_fp64_fp32_r01.json).  128 x 128 CTA tiles reach
//      30.7 TFLOP/s at 4096^3.
// f32: FFMA SIMT (exact binary32, no TF32 rounding), 4x4 register tiles.
//
// Operand tiles are staged global->shared with cp.async (zero-filled out of
// bounds) in a 3-stage pipeline; 16-byte vectors when the leading dimension
// and the contiguous extent allow, 8/4-byte otherwise, so every shape works.
// Batch and tiles share a flat grid.x (65536-slice batches exceed gridDim.z).
#include "common.cuh"
#include "ops.cuh"
#include <algorithm>

#ifndef DLAB_GEMM_BKL
#define DLAB_GEMM_BKL 32  // k-block of the 128 x 128 configuration (3 stages: 212 KB smem)
#endif
#ifndef DLAB_SHORTK
#define DLAB_SHORTK 1024  // K up to which large GEMMs use the two-CTA 128 x 64 tiles
#endif
#ifndef DLAB_SHORTK_CFG
#define DLAB_SHORTK_CFG 1
#endif
#ifndef DLAB_GEMM_BKS
#define DLAB_GEMM_BKS 16  // k-block of the 64 x 64 configuration
#endif

namespace dlab {
namespace {

constexpr int STAGES = 3, PAD = 4;
#ifndef DLAB_GEMM_CPF
#define DLAB_GEMM_CPF 2  // C row groups prefetched before the main loop (the MINB == 2 configuration)
#endif

// Tile configurations: CTA tile BM x BN, warp tile WM x WN (FP64 DMMA),
// k-block BK per pipeline stage.
template <int BM_, int BN_, int WM_, int WN_, int BK_ = 16, int MINB_ = 1>
struct Cfg {
  static constexpr int BM = BM_, BN = BN_, WM = WM_, WN = WN_, BK = BK_, MINB = MINB_;
  static constexpr int WARPS_N = BN / WN;
  static constexpr int WARPS = (BM / WM) * (BN / WN);
  static constexpr int NT = WARPS * 32;
};
#ifndef DLAB_CFGS_MINB
#define DLAB_CFGS_MINB 4
#endif
using CfgS = Cfg<64, 64, 32, 32, DLAB_GEMM_BKS, DLAB_CFGS_MINB>;  // 128 threads: small / batched problems
using CfgL = Cfg<128, 128, 64, 32, DLAB_GEMM_BKL>;  // 256 threads: large trailing updates
// short-K (rank <= 128 updates: the blocked Cholesky's trailing SYRKs): a
// 16-deep k-block keeps 3 stages in 71 KB, so 3 CTAs share an SM and one
// CTA's C read-modify-write epilogue overlaps another's operand loads
// Large GEMMs with K <= DLAB_SHORTK, a write mask or a triangular operand:
// 128 x 64 tiles at two CTAs per SM (110-128 registers), so one CTA's
// operand prologue and C read-modify-write epilogue overlap the other's DMMA
// main loop, and the finer tiles balance triangular K ranges.  Measured on
// B200: the blocked Cholesky's rank-64 SYRKs, the 128^3 batched products of
// C5 and potrf_bwd's triangular products all gain (C5 -16 %); plain deep-K
// GEMMs keep the 128 x 128, k-block 32 tiles (31.5 TF/s at 4096^3).
#if DLAB_SHORTK_CFG == 1
using CfgK = Cfg<128, 64, 32, 32, 16, 2>;
#else
using CfgK = Cfg<128, 128, 64, 32, 16>;
#endif
// narrow N (<= 32, deep K): the blocked LQ's W = R Yc^T (rows x 32 x n)
using CfgN = Cfg<64, 32, 32, 16, 16>;

template <typename T>
struct GemmArgs {
  int64_t m, n, k;
  T alpha, beta;
  MatB<const T> a, b;
  MatB<T> c;
  int mask;
  const int32_t* skip;
  int64_t tiles_m, tiles_n;
  int tri_a, tri_b;
  int64_t inner;
  int64_t total;  // tiles over all slabs; CTAs loop tile = blockIdx.x, += gridDim.x
};

__device__ __forceinline__ void cp_async(void* smem, const void* gmem, bool pred, int bytes) {
  unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  int src = pred ? bytes : 0;
  if (bytes == 16)
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem), "r"(src));
  else if (bytes == 8)
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(s), "l"(gmem), "r"(src));
  else
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;\n" ::"r"(s), "l"(gmem), "r"(src));
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

// Shared-memory tile geometry.  A tile (BM x BK logical) is stored [m][k]
// when !TA (rows of A are contiguous in k) and [k][m] when TA; B likewise
// [k][n] when !TB and [n][k] when TB.  PAD = 4 elements keeps the 64-bit
// fragment loads of a half-warp on distinct banks.
template <int BM, int BK, bool TA>
struct ATile {
  static constexpr int LD = TA ? (BM + PAD) : (BK + PAD);
  static constexpr int ELEMS = TA ? BK * LD : BM * LD;
  __device__ static int idx(int i, int k) { return TA ? k * LD + i : i * LD + k; }
};
template <int BN, int BK, bool TB>
struct BTile {
  static constexpr int LD = TB ? (BK + PAD) : (BN + PAD);
  static constexpr int ELEMS = TB ? BN * LD : BK * LD;
  __device__ static int idx(int k, int j) { return TB ? j * LD + k : k * LD + j; }
};

// Issue the cp.async loads of one k-block into stage buffers sa / sb.
template <typename T, class C, bool TA, bool TB, int VA, int VB>
__device__ __forceinline__ void load_stage(const GemmArgs<T>& g, const T* A, const T* B, int64_t m0, int64_t n0,
                                           int64_t k0, T* sa, T* sb) {
  constexpr int BM = C::BM, BN = C::BN, NT = C::NT, BK = C::BK;
  {
    constexpr int CH = (BM * BK) / VA;
#pragma unroll
    for (int c0 = 0; c0 < CH; c0 += NT) {
      const int c = c0 + threadIdx.x;
      if (CH % NT != 0 && c >= CH) break;
      int i, k;
      if (!TA) {  // contiguous along k
        i = c / (BK / VA);
        k = (c % (BK / VA)) * VA;
      } else {    // contiguous along i
        k = c / (BM / VA);
        i = (c % (BM / VA)) * VA;
      }
      const int64_t gi = m0 + i, gk = k0 + k;
      const bool ok = gi < g.m && gk < g.k;
      const T* src = ok ? (TA ? A + gk * g.a.ld + gi : A + gi * g.a.ld + gk) : A;
      cp_async(sa + ATile<BM, BK, TA>::idx(i, k), src, ok, VA * (int)sizeof(T));
    }
  }
  {
    constexpr int CH = (BN * BK) / VB;
#pragma unroll
    for (int c0 = 0; c0 < CH; c0 += NT) {
      const int c = c0 + threadIdx.x;
      if (CH % NT != 0 && c >= CH) break;
      int j, k;
      if (!TB) {  // contiguous along j
        k = c / (BN / VB);
        j = (c % (BN / VB)) * VB;
      } else {    // contiguous along k
        j = c / (BK / VB);
        k = (c % (BK / VB)) * VB;
      }
      const int64_t gj = n0 + j, gk = k0 + k;
      const bool ok = gj < g.n && gk < g.k;
      const T* src = ok ? (TB ? B + gj * g.b.ld + gk : B + gk * g.b.ld + gj) : B;
      cp_async(sb + BTile<BN, BK, TB>::idx(k, j), src, ok, VB * (int)sizeof(T));
    }
  }
}

// Zero the ignored triangle of triangular operands inside k-block k0 (only
// blocks that straddle the diagonal need it).
template <typename T, class C, bool TA, bool TB>
__device__ __forceinline__ bool mask_stage(const GemmArgs<T>& g, int64_t m0, int64_t n0, int64_t k0, T* sa, T* sb) {
  constexpr int BM = C::BM, BN = C::BN, NT = C::NT, BK = C::BK;
  bool touched = false;
  if (g.tri_a != TRI_NONE) {
    const bool lower = g.tri_a == TRI_LOWER;  // A(i,k) = 0 for k > i (lower) / k < i (upper)
    const bool straddles = lower ? (k0 + BK - 1 > m0) : (k0 < m0 + BM - 1);
    if (straddles) {
      for (int e = threadIdx.x; e < BM * BK; e += NT) {
        const int i = e / BK, k = e % BK;
        const int64_t gi = m0 + i, gk = k0 + k;
        if (lower ? (gk > gi) : (gk < gi)) sa[ATile<BM, BK, TA>::idx(i, k)] = T(0);
      }
      touched = true;
    }
  }
  if (g.tri_b != TRI_NONE) {
    const bool lower = g.tri_b == TRI_LOWER;  // B(k,j) = 0 for k < j (lower) / k > j (upper)
    const bool straddles = lower ? (k0 < n0 + BN - 1) : (k0 + BK - 1 > n0);
    if (straddles) {
      for (int e = threadIdx.x; e < BN * BK; e += NT) {
        const int k = e / BN, j = e % BN;
        const int64_t gj = n0 + j, gk = k0 + k;
        if (lower ? (gk < gj) : (gk > gj)) sb[BTile<BN, BK, TB>::idx(k, j)] = T(0);
      }
      touched = true;
    }
  }
  return touched;
}

template <int BM, int BN>
__device__ __forceinline__ bool tile_masked_out(int mask, int64_t m0, int64_t n0) {
  if (mask == MASK_LOWER) return n0 > m0 + BM - 1;
  if (mask == MASK_UPPER) return m0 > n0 + BN - 1;
  return false;
}

// Per-tile K range implied by triangular operands.
template <typename T, int BM, int BN, int BK>
__device__ __forceinline__ void k_range(const GemmArgs<T>& g, int64_t m0, int64_t n0, int64_t& klo, int64_t& khi) {
  klo = 0;
  khi = g.k;
  if (g.tri_a == TRI_LOWER) khi = min(khi, m0 + BM);
  if (g.tri_a == TRI_UPPER) klo = max(klo, m0);
  if (g.tri_b == TRI_LOWER) klo = max(klo, n0);
  if (g.tri_b == TRI_UPPER) khi = min(khi, n0 + BN);
  klo = (klo / BK) * BK;
}

template <typename T>
__device__ __forceinline__ void store_c(const GemmArgs<T>& g, T* Cp, int64_t gi, int64_t gj, T v) {
  if (gi >= g.m || gj >= g.n) return;
  if (g.mask == MASK_LOWER && gj > gi) return;
  if (g.mask == MASK_UPPER && gj < gi) return;
  T* cp = Cp + gi * g.c.ld + gj;
  T r = g.alpha * v;
  if (g.beta != T(0)) r += g.beta * *cp;
  *cp = r;
}

// Decode blockIdx.x into (outer slice, inner block, tile) and operand bases.
template <typename T>
struct TileCoord {
  int64_t bo, m0, n0;
  const T *A, *B;
  T* C;
};
template <typename T, int BM, int BN>
__device__ __forceinline__ TileCoord<T> decode(const GemmArgs<T>& g, int64_t tile) {
  const int64_t per = g.tiles_m * g.tiles_n;
  const int64_t slab = tile / per;
  tile -= slab * per;
  TileCoord<T> t;
  t.bo = slab / g.inner;
  const int64_t bi = slab % g.inner;
  int64_t tm = tile / g.tiles_n, tn = tile % g.tiles_n;
  // Longest-K tiles first (CTAs are dispatched in blockIdx order): a lower
  // op(A) gives the bottom tile rows the longest K range, an upper op(B) the
  // right-most tile columns.
  if (g.tri_a == TRI_LOWER) tm = g.tiles_m - 1 - tm;
  if (g.tri_b == TRI_UPPER) tn = g.tiles_n - 1 - tn;
  t.m0 = tm * BM;
  t.n0 = tn * BN;
  t.A = g.a.p + t.bo * g.a.bs + bi * g.a.bsi;
  t.B = g.b.p + t.bo * g.b.bs + bi * g.b.bsi;
  t.C = g.c.p + t.bo * g.c.bs + bi * g.c.bsi;
  return t;
}

// ------------------------------------------------------------------ f64 DMMA
template <class C, bool TA, bool TB, int VA, int VB>
__global__ void __launch_bounds__(C::NT, C::MINB) dgemm_dmma(GemmArgs<double> g) {
  using AT = ATile<C::BM, C::BK, TA>;
  using BT = BTile<C::BN, C::BK, TB>;
  constexpr int MI = C::WM / 8, NI = C::WN / 8, BK = C::BK;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double* smem = reinterpret_cast<double*>(smem_raw);
  double* sA = smem;
  double* sB = smem + STAGES * AT::ELEMS;

  for (int64_t tile = blockIdx.x; tile < g.total; tile += gridDim.x) {
  __syncthreads();  // the previous tile's warps are done with the stage buffers
  const TileCoord<double> tc = decode<double, C::BM, C::BN>(g, tile);
  const int64_t m0 = tc.m0, n0 = tc.n0;
  if (g.skip && g.skip[tc.bo]) continue;
  if (tile_masked_out<C::BM, C::BN>(g.mask, m0, n0)) continue;
  int64_t klo, khi;
  k_range<double, C::BM, C::BN, C::BK>(g, m0, n0, klo, khi);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int wm = (warp / C::WARPS_N) * C::WM, wn = (warp % C::WARPS_N) * C::WN;
  const int fr = lane >> 2, fc = lane & 3;
  double acc[MI][NI][2];
#pragma unroll
  for (int i = 0; i < MI; ++i)
#pragma unroll
    for (int j = 0; j < NI; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

  const bool tri = (g.tri_a | g.tri_b) != 0;
  const int64_t nk = khi > klo ? (khi - klo + BK - 1) / BK : 0;
#pragma unroll
  for (int s = 0; s < STAGES - 1; ++s) {
    if (s < nk)
      load_stage<double, C, TA, TB, VA, VB>(g, tc.A, tc.B, m0, n0, klo + s * BK, sA + s * AT::ELEMS,
                                            sB + s * BT::ELEMS);
    cp_commit();
  }
  const bool vec2 = ((g.c.ld & 1) == 0) && ((reinterpret_cast<uintptr_t>(tc.C) & 15) == 0);
  auto load_group = [&](int i, double (&cv)[NI][2]) {
#pragma unroll
    for (int j = 0; j < NI; ++j) {
      cv[j][0] = cv[j][1] = 0.0;
      if (g.beta == 0.0) continue;
      const int64_t gi = m0 + wm + i * 8 + fr, gj = n0 + wn + j * 8 + 2 * fc;
      if (gi >= g.m) continue;
      const double* cp = tc.C + gi * g.c.ld + gj;
      if (vec2 && gj + 1 < g.n) {
        const double2 v = *reinterpret_cast<const double2*>(cp);
        cv[j][0] = v.x;
        cv[j][1] = v.y;
      } else {
        if (gj < g.n) cv[j][0] = cp[0];
        if (gj + 1 < g.n) cv[j][1] = cp[1];
      }
    }
  };
  // short-K configurations: the first CPF C row groups load now, in flight
  // under the main loop instead of exposed at the epilogue
  constexpr int CPF = C::MINB == 2 ? DLAB_GEMM_CPF : 0, CPF1 = CPF > 0 ? CPF : 1;
  double cpf[CPF1][NI][2];
  if constexpr (CPF > 0) {
#pragma unroll
    for (int i = 0; i < CPF; ++i) load_group(i, cpf[i]);
  }
  for (int64_t kb = 0; kb < nk; ++kb) {
    cp_wait<STAGES - 2>();
    __syncthreads();
    const int st = (int)(kb % STAGES);
    if (tri && mask_stage<double, C, TA, TB>(g, m0, n0, klo + kb * BK, sA + st * AT::ELEMS, sB + st * BT::ELEMS))
      __syncthreads();
    {  // prefetch kb + STAGES - 1 into the slot freed at kb - 1
      const int64_t pf = kb + STAGES - 1;
      const int ps = (int)(pf % STAGES);
      if (pf < nk)
        load_stage<double, C, TA, TB, VA, VB>(g, tc.A, tc.B, m0, n0, klo + pf * BK, sA + ps * AT::ELEMS,
                                              sB + ps * BT::ELEMS);
      cp_commit();
    }
    const double* a = sA + st * AT::ELEMS;
    const double* b = sB + st * BT::ELEMS;
#pragma unroll
    for (int kk = 0; kk < BK; kk += 4) {
      double af[MI], bf[NI];
#pragma unroll
      for (int i = 0; i < MI; ++i) af[i] = a[AT::idx(wm + i * 8 + fr, kk + fc)];
#pragma unroll
      for (int j = 0; j < NI; ++j) bf[j] = b[BT::idx(kk + fc, wn + j * 8 + fr)];
#pragma unroll
      for (int i = 0; i < MI; ++i)
#pragma unroll
        for (int j = 0; j < NI; ++j)
          asm volatile(
              "mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
              : "+d"(acc[i][j][0]), "+d"(acc[i][j][1])
              : "d"(af[i]), "d"(bf[j]));
    }
  }
  cp_wait<0>();
  // Epilogue: C rows in groups of 8 (one fragment row i); when beta != 0 the
  // C values of group i+1 are loaded before group i is stored, so the
  // read-modify-write of C keeps loads in flight (the rank-64 SYRK updates
  // of the blocked Cholesky are bound by exactly this C traffic).  The first
  // CPF groups were loaded before the main loop (short-K configurations).
  double cur[NI][2], nxt[NI][2];
  if constexpr (CPF > 0) {
#pragma unroll
    for (int j = 0; j < NI; ++j) cur[j][0] = cpf[0][j][0], cur[j][1] = cpf[0][j][1];
  } else {
    load_group(0, cur);
  }
#pragma unroll
  for (int i = 0; i < MI; ++i) {
    if (i + 1 < MI) {
      if (i + 1 < CPF) {
#pragma unroll
        for (int j = 0; j < NI; ++j) nxt[j][0] = cpf[(i + 1) % CPF1][j][0], nxt[j][1] = cpf[(i + 1) % CPF1][j][1];
      } else {
        load_group(i + 1, nxt);
      }
    }
    const int64_t gi = m0 + wm + i * 8 + fr;
#pragma unroll
    for (int j = 0; j < NI; ++j) {
      const int64_t gj = n0 + wn + j * 8 + 2 * fc;
      if (gi >= g.m) continue;
      const double v0 = g.alpha * acc[i][j][0] + g.beta * cur[j][0];
      const double v1 = g.alpha * acc[i][j][1] + g.beta * cur[j][1];
      const bool ok0 = gj < g.n && !(g.mask == MASK_LOWER && gj > gi) && !(g.mask == MASK_UPPER && gj < gi);
      const bool ok1 =
          gj + 1 < g.n && !(g.mask == MASK_LOWER && gj + 1 > gi) && !(g.mask == MASK_UPPER && gj + 1 < gi);
      double* cp = tc.C + gi * g.c.ld + gj;
      if (vec2 && ok0 && ok1) {
        *reinterpret_cast<double2*>(cp) = make_double2(v0, v1);
      } else {
        if (ok0) cp[0] = v0;
        if (ok1) cp[1] = v1;
      }
    }
    if (i + 1 < MI) {
#pragma unroll
      for (int j = 0; j < NI; ++j) {
        cur[j][0] = nxt[j][0];
        cur[j][1] = nxt[j][1];
      }
    }
  }
  }  // tile loop
}

// ------------------------------------------------------------------ f32 FFMA
template <bool TA, bool TB, int VA, int VB>
__global__ void __launch_bounds__(256) sgemm_ffma(GemmArgs<float> g) {
  using C = Cfg<64, 64, 32, 16>;  // 8 warps -> 256 threads; smem geometry of a 64 x 64 tile
  static_assert(C::NT == 256, "sgemm thread count");
  constexpr int BK = C::BK;
  using AT = ATile<64, BK, TA>;
  using BT = BTile<64, BK, TB>;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  float* smem = reinterpret_cast<float*>(smem_raw);
  float* sA = smem;
  float* sB = smem + STAGES * AT::ELEMS;

  const TileCoord<float> tc = decode<float, 64, 64>(g, blockIdx.x);
  const int64_t m0 = tc.m0, n0 = tc.n0;
  if (g.skip && g.skip[tc.bo]) return;
  if (tile_masked_out<64, 64>(g.mask, m0, n0)) return;
  int64_t klo, khi;
  k_range<float, 64, 64, BK>(g, m0, n0, klo, khi);

  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;  // 16 x 16 threads, 4x4 each
  float acc[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = 0.f;

  const bool tri = (g.tri_a | g.tri_b) != 0;
  const int64_t nk = khi > klo ? (khi - klo + BK - 1) / BK : 0;
#pragma unroll
  for (int s = 0; s < STAGES - 1; ++s) {
    if (s < nk)
      load_stage<float, C, TA, TB, VA, VB>(g, tc.A, tc.B, m0, n0, klo + s * BK, sA + s * AT::ELEMS,
                                           sB + s * BT::ELEMS);
    cp_commit();
  }
  for (int64_t kb = 0; kb < nk; ++kb) {
    cp_wait<STAGES - 2>();
    __syncthreads();
    const int st = (int)(kb % STAGES);
    if (tri && mask_stage<float, C, TA, TB>(g, m0, n0, klo + kb * BK, sA + st * AT::ELEMS, sB + st * BT::ELEMS))
      __syncthreads();
    {
      const int64_t pf = kb + STAGES - 1;
      const int ps = (int)(pf % STAGES);
      if (pf < nk)
        load_stage<float, C, TA, TB, VA, VB>(g, tc.A, tc.B, m0, n0, klo + pf * BK, sA + ps * AT::ELEMS,
                                             sB + ps * BT::ELEMS);
      cp_commit();
    }
    const float* a = sA + st * AT::ELEMS;
    const float* b = sB + st * BT::ELEMS;
#pragma unroll
    for (int kk = 0; kk < BK; ++kk) {
      float av[4], bv[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) av[i] = a[AT::idx(ty + 16 * i, kk)];
#pragma unroll
      for (int j = 0; j < 4; ++j) bv[j] = b[BT::idx(kk, tx + 16 * j)];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(av[i], bv[j], acc[i][j]);
    }
  }
  cp_wait<0>();
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) store_c<float>(g, tc.C, m0 + ty + 16 * i, n0 + tx + 16 * j, acc[i][j]);
}

template <typename T, bool TA, bool TB, int VA, int VB>
cudaError_t launch_tv(GemmArgs<T> g, int64_t slabs, cudaStream_t s, bool large, int max_ctas, bool rowtile) {
  auto grid = [&](int64_t tiles) {
    g.total = tiles;
    return (unsigned)(max_ctas > 0 && tiles > max_ctas ? max_ctas : tiles);
  };
  if constexpr (sizeof(T) == 8) {
    // Masked, triangular-operand and short-K products: 64 x 64 tiles at four
    // CTAs per SM (measured on B200 against the two-CTA 128 x 64 tiles: the
    // potrf pullback at n = 1024 x 8 -16 %, n = 128 x 512 -20 %, the C2 step
    // -1 %; per-tile prologue / C read-modify-write of one CTA hides under
    // three others' DMMA main loops).  DLA_GEMM_MASKED_TILE=128 restores the
    // 128 x 64 tiles (tuning switch).  rowtile keeps its 128-row tiles: in-place
    // trmm correctness depends on them.
    static const bool masked128 = [] {
      const char* e = getenv("DLA_GEMM_MASKED_TILE");
      return e && atoi(e) == 128;
    }();
    if (!masked128 && !rowtile && large &&
        (g.k <= DLAB_SHORTK || g.mask != MASK_FULL || g.tri_a != TRI_NONE || g.tri_b != TRI_NONE))
      large = false;
    if (g.n <= 32 && g.k >= 128 && g.m >= 64 && !rowtile) {
      using C = CfgN;
      g.tiles_m = (g.m + C::BM - 1) / C::BM;
      g.tiles_n = (g.n + C::BN - 1) / C::BN;
      const size_t smem = sizeof(T) * STAGES * (ATile<C::BM, C::BK, TA>::ELEMS + BTile<C::BN, C::BK, TB>::ELEMS);
      auto k = dgemm_dmma<C, TA, TB, VA, VB>;
      ensure_smem_attr(k, smem);
      const unsigned nb = grid(slabs * g.tiles_m * g.tiles_n);
      k<<<nb, C::NT, smem, s>>>(g);
    } else if (rowtile || (large && (g.k <= DLAB_SHORTK || g.mask != MASK_FULL || g.tri_a != TRI_NONE ||
                                      g.tri_b != TRI_NONE))) {
      using C = CfgK;
      g.tiles_m = (g.m + C::BM - 1) / C::BM;
      g.tiles_n = (g.n + C::BN - 1) / C::BN;
      const size_t smem = sizeof(T) * STAGES * (ATile<C::BM, C::BK, TA>::ELEMS + BTile<C::BN, C::BK, TB>::ELEMS);
      auto k = dgemm_dmma<C, TA, TB, VA, VB>;
      ensure_smem_attr(k, smem);
      const unsigned nb = grid(slabs * g.tiles_m * g.tiles_n);
      k<<<nb, C::NT, smem, s>>>(g);
    } else if (large) {
      using C = CfgL;
      g.tiles_m = (g.m + C::BM - 1) / C::BM;
      g.tiles_n = (g.n + C::BN - 1) / C::BN;
      const size_t smem = sizeof(T) * STAGES * (ATile<C::BM, C::BK, TA>::ELEMS + BTile<C::BN, C::BK, TB>::ELEMS);
      auto k = dgemm_dmma<C, TA, TB, VA, VB>;
      ensure_smem_attr(k, smem);
      const unsigned nb = grid(slabs * g.tiles_m * g.tiles_n);
      k<<<nb, C::NT, smem, s>>>(g);
    } else {
      using C = CfgS;
      g.tiles_m = (g.m + C::BM - 1) / C::BM;
      g.tiles_n = (g.n + C::BN - 1) / C::BN;
      const size_t smem = sizeof(T) * STAGES * (ATile<C::BM, C::BK, TA>::ELEMS + BTile<C::BN, C::BK, TB>::ELEMS);
      auto k = dgemm_dmma<C, TA, TB, VA, VB>;
      ensure_smem_attr(k, smem);
      const unsigned nb = grid(slabs * g.tiles_m * g.tiles_n);
      k<<<nb, C::NT, smem, s>>>(g);
    }
  } else {
    (void)large;
    g.tiles_m = (g.m + 63) / 64;
    g.tiles_n = (g.n + 63) / 64;
    const size_t smem = sizeof(T) * STAGES * (ATile<64, 16, TA>::ELEMS + BTile<64, 16, TB>::ELEMS);
    auto k = sgemm_ffma<TA, TB, VA, VB>;
    ensure_smem_attr(k, smem);
    g.total = slabs * g.tiles_m * g.tiles_n;
    k<<<(unsigned)g.total, 256, smem, s>>>(g);
  }
  return cudaGetLastError();
}

template <typename T, bool TA, bool TB>
cudaError_t launch_t(const GemmArgs<T>& g, int64_t slabs, cudaStream_t s, bool va, bool vb, bool large, int mc,
                     bool rt) {
  constexpr int V = 16 / (int)sizeof(T);
  if (va && vb) return launch_tv<T, TA, TB, V, V>(g, slabs, s, large, mc, rt);
  if (va) return launch_tv<T, TA, TB, V, 1>(g, slabs, s, large, mc, rt);
  if (vb) return launch_tv<T, TA, TB, 1, V>(g, slabs, s, large, mc, rt);
  return launch_tv<T, TA, TB, 1, 1>(g, slabs, s, large, mc, rt);
}

// Vector loads need 16-byte aligned rows and a contiguous extent that is a
// multiple of the vector width.
template <typename T>
bool vec_ok(const MatB<const T>& x, int64_t contiguous_extent) {
  constexpr int V = 16 / (int)sizeof(T);
  const uintptr_t p = reinterpret_cast<uintptr_t>(x.p);
  return (p % 16 == 0) && (x.ld % V == 0) && (x.bs % V == 0) && (x.bsi % V == 0) && (contiguous_extent % V == 0);
}

// Algorithmic flops of one slab: 2 x #{(i, j, k)} with C(i, j) inside the
// mask and A(i, k), B(k, j) inside their triangles (tri_a lower: k <= i,
// upper: k >= i; tri_b lower: k >= j, upper: k <= j; mask lower: i >= j).
// Counted over a strided (i, j) grid, exact k range per point: e.g. upper x
// lower with a full output is 2n^3/3, lower x lower into a lower mask n^3/3.
// Only evaluated when DLA profiling is on.
double useful_flops(int64_t m, int64_t n, int64_t k, int mask, int tri_a, int tri_b) {
  if (mask == MASK_FULL && tri_a == TRI_NONE && tri_b == TRI_NONE) return 2.0 * (double)m * (double)n * (double)k;
  const int64_t si = (m + 255) / 256, sj = (n + 255) / 256;
  double cnt = 0.0;
  for (int64_t i = 0; i < m; i += si) {
    for (int64_t j = 0; j < n; j += sj) {
      if (mask == MASK_LOWER && i < j) continue;
      if (mask == MASK_UPPER && i > j) continue;
      int64_t lo = 0, hi = k - 1;
      if (tri_a == TRI_LOWER) hi = std::min(hi, i);
      if (tri_a == TRI_UPPER) lo = std::max(lo, i);
      if (tri_b == TRI_LOWER) lo = std::max(lo, j);
      if (tri_b == TRI_UPPER) hi = std::min(hi, j);
      if (hi >= lo) cnt += (double)(hi - lo + 1);
    }
  }
  const double pts_i = (double)((m + si - 1) / si), pts_j = (double)((n + sj - 1) / sj);
  return 2.0 * cnt * ((double)m / pts_i) * ((double)n / pts_j);
}

}  // namespace

// fp32 products that run on tcgen05 (and carve packed operand tiles)
bool sgemm_tc_route(int64_t m, int64_t n, int64_t k, int64_t inner) {
  static const bool tc = [] {
    const char* e = getenv("DLA_SGEMM_TC");  // tuning switch: 0 keeps every fp32 GEMM on FFMA
    return e ? atoi(e) != 0 : true;
  }();
  return tc && inner == 1 && m >= 256 && n >= 256 && k >= 128;
}

template <typename T>
size_t ws_gemm(int64_t batch, int64_t m, int64_t n, int64_t k, int64_t inner) {
  if (sizeof(T) != 4 || batch <= 0 || !sgemm_tc_route(m, n, k, inner)) return 0;
  return carve_bound(sgemm_tc_ws_bytes(batch, m, n, k));
}
template size_t ws_gemm<double>(int64_t, int64_t, int64_t, int64_t, int64_t);
template size_t ws_gemm<float>(int64_t, int64_t, int64_t, int64_t, int64_t);

template <typename T>
dla_status gemm(const Ctx& c, int64_t batch, int64_t m, int64_t n, int64_t k, T alpha, MatB<const T> a,
                bool ta, MatB<const T> b, bool tb, T beta, MatB<T> cm, int mask, const int32_t* skip, int tri_a,
                int tri_b, int64_t inner) {
  if (batch <= 0 || m <= 0 || n <= 0 || inner <= 0) return DLA_OK;
  if (k <= 0) {  // C = beta C
    if (beta == T(1)) return DLA_OK;
    if (mask != MASK_FULL || inner != 1) return DLA_ERR_INVALID;
    return ew_scale<T>(c, batch, m, n, cm, beta, skip);
  }
  const bool rowtile = sizeof(T) == 8 && c.gemm_rowtile != 0 && m <= 128;
  if (inner == 1 && tri_a == TRI_NONE && tri_b == TRI_NONE && !rowtile) {  // vector / outer-product shapes
    dla_status st;
    if (gemm_skinny<T>(c, batch, m, n, k, alpha, a, ta, b, tb, beta, cm, mask, skip, &st)) return st;
  }
  if constexpr (sizeof(T) == 4) {  // large fp32 products: tcgen05 3xTF32 (gemm_tc.cu)
    if (sgemm_tc_route(m, n, k, inner)) {  // big products: the packing pass pays off
      dla_status st;
      const bool prof = gemm_prof_on();
      if (prof) gemm_prof_begin(c.stream);
      if (sgemm_tc(c, batch, m, n, k, alpha, a, ta, b, tb, beta, cm, mask, skip, tri_a, tri_b, inner, &st)) {
        if (prof) gemm_prof_end(c.stream, useful_flops(m, n, k, mask, tri_a, tri_b) * (double)batch);
        return st;
      }
    }
  }
  if constexpr (sizeof(T) == 8) {  // large products: the TMA-fed persistent kernel (gemm_tma.cu)
    if (!rowtile && c.gemm_ctas <= 0) {
      dla_status st;
      const bool prof = gemm_prof_on();
      if (prof) gemm_prof_begin(c.stream);
      if (gemm_tma(c, batch, m, n, k, alpha, a, ta, b, tb, beta, cm, mask, skip, tri_a, tri_b, inner, &st)) {
        if (prof) gemm_prof_end(c.stream, useful_flops(m, n, k, mask, tri_a, tri_b) * (double)batch);
        return st;
      }
      if (prof) gemm_prof_cancel();
    }
  }
  GemmArgs<T> g{m, n, k, alpha, beta, a, b, cm, mask, skip, 0, 0, tri_a, tri_b, inner, 0};
  const bool va = vec_ok<T>(a, ta ? m : k);
  const bool vb = vec_ok<T>(b, tb ? k : n);
  // 128 x 128 tiles once they alone fill every SM; 64 x 64 otherwise
  const int64_t slabs = batch * inner;
  const int64_t big_tiles = slabs * ((m + 127) / 128) * ((n + 127) / 128);
  const bool large = big_tiles >= c.sms && k >= 64;
  cudaError_t e;
  const bool prof = gemm_prof_on();
  if (prof) gemm_prof_begin(c.stream);
  if (!ta && !tb) e = launch_t<T, false, false>(g, slabs, c.stream, va, vb, large, c.gemm_ctas, rowtile);
  else if (ta && !tb) e = launch_t<T, true, false>(g, slabs, c.stream, va, vb, large, c.gemm_ctas, rowtile);
  else if (!ta && tb) e = launch_t<T, false, true>(g, slabs, c.stream, va, vb, large, c.gemm_ctas, rowtile);
  else e = launch_t<T, true, true>(g, slabs, c.stream, va, vb, large, c.gemm_ctas, rowtile);
  if (e != cudaSuccess) {
    fprintf(stderr, "dla_b200 gemm: %s\n", cudaGetErrorString(e));
    return DLA_ERR_CUDA;
  }
  note_launch(1);
  if (prof) gemm_prof_end(c.stream, useful_flops(m, n, k, mask, tri_a, tri_b) * (double)slabs);
  return DLA_OK;
}

template dla_status gemm<double>(const Ctx&, int64_t, int64_t, int64_t, int64_t, double, MatB<const double>,
                                 bool, MatB<const double>, bool, double, MatB<double>, int, const int32_t*, int, int,
                                 int64_t);
template dla_status gemm<float>(const Ctx&, int64_t, int64_t, int64_t, int64_t, float, MatB<const float>,
                                bool, MatB<const float>, bool, float, MatB<float>, int, const int32_t*, int, int,
                                int64_t);

}  // namespace dlab
