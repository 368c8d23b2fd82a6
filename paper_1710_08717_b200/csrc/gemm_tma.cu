// TMA-fed, warp-specialised persistent FP64 GEMM for the large products of
// the potrf pullback and the GP step (f64, one slab per matrix):
//
//     C = alpha op(A) op(B) + beta C,  triangular operands / lower-upper masks
//
// (the blocked algorithms' P' = tril(L^T Lbar), W = P' L^-1, Z = L^-T W,
// dl/adjoints.hpp:175-191 as restated in inv.cu).  One CTA per SM walks the
// 128 x 128 output tiles in longest-K-first order:
//
//   * warp 8 (producer; its warpgroup gives its registers to the consumers
//     by setmaxnreg): cp.async.bulk.tensor (SASS UTMALDG) of each tile's
//     16-deep k-chunks into a STAGES-deep ring of 128B-swizzled buffers,
//     mbarrier transaction counts; the ring runs across tile boundaries, so
//     the next tile's operands land while the current tile's epilogue runs.
//     K-major operands (rows contiguous in k) load as one [128 rows][16 k]
//     box, M/N-major operands (contiguous in m / n) as eight [16 k][16 mn]
//     boxes; the 128B swizzle makes both fragment orientations conflict-free.
//   * warps 0-7 (consumers, 2 x 4 warp grid of 64 x 32 warp tiles): FP64
//     DMMA m8n8k4 from the ring, the ignored triangle of a triangular operand
//     masked to zero in the fragments of the chunks that straddle its
//     diagonal, one mbarrier arrive per warp per chunk; the epilogue stores
//     alpha acc (+ beta C) straight from registers (16-byte stores).
//
// The generic cp.async kernel (gemm.cu) keeps every other shape.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <atomic>
#include <cmath>

#include "common.cuh"
#include "ops.cuh"

namespace dlab {
namespace {

constexpr int TK = 16;          // k per chunk (one 128-byte swizzle row of doubles)
constexpr int TBM = 128;  // CTA tile rows; columns BN = 128 (plain) or 64 (triangular / masked)
constexpr int TCONS = 8;        // consumer warps
constexpr int TTHREADS = (TCONS + 4) * 32;  // + one producer warpgroup (warp 8 issues, 9-11 idle)
constexpr int TWN = 32, TNI = TWN / 8;
constexpr int T_ABYTES = TBM * TK * 8;
template <int BN>
struct TT {  // per-width geometry: 2 x 4 warps of 64 x 32 (BN 128) / 4 x 2 of 32 x 32 (BN 64)
  static constexpr int WM = BN == 128 ? 64 : 32, MI = WM / 8, BBYTES = BN * TK * 8, STAGE = T_ABYTES + BBYTES;
  static constexpr int STAGES = BN == 128 ? 5 : 7;
  static constexpr size_t SMEM = (size_t)STAGES * STAGE + 1024 + 2 * STAGES * 8 + 2 * 4 * 8 + 4 * 8;
};

struct TmaArgs {
  int64_t m, n, k, batch;
  int64_t tm, tn;        // tiles per slab
  int64_t per;           // enumerated tiles per slab
  int64_t ratio;         // 128 / tile width (lower-masked enumeration)
  int64_t total;
  double alpha, beta;
  MatB<double> c;
  int mask, tri_a, tri_b;
  const int32_t* skip;
};

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbw(uint32_t bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "W_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra W_%=;\n\t}\n" ::"r"(bar),
      "r"(parity)
      : "memory");
}

__device__ __forceinline__ void tma_ld(uint32_t dst, const CUtensorMap* map, int c0, int c1, int c2, uint32_t bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];\n" ::"r"(
          dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(bar)
      : "memory");
}

// byte offset of (row, col) in a [rows][16 doubles] 128B-swizzled box
__device__ __forceinline__ uint32_t swz16(int row, int col) {
  return (uint32_t)(row * 128 + ((((col >> 1) ^ (row & 7))) << 4) + ((col & 1) << 3));
}
// element (mn, k) of a 128 x 16 operand chunk: K-major = one [128][16] box,
// MN-major = eight [16 k][16 mn] boxes
template <bool MN>
__device__ __forceinline__ uint32_t opoff(int mn, int k) {
  return MN ? (uint32_t)((mn >> 4) * 2048) + swz16(k, mn & 15) : swz16(mn, k);
}

// Tile t of a slab in (roughly) longest-K-first order; the tiles are handed
// out dynamically, so long tiles start first and short ones fill the tail.
// Lower-masked outputs enumerate only the tiles on or below the diagonal:
// row tm (128 rows) holds R (tm + 1) column tiles of width 128 / R, rows from
// the top (K from m0 on: P' = L^T Lbar) or, for a lower op(A) (K up to
// m0 + 128: W = P' L^-1), from the bottom.
__device__ __forceinline__ int64_t tri_row(int64_t t, int64_t R) {
  int64_t r = (int64_t)((sqrt(8.0 * (double)t / (double)R + 1.0) - 1.0) * 0.5);
  while (R * r * (r + 1) / 2 > t) --r;
  while (R * (r + 1) * (r + 2) / 2 <= t) ++r;
  return r;
}
__device__ __forceinline__ void tile_of(const TmaArgs& g, int64_t t, int64_t& b, int64_t& tm, int64_t& tn) {
  b = t / g.per;
  t -= b * g.per;
  if (g.mask == MASK_LOWER) {
    const int64_t R = g.ratio;
    if (g.tri_a == TRI_LOWER) t = g.per - 1 - t;
    tm = tri_row(t, R);
    tn = t - R * tm * (tm + 1) / 2;
  } else {
    tm = t / g.tn;
    tn = t % g.tn;
    if (g.tri_a == TRI_LOWER) tm = g.tm - 1 - tm;
    if (g.tri_b == TRI_UPPER) tn = g.tn - 1 - tn;
  }
}

__device__ __forceinline__ void krange(const TmaArgs& g, int64_t m0, int64_t n0, int bn, int64_t& klo, int64_t& khi) {
  klo = 0;
  khi = g.k;
  if (g.tri_a == TRI_LOWER) khi = min(khi, m0 + TBM);
  if (g.tri_a == TRI_UPPER) klo = max(klo, m0);
  if (g.tri_b == TRI_LOWER) klo = max(klo, n0);
  if (g.tri_b == TRI_UPPER) khi = min(khi, n0 + bn);
  klo = (klo / TK) * TK;
}

// Fragment row (A) / column (B) -> tile-local index.  K-major operands: the
// identity (8 consecutive rows of the swizzled [rows][16 k] box are
// conflict-free).  MN-major operands hold 16 m (n) per 128-byte row, and the
// 128B swizzle only permutes 16-byte chunks within a row: 8 consecutive m at
// 4 consecutive k would put two k rows on the same banks.  The fragment rows
// of half-warp h therefore take m = {0,1,8,9} + 2h (+ 4 for the odd fragment
// of a 16-row group) -- chunks c and c + 4, which the row XOR spreads over all
// 32 banks.  The accumulator rows / columns follow the same map.
// K-major boxes hold one row per m (n): rows m and m ^ 1 share the XOR
// pair of chunks, so half-warp h takes rows {0, 2, 4, 6} + h of each 8-row
// group (four disjoint 32-byte bank segments).
template <bool MN>
__device__ __forceinline__ int fidx(int f8, int fr) {  // f8: fragment index (8 rows / cols each)
  if (!MN) return f8 * 8 + 2 * (fr & 3) + (fr >> 2);
  return (f8 >> 1) * 16 + (f8 & 1) * 4 + ((fr & 1) | ((fr & 2) << 2) | ((fr & 4) >> 1));
}

// Per-launch tile counters (dynamic scheduling: longest-K-first tiles are
// taken in order by whichever CTA is free -- LPT); a launch uses slot
// `slot`, the last CTA to finish resets it.  64 slots: concurrent launches on
// different streams (the look-ahead / inverse side streams) never share one.
constexpr int TSLOTS = 64;
__device__ unsigned int g_tma_tiles[TSLOTS][2];
constexpr int TQ = 4;  // tile-id ring between the producer and the consumers

template <bool AMN, bool BMN, int BN>
__global__ void __launch_bounds__(TTHREADS, 1)
    k_dgemm_tma(const __grid_constant__ CUtensorMap map_a, const __grid_constant__ CUtensorMap map_b, TmaArgs g,
                int slot) {
  constexpr int TSTAGES = TT<BN>::STAGES, T_STAGE = TT<BN>::STAGE, TWM = TT<BN>::WM, TMI = TT<BN>::MI, TBN = BN;
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* smem = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~(uintptr_t)1023);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + TSTAGES * T_STAGE);
  uint64_t* empty = full + TSTAGES;
  uint64_t* tfull = empty + TSTAGES;
  uint64_t* tempty = tfull + TQ;
  int64_t* tids = reinterpret_cast<int64_t*>(tempty + TQ);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < TSTAGES; ++s) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(su32(&full[s])));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(su32(&empty[s])), "r"(TCONS));
    }
    for (int q = 0; q < TQ; ++q) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(su32(&tfull[q])));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(su32(&tempty[q])), "r"(TCONS));
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();

  if (warp >= TCONS) {  // ------------------------------------------------ producer warpgroup
    // hand the registers to the consumers (setmaxnreg works per warpgroup)
    asm volatile("setmaxnreg.dec.sync.aligned.u32 40;\n" ::: "memory");
    if (warp == TCONS && lane == 0) {
      asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<uint64_t>(&map_a)) : "memory");
      asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<uint64_t>(&map_b)) : "memory");
      uint32_t it = 0;
      for (uint32_t ti = 0;; ++ti) {
        const int64_t t = (int64_t)atomicAdd(&g_tma_tiles[slot][0], 1u);
        const uint32_t q = ti % TQ;
        mbw(su32(&tempty[q]), ((ti / TQ) & 1) ^ 1);
        tids[q] = t;
        asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];\n" ::"r"(su32(&tfull[q])) : "memory");
        if (t >= g.total) break;
        int64_t b, tm, tn;
        tile_of(g, t, b, tm, tn);
        if (g.skip && g.skip[b]) continue;
        const int64_t m0 = tm * TBM, n0 = tn * TBN;
        int64_t klo, khi;
        krange(g, m0, n0, BN, klo, khi);
        for (int64_t k0 = klo; k0 < khi; k0 += TK, ++it) {
          const uint32_t s = it % TSTAGES, ph = (it / TSTAGES) & 1;
          mbw(su32(&empty[s]), ph ^ 1);
          const uint32_t bar = su32(&full[s]);
          asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(bar), "r"(T_STAGE)
                       : "memory");
          const uint32_t dst = su32(smem + s * T_STAGE);
          if (AMN) {
#pragma unroll
            for (int x = 0; x < TBM / 16; ++x) tma_ld(dst + x * 2048, &map_a, (int)m0 + 16 * x, (int)k0, (int)b, bar);
          } else {
            tma_ld(dst, &map_a, (int)k0, (int)m0, (int)b, bar);
          }
          if (BMN) {
#pragma unroll
            for (int x = 0; x < TBN / 16; ++x)
              tma_ld(dst + T_ABYTES + x * 2048, &map_b, (int)n0 + 16 * x, (int)k0, (int)b, bar);
          } else {
            tma_ld(dst + T_ABYTES, &map_b, (int)k0, (int)n0, (int)b, bar);
          }
        }
      }
    }
  } else {
    // ------------------------------------------------------------------ consumers
    asm volatile("setmaxnreg.inc.sync.aligned.u32 232;\n" ::: "memory");
    const int wm = (warp / (TBN / TWN)) * TWM, wn = (warp % (TBN / TWN)) * TWN;
    const int fr = lane >> 2, fc = lane & 3;
    uint32_t it = 0;
    for (uint32_t ti = 0;; ++ti) {
      const uint32_t q = ti % TQ;
      mbw(su32(&tfull[q]), (ti / TQ) & 1);
      const int64_t t = *reinterpret_cast<volatile int64_t*>(&tids[q]);
      __syncwarp();
      if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(su32(&tempty[q])) : "memory");
      if (t >= g.total) break;
      int64_t b, tm, tn;
      tile_of(g, t, b, tm, tn);
      if (g.skip && g.skip[b]) continue;
      const int64_t m0 = tm * TBM, n0 = tn * TBN;
      int64_t klo, khi;
      krange(g, m0, n0, BN, klo, khi);
      double acc[TMI][TNI][2];
#pragma unroll
      for (int i = 0; i < TMI; ++i)
#pragma unroll
        for (int j = 0; j < TNI; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
      for (int64_t k0 = klo; k0 < khi; k0 += TK, ++it) {
        const uint32_t s = it % TSTAGES, ph = (it / TSTAGES) & 1;
        mbw(su32(&full[s]), ph);
        const unsigned char* sa = smem + s * T_STAGE;
        const unsigned char* sb = sa + T_ABYTES;
        // chunks that straddle a triangular operand's diagonal mask the
        // ignored triangle in the fragments (A lower: A(i,k) = 0 for k > i;
        // upper k < i; B lower: B(k,j) = 0 for k < j; upper k > j)
        const bool ma =
            (g.tri_a == TRI_LOWER && k0 + TK - 1 > m0 + wm) || (g.tri_a == TRI_UPPER && k0 < m0 + wm + TWM - 1);
        const bool mb =
            (g.tri_b == TRI_LOWER && k0 < n0 + wn + TWN - 1) || (g.tri_b == TRI_UPPER && k0 + TK - 1 > n0 + wn);
        if (!(ma || mb)) {  // the common case: plain loads, no per-element tests
#pragma unroll
          for (int kk = 0; kk < TK; kk += 4) {
            double af[TMI], bf[TNI];
#pragma unroll
            for (int i = 0; i < TMI; ++i)
              af[i] = *reinterpret_cast<const double*>(sa + opoff<AMN>(wm + fidx<AMN>(i, fr), kk + fc));
#pragma unroll
            for (int j = 0; j < TNI; ++j)
              bf[j] = *reinterpret_cast<const double*>(sb + opoff<BMN>(wn + fidx<BMN>(j, fr), kk + fc));
#pragma unroll
            for (int i = 0; i < TMI; ++i)
#pragma unroll
              for (int j = 0; j < TNI; ++j)
                asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                             : "+d"(acc[i][j][0]), "+d"(acc[i][j][1])
                             : "d"(af[i]), "d"(bf[j]));
          }
        } else {  // a chunk on a triangular operand's diagonal: mask the ignored triangle
          const int ko = (int)(k0 - m0), kn = (int)(k0 - n0);  // chunk k relative to the tile corner
#pragma unroll
          for (int kk = 0; kk < TK; kk += 4) {
            double af[TMI], bf[TNI];
#pragma unroll
            for (int i = 0; i < TMI; ++i) {
              const int r = wm + fidx<AMN>(i, fr), kr = ko + kk + fc;  // k - m0 vs row r
              double v = *reinterpret_cast<const double*>(sa + opoff<AMN>(r, kk + fc));
              if (g.tri_a == TRI_LOWER ? kr > r : (g.tri_a == TRI_UPPER && kr < r)) v = 0.0;
              af[i] = v;
            }
#pragma unroll
            for (int j = 0; j < TNI; ++j) {
              const int cc = wn + fidx<BMN>(j, fr), kc = kn + kk + fc;
              double v = *reinterpret_cast<const double*>(sb + opoff<BMN>(cc, kk + fc));
              if (g.tri_b == TRI_LOWER ? kc < cc : (g.tri_b == TRI_UPPER && kc > cc)) v = 0.0;
              bf[j] = v;
            }
#pragma unroll
            for (int i = 0; i < TMI; ++i)
#pragma unroll
              for (int j = 0; j < TNI; ++j)
                asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                             : "+d"(acc[i][j][0]), "+d"(acc[i][j][1])
                             : "d"(af[i]), "d"(bf[j]));
          }
        }
        __syncwarp();
        if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(su32(&empty[s])) : "memory");
      }
      // epilogue straight from registers (the producer is already filling the
      // ring with the next tile's chunks)
      double* C = g.c.p + b * g.c.bs;
      const bool vec = ((g.c.ld & 1) == 0) && ((reinterpret_cast<uintptr_t>(C) & 15) == 0);
#pragma unroll
      for (int i = 0; i < TMI; ++i) {
        const int64_t gi = m0 + wm + fidx<AMN>(i, fr);
        if (gi >= g.m) continue;
#pragma unroll
        for (int j = 0; j < TNI; ++j) {
          // C fragment columns 2 fc, 2 fc + 1 are B fragment columns (adjacent
          // in memory for MN-major B, 2 apart for K-major B)
          const int64_t gj0 = n0 + wn + fidx<BMN>(j, 2 * fc), gj1 = n0 + wn + fidx<BMN>(j, 2 * fc + 1);
          const bool ok0 = gj0 < g.n && !(g.mask == MASK_LOWER && gj0 > gi) && !(g.mask == MASK_UPPER && gj0 < gi);
          const bool ok1 = gj1 < g.n && !(g.mask == MASK_LOWER && gj1 > gi) && !(g.mask == MASK_UPPER && gj1 < gi);
          double* c0 = C + gi * g.c.ld + gj0;
          double* c1 = C + gi * g.c.ld + gj1;
          double v0 = g.alpha * acc[i][j][0], v1 = g.alpha * acc[i][j][1];
          if (g.beta != 0.0) {
            if (ok0) v0 += g.beta * *c0;
            if (ok1) v1 += g.beta * *c1;
          }
          if (BMN && vec && ok0 && ok1) {
            *reinterpret_cast<double2*>(c0) = make_double2(v0, v1);
          } else {
            if (ok0) *c0 = v0;
            if (ok1) *c1 = v1;
          }
        }
      }
    }
  }
  // the last CTA out re-arms the launch's counter slot
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    if (atomicAdd(&g_tma_tiles[slot][1], 1u) == gridDim.x - 1) {
      g_tma_tiles[slot][0] = 0;
      g_tma_tiles[slot][1] = 0;
      __threadfence();
    }
  }
}

PFN_cuTensorMapEncodeTiled_v12000 encode() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      p = nullptr;
    return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }();
  return fn;
}

// 3-D map (inner, outer, batch) over a row-major operand with leading
// dimension ld (the inner index contiguous); box = [box_outer][16 inner].
bool map3(CUtensorMap* map, const double* p, int64_t inner, int64_t outer, int64_t ld, int64_t bs, int64_t batch,
          int box_outer) {
  auto enc = encode();
  if (!enc) return false;
  cuuint64_t dims[3] = {(cuuint64_t)inner, (cuuint64_t)outer, (cuuint64_t)batch};
  cuuint64_t strides[2] = {(cuuint64_t)ld * 8, (cuuint64_t)(batch > 1 ? bs : outer * ld) * 8};
  cuuint32_t box[3] = {(cuuint32_t)TK, (cuuint32_t)box_outer, 1};
  cuuint32_t es[3] = {1, 1, 1};
  return enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, const_cast<double*>(p), dims, strides, box, es,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

std::atomic<unsigned> g_next_slot{0};
template <bool AMN, bool BMN, int BN>
void launch(const CUtensorMap& ma, const CUtensorMap& mb, const TmaArgs& g, int grid, cudaStream_t s) {
  const int slot = (int)(g_next_slot.fetch_add(1u) % TSLOTS);
  ensure_smem_attr(k_dgemm_tma<AMN, BMN, BN>, TT<BN>::SMEM);
  k_dgemm_tma<AMN, BMN, BN><<<grid, TTHREADS, TT<BN>::SMEM, s>>>(ma, mb, g, slot);
}
template <bool AMN, bool BMN>
void launch_bn(const CUtensorMap& ma, const CUtensorMap& mb, const TmaArgs& g, int grid, cudaStream_t s, int bn) {
  if (bn == 64) launch<AMN, BMN, 64>(ma, mb, g, grid, s);
  else launch<AMN, BMN, 128>(ma, mb, g, grid, s);
}

bool aligned_op(const MatB<const double>& x, int64_t batch) {
  return (reinterpret_cast<uintptr_t>(x.p) & 15) == 0 && (x.ld & 1) == 0 && (batch == 1 || (x.bs & 1) == 0) &&
         x.ld < ((int64_t)1 << 31) && x.bsi == 0;
}

}  // namespace

// Large fp64 products on the TMA kernel; false = not taken (the caller runs
// the generic kernel).  DLA_GEMM_TMA (tuning switch): 1 (default) plain
// products with >= 2 waves of 128 x 128 tiles, 2 every single-slab product
// with m, n, k >= 256 (tests), 0 never.
bool gemm_tma(const Ctx& c, int64_t batch, int64_t m, int64_t n, int64_t k, double alpha, MatB<const double> a,
              bool ta, MatB<const double> b, bool tb, double beta, MatB<double> cm, int mask, const int32_t* skip,
              int tri_a, int tri_b, int64_t inner, dla_status* st) {
  static const int on = [] {
    const char* e = getenv("DLA_GEMM_TMA");  // tuning switch: 0 = the cp.async kernel for every product
    return e ? atoi(e) : 1;
  }();
  if (!on || inner != 1 || k < 256 || m < 256 || n < 256 || batch > 65535) return false;
  // Measured against the cp.async kernel (tools/gemm_tri_time.py): plain
  // products with >= 2 waves of 128 x 128 tiles gain (4096^3: 32.3 vs 31.3
  // TF/s); the potrf pullback's triangular products run at parity or 2 %
  // behind (Z at n = 4096: 30.2 vs 31.0 TF/s) and batched 1024^3 products lose
  // to the finer 64 x 64 tiles -- so by default only the former take it
  // (DLA_GEMM_TMA=2: every eligible product).
  const bool plain = mask == MASK_FULL && tri_a == TRI_NONE && tri_b == TRI_NONE;
  if (on < 2 && (!plain || batch * ((m + TBM - 1) / TBM) * ((n + 127) / 128) < 2 * (int64_t)c.sms)) return false;
  if (mask == MASK_UPPER || (mask == MASK_LOWER && m != n)) return false;
  // triangular operands / masks: 128 x 64 tiles (half the wasted work on the
  // diagonal, twice the tiles to balance); plain products 128 x 128
  static const int bn_env = [] {
    const char* e = getenv("DLA_GEMM_TMA_BN");  // tuning switch: 64 / 128 force the tile width
    return e ? atoi(e) : 0;
  }();
  const int bn = bn_env == 64 || bn_env == 128
                     ? bn_env
                     : ((tri_a != TRI_NONE || tri_b != TRI_NONE || mask != MASK_FULL) ? 64 : 128);
  const int64_t tm = (m + TBM - 1) / TBM, tn = (n + bn - 1) / bn;
  // lower-masked: tile rows of 128 against columns of bn (bn divides 128)
  const int64_t per = mask == MASK_FULL ? tm * tn : (128 / bn) * tm * (tm + 1) / 2;
  if (batch * per < (int64_t)c.sms && on < 2) return false;
  if (!aligned_op(a, batch) || !aligned_op(b, batch)) return false;
  if ((reinterpret_cast<uintptr_t>(cm.p) & 15) != 0 || (cm.ld & 1) != 0 || (batch > 1 && (cm.bs & 1) != 0))
    return false;
  if (!encode()) return false;
  CUtensorMap ma, mb;
  // A: op(A)(i, k); !ta: A is m x k row-major (K-major); ta: A is k x m (M-major)
  const bool okA = !ta ? map3(&ma, a.p, k, m, a.ld, a.bs, batch, TBM) : map3(&ma, a.p, m, k, a.ld, a.bs, batch, TK);
  // B: op(B)(k, j); !tb: B is k x n (N-major); tb: B is n x k (K-major)
  const bool okB = !tb ? map3(&mb, b.p, n, k, b.ld, b.bs, batch, TK) : map3(&mb, b.p, k, n, b.ld, b.bs, batch, bn);
  if (!okA || !okB) return false;
  TmaArgs g;
  g.m = m;
  g.n = n;
  g.k = k;
  g.batch = batch;
  g.tm = tm;
  g.tn = tn;
  g.per = per;
  g.ratio = 128 / bn;
  g.total = per * batch;
  g.alpha = alpha;
  g.beta = beta;
  g.c = cm;
  g.mask = mask;
  g.tri_a = tri_a;
  g.tri_b = tri_b;
  g.skip = skip;
  const int grid = (int)std::min<int64_t>(g.total, c.sms);
  if (!ta && !tb) launch_bn<false, true>(ma, mb, g, grid, c.stream, bn);
  else if (ta && !tb) launch_bn<true, true>(ma, mb, g, grid, c.stream, bn);
  else if (!ta && tb) launch_bn<false, false>(ma, mb, g, grid, c.stream, bn);
  else launch_bn<true, false>(ma, mb, g, grid, c.stream, bn);
  const cudaError_t e = cudaGetLastError();
  *st = e == cudaSuccess ? DLA_OK : DLA_ERR_CUDA;
  note_launch(1);
  return true;
}

}  // namespace dlab
