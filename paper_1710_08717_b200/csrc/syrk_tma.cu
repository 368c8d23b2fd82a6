// Trailing rank-K update of the blocked Cholesky (f64), TMA-fed and
// warp-specialised:   C[lower] = alpha * P P^T + beta * C,   P = m x K.
//
// The right-looking factorization (dl/cholesky.hpp:43-70) re-reads and
// re-writes the whole trailing triangle once per 64-column panel.  At
// K = 64 each 128 x 64 C tile carries only 1 MFLOP against 64 KB of C read +
// 64 KB written, so a tile-per-CTA GEMM serialises its operand prologue, its
// DMMA main loop and its C read-modify-write (ncu: tensor pipe ~48 % active).
// Here one persistent CTA per SM streams tile after tile:
//
//   * warp 8 (producer): cp.async.bulk.tensor (TMA, SASS UTMALDG) of the
//     16-column k-chunks of P's tile rows (A: 128 rows, B: 64 rows) into a
//     4-stage ring of 128B-swizzled shared buffers, mbarrier transaction
//     counts; the ring runs across tile boundaries, so the next tile's
//     operands land while the current tile finishes;
//     After a tile's k-chunks it also loads that tile's C (4 swizzled 128 x 16
//     boxes, 64 KB) into a C buffer, which lands under the tile's main loop;
//   * warps 0-7 (consumers, 4 x 2 of 32 x 32 warp tiles): FP64 DMMA
//     (mma.sync m8n8k4) from the swizzled buffers (conflict-free fragment
//     loads: the 128B swizzle XORs the 16-byte chunk with row & 7), release
//     each stage with one arrive per warp, then C = alpha acc + beta C from
//     the C buffer, stored (lower triangle only) straight from registers.
//
// Only the lower tiles are enumerated (no dead CTAs); rows / k beyond the
// operand are zero-filled by the TMA unit.  The grid may be capped so the
// concurrently running panel kernel of the look-ahead keeps its SMs.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <cmath>
#include <mutex>

#include "common.cuh"
#include "ops.cuh"

namespace dlab {
namespace {

constexpr int SKC = 16;

// CTA tile 128 x BN, consumer warp tile WM x WN (8 warps), ST k-chunk stages.
template <int BM_, int BN_, int WM_, int WN_, int ST_, int NCB_, int MINB_>
struct SCfg {
  static constexpr int BM = BM_, BN = BN_, WM = WM_, WN = WN_, ST = ST_, NCB = NCB_, MINB = MINB_;
  static constexpr int CONS = (BM / WM) * (BN / WN);  // consumer warps; + one producer warp
  static constexpr int THREADS = (CONS + 1) * 32;
  static constexpr int WARPS_N = BN / WN, MI = WM / 8, NI = WN / 8;
  static constexpr int A_BYTES = BM * SKC * 8, B_BYTES = BN * SKC * 8;
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int C_BYTES = BM * BN * 8;  // BN / 16 swizzled BM x 16 boxes
  static constexpr size_t SMEM = (size_t)ST * STAGE_BYTES + NCB * C_BYTES + 1024 + (2 * ST + 2 * NCB) * 8;
};
using SCfgA = SCfg<128, 64, 32, 32, 4, 2, 1>;  // 128 x 64 tiles, 8 consumer warps, double-buffered C, 1 CTA/SM
using SCfgB = SCfg<64, 64, 32, 32, 4, 1, 2>;   // 64 x 64 tiles, 4 consumer warps, 2 CTAs/SM (epilogues interleave)

struct SyrkArgs {
  int64_t m, k, batch;
  int64_t tm;        // tile rows per slice
  int64_t tn;        // tile columns per slice
  int64_t ratio;     // BM / BN: row r of tiles holds ratio * (r + 1) lower tiles
  int64_t per;       // lower tiles per slice
  int64_t total;     // per * batch
  double alpha, beta;
  MatB<double> c;    // C (m x m, lower)
};

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mb_wait(uint32_t bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "W_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra W_%=;\n\t}\n" ::"r"(bar),
      "r"(parity)
      : "memory");
}

__device__ __forceinline__ void tma3(uint32_t dst, const CUtensorMap* map, int c0, int c1, int c2, uint32_t bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];\n" ::"r"(
          dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(bar)
      : "memory");
}

// Lower tile `t` of a slice (row-major over tile rows; row r holds tiles
// 0 .. min(R (r + 1), tn) - 1 with R = BM / BN).
__device__ __forceinline__ bool decode_lower(const SyrkArgs& g, int64_t t, int64_t& b, int64_t& tm, int64_t& tnn) {
  b = t / g.per;
  t -= b * g.per;
  const int64_t R = g.ratio;
  int64_t r = (int64_t)((sqrt(8.0 * (double)t / (double)R + 1.0) - 1.0) * 0.5);
  while (R * r * (r + 1) / 2 > t) --r;
  while (R * (r + 1) * (r + 2) / 2 <= t) ++r;
  tm = r;
  tnn = t - R * r * (r + 1) / 2;
  return tnn < g.tn;
}


// Fragment row fr -> box row: rows r and r ^ 1 of a [rows][16] 128B-swizzled
// box share their XOR'd chunk pair, so 8 consecutive rows at 4 consecutive k
// take each bank segment twice; half-warp h takes rows {0, 2, 4, 6} + h of
// the 8-row group instead (four disjoint 32-byte segments: conflict-free).
__device__ __forceinline__ int fperm(int fr) { return 2 * (fr & 3) + (fr >> 2); }

// byte offset of element (row, k) in a [rows][16 doubles] 128B-swizzled box
__device__ __forceinline__ uint32_t swz(int row, int k) {
  return (uint32_t)(row * 128 + ((((k >> 1) ^ (row & 7))) << 4) + ((k & 1) << 3));
}

__device__ __forceinline__ void tma3_store(const CUtensorMap* map, int c0, int c1, int c2, uint32_t src) {
  asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%1, %2, %3}], [%4];\n" ::"l"(
                   reinterpret_cast<uint64_t>(map)),
               "r"(c0), "r"(c1), "r"(c2), "r"(src)
               : "memory");
}

template <class CF>
__global__ void __launch_bounds__(CF::THREADS, CF::MINB)
    k_syrk_tma(const __grid_constant__ CUtensorMap map_a, const __grid_constant__ CUtensorMap map_b,
               const __grid_constant__ CUtensorMap map_c, SyrkArgs g) {
  constexpr int SBM = CF::BM, SCONS = CF::CONS;
  constexpr int SBN = CF::BN, SST = CF::ST, NCB = CF::NCB, A_BYTES = CF::A_BYTES, STAGE_BYTES = CF::STAGE_BYTES,
                C_BYTES = CF::C_BYTES, MI = CF::MI, NI = CF::NI;
  constexpr int BOX = SBM * SKC * 8;  // one BM x 16 swizzled box
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* smem = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~(uintptr_t)1023);
  unsigned char* csm0 = smem + SST * STAGE_BYTES;
  uint64_t* full = reinterpret_cast<uint64_t*>(csm0 + NCB * C_BYTES);
  uint64_t* empty = full + SST;
  uint64_t* cfull = empty + SST;
  uint64_t* cempty = cfull + NCB;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nk = (int)((g.k + SKC - 1) / SKC);
  const bool use_c = g.beta != 0.0;
  const int64_t ntile = g.total > blockIdx.x ? (g.total - 1 - blockIdx.x) / gridDim.x + 1 : 0;
  if (threadIdx.x == 0) {
    for (int s = 0; s < SST; ++s) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(su32(&full[s])));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(su32(&empty[s])), "r"(SCONS));
    }
    for (int q = 0; q < NCB; ++q) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(su32(&cfull[q])));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(su32(&cempty[q])));
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();

  if (warp == SCONS) {  // ---------------------------------------------- producer
    if (lane == 0) {
      asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<uint64_t>(&map_a)) : "memory");
      asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<uint64_t>(&map_b)) : "memory");
      asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<uint64_t>(&map_c)) : "memory");
      uint32_t it = 0;
      for (int64_t ti = 0; ti < ntile; ++ti) {
        int64_t b, tm, tnn;
        decode_lower(g, blockIdx.x + ti * gridDim.x, b, tm, tnn);  // clipped tiles: zero operands, nothing stored
        for (int kc = 0; kc < nk; ++kc, ++it) {
          const uint32_t s = it % SST, ph = (it / SST) & 1;
          mb_wait(su32(&empty[s]), ph ^ 1);
          const uint32_t bar = su32(&full[s]);
          asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(bar), "r"(STAGE_BYTES)
                       : "memory");
          const uint32_t dst = su32(smem + s * STAGE_BYTES);
          tma3(dst, &map_a, kc * SKC, (int)(tm * SBM), (int)b, bar);
          tma3(dst + A_BYTES, &map_b, kc * SKC, (int)(tnn * SBN), (int)b, bar);
        }
        if (use_c) {  // the tile's C, into C buffer ti % NCB once its previous store has been read out
          const int q = (int)(ti % NCB);
          mb_wait(su32(&cempty[q]), (uint32_t)(((ti / NCB) & 1) ^ 1));
          const uint32_t bar = su32(&cfull[q]);
          asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(bar), "r"(C_BYTES) : "memory");
#pragma unroll
          for (int x = 0; x < SBN / SKC; ++x)
            tma3(su32(csm0 + q * C_BYTES + x * BOX), &map_c, (int)(tnn * SBN) + x * SKC, (int)(tm * SBM), (int)b, bar);
        }
      }
    }
    return;
  }

  // ------------------------------------------------------------------ consumers
  const int wm = (warp / CF::WARPS_N) * CF::WM, wn = (warp % CF::WARPS_N) * CF::WN;
  const int fr = lane >> 2, fc = lane & 3;
  uint32_t it = 0;
  for (int64_t ti = 0; ti < ntile; ++ti) {
    int64_t b, tm, tnn;
    decode_lower(g, blockIdx.x + ti * gridDim.x, b, tm, tnn);
    const int64_t m0 = tm * SBM, n0 = tnn * SBN;
    double acc[MI][NI][2];
#pragma unroll
    for (int i = 0; i < MI; ++i)
#pragma unroll
      for (int j = 0; j < NI; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
    for (int kc = 0; kc < nk; ++kc, ++it) {
      const uint32_t s = it % SST, ph = (it / SST) & 1;
      mb_wait(su32(&full[s]), ph);
      const unsigned char* sa = smem + s * STAGE_BYTES;
      const unsigned char* sb = sa + A_BYTES;
#pragma unroll
      for (int kk = 0; kk < SKC; kk += 4) {
        double af[MI], bf[NI];
#pragma unroll
        for (int i = 0; i < MI; ++i)
          af[i] = *reinterpret_cast<const double*>(sa + swz(wm + i * 8 + fperm(fr), kk + fc));
#pragma unroll
        for (int j = 0; j < NI; ++j)
          bf[j] = *reinterpret_cast<const double*>(sb + swz(wn + j * 8 + fperm(fr), kk + fc));
#pragma unroll
        for (int i = 0; i < MI; ++i)
#pragma unroll
          for (int j = 0; j < NI; ++j)
            asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                         : "+d"(acc[i][j][0]), "+d"(acc[i][j][1])
                         : "d"(af[i]), "d"(bf[j]));
      }
      __syncwarp();
      if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(su32(&empty[s])) : "memory");
    }
    // Epilogue, in place in C buffer q: alpha acc + beta C on the lower
    // triangle, C (beta != 0) or the symmetric product itself (beta == 0, the
    // caller mirrors) above it; then ONE thread stores the tile with TMA
    // (out-of-range rows / columns are clipped by the unit) and the warps move
    // on to the next tile while the store drains.
    const int q = (int)(ti % NCB);
    unsigned char* cb = csm0 + q * C_BYTES;
    if (use_c) mb_wait(su32(&cfull[q]), (uint32_t)((ti / NCB) & 1));
    else asm volatile("bar.sync 1, %0;\n" ::"n"(SCONS * 32) : "memory");  // buffer q's last store has been read out
#pragma unroll
    for (int i = 0; i < MI; ++i) {
      const int rl = wm + i * 8 + fperm(fr);  // tile row of this lane's accumulator row
      const int64_t gi = m0 + rl;
#pragma unroll
      for (int j = 0; j < NI; ++j) {
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int cl = wn + j * 8 + fperm(2 * fc + e);  // accumulator column -> tile column
          const int64_t gj = n0 + cl;
          double* cp = reinterpret_cast<double*>(cb + (cl >> 4) * BOX + swz(rl, cl & 15));
          double v;
          if (use_c) {
            const double cv = *cp;
            v = gj <= gi ? g.alpha * acc[i][j][e] + g.beta * cv : cv;
          } else {
            v = g.alpha * acc[i][j][e];
          }
          *cp = v;
        }
      }
    }
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
    asm volatile("bar.sync 1, %0;\n" ::"n"(SCONS * 32) : "memory");
    if (threadIdx.x == 0) {
#pragma unroll
      for (int x = 0; x < SBN / SKC; ++x)
        tma3_store(&map_c, (int)n0 + x * SKC, (int)m0, (int)b, su32(cb + x * BOX));
      asm volatile("cp.async.bulk.commit_group;\n" ::: "memory");
      // the store issued NCB - 1 tiles ago has been read out of its buffer
      asm volatile("cp.async.bulk.wait_group.read %0;\n" ::"n"(NCB - 1) : "memory");
      if (use_c && ti + 1 >= NCB) {
        const int qp = (int)((ti + 1) % NCB);
        asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(su32(&cempty[qp])) : "memory");
      }
    }
  }
  if (threadIdx.x == 0) asm volatile("cp.async.bulk.wait_group 0;\n" ::: "memory");
}

// cuTensorMapEncodeTiled through the runtime's driver entry point (no -lcuda).
PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
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

bool make_map(CUtensorMap* map, const double* p, int64_t rows, int64_t cols, int64_t ld, int64_t bs, int64_t batch,
              int box_rows) {
  auto enc = encode_fn();
  if (!enc) return false;
  cuuint64_t dims[3] = {(cuuint64_t)cols, (cuuint64_t)rows, (cuuint64_t)batch};
  cuuint64_t strides[2] = {(cuuint64_t)ld * 8, (cuuint64_t)(batch > 1 ? bs : rows * ld) * 8};
  cuuint32_t box[3] = {(cuuint32_t)SKC, (cuuint32_t)box_rows, 1};
  cuuint32_t es[3] = {1, 1, 1};
  return enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, const_cast<double*>(p), dims, strides, box, es,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

}  // namespace

bool syrk_tma_eligible(int64_t m, int64_t k, const MatB<const double>& p, const MatB<double>& c, int64_t batch) {
  static const bool on = [] {
    const char* e = getenv("DLA_SYRK_TMA");  // tuning switch: 0 keeps the trailing update on the generic GEMM
    return e ? atoi(e) != 0 : true;
  }();
  if (!on || m < 256 || k < 1 || k > 256) return false;
  if ((reinterpret_cast<uintptr_t>(p.p) & 15) != 0 || (p.ld & 1) != 0 || (batch > 1 && (p.bs & 1) != 0)) return false;
  if ((reinterpret_cast<uintptr_t>(c.p) & 15) != 0 || (c.ld & 1) != 0 || (batch > 1 && (c.bs & 1) != 0)) return false;
  if (m > (int64_t)1 << 31 || batch > 65535) return false;
  return encode_fn() != nullptr;
}

// C[lower] = alpha P P^T + beta C; P m x k (row-major, ld), C m x m.
// max_ctas > 0 caps the persistent grid (the look-ahead leaves the panel its SMs).
dla_status syrk_tma(const Ctx& c, int64_t batch, int64_t m, int64_t k, double alpha, MatB<const double> p, double beta,
                    MatB<double> cm, int max_ctas) {
  if (batch <= 0 || m <= 0) return DLA_OK;
  static const int cfg = [] {
    const char* e = getenv("DLA_SYRK_CFG");  // tuning switch: 0 = 128 x 64 tiles, 1 = 128 x 128 tiles
    return e ? atoi(e) : 0;
  }();
  const int bm = cfg == 1 ? SCfgB::BM : SCfgA::BM, bn = cfg == 1 ? SCfgB::BN : SCfgA::BN;
  const int per_sm = cfg == 1 ? SCfgB::MINB : SCfgA::MINB;
  CUtensorMap ma, mb, mc;
  if (!make_map(&ma, p.p, m, k, p.ld, p.bs, batch, bm) || !make_map(&mb, p.p, m, k, p.ld, p.bs, batch, bn) ||
      !make_map(&mc, cm.p, m, m, cm.ld, cm.bs, batch, bm))
    return DLA_ERR_CUDA;
  SyrkArgs g;
  g.m = m;
  g.k = k;
  g.batch = batch;
  g.tm = (m + bm - 1) / bm;
  g.tn = (m + bn - 1) / bn;
  g.ratio = bm / bn;
  g.per = g.ratio * g.tm * (g.tm + 1) / 2;
  g.total = g.per * batch;
  g.alpha = alpha;
  g.beta = beta;
  g.c = cm;
  int grid = c.sms * per_sm;
  if (max_ctas > 0 && max_ctas * per_sm < grid) grid = max_ctas * per_sm;
  if ((int64_t)grid > g.total) grid = (int)g.total;
  if (cfg == 1) {
    ensure_smem_attr(k_syrk_tma<SCfgB>, SCfgB::SMEM);
    k_syrk_tma<SCfgB><<<grid, SCfgB::THREADS, SCfgB::SMEM, c.stream>>>(ma, mb, mc, g);
  } else {
    ensure_smem_attr(k_syrk_tma<SCfgA>, SCfgA::SMEM);
    k_syrk_tma<SCfgA><<<grid, SCfgA::THREADS, SCfgA::SMEM, c.stream>>>(ma, mb, mc, g);
  }
  DLAB_LAUNCH_CHECK();
  note_launch(1);
  return DLA_OK;
}

}  // namespace dlab
