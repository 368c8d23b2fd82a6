// fp32 GEMM on the 5th-generation tensor cores: tcgen05.mma kind::tf32 with
// 3xTF32 splitting (a = a_hi + a_lo, both TF32; C += a_hi b_hi + a_hi b_lo +
// a_lo b_hi), which keeps binary32-level accuracy (the dropped a_lo b_lo term
// is ~2^-22 relative) while running on the tensor pipe.  This is the fp32
// policy of the large products; small / skinny fp32 products
// stay on the exact FFMA kernels.
//
// A packing pass writes each operand once as TF32 hi / lo tiles (128 x 32,
// the canonical no-swizzle K-major UMMA layout, zero-padded, transposed when
// the operand's m / n is the contiguous dimension).  The GEMM then moves
// whole tiles with bulk async copies (TMA bulk engine) into a 4-stage shared
// ring (k-block 16), one lane issues tcgen05.mma (UMMA 128 x 256 x 8, three
// products per k-step) with the accumulator in TMEM (256 columns), and 4 warps
// run the epilogue.  One CTA per 128 x 256 output tile.  Measured on B200 at
// 4096^3: 201.8 TFLOP/s fp32-accurate (128 x 128 tiles / k-block 32 / 3
// stages: 190.7; k-block 8 / 8 stages: 140).
// Triangular operands, batching, alpha / beta and the lower / upper write
// masks are handled in staging and in the epilogue, like gemm.cu.
#include "common.cuh"

namespace dlab {
namespace {

#ifndef DLAB_TC_TK
#define DLAB_TC_TK 16
#endif
#ifndef DLAB_TC_ST
#define DLAB_TC_ST 4
#endif
constexpr int TM = 128, TN = 128, TK = DLAB_TC_TK, TT = 128;
constexpr uint32_t KSBO = (TK / 4) * 128;  // K-major tile: bytes between 8-row groups
constexpr int TNC = 256;  // CTA tile N: two packed 128-row B tiles per MMA (UMMA N = 256)
constexpr int TILE_F = TM * TK;  // floats per staged operand tile (A and B tiles are the same size)

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ float tf32_rna(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return __uint_as_float(r);
}

// Canonical no-swizzle K-major layout (uint128 = 4 floats): core matrix =
// 8 rows x 4 k, [row/8][k/4][row%8][k%4]; LBO (k direction) = 128 B, SBO (row
// direction) = 8 * 128 B.  Operands whose m / n is the contiguous global
// dimension are loaded along it (coalesced) and transposed on the store.
__device__ __forceinline__ int off_kmajor(int row, int k) {
  return ((row >> 3) * (TK / 4) + (k >> 2)) * 32 + (row & 7) * 4 + (k & 3);
}

__device__ __forceinline__ uint64_t make_sdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;  // descriptor version (sm_100)
  // base offset 0, legacy LBO mode, layout type 0 = SWIZZLE_NONE
  return d;
}

__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n\t}\n" ::"r"(bar),
      "r"(parity));
}

__device__ __forceinline__ void mma_tf32(uint32_t tmem, uint64_t da, uint64_t db, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem),
      "l"(da), "l"(db), "r"(idesc), "r"(acc));
}

// ---------------------------------------------------------------- packing
// op(X) (rows x kdim, batch) -> tiles [batch][rt][kt][hi | lo][TILE_F] in the
// canonical K-major order, split into TF32 hi / lo, zero-padded, triangle
// masked.  One CTA per 128 x 32 tile; coalesced loads along X's contiguous
// dimension through a padded shared tile, coalesced float4 stores.
template <bool KCONTIG>
__global__ void __launch_bounds__(256) k_tf32_pack(const float* X, int64_t ld, int64_t xbs, int64_t rows, int64_t kdim,
                                                   int tri, int64_t rt_n, int64_t kt_n, const int32_t* skip,
                                                   float* out) {
  __shared__ float T[TM][TK + 1];
  int64_t t = blockIdx.x;
  const int64_t kt = t % kt_n;
  t /= kt_n;
  const int64_t rt = t % rt_n, b = t / rt_n;
  float* o = out + (size_t)blockIdx.x * 2 * TILE_F;
  if (skip && skip[b]) return;
  const float* Xb = X + b * xbs;
  const int64_t r0 = rt * TM, k0 = kt * TK;
  for (int e = threadIdx.x; e < TM * TK; e += 256) {
    int row, k;
    if (KCONTIG) {
      row = e / TK;
      k = e % TK;
    } else {
      k = e / TM;
      row = e % TM;
    }
    const int64_t gr = r0 + row, gk = k0 + k;
    bool ok = gr < rows && gk < kdim;
    if (tri == TRI_LOWER) ok = ok && gk <= gr;
    if (tri == TRI_UPPER) ok = ok && gk >= gr;
    T[row][k] = ok ? (KCONTIG ? Xb[gr * ld + gk] : Xb[gk * ld + gr]) : 0.f;
  }
  __syncthreads();
  for (int g4 = threadIdx.x; g4 < TILE_F / 4; g4 += 256) {
    const int cm = g4 >> 3, r8 = g4 & 7;
    const int row = (cm / (TK / 4)) * 8 + r8, k = (cm % (TK / 4)) * 4;
    float h[4], l[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const float v = T[row][k + e];
      h[e] = tf32_rna(v);
      l[e] = tf32_rna(v - h[e]);
    }
    reinterpret_cast<float4*>(o)[g4] = make_float4(h[0], h[1], h[2], h[3]);
    reinterpret_cast<float4*>(o + TILE_F)[g4] = make_float4(l[0], l[1], l[2], l[3]);
  }
}

// ------------------------------------------------------------------ GEMM
// Warp-specialised pipeline over packed tiles: warp 0 (one lane) moves each
// k-block's four 16 KB tiles (A hi/lo, B hi/lo) into a 3-stage shared ring
// with bulk async copies (TMA bulk engine, mbarrier transaction counts);
// warp 1 (one lane) issues the 12 tcgen05.mma of a stage and commits them to
// the stage's "empty" barrier; all four warps run the TMEM epilogue.
constexpr int TCST = DLAB_TC_ST;
constexpr uint32_t A_BYTES = 2 * TILE_F * 4;                // A hi | A lo (128 rows)
constexpr uint32_t B_BYTES = 2 * (TNC / TN) * TILE_F * 4;   // B hi (256 rows) | B lo (256 rows)
constexpr uint32_t STAGE_BYTES = A_BYTES + B_BYTES;

struct TcArgs2 {
  int64_t m, n;
  float alpha, beta;
  const float *ap, *bp;  // packed operands
  int64_t art, akt, brt, bkt;
  MatB<float> c;
  int mask;
  const int32_t* skip;
  int64_t tiles_m, tiles_n;
  int tri_a, tri_b;
  int64_t kdim;
};

__device__ __forceinline__ void mbar_arrive_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(dst),
               "l"(src), "r"(bytes), "r"(bar)
               : "memory");
}

__global__ void __launch_bounds__(TT, 1) k_sgemm_tc(TcArgs2 g) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  __shared__ __align__(8) uint64_t full[TCST], empty[TCST], done;
  __shared__ uint32_t tmem_base;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  int64_t tile = blockIdx.x;
  const int64_t per = g.tiles_m * g.tiles_n;
  const int64_t b = tile / per;
  tile -= b * per;
  const int64_t mt = tile / g.tiles_n, nt = tile % g.tiles_n;
  const int64_t m0 = mt * TM, n0 = nt * TNC;
  if (g.skip && g.skip[b]) return;
  if (g.mask == MASK_LOWER && n0 > m0 + TM - 1) return;
  if (g.mask == MASK_UPPER && m0 > n0 + TNC - 1) return;
  int64_t klo = 0, khi = g.kdim;
  if (g.tri_a == TRI_LOWER) khi = min(khi, m0 + TM);
  if (g.tri_a == TRI_UPPER) klo = max(klo, m0);
  if (g.tri_b == TRI_LOWER) klo = max(klo, n0);
  if (g.tri_b == TRI_UPPER) khi = min(khi, n0 + TNC);
  const int64_t kt0 = klo / TK;
  const int64_t nk = khi > kt0 * TK ? (khi - kt0 * TK + TK - 1) / TK : 0;

  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_u32(&tmem_base)),
                 "r"(TNC));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  if (tid == 0) {
    for (int s = 0; s < TCST; ++s) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(smem_u32(&full[s])));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(smem_u32(&empty[s])));
    }
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(smem_u32(&done)));
    asm volatile("fence.mbarrier_init.release.cluster;\n");
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n");
  const uint32_t tmem = tmem_base;
  const uint32_t sbase = smem_u32(smem_raw);

  if (warp == 0 && lane == 0) {  // producer
    const float* at = g.ap + (size_t)((b * g.art + mt) * g.akt) * 2 * TILE_F;
    const int64_t rt0 = nt * (TNC / TN);
    const int nsub = (int)min((int64_t)(TNC / TN), g.brt - rt0);  // B sub-tiles that exist (the rest: unused columns)
    for (int64_t kb = 0; kb < nk; ++kb) {
      const int s = (int)(kb % TCST);
      if (kb >= TCST) mbar_wait(smem_u32(&empty[s]), (uint32_t)(((kb / TCST) - 1) & 1));
      const uint32_t dst = sbase + (uint32_t)s * STAGE_BYTES;
      mbar_arrive_tx(smem_u32(&full[s]), A_BYTES + (uint32_t)nsub * 2 * TILE_F * 4);
      bulk_g2s(dst, at + (size_t)(kt0 + kb) * 2 * TILE_F, A_BYTES, smem_u32(&full[s]));
      for (int j = 0; j < nsub; ++j) {
        const float* bt = g.bp + (size_t)(((b * g.brt + rt0 + j) * g.bkt) + kt0 + kb) * 2 * TILE_F;
        bulk_g2s(dst + A_BYTES + j * TILE_F * 4, bt, TILE_F * 4, smem_u32(&full[s]));
        bulk_g2s(dst + A_BYTES + B_BYTES / 2 + j * TILE_F * 4, bt + TILE_F, TILE_F * 4, smem_u32(&full[s]));
      }
    }
  } else if (warp == 1 && lane == 0) {  // MMA issuer
    const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(TNC >> 3) << 17) | ((uint32_t)(TM >> 4) << 24);
    for (int64_t kb = 0; kb < nk; ++kb) {
      const int s = (int)(kb % TCST);
      mbar_wait(smem_u32(&full[s]), (uint32_t)((kb / TCST) & 1));
      asm volatile("tcgen05.fence::after_thread_sync;\n");
      const uint32_t st = sbase + (uint32_t)s * STAGE_BYTES;
      const uint32_t ahi = st, alo = st + TILE_F * 4, bhi = st + A_BYTES, blo = st + A_BYTES + B_BYTES / 2;
#pragma unroll
      for (int ks = 0; ks < TK / 8; ++ks) {
        const uint64_t dah = make_sdesc(ahi + ks * 256, 128, KSBO);
        const uint64_t dal = make_sdesc(alo + ks * 256, 128, KSBO);
        const uint64_t dbh = make_sdesc(bhi + ks * 256, 128, KSBO);
        const uint64_t dbl = make_sdesc(blo + ks * 256, 128, KSBO);
        const uint32_t acc = (kb == 0 && ks == 0) ? 0u : 1u;
        mma_tf32(tmem, dal, dbh, idesc, acc);  // small terms first
        mma_tf32(tmem, dah, dbl, idesc, 1u);
        mma_tf32(tmem, dah, dbh, idesc, 1u);
      }
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
          smem_u32(&empty[s])));
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
        smem_u32(&done)));
  }
  __syncwarp();
  if (nk > 0) mbar_wait(smem_u32(&done), 0u);
  asm volatile("tcgen05.fence::after_thread_sync;\n");

  // epilogue: warp w owns TMEM lanes (= rows) 32w .. 32w+31
  const int64_t gi = m0 + warp * 32 + lane;
  float* C = g.c.p + b * g.c.bs;
  for (int c0 = 0; c0 < TNC; c0 += 32) {
    uint32_t r[32];
    const uint32_t taddr = tmem + ((uint32_t)(warp * 32) << 16) + (uint32_t)c0;
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,"
        "%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];\n"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
          "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]),
          "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
          "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;\n");
    if (gi < g.m) {
      float* crow = C + gi * g.c.ld;
#pragma unroll
      for (int j = 0; j < 32; ++j) {
        const int64_t gj = n0 + c0 + j;
        if (gj >= g.n) break;
        if (g.mask == MASK_LOWER && gj > gi) continue;
        if (g.mask == MASK_UPPER && gj < gi) continue;
        float v = g.alpha * (nk > 0 ? __uint_as_float(r[j]) : 0.f);
        if (g.beta != 0.f) v += g.beta * crow[gj];
        crow[gj] = v;
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "r"(TNC));
}

}  // namespace

// Packed hi/lo TF32 operand tiles of one call (the k_tf32_pack output).
size_t sgemm_tc_ws_bytes(int64_t batch, int64_t m, int64_t n, int64_t k) {
  const int64_t art = (m + TM - 1) / TM, brt = (n + TN - 1) / TN, kt = (k + TK - 1) / TK;
  return sizeof(float) * 2 * TILE_F * (size_t)(batch * kt * (art + brt));
}

// C = alpha op(A) op(B) + beta C on tcgen05 (3xTF32).  Returns false if the
// problem is outside this kernel's scope (the caller uses the FFMA GEMM).
bool sgemm_tc(const Ctx& c, int64_t batch, int64_t m, int64_t n, int64_t k, float alpha, MatB<const float> a, bool ta,
              MatB<const float> b, bool tb, float beta, MatB<float> cm, int mask, const int32_t* skip, int tri_a,
              int tri_b, int64_t inner, dla_status* st) {
  if (inner != 1) return false;
  *st = DLA_OK;
  const int64_t art = (m + TM - 1) / TM, brt = (n + TN - 1) / TN, kt = (k + TK - 1) / TK;
  Scratch ws(c, sgemm_tc_ws_bytes(batch, m, n, k));
  if (!ws.ok) {
    *st = DLA_ERR_WORKSPACE;
    return true;
  }
  float* apk = ws.as<float>();
  float* bpk = apk + (size_t)(batch * art * kt) * 2 * TILE_F;
  // op(A) rows x k: k contiguous iff !ta; the B operand is op(B)^T (n x k): k contiguous iff tb
  const int tri_bv = tri_b == TRI_LOWER ? TRI_UPPER : (tri_b == TRI_UPPER ? TRI_LOWER : TRI_NONE);
  if (!ta)
    k_tf32_pack<true><<<(unsigned)(batch * art * kt), 256, 0, c.stream>>>(a.p, a.ld, a.bs, m, k, tri_a, art, kt, skip, apk);
  else
    k_tf32_pack<false><<<(unsigned)(batch * art * kt), 256, 0, c.stream>>>(a.p, a.ld, a.bs, m, k, tri_a, art, kt, skip, apk);
  if (tb)
    k_tf32_pack<true><<<(unsigned)(batch * brt * kt), 256, 0, c.stream>>>(b.p, b.ld, b.bs, n, k, tri_bv, brt, kt, skip, bpk);
  else
    k_tf32_pack<false><<<(unsigned)(batch * brt * kt), 256, 0, c.stream>>>(b.p, b.ld, b.bs, n, k, tri_bv, brt, kt, skip, bpk);
  const int64_t ctn = (n + TNC - 1) / TNC;
  TcArgs2 g{m, n, alpha, beta, apk, bpk, art, kt, brt, kt, cm, mask, skip, art, ctn, tri_a, tri_b, k};
  const size_t smem = (size_t)TCST * STAGE_BYTES;
  ensure_smem_attr(k_sgemm_tc, smem);
  k_sgemm_tc<<<(unsigned)(batch * art * ctn), TT, smem, c.stream>>>(g);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    fprintf(stderr, "dla_b200 sgemm_tc: %s\n", cudaGetErrorString(e));
    *st = DLA_ERR_CUDA;
  }
  note_launch(3);
  return true;
}

}  // namespace dlab
