// Cholesky of one n <= 64 block held in shared memory by a CTA of >= 64
// threads (dl/cholesky.hpp:35-72 reordered for the GPU).
//
// The pivot chain is the critical path of any Cholesky (n dependent
// sqrt/div pairs).  Here it never crosses a block barrier: the block is
// processed in 16-column panels, each factored by ONE warp entirely in
// registers (lane l holds panel rows l and l + 32; pivots and multipliers move
// by warp shuffles; every lane takes the sqrt and the reciprocal itself), and
// the CTA's warps then apply the panel to the trailing lower triangle with
// plain DFMA.  Two barriers per 16 columns instead of one per column.
#pragma once

#include "common.cuh"

namespace dlab {

constexpr int CH_LD = 65;  // smem row stride for a 64 x 64 block

// S: n x n block in shared memory (row stride CH_LD), lower triangle valid.
// On return S holds L in its lower triangle.  Returns the first failing pivot
// (uniform across the CTA) or -1.  `flag` is one shared int.
template <typename T>
__device__ __forceinline__ int chol_smem64(T* S, int n, int* flag) {
  constexpr int W = 16;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nthreads = blockDim.x;
  if (threadIdx.x == 0) *flag = -1;
  __syncthreads();
  for (int p0 = 0; p0 < n; p0 += W) {
    const int w = min(W, n - p0);  // panel width
    if (warp == 0) {
      // panel rows p0 + lane (slot 0) and p0 + lane + 32 (slot 1)
      T r0[W], r1[W];
      const int i0 = p0 + lane, i1 = p0 + lane + 32;
#pragma unroll
      for (int c = 0; c < W; ++c) {
        r0[c] = (i0 < n && c < w) ? S[i0 * CH_LD + p0 + c] : T(0);
        r1[c] = (i1 < n && c < w) ? S[i1 * CH_LD + p0 + c] : T(0);
      }
      int failed = -1;
#pragma unroll
      for (int j = 0; j < W; ++j) {
        if (j < w && failed < 0) {
          const T d = __shfl_sync(0xffffffffu, r0[j], j);  // pivot row p0 + j lives on lane j
          if (!(d > T(0))) {
            failed = p0 + j;
          } else {
            // 1/sqrt(d) directly (one MUFU + Newton, ~75 cycles) keeps the
            // serial pivot chain short; L(j,j) = d * (1/sqrt d) is off the
            // chain.  Differs from sqrt-then-divide by <= 1 ulp.
            const T inv = Num<T>::rsqrt_(d);
            const T rt = d * inv;
            // column j: L(i, j) = a(i, j) / L(j, j) for rows below the pivot
            const T l0 = (lane > j) ? r0[j] * inv : (lane == j ? rt : r0[j]);
            const T l1 = r1[j] * inv;
            r0[j] = l0;
            r1[j] = l1;
#pragma unroll
            for (int k = j + 1; k < W; ++k) {
              const T lkj = __shfl_sync(0xffffffffu, l0, k);  // L(p0 + k, j) on lane k
              if (lane >= k) r0[k] -= l0 * lkj;              // rows at/below the diagonal of col k
              r1[k] -= l1 * lkj;
            }
          }
        }
      }
#pragma unroll
      for (int c = 0; c < W; ++c) {
        if (c < w) {
          if (i0 < n && lane >= c) S[i0 * CH_LD + p0 + c] = r0[c];
          if (i1 < n) S[i1 * CH_LD + p0 + c] = r1[c];
        }
      }
      if (lane == 0 && failed >= 0) *flag = failed;
    }
    __syncthreads();
    if (*flag >= 0) return *flag;
    // trailing update: A(i, k) -= sum_c L(i, p0+c) L(k, p0+c) for p0+w <= k <= i < n
    const int t0 = p0 + w;
    const int m = n - t0;
    if (m > 0) {
      if constexpr (sizeof(T) == 8) {
        // 8x8 lower tiles on FP64 DMMA (m8n8k4), K = panel width; entries of
        // diagonal tiles above the diagonal are scratch (never stored).
        const int nw = nthreads >> 5, fr = lane >> 2, fc = lane & 3;
        const int mt = (m + 7) / 8;
        const int ntiles = mt * (mt + 1) / 2;
        for (int tile = warp; tile < ntiles; tile += nw) {
          int a = 0;
          while ((a + 1) * (a + 2) / 2 <= tile) ++a;
          const int b = tile - a * (a + 1) / 2;
          double c0 = 0.0, c1 = 0.0;
#pragma unroll
          for (int kk = 0; kk < W; kk += 4) {
            const bool ok = kk + fc < w;
            const double af = ok ? S[(t0 + 8 * a + fr) * CH_LD + p0 + kk + fc] : 0.0;
            const double bf = ok ? S[(t0 + 8 * b + fr) * CH_LD + p0 + kk + fc] : 0.0;
            asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                         : "+d"(c0), "+d"(c1)
                         : "d"(af), "d"(bf));
          }
          T* crow = S + (t0 + 8 * a + fr) * CH_LD + t0 + 8 * b + 2 * fc;
          crow[0] -= c0;
          crow[1] -= c1;
        }
      } else {
        for (int e = threadIdx.x; e < m * m; e += nthreads) {
          const int i = t0 + e / m, k = t0 + e % m;
          if (k > i) continue;
          const T* li = S + i * CH_LD + p0;
          const T* lk = S + k * CH_LD + p0;
          T acc = S[i * CH_LD + k];
#pragma unroll
          for (int c = 0; c < W; ++c)
            if (c < w) acc -= li[c] * lk[c];
          S[i * CH_LD + k] = acc;
        }
      }
    }
    __syncthreads();
  }
  return -1;
}

}  // namespace dlab
