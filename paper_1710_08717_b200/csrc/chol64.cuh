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

// Column J of a W-wide register panel (template recursion keeps every
// register index a compile-time constant).  Straight-line: a failed pivot is
// only recorded; the NaNs it creates never leave the CTA.
template <typename T, int W, int J>
__device__ __forceinline__ void panel_cols(T (&r0)[W], T (&r1)[W], int lane, int w, int p0, int& failed) {
  if constexpr (J < W) {
    const T d = __shfl_sync(0xffffffffu, r0[J], J);  // pivot row p0 + J lives on lane J
    if (!(d > T(0)) && failed < 0 && J < w) failed = p0 + J;
    // 1/sqrt(d) directly (one MUFU + Newton, ~75 cycles) keeps the serial
    // pivot chain short; L(J,J) = d * (1/sqrt d) is off the chain.  Differs
    // from sqrt-then-divide by <= 1 ulp.
    const T inv = Num<T>::rsqrt_(d);
    const T rt = d * inv;
    // column J: L(i, J) = a(i, J) / L(J, J) for rows below the pivot
    const T l0 = (lane > J) ? r0[J] * inv : (lane == J ? rt : r0[J]);
    const T l1 = r1[J] * inv;
    r0[J] = l0;
    r1[J] = l1;
#pragma unroll
    for (int k = J + 1; k < W; ++k) {
      const T lkj = __shfl_sync(0xffffffffu, l0, k);  // L(p0 + k, J) on lane k
      if (lane >= k) r0[k] -= l0 * lkj;              // rows at/below the diagonal of col k
      r1[k] -= l1 * lkj;
    }
    panel_cols<T, W, J + 1>(r0, r1, lane, w, p0, failed);
  }
}

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
      // The padded columns of a narrow last panel factor an identity block.
#pragma unroll
      for (int c = 0; c < W; ++c)
        if (c >= w && lane == c) r0[c] = T(1);
      panel_cols<T, W, 0>(r0, r1, lane, w, p0, failed);
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

// Forward substitution S y = v for nv <= 64 vectors held vector-major in
// shared memory (V[v * CH_LD + i]); S lower triangular, 64 x 64 (zero padded
// beyond nb), rd[i] = 1 / S(i,i).  8-row blocks: the 8 x 8 diagonal block is
// solved per vector (one thread per vector), the rows below are updated by an
// (rows x 8) x (8 x 64) FP64 DMMA product.  Needs >= 64 threads, ends synced.
template <typename T>
__device__ __forceinline__ void blocked_fwd_subst(const T* S, T* V, const T* rd, int nb, int nv) {
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, fr = lane >> 2, fc = lane & 3;
  const int nw = blockDim.x >> 5;
  for (int c0 = 0; c0 < nb; c0 += 8) {
    if (tid < nv) {
      T* xv = V + tid * CH_LD;
      for (int i = c0; i < c0 + 8 && i < nb; ++i) {
        T acc = xv[i];
        for (int p = c0; p < i; ++p) acc -= S[i * CH_LD + p] * xv[p];
        xv[i] = acc * rd[i];
      }
    }
    __syncthreads();
    const int r0 = c0 + 8;
    const int rtiles = (nb - r0 + 7) / 8;
    if constexpr (sizeof(T) == 8) {
      for (int tile = warp; tile < rtiles * 8; tile += nw) {
        const int rt = r0 + (tile >> 3) * 8, nt = (tile & 7) * 8;
        double acc0 = 0.0, acc1 = 0.0;
#pragma unroll
        for (int kk = 0; kk < 8; kk += 4) {
          const double af = S[(rt + fr) * CH_LD + c0 + kk + fc];
          const double bf = V[(nt + fr) * CH_LD + c0 + kk + fc];
          asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                       : "+d"(acc0), "+d"(acc1)
                       : "d"(af), "d"(bf));
        }
        V[(nt + 2 * fc) * CH_LD + rt + fr] -= acc0;
        V[(nt + 2 * fc + 1) * CH_LD + rt + fr] -= acc1;
      }
    } else {
      for (int e = tid; e < rtiles * 8 * 64; e += blockDim.x) {
        const int r = r0 + e / 64, v = e % 64;
        T acc = T(0);
#pragma unroll
        for (int p = 0; p < 8; ++p) acc += S[r * CH_LD + c0 + p] * V[v * CH_LD + c0 + p];
        V[v * CH_LD + r] -= acc;
      }
    }
    __syncthreads();
  }
}

}  // namespace dlab
