// Cholesky of one n <= NMAX (64 or 128) block held in shared memory by a CTA
// of >= 64 threads (dl/cholesky.hpp:35-72 reordered for the GPU).
//
// The pivot chain is the critical path of any Cholesky (n dependent
// sqrt/div pairs).  Here it never crosses a block barrier: see chol_smem.
#pragma once

#include "common.cuh"

namespace dlab {

constexpr int CH_LD = 65;  // smem row stride for a 64 x 64 block

#ifndef DLAB_CHOL_W
#define DLAB_CHOL_W(NMAX) 16  // warp-panel width of chol_smem
#endif

// Column J of a W-wide register panel (template recursion keeps every
// register index a compile-time constant).  Lane l holds panel rows
// p0 + l + 32 q in slot q.  Straight-line: a failed pivot is only recorded;
// the NaNs it creates never leave the CTA.
template <typename T, int W, int Q, int J>
__device__ __forceinline__ void panel_cols(T (&r)[Q][W], int lane, int w, int p0, int& failed, T dcur, T* cbuf) {
  if constexpr (J < W) {
    // dcur: this lane's candidate for pivot J (meaningful on lane J), formed
    // at column J-1 straight from the lane's own multiplier, so the serial
    // chain per column is shuffle -> rsqrt -> multiply -> FMA and never waits
    // for the broadcast of the other multipliers.
    const T d = __shfl_sync(0xffffffffu, dcur, J);  // pivot row p0 + J lives on lane J
    if (!(d > T(0)) && failed < 0 && J < w) failed = p0 + J;
    // 1/sqrt(d) directly (one MUFU + Newton, ~75 cycles) keeps the serial
    // pivot chain short; L(J,J) = d * (1/sqrt d) is off the chain.  Differs
    // from sqrt-then-divide by <= 1 ulp.
    const T inv = Num<T>::rsqrt_(d);
    const T rt = d * inv;
    // column J: L(i, J) = a(i, J) / L(J, J) for rows below the pivot
    T l[Q];
    l[0] = (lane > J) ? r[0][J] * inv : (lane == J ? rt : r[0][J]);
    T dnext = T(0);
    if constexpr (J + 1 < W) dnext = r[0][J + 1] - l[0] * l[0];  // pivot J+1 on lane J+1
#pragma unroll
    for (int q = 1; q < Q; ++q) l[q] = r[q][J] * inv;
#pragma unroll
    for (int q = 0; q < Q; ++q) r[q][J] = l[q];
#ifdef DLAB_PANEL_SHFL
#pragma unroll
    for (int k = J + 1; k < W; ++k) {
      const T lkj = __shfl_sync(0xffffffffu, l[0], k);  // L(p0 + k, J) on lane k
      if (lane >= k) r[0][k] -= l[0] * lkj;            // rows at/below the diagonal of col k
#pragma unroll
      for (int q = 1; q < Q; ++q) r[q][k] -= l[q] * lkj;
    }
#else
    // the column's panel multipliers L(p0 + k, J), k > J, are broadcast
    // through a double-buffered shared vector: one STS + vector LDS per pair
    // instead of two SHFLs per value
    if constexpr (J + 1 < W) {
      T* cb = cbuf + (J & 1) * 32;
      if (lane < W) cb[lane] = l[0];
      __syncwarp();
      constexpr int VN = 16 / sizeof(T);
#pragma unroll
      for (int k0 = ((J + 1) / VN) * VN; k0 < W; k0 += VN) {
        T v[VN];
        if constexpr (VN == 2) {
          const double2 t2 = *reinterpret_cast<const double2*>(cb + k0);
          v[0] = t2.x;
          v[1] = t2.y;
        } else {
          const float4 t4 = *reinterpret_cast<const float4*>(cb + k0);
          v[0] = t4.x;
          v[1] = t4.y;
          v[2] = t4.z;
          v[3] = t4.w;
        }
#pragma unroll
        for (int u = 0; u < VN; ++u) {
          const int k = k0 + u;
          if (k > J) {
            if (lane >= k) r[0][k] -= l[0] * v[u];
#pragma unroll
            for (int q = 1; q < Q; ++q) r[q][k] -= l[q] * v[u];
          }
        }
      }
    }
#endif
    panel_cols<T, W, Q, J + 1>(r, lane, w, p0, failed, dnext, cbuf);
  }
}

// One warp factors the W-wide panel at column p0 (rows p0 .. n-1, Q slots of
// 32 rows per lane) in registers and writes it back.  Returns the failing
// pivot or -1.
template <typename T, int LD, int W, int Q>
__device__ __forceinline__ int panel_warp(T* S, int n, int p0, int w, int lane) {
  T r[Q][W];
#pragma unroll
  for (int q = 0; q < Q; ++q) {
    const int i = p0 + lane + 32 * q;
#pragma unroll
    for (int c = 0; c < W; ++c) r[q][c] = (i < n && c < w) ? S[i * LD + p0 + c] : T(0);
  }
  // The padded columns of a narrow last panel factor an identity block.
#pragma unroll
  for (int c = 0; c < W; ++c)
    if (c >= w && lane == c) r[0][c] = T(1);
  int failed = -1;
  __shared__ __align__(16) T cbuf[64];
  panel_cols<T, W, Q, 0>(r, lane, w, p0, failed, r[0][0], cbuf);
#pragma unroll
  for (int q = 0; q < Q; ++q) {
    const int i = p0 + lane + 32 * q;
#pragma unroll
    for (int c = 0; c < W; ++c)
      if (c < w && i < n && (q > 0 || lane >= c)) S[i * LD + p0 + c] = r[q][c];
  }
  return failed;
}

// Dispatch on the number of live 32-row slots (the panel shrinks as p0
// advances; dead slots would only burn the serial chain).
template <typename T, int LD, int W, int Q>
__device__ __forceinline__ int panel_warp_n(T* S, int n, int p0, int w, int lane, int qa) {
  if constexpr (Q > 1) {
    if (qa < Q) return panel_warp_n<T, LD, W, Q - 1>(S, n, p0, w, lane, qa);
  }
  return panel_warp<T, LD, W, Q>(S, n, p0, w, lane);
}

// S: n x n block in shared memory (row stride NMAX + 1), n <= NMAX, lower
// triangle valid.  On return S holds L in its lower triangle.  Returns the
// first failing pivot (uniform across the CTA) or -1.  `flag` is one shared
// int.  Processed in 16-column panels, each factored by ONE warp entirely in
// registers (pivots and multipliers move by warp shuffles; every lane takes
// the reciprocal square root itself); the CTA's warps then apply the panel to
// the trailing lower triangle (8 x 8 DMMA tiles for f64).  Two barriers per
// 16 columns instead of one per column.
#ifdef DLAB_PANEL_PROF
__device__ unsigned long long g_cprof[128][16];
__device__ int g_prof_row;
#define CSTAMP(i)                                                                     \
  do {                                                                                \
    if (gridDim.x >= 16 && blockIdx.x == 0 && threadIdx.x == 0) {                     \
      unsigned long long t_;                                                          \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                          \
      g_cprof[g_prof_row & 127][i] = t_;                                              \
    }                                                                                 \
  } while (0)
#else
#define CSTAMP(i)
#endif
struct NoSide {
  __device__ void operator()(int) const {}
};

// `side(warp)` runs on warps 1.. while warp 0 factors the first 16-column
// panel (the only phase in which they would otherwise wait at a barrier);
// it must not touch S.
template <typename T, int NMAX, typename F = NoSide>
__device__ __forceinline__ int chol_smem(T* S, int n, int* flag, F side = F()) {
  constexpr int W = DLAB_CHOL_W(NMAX), LD = NMAX + 1, Q = NMAX / 32;
  static_assert(NMAX % 32 == 0, "32-row slots");
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nthreads = blockDim.x;
  if (threadIdx.x == 0) *flag = -1;
  __syncthreads();
  CSTAMP(0);
  for (int p0 = 0; p0 < n; p0 += W) {
    const int w = min(W, n - p0);  // panel width
    if (warp == 0) {
      const int failed = panel_warp_n<T, LD, W, Q>(S, n, p0, w, lane, (n - p0 + 31) >> 5);
      if (lane == 0 && failed >= 0) *flag = failed;
      if (p0 == 0) CSTAMP(9);
    } else if (p0 == 0) {
      side(warp);
    }
    __syncthreads();
    CSTAMP(1 + 2 * (p0 / W));
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
            const double af = ok ? S[(t0 + 8 * a + fr) * LD + p0 + kk + fc] : 0.0;
            const double bf = ok ? S[(t0 + 8 * b + fr) * LD + p0 + kk + fc] : 0.0;
            asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                         : "+d"(c0), "+d"(c1)
                         : "d"(af), "d"(bf));
          }
          T* crow = S + (t0 + 8 * a + fr) * LD + t0 + 8 * b + 2 * fc;
          crow[0] -= c0;
          crow[1] -= c1;
        }
      } else {
        for (int e = threadIdx.x; e < m * m; e += nthreads) {
          const int i = t0 + e / m, k = t0 + e % m;
          if (k > i) continue;
          const T* li = S + i * LD + p0;
          const T* lk = S + k * LD + p0;
          T acc = S[i * LD + k];
#pragma unroll
          for (int c = 0; c < W; ++c)
            if (c < w) acc -= li[c] * lk[c];
          S[i * LD + k] = acc;
        }
      }
    }
    __syncthreads();
    CSTAMP(2 + 2 * (p0 / W));
  }
  return -1;
}

// Blocked-potrf panel step, fp64: factor A11 (S, nb x nb, nb <= 64) AND
// solve the CTA's chunk rows V <- V L11^{-T} (nv <= 64 rows, stride LD) in
// one interleaved pass.  While warp 0 factors 16-column panel j of A11 (the
// pivot chain), warps {1,2,3,5,6,7} (not warp 4: it shares warp 0's issue
// slots) solve V's columns of panel j-1 against its 16 x 16 diagonal block
// and apply them to V's later columns (DMMA) -- so the chunk solve rides
// under the factorization instead of following it.  `pre(warp)` (the fused
// look-ahead update of V) runs in that slot for j = 0.  Returns the failing
// pivot (uniform) or -1; on success V holds L21's rows.
template <int LD, typename F>
__device__ __forceinline__ int chol_tall64(double* S, double* V, int nb, int nv, int* flag, F pre) {
  constexpr int W = 16, Q = 2;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, fr = lane >> 2, fc = lane & 3;
  if (threadIdx.x == 0) *flag = -1;
  __syncthreads();
  CSTAMP(0);
  const int np = (nb + W - 1) / W;
  // V work group: 6 warps, a named barrier of 192 threads
  const int vw = warp < 4 ? warp - 1 : warp - 2;  // 0..5 for warps 1-3, 5-7
  for (int j = 0; j <= np; ++j) {
    const int p0 = j * W;
    if (warp == 0) {
      if (j < np) {
        const int failed = panel_warp_n<double, LD, W, Q>(S, nb, p0, min(W, nb - p0), lane, (nb - p0 + 31) >> 5);
        if (lane == 0 && failed >= 0) *flag = failed;
      }
    } else if (j == 0) {
      pre(warp);
    } else if (warp != 4 && nv > 0) {
      const int c0 = p0 - W, w = min(W, nb - c0);
      // (1) rows of V: x L(c0.., c0..)^T = v on the 16 x 16 diagonal block
      const int v = threadIdx.x - 32;  // warps 1, 2
      if (v < nv && v >= 0) {
        double x[W], rdl[W];
#pragma unroll
        for (int i = 0; i < W; ++i) {
          x[i] = i < w ? V[v * LD + c0 + i] : 0.0;
          rdl[i] = i < w ? 1.0 / S[(c0 + i) * LD + c0 + i] : 0.0;
        }
#pragma unroll
        for (int p = 0; p < W; ++p) {
          x[p] *= rdl[p];
#pragma unroll
          for (int i = p + 1; i < W; ++i)
            if (i < w) x[i] -= S[(c0 + i) * LD + c0 + p] * x[p];
        }
#pragma unroll
        for (int i = 0; i < W; ++i)
          if (i < w) V[v * LD + c0 + i] = x[i];
      }
      asm volatile("bar.sync 1, 192;" ::: "memory");
      // (2) V(:, c0+W .. nb) -= X L(c0+W .. nb, c0 .. c0+W)^T  (8 x 8 DMMA tiles)
      const int t0 = c0 + W;
      if (t0 < nb) {
        const int rts = (nv + 7) / 8, cts = (nb - t0 + 7) / 8;
        for (int tile = vw; tile < rts * cts; tile += 6) {
          const int rt = tile / cts, ct = t0 / 8 + tile % cts;
          double a0 = 0.0, a1 = 0.0;
#pragma unroll
          for (int s = 0; s < 4; ++s) {  // k-column 4 fc + s: conflict-free with stride 65
            const bool ok = 4 * fc + s < w;
            const double af = ok ? V[(8 * rt + fr) * LD + c0 + 4 * fc + s] : 0.0;
            const double bf = ok ? S[(8 * ct + fr) * LD + c0 + 4 * fc + s] : 0.0;
            asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                         : "+d"(a0), "+d"(a1)
                         : "d"(af), "d"(bf));
          }
          double* crow = V + (8 * rt + fr) * LD + 8 * ct + 2 * fc;
          crow[0] -= a0;
          crow[1] -= a1;
        }
      }
    }
    __syncthreads();
    CSTAMP(1 + 2 * j);
    if (*flag >= 0) return *flag;
    if (j == np) break;
    // A11 trailing update with panel j: A(i, k) -= L(i, p0..) L(k, p0..), t0 <= k <= i < nb
    const int w = min(W, nb - p0), t0 = p0 + w, m = nb - t0;
    if (m > 0) {
      const int mt = (m + 7) / 8, ntiles = mt * (mt + 1) / 2;
      for (int tile = warp; tile < ntiles; tile += 8) {
        int a = 0;
        while ((a + 1) * (a + 2) / 2 <= tile) ++a;
        const int b = tile - a * (a + 1) / 2;
        double c0 = 0.0, c1 = 0.0;
#pragma unroll
        for (int s = 0; s < 4; ++s) {
          const bool ok = 4 * fc + s < w;
          const double af = ok ? S[(t0 + 8 * a + fr) * LD + p0 + 4 * fc + s] : 0.0;
          const double bf = ok ? S[(t0 + 8 * b + fr) * LD + p0 + 4 * fc + s] : 0.0;
          asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                       : "+d"(c0), "+d"(c1)
                       : "d"(af), "d"(bf));
        }
        double* crow = S + (t0 + 8 * a + fr) * LD + t0 + 8 * b + 2 * fc;
        crow[0] -= c0;
        crow[1] -= c1;
      }
      __syncthreads();
      CSTAMP(2 + 2 * j);
    }
  }
  return -1;
}

template <typename T>
__device__ __forceinline__ int chol_smem64(T* S, int n, int* flag) {
  return chol_smem<T, 64>(S, n, flag);
}

// ------------------------------------------------ warp-register Cholesky
// Row-per-lane factorization of a 32 x 32 block held in registers (lane l
// owns row l).  Values every lane needs are broadcast from shared memory
// with 16-byte loads (Bc): one LDS.128 carries 2 doubles where a 64-bit
// shuffle costs two SHFLs per value.
constexpr int WCH = 32;

template <typename T>
struct Bc;
template <>
struct Bc<double> {
  static constexpr int N = 2;
  static constexpr int LLD = 34;  // broadcast tiles: 16-byte aligned rows
  __device__ static void ld(const double* p, double (&v)[2]) {
    const double2 t = *reinterpret_cast<const double2*>(p);
    v[0] = t.x;
    v[1] = t.y;
  }
};
template <>
struct Bc<float> {
  static constexpr int N = 4;
  static constexpr int LLD = 36;
  __device__ static void ld(const float* p, float (&v)[4]) {
    const float4 t = *reinterpret_cast<const float4*>(p);
    v[0] = t.x;
    v[1] = t.y;
    v[2] = t.z;
    v[3] = t.w;
  }
};

// Column J of the row-per-lane Cholesky (dl/cholesky.hpp:35-72): the pivot
// moves by one shuffle, the column's multipliers through a double-buffered
// shared vector (one __syncwarp per column).
// sink != nullptr: each finished multiplier r[J] is also stored to sink[J]
// (the caller's shared-memory row) as its column completes, so callers that
// only store L afterwards let the register die instead of carrying (and
// spilling) the finished part of the row through the rest of the chain.
template <typename T, int J>
__device__ __forceinline__ void wchol_col(T (&r)[WCH], int lane, int n, T* buf, int& failed, T dcur,
                                          T* sink = nullptr) {
  if constexpr (J < WCH) {
    // dcur: pivot candidate formed from this lane's own multiplier at column
    // J-1 (see panel_cols): the serial chain is shuffle -> rsqrt -> mul -> FMA.
    const T d = __shfl_sync(0xffffffffu, dcur, J);
    if (!(d > T(0)) && failed < 0 && J < n) failed = J;
    const T inv = Num<T>::rsqrt_(d);
    const T rt = d * inv;
    const T l = (lane > J) ? r[J] * inv : (lane == J ? rt : r[J]);
    r[J] = l;
    if (sink) sink[J] = l;
    T dnext = T(0);
    if constexpr (J + 1 < WCH) {
      dnext = r[J + 1] - l * l;
      constexpr int VN = Bc<T>::N;
      T* cb = buf + (J & 1) * WCH;
      cb[lane] = l;
      __syncwarp();
#pragma unroll
      for (int k0 = ((J + 1) / VN) * VN; k0 < WCH; k0 += VN) {
        T v[VN];
        Bc<T>::ld(cb + k0, v);
#pragma unroll
        for (int u = 0; u < VN; ++u)  // lanes above row k0+u only touch unused upper entries
          if (k0 + u > J) r[k0 + u] -= l * v[u];
      }
    }
    wchol_col<T, J + 1>(r, lane, n, buf, failed, dnext, sink);
  }
}

// Forward substitution S y = v for nv <= 64 vectors held vector-major in
// shared memory (V[v * LD + i]); S lower triangular, nb x nb at row stride
// LD, rd[i] = 1 / S(i,i).  8-row blocks: the 8 x 8 diagonal block is
// solved per vector (one thread per vector), the rows below are updated by an
// (rows x 8) x (8 x 64) FP64 DMMA product.  Needs >= 64 threads, ends synced.
template <typename T, int LD = CH_LD>
__device__ __forceinline__ void blocked_fwd_subst(const T* S, T* V, const T* rd, int nb, int nv) {
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, fr = lane >> 2, fc = lane & 3;
  const int nw = blockDim.x >> 5;
  for (int c0 = 0; c0 < nb; c0 += 8) {
    if (tid < nv) {
      // right-looking in registers: the serial chain is one multiply and one
      // FMA per row; the S loads are independent of it
      T* xv = V + tid * LD;
      T x[8];
#pragma unroll
      for (int r = 0; r < 8; ++r) x[r] = (c0 + r < nb) ? xv[c0 + r] : T(0);
#pragma unroll
      for (int p = 0; p < 8; ++p) {
        x[p] *= (c0 + p < nb) ? rd[c0 + p] : T(0);
#pragma unroll
        for (int i = p + 1; i < 8; ++i)
          if (c0 + i < nb) x[i] -= S[(c0 + i) * LD + c0 + p] * x[p];
      }
#pragma unroll
      for (int r = 0; r < 8; ++r)
        if (c0 + r < nb) xv[c0 + r] = x[r];
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
          const double af = S[(rt + fr) * LD + c0 + kk + fc];
          const double bf = V[(nt + fr) * LD + c0 + kk + fc];
          asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                       : "+d"(acc0), "+d"(acc1)
                       : "d"(af), "d"(bf));
        }
        V[(nt + 2 * fc) * LD + rt + fr] -= acc0;
        V[(nt + 2 * fc + 1) * LD + rt + fr] -= acc1;
      }
    } else {
      for (int e = tid; e < rtiles * 8 * 64; e += blockDim.x) {
        const int r = r0 + e / 64, v = e % 64;
        T acc = T(0);
#pragma unroll
        for (int p = 0; p < 8; ++p) acc += S[r * LD + c0 + p] * V[v * LD + c0 + p];
        V[v * LD + r] -= acc;
      }
    }
    __syncthreads();
  }
}

}  // namespace dlab
