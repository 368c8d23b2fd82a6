// Register-blocked right-looking Cholesky of one n <= 64 block by a 256-thread
// CTA: thread (ty, tx) of a 16 x 16 grid owns elements (ty + 16a, tx + 16b),
// a, b in 0..3, in registers.  Each step publishes the pivot column through a
// double-buffered shared vector, so a column costs ONE barrier (the scalar
// reference loop, dl/cholesky.hpp:44-58, is the same recurrence reordered).
#pragma once

#include "common.cuh"

namespace dlab {

template <typename T>
struct Chol64 {
  T r[4][4];
  int ty, tx;

  __device__ Chol64() : ty(threadIdx.x >> 4), tx(threadIdx.x & 15) {}

  // load the lower triangle of an n x n block (rows ld apart); others = 0
  __device__ __forceinline__ void load(const T* a, int64_t ld, int n) {
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int k = ty + 16 * i, l = tx + 16 * j;
        r[i][j] = (k < n && l <= k) ? a[k * ld + l] : T(0);
      }
  }

  // Factor in place; colbuf: 2 x 66 shared.  Returns the failing step or -1
  // (uniform across the CTA).
  __device__ __forceinline__ int factor(int n, T* colbuf) {
    for (int j = 0; j < n; ++j) {
      T* cb = colbuf + (j & 1) * 66;
      if (tx == (j & 15)) {
        const int q = j >> 4;  // register column, selected without dynamic indexing
        T own = T(0);
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const T v = q == 0 ? r[i][0] : q == 1 ? r[i][1] : q == 2 ? r[i][2] : r[i][3];
          cb[ty + 16 * i] = v;
          if (i == q) own = v;
        }
        // the pivot's owner alone takes the (slow-path-carrying) sqrt and divide
        if (ty == (j & 15) && own > T(0)) {
          const T rt = Num<T>::sqrt_(own);
          cb[64] = rt;
          cb[65] = T(1) / rt;
        }
      }
      __syncthreads();
      const T d = cb[j];
      if (!(d > T(0))) return j;
      const T rt = cb[64];
      const T inv = cb[65];
      T lk[4], ll[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        lk[i] = cb[ty + 16 * i] * inv;
        ll[i] = cb[tx + 16 * i] * inv;
      }
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          const int k = ty + 16 * i, l = tx + 16 * c;
          if (l > j && k >= l) r[i][c] -= lk[i] * ll[c];
          else if (l == j) r[i][c] = (k == j) ? rt : (k > j ? lk[i] : r[i][c]);
        }
    }
    return -1;
  }

  // store L (lower) or R = L^T (upper) with the opposite triangle zeroed
  __device__ __forceinline__ void store(T* a, int64_t ld, int n, bool lower) const {
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int k = ty + 16 * i, l = tx + 16 * j;
        if (k >= n || l >= n) continue;
        const T v = (l <= k) ? r[i][j] : T(0);
        if (lower) a[k * ld + l] = v;
        else a[l * ld + k] = v;
      }
  }
};

}  // namespace dlab
