// Per-phase cycle accounting of the Chol64 column loop (thread 0 view).
#include <cstdio>
#include <cuda_runtime.h>
#include "chol64.cuh"
namespace dlab { void note_launch(int) {} }
using T = double;
__global__ void k(double* a, int n, long long* t, int variant) {
  __shared__ double colbuf[2 * 66];
  dlab::Chol64<double> ch;
  ch.load(a, n, n);
  __syncthreads();
  const int ty = ch.ty, tx = ch.tx;
  long long acc_top = 0, acc_bar = 0, acc_upd = 0;
  for (int j = 0; j < n; ++j) {
    long long c0 = clock64();
    T* cb = colbuf + (j & 1) * 66;
    if (tx == (j & 15)) {
      const int q = j >> 4;
      T own = 0;
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const T v = q == 0 ? ch.r[i][0] : q == 1 ? ch.r[i][1] : q == 2 ? ch.r[i][2] : ch.r[i][3];
        cb[ty + 16 * i] = v;
        if (i == q) own = v;
      }
      if (ty == (j & 15) && own > 0) {
        T rt, inv;
        if (variant == 0) { rt = sqrt(own); inv = 1.0 / rt; }
        else { inv = rsqrt(own); rt = own * inv; }
        cb[64] = rt; cb[65] = inv;
      }
    }
    long long c1 = clock64();
    __syncthreads();
    long long c2 = clock64();
    const T d = cb[j];
    if (!(d > 0)) break;
    const T rt = cb[64], inv = cb[65];
    T lk[4], ll[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const T vk = cb[ty + 16 * i] * inv; lk[i] = (ty + 16 * i > j) ? vk : 0;
      const T vl = cb[tx + 16 * i] * inv; ll[i] = (tx + 16 * i > j) ? vl : 0;
    }
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int c = 0; c < 4; ++c) ch.r[i][c] -= lk[i] * ll[c];
    if (tx == (j & 15)) {
      const int q = j >> 4;
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int kk = ty + 16 * i;
        const T v = (kk == j) ? rt : (kk > j ? lk[i] : 0);
#pragma unroll
        for (int c = 0; c < 4; ++c) if (c == q) ch.r[i][c] = v;
      }
    }
    long long c3 = clock64();
    acc_top += c1 - c0; acc_bar += c2 - c1; acc_upd += c3 - c2;
  }
  __syncthreads();
  ch.store(a, n, n, true);
  if (threadIdx.x == 0 || threadIdx.x == 17) {
    t[threadIdx.x == 0 ? 0 : 3] = acc_top; t[threadIdx.x == 0 ? 1 : 4] = acc_bar; t[threadIdx.x == 0 ? 2 : 5] = acc_upd;
  }
}
int main() {
  const int n = 64; double h[n * n];
  for (int i = 0; i < n; ++i) for (int j = 0; j < n; ++j) h[i * n + j] = (i == j ? n + 1.0 : 1.0 / (1 + i + j));
  double* d; long long* t; cudaMalloc(&d, sizeof(h)); cudaMalloc(&t, 64);
  for (int v = 0; v < 2; ++v) for (int r = 0; r < 2; ++r) {
    cudaMemcpy(d, h, sizeof(h), cudaMemcpyHostToDevice);
    k<<<1, 256>>>(d, n, t, v);
    long long ht[6]; cudaMemcpy(ht, t, sizeof(ht), cudaMemcpyDeviceToHost);
    printf("{\"variant\": %d, \"t0_top\": %.0f, \"t0_bar\": %.0f, \"t0_upd\": %.0f, \"t17_top\": %.0f, \"t17_bar\": %.0f, \"t17_upd\": %.0f}\n",
           v, ht[0] / 64.0, ht[1] / 64.0, ht[2] / 64.0, ht[3] / 64.0, ht[4] / 64.0, ht[5] / 64.0);
  }
}
