// Where do the cycles of a 16-column warp-panel Cholesky go?  One warp,
// variants: 0 full, 1 no rsqrt (cheap reciprocal), 2 no update loop,
// 3 no smem publication (values only in registers).
#include <cstdio>
#include <cuda_runtime.h>

constexpr int W = 16, LD = 65;

template <int V>
__global__ void panel(double* g, long long* t) {
  __shared__ double S[64 * LD];
  const int lane = threadIdx.x;
  for (int e = lane; e < 64 * 64; e += 32) S[(e / 64) * LD + e % 64] = g[e];
  __syncwarp();
  double r0[W], r1[W];
  for (int c = 0; c < W; ++c) {
    r0[c] = S[lane * LD + c];
    r1[c] = S[(lane + 32) * LD + c];
  }
  long long t0 = clock64();
#pragma unroll
  for (int j = 0; j < W; ++j) {
    const double d = (V == 3) ? __shfl_sync(0xffffffffu, r0[j], j) : S[j * LD + j];
    double inv;
    if (V == 1) inv = (double)(1.0f / sqrtf((float)d));
    else inv = rsqrt(d);
    const double rt = d * inv;
    const double l0 = (lane > j) ? r0[j] * inv : (lane == j ? rt : r0[j]);
    const double l1 = r1[j] * inv;
    r0[j] = l0;
    r1[j] = l1;
    if (V != 3) {
      if (lane < W) S[lane * LD + j] = l0;
      __syncwarp();
    }
    if (V != 2) {
#pragma unroll
      for (int k = j + 1; k < W; ++k) {
        const double lkj = (V == 3) ? __shfl_sync(0xffffffffu, l0, k) : S[k * LD + j];
        if (lane >= k) r0[k] -= l0 * lkj;
        r1[k] -= l1 * lkj;
      }
    }
    if (V != 3) {
      if (j + 1 < W && lane == j + 1) S[lane * LD + j + 1] = r0[j + 1];
      __syncwarp();
    }
  }
  long long t1 = clock64();
  double s = 0;
  for (int c = 0; c < W; ++c) s += r0[c] + r1[c];
  g[lane] = s;
  if (lane == 0) t[V] = t1 - t0;
}

int main() {
  double h[64 * 64];
  for (int i = 0; i < 64; ++i)
    for (int j = 0; j < 64; ++j) h[i * 64 + j] = (i == j ? 65.0 : 1.0 / (1 + i + j));
  double* g;
  long long* t;
  cudaMalloc(&g, sizeof(h));
  cudaMalloc(&t, 64);
  long long ht[4];
  for (int rep = 0; rep < 2; ++rep) {
    cudaMemcpy(g, h, sizeof(h), cudaMemcpyHostToDevice);
    panel<0><<<1, 32>>>(g, t);
    cudaMemcpy(g, h, sizeof(h), cudaMemcpyHostToDevice);
    panel<1><<<1, 32>>>(g, t);
    cudaMemcpy(g, h, sizeof(h), cudaMemcpyHostToDevice);
    panel<2><<<1, 32>>>(g, t);
    cudaMemcpy(g, h, sizeof(h), cudaMemcpyHostToDevice);
    panel<3><<<1, 32>>>(g, t);
    cudaMemcpy(ht, t, sizeof(ht), cudaMemcpyDeviceToHost);
    printf("{\"full\": %.0f, \"cheap_rcp\": %.0f, \"no_update\": %.0f, \"shfl_only\": %.0f}  (cycles per column)\n",
           ht[0] / 16.0, ht[1] / 16.0, ht[2] / 16.0, ht[3] / 16.0);
  }
  return 0;
}
