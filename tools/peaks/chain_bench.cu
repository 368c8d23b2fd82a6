// Latency of the Cholesky pivot chain primitives on one warp (cycles/step):
// shuffle -> rsqrt (MUFU seed + Newton) -> multiply -> FMA, with and without
// extra independent work per step.
#include <cstdio>
#include <cuda_runtime.h>

#include "common.cuh"

namespace dlab {
void note_launch(int) {}
}

template <int EXTRA>
__global__ void k(double* out, long long* t) {
  const int lane = threadIdx.x;
  double r = 2.0 + lane, x = 3.0 + lane;
  double acc[16];
#pragma unroll
  for (int u = 0; u < 16; ++u) acc[u] = lane + u;
  long long t0 = clock64();
#pragma unroll 1
  for (int it = 0; it < 256; ++it) {
    const double d = __shfl_sync(0xffffffffu, x, it & 31);
    const double inv = dlab::Num<double>::rsqrt_(d);
    const double l = r * inv;
    x = fma(-l, l, x + 1.0);
#pragma unroll
    for (int u = 0; u < EXTRA; ++u) {
      const double v = __shfl_sync(0xffffffffu, l, u);
      acc[u] = fma(-l, v, acc[u]);
    }
  }
  long long t1 = clock64();
  double s = x;
#pragma unroll
  for (int u = 0; u < 16; ++u) s += acc[u];
  out[lane] = s;
  if (lane == 0) *t = t1 - t0;
}

int main() {
  double* o;
  long long* t;
  cudaMalloc(&o, 256 * 8);
  cudaMalloc(&t, 8);
  long long h;
  k<0><<<1, 32>>>(o, t);
  cudaMemcpy(&h, t, 8, cudaMemcpyDeviceToHost);
  printf("{\"extra\": 0, \"cycles_per_step\": %.1f}\n", h / 256.0);
  k<8><<<1, 32>>>(o, t);
  cudaMemcpy(&h, t, 8, cudaMemcpyDeviceToHost);
  printf("{\"extra\": 8, \"cycles_per_step\": %.1f}\n", h / 256.0);
  k<16><<<1, 32>>>(o, t);
  cudaMemcpy(&h, t, 8, cudaMemcpyDeviceToHost);
  printf("{\"extra\": 16, \"cycles_per_step\": %.1f}\n", h / 256.0);
  return 0;
}
