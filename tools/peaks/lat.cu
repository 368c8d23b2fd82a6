// Dependent-chain latencies of FP64 ops on B200 (one warp), in SM cycles.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o lat lat.cu && ./lat
#include <cstdio>
#include <cuda_runtime.h>

constexpr int N = 1024;

__global__ void chains(double x0, long long* out, double* sink) {
  double x = x0 + threadIdx.x * 1e-9;
  long long t0 = clock64();
  for (int i = 0; i < N; ++i) x = fma(x, 0.999999, 1e-7);
  long long t1 = clock64();
  for (int i = 0; i < N; ++i) x = sqrt(x) + 0.5;
  long long t2 = clock64();
  for (int i = 0; i < N; ++i) x = 1.0 / x + 0.5;
  long long t3 = clock64();
  for (int i = 0; i < N; ++i) x = rsqrt(x) + 0.5;
  long long t4 = clock64();
  for (int i = 0; i < N; ++i) x = __drcp_rn(x) + 0.5;
  long long t5 = clock64();
  float y = (float)x;
  for (int i = 0; i < N; ++i) y = fmaf(y, 0.999f, 1e-4f);
  long long t6 = clock64();
  __shared__ double s[64];
  s[threadIdx.x & 63] = x;
  __syncthreads();
  long long t7 = clock64();
  for (int i = 0; i < N; ++i) __syncthreads();
  long long t8 = clock64();
  if (threadIdx.x == 0) {
    out[0] = t1 - t0; out[1] = t2 - t1; out[2] = t3 - t2; out[3] = t4 - t3; out[4] = t5 - t4;
    out[5] = t6 - t5; out[6] = t8 - t7;
  }
  sink[threadIdx.x] = x + y + s[(threadIdx.x + 1) & 63];
}

int main() {
  long long* d; double* s;
  cudaMalloc(&d, 64); cudaMalloc(&s, 256 * 8);
  for (int threads : {32, 256}) {
    chains<<<1, threads>>>(1.5, d, s);
    long long h[7];
    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    printf("{\"threads\": %d, \"dfma\": %.1f, \"dsqrt\": %.1f, \"ddiv\": %.1f, \"drsqrt\": %.1f, \"drcp\": %.1f, "
           "\"ffma\": %.1f, \"bar_sync\": %.1f}\n", threads,
           h[0] / (double)N, h[1] / (double)N, h[2] / (double)N, h[3] / (double)N, h[4] / (double)N,
           h[5] / (double)N, h[6] / (double)N);
  }
  return 0;
}
