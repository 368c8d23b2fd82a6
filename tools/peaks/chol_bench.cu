// Cycle count of the shared-memory Cholesky leaf (chol_smem64) on one CTA.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I../../paper_1710_08717_b200/csrc -o chol_bench chol_bench.cu
#include <cstdio>
#include <cuda_runtime.h>

#include "chol64.cuh"

namespace dlab {
void note_launch(int) {}
}

template <int NMAX>
__global__ void k(double* a, int n, long long* t) {
  constexpr int LD = NMAX + 1;
  extern __shared__ double S[];
  __shared__ int flag;
  for (int e = threadIdx.x; e < n * n; e += blockDim.x) S[(e / n) * LD + e % n] = a[e];
  __syncthreads();
  long long t0 = clock64();
  int f = dlab::chol_smem<double, NMAX>(S, n, &flag);
  __syncthreads();
  long long t1 = clock64();
  for (int e = threadIdx.x; e < n * n; e += blockDim.x) {
    const int i = e / n, j = e % n;
    a[e] = j <= i ? S[i * LD + j] : 0.0;
  }
  if (threadIdx.x == 0) {
    t[0] = t1 - t0;
    t[1] = f;
  }
}

int main() {
  for (int n : {128, 96, 64, 32}) {
    static double h[128 * 128], ref[128 * 128], out[128 * 128];
    for (int i = 0; i < n; ++i)
      for (int j = 0; j < n; ++j) h[i * n + j] = (i == j ? n + 1.0 : 1.0 / (1 + i + j));
    // host Cholesky for checking
    for (int i = 0; i < n * n; ++i) ref[i] = h[i];
    for (int j = 0; j < n; ++j) {
      double d = ref[j * n + j];
      for (int p = 0; p < j; ++p) d -= ref[j * n + p] * ref[j * n + p];
      d = sqrt(d);
      ref[j * n + j] = d;
      for (int i = j + 1; i < n; ++i) {
        double s = ref[i * n + j];
        for (int p = 0; p < j; ++p) s -= ref[i * n + p] * ref[j * n + p];
        ref[i * n + j] = s / d;
      }
    }
    double* d;
    long long* t;
    cudaMalloc(&d, sizeof(h));
    cudaMalloc(&t, 64);
    cudaFuncSetAttribute(k<128>, cudaFuncAttributeMaxDynamicSharedMemorySize, 140000);
    for (int threads : {64, 128, 256, 512}) {
      cudaMemcpy(d, h, sizeof(double) * n * n, cudaMemcpyHostToDevice);
      for (int rep = 0; rep < 2; ++rep) {
        cudaMemcpy(d, h, sizeof(double) * n * n, cudaMemcpyHostToDevice);
        if (n <= 64)
          k<64><<<1, threads, 8 * 64 * 65>>>(d, n, t);
        else
          k<128><<<1, threads, 8 * 128 * 129>>>(d, n, t);
      }
      long long ht[2];
      cudaMemcpy(ht, t, sizeof(ht), cudaMemcpyDeviceToHost);
      cudaMemcpy(out, d, sizeof(double) * n * n, cudaMemcpyDeviceToHost);
      double err = 0;
      for (int i = 0; i < n; ++i)
        for (int j = 0; j <= i; ++j) err = fmax(err, fabs(out[i * n + j] - ref[i * n + j]));
      printf("{\"nmax\": %d, \"n\": %d, \"threads\": %d, \"factor_cycles\": %lld, \"per_col\": %.1f, \"fail\": %lld, \"maxerr\": %.2e}\n",
             n <= 64 ? 64 : 128, n, threads, ht[0], ht[0] / (double)n, ht[1], err);
    }
  }
  return 0;
}
