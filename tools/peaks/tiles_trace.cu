// Timeline of the persistent tile Cholesky (potrf_tiles.cu) on one SPD matrix:
// per task (grab, update done, end, SM, i, j) from %globaltimer.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 --expt-relaxed-constexpr \
//        -DDLAB_TILES_TRACE -I../../paper_1710_08717_b200/csrc -o tiles_trace tiles_trace.cu
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "potrf_tiles.cu"

namespace dlab {
void note_launch(int) {}
}

int main(int argc, char** argv) {
  const int n = argc > 1 ? atoi(argv[1]) : 4096;
  std::vector<double> h((size_t)n * n);
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j) h[(size_t)i * n + j] = (i == j ? n : 0.0) + 1.0 / (1.0 + i + j);
  double* d;
  cudaMalloc(&d, sizeof(double) * n * n);
  const int nt = (n + 63) / 64, tasks = nt * (nt + 1) / 2;
  long long* tr;
  cudaMalloc(&tr, sizeof(long long) * 6 * tasks);
  cudaMemcpyToSymbol(dlab::dlab_tiles_trace, &tr, sizeof(tr));
  cudaDeviceProp p;
  cudaGetDeviceProperties(&p, 0);
  dlab::Ctx c{nullptr, p.multiProcessorCount, nullptr};
  for (int rep = 0; rep < 3; ++rep) {
    cudaMemcpy(d, h.data(), sizeof(double) * n * n, cudaMemcpyHostToDevice);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    dlab::potrf_tiles(c, 1, n, dlab::MatB<double>{d, n, (int64_t)n * n}, 0);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    fprintf(stderr, "rep %d: %.3f ms (%s)\n", rep, ms, cudaGetErrorString(cudaGetLastError()));
  }
  std::vector<long long> ht((size_t)6 * tasks);
  cudaMemcpy(ht.data(), tr, sizeof(long long) * 6 * tasks, cudaMemcpyDeviceToHost);
  long long t0 = ht[0];
  for (int t = 0; t < tasks; ++t) t0 = ht[6 * t] < t0 ? ht[6 * t] : t0;
  printf("ticket,i,j,sm,grab_us,update_us,end_us\n");
  for (int t = 0; t < tasks; ++t)
    printf("%d,%lld,%lld,%lld,%.2f,%.2f,%.2f\n", t, ht[6 * t + 4], ht[6 * t + 5], ht[6 * t + 3],
           (ht[6 * t] - t0) / 1e3, (ht[6 * t + 1] - t0) / 1e3, (ht[6 * t + 2] - t0) / 1e3);
  return 0;
}
