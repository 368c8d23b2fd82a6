// Microbenchmarks for the FP64/FP32 roofline denominators on B200 (sm_100a).
// MEASURED_PEAKS.json (driver-written) holds HBM copy and bf16 GEMM only; the
// linear-algebra path needs the FP64 DFMA / DMMA and FP32 FFMA ceilings.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o peaks peaks.cu
//   ./peaks  -> one JSON line
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { \
  fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_)); return 1; } } while (0)

constexpr int ITERS = 4096;

__global__ void dfma_loop(double* out, double s) {
  double a[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) a[i] = threadIdx.x * 1e-3 + i;
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) a[i] = fma(a[i], s, 0.5);
  }
  double r = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) r += a[i];
  if (r == 1234.5) out[0] = r;
}

__global__ void ffma_loop(float* out, float s) {
  float a[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) a[i] = threadIdx.x * 1e-3f + i;
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < 16; ++i) a[i] = fmaf(a[i], s, 0.5f);
  }
  float r = 0;
#pragma unroll
  for (int i = 0; i < 16; ++i) r += a[i];
  if (r == 1234.5f) out[0] = r;
}

// m8n8k4 f64: 8*8*4 = 256 FMA per warp-instruction. 4 independent accumulators.
__global__ void dmma884_loop(double* out) {
  double a = threadIdx.x * 1e-3, b = 1.0 - threadIdx.x * 1e-4;
  double c[4][2] = {};
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < 4; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
  }
  double r = 0;
#pragma unroll
  for (int i = 0; i < 4; ++i) r += c[i][0] + c[i][1];
  if (r == 1234.5) out[0] = r;
}

// m16n8k16 f64 (PTX 7.8+, sm_90+): 16*8*16 = 2048 FMA per warp-instruction.
__global__ void dmma16816_loop(double* out) {
  double a[8], b[4];
#pragma unroll
  for (int i = 0; i < 8; ++i) a[i] = threadIdx.x * 1e-3 + i * 1e-2;
#pragma unroll
  for (int i = 0; i < 4; ++i) b[i] = 1.0 - threadIdx.x * 1e-4 - i * 1e-3;
  double c[2][4] = {};
  for (int it = 0; it < ITERS / 8; ++it) {
#pragma unroll
    for (int i = 0; i < 2; ++i)
      asm volatile(
          "mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, "
          "{%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};\n"
          : "+d"(c[i][0]), "+d"(c[i][1]), "+d"(c[i][2]), "+d"(c[i][3])
          : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]),
            "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
  }
  double r = 0;
#pragma unroll
  for (int i = 0; i < 2; ++i) r += c[i][0] + c[i][1] + c[i][2] + c[i][3];
  if (r == 1234.5) out[0] = r;
}

template <typename F>
float time_it(F f) {
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  f();  // warm
  cudaDeviceSynchronize();
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(a);
    f();
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    if (ms < best) best = ms;
  }
  return best;
}

int main() {
  int sms = 0; CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  double* d; float* f; CK(cudaMalloc(&d, 64)); CK(cudaMalloc(&f, 64));
  const int blocks = sms * 8, threads = 256;
  const double warps = double(blocks) * threads / 32;
  float t_dfma = time_it([&] { dfma_loop<<<blocks, threads>>>(d, 0.999); });
  double dfma_tf = double(blocks) * threads * ITERS * 8 * 2 / (t_dfma * 1e-3) / 1e12;
  float t_ffma = time_it([&] { ffma_loop<<<blocks, threads>>>(f, 0.999f); });
  double ffma_tf = double(blocks) * threads * ITERS * 16 * 2 / (t_ffma * 1e-3) / 1e12;
  float t_884 = time_it([&] { dmma884_loop<<<blocks, threads>>>(d); });
  double d884_tf = warps * ITERS * 4 * 256 * 2 / (t_884 * 1e-3) / 1e12;
  float t_16816 = time_it([&] { dmma16816_loop<<<blocks, threads>>>(d); });
  double d16816_tf = warps * (ITERS / 8) * 2 * 2048 * 2 / (t_16816 * 1e-3) / 1e12;
  CK(cudaGetLastError());
  int clk = 0; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  printf("{\"sms\": %d, \"dfma_tflops\": %.2f, \"ffma_tflops\": %.2f, \"dmma_m8n8k4_tflops\": %.2f, "
         "\"dmma_m16n8k16_tflops\": %.2f, \"clock_khz_attr\": %d}\n",
         sms, dfma_tf, ffma_tf, d884_tf, d16816_tf, clk);
  return 0;
}
