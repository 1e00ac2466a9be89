// FP64 SIMT peak microbenchmark for the roofline denominator (B200 has no
// driver-measured FP64 figure in MEASURED_PEAKS.json).  8 independent DFMA
// chains per thread, grid = 148 SMs x 8 CTAs x 256 threads.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 tools/fp64_peak.cu -o tools/fp64_peak
#include <cstdio>
#include <cuda_runtime.h>

__global__ void dfma_loop(double* out, int iters, double a, double b) {
  double x[8];
  for (int i = 0; i < 8; ++i) x[i] = threadIdx.x * 1e-3 + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] = fma(x[i], a, b);
  }
  double s = 0;
  for (int i = 0; i < 8; ++i) s += x[i];
  if (s == 12345.678) out[0] = s;
}

__global__ void dmul_dadd_loop(double* out, int iters, double a, double b) {
  double x[8];
  for (int i = 0; i < 8; ++i) x[i] = threadIdx.x * 1e-3 + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] = __dadd_rn(__dmul_rn(x[i], a), b);
  }
  double s = 0;
  for (int i = 0; i < 8; ++i) s += x[i];
  if (s == 12345.678) out[0] = s;
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* d;
  cudaMalloc(&d, 8);
  const int blocks = sms * 8, threads = 256, iters = 1 << 14;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  double best_fma = 0, best_ma = 0;
  for (int rep = 0; rep < 5; ++rep) {
    float ms;
    cudaEventRecord(e0);
    dfma_loop<<<blocks, threads>>>(d, iters, 0.999999, 1e-7);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    double fl = 2.0 * 8 * (double)iters * blocks * threads;
    if (rep) best_fma = fl / (ms * 1e-3) / 1e12 > best_fma ? fl / (ms * 1e-3) / 1e12 : best_fma;
    cudaEventRecord(e0);
    dmul_dadd_loop<<<blocks, threads>>>(d, iters, 0.999999, 1e-7);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    if (rep) best_ma = fl / (ms * 1e-3) / 1e12 > best_ma ? fl / (ms * 1e-3) / 1e12 : best_ma;
  }
  int clk = 0;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  printf("{\"fp64_tflops\": %.3f, \"fp64_mul_add_tflops\": %.3f, \"sms\": %d, "
         "\"clock_khz_attr\": %d, \"how\": \"8 independent DFMA (resp. DMUL+DADD) chains per "
         "thread, %d CTAs x %d threads x %d iters, best of 4, CUDA events\"}\n",
         best_fma, best_ma, sms, clk, blocks, threads, iters);
  return 0;
}
