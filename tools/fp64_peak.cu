// FP64 (DFMA) peak microbenchmark for the roofline denominator of the FP64-bound kernels.
// Each thread runs 8 independent DFMA chains; grid = 148 SMs x 8 blocks x 256 threads.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(double* out, int iters, double a, double b) {
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
int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  double* out; cudaMalloc(&out, 8);
  int iters = 1 << 20, blocks = sms * 8, threads = 256;
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  k<<<blocks, threads>>>(out, 1024, 0.999999, 1e-7);
  double best = 0;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(e0);
    k<<<blocks, threads>>>(out, iters, 0.999999, 1e-7);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double fl = 2.0 * 8 * (double)iters * blocks * threads;
    double tf = fl / (ms * 1e-3) / 1e12;
    if (tf > best) best = tf;
  }
  printf("{\"fp64_tflops\": %.3f, \"sms\": %d, \"clock_khz_attr\": %d, \"how\": \"8 independent DFMA chains/thread, %d blocks x %d threads, best of 5\"}\n", best, sms, clk, blocks, threads);
  return 0;
}
