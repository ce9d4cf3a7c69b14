// Development probe: gap between dependent tiny kernels with and without programmatic
// dependent launch (PDL) on this GPU.
#include <cstdio>
#include <ctime>
#include <cuda_runtime.h>
__global__ void k_tiny(int* x, int n) {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;");
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) x[i] += 1;
}
__device__ __forceinline__ unsigned long long gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__global__ void k_work(int* x, int n) {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  unsigned long long t0 = gtime(), d = 1000ull * (blockIdx.x % 7 + 1);
  while (gtime() - t0 < d) {
  }
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) x[i] += 1;
}
int main() {
  int* x;
  cudaMalloc(&x, sizeof(int) * (1 << 20));
  cudaStream_t s;
  cudaStreamCreate(&s);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int pdl = 0; pdl < 2; ++pdl) {
    for (int blocks : {1, 64, 1024}) {
      for (int rep = 0; rep < 2; ++rep) {
        cudaEventRecord(a, s);
        for (int k = 0; k < 100; ++k) {
          cudaLaunchConfig_t cfg = {};
          cfg.gridDim = blocks;
          cfg.blockDim = 256;
          cfg.stream = s;
          cudaLaunchAttribute at[1];
          at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
          at[0].val.programmaticStreamSerializationAllowed = 1;
          cfg.attrs = at;
          cfg.numAttrs = pdl;
          cudaLaunchKernelEx(&cfg, k_tiny, x, blocks * 256);
        }
        cudaEventRecord(b, s);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        if (rep) printf("pdl %d blocks %d: %.2f us per kernel\n", pdl, blocks, ms * 10.0f);
      }
    }
  }
  // the same 100 launches captured once into a CUDA graph and replayed
  for (int blocks : {1, 64, 1024}) {
    cudaGraph_t g;
    cudaGraphExec_t ge;
    cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal);
    for (int k = 0; k < 100; ++k) k_tiny<<<blocks, 256, 0, s>>>(x, blocks * 256);
    cudaStreamEndCapture(s, &g);
    cudaGraphInstantiate(&ge, g, 0);
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(a, s);
      cudaGraphLaunch(ge, s);
      cudaEventRecord(b, s);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      if (rep) printf("graph blocks %d: %.2f us per kernel\n", blocks, ms * 10.0f);
    }
  }
  // the same with programmatic edges inside the captured graph (PDL launches under capture),
  // and a kernel with real work and a ragged tail (block b spins (b % 7 + 1) us)
  for (int work = 0; work < 2; ++work) {
    for (int pdl = 0; pdl < 2; ++pdl) {
      for (int blocks : {1, 148, 296, 1024}) {
        cudaGraph_t g;
        cudaGraphExec_t ge;
        cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal);
        for (int k = 0; k < 100; ++k) {
          cudaLaunchConfig_t cfg = {};
          cfg.gridDim = blocks;
          cfg.blockDim = 256;
          cfg.stream = s;
          cudaLaunchAttribute at[1];
          at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
          at[0].val.programmaticStreamSerializationAllowed = 1;
          cfg.attrs = at;
          cfg.numAttrs = pdl;
          if (work) cudaLaunchKernelEx(&cfg, k_work, x, blocks * 256);
          else cudaLaunchKernelEx(&cfg, k_tiny, x, blocks * 256);
        }
        cudaError_t e = cudaStreamEndCapture(s, &g);
        if (e != cudaSuccess) { printf("capture failed: %s\n", cudaGetErrorString(e)); return 1; }
        cudaGraphInstantiate(&ge, g, 0);
        for (int rep = 0; rep < 3; ++rep) {
          cudaEventRecord(a, s);
          cudaGraphLaunch(ge, s);
          cudaEventRecord(b, s);
          cudaEventSynchronize(b);
          float ms;
          cudaEventElapsedTime(&ms, a, b);
          if (rep == 2) printf("graph %s pdl %d blocks %d: %.2f us per kernel\n",
                               work ? "work" : "tiny", pdl, blocks, ms * 10.0f);
        }
        cudaGraphExecDestroy(ge);
        cudaGraphDestroy(g);
      }
    }
  }
  printf("last error: %s\n", cudaGetErrorString(cudaGetLastError()));
  // host cost of one plain launch
  {
    cudaStreamSynchronize(s);
    cudaEvent_t c0;
    cudaEventCreate(&c0);
    auto t0 = clock();
    for (int k = 0; k < 1000; ++k) k_tiny<<<1, 256, 0, s>>>(x, 256);
    auto t1 = clock();
    cudaStreamSynchronize(s);
    printf("host launch cost %.2f us\n", 1e6 * double(t1 - t0) / CLOCKS_PER_SEC / 1000.0);
  }
  return 0;
}
