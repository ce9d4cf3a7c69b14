#include <stdio.h>
#include "../../paper_2403_18761_b200/csrc/rpd_internal.cuh"
using namespace rpd;
__host__ __device__ void probe(const XPlane* P, int* out) {
  XPlane one;
  for (int k = 0; k < 4; ++k) one.a[k] = 1;
  one.n[0] = one.n[1] = one.n[2] = 0;
  one.radical = 0;
  one.rank = 0;
  const XPlane* d3[4] = {&P[0], &P[1], &P[2], &one};
  out[0] = det4_sign(d3);
  const XPlane* d4[4] = {&P[0], &P[1], &P[2], &P[3]};
  out[1] = det4_sign(d4);
  for (int k = 0; k < 4; ++k) {
    const XPlane* rr[4] = {&P[0], &P[1], &P[2], &P[3]};
    rr[k] = &one;
    out[2 + k] = det4_sign(rr);
  }
  int zh = 0;
  out[6] = sos_sign_exact(P[0], P[1], P[2], P[3], &zh);
  out[7] = zh;
}
__global__ void k(const XPlane* P, int* out) { probe(P, out); }
int main() {
  long long v[36] = {1, -458752, 1114112, 65536, 589824, 512, -512, 1024, 6,
                     1, -147456, 376832, 376832, 376832, 512, 0, 0, 14,
                     1, -786432, -262144, -1310720, 262144, -512, 512, 1024, 4,
                     0, 0, 1, 0, 0, 0, 0, 0, 17};
  XPlane P[4];
  for (int k = 0; k < 4; ++k) {
    P[k].radical = (int)v[9 * k];
    for (int c = 0; c < 4; ++c) P[k].a[c] = v[9 * k + 1 + c];
    for (int c = 0; c < 3; ++c) P[k].n[c] = v[9 * k + 5 + c];
    P[k].rank = v[9 * k + 8];
  }
  int h[8], d[8];
  probe(P, h);
  XPlane* dP; int* dO;
  cudaMalloc(&dP, sizeof P); cudaMalloc(&dO, sizeof d);
  cudaMemcpy(dP, P, sizeof P, cudaMemcpyHostToDevice);
  k<<<1, 1>>>(dP, dO);
  cudaMemcpy(d, dO, sizeof d, cudaMemcpyDeviceToHost);
  printf("sizeof XPlane %zu\n", sizeof(XPlane));
  for (int i = 0; i < 8; ++i) printf("%d: host %d device %d\n", i, h[i], d[i]);
  return 0;
}
