// Device twin of pred_harness.cu: evaluates the exact predicates of rpd_internal.cuh in a
// kernel (one thread per case) so host and device results can be compared.
#include <stdio.h>
#include <vector>
#include "../../paper_2403_18761_b200/csrc/rpd_internal.cuh"
using namespace rpd;
__global__ void k(const XPlane* P, int n, int* out) {
  int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= n) return;
  const XPlane* r[4] = {&P[4 * c], &P[4 * c + 1], &P[4 * c + 2], &P[4 * c + 3]};
  int zh = 0;
  out[3 * c] = det4_sign(r);
  out[3 * c + 1] = sos_sign_exact(P[4 * c], P[4 * c + 1], P[4 * c + 2], P[4 * c + 3], &zh);
  out[3 * c + 2] = det4_is_zero(P[4 * c], P[4 * c + 1], P[4 * c + 2], P[4 * c + 3]);
}
int main() {
  std::vector<XPlane> P;
  while (true) {
    XPlane x;
    int rad;
    if (scanf("%d %lld %lld %lld %lld %lld %lld %lld %lld", &rad, &x.a[0], &x.a[1], &x.a[2],
              &x.a[3], &x.n[0], &x.n[1], &x.n[2], &x.rank) != 9)
      break;
    x.radical = rad;
    P.push_back(x);
  }
  int n = (int)P.size() / 4;
  XPlane* dP;
  int* dO;
  cudaMalloc(&dP, sizeof(XPlane) * P.size() + 1);
  cudaMalloc(&dO, sizeof(int) * 3 * n + 4);
  cudaMemcpy(dP, P.data(), sizeof(XPlane) * P.size(), cudaMemcpyHostToDevice);
  k<<<(n + 127) / 128, 128>>>(dP, n, dO);
  std::vector<int> o(3 * n);
  cudaMemcpy(o.data(), dO, sizeof(int) * 3 * n, cudaMemcpyDeviceToHost);
  for (int c = 0; c < n; ++c) printf("%d %d %d\n", o[3 * c], o[3 * c + 1], o[3 * c + 2]);
  return 0;
}
