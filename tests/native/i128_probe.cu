// Probe: host vs device __int128 arithmetic used by the exact predicates.
#include <stdio.h>
#include "../../paper_2403_18761_b200/csrc/rpd_internal.cuh"
using namespace rpd;
__host__ __device__ void probe(const long long* r1, const long long* r2, const long long* r3, long long* out) {
  // det4 with ONE row first, per-column minors
  for (int c = 0; c < 4; ++c) {
    long long a[3], b[3], d[3];
    int n = 0;
    for (int k = 0; k < 4; ++k)
      if (k != c) { a[n] = r1[k]; b[n] = r2[k]; d[n] = r3[k]; ++n; }
    i128 m = det3_i(a, b, d);
    out[2 * c] = (long long)(m >> 64);
    out[2 * c + 1] = (long long)(unsigned long long)m;
  }
  long long one[4] = {1, 1, 1, 1};
  i128 D = det4_small_row0(one, r1, r2, r3);
  out[8] = (long long)(D >> 64);
  out[9] = (long long)(unsigned long long)D;
  i128 x = (i128)r1[0] * r2[1];
  i128 y = (i128)r1[0] * ((i128)r2[1] * r3[2]);
  out[10] = (long long)(x >> 64); out[11] = (long long)(unsigned long long)x;
  out[12] = (long long)(y >> 64); out[13] = (long long)(unsigned long long)y;
}
__global__ void k(const long long* r, long long* out) { probe(r, r + 4, r + 8, out); }
int main() {
  long long r[12] = {-458752, 1114112, 65536, 589824, -147456, 376832, 376832, 376832,
                     -786432, -262144, -1310720, 262144};
  long long h[14], d[14];
  probe(r, r + 4, r + 8, h);
  long long *dr, *dout;
  cudaMalloc(&dr, sizeof r); cudaMalloc(&dout, sizeof d);
  cudaMemcpy(dr, r, sizeof r, cudaMemcpyHostToDevice);
  k<<<1, 1>>>(dr, dout);
  cudaMemcpy(d, dout, sizeof d, cudaMemcpyDeviceToHost);
  for (int i = 0; i < 14; i += 2) printf("host %lld:%llu  device %lld:%llu\n", h[i], (unsigned long long)h[i+1], d[i], (unsigned long long)d[i+1]);
  return 0;
}
