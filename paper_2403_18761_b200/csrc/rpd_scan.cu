// rpd_scan.cu -- exclusive prefix sums used by the compaction steps:
// out[k] = sum_{m<k} in[m] for k in [0, n], out[n] = total.  Three phases: per-tile reduce,
// one-block scan of tile sums, per-tile scan + offset.  Deterministic (integer).
#include "rpd_ctx.h"

namespace rpd {

constexpr int SCAN_THREADS = 256;
constexpr int SCAN_ITEMS = 16;
constexpr int SCAN_TILE = SCAN_THREADS * SCAN_ITEMS;  // 4096

template <class T>
__device__ inline int load_item(const T* in, int64_t k, int64_t n) {
  return k < n ? (int)in[k] : 0;
}

__device__ inline int block_exclusive_scan(int v, int* smem, int* total) {
  // warp scan
  int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  int x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    int y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) smem[w] = x;
  __syncthreads();
  if (w == 0) {
    int nw = blockDim.x >> 5;
    int s = lane < nw ? smem[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      int y = __shfl_up_sync(0xffffffffu, s, o);
      if (lane >= o) s += y;
    }
    if (lane < nw) smem[lane] = s;
  }
  __syncthreads();
  int base = w > 0 ? smem[w - 1] : 0;
  *total = smem[(blockDim.x >> 5) - 1];
  __syncthreads();
  return base + x - v;
}

template <class T>
__global__ void k_scan_reduce(const T* __restrict__ in, int64_t n, int* __restrict__ sums) {
  __shared__ int sm[32];
  int64_t base = (int64_t)blockIdx.x * SCAN_TILE + threadIdx.x * SCAN_ITEMS;
  int s = 0;
#pragma unroll
  for (int k = 0; k < SCAN_ITEMS; ++k) s += load_item(in, base + k, n);
  int tot;
  block_exclusive_scan(s, sm, &tot);
  if (threadIdx.x == 0) sums[blockIdx.x] = tot;
}

__global__ void k_scan_sums(int* __restrict__ sums, int nb) {
  __shared__ int sm[32];
  int carry = 0;
  for (int b0 = 0; b0 < nb; b0 += blockDim.x) {
    int k = b0 + threadIdx.x;
    int v = k < nb ? sums[k] : 0;
    int tot;
    int ex = block_exclusive_scan(v, sm, &tot);
    if (k < nb) sums[k] = carry + ex;
    carry += tot;
  }
  if (threadIdx.x == 0) sums[nb] = carry;
}

template <class T>
__global__ void k_scan_apply(const T* __restrict__ in, int64_t n, const int* __restrict__ sums,
                             int* __restrict__ out, int nb) {
  __shared__ int sm[32];
  int64_t base = (int64_t)blockIdx.x * SCAN_TILE + threadIdx.x * SCAN_ITEMS;
  int v[SCAN_ITEMS];
  int s = 0;
#pragma unroll
  for (int k = 0; k < SCAN_ITEMS; ++k) {
    v[k] = load_item(in, base + k, n);
    s += v[k];
  }
  int tot;
  int ex = block_exclusive_scan(s, sm, &tot) + sums[blockIdx.x];
#pragma unroll
  for (int k = 0; k < SCAN_ITEMS; ++k) {
    if (base + k < n) out[base + k] = ex;
    ex += v[k];
  }
  if (blockIdx.x == nb - 1 && threadIdx.x == 0) out[n] = sums[nb];
}

template <class T>
static cudaError_t scan_impl(rpd_ctx* c, const T* in, int32_t* out, int64_t n) {
  if (n == 0) {
    return cudaMemsetAsync(out, 0, sizeof(int32_t), c->stream);
  }
  int nb = (int)((n + SCAN_TILE - 1) / SCAN_TILE);
  cudaError_t e = c->scratch.ensure(sizeof(int) * (nb + 1));
  if (e) return e;
  int* sums = c->scratch.as<int>();
  k_scan_reduce<T><<<nb, SCAN_THREADS, 0, c->stream>>>(in, n, sums);
  k_scan_sums<<<1, 1024, 0, c->stream>>>(sums, nb);
  k_scan_apply<T><<<nb, SCAN_THREADS, 0, c->stream>>>(in, n, sums, out, nb);
  c->launches += 3;
  return cudaGetLastError();
}

cudaError_t launch_scan_i32(rpd_ctx* c, const int32_t* in, int32_t* out, int64_t n) {
  return scan_impl<int32_t>(c, in, out, n);
}
cudaError_t launch_scan_u8(rpd_ctx* c, const uint8_t* in, int32_t* out, int64_t n) {
  return scan_impl<uint8_t>(c, in, out, n);
}

}  // namespace rpd
