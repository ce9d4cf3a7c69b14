// rpd_scan.cu -- exclusive prefix sums used by the compaction steps:
// out[k] = sum_{m<k} in[m] for k in [0, n], out[n] = total.  One launch per scan, or per group of up to
// five equal-length scans (decoupled look-back over 4096-element tiles).  Deterministic (integer).
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

// Single pass (decoupled look-back): tiles take tickets in launch order, publish their
// aggregate, then warp 0 walks back over the predecessors' published aggregates / inclusive
// prefixes.  Each state word packs {call epoch (30 bit), flag (2 bit), value (32 bit)} so that
// stale words of earlier calls read as "not yet published" and no reset launch is needed.
constexpr unsigned long long F_AGG = 1ull, F_INC = 2ull;

__device__ __forceinline__ unsigned long long st_pack(unsigned epoch, unsigned long long f,
                                                      int v) {
  return ((unsigned long long)epoch << 34) | (f << 32) | (unsigned)v;
}

// K <= 5 arrays of n elements (io.in[a] -> io.out[a]) in one launch: ticket q is tile q % nb
// of array q / nb, so every tile's look-back predecessors hold smaller tickets.
template <class T>
struct ScanIO {
  const T* in[5];
  int* out[5];
};

template <class T>
__global__ void __launch_bounds__(SCAN_THREADS) k_scan(ScanIO<T> io, int64_t n, int nb,
                                                      unsigned long long* __restrict__ ticket,
                                                      unsigned long long ticket_base,
                                                      unsigned long long* state_base,
                                                      unsigned epoch, const int* n_dev) {
  __shared__ int sm[32];
  __shared__ int s_tile, s_prefix;
  if (threadIdx.x == 0) s_tile = (int)(atomicAdd(ticket, 1ull) - ticket_base);
  __syncthreads();
  const int arr = s_tile / nb;
  const int tile = s_tile - arr * nb;
  // device-driven length (nb tiles per array launched for a bound): the tiles beyond it leave
  // at once (no successor waits on them: look-back only reads smaller tickets)
  int nb_act = nb;
  if (n_dev) {
    n = *n_dev;
    nb_act = n > 0 ? (int)((n + SCAN_TILE - 1) / SCAN_TILE) : 1;
    if (tile >= nb_act) return;
  }
  const T* __restrict__ in = io.in[arr];
  int* __restrict__ out = io.out[arr];
  unsigned long long* state = state_base + (int64_t)arr * nb;
  const int64_t base = (int64_t)tile * SCAN_TILE + threadIdx.x * SCAN_ITEMS;
  int v[SCAN_ITEMS];
  int s = 0;
#pragma unroll
  for (int k = 0; k < SCAN_ITEMS; ++k) {
    v[k] = load_item(in, base + k, n);
    s += v[k];
  }
  int tot;
  int ex = block_exclusive_scan(s, sm, &tot);
  if (threadIdx.x < 32) {
    const int lane = threadIdx.x;
    int prefix = 0;
    if (tile == 0) {
      if (lane == 0) atomicExch(state, st_pack(epoch, F_INC, tot));
    } else {
      if (lane == 0) atomicExch(state + tile, st_pack(epoch, F_AGG, tot));
      int j = tile - 1;
      while (true) {
        const int idx = j - lane;
        unsigned long long w = 0;
        unsigned f = 0;
        if (idx >= 0) {
          do {
            w = *(volatile unsigned long long*)(state + idx);
            f = (unsigned)(w >> 34) == epoch ? (unsigned)(w >> 32) & 3u : 0u;
          } while (f == 0);
        }
        const int val = idx >= 0 ? (int)(unsigned)w : 0;
        const unsigned inc = __ballot_sync(0xffffffffu, f == F_INC);
        // lanes up to (and including) the nearest inclusive prefix contribute
        const int stop = inc ? __ffs(inc) - 1 : 31;
        int x = lane <= stop ? val : 0;
#pragma unroll
        for (int d = 16; d > 0; d >>= 1) x += __shfl_xor_sync(0xffffffffu, x, d);
        prefix += x;
        if (inc) break;
        j -= 32;
      }
      if (lane == 0) atomicExch(state + tile, st_pack(epoch, F_INC, prefix + tot));
    }
    if (lane == 0) s_prefix = prefix;
  }
  __syncthreads();
  ex += s_prefix;
#pragma unroll
  for (int k = 0; k < SCAN_ITEMS; ++k) {
    if (base + k < n) out[base + k] = ex;
    ex += v[k];
  }
  if (tile == nb_act - 1 && threadIdx.x == 0) out[n] = s_prefix + tot;
}

// n_dev (device-driven update): the length is read on the device; n is its bound.  Inside a
// captured graph (c->pdd) the look-back state is a fresh region reset by a memset node (ticket
// base 0, epoch 1), so that every replay starts clean.
template <class T>
static cudaError_t scan_impl(rpd_ctx* c, const ScanIO<T>& io, int K, int64_t n,
                             const int* n_dev = nullptr) {
  if (n == 0 && !n_dev) {
    for (int a = 0; a < K; ++a) {
      cudaError_t e = cudaMemsetAsync(io.out[a], 0, sizeof(int32_t), c->stream);
      if (e) return e;
    }
    return cudaSuccess;
  }
  const int nb = n > 0 ? (int)((n + SCAN_TILE - 1) / SCAN_TILE) : 1;
  if (c->pdd) {
    const size_t words = 1 + (size_t)K * nb;
    if ((c->g_scan_used + words) * sizeof(unsigned long long) > c->g_scan.cap)
      return cudaErrorInvalidValue;  // (the prologue sizes the region: a bug if reached)
    unsigned long long* r = c->g_scan.as<unsigned long long>() + c->g_scan_used;
    c->g_scan_used += words;
    cudaError_t e = cudaMemsetAsync(r, 0, words * sizeof(unsigned long long), c->stream);
    if (e) return e;
    k_scan<T><<<nb * K, SCAN_THREADS, 0, c->stream>>>(io, n, nb, r, 0ull, r + 1, 1u, n_dev);
    ++c->launches;
    return cudaGetLastError();
  }
  const size_t bytes = sizeof(unsigned long long) * ((size_t)K * nb + 1);
  if (bytes > c->scratch.cap || !c->scratch.p) {
    cudaError_t e = c->scratch.ensure(bytes);
    if (e) return e;
    e = cudaMemsetAsync(c->scratch.p, 0, c->scratch.cap, c->stream);
    if (e) return e;
    c->scan_ticket = 0;
  }
  unsigned long long* ticket = c->scratch.as<unsigned long long>();
  c->scan_epoch = (c->scan_epoch + 1) & ((1u << 30) - 1);
  if (c->scan_epoch == 0) c->scan_epoch = 1;
  k_scan<T><<<nb * K, SCAN_THREADS, 0, c->stream>>>(io, n, nb, ticket,
                                                     c->scan_ticket, ticket + 1, c->scan_epoch,
                                                     n_dev);
  c->scan_ticket += (unsigned long long)nb * K;
  ++c->launches;
  return cudaGetLastError();
}

cudaError_t launch_scan_i32(rpd_ctx* c, const int32_t* in, int32_t* out, int64_t n,
                            const int* n_dev) {
  return scan_impl<int32_t>(c, ScanIO<int32_t>{{in}, {out}}, 1, n, n_dev);
}
cudaError_t launch_scan_u8(rpd_ctx* c, const uint8_t* in, int32_t* out, int64_t n,
                           const int* n_dev) {
  return scan_impl<uint8_t>(c, ScanIO<uint8_t>{{in}, {out}}, 1, n, n_dev);
}
// K <= 5 equal-length int32 scans in[a] -> out[a] in one launch
cudaError_t launch_scan_i32_multi(rpd_ctx* c, const int32_t* const* in, int32_t* const* out,
                                  int K, int64_t n, const int* n_dev) {
  ScanIO<int32_t> io{};
  for (int a = 0; a < K; ++a) {
    io.in[a] = in[a];
    io.out[a] = out[a];
  }
  return scan_impl<int32_t>(c, io, K, n, n_dev);
}

}  // namespace rpd
