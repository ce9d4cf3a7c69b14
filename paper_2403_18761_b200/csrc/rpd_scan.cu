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
// A scan fused with its producer and consumer (one launch instead of flag -> scan -> scatter):
// op.load(k) gives element k's value, op.emit(k, exclusive prefix, value, acc) consumes it,
// op.flush(acc) ends a thread (acc: a per-thread accumulator), op.total(n, total) stores the
// total.  Same single-pass decoupled look-back as k_scan (one array).
template <class Op>
__global__ void __launch_bounds__(SCAN_THREADS) k_scan_op(Op op, int64_t n, int nb,
                                                         unsigned long long* __restrict__ ticket,
                                                         unsigned long long ticket_base,
                                                         unsigned long long* state,
                                                         unsigned epoch, const int* n_dev) {
  __shared__ int sm[32];
  __shared__ int s_tile, s_prefix;
  if (threadIdx.x == 0) s_tile = (int)(atomicAdd(ticket, 1ull) - ticket_base);
  __syncthreads();
  const int tile = s_tile;
  int nb_act = nb;
  if (n_dev) {
    n = *n_dev;
    nb_act = n > 0 ? (int)((n + SCAN_TILE - 1) / SCAN_TILE) : 1;
    if (tile >= nb_act) return;
  }
  op.init();
  const int64_t base = (int64_t)tile * SCAN_TILE + threadIdx.x * SCAN_ITEMS;
  int v[SCAN_ITEMS];
  int s = 0;
#pragma unroll
  for (int k = 0; k < SCAN_ITEMS; ++k) {
    v[k] = base + k < n ? op.load(base + k) : 0;
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
  typename Op::Acc acc = Op::acc0();
#pragma unroll
  for (int k = 0; k < SCAN_ITEMS; ++k) {
    if (base + k < n) op.emit(base + k, ex, v[k], acc);
    ex += v[k];
  }
  op.flush(acc);
  if (tile == nb_act - 1 && threadIdx.x == 0) op.total(n, s_prefix + tot);
}

// dirty tets (partial update): flag = the tet relates to a new sphere (count > 0); the list
// (ascending), the oldest candidate-list epoch of the dirty tets (whose
// lists are re-stamped with the current epoch), the count at scan_out[T] (and in pd)
struct DirtyOp {
  const int32_t* count;
  int32_t* list;
  int32_t* cepoch;
  int* min_epoch;
  int epoch;
  int32_t* scan_out;
  PDyn* pd;
  int* qhdr;  // graph: the BVH work-queue header, zeroed for the re-filter that follows
  typedef int Acc;
  __device__ static Acc acc0() { return 0x7fffffff; }
  __device__ void init() {
    if (pd) epoch = pd->epoch;
  }
  __device__ int load(int64_t t) const { return count[t] > 0; }
  __device__ void emit(int64_t t, int p, int f, Acc& acc) const {
    if (f) {
      list[p] = (int32_t)t;
      acc = min(acc, cepoch[t]);
      cepoch[t] = epoch;
    }
  }
  __device__ void flush(Acc acc) const {
    acc = __reduce_min_sync(0xffffffffu, acc);  // one atomic per warp
    if ((threadIdx.x & 31) == 0 && acc != 0x7fffffff) atomicMin(min_epoch, acc);
  }
  __device__ void total(int64_t n, int tot) const {
    scan_out[n] = tot;
    if (pd) pd->nd = pd->nb = tot;
    if (qhdr) qhdr[0] = qhdr[1] = 0;
  }
};

// spheres whose rows were rebuilt after the oldest candidate list of the dirty tets (the
// restricted re-filter traverses only these); count at scan_out[N] (and in pd)
struct ChangedOp {
  const int32_t* repoch;
  const int* min_epoch;
  int32_t* list;
  int32_t* scan_out;
  PDyn* pd;
  int me;
  typedef int Acc;
  __device__ static Acc acc0() { return 0; }
  __device__ void init() { me = *min_epoch; }
  __device__ int load(int64_t i) const { return repoch[i] > me; }
  __device__ void emit(int64_t i, int p, int f, Acc&) const {
    if (f) list[p] = (int32_t)i;
  }
  __device__ void flush(Acc) const {}
  __device__ void total(int64_t n, int tot) const {
    scan_out[n] = tot;
    if (pd) pd->n_chg = tot;
  }
};

// the positions of the flags equal to val (val < 0: any non-zero flag), ascending; the
// count at *count
struct FlagListOp {
  const uint8_t* flag;
  int32_t* list;
  int* count;
  int val;
  typedef int Acc;
  __device__ static Acc acc0() { return 0; }
  __device__ void init() {}
  __device__ int load(int64_t i) const { return val < 0 ? flag[i] != 0 : flag[i] == val; }
  __device__ void emit(int64_t i, int p, int f, Acc&) const {
    if (f) list[p] = (int32_t)i;
  }
  __device__ void flush(Acc) const {}
  __device__ void total(int64_t, int tot) const { *count = tot; }
};

template <class Op>
static cudaError_t scan_op_impl(rpd_ctx* c, const Op& op, int64_t n, const int* n_dev) {
  const int nb = n > 0 ? (int)((n + SCAN_TILE - 1) / SCAN_TILE) : 1;
  unsigned long long *ticket, *state, base;
  unsigned epoch;
  cudaError_t e;
  if (c->pdd) {  // (inside a captured graph: a fresh region, see scan_impl)
    const size_t words = 1 + (size_t)nb;
    if ((c->g_scan_used + words) * sizeof(unsigned long long) > c->g_scan.cap)
      return cudaErrorInvalidValue;
    ticket = c->g_scan.as<unsigned long long>() + c->g_scan_used;
    c->g_scan_used += words;  // (zeroed by k_pd_init)
    state = ticket + 1;
    base = 0;
    epoch = 1;
  } else {
    const size_t bytes = sizeof(unsigned long long) * ((size_t)nb + 1);
    if (bytes > c->scratch.cap || !c->scratch.p) {
      if ((e = c->scratch.ensure(bytes))) return e;
      if ((e = cudaMemsetAsync(c->scratch.p, 0, c->scratch.cap, c->stream))) return e;
      c->scan_ticket = 0;
    }
    ticket = c->scratch.as<unsigned long long>();
    state = ticket + 1;
    base = c->scan_ticket;
    c->scan_epoch = (c->scan_epoch + 1) & ((1u << 30) - 1);
    if (c->scan_epoch == 0) c->scan_epoch = 1;
    epoch = c->scan_epoch;
    c->scan_ticket += (unsigned long long)nb;
  }
  k_scan_op<Op><<<nb, SCAN_THREADS, 0, c->stream>>>(op, n, nb, ticket, base, state, epoch, n_dev);
  ++c->launches;
  return cudaGetLastError();
}

cudaError_t launch_flag_list(rpd_ctx* c, const uint8_t* flag, int64_t n, int32_t* list,
                             int* count, int val) {
  if (n == 0) return cudaMemsetAsync(count, 0, sizeof(int), c->stream);
  return scan_op_impl(c, FlagListOp{flag, list, count, val}, n, nullptr);
}

cudaError_t launch_dirty_scan(rpd_ctx* c, int64_t T) {
  PDyn* pd = c->pdd;
  DirtyOp op{c->d_count.as<int32_t>(), c->d_list.as<int32_t>(),
             c->cepoch.as<int32_t>(), c->min_epoch.as<int>(), c->epoch,
             c->d_scan.as<int32_t>(), pd, pd ? c->bvh_items.as<int>() : nullptr};
  return scan_op_impl(c, op, T, nullptr);
}

cudaError_t launch_changed_scan(rpd_ctx* c, int64_t N) {
  PDyn* pd = c->pdd;
  ChangedOp op{c->st.repoch.as<int32_t>(), c->min_epoch.as<int>(), c->c_list.as<int32_t>(),
               c->c_scan.as<int32_t>(), pd, 0};
  return scan_op_impl(c, op, N, pd ? &pd->N : nullptr);
}

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
    c->g_scan_used += words;  // (zeroed by k_pd_init at the start of every replay)
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
