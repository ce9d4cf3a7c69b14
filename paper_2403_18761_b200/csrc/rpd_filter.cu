// rpd_filter.cu -- SURVEY.md §8(a) rows a2 (Alg. 1 relation filter) and a3 (per-tet k_tet
// candidate compaction).
//
// Alg. 1, prose reading (R1), strict (R2), hidden spheres (R4):
//   k_site(i) = 0:  rel(t, i) = (N == 1)
//   otherwise:      rel(t, i) = for all j in N(i): exists vertex v of t with h_ij(v) > 0,
//                   h_ij = PD_j - PD_i (v strictly power-closer to m_i than to m_j).
// Every h_ij(v) is an integer-valued double < 2^35.4 computed exactly (three FMAs on exact
// integer operands with exact partial sums), so the booleans are exact; the "> 0" test reads
// the fp64 bit pattern as int64, which keeps the compares off the FP64 pipe.
//
// Two kernels compute the same booleans:
//  * k_filter_allpairs -- literal "every pair of tet-sphere": lane = tet
//    (Morton order), the warp sweeps all spheres and their planes with a warp-uniform early
//    exit.
//  * k_filter_bvh (RPD_FILTER_PRUNED) -- sphere-centric traversal of a 2-level box hierarchy
//    over the Morton-ordered tets (leaves = 32 tets, super nodes = 32 leaves).  A node is
//    skipped when some plane h_ij has max over the node's exact lattice AABB <= 0: then every
//    vertex of every tet below fails that plane and Alg. 1 rejects them all.  Leaves that
//    survive run the exact Alg. 1, lane = tet.  Work is proportional to the relations, not to
//    T x N.
// Positive pairs go to a per-tet slab slab[a * cap + c]; the compaction sorts each tet's list
// (ascending sphere id, R9) and writes the CSR.
#include "rpd_ctx.h"
#include "rpd_internal.cuh"

namespace rpd {

__device__ __forceinline__ bool pos(double h) { return __double_as_longlong(h) > 0; }

// ------------------------------------------------------------------ literal all-pairs

__global__ void __launch_bounds__(256) k_filter_allpairs(
    const double* __restrict__ tx, int64_t T, const int32_t* __restrict__ tet_ids, int64_t n,
    const int32_t* __restrict__ nbr_off, const double4* __restrict__ planes, int N, int lo,
    int hi, int cap, int32_t* __restrict__ k_tet, int32_t* __restrict__ slab,
    int32_t* __restrict__ k_words, unsigned long long* __restrict__ stats) {
  int64_t a = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  bool valid = a < n;
  int64_t t = valid ? (tet_ids ? (int64_t)tet_ids[a] : a) : 0;
  double X[4], Y[4], Z[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    X[k] = valid ? tx[(3 * k + 0) * T + t] : 0.0;
    Y[k] = valid ? tx[(3 * k + 1) * T + t] : 0.0;
    Z[k] = valid ? tx[(3 * k + 2) * T + t] : 0.0;
  }
  int cnt = 0, words = 0;
  long long ntests = 0;  // literal Alg. 1 vertex tests of this lane
  for (int i = lo; i < hi; ++i) {
    int e0 = __ldg(nbr_off + i), e1 = __ldg(nbr_off + i + 1);
    bool alive = valid;
    if (e0 == e1) {
      alive = alive && (N == 1);
    } else {
      for (int e = e0; e < e1; ++e) {
        double4 p = planes[e];
        bool hk[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          double h = fma(p.x, X[k], fma(p.y, Y[k], fma(p.z, Z[k], p.w)));
          hk[k] = pos(h);
        }
        const bool hit = hk[0] | hk[1] | hk[2] | hk[3];
        if (alive) ntests += hk[0] ? 1 : (hk[1] ? 2 : (hk[2] ? 3 : 4));
        alive = alive && hit;
        if (!__any_sync(0xffffffffu, alive)) break;
      }
    }
    if (alive) {
      if (cnt < cap) slab[a * cap + cnt] = i;
      ++cnt;
      words += (e1 - e0 + 31) >> 5;  // incidence-mask words of this candidate pair
    }
  }
  if (valid) {
    k_tet[a] = cnt;
    if (k_words) k_words[a] = words;
  }
  int m = cnt;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    m = max(m, __shfl_xor_sync(0xffffffffu, m, o));
    ntests += __shfl_xor_sync(0xffffffffu, ntests, o);
  }
  if ((threadIdx.x & 31) == 0) {
    atomicMax(stats + ST_MAXK, (unsigned long long)m);
    atomicAdd(stats + ST_REL_TESTS, (unsigned long long)ntests);
  }
}

// ------------------------------------------------------------------ box hierarchy

constexpr int BVH_LEAF = 32;    // tets per leaf (one warp)
constexpr int BVH_FAN = 32;     // leaves per super node
constexpr int BVH_PCAP = 64;    // planes of a sphere staged in shared memory (super level)
constexpr int BVH_LCAP = 256;   // planes staged per warp in the leaf kernel

// exact lattice AABB of every leaf (32 consecutive tets of the list)
__global__ void k_leaf_boxes(const double* __restrict__ tx, int64_t T,
                             const int32_t* __restrict__ tet_ids, int64_t n,
                             double* __restrict__ leaf, int64_t n_leaf) {
  const int64_t a = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int lane = threadIdx.x & 31;
  const bool valid = a < n;
  const int64_t t = valid ? (tet_ids ? (int64_t)tet_ids[a] : a) : 0;
  double bl[3] = {1e300, 1e300, 1e300}, bh[3] = {-1e300, -1e300, -1e300};
  if (valid) {
#pragma unroll
    for (int k = 0; k < 4; ++k)
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        const double x = tx[(3 * k + c) * T + t];
        bl[c] = fmin(bl[c], x);
        bh[c] = fmax(bh[c], x);
      }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1)
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      bl[c] = fmin(bl[c], __shfl_xor_sync(0xffffffffu, bl[c], o));
      bh[c] = fmax(bh[c], __shfl_xor_sync(0xffffffffu, bh[c], o));
    }
  const int64_t l = a / BVH_LEAF;
  if (lane == 0 && l < n_leaf) {
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      leaf[6 * l + c] = bl[c];
      leaf[6 * l + 3 + c] = bh[c];
    }
  }
}

// AABB of every super node (32 consecutive leaves)
__global__ void k_super_boxes(const double* __restrict__ leaf, int64_t n_leaf,
                              double* __restrict__ sup, int64_t n_sup) {
  const int64_t l = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int lane = threadIdx.x & 31;
  double bl[3] = {1e300, 1e300, 1e300}, bh[3] = {-1e300, -1e300, -1e300};
  if (l < n_leaf) {
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      bl[c] = leaf[6 * l + c];
      bh[c] = leaf[6 * l + 3 + c];
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1)
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      bl[c] = fmin(bl[c], __shfl_xor_sync(0xffffffffu, bl[c], o));
      bh[c] = fmax(bh[c], __shfl_xor_sync(0xffffffffu, bh[c], o));
    }
  const int64_t s = l / BVH_FAN;
  if (lane == 0 && s < n_sup) {
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      sup[6 * s + c] = bl[c];
      sup[6 * s + 3 + c] = bh[c];
    }
  }
}

// Can some tet inside the lane's box B pass the first min(k, BVH_PCAP) planes of the sphere?
// (exact and conservative: passing a subset of the planes is necessary for passing all; the
// leaf kernel checks every plane).  The planes are staged in shared memory once per sphere.
__device__ __forceinline__ bool box_passes_w(const double* __restrict__ B, bool valid,
                                             const double4* __restrict__ sp, int k) {
  if (!valid) return false;
  const double l0 = B[0], l1 = B[1], l2 = B[2], h0 = B[3], h1 = B[4], h2 = B[5];
  const int ce = min(k, BVH_PCAP);
  for (int e = 0; e < ce; ++e) {
    const double4 p = sp[e];
    const double mh =
        p.w + fmax(p.x * l0, p.x * h0) + fmax(p.y * l1, p.y * h1) + fmax(p.z * l2, p.z * h2);
    if (!pos(mh)) return false;
  }
  return true;
}

__device__ __forceinline__ void stage_planes(double4* __restrict__ sp,
                                             const double4* __restrict__ gp, int k) {
  const int lane = threadIdx.x & 31;
  __syncwarp();
  for (int e = lane; e < BVH_PCAP && e < k; e += 32) sp[e] = gp[e];
  __syncwarp();
}

constexpr int BVH_WARPS = 4;

// phase 1: one warp per sphere tests the super-node boxes and queues (sphere, super node)
// work items (a sphere with a huge cell becomes many items: load balance)
__global__ void __launch_bounds__(BVH_WARPS * 32) k_bvh_super(
    const double* __restrict__ sup, int64_t n_sup, const double* __restrict__ leaf,
    int64_t n_leaf, const int32_t* __restrict__ nbr_off,
    const double4* __restrict__ planes, int N, int lo, int hi, int2* __restrict__ items,
    int cap_items, int* __restrict__ n_items, const int32_t* __restrict__ list,
    const int* __restrict__ n_list_dev) {
  if (n_list_dev) hi = lo + *n_list_dev;
  __shared__ double4 s_pl[BVH_WARPS][BVH_PCAP];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const unsigned FULL = 0xffffffffu;
  double4* sp = s_pl[warp];
  const int64_t gw = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t ii = lo + gw; ii < hi; ii += nw) {
    const int i = list ? list[ii] : (int)ii;
    const int e0 = __ldg(nbr_off + i), e1 = __ldg(nbr_off + i + 1);
    const int k = e1 - e0;
    if (k == 0 && N != 1) continue;  // hidden sphere (R4): relates to no tet
    const double4* gp = planes + e0;
    stage_planes(sp, gp, k);
    for (int64_t s0 = 0; s0 < n_sup; s0 += 32) {
      const int64_t s = s0 + lane;
      unsigned sm = __ballot_sync(FULL, box_passes_w(sup + 6 * s, s < n_sup, sp, k));
      while (sm) {
        const int64_t sl = s0 + __ffs(sm) - 1;
        sm &= sm - 1;
        // leaves of the surviving super node (lane = leaf) -> (sphere, leaf) work items
        const int64_t l = sl * BVH_FAN + lane;
        const bool ok = box_passes_w(leaf + 6 * l, l < n_leaf, sp, k);
        const unsigned lm = __ballot_sync(FULL, ok);
        if (!lm) continue;
        int base = 0;
        if (lane == 0) base = atomicAdd(n_items, __popc(lm));
        base = __shfl_sync(FULL, base, 0);
        if (ok) {
          const int slot = base + __popc(lm & ((1u << lane) - 1u));
          if (slot < cap_items) items[slot] = make_int2(i, (int)l);
        }
      }
    }
  }
}

// phase 2: one warp per (sphere, super node) item: leaf boxes, then the exact Alg. 1
// (lane = tet) on the surviving leaves
__global__ void __launch_bounds__(BVH_WARPS * 32) k_bvh_leaf(
    const double* __restrict__ tx, int64_t T, const int32_t* __restrict__ tet_ids, int64_t n,
    const double* __restrict__ leaf, int64_t n_leaf, const int32_t* __restrict__ nbr_off,
    const double4* __restrict__ planes, const int2* __restrict__ items,
    const int* __restrict__ n_items_p, int cap_items, int cap, int32_t* __restrict__ k_tet,
    int32_t* __restrict__ slab, int32_t* __restrict__ k_words,
    unsigned long long* __restrict__ stats) {
  extern __shared__ double4 s_lpl[];  // BVH_WARPS x BVH_LCAP planes
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const unsigned FULL = 0xffffffffu;
  double4* sp = s_lpl + warp * BVH_LCAP;
  long long ntests = 0, npairs = 0;
  const int n_items = min(*n_items_p, cap_items);
  const int64_t gw = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  int cur_i = -1;
  for (int64_t it = gw; it < n_items; it += nw) {
#ifdef RPD_DEBUG_BVH
    const long long t_start = clock64();
    int dbg_leaves = 0, dbg_cross = 0;
#endif
    const int2 item = items[it];
    const int i = item.x;
    const int64_t sl = item.y;  // leaf index
    const int e0 = __ldg(nbr_off + i), e1 = __ldg(nbr_off + i + 1);
    const int k = e1 - e0;
    const double4* gp = planes + e0;
    if (i != cur_i) {
      __syncwarp();
      for (int e = lane; e < BVH_LCAP && e < k; e += 32) sp[e] = gp[e];
      __syncwarp();
      cur_i = i;
    }
    const int words = (k + 31) >> 5;
    {
      const int64_t ll = sl;  // the item's leaf (its box passed the first planes)
      const double* B = leaf + 6 * ll;
      const double l0 = B[0], l1 = B[1], l2 = B[2], h0 = B[3], h1 = B[4], h2 = B[5];
      if (k > BVH_PCAP) {
        // the box test saw only the first BVH_PCAP planes: check the rest (lane = plane)
        bool rej = false;
        for (int ec = BVH_PCAP + lane; ec < k; ec += 32) {
          const double4 p = ec < BVH_LCAP ? sp[ec] : gp[ec];
          const double mx = p.w + fmax(p.x * l0, p.x * h0) + fmax(p.y * l1, p.y * h1) +
                            fmax(p.z * l2, p.z * h2);
          rej |= !pos(mx);
        }
        if (__any_sync(FULL, rej)) continue;  // next item
      }
      const int64_t a = ll * BVH_LEAF + lane;
      const bool valid = a < n;
      const int64_t t = valid ? (tet_ids ? (int64_t)tet_ids[a] : a) : 0;
      double X[4], Y[4], Z[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        X[q] = valid ? tx[(3 * q + 0) * T + t] : 0.0;
        Y[q] = valid ? tx[(3 * q + 1) * T + t] : 0.0;
        Z[q] = valid ? tx[(3 * q + 2) * T + t] : 0.0;
      }
      // planes with min over the leaf box > 0 hold at every vertex of every tet of the leaf;
      // only the planes crossing the box are tested per tet
      bool alive = valid;
      for (int c0 = 0; c0 < k; c0 += 32) {
        const int ec = c0 + lane;
        bool crosses = false;
        if (ec < k) {
          const double4 p = ec < BVH_LCAP ? sp[ec] : gp[ec];
          const double mn = p.w + fmin(p.x * l0, p.x * h0) + fmin(p.y * l1, p.y * h1) +
                            fmin(p.z * l2, p.z * h2);
          crosses = !pos(mn);
        }
        unsigned cm = __ballot_sync(FULL, crosses);
#ifdef RPD_DEBUG_BVH
        dbg_cross += __popc(cm);
#endif
        while (cm) {
          const int e = c0 + __ffs(cm) - 1;
          cm &= cm - 1;
          const double4 p = e < BVH_LCAP ? sp[e] : gp[e];
          bool hk[4];
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const double h = fma(p.x, X[q], fma(p.y, Y[q], fma(p.z, Z[q], p.w)));
            hk[q] = pos(h);
          }
          const bool hit = hk[0] | hk[1] | hk[2] | hk[3];
          if (alive) ntests += hk[0] ? 1 : (hk[1] ? 2 : (hk[2] ? 3 : 4));
          alive = alive && hit;
          if (!__any_sync(FULL, alive)) break;
        }
        if (!__any_sync(FULL, alive)) break;
      }
      npairs += valid;
#ifdef RPD_DEBUG_BVH
      ++dbg_leaves;
#endif
      if (alive) {
        const int slot = atomicAdd(k_tet + a, 1);
        if (slot < cap) slab[a * cap + slot] = i;
        if (k_words) atomicAdd(k_words + a, words);
      }
    }
#ifdef RPD_DEBUG_BVH
    const long long dt = clock64() - t_start;
    if (lane == 0 && dt > 40000)
      printf("bvh_leaf item %lld of %d: sphere %d k %d super %lld leaves %d crossing %d cycles %lld\n",
             (long long)it, n_items, i, k, (long long)sl, dbg_leaves, dbg_cross, dt);
#endif
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    ntests += __shfl_xor_sync(FULL, ntests, o);
    npairs += __shfl_xor_sync(FULL, npairs, o);
  }
  if (lane == 0) {
    atomicAdd(stats + ST_REL_TESTS, (unsigned long long)ntests);
    atomicAdd(stats + ST_TESTED, (unsigned long long)npairs);
  }
}

__global__ void k_max_ktet(int64_t n, const int32_t* __restrict__ k_tet,
                           unsigned long long* __restrict__ stats) {
  int64_t a = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  int m = a < n ? k_tet[a] : 0;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0 && m > 0) atomicMax(stats + ST_MAXK, (unsigned long long)m);
}

// ------------------------------------------------------------------ compaction

__global__ void k_compact_cands(int64_t n, int cap, const int32_t* __restrict__ k_tet,
                                int32_t* __restrict__ slab, const int32_t* __restrict__ cand_off,
                                int32_t* __restrict__ cand_idx, int32_t* __restrict__ pair_tet,
                                const int32_t* __restrict__ w_off, int32_t* __restrict__ p_moff,
                                const int32_t* __restrict__ nbr_off, int64_t n_pairs) {
  int64_t a = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (a >= n) return;
  const int k = min(k_tet[a], cap);
  int32_t* s = slab + a * cap;
  // ascending sphere id (the BVH filter appends in arbitrary order)
  for (int x = 1; x < k; ++x) {
    const int v = s[x];
    int y = x;
    while (y > 0 && s[y - 1] > v) {
      s[y] = s[y - 1];
      --y;
    }
    s[y] = v;
  }
  const int o = cand_off[a];
  int w = w_off ? w_off[a] : 0;
  for (int c = 0; c < k; ++c) {
    const int i = s[c];
    cand_idx[o + c] = i;
    if (pair_tet) pair_tet[o + c] = (int32_t)a;
    if (p_moff) {
      p_moff[o + c] = w;
      w += (nbr_off[i + 1] - nbr_off[i] + 31) >> 5;
    }
  }
  if (p_moff && a == n - 1) p_moff[n_pairs] = w;
}

static inline unsigned nblk(int64_t n, int b) { return (unsigned)((n + b - 1) / b); }

// Dirty tet a keeps its old candidates i whose neighbour row is unchanged: rel(t, i) only
// depends on t and N(i), so the boolean is the same as before (R11).
__global__ void k_keep_old(int64_t n, const int32_t* __restrict__ dirty,
                           const int32_t* __restrict__ co_off, const int32_t* __restrict__ co_idx,
                           const int32_t* __restrict__ repoch, const int* __restrict__ min_epoch,
                           const int32_t* __restrict__ nbr_off, int cap,
                           int32_t* __restrict__ k_tet, int32_t* __restrict__ slab,
                           int32_t* __restrict__ k_words) {
  const int64_t a = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (a >= n) return;
  const int t = dirty[a];
  const int me = *min_epoch;
  for (int q = co_off[t]; q < co_off[t + 1]; ++q) {
    const int i = co_idx[q];
    if (repoch[i] > me) continue;  // re-tested by the traversal
    const int slot = atomicAdd(k_tet + a, 1);
    if (slot < cap) slab[a * cap + slot] = i;
    atomicAdd(k_words + a, (nbr_off[i + 1] - nbr_off[i] + 31) >> 5);
  }
}

cudaError_t launch_keep_old(rpd_ctx* c, const int32_t* dirty, int64_t n_dirty,
                            const CandSet& co, int cap, int32_t* k_tet, int32_t* slab,
                            int32_t* k_words) {
  if (n_dirty == 0) return cudaSuccess;
  k_keep_old<<<nblk(n_dirty, 256), 256, 0, c->stream>>>(
      n_dirty, dirty, co.off.as<int32_t>(), co.idx.as<int32_t>(), c->st.repoch.as<int32_t>(),
      c->min_epoch.as<int>(), c->st.nbr_off.as<int32_t>(), cap, k_tet, slab, k_words);
  ++c->launches;
  return cudaGetLastError();
}

__global__ void k_chg_flags(int64_t N, const int32_t* __restrict__ repoch,
                            const int* __restrict__ min_epoch, uint8_t* __restrict__ flag) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < N) flag[i] = repoch[i] > *min_epoch;
}

__global__ void k_chg_list(int64_t N, const uint8_t* __restrict__ flag,
                           const int32_t* __restrict__ scan, int32_t* __restrict__ list) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < N && flag[i]) list[scan[i]] = (int32_t)i;
}

// list of the spheres whose rows changed (count at c_scan[N])
cudaError_t launch_max_ktet(rpd_ctx* c, int64_t n, const int32_t* k_tet) {
  if (n == 0) return cudaSuccess;
  k_max_ktet<<<nblk(n, 256), 256, 0, c->stream>>>(n, k_tet, c->stats.as<unsigned long long>());
  ++c->launches;
  return cudaGetLastError();
}

cudaError_t launch_changed_list(rpd_ctx* c, int64_t N) {
  if (N > 0) {
    k_chg_flags<<<nblk(N, 256), 256, 0, c->stream>>>(N, c->st.repoch.as<int32_t>(),
                                                     c->min_epoch.as<int>(),
                                                     c->c_flag.as<uint8_t>());
    ++c->launches;
  }
  cudaError_t e = launch_scan_u8(c, c->c_flag.as<uint8_t>(), c->c_scan.as<int32_t>(), N);
  if (e || N == 0) return e;
  k_chg_list<<<nblk(N, 256), 256, 0, c->stream>>>(N, c->c_flag.as<uint8_t>(),
                                                  c->c_scan.as<int32_t>(),
                                                  c->c_list.as<int32_t>());
  ++c->launches;
  return cudaGetLastError();
}

cudaError_t launch_filter(rpd_ctx* c, const int32_t* tet_ids, int64_t n_tets, int cap,
                          int sphere_lo, int sphere_hi, int32_t* k_tet, int32_t* slab,
                          int32_t* k_words, const int32_t* sphere_list,
                          const int* n_list_dev) {
  if (n_tets == 0) return cudaSuccess;
  if (c->filter_mode == RPD_FILTER_PRUNED) {
    const int64_t n_leaf = (n_tets + BVH_LEAF - 1) / BVH_LEAF;
    const int64_t n_sup = (n_leaf + BVH_FAN - 1) / BVH_FAN;
    cudaError_t e = c->bvh.ensure(sizeof(double) * 6 * (n_leaf + n_sup));
    if (e) return e;
    double* leaf = c->bvh.as<double>();
    double* sup = leaf + 6 * n_leaf;
    e = cudaMemsetAsync(k_tet, 0, sizeof(int32_t) * n_tets, c->stream);
    if (!e && k_words) e = cudaMemsetAsync(k_words, 0, sizeof(int32_t) * n_tets, c->stream);
    if (e) return e;
    k_leaf_boxes<<<nblk(n_leaf * BVH_LEAF, 256), 256, 0, c->stream>>>(
        c->st.tx.as<double>(), c->st.T, tet_ids, n_tets, leaf, n_leaf);
    k_super_boxes<<<nblk(n_sup * BVH_FAN, 256), 256, 0, c->stream>>>(leaf, n_leaf, sup, n_sup);
    c->launches += 2;
    const int64_t ns = sphere_hi - sphere_lo;
    if (ns > 0) {
      int sms = 148;
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, c->device);
      // work-item queue: [0] = count, then int2 items
      int64_t cap_items = 48 * ns + 4 * n_leaf + 4096;
      if (cap_items < c->bvh_min_items) cap_items = c->bvh_min_items;
      if (cap_items > (1 << 30)) cap_items = 1 << 30;
      e = c->bvh_items.ensure(sizeof(int2) * (cap_items + 1));
      if (e) return e;
      int* n_items = c->bvh_items.as<int>();
      int2* items = reinterpret_cast<int2*>(c->bvh_items.as<char>() + sizeof(int2));
      e = cudaMemsetAsync(n_items, 0, sizeof(int), c->stream);
      if (e) return e;
      int64_t blocks = (ns + BVH_WARPS - 1) / BVH_WARPS;
      if (blocks > (int64_t)sms * 16) blocks = (int64_t)sms * 16;
      k_bvh_super<<<(unsigned)blocks, BVH_WARPS * 32, 0, c->stream>>>(
          sup, n_sup, leaf, n_leaf, c->st.nbr_off.as<int32_t>(), c->st.planes.as<double4>(), (int)c->st.N,
          sphere_lo, sphere_hi, items, (int)cap_items, n_items, sphere_list, n_list_dev);
      static bool attr_set = false;
      const int lsmem = (int)(sizeof(double4) * BVH_LCAP * BVH_WARPS);
      if (!attr_set) {
        e = cudaFuncSetAttribute(k_bvh_leaf, cudaFuncAttributeMaxDynamicSharedMemorySize, lsmem);
        if (e) return e;
        attr_set = true;
      }
      k_bvh_leaf<<<(unsigned)(sms * 16), BVH_WARPS * 32, lsmem, c->stream>>>(
          c->st.tx.as<double>(), c->st.T, tet_ids, n_tets, leaf, n_leaf,
          c->st.nbr_off.as<int32_t>(), c->st.planes.as<double4>(), items, n_items,
          (int)cap_items, cap, k_tet, slab, k_words, c->stats.as<unsigned long long>());
      c->launches += 2;
      c->bvh_cap_items = cap_items;
    }
    k_max_ktet<<<nblk(n_tets, 256), 256, 0, c->stream>>>(n_tets, k_tet,
                                                        c->stats.as<unsigned long long>());
    ++c->launches;
    return cudaGetLastError();
  }
  k_filter_allpairs<<<nblk(n_tets, 256), 256, 0, c->stream>>>(
      c->st.tx.as<double>(), c->st.T, tet_ids, n_tets, c->st.nbr_off.as<int32_t>(),
      c->st.planes.as<double4>(), (int)c->st.N, sphere_lo, sphere_hi, cap, k_tet, slab,
      k_words, c->stats.as<unsigned long long>());
  ++c->launches;
  return cudaGetLastError();
}

cudaError_t launch_compact_cands(rpd_ctx* c, int64_t n, int cap, const int32_t* k_tet,
                                 int32_t* slab, const int32_t* cand_off, int32_t* cand_idx,
                                 int32_t* pair_tet, const int32_t* w_off, int32_t* p_moff,
                                 int64_t n_pairs) {
  if (n == 0) {
    if (p_moff) return cudaMemsetAsync(p_moff, 0, sizeof(int32_t), c->stream);
    return cudaSuccess;
  }
  k_compact_cands<<<nblk(n, 256), 256, 0, c->stream>>>(n, cap, k_tet, slab, cand_off, cand_idx,
                                                       pair_tet, w_off, p_moff,
                                                       c->st.nbr_off.as<int32_t>(), n_pairs);
  ++c->launches;
  return cudaGetLastError();
}

}  // namespace rpd
