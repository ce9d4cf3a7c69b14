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
#include <mutex>

#include "rpd_ctx.h"
#include "rpd_internal.cuh"

namespace rpd {

__device__ __forceinline__ bool pos(double h) { return __double_as_longlong(h) > 0; }

// ------------------------------------------------------------------ literal all-pairs

__global__ void __launch_bounds__(256) k_filter_allpairs(
    const double* __restrict__ tx, int64_t T, const int32_t* __restrict__ tet_ids, int64_t n,
    const int32_t* __restrict__ nbr_off, const double4* __restrict__ planes, int N, int lo,
    int hi, int cap, int32_t* __restrict__ k_tet, int32_t* __restrict__ slab,
    uint2* __restrict__ slab_m, int32_t* __restrict__ k_words,
    unsigned long long* __restrict__ stats) {
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
    uint2 cm = make_uint2(0u, 0u);  // cut mask: planes (first 64) not positive at all corners
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
        const int q = e - e0;
        if (!(hk[0] & hk[1] & hk[2] & hk[3]) && q < 64) {
          if (q < 32) cm.x |= 1u << q;
          else cm.y |= 1u << (q - 32);
        }
        if (alive) ntests += hk[0] ? 1 : (hk[1] ? 2 : (hk[2] ? 3 : 4));
        alive = alive && hit;
        if (!__any_sync(0xffffffffu, alive)) break;
      }
    }
    if (alive) {
      if (cnt < cap) {
        slab[a * cap + cnt] = i;
        if (slab_m) slab_m[a * cap + cnt] = cm;
      }
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
  {
    const int slot[2] = {ST_MAXK, ST_REL_TESTS}, kind[2] = {1, 0};
    const unsigned long long v[2] = {(unsigned long long)m, (unsigned long long)ntests};
    block_stats<2>(stats, slot, kind, v);
  }
}

// ------------------------------------------------------------------ box hierarchy

constexpr int BVH_LEAF = 32;    // tets per leaf (one warp)
constexpr int BVH_FAN = 32;     // leaves per super node
constexpr int BVH_PCAP = 64;    // planes of a sphere staged in shared memory (super level)
constexpr int BVH_LCAP = 256;   // planes staged per warp in the leaf kernel
// work distribution of the BVH kernels: 1 = contiguous item ranges per warp (staged planes
// reused across consecutive items of one sphere), 0 = grid-stride (better load balance)
#ifndef RPD_BVH_CONTIG_TOP
#define RPD_BVH_CONTIG_TOP 1
#endif
#ifndef RPD_BVH_CONTIG_SUPER
#define RPD_BVH_CONTIG_SUPER 0
#endif
#ifndef RPD_BVH_CONTIG_LEAF
#define RPD_BVH_CONTIG_LEAF 0
#endif
// top level: test a sphere's staged planes nearest-to-its-centre first (with more than
// BVH_PCAP planes the nearest BVH_PCAP are the ones tested -- still a subset, still exact).
// Off: measured slower at C5 (the warp waits for its slowest lane's failing plane either way)
#ifndef RPD_BVH_SORT
#define RPD_BVH_SORT 0
#endif

// exact lattice AABB of every leaf (32 consecutive tets of the list)
__global__ void k_leaf_boxes(const double* __restrict__ tx, int64_t T,
                             const int32_t* __restrict__ tet_ids, int64_t n,
                             double* __restrict__ leaf, int64_t n_leaf,
                             const int* __restrict__ n_dev, int32_t* __restrict__ zero_a,
                             int32_t* __restrict__ zero_b) {
  if (n_dev) {  // device-driven update: the list length from the device
    n = *n_dev;
    n_leaf = (n + BVH_LEAF - 1) / BVH_LEAF;
  }
  const int64_t a = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (zero_a && a < n) {  // (graph: the counters of the subset, instead of memsets over T)
    zero_a[a] = 0;
    if (zero_b) zero_b[a] = 0;
  }
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
                              double* __restrict__ sup, int64_t n_sup,
                              const int* __restrict__ n_dev) {
  if (n_dev) {
    n_leaf = (*n_dev + BVH_LEAF - 1) / BVH_LEAF;
    n_sup = (n_leaf + BVH_FAN - 1) / BVH_FAN;
  }
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

// phase 1: one warp per (sphere, chunk of 32 super nodes) tests the super-node boxes and queues
// (sphere, super node) items; a sphere with a huge cell becomes many items (load balance).
// Every warp takes a contiguous range of the (sphere, chunk) work so that consecutive chunks
// share the sphere's staged planes (staged once per sphere per warp, not once per chunk), and
// skips the rest of a hidden sphere's chunks at once.
__global__ void __launch_bounds__(BVH_WARPS * 32) k_bvh_top(
    const double* __restrict__ sup, int64_t n_sup, const int32_t* __restrict__ nbr_off,
    const double4* __restrict__ planes, int N, int lo, int hi, int2* __restrict__ items,
    int cap_items, int* __restrict__ n_items, const int32_t* __restrict__ list,
    const int* __restrict__ n_list_dev, const double4* __restrict__ sw,
    const PDyn* __restrict__ pd, int sub) {
  if (pd) {  // device-driven update: sphere range / count and the subset's size from the device
    N = pd->N;
    if (!list) {
      lo = pd->N_old;
      hi = pd->N;
    }
    if (sub) n_sup = ((pd->nb + BVH_LEAF - 1) / BVH_LEAF + BVH_FAN - 1) / BVH_FAN;
  }
  if (n_list_dev) hi = lo + *n_list_dev;
  __shared__ double4 s_pl[BVH_WARPS][BVH_PCAP];
#if RPD_BVH_SORT
  __shared__ double4 s_all[BVH_WARPS][2 * BVH_PCAP];  // staging before the ordering
  __shared__ double s_key[BVH_WARPS][2 * BVH_PCAP];
#endif
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const unsigned FULL = 0xffffffffu;
  double4* sp = s_pl[warp];
  const int64_t n_chunk = (n_sup + 31) >> 5;
  const int64_t gw = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int64_t n_work = (int64_t)(hi - lo) * n_chunk;
  const int64_t per = RPD_BVH_CONTIG_TOP ? (n_work + nw - 1) / nw : 1;
  const int64_t w_end = RPD_BVH_CONTIG_TOP ? min(n_work, (gw + 1) * per) : n_work;
  const int64_t w_step = RPD_BVH_CONTIG_TOP ? 1 : nw;
  int cur_i = -1, k = 0;
  for (int64_t w = gw * per; w < w_end; w += w_step) {
    const int64_t ii = lo + w / n_chunk;
    const int64_t s = (w % n_chunk) * 32 + lane;
    const int i = list ? list[ii] : (int)ii;
    if (i != cur_i) {
      const int e0 = __ldg(nbr_off + i), e1 = __ldg(nbr_off + i + 1);
      k = e1 - e0;
      cur_i = i;
      if (k == 0 && N != 1) {  // hidden sphere (R4): relates to no tet
        if (RPD_BVH_CONTIG_TOP) w = (w / n_chunk + 1) * n_chunk - 1;  // its other chunks
        continue;
      }
#if RPD_BVH_SORT
      if (k > 1) {
        // the first 2 BVH_PCAP planes, keyed by their distance from the sphere's centre
        // h(theta_i) / |n| (integer-valued plane, exact h), the nearest BVH_PCAP kept in order
        const int ks = min(k, 2 * BVH_PCAP);
        const double4 ci = sw[i];
        __syncwarp();
        for (int e = lane; e < ks; e += 32) {
          const double4 p = planes[e0 + e];
          s_all[warp][e] = p;
          const double h = fma(p.x, ci.x, fma(p.y, ci.y, fma(p.z, ci.z, p.w)));
          s_key[warp][e] = h * rsqrt(fma(p.x, p.x, fma(p.y, p.y, p.z * p.z)));
        }
        __syncwarp();
        for (int e = lane; e < ks; e += 32) {
          const double ke = s_key[warp][e];
          int rk = 0;
          for (int f = 0; f < ks; ++f) {
            const double kf = s_key[warp][f];
            rk += kf < ke || (kf == ke && f < e);
          }
          if (rk < BVH_PCAP) sp[rk] = s_all[warp][e];
        }
        __syncwarp();
        if (k > 2 * BVH_PCAP) k = BVH_PCAP;  // (test the nearest BVH_PCAP of the first 128)
      } else {
        stage_planes(sp, planes + e0, k);
      }
#else
      stage_planes(sp, planes + e0, k);
#endif
    } else if (k == 0 && N != 1) {
      continue;
    }
    const bool ok = box_passes_w(sup + 6 * s, s < n_sup, sp, k);
    const unsigned sm = __ballot_sync(FULL, ok);
    if (!sm) continue;
    int base = 0;
    if (lane == 0) base = atomicAdd(n_items, __popc(sm));
    base = __shfl_sync(FULL, base, 0);
    if (ok) {
      const int slot = base + __popc(sm & ((1u << lane) - 1u));
      if (slot < cap_items) items[slot] = make_int2(i, (int)s);
    }
  }
}

// phase 2: one warp per (sphere, super node) item tests the 32 leaf boxes of the super node
// and queues (sphere, leaf) items
__global__ void __launch_bounds__(BVH_WARPS * 32) k_bvh_super(
    const double* __restrict__ leaf, int64_t n_leaf, const int32_t* __restrict__ nbr_off,
    const double4* __restrict__ planes, const int2* __restrict__ sitems,
    const int* __restrict__ n_sitems_p, int cap_sitems, int2* __restrict__ items,
    int cap_items, int* __restrict__ n_items, const int* __restrict__ n_dev) {
  if (n_dev) n_leaf = (*n_dev + BVH_LEAF - 1) / BVH_LEAF;
  __shared__ double4 s_pl[BVH_WARPS][BVH_PCAP];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const unsigned FULL = 0xffffffffu;
  double4* sp = s_pl[warp];
  const int n_sitems = min(*n_sitems_p, cap_sitems);
  const int64_t gw = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  // contiguous item ranges per warp (RPD_BVH_CONTIG_SUPER): the items of one sphere are
  // queued in runs, so the staged planes are reused across consecutive items
  const int64_t per = RPD_BVH_CONTIG_SUPER ? (n_sitems + nw - 1) / nw : 1;
  const int64_t it_end = RPD_BVH_CONTIG_SUPER ? min((int64_t)n_sitems, (gw + 1) * per) : n_sitems;
  int cur_i = -1;
  for (int64_t it = gw * per; it < it_end; it += RPD_BVH_CONTIG_SUPER ? 1 : nw) {
    const int2 item = sitems[it];
    const int i = item.x;
    const int e0 = __ldg(nbr_off + i), e1 = __ldg(nbr_off + i + 1);
    const int k = e1 - e0;
    if (i != cur_i) {
      stage_planes(sp, planes + e0, k);
      cur_i = i;
    }
    const int64_t l = (int64_t)item.y * BVH_FAN + lane;
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

// phase 3: one warp per (sphere, leaf) item: the remaining planes on the leaf box, then the
// exact Alg. 1 (lane = tet)
#ifndef RPD_BVH_LEAF_MINB
#define RPD_BVH_LEAF_MINB 1  // min resident blocks of k_bvh_leaf (a register cap; A/B knob)
#endif
__global__ void __launch_bounds__(BVH_WARPS * 32, RPD_BVH_LEAF_MINB) k_bvh_leaf(
    const double* __restrict__ tx, int64_t T, const int32_t* __restrict__ tet_ids, int64_t n,
    const double* __restrict__ leaf, int64_t n_leaf, const int32_t* __restrict__ nbr_off,
    const double4* __restrict__ planes, const int2* __restrict__ items,
    const int* __restrict__ n_items_p, int cap_items, int cap, int32_t* __restrict__ k_tet,
    int32_t* __restrict__ slab, uint2* __restrict__ slab_m, int32_t* __restrict__ k_words,
    unsigned long long* __restrict__ stats, const int* __restrict__ n_dev) {
  if (n_dev) {
    n = *n_dev;
    n_leaf = (n + BVH_LEAF - 1) / BVH_LEAF;
  }
  extern __shared__ double4 s_lpl[];  // BVH_WARPS x BVH_LCAP planes
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const unsigned FULL = 0xffffffffu;
  double4* sp = s_lpl + warp * BVH_LCAP;
  long long ntests = 0, npairs = 0;
  const int n_items = min(*n_items_p, cap_items);
  const int64_t gw = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int64_t per = RPD_BVH_CONTIG_LEAF ? (n_items + nw - 1) / nw : 1;  // (see k_bvh_super)
  const int64_t it_end = RPD_BVH_CONTIG_LEAF ? min((int64_t)n_items, (gw + 1) * per) : n_items;
  int cur_i = -1;
  for (int64_t it = gw * per; it < it_end; it += RPD_BVH_CONTIG_LEAF ? 1 : nw) {
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
      uint2 cutm = make_uint2(0u, 0u);  // cut mask (first 64 planes): crossing planes not
                                      // positive at all 4 corners of this lane's tet
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
          if (!(hk[0] & hk[1] & hk[2] & hk[3]) && e < 64) {
            if (e < 32) cutm.x |= 1u << e;
            else cutm.y |= 1u << (e - 32);
          }
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
        if (slot < cap) {
          slab[a * cap + slot] = i;
          if (slab_m) slab_m[a * cap + slot] = cutm;
        }
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
  {
    const int slot[2] = {ST_REL_TESTS, ST_TESTED}, kind[2] = {0, 0};
    const unsigned long long v[2] = {(unsigned long long)ntests, (unsigned long long)npairs};
    block_stats<2>(stats, slot, kind, v);
  }
}

__global__ void k_max_ktet(int64_t n, const int32_t* __restrict__ k_tet,
                           unsigned long long* __restrict__ stats, const int* __restrict__ n_dev) {
  if (n_dev) n = *n_dev;
  int64_t a = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  int m = a < n ? k_tet[a] : 0;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, o));
  const int slot[1] = {ST_MAXK}, kind[1] = {1};
  const unsigned long long v[1] = {(unsigned long long)(m > 0 ? m : 0)};
  block_stats<1>(stats, slot, kind, v);
}

// ------------------------------------------------------------------ compaction

// Candidate ids of a tet (distinct) sorted ascending (the BVH filter appends them in arbitrary
// order) with the incidence-mask word offsets of the pairs in sorted order.
// One thread per tet (most lists are short: k_tet mean 2-4, p99 ~11): the tet's slab entries
// are loaded into registers (<= CC_REG of them), each one's rank among them (and the prefix of
// the incidence-mask words of the smaller ids) counted by compare loops, and written to its
// sorted position -- no warp-wide shuffles for lists of one or two entries.  Longer lists go
// to a warp each (second kernel).
// the pair's cut-mask words (incidence-mask layout): the filter's 64-plane mask, all ones
// beyond it (the clip then classifies those planes itself; any superset is safe, the clip
// re-checks every selected plane)
__device__ __forceinline__ void write_cut(unsigned* dst, int words, const uint2* m) {
  const uint2 v = m ? *m : make_uint2(~0u, ~0u);
  for (int w = 0; w < words; ++w) dst[w] = w == 0 ? v.x : (w == 1 ? v.y : ~0u);
}

constexpr int CC_REG = 16;
__global__ void __launch_bounds__(256) k_compact_cands_t(
    int64_t n, int cap, const int32_t* __restrict__ k_tet, const int32_t* __restrict__ slab,
    const int32_t* __restrict__ cand_off, int32_t* __restrict__ cand_idx,
    int32_t* __restrict__ pair_tet, const int32_t* __restrict__ w_off,
    int32_t* __restrict__ p_moff, const int32_t* __restrict__ nbr_off, int64_t n_pairs,
    int32_t* __restrict__ long_list, int* __restrict__ n_long, const uint2* __restrict__ slab_m,
    unsigned* __restrict__ p_cut, const PDyn* __restrict__ pd) {
  const int64_t a = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (pd) {  // device-driven update: batch sizes and the pool tail from the device
    n = pd->nb;
    n_pairs = pd->nc;
    cand_idx += pd->fill_c;
    if (n == 0 && a == 0 && p_moff) p_moff[0] = 0;
  }
  if (a >= n) return;
  const int k = min(k_tet[a], cap);
  const int32_t* s = slab + a * cap;
  const int o = cand_off[a];
  const int w0 = w_off ? w_off[a] : 0;
  if (k <= CC_REG) {
    int v[CC_REG], wd[CC_REG];
#pragma unroll
    for (int m = 0; m < CC_REG; ++m) {
      v[m] = m < k ? __ldg(s + m) : INT_MAX;
      wd[m] = 0;
    }
    if (p_moff) {
#pragma unroll
      for (int m = 0; m < CC_REG; ++m)
        if (m < k) wd[m] = (__ldg(nbr_off + v[m] + 1) - __ldg(nbr_off + v[m]) + 31) >> 5;
    }
#pragma unroll
    for (int j = 0; j < CC_REG; ++j) {
      if (j >= k) break;
      int rank = 0, pre = 0;
#pragma unroll
      for (int m = 0; m < CC_REG; ++m) {
        const bool lt = v[m] < v[j];
        rank += lt;
        pre += lt ? wd[m] : 0;
      }
      cand_idx[o + rank] = v[j];
      if (pair_tet) pair_tet[o + rank] = (int32_t)a;
      if (p_moff) p_moff[o + rank] = w0 + pre;
      if (p_cut) write_cut(p_cut + w0 + pre, wd[j], slab_m + a * cap + j);
    }
  } else {  // a long list: one warp per tet in k_compact_cands_w (rare)
    long_list[atomicAdd(n_long, 1)] = (int32_t)a;
  }
  if (p_moff && a == n - 1) {  // terminal word offset
    int tot = 0;
    for (int m = 0; m < k; ++m) {
      const int vm = s[m];
      tot += (__ldg(nbr_off + vm + 1) - __ldg(nbr_off + vm) + 31) >> 5;
    }
    p_moff[n_pairs] = w0 + tot;
  }
}

// the long lists: rank-sorted by a warp each (their ids distinct), then the incidence-word
// offsets of the pairs by a running warp scan in sorted order
__global__ void k_compact_cands_w(const int32_t* __restrict__ list, const int* __restrict__ n_list,
                                  int64_t n, int cap, const int32_t* __restrict__ k_tet,
                                const int32_t* __restrict__ slab,
                                const int32_t* __restrict__ cand_off,
                                int32_t* __restrict__ cand_idx, int32_t* __restrict__ pair_tet,
                                const int32_t* __restrict__ w_off, int32_t* __restrict__ p_moff,
                                const int32_t* __restrict__ nbr_off, int64_t n_pairs,
                                const uint2* __restrict__ slab_m, unsigned* __restrict__ p_cut,
                                const PDyn* __restrict__ pd) {
  if (pd) cand_idx += pd->fill_c;
  const int lane = threadIdx.x & 31;
  const unsigned FULL = 0xffffffffu;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int64_t nl = *n_list;
  for (int64_t li = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; li < nl; li += nw) {
  const int64_t a = list[li];
  const int k = min(k_tet[a], cap);
  const int32_t* s = slab + a * cap;
  const int o = cand_off[a];
  for (int r0 = 0; r0 < k; r0 += 32) {
    const int j = r0 + lane;
    const int v = j < k ? s[j] : INT_MAX;
    int rank = 0;
    for (int q0 = 0; q0 < k; q0 += 32) {
      const int u = q0 + lane < k ? s[q0 + lane] : INT_MAX;
#pragma unroll 8
      for (int m = 0; m < 32; ++m) rank += __shfl_sync(FULL, u, m) < v;
    }
    if (j < k) {
      cand_idx[o + rank] = v;
      if (pair_tet) pair_tet[o + rank] = (int32_t)a;
    }
  }
  if (!p_moff) continue;
  __syncwarp();
  int w = w_off ? w_off[a] : 0;
  for (int r0 = 0; r0 < k; r0 += 32) {
    const int j = r0 + lane;
    int words = 0;
    if (j < k) {
      const int i = cand_idx[o + j];
      words = (__ldg(nbr_off + i + 1) - __ldg(nbr_off + i) + 31) >> 5;
    }
    int x = words;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const int y = __shfl_up_sync(FULL, x, d);
      if (lane >= d) x += y;
    }
    if (j < k) {
      p_moff[o + j] = w + x - words;
      if (p_cut) {  // the cut mask of sorted candidate j: found by its id in the slab
        const int i = cand_idx[o + j];
        int src = 0;
        for (int m = 0; m < k; ++m) src = s[m] == i ? m : src;
        write_cut(p_cut + w + x - words, words, slab_m + a * cap + src);
      }
    }
    w += __shfl_sync(FULL, x, 31);
  }
  __syncwarp();
  }  // (the terminal word offset is written by k_compact_cands_t)
}


static inline unsigned nblk(int64_t n, int b) { return (unsigned)((n + b - 1) / b); }

// Dirty tet a keeps its old candidates i whose neighbour row is unchanged: rel(t, i) only
// depends on t and N(i), so the boolean is the same as before (R11).
__global__ void k_keep_old(int64_t n, const int32_t* __restrict__ dirty,
                           const int2* __restrict__ co_rows, const int32_t* __restrict__ co_idx,
                           const int32_t* __restrict__ repoch, const int* __restrict__ min_epoch,
                           const int32_t* __restrict__ nbr_off, int cap,
                           int32_t* __restrict__ k_tet, int32_t* __restrict__ slab,
                           uint2* __restrict__ slab_m, int32_t* __restrict__ k_words,
                           const int* __restrict__ n_dev) {
  if (n_dev) n = *n_dev;
  const int lane = threadIdx.x & 31;
  const unsigned FULL = 0xffffffffu;
  const int64_t nwarp = ((int64_t)gridDim.x * blockDim.x) >> 5;
  // warp per tet (grid-stride)
  for (int64_t a = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; a < n; a += nwarp) {
  const int t = dirty[a];
  const int me = *min_epoch;
  const int2 rw = co_rows[t];  // the tet's old candidates in the state pool
  const int q0 = rw.x, q1 = rw.y;
  for (int qb = q0; qb < q1; qb += 32) {
    const int q = qb + lane;
    const int i = q < q1 ? co_idx[q] : 0;
    const bool keep = q < q1 && repoch[i] <= me;  // else re-tested by the traversal
    const unsigned km = __ballot_sync(FULL, keep);
    if (!km) continue;
    int words = keep ? (nbr_off[i + 1] - nbr_off[i] + 31) >> 5 : 0;
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) words += __shfl_xor_sync(FULL, words, d);
    int base = 0;
    if (lane == 0) {
      base = atomicAdd(k_tet + a, __popc(km));
      atomicAdd(k_words + a, words);
    }
    base = __shfl_sync(FULL, base, 0);
    if (keep) {
      const int slot = base + __popc(km & ((1u << lane) - 1u));
      if (slot < cap) {
        slab[a * cap + slot] = i;
        if (slab_m) slab_m[a * cap + slot] = make_uint2(~0u, ~0u);  // (no mask: all planes)
      }
    }
  }
  }
}

cudaError_t launch_keep_old(rpd_ctx* c, const int32_t* dirty, int64_t n_dirty,
                            const CandSet& co, int cap, int32_t* k_tet, int32_t* slab,
                            int32_t* k_words) {
  if (n_dirty == 0) return cudaSuccess;
  const PDyn* pd = c->pdd;
  unsigned grid = nblk(n_dirty * 32, 256);
  if (pd && grid > (unsigned)c->sms * 8) grid = c->sms * 8;  // (grid-stride over the bound)
  k_keep_old<<<grid, 256, 0, c->stream>>>(
      n_dirty, dirty, co.rows.as<int2>(), co.idx.as<int32_t>(), c->st.repoch.as<int32_t>(),
      c->min_epoch.as<int>(), c->st.nbr_off.as<int32_t>(), cap, k_tet, slab,
      slab ? c->slab_m.as<uint2>() : nullptr, k_words, pd ? &pd->nb : nullptr);
  ++c->launches;
  return cudaGetLastError();
}

// list of the spheres whose rows changed (count at c_scan[N])
cudaError_t launch_max_ktet(rpd_ctx* c, int64_t n, const int32_t* k_tet) {
  if (n == 0) return cudaSuccess;
  k_max_ktet<<<nblk(n, 256), 256, 0, c->stream>>>(n, k_tet, c->stats.as<unsigned long long>(),
                                                 c->pdd ? &c->pdd->nb : nullptr);
  ++c->launches;
  return cudaGetLastError();
}

cudaError_t launch_changed_list(rpd_ctx* c, int64_t N) {
  // (device-driven update: N is the grid's bound, the count comes from the device)
  if (N == 0) return cudaMemsetAsync(c->c_scan.p, 0, sizeof(int32_t), c->stream);
  return launch_changed_scan(c, N);
}

cudaError_t launch_filter(rpd_ctx* c, const int32_t* tet_ids, int64_t n_tets, int cap,
                          int sphere_lo, int sphere_hi, int32_t* k_tet, int32_t* slab,
                          int32_t* k_words, const int32_t* sphere_list,
                          const int* n_list_dev) {
  if (n_tets == 0) return cudaSuccess;
  // device-driven update (c->pdd): n_tets is the grids' bound; a tet subset's length and the
  // sphere range come from the device, the work-queue capacities from the host prologue
  PDyn* pd = c->pdd;
  const int* nsub = pd && tet_ids ? &pd->nb : nullptr;
  if (c->filter_mode == RPD_FILTER_PRUNED) {
    const int64_t n_leaf = (n_tets + BVH_LEAF - 1) / BVH_LEAF;
    const int64_t n_sup = (n_leaf + BVH_FAN - 1) / BVH_FAN;
    // boxes of the whole mesh depend on the mesh only: built once per rpd_relations and
    // reused by the dirty-tet detection of every partial update; subsets are rebuilt
    DevBuf& bb = tet_ids ? c->bvh : c->bvh_all;
    cudaError_t e = bb.ensure(sizeof(double) * 6 * (n_leaf + n_sup));
    if (e) return e;
    double* leaf = bb.as<double>();
    double* sup = leaf + 6 * n_leaf;
    if (!nsub) {  // (a graph's subset: zeroed by k_leaf_boxes)
      e = cudaMemsetAsync(k_tet, 0, sizeof(int32_t) * n_tets, c->stream);
      if (!e && k_words) e = cudaMemsetAsync(k_words, 0, sizeof(int32_t) * n_tets, c->stream);
      if (e) return e;
    }
    if (tet_ids || !c->bvh_all_valid) {
      k_leaf_boxes<<<nblk(n_leaf * BVH_LEAF, 256), 256, 0, c->stream>>>(
          c->st.tx.as<double>(), c->st.T, tet_ids, n_tets, leaf, n_leaf, nsub,
          nsub ? k_tet : nullptr, nsub ? k_words : nullptr);
      k_super_boxes<<<nblk(n_sup * BVH_FAN, 256), 256, 0, c->stream>>>(leaf, n_leaf, sup, n_sup,
                                                                      nsub);
      c->launches += 2;
      if (!tet_ids) c->bvh_all_valid = true;
    }
    const int64_t ns = sphere_hi - sphere_lo;
    if (ns > 0) {
      const int sms = c->sms;
      // work-item queues: int2 header {leaf items, super items}, leaf items, super items
      int64_t cap_items = 48 * ns + 4 * n_leaf + 4096;
      int64_t cap_sup = 8 * ns + 4 * n_sup + 4096;
      if (cap_items < c->bvh_min_items) cap_items = c->bvh_min_items;
      if (cap_sup < c->bvh_min_items) cap_sup = c->bvh_min_items;
      if (cap_items > (1 << 30)) cap_items = 1 << 30;
      if (cap_sup > (1 << 30)) cap_sup = 1 << 30;
      if (pd) {
        cap_items = c->dd_cap[tet_ids ? 1 : 0][0];
        cap_sup = c->dd_cap[tet_ids ? 1 : 0][1];
      }
      e = c->bvh_items.ensure(sizeof(int2) * (cap_items + cap_sup + 1));
      if (e) return e;
      int* n_items = c->bvh_items.as<int>();
      int* n_sitems = n_items + 1;
      int2* items = reinterpret_cast<int2*>(c->bvh_items.as<char>() + sizeof(int2));
      int2* sitems = items + cap_items;
      if (!pd) {  // (a graph: zeroed by k_pd_init / the dirty scan)
        e = cudaMemsetAsync(n_items, 0, sizeof(int2), c->stream);
        if (e) return e;
      }
      const int64_t n_chunk = (n_sup + 31) / 32;
      int64_t blocks = (ns * n_chunk + BVH_WARPS - 1) / BVH_WARPS;
      if (blocks > (int64_t)sms * (pd ? 4 : 16)) blocks = (int64_t)sms * (pd ? 4 : 16);
      k_bvh_top<<<(unsigned)blocks, BVH_WARPS * 32, 0, c->stream>>>(
          sup, n_sup, c->st.nbr_off.as<int32_t>(), c->st.planes.as<double4>(), (int)c->st.N,
          sphere_lo, sphere_hi, sitems, (int)cap_sup, n_sitems, sphere_list, n_list_dev,
          c->st.sw.as<double4>(), pd, tet_ids != nullptr);
      k_bvh_super<<<(unsigned)(sms * 16), BVH_WARPS * 32, 0, c->stream>>>(
          leaf, n_leaf, c->st.nbr_off.as<int32_t>(), c->st.planes.as<double4>(), sitems,
          n_sitems, (int)cap_sup, items, (int)cap_items, n_items, nsub);
      // the smem attribute is per device (set once per device, guarded across threads)
      static bool attr_set[RPD_MAX_DEVICES] = {};
      static std::mutex mu;
      const int lsmem = (int)(sizeof(double4) * BVH_LCAP * BVH_WARPS);
      if (c->device < 0 || c->device >= RPD_MAX_DEVICES) return cudaErrorInvalidDevice;
      {
        std::lock_guard<std::mutex> g(mu);
        if (!attr_set[c->device]) {
          e = cudaFuncSetAttribute(k_bvh_leaf, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   lsmem);
          if (e) return e;
          attr_set[c->device] = true;
        }
      }
      k_bvh_leaf<<<(unsigned)(sms * 16), BVH_WARPS * 32, lsmem, c->stream>>>(
          c->st.tx.as<double>(), c->st.T, tet_ids, n_tets, leaf, n_leaf,
          c->st.nbr_off.as<int32_t>(), c->st.planes.as<double4>(), items, n_items,
          (int)cap_items, cap, k_tet, slab, slab ? c->slab_m.as<uint2>() : nullptr, k_words,
          c->stats.as<unsigned long long>(), nsub);
      c->launches += 3;
      c->bvh_cap_items = cap_items < cap_sup ? cap_items : cap_sup;
    }
    if (slab && !nsub) {  // (count-only dirty detection: no maximum; a graph's re-filter takes
                          // it after keep_old)
      k_max_ktet<<<nblk(n_tets, 256), 256, 0, c->stream>>>(n_tets, k_tet,
                                                          c->stats.as<unsigned long long>(), nsub);
      ++c->launches;
    }
    return cudaGetLastError();
  }
  k_filter_allpairs<<<nblk(n_tets, 256), 256, 0, c->stream>>>(
      c->st.tx.as<double>(), c->st.T, tet_ids, n_tets, c->st.nbr_off.as<int32_t>(),
      c->st.planes.as<double4>(), (int)c->st.N, sphere_lo, sphere_hi, cap, k_tet, slab,
      slab ? c->slab_m.as<uint2>() : nullptr, k_words, c->stats.as<unsigned long long>());
  ++c->launches;
  return cudaGetLastError();
}

cudaError_t launch_compact_cands(rpd_ctx* c, int64_t n, int cap, const int32_t* k_tet,
                                 int32_t* slab, const int32_t* cand_off, int32_t* cand_idx,
                                 int32_t* pair_tet, const int32_t* w_off, int32_t* p_moff,
                                 int64_t n_pairs, unsigned* p_cut) {
  const PDyn* pd = c->pdd;  // device-driven update: n, n_pairs are bounds (kernels read pd)
  if (n == 0) {
    if (p_moff) return cudaMemsetAsync(p_moff, 0, sizeof(int32_t), c->stream);
    return cudaSuccess;
  }
  cudaError_t e = c->cand_long.ensure(sizeof(int32_t) * (n + 1));
  if (e) return e;
  int* n_long = c->cand_long.as<int>();
  int32_t* long_list = c->cand_long.as<int32_t>() + 1;
  if (!pd && (e = cudaMemsetAsync(n_long, 0, sizeof(int), c->stream))) return e;
  const uint2* slab_m = p_cut ? c->slab_m.as<uint2>() : nullptr;
  k_compact_cands_t<<<nblk(n, 256), 256, 0, c->stream>>>(n, cap, k_tet, slab, cand_off,
                                                        cand_idx, pair_tet, w_off, p_moff,
                                                        c->st.nbr_off.as<int32_t>(), n_pairs,
                                                        long_list, n_long, slab_m, p_cut, pd);
  // (grid for every list, exits on the device count: long lists are rare)
  k_compact_cands_w<<<(unsigned)c->sms * 4, 256, 0, c->stream>>>(
      long_list, n_long, n, cap, k_tet, slab, cand_off, cand_idx, pair_tet, w_off, p_moff,
      c->st.nbr_off.as<int32_t>(), n_pairs, slab_m, p_cut, pd);
  c->launches += 2;
  return cudaGetLastError();
}

}  // namespace rpd
