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
// Kernel shape: lane = tet (tets are Morton-sorted, so a warp covers a compact region), the
// warp sweeps all spheres in id order and, per sphere, its planes in CSR order until every
// lane has failed a plane (warp-uniform early exit, the paper's outer loop); planes are
// warp-uniform broadcast loads.  Positive spheres are appended to a per-tet slab
// slab[c * n + t] (c < cap, coalesced over t), already in ascending sphere id.
#include "rpd_ctx.h"
#include "rpd_internal.cuh"

namespace rpd {

__device__ __forceinline__ bool pos(double h) { return __double_as_longlong(h) > 0; }

// Alg. 1 for sphere i and this lane's tet (warp-uniform i; all 32 lanes must call).  The
// loop over neighbours stops when every lane of the warp has failed a plane.
__device__ __forceinline__ bool alg1_warp(int i, const double (&X)[4], const double (&Y)[4],
                                          const double (&Z)[4], bool valid,
                                          const int32_t* __restrict__ nbr_off,
                                          const double4* __restrict__ planes, int N,
                                          long long& ntests, int& e0_out, int& e1_out) {
  const int e0 = __ldg(nbr_off + i), e1 = __ldg(nbr_off + i + 1);
  e0_out = e0;
  e1_out = e1;
  bool alive = valid;
  if (e0 == e1) return alive && (N == 1);
  for (int e = e0; e < e1; ++e) {
    const double4 p = planes[e];
    bool hk[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const double h = fma(p.x, X[k], fma(p.y, Y[k], fma(p.z, Z[k], p.w)));
      hk[k] = pos(h);
    }
    const bool hit = hk[0] | hk[1] | hk[2] | hk[3];
    if (alive) ntests += hk[0] ? 1 : (hk[1] ? 2 : (hk[2] ? 3 : 4));
    alive = alive && hit;
    if (!__any_sync(0xffffffffu, alive)) break;
  }
  return alive;
}

// ------------------------------------------------------------------ pruned filter
// Same booleans as the all-pairs kernel, without evaluating pairs that provably fail:
// a CTA of PF_T Morton-consecutive tets computes the exact lattice AABB B of their vertices;
// sphere i can relate to one of them only if every plane h_ij has max_B h_ij > 0 (if some
// plane has max_B h_ij <= 0, every vertex of every tet of the CTA fails that plane, so Alg. 1
// rejects all of them).  max_B h = d + sum_c max(n_c lo_c, n_c hi_c) is exact (integers).
// The CTA sweeps all spheres with lane = sphere (level 1), compacts the survivors in
// ascending id into shared memory, and its warps then run the exact Alg. 1 (lane = tet) on
// the survivors only (level 2).  DESIGN.md §Prune.
constexpr int PF_T = 128;
constexpr int PF_LIST = 3072;

__global__ void __launch_bounds__(PF_T) k_filter_pruned(
    const double* __restrict__ tx, int64_t T, const int32_t* __restrict__ tet_ids, int64_t n,
    const int32_t* __restrict__ nbr_off, const double4* __restrict__ planes, int N, int lo,
    int hi, int cap, int32_t* __restrict__ k_tet, int32_t* __restrict__ slab,
    int32_t* __restrict__ k_words, unsigned long long* __restrict__ stats) {
  __shared__ double s_box[PF_T / 32][6];
  __shared__ int s_list[PF_LIST];
  __shared__ int s_wc[PF_T / 32];
  __shared__ int s_cnt;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const unsigned FULL = 0xffffffffu;
  const int64_t a = blockIdx.x * (int64_t)PF_T + tid;
  const bool valid = a < n;
  const int64_t t = valid ? (tet_ids ? (int64_t)tet_ids[a] : a) : 0;
  double X[4], Y[4], Z[4];
  double bl[3] = {1e300, 1e300, 1e300}, bh[3] = {-1e300, -1e300, -1e300};
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    X[k] = valid ? tx[(3 * k + 0) * T + t] : 0.0;
    Y[k] = valid ? tx[(3 * k + 1) * T + t] : 0.0;
    Z[k] = valid ? tx[(3 * k + 2) * T + t] : 0.0;
    if (valid) {
      bl[0] = fmin(bl[0], X[k]);
      bh[0] = fmax(bh[0], X[k]);
      bl[1] = fmin(bl[1], Y[k]);
      bh[1] = fmax(bh[1], Y[k]);
      bl[2] = fmin(bl[2], Z[k]);
      bh[2] = fmax(bh[2], Z[k]);
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1)
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      bl[c] = fmin(bl[c], __shfl_xor_sync(FULL, bl[c], o));
      bh[c] = fmax(bh[c], __shfl_xor_sync(FULL, bh[c], o));
    }
  if (lane == 0) {
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      s_box[warp][c] = bl[c];
      s_box[warp][3 + c] = bh[c];
    }
  }
  if (tid == 0) s_cnt = 0;
  __syncthreads();
#pragma unroll
  for (int w = 0; w < PF_T / 32; ++w)
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      bl[c] = fmin(bl[c], s_box[w][c]);
      bh[c] = fmax(bh[c], s_box[w][3 + c]);
    }

  int cnt = 0, words = 0;
  long long ntests = 0, npairs = 0;
  for (int base = lo; base < hi; base += PF_T) {
    // ---- level 1: lane = sphere, exact box rejection
    const int i = base + tid;
    bool pass = false;
    if (i < hi) {
      const int e0 = __ldg(nbr_off + i), e1 = __ldg(nbr_off + i + 1);
      if (e0 == e1) {
        pass = (N == 1);
      } else {
        pass = true;
        for (int e = e0; e < e1; ++e) {
          const double4 p = planes[e];
          const double mh = p.w + fmax(p.x * bl[0], p.x * bh[0]) +
                            fmax(p.y * bl[1], p.y * bh[1]) + fmax(p.z * bl[2], p.z * bh[2]);
          if (!pos(mh)) {
            pass = false;
            break;
          }
        }
      }
    }
    const unsigned b = __ballot_sync(FULL, pass);
    if (lane == 0) s_wc[warp] = __popc(b);
    __syncthreads();
    int off = s_cnt, tot = 0;
#pragma unroll
    for (int w = 0; w < PF_T / 32; ++w) {
      if (w < warp) off += s_wc[w];
      tot += s_wc[w];
    }
    if (pass) s_list[off + __popc(b & ((1u << lane) - 1u))] = i;
    __syncthreads();
    if (tid == 0) s_cnt += tot;
    __syncthreads();
    // ---- level 2: exact Alg. 1 on the survivors, lane = tet
    const int nl = s_cnt;
    if (nl > PF_LIST - PF_T || base + PF_T >= hi) {
      for (int q = 0; q < nl; ++q) {
        const int si = s_list[q];
        int e0, e1;
        const bool alive = alg1_warp(si, X, Y, Z, valid, nbr_off, planes, N, ntests, e0, e1);
        npairs += valid;
        if (alive) {
          if (cnt < cap) slab[(int64_t)cnt * n + a] = si;
          ++cnt;
          words += (e1 - e0 + 31) >> 5;
        }
      }
      __syncthreads();
      if (tid == 0) s_cnt = 0;
      __syncthreads();
    }
  }
  if (valid) {
    k_tet[a] = cnt;
    if (k_words) k_words[a] = words;
  }
  int m = cnt;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    m = max(m, __shfl_xor_sync(FULL, m, o));
    ntests += __shfl_xor_sync(FULL, ntests, o);
    npairs += __shfl_xor_sync(FULL, npairs, o);
  }
  if (lane == 0) {
    atomicMax(stats + ST_MAXK, (unsigned long long)m);
    atomicAdd(stats + ST_REL_TESTS, (unsigned long long)ntests);
    atomicAdd(stats + ST_TESTED, (unsigned long long)npairs);
  }
}

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
      if (cnt < cap) slab[(int64_t)cnt * n + a] = i;
      ++cnt;
      words += (e1 - e0 + 31) >> 5;  // incidence-mask words of this candidate pair
    }
  }
  if (valid) {
    k_tet[a] = cnt;
    if (k_words) k_words[a] = words;
  }
  // max k_tet (warp-aggregated)
  int m = cnt;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, o));
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) ntests += __shfl_xor_sync(0xffffffffu, ntests, o);
  if ((threadIdx.x & 31) == 0) {
    atomicMax(stats + ST_MAXK, (unsigned long long)m);
    atomicAdd(stats + ST_REL_TESTS, (unsigned long long)ntests);
  }
}

__global__ void k_compact_cands(int64_t n, int cap, const int32_t* __restrict__ k_tet,
                                const int32_t* __restrict__ slab,
                                const int32_t* __restrict__ cand_off,
                                int32_t* __restrict__ cand_idx, int32_t* __restrict__ pair_tet,
                                const int32_t* __restrict__ w_off, int32_t* __restrict__ p_moff,
                                const int32_t* __restrict__ nbr_off, int64_t n_pairs) {
  int64_t a = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (a >= n) return;
  int k = k_tet[a];
  int o = cand_off[a];
  int w = w_off ? w_off[a] : 0;
  for (int c = 0; c < k && c < cap; ++c) {
    int i = slab[(int64_t)c * n + a];
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

cudaError_t launch_filter(rpd_ctx* c, const int32_t* tet_ids, int64_t n_tets, int cap,
                          int sphere_lo, int sphere_hi, int32_t* k_tet, int32_t* slab,
                          int32_t* k_words) {
  if (n_tets == 0) return cudaSuccess;
  if (c->filter_mode == RPD_FILTER_PRUNED) {
    k_filter_pruned<<<nblk(n_tets, PF_T), PF_T, 0, c->stream>>>(
        c->st.tx.as<double>(), c->st.T, tet_ids, n_tets, c->st.nbr_off.as<int32_t>(),
        c->st.planes.as<double4>(), (int)c->st.N, sphere_lo, sphere_hi, cap, k_tet, slab,
        k_words, c->stats.as<unsigned long long>());
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
                                 const int32_t* slab, const int32_t* cand_off,
                                 int32_t* cand_idx, int32_t* pair_tet, const int32_t* w_off,
                                 int32_t* p_moff, int64_t n_pairs) {
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
