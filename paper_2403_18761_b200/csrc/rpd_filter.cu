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
