// rpd_euler.cu -- SURVEY.md §8(f) NEXT-1: fractional Euler characteristics of the restricted
// power elements, computed on the fly by the clip kernel (Sec. 4.1.2).
//
// "such fractional Euler characteristics are inputted together with the mesh, based on the
// combinatorial structure of the tetrahedral mesh": every vertex, edge and face
// of the tet complex carries 1 / (number of tets sharing it) inside each tet, a tet carries 1.
// This file builds those payloads once per mesh:
//
//   * sharing counts: vertices by atomic counters, edges and faces by open-addressing hash
//     tables of their sorted vertex keys (atomicCAS insert + atomicAdd count);
//   * per ctx-local tet a 16-byte record of its 14 sharing counts (4 corners, 6 edges in
//     corner-pair order 01 02 03 12 13 23, 4 faces, face k opposite corner k);
//   * exact arithmetic: every payload is the integer numerator L / count over the common
//     denominator L = lcm of the counts present (one thread, L < 2^50), so the per-piece and
//     per-sphere sums are exact integers -- order-independent, hence bit-identical across
//     launches, kernels and ranks;
//
// and, after every clip / partial update, the per-sphere sums ("For each medial sphere, we
// collect the fractional Euler characteristics for all of its restricted elements",
// PAPER.md:506): Euler(RPC(m_i)) over the pieces of m_i and Euler(RPF(m_i, m_j)) over their
// facets on h_ij, by integer atomics into arrays aligned with the sphere ids and the CSR.
#include "rpd_ctx.h"
#include "rpd_internal.cuh"

namespace rpd {

static inline unsigned nblk(int64_t n, int b) { return (unsigned)((n + b - 1) / b); }

constexpr unsigned long long EMPTY_KEY = ~0ull;
__constant__ int EU_EDGE[6][2] = {{0, 1}, {0, 2}, {0, 3}, {1, 2}, {1, 3}, {2, 3}};

__device__ __forceinline__ unsigned long long mix64(unsigned long long x) {
  x ^= x >> 33;
  x *= 0xff51afd7ed558ccdull;
  x ^= x >> 33;
  x *= 0xc4ceb9fe1a85ec53ull;
  x ^= x >> 33;
  return x;
}

// insert-or-count; returns false if the table is full (never with the sizing below)
__device__ bool ht_add(unsigned long long* keys, unsigned* cnt, unsigned long long mask,
                       unsigned long long key) {
  unsigned long long h = mix64(key) & mask;
  for (unsigned long long probe = 0; probe <= mask; ++probe) {
    const unsigned long long prev = atomicCAS(keys + h, EMPTY_KEY, key);
    if (prev == EMPTY_KEY || prev == key) {
      atomicAdd(cnt + h, 1u);
      return true;
    }
    h = (h + 1) & mask;
  }
  return false;
}

__device__ unsigned ht_get(const unsigned long long* keys, const unsigned* cnt,
                           unsigned long long mask, unsigned long long key) {
  unsigned long long h = mix64(key) & mask;
  for (unsigned long long probe = 0; probe <= mask; ++probe) {
    const unsigned long long k = keys[h];
    if (k == key) return cnt[h];
    if (k == EMPTY_KEY) return 0u;
    h = (h + 1) & mask;
  }
  return 0u;
}

__device__ __forceinline__ void sort3(long long& a, long long& b, long long& c) {
  long long t;
  if (b < a) { t = a; a = b; b = t; }
  if (c < b) { t = b; b = c; c = t; }
  if (b < a) { t = a; a = b; b = t; }
}

// counts of every vertex (atomics), edge and face (hash tables) over all tets of the mesh
__global__ void k_eu_count(int64_t T, const int32_t* __restrict__ tets, int64_t V,
                           unsigned* __restrict__ vcnt, unsigned long long* ekeys,
                           unsigned* ecnt, unsigned long long emask, unsigned long long* fkeys,
                           unsigned* fcnt, unsigned long long fmask, int* err) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= T) return;
  const int4 q = reinterpret_cast<const int4*>(tets)[t];
  const long long v[4] = {q.x, q.y, q.z, q.w};
  bool ok = true;
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    if (v[k] < 0 || v[k] >= V) {
      if (atomicCAS(err, 0, (int)RPD_EINVAL) == 0) {
        err[1] = ERR_TET_INDEX;
        err[2] = (int)t;
      }
      return;
    }
  }
#pragma unroll
  for (int k = 0; k < 4; ++k) atomicAdd(vcnt + v[k], 1u);
#pragma unroll
  for (int e = 0; e < 6; ++e) {
    long long a = v[EU_EDGE[e][0]], b = v[EU_EDGE[e][1]];
    if (b < a) { const long long x = a; a = b; b = x; }
    ok &= ht_add(ekeys, ecnt, emask, (unsigned long long)(a * V + b));
  }
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    long long a = v[k == 0 ? 1 : 0], b = v[k <= 1 ? 2 : 1], c = v[k <= 2 ? 3 : 2];
    sort3(a, b, c);
    ok &= ht_add(fkeys, fcnt, fmask, (unsigned long long)((a * V + b) * V + c));
  }
  if (!ok && atomicCAS(err, 0, (int)RPD_ENOMEM) == 0) err[1] = 0;
}

// per ctx-local tet: the 14 sharing counts as bytes; the set of counts present (bitmap)
__global__ void k_eu_records(int64_t T_local, const int32_t* __restrict__ local_ids,
                             const int32_t* __restrict__ tets, int64_t V,
                             const unsigned* __restrict__ vcnt,
                             const unsigned long long* __restrict__ ekeys,
                             const unsigned* __restrict__ ecnt, unsigned long long emask,
                             const unsigned long long* __restrict__ fkeys,
                             const unsigned* __restrict__ fcnt, unsigned long long fmask,
                             uint4* __restrict__ rec, unsigned* __restrict__ present, int* err) {
  const int64_t l = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (l >= T_local) return;
  const int64_t t = local_ids ? (int64_t)local_ids[l] : l;
  const int4 q = reinterpret_cast<const int4*>(tets)[t];
  const long long v[4] = {q.x, q.y, q.z, q.w};
  unsigned c[16];
#pragma unroll
  for (int k = 0; k < 4; ++k) c[k] = vcnt[v[k]];
#pragma unroll
  for (int e = 0; e < 6; ++e) {
    long long a = v[EU_EDGE[e][0]], b = v[EU_EDGE[e][1]];
    if (b < a) { const long long x = a; a = b; b = x; }
    c[4 + e] = ht_get(ekeys, ecnt, emask, (unsigned long long)(a * V + b));
  }
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    long long a = v[k == 0 ? 1 : 0], b = v[k <= 1 ? 2 : 1], cc = v[k <= 2 ? 3 : 2];
    sort3(a, b, cc);
    c[10 + k] = ht_get(fkeys, fcnt, fmask, (unsigned long long)((a * V + b) * V + cc));
  }
  c[14] = c[15] = 0u;
  unsigned w[4] = {0u, 0u, 0u, 0u};
#pragma unroll
  for (int m = 0; m < 14; ++m) {
    if (c[m] == 0u || c[m] > 255u) {
      if (atomicCAS(err, 0, (int)RPD_EOVERFLOW) == 0) {
        err[1] = 200;  // an element shared by more than 255 tets
        err[2] = (int)l;
      }
      return;
    }
    w[m >> 2] |= c[m] << (8 * (m & 3));
    atomicOr(present + (c[m] >> 5), 1u << (c[m] & 31));
  }
  rec[l] = make_uint4(w[0], w[1], w[2], w[3]);
}

__device__ long long gcd_ll(long long a, long long b) {
  while (b) {
    const long long t = a % b;
    a = b;
    b = t;
  }
  return a;
}

// L = lcm of the counts present; A[n] = L / n (payload numerators); out[0] = L or -1
__global__ void k_eu_lcm(const unsigned* __restrict__ present, long long* __restrict__ A,
                         long long* __restrict__ Lout) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  long long L = 1;
  for (int n = 1; n < 256; ++n) {
    if (!((present[n >> 5] >> (n & 31)) & 1u)) continue;
    const long long g = gcd_ll(L, n);
    if (L / g > (1ll << 50) / n) {
      *Lout = -1;
      return;
    }
    L = L / g * n;
  }
  for (int n = 0; n < 256; ++n) A[n] = n > 0 ? L / n : 0;
  *Lout = L;
}

cudaError_t launch_euler_setup(rpd_ctx* c, const int32_t* tets_all, int64_t T_all, int64_t V,
                               const int32_t* local_ids, int64_t T_local) {
  unsigned long long he = 1, hf = 1;
  while (he <= (unsigned long long)(6 * T_all)) he <<= 1;  // load <= 1/2 even for a tet soup
  while (hf <= (unsigned long long)(4 * T_all)) hf <<= 1;
  he <<= 1;
  hf <<= 1;
  cudaError_t e;
  if ((e = c->eu_tab.ensure((he + hf) * (sizeof(unsigned long long) + sizeof(unsigned)) +
                            sizeof(unsigned) * (V > 0 ? V : 1))))
    return e;
  unsigned long long* ekeys = c->eu_tab.as<unsigned long long>();
  unsigned long long* fkeys = ekeys + he;
  unsigned* ecnt = reinterpret_cast<unsigned*>(fkeys + hf);
  unsigned* fcnt = ecnt + he;
  unsigned* vcnt = fcnt + hf;
  if ((e = cudaMemsetAsync(ekeys, 0xff, sizeof(unsigned long long) * (he + hf), c->stream))) return e;
  if ((e = cudaMemsetAsync(ecnt, 0, sizeof(unsigned) * (he + hf + (V > 0 ? V : 1)), c->stream)))
    return e;
  if ((e = c->eu_rec.ensure(sizeof(uint4) * (T_local > 0 ? T_local : 1)))) return e;
  if ((e = c->eu_A.ensure(sizeof(long long) * 256 + sizeof(unsigned) * 8 + sizeof(long long))))
    return e;
  unsigned* present = reinterpret_cast<unsigned*>(c->eu_A.as<long long>() + 257);
  if ((e = cudaMemsetAsync(present, 0, sizeof(unsigned) * 8, c->stream))) return e;
  int* err = c->errw.as<int>();
  if (T_all > 0) {
    k_eu_count<<<nblk(T_all, 256), 256, 0, c->stream>>>(T_all, tets_all, V, vcnt, ekeys, ecnt,
                                                        he - 1, fkeys, fcnt, hf - 1, err);
    ++c->launches;
  }
  if (T_local > 0) {
    k_eu_records<<<nblk(T_local, 256), 256, 0, c->stream>>>(
        T_local, local_ids, tets_all, V, vcnt, ekeys, ecnt, he - 1, fkeys, fcnt, hf - 1,
        c->eu_rec.as<uint4>(), present, err);
    ++c->launches;
  }
  k_eu_lcm<<<1, 32, 0, c->stream>>>(present, c->eu_A.as<long long>(),
                                    c->eu_A.as<long long>() + 256);
  ++c->launches;
  return cudaGetLastError();
}

// ---------------------------------------------------------------- per-sphere sums

// rpc[i] += Euler of every piece of sphere i; rpf[e] += Euler of every radical facet whose
// neighbour j sits at CSR entry e of row i (binary search: rows are sorted ascending).
// Integer atomics: the sums are exact and independent of the order.
__global__ void k_eu_sums(int64_t n_pieces, const int32_t* __restrict__ sphere,
                          const long long* __restrict__ peu, const int32_t* __restrict__ roff,
                          const int32_t* __restrict__ rj, const long long* __restrict__ re,
                          const int32_t* __restrict__ nbr_off, const int32_t* __restrict__ nbr_idx,
                          unsigned long long* __restrict__ rpc, unsigned long long* __restrict__ rpf,
                          unsigned long long* __restrict__ miss) {
  const int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (q >= n_pieces) return;
  const int i = sphere[q];
  atomicAdd(rpc + i, (unsigned long long)peu[q]);
  const int e0 = nbr_off[i], e1 = nbr_off[i + 1];
  for (int r = roff[q]; r < roff[q + 1]; ++r) {
    const int j = rj[r];
    int lo = e0, hi = e1;  // first entry >= j
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if (nbr_idx[mid] < j) lo = mid + 1;
      else hi = mid;
    }
    if (lo < e1 && nbr_idx[lo] == j) atomicAdd(rpf + lo, (unsigned long long)re[r]);
    else atomicAdd(miss, 1ull);  // a kept facet whose neighbour left the row (R12 degenerate)
  }
}

cudaError_t launch_euler_sums(rpd_ctx* c, const PieceSet& ps) {
  const int64_t N = c->st.N, E = c->st.E;
  cudaError_t e;
  if ((e = c->eu_sum.ensure(sizeof(long long) * (N + E + 1)))) return e;
  long long* rpc = c->eu_sum.as<long long>();
  if ((e = cudaMemsetAsync(rpc, 0, sizeof(long long) * (N + E + 1), c->stream))) return e;
  if (ps.n_pieces > 0) {
    k_eu_sums<<<nblk(ps.n_pieces, 256), 256, 0, c->stream>>>(
        ps.n_pieces, ps.sphere.as<int32_t>(), ps.eu.as<long long>(), ps.rpf_off.as<int32_t>(),
        ps.rpf_j.as<int32_t>(), ps.rpf_e.as<long long>(), c->st.nbr_off.as<int32_t>(),
        c->st.nbr_idx.as<int32_t>(), reinterpret_cast<unsigned long long*>(rpc),
        reinterpret_cast<unsigned long long*>(rpc + N),
        reinterpret_cast<unsigned long long*>(rpc + N + E));
    ++c->launches;
  }
  return cudaGetLastError();
}

}  // namespace rpd
