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
#include <cub/cub.cuh>

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

// insert-or-count; returns the slot (and the count before this insertion in *before), or -1
// if the table is full (never with the sizing below)
__device__ long long ht_add(unsigned long long* keys, unsigned* cnt, unsigned long long mask,
                            unsigned long long key, unsigned* before = nullptr) {
  unsigned long long h = mix64(key) & mask;
  for (unsigned long long probe = 0; probe <= mask; ++probe) {
    const unsigned long long prev = atomicCAS(keys + h, EMPTY_KEY, key);
    if (prev == EMPTY_KEY || prev == key) {
      const unsigned b = atomicAdd(cnt + h, 1u);
      if (before) *before = b;
      return (long long)h;
    }
    h = (h + 1) & mask;
  }
  return -1;
}

__device__ long long ht_find(const unsigned long long* keys, unsigned long long mask,
                             unsigned long long key) {
  unsigned long long h = mix64(key) & mask;
  for (unsigned long long probe = 0; probe <= mask; ++probe) {
    const unsigned long long k = keys[h];
    if (k == key) return (long long)h;
    if (k == EMPTY_KEY) return -1;
    h = (h + 1) & mask;
  }
  return -1;
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
                           unsigned* fcnt, unsigned long long fmask, int* fown, int* err) {
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
    ok &= ht_add(ekeys, ecnt, emask, (unsigned long long)(a * V + b)) >= 0;
  }
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    long long a = v[k == 0 ? 1 : 0], b = v[k <= 1 ? 2 : 1], c = v[k <= 2 ? 3 : 2];
    sort3(a, b, c);
    unsigned before = 0u;
    const long long h = ht_add(fkeys, fcnt, fmask, (unsigned long long)((a * V + b) * V + c),
                               &before);
    ok &= h >= 0;
    if (h >= 0 && before < 2u) fown[2 * h + before] = (int)(4 * t + k);  // face owners
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
                             const int* __restrict__ fown, int* __restrict__ adj,
                             uint4* __restrict__ rec, long long* __restrict__ Lt,
                             unsigned* __restrict__ present, int* err) {
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
    const long long h = ht_find(fkeys, fmask, (unsigned long long)((a * V + b) * V + cc));
    c[10 + k] = h >= 0 ? fcnt[h] : 0u;
    // face neighbour (4 t' + k'), -1 on the boundary or at a non-manifold face
    int nb = -1;
    if (h >= 0 && c[10 + k] == 2u) {
      const int o0 = fown[2 * h], o1 = fown[2 * h + 1];
      nb = o0 == (int)(4 * t + k) ? o1 : o0;
    }
    adj[4 * l + k] = nb;
  }
  c[14] = c[15] = 0u;
  unsigned w[4] = {0u, 0u, 0u, 0u};
  long long L = 1;  // the tet's denominator: lcm of its 14 sharing counts
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
    const long long n = c[m];
    long long a = L, b = n;
    while (b) {
      const long long r = a % b;
      a = b;
      b = r;
    }
    if (L / a > (1ll << 62) / n) {
      if (atomicCAS(err, 0, (int)RPD_EOVERFLOW) == 0) {
        err[1] = 201;  // L_t > 2^62
        err[2] = (int)l;
      }
      return;
    }
    L = L / a * n;
  }
  rec[l] = make_uint4(w[0], w[1], w[2], w[3]);
  Lt[l] = L;
}

__device__ long long gcd_ll(long long a, long long b) {
  while (b) {
    const long long t = a % b;
    a = b;
    b = t;
  }
  return a;
}

// The primes p <= 255 dividing some sharing count present, with p^E the largest power of p
// <= 255 (every denominator's p-part divides it): table[j] = p, table[64 + j] = p^E,
// table[128] = P.  The per-sphere sums keep one residue modulo p^E per prime (see k_eu_sums).
__global__ void k_eu_primes(const unsigned* __restrict__ present, long long* __restrict__ table) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  int P = 0;
  for (int p = 2; p < 256; ++p) {
    bool prime = true;
    for (int d = 2; d * d <= p && prime; ++d) prime = p % d != 0;
    if (!prime) continue;
    bool used = false;
    for (int n = p; n < 256 && !used; n += p) used = (present[n >> 5] >> (n & 31)) & 1u;
    if (!used) continue;
    long long pe = p;
    while (pe * p <= 255) pe *= p;
    table[P] = p;
    table[64 + P] = pe;
    ++P;
  }
  table[128] = P;
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
                            sizeof(unsigned) * (V > 0 ? V : 1) + sizeof(int) * 2 * hf)))
    return e;
  unsigned long long* ekeys = c->eu_tab.as<unsigned long long>();
  unsigned long long* fkeys = ekeys + he;
  unsigned* ecnt = reinterpret_cast<unsigned*>(fkeys + hf);
  unsigned* fcnt = ecnt + he;
  unsigned* vcnt = fcnt + hf;
  int* fown = reinterpret_cast<int*>(vcnt + (V > 0 ? V : 1));
  if ((e = cudaMemsetAsync(ekeys, 0xff, sizeof(unsigned long long) * (he + hf), c->stream))) return e;
  if ((e = cudaMemsetAsync(ecnt, 0, sizeof(unsigned) * (he + hf + (V > 0 ? V : 1)), c->stream)))
    return e;
  if ((e = c->eu_rec.ensure(sizeof(uint4) * (T_local > 0 ? T_local : 1)))) return e;
  if ((e = c->eu_adj.ensure(sizeof(int) * 4 * (T_local > 0 ? T_local : 1)))) return e;
  if ((e = c->eu_A.ensure(sizeof(long long) * 512))) return e;
  if ((e = c->eu_Lt.ensure(sizeof(long long) * (T_local > 0 ? T_local : 1)))) return e;
  unsigned* present = reinterpret_cast<unsigned*>(c->eu_A.as<long long>() + 257);
  if ((e = cudaMemsetAsync(present, 0, sizeof(unsigned) * 8, c->stream))) return e;
  int* err = c->errw.as<int>();
  if (T_all > 0) {
    k_eu_count<<<nblk(T_all, 256), 256, 0, c->stream>>>(T_all, tets_all, V, vcnt, ekeys, ecnt,
                                                        he - 1, fkeys, fcnt, hf - 1, fown, err);
    ++c->launches;
  }
  if (T_local > 0) {
    k_eu_records<<<nblk(T_local, 256), 256, 0, c->stream>>>(
        T_local, local_ids, tets_all, V, vcnt, ekeys, ecnt, he - 1, fkeys, fcnt, hf - 1, fown,
        c->eu_adj.as<int>(), c->eu_rec.as<uint4>(), c->eu_Lt.as<long long>(), present, err);
    ++c->launches;
  }
  k_eu_primes<<<1, 32, 0, c->stream>>>(present, c->eu_A.as<long long>());
  ++c->launches;
  return cudaGetLastError();
}

// ---------------------------------------------------------------- per-sphere sums

// Exact sums of fractions with different denominators, for any mesh (no common denominator of
// the whole mesh): a value num / L_t is split by partial fractions into an integer K plus, for
// every prime power q = p^e exactly dividing L_t, a residue a / q (0 <= a < q), scaled to the
// prime's fixed power p^E (the largest <= 255, which every sharing count's p-part divides).  The
// accumulator row of a sum is [K, R_1 .. R_P] (integer adds, order-independent); the value is
// K + sum_j R_j / p_j^E, an integer iff every R_j is a multiple of p_j^E (partial fractions
// are unique), then carried into K (k_eu_final).
struct EuTable {
  int P;
  int p[64];
  int pe[64];
};

__device__ __forceinline__ long long inv_mod(long long a, long long m) {  // a, m coprime
  long long g = m, x = 0, x1 = 1, b = a % m;
  while (b) {  // extended Euclid on (m, b)
    const long long qq = g / b, t = g - qq * b;
    g = b;
    b = t;
    const long long tx = x - qq * x1;
    x = x1;
    x1 = tx;
  }
  x %= m;
  return x < 0 ? x + m : x;
}

// the partial-fraction factors of a tet's denominator L_t (computed once per tet): for every
// prime p_j | L_t, q = p_j^e exactly dividing L_t, m = L_t / q, inv = m^{-1} mod q, and the
// scale p^E / q of the residue; at most 15 distinct primes (14 counts <= 255)
struct FracFactors {
  int n;
  int slot[16];
  long long q[16], m[16], inv[16], sc[16];
};

__device__ void frac_factors(long long L, const EuTable& tb, FracFactors& f) {
  f.n = 0;
  long long r = L;
  for (int j = 0; j < tb.P && r > 1 && f.n < 16; ++j) {
    const long long p = tb.p[j];
    if (r % p) continue;
    long long q = 1;
    while (r % p == 0) {
      r /= p;
      q *= p;
    }
    const int k = f.n++;
    f.slot[k] = j;
    f.q[k] = q;
    f.m[k] = L / q;
    f.inv[k] = inv_mod(f.m[k] % q, q);
    f.sc[k] = tb.pe[j] / q;
  }
}

// acc[0..P] += num / L as integer part + residues (num / L = K + sum_k a_k / q_k)
__device__ void frac_add(unsigned long long* acc, long long num, long long L,
                         const FracFactors& f) {
  long long s = 0;      // sum_k a_k m_k (each term < L)
  __int128 s128 = 0;    // (when L is large)
  const bool big = L > (1ll << 58);
  for (int k = 0; k < f.n; ++k) {
    long long nm = num % f.q[k];
    if (nm < 0) nm += f.q[k];
    const long long a = nm * f.inv[k] % f.q[k];
    if (big) s128 += (__int128)a * f.m[k];
    else s += a * f.m[k];
    if (a) atomicAdd(acc + 1 + f.slot[k], (unsigned long long)(a * f.sc[k]));
  }
  // K = (num - s) / L exactly (partial fractions); floor division of exact multiples
  const long long K = big ? (long long)(((__int128)num - s128) / L) : (num - s) / L;
  if (K) atomicAdd(acc, (unsigned long long)K);
}

// one thread per tet: every piece's Euler into its sphere's row, every radical facet's into the
// row of the CSR entry of (i, j) (binary search: rows are sorted ascending)
__global__ void k_eu_sums(int64_t T, const int32_t* __restrict__ poff,
                          const int32_t* __restrict__ sphere, const long long* __restrict__ peu,
                          const int32_t* __restrict__ roff, const int32_t* __restrict__ rj,
                          const long long* __restrict__ re, const long long* __restrict__ Lt,
                          const int32_t* __restrict__ nbr_off, const int32_t* __restrict__ nbr_idx,
                          int64_t N, unsigned long long* __restrict__ acc, EuTable tb,
                          unsigned long long* __restrict__ miss) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= T) return;
  const int q0 = poff[t], q1 = poff[t + 1];
  if (q0 == q1) return;
  const long long L = Lt[t];
  FracFactors f;
  frac_factors(L, tb, f);
  const int W = 1 + tb.P;
  for (int q = q0; q < q1; ++q) {
    const int i = sphere[q];
    frac_add(acc + (int64_t)W * i, peu[q], L, f);
    const int e0 = nbr_off[i], e1 = nbr_off[i + 1];
    for (int r = roff[q]; r < roff[q + 1]; ++r) {
      const int j = rj[r];
      int lo = e0, hi = e1;  // first entry >= j
      while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (nbr_idx[mid] < j) lo = mid + 1;
        else hi = mid;
      }
      if (lo < e1 && nbr_idx[lo] == j) frac_add(acc + (int64_t)W * (N + lo), re[r], L, f);
      else atomicAdd(miss, 1ull);  // a kept facet whose neighbour left the row (R12 degenerate)
    }
  }
}

// accumulator rows -> integer value (exact when `exact`), value as a double
__global__ void k_eu_final(int64_t n, const unsigned long long* __restrict__ acc, EuTable tb,
                           long long* __restrict__ vi, double* __restrict__ vd,
                           uint8_t* __restrict__ ex) {
  const int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (x >= n) return;
  const unsigned long long* a = acc + (int64_t)(1 + tb.P) * x;
  long long K = (long long)a[0];
  double frac = 0.0;
  bool exact = true;
  for (int j = 0; j < tb.P; ++j) {
    const unsigned long long R = a[1 + j], pe = (unsigned long long)tb.pe[j];
    K += (long long)(R / pe);
    const unsigned long long rho = R % pe;
    exact &= rho == 0ull;
    frac += (double)rho / (double)pe;
  }
  vi[x] = K;
  vd[x] = (double)K + frac;
  ex[x] = exact ? 1 : 0;
}

static EuTable eu_table(rpd_ctx* c) {
  EuTable tb{};
  tb.P = c->eu_P;
  for (int j = 0; j < c->eu_P && j < 64; ++j) {
    tb.p[j] = c->eu_primes[j];
    tb.pe[j] = c->eu_ppow[j];
  }
  return tb;
}

cudaError_t launch_euler_final(rpd_ctx* c, const unsigned long long* acc, int64_t n,
                               long long* vi, double* vd, uint8_t* ex) {
  if (n <= 0) return cudaSuccess;
  k_eu_final<<<nblk(n, 256), 256, 0, c->stream>>>(n, acc, eu_table(c), vi, vd, ex);
  ++c->launches;
  return cudaGetLastError();
}

// eu_acc [(N + E) (1 + P)] accumulators; eu_fin: int64 [N+E] values, double [N+E], uint8 [N+E]
// exactness, and one miss counter
cudaError_t launch_euler_sums(rpd_ctx* c, const PieceSet& ps) {
  const int64_t N = c->st.N, E = c->st.E, W = 1 + c->eu_P, rows = N + E;
  cudaError_t e;
  if ((e = c->eu_acc.ensure(sizeof(long long) * (W * rows + 1)))) return e;
  if ((e = c->eu_fin.ensure((sizeof(long long) + sizeof(double) + 1) * (rows + 1) + 64))) return e;
  unsigned long long* acc = c->eu_acc.as<unsigned long long>();
  if ((e = cudaMemsetAsync(acc, 0, sizeof(long long) * (W * rows + 1), c->stream))) return e;
  const int64_t T = ps.n_tets;
  if (T > 0 && ps.n_pieces > 0) {
    k_eu_sums<<<nblk(T, 128), 128, 0, c->stream>>>(
        T, ps.off.as<int32_t>(), ps.sphere.as<int32_t>(), ps.eu.as<long long>(),
        ps.rpf_off.as<int32_t>(), ps.rpf_j.as<int32_t>(), ps.rpf_e.as<long long>(),
        c->eu_Lt.as<long long>(), c->st.nbr_off.as<int32_t>(), c->st.nbr_idx.as<int32_t>(), N,
        acc, eu_table(c), acc + W * rows);
    ++c->launches;
  }
  long long* vi = c->eu_fin.as<long long>();
  double* vd = reinterpret_cast<double*>(vi + rows + 1);
  uint8_t* ex = reinterpret_cast<uint8_t*>(vd + rows + 1);
  return launch_euler_final(c, acc, rows, vi, vd, ex);
}

// per piece its tet's denominator (rpd_get_euler)
__global__ void k_piece_den(int64_t T, const int32_t* __restrict__ poff,
                            const long long* __restrict__ Lt, long long* __restrict__ den) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= T) return;
  for (int q = poff[t]; q < poff[t + 1]; ++q) den[q] = Lt[t];
}

cudaError_t launch_piece_den(rpd_ctx* c, const PieceSet& ps) {
  cudaError_t e = c->eu_den.ensure(sizeof(long long) * (ps.n_pieces > 0 ? ps.n_pieces : 1));
  if (e || ps.n_tets == 0) return e;
  k_piece_den<<<nblk(ps.n_tets, 256), 256, 0, c->stream>>>(
      ps.n_tets, ps.off.as<int32_t>(), c->eu_Lt.as<long long>(), c->eu_den.as<long long>());
  ++c->launches;
  return cudaGetLastError();
}


// ---------------------------------------------------------------- CC numbers (NEXT-2)
//
// "we can trace their CC numbers using a simple traversal algorithm".  The
// pieces of sphere i are the nodes of RPC(m_i); two pieces in tets sharing face f are joined
// when f is an SoS facet of both (the perturbed cell meets f in a 2-face).  The radical facets
// of m_i on h_ij are the nodes of RPF(m_i, m_j); two in face-adjacent tets are joined when both
// have an edge on the shared face.  Union-find with atomic hooking of the larger root onto the
// smaller (lock-free, the result is the same partition whatever the order), then one count
// per root.

__device__ __forceinline__ int uf_find(int* par, int x) {
  while (true) {
    const int y = par[x];
    if (y == x) return x;
    const int z = par[y];
    if (z != y) par[x] = z;  // path halving (a benign race: z is an ancestor of x)
    x = y;
  }
}

__device__ void uf_union(int* par, int a, int b) {
  while (true) {
    a = uf_find(par, a);
    b = uf_find(par, b);
    if (a == b) return;
    if (a < b) {
      const int t = a;
      a = b;
      b = t;
    }
    if (atomicCAS(par + a, a, b) == a) return;
  }
}

__global__ void k_cc_init(int64_t n, int* __restrict__ par) {
  const int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (x < n) par[x] = (int)x;
}

// index in [lo, hi) of v in an ascending array, or -1
__device__ __forceinline__ int find_sorted(const int32_t* a, int lo, int hi, int v) {
  const int end = hi;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (a[mid] < v) lo = mid + 1;
    else hi = mid;
  }
  return (lo < end && a[lo] == v) ? lo : -1;
}

// one thread per tet: joins its pieces (and their radical facets) with the face neighbours'
// of larger index
__global__ void k_cc_link(int64_t T, const int* __restrict__ adj, const int32_t* __restrict__ poff,
                          const int32_t* __restrict__ psph, const uint8_t* __restrict__ sfm,
                          const int32_t* __restrict__ roff, const int32_t* __restrict__ rj,
                          const uint8_t* __restrict__ rfm, int* __restrict__ par_c,
                          int* __restrict__ par_f) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= T) return;
  const int p0 = poff[t], p1 = poff[t + 1];
  if (p0 == p1) return;
  for (int k = 0; k < 4; ++k) {
    const int nb = adj[4 * t + k];
    if (nb < 0 || (nb >> 2) < t) continue;  // each shared face once
    const int t2 = nb >> 2, k2 = nb & 3;
    const int q0 = poff[t2], q1 = poff[t2 + 1];
    for (int q = p0; q < p1; ++q) {
      const int i = psph[q];
      const int q2 = find_sorted(psph, q0, q1, i);
      if (q2 < 0) continue;
      if (((sfm[q] >> k) & 1) && ((sfm[q2] >> k2) & 1)) uf_union(par_c, q, q2);
      const int r20 = roff[q2], r21 = roff[q2 + 1];
      for (int r = roff[q]; r < roff[q + 1]; ++r) {
        if (!((rfm[r] >> k) & 1)) continue;
        const int r2 = find_sorted(rj, r20, r21, rj[r]);
        if (r2 >= 0 && ((rfm[r2] >> k2) & 1)) uf_union(par_f, r, r2);
      }
    }
  }
}

// one thread per piece: a root piece counts one RPC component of its sphere, a root facet one
// RPF component at the CSR entry of (i, j); comp = the root (smallest index of the component)
__global__ void k_cc_count(int64_t n_pieces, const int32_t* __restrict__ psph,
                           const int32_t* __restrict__ roff, const int32_t* __restrict__ rj,
                           const int32_t* __restrict__ nbr_off,
                           const int32_t* __restrict__ nbr_idx, int* __restrict__ par_c,
                           int* __restrict__ par_f, int* __restrict__ rpc_cc,
                           int* __restrict__ rpf_cc) {
  const int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (q >= n_pieces) return;
  const int i = psph[q];
  const int rc = uf_find(par_c, (int)q);
  if (rc == q) atomicAdd(rpc_cc + i, 1);
  const int e0 = nbr_off[i], e1 = nbr_off[i + 1];
  for (int r = roff[q]; r < roff[q + 1]; ++r) {
    if (uf_find(par_f, r) != r) continue;
    const int e = find_sorted(nbr_idx, e0, e1, rj[r]);
    if (e >= 0) atomicAdd(rpf_cc + e, 1);
  }
}

// final labels (a second pass: roots are final once every union has returned)
__global__ void k_cc_label(int64_t n, int* __restrict__ par) {
  const int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (x < n) par[x] = uf_find(par, (int)x);
}

// cc_out layout: rpc_cc [N], rpf_cc [E]; cc_par: piece parents [n_pieces], facet parents [n_rpf]
cudaError_t launch_cc(rpd_ctx* c, const PieceSet& ps) {
  const int64_t N = c->st.N, E = c->st.E, T = ps.n_tets, np = ps.n_pieces, nr = ps.n_rpf;
  cudaError_t e;
  if ((e = c->cc_par.ensure(sizeof(int) * (np + nr + 1)))) return e;
  if ((e = c->cc_out.ensure(sizeof(int) * (N + E + 1)))) return e;
  int* par_c = c->cc_par.as<int>();
  int* par_f = par_c + np;
  int* rpc_cc = c->cc_out.as<int>();
  if ((e = cudaMemsetAsync(rpc_cc, 0, sizeof(int) * (N + E + 1), c->stream))) return e;
  if (np > 0) {  // (separate index spaces: pieces and radical facets)
    k_cc_init<<<nblk(np, 256), 256, 0, c->stream>>>(np, par_c);
    ++c->launches;
  }
  if (nr > 0) {
    k_cc_init<<<nblk(nr, 256), 256, 0, c->stream>>>(nr, par_f);
    ++c->launches;
  }
  if (T > 0 && np > 0) {
    k_cc_link<<<nblk(T, 128), 128, 0, c->stream>>>(
        T, c->eu_adj.as<int>(), ps.off.as<int32_t>(), ps.sphere.as<int32_t>(),
        ps.sfm.as<uint8_t>(), ps.rpf_off.as<int32_t>(), ps.rpf_j.as<int32_t>(),
        ps.rfm.as<uint8_t>(), par_c, par_f);
    ++c->launches;
    k_cc_count<<<nblk(np, 256), 256, 0, c->stream>>>(
        np, ps.sphere.as<int32_t>(), ps.rpf_off.as<int32_t>(), ps.rpf_j.as<int32_t>(),
        c->st.nbr_off.as<int32_t>(), c->st.nbr_idx.as<int32_t>(), par_c, par_f, rpc_cc,
        rpc_cc + N);
    ++c->launches;
    k_cc_label<<<nblk(np, 256), 256, 0, c->stream>>>(np, par_c);
    ++c->launches;
    if (nr > 0) {
      k_cc_label<<<nblk(nr, 256), 256, 0, c->stream>>>(nr, par_f);
      ++c->launches;
    }
  }
  return cudaGetLastError();
}

// ---------------------------------------------------------------- CC numbers of a sharded job
//
// The tets are sharded over ranks (rpd_set_euler with local_ids; face neighbours are global
// tet ids).  A distributed union-find (DESIGN.md §10 "CC numbers of a sharded job"):
//   1. every rank joins its own pieces (and radical facets) across its interior faces, as
//      launch_cc, and labels each by the global id of its local component's root (its rank's
//      base + the smallest local index: roots are component minima whatever the order);
//   2. for each shard-boundary face f (the neighbour tet is on another rank) every piece of m_i
//      with f as a facet emits a record (key = (f, i), label), every radical facet on h_ij with
//      an edge on f a record (key = (f, i), j, label) -- f = the smaller of the two 4 t + k ids
//      of the shared face, so both sides produce the same key;
//   3. the records of all ranks (all-gathered by the caller) are sorted by key and equal keys
//      (and equal j) joined in a union-find over the global ids -- every rank runs the same
//      unions, and the roots are the component minima, so the partition is the same on all;
//   4. each rank counts its local roots that are global roots (a global component's minimum is
//      its local component's minimum): the sums over ranks are the CC numbers.

__global__ void k_g2l(int64_t T_local, const int32_t* __restrict__ local_ids,
                      int32_t* __restrict__ g2l) {
  const int64_t l = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (l < T_local) g2l[local_ids[l]] = (int32_t)l;
}

// k_cc_link on a shard: the face neighbour's local index through g2l (remote ones skipped)
__global__ void k_cc_link_sh(int64_t T, const int* __restrict__ adj, const int32_t* __restrict__ g2l,
                             const int32_t* __restrict__ poff, const int32_t* __restrict__ psph,
                             const uint8_t* __restrict__ sfm, const int32_t* __restrict__ roff,
                             const int32_t* __restrict__ rj, const uint8_t* __restrict__ rfm,
                             int* __restrict__ par_c, int* __restrict__ par_f) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= T) return;
  const int p0 = poff[t], p1 = poff[t + 1];
  if (p0 == p1) return;
  for (int k = 0; k < 4; ++k) {
    const int nb = adj[4 * t + k];
    if (nb < 0) continue;
    const int t2 = g2l[nb >> 2], k2 = nb & 3;
    if (t2 < 0 || t2 < t) continue;  // remote, or this face from the other side
    const int q0 = poff[t2], q1 = poff[t2 + 1];
    for (int q = p0; q < p1; ++q) {
      const int i = psph[q];
      const int q2 = find_sorted(psph, q0, q1, i);
      if (q2 < 0) continue;
      if (((sfm[q] >> k) & 1) && ((sfm[q2] >> k2) & 1)) uf_union(par_c, q, q2);
      const int r20 = roff[q2], r21 = roff[q2 + 1];
      for (int r = roff[q]; r < roff[q + 1]; ++r) {
        if (!((rfm[r] >> k) & 1)) continue;
        const int r2 = find_sorted(rj, r20, r21, rj[r]);
        if (r2 >= 0 && ((rfm[r2] >> k2) & 1)) uf_union(par_f, r, r2);
      }
    }
  }
}

// boundary records of the shard (atomic append; sorted later): RPC key (f << 21 | i), label;
// RPF key (f << 21 | i), j, label.  Labels: global ids of the local roots.
__global__ void k_cc_bnd(int64_t T, const int32_t* __restrict__ local_ids,
                         const int* __restrict__ adj, const int32_t* __restrict__ g2l,
                         const int32_t* __restrict__ poff, const int32_t* __restrict__ psph,
                         const uint8_t* __restrict__ sfm, const int32_t* __restrict__ roff,
                         const int32_t* __restrict__ rj, const uint8_t* __restrict__ rfm,
                         int* __restrict__ par_c, int* __restrict__ par_f, long long base_c,
                         long long base_f, unsigned long long* __restrict__ key_c,
                         int32_t* __restrict__ lab_c, unsigned long long* __restrict__ key_f,
                         int32_t* __restrict__ j_f, int32_t* __restrict__ lab_f,
                         int* __restrict__ n_rec) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= T) return;
  const int p0 = poff[t], p1 = poff[t + 1];
  if (p0 == p1) return;
  const long long tg = local_ids[t];
  for (int k = 0; k < 4; ++k) {
    const int nb = adj[4 * t + k];
    if (nb < 0 || g2l[nb >> 2] >= 0) continue;  // boundary of the mesh, or an interior face
    const unsigned long long f = (unsigned long long)min(4 * tg + k, (long long)nb);
    for (int q = p0; q < p1; ++q) {
      const unsigned long long key = (f << 21) | (unsigned long long)psph[q];
      if ((sfm[q] >> k) & 1) {
        const int s = atomicAdd(n_rec, 1);
        key_c[s] = key;
        lab_c[s] = (int32_t)(base_c + uf_find(par_c, q));
      }
      for (int r = roff[q]; r < roff[q + 1]; ++r) {
        if (!((rfm[r] >> k) & 1)) continue;
        const int s = atomicAdd(n_rec + 1, 1);
        key_f[s] = key;
        j_f[s] = rj[r];
        lab_f[s] = (int32_t)(base_f + uf_find(par_f, r));
      }
    }
  }
}

__global__ void k_cc_init_range(int64_t n, int* __restrict__ par) {
  for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < n;
       x += (int64_t)gridDim.x * blockDim.x)
    par[x] = (int)x;
}

// sorted RPC records: equal neighbouring keys are the two sides of a face -> join
__global__ void k_cc_join_c(int64_t n, const unsigned long long* __restrict__ key,
                            const int32_t* __restrict__ lab, int* __restrict__ par) {
  for (int64_t p = 1 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < n;
       p += (int64_t)gridDim.x * blockDim.x)
    if (key[p] == key[p - 1]) uf_union(par, lab[p], lab[p - 1]);
}

// sorted RPF records (value = record index): within a run of equal keys, equal j -> join
__global__ void k_cc_join_f(int64_t n, const unsigned long long* __restrict__ key,
                            const int32_t* __restrict__ idx, const int32_t* __restrict__ jf,
                            const int32_t* __restrict__ lab, int* __restrict__ par) {
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < n;
       p += (int64_t)gridDim.x * blockDim.x) {
    const int a = idx[p];
    for (int64_t q = p + 1; q < n && key[q] == key[p]; ++q) {
      const int b = idx[q];
      if (jf[a] == jf[b]) uf_union(par, lab[a], lab[b]);
    }
  }
}

// this rank's contributions: its local roots that are global roots, per sphere / CSR entry
__global__ void k_cc_count_sh(int64_t n_pieces, const int32_t* __restrict__ psph,
                              const int32_t* __restrict__ roff, const int32_t* __restrict__ rj,
                              const int32_t* __restrict__ nbr_off,
                              const int32_t* __restrict__ nbr_idx, int* __restrict__ lpar_c,
                              int* __restrict__ lpar_f, int* __restrict__ gpar_c,
                              int* __restrict__ gpar_f, long long base_c, long long base_f,
                              int* __restrict__ rpc_cc, int* __restrict__ rpf_cc) {
  const int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (q >= n_pieces) return;
  const int i = psph[q];
  if (uf_find(lpar_c, (int)q) == q && uf_find(gpar_c, (int)(base_c + q)) == base_c + q)
    atomicAdd(rpc_cc + i, 1);
  const int e0 = nbr_off[i], e1 = nbr_off[i + 1];
  for (int r = roff[q]; r < roff[q + 1]; ++r) {
    if (uf_find(lpar_f, r) != r || uf_find(gpar_f, (int)(base_f + r)) != base_f + r) continue;
    const int e = find_sorted(nbr_idx, e0, e1, rj[r]);
    if (e >= 0) atomicAdd(rpf_cc + e, 1);
  }
}

cudaError_t launch_g2l(rpd_ctx* c, const int32_t* local_ids, int64_t T_local, int64_t T_all) {
  cudaError_t e = c->eu_g2l.ensure(sizeof(int32_t) * (T_all > 0 ? T_all : 1));
  if (e) return e;
  if ((e = cudaMemsetAsync(c->eu_g2l.p, 0xff, sizeof(int32_t) * (T_all > 0 ? T_all : 1),
                           c->stream)))
    return e;
  if (T_local > 0 && local_ids) {
    k_g2l<<<nblk(T_local, 256), 256, 0, c->stream>>>(T_local, local_ids, c->eu_g2l.as<int32_t>());
    ++c->launches;
  }
  return cudaGetLastError();
}

// step 1 + 2: local union-find (cc_par: pieces, then radical facets) and the boundary records
// into cc_bnd (counts at n_rec[0..1] on the device)
cudaError_t launch_cc_shard(rpd_ctx* c, const PieceSet& ps, long long base_c, long long base_f,
                            int* n_rec) {
  const int64_t T = ps.n_tets, np = ps.n_pieces, nr = ps.n_rpf;
  cudaError_t e;
  if ((e = c->cc_par.ensure(sizeof(int) * (np + nr + 1)))) return e;
  int* par_c = c->cc_par.as<int>();
  int* par_f = par_c + np;
  // record buffers: at most 4 per piece / per radical facet
  const size_t nc = 4 * (size_t)np + 1, nf = 4 * (size_t)nr + 1;
  if ((e = c->cc_bnd.ensure(nc * 12 + nf * 16 + 64))) return e;
  unsigned long long* key_c = c->cc_bnd.as<unsigned long long>();
  unsigned long long* key_f = key_c + nc;
  int32_t* lab_c = reinterpret_cast<int32_t*>(key_f + nf);
  int32_t* j_f = lab_c + nc;
  int32_t* lab_f = j_f + nf;
  if ((e = cudaMemsetAsync(n_rec, 0, sizeof(int) * 2, c->stream))) return e;
  if (np > 0) {
    k_cc_init_range<<<nblk(np, 256), 256, 0, c->stream>>>(np, par_c);
    ++c->launches;
  }
  if (nr > 0) {
    k_cc_init_range<<<nblk(nr, 256), 256, 0, c->stream>>>(nr, par_f);
    ++c->launches;
  }
  if (T > 0 && np > 0) {
    k_cc_link_sh<<<nblk(T, 128), 128, 0, c->stream>>>(
        T, c->eu_adj.as<int>(), c->eu_g2l.as<int32_t>(), ps.off.as<int32_t>(),
        ps.sphere.as<int32_t>(), ps.sfm.as<uint8_t>(), ps.rpf_off.as<int32_t>(),
        ps.rpf_j.as<int32_t>(), ps.rfm.as<uint8_t>(), par_c, par_f);
    k_cc_bnd<<<nblk(T, 128), 128, 0, c->stream>>>(
        T, c->eu_ids.as<int32_t>(), c->eu_adj.as<int>(), c->eu_g2l.as<int32_t>(),
        ps.off.as<int32_t>(), ps.sphere.as<int32_t>(), ps.sfm.as<uint8_t>(),
        ps.rpf_off.as<int32_t>(), ps.rpf_j.as<int32_t>(), ps.rfm.as<uint8_t>(), par_c, par_f,
        base_c, base_f, key_c, lab_c, key_f, j_f, lab_f, n_rec);
    c->launches += 2;
  }
  return cudaGetLastError();
}

// step 3 + 4 on this rank: the gathered records of all ranks -> this rank's counts [N + E]
cudaError_t launch_cc_merge(rpd_ctx* c, const PieceSet& ps, const unsigned long long* key_c,
                            const int32_t* lab_c, int64_t n_c, const unsigned long long* key_f,
                            const int32_t* j_f, const int32_t* lab_f, int64_t n_f,
                            int64_t tot_c, int64_t tot_f, long long base_c, long long base_f,
                            int32_t* counts) {
  const int64_t N = c->st.N, E = c->st.E, np = ps.n_pieces;
  cudaError_t e;
  const size_t nc1 = n_c > 0 ? n_c : 1, nf1 = n_f > 0 ? n_f : 1;
  if ((e = c->cc_gpar.ensure(sizeof(int) * (tot_c + tot_f + 2)))) return e;
  if ((e = c->cc_sort.ensure(nc1 * 12 + nf1 * 16 + 64))) return e;
  int* gpar_c = c->cc_gpar.as<int>();
  int* gpar_f = gpar_c + tot_c + 1;
  unsigned long long* sk_c = c->cc_sort.as<unsigned long long>();
  unsigned long long* sk_f = sk_c + nc1;
  int32_t* sl_c = reinterpret_cast<int32_t*>(sk_f + nf1);
  int32_t* si_f = sl_c + nc1;
  int32_t* ix_f = si_f + nf1;  // record indices (values of the RPF sort)
  const int g = 8 * c->sms;
  k_cc_init_range<<<g, 256, 0, c->stream>>>(tot_c, gpar_c);
  k_cc_init_range<<<g, 256, 0, c->stream>>>(tot_f, gpar_f);
  c->launches += 2;
  size_t b1 = 0, b2 = 0;
  if (n_c > 0 &&
      (e = cub::DeviceRadixSort::SortPairs(nullptr, b1, key_c, sk_c, lab_c, sl_c, (int)n_c, 0, 64,
                                           c->stream)))
    return e;
  if (n_f > 0 &&
      (e = cub::DeviceRadixSort::SortPairs(nullptr, b2, key_f, sk_f, ix_f, si_f, (int)n_f, 0, 64,
                                           c->stream)))
    return e;
  if ((e = c->mm_tmp.ensure((b1 > b2 ? b1 : b2) + 16))) return e;
  if (n_c > 0) {
    size_t bt = c->mm_tmp.cap;
    if ((e = cub::DeviceRadixSort::SortPairs(c->mm_tmp.p, bt, key_c, sk_c, lab_c, sl_c, (int)n_c,
                                             0, 64, c->stream)))
      return e;
    k_cc_join_c<<<g, 256, 0, c->stream>>>(n_c, sk_c, sl_c, gpar_c);
    c->launches += 2;
  }
  if (n_f > 0) {
    k_cc_init_range<<<g, 256, 0, c->stream>>>(n_f, ix_f);  // (identity indices)
    size_t bt = c->mm_tmp.cap;
    if ((e = cub::DeviceRadixSort::SortPairs(c->mm_tmp.p, bt, key_f, sk_f, ix_f, si_f, (int)n_f,
                                             0, 64, c->stream)))
      return e;
    k_cc_join_f<<<g, 256, 0, c->stream>>>(n_f, sk_f, si_f, j_f, lab_f, gpar_f);
    c->launches += 3;
  }
  if ((e = cudaMemsetAsync(counts, 0, sizeof(int32_t) * (N + E), c->stream))) return e;
  if (np > 0) {
    int* lpar_c = c->cc_par.as<int>();
    k_cc_count_sh<<<nblk(np, 256), 256, 0, c->stream>>>(
        np, ps.sphere.as<int32_t>(), ps.rpf_off.as<int32_t>(), ps.rpf_j.as<int32_t>(),
        c->st.nbr_off.as<int32_t>(), c->st.nbr_idx.as<int32_t>(), lpar_c, lpar_c + np, gpar_c,
        gpar_f, base_c, base_f, counts, counts + N);
    ++c->launches;
  }
  return cudaGetLastError();
}

// ---------------------------------------------------------------- dual medial mesh (NEXT-2)
//
// RPC -> vertex, RPF(m_i, m_j) -> edge e_ij, RPE(m_i, m_j, m_k) -> triangle
// f_ijk.  One thread per piece emits an edge key per radical facet and a triangle key per pair
// of its radical facets that share an edge (rpf_adj); keys are sorted and deduplicated with
// CUB's radix sort / unique (library primitives) and decoded.

__global__ void k_mm_count(int64_t n_pieces, const int32_t* __restrict__ roff,
                           const unsigned long long* __restrict__ radj, int32_t* __restrict__ cnt) {
  const int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (q >= n_pieces) return;
  int n = 0;
  for (int r = roff[q]; r < roff[q + 1]; ++r) {
    const int a = r - roff[q];
    n += a < 63 ? __popcll(radj[r] >> (a + 1)) : 0;
  }
  cnt[q] = n;
}

__global__ void k_mm_emit(int64_t n_pieces, const int32_t* __restrict__ psph,
                          const int32_t* __restrict__ roff, const int32_t* __restrict__ rj,
                          const unsigned long long* __restrict__ radj,
                          const int32_t* __restrict__ foff, unsigned long long* __restrict__ ekeys,
                          unsigned long long* __restrict__ fkeys) {
  const int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (q >= n_pieces) return;
  const long long i = psph[q];
  const int r0 = roff[q], r1 = roff[q + 1];
  int m = foff[q];
  for (int r = r0; r < r1; ++r) {
    const long long j = rj[r];
    ekeys[r] = ((unsigned long long)min(i, j) << 32) | (unsigned long long)max(i, j);
    const int a = r - r0;
    unsigned long long bits = a < 63 ? radj[r] >> (a + 1) : 0ull;
    while (bits) {
      const int b = a + __ffsll((long long)bits);  // (a + 1) + bit index
      bits &= bits - 1ull;
      long long x = i, y = j, z = rj[r0 + b];
      sort3(x, y, z);
      fkeys[m++] = ((unsigned long long)x << 42) | ((unsigned long long)y << 21) |
                   (unsigned long long)z;
    }
  }
}

__global__ void k_mm_decode(int64_t ne, const unsigned long long* __restrict__ ek, int64_t nf,
                            const unsigned long long* __restrict__ fk, int32_t* __restrict__ out) {
  const int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (x < ne) {
    out[2 * x] = (int32_t)(ek[x] >> 32);
    out[2 * x + 1] = (int32_t)(ek[x] & 0xffffffffull);
  } else if (x < ne + nf) {
    const int64_t f = x - ne;
    const unsigned long long k = fk[f];
    int32_t* o = out + 2 * ne + 3 * f;
    o[0] = (int32_t)(k >> 42);
    o[1] = (int32_t)((k >> 21) & 0x1fffffull);
    o[2] = (int32_t)(k & 0x1fffffull);
  }
}

// sorted unique keys: in -> out (count to *n_out, device), temp in c->mm_tmp
static cudaError_t sort_unique(rpd_ctx* c, unsigned long long* keys, unsigned long long* tmp_keys,
                               int64_t n, int* n_out) {
  size_t b1 = 0, b2 = 0;
  cudaError_t e = cub::DeviceRadixSort::SortKeys(nullptr, b1, keys, tmp_keys, (int)n, 0, 64,
                                                 c->stream);
  if (e) return e;
  e = cub::DeviceSelect::Unique(nullptr, b2, tmp_keys, keys, n_out, (int)n, c->stream);
  if (e) return e;
  if ((e = c->mm_tmp.ensure(b1 > b2 ? b1 : b2))) return e;
  size_t bt = c->mm_tmp.cap;
  if ((e = cub::DeviceRadixSort::SortKeys(c->mm_tmp.p, bt, keys, tmp_keys, (int)n, 0, 64,
                                          c->stream)))
    return e;
  bt = c->mm_tmp.cap;
  e = cub::DeviceSelect::Unique(c->mm_tmp.p, bt, tmp_keys, keys, n_out, (int)n, c->stream);
  c->launches += 2;
  return e;
}

cudaError_t launch_medial_mesh(rpd_ctx* c, const PieceSet& ps, int64_t* n_edges,
                               int64_t* n_faces) {
  const int64_t np = ps.n_pieces, nr = ps.n_rpf;
  cudaError_t e;
  // face counts per piece -> offsets (total read back)
  if ((e = c->cc_par.ensure(sizeof(int32_t) * (2 * np + 2)))) return e;
  int32_t* cnt = c->cc_par.as<int32_t>();
  int32_t* foff = cnt + np + 1;
  if (np > 0) {
    k_mm_count<<<nblk(np, 256), 256, 0, c->stream>>>(np, ps.rpf_off.as<int32_t>(),
                                                     ps.radj.as<unsigned long long>(), cnt);
    ++c->launches;
  }
  if ((e = launch_scan_i32(c, cnt, foff, np))) return e;
  int32_t nf_all = 0;
  if ((e = cudaMemcpyAsync(&nf_all, foff + np, sizeof(int32_t), cudaMemcpyDeviceToHost,
                           c->stream)))
    return e;
  if ((e = cudaStreamSynchronize(c->stream))) return e;
  const int64_t tot = nr + nf_all;
  if ((e = c->mm_keys.ensure(sizeof(unsigned long long) * 2 * (tot > 0 ? tot : 1) + 64)))
    return e;
  unsigned long long* ek = c->mm_keys.as<unsigned long long>();
  unsigned long long* fk = ek + nr;
  unsigned long long* tk = ek + tot;  // sort output scratch
  int* n_sel = reinterpret_cast<int*>(tk + (tot > 0 ? tot : 1));
  if (np > 0) {
    k_mm_emit<<<nblk(np, 256), 256, 0, c->stream>>>(
        np, ps.sphere.as<int32_t>(), ps.rpf_off.as<int32_t>(), ps.rpf_j.as<int32_t>(),
        ps.radj.as<unsigned long long>(), foff, ek, fk);
    ++c->launches;
  }
  int hs[2] = {0, 0};
  if (nr > 0) {
    if ((e = sort_unique(c, ek, tk, nr, n_sel))) return e;
    if ((e = cudaMemcpyAsync(hs, n_sel, sizeof(int), cudaMemcpyDeviceToHost, c->stream)))
      return e;
  }
  if (nf_all > 0) {
    if ((e = sort_unique(c, fk, tk, nf_all, n_sel + 1))) return e;
    if ((e = cudaMemcpyAsync(hs + 1, n_sel + 1, sizeof(int), cudaMemcpyDeviceToHost, c->stream)))
      return e;
  }
  if ((e = cudaStreamSynchronize(c->stream))) return e;
  const int64_t ne = hs[0], nf = hs[1];
  if ((e = c->mm_out.ensure(sizeof(int32_t) * (2 * ne + 3 * nf + 1)))) return e;
  if (ne + nf > 0) {
    k_mm_decode<<<nblk(ne + nf, 256), 256, 0, c->stream>>>(ne, ek, nf, fk,
                                                           c->mm_out.as<int32_t>());
    ++c->launches;
  }
  *n_edges = ne;
  *n_faces = nf;
  return cudaGetLastError();
}

// ---------------------------------------------------------------- restricted power edges
//
// RPE(m_i, m_j, m_k) seen from m_i ("we are expecting each restricted element
// (i.e., RPC, RPF, RPE) to have CC=1 and Euler=1", 497, 506): in every piece of m_i the edge
// on the radical planes h_ij and h_ik (j < k).  The clip records, per radical facet x, which
// other radical facets y share an edge with it (rpf_adj) and on which tet faces those edges
// end (rep: 16 bits per face holding the ranks + 1 of at most two y).  Here one thread per
// tet expands them into the per-piece RPE list (ascending (j, k)) with the edge's fractional
// Euler characteristic V - E = pay(end 1) + pay(end 2) - pay(edge): the edge lies inside the
// tet (payload 1), an end on tet face f carries f's payload, an end inside the tet 1.  Per-
// (i, j, k) sums by CUB sort + reduce-by-key (library primitives); CC numbers by union-find
// over the per-piece edges, two joined across a shared tet face when both end on it (a line
// meets the face's plane once, so the two ends are the same point).

__device__ __forceinline__ unsigned rep_faces(unsigned long long rep, int b) {
  unsigned F = 0u;
#pragma unroll
  for (int f = 0; f < 4; ++f) {
    const unsigned w = (unsigned)(rep >> (16 * f)) & 0xffffu;
    if ((w & 0xffu) == (unsigned)(b + 1) || ((w >> 8) & 0xffu) == (unsigned)(b + 1)) F |= 1u << f;
  }
  return F;
}

// one thread per tet: the RPE list of each of its pieces (count at rpe_off, emitted in
// (rank a, rank b) order = ascending (j, k)); keys (i << 42 | j << 21 | k) and values for the
// per-(i, j, k) sums
__global__ void k_rpe_emit(int64_t T, const int32_t* __restrict__ poff,
                           const int32_t* __restrict__ psph, const int32_t* __restrict__ roff,
                           const int32_t* __restrict__ rj,
                           const unsigned long long* __restrict__ radj,
                           const unsigned long long* __restrict__ rep,
                           const int32_t* __restrict__ eoff, const uint4* __restrict__ rec,
                           const long long* __restrict__ Lt,
                           int32_t* __restrict__ ej, int32_t* __restrict__ ek,
                           long long* __restrict__ ee, uint8_t* __restrict__ efm,
                           unsigned long long* __restrict__ keys, long long* __restrict__ vals) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= T) return;
  const uint4 rc = rec[t];
  const long long L = Lt[t];
  long long h2[4];  // twice the payload of the tet's 4 faces minus 2: 2 / count - 2 (0 or -1)
#pragma unroll
  for (int f = 0; f < 4; ++f) {
    const int m = 10 + f;
    const unsigned w = m < 12 ? rc.z : rc.w;
    h2[f] = 2 / (long long)((w >> (8 * (m & 3))) & 0xffu) - 2;
  }
  for (int q = poff[t]; q < poff[t + 1]; ++q) {
    const long long i = psph[q];
    const int r0 = roff[q], r1 = roff[q + 1];
    int m = eoff[q];
    for (int r = r0; r < r1; ++r) {
      const int a = r - r0;
      unsigned long long bits = a < 63 ? radj[r] >> (a + 1) : 0ull;
      while (bits) {
        const int b = a + __ffsll((long long)bits);
        bits &= bits - 1ull;
        const unsigned F = rep_faces(rep[r], b);
        long long v2 = 2;  // twice V - E: 2 (1 - |F|) + sum of twice the faces' payloads
        for (int f = 0; f < 4; ++f)
          if ((F >> f) & 1u) v2 += h2[f];
        const long long j = rj[r], k = rj[r0 + b];
        ej[m] = (int32_t)j;
        ek[m] = (int32_t)k;
        // numerator over L_t: (v2 / 2) L_t (v2 odd only with a face of count 2: L_t even)
        ee[m] = (L & 1) ? (v2 / 2) * L : v2 * (L / 2);
        efm[m] = (uint8_t)F;
        keys[m] = ((unsigned long long)i << 42) | ((unsigned long long)j << 21) |
                  (unsigned long long)k;
        vals[m] = v2;
        ++m;
      }
    }
  }
}

// index of RPE (j, k) in a piece's list [lo, hi), or -1 (lists are short)
__device__ __forceinline__ int rpe_find(const int32_t* ej, const int32_t* ek, int lo, int hi,
                                        int j, int k) {
  for (int m = lo; m < hi; ++m)
    if (ej[m] == j && ek[m] == k) return m;
  return -1;
}

__global__ void k_rpe_link(int64_t T, const int* __restrict__ adj, const int32_t* __restrict__ poff,
                           const int32_t* __restrict__ psph, const int32_t* __restrict__ eoff,
                           const int32_t* __restrict__ ej, const int32_t* __restrict__ ek,
                           const uint8_t* __restrict__ efm, int* __restrict__ par) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= T) return;
  const int p0 = poff[t], p1 = poff[t + 1];
  for (int f = 0; f < 4; ++f) {
    const int nb = adj[4 * t + f];
    if (nb < 0 || (nb >> 2) < t) continue;  // each shared face once
    const int t2 = nb >> 2, f2 = nb & 3;
    const int q0 = poff[t2], q1 = poff[t2 + 1];
    for (int q = p0; q < p1; ++q) {
      const int q2 = find_sorted(psph, q0, q1, psph[q]);
      if (q2 < 0) continue;
      for (int m = eoff[q]; m < eoff[q + 1]; ++m) {
        if (!((efm[m] >> f) & 1)) continue;
        const int m2 = rpe_find(ej, ek, eoff[q2], eoff[q2 + 1], ej[m], ek[m]);
        if (m2 >= 0 && ((efm[m2] >> f2) & 1)) uf_union(par, m, m2);
      }
    }
  }
}

// a root edge counts one component of its (i, j, k): binary search of its key among the
// sorted unique keys
__global__ void k_rpe_cc(int64_t n, int* __restrict__ par, const unsigned long long* __restrict__ keys,
                         const unsigned long long* __restrict__ ukeys, int64_t nu,
                         int* __restrict__ cc) {
  const int64_t m = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (m >= n || uf_find(par, (int)m) != m) return;
  const unsigned long long key = keys[m];
  int64_t lo = 0, hi = nu;
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (ukeys[mid] < key) lo = mid + 1;
    else hi = mid;
  }
  if (lo < nu && ukeys[lo] == key) atomicAdd(cc + lo, 1);
}

__global__ void k_rpe_decode(int64_t nu, const unsigned long long* __restrict__ uk,
                             int32_t* __restrict__ tri) {
  const int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (x >= nu) return;
  const unsigned long long k = uk[x];
  tri[3 * x] = (int32_t)(k >> 42);
  tri[3 * x + 1] = (int32_t)((k >> 21) & 0x1fffffull);
  tri[3 * x + 2] = (int32_t)(k & 0x1fffffull);
}

// the per-piece RPE lists, their per-(i, j, k) sums and (with_cc) CC numbers.  Layout in
// c->rpe_buf: eoff [np+1] | ej, ek [n] | efm [n] | ee [n] | keys, vals, sorted keys / vals
// [n] | unique keys, sums [n] | cc [n] | tri [3n] | union-find parents [n]
cudaError_t launch_rpe(rpd_ctx* c, const PieceSet& ps, bool with_cc, int64_t* n_rpe,
                       int64_t* n_tri) {
  const int64_t np = ps.n_pieces, nr = ps.n_rpf, T = ps.n_tets;
  cudaError_t e;
  if ((e = c->cc_par.ensure(sizeof(int32_t) * (2 * np + 2)))) return e;
  int32_t* cnt = c->cc_par.as<int32_t>();
  if ((e = c->rpe_off.ensure(sizeof(int32_t) * (np + 1)))) return e;
  int32_t* eoff = c->rpe_off.as<int32_t>();
  if (np > 0) {
    k_mm_count<<<nblk(np, 256), 256, 0, c->stream>>>(np, ps.rpf_off.as<int32_t>(),
                                                     ps.radj.as<unsigned long long>(), cnt);
    ++c->launches;
  }
  if ((e = launch_scan_i32(c, cnt, eoff, np))) return e;
  int32_t nn = 0;
  if ((e = cudaMemcpyAsync(&nn, eoff + np, sizeof(int32_t), cudaMemcpyDeviceToHost, c->stream)))
    return e;
  if ((e = cudaStreamSynchronize(c->stream))) return e;
  const int64_t n = nn, n1 = n > 0 ? n : 1;
  // 8-byte arrays first, then 4-byte, then bytes
  const size_t bytes = 8 * (6 * n1) + 4 * (2 * n1 + n1 + 3 * n1 + n1) + n1 + 64;
  if ((e = c->rpe_buf.ensure(bytes))) return e;
  unsigned long long* keys = c->rpe_buf.as<unsigned long long>();
  long long* vals = reinterpret_cast<long long*>(keys + n1);
  unsigned long long* skeys = keys + 2 * n1;
  long long* svals = reinterpret_cast<long long*>(keys + 3 * n1);
  unsigned long long* ukeys = keys + 4 * n1;
  long long* usums = reinterpret_cast<long long*>(keys + 5 * n1);
  int32_t* ej = reinterpret_cast<int32_t*>(keys + 6 * n1);
  int32_t* ek = ej + n1;
  int32_t* cc = ek + n1;
  int32_t* tri = cc + n1;
  int32_t* par = tri + 3 * n1;
  uint8_t* efm = reinterpret_cast<uint8_t*>(par + n1);
  if ((e = c->rpe_ee.ensure(sizeof(long long) * n1))) return e;
  long long* ee = c->rpe_ee.as<long long>();
  if (T > 0 && np > 0) {
    k_rpe_emit<<<nblk(T, 128), 128, 0, c->stream>>>(
        T, ps.off.as<int32_t>(), ps.sphere.as<int32_t>(), ps.rpf_off.as<int32_t>(),
        ps.rpf_j.as<int32_t>(), ps.radj.as<unsigned long long>(),
        ps.rep.as<unsigned long long>(), eoff, c->eu_rec.as<uint4>(), c->eu_Lt.as<long long>(),
        ej, ek, ee, efm, keys, vals);
    ++c->launches;
  }
  int64_t nu = 0;
  if (n > 0) {
    // per-(i, j, k) sums: sort by key, reduce by key (CUB)
    size_t b1 = 0, b2 = 0;
    int* d_nu = par;  // (scratch: parents are initialised below)
    if ((e = cub::DeviceRadixSort::SortPairs(nullptr, b1, keys, skeys, vals, svals, (int)n, 0,
                                             63, c->stream)))
      return e;
    if ((e = cub::DeviceReduce::ReduceByKey(nullptr, b2, skeys, ukeys, svals, usums, d_nu,
                                            cuda::std::plus<long long>(), (int)n, c->stream)))
      return e;
    if ((e = c->mm_tmp.ensure(b1 > b2 ? b1 : b2))) return e;
    size_t bt = c->mm_tmp.cap;
    if ((e = cub::DeviceRadixSort::SortPairs(c->mm_tmp.p, bt, keys, skeys, vals, svals, (int)n,
                                             0, 63, c->stream)))
      return e;
    bt = c->mm_tmp.cap;
    if ((e = cub::DeviceReduce::ReduceByKey(c->mm_tmp.p, bt, skeys, ukeys, svals, usums, d_nu,
                                            cuda::std::plus<long long>(), (int)n, c->stream)))
      return e;
    c->launches += 2;
    int hnu = 0;
    if ((e = cudaMemcpyAsync(&hnu, d_nu, sizeof(int), cudaMemcpyDeviceToHost, c->stream)))
      return e;
    if ((e = cudaStreamSynchronize(c->stream))) return e;
    nu = hnu;
    if ((e = cudaMemsetAsync(cc, 0, sizeof(int32_t) * n1, c->stream))) return e;
    k_rpe_decode<<<nblk(nu, 256), 256, 0, c->stream>>>(nu, ukeys, tri);
    ++c->launches;
    if (with_cc) {
      k_cc_init<<<nblk(n, 256), 256, 0, c->stream>>>(n, par);
      k_rpe_link<<<nblk(T, 128), 128, 0, c->stream>>>(
          T, c->eu_adj.as<int>(), ps.off.as<int32_t>(), ps.sphere.as<int32_t>(), eoff, ej, ek,
          efm, par);
      k_rpe_cc<<<nblk(n, 256), 256, 0, c->stream>>>(n, par, keys, ukeys, nu, cc);
      c->launches += 3;
    }
  }
  c->rpe_n = n;
  c->rpe_nu = nu;
  *n_rpe = n;
  *n_tri = nu;
  return cudaGetLastError();
}

// ---------------------------------------------------------------- RPEs of a sharded job
//
// As the CC numbers of RPCs / RPFs (rpd_cc_shard / rpd_cc_merge): the rank's RPE parts joined
// across its interior faces (k_rpe_link through the global -> local tet map), records of its
// shard-boundary faces, a global union-find over the gathered records, and per rank the
// components whose smallest global id it holds, counted per (i, j, k); the ranks' per-key
// lists (Euler numerators, component counts) are summed by key (rpd_reduce_by_key).

__global__ void k_rpe_link_sh(int64_t T, const int* __restrict__ adj,
                              const int32_t* __restrict__ g2l, const int32_t* __restrict__ poff,
                              const int32_t* __restrict__ psph, const int32_t* __restrict__ eoff,
                              const int32_t* __restrict__ ej, const int32_t* __restrict__ ek,
                              const uint8_t* __restrict__ efm, int* __restrict__ par) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= T) return;
  const int p0 = poff[t], p1 = poff[t + 1];
  for (int f = 0; f < 4; ++f) {
    const int nb = adj[4 * t + f];
    if (nb < 0) continue;
    const int t2 = g2l[nb >> 2], f2 = nb & 3;
    if (t2 < 0 || t2 < t) continue;  // remote, or this face from the other side
    const int q0 = poff[t2], q1 = poff[t2 + 1];
    for (int q = p0; q < p1; ++q) {
      const int q2 = find_sorted(psph, q0, q1, psph[q]);
      if (q2 < 0) continue;
      for (int m = eoff[q]; m < eoff[q + 1]; ++m) {
        if (!((efm[m] >> f) & 1)) continue;
        const int m2 = rpe_find(ej, ek, eoff[q2], eoff[q2 + 1], ej[m], ek[m]);
        if (m2 >= 0 && ((efm[m2] >> f2) & 1)) uf_union(par, m, m2);
      }
    }
  }
}

// records of the RPE parts with an endpoint on a shard-boundary face: key (f << 21 | i), the
// pair (j << 21 | k), label = global id of the local root
__global__ void k_rpe_bnd(int64_t T, const int32_t* __restrict__ local_ids,
                          const int* __restrict__ adj, const int32_t* __restrict__ g2l,
                          const int32_t* __restrict__ poff, const int32_t* __restrict__ psph,
                          const int32_t* __restrict__ eoff, const int32_t* __restrict__ ej,
                          const int32_t* __restrict__ ek, const uint8_t* __restrict__ efm,
                          int* __restrict__ par, long long base,
                          unsigned long long* __restrict__ key_b,
                          unsigned long long* __restrict__ jk_b, int32_t* __restrict__ lab_b,
                          int* __restrict__ n_rec) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= T) return;
  const int p0 = poff[t], p1 = poff[t + 1];
  const long long tg = local_ids[t];
  for (int f = 0; f < 4; ++f) {
    const int nb = adj[4 * t + f];
    if (nb < 0 || g2l[nb >> 2] >= 0) continue;
    const unsigned long long fid = (unsigned long long)min(4 * tg + f, (long long)nb);
    for (int q = p0; q < p1; ++q)
      for (int m = eoff[q]; m < eoff[q + 1]; ++m) {
        if (!((efm[m] >> f) & 1)) continue;
        const int s = atomicAdd(n_rec, 1);
        key_b[s] = (fid << 21) | (unsigned long long)psph[q];
        jk_b[s] = ((unsigned long long)ej[m] << 21) | (unsigned long long)ek[m];
        lab_b[s] = (int32_t)(base + uf_find(par, m));
      }
  }
}

// sorted boundary records (value = record index): equal key and pair -> join
__global__ void k_rpe_join(int64_t n, const unsigned long long* __restrict__ key,
                           const int32_t* __restrict__ idx, const unsigned long long* __restrict__ jk,
                           const int32_t* __restrict__ lab, int* __restrict__ par) {
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < n;
       p += (int64_t)gridDim.x * blockDim.x) {
    const int a = idx[p];
    for (int64_t q = p + 1; q < n && key[q] == key[p]; ++q) {
      const int b = idx[q];
      if (jk[a] == jk[b]) uf_union(par, lab[a], lab[b]);
    }
  }
}

// this rank's RPE parts that are local and global roots: (triple key, 1) pairs (0 elsewhere)
__global__ void k_rpe_roots(int64_t n, const unsigned long long* __restrict__ keys,
                            int* __restrict__ lpar, int* __restrict__ gpar, long long base,
                            unsigned long long* __restrict__ out_k, long long* __restrict__ out_v) {
  const int64_t m = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (m >= n) return;
  const bool root = uf_find(lpar, (int)m) == m && uf_find(gpar, (int)(base + m)) == base + m;
  out_k[m] = keys[m];
  out_v[m] = root ? 1 : 0;
}

// sum of vals per key, keys ascending (CUB radix sort + reduce-by-key); *n_out on the device
cudaError_t launch_reduce_by_key(rpd_ctx* c, const unsigned long long* keys, const long long* vals,
                                 int64_t n, unsigned long long* out_k, long long* out_v,
                                 int* n_out) {
  cudaError_t e;
  if (n <= 0) return cudaMemsetAsync(n_out, 0, sizeof(int), c->stream);
  if ((e = c->rk_buf.ensure(16 * (size_t)n + 64))) return e;
  unsigned long long* sk = c->rk_buf.as<unsigned long long>();
  long long* sv = reinterpret_cast<long long*>(sk + n);
  size_t b1 = 0, b2 = 0;
  if ((e = cub::DeviceRadixSort::SortPairs(nullptr, b1, keys, sk, vals, sv, (int)n, 0, 64,
                                           c->stream)))
    return e;
  if ((e = cub::DeviceReduce::ReduceByKey(nullptr, b2, sk, out_k, sv, out_v, n_out,
                                          cuda::std::plus<long long>(), (int)n, c->stream)))
    return e;
  if ((e = c->mm_tmp.ensure((b1 > b2 ? b1 : b2) + 16))) return e;
  size_t bt = c->mm_tmp.cap;
  if ((e = cub::DeviceRadixSort::SortPairs(c->mm_tmp.p, bt, keys, sk, vals, sv, (int)n, 0, 64,
                                           c->stream)))
    return e;
  bt = c->mm_tmp.cap;
  if ((e = cub::DeviceReduce::ReduceByKey(c->mm_tmp.p, bt, sk, out_k, sv, out_v, n_out,
                                          cuda::std::plus<long long>(), (int)n, c->stream)))
    return e;
  c->launches += 2;
  return cudaGetLastError();
}

// rpd_rpe_shard: launch_rpe (per-piece lists, per-key sums) + local union + boundary records
// into c->rpe_bnd (count at n_rec on the device)
cudaError_t launch_rpe_shard(rpd_ctx* c, const PieceSet& ps, long long base, int* n_rec,
                             int64_t* n_rpe, int64_t* n_tri) {
  cudaError_t e = launch_rpe(c, ps, false, n_rpe, n_tri);
  if (e) return e;
  const int64_t n = *n_rpe, n1 = n > 0 ? n : 1, T = ps.n_tets, np = ps.n_pieces;
  unsigned long long* keys = c->rpe_buf.as<unsigned long long>();
  int32_t* ej = reinterpret_cast<int32_t*>(keys + 6 * n1);
  int32_t* ek = ej + n1;
  int32_t* par = ek + n1 + n1 + 3 * n1;  // (layout of launch_rpe)
  uint8_t* efm = reinterpret_cast<uint8_t*>(par + n1);
  const int32_t* eoff = c->rpe_off.as<int32_t>();
  const size_t nb = 4 * (size_t)n1;  // at most 2 endpoint faces per part, each on <= 2 faces
  if ((e = c->rpe_bnd.ensure(nb * 20 + 64))) return e;
  unsigned long long* key_b = c->rpe_bnd.as<unsigned long long>();
  unsigned long long* jk_b = key_b + nb;
  int32_t* lab_b = reinterpret_cast<int32_t*>(jk_b + nb);
  if ((e = cudaMemsetAsync(n_rec, 0, sizeof(int), c->stream))) return e;
  if (n > 0) {
    k_cc_init<<<nblk(n, 256), 256, 0, c->stream>>>(n, par);
    ++c->launches;
  }
  if (T > 0 && np > 0 && n > 0) {
    k_rpe_link_sh<<<nblk(T, 128), 128, 0, c->stream>>>(
        T, c->eu_adj.as<int>(), c->eu_g2l.as<int32_t>(), ps.off.as<int32_t>(),
        ps.sphere.as<int32_t>(), eoff, ej, ek, efm, par);
    k_rpe_bnd<<<nblk(T, 128), 128, 0, c->stream>>>(
        T, c->eu_ids.as<int32_t>(), c->eu_adj.as<int>(), c->eu_g2l.as<int32_t>(),
        ps.off.as<int32_t>(), ps.sphere.as<int32_t>(), eoff, ej, ek, efm, par, base, key_b,
        jk_b, lab_b, n_rec);
    c->launches += 2;
  }
  return cudaGetLastError();
}

// rpd_rpe_merge: the gathered records -> global union -> this rank's (key, count) of its
// global-root parts, reduced by key into c->rpe_cnt (keys [.], counts [.], *n_out on device)
cudaError_t launch_rpe_merge(rpd_ctx* c, const unsigned long long* key_b,
                             const unsigned long long* jk_b, const int32_t* lab_b, int64_t n_b,
                             int64_t total, long long base, int* n_out) {
  const int64_t n = c->rpe_n, n1 = n > 0 ? n : 1, nb1 = n_b > 0 ? n_b : 1;
  cudaError_t e;
  if ((e = c->cc_gpar.ensure(sizeof(int) * (total + 1)))) return e;
  if ((e = c->cc_sort.ensure(nb1 * 16 + 64))) return e;
  int* gpar = c->cc_gpar.as<int>();
  unsigned long long* sk = c->cc_sort.as<unsigned long long>();
  int32_t* ix = reinterpret_cast<int32_t*>(sk + nb1);
  int32_t* six = ix + nb1;
  const int g = 8 * c->sms;
  k_cc_init_range<<<g, 256, 0, c->stream>>>(total, gpar);
  ++c->launches;
  if (n_b > 0) {
    k_cc_init_range<<<g, 256, 0, c->stream>>>(n_b, ix);
    size_t b1 = 0;
    if ((e = cub::DeviceRadixSort::SortPairs(nullptr, b1, key_b, sk, ix, six, (int)n_b, 0, 64,
                                             c->stream)))
      return e;
    if ((e = c->mm_tmp.ensure(b1 + 16))) return e;
    size_t bt = c->mm_tmp.cap;
    if ((e = cub::DeviceRadixSort::SortPairs(c->mm_tmp.p, bt, key_b, sk, ix, six, (int)n_b, 0,
                                             64, c->stream)))
      return e;
    k_rpe_join<<<g, 256, 0, c->stream>>>(n_b, sk, six, jk_b, lab_b, gpar);
    c->launches += 3;
  }
  // this rank's root parts per triple key
  unsigned long long* keys = c->rpe_buf.as<unsigned long long>();
  int32_t* ej = reinterpret_cast<int32_t*>(keys + 6 * n1);
  int32_t* lpar = ej + n1 + n1 + n1 + 3 * n1;
  if ((e = c->rpe_cnt.ensure(32 * (size_t)n1 + 64))) return e;
  unsigned long long* rk = c->rpe_cnt.as<unsigned long long>();
  long long* rv = reinterpret_cast<long long*>(rk + n1);
  unsigned long long* ok = rk + 2 * n1;
  long long* ov = reinterpret_cast<long long*>(rk + 3 * n1);
  if (n > 0) {
    k_rpe_roots<<<nblk(n, 256), 256, 0, c->stream>>>(n, keys, lpar, gpar, base, rk, rv);
    ++c->launches;
  }
  return launch_reduce_by_key(c, rk, rv, n, ok, ov, n_out);
}

}  // namespace rpd
