// rpd_internal.cuh -- shared device/host internals of librpd (CUDA path only; the oracle
// under oracle/ shares nothing with this file).
//
// Units.  Inputs are real coordinates on the 2^-10 lattice; the stage kernel rescales them
// by 2^10 (exact) so every coordinate is an integer-valued double ("lattice units").  With
// |X| < 2^16 and r < 2^16 every power-distance difference at a vertex is an integer of
// magnitude < 2^35.4 and is computed EXACTLY in fp64 (all partial sums < 2^53).
//
// Planes.  For sphere i and neighbour j (CSR entry e):
//     h_ij(X) = PD_j(X) - PD_i(X) = n . X + d,   n = 2 (Theta_i - Theta_j),  d = W_j - W_i,
//     W = |Theta|^2 - R^2
// h_ij > 0  <=>  X is strictly power-closer to m_i than to m_j (Alg. 1, R1/R2).
//
// Clip frame.  A piece lives in the barycentric coordinates of its
// tet: tet face k is the 4-vector e_k, radical plane j is g_j = (h_ij(V0..V3)) (exact
// integers).  A vertex is the intersection of 3 planes and is stored as the homogeneous
// 4-vector K = cross(a_p, a_q, a_r) (a . K = det[a_p; a_q; a_r; a]) scaled so sum(K) > 0;
// then sign(h_s at v) = sign(g_s . K).  fp64 K carries an error bound; undecided signs go to
// an exact int128 evaluation with symbolic perturbation (inward, rank(radical j) = j,
// rank(face k) = N + k).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

typedef __int128 i128;

#define RPD_LATTICE 1024.0
#define RPD_MAXV 32     // vertices per piece held by the warp (lane = vertex)
#define RPD_MAXP 32     // planes per piece (4 tet faces + cutting radical planes)
#define RPD_INC_CAP 32  // incidences per piece in the per-pair slab

namespace rpd {

constexpr double U = 1.1102230246251565e-16;  // 2^-53

// ------------------------------------------------------------------ exact helpers (int128)

__host__ __device__ inline long long d2ll(double x) { return (long long)x; }

// det of 3x3 integer matrix rows a,b,c (int64 entries, result must fit int128)
__host__ __device__ inline i128 det3_i(const long long* a, const long long* b, const long long* c) {
  i128 m0 = (i128)b[1] * c[2] - (i128)b[2] * c[1];
  i128 m1 = (i128)b[0] * c[2] - (i128)b[2] * c[0];
  i128 m2 = (i128)b[0] * c[1] - (i128)b[1] * c[0];
  return (i128)a[0] * m0 - (i128)a[1] * m1 + (i128)a[2] * m2;
}

// det of a 4x4 integer matrix whose row 0 has entries in {-1,0,1} (a tet face e_k or the
// all-ones row): Laplace along row 0, 3x3 minors of rows 1..3 fit int128 (<= 2^110.6).
__host__ __device__ inline i128 det4_small_row0(const long long* r0, const long long* r1,
                                       const long long* r2, const long long* r3) {
  i128 acc = 0;
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    if (r0[c] == 0) continue;
    long long a[3], b[3], d[3];
    int n = 0;
#pragma unroll
    for (int k = 0; k < 4; ++k)
      if (k != c) {
        a[n] = r1[k];
        b[n] = r2[k];
        d[n] = r3[k];
        ++n;
      }
    i128 m = det3_i(a, b, d);
    if (c & 1) m = -m;
    acc += r0[c] > 0 ? m : -m;
  }
  return acc;
}

__host__ __device__ inline int sgn128(i128 x) { return x > 0 ? 1 : (x < 0 ? -1 : 0); }

// A plane of the current piece as exact integers.
struct XPlane {
  long long a[4];   // barycentric vector
  long long n[3];   // Cartesian normal (radical only)
  long long rank;   // SoS rank
  int radical;      // 1 radical, 0 tet face / all-ones row
};

__host__ __device__ inline bool is_small(const XPlane& p) { return !p.radical; }

// det[r0; r1; r2; r3] in the barycentric frame, exact sign.  At most three radical rows is
// evaluated directly; four radical rows use the Cartesian identity
//   det_bary = det(M) * det_cart[(n, d')],  M = [V0 V1 V2 V3; 1 1 1 1],  d' = a[0] = h(V0),
// where det(M) = -6 vol(t) < 0 for a positively oriented tet,
// whose entries are <= 2^17 (n) and <= 2^35.4 (d') so the Cartesian det fits int128.
__host__ __device__ inline int det4_sign(const XPlane* r[4]) {
  int small = -1;
#pragma unroll
  for (int k = 0; k < 4; ++k)
    if (small < 0 && is_small(*r[k])) small = k;
  if (small >= 0) {
    const long long* rows[4];
    int n = 1;
    rows[0] = r[small]->a;
    for (int k = 0; k < 4; ++k)
      if (k != small) rows[n++] = r[k]->a;
    // moving row `small` to the top is `small` adjacent swaps
    i128 d = det4_small_row0(rows[0], rows[1], rows[2], rows[3]);
    return (small & 1) ? -sgn128(d) : sgn128(d);
  }
  // all radical: Laplace along the d' column (column 3 of the Cartesian 4x4)
  i128 acc = 0;
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const long long* m[3];
    int n = 0;
    for (int q = 0; q < 4; ++q)
      if (q != k) m[n++] = r[q]->n;
    long long c3 = 0;
    {
      // 3x3 det of normals fits int64 (<= 6 * 2^51)
      c3 = m[0][0] * (m[1][1] * m[2][2] - m[1][2] * m[2][1]) -
           m[0][1] * (m[1][0] * m[2][2] - m[1][2] * m[2][0]) +
           m[0][2] * (m[1][0] * m[2][1] - m[1][1] * m[2][0]);
    }
    // cofactor sign of entry (k, 3): (-1)^(k+3)
    i128 term = (i128)r[k]->a[0] * c3;
    acc += ((k + 3) & 1) ? -term : term;
  }
  return -sgn128(acc);  // det(M) < 0
}

// Exact SoS sign of plane s at the vertex (p, q, r):  sign(D4(eps)) * sign(D3).
// zero_hit is set when D4 == 0 exactly.
static __host__ __device__ __noinline__ int sos_sign_exact(const XPlane& p, const XPlane& q, const XPlane& r,
                                     const XPlane& s, int* zero_hit) {
  XPlane one;
  one.a[0] = one.a[1] = one.a[2] = one.a[3] = 1;
  one.n[0] = one.n[1] = one.n[2] = 0;
  one.radical = 0;
  one.rank = 0;
  const XPlane* rows3[4] = {&p, &q, &r, &one};
  int sD3 = det4_sign(rows3);
  const XPlane* rows[4] = {&p, &q, &r, &s};
  int sD4 = det4_sign(rows);
  if (sD4 != 0) return sD4 * sD3;
  *zero_hit = 1;
  // inward perturbation a_k -> a_k - eps^rank(k) * 1:  D4(eps) = D4 - sum eps^rank C_k;
  // visit the rows in increasing rank (selection by mask: an in-place insertion sort of a
  // local index array was observed to be evaluated differently on sm_100a than on the host,
  // see tests/native/sos_probe.cu)
  unsigned used = 0u;
  for (int o = 0; o < 4; ++o) {
    int best = -1;
    long long br = 0;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const bool free_k = ((used >> k) & 1u) == 0u;
      if (free_k && (best < 0 || rows[k]->rank < br)) {
        best = k;
        br = rows[k]->rank;
      }
    }
    used |= 1u << best;
    const XPlane* rr[4] = {best == 0 ? &one : rows[0], best == 1 ? &one : rows[1],
                           best == 2 ? &one : rows[2], best == 3 ? &one : rows[3]};
    int sC = det4_sign(rr);
    if (sC != 0) return -sC * sD3;
  }
  return 0;  // unreachable: C_s = D3 != 0
}

// exact zero test of det[p; q; r; s] (no perturbation)
static __host__ __device__ __noinline__ bool det4_is_zero(const XPlane& p, const XPlane& q, const XPlane& r,
                                    const XPlane& s) {
  const XPlane* rows[4] = {&p, &q, &r, &s};
  return det4_sign(rows) == 0;
}

// int128 -> double via the magnitude: hi * 2^64 + lo (relative error <= 2^-52)
__host__ __device__ inline double i128_to_double(i128 v) {
  bool neg = v < 0;
  unsigned __int128 u = neg ? (unsigned __int128)(-v) : (unsigned __int128)v;
  double d = (double)(unsigned long long)(u >> 64) * 18446744073709551616.0 +
             (double)(unsigned long long)u;
  return neg ? -d : d;
}

// exact homogeneous vertex K = cross(a_p, a_q, a_r), normalised to sum(K) > 0, as doubles
static __host__ __device__ __noinline__ void exact_vertex(const XPlane& p, const XPlane& q, const XPlane& r,
                                    double K[4]) {
  i128 Ki[4];
  i128 sum = 0;
#pragma unroll
  for (int m = 0; m < 4; ++m) {
    long long a[3], b[3], c[3];
    int n = 0;
    for (int k = 0; k < 4; ++k)
      if (k != m) {
        a[n] = p.a[k];
        b[n] = q.a[k];
        c[n] = r.a[k];
        ++n;
      }
    i128 d = det3_i(a, b, c);
    Ki[m] = ((3 + m) & 1) ? -d : d;
    sum += Ki[m];
  }
  bool flip = sum < 0;
#pragma unroll
  for (int m = 0; m < 4; ++m) {
    i128 v = flip ? -Ki[m] : Ki[m];
    K[m] = i128_to_double(v);
  }
}

// Statistics counters of a kernel: every thread passes its warp-reduced values (only the
// warp leader's count); warp leaders combine them in shared memory and one thread per block
// issues one global atomic per non-zero counter.  Must be called by every thread of the block.
// (Per-warp atomics on the same few addresses serialise in L2: tens of microseconds per
// launch.)  kind[k]: 0 = add, 1 = max.
template <int K>
__device__ inline void block_stats(unsigned long long* stats, const int (&slot)[K],
                                   const int (&kind)[K], const unsigned long long (&v)[K]) {
  __shared__ unsigned long long s_red[K];
  if (threadIdx.x < K) s_red[threadIdx.x] = 0ull;
  __syncthreads();
  if ((threadIdx.x & 31) == 0) {
#pragma unroll
    for (int k = 0; k < K; ++k)
      if (v[k]) {
        if (kind[k]) atomicMax(&s_red[k], v[k]);
        else atomicAdd(&s_red[k], v[k]);
      }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
#pragma unroll
    for (int k = 0; k < K; ++k)
      if (s_red[k]) {
        if (kind[k]) atomicMax(stats + slot[k], s_red[k]);
        else atomicAdd(stats + slot[k], s_red[k]);
      }
  }
}

}  // namespace rpd
