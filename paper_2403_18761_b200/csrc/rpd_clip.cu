// rpd_clip.cu -- SURVEY.md §8(a) rows a4 (Tet-Cell clipping) and a5 (piece output).
//
// For every candidate pair (t, i) of the relation filter the piece
//     P(t, i) = t  n  { x : PD_i(x) <= PD_j(x), j in N(i) }
// is built by sequential convex clipping of the tet by the radical half-spaces of sphere i
// against all of its power neighbours.  Polytope representation after Ray et al.
// (PAPER.md:382): half-spaces as 4 coefficients, every vertex = the triplet of half-spaces
// through it, kept as an oriented triangle of the dual triangulation so that clipping is a
// local re-triangulation of the conflict region and facets can be walked.
//
// B200 mapping: a group of GW lanes per pair (GW = 16: two pairs per warp run in lockstep),
// VPL vertex slots per lane (slot v = GW k + lane), the polytope in per-group shared memory
// (vertex slots updated in place, a live-slot mask, explicit dual-edge links).  The fast kernel has GW = 16,
// VPL = 1 (<= 16 vertices and planes); pairs that exceed it are re-run by the same kernel
// instantiated with GW = 32, VPL = 4 (<= 128).  The k_site planes are first classified GW at a
// time, one per lane, from their exact values at the 4 tet corners:
// planes with all four values > 0 cannot cut (most of them), a plane with all four < 0
// empties the piece; only the remaining planes run the per-vertex sign pass.
//
// Signs: the plane value at a vertex is g_s . K with K the fp64
// homogeneous vertex (3x3 cofactors of its planes' barycentric 4-vectors) and a running
// error bound F; |g_s . K| > |g_s|_1 * F decides it, otherwise the exact int128 path
// evaluates det[a_p; a_q; a_r; a_s] and applies the inward symbolic perturbation.
//
// Outputs per pair: non-empty flag, volume, first moment (facet fans, deterministic warp
// reduction), tet-face mask and incidences as a bitmask over the positions of N(i)
// (positive-area SoS facets expanded by exactly coincident sources, R7).
#include <mutex>

#include "rpd_ctx.h"
#include "rpd_internal.cuh"

#ifndef RPD_CLIP_GW
#define RPD_CLIP_GW 16   // lanes per pair in the fast kernel (2 pairs per warp)
#endif
#ifndef RPD_CLIP_VPL
#define RPD_CLIP_VPL 1   // vertex slots per lane in the fast kernel
#endif
#ifndef RPD_CLIP_MINB
#define RPD_CLIP_MINB 2  // min resident blocks per SM for the fast kernel
#endif
#ifndef RPD_CLIP_STATIC
#define RPD_CLIP_STATIC 90  // percent of the fast kernel's pairs assigned grid-stride
#endif
#ifndef RPD_CLIP_THREADS
#define RPD_CLIP_THREADS 256  // threads per block of the fast kernel
#endif

#ifndef RPD_CLIP_MID_VPL
#define RPD_CLIP_MID_VPL 2  // vertex slots per lane of the middle (first overflow) tier, GW = 32
#endif
#ifndef RPD_CLIP_MID32
#define RPD_CLIP_MID32 0    // 1: a 32-slot tier (GW = 32, one slot per lane) before the middle one (measured slower)
#endif

namespace rpd {

template <int GW, int VPL>
struct alignas(16) WarpState {  // (16-byte aligned: double2 accesses)
  static constexpr int MAXV = GW * VPL;
  static constexpr int MAXP = GW * VPL;
  double g[MAXP][4];       // barycentric plane vectors (exact integers)
  double gb[GW][4];        // the current batch of classified planes (one per lane)
  double K[MAXV][4];       // homogeneous vertices (slots; the live set is a group mask)
  double F[MAXV];          // error scalars
  double KM[MAXV];         // max |K_m| of every vertex
  double x[MAXV][3];       // final vertex coordinates (lattice units, relative to V0)
  double V[4][3];          // tet corners (lattice units)
  double val[MAXV];        // plane value g_s . K of every vertex in the current sign pass
  unsigned tri[MAXV];      // oriented plane triplet of every vertex (3 x 8 bits)
  unsigned char nb[MAXV][4];  // vertex across edge r = (tri[r], tri[r+1]) of the dual
  unsigned char vx[MAXV];  // 1 if the current sign was decided by the exact path
  static constexpr int MAXS = VPL > 1 ? MAXV : 1;
  double Kn[MAXS][4];      // staging of the new vertices of a cut when they outnumber the lanes
  double Fn[MAXS];
  double KMn[MAXS];
  unsigned dsc[MAXV];      // new-vertex descriptors: u | v << 8 | x << 16 | y << 24
  unsigned short dq[MAXV];  // and their target slot codes (slot, or MAXV + extra number)
  unsigned char xs[MAXV];  // slot of every extra new vertex of the current cut
  unsigned char c0[MAXP];  // cut step: the new vertex whose first (second) plane is p
  unsigned char c1[MAXP];
  int src[MAXP];           // radical: sphere j; tet face k: -1-k
  int eidx[MAXP];          // CSR entry of a radical plane, -1 for faces
  int tw[MAXP];            // twin[eidx] (next coincident CSR entry of the row), -1 if none
  int ref[MAXP];           // reference vertex of every facet (fan apex)
  long long pay[16];       // Euler payload numerators of the tet's elements (rpd_euler.cu)
};

// oriented dual triangles of the 4 tet corners (corner k = faces != k); this orientation
// makes the facet walk below produce positive volumes for positively oriented tets
__constant__ unsigned CORNER_TRI[4] = {
    1u | (3u << 8) | (2u << 16), 0u | (2u << 8) | (3u << 16), 0u | (3u << 8) | (1u << 16),
    0u | (1u << 8) | (2u << 16)};

__device__ __forceinline__ int tri_at(unsigned tr, int k) { return (tr >> (8 * k)) & 0xff; }
__device__ __forceinline__ bool tri_has(unsigned tr, int p) {
  return tri_at(tr, 0) == p || tri_at(tr, 1) == p || tri_at(tr, 2) == p;
}
__device__ __forceinline__ unsigned tri_pack(int a, int b, int c) {
  return (unsigned)a | ((unsigned)b << 8) | ((unsigned)c << 16);
}

// neighbours of the 4 tet corners across their dual edges (CORNER_TRI orientation)
__constant__ unsigned char CORNER_NB[4][3] = {{2, 1, 3}, {3, 0, 2}, {1, 0, 3}, {2, 0, 1}};

// max(|a|, |b|) of doubles through their bit patterns (no FP64 min/max instructions)
__device__ __forceinline__ double absmax(double a, double b) {
  const long long x = __double_as_longlong(a) & 0x7fffffffffffffffll;
  const long long y = __double_as_longlong(b) & 0x7fffffffffffffffll;
  return __longlong_as_double(x > y ? x : y);
}
// 2^-e with 2^(e-1) <= m < 2^e for a normal m > 0 (so m * scale is in [0.5, 1))
__device__ __forceinline__ double inv_pow2_ceil(double m) {
  const long long ex = ((__double_as_longlong(m) >> 52) & 0x7ff) - 1022;
  return __longlong_as_double((1023 - ex) << 52);
}

template <int W>
struct Bits {
  unsigned w[W];
  __device__ void clear() {
#pragma unroll
    for (int k = 0; k < W; ++k) w[k] = 0u;
  }
  __device__ void set(int p) { w[p >> 5] |= 1u << (p & 31); }
  __device__ bool has(int p) const { return (w[p >> 5] >> (p & 31)) & 1u; }
  __device__ void set_tri(unsigned tr) {
    set(tri_at(tr, 0));
    set(tri_at(tr, 1));
    set(tri_at(tr, 2));
  }
  __device__ void warp_or(unsigned mask) {
#pragma unroll
    for (int k = 0; k < W; ++k) w[k] = __reduce_or_sync(mask, w[k]);
  }
  // next set bit >= from, or -1
  __device__ int next(int from) const {
    for (int k = from >> 5; k < W; ++k) {
      unsigned m = w[k];
      if (k == (from >> 5)) m &= (from & 31) ? (~0u << (from & 31)) : ~0u;
      if (m) return 32 * k + __ffs(m) - 1;
    }
    return -1;
  }
};

// slot masks: word k, bit l <-> slot GW k + l (group-local bits)
template <int VPL>
__device__ __forceinline__ int mask_count(const unsigned (&m)[VPL]) {
  int c = 0;
#pragma unroll
  for (int k = 0; k < VPL; ++k) c += __popc(m[k]);
  return c;
}
// slot of the j-th (0-based) set bit (j is small: clear the j lowest bits, take the next)
template <int GW, int VPL>
__device__ __forceinline__ int mask_nth(const unsigned (&m)[VPL], int j) {
#pragma unroll
  for (int k = 0; k < VPL; ++k) {
    const int c = __popc(m[k]);
    if (j < c) {
      unsigned w = m[k];
      for (int q = 0; q < j; ++q) w &= w - 1u;
      return GW * k + __ffs(w) - 1;
    }
    j -= c;
  }
  return -1;
}
template <int GW>
__device__ __forceinline__ bool slot_in(const unsigned* m, int v) {
  return (m[v / GW] >> (v % GW)) & 1u;
}

struct ClipCtx {
  const double4* planes;   // global plane table (for Cartesian normals)
  long long N;             // sphere count (SoS rank of tet faces = N + k)
};

template <int GW, int VPL>
__device__ inline void make_xplane(const WarpState<GW, VPL>& S, const ClipCtx& C, int id,
                                   XPlane* xp) {
#pragma unroll
  for (int k = 0; k < 4; ++k) xp->a[k] = (long long)S.g[id][k];
  int src = S.src[id];
  if (src >= 0) {
    double4 p = C.planes[S.eidx[id]];
    xp->n[0] = (long long)p.x;
    xp->n[1] = (long long)p.y;
    xp->n[2] = (long long)p.z;
    xp->radical = 1;
    xp->rank = src;
  } else {
    xp->n[0] = xp->n[1] = xp->n[2] = 0;
    xp->radical = 0;
    xp->rank = C.N + (-1 - src);
  }
}

// ---- exact slow paths (out of line, so their int128 state does not weigh on the kernel)

// SoS sign of the plane s (table id sid, or a new plane given by its vector, CSR entry and
// rank when sid < 0) at the vertex with planes tr
template <int GW, int VPL>
__device__ __noinline__ int exact_sign(const WarpState<GW, VPL>& S, const ClipCtx& C, unsigned tr,
                                       int sid, const double* s, int es, int rank,
                                       int* zero_hit) {
  XPlane xa, xb, xc, xs;
  make_xplane(S, C, tri_at(tr, 0), &xa);
  make_xplane(S, C, tri_at(tr, 1), &xb);
  make_xplane(S, C, tri_at(tr, 2), &xc);
  if (sid >= 0) {
    make_xplane(S, C, sid, &xs);
  } else {
#pragma unroll
    for (int q = 0; q < 4; ++q) xs.a[q] = (long long)s[q];
    const double4 pl = C.planes[es];
    xs.n[0] = (long long)pl.x;
    xs.n[1] = (long long)pl.y;
    xs.n[2] = (long long)pl.z;
    xs.radical = 1;
    xs.rank = rank;
  }
  return sos_sign_exact(xa, xb, xc, xs, zero_hit);
}

template <int GW, int VPL>
__device__ __noinline__ bool exact_is_zero(const WarpState<GW, VPL>& S, const ClipCtx& C,
                                           unsigned tr, int q) {
  XPlane xa, xb, xc, xq;
  make_xplane(S, C, tri_at(tr, 0), &xa);
  make_xplane(S, C, tri_at(tr, 1), &xb);
  make_xplane(S, C, tri_at(tr, 2), &xc);
  make_xplane(S, C, q, &xq);
  return det4_is_zero(xa, xb, xc, xq);
}

template <int GW, int VPL>
__device__ __noinline__ void exact_vertex_of(const WarpState<GW, VPL>& S, const ClipCtx& C, int a,
                                             int b, int c, double* K) {
  XPlane pa, pb, pc;
  make_xplane(S, C, a, &pa);
  make_xplane(S, C, b, &pb);
  make_xplane(S, C, c, &pc);
  exact_vertex(pa, pb, pc, K);
}

// fp64 homogeneous vertex of planes (a, b, c), normalised to sum(K) > 0, with the error
// scalar F such that |g . K~ - g . K| <= |g|_1 F for every plane vector g.
template <int GW, int VPL>
__device__ inline void vertex_from_planes(const WarpState<GW, VPL>& S, const ClipCtx& C, int a,
                                          int b, int c, double K[4], double* F, double* KMo,
                                          int* nexact) {
  const double* ra = S.g[a];
  const double* rb = S.g[b];
  const double* rc = S.g[c];
  double E = 0.0, Kmax = 0.0, sum = 0.0, sabs = 0.0;
#pragma unroll
  for (int m = 0; m < 4; ++m) {
    const int c0 = m == 0 ? 1 : 0;
    const int c1 = m <= 1 ? 2 : 1;
    const int c2 = m <= 2 ? 3 : 2;
    double m0 = fma(rb[c1], rc[c2], -rb[c2] * rc[c1]);
    double m1 = fma(rb[c0], rc[c2], -rb[c2] * rc[c0]);
    double m2 = fma(rb[c0], rc[c1], -rb[c1] * rc[c0]);
    double d = fma(ra[c0], m0, fma(-ra[c1], m1, ra[c2] * m2));
    double p0 = fabs(rb[c1] * rc[c2]) + fabs(rb[c2] * rc[c1]);
    double p1 = fabs(rb[c0] * rc[c2]) + fabs(rb[c2] * rc[c0]);
    double p2 = fabs(rb[c0] * rc[c1]) + fabs(rb[c1] * rc[c0]);
    double perm = fabs(ra[c0]) * p0 + fabs(ra[c1]) * p1 + fabs(ra[c2]) * p2;
    K[m] = (m & 1) ? d : -d;  // (-1)^(3+m)
    E = absmax(E, perm);
    Kmax = absmax(Kmax, d);
    sum += K[m];
    sabs += fabs(K[m]);
  }
  E *= 10.0 * U;
  // certify sign(sum K) = sign(D3)
  double sb = (4.0 * E + 4.0 * U * sabs) * (1.0 + 1e-9);
  if (!(fabs(sum) > sb)) {
    exact_vertex_of(S, C, a, b, c, K);  // normalised, each component within 2^-52 relative
    ++*nexact;
    const double km = absmax(absmax(K[0], K[1]), absmax(K[2], K[3]));
    *F = 9.0 * U * km * (1.0 + 1e-9);
    *KMo = km;
    return;
  }
  if (sum < 0.0) {
#pragma unroll
    for (int m = 0; m < 4; ++m) K[m] = -K[m];
  }
  *F = (E + 5.0 * U * Kmax) * (1.0 + 1e-9);
  *KMo = Kmax;
}

// New vertex on the edge from the kept vertex u to the removed vertex v where plane s
// vanishes: K = val_u K_v - val_v K_u (a positive combination; g_s . K = 0).  Error bound
// from the endpoints' bounds and the plane values' bounds; rescaled by a power of two.
// Falls back to the exact-cofactor construction from the three planes when an endpoint's
// sign came from the exact path or the bound is too loose.
template <int GW, int VPL>
__device__ inline int new_vertex(const WarpState<GW, VPL>& S, const ClipCtx& C, int u,
                                 int v, int x, int y, int sid, double sabs, double K[4],
                                 double* F, double* KMo, int* nexact) {
  if (!S.vx[u] && !S.vx[v]) {
    const double vu = S.val[u], avv = -S.val[v];  // vu > B_u > 0, -val_v > B_v > 0
    const double* Ku = S.K[u];
    const double* Kv = S.K[v];
    const double Fu = S.F[u], Fv = S.F[v];
    const double ku = S.KM[u], kv = S.KM[v];
#pragma unroll
    for (int m = 0; m < 4; ++m) K[m] = fma(vu, Kv[m], avv * Ku[m]);
    const double km = absmax(absmax(K[0], K[1]), absmax(K[2], K[3]));
    const double Bu = sabs * Fu, Bv = sabs * Fv;
    const double E = Bu * kv + (vu + Bu) * Fv + Bv * ku + (avv + Bv) * Fu +
                     3.0 * U * (vu * kv + avv * ku);
    const double Fn = (E + 5.0 * U * km) * (1.0 + 1e-9);
    if (Fn <= 1e-6 * km && km > 1e-300) {
      const double sc = inv_pow2_ceil(km);  // exact power-of-two rescale to [0.5, 1)
#pragma unroll
      for (int m = 0; m < 4; ++m) K[m] *= sc;
      *F = Fn * sc;
      *KMo = km * sc;
      return 0;
    }
  }
  vertex_from_planes(S, C, x, y, sid, K, F, KMo, nexact);
  return 1;
}

enum { ST_ALIVE = 0, ST_EMPTY = 1, ST_OVER = 2 };
constexpr int ST_N_CLIP = 13;  // statistics counters reduced by the clip kernels

#ifdef RPD_CLIP_PHASES
// development aid: cycles per clip phase summed over groups (lane 0 of each group)
__device__ unsigned long long g_phase[8];
#define PHASE_MARK(k)                      \
  do {                                     \
    const long long _t = clock64();        \
    ph[k] += _t - ph_t;                    \
    ph_t = _t;                             \
  } while (0)
#else
#define PHASE_MARK(k) \
  do {                \
  } while (0)
#endif

// fractional Euler characteristics: carrier of a piece element from the
// tet faces among its planes (bit k = tet face k) -> index into WarpState::pay: 14 = inside
// the tet (payload 1 = L), 10 + k = face k, 4 + e = tet edge e (corner pairs 01 02 03 12 13 23)
// when two faces meet, corner c when three do
__constant__ unsigned char EU_BIDX[16] = {14, 10, 11, 9, 12, 8, 6, 3, 13, 7, 5, 2, 4, 1, 0, 14};
__device__ __forceinline__ unsigned eu_pm(int p) { return p < 4 ? 1u << p : 0u; }
// the RPE endpoint record of radical plane x: 16 bits per tet face (ranks + 1 of two planes)
__device__ __forceinline__ unsigned long long rep_of(const unsigned* epw, int x) {
  unsigned long long r = 0ull;
#pragma unroll
  for (int f = 0; f < 4; ++f) r |= (unsigned long long)((epw[4 * x + f] >> 8) & 0xffffu) << (16 * f);
  return r;
}

struct PairOut {
  double* vol;
  double* m1;
  uint8_t* flag;       // 0 empty, 1 non-empty, 2 overflow (re-run by the wide kernel)
  uint8_t* fm;
  unsigned* incmask;   // incidence bitmask words of every pair (positions in N(i))
  const int32_t* mask_off;
  const unsigned* cut; // per pair (mask_off layout): the planes that can cut (filter values)
  int32_t* over_list;  // pairs that overflowed (re-run by the next wider kernel)
  int32_t* over_count;
  // Euler (eu_rec == nullptr: off)
  const uint4* eu_rec;      // per ctx-local tet: the 14 sharing counts of its elements
  const long long* eu_Lt;   // per ctx-local tet: its denominator L_t = lcm of its 14 counts
  long long* eu_piece;      // per pair: Euler of the piece x L
  unsigned* rmask;          // per pair: SoS radical facets (bits over N(i), incmask layout)
  long long* rval;          // per (pair, row position): Euler of that facet x L
  uint8_t* sfm;             // per pair: tet faces that are SoS facets (CC numbers, NEXT-2)
  uint8_t* rfm;             // per (pair, row position): tet faces the facet has an edge on
  unsigned long long* radj; // per (pair, row position): radical facets sharing an edge (rank)
  unsigned long long* rep;  // per (pair, row position): RPE endpoint faces (rpd_ctx.h PieceSet)
};

// EU: also the fractional Euler characteristics (a separate instantiation, so that the plain
// clip keeps its register allocation)
template <int GW, int VPL, bool EU>
__global__ void __launch_bounds__(VPL == 1 && GW == RPD_CLIP_GW ? RPD_CLIP_THREADS
                                  : (VPL <= 2 ? 256 : (VPL <= 4 ? 64 : 32)),
                                  VPL == 1 && GW == RPD_CLIP_GW ? RPD_CLIP_MINB : (VPL <= 2 ? 2 : 1)) k_clip(
    int64_t n_pairs, const int32_t* __restrict__ pair_list, const int32_t* __restrict__ pair_tet,
    const int32_t* __restrict__ tet_ids, const int32_t* __restrict__ cand_idx,
    const double* __restrict__ tx, int64_t T, const int32_t* __restrict__ nbr_off,
    const int32_t* __restrict__ nbr_idx, const double4* __restrict__ planes,
    const int32_t* __restrict__ twin, long long N, PairOut out,
    unsigned long long* __restrict__ stats, const int32_t* __restrict__ n_dev,
    int* __restrict__ dyn, const PDyn* __restrict__ pd) {
  using WS = WarpState<GW, VPL>;
  if (n_dev) n_pairs = *n_dev;
  if (pd) {  // device-driven update: the sphere count and the pool tail from the device
    N = pd->N;
    cand_idx += pd->fill_c;
  }
  constexpr int MAXP = WS::MAXP;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  WS& S = reinterpret_cast<WS*>(smem_raw)[threadIdx.x / GW];
  // GW lanes clip one pair (a "group"); 32 / GW groups per warp run in lockstep
  const int lane = threadIdx.x & (GW - 1);
  const int grp = (threadIdx.x & 31) / GW;
  const unsigned GLOW = GW == 32 ? 0xffffffffu : ((1u << GW) - 1u);
  const unsigned FULL = GLOW << (GW * grp);  // this group's lanes
  ClipCtx C{planes, N};
  const int64_t gw = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) / GW;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) / GW;
  int n_exact = 0, n_zero = 0, max_v = 0, max_p = 0, n_over = 0;
  int d_sign = 0, d_out = 0, d_fb = 0;  // diagnostics
  int n_euover = 0;  // pieces with more than 64 radical facets (Euler/topology mode)
  // algorithmic work (warp-uniform quantities, counted once per warp)
  unsigned c_planes = 0, c_tests = 0, c_constr = 0, c_fan = 0;  // per group: small
#ifdef RPD_CLIP_PHASES
  long long ph[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  long long ph_t = clock64();
#endif

  // software pipeline of the pair's index loads: level 1 (pair -> tet, sphere) is fetched one
  // pair ahead at the top of the loop, level 2 (tet corners, CSR row bounds) once the plane
  // loop is done, so the dependent global loads overlap the previous pair's work
  int64_t pf_p = 0, pf_t = 0;
  int pf_a = 0, pf_i = 0, pf_e0 = 0, pf_e1 = 0, pf_mo = 0;
  constexpr int NTX = (12 + GW - 1) / GW;  // tet corner coordinates per lane
  double pf_tx[NTX];
  auto fetch1 = [&](int64_t pj) {
    pf_p = pair_list ? (int64_t)pair_list[pj] : pj;
    pf_a = pair_tet[pf_p];
    pf_i = cand_idx[pf_p];
    pf_mo = out.mask_off[pf_p];
  };
  auto fetch2 = [&]() {
    const int64_t t = tet_ids ? (int64_t)tet_ids[pf_a] : (int64_t)pf_a;
    pf_t = t;
#pragma unroll
    for (int q = 0; q < NTX; ++q)
      if (lane + GW * q < 12) pf_tx[q] = __ldg(tx + (lane + GW * q) * T + t);
    pf_e0 = __ldg(nbr_off + pf_i);
    pf_e1 = __ldg(nbr_off + pf_i + 1);
  };
  // pair order: the first RPD_CLIP_STATIC percent grid-stride (no atomics), the rest taken
  // one at a time from a counter (dyn), so that the groups finish together instead of the
  // kernel waiting for the groups whose static share drew the most expensive pieces
  const int64_t n_static = dyn ? n_pairs * RPD_CLIP_STATIC / 100 : n_pairs;
  auto next_of = [&](int64_t cur) -> int64_t {
    if (cur + nw < n_static) return cur + nw;
    if (!dyn) return n_pairs;
    long long v = 0;
    if (lane == 0) v = n_static + atomicAdd(dyn, 1);
    return (int64_t)__shfl_sync(FULL, v, 0, GW);
  };
  const int64_t first = gw < n_static ? gw : next_of(n_pairs);
  if (first < n_pairs) {
    fetch1(first);
    fetch2();
  }
  int64_t nxt = n_pairs;
  for (int64_t pi = first; pi < n_pairs; pi = nxt) {
    nxt = next_of(pi);
    const int64_t p = pf_p, t_cur = pf_t;
    const int e0 = pf_e0, e1 = pf_e1, mo = pf_mo;
    const int nwp = (e1 - e0 + 31) >> 5;  // incidence-mask words of the pair
#pragma unroll
    for (int q = 0; q < NTX; ++q)
      if (lane + GW * q < 12) (&S.V[0][0])[lane + GW * q] = pf_tx[q];
    const bool has_next = nxt < n_pairs;
    if (has_next) fetch1(nxt);
    if (lane < 4) {
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        S.g[lane][k] = (k == lane) ? 1.0 : 0.0;
        S.K[lane][k] = (k == lane) ? 1.0 : 0.0;
      }
      S.src[lane] = -1 - lane;
      S.eidx[lane] = -1;
      S.tw[lane] = -1;
      S.F[lane] = 0.0;
      S.KM[lane] = 1.0;
      S.tri[lane] = CORNER_TRI[lane];
#pragma unroll
      for (int r = 0; r < 3; ++r) S.nb[lane][r] = CORNER_NB[lane][r];
    }
    __syncwarp(FULL);
    PHASE_MARK(0);
    int np = 4, nv = 4, status = ST_ALIVE, zero_hit = 0;
    unsigned live[VPL];  // live vertex slots (group-uniform)
#pragma unroll
    for (int k = 0; k < VPL; ++k) live[k] = k == 0 ? 0xfu : 0u;
    // the planes to classify: the pair's cut mask (planes with a corner value <= 0, from the
    // relation filter's exact Alg. 1 values), taken GW set bits at a time in
    // CSR order; each selected plane is still checked here (a superset mask is safe)
    const int kp = e1 - e0;
    int cw = 0;                       // current mask word
    unsigned cmask = 0u;              // its unprocessed bits
    if (kp > 0) {
      cmask = out.cut[mo];
      if (kp < 32) cmask &= (1u << kp) - 1u;
    }
    while (status == ST_ALIVE) {
      while (cmask == 0u && ++cw < nwp) {
        cmask = out.cut[mo + cw];
        if (kp - 32 * cw < 32) cmask &= (1u << (kp - 32 * cw)) - 1u;
      }
      if (cmask == 0u) break;
      const int nset = __popc(cmask);
      const bool have = lane < nset;
      const int bit = have ? (int)__fns(cmask, 0, lane + 1) : 0;
      const int e = e0 + 32 * cw + bit;
      {  // drop the bits taken by this batch
        const int last = __shfl_sync(FULL, bit, min(nset, GW) - 1, GW);
        cmask = nset <= GW ? 0u : (cmask & ~((2u << last) - 1u));
      }
      c_planes += min(nset, GW);
      double g[4];
      bool allpos = false;
      if (have) {
        const double4 pl = planes[e];
        allpos = true;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          g[k] = fma(pl.x, S.V[k][0], fma(pl.y, S.V[k][1], fma(pl.z, S.V[k][2], pl.w)));
          allpos &= g[k] > 0.0;
        }
        if (!allpos) {  // staged for the sign passes (read by all lanes after the sync)
          reinterpret_cast<double2*>(S.gb[lane])[0] = make_double2(g[0], g[1]);
          reinterpret_cast<double2*>(S.gb[lane])[1] = make_double2(g[2], g[3]);
        }
      }
      // (no "negative at all four corners" early exit: Alg. 1 admits a candidate only if
      // every plane is positive at some corner -- the same exact values -- and such a plane
      // would empty the piece in its sign pass anyway)
      unsigned act = (__ballot_sync(FULL, have && !allpos) >> (GW * grp)) & GLOW;
      if (act) __syncwarp(FULL);
      PHASE_MARK(1);
      while (act && status == ST_ALIVE) {
        const int l = __ffs(act) - 1;
        act &= act - 1;
#ifdef RPD_CLIP_PHASES
        ++ph[6];
#endif
        double s[4];  // the plane's values at the 4 tet corners (its barycentric vector)
        {
          const double2 a = reinterpret_cast<const double2*>(S.gb[l])[0];
          const double2 b = reinterpret_cast<const double2*>(S.gb[l])[1];
          s[0] = a.x;
          s[1] = a.y;
          s[2] = b.x;
          s[3] = b.y;
        }
        const int es = __shfl_sync(FULL, e, l, GW);
        const int js = __ldg(nbr_idx + es);
        const int tws = __ldg(twin + es);
        const double sabs = fabs(s[0]) + fabs(s[1]) + fabs(s[2]) + fabs(s[3]);

        // ---- sign of every vertex slot
        int sg[VPL];
        double valr[VPL];
        unsigned char vxr[VPL];
        unsigned negm[VPL], posm[VPL];
#pragma unroll
        for (int k = 0; k < VPL; ++k) negm[k] = posm[k] = 0u;
        bool anyneg = false, anypos = false;
#pragma unroll
        for (int k = 0; k < VPL; ++k) {
          sg[k] = 0;
          if (!live[k]) continue;  // no live slot in this word (group-uniform)
          const int v = GW * k + lane;
          const bool valid = (live[k] >> lane) & 1u;
          if (valid) {
            const double2 k01 = reinterpret_cast<const double2*>(S.K[v])[0];
            const double2 k23 = reinterpret_cast<const double2*>(S.K[v])[1];
            const double val = fma(s[0], k01.x, fma(s[1], k01.y, fma(s[2], k23.x, s[3] * k23.y)));
            const double B = sabs * S.F[v];
            valr[k] = val;
            vxr[k] = 0;
            if (val > B) sg[k] = 1;
            else if (val < -B) sg[k] = -1;
            else {
              int zh = 0;
              sg[k] = exact_sign(S, C, S.tri[v], -1, s, es, js, &zh);
              vxr[k] = 1;
              ++n_exact;
              ++d_sign;
              if (zh) {
                ++n_zero;
                zero_hit = 1;
              }
            }
          }
          // (signs are never zero: the SoS rule decides every tie)
          posm[k] = (__ballot_sync(FULL, valid && sg[k] > 0) >> (GW * grp)) & GLOW;
          negm[k] = live[k] & ~posm[k];
          anyneg |= negm[k] != 0u;
          anypos |= posm[k] != 0u;
        }
        c_tests += nv;
#ifdef RPD_TRACE
        if (p == RPD_TRACE) {
          for (int k = 0; k < VPL; ++k) {
            int v = GW * k + lane;
            if ((live[k] >> lane) & 1u) {
              unsigned tr = S.tri[v];
              printf("plane j=%d es=%d v=%d tri=(%d,%d,%d) sg=%d K=(%g,%g,%g,%g) F=%g\n",
                     nbr_idx[es], es, v, tri_at(tr, 0), tri_at(tr, 1), tri_at(tr, 2), sg[k],
                     S.K[v][0], S.K[v][1], S.K[v][2], S.K[v][3], S.F[v]);
            }
          }
        }
#endif
        PHASE_MARK(2);
        if (!anyneg) continue;  // the plane does not cut: skip it
        if (anypos) {  // a cut: the signs' values for the new-vertex construction
#pragma unroll
          for (int k = 0; k < VPL; ++k) {
            const int v = GW * k + lane;
            if ((live[k] >> lane) & 1u) {
              S.val[v] = valr[k];
              S.vx[v] = vxr[k];
            }
          }
        }
        if (!anypos) {
          status = ST_EMPTY;
          break;
        }
        if (np >= MAXP) {
          status = ST_OVER;
          break;
        }
        const int sid = np++;
#ifdef RPD_CLIP_PHASES
        ++ph[7];
#endif
        if (lane == 0) {  // (read by other lanes only after the descriptor sync below)
#pragma unroll
          for (int k = 0; k < 4; ++k) S.g[sid][k] = s[k];
          S.src[sid] = js;
          S.eidx[sid] = es;
          S.tw[sid] = tws;
        }
        // ---- new vertices, in place: one per boundary edge of the conflict region (a removed
        // vertex v with a kept neighbour u across its dual edge (x, y)), oriented as that edge:
        // (x, y, s).  Kept vertices stay in their slots; the first new vertex of v takes v's
        // slot, further ones ("extras") take free slots (holes, removed vertices without new
        // ones).  Links: across (x, y) -> u; across (y, s) and (s, x) -> the neighbouring new
        // vertices around the new facet s, found through per-plane tables.
        const unsigned lt = (1u << lane) - 1u;  // group lanes below this one
        unsigned nbw[VPL], hasnew[VPL], extra[VPL], keptr[VPL];
        int ex_idx[VPL];
        int ex_base = 0;
#pragma unroll
        for (int k = 0; k < VPL; ++k) {
          keptr[k] = 0u;  // bit r: the neighbour across dual edge r is kept
          nbw[k] = 0u;
          ex_idx[k] = 0;
          hasnew[k] = 0u;
          if (!live[k]) continue;
          const int v = GW * k + lane;
          if ((negm[k] >> lane) & 1u) {
            nbw[k] = *reinterpret_cast<const unsigned*>(S.nb[v]);
#pragma unroll
            for (int r = 0; r < 3; ++r)
              keptr[k] |= (unsigned)slot_in<GW>(posm, (nbw[k] >> (8 * r)) & 0xff) << r;
          }
          // extras per removed vertex: ex = nnew - 1 in {0, 1, 2}; prefix over the lanes by
          // its two bit planes
          const int nnew = __popc(keptr[k]);
          const int ex = nnew > 0 ? nnew - 1 : 0;
          hasnew[k] = (__ballot_sync(FULL, nnew > 0) >> (GW * grp)) & GLOW;
          const unsigned b0 = (__ballot_sync(FULL, ex & 1) >> (GW * grp)) & GLOW;
          const unsigned b1 = (__ballot_sync(FULL, ex & 2) >> (GW * grp)) & GLOW;
          ex_idx[k] = ex_base + __popc(b0 & lt) + 2 * __popc(b1 & lt);
          ex_base += __popc(b0) + 2 * __popc(b1);
        }
        // the lowest ex_base free slots take the extras: the free slot of rank r (in slot order)
        // holds extra r; S.xs maps extra numbers to slots
        {
          int rank_base = 0;
#pragma unroll
          for (int k = 0; k < VPL; ++k) {
            const unsigned f = ~(posm[k] | hasnew[k]) & GLOW;
            const int rk = rank_base + __popc(f & lt);
            const bool mine = ((f >> lane) & 1u) && rk < ex_base;
            if (mine) S.xs[rk] = (unsigned char)(GW * k + lane);
            extra[k] = (__ballot_sync(FULL, mine) >> (GW * grp)) & GLOW;
            rank_base += __popc(f);
          }
          if (rank_base < ex_base) {  // more than MAXV vertices
            status = ST_OVER;
            break;
          }
        }
        // descriptors of the new vertices (edge (u, v), planes (x, y), target slot code:
        // the slot v, or MAXV + extra number), numbered in slot order of v; then one lane per
        // new vertex builds it (slot v may be read as an edge endpoint until the following sync)
        {
          int hb = 0;
#pragma unroll
          for (int k = 0; k < VPL; ++k) {
            const int d0 = ex_idx[k] + hb + __popc(hasnew[k] & lt);
            hb += __popc(hasnew[k]);
            if (!keptr[k]) continue;
            const int v = GW * k + lane;
            const unsigned tr = S.tri[v];
            int j = 0;
#pragma unroll
            for (int r = 0; r < 3; ++r) {
              if (!((keptr[k] >> r) & 1u)) continue;
              const int u = (nbw[k] >> (8 * r)) & 0xff;
              const int qc = j == 0 ? v : WS::MAXV + ex_idx[k] + j - 1;
              const int x = tri_at(tr, r), y = tri_at(tr, (r + 1) % 3);
              S.dsc[d0 + j] = (unsigned)u | ((unsigned)v << 8) | ((unsigned)x << 16) |
                              ((unsigned)y << 24);
              S.dq[d0 + j] = (unsigned short)qc;
              ++j;
            }
          }
        }
        const int n_new = mask_count<VPL>(hasnew) + ex_base;
        __syncwarp(FULL);
        if (VPL == 1 || n_new <= GW) {  // (VPL == 1: n_new <= MAXV = GW always)
          // one new vertex per lane, held in registers across the sync
          double K[4], F = 0.0, KMv = 0.0;
          unsigned ds = 0u;
          int q = 0;
          if (lane < n_new) {
            ds = S.dsc[lane];
            q = S.dq[lane];
            if (q >= WS::MAXV) q = S.xs[q - WS::MAXV];
            const int u = ds & 0xff, v = (ds >> 8) & 0xff, x = (ds >> 16) & 0xff, y = ds >> 24;
            d_fb += new_vertex(S, C, u, v, x, y, sid, sabs, K, &F, &KMv, &n_exact);
            // u's link across the edge to v now leads to the new vertex (only this lane
            // touches that byte; the entries other lanes search for are never equal to v)
            const int ru = S.nb[u][0] == v ? 0 : (S.nb[u][1] == v ? 1 : 2);
            S.nb[u][ru] = (unsigned char)q;
          }
          __syncwarp(FULL);
          if (lane < n_new) {
            const int x = (ds >> 16) & 0xff, y = ds >> 24;
#pragma unroll
            reinterpret_cast<double2*>(S.K[q])[0] = make_double2(K[0], K[1]);
            reinterpret_cast<double2*>(S.K[q])[1] = make_double2(K[2], K[3]);
            S.F[q] = F;
            S.KM[q] = KMv;
            S.tri[q] = tri_pack(x, y, sid);
            S.nb[q][0] = (unsigned char)(ds & 0xff);
            S.c0[x] = (unsigned char)q;  // the new vertex whose first plane is x
            S.c1[y] = (unsigned char)q;  // ... whose second plane is y
          }
          __syncwarp(FULL);
          // close the cycle around the new facet s: across (y, s) the new vertex (y, ., s),
          // across (s, x) the new vertex (., x, s)
          if (lane < n_new) {
            const int x = (ds >> 16) & 0xff, y = ds >> 24;
            S.nb[q][1] = S.c0[y];
            S.nb[q][2] = S.c1[x];
          }
        } else {
          // more new vertices than lanes (wide kernels only): staged in shared memory
          for (int d = lane; d < n_new; d += GW) {
            const unsigned ds = S.dsc[d];
            const int u = ds & 0xff, v = (ds >> 8) & 0xff, x = (ds >> 16) & 0xff, y = ds >> 24;
            double K[4], F, KMv;
            d_fb += new_vertex(S, C, u, v, x, y, sid, sabs, K, &F, &KMv, &n_exact);
#pragma unroll
            for (int m = 0; m < 4; ++m) S.Kn[d][m] = K[m];
            S.Fn[d] = F;
            S.KMn[d] = KMv;
            int qd = S.dq[d];
            if (qd >= WS::MAXV) qd = S.xs[qd - WS::MAXV];
            S.dq[d] = (unsigned short)qd;  // decoded for the store loop below
            const int ru = S.nb[u][0] == v ? 0 : (S.nb[u][1] == v ? 1 : 2);
            S.nb[u][ru] = (unsigned char)qd;
          }
          __syncwarp(FULL);
          for (int d = lane; d < n_new; d += GW) {
            const unsigned ds = S.dsc[d];
            const int q = S.dq[d];
            const int x = (ds >> 16) & 0xff, y = ds >> 24;
#pragma unroll
            for (int m = 0; m < 4; ++m) S.K[q][m] = S.Kn[d][m];
            S.F[q] = S.Fn[d];
            S.KM[q] = S.KMn[d];
            S.tri[q] = tri_pack(x, y, sid);
            S.nb[q][0] = (unsigned char)(ds & 0xff);
            S.c0[x] = (unsigned char)q;
            S.c1[y] = (unsigned char)q;
          }
          __syncwarp(FULL);
          for (int d = lane; d < n_new; d += GW) {
            const unsigned ds = S.dsc[d];
            const int q = S.dq[d];
            const int x = (ds >> 16) & 0xff, y = ds >> 24;
            S.nb[q][1] = S.c0[y];
            S.nb[q][2] = S.c1[x];
          }
        }
#pragma unroll
        for (int k = 0; k < VPL; ++k) live[k] = posm[k] | hasnew[k] | extra[k];
        c_constr += n_new;
        nv = mask_count<VPL>(live);
        __syncwarp(FULL);
        PHASE_MARK(3);
      }
    }

    if (has_next) fetch2();
    // ------------------------------------------------------------------ outputs
    if (status != ST_ALIVE) {
      if (status == ST_OVER) {
        ++n_over;
        if (lane == 0 && out.over_list) {
          const int slot = atomicAdd(out.over_count, 1);
          out.over_list[slot] = (int32_t)p;
        }
      }
      if (lane == 0) out.flag[p] = status == ST_OVER ? 2 : 0;
      __syncwarp(FULL);
      continue;
    }
    max_v = max(max_v, nv);
    max_p = max(max_p, np);
    unsigned mytri[VPL];
    Bits<VPL> facets_all;
    facets_all.clear();
#pragma unroll
    for (int k = 0; k < VPL; ++k) {
      const int v = GW * k + lane;
      const bool lv = (live[k] >> lane) & 1u;
      mytri[k] = lv ? S.tri[v] : 0xffffffu;
      if (lv) facets_all.set_tri(mytri[k]);
    }
    facets_all.warp_or(FULL);
    Bits<VPL> facets = facets_all;
    {
      int nf = 0;
#pragma unroll
      for (int k = 0; k < VPL; ++k) nf += __popc(facets_all.w[k]);
      c_fan += 3 * nv - 2 * nf;  // sum over facets of (vertices - 2)
    }

    // zero-area SoS facets (only possible after an exact-zero predicate; C1.7)
    zero_hit = __any_sync(FULL, zero_hit);  // (per lane until here)
    if (zero_hit) {
      for (int f = facets_all.next(0); f >= 0; f = facets_all.next(f + 1)) {
        Bits<VPL> Q;
        Q.clear();
#pragma unroll
        for (int k = 0; k < VPL; ++k)
          if (((live[k] >> lane) & 1u) && tri_has(mytri[k], f)) Q.set_tri(mytri[k]);
        Q.warp_or(FULL);
        Q.w[f >> 5] &= ~(1u << (f & 31));
        bool zero_area = false;
        for (int q = Q.next(0); q >= 0 && !zero_area; q = Q.next(q + 1)) {
          bool on = true;
#pragma unroll
          for (int k = 0; k < VPL; ++k) {
            const int v = GW * k + lane;
            if (((live[k] >> lane) & 1u) && tri_has(mytri[k], f) && !tri_has(mytri[k], q)) {
              const double* K = S.K[v];
              const double* gq = S.g[q];
              const double val =
                  fma(gq[0], K[0], fma(gq[1], K[1], fma(gq[2], K[2], gq[3] * K[3])));
              const double sa = fabs(gq[0]) + fabs(gq[1]) + fabs(gq[2]) + fabs(gq[3]);
              if (fabs(val) > sa * S.F[v]) {
                on = false;
              } else {
                on = on && exact_is_zero(S, C, mytri[k], q);
                ++n_exact;
              }
            }
          }
          zero_area = __all_sync(FULL, on);
        }
        if (zero_area) facets.w[f >> 5] &= ~(1u << (f & 31));
      }
    }

    // incidences: every positive-area facet plus its exactly coincident sources
    unsigned fmask_bits = 0, ibits = 0;
    unsigned* words = out.incmask + mo;
    // k_site <= 32 (one mask word, most pairs): bits or-reduced over the group and stored
    // once; otherwise the words are zeroed here (no memset pass) and then set by
    // fire-and-forget atomics (the zero stores are ordered before them by the warp sync)
    const bool one_word = nwp == 1;
    if (!one_word) {
      for (int w = lane; w < nwp; w += GW) words[w] = 0u;
      __syncwarp(FULL);
    }
#pragma unroll
    for (int k = 0; k < VPL; ++k) {
      const int pl = GW * k + lane;
      if (pl < np) S.ref[pl] = 0x7fffffff;
      if (pl < np && facets.has(pl)) {
        const int src = S.src[pl];
        if (src < 0) {
          fmask_bits |= 1u << (-1 - src);
        } else {
          // radical plane coinciding with tet face a: g = c e_a, c > 0
          const double* gg = S.g[pl];
          int nz = 0, az = 0;
#pragma unroll
          for (int q = 0; q < 4; ++q)
            if (gg[q] != 0.0) {
              ++nz;
              az = q;
            }
          if (nz == 1 && gg[az] > 0.0) fmask_bits |= 1u << az;
          int e = S.eidx[pl];
          int nx = S.tw[pl];
          while (e >= 0) {
            const int pos = e - e0;
            if (one_word) ibits |= 1u << pos;
            else atomicOr(words + (pos >> 5), 1u << (pos & 31));
            e = nx;
            if (e >= 0) nx = twin[e];
          }
        }
      }
    }
    const unsigned facemask = __reduce_or_sync(FULL, fmask_bits);
    if (one_word) {
      const unsigned w = __reduce_or_sync(FULL, ibits);
      if (lane == 0) words[0] = w;
    }
    __syncwarp(FULL);
    PHASE_MARK(4);

    // ---- fractional Euler characteristics (Eq. (1)) of the SoS polytope:
    // Euler(piece) = sum_v pay(v) - sum_e pay(e) + sum_f pay(f) - 1 and, per radical facet f,
    // Euler(f) = sum_{v on f} pay(v) - sum_{e on f} pay(e) + pay(f).  Every vertex is simple
    // (3 planes), so each of its 3 plane pairs is an edge counted at both of its ends: edges
    // enter as halves, accumulated doubled (exact integers over L).  The payload of an element
    // is inherited from the smallest tet simplex holding it: new vertices from
    // the edge they cut, new edges from the face they cut, new facets from the cell.
    if constexpr (EU) {
      long long* acc = reinterpret_cast<long long*>(S.val);  // per plane: doubled facet sums
      {
        // payload numerators over the tet's own denominator L_t: L_t / count (any mesh: no
        // common denominator of the whole mesh is formed)
        const uint4 rc = __ldg(out.eu_rec + t_cur);
        const long long Lt = __ldg(out.eu_Lt + t_cur);
        if (lane < 14) {
          const unsigned w = lane < 4 ? rc.x : (lane < 8 ? rc.y : (lane < 12 ? rc.z : rc.w));
          S.pay[lane] = Lt / (long long)((w >> (8 * (lane & 3))) & 0xffu);
        } else if (lane == 14) {
          S.pay[14] = Lt;
        }
#pragma unroll
        for (int k = 0; k < VPL; ++k) {
          const int pl = GW * k + lane;
          if (pl < np) {
            acc[pl] = 0;
            S.dsc[pl] = 0u;  // (free after the cuts) tet faces next to each facet
            reinterpret_cast<unsigned long long*>(S.KM)[pl] = 0ull;  // adjacent radical facets
            // rank of a radical facet among the piece's radical facets by ascending j (the
            // order of the compacted rpf entries): the cutting planes were added in CSR order,
            // i.e. ascending j, so it is the number of radical facets with a smaller plane id
            if (pl >= 4 && facets_all.has(pl)) {
              int rk = 0;
#pragma unroll
              for (int w = 0; w < VPL; ++w) {
                const int lo = 32 * w, hi = lo + 32;
                unsigned m = facets_all.w[w];
                if (lo < 4) m &= ~0xfu;                       // radical planes only
                if (pl < hi) m &= pl > lo ? (1u << (pl - lo)) - 1u : 0u;  // below pl
                rk += __popc(m);
              }
              S.c0[pl] = (unsigned char)(rk < 64 ? rk : 255);
            }
          }
        }
      }
      // RPE endpoint faces: per (radical plane x, tet face f) a count byte and the ranks + 1 of
      // the (at most two) radical planes y whose edge with x ends on f (free scratch: the
      // classification batch / the cut staging, unused after the cuts)
      unsigned* epw = VPL == 1 ? reinterpret_cast<unsigned*>(&S.gb[0][0])
                               : reinterpret_cast<unsigned*>(&S.Kn[0][0]);
      static_assert(VPL == 1 ? (int)sizeof(S.gb) >= 16 * MAXP : (int)sizeof(S.Kn) >= 16 * MAXP,
                    "RPE endpoint scratch");
#pragma unroll
      for (int k = 0; k < VPL; ++k) {
        const int pl = GW * k + lane;
        if (pl < np) reinterpret_cast<uint4*>(epw)[pl] = make_uint4(0u, 0u, 0u, 0u);
      }
      __syncwarp(FULL);
      unsigned long long* adj = reinterpret_cast<unsigned long long*>(S.KM);
      long long c2 = 0, cf = 0;
#pragma unroll
      for (int k = 0; k < VPL; ++k) {
        if (!((live[k] >> lane) & 1u)) continue;
        const int a = tri_at(mytri[k], 0), b = tri_at(mytri[k], 1), cc = tri_at(mytri[k], 2);
        const unsigned ma = eu_pm(a), mb = eu_pm(b), mc = eu_pm(cc);
        const long long pv2 = 2 * S.pay[EU_BIDX[ma | mb | mc]];
        const long long pab = S.pay[EU_BIDX[ma | mb]], pbc = S.pay[EU_BIDX[mb | mc]],
                        pca = S.pay[EU_BIDX[mc | ma]];
        c2 += pv2 - pab - pbc - pca;
        if (a >= 4) atomicAdd(reinterpret_cast<unsigned long long*>(acc + a),
                              (unsigned long long)(pv2 - pab - pca));
        if (b >= 4) atomicAdd(reinterpret_cast<unsigned long long*>(acc + b),
                              (unsigned long long)(pv2 - pab - pbc));
        if (cc >= 4) atomicAdd(reinterpret_cast<unsigned long long*>(acc + cc),
                               (unsigned long long)(pv2 - pbc - pca));
        // CC numbers: every plane pair of the triplet is an edge, so a radical facet has an
        // edge on each tet face of its vertices' triplets
        if (a >= 4 && (mb | mc)) atomicOr(S.dsc + a, mb | mc);
        if (b >= 4 && (ma | mc)) atomicOr(S.dsc + b, ma | mc);
        if (cc >= 4 && (ma | mb)) atomicOr(S.dsc + cc, ma | mb);
        // medial mesh: a plane pair of the triplet on two radical planes is a restricted power
        // edge RPE(m_i, m_j, m_k) (a triangle of the dual medial mesh)
        const int pr[3][3] = {{a, b, cc}, {b, cc, a}, {cc, a, b}};
#pragma unroll
        for (int r = 0; r < 3; ++r) {
          const int x = pr[r][0], y = pr[r][1], z = pr[r][2];
          if (x >= 4 && y >= 4) {
            const int rx = S.c0[x], ry = S.c0[y];
            if (rx < 64 && ry < 64) {
              atomicOr(adj + x, 1ull << ry);
              atomicOr(adj + y, 1ull << rx);
              if (z < 4) {  // this vertex is an endpoint of RPE (x, y) on tet face z
                const unsigned sx = atomicAdd(epw + 4 * x + z, 1u) & 0xffu;
                const unsigned sy = atomicAdd(epw + 4 * y + z, 1u) & 0xffu;
                if (sx < 2) atomicOr(epw + 4 * x + z, (unsigned)(ry + 1) << (8 * (1 + sx)));
                if (sy < 2) atomicOr(epw + 4 * y + z, (unsigned)(rx + 1) << (8 * (1 + sy)));
                if (sx >= 2 || sy >= 2) ++n_euover;  // (not with SoS: a line meets f once)
              }
            } else {
              ++n_euover;
            }
          }
        }
      }
      __syncwarp(FULL);
      unsigned* rw = out.rmask + mo;
      long long* rv = out.rval + 32 * (int64_t)mo;
      if (!one_word) {
        for (int w = lane; w < nwp; w += GW) rw[w] = 0u;
        __syncwarp(FULL);
      }
      unsigned rbits = 0u, sbits = 0u;
#pragma unroll
      for (int k = 0; k < VPL; ++k) {
        const int pl = GW * k + lane;
        if (pl < np && facets_all.has(pl)) {
          cf += S.pay[EU_BIDX[eu_pm(pl)]];
          sbits |= eu_pm(pl);
          if (pl >= 4) {  // radical facet: its part of the RPF between m_i and m_j
            const int pos = S.eidx[pl] - e0;
            rv[pos] = acc[pl] / 2 + S.pay[14];
            out.rfm[32 * (int64_t)mo + pos] = (uint8_t)S.dsc[pl];
            out.radj[32 * (int64_t)mo + pos] = adj[pl];
            out.rep[32 * (int64_t)mo + pos] = rep_of(epw, pl);
            if (one_word) rbits |= 1u << pos;
            else atomicOr(rw + (pos >> 5), 1u << (pos & 31));
          }
        }
      }
#pragma unroll
      for (int o = GW / 2; o > 0; o >>= 1) {
        c2 += __shfl_xor_sync(FULL, c2, o, GW);
        cf += __shfl_xor_sync(FULL, cf, o, GW);
      }
      if (one_word) {
        const unsigned w = __reduce_or_sync(FULL, rbits);
        if (lane == 0) rw[0] = w;
      }
      sbits = __reduce_or_sync(FULL, sbits);
      if (lane == 0) {
        out.eu_piece[p] = c2 / 2 + cf - S.pay[14];
        out.sfm[p] = (uint8_t)sbits;
      }
      __syncwarp(FULL);
    }

    // ---- geometry: vertex coordinates relative to V0 (lattice units); facet fan apex =
    // lowest vertex of the facet
#pragma unroll
    for (int k = 0; k < VPL; ++k) {
      const int v = GW * k + lane;
      if ((live[k] >> lane) & 1u) {
        double K[4];
#pragma unroll
        for (int m = 0; m < 4; ++m) K[m] = S.K[v][m];
        double sum = K[0] + K[1] + K[2] + K[3];
        // coordinates need |dx| <= 1.5e-11 diam(t): 15 F / sum <= 1.5e-11;
        // edge-interpolated vertices that miss it are rebuilt from their planes, then exactly
        if (16.0 * S.F[v] > 1e-12 * sum) {
          double F2, KM2;
          int dummy = 0;
          vertex_from_planes(S, C, tri_at(mytri[k], 0), tri_at(mytri[k], 1),
                             tri_at(mytri[k], 2), K, &F2, &KM2, &dummy);
          sum = K[0] + K[1] + K[2] + K[3];
          if (16.0 * F2 > 1e-12 * sum) {
            exact_vertex_of(S, C, tri_at(mytri[k], 0), tri_at(mytri[k], 1), tri_at(mytri[k], 2),
                            K);
            sum = K[0] + K[1] + K[2] + K[3];
            ++n_exact;
            ++d_out;
          }
        }
        const double inv = 1.0 / sum;
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          double acc = 0.0;
#pragma unroll
          for (int q = 1; q < 4; ++q) acc = fma(K[q] * inv, S.V[q][c] - S.V[0][c], acc);
          S.x[v][c] = acc;
        }
#pragma unroll
        for (int r = 0; r < 3; ++r) atomicMin(&S.ref[tri_at(mytri[k], r)], v);
      }
    }
    __syncwarp(FULL);
    double vol6 = 0.0, m24[3] = {0.0, 0.0, 0.0};
#pragma unroll
    for (int k = 0; k < VPL; ++k) {
      const int v = GW * k + lane;
      if ((live[k] >> lane) & 1u) {
        const double* xv = S.x[v];
#pragma unroll
        for (int r = 0; r < 3; ++r) {
          const int f = tri_at(mytri[k], r);
          const int w = S.nb[v][(r + 2) % 3];  // next vertex of facet f (edge (., f))
          const double* xr = S.x[S.ref[f]];
          const double* xw = S.x[w];
          const double det = xr[0] * (xv[1] * xw[2] - xv[2] * xw[1]) -
                             xr[1] * (xv[0] * xw[2] - xv[2] * xw[0]) +
                             xr[2] * (xv[0] * xw[1] - xv[1] * xw[0]);
          vol6 += det;
#pragma unroll
          for (int c = 0; c < 3; ++c) m24[c] += det * (xr[c] + xv[c] + xw[c]);
        }
      }
    }
#pragma unroll
    for (int o = GW / 2; o > 0; o >>= 1) {
      vol6 += __shfl_xor_sync(FULL, vol6, o, GW);
#pragma unroll
      for (int c = 0; c < 3; ++c) m24[c] += __shfl_xor_sync(FULL, m24[c], o, GW);
    }
    if (lane == 0) {
      const double L = 1.0 / RPD_LATTICE;
      const double vol = vol6 * (L * L * L / 6.0);
      out.vol[p] = vol;
#pragma unroll
      for (int c = 0; c < 3; ++c)
        out.m1[3 * p + c] = m24[c] * (L * L * L * L / 24.0) + vol * (S.V[0][c] * L);
      out.flag[p] = 1;
      out.fm[p] = (uint8_t)facemask;
    }
    __syncwarp(FULL);
    PHASE_MARK(5);
  }
#ifdef RPD_CLIP_PHASES
  if (lane == 0)
    for (int k = 0; k < 8; ++k) atomicAdd(&g_phase[k], (unsigned long long)ph[k]);
#endif
  // statistics: per-lane counters summed over the warp, group-uniform ones over the warp's
  // group leaders, then one global atomic per non-zero counter per block (block_stats)
  const bool lead = lane == 0;
  unsigned long long v[ST_N_CLIP] = {(unsigned long long)n_exact, (unsigned long long)n_zero,
                                     (unsigned long long)d_sign,  (unsigned long long)d_out,
                                     (unsigned long long)d_fb,    lead ? c_planes : 0u,
                                     lead ? c_tests : 0u,         lead ? c_constr : 0u,
                                     lead ? c_fan : 0u,
                                     lead && !out.over_list ? (unsigned long long)n_over : 0ull,
                                     (unsigned long long)n_euover,
                                     (unsigned long long)max_v,   (unsigned long long)max_p};
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
#pragma unroll
    for (int k = 0; k < 11; ++k) v[k] += __shfl_xor_sync(0xffffffffu, v[k], o);
#pragma unroll
    for (int k = 11; k < 13; ++k) v[k] = max(v[k], __shfl_xor_sync(0xffffffffu, v[k], o));
  }
  const int slot[ST_N_CLIP] = {ST_EXACT,    ST_ZERO,        12,            13,
                               14,          ST_CLIP_PLANES, ST_CLIP_TESTS, ST_CLIP_CONSTR,
                               ST_CLIP_FAN, ST_OVERFLOW,    ST_EU_OVER,    ST_MAXV,
                               ST_MAXP};
  const int kind[ST_N_CLIP] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 1, 1};
  block_stats<ST_N_CLIP>(stats, slot, kind, v);
}

// incidences per pair (0 for empty pairs)
__global__ void k_count_inc(int64_t n_pairs, const uint8_t* __restrict__ flag,
                            const int32_t* __restrict__ mask_off,
                            const unsigned* __restrict__ mask, int32_t* __restrict__ ninc,
                            int32_t* __restrict__ f01, const unsigned* __restrict__ rmask,
                            int32_t* __restrict__ nrpf, const int* __restrict__ n_dev) {
  if (n_dev) n_pairs = *n_dev;
  int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (p >= n_pairs) return;
  int n = 0, r = 0;
  const bool ne = flag[p] == 1;
  if (ne)
    for (int w = mask_off[p]; w < mask_off[p + 1]; ++w) {
      n += __popc(mask[w]);
      if (rmask) r += __popc(rmask[w]);
    }
  ninc[p] = n;
  f01[p] = ne;
  if (rmask) nrpf[p] = r;
}

struct EuCompact {
  const unsigned* rmask;     // nullptr: Euler off
  const long long* rval;
  const long long* p_eu;
  const int32_t* rscan;
  long long* piece;
  int32_t *rpf_off, *rpf_j;
  long long* rpf_e;
  const uint8_t *p_sfm, *p_rfm;  // CC flags (per pair, per pair slot)
  uint8_t *sfm, *rfm;            // ... compacted (per piece, per radical facet)
  const unsigned long long* p_radj;  // radical-facet adjacency (per pair slot)
  unsigned long long* radj;          // ... compacted (per radical facet)
  const unsigned long long* p_rep;   // RPE endpoint faces (per pair slot)
  unsigned long long* rep;           // ... compacted (per radical facet)
  int32_t inc_base, rpf_base;        // value offsets of inc_off / rpf_off (pool append)
};

__global__ void k_compact_pieces(int64_t n_pairs, const int32_t* __restrict__ cand_idx,
                                 const int32_t* __restrict__ nbr_off,
                                 const int32_t* __restrict__ nbr_idx,
                                 const uint8_t* __restrict__ flag, const int32_t* __restrict__ pscan,
                                 const int32_t* __restrict__ iscan, const double* __restrict__ pvol,
                                 const double* __restrict__ pm1, const uint8_t* __restrict__ pfm,
                                 const int32_t* __restrict__ mask_off,
                                 const unsigned* __restrict__ mask,
                                 int32_t* __restrict__ piece_sphere, double* __restrict__ piece_vol,
                                 double* __restrict__ piece_m1, uint8_t* __restrict__ piece_fm,
                                 int32_t* __restrict__ inc_off, int32_t* __restrict__ inc_sphere,
                                 EuCompact eu, const PDyn* __restrict__ pd,
                                 const int32_t* __restrict__ cand_off,
                                 int32_t* __restrict__ piece_off) {
  if (pd) {  // (graph: the batch's per-tet piece offsets too -- k_piece_off of the eager path)
    const int64_t nt = pd->nb;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t <= nt;
         t += (int64_t)gridDim.x * blockDim.x)
      piece_off[t] = pscan[cand_off[t]];
  }
  if (pd) {  // device-driven update: the batch size and the pool tails from the device
    n_pairs = pd->nc;
    cand_idx += pd->fill_c;
    piece_sphere += pd->fill_p;
    piece_vol += pd->fill_p;
    piece_m1 += 3 * (int64_t)pd->fill_p;
    piece_fm += pd->fill_p;
    inc_off += pd->fill_p;
    inc_sphere += pd->fill_i;
    eu.inc_base = pd->fill_i;
    if (n_pairs == 0 && blockIdx.x == 0 && threadIdx.x == 0) inc_off[0] = eu.inc_base;
  }
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < n_pairs; p += stride) {
  if (p == n_pairs - 1) {
    inc_off[pscan[n_pairs]] = eu.inc_base + iscan[n_pairs];
    if (eu.rmask) eu.rpf_off[pscan[n_pairs]] = eu.rpf_base + eu.rscan[n_pairs];
  }
  if (flag[p] != 1) continue;
  const int q = pscan[p];
  const int i = cand_idx[p];
  piece_sphere[q] = i;
  piece_vol[q] = pvol[p];
  piece_m1[3 * q + 0] = pm1[3 * p + 0];
  piece_m1[3 * q + 1] = pm1[3 * p + 1];
  piece_m1[3 * q + 2] = pm1[3 * p + 2];
  piece_fm[q] = pfm[p];
  int o = iscan[p];
  inc_off[q] = eu.inc_base + o;
  const int e0 = nbr_off[i];
  const int w0 = mask_off[p];
  for (int w = w0; w < mask_off[p + 1]; ++w) {
    unsigned m = mask[w];
    while (m) {
      int b = __ffs(m) - 1;
      m &= m - 1;
      inc_sphere[o++] = nbr_idx[e0 + 32 * (w - w0) + b];
    }
  }
  if (eu.rmask) {  // Euler: the piece's value and its radical facets, ascending neighbour id
    eu.piece[q] = eu.p_eu[p];
    eu.sfm[q] = eu.p_sfm[p];
    int r = eu.rscan[p];
    eu.rpf_off[q] = eu.rpf_base + r;
    for (int w = w0; w < mask_off[p + 1]; ++w) {
      unsigned m = eu.rmask[w];
      while (m) {
        const int b = __ffs(m) - 1;
        m &= m - 1;
        const int pos = 32 * (w - w0) + b;
        eu.rpf_j[r] = nbr_idx[e0 + pos];
        eu.rpf_e[r] = eu.rval[32 * (int64_t)w0 + pos];
        eu.rfm[r] = eu.p_rfm[32 * (int64_t)w0 + pos];
        eu.radj[r] = eu.p_radj[32 * (int64_t)w0 + pos];
        eu.rep[r] = eu.p_rep[32 * (int64_t)w0 + pos];
        ++r;
      }
    }
  }
  }
}

__global__ void k_piece_off(int64_t T, const int32_t* __restrict__ cand_off,
                            const int32_t* __restrict__ pscan, int32_t* __restrict__ piece_off,
                            const int* __restrict__ n_dev) {
  if (n_dev) T = *n_dev;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t <= T; t += stride)
    piece_off[t] = pscan[cand_off[t]];
}

static inline unsigned nblk(int64_t n, int b) { return (unsigned)((n + b - 1) / b); }

void clip_phase_dump() {
#ifdef RPD_CLIP_PHASES
  unsigned long long h[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  cudaMemcpyFromSymbol(h, g_phase, sizeof(h));
  const unsigned long long z[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  cudaMemcpyToSymbol(g_phase, z, sizeof(z));
  double tot = 0;
  for (int k = 0; k < 6; ++k) tot += (double)h[k];
  const char* nm[6] = {"setup", "classify", "sign", "cut", "facets+inc", "geometry+store"};
  fprintf(stderr, "[rpd clip phases] group-cycles");
  for (int k = 0; k < 6; ++k) fprintf(stderr, "  %s %.1f%%", nm[k], 100.0 * h[k] / (tot > 0 ? tot : 1));
  fprintf(stderr, "  total %.3e  sign-passes %llu cuts %llu\n", tot, h[6], h[7]);
#endif
}

template <int GW, int VPL, bool EU>
static cudaError_t launch_clip_t(rpd_ctx* c, int64_t n, const int32_t* pair_list,
                                 const int32_t* pair_tet, const int32_t* tet_ids,
                                 const int32_t* cand_idx, const int32_t* moff,
                                 const unsigned* cut, int32_t* over, const int32_t* n_dev,
                                 int* dyn = nullptr, int64_t grid_cap = 0) {
  constexpr int THREADS = VPL == 1 && GW == RPD_CLIP_GW ? RPD_CLIP_THREADS
                         : (VPL <= 2 ? 256 : (VPL <= 4 ? 64 : 32));
  constexpr int GROUPS = THREADS / GW;  // pairs in flight per block
  size_t smem = sizeof(WarpState<GW, VPL>) * GROUPS;
  // kernel attributes are per device: set / queried once per (instantiation, device) (host API
  // calls cost microseconds per launch); the table is guarded for ctxs on several threads
  static int occ_dev[RPD_MAX_DEVICES] = {};
  static std::mutex mu;
  if (c->device < 0 || c->device >= RPD_MAX_DEVICES) return cudaErrorInvalidDevice;
  int occ;
  {
    std::lock_guard<std::mutex> g(mu);
    occ = occ_dev[c->device];
    if (occ == 0) {
      cudaError_t e = cudaFuncSetAttribute(k_clip<GW, VPL, EU>,
                                           cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      if (e) return e;
      int o = 1;
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, k_clip<GW, VPL, EU>, THREADS, smem);
      occ = occ_dev[c->device] = o < 1 ? 1 : o;
    }
  }
  const int sms = c->sms;
  int64_t want = (n + GROUPS - 1) / GROUPS;
  int64_t grid = (int64_t)sms * occ;
  if (want < grid) grid = want;
  // the 128- and 256-slot tiers over an overflow list (a handful of pairs, often none; the
  // count is read on the device): one block per SM, so an empty launch costs little
  if (pair_list && VPL >= 4 && grid > sms) grid = sms;
  if (grid_cap > 0 && grid > grid_cap) grid = grid_cap;
  if (grid < 1) grid = 1;
  PairOut o{c->p_vol.as<double>(),   c->p_m1.as<double>(),    c->p_flag.as<uint8_t>(),
            c->p_fm.as<uint8_t>(),   c->p_mask.as<unsigned>(), moff, cut,
            over ? over + 1 : nullptr, over,
            c->euler ? c->eu_rec.as<uint4>() : nullptr, c->eu_Lt.as<long long>(),
            c->p_eu.as<long long>(), c->p_rmask.as<unsigned>(), c->p_rval.as<long long>(),
            c->p_sfm.as<uint8_t>(), c->p_rfm.as<uint8_t>(),
            c->p_radj.as<unsigned long long>(), c->p_rep.as<unsigned long long>()};
  k_clip<GW, VPL, EU><<<(unsigned)grid, THREADS, smem, c->stream>>>(
      n, pair_list, pair_tet, tet_ids, cand_idx, c->st.tx.as<double>(), c->st.T,
      c->st.nbr_off.as<int32_t>(), c->st.nbr_idx.as<int32_t>(), c->st.planes.as<double4>(),
      c->st.twin.as<int32_t>(), (long long)c->st.N, o, c->stats.as<unsigned long long>(),
      n_dev, dyn, c->pdd);
  ++c->launches;
  return cudaGetLastError();
}

// fast kernel over all pairs (overflowing pairs are listed in p_over[1..], count p_over[0]),
// or the widest kernel over all pairs when `wide`
template <bool EU>
static cudaError_t launch_clip_eu(rpd_ctx* c, int64_t n_pairs, const int32_t* pair_tet,
                                  const int32_t* tet_ids, const int32_t* cand_idx,
                                  const int32_t* moff, const unsigned* cut, int wide) {
  if (wide)
    return launch_clip_t<32, 4, EU>(c, n_pairs, nullptr, pair_tet, tet_ids, cand_idx, moff, cut,
                                    c->p_over3.as<int32_t>(), nullptr);
  cudaError_t e = c->p_dyn.ensure(sizeof(int));
  if (e) return e;
  if ((e = cudaMemsetAsync(c->p_dyn.p, 0, sizeof(int), c->stream))) return e;
  return launch_clip_t<RPD_CLIP_GW, RPD_CLIP_VPL, EU>(c, n_pairs, nullptr, pair_tet, tet_ids,
                                                      cand_idx, moff, cut, c->p_over.as<int32_t>(),
                                                      nullptr, c->p_dyn.as<int>());
}

// graph path: the fast tier's pairs split by their number of cut planes (cut-mask bits within
// the row): more than `thresh` -> the big list (clipped by the 64-slot tier concurrently with
// the fast tier), else the small list (warp-aggregated appends; order is irrelevant)
__global__ void k_pair_route(const PDyn* __restrict__ pd, const int32_t* __restrict__ moff,
                             const unsigned* __restrict__ cut, const int32_t* __restrict__ cand_idx,
                             const int32_t* __restrict__ nbr_off, int thresh,
                             int32_t* __restrict__ route) {
  const int n = pd->nc_fast;
  cand_idx += pd->fill_c;
  int* n_small = route;
  int* n_big = route + 1;
  int32_t* small_list = route + 2;
  int32_t* big_list = small_list + pd->nc_max;
  const int lane = threadIdx.x & 31;
  for (int64_t p0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) - lane; p0 < n;
       p0 += (int64_t)gridDim.x * blockDim.x) {
    const int64_t p = p0 + lane;
    bool big = false;
    if (p < n) {
      const int i = cand_idx[p];
      const int kp = nbr_off[i + 1] - nbr_off[i];
      int pc = 0;
      for (int w = moff[p], q = 0; w < moff[p + 1]; ++w, ++q) {
        unsigned m = cut[w];
        if (kp - 32 * q < 32) m &= (1u << (kp - 32 * q)) - 1u;
        pc += __popc(m);
      }
      big = pc > thresh;
    }
    const unsigned bm = __ballot_sync(0xffffffffu, big && p < n);
    const unsigned sm = __ballot_sync(0xffffffffu, !big && p < n);
    int bb = 0, sb = 0;
    if (lane == 0) {
      if (bm) bb = atomicAdd(n_big, __popc(bm));
      if (sm) sb = atomicAdd(n_small, __popc(sm));
    }
    bb = __shfl_sync(0xffffffffu, bb, 0);
    sb = __shfl_sync(0xffffffffu, sb, 0);
    if (p < n) {
      if (big) big_list[bb + __popc(bm & ((1u << lane) - 1u))] = (int32_t)p;
      else small_list[sb + __popc(sm & ((1u << lane) - 1u))] = (int32_t)p;
    }
  }
}

// fast kernel over all pairs (overflowing pairs are listed in p_over[1..], count p_over[0]),
// or the widest kernel over all pairs when `wide`
cudaError_t launch_clip(rpd_ctx* c, int64_t n_pairs, const int32_t* pair_tet,
                        const int32_t* tet_ids, const int32_t* cand_idx, const int32_t* moff,
                        const unsigned* cut, int wide) {
  c->clip_small = 0;
  if (n_pairs == 0) return cudaSuccess;
  if (c->pdd) {
    // device-driven update: n_pairs is the grids' bound; the count is read on the device by
    // both entry tiers, and only the one the eager path would choose gets it (nc_fast /
    // nc_small, the other sees 0).  The fast tier's overflows go down the usual cascade.
    // (the pair counter p_dyn is zeroed by k_pd_init)
    cudaError_t e;
    if (c->clip_route > 0) {
      // the pairs with many cut planes (the fast tier's likely overflows) clipped by the
      // 64-slot tier in a concurrent branch of the graph, the others by the fast tier
      int32_t* route = c->p_route.as<int32_t>();
      const int32_t* small_list = route + 2;
      const int32_t* big_list = small_list + c->pdd_nc_max;
      k_pair_route<<<(unsigned)(c->sms * 4), 256, 0, c->stream>>>(
          c->pdd, moff, cut, cand_idx, c->st.nbr_off.as<int32_t>(), c->clip_route, route);
      ++c->launches;
      if ((e = cudaEventRecord(c->g_fork, c->stream))) return e;
      if ((e = cudaStreamWaitEvent(c->side_stream, c->g_fork, 0))) return e;
      cudaStream_t main = c->stream;
      c->stream = c->side_stream;
      e = launch_clip_t<32, RPD_CLIP_MID_VPL, false>(c, n_pairs, big_list, pair_tet, tet_ids,
                                                     cand_idx, moff, cut, c->p_over2.as<int32_t>(),
                                                     route + 1, nullptr, c->sms);
      c->stream = main;
      if (e) return e;
      if ((e = cudaEventRecord(c->g_join, c->side_stream))) return e;
      e = launch_clip_t<RPD_CLIP_GW, RPD_CLIP_VPL, false>(c, n_pairs, small_list, pair_tet,
                                                         tet_ids, cand_idx, moff, cut,
                                                         c->p_over.as<int32_t>(), route,
                                                         c->p_dyn.as<int>());
      if (e) return e;
      if ((e = cudaStreamWaitEvent(c->stream, c->g_join, 0))) return e;
    } else {
      e = launch_clip_t<RPD_CLIP_GW, RPD_CLIP_VPL, false>(c, n_pairs, nullptr, pair_tet, tet_ids,
                                                         cand_idx, moff, cut,
                                                         c->p_over.as<int32_t>(),
                                                         &c->pdd->nc_fast, c->p_dyn.as<int>());
    }
    if (e) return e;
    return launch_clip_t<32, RPD_CLIP_MID_VPL, false>(c, n_pairs < RPD_CLIP_SMALL ? n_pairs : RPD_CLIP_SMALL,
                                                      nullptr, pair_tet, tet_ids, cand_idx, moff,
                                                      cut, c->p_over2.as<int32_t>(),
                                                      &c->pdd->nc_small);
  }
  if (!wide && n_pairs < RPD_CLIP_SMALL && !c->clip_tiers) {
    // few pairs (small partial updates): latency, not throughput -- one pass of the 64-slot
    // tier over every pair instead of the fast tier plus a re-run of its overflows
    c->clip_small = 1;
    return c->euler
               ? launch_clip_t<32, RPD_CLIP_MID_VPL, true>(c, n_pairs, nullptr, pair_tet, tet_ids,
                                                           cand_idx, moff, cut,
                                                           c->p_over2.as<int32_t>(), nullptr)
               : launch_clip_t<32, RPD_CLIP_MID_VPL, false>(c, n_pairs, nullptr, pair_tet,
                                                            tet_ids, cand_idx, moff, cut,
                                                            c->p_over2.as<int32_t>(), nullptr);
  }
  return c->euler ? launch_clip_eu<true>(c, n_pairs, pair_tet, tet_ids, cand_idx, moff, cut, wide)
                  : launch_clip_eu<false>(c, n_pairs, pair_tet, tet_ids, cand_idx, moff, cut, wide);
}

// the overflow list p_over[1 .. p_over[0]] (count read on the device) is re-run by the
// 64-slot kernel <32, RPD_CLIP_MID_VPL = 2>; its own overflows (p_over2) by the 128-slot <32, 4>
// the slow path: the 128-slot tier's overflows (list p_over3) re-run with 256 vertex / plane
// slots (one 32-lane group per block, ~45 KB of shared memory); beyond that the clip fails
// with RPD_EOVERFLOW (8-bit vertex and plane ids)
template <bool EU>
static cudaError_t launch_slow(rpd_ctx* c, const int32_t* pair_tet, const int32_t* tet_ids,
                               const int32_t* cand_idx, const int32_t* moff,
                               const unsigned* cut) {
  return launch_clip_t<32, 8, EU>(c, 1 << 30, c->p_over3.as<int32_t>() + 1, pair_tet, tet_ids,
                                  cand_idx, moff, cut, nullptr, c->p_over3.as<int32_t>());
}

template <bool EU>
static cudaError_t launch_overflow_eu(rpd_ctx* c, const int32_t* pair_tet, const int32_t* tet_ids,
                                      const int32_t* cand_idx, const int32_t* moff,
                                      const unsigned* cut) {
  cudaError_t e;
#if RPD_CLIP_MID32
  // 32-slot tier (one slot per lane: the fast tier's program on a full warp) for the fast
  // tier's overflows; its own overflows go on to the 64-slot tier
  e = launch_clip_t<32, 1, EU>(c, 1 << 30, c->p_over.as<int32_t>() + 1, pair_tet, tet_ids,
                               cand_idx, moff, cut, c->p_over3.as<int32_t>(), c->p_over.as<int32_t>());
  if (e) return e;
  e = launch_clip_t<32, RPD_CLIP_MID_VPL, EU>(
      c, 1 << 30, c->p_over3.as<int32_t>() + 1, pair_tet, tet_ids, cand_idx, moff, cut,
      c->p_over2.as<int32_t>(), c->p_over3.as<int32_t>());
#else
  e = launch_clip_t<32, RPD_CLIP_MID_VPL, EU>(
      c, 1 << 30, c->p_over.as<int32_t>() + 1, pair_tet, tet_ids, cand_idx, moff, cut,
      c->p_over2.as<int32_t>(), c->p_over.as<int32_t>());
#endif
  if (e) return e;
  e = launch_clip_t<32, 4, EU>(c, 1 << 30, c->p_over2.as<int32_t>() + 1, pair_tet, tet_ids,
                               cand_idx, moff, cut, c->p_over3.as<int32_t>(),
                               c->p_over2.as<int32_t>());
  if (e) return e;
  return launch_slow<EU>(c, pair_tet, tet_ids, cand_idx, moff, cut);
}

cudaError_t launch_clip_overflow(rpd_ctx* c, const int32_t* pair_tet, const int32_t* tet_ids,
                                 const int32_t* cand_idx, const int32_t* moff,
                                 const unsigned* cut) {
  if (c->clip_small) {  // only the 64-slot tier's overflows remain: 128 slots, then 256
    cudaError_t e =
        c->euler ? launch_clip_t<32, 4, true>(c, 1 << 30, c->p_over2.as<int32_t>() + 1,
                                              pair_tet, tet_ids, cand_idx, moff, cut,
                                              c->p_over3.as<int32_t>(), c->p_over2.as<int32_t>())
                 : launch_clip_t<32, 4, false>(c, 1 << 30, c->p_over2.as<int32_t>() + 1,
                                               pair_tet, tet_ids, cand_idx, moff, cut,
                                               c->p_over3.as<int32_t>(), c->p_over2.as<int32_t>());
    if (e) return e;
    return c->euler ? launch_slow<true>(c, pair_tet, tet_ids, cand_idx, moff, cut)
                    : launch_slow<false>(c, pair_tet, tet_ids, cand_idx, moff, cut);
  }
  if (c->clip_wide)  // the 128-slot tier ran on every pair: its overflows
    return c->euler ? launch_slow<true>(c, pair_tet, tet_ids, cand_idx, moff, cut)
                    : launch_slow<false>(c, pair_tet, tet_ids, cand_idx, moff, cut);
  return c->euler ? launch_overflow_eu<true>(c, pair_tet, tet_ids, cand_idx, moff, cut)
                  : launch_overflow_eu<false>(c, pair_tet, tet_ids, cand_idx, moff, cut);
}

// (device-driven update: n_pairs is the bound, the count is pd->nc)
cudaError_t launch_piece_scans(rpd_ctx* c, int64_t n_pairs, const int32_t* moff) {
  const int* n_dev = c->pdd ? &c->pdd->nc : nullptr;
  if (n_pairs > 0) {
    k_count_inc<<<nblk(n_pairs, 256), 256, 0, c->stream>>>(
        n_pairs, c->p_flag.as<uint8_t>(), moff, c->p_mask.as<unsigned>(),
        c->p_ninc.as<int32_t>(), c->p_f01.as<int32_t>(),
        c->euler ? c->p_rmask.as<unsigned>() : nullptr, c->p_nrpf.as<int32_t>(), n_dev);
    ++c->launches;
  }
  const int32_t* in[3] = {c->p_f01.as<int32_t>(), c->p_ninc.as<int32_t>(), c->p_nrpf.as<int32_t>()};
  int32_t* out[3] = {c->p_scan.as<int32_t>(), c->i_scan.as<int32_t>(), c->r_scan.as<int32_t>()};
  return launch_scan_i32_multi(c, in, out, c->euler ? 3 : 2, n_pairs, n_dev);
}

cudaError_t launch_compact_pieces(rpd_ctx* c, int64_t n_tets, int64_t n_pairs,
                                  const int32_t* cand_off, const int32_t* cand_idx,
                                  const int32_t* moff, const PieceDst& d) {
  const PDyn* pd = c->pdd;  // device-driven update: bounds here, counts / pool tails in pd
  if (n_pairs > 0 || pd) {
    unsigned grid = nblk(n_pairs > 0 ? n_pairs : 1, 256);
    if (pd && grid > (unsigned)c->sms * 4) grid = c->sms * 4;  // (grid-stride over the bound)
    k_compact_pieces<<<grid, 256, 0, c->stream>>>(
        n_pairs, cand_idx, c->st.nbr_off.as<int32_t>(), c->st.nbr_idx.as<int32_t>(),
        c->p_flag.as<uint8_t>(), c->p_scan.as<int32_t>(), c->i_scan.as<int32_t>(),
        c->p_vol.as<double>(), c->p_m1.as<double>(), c->p_fm.as<uint8_t>(),
        moff, c->p_mask.as<unsigned>(), d.sphere, d.vol, d.m1, d.fm,
        d.inc_off, d.inc,
        EuCompact{c->euler ? c->p_rmask.as<unsigned>() : nullptr, c->p_rval.as<long long>(),
                  c->p_eu.as<long long>(), c->r_scan.as<int32_t>(), d.eu, d.rpf_off, d.rpf_j,
                  d.rpf_e, c->p_sfm.as<uint8_t>(), c->p_rfm.as<uint8_t>(), d.sfm, d.rfm,
                  c->p_radj.as<unsigned long long>(), d.radj, c->p_rep.as<unsigned long long>(),
                  d.rep, d.inc_base, d.rpf_base}, pd, cand_off, d.off);
    ++c->launches;
    if (pd) return cudaGetLastError();
  } else {
    // the terminal offsets of an empty batch (the pool's current fill levels)
    cudaMemcpyAsync(d.inc_off, &d.inc_base, sizeof(int32_t), cudaMemcpyHostToDevice, c->stream);
    if (c->euler)
      cudaMemcpyAsync(d.rpf_off, &d.rpf_base, sizeof(int32_t), cudaMemcpyHostToDevice, c->stream);
  }
  unsigned g2 = nblk(n_tets + 1, 256);
  if (pd && g2 > (unsigned)c->sms * 2) g2 = c->sms * 2;
  k_piece_off<<<g2, 256, 0, c->stream>>>(n_tets, cand_off, c->p_scan.as<int32_t>(), d.off,
                                         pd ? &pd->nb : nullptr);
  ++c->launches;
  return cudaGetLastError();
}

}  // namespace rpd
