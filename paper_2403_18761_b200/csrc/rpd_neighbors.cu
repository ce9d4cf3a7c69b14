// rpd_neighbors.cu -- SURVEY.md §8(f) NEXT-3: the sphere neighbour lists (k_site) on the GPU,
// the step right before the RPD (the 'Security Radius' criterion "is not
// sufficient anymore", so "we use the Regular Triangulation in CGAL to compute all possible
// neighbors (k_site) of a given sphere").  Instead of a regular triangulation we compute a *certified superset* of the
// neighbours whose power cell facets meet the domain box B (DESIGN.md §10 "Sphere
// neighbours"): every sphere j whose radical plane holds a positive-area facet of C_i ∩ B is
// listed.  The RPD restricted to tets inside B is unchanged by redundant planes (SURVEY §8(c)
// C0: "supersets are harmless"), so the pieces equal those of the regular-triangulation lists.
//
// Per sphere i (one warp), in coordinates y = x - theta_i:
//   1. K = the KSEL spheres of smallest power distance PD_j(theta_i) found in the grid rings
//      around i (a heuristic choice: correctness does not depend on it);
//   2. P_K = B ∩ ⋂_{k∈K} {h_ik >= 0} ⊇ C_i ∩ B; its vertices by a sequential clip of B's
//      corners, one plane at a time (triples only from the plane pairs tight at a vertex the
//      plane may remove; or, RPD_NB_SEQ=0, by enumeration of all plane triples), in fp64,
//      each vertex with an error radius e_v from its conditioning, kept when every half-space
//      holds within e_v + tol0 (so no true vertex is lost); refined over rounds by the planes
//      that cut it deepest;
//   3. j is listed iff h_ij(v) <= e_v + tol0 at some vertex v of P_K (convexity: if h_ij > 0 at
//      every vertex, the plane misses P_K ⊇ C_i ∩ B); only spheres in the ball
//      |theta_j - theta_i| <= rho + sqrt(PDmax + rmax^2) (+ margins) can pass, found through
//      the uniform grid.
// Special cases: a sphere with the same centre and a larger radius (or the same radius and a
// smaller id) hides i (empty row); a non-empty P_K with no cutting plane and N > 1 (i's cell
// covers B) lists its nearest sphere, a redundant plane, so that R4 (k_site = 0 -> no
// relation) does not apply.  If the vertex list overflows, P_K is replaced by B (conservative).
//
// Passes: bounds (centre box, r_max) -> grid counting sort -> pass 1 (count, rows <= CAP1 kept)
// -> scan -> pass 2 (recompute rows > CAP1) -> per-row rank sort into ascending CSR.
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>

#include "rpd_ctx.h"

namespace rpd {
namespace {

#ifndef RPD_NB_KSEL0
#define RPD_NB_KSEL0 56
#endif
constexpr int NB_KSEL0 = RPD_NB_KSEL0;    // planes of the first P_K besides the 6 box planes
#ifndef RPD_NB_KSEL
#define RPD_NB_KSEL 64
#endif
constexpr int NB_KSEL = RPD_NB_KSEL;      // planes of a refined P_K (facets + deepest cuts), <= 64
constexpr int NB_MAXP = 6 + NB_KSEL;      // (< 128: the tight-plane masks below)
constexpr int NB_MAXV = NB_KSEL > 48 ? 200 : 224;  // vertex candidates of P_K per sphere
constexpr int NB_CAPC = 128;              // selection candidates: 4 per lane
constexpr int NB_CAP1 = 256;              // row entries kept by pass 1
constexpr int NB_WARPS = 4;               // warps per block of the main kernel
#ifndef RPD_NB_BT
#define RPD_NB_BT 256
#endif
constexpr int NB_BT = RPD_NB_BT;          // threads per sphere of the heavy-row kernel (A/B knob)
constexpr int NB_GMAX = 160;              // grid cells per axis (max)
constexpr int NB_RB = 256;                // radius buckets of the work order
constexpr int NB_ROUNDS = 6;              // polytope refinements (the last one lists)
#ifndef RPD_NB_HCAP
#define RPD_NB_HCAP 16384
#endif
constexpr int NB_HCAP = RPD_NB_HCAP;      // hit list of a round (per warp slot, global memory)

struct NbGrid {
  double lo[3], h[3];
  double rmax;
  int G;
};

struct NbSmem {
  int cid[NB_CAPC];
  double key[NB_CAPC];
  double4 pl[NB_MAXP];        // unit normal a, offset b: a.y + b >= 0 inside
  double4 vx[NB_MAXV];        // y, error radius
  int out[NB_CAP1];
  int kid[NB_KSEL];
  int n_v, n_o, flags, first, n_pair;
};

// per-lane smallest NB_TOPL keys (ties: smaller id), kept sorted; deterministic because every
// lane visits its cells and their (id-sorted) spheres in a fixed order
struct LaneTop {
  double k[4];
  int j[4];
  __device__ void init() {
    for (int t = 0; t < 4; ++t) {
      k[t] = 1e300;
      j[t] = -1;
    }
  }
  __device__ void push(double key, int id) {
    if (!(key < k[3] || (key == k[3] && id < j[3]))) return;
    int t = 3;
    while (t > 0 && (key < k[t - 1] || (key == k[t - 1] && id < j[t - 1]))) {
      k[t] = k[t - 1];
      j[t] = j[t - 1];
      --t;
    }
    k[t] = key;
    j[t] = id;
  }
};

__device__ __forceinline__ double warp_max(double v) {
  for (int o = 16; o; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

__global__ void k_nb_bounds(const double* __restrict__ sph, int64_t N, int G, NbGrid* g) {
  __shared__ double s[6][32];
  double mn[3] = {1e300, 1e300, 1e300}, mx[3] = {-1e300, -1e300, -1e300}, rm = 0.0;
  for (int64_t i = threadIdx.x; i < N; i += blockDim.x) {
    for (int k = 0; k < 3; ++k) {
      const double c = sph[4 * i + k];
      mn[k] = fmin(mn[k], c);
      mx[k] = fmax(mx[k], c);
    }
    rm = fmax(rm, sph[4 * i + 3]);
  }
  double v[7] = {-mn[0], -mn[1], -mn[2], mx[0], mx[1], mx[2], rm};
  for (int k = 0; k < 7; ++k) v[k] = warp_max(v[k]);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31, nw = blockDim.x >> 5;
  __shared__ double s7[32];
  if (l == 0) {
    for (int k = 0; k < 6; ++k) s[k][w] = v[k];
    s7[w] = v[6];
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double r[7] = {-1e300, -1e300, -1e300, -1e300, -1e300, -1e300, 0.0};
    for (int q = 0; q < nw; ++q) {
      for (int k = 0; k < 6; ++k) r[k] = fmax(r[k], s[k][q]);
      r[6] = fmax(r[6], s7[q]);
    }
    for (int k = 0; k < 3; ++k) {
      const double lo = -r[k], hi = r[3 + k];
      const double ext = hi - lo;
      g->lo[k] = lo;
      g->h[k] = ext > 0 ? ext * (1.0 + 1e-12) / G : 1.0;
    }
    g->rmax = r[6];
    g->G = G;
  }
}

// NaN / Inf coordinates or a negative radius -> RPD_EINVAL (error word, first offender)
__global__ void k_nb_check(const double* __restrict__ sph, int64_t N, int* __restrict__ err) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < N;
       i += (int64_t)gridDim.x * blockDim.x) {
    const double x = sph[4 * i], y = sph[4 * i + 1], z = sph[4 * i + 2], r = sph[4 * i + 3];
    const bool bad_nan = !isfinite(x) || !isfinite(y) || !isfinite(z) || !isfinite(r);
    if (bad_nan || r < 0) {
      if (atomicCAS(&err[0], 0, (int)RPD_EINVAL) == 0) {
        err[1] = bad_nan ? ERR_SPHERE_NAN : ERR_RADIUS_NEG;
        err[2] = (int)i;
      }
    }
  }
}

__device__ __forceinline__ int nb_cell_axis(double c, const NbGrid& g, int k) {
  int q = (int)floor((c - g.lo[k]) / g.h[k]);
  return q < 0 ? 0 : (q >= g.G ? g.G - 1 : q);
}

__global__ void k_nb_count(const double* __restrict__ sph, int64_t N, const NbGrid* __restrict__ gp,
                           int32_t* __restrict__ cnt, int32_t* __restrict__ cell_of) {
  const NbGrid g = *gp;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < N;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int cx = nb_cell_axis(sph[4 * i], g, 0), cy = nb_cell_axis(sph[4 * i + 1], g, 1),
              cz = nb_cell_axis(sph[4 * i + 2], g, 2);
    const int c = (cz * g.G + cy) * g.G + cx;
    cell_of[i] = c;
    atomicAdd(&cnt[c], 1);
  }
}

__global__ void k_nb_scatter(int64_t N, const int32_t* __restrict__ cell_of,
                             const int32_t* __restrict__ start, int32_t* __restrict__ fill,
                             int32_t* __restrict__ items) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < N;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int c = cell_of[i];
    items[start[c] + atomicAdd(&fill[c], 1)] = (int)i;
  }
}

// deterministic cell contents: insertion sort of each (small) cell by sphere id
__global__ void k_nb_cellsort(int64_t n_cells, const int32_t* __restrict__ start,
                              int32_t* __restrict__ items) {
  for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < n_cells;
       c += (int64_t)gridDim.x * blockDim.x) {
    const int a = start[c], b = start[c + 1];
    for (int p = a + 1; p < b; ++p) {
      const int v = items[p];
      int q = p - 1;
      while (q >= a && items[q] > v) {
        items[q + 1] = items[q];
        --q;
      }
      items[q + 1] = v;
    }
  }
}

__global__ void k_nb_gather(int64_t N, const int32_t* __restrict__ items,
                            const double* __restrict__ sph, double4* __restrict__ sorted) {
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < N;
       p += (int64_t)gridDim.x * blockDim.x) {
    const int j = items[p];
    sorted[p] = make_double4(sph[4 * j], sph[4 * j + 1], sph[4 * j + 2], sph[4 * j + 3]);
  }
}

// work order: spheres by descending radius (the big spheres have the big cells and the long
// scans), taken from a counter, so that the longest rows start first
// work order: descending radius (the big spheres have the big cells and the long scans; the
// near-zero ones are heavy too, but moving them first or going ascending measured no better:
// DESIGN.md "Sphere neighbours")
#ifndef RPD_NB_TINY_FIRST
#define RPD_NB_TINY_FIRST 0  // the smallest radius bucket first, then descending (A/B knob)
#endif
__device__ __forceinline__ int nb_rbucket(double r, double rmax) {
  int b = rmax > 0 ? (int)((1.0 - r / rmax) * NB_RB) : 0;
  b = b < 0 ? 0 : (b >= NB_RB ? NB_RB - 1 : b);
  if (RPD_NB_TINY_FIRST) b = b == NB_RB - 1 ? 0 : b + 1;
  return b;
}
__global__ void k_nb_rcount(const double* __restrict__ sph, int64_t N, const NbGrid* __restrict__ g,
                            int32_t* __restrict__ cnt) {
  const double rmax = g->rmax;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < N;
       i += (int64_t)gridDim.x * blockDim.x)
    atomicAdd(&cnt[nb_rbucket(sph[4 * i + 3], rmax)], 1);
}
__global__ void k_nb_rscatter(const double* __restrict__ sph, int64_t N,
                              const NbGrid* __restrict__ g, const int32_t* __restrict__ start,
                              int32_t* __restrict__ fill, int32_t* __restrict__ order) {
  const double rmax = g->rmax;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < N;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int b = nb_rbucket(sph[4 * i + 3], rmax);
    order[start[b] + atomicAdd(&fill[b], 1)] = (int)i;
  }
}

struct NbArgs {
  const double* sph;
  int64_t N;
  const NbGrid* grid;
  const int32_t* start;   // [G^3 + 1]
  const int32_t* items;   // spheres by cell
  const double4* sorted;  // their (x, y, z, r), same order
  double blo[3], bhi[3];  // the domain box B
  double tol0;            // absolute slack (distance units)
  int32_t* cnt;           // [N] row lengths (pass 1 writes)
  int32_t* slab;          // [N][CAP1] pass-1 rows (unsorted)
  const int32_t* off;     // [N+1] (pass 2)
  int32_t* tmp;           // [E] pass-2 rows (unsorted)
  int32_t* n_long;        // rows longer than CAP1: count, then ids
  int32_t* long_ids;
  unsigned long long* stats;  // [0] vertex overflows, [1] hidden, [2] triples, [3] block rows
  int* err;
  const int32_t* order;   // work order (pass 1)
  int32_t* work;          // work counter (pass 1)
  int64_t n_work;         // pass 1 rows: order[0, n_work) (0: all N) ...
  const int32_t* n_work_dev;  // ... or a device count (incremental update)
  long long* dbg;  // development aid (RPD_NB_DEBUG): per sphere 8 counters, or null
  double4* ball;   // [2N] per row: bounding ball of its final P_K (center, radius; r < 0:
                   // empty), then the half extents of P_K's vertex box around that centre
  int32_t* hits;   // [warp slots][NB_HCAP] positions (cell-sorted arrays) of a round's hits
  // heavy rows: pass 1 (a warp per sphere) hands a sphere whose round-0 search ball holds more
  // than heavy_items grid entries to the block kernel (a block of NB_BT threads per sphere)
  int heavy_items;    // 0: off
  int32_t* heavy_ids;  // [N]
  int32_t* n_heavy;    // their count
  int32_t* work2;      // the block kernel's work counter
  int ball_test;       // enumeration: skip plane pairs whose line misses the previous ball
};

// The per-sphere computation runs on a warp (NT = 32) or on a block of NT threads (heavy
// rows).  Both give the same row, bit for bit: the block's extra warps only share the loops
// whose results do not depend on which thread did what (the vertex enumeration, whose vertex
// SET is the result -- nothing downstream depends on the vertex order -- and the scans, whose
// per-thread candidate lists are merged into the 32 "virtual lanes" the warp would have had,
// t mod 32, and whose hit lists are compacted in scan order); everything else is done by warp
// 0 with the warp's code and broadcast through shared memory.
template <int NT>
struct NbBlk {
  double tk[4 * NT];  // per-thread LaneTop (merged into the 32 virtual lanes)
  int tj[4 * NT];
  int wc[NT / 32];    // per-warp counts (ordered compaction)
};
template <>
struct NbBlk<32> {};

struct NbBc {  // warp 0 -> the block
  double R, rho_v, pdm_v, evm_v, cx, cy, cz, rs, bc[3], be[3];
  int nK, first_new, n_deep;
};

template <int NT>
struct NbSm {
  NbSmem s;
  NbBc b;
  NbBlk<NT> k;
};

// One group (warp or block) computes sphere i's row.  PASS2: writes the row into tmp at off[i]
// (rows > CAP1).
template <int NT, bool PASS2>
__device__ void nb_row(const NbArgs& A, NbSm<NT>& SM, int i, int tid, int32_t* __restrict__ hb) {
  constexpr bool BLK = NT > 32;
  NbSmem& S = SM.s;
  NbBc& Bc = SM.b;
  const int lane = tid & 31, warp = tid >> 5;
  const bool w0 = warp == 0;
  auto gsync = [&]() {
    if constexpr (BLK) __syncthreads();
    else __syncwarp();
  };
  const NbGrid& g = *A.grid;
  const double4 si = make_double4(A.sph[4 * i], A.sph[4 * i + 1], A.sph[4 * i + 2], A.sph[4 * i + 3]);
  const int G = g.G;
  const int ci[3] = {nb_cell_axis(si.x, g, 0), nb_cell_axis(si.y, g, 1), nb_cell_axis(si.z, g, 2)};
  if (tid == 0) {
    S.n_v = 0;
    S.n_o = 0;
    S.flags = 0;
  }
  gsync();
  LaneTop top;
  top.init();
  const long long t_start = clock64();
  unsigned long long g_start = 0;
  if (!BLK && A.dbg) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g_start));
  long long dbg_scan = 0, dbg_cells = 0, dbg_vloop = 0, dbg_enum = 0, dbg_sclk = 0;
  int dbg_rounds = 0;
  // ---- 1. ring collection of candidates for K (and the hiding test): warp 0
  if (w0) {
    int n_seen = 0;
    for (int r = 0;; ++r) {
      const int w = 2 * r + 1, nc = w * w * w;
      for (int q = lane; q < nc; q += 32) {
        const int dx = q % w - r, dy = (q / w) % w - r, dz = q / (w * w) - r;
        if (max(abs(dx), max(abs(dy), abs(dz))) != r) continue;
        const int x = ci[0] + dx, y = ci[1] + dy, z = ci[2] + dz;
        if (x < 0 || y < 0 || z < 0 || x >= G || y >= G || z >= G) continue;
        const int c = (z * G + y) * G + x;
        for (int p = A.start[c]; p < A.start[c + 1]; ++p) {
          const int j = A.items[p];
          if (j == i) continue;
          const double4 sj = make_double4(A.sph[4 * j], A.sph[4 * j + 1], A.sph[4 * j + 2], A.sph[4 * j + 3]);
          const double ux = sj.x - si.x, uy = sj.y - si.y, uz = sj.z - si.z;
          const double d2 = ux * ux + uy * uy + uz * uz;
          if (d2 == 0.0) {
            if (sj.w > si.w || (sj.w == si.w && j < i)) atomicOr(&S.flags, 1);  // hidden
            continue;
          }
          top.push(d2 - sj.w * sj.w, j);
          ++n_seen;
        }
      }
      int n = n_seen;
      for (int o = 16; o; o >>= 1) n += __shfl_xor_sync(0xffffffffu, n, o);
      if (n >= NB_KSEL0 + 8 || r >= G) break;
    }
    for (int t = 0; t < 4; ++t) {
      S.cid[4 * lane + t] = top.j[t];
      S.key[4 * lane + t] = top.k[t];
    }
  }
  gsync();
  if (S.flags & 1) {
    if (!PASS2 && tid == 0) {
      A.cnt[i] = 0;
      atomicAdd(&A.stats[1], 1ull);
      if (A.ball) A.ball[2 * i] = make_double4(0.0, 0.0, 0.0, -1.0);  // (empty cell)
    }
    return;
  }
  // box planes (fixed), then rounds: select KSEL planes, enumerate P_K, scan the ball
  if (tid < 6) {
    const int k = tid >> 1;
    const double cth = k == 0 ? si.x : (k == 1 ? si.y : si.z);
    // lo: y_k + (cth - lo) >= 0 ; hi: -y_k + (hi - cth) >= 0
    double4 p = make_double4(0, 0, 0, 0);
    const double sgn = (tid & 1) ? -1.0 : 1.0;
    if (k == 0) p.x = sgn;
    if (k == 1) p.y = sgn;
    if (k == 2) p.z = sgn;
    p.w = (tid & 1) ? (A.bhi[k] - cth) : (cth - A.blo[k]);
    S.pl[tid] = p;
  }
  const double L = sqrt((A.bhi[0] - A.blo[0]) * (A.bhi[0] - A.blo[0]) +
                        (A.bhi[1] - A.blo[1]) * (A.bhi[1] - A.blo[1]) +
                        (A.bhi[2] - A.blo[2]) * (A.bhi[2] - A.blo[2]));
  const int base = PASS2 ? A.off[i] : 0;
  const int cap2 = PASS2 ? A.cnt[i] : 0;  // pass 2: the pass-1 length bounds the writes

  // select up to `want` planes from the candidates S.cid / S.key (smallest key first, ties:
  // smaller id), appended after the nK kept ones (warp 0)
  auto select = [&](int nK, int want) {
    int sel = nK;
    for (; sel < want; ++sel) {
      double bk = 1e300;
      int bi = 0x7fffffff, bs = -1;
      for (int s2 = lane; s2 < NB_CAPC; s2 += 32) {
        const int j = S.cid[s2];
        if (j < 0) continue;
        const double k = S.key[s2];
        if (k < bk || (k == bk && j < bi)) {
          bk = k;
          bi = j;
          bs = s2;
        }
      }
      for (int o = 16; o; o >>= 1) {
        const double ok = __shfl_xor_sync(0xffffffffu, bk, o);
        const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
        const int os = __shfl_xor_sync(0xffffffffu, bs, o);
        if (ok < bk || (ok == bk && oi < bi)) {
          bk = ok;
          bi = oi;
          bs = os;
        }
      }
      if (bs < 0) break;
      if (lane == 0) {
        const int j = S.cid[bs];
        S.cid[bs] = -1;
        const double ux = A.sph[4 * j] - si.x, uy = A.sph[4 * j + 1] - si.y,
                     uz = A.sph[4 * j + 2] - si.z, rj = A.sph[4 * j + 3];
        const double u2 = ux * ux + uy * uy + uz * uz, un = sqrt(u2);
        // h_ij(y) = -2 u.y + |u|^2 - r_j^2 + r_i^2 >= 0, normalised by 2|u|
        S.pl[6 + sel] = make_double4(-ux / un, -uy / un, -uz / un,
                                     (u2 - rj * rj + si.w * si.w) / (2.0 * un));
        S.kid[sel] = j;
      }
      __syncwarp();
    }
    return sel;
  };
  // round 0: K = the KSEL smallest power distances at theta_i.  Later rounds (monotone, the
  // polytope only shrinks): K = the planes of K that are facets of P_K (the others are
  // redundant for it) + the deepest cuts into P_K among the ball's spheres.  Converged when no
  // sphere cuts deeper than tolF: the final scan lists the hits.
  int nK = 0;
  if (w0) {
    nK = select(0, NB_KSEL0);
    if (lane == 0) S.first = nK > 0 ? S.kid[0] : -1;
  }
  if constexpr (BLK) {
    if (tid == 0) Bc.nK = nK;
    __syncthreads();
    nK = Bc.nK;
  } else {
    __syncwarp();
  }
  const int n_sel = nK;
  int n_v = 0;
  double R = 0.0, cx = 0.0, cy = 0.0, cz = 0.0, rs = 0.0;
  double bc[3] = {0, 0, 0}, be[3] = {0, 0, 0}, rho_v = 0.0, pdm_v = 0.0, evm_v = 0.0;
  unsigned long long n_tri = 0;
  const double tolF = 1e-6 * L + 1e-9;
  bool converged = false;
  bool list_exact = true;  // S.vx holds the vertices of P_K (not the box fallback)
  int first_new = 0;
  int n_list = -1;  // hits of the previous round in hb (-1: none, scan the grid)
  auto flush_tri = [&]() {  // (per warp)
    if constexpr (!PASS2) {
      for (int o = 16; o; o >>= 1) n_tri += __shfl_xor_sync(0xffffffffu, n_tri, o);
      if (lane == 0 && n_tri) atomicAdd(&A.stats[2], n_tri);
    }
  };
  for (int round = 0;; ++round) {
    const bool final_round = converged || round == NB_ROUNDS - 1;
    if (!converged) {
    const long long t_enum = clock64();
    const int M = 6 + nK;
    // ---- 3. vertices of P_K.  Round 0: every plane triple a < b < c.  Later rounds (P_K =
    // P_old ∩ new planes, planes [first_new, M) new): the old vertices that satisfy the new
    // planes (every old vertex lies on >= 3 kept facet planes), plus the triples whose largest
    // index is a new plane.  thread = pair (a, b)
    if (A.ball_test & 2) {
      // Sequential clip (default): P_K is cut by one new plane c at a time.  A vertex of
      // P ∩ {h_c >= 0} is a vertex of P on the kept side or lies on an edge a ∩ b of P that
      // crosses h_c = 0, whose removed endpoint u is a vertex of P tight at a and b.  So the
      // new vertices are the triples (a, b, c) over the pairs of planes tight at the vertices
      // that h_c may remove -- with margins: "may remove" is h_c < 2 m_v, "tight" |h| <= 2 m_v,
      // kept is h_c >= -m_v (m_v = e_v + tol0 + 8 eps |w|, the keep margin of the enumeration).
      // Every true vertex of the true polytope stays recorded within its error radius after
      // each cut, as with the triple enumeration, whose
      // triples (a, b, c) below are a subset; runs on warp 0.
      if (w0) {
        unsigned* const pm = reinterpret_cast<unsigned*>(S.key);  // pair bits (S.key free here)
        int* const plist = S.out;                                  // pair list (free here)
        constexpr double EPS = 1.1102230246251565e-16;
        // the triple a ∩ b ∩ c: y, error radius; false if (near) singular
        auto solve3 = [&](const double4& pa, const double4& pb, const double4& pc,
                          double4& y) -> bool {
          const double ab_x = pa.y * pb.z - pa.z * pb.y, ab_y = pa.z * pb.x - pa.x * pb.z,
                       ab_z = pa.x * pb.y - pa.y * pb.x;
          const double det = pc.x * ab_x + pc.y * ab_y + pc.z * ab_z;
          if (fabs(det) < 1e-13) return false;
          const double bc_x = pb.y * pc.z - pb.z * pc.y, bc_y = pb.z * pc.x - pb.x * pc.z,
                       bc_z = pb.x * pc.y - pb.y * pc.x;
          const double ca_x = pc.y * pa.z - pc.z * pa.y, ca_y = pc.z * pa.x - pc.x * pa.z,
                       ca_z = pc.x * pa.y - pc.y * pa.x;
          const double inv = -1.0 / det;
          y.x = (pa.w * bc_x + pb.w * ca_x + pc.w * ab_x) * inv;
          y.y = (pa.w * bc_y + pb.w * ca_y + pc.w * ab_y) * inv;
          y.z = (pa.w * bc_z + pb.w * ca_z + pc.w * ab_z) * inv;
          y.w = 64.0 * EPS * (fabs(pa.w) + fabs(pb.w) + fabs(pc.w) + L) / fabs(det);
          return true;
        };
        int nv = n_v, c0 = first_new;
        bool over = false;
        if (first_new == 0) {  // round 0 (or after a box fallback): start from the box
          if (lane < 8) {
            double4 y;
            solve3(S.pl[lane & 1], S.pl[2 + ((lane >> 1) & 1)], S.pl[4 + ((lane >> 2) & 1)], y);
            S.vx[lane] = y;
          }
          nv = 8;
          c0 = 6;
          __syncwarp();
        }
        for (int c = c0; c < M && nv > 0 && !over; ++c) {
          const double4 pc = S.pl[c];
          const double mc = A.tol0 + 8.0 * EPS * fabs(pc.w);
          const int nwp = (c * (c - 1) / 2 + 31) >> 5;
          for (int q = lane; q < nwp; q += 32) pm[q] = 0u;
          if (lane == 0) S.n_pair = 0;
          __syncwarp();
          // (a) the pairs of planes tight at the vertices h_c may remove (deduplicated)
          bool cuts = false;
          for (int s2 = lane; s2 < nv; s2 += 32) {
            const double4 v = S.vx[s2];
            if (pc.x * v.x + pc.y * v.y + pc.z * v.z + pc.w >= 2.0 * (v.w + mc)) continue;
            cuts = true;
            unsigned long long tm[2] = {0ull, 0ull};  // planes [0, 64), [64, 128)
            for (int k = 0; k < c; ++k) {
              const double4 pk = S.pl[k];
              const double h = pk.x * v.x + pk.y * v.y + pk.z * v.z + pk.w;
              if (h <= 2.0 * (v.w + A.tol0 + 8.0 * EPS * fabs(pk.w)))
                tm[k >> 6] |= 1ull << (k & 63);
            }
            for (int wa = 0; wa < 2; ++wa)
              for (unsigned long long ma = tm[wa]; ma; ma &= ma - 1) {
                const int a = __ffsll((long long)ma) - 1 + 64 * wa;
                for (int wb = wa; wb < 2; ++wb)
                  for (unsigned long long mb = wb == wa ? (ma & (ma - 1)) : tm[1]; mb;
                       mb &= mb - 1) {
                    const int b = __ffsll((long long)mb) - 1 + 64 * wb;
                    const int q = a * (2 * c - a - 1) / 2 + (b - a - 1);
                    const unsigned bit = 1u << (q & 31);
                    if (!(atomicOr(&pm[q >> 5], bit) & bit)) {
                      const int t = atomicAdd(&S.n_pair, 1);
                      if (t < NB_CAP1) plist[t] = a | (b << 8);
                    }
                  }
              }
          }
          __syncwarp();
          if (!__any_sync(0xffffffffu, cuts)) continue;  // h_c >= 2 m_v at every vertex: P unchanged
          const int np = S.n_pair;
          if (np > NB_CAP1) {
            over = true;
            break;
          }
          // (b) the kept vertices, compacted in place (in order)
          int kept = 0;
          for (int b0 = 0; b0 < nv; b0 += 32) {
            const int s2 = b0 + lane;
            double4 v = make_double4(0, 0, 0, 0);
            bool ok = false;
            if (s2 < nv) {
              v = S.vx[s2];
              ok = pc.x * v.x + pc.y * v.y + pc.z * v.z + pc.w >= -(v.w + mc);
            }
            const unsigned m = __ballot_sync(0xffffffffu, ok);
            __syncwarp();
            if (ok) S.vx[kept + __popc(m & ((1u << lane) - 1u))] = v;
            kept += __popc(m);
            __syncwarp();
          }
          if (lane == 0) S.n_v = kept;
          __syncwarp();
          // (c) the new vertices (a, b, c) that hold every plane up to c within their margin
          for (int t = lane; t < np; t += 32) {
            const int a = plist[t] & 0xff, b = plist[t] >> 8;
            double4 y;
            ++n_tri;
            if (!solve3(S.pl[a], S.pl[b], pc, y)) continue;
            bool ok = true;
            for (int k = 0; k < c && ok; ++k) {
              const double4 pk = S.pl[k];
              ok = pk.x * y.x + pk.y * y.y + pk.z * y.z + pk.w >=
                   -(y.w + A.tol0 + 8.0 * EPS * fabs(pk.w));
            }
            if (!ok) continue;
            const int s2 = atomicAdd(&S.n_v, 1);
            if (s2 < NB_MAXV) S.vx[s2] = y;
          }
          __syncwarp();
          nv = S.n_v;
          if (nv > NB_MAXV) over = true;
          __syncwarp();
        }
        if (lane == 0) S.n_v = over ? NB_MAXV + 1 : nv;
      }
      gsync();
    } else {  // the triple enumeration (RPD_NB_SEQ=0)
      if (w0) {
        if (first_new > 0) {
          int kept = 0;
          for (int c0 = 0; c0 < n_v; c0 += 32) {
            const int s2 = c0 + lane;
            bool ok = false;
            double4 v = make_double4(0, 0, 0, 0);
            if (s2 < n_v) {
              v = S.vx[s2];
              ok = true;
              for (int k = first_new; k < M && ok; ++k) {
                const double4 pk = S.pl[k];
                ok = pk.x * v.x + pk.y * v.y + pk.z * v.z + pk.w >=
                     -(v.w + A.tol0 + 8.0 * 1.1102230246251565e-16 * fabs(pk.w));
              }
            }
            const unsigned m = __ballot_sync(0xffffffffu, ok);
            __syncwarp();
            if (ok) S.vx[kept + __popc(m & ((1u << lane) - 1u))] = v;  // in place: <= s2
            kept += __popc(m);
            __syncwarp();
          }
          if (lane == 0) S.n_v = kept;
        } else if (lane == 0) {
          S.n_v = 0;
        }
      }
      gsync();
      const int n_pairs = M * (M - 1) / 2;
      const bool ball_ok = (A.ball_test & 1) && first_new > 0;  // (a previous round's ball exists)
      for (int q = tid; q < n_pairs; q += NT) {
        int a = 0, rem = q;
        while (rem >= M - 1 - a) {
          rem -= M - 1 - a;
          ++a;
        }
        const int b = a + 1 + rem;
        const double4 pa = S.pl[a], pb = S.pl[b];
        const double ab_x = pa.y * pb.z - pa.z * pb.y, ab_y = pa.z * pb.x - pa.x * pb.z,
                     ab_z = pa.x * pb.y - pa.y * pb.x;
        if (ball_ok) {
          // refinement rounds: P_K only shrinks, so every vertex of the new P_K lies in the
          // previous round's ball (centre c, radius rs: error radii included); a pair whose
          // line a ∩ b passes farther from c than rs (+ slack) carries none.  Squared distance
          // of c to the line, no division: (ha^2 + hb^2 - 2 cab ha hb) / |n_a x n_b|^2
          const double D2 = ab_x * ab_x + ab_y * ab_y + ab_z * ab_z;
          if (D2 >= 1e-6) {
            const double ha = pa.x * cx + pa.y * cy + pa.z * cz + pa.w;
            const double hb = pb.x * cx + pb.y * cy + pb.z * cz + pb.w;
            const double cab = pa.x * pb.x + pa.y * pb.y + pa.z * pb.z;
            const double rr = rs + 1e-7 * (L + fabs(pa.w) + fabs(pb.w));
            if (ha * ha + hb * hb - 2.0 * cab * ha * hb > rr * rr * D2) continue;
          }
        }
        for (int cc = max(b + 1, first_new); cc < M; ++cc) {
          const double4 pc = S.pl[cc];
          ++n_tri;
          const double det = pc.x * ab_x + pc.y * ab_y + pc.z * ab_z;
          if (fabs(det) < 1e-13) continue;
          const double bc_x = pb.y * pc.z - pb.z * pc.y, bc_y = pb.z * pc.x - pb.x * pc.z,
                       bc_z = pb.x * pc.y - pb.y * pc.x;
          const double ca_x = pc.y * pa.z - pc.z * pa.y, ca_y = pc.z * pa.x - pc.x * pa.z,
                       ca_z = pc.x * pa.y - pc.y * pa.x;
          const double inv = -1.0 / det;
          const double yx = (pa.w * bc_x + pb.w * ca_x + pc.w * ab_x) * inv;
          const double yy = (pa.w * bc_y + pb.w * ca_y + pc.w * ab_y) * inv;
          const double yz = (pa.w * bc_z + pb.w * ca_z + pc.w * ab_z) * inv;
          // error radius: rounding of the offsets and cofactors amplified by 1/|det|
          const double ev = 64.0 * 1.1102230246251565e-16 *
                            (fabs(pa.w) + fabs(pb.w) + fabs(pc.w) + L) / fabs(det);
          bool ok = true;
          for (int k = 0; k < M && ok; ++k) {
            const double4 pk = S.pl[k];
            const double h = pk.x * yx + pk.y * yy + pk.z * yz + pk.w;
            ok = h >= -(ev + A.tol0 + 8.0 * 1.1102230246251565e-16 * fabs(pk.w));
          }
          if (!ok) continue;
          const int s2 = atomicAdd(&S.n_v, 1);
          if (s2 < NB_MAXV) S.vx[s2] = make_double4(yx, yy, yz, ev);
        }
      }
      gsync();
    }
    dbg_enum += clock64() - t_enum;
    n_v = S.n_v;
    if (n_v == 0) {  // P_K empty: C_i ∩ B is empty
      if (!PASS2 && tid == 0) {
        A.cnt[i] = 0;
        if (A.ball) A.ball[2 * i] = make_double4(0.0, 0.0, 0.0, -1.0);
      }
      flush_tri();
      return;
    }
    if (n_v > NB_MAXV) {  // conservative fallback: the box corners
      list_exact = false;
      if (tid < 8)
        S.vx[tid] = make_double4(((tid & 1) ? A.bhi[0] : A.blo[0]) - si.x,
                                 ((tid & 2) ? A.bhi[1] : A.blo[1]) - si.y,
                                 ((tid & 4) ? A.bhi[2] : A.blo[2]) - si.z, A.tol0);
      if (!PASS2 && tid == 0 && final_round) atomicAdd(&A.stats[0], 1ull);
      n_v = 8;
      gsync();
    }
    // ---- 4. search ball (warp 0): radius R around theta_i; a bounding ball of P_K around the
    // centre of its vertex box (a plane farther than its radius from the centre misses P_K: one
    // dot product instead of a loop over the vertices) and the vertex box itself.  Only max /
    // min reductions: independent of the vertex order.
    if (w0) {
      double rho = 0.0, pdm = -1e300, evm = 0.0;
      for (int s2 = lane; s2 < n_v; s2 += 32) {
        const double4 v = S.vx[s2];
        const double d2 = v.x * v.x + v.y * v.y + v.z * v.z, d = sqrt(d2) + v.w;
        rho = fmax(rho, d);
        pdm = fmax(pdm, d * d - si.w * si.w);
        evm = fmax(evm, v.w);
      }
      rho = warp_max(rho);
      pdm = warp_max(pdm);
      evm = warp_max(evm);
      R = (rho + sqrt(fmax(pdm, 0.0) + g.rmax * g.rmax)) * (1.0 + 1e-9) +
          4.0 * (evm + A.tol0) + 1e-9 * L;
      // axis box of the vertices (grown by their error radii): centre bc, half extents be
      double mn[3] = {1e300, 1e300, 1e300}, mx[3] = {-1e300, -1e300, -1e300};
      for (int s2 = lane; s2 < n_v; s2 += 32) {
        const double4 v = S.vx[s2];
        mn[0] = fmin(mn[0], v.x - v.w);
        mn[1] = fmin(mn[1], v.y - v.w);
        mn[2] = fmin(mn[2], v.z - v.w);
        mx[0] = fmax(mx[0], v.x + v.w);
        mx[1] = fmax(mx[1], v.y + v.w);
        mx[2] = fmax(mx[2], v.z + v.w);
      }
      for (int k = 0; k < 3; ++k) {
        mn[k] = -warp_max(-mn[k]);
        mx[k] = warp_max(mx[k]);
        bc[k] = 0.5 * (mn[k] + mx[k]);
        be[k] = 0.5 * (mx[k] - mn[k]) * (1.0 + 1e-12) + 1e-12 * L;
      }
      cx = bc[0];
      cy = bc[1];
      cz = bc[2];
      double rr = 0.0;
      for (int s2 = lane; s2 < n_v; s2 += 32) {
        const double4 v = S.vx[s2];
        const double dx = v.x - cx, dy = v.y - cy, dz = v.z - cz;
        rr = fmax(rr, sqrt(dx * dx + dy * dy + dz * dz) + v.w);
      }
      rs = warp_max(rr) * (1.0 + 1e-12) + 1e-12 * L;
      rho_v = rho;
      pdm_v = pdm;
      evm_v = evm;
    }
    if constexpr (BLK) {
      if (tid == 0) {
        Bc.R = R;
        Bc.rho_v = rho_v;
        Bc.pdm_v = pdm_v;
        Bc.evm_v = evm_v;
        Bc.cx = cx;
        Bc.cy = cy;
        Bc.cz = cz;
        Bc.rs = rs;
        for (int k = 0; k < 3; ++k) {
          Bc.bc[k] = bc[k];
          Bc.be[k] = be[k];
        }
      }
      __syncthreads();
      if (!w0) {
        R = Bc.R;
        rho_v = Bc.rho_v;
        pdm_v = Bc.pdm_v;
        evm_v = Bc.evm_v;
        cx = Bc.cx;
        cy = Bc.cy;
        cz = Bc.cz;
        rs = Bc.rs;
        for (int k = 0; k < 3; ++k) {
          bc[k] = Bc.bc[k];
          be[k] = Bc.be[k];
        }
      }
    }
    }  // !converged
    // the search ball's cell box and its rows of cells (fixed y, z: contiguous in the
    // cell-sorted arrays)
    int lo[3], hi[3];
    {
      const double c[3] = {si.x, si.y, si.z};
      for (int k = 0; k < 3; ++k) {
        lo[k] = nb_cell_axis(c[k] - R, g, k);
        hi[k] = nb_cell_axis(c[k] + R, g, k);
      }
    }
    const int ny = hi[1] - lo[1] + 1, nz = hi[2] - lo[2] + 1, nrows = ny * nz;
    // lane = row r0 + lane of a 32-row chunk: its position range [pb, pe) (empty if the row's
    // (y, z) extent is beyond R)
    auto row_range = [&](int r0, int& pb, int& pe) {
      pb = pe = 0;
      const int rr = r0 + lane;
      if (rr < nrows) {
        const int y = lo[1] + rr % ny, z = lo[2] + rr / ny;
        double dd = 0.0;  // distance from theta_i to the row's (y, z) extent
        {
          const double ay0 = g.lo[1] + y * g.h[1], ay1 = ay0 + g.h[1];
          const double az0 = g.lo[2] + z * g.h[2], az1 = az0 + g.h[2];
          const double ey = si.y < ay0 ? ay0 - si.y : (si.y > ay1 ? si.y - ay1 : 0.0);
          const double ez = si.z < az0 ? az0 - si.z : (si.z > az1 ? si.z - az1 : 0.0);
          dd = ey * ey + ez * ez;
        }
        if (dd <= R * R * (1.0 + 1e-9)) {
          const int c0 = (z * G + y) * G;
          pb = A.start[c0 + lo[0]];
          pe = A.start[c0 + hi[0] + 1];
        }
      }
    };
    if constexpr (!BLK) {
      // heavy row (pass 1, round 0): more than heavy_items grid entries in the search ball --
      // handed to the block kernel, which recomputes it from the start (same row)
      if (!PASS2 && round == 0 && !final_round && A.heavy_items != 0 && n_list < 0) {
        int tot = 0;
        for (int r0 = 0; r0 < nrows; r0 += 32) {
          int pb, pe;
          row_range(r0, pb, pe);
          tot += pe - pb;
        }
        for (int o = 16; o; o >>= 1) tot += __shfl_xor_sync(0xffffffffu, tot, o);
        if (tot > A.heavy_items) {
          if (lane == 0) A.heavy_ids[atomicAdd(A.n_heavy, 1)] = i;
          return;
        }
      }
    }
    unsigned long long fmask = 0;  // facets of P_K among the K planes (lane = plane; warp 0)
    if (!final_round && w0) {
      for (int p0 = 0; p0 < nK; p0 += 32) {
        const int p = p0 + lane;
        bool facet = false;
        if (p < nK) {
          const double4 pk = S.pl[6 + p];
          const double slack = A.tol0 + 8.0 * 1.1102230246251565e-16 * fabs(pk.w);
          double depth = 1e300;
          for (int s2 = 0; s2 < n_v && depth > slack; ++s2) {
            const double4 v = S.vx[s2];
            depth = fmin(depth, pk.x * v.x + pk.y * v.y + pk.z * v.z + pk.w - v.w);
          }
          facet = depth <= slack;
        }
        fmask |= (unsigned long long)__ballot_sync(0xffffffffu, facet) << p0;
      }
    }
    if (!final_round) top.init();
    // ---- 5. every sphere of the ball whose plane reaches a vertex of P_K: collected with its
    // depth (selection of the next round) or, in the final round, listed.  The hits of a round
    // (some vertex within slack) are kept in hb: P_K only shrinks, so a plane that reaches a
    // later P_K (or cuts it) reached this one, and the next round scans the list, not the grid
    // (sound for any list that holds every hit; a full list falls back to the grid)
    // visit position p: bit 0 = hit, bit 1 = deep cut (not in the final round)
    auto visit = [&](int p, double& key, int& jo) -> int {
      const int j = A.items[p];
      jo = j;
      dbg_cells += 1 + (n_list < 0 ? (1ll << 32) : 0ll);
      if (j == i) return 0;
      const double4 sj = A.sorted[p];
      const double ux = sj.x - si.x, uy = sj.y - si.y, uz = sj.z - si.z, rj = sj.w;
      const double u2 = ux * ux + uy * uy + uz * uz;
      if (u2 == 0.0 || u2 > R * R) return 0;
      const double un = sqrt(u2);
      {  // j reaches a vertex v only if |v - theta_j|^2 <= PD_i(v) + r_j^2 (+ slack):
         // |theta_j - theta_i| <= (rho + sqrt(PDmax + r_j^2)) (1 + 1e-9) + 4 (e_max + tol0) + 1e-9 L,
         // tested without a second square root (the right side's relative margin doubled)
        const double d = un - rho_v * (1.0 + 1e-9) - 4.0 * (evm_v + A.tol0) - 1e-9 * L;
        if (d > 0.0 && d * d > (fmax(pdm_v, 0.0) + rj * rj) * ((1.0 + 2e-9) * (1.0 + 2e-9)))
          return 0;
      }
      const double iun = 1.0 / un;
      const double ax = -ux * iun, ay = -uy * iun, az = -uz * iun;
      const double bw = (u2 - rj * rj + si.w * si.w) * (0.5 * iun);
      const double slack = A.tol0 + 8.0 * 1.1102230246251565e-16 * fabs(bw);
      ++dbg_scan;
      const double hcen = ax * cx + ay * cy + az * cz + bw;  // plane value at the centre
      // lower bounds of the plane's minimum over P_K: the centre ball and the vertex box
      const double lb = fmax(hcen - rs, ax * bc[0] + ay * bc[1] + az * bc[2] + bw -
                                            (fabs(ax) * be[0] + fabs(ay) * be[1] + fabs(az) * be[2]));
      if (lb > slack) return 0;
      // final round: a hit once some vertex is within slack; earlier rounds: a deep cut once
      // some vertex is cut by more than tolF (ranked by the value at the centre)
      const double thr = final_round ? slack : -tolF;
      // (4 vertices per step: the test after a step only sees a smaller minimum, so both
      // result bits are those of the vertex-by-vertex loop)
      double depth = 1e300;
      int s2 = 0;
      bool stop = false;
      for (; s2 + 4 <= n_v && !stop; s2 += 4) {
        const double4 v0 = S.vx[s2], v1 = S.vx[s2 + 1], v2 = S.vx[s2 + 2], v3 = S.vx[s2 + 3];
        const double h0 = ax * v0.x + ay * v0.y + az * v0.z + bw - v0.w;
        const double h1 = ax * v1.x + ay * v1.y + az * v1.z + bw - v1.w;
        const double h2 = ax * v2.x + ay * v2.y + az * v2.z + bw - v2.w;
        const double h3 = ax * v3.x + ay * v3.y + az * v3.z + bw - v3.w;
        depth = fmin(depth, fmin(fmin(h0, h1), fmin(h2, h3)));
        dbg_vloop += 4;
        stop = final_round ? depth <= thr : depth < thr;
      }
      for (; s2 < n_v && !stop; ++s2) {
        const double4 v = S.vx[s2];
        depth = fmin(depth, ax * v.x + ay * v.y + az * v.z + bw - v.w);
        ++dbg_vloop;
        stop = final_round ? depth <= thr : depth < thr;
      }
      key = hcen;
      return (depth <= slack ? 1 : 0) | (!final_round && depth < -tolF ? 2 : 0);
    };
    auto take = [&](int code, double key, int j) {
      if (final_round) {
        if (code & 1) {
          const int s2 = atomicAdd(&S.n_o, 1);
          if (PASS2) {
            if (s2 < cap2) A.tmp[base + s2] = j;
          } else if (s2 < NB_CAP1) {
            S.out[s2] = j;
          }
        }
      } else if (code & 2) {
        top.push(key, j);
      }
    };
    // ordered compaction of a step's hits into hb (in place: a hit's new index <= its old one)
    auto compact = [&](bool f, int p, int nh) -> int {
      const unsigned m = __ballot_sync(0xffffffffu, f);
      if constexpr (!BLK) {
        const int at = nh + __popc(m & ((1u << lane) - 1u));
        if (f && at < NB_HCAP) hb[at] = p;
        return nh + __popc(m);
      } else {
        if (lane == 0) SM.k.wc[warp] = __popc(m);
        __syncthreads();
        int before = 0, tot = 0;
#pragma unroll
        for (int w = 0; w < NT / 32; ++w) {
          const int c = SM.k.wc[w];
          before += w < warp ? c : 0;
          tot += c;
        }
        const int at = nh + before + __popc(m & ((1u << lane) - 1u));
        if (f && at < NB_HCAP) hb[at] = p;
        __syncthreads();  // (wc is reused by the next step)
        return nh + tot;
      }
    };
    int n_hit = 0;  // hits recorded this round (> NB_HCAP: overflow)
    const long long t_scan = clock64();
    if (n_list >= 0) {  // ---- scan the previous round's hits, compacted in place
      ++dbg_rounds;
      for (int t0 = 0; t0 < n_list; t0 += NT) {
        const int t = t0 + tid;
        int code = 0, j = -1, p = 0;
        double key = 0.0;
        if (t < n_list) {
          p = hb[t];
          code = visit(p, key, j);
          take(code, key, j);
        }
        if (!final_round) n_hit = compact(code & 1, p, n_hit);
      }
    } else {
      ++dbg_rounds;
      // every warp walks the same 32-row chunks: lane = row for the ranges, then the group
      // walks the concatenated ranges (coalesced id / sphere loads), item t on thread t mod NT
      for (int r0 = 0; r0 < nrows; r0 += 32) {
        int pb = 0, pe = 0;
        row_range(r0, pb, pe);
        const int len = pe - pb;
        int incl = len;
        for (int o = 1; o < 32; o <<= 1) {
          const int t = __shfl_up_sync(0xffffffffu, incl, o);
          if (lane >= o) incl += t;
        }
        const int total = __shfl_sync(0xffffffffu, incl, 31);
        const int excl = incl - len;
        for (int t0 = 0; t0 < total; t0 += NT) {
          const int t = t0 + tid;
          int k = 0;  // the row holding t: the largest k with excl_k <= t
          for (int step = 16; step; step >>= 1) {
            const int e = __shfl_sync(0xffffffffu, excl, k + step);
            if (e <= t) k += step;
          }
          const int pbk = __shfl_sync(0xffffffffu, pb, k), exk = __shfl_sync(0xffffffffu, excl, k);
          int code = 0, j = -1, p = 0;
          double key = 0.0;
          if (t < total) {
            p = pbk + (t - exk);
            code = visit(p, key, j);
            take(code, key, j);
          }
          if (!final_round) n_hit = compact(code & 1, p, n_hit);
        }
      }
    }
    n_list = n_hit <= NB_HCAP ? n_hit : -1;
    gsync();
    dbg_sclk += clock64() - t_scan;
    if (final_round) break;
    if constexpr (BLK) {  // the 32 virtual lanes' candidate lists: thread t -> lane t mod 32
      for (int t = 0; t < 4; ++t) {
        SM.k.tk[4 * tid + t] = top.k[t];
        SM.k.tj[4 * tid + t] = top.j[t];
      }
      __syncthreads();
      if (w0) {
        for (int w = 1; w < NT / 32; ++w)
          for (int t = 0; t < 4; ++t) {
            const int s = 4 * (32 * w + lane) + t;
            if (SM.k.tj[s] >= 0) top.push(SM.k.tk[s], SM.k.tj[s]);
          }
      }
    }
    int n_deep = 0;
    if (w0) {
      for (int t = 0; t < 4; ++t) {
        S.cid[4 * lane + t] = top.j[t];
        S.key[4 * lane + t] = top.k[t];
        n_deep += top.j[t] >= 0;
      }
      for (int o = 16; o; o >>= 1) n_deep += __shfl_xor_sync(0xffffffffu, n_deep, o);
      __syncwarp();
      if (n_deep > 0) {
        // keep the facet planes (compacted in order), then the deepest cuts
        if (lane == 0) {
          int q = 0;
          for (int p = 0; p < nK; ++p)
            if (fmask >> p & 1ull) {
              S.pl[6 + q] = S.pl[6 + p];
              S.kid[q] = S.kid[p];
              ++q;
            }
        }
        __syncwarp();
        nK = select(__popcll(fmask), NB_KSEL);
        first_new = list_exact ? 6 + __popcll(fmask) : 0;
      }
    }
    if constexpr (BLK) {
      if (tid == 0) {
        Bc.n_deep = n_deep;
        Bc.nK = nK;
        Bc.first_new = first_new;
      }
      __syncthreads();
      nK = Bc.nK;
      first_new = Bc.first_new;
      n_deep = Bc.n_deep;
      __syncthreads();  // (Bc is rewritten by the next round)
    }
    if (n_deep == 0) converged = true;
    if (converged && n_list >= 0 && (A.ball_test & 4)) {
      // the final list is this round's hit list: the listing round would scan exactly these
      // positions against the same P_K with the same test (some vertex within slack; this
      // round's loop only stopped early on a deep cut, which there is none of), so every one
      // is listed (RPD_NB_REUSE=0: the listing scan)
      for (int t = tid; t < n_list; t += NT) {
        const int j = A.items[hb[t]];
        if (PASS2) {
          if (t < cap2) A.tmp[base + t] = j;
        } else if (t < NB_CAP1) {
          S.out[t] = j;
        }
      }
      if (tid == 0) S.n_o = n_list;
      gsync();
      break;
    }
  }
  flush_tri();
  gsync();
  int n_o = S.n_o;
  if (n_o == 0 && A.N > 1) {  // i's cell covers B: list the nearest sphere (redundant plane)
    if (n_sel > 0 && tid == 0) {  // not hit: h_ij > 0 on P_K, so the plane is redundant
      if (PASS2) {
        if (cap2 > 0) A.tmp[base] = S.first;
      } else {
        S.out[0] = S.first;
      }
      S.n_o = 1;
    }
    gsync();
    n_o = S.n_o;
  }
  if (PASS2 && n_o != cap2 && tid == 0 && atomicCAS(A.err, 0, (int)RPD_EOVERFLOW) == 0) {
    A.err[1] = ERR_NB_RECOMPUTE;
    A.err[2] = i;
  }
  if (!BLK && A.dbg && !PASS2) {
    for (int o = 16; o; o >>= 1) {
      dbg_scan += __shfl_xor_sync(0xffffffffu, dbg_scan, o);
      dbg_vloop += __shfl_xor_sync(0xffffffffu, dbg_vloop, o);
      dbg_cells += __shfl_xor_sync(0xffffffffu, dbg_cells, o);
    }
    if (lane == 0) {
      long long* d = A.dbg + 8 * (long long)i;
      d[0] = clock64() - t_start;
      d[1] = dbg_rounds;
      d[2] = dbg_enum;  // cycles in the vertex enumeration (lane 0)
      d[3] = dbg_sclk;  // cycles in the ball scans (lane 0)
      d[4] = dbg_vloop;
      d[5] = n_v;
      d[6] = dbg_cells;  // items visited by the scans (grid scans << 32)
      d[7] = (long long)g_start;  // start (ns, global timer)
    }
  }
  if (!PASS2) {
    if (tid == 0) {
      A.cnt[i] = n_o;
      // a ball around P_K ⊇ C_i ∩ B (world coordinates; incremental updates test it)
      if (A.ball) {  // and the half extents of its vertex box (same centre)
        A.ball[2 * i] = make_double4(si.x + cx, si.y + cy, si.z + cz, rs + A.tol0);
        A.ball[2 * i + 1] = make_double4(be[0] + A.tol0, be[1] + A.tol0, be[2] + A.tol0, 0.0);
      }
      if (n_o > NB_CAP1) A.long_ids[atomicAdd(A.n_long, 1)] = i;
    }
    if (n_o <= NB_CAP1)
      for (int s = tid; s < n_o; s += NT) A.slab[(int64_t)i * NB_CAP1 + s] = S.out[s];
  }
}

#ifdef RPD_NB_MINB  // min resident blocks of pass 1 (a register budget; A/B knob)
#define NB_PASS1_BOUNDS __launch_bounds__(32 * NB_WARPS, RPD_NB_MINB)
#else
#define NB_PASS1_BOUNDS __launch_bounds__(32 * NB_WARPS)
#endif
__global__ void NB_PASS1_BOUNDS k_nb_pass1(NbArgs A) {
  __shared__ NbSm<32> sm[NB_WARPS];
  if (*(volatile int*)A.err != 0) {  // invalid input: empty rows, no dereference of NaN cells
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < A.N;
         i += (int64_t)gridDim.x * blockDim.x)
      A.cnt[i] = 0;
    return;
  }
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t nwork = A.n_work_dev ? *A.n_work_dev : (A.n_work > 0 ? A.n_work : A.N);
  for (;;) {
    int q = 0;
    if (lane == 0) q = atomicAdd(A.work, 1);
    q = __shfl_sync(0xffffffffu, q, 0);
    if (q >= nwork) break;
    nb_row<32, false>(A, sm[w], A.order[q], lane,
                      A.hits + (size_t)(blockIdx.x * NB_WARPS + w) * NB_HCAP);
  }
}

// the heavy rows handed over by pass 1: a block per sphere, taken from a counter
__global__ void __launch_bounds__(NB_BT) k_nb_heavy(NbArgs A) {
  __shared__ NbSm<NB_BT> sm;
  __shared__ int q_s;
  const int n = *A.n_heavy;
  if (*(volatile int*)A.err != 0) {  // invalid input: empty rows (as pass 1)
    for (int q = blockIdx.x * blockDim.x + threadIdx.x; q < n; q += gridDim.x * blockDim.x)
      A.cnt[A.heavy_ids[q]] = 0;
    return;
  }
  for (;;) {
    if (threadIdx.x == 0) q_s = atomicAdd(A.work2, 1);
    __syncthreads();
    const int q = q_s;
    __syncthreads();
    if (q >= n) break;
    if (threadIdx.x == 0) atomicAdd(&A.stats[3], 1ull);
    nb_row<NB_BT, false>(A, sm, A.heavy_ids[q], threadIdx.x,
                         A.hits + (size_t)blockIdx.x * NB_HCAP);
    __syncthreads();
  }
}

__global__ void __launch_bounds__(32 * NB_WARPS) k_nb_pass2(NbArgs A) {
  __shared__ NbSm<32> sm[NB_WARPS];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int n = *A.n_long;
  for (int q = blockIdx.x * NB_WARPS + w; q < n; q += gridDim.x * NB_WARPS)
    nb_row<32, true>(A, sm[w], A.long_ids[q], lane,
                     A.hits + (size_t)(blockIdx.x * NB_WARPS + w) * NB_HCAP);
}

// rows into ascending order: rank of each entry among its row (entries are distinct)
__global__ void k_nb_sort(int64_t N, const int32_t* __restrict__ off, const int32_t* __restrict__ slab,
                          const int32_t* __restrict__ tmp, int32_t* __restrict__ idx) {
  const int lane = threadIdx.x & 31;
  for (int64_t i = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; i < N;
       i += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    const int a = off[i], n = off[i + 1] - a;
    const int32_t* src = n <= NB_CAP1 ? slab + i * NB_CAP1 : tmp + a;
    for (int s = lane; s < n; s += 32) {
      const int v = src[s];
      int rk = 0;
      for (int t = 0; t < n; ++t) rk += src[t] < v;
      idx[a + rk] = v;
    }
  }
}

}  // namespace

size_t nb_grid_cells(int64_t N) {
  int G = 1;
  while ((int64_t)G * G * G * 2 < N && G < NB_GMAX) ++G;
  return (size_t)G * G * G;
}

// heavy-row hand-off threshold (grid entries in a row's round-0 search ball; RPD_NB_HEAVY,
// 0 = every row on a warp, -1 = every row on a block: the equivalence tests)
static int nb_heavy_items(int dflt) {
  const char* s = getenv("RPD_NB_HEAVY");
  return s ? atoi(s) : dflt;
}
constexpr int NB_HEAVY_DEFAULT = 0;  // no hand-off in a full recompute (C3 / C5 sweep: DESIGN.md §10)
constexpr int NB_HEAVY_UPDATE = 2048;   // incremental updates with more new rows than:
constexpr int NB_UPDATE_ALL_BLOCKS = 2048;

// the block kernel over the heavy rows (device count; persistent grid, at most n_max blocks)
static cudaError_t nb_launch_heavy(rpd_ctx* c, const NbArgs& A, int64_t n_max) {
  if (A.heavy_items == 0 || n_max <= 0) return cudaSuccess;
  static int occ[RPD_MAX_DEVICES] = {};
  int& o = occ[c->device < RPD_MAX_DEVICES ? c->device : 0];
  if (o == 0 && (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, k_nb_heavy, NB_BT, 0) || o < 1))
    o = 1;
  // (one hit-list slot per block: nb_build allocates at least 2 * sms * NB_WARPS slots)
  const int64_t g = std::min<int64_t>(n_max, (int64_t)std::min(o, 2 * NB_WARPS) * c->sms);
  k_nb_heavy<<<(int)g, NB_BT, 0, c->stream>>>(A);
  ++c->launches;
  return cudaGetLastError();
}

// The uniform grid of the spheres, their cell-ordered copy and the radius work order; the
// pass arguments in *A and the pass-1 grid size in *mb.  Buffers in c->nb_buf.
static cudaError_t nb_build(rpd_ctx* c, const double* sph, int64_t N, const double box[6],
                            int32_t* cnt, NbArgs* Ap, int* mbp) {
  int G = 1;
  while ((int64_t)G * G * G * 2 < N && G < NB_GMAX) ++G;
  const int64_t ncell = (int64_t)G * G * G;
  const size_t bytes = sizeof(NbGrid) + 16 + sizeof(int32_t) * (3 * (ncell + 1) + 2 * (N + 1) + 2) +
                       sizeof(int32_t) * (size_t)N * NB_CAP1 + sizeof(unsigned long long) * 4 +
                       sizeof(double4) * (N + 1) + sizeof(int32_t) * (3 * (NB_RB + 1) + 2 + N + 1) +
                       sizeof(int32_t) * (N + 1 + 4) + 1024;
  // (2x on a reallocation: incremental updates grow N a batch at a time)
  cudaError_t e = c->nb_buf.ensure_slack(bytes, 2);
  if (e) return e;
  char* b = c->nb_buf.as<char>();
  auto take = [&](size_t n) {
    char* r = b;
    b += (n + 15) & ~size_t(15);
    return r;
  };
  NbGrid* g = reinterpret_cast<NbGrid*>(take(sizeof(NbGrid)));
  unsigned long long* st = reinterpret_cast<unsigned long long*>(take(8 * 4));
  int32_t* ccnt = reinterpret_cast<int32_t*>(take(4 * (ncell + 1)));
  int32_t* start = reinterpret_cast<int32_t*>(take(4 * (ncell + 1)));
  int32_t* fill = reinterpret_cast<int32_t*>(take(4 * (ncell + 1)));
  int32_t* cell_of = reinterpret_cast<int32_t*>(take(4 * (N + 1)));
  int32_t* items = reinterpret_cast<int32_t*>(take(4 * (N + 1)));
  int32_t* nlong = reinterpret_cast<int32_t*>(take(4 * 2));
  int32_t* rb = reinterpret_cast<int32_t*>(take(4 * (3 * (NB_RB + 1) + 2)));  // cnt, start, fill, work
  int32_t* order = reinterpret_cast<int32_t*>(take(4 * (N + 1)));
  int32_t* slab = reinterpret_cast<int32_t*>(take(4 * (size_t)N * NB_CAP1));
  double4* sorted = reinterpret_cast<double4*>(take(sizeof(double4) * (N + 1)));
  int32_t* hvy = reinterpret_cast<int32_t*>(take(4 * 4));  // n_heavy, work2
  int32_t* hvy_ids = reinterpret_cast<int32_t*>(take(4 * (N + 1)));
  c->nb_grid = g;
  c->nb_stats = st;
  c->nb_start = start;
  c->nb_items = items;
  c->nb_long = nlong;
  c->nb_slab = slab;
  c->nb_long_ids = cell_of;
  c->nb_sorted = sorted;
  if ((e = cudaMemsetAsync(ccnt, 0, 4 * (ncell + 1), c->stream))) return e;
  if ((e = cudaMemsetAsync(fill, 0, 4 * (ncell + 1), c->stream))) return e;
  if ((e = cudaMemsetAsync(st, 0, 8 * 4, c->stream))) return e;
  if ((e = cudaMemsetAsync(nlong, 0, 8, c->stream))) return e;
  if ((e = cudaMemsetAsync(hvy, 0, 16, c->stream))) return e;
  if ((e = cudaMemsetAsync(rb, 0, 4 * (3 * (NB_RB + 1) + 2), c->stream))) return e;
  const int blocks = (int)std::min<int64_t>((N + 255) / 256, 8 * (int64_t)c->sms) + 1;
  k_nb_check<<<blocks, 256, 0, c->stream>>>(sph, N, c->errw.as<int>());
  ++c->launches;
  k_nb_bounds<<<1, 1024, 0, c->stream>>>(sph, N, G, g);
  ++c->launches;
  k_nb_count<<<blocks, 256, 0, c->stream>>>(sph, N, g, ccnt, cell_of);
  ++c->launches;
  if ((e = launch_scan_i32(c, ccnt, start, ncell))) return e;
  k_nb_scatter<<<blocks, 256, 0, c->stream>>>(N, cell_of, start, fill, items);
  ++c->launches;
  k_nb_cellsort<<<(int)std::min<int64_t>((ncell + 255) / 256, 8 * (int64_t)c->sms), 256, 0,
                  c->stream>>>(ncell, start, items);
  ++c->launches;
  k_nb_gather<<<blocks, 256, 0, c->stream>>>(N, items, sph, sorted);
  ++c->launches;
  k_nb_rcount<<<blocks, 256, 0, c->stream>>>(sph, N, g, rb);
  ++c->launches;
  if ((e = launch_scan_i32(c, rb, rb + (NB_RB + 1), NB_RB))) return e;
  k_nb_rscatter<<<blocks, 256, 0, c->stream>>>(sph, N, g, rb + (NB_RB + 1), rb + 2 * (NB_RB + 1),
                                                order);
  ++c->launches;
  NbArgs A{};
  A.sph = sph;
  A.N = N;
  A.grid = g;
  A.start = start;
  A.items = items;
  A.sorted = sorted;
  A.order = order;
  A.work = rb + 3 * (NB_RB + 1);
  double L2 = 0.0;
  for (int k = 0; k < 3; ++k) {
    A.blo[k] = box[k];
    A.bhi[k] = box[3 + k];
    L2 += (box[3 + k] - box[k]) * (box[3 + k] - box[k]);
  }
  A.tol0 = 1e-9 * sqrt(L2) + 1e-12;
  A.cnt = cnt;
  A.slab = slab;
  A.n_long = nlong;
  A.long_ids = reinterpret_cast<int32_t*>(cell_of);  // cell_of is dead after the scatter
  A.stats = st;
  A.err = c->errw.as<int>();
  A.dbg = (long long*)c->nb_dbg;
  A.ball = c->nb_ball.as<double4>();
  A.heavy_items = nb_heavy_items(NB_HEAVY_DEFAULT);
  {
    // bit 0: the ball pre-test of the triple enumeration's refinement pairs; bit 1: the
    // sequential clip in place of the triple enumeration (RPD_NB_SEQ=0: the enumeration);
    // bit 2: the converged round's hit list taken as the row (RPD_NB_REUSE=0: a listing scan)
    const char* bt = getenv("RPD_NB_BALLT");
    const char* sq = getenv("RPD_NB_SEQ");
    const char* ru = getenv("RPD_NB_REUSE");
    A.ball_test = (bt ? (atoi(bt) & 1) : 1) | ((sq ? atoi(sq) : 1) ? 2 : 0) |
                  ((ru ? atoi(ru) : 1) ? 4 : 0);
  }
  c->nb_ball_test = A.ball_test;
  A.heavy_ids = hvy_ids;
  A.n_heavy = hvy;
  A.work2 = hvy + 1;
  c->nb_args_tol0 = A.tol0;
  int occ = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_nb_pass1, 32 * NB_WARPS, 0) || occ < 1)
    occ = 4;
  const int mb = (int)std::min<int64_t>((N + NB_WARPS - 1) / NB_WARPS, (int64_t)occ * c->sms);
  // hit lists: one per warp slot of pass 1 or pass 2 (2 * sms blocks)
  const size_t slots = (size_t)std::max(mb, 2 * c->sms) * NB_WARPS;
  if ((e = c->nb_hits.ensure(sizeof(int32_t) * NB_HCAP * slots))) return e;
  A.hits = c->nb_hits.as<int32_t>();
  c->nb_work = A.work;
  c->nb_order = order;
  *Ap = A;
  *mbp = mb;
  return cudaGetLastError();
}

// Pass 1 and the scan; *E_dev = total entries (off[N]).
cudaError_t launch_neighbors_pass1(rpd_ctx* c, const double* sph, int64_t N, const double box[6],
                                   int32_t* cnt, int32_t* off) {
  NbArgs A{};
  int mb = 0;
  cudaError_t e = nb_build(c, sph, N, box, cnt, &A, &mb);
  if (e) return e;
  k_nb_pass1<<<mb > 0 ? mb : 1, 32 * NB_WARPS, 0, c->stream>>>(A);
  ++c->launches;
  if ((e = cudaGetLastError())) return e;
  if ((e = nb_launch_heavy(c, A, N))) return e;
  if ((e = launch_scan_i32(c, cnt, off, N))) return e;
  return cudaGetLastError();
}

// pass 2 (rows longer than the pass-1 slab, into tmp at off) and the ascending sort
cudaError_t launch_neighbors_pass2(rpd_ctx* c, const double* sph, int64_t N, const double box[6],
                                   int32_t* cnt, const int32_t* off, int32_t* tmp, int32_t* idx) {
  cudaError_t e = launch_neighbors_pass2_rows(c, sph, N, box, cnt, off, tmp);
  if (e) return e;
  const int sb = (int)std::min<int64_t>((N * 32 + 255) / 256, 16 * (int64_t)c->sms);
  k_nb_sort<<<sb > 0 ? sb : 1, 256, 0, c->stream>>>(N, off, c->nb_slab, tmp, idx);
  ++c->launches;
  return cudaGetLastError();
}

cudaError_t launch_neighbors_pass2_rows(rpd_ctx* c, const double* sph, int64_t N,
                                        const double box[6], int32_t* cnt, const int32_t* off,
                                        int32_t* tmp) {
  NbArgs A{};
  A.sph = sph;
  A.N = N;
  A.grid = reinterpret_cast<const NbGrid*>(c->nb_grid);
  A.start = c->nb_start;
  A.items = c->nb_items;
  A.sorted = reinterpret_cast<const double4*>(c->nb_sorted);
  for (int k = 0; k < 3; ++k) {
    A.blo[k] = box[k];
    A.bhi[k] = box[3 + k];
  }
  A.tol0 = c->nb_args_tol0;
  A.ball_test = c->nb_ball_test;
  A.cnt = cnt;
  A.slab = c->nb_slab;
  A.off = off;
  A.tmp = tmp;
  A.n_long = c->nb_long;
  A.long_ids = c->nb_long_ids;
  A.stats = c->nb_stats;
  A.hits = c->nb_hits.as<int32_t>();
  k_nb_pass2<<<2 * c->sms, 32 * NB_WARPS, 0, c->stream>>>(A);
  ++c->launches;
  return cudaGetLastError();
}

// ---------------------------------------------------------------- incremental update
//
// After M spheres are appended (DESIGN.md §10 "Sphere neighbours", reading R34) the cells only
// shrink: a facet of the new cell C_i ∩ B between i and an old sphere k is part of an old facet,
// so the new neighbours of an old sphere i are among its old neighbours and the new spheres.
// And a new sphere j can cut C_i ∩ B only where h_ij < 0; every row stores a ball around its
// last bounding polytope P_K ⊇ C_i ∩ B.  So the row of an old sphere becomes its old row
// followed by the new spheres whose radical plane reaches its ball (ids > N_old: the row stays
// ascending) -- a certified superset again: B ∩ (planes of the row) = the new cell exactly,
// since the new spheres that miss the ball do not cut the old cell.  A new sphere with the same
// centre that hides i (larger radius) empties i's row.  The new spheres' rows are computed by
// pass 1 / pass 2.  Rows only grow; a full rpd_neighbors tightens them again.

static __global__ void k_nb_same(const double* __restrict__ sph, const double* __restrict__ prev,
                                 int64_t n4, int* __restrict__ err) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n4;
       k += (int64_t)gridDim.x * blockDim.x)
    if (!(sph[k] == prev[k]) && atomicCAS(&err[0], 0, (int)RPD_EINVAL) == 0) {
      err[1] = ERR_SPHERE_CHANGED;
      err[2] = (int)(k / 4);
    }
}

static __global__ void k_nb_iota(int32_t* __restrict__ list, int64_t base, int64_t n,
                                 int32_t* __restrict__ count) {
  if (count && blockIdx.x == 0 && threadIdx.x == 0) *count = (int32_t)n;
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n;
       k += (int64_t)gridDim.x * blockDim.x)
    list[k] = (int32_t)(base + k);
}

// old sphere i against the new spheres (tiles in shared memory): WRITE = false counts the new
// spheres whose plane reaches i's ball into len[i] (+ the old row; 0 when a new sphere hides
// i, whose ball is then emptied) and flags the extended rows; WRITE = true appends their ids
constexpr int NB_AT = 256;
template <bool WRITE>
static __global__ void __launch_bounds__(NB_AT) k_nb_extend(
    int64_t N_old, int64_t N, const double* __restrict__ sph, double4* __restrict__ ball,
    double margin, const int32_t* __restrict__ old_off, int32_t* __restrict__ len,
    uint8_t* __restrict__ flag, const int32_t* __restrict__ off, int32_t* __restrict__ idx) {
  __shared__ double4 s_new[NB_AT];
  for (int64_t i0 = (int64_t)blockIdx.x * blockDim.x; i0 < N_old;
       i0 += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = i0 + threadIdx.x;
    double4 b = make_double4(0, 0, 0, -1.0), bx = make_double4(0, 0, 0, 0),
            si = make_double4(0, 0, 0, 0);
    if (i < N_old) {
      b = ball[2 * i];
      bx = ball[2 * i + 1];
      si = make_double4(sph[4 * i], sph[4 * i + 1], sph[4 * i + 2], sph[4 * i + 3]);
    }
    const int o0 = i < N_old ? old_off[i] : 0, o1 = i < N_old ? old_off[i + 1] : 0;
    int n_hit = 0, pos = WRITE && i < N_old ? off[i] + (o1 - o0) : 0;
    bool hidden = false;
    for (int64_t j0 = N_old; j0 < N; j0 += NB_AT) {
      __syncthreads();
      if (j0 + threadIdx.x < N) {
        const int64_t j = j0 + threadIdx.x;
        s_new[threadIdx.x] = make_double4(sph[4 * j], sph[4 * j + 1], sph[4 * j + 2], sph[4 * j + 3]);
      }
      __syncthreads();
      const int nj = (int)(N - j0 < NB_AT ? N - j0 : NB_AT);
      if (b.w < 0.0 || hidden) continue;  // (an empty cell stays empty)
      for (int q = 0; q < nj; ++q) {
        const double4 sj = s_new[q];
        const double ux = sj.x - si.x, uy = sj.y - si.y, uz = sj.z - si.z;
        const double u2 = ux * ux + uy * uy + uz * uz;
        if (u2 == 0.0) {  // same centre: the larger radius hides the other (ties: smaller id, i)
          if (sj.w > si.w) {
            hidden = true;
            break;
          }
          continue;
        }
        // h_ij(x) = (-u.(x - theta_i) + (|u|^2 - r_j^2 + r_i^2) / 2) / |u| >= 0 on C_i: its
        // minimum over the ball is the value at the centre minus the radius, over the vertex
        // box the value at the centre minus sum |u_k| e_k / |u|; both bound it over P_K
        const double un = sqrt(u2);
        const double yx = b.x - si.x, yy = b.y - si.y, yz = b.z - si.z;
        const double hc =
            (-(ux * yx + uy * yy + uz * yz) + 0.5 * (u2 - sj.w * sj.w + si.w * si.w)) / un;
        const double hb = hc - (fabs(ux) * bx.x + fabs(uy) * bx.y + fabs(uz) * bx.z) / un;
        if (hc - b.w <= margin && hb <= margin) {
          if (WRITE) idx[pos++] = (int32_t)(j0 + q);
          ++n_hit;
        }
      }
    }
    if (!WRITE && i < N_old) {
      len[i] = hidden ? 0 : (o1 - o0) + n_hit;
      flag[i] = hidden || n_hit > 0;
      if (hidden) ball[2 * i] = make_double4(0.0, 0.0, 0.0, -1.0);
    }
  }
}

// warp per row: the old rows' kept entries (copied; the appended ones are written by
// k_nb_extend<true>), the new rows rank-sorted from the slab / pass-2 rows
static __global__ void k_nb_merge(int64_t N, int64_t N_old, const int32_t* __restrict__ len,
                                  const int32_t* __restrict__ old_off,
                                  const int32_t* __restrict__ old_idx,
                                  const int32_t* __restrict__ off, const int32_t* __restrict__ slab,
                                  const int32_t* __restrict__ tmp, int32_t* __restrict__ idx) {
  const int lane = threadIdx.x & 31;
  for (int64_t i = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; i < N;
       i += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    const int a = off[i], n = off[i + 1] - a;
    if (i < N_old) {
      if (len[i] == 0) continue;  // (hidden)
      const int o = old_off[i], k = old_off[i + 1] - o;
      for (int s = lane; s < k; s += 32) idx[a + s] = old_idx[o + s];
      continue;
    }
    const int32_t* src = n <= NB_CAP1 ? slab + i * NB_CAP1 : tmp + a;
    for (int s = lane; s < n; s += 32) {
      const int v = src[s];
      int rk = 0;
      for (int t = 0; t < n; ++t) rk += src[t] < v;
      idx[a + rk] = v;
    }
  }
}

// new rows' lengths from pass 1
static __global__ void k_nb_newlen(int64_t N_old, int64_t N, const int32_t* __restrict__ cnt,
                                   int32_t* __restrict__ len) {
  for (int64_t i = N_old + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < N;
       i += (int64_t)gridDim.x * blockDim.x)
    len[i] = cnt[i];
}

static double nb_margin(const double box[6]) {
  double L2 = 0.0;
  for (int k = 0; k < 3; ++k) L2 += (box[3 + k] - box[k]) * (box[3 + k] - box[k]);
  return 1e-9 * sqrt(L2) + 1e-12;
}

// Part 1 of an incremental update: grid, the new rows (pass 1), the old rows' lengths, the
// merged offsets (off[N] = E); misc[0] = old rows extended or emptied (flag)
cudaError_t launch_nb_update1(rpd_ctx* c, const double* sph, int64_t N, int64_t N_old,
                              const double box[6], const double* prev, int32_t* cnt,
                              uint8_t* flag, int32_t* list, int32_t* len,
                              const int32_t* old_off, int32_t* off, int* misc) {
  cudaError_t e;
  const int blocks = (int)std::min<int64_t>((N + 255) / 256, 8 * (int64_t)c->sms) + 1;
  k_nb_same<<<blocks, 256, 0, c->stream>>>(sph, prev, 4 * N_old, c->errw.as<int>());
  ++c->launches;
  NbArgs A{};
  int mb = 0;
  if ((e = nb_build(c, sph, N, box, cnt, &A, &mb))) return e;
  const int64_t M = N - N_old;
  // few new rows (latency): every one on a block; else pass 1 with the heavy-row hand-off at
  // a lower threshold than the full recompute's (the GPU is not full: latency decides)
  A.heavy_items = nb_heavy_items(M <= NB_UPDATE_ALL_BLOCKS ? -1 : NB_HEAVY_UPDATE);
  const int ib = (int)std::min<int64_t>((M + 255) / 256 + 1, 4 * (int64_t)c->sms);
  if (A.heavy_items < 0) {
    k_nb_iota<<<ib, 256, 0, c->stream>>>(A.heavy_ids, N_old, M, A.n_heavy);
    ++c->launches;
  } else {
    k_nb_iota<<<ib, 256, 0, c->stream>>>(list, N_old, M, nullptr);
    ++c->launches;
    A.order = list;
    A.n_work = M;
    if ((e = cudaMemsetAsync(A.work, 0, sizeof(int32_t), c->stream))) return e;
    const int mb1 = (int)std::max<int64_t>(1, std::min<int64_t>((M + NB_WARPS - 1) / NB_WARPS, mb));
    k_nb_pass1<<<mb1, 32 * NB_WARPS, 0, c->stream>>>(A);
    ++c->launches;
  }
  if ((e = nb_launch_heavy(c, A, M))) return e;
  k_nb_newlen<<<(int)std::min<int64_t>((M + 255) / 256 + 1, 4 * (int64_t)c->sms), 256, 0,
                c->stream>>>(N_old, N, cnt, len);
  ++c->launches;
  const int eb = (int)std::max<int64_t>(1, std::min<int64_t>((N_old + NB_AT - 1) / NB_AT,
                                                             8 * (int64_t)c->sms));
  k_nb_extend<false><<<eb, NB_AT, 0, c->stream>>>(N_old, N, sph, c->nb_ball.as<double4>(),
                                                  nb_margin(box), old_off, len, flag, nullptr,
                                                  nullptr);
  ++c->launches;
  if ((e = launch_flag_list(c, flag, N_old, list, misc, -1))) return e;  // (the count)
  if ((e = launch_scan_i32(c, len, off, N))) return e;
  return cudaGetLastError();
}

// Part 2: the new long rows (pass 2) and the merged, ascending CSR
cudaError_t launch_nb_update2(rpd_ctx* c, const double* sph, int64_t N, int64_t N_old,
                              const double box[6], int32_t* cnt, const int32_t* len,
                              const int32_t* old_off, const int32_t* old_idx, const int32_t* off,
                              int32_t* tmp, int32_t* idx) {
  cudaError_t e = launch_neighbors_pass2_rows(c, sph, N, box, cnt, off, tmp);
  if (e) return e;
  const int sb = (int)std::min<int64_t>((N * 32 + 255) / 256, 16 * (int64_t)c->sms);
  k_nb_merge<<<sb > 0 ? sb : 1, 256, 0, c->stream>>>(N, N_old, len, old_off, old_idx, off,
                                                      c->nb_slab, tmp, idx);
  ++c->launches;
  const int eb = (int)std::max<int64_t>(1, std::min<int64_t>((N_old + NB_AT - 1) / NB_AT,
                                                             8 * (int64_t)c->sms));
  k_nb_extend<true><<<eb, NB_AT, 0, c->stream>>>(N_old, N, sph, c->nb_ball.as<double4>(),
                                                 nb_margin(box), old_off, nullptr, nullptr, off,
                                                 idx);
  ++c->launches;
  return cudaGetLastError();
}

}  // namespace rpd
