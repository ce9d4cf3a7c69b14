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
// B200 mapping: one warp per pair, lane = vertex (<= 32 vertices, <= 32 planes), polytope
// in per-warp shared memory (double-buffered vertex table).  The k_site planes are first
// classified 32 at a time, one per lane, from their exact values at the 4 tet corners:
// planes with all four values > 0 cannot cut (most of them), a plane with all four < 0
// empties the piece; only the remaining planes run the per-vertex sign pass.
//
// Signs: the plane value at a vertex is g_s . K with K the fp64
// homogeneous vertex (3x3 cofactors of its planes' barycentric 4-vectors) and a running
// error bound F; |g_s . K| > |g_s|_1 * F decides it, otherwise the exact int128 path
// evaluates det[a_p; a_q; a_r; a_s] and applies the inward symbolic perturbation.
//
// Outputs per pair: non-empty flag, volume, first moment (facet fans, deterministic warp
// reduction), tet-face mask and incidences (positive-area SoS facets expanded by exactly
// coincident sources, R7).
#include "rpd_ctx.h"
#include "rpd_internal.cuh"

namespace rpd {

constexpr int CLIP_WARPS = 8;  // warps per block

struct WarpState {
  double g[RPD_MAXP][4];   // barycentric plane vectors (exact integers)
  double K[2][RPD_MAXV][4];
  double F[2][RPD_MAXV];
  double x[RPD_MAXV][3];   // final vertex coordinates (lattice units, relative to V0)
  unsigned tri[2][RPD_MAXV];
  int src[RPD_MAXP];       // radical: sphere j; tet face k: -1-k
  int eidx[RPD_MAXP];      // CSR entry of a radical plane, -1 for faces
  int ref[RPD_MAXP];       // reference vertex of every facet (fan apex)
  int inc[RPD_INC_CAP];
  int ninc;
};

// oriented dual triangles of the 4 tet corners (corner k = faces != k)
__constant__ unsigned CORNER_TRI[4] = {
    1u | (2u << 8) | (3u << 16), 0u | (3u << 8) | (2u << 16), 0u | (1u << 8) | (3u << 16),
    0u | (2u << 8) | (1u << 16)};

__device__ __forceinline__ int tri_at(unsigned tr, int k) { return (tr >> (8 * k)) & 0xff; }
__device__ __forceinline__ bool tri_has(unsigned tr, int p) {
  return tri_at(tr, 0) == p || tri_at(tr, 1) == p || tri_at(tr, 2) == p;
}
__device__ __forceinline__ unsigned tri_pack(int a, int b, int c) {
  return (unsigned)a | ((unsigned)b << 8) | ((unsigned)c << 16);
}
__device__ __forceinline__ unsigned tri_bits(unsigned tr) {
  return (1u << tri_at(tr, 0)) | (1u << tri_at(tr, 1)) | (1u << tri_at(tr, 2));
}

// vertex u != self of the current table containing planes a and b (-1 if none)
__device__ inline int find_edge_nb(const unsigned* tri, int nv, int self, int a, int b) {
  for (int u = 0; u < nv; ++u)
    if (u != self && tri_has(tri[u], a) && tri_has(tri[u], b)) return u;
  return -1;
}

struct ClipCtx {
  const double4* planes;   // global plane table (for Cartesian normals)
  long long N;             // sphere count (SoS rank of tet faces = N + k)
};

__device__ inline void make_xplane(const WarpState& S, const ClipCtx& C, int id, XPlane* xp) {
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

// fp64 homogeneous vertex of planes (a, b, c) with error bound; returns false if the sign of
// sum(K) could not be certified (caller then uses the exact vertex)
__device__ inline void vertex_from_planes(const WarpState& S, const ClipCtx& C, int a, int b,
                                          int c, double K[4], double* F, int* nexact) {
  const double* ra = S.g[a];
  const double* rb = S.g[b];
  const double* rc = S.g[c];
  double E = 0.0, Kmax = 0.0, sum = 0.0, sabs = 0.0;
#pragma unroll
  for (int m = 0; m < 4; ++m) {
    int c0 = m == 0 ? 1 : 0;
    int c1 = m <= 1 ? 2 : 1;
    int c2 = m <= 2 ? 3 : 2;
    double m0 = fma(rb[c1], rc[c2], -rb[c2] * rc[c1]);
    double m1 = fma(rb[c0], rc[c2], -rb[c2] * rc[c0]);
    double m2 = fma(rb[c0], rc[c1], -rb[c1] * rc[c0]);
    double d = fma(ra[c0], m0, fma(-ra[c1], m1, ra[c2] * m2));
    double p0 = fabs(rb[c1] * rc[c2]) + fabs(rb[c2] * rc[c1]);
    double p1 = fabs(rb[c0] * rc[c2]) + fabs(rb[c2] * rc[c0]);
    double p2 = fabs(rb[c0] * rc[c1]) + fabs(rb[c1] * rc[c0]);
    double perm = fabs(ra[c0]) * p0 + fabs(ra[c1]) * p1 + fabs(ra[c2]) * p2;
    K[m] = (m & 1) ? d : -d;  // (-1)^(3+m)
    E = fmax(E, perm);
    Kmax = fmax(Kmax, fabs(d));
    sum += K[m];
    sabs += fabs(K[m]);
  }
  E *= 10.0 * U;
  // certify sign(sum K) = sign(D3)
  double sb = (4.0 * E + 4.0 * U * sabs) * (1.0 + 1e-9);
  if (!(fabs(sum) > sb)) {
    XPlane pa, pb, pc;
    make_xplane(S, C, a, &pa);
    make_xplane(S, C, b, &pb);
    make_xplane(S, C, c, &pc);
    exact_vertex(pa, pb, pc, K);  // normalised, sum > 0
    ++*nexact;
    // exact to 2^-52 relative per component
    double km = fmax(fmax(fabs(K[0]), fabs(K[1])), fmax(fabs(K[2]), fabs(K[3])));
    *F = 4.0 * U * km * (1.0 + 1e-9) + 5.0 * U * km;
    return;
  }
  if (sum < 0.0) {
#pragma unroll
    for (int m = 0; m < 4; ++m) K[m] = -K[m];
  }
  *F = (E + 5.0 * U * Kmax) * (1.0 + 1e-9);
}

enum { ST_ALIVE = 0, ST_EMPTY = 1, ST_OVER = 2 };

struct PairOut {
  double* vol;
  double* m1;
  uint8_t* flag;
  uint8_t* fm;
  int32_t* ninc;
  int32_t* inc;
};

__global__ void __launch_bounds__(CLIP_WARPS * 32) k_clip(
    int64_t n_pairs, const int32_t* __restrict__ pair_tet, const int32_t* __restrict__ tet_ids,
    const int32_t* __restrict__ cand_idx, const double* __restrict__ tx, int64_t T,
    const int32_t* __restrict__ nbr_off, const int32_t* __restrict__ nbr_idx,
    const double4* __restrict__ planes, const int32_t* __restrict__ twin, long long N,
    PairOut out, unsigned long long* __restrict__ stats) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  WarpState& S = reinterpret_cast<WarpState*>(smem_raw)[threadIdx.x >> 5];
  const int lane = threadIdx.x & 31;
  const unsigned FULL = 0xffffffffu;
  const unsigned lt_mask = (1u << lane) - 1u;
  ClipCtx C{planes, N};
  int64_t gw = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  int n_exact = 0, n_zero = 0, max_v = 0, max_p = 0, n_over = 0;

  for (int64_t p = gw; p < n_pairs; p += nw) {
    int64_t a = pair_tet[p];
    int64_t t = tet_ids ? (int64_t)tet_ids[a] : a;
    int i = cand_idx[p];
    double V[4][3];
#pragma unroll
    for (int k = 0; k < 4; ++k)
#pragma unroll
      for (int c = 0; c < 3; ++c) V[k][c] = __ldg(tx + (3 * k + c) * T + t);

    if (lane < 4) {
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        S.g[lane][k] = (k == lane) ? 1.0 : 0.0;
        S.K[0][lane][k] = (k == lane) ? 1.0 : 0.0;
      }
      S.src[lane] = -1 - lane;
      S.eidx[lane] = -1;
      S.F[0][lane] = 0.0;
      S.tri[0][lane] = CORNER_TRI[lane];
    }
    __syncwarp();
    int np = 4, nv = 4, cur = 0, status = ST_ALIVE, zero_hit = 0;
    const int e0 = __ldg(nbr_off + i), e1 = __ldg(nbr_off + i + 1);

    for (int base = e0; base < e1 && status == ST_ALIVE; base += 32) {
      const int e = base + lane;
      const bool have = e < e1;
      double g[4] = {0.0, 0.0, 0.0, 0.0};
      bool allpos = false, allneg = false;
      if (have) {
        double4 pl = planes[e];
        allpos = true;
        allneg = true;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          g[k] = fma(pl.x, V[k][0], fma(pl.y, V[k][1], fma(pl.z, V[k][2], pl.w)));
          allpos &= g[k] > 0.0;
          allneg &= g[k] < 0.0;
        }
      }
      if (__any_sync(FULL, allneg)) {
        status = ST_EMPTY;
        break;
      }
      unsigned act = __ballot_sync(FULL, have && !allpos);
      while (act && status == ST_ALIVE) {
        const int l = __ffs(act) - 1;
        act &= act - 1;
        double s[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) s[k] = __shfl_sync(FULL, g[k], l);
        const int es = base + l;
        const double sabs = fabs(s[0]) + fabs(s[1]) + fabs(s[2]) + fabs(s[3]);

        // ---- sign of every vertex
        const bool valid = lane < nv;
        int sg = 0;
        if (valid) {
          const double* K = S.K[cur][lane];
          double val = fma(s[0], K[0], fma(s[1], K[1], fma(s[2], K[2], s[3] * K[3])));
          double B = sabs * S.F[cur][lane];
          if (val > B) sg = 1;
          else if (val < -B) sg = -1;
          else {
            // exact path
            XPlane xa, xb, xc, xs;
            unsigned tr = S.tri[cur][lane];
            make_xplane(S, C, tri_at(tr, 0), &xa);
            make_xplane(S, C, tri_at(tr, 1), &xb);
            make_xplane(S, C, tri_at(tr, 2), &xc);
#pragma unroll
            for (int k = 0; k < 4; ++k) xs.a[k] = (long long)s[k];
            double4 pl = planes[es];
            xs.n[0] = (long long)pl.x;
            xs.n[1] = (long long)pl.y;
            xs.n[2] = (long long)pl.z;
            xs.radical = 1;
            xs.rank = nbr_idx[es];
            int zh = 0;
            sg = sos_sign_exact(xa, xb, xc, xs, &zh);
            ++n_exact;
            if (zh) {
              ++n_zero;
              zero_hit = 1;
            }
          }
        }
        zero_hit = __any_sync(FULL, zero_hit);
        const unsigned negm = __ballot_sync(FULL, valid && sg < 0);
        const unsigned posm = __ballot_sync(FULL, valid && sg > 0);
        if (!negm) continue;  // plane does not cut: skip
        if (!posm) {
          status = ST_EMPTY;
          break;
        }
        if (np >= RPD_MAXP) {
          status = ST_OVER;
          break;
        }
        const int sid = np++;
        if (lane == 0) {
#pragma unroll
          for (int k = 0; k < 4; ++k) S.g[sid][k] = s[k];
          S.src[sid] = nbr_idx[es];
          S.eidx[sid] = es;
        }
        __syncwarp();
        // ---- new vertices: for every edge of a removed vertex whose neighbour is kept
        unsigned newtri[3];
        int nnew = 0;
        if (valid && sg < 0) {
          unsigned tr = S.tri[cur][lane];
#pragma unroll
          for (int r = 0; r < 3; ++r) {
            int x = tri_at(tr, r), y = tri_at(tr, (r + 1) % 3);
            int u = find_edge_nb(S.tri[cur], nv, lane, x, y);
            if (u >= 0 && ((posm >> u) & 1u)) newtri[nnew++] = tri_pack(x, y, sid);
          }
        }
        int incl = nnew;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          int y = __shfl_up_sync(FULL, incl, o);
          if (lane >= o) incl += y;
        }
        const int total_new = __shfl_sync(FULL, incl, 31);
        const int nkept = __popc(posm);
        const int nv2 = nkept + total_new;
        if (nv2 > RPD_MAXV) {
          status = ST_OVER;
          break;
        }
        const int nxt = cur ^ 1;
        if (valid && sg > 0) {
          int k = __popc(posm & lt_mask);
#pragma unroll
          for (int m = 0; m < 4; ++m) S.K[nxt][k][m] = S.K[cur][lane][m];
          S.F[nxt][k] = S.F[cur][lane];
          S.tri[nxt][k] = S.tri[cur][lane];
        }
        for (int q = 0; q < nnew; ++q) {
          int k = nkept + incl - nnew + q;
          unsigned tr = newtri[q];
          double K[4], F;
          vertex_from_planes(S, C, tri_at(tr, 0), tri_at(tr, 1), tri_at(tr, 2), K, &F, &n_exact);
#pragma unroll
          for (int m = 0; m < 4; ++m) S.K[nxt][k][m] = K[m];
          S.F[nxt][k] = F;
          S.tri[nxt][k] = tr;
        }
        nv = nv2;
        cur = nxt;
        __syncwarp();
      }
    }

    // ------------------------------------------------------------------ outputs
    if (status == ST_OVER) ++n_over;
    if (status != ST_ALIVE) {
      if (lane == 0) {
        out.flag[p] = 0;
        out.ninc[p] = 0;
      }
      __syncwarp();
      continue;
    }
    max_v = max(max_v, nv);
    max_p = max(max_p, np);
    const bool valid = lane < nv;
    const unsigned mytri = valid ? S.tri[cur][lane] : 0u;
    const unsigned facets_all = __reduce_or_sync(FULL, valid ? tri_bits(mytri) : 0u);
    unsigned facets = facets_all;

    // zero-area SoS facets (only possible after an exact-zero predicate; C1.7)
    if (zero_hit) {
      unsigned fl = facets_all;
      while (fl) {
        const int f = __ffs(fl) - 1;
        fl &= fl - 1;
        const bool onf = valid && tri_has(mytri, f);
        unsigned Q = __reduce_or_sync(FULL, onf ? tri_bits(mytri) : 0u) & ~(1u << f);
        bool zero_area = false;
        while (Q && !zero_area) {
          const int q = __ffs(Q) - 1;
          Q &= Q - 1;
          bool on = true;
          if (onf && !tri_has(mytri, q)) {
            const double* K = S.K[cur][lane];
            const double* gq = S.g[q];
            double val = fma(gq[0], K[0], fma(gq[1], K[1], fma(gq[2], K[2], gq[3] * K[3])));
            double sa = fabs(gq[0]) + fabs(gq[1]) + fabs(gq[2]) + fabs(gq[3]);
            if (fabs(val) > sa * S.F[cur][lane]) {
              on = false;
            } else {
              XPlane xa, xb, xc, xq;
              make_xplane(S, C, tri_at(mytri, 0), &xa);
              make_xplane(S, C, tri_at(mytri, 1), &xb);
              make_xplane(S, C, tri_at(mytri, 2), &xc);
              make_xplane(S, C, q, &xq);
              on = det4_is_zero(xa, xb, xc, xq);
              ++n_exact;
            }
          }
          zero_area = __all_sync(FULL, on);
        }
        if (zero_area) facets &= ~(1u << f);
      }
    }

    // incidences: every positive-area facet plus its exactly coincident sources
    if (lane == 0) S.ninc = 0;
    __syncwarp();
    unsigned fmask_bits = 0;
    if (lane < np && ((facets >> lane) & 1u)) {
      const int src = S.src[lane];
      if (src < 0) {
        fmask_bits |= 1u << (-1 - src);
      } else {
        // radical plane coinciding with tet face a: g = c e_a, c > 0
        const double* gg = S.g[lane];
        int nz = 0, az = -1;
#pragma unroll
        for (int k = 0; k < 4; ++k)
          if (gg[k] != 0.0) {
            ++nz;
            az = k;
          }
        if (nz == 1 && gg[az] > 0.0) fmask_bits |= 1u << az;
        int e = S.eidx[lane];
        while (e >= 0) {
          int slot = atomicAdd(&S.ninc, 1);
          if (slot < RPD_INC_CAP) S.inc[slot] = nbr_idx[e];
          e = twin[e];
        }
      }
    }
    const unsigned facemask = __reduce_or_sync(FULL, fmask_bits);
    __syncwarp();
    const int ninc = S.ninc;
    if (ninc > RPD_INC_CAP) {
      ++n_over;
      if (lane == 0) {
        out.flag[p] = 0;
        out.ninc[p] = 0;
      }
      __syncwarp();
      continue;
    }
    // rank sort of the incidence list (distinct ids)
    int my = lane < ninc ? S.inc[lane] : 0;
    int rank = 0;
    for (int q = 0; q < ninc; ++q) rank += S.inc[q] < my;
    __syncwarp();
    if (lane < ninc) out.inc[p * RPD_INC_CAP + rank] = my;

    // ---- geometry: vertex coordinates relative to V0 (lattice units)
    if (valid) {
      double K[4];
#pragma unroll
      for (int m = 0; m < 4; ++m) K[m] = S.K[cur][lane][m];
      double sum = K[0] + K[1] + K[2] + K[3];
      if (16.0 * S.F[cur][lane] > 1e-12 * sum) {
        XPlane xa, xb, xc;
        make_xplane(S, C, tri_at(mytri, 0), &xa);
        make_xplane(S, C, tri_at(mytri, 1), &xb);
        make_xplane(S, C, tri_at(mytri, 2), &xc);
        exact_vertex(xa, xb, xc, K);
        sum = K[0] + K[1] + K[2] + K[3];
        ++n_exact;
      }
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        double acc = 0.0;
#pragma unroll
        for (int k = 1; k < 4; ++k) acc = fma(K[k] / sum, V[k][c] - V[0][c], acc);
        S.x[lane][c] = acc;
      }
    }
    {
      unsigned fl = facets_all;
      while (fl) {
        const int f = __ffs(fl) - 1;
        fl &= fl - 1;
        unsigned on = __ballot_sync(FULL, valid && tri_has(mytri, f));
        if (lane == 0) S.ref[f] = __ffs(on) - 1;
      }
    }
    __syncwarp();
    double vol6 = 0.0, m24[3] = {0.0, 0.0, 0.0};
    if (valid) {
      const double* xv = S.x[lane];
#pragma unroll
      for (int r = 0; r < 3; ++r) {
        const int f = tri_at(mytri, r);
        const int zc = tri_at(mytri, (r + 2) % 3);
        const int w = find_edge_nb(S.tri[cur], nv, lane, zc, f);
        const int rf = S.ref[f];
        const double* xr = S.x[rf];
        const double* xw = S.x[w];
        double det = xr[0] * (xv[1] * xw[2] - xv[2] * xw[1]) -
                     xr[1] * (xv[0] * xw[2] - xv[2] * xw[0]) +
                     xr[2] * (xv[0] * xw[1] - xv[1] * xw[0]);
        vol6 += det;
#pragma unroll
        for (int c = 0; c < 3; ++c) m24[c] += det * (xr[c] + xv[c] + xw[c]);
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      vol6 += __shfl_xor_sync(FULL, vol6, o);
#pragma unroll
      for (int c = 0; c < 3; ++c) m24[c] += __shfl_xor_sync(FULL, m24[c], o);
    }
    if (lane == 0) {
      const double L = 1.0 / RPD_LATTICE;
      const double vol = (vol6 / 6.0) * (L * L * L);
      out.vol[p] = vol;
#pragma unroll
      for (int c = 0; c < 3; ++c)
        out.m1[3 * p + c] = (m24[c] / 24.0) * (L * L * L * L) + vol * (V[0][c] * L);
      out.flag[p] = 1;
      out.fm[p] = (uint8_t)facemask;
      out.ninc[p] = ninc;
    }
    __syncwarp();
  }
  // statistics (warp-aggregated)
  for (int o = 16; o > 0; o >>= 1) {
    n_exact += __shfl_xor_sync(0xffffffffu, n_exact, o);
    n_zero += __shfl_xor_sync(0xffffffffu, n_zero, o);
  }
  if (lane == 0) {
    if (n_exact) atomicAdd(stats + ST_EXACT, (unsigned long long)n_exact);
    if (n_zero) atomicAdd(stats + ST_ZERO, (unsigned long long)n_zero);
    if (n_over) atomicAdd(stats + ST_OVERFLOW, (unsigned long long)n_over);
    atomicMax(stats + ST_MAXV, (unsigned long long)max_v);
    atomicMax(stats + ST_MAXP, (unsigned long long)max_p);
  }
}

__global__ void k_compact_pieces(int64_t n_pairs, const int32_t* __restrict__ cand_idx,
                                 const uint8_t* __restrict__ flag, const int32_t* __restrict__ pscan,
                                 const int32_t* __restrict__ iscan, const double* __restrict__ pvol,
                                 const double* __restrict__ pm1, const uint8_t* __restrict__ pfm,
                                 const int32_t* __restrict__ pninc, const int32_t* __restrict__ pinc,
                                 int32_t* __restrict__ piece_sphere, double* __restrict__ piece_vol,
                                 double* __restrict__ piece_m1, uint8_t* __restrict__ piece_fm,
                                 int32_t* __restrict__ inc_off, int32_t* __restrict__ inc_sphere) {
  int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (p >= n_pairs) return;
  if (p == n_pairs - 1) inc_off[pscan[n_pairs]] = iscan[n_pairs];
  if (!flag[p]) return;
  int q = pscan[p];
  piece_sphere[q] = cand_idx[p];
  piece_vol[q] = pvol[p];
  piece_m1[3 * q + 0] = pm1[3 * p + 0];
  piece_m1[3 * q + 1] = pm1[3 * p + 1];
  piece_m1[3 * q + 2] = pm1[3 * p + 2];
  piece_fm[q] = pfm[p];
  int o = iscan[p];
  inc_off[q] = o;
  int n = pninc[p];
  for (int k = 0; k < n; ++k) inc_sphere[o + k] = pinc[p * RPD_INC_CAP + k];
}

__global__ void k_piece_off(int64_t T, const int32_t* __restrict__ cand_off,
                            const int32_t* __restrict__ pscan, int32_t* __restrict__ piece_off) {
  int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t > T) return;
  piece_off[t] = pscan[cand_off[t]];
}

static inline unsigned nblk(int64_t n, int b) { return (unsigned)((n + b - 1) / b); }

cudaError_t launch_clip(rpd_ctx* c, int64_t n_pairs, const int32_t* pair_tet,
                        const int32_t* tet_ids, const int32_t* cand_idx) {
  if (n_pairs == 0) return cudaSuccess;
  size_t smem = sizeof(WarpState) * CLIP_WARPS;
  cudaError_t e = cudaFuncSetAttribute(k_clip, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)smem);
  if (e) return e;
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, c->device);
  int occ = 1;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_clip, CLIP_WARPS * 32, smem);
  if (occ < 1) occ = 1;
  int64_t want = (n_pairs + CLIP_WARPS - 1) / CLIP_WARPS;
  int64_t grid = (int64_t)sms * occ;
  if (want < grid) grid = want;
  PairOut o{c->p_vol.as<double>(), c->p_m1.as<double>(), c->p_flag.as<uint8_t>(),
            c->p_fm.as<uint8_t>(), c->p_ninc.as<int32_t>(), c->p_inc.as<int32_t>()};
  k_clip<<<(unsigned)grid, CLIP_WARPS * 32, smem, c->stream>>>(
      n_pairs, pair_tet, tet_ids, cand_idx, c->st.tx.as<double>(), c->st.T,
      c->st.nbr_off.as<int32_t>(), c->st.nbr_idx.as<int32_t>(), c->st.planes.as<double4>(),
      c->st.twin.as<int32_t>(), (long long)c->st.N, o, c->stats.as<unsigned long long>());
  ++c->launches;
  return cudaGetLastError();
}

cudaError_t launch_piece_scans(rpd_ctx* c, int64_t n_pairs) {
  cudaError_t e = launch_scan_u8(c, c->p_flag.as<uint8_t>(), c->p_scan.as<int32_t>(), n_pairs);
  if (e) return e;
  return launch_scan_i32(c, c->p_ninc.as<int32_t>(), c->i_scan.as<int32_t>(), n_pairs);
}

cudaError_t launch_compact_pieces(rpd_ctx* c, int64_t n_tets, int64_t n_pairs,
                                  const int32_t* cand_off, const int32_t* cand_idx,
                                  const PieceDst& d) {
  if (n_pairs > 0) {
    k_compact_pieces<<<nblk(n_pairs, 256), 256, 0, c->stream>>>(
        n_pairs, cand_idx, c->p_flag.as<uint8_t>(), c->p_scan.as<int32_t>(),
        c->i_scan.as<int32_t>(), c->p_vol.as<double>(), c->p_m1.as<double>(),
        c->p_fm.as<uint8_t>(), c->p_ninc.as<int32_t>(), c->p_inc.as<int32_t>(), d.sphere, d.vol,
        d.m1, d.fm, d.inc_off, d.inc);
    ++c->launches;
  } else {
    cudaMemsetAsync(d.inc_off, 0, sizeof(int32_t), c->stream);
  }
  k_piece_off<<<nblk(n_tets + 1, 256), 256, 0, c->stream>>>(n_tets, cand_off,
                                                          c->p_scan.as<int32_t>(), d.off);
  ++c->launches;
  return cudaGetLastError();
}

}  // namespace rpd
