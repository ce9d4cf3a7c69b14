// rpd_envelope.cu -- SURVEY.md §8(f) NEXT-4: geometry preservation, the paper's second GPU
// workload (Sec. 4.3): "For each surface sample, we compute its distance to
// the closest enveloping volume of the medial mesh (sphere, cone, slab ...) in GPU".
//
// A medial cone is the family of spheres linearly interpolated between two medial spheres, a
// slab between three.  The value of a primitive at p is
//     g = min over the interpolation parameters of |p - c| - r,
// convex in the parameters; the envelope distance of a sample is max(min over primitives, 0).
// Closed forms (fp64):
//   sphere  g = |p - c| - r
//   cone    with d = c2 - c1, L = |d|, dr = r2 - r1, q = p - c1, a = q.d / L, h = dist to the
//           axis: the stationary t = (a + dr h / sqrt(L^2 - dr^2)) / L (|n.d| = -dr for the unit
//           normal n of the tangent direction), clamped to [0, 1] (1-D convex); if |dr| >= L one
//           end sphere contains the other: the better end
//   slab    the unit normal n of the stationary sphere satisfies n.e1 = -dr1, n.e2 = -dr2 (its
//           in-plane part from the 2x2 Gram system), its out-of-plane part points to p's side;
//           the touching centre c = p - rho n lies in the plane; if its (u, v) is inside the
//           triangle that is the minimum, otherwise the minimum is on one of the three cones.
//
// B200 mapping: samples and primitives are sorted by the Morton code of their position (CUB
// radix sort, a library primitive; primitives by kind first), primitives in tiles of 32 of
// one kind with the boxes of their balls and of their centres.  A warp takes 32
// Morton-consecutive samples (lane = sample) and, per kind (spheres first: cheap, and a good
// first bound), walks that kind's tiles outward from its own place in the Morton order.  A
// tile is skipped when every lane's lower bound exceeds the lane's best: outside the box of
// the balls the distance to it (a cone or slab is the convex hull of its balls), inside the
// distance to the box of the centres minus the largest radius.  Otherwise each lane loads one
// member and the warp evaluates all 32 members for each needing sample in turn, with a warp
// min-reduce of (value, id): no idle lanes, no divergence by kind.  Work per evaluated
// (sample, primitive) pair: ~10 (sphere), ~40 (cone), ~100 (slab) fp64 flops plus 1-5 fp64
// square roots and divisions.
#include <cub/cub.cuh>

#include "rpd_ctx.h"

namespace rpd {

static inline unsigned nblk(int64_t n, int b) { return (unsigned)((n + b - 1) / b); }

constexpr int ENV_TILE = 32;
#ifndef RPD_ENV_SMEM
#define RPD_ENV_SMEM 1  // members' records read from shared memory (fewer registers)
#endif
constexpr int ENV_WARPS = 4;

struct EnvPrim {      // one primitive: up to three spheres (x, y, z, r); kind = #spheres - 1
  double s[3][4];
  double k[12];       // per-primitive constants of the closed forms (env_prep)
  double ek[3][3];    // slab: the constants k0..k2 of its three edge cones (s0s1, s0s2, s1s2)
  int kind, id;       // id: the primitive's index in the caller's numbering
};

struct EnvTile {      // box of the tile's balls (centre -/+ radius), of its centres, largest radius
  double lo[3], hi[3], clo[3], chi[3], rmax;
  int first, count, kind;
};

__device__ __forceinline__ double env_norm(double x, double y, double z) {
  return sqrt(fma(x, x, fma(y, y, z * z)));
}

__device__ __forceinline__ double env_sphere(const double* p, const double* s) {
  return env_norm(p[0] - s[0], p[1] - s[1], p[2] - s[2]) - s[3];
}

__device__ double env_cone(const double* p, const double* s1, const double* s2) {
  const double d0 = s2[0] - s1[0], d1 = s2[1] - s1[1], d2 = s2[2] - s1[2];
  const double dr = s2[3] - s1[3];
  const double L2 = fma(d0, d0, fma(d1, d1, d2 * d2));
  if (!(dr * dr < L2))  // nested end spheres (or coincident centres): the better end
    return fmin(env_sphere(p, s1), env_sphere(p, s2));
  const double q0 = p[0] - s1[0], q1 = p[1] - s1[1], q2 = p[2] - s1[2];
  const double L = sqrt(L2);
  const double a = fma(q0, d0, fma(q1, d1, q2 * d2)) / L;
  const double h = sqrt(fmax(fma(q0, q0, fma(q1, q1, q2 * q2)) - a * a, 0.0));
  double t = (a + dr * h / sqrt(L2 - dr * dr)) / L;
  t = fmin(fmax(t, 0.0), 1.0);
  // (the clamped stationary point is the minimum of the convex g(t) on [0, 1], the ends
  // included)
  return env_norm(q0 - t * d0, q1 - t * d1, q2 - t * d2) - fma(t, dr, s1[3]);
}

__device__ double env_slab(const double* p, const double* s1, const double* s2,
                           const double* s3) {
  const double e1[3] = {s2[0] - s1[0], s2[1] - s1[1], s2[2] - s1[2]};
  const double e2[3] = {s3[0] - s1[0], s3[1] - s1[1], s3[2] - s1[2]};
  const double dr1 = s2[3] - s1[3], dr2 = s3[3] - s1[3];
  const double g11 = fma(e1[0], e1[0], fma(e1[1], e1[1], e1[2] * e1[2]));
  const double g12 = fma(e1[0], e2[0], fma(e1[1], e2[1], e1[2] * e2[2]));
  const double g22 = fma(e2[0], e2[0], fma(e2[1], e2[1], e2[2] * e2[2]));
  const double det = g11 * g22 - g12 * g12;
  // the minimum is the interior stationary point when it exists inside the triangle (g is
  // convex), otherwise on the boundary: the three cones
#define EDGES fmin(env_cone(p, s1, s2), fmin(env_cone(p, s1, s3), env_cone(p, s2, s3)))
  if (!(det > 1e-14 * g11 * g22)) return EDGES;  // (nearly) collinear centres
  // in-plane part of the stationary sphere's unit normal: G [al, be] = [-dr1, -dr2]
  const double al = (-dr1 * g22 + dr2 * g12) / det, be = (-dr2 * g11 + dr1 * g12) / det;
  const double np2 = -al * dr1 - be * dr2;  // |n_plane|^2
  if (!(np2 < 1.0)) return EDGES;
  double N[3] = {e1[1] * e2[2] - e1[2] * e2[1], e1[2] * e2[0] - e1[0] * e2[2],
                 e1[0] * e2[1] - e1[1] * e2[0]};
  const double nl = env_norm(N[0], N[1], N[2]);
  N[0] /= nl;
  N[1] /= nl;
  N[2] /= nl;
  const double q[3] = {p[0] - s1[0], p[1] - s1[1], p[2] - s1[2]};
  const double z = fma(q[0], N[0], fma(q[1], N[1], q[2] * N[2]));
  if (z == 0.0) return EDGES;
  const double w = sqrt(1.0 - np2);
  const double rho = fabs(z) / w;
  const double sg = z > 0.0 ? 1.0 : -1.0;
  double c[3];  // touching centre relative to s1: q - rho n
#pragma unroll
  for (int k = 0; k < 3; ++k) c[k] = q[k] - rho * (al * e1[k] + be * e2[k] + sg * w * N[k]);
  const double b1 = fma(c[0], e1[0], fma(c[1], e1[1], c[2] * e1[2]));
  const double b2 = fma(c[0], e2[0], fma(c[1], e2[1], c[2] * e2[2]));
  const double u = (b1 * g22 - b2 * g12) / det, v = (b2 * g11 - b1 * g12) / det;
  if (u >= 0.0 && v >= 0.0 && u + v <= 1.0) return rho - (s1[3] + u * dr1 + v * dr2);
  return EDGES;
#undef EDGES
}

// Per-primitive constants, so that an evaluation needs no division and at most two square
// roots (the interior case of a slab none):
//   cone  k0 = 1 / L^2, k1 = dr / (L sqrt(L^2 - dr^2)), k2 = 1 if the end spheres are nested:
//         t = (q.d) k0 + k1 h, h = sqrt(|q|^2 - (q.d)^2 k0)
//   slab  k0..2 = the inverse Gram matrix (i11, i12, i22), k3..5 = the in-plane part of the
//         stationary normal, k6..8 = the unit plane normal N, k9 = w = sqrt(1 - |n_plane|^2),
//         k10 = 1 / w, k11 = 1 if an interior stationary point can exist
__device__ void cone_consts(const double* s1, const double* s2, double* k) {
  const double d0 = s2[0] - s1[0], d1 = s2[1] - s1[1], d2 = s2[2] - s1[2];
  const double dr = s2[3] - s1[3];
  const double L2 = d0 * d0 + d1 * d1 + d2 * d2;
  k[0] = k[1] = k[2] = 0.0;
  if (!(dr * dr < L2)) {
    k[2] = 1.0;
    return;
  }
  k[0] = 1.0 / L2;
  k[1] = dr / (sqrt(L2) * sqrt(L2 - dr * dr));
}

__device__ __forceinline__ double cone_eval(const double* p, const double* s1, const double* s2,
                                            const double* k) {
  if (k[2] != 0.0) return fmin(env_sphere(p, s1), env_sphere(p, s2));
  const double d0 = s2[0] - s1[0], d1 = s2[1] - s1[1], d2 = s2[2] - s1[2];
  const double q0 = p[0] - s1[0], q1 = p[1] - s1[1], q2 = p[2] - s1[2];
  const double qd = fma(q0, d0, fma(q1, d1, q2 * d2));
  const double h = sqrt(fmax(fma(q0, q0, fma(q1, q1, q2 * q2)) - qd * qd * k[0], 0.0));
  const double t = fmin(fmax(fma(qd, k[0], k[1] * h), 0.0), 1.0);
  return env_norm(q0 - t * d0, q1 - t * d1, q2 - t * d2) - fma(t, s2[3] - s1[3], s1[3]);
}

__device__ void env_prep(EnvPrim& e) {
  for (int q = 0; q < 12; ++q) e.k[q] = 0.0;
  if (e.kind == 2) {
    cone_consts(e.s[0], e.s[1], e.ek[0]);
    cone_consts(e.s[0], e.s[2], e.ek[1]);
    cone_consts(e.s[1], e.s[2], e.ek[2]);
  }
  if (e.kind == 1) {
    const double* s1 = e.s[0];
    const double* s2 = e.s[1];
    const double d0 = s2[0] - s1[0], d1 = s2[1] - s1[1], d2 = s2[2] - s1[2];
    const double dr = s2[3] - s1[3];
    const double L2 = d0 * d0 + d1 * d1 + d2 * d2;
    if (!(dr * dr < L2)) {
      e.k[2] = 1.0;
      return;
    }
    e.k[0] = 1.0 / L2;
    e.k[1] = dr / (sqrt(L2) * sqrt(L2 - dr * dr));
  } else if (e.kind == 2) {
    const double* s1 = e.s[0];
    const double e1[3] = {e.s[1][0] - s1[0], e.s[1][1] - s1[1], e.s[1][2] - s1[2]};
    const double e2[3] = {e.s[2][0] - s1[0], e.s[2][1] - s1[1], e.s[2][2] - s1[2]};
    const double dr1 = e.s[1][3] - s1[3], dr2 = e.s[2][3] - s1[3];
    const double g11 = e1[0] * e1[0] + e1[1] * e1[1] + e1[2] * e1[2];
    const double g12 = e1[0] * e2[0] + e1[1] * e2[1] + e1[2] * e2[2];
    const double g22 = e2[0] * e2[0] + e2[1] * e2[1] + e2[2] * e2[2];
    const double det = g11 * g22 - g12 * g12;
    if (!(det > 1e-14 * g11 * g22)) return;  // (nearly) collinear centres: edges only
    const double al = (-dr1 * g22 + dr2 * g12) / det, be = (-dr2 * g11 + dr1 * g12) / det;
    const double np2 = -al * dr1 - be * dr2;
    if (!(np2 < 1.0)) return;
    double N[3] = {e1[1] * e2[2] - e1[2] * e2[1], e1[2] * e2[0] - e1[0] * e2[2],
                   e1[0] * e2[1] - e1[1] * e2[0]};
    const double nl = sqrt(N[0] * N[0] + N[1] * N[1] + N[2] * N[2]);
    e.k[0] = g22 / det;
    e.k[1] = -g12 / det;
    e.k[2] = g11 / det;
    for (int c = 0; c < 3; ++c) {
      e.k[3 + c] = al * e1[c] + be * e2[c];
      e.k[6 + c] = N[c] / nl;
    }
    e.k[9] = sqrt(1.0 - np2);
    e.k[10] = 1.0 / e.k[9];
    e.k[11] = 1.0;
  }
}

__device__ __forceinline__ double env_cone_k(const double* p, const EnvPrim& e) {
  const double* s1 = e.s[0];
  const double* s2 = e.s[1];
  if (e.k[2] != 0.0) return fmin(env_sphere(p, s1), env_sphere(p, s2));
  const double d0 = s2[0] - s1[0], d1 = s2[1] - s1[1], d2 = s2[2] - s1[2];
  const double q0 = p[0] - s1[0], q1 = p[1] - s1[1], q2 = p[2] - s1[2];
  const double qd = fma(q0, d0, fma(q1, d1, q2 * d2));
  const double h = sqrt(fmax(fma(q0, q0, fma(q1, q1, q2 * q2)) - qd * qd * e.k[0], 0.0));
  const double t = fmin(fmax(fma(qd, e.k[0], e.k[1] * h), 0.0), 1.0);
  return env_norm(q0 - t * d0, q1 - t * d1, q2 - t * d2) - fma(t, s2[3] - s1[3], s1[3]);
}

__device__ __forceinline__ double env_slab_k(const double* p, const EnvPrim& e) {
  const double* s1 = e.s[0];
  if (e.k[11] != 0.0) {
    const double q[3] = {p[0] - s1[0], p[1] - s1[1], p[2] - s1[2]};
    const double z = fma(q[0], e.k[6], fma(q[1], e.k[7], q[2] * e.k[8]));
    if (z != 0.0) {
      const double rho = fabs(z) * e.k[10];
      const double sw = z > 0.0 ? e.k[9] : -e.k[9];
      double c[3];
#pragma unroll
      for (int a = 0; a < 3; ++a) c[a] = q[a] - rho * fma(sw, e.k[6 + a], e.k[3 + a]);
      const double b1 = (c[0] * (e.s[1][0] - s1[0]) + c[1] * (e.s[1][1] - s1[1])) +
                        c[2] * (e.s[1][2] - s1[2]);
      const double b2 = (c[0] * (e.s[2][0] - s1[0]) + c[1] * (e.s[2][1] - s1[1])) +
                        c[2] * (e.s[2][2] - s1[2]);
      const double u = fma(e.k[0], b1, e.k[1] * b2), v = fma(e.k[1], b1, e.k[2] * b2);
      if (u >= 0.0 && v >= 0.0 && u + v <= 1.0)
        return rho - (s1[3] + u * (e.s[1][3] - s1[3]) + v * (e.s[2][3] - s1[3]));
    }
  }
  return fmin(cone_eval(p, e.s[0], e.s[1], e.ek[0]),
              fmin(cone_eval(p, e.s[0], e.s[2], e.ek[1]), cone_eval(p, e.s[1], e.s[2], e.ek[2])));
}

__device__ __forceinline__ double env_eval(const double* p, const EnvPrim& e) {
  if (e.kind == 0) return env_sphere(p, e.s[0]);
  if (e.kind == 1) return env_cone_k(p, e);
  return env_slab_k(p, e);
}

// ---- Morton ordering

__device__ __forceinline__ unsigned long long spread3(unsigned long long x) {  // 20 bits used
  x &= 0x1fffffull;
  x = (x | x << 32) & 0x1f00000000ffffull;
  x = (x | x << 16) & 0x1f0000ff0000ffull;
  x = (x | x << 8) & 0x100f00f00f00f00full;
  x = (x | x << 4) & 0x10c30c30c30c30c3ull;
  x = (x | x << 2) & 0x1249249249249249ull;
  return x;
}

__device__ __forceinline__ unsigned long long morton(const double* x, const double* lo,
                                                     double inv) {
  unsigned long long m = 0;
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    double f = (x[k] - lo[k]) * inv;
    f = fmin(fmax(f, 0.0), 1048575.0);
    m |= spread3((unsigned long long)f) << k;
  }
  return m;
}

// primitives of one kind -> records + Morton keys of their centroid (kind in the top bits)
__global__ void k_env_prims(int kind, int64_t n, int64_t id0, const double* __restrict__ sph,
                            const int32_t* __restrict__ ids, EnvPrim* __restrict__ prims,
                            unsigned long long* __restrict__ keys, int32_t* __restrict__ idx,
                            const double* __restrict__ box, int64_t out0) {
  const int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (x >= n) return;
  EnvPrim e;
  e.kind = kind;
  e.id = (int)(id0 + x);
  double cen[3] = {0.0, 0.0, 0.0};
  for (int a = 0; a < 3; ++a) {
    const int64_t sid = kind == 0 ? x : (a <= kind ? (int64_t)ids[(kind + 1) * x + a] : -1);
    const int64_t src = sid >= 0 ? sid : (kind == 0 ? x : (int64_t)ids[(kind + 1) * x]);
#pragma unroll
    for (int c = 0; c < 4; ++c) e.s[a][c] = sph[4 * src + c];
    if (a <= kind)
#pragma unroll
      for (int c = 0; c < 3; ++c) cen[c] += e.s[a][c] / (kind + 1);
  }
  env_prep(e);
  prims[out0 + x] = e;
  keys[out0 + x] = ((unsigned long long)kind << 62) | morton(cen, box, box[3]);
  idx[out0 + x] = (int32_t)(out0 + x);
}

__global__ void k_env_sample_keys(int64_t S, const double* __restrict__ smp,
                                  const double* __restrict__ box,
                                  unsigned long long* __restrict__ keys,
                                  int32_t* __restrict__ idx) {
  const int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (x >= S) return;
  keys[x] = morton(smp + 3 * x, box, box[3]);
  idx[x] = (int32_t)x;
}

// every sphere id of the cones and slabs in [0, N)
__global__ void k_env_check(int64_t n, const int32_t* __restrict__ ids, int64_t N, int* err) {
  const int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (x < n && (ids[x] < 0 || ids[x] >= N) && atomicCAS(err, 0, (int)RPD_EINVAL) == 0) {
    err[1] = ERR_NBR_INDEX;
    err[2] = (int)x;
  }
}

// bounding box of the samples and sphere centres (lo[3], 1 / cell) -- one block
__global__ void k_env_box(int64_t S, const double* __restrict__ smp, int64_t N,
                          const double* __restrict__ sph, double* __restrict__ box) {
  double lo[3] = {1e300, 1e300, 1e300}, hi[3] = {-1e300, -1e300, -1e300};
  for (int64_t x = threadIdx.x; x < S + N; x += blockDim.x) {
    const double* v = x < S ? smp + 3 * x : sph + 4 * (x - S);
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      lo[c] = fmin(lo[c], v[c]);
      hi[c] = fmax(hi[c], v[c]);
    }
  }
  __shared__ double s_lo[3][32], s_hi[3][32];
#pragma unroll
  for (int c = 0; c < 3; ++c)
    for (int o = 16; o > 0; o >>= 1) {
      lo[c] = fmin(lo[c], __shfl_xor_sync(0xffffffffu, lo[c], o));
      hi[c] = fmax(hi[c], __shfl_xor_sync(0xffffffffu, hi[c], o));
    }
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  if (l == 0)
    for (int c = 0; c < 3; ++c) {
      s_lo[c][w] = lo[c];
      s_hi[c][w] = hi[c];
    }
  __syncthreads();
  if (threadIdx.x == 0) {
    double ext = 0.0;
    for (int c = 0; c < 3; ++c) {
      double a = s_lo[c][0], b = s_hi[c][0];
      for (int k = 1; k < (int)(blockDim.x >> 5); ++k) {
        a = fmin(a, s_lo[c][k]);
        b = fmax(b, s_hi[c][k]);
      }
      box[c] = a;
      ext = fmax(ext, b - a);
    }
    box[3] = ext > 0.0 ? 1048575.0 / ext : 1.0;  // 20 bits per axis (the kind in bits 62-63)
  }
}

struct TileRanges {
  int64_t tb[4];   // kind k owns tiles [tb[k], tb[k+1])
  int64_t pb[4];   // and sorted primitives [pb[k], pb[k+1])
  int64_t sb[4];   // and super tiles [sb[k], sb[k+1]) (ENV_SUP consecutive tiles each)
};

#ifndef RPD_ENV_SUP
#define RPD_ENV_SUP 16  // tiles per super tile (0: no super tiles; A/B knob)
#endif
constexpr int ENV_SUP = RPD_ENV_SUP > 0 ? RPD_ENV_SUP : 1;

constexpr unsigned long long MORTON_MASK = (1ull << 62) - 1ull;

// tiles of ENV_TILE consecutive Morton-sorted primitives of one kind (the sort key leads with
// the kind), with the box of their balls
__global__ void k_env_tiles(TileRanges R, const EnvPrim* __restrict__ prims,
                            const int32_t* __restrict__ order,
                            const unsigned long long* __restrict__ keys,
                            EnvPrim* __restrict__ sorted, EnvTile* __restrict__ tiles,
                            unsigned long long* __restrict__ tile_key) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= R.tb[3]) return;
  int kind = 0;
  while (kind < 2 && t >= R.tb[kind + 1]) ++kind;
  const int64_t begin = R.pb[kind] + (t - R.tb[kind]) * ENV_TILE;
  const int64_t end = min(begin + ENV_TILE, R.pb[kind + 1]);
  EnvTile T;
  for (int c = 0; c < 3; ++c) {
    T.lo[c] = T.clo[c] = 1e300;
    T.hi[c] = T.chi[c] = -1e300;
  }
  T.rmax = -1e300;
  T.first = (int)begin;
  T.count = (int)(end - begin);
  T.kind = kind;
  for (int64_t x = begin; x < end; ++x) {
    const EnvPrim e = prims[order[x]];
    sorted[x] = e;
    for (int a = 0; a <= e.kind; ++a) {
      for (int c = 0; c < 3; ++c) {  // box of the balls: it holds their convex hull
        T.lo[c] = fmin(T.lo[c], e.s[a][c] - e.s[a][3]);
        T.hi[c] = fmax(T.hi[c], e.s[a][c] + e.s[a][3]);
        T.clo[c] = fmin(T.clo[c], e.s[a][c]);
        T.chi[c] = fmax(T.chi[c], e.s[a][c]);
      }
      T.rmax = fmax(T.rmax, e.s[a][3]);
    }
  }
  tiles[t] = T;
  tile_key[t] = keys[begin] & MORTON_MASK;
}

// super tiles: ENV_SUP consecutive tiles of one kind, the union of their boxes and their
// largest radius (first / count: the tile range)
__global__ void k_env_supers(TileRanges R, const EnvTile* __restrict__ tiles,
                             EnvTile* __restrict__ sup) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= R.sb[3]) return;
  int kind = 0;
  while (kind < 2 && t >= R.sb[kind + 1]) ++kind;
  const int64_t begin = R.tb[kind] + (t - R.sb[kind]) * ENV_SUP;
  const int64_t end = min(begin + (int64_t)ENV_SUP, R.tb[kind + 1]);
  EnvTile U;
  for (int c = 0; c < 3; ++c) {
    U.lo[c] = U.clo[c] = 1e300;
    U.hi[c] = U.chi[c] = -1e300;
  }
  U.rmax = -1e300;
  U.first = (int)begin;
  U.count = (int)(end - begin);
  U.kind = kind;
  for (int64_t x = begin; x < end; ++x) {
    const EnvTile T = tiles[x];
    for (int c = 0; c < 3; ++c) {
      U.lo[c] = fmin(U.lo[c], T.lo[c]);
      U.hi[c] = fmax(U.hi[c], T.hi[c]);
      U.clo[c] = fmin(U.clo[c], T.clo[c]);
      U.chi[c] = fmax(U.chi[c], T.chi[c]);
    }
    U.rmax = fmax(U.rmax, T.rmax);
  }
  sup[t] = U;
}

// a lower bound of the value of every member under box T at p: outside the box of the balls
// the distance to it (a member lies in the convex hull of its balls, inside that box); inside,
// the distance to the box of the centres minus the largest radius.  Valid for a super tile's
// union boxes as well (every member lies in one of its tiles' boxes).
__device__ __forceinline__ double env_tile_lb(const EnvTile& T, const double* p) {
  const double db = env_norm(fmax(fmax(T.lo[0] - p[0], p[0] - T.hi[0]), 0.0),
                             fmax(fmax(T.lo[1] - p[1], p[1] - T.hi[1]), 0.0),
                             fmax(fmax(T.lo[2] - p[2], p[2] - T.hi[2]), 0.0));
  if (db > 0.0) return db;
  return env_norm(fmax(fmax(T.clo[0] - p[0], p[0] - T.chi[0]), 0.0),
                  fmax(fmax(T.clo[1] - p[1], p[1] - T.chi[1]), 0.0),
                  fmax(fmax(T.clo[2] - p[2], p[2] - T.chi[2]), 0.0)) -
         T.rmax;
}

// One warp per 32 Morton-consecutive samples (lane = sample).  Per kind (spheres, then cones,
// then slabs) the kind's tiles are visited outward from the warp's place in their Morton
// order; a tile is skipped when for every lane the distance to the box of its balls exceeds
// the lane's best (a cone or slab is the convex hull of its balls, so that distance bounds
// every member's value), else every lane loads one member and the warp evaluates the 32
// members for each sample that needs the tile in turn (one member per lane, a warp min-reduce
// of (value, id)): full lanes whatever the number of samples needing the tile.
__global__ void __launch_bounds__(ENV_WARPS * 32) k_env_dist(
    int64_t S, const double* __restrict__ smp, const int32_t* __restrict__ sorder,
    const unsigned long long* __restrict__ skey, TileRanges R,
    const EnvTile* __restrict__ tiles, const unsigned long long* __restrict__ tile_key,
    const EnvTile* __restrict__ sup, const EnvPrim* __restrict__ prims, double* __restrict__ g_out,
    int32_t* __restrict__ prim_out, unsigned long long* __restrict__ n_eval) {
  const unsigned FULL = 0xffffffffu;
  const int lane = threadIdx.x & 31;
#if RPD_ENV_SMEM
  __shared__ EnvPrim s_rec[ENV_WARPS][ENV_TILE];
  EnvPrim& e_sm = s_rec[threadIdx.x >> 5][lane];
#endif
  const int64_t gw = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  unsigned long long evals = 0;
  for (int64_t base = gw * 32; base < S; base += nw * 32) {
    const int64_t si = base + lane;
    const bool valid = si < S;
    const int64_t o = valid ? sorder[si] : 0;
    const double p[3] = {valid ? smp[3 * o] : 0.0, valid ? smp[3 * o + 1] : 0.0,
                         valid ? smp[3 * o + 2] : 0.0};
    double best = valid ? 1e300 : -1e300;
    int arg = 0x7fffffff;
    const unsigned long long k0 = skey[base];
    for (int kind = 0; kind < 3; ++kind) {
      const int64_t lo_t = R.tb[kind], hi_t = R.tb[kind + 1];
      if (lo_t == hi_t) continue;
      int64_t lo = lo_t, hi = hi_t;
      while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        if (tile_key[mid] <= k0) lo = mid + 1;
        else hi = mid;
      }
      const int64_t t0 = lo > lo_t ? lo - 1 : lo_t;
      // super tiles outward from the warp's place (RPD_ENV_SUP > 0), each needed one's tiles
      // in order; or every tile outward (RPD_ENV_SUP = 0).  Any visiting order and any valid
      // culling give the same result: a culled member's value exceeds the lane's best
      const bool use_sup = RPD_ENV_SUP > 0;
      const int64_t lo_u = use_sup ? R.sb[kind] : lo_t, hi_u = use_sup ? R.sb[kind + 1] : hi_t;
      const int64_t u0 = use_sup ? R.sb[kind] + (t0 - lo_t) / ENV_SUP : t0;
      int64_t t = 0, t_end = 0;  // the current super tile's remaining tiles
      for (int64_t j = 0;;) {
        if (t >= t_end) {  // next super tile (or tile) outward
          const int64_t up = u0 + (j >> 1), dn = u0 - 1 - (j >> 1);
          if (up >= hi_u && dn < lo_u) break;
          const int64_t u = (j & 1) ? dn : up;
          ++j;
          if (u < lo_u || u >= hi_u) continue;
          if (!use_sup) {
            t = u;
            t_end = u + 1;
          } else {
            const EnvTile U = sup[u];
            const bool need_u = env_tile_lb(U, p) <= best + 1e-9 * (fabs(best) + 1.0);
            if (!__any_sync(FULL, need_u)) continue;
            t = U.first;
            t_end = U.first + U.count;
          }
        }
        const EnvTile T = tiles[t++];
        // (exact up to rounding: a small margin keeps the culling safe)
        const bool need = env_tile_lb(T, p) <= best + 1e-9 * (fabs(best) + 1.0);
        unsigned m = __ballot_sync(FULL, need);
        if (!m) continue;
        const bool has = lane < T.count;
#if RPD_ENV_SMEM
        __syncwarp();
        if (has) e_sm = prims[T.first + lane];
        __syncwarp();
        const EnvPrim& e = e_sm;
#else
        EnvPrim e;
        if (has) e = prims[T.first + lane];
        else e.kind = kind;
#endif
        const int my_id = has ? e.id : 0x7fffffff;
        evals += (unsigned long long)__popc(m) * T.count;
        while (m) {
          const int l = __ffs(m) - 1;
          m &= m - 1;
          const double q[3] = {__shfl_sync(FULL, p[0], l), __shfl_sync(FULL, p[1], l),
                               __shfl_sync(FULL, p[2], l)};
          double g = has ? env_eval(q, e) : 1e300;
          int id = my_id;
#pragma unroll
          for (int off = 16; off > 0; off >>= 1) {
            const double og = __shfl_xor_sync(FULL, g, off);
            const int oid = __shfl_xor_sync(FULL, id, off);
            if (og < g || (og == g && oid < id)) {
              g = og;
              id = oid;
            }
          }
          if (lane == l && (g < best || (g == best && id < arg))) {
            best = g;
            arg = id;
          }
        }
      }
    }
    if (valid) {
      g_out[o] = best;
      prim_out[o] = arg;
    }
  }
  if (lane == 0 && evals) atomicAdd(n_eval, evals);
}

// validation of the primitives' sphere ids (before any kernel dereferences them)
cudaError_t launch_envelope_check(rpd_ctx* c, int64_t N, const int32_t* edges, int64_t NE,
                                  const int32_t* faces, int64_t NF) {
  if (NE > 0) {
    k_env_check<<<nblk(2 * NE, 256), 256, 0, c->stream>>>(2 * NE, edges, N, c->errw.as<int>());
    ++c->launches;
  }
  if (NF > 0) {
    k_env_check<<<nblk(3 * NF, 256), 256, 0, c->stream>>>(3 * NF, faces, N, c->errw.as<int>());
    ++c->launches;
  }
  return cudaGetLastError();
}

template <class K, class V>
static cudaError_t sort_pairs(rpd_ctx* c, K* k_in, K* k_out, V* v_in, V* v_out, int64_t n) {
  size_t bytes = 0;
  cudaError_t e = cub::DeviceRadixSort::SortPairs(nullptr, bytes, k_in, k_out, v_in, v_out,
                                                  (int)n, 0, 64, c->stream);
  if (e) return e;
  if ((e = c->mm_tmp.ensure(bytes))) return e;
  bytes = c->mm_tmp.cap;
  e = cub::DeviceRadixSort::SortPairs(c->mm_tmp.p, bytes, k_in, k_out, v_in, v_out, (int)n, 0,
                                      64, c->stream);
  ++c->launches;
  return e;
}

cudaError_t launch_envelope(rpd_ctx* c, const double* smp, int64_t S, const double* sph,
                            int64_t N, const int32_t* edges, int64_t NE, const int32_t* faces,
                            int64_t NF, double* g_out, int32_t* prim_out,
                            unsigned long long* n_eval) {
  const int64_t P = N + NE + NF;
  TileRanges R;
  {
    const int64_t cnt[3] = {N, NE, NF};
    R.tb[0] = 0;
    R.pb[0] = 0;
    for (int k = 0; k < 3; ++k) {
      R.tb[k + 1] = R.tb[k] + (cnt[k] + ENV_TILE - 1) / ENV_TILE;
      R.pb[k + 1] = R.pb[k] + cnt[k];
    }
    R.sb[0] = 0;
    for (int k = 0; k < 3; ++k) R.sb[k + 1] = R.sb[k] + (R.tb[k + 1] - R.tb[k] + ENV_SUP - 1) / ENV_SUP;
  }
  const int64_t n_tiles = R.tb[3], n_sup = R.sb[3];
  const size_t bytes = sizeof(EnvPrim) * 2 * (P + 1) + sizeof(EnvTile) * (n_tiles + n_sup + 2) +
                       sizeof(unsigned long long) * 2 * (P + S + 2) +
                       sizeof(int32_t) * 2 * (P + S + 2) + sizeof(double) * 8 +
                       sizeof(unsigned long long) * (n_tiles + 1) + 512;
  cudaError_t e = c->env_buf.ensure(bytes);
  if (e) return e;
  char* b = c->env_buf.as<char>();
  auto take = [&](size_t n) {
    char* r = b;
    b += (n + 15) & ~size_t(15);
    return r;
  };
  EnvPrim* prims = reinterpret_cast<EnvPrim*>(take(sizeof(EnvPrim) * (P + 1)));
  EnvPrim* sorted = reinterpret_cast<EnvPrim*>(take(sizeof(EnvPrim) * (P + 1)));
  EnvTile* tiles = reinterpret_cast<EnvTile*>(take(sizeof(EnvTile) * (n_tiles + 1)));
  EnvTile* sup = reinterpret_cast<EnvTile*>(take(sizeof(EnvTile) * (n_sup + 1)));
  unsigned long long* pk = reinterpret_cast<unsigned long long*>(take(8 * (P + 1)));
  unsigned long long* pk2 = reinterpret_cast<unsigned long long*>(take(8 * (P + 1)));
  int32_t* pi = reinterpret_cast<int32_t*>(take(4 * (P + 1)));
  int32_t* pi2 = reinterpret_cast<int32_t*>(take(4 * (P + 1)));
  unsigned long long* sk = reinterpret_cast<unsigned long long*>(take(8 * (S + 1)));
  unsigned long long* sk2 = reinterpret_cast<unsigned long long*>(take(8 * (S + 1)));
  int32_t* si = reinterpret_cast<int32_t*>(take(4 * (S + 1)));
  int32_t* si2 = reinterpret_cast<int32_t*>(take(4 * (S + 1)));
  double* box = reinterpret_cast<double*>(take(sizeof(double) * 8));
  unsigned long long* tile_key = reinterpret_cast<unsigned long long*>(take(8 * (n_tiles + 1)));
  k_env_box<<<1, 1024, 0, c->stream>>>(S, smp, N, sph, box);
  ++c->launches;
  const int32_t* ids[3] = {nullptr, edges, faces};
  const int64_t cnt[3] = {N, NE, NF};
  int64_t off = 0;
  for (int k = 0; k < 3; ++k) {
    if (cnt[k] > 0) {
      k_env_prims<<<nblk(cnt[k], 256), 256, 0, c->stream>>>(k, cnt[k], off, sph, ids[k], prims,
                                                            pk, pi, box, off);
      ++c->launches;
    }
    off += cnt[k];
  }
  if (P > 0 && (e = sort_pairs(c, pk, pk2, pi, pi2, P))) return e;
  if (n_tiles > 0) {
    k_env_tiles<<<nblk(n_tiles, 128), 128, 0, c->stream>>>(R, prims, pi2, pk2, sorted, tiles,
                                                           tile_key);
    ++c->launches;
    if (RPD_ENV_SUP > 0) {
      k_env_supers<<<nblk(n_sup, 128), 128, 0, c->stream>>>(R, tiles, sup);
      ++c->launches;
    }
  }
  if (S == 0) return cudaGetLastError();
  k_env_sample_keys<<<nblk(S, 256), 256, 0, c->stream>>>(S, smp, box, sk, si);
  ++c->launches;
  if ((e = sort_pairs(c, sk, sk2, si, si2, S))) return e;
  int64_t blocks = (S + 32 * ENV_WARPS - 1) / (32 * ENV_WARPS);
  if (blocks > (int64_t)c->sms * 16) blocks = (int64_t)c->sms * 16;
  k_env_dist<<<(unsigned)blocks, ENV_WARPS * 32, 0, c->stream>>>(
      S, smp, si2, sk2, R, tiles, tile_key, sup, sorted, g_out, prim_out, n_eval);
  ++c->launches;
  return cudaGetLastError();
}

}  // namespace rpd
