// rpd_stage.cu -- SURVEY.md §8(a) row a1: input validation and staging.
//
// Converts inputs to lattice units (x * 2^10, exact), gathers tet corner coordinates into a
// coalesced SoA table, builds W = |Theta|^2 - R^2 per sphere, sorts each neighbour row
// ascending, and builds the radical plane h_ij = n . X + d of every CSR entry
// (n = 2 (Theta_i - Theta_j), d = W_j - W_i) plus the
// "twin" chain of entries of the same row whose oriented planes coincide (R7).
// Every value is an integer-valued double below 2^53, so all of it is exact.
#include <math.h>

#include <utility>

#include "rpd_ctx.h"
#include "rpd_internal.cuh"

namespace rpd {

__device__ inline void report(int* err, int status, int kind, long long idx) {
  if (atomicCAS(err, 0, status) == 0) {
    err[1] = kind;
    err[2] = (int)(idx > 0x7fffffff ? 0x7fffffff : idx);
  }
}

// x real -> lattice; returns false if off the 2^-10 lattice box [0, 64)
__device__ inline bool to_lat(double x, double* X) {
  double v = x * RPD_LATTICE;
  *X = v;
  return (x >= 0.0) && (x < 64.0) && (v == rint(v));
}

__global__ void k_check_verts(const double* __restrict__ verts, int64_t n, int* err) {
  int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (k >= n) return;
  double x = verts[k], X;
  if (!isfinite(x)) report(err, RPD_EINVAL, ERR_VERT_NAN, k / 3);
  else if (!to_lat(x, &X)) report(err, RPD_ENOTEXACT, ERR_VERT_LATTICE, k / 3);
}

__global__ void k_stage_tets(const double* __restrict__ verts, int64_t V,
                             const int32_t* __restrict__ tets, int64_t T,
                             double* __restrict__ tx, int* err) {
  int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= T) return;
  double P[4][3];
  bool ok = true;
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    int32_t v = tets[4 * t + k];
    if (v < 0 || v >= V) {
      ok = false;
      v = 0;
    }
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      P[k][c] = verts[3 * (int64_t)v + c] * RPD_LATTICE;
      tx[(3 * k + c) * T + t] = P[k][c];
    }
  }
  if (!ok) {
    report(err, RPD_EINVAL, ERR_TET_INDEX, t);
    return;
  }
  // orientation: det(V1-V0, V2-V0, V3-V0) > 0, exact (integers, partial sums < 2^53)
  double a[3], b[3], d[3];
  for (int c = 0; c < 3; ++c) {
    a[c] = P[1][c] - P[0][c];
    b[c] = P[2][c] - P[0][c];
    d[c] = P[3][c] - P[0][c];
  }
  double det = a[0] * (b[1] * d[2] - b[2] * d[1]) - a[1] * (b[0] * d[2] - b[2] * d[0]) +
               a[2] * (b[0] * d[1] - b[1] * d[0]);
  if (!(det > 0.0)) report(err, RPD_EINVAL, ERR_TET_ORIENT, t);
}

// old_sw (partial updates): the previous staging of spheres [0, N_old), which must not change
// (rpd.h: new spheres are appended; their rows and planes are reused)
__global__ void k_stage_spheres(const double* __restrict__ spheres, int64_t N,
                                double4* __restrict__ sw, const double4* __restrict__ old_sw,
                                int64_t N_old, int* err, const PDyn* __restrict__ pd) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (pd) {  // device-driven update: inputs and sizes from the device (grid sized by a bound)
    spheres = pd->spheres;
    N = pd->N;
    N_old = pd->N_old;
    // ... and the new ids must be the appended range (k_check_new_ids of the eager path)
    if (i < pd->M && pd->new_ids[i] != N_old + i && atomicCAS(err, 0, (int)RPD_EINVAL) == 0) {
      err[1] = 100;
      err[2] = (int)i;
    }
  }
  if (i >= N) return;
  double S[4];
  for (int c = 0; c < 4; ++c) {
    double x = spheres[4 * i + c];
    if (!isfinite(x)) {
      report(err, RPD_EINVAL, ERR_SPHERE_NAN, i);
      return;
    }
    if (c == 3 && x < 0.0) {
      report(err, RPD_EINVAL, ERR_RADIUS_NEG, i);
      return;
    }
    if (!to_lat(x, &S[c])) {
      report(err, RPD_ENOTEXACT, ERR_SPHERE_LATTICE, i);
      return;
    }
  }
  double W = S[0] * S[0] + S[1] * S[1] + S[2] * S[2] - S[3] * S[3];
  const double4 v = make_double4(S[0], S[1], S[2], W);
  if (old_sw && i < N_old) {
    const double4 o = old_sw[i];
    if (o.x != v.x || o.y != v.y || o.z != v.z || o.w != v.w) {
      report(err, RPD_EINVAL, ERR_SPHERE_CHANGED, i);
      return;
    }
  }
  sw[i] = v;
}

struct OldRows {  // previous staged CSR (partial updates: unchanged rows are copied)
  const int32_t* off;
  const int32_t* idx;
  const double4* planes;
  const int32_t* twin;
  const unsigned long long* hkey;
  const int32_t* repoch;
  int64_t N;
};

// The lanes that build one row: a group of RG lanes of a warp (k_stage_rows) or a whole block
// (k_stage_long, the long rows of a partial update); same code, different votes and barriers.
template <int RG>
struct WarpRows {
  int lane;
  unsigned full;
  static constexpr int size = RG;
  __device__ bool all(bool x) const { return __all_sync(full, x); }
  __device__ bool any(bool x) const { return __any_sync(full, x); }
  __device__ void sync() const { __syncwarp(full); }
};
struct BlockRows {
  int lane;
  int size;
  __device__ bool all(bool x) const { return __syncthreads_and(x); }
  __device__ bool any(bool x) const { return __syncthreads_or(x); }
  __device__ void sync() const { __syncthreads(); }
};

// Build row i (entries [e0, e1)): validation, ascending order (input order kept when sorted,
// else rank sort), radical planes, twin keys and twins.  tab: the row's duplicate-key hash
// table (at least pow2 >= 2k entries; global scratch or shared memory).
template <class G>
__device__ void stage_build(const G& g, int64_t i, int32_t e0, int32_t e1, bool sorted,
                            int64_t N, const int32_t* __restrict__ idx_in,
                            const double4* __restrict__ sw, int32_t* __restrict__ idx_out,
                            double4* __restrict__ planes, int32_t* __restrict__ twin,
                            unsigned long long* __restrict__ hkey, int32_t* __restrict__ repoch,
                            int epoch, unsigned long long* tab, int* err) {
  const int lane = g.lane, S = g.size;
  const int k = e1 - e0;
  if (lane == 0) repoch[i] = epoch;
  bool bad = false;
  for (int32_t e = e0 + lane; e < e1; e += S) {
    const int32_t j = idx_in[e];
    if (j < 0 || j >= N) {
      report(err, RPD_EINVAL, ERR_NBR_INDEX, i);
      bad = true;
      break;
    }
    if (j == i) {
      report(err, RPD_EINVAL, ERR_NBR_SELF, i);
      bad = true;
      break;
    }
    if (sorted) {
      idx_out[e] = j;
      continue;
    }
    int rank = 0;
    for (int32_t f = e0; f < e1; ++f) {
      const int32_t x = idx_in[f];
      if (x == j && f != e) {
        report(err, RPD_EINVAL, ERR_NBR_DUP, i);
        bad = true;
      }
      rank += x < j;
    }
    if (bad) break;
    idx_out[e0 + rank] = j;
  }
  if (g.any(bad)) return;
  g.sync();
  const double4 si = sw[i];
  // planes, and the twin key: bit patterns of the ratios to the first non-zero normal
  // component (correctly rounded quotients of exactly proportional integers are equal)
  for (int32_t e = e0 + lane; e < e1; e += S) {
    const int32_t j = idx_out[e];
    const double4 sj = sw[j];
    const double nx = 2.0 * (si.x - sj.x), ny = 2.0 * (si.y - sj.y), nz = 2.0 * (si.z - sj.z);
    if (nx == 0.0 && ny == 0.0 && nz == 0.0) report(err, RPD_EINVAL, ERR_NBR_SAME_CENTRE, i);
    const double4 a = make_double4(nx, ny, nz, sj.w - si.w);
    planes[e] = a;
    const double piv = fabs(a.x != 0.0 ? a.x : (a.y != 0.0 ? a.y : a.z));
    const int which = a.x != 0.0 ? 0 : (a.y != 0.0 ? 1 : 2);
    unsigned long long h = 1469598103934665603ull ^ (unsigned long long)which;
    h = (h ^ (unsigned long long)__double_as_longlong(a.x / piv)) * 1099511628211ull;
    h = (h ^ (unsigned long long)__double_as_longlong(a.y / piv)) * 1099511628211ull;
    h = (h ^ (unsigned long long)__double_as_longlong(a.z / piv)) * 1099511628211ull;
    h = (h ^ (unsigned long long)__double_as_longlong(a.w / piv)) * 1099511628211ull;
    // final avalanche (the ratios of small integers have all-zero low mantissa bits, so the
    // low bits of the raw product barely vary and would cluster the hash-table slots)
    h ^= h >> 33;
    h *= 0xff51afd7ed558ccdull;
    h ^= h >> 33;
    h *= 0xc4ceb9fe1a85ec53ull;
    h ^= h >> 33;
    hkey[e] = h;
  }
  g.sync();
  // twins: next entry of the row with the same oriented plane (equal keys compared exactly).
  // Long rows first check for a repeated key with the row's hash table; without a repeat every
  // entry has no twin.
  bool maybe = true;
  if (k > 64) {
    int tsz = 1;
    while (tsz < 2 * k) tsz <<= 1;
    for (int q = lane; q < tsz; q += S) tab[q] = 0ull;
    g.sync();
    bool dup = false;
    for (int32_t e = e0 + lane; e < e1; e += S) {
      const unsigned long long h = hkey[e] | 1ull;
      int slot = (int)(h & (unsigned long long)(tsz - 1));
      while (true) {
        const unsigned long long prev = atomicCAS(tab + slot, 0ull, h);
        if (prev == 0ull) break;
        if (prev == h) {
          dup = true;
          break;
        }
        slot = (slot + 1) & (tsz - 1);
      }
    }
    maybe = g.any(dup);
  }
  for (int32_t e = e0 + lane; e < e1; e += S) {
    int32_t tw = -1;
    if (maybe) {
      const unsigned long long h = hkey[e];
      for (int32_t f = e + 1; f < e1 && tw < 0; f += 4) {
        unsigned long long hf[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) hf[q] = f + q < e1 ? hkey[f + q] : ~h;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          if (tw >= 0 || hf[q] != h) continue;
          const double4 a = planes[e], b = planes[f + q];
          const bool prop = a.x * b.y == a.y * b.x && a.x * b.z == a.z * b.x &&
                            a.y * b.z == a.z * b.y && a.x * b.w == a.w * b.x &&
                            a.y * b.w == a.w * b.y && a.z * b.w == a.w * b.z;
          const double dot = a.x * b.x + a.y * b.y + a.z * b.z;
          if (prop && dot > 0.0) tw = f + q;
        }
      }
    }
    twin[e] = tw;
  }
}

#ifndef RPD_STAGE_LONG
#define RPD_STAGE_LONG 96  // rows longer than this that need building go to k_stage_long
#endif
constexpr int STAGE_LONG_THREADS = 256;
constexpr int STAGE_LONG_TAB = 2048;  // shared hash slots of k_stage_long (rows up to 1024)

// One group of RG lanes per sphere row (STAGE_RG): validation, ascending order, radical planes
// and twins (stage_build).  In a partial update a row of an old sphere whose neighbour list is
// unchanged is copied from the previous stage instead, and a long row that must be built is
// deferred to k_stage_long (a block per row: its hash table in shared memory) when long_list
// is given.
#ifndef RPD_STAGE_MINB
#define RPD_STAGE_MINB 1  // min resident blocks of k_stage_rows (a register cap; A/B knob)
#endif
template <int RG>
__global__ void __launch_bounds__(256, RPD_STAGE_MINB) k_stage_rows(const int32_t* __restrict__ off_in, const int32_t* __restrict__ idx_in,
                             int64_t N, int64_t E, const double4* __restrict__ sw,
                             int32_t* __restrict__ off_out, int32_t* __restrict__ idx_out,
                             double4* __restrict__ planes, int32_t* __restrict__ twin,
                             unsigned long long* __restrict__ hkey, int32_t* __restrict__ repoch,
                             int epoch, unsigned long long* __restrict__ htab, OldRows old,
                             int* err, const PDyn* __restrict__ pd, int32_t* __restrict__ long_list,
                             int* __restrict__ n_long) {
  if (pd) {  // device-driven update (see k_stage_spheres)
    off_in = pd->nbr_off;
    idx_in = pd->nbr_idx;
    N = pd->N;
    E = pd->E;
    old.N = pd->N_old;
    epoch = pd->epoch;
  }
  const int64_t i = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) / RG;
  const int lane = threadIdx.x & (RG - 1);
  const unsigned FULL = (RG == 32 ? 0xffffffffu : ((1u << RG) - 1u))
                        << (RG * ((threadIdx.x & 31) / RG));  // this row's lanes
  if (i >= N) return;
  const int32_t e0 = off_in[i], e1 = off_in[i + 1];
  // the previous stage's row bounds, loaded together with the new ones (partial updates)
  const bool has_old = old.off && i < old.N;
  const int32_t o0 = has_old ? old.off[i] : 0, o1 = has_old ? old.off[i + 1] : 0;
  if (lane == 0) {
    off_out[i] = e0;
    if (i == N - 1) off_out[N] = e1;
  }
  if (e0 < 0 || e1 < e0 || e1 > E || (i == 0 && e0 != 0) || (i == N - 1 && e1 != E)) {
    if (lane == 0) report(err, RPD_EINVAL, ERR_NBR_OFF, i);
    return;
  }
  const int k = e1 - e0;
  // sorted strictly ascending?  (then no duplicates either); rows of at most RG entries hold
  // one entry per lane, and the old row's entries are loaded alongside for the reuse test
  bool sorted = true, same = has_old && (o1 - o0) == k;
  if (k <= RG) {
    const bool have = lane < k;
    const int32_t x = have ? idx_in[e0 + lane] : 0;
    const int32_t ox = have && same ? old.idx[o0 + lane] : 0;
    const int32_t xn = __shfl_down_sync(FULL, x, 1, RG);
    sorted = !(have && lane + 1 < k) || x < xn;
    same = same && (!have || ox == x);
  } else {
    for (int32_t e = e0 + lane; e + 1 < e1; e += RG) sorted &= idx_in[e] < idx_in[e + 1];
    for (int32_t q = lane; same && q < k; q += RG) same = old.idx[o0 + q] == idx_in[e0 + q];
  }
  sorted = __all_sync(FULL, sorted);
  // unchanged row of an old sphere: copy the previous stage
  // (empty rows are never reused: their Alg. 1 boolean depends on N, R4)
  if (has_old && sorted && k > 0) {
    if (__all_sync(FULL, same)) {
      if (lane == 0) repoch[i] = old.repoch[i];
      for (int32_t q = lane; q < k; q += RG) {
        idx_out[e0 + q] = old.idx[o0 + q];
        planes[e0 + q] = old.planes[o0 + q];
        hkey[e0 + q] = old.hkey[o0 + q];
        const int32_t tw = old.twin[o0 + q];
        twin[e0 + q] = tw < 0 ? -1 : tw - o0 + e0;
      }
      return;
    }
  }
  if (long_list && k > RPD_STAGE_LONG) {  // a long row to build: a block of its own
    if (lane == 0) long_list[atomicAdd(n_long, 1)] = (int32_t)i;
    return;
  }
#ifdef RPD_DEBUG_STAGE
  const long long t0 = clock64();
#endif
  stage_build(WarpRows<RG>{lane, FULL}, i, e0, e1, sorted, N, idx_in, sw, idx_out, planes, twin,
              hkey, repoch, epoch, htab + 4 * (int64_t)e0, err);
#ifdef RPD_DEBUG_STAGE
  const long long dt = clock64() - t0;
  if (lane == 0 && dt > RPD_DEBUG_STAGE_MIN)
    printf("stage row %lld k %d sorted %d cycles %lld\n", (long long)i, k, (int)sorted, dt);
#endif
}

// The deferred long rows of a partial update: a block per row (grid-stride over the list)
__global__ void __launch_bounds__(STAGE_LONG_THREADS) k_stage_long(
    const int32_t* __restrict__ off_in, const int32_t* __restrict__ idx_in, int64_t N,
    const double4* __restrict__ sw, int32_t* __restrict__ idx_out, double4* __restrict__ planes,
    int32_t* __restrict__ twin, unsigned long long* __restrict__ hkey,
    int32_t* __restrict__ repoch, int epoch, unsigned long long* __restrict__ htab, int* err,
    const PDyn* __restrict__ pd, const int32_t* __restrict__ long_list,
    const int* __restrict__ n_long) {
  __shared__ unsigned long long s_tab[STAGE_LONG_TAB];
  if (pd) {
    off_in = pd->nbr_off;
    idx_in = pd->nbr_idx;
    N = pd->N;
    epoch = pd->epoch;
  }
  const int n = *n_long;
  const BlockRows g{(int)threadIdx.x, (int)blockDim.x};
  for (int q = blockIdx.x; q < n; q += gridDim.x) {
    const int64_t i = long_list[q];
    const int32_t e0 = off_in[i], e1 = off_in[i + 1];
    bool sorted = true;
    for (int32_t e = e0 + g.lane; e + 1 < e1; e += g.size) sorted &= idx_in[e] < idx_in[e + 1];
    sorted = g.all(sorted);
    unsigned long long* tab = 2 * (e1 - e0) <= STAGE_LONG_TAB ? s_tab : htab + 4 * (int64_t)e0;
    stage_build(g, i, e0, e1, sorted, N, idx_in, sw, idx_out, planes, twin, hkey, repoch, epoch,
                tab, err);
    g.sync();  // (the shared table is reused by the next row)
  }
}

#ifndef STAGE_RG
#define STAGE_RG 32  // lanes per row of k_stage_rows (8 and 16 measured slower)
#endif

static inline unsigned nblk(int64_t n, int b) { return (unsigned)((n + b - 1) / b); }

cudaError_t launch_stage_mesh(rpd_ctx* c, const double* verts, int64_t V, const int32_t* tets,
                              int64_t T) {
  Stage& s = c->st;
  cudaError_t e = s.tx.ensure(sizeof(double) * 12 * (T > 0 ? T : 1));
  if (e) return e;
  s.T = T;
  s.V = V;
  c->bvh_all_valid = false;
  int* err = c->errw.as<int>();
  if (c->validate && V > 0) {
    k_check_verts<<<nblk(3 * V, 256), 256, 0, c->stream>>>(verts, 3 * V, err);
    ++c->launches;
  }
  if (T > 0) {
    k_stage_tets<<<nblk(T, 256), 256, 0, c->stream>>>(verts, V, tets, T, s.tx.as<double>(), err);
    ++c->launches;
  }
  return cudaGetLastError();
}

// host part of a sphere staging: the previous rows become the "old" buffers (copied for
// unchanged rows when reusing), the buffers are sized for N spheres / E entries
cudaError_t stage_prepare(rpd_ctx* c, int64_t N, int64_t E) {
  Stage& s = c->st;
  cudaError_t e;
  std::swap(s.nbr_off, s.old_off);
  std::swap(s.nbr_idx, s.old_idx);
  std::swap(s.planes, s.old_planes);
  std::swap(s.twin, s.old_twin);
  std::swap(s.hkey, s.old_hkey);
  std::swap(s.repoch, s.old_repoch);
  std::swap(s.sw, s.old_sw);
  s.N_prev = s.N;
  if ((e = s.sw.ensure(sizeof(double4) * (N > 0 ? N : 1)))) return e;
  if ((e = s.nbr_off.ensure(sizeof(int32_t) * (N + 1)))) return e;
  if ((e = s.nbr_idx.ensure(sizeof(int32_t) * (E > 0 ? E : 1)))) return e;
  if ((e = s.planes.ensure(sizeof(double4) * (E > 0 ? E : 1)))) return e;
  if ((e = s.twin.ensure(sizeof(int32_t) * (E > 0 ? E : 1)))) return e;
  if ((e = s.hkey.ensure(sizeof(unsigned long long) * (E > 0 ? E : 1)))) return e;
  if ((e = s.repoch.ensure(sizeof(int32_t) * (N > 0 ? N : 1)))) return e;
  if ((e = s.htab.ensure(sizeof(unsigned long long) * 4 * (E > 0 ? E : 1)))) return e;
  if ((e = s.long_rows.ensure(sizeof(int32_t) * (N + 2)))) return e;  // (list + its count)
  s.N = N;
  s.E = E;
  return cudaSuccess;
}

// the staging kernels (after stage_prepare).  Device-driven mode (c->pdd): inputs and sizes
// come from the device, the grids cover the buffers' capacity
cudaError_t stage_launch(rpd_ctx* c, const double* spheres, const int32_t* nbr_off,
                         const int32_t* nbr_idx, bool reuse_rows, int epoch) {
  Stage& s = c->st;
  const int64_t N = s.N, E = s.E, N_old = s.N_prev;
  const PDyn* pd = c->pdd;
  OldRows old{nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, 0};
  if (reuse_rows && s.old_off.p)
    old = OldRows{s.old_off.as<int32_t>(),  s.old_idx.as<int32_t>(),
                  s.old_planes.as<double4>(), s.old_twin.as<int32_t>(),
                  s.old_hkey.as<unsigned long long>(), s.old_repoch.as<int32_t>(), N_old};
  int* err = c->errw.as<int>();
  const int64_t Ng = pd ? (int64_t)(s.sw.cap / sizeof(double4)) : N;  // grid rows
  if (N > 0) {
    k_stage_spheres<<<nblk(Ng, 256), 256, 0, c->stream>>>(
        spheres, N, s.sw.as<double4>(), old.off ? s.old_sw.as<double4>() : nullptr, N_old, err,
        pd);
    ++c->launches;
    // partial updates defer the long rows that must be built to a block each
    int32_t* long_list = nullptr;
    int* n_long = nullptr;
    if (old.off) {
      long_list = s.long_rows.as<int32_t>();
      n_long = long_list + (s.long_rows.cap / sizeof(int32_t)) - 1;  // (count: the last word)
      if (!pd) {  // (a graph: zeroed by k_pd_init)
        cudaError_t e = cudaMemsetAsync(n_long, 0, sizeof(int), c->stream);
        if (e) return e;
      }
    }
    k_stage_rows<STAGE_RG><<<nblk(STAGE_RG * Ng, 256), 256, 0, c->stream>>>(
        nbr_off, nbr_idx, N, E, s.sw.as<double4>(), s.nbr_off.as<int32_t>(),
        s.nbr_idx.as<int32_t>(), s.planes.as<double4>(), s.twin.as<int32_t>(),
        s.hkey.as<unsigned long long>(), s.repoch.as<int32_t>(), epoch,
        s.htab.as<unsigned long long>(), old, err, pd, long_list, n_long);
    ++c->launches;
    if (long_list) {
      k_stage_long<<<c->sms, STAGE_LONG_THREADS, 0, c->stream>>>(
          nbr_off, nbr_idx, N, s.sw.as<double4>(), s.nbr_idx.as<int32_t>(),
          s.planes.as<double4>(), s.twin.as<int32_t>(), s.hkey.as<unsigned long long>(),
          s.repoch.as<int32_t>(), epoch, s.htab.as<unsigned long long>(), err, pd, long_list,
          n_long);
      ++c->launches;
    }
  } else {
    cudaError_t e = cudaMemsetAsync(s.nbr_off.p, 0, sizeof(int32_t), c->stream);
    if (e) return e;
  }
  return cudaGetLastError();
}

cudaError_t launch_stage_spheres(rpd_ctx* c, const double* spheres, int64_t N,
                                 const int32_t* nbr_off, const int32_t* nbr_idx, int64_t E,
                                 bool reuse_rows, int epoch) {
  cudaError_t e = stage_prepare(c, N, E);
  if (e) return e;
  return stage_launch(c, spheres, nbr_off, nbr_idx, reuse_rows, epoch);
}

}  // namespace rpd
