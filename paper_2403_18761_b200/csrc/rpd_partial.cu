// rpd_partial.cu -- SURVEY.md §8(a) row a6: partial RPD update.
//
// "We only select a subset of tets from T relating to new spheres {m_j} and compute the
// intersection among them.  Thus, the RPD is updated partially instead of re-computing as a
// whole" (also 384, 396).  Reading R11: dirty tets are the tets that
// Alg. 1 relates to at least one new sphere; they are re-filtered against all spheres and
// re-clipped with the new neighbour lists, every other tet keeps its candidates and pieces.
//
// Kernels here: new-id validation, dirty-tet list (flag -> scan -> ascending list + position
// map) and the two-phase CSR merge (per-tet counts -> scans -> element copies) of the clean
// old tets and the re-clipped dirty tets, incidence-mask word offsets included.
#include "rpd_ctx.h"
#include "rpd_internal.cuh"

namespace rpd {

static inline unsigned nblk(int64_t n, int b) { return (unsigned)((n + b - 1) / b); }

__global__ void k_check_new_ids(const int32_t* __restrict__ new_ids, int64_t M, int64_t N_old,
                                int* err) {
  int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (k >= M) return;
  if (new_ids[k] != N_old + k && atomicCAS(err, 0, (int)RPD_EINVAL) == 0) {
    err[1] = 100;  // new ids not the appended range
    err[2] = (int)k;
  }
}

__global__ void k_dirty_flag(int64_t T, const int32_t* __restrict__ count,
                             uint8_t* __restrict__ flag) {
  int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t < T) flag[t] = count[t] > 0;
}

// dirty list + position map; the oldest candidate-list epoch among the dirty tets, whose
// lists are re-stamped with the current epoch
__global__ void k_dirty_list(int64_t T, const uint8_t* __restrict__ flag,
                             const int32_t* __restrict__ scan, int32_t* __restrict__ list,
                             int32_t* __restrict__ pos, int32_t* __restrict__ cepoch,
                             int* __restrict__ min_epoch, int epoch) {
  int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= T) return;
  if (flag[t]) {
    list[scan[t]] = (int32_t)t;
    pos[t] = scan[t];
    atomicMin(min_epoch, cepoch[t]);
    cepoch[t] = epoch;
  } else {
    pos[t] = -1;
  }
}

cudaError_t launch_check_new_ids(rpd_ctx* c, const int32_t* new_ids, int64_t M, int64_t N_old) {
  if (M == 0) return cudaSuccess;
  k_check_new_ids<<<nblk(M, 256), 256, 0, c->stream>>>(new_ids, M, N_old, c->errw.as<int>());
  ++c->launches;
  return cudaGetLastError();
}

// d_count (filter counts over the new spheres) -> d_flag -> d_scan -> d_list, d_pos
cudaError_t launch_dirty_list(rpd_ctx* c, int64_t T) {
  if (T == 0) return cudaMemsetAsync(c->d_scan.p, 0, sizeof(int32_t), c->stream);
  k_dirty_flag<<<nblk(T, 256), 256, 0, c->stream>>>(T, c->d_count.as<int32_t>(),
                                                    c->d_flag.as<uint8_t>());
  ++c->launches;
  cudaError_t e = launch_scan_u8(c, c->d_flag.as<uint8_t>(), c->d_scan.as<int32_t>(), T);
  if (e) return e;
  e = cudaMemsetAsync(c->min_epoch.p, 0x7f, sizeof(int), c->stream);
  if (e) return e;
  k_dirty_list<<<nblk(T, 256), 256, 0, c->stream>>>(
      T, c->d_flag.as<uint8_t>(), c->d_scan.as<int32_t>(), c->d_list.as<int32_t>(),
      c->d_pos.as<int32_t>(), c->cepoch.as<int32_t>(), c->min_epoch.as<int>(), c->epoch);
  ++c->launches;
  return cudaGetLastError();
}

// ---------------------------------------------------------------- merge

struct MergeSrc {
  const int32_t *c_off, *c_idx, *c_moff;
  const int32_t *p_off, *p_sphere, *p_inc_off, *p_inc;
  const double *p_vol, *p_m1;
  const uint8_t* p_fm;
};

__device__ inline MergeSrc pick(int d, const MergeSrc& o, const MergeSrc& n) {
  return d >= 0 ? n : o;
}

// per-tet counts of the merged sets: candidates, pieces, incidences, incidence-mask words
__global__ void k_merge_counts(int64_t T, const int32_t* __restrict__ dpos, MergeSrc o,
                               MergeSrc n, int32_t* __restrict__ cnt) {
  int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= T) return;
  const int d = dpos[t];
  const MergeSrc s = pick(d, o, n);
  const int64_t k = d >= 0 ? d : t;
  const int p0 = s.p_off[k], p1 = s.p_off[k + 1];
  const int c0 = s.c_off[k], c1 = s.c_off[k + 1];
  cnt[t] = c1 - c0;
  cnt[T + t] = p1 - p0;
  cnt[2 * T + t] = s.p_inc_off[p1] - s.p_inc_off[p0];
  cnt[3 * T + t] = s.c_moff[c1] - s.c_moff[c0];
}

struct MergeDst {
  const int32_t *c_off, *p_off, *i_tet, *w_tet;  // scans of the counts (new offsets)
  int32_t *c_idx, *pair_tet, *c_moff, *p_sphere, *p_inc_off, *p_inc;
  double *p_vol, *p_m1;
  uint8_t* p_fm;
  int32_t* src_piece;  // per new piece: source piece index, +(1 << 30) when from the dirty set
};

// last index t in [0, n) with off[t] <= q (off non-decreasing, off[0] = 0)
__device__ __forceinline__ int64_t seg_of(const int32_t* __restrict__ off, int64_t n, int64_t q) {
  int64_t lo = 0, hi = n;  // invariant: off[lo] <= q < off[hi]
  while (hi - lo > 1) {
    const int64_t mid = (lo + hi) >> 1;
    if (off[mid] <= q) lo = mid;
    else hi = mid;
  }
  return lo;
}

// The copy kernels read their element counts from the device scans (no host round trip) and
// stride over them with a grid sized from a host upper bound.

// one thread per merged candidate (+ its incidence-mask word offset)
__global__ void k_merge_cands(int64_t T, const int32_t* __restrict__ dpos, MergeSrc o,
                              MergeSrc n, MergeDst D) {
  const int64_t n_new = D.c_off[T];
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < n_new; q += stride) {
    const int64_t t = seg_of(D.c_off, T, q);
    const int d = dpos[t];
    const MergeSrc& s = d >= 0 ? n : o;
    const int64_t k = d >= 0 ? d : t;
    const int64_t src = s.c_off[k] + (q - D.c_off[t]);
    D.c_idx[q] = s.c_idx[src];
    D.pair_tet[q] = (int32_t)t;
    D.c_moff[q] = D.w_tet[t] + (s.c_moff[src] - s.c_moff[s.c_off[k]]);
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) D.c_moff[n_new] = D.w_tet[T];
}

// one thread per merged piece
__global__ void k_merge_pieces(int64_t T, const int32_t* __restrict__ dpos, MergeSrc o,
                               MergeSrc n, MergeDst D) {
  const int64_t n_new = D.p_off[T];
  if (blockIdx.x == 0 && threadIdx.x == 0) D.p_inc_off[n_new] = D.i_tet[T];
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < n_new; q += stride) {
    const int64_t t = seg_of(D.p_off, T, q);
    const int d = dpos[t];
    const MergeSrc& s = d >= 0 ? n : o;
    const int64_t k = d >= 0 ? d : t;
    const int p0 = s.p_off[k];
    const int sp = p0 + (int)(q - D.p_off[t]);
    D.p_sphere[q] = s.p_sphere[sp];
    D.p_vol[q] = s.p_vol[sp];
    D.p_m1[3 * q + 0] = s.p_m1[3 * sp + 0];
    D.p_m1[3 * q + 1] = s.p_m1[3 * sp + 1];
    D.p_m1[3 * q + 2] = s.p_m1[3 * sp + 2];
    D.p_fm[q] = s.p_fm[sp];
    D.p_inc_off[q] = D.i_tet[t] + (s.p_inc_off[sp] - s.p_inc_off[p0]);
    D.src_piece[q] = sp + (d >= 0 ? (1 << 30) : 0);
  }
}

// one thread per merged incidence (after k_merge_pieces: needs p_inc_off and src_piece)
__global__ void k_merge_incs(int64_t T, MergeSrc o, MergeSrc n, MergeDst D) {
  const int64_t n_pieces_new = D.p_off[T], n_inc_new = D.i_tet[T];
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n_inc_new; r += stride) {
    const int64_t q = seg_of(D.p_inc_off, n_pieces_new, r);
    const int code = D.src_piece[q];
    const MergeSrc& s = code >= (1 << 30) ? n : o;
    const int sp = code & ((1 << 30) - 1);
    D.p_inc[r] = s.p_inc[s.p_inc_off[sp] + (r - D.p_inc_off[q])];
  }
}

static MergeSrc src_of(const CandSet& cs, const PieceSet& ps) {
  return MergeSrc{cs.off.as<int32_t>(),     cs.idx.as<int32_t>(),     cs.moff.as<int32_t>(),
                  ps.off.as<int32_t>(),     ps.sphere.as<int32_t>(),  ps.inc_off.as<int32_t>(),
                  ps.inc.as<int32_t>(),     ps.vol.as<double>(),      ps.m1.as<double>(),
                  ps.fm.as<uint8_t>()};
}

static inline unsigned grid_for(int64_t n_ub) {
  const int64_t g = (n_ub + 255) / 256;
  return (unsigned)(g < 1 ? 1 : (g > 148 * 32 ? 148 * 32 : g));
}

// phase 0: per-tet counts and their scans (new cand offsets -> cn.off, new piece offsets ->
// pn.off, tet-level incidence offsets -> m_off, tet-level mask-word offsets -> m_off + T + 1);
// totals at [T] of each.
// phase 1: copies into cn / pn, sized by the host upper bounds cn.n, pn.n_pieces, pn.n_inc
// (exact totals are read back by the caller after the copies).
cudaError_t launch_merge(rpd_ctx* c, int64_t T, const CandSet& co, const PieceSet& po,
                         const CandSet& cd, const PieceSet& pd, CandSet& cn, PieceSet& pn,
                         int phase) {
  MergeSrc o = src_of(co, po), n = src_of(cd, pd);
  int32_t* m_off = c->m_off.as<int32_t>();
  int32_t* w_off = m_off + (T + 1);
  if (phase == 0) {
    if (T > 0) {
      k_merge_counts<<<nblk(T, 256), 256, 0, c->stream>>>(T, c->d_pos.as<int32_t>(), o, n,
                                                          c->m_cnt.as<int32_t>());
      ++c->launches;
    }
    cudaError_t e;
    if ((e = launch_scan_i32(c, c->m_cnt.as<int32_t>(), cn.off.as<int32_t>(), T))) return e;
    if ((e = launch_scan_i32(c, c->m_cnt.as<int32_t>() + T, pn.off.as<int32_t>(), T))) return e;
    if ((e = launch_scan_i32(c, c->m_cnt.as<int32_t>() + 2 * T, m_off, T))) return e;
    return launch_scan_i32(c, c->m_cnt.as<int32_t>() + 3 * T, w_off, T);
  }
  cudaError_t e = c->m_src.ensure(sizeof(int32_t) * (pn.n_pieces > 0 ? pn.n_pieces : 1));
  if (e) return e;
  MergeDst D{cn.off.as<int32_t>(),     pn.off.as<int32_t>(),      m_off,
             w_off,                    cn.idx.as<int32_t>(),      cn.pair_tet.as<int32_t>(),
             cn.moff.as<int32_t>(),    pn.sphere.as<int32_t>(),   pn.inc_off.as<int32_t>(),
             pn.inc.as<int32_t>(),     pn.vol.as<double>(),       pn.m1.as<double>(),
             pn.fm.as<uint8_t>(),      c->m_src.as<int32_t>()};
  const int32_t* dpos = c->d_pos.as<int32_t>();
  k_merge_cands<<<grid_for(cn.n), 256, 0, c->stream>>>(T, dpos, o, n, D);
  k_merge_pieces<<<grid_for(pn.n_pieces), 256, 0, c->stream>>>(T, dpos, o, n, D);
  k_merge_incs<<<grid_for(pn.n_inc), 256, 0, c->stream>>>(T, o, n, D);
  c->launches += 3;
  return cudaGetLastError();
}

}  // namespace rpd
