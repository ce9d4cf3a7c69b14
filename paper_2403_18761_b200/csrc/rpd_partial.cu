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
  int ep = 0x7fffffff;
  if (t < T) {
    if (flag[t]) {
      list[scan[t]] = (int32_t)t;
      pos[t] = scan[t];
      ep = cepoch[t];
      cepoch[t] = epoch;
    } else {
      pos[t] = -1;
    }
  }
  // one atomic per warp (per-tet atomics on one address serialise in L2)
  ep = __reduce_min_sync(0xffffffffu, ep);
  if ((threadIdx.x & 31) == 0 && ep != 0x7fffffff) atomicMin(min_epoch, ep);
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
  const int32_t *c_off, *c_idx, *c_moff, *c_pt;
  const int32_t *p_off, *p_sphere, *p_inc_off, *p_inc;
  const double *p_vol, *p_m1;
  const uint8_t* p_fm;
  // Euler mode (p_eu == nullptr: off): per-piece value and the radical-facet CSR
  const long long* p_eu;
  const int32_t *p_rpf_off, *p_rpf_j;
  const long long* p_rpf_e;
  const uint8_t *p_sfm, *p_rfm;
  const unsigned long long* p_radj;
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
  if (s.p_eu) cnt[4 * T + t] = s.p_rpf_off[p1] - s.p_rpf_off[p0];
}

struct MergeDst {
  const int32_t *c_off, *p_off, *i_tet, *w_tet;  // scans of the counts (new offsets)
  int32_t *c_idx, *pair_tet, *c_moff, *p_sphere, *p_inc_off, *p_inc;
  double *p_vol, *p_m1;
  uint8_t* p_fm;
  const int32_t* r_tet;  // Euler mode: scan of the per-tet radical-facet counts
  long long* p_eu;
  int32_t *p_rpf_off, *p_rpf_j;
  long long* p_rpf_e;
  uint8_t *p_sfm, *p_rfm;
  unsigned long long* p_radj;
};

#ifndef RPD_MERGE_MT
#define RPD_MERGE_MT 256
#endif
constexpr int MT = RPD_MERGE_MT;  // tets per merge tile (one block of MT threads)

// block-wide copy dst[k] = f(src[k]), k < n, with 8 independent loads in flight per thread
// before their stores (the source and destination sets never overlap)
template <class T, class F>
__device__ __forceinline__ void tile_copy(T* __restrict__ dst, const T* __restrict__ src, int n,
                                          F f) {
  constexpr int U = 8;
  for (int k0 = threadIdx.x; k0 < n; k0 += U * blockDim.x) {
    T v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int k = k0 + u * blockDim.x;
      if (k < n) v[u] = __ldg(src + k);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int k = k0 + u * blockDim.x;
      if (k < n) dst[k] = f(v[u]);
    }
  }
}

// upper_bound(off[0..n], q) - 1 in shared memory: the tile-local tet of element q
__device__ __forceinline__ int tile_seg(const int* off, int n, int q) {
  int lo = 0, hi = n;  // off[lo] <= q < off[hi]
  while (hi - lo > 1) {
    const int mid = (lo + hi) >> 1;
    if (off[mid] <= q) lo = mid;
    else hi = mid;
  }
  return lo;
}

// One block per tile of MT consecutive tets: the tile's per-tet destination offsets and
// source bases (clean tet: old set at t, dirty tet: re-clipped set at its dirty position) are
// staged in shared memory, then the block copies the tile's candidates, pieces and incidences
// (each a contiguous destination range) with coalesced element loops; an element's tet is
// found by binary search over the staged offsets (no global-memory searches).
__global__ void __launch_bounds__(MT) k_merge_copy(int64_t T, const int32_t* __restrict__ dpos,
                                                    MergeSrc o, MergeSrc n, MergeDst D) {
  __shared__ int s_nc[MT + 1], s_np[MT + 1], s_ni[MT + 1];
  __shared__ int s_sc[MT], s_sp[MT], s_si[MT], s_nw[MT], s_sw[MT];
  __shared__ int s_nr[MT + 1], s_sr[MT];
  const bool eu = D.p_eu != nullptr;
  __shared__ unsigned char s_dirty[MT];
  const int64_t t0 = (int64_t)blockIdx.x * MT;
  const int nt = (int)min((int64_t)MT, T - t0);
  for (int l = threadIdx.x; l <= nt; l += blockDim.x) {
    const int64_t t = t0 + l;
    s_nc[l] = D.c_off[t];
    s_np[l] = D.p_off[t];
    s_ni[l] = D.i_tet[t];
    if (eu) s_nr[l] = D.r_tet[t];
    if (l < nt) {
      const int d = dpos[t];
      const MergeSrc& s = d >= 0 ? n : o;
      const int64_t k = d >= 0 ? d : t;
      const int c0 = s.c_off[k], p0 = s.p_off[k];
      s_dirty[l] = d >= 0;
      s_sc[l] = c0;
      s_sp[l] = p0;
      s_si[l] = s.p_inc_off[p0];
      s_nw[l] = D.w_tet[t];
      s_sw[l] = s.c_moff[c0];
      if (eu) s_sr[l] = s.p_rpf_off[p0];
    }
  }
  // a tile without dirty tets is one contiguous range of the old set in every array, moved
  // by a constant offset: straight streaming copies (most tiles: insertions are local)
  // (also the barrier after the staging; blockDim.x == MT, so thread l staged s_dirty[l])
  const int any_dirty = __syncthreads_or(threadIdx.x < nt && s_dirty[threadIdx.x]);
  if (!any_dirty) {
    const int nc = s_nc[nt] - s_nc[0], npc = s_np[nt] - s_np[0], ni = s_ni[nt] - s_ni[0];
    const int c_src = s_sc[0], p_src = s_sp[0], i_src = s_si[0];
    const int c_dst = s_nc[0], p_dst = s_np[0], i_dst = s_ni[0];
    const int wshift = s_nw[0] - s_sw[0], ishift = s_ni[0] - s_si[0];
    auto same = [](auto x) { return x; };
    tile_copy(D.c_idx + c_dst, o.c_idx + c_src, nc, same);
    tile_copy(D.pair_tet + c_dst, o.c_pt + c_src, nc, same);
    tile_copy(D.c_moff + c_dst, o.c_moff + c_src, nc, [=](int32_t x) { return x + wshift; });
    tile_copy(D.p_sphere + p_dst, o.p_sphere + p_src, npc, same);
    tile_copy(D.p_vol + p_dst, o.p_vol + p_src, npc, same);
    tile_copy(D.p_fm + p_dst, o.p_fm + p_src, npc, same);
    tile_copy(D.p_inc_off + p_dst, o.p_inc_off + p_src, npc, [=](int32_t x) { return x + ishift; });
    tile_copy(D.p_m1 + 3 * (int64_t)p_dst, o.p_m1 + 3 * (int64_t)p_src, 3 * npc, same);
    tile_copy(D.p_inc + i_dst, o.p_inc + i_src, ni, same);
    if (eu) {
      const int nr = s_nr[nt] - s_nr[0], r_src = s_sr[0], r_dst = s_nr[0];
      const int rshift = s_nr[0] - s_sr[0];
      tile_copy(D.p_eu + p_dst, o.p_eu + p_src, npc, same);
      tile_copy(D.p_sfm + p_dst, o.p_sfm + p_src, npc, same);
      tile_copy(D.p_rfm + r_dst, o.p_rfm + r_src, nr, same);
      tile_copy(D.p_radj + r_dst, o.p_radj + r_src, nr, same);
      tile_copy(D.p_rpf_off + p_dst, o.p_rpf_off + p_src, npc,
                [=](int32_t x) { return x + rshift; });
      tile_copy(D.p_rpf_j + r_dst, o.p_rpf_j + r_src, nr, same);
      tile_copy(D.p_rpf_e + r_dst, o.p_rpf_e + r_src, nr, same);
    }
    if (t0 + nt == T && threadIdx.x == 0) {
      D.c_moff[s_nc[nt]] = D.w_tet[T];
      D.p_inc_off[s_np[nt]] = s_ni[nt];
      if (eu) D.p_rpf_off[s_np[nt]] = s_nr[nt];
    }
    return;
  }
  // candidates (+ their incidence-mask word offsets)
  for (int q = s_nc[0] + threadIdx.x; q < s_nc[nt]; q += blockDim.x) {
    const int l = tile_seg(s_nc, nt, q);
    const MergeSrc& s = s_dirty[l] ? n : o;
    const int src = s_sc[l] + (q - s_nc[l]);
    D.c_idx[q] = s.c_idx[src];
    D.pair_tet[q] = (int32_t)(t0 + l);
    D.c_moff[q] = s_nw[l] + (s.c_moff[src] - s_sw[l]);
  }
  // pieces
  for (int q = s_np[0] + threadIdx.x; q < s_np[nt]; q += blockDim.x) {
    const int l = tile_seg(s_np, nt, q);
    const MergeSrc& s = s_dirty[l] ? n : o;
    const int sp = s_sp[l] + (q - s_np[l]);
    D.p_sphere[q] = s.p_sphere[sp];
    D.p_vol[q] = s.p_vol[sp];
    D.p_m1[3 * (int64_t)q + 0] = s.p_m1[3 * (int64_t)sp + 0];
    D.p_m1[3 * (int64_t)q + 1] = s.p_m1[3 * (int64_t)sp + 1];
    D.p_m1[3 * (int64_t)q + 2] = s.p_m1[3 * (int64_t)sp + 2];
    D.p_fm[q] = s.p_fm[sp];
    D.p_inc_off[q] = s_ni[l] + (s.p_inc_off[sp] - s_si[l]);
    if (eu) {
      D.p_eu[q] = s.p_eu[sp];
      D.p_sfm[q] = s.p_sfm[sp];
      D.p_rpf_off[q] = s_nr[l] + (s.p_rpf_off[sp] - s_sr[l]);
    }
  }
  // radical facets of the pieces (Euler mode)
  if (eu)
    for (int r = s_nr[0] + threadIdx.x; r < s_nr[nt]; r += blockDim.x) {
      const int l = tile_seg(s_nr, nt, r);
      const MergeSrc& s = s_dirty[l] ? n : o;
      const int src = s_sr[l] + (r - s_nr[l]);
      D.p_rpf_j[r] = s.p_rpf_j[src];
      D.p_rpf_e[r] = s.p_rpf_e[src];
      D.p_rfm[r] = s.p_rfm[src];
      D.p_radj[r] = s.p_radj[src];
    }
  // incidences (a tet's incidences are contiguous in its source set)
  for (int r = s_ni[0] + threadIdx.x; r < s_ni[nt]; r += blockDim.x) {
    const int l = tile_seg(s_ni, nt, r);
    const MergeSrc& s = s_dirty[l] ? n : o;
    D.p_inc[r] = s.p_inc[s_si[l] + (r - s_ni[l])];
  }
  if (t0 + nt == T && threadIdx.x == 0) {  // terminal entries
    D.c_moff[s_nc[nt]] = D.w_tet[T];
    D.p_inc_off[s_np[nt]] = s_ni[nt];
    if (eu) D.p_rpf_off[s_np[nt]] = s_nr[nt];
  }
}

static MergeSrc src_of(const CandSet& cs, const PieceSet& ps, bool eu) {
  return MergeSrc{cs.off.as<int32_t>(),     cs.idx.as<int32_t>(),     cs.moff.as<int32_t>(),
                  cs.pair_tet.as<int32_t>(),
                  ps.off.as<int32_t>(),     ps.sphere.as<int32_t>(),  ps.inc_off.as<int32_t>(),
                  ps.inc.as<int32_t>(),     ps.vol.as<double>(),      ps.m1.as<double>(),
                  ps.fm.as<uint8_t>(),
                  eu ? ps.eu.as<long long>() : nullptr, ps.rpf_off.as<int32_t>(),
                  ps.rpf_j.as<int32_t>(),   ps.rpf_e.as<long long>(), ps.sfm.as<uint8_t>(),
                  ps.rfm.as<uint8_t>(),     ps.radj.as<unsigned long long>()};
}

// phase 0: per-tet counts and their scans (new cand offsets -> cn.off, new piece offsets ->
// pn.off, tet-level incidence offsets -> m_off, tet-level mask-word offsets -> m_off + T + 1);
// totals at [T] of each.
// phase 1: the tiled copy into cn / pn (allocated by the caller from host upper bounds; the
// exact totals are read back after the copy).
cudaError_t launch_merge(rpd_ctx* c, int64_t T, const CandSet& co, const PieceSet& po,
                         const CandSet& cd, const PieceSet& pd, CandSet& cn, PieceSet& pn,
                         int phase) {
  const bool eu = c->euler != 0;
  MergeSrc o = src_of(co, po, eu), n = src_of(cd, pd, eu);
  int32_t* m_off = c->m_off.as<int32_t>();
  int32_t* w_off = m_off + (T + 1);
  int32_t* r_off = m_off + 2 * (T + 1);
  if (phase == 0) {
    if (T > 0) {
      k_merge_counts<<<nblk(T, 256), 256, 0, c->stream>>>(T, c->d_pos.as<int32_t>(), o, n,
                                                          c->m_cnt.as<int32_t>());
      ++c->launches;
    }
    const int32_t* cnt = c->m_cnt.as<int32_t>();
    const int32_t* in[5] = {cnt, cnt + T, cnt + 2 * T, cnt + 3 * T, cnt + 4 * T};
    int32_t* out[5] = {cn.off.as<int32_t>(), pn.off.as<int32_t>(), m_off, w_off, r_off};
    return launch_scan_i32_multi(c, in, out, eu ? 5 : 4, T);
  }
  MergeDst D{cn.off.as<int32_t>(),     pn.off.as<int32_t>(),      m_off,
             w_off,                    cn.idx.as<int32_t>(),      cn.pair_tet.as<int32_t>(),
             cn.moff.as<int32_t>(),    pn.sphere.as<int32_t>(),   pn.inc_off.as<int32_t>(),
             pn.inc.as<int32_t>(),     pn.vol.as<double>(),       pn.m1.as<double>(),
             pn.fm.as<uint8_t>(),      r_off,
             eu ? pn.eu.as<long long>() : nullptr, pn.rpf_off.as<int32_t>(),
             pn.rpf_j.as<int32_t>(),   pn.rpf_e.as<long long>(), pn.sfm.as<uint8_t>(),
             pn.rfm.as<uint8_t>(),     pn.radj.as<unsigned long long>()};
  if (T > 0) {
    k_merge_copy<<<nblk(T, MT), MT, 0, c->stream>>>(T, c->d_pos.as<int32_t>(), o, n, D);
    ++c->launches;
  }
  return cudaGetLastError();
}

}  // namespace rpd
