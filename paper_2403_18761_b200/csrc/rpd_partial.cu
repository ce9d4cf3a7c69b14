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
                                int* err, const PDyn* __restrict__ pd) {
  if (pd) {  // device-driven update (grid sized for the largest M of the graph path)
    new_ids = pd->new_ids;
    M = pd->M;
    N_old = pd->N_old;
  }
  int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (k >= M) return;
  if (new_ids[k] != N_old + k && atomicCAS(err, 0, (int)RPD_EINVAL) == 0) {
    err[1] = 100;  // new ids not the appended range
    err[2] = (int)k;
  }
}

cudaError_t launch_check_new_ids(rpd_ctx* c, const int32_t* new_ids, int64_t M, int64_t N_old) {
  if (M == 0) return cudaSuccess;
  k_check_new_ids<<<nblk(M, 256), 256, 0, c->stream>>>(new_ids, M, N_old, c->errw.as<int>(),
                                                       c->pdd);
  ++c->launches;
  return cudaGetLastError();
}

// d_count (filter counts over the new spheres) -> d_list, d_scan[T] = count, cepoch
// re-stamped, min_epoch: one fused scan (rpd_scan.cu)
cudaError_t launch_dirty_list(rpd_ctx* c, int64_t T) {
  if (T == 0) return cudaMemsetAsync(c->d_scan.p, 0, sizeof(int32_t), c->stream);
  if (!c->pdd) {  // (in a graph k_pd_init sets it)
    cudaError_t e = cudaMemsetAsync(c->min_epoch.p, 0x7f, sizeof(int), c->stream);
    if (e) return e;
  }
  return launch_dirty_scan(c, T);
}

// ---------------------------------------------------------------- state pools

__global__ void k_rows_from_off(int64_t T, const int32_t* __restrict__ coff,
                                int2* __restrict__ crow, const int32_t* __restrict__ poff,
                                int2* __restrict__ prow) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= T) return;
  if (crow) crow[t] = make_int2(coff[t], coff[t + 1]);
  if (prow) prow[t] = make_int2(poff[t], poff[t + 1]);
}

cudaError_t launch_rows_from_off(rpd_ctx* c, int64_t T, const CandSet* cs, PieceSet* ps,
                                 CandSet* cs_rows) {
  cudaError_t e;
  if (cs && (e = cs_rows->rows.ensure(sizeof(int2) * (T > 0 ? T : 1)))) return e;
  if (ps && (e = ps->rows.ensure(sizeof(int2) * (T > 0 ? T : 1)))) return e;
  if (T == 0) return cudaSuccess;
  k_rows_from_off<<<nblk(T, 256), 256, 0, c->stream>>>(
      T, cs ? cs->off.as<int32_t>() : nullptr, cs ? cs_rows->rows.as<int2>() : nullptr,
      ps ? ps->off.as<int32_t>() : nullptr, ps ? ps->rows.as<int2>() : nullptr);
  ++c->launches;
  return cudaGetLastError();
}

// dirty tet a (tet t = dirty[a]): its old segments are counted as removed, its rows re-pointed
// at the batch appended at (cbase, pbase) of the pools
__global__ void k_rows_update(int64_t nd, const int32_t* __restrict__ dirty,
                              int2* __restrict__ crow, int2* __restrict__ prow,
                              const int32_t* __restrict__ inc_off,
                              const int32_t* __restrict__ rpf_off,
                              const int32_t* __restrict__ dc_off, const int32_t* __restrict__ dp_off,
                              int cbase, int pbase, unsigned long long* __restrict__ rm,
                              const PDyn* __restrict__ pd) {
  if (pd) {  // device-driven update: batch size and pool fill levels from the device
    nd = pd->nb;
    cbase = pd->fill_c;
    pbase = pd->fill_p;
  }
  unsigned long long v[4] = {0, 0, 0, 0};
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t a = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; a < nd; a += stride) {
    const int t = dirty[a];
    const int2 oc = crow[t], op = prow[t];
    v[0] += oc.y - oc.x;
    v[1] += op.y - op.x;
    if (op.y > op.x) {
      v[2] += inc_off[op.y] - inc_off[op.x];
      if (rpf_off) v[3] += rpf_off[op.y] - rpf_off[op.x];
    }
    crow[t] = make_int2(cbase + dc_off[a], cbase + dc_off[a + 1]);
    prow[t] = make_int2(pbase + dp_off[a], pbase + dp_off[a + 1]);
  }
#pragma unroll
  for (int k = 0; k < 4; ++k) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v[k] += __shfl_xor_sync(0xffffffffu, v[k], o);
  }
  if ((threadIdx.x & 31) == 0)
    for (int k = 0; k < 4; ++k)
      if (v[k]) atomicAdd(rm + k, v[k]);
}

cudaError_t launch_rows_update(rpd_ctx* c, const int32_t* dirty, int64_t nd, CandSet& pool_c,
                               PieceSet& pool_p, const CandSet& cd, const PieceSet& pd,
                               int64_t cbase, int64_t pbase, unsigned long long* rm) {
  cudaError_t e = c->pdd ? cudaSuccess  // (in a graph k_pd_init zeroes rm)
                         : cudaMemsetAsync(rm, 0, sizeof(unsigned long long) * 4, c->stream);
  if (e || nd == 0) return e;
  unsigned grid = nblk(nd, 256);
  if (c->pdd && grid > (unsigned)c->sms * 2) grid = c->sms * 2;  // (grid-stride over the bound)
  k_rows_update<<<grid, 256, 0, c->stream>>>(
      nd, dirty, pool_c.rows.as<int2>(), pool_p.rows.as<int2>(), pool_p.inc_off.as<int32_t>(),
      c->euler ? pool_p.rpf_off.as<int32_t>() : nullptr, cd.off.as<int32_t>(),
      pd.off.as<int32_t>(), (int)cbase, (int)pbase, rm, c->pdd);
  ++c->launches;
  return cudaGetLastError();
}

// ---------------------------------------------------------------- validation aggregates

// per-sphere RPC volume: every tet's piece slots (state rows) added to their spheres
__global__ void k_sphere_vol(int64_t T, const int2* __restrict__ prow,
                             const int32_t* __restrict__ psph, const double* __restrict__ pvol,
                             double* __restrict__ out) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < T;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int2 r = prow[t];
    for (int q = r.x; q < r.y; ++q) atomicAdd(out + psph[q], pvol[q]);
  }
}

cudaError_t launch_sphere_volumes(rpd_ctx* c, double* out) {
  const PieceSet& ps = c->pcs[c->cur];
  const int64_t T = c->st.T, N = c->st.N;
  cudaError_t e = cudaMemsetAsync(out, 0, sizeof(double) * (N > 0 ? N : 1), c->stream);
  if (e || T == 0) return e;
  k_sphere_vol<<<nblk(T, 256), 256, 0, c->stream>>>(T, ps.rows.as<int2>(), ps.sphere.as<int32_t>(),
                                                    ps.vol.as<double>(), out);
  ++c->launches;
  return cudaGetLastError();
}

// ---------------------------------------------------------------- device-driven updates

// the inputs of this update from the mapped pinned mirror; the outputs cleared; and every
// small counter / flag the graph's kernels accumulate into, zeroed here in one launch instead
// of ~20 memset nodes (the eager path's memsets): error word, stats, overflow lists' counts,
// the pair counter, the work-queue header, the removed-segment sums, min epoch, the look-back
// state of the graph's scans
struct PdZero {
  int* errw;
  unsigned long long* stats;
  int* min_epoch;
  int32_t *over1, *over2, *over3;
  int* pair_ctr;
  int* n_long;
  int* qhdr;
  int* n_stage_long;
  int* route;  // the routed-pair counts (2)
  unsigned long long* rm;
  unsigned long long* scan_state;
  int64_t scan_words;
};
__global__ void k_pd_init(PDyn* __restrict__ pd, const PDyn* __restrict__ host, PdZero z) {
  if (threadIdx.x == 0) {
    PDyn v = *host;
    v.nd = v.nb = v.n_chg = v.nc = v.nw = v.np = v.ni = v.maxk = v.need = v.abort = 0;
    v.nc_fast = v.nc_small = v.nc_req = v.nw_req = 0;
    for (int k = 0; k < 6; ++k) v.stamp[k] = 0;
    *pd = v;
    *z.min_epoch = 0x7f7f7f7f;
    *z.over1 = *z.over2 = *z.over3 = 0;
    *z.pair_ctr = 0;
    *z.n_long = 0;
    z.qhdr[0] = z.qhdr[1] = 0;
    *z.n_stage_long = 0;
    z.route[0] = z.route[1] = 0;
  }
  if (threadIdx.x < 4) {
    z.errw[threadIdx.x] = 0;
    z.rm[threadIdx.x] = 0ull;
  }
  if (threadIdx.x < ST_N) z.stats[threadIdx.x] = 0ull;
  for (int64_t k = threadIdx.x; k < z.scan_words; k += blockDim.x) z.scan_state[k] = 0ull;
}

// after the batch's re-filter and scans: its candidate / mask-word totals, and the checks the
// eager path makes on the host (slab capacity, work queues, batch bounds, pool room).  Any
// failure aborts the rest of the graph (batch sizes set to 0) and the host redoes the batch
__global__ void k_pd_check(PDyn* __restrict__ pd, const int32_t* __restrict__ c_off,
                           const int32_t* __restrict__ w_off,
                           const unsigned long long* __restrict__ stats,
                           const int* __restrict__ queue, const int* __restrict__ err,
                           int slab_cap) {
  if (threadIdx.x != 0) return;
  const int nb = pd->nb;
  int nc = c_off[nb], nw = w_off[nb], ab = 0;
  const int maxk = (int)stats[ST_MAXK];
  if (maxk > slab_cap) ab |= PD_SLAB;
  if (queue[0] > pd->cap_items || queue[1] > pd->cap_sup) ab |= PD_QUEUE;
  if (nc > pd->nc_max || nw > pd->nw_max) ab |= PD_BATCH;
  if ((long long)pd->fill_c + nc > pd->room_c || (long long)pd->fill_p + nc > pd->room_p ||
      (long long)pd->fill_i + 32ll * nw > pd->room_i)
    ab |= PD_POOL;
  if (err[0] != 0) ab |= PD_ERR;
  pd->maxk = maxk;
  pd->need = max(queue[0], queue[1]);
  pd->nc_req = nc;
  pd->nw_req = nw;
  if (ab) {
    pd->abort = ab;
    pd->nb = 0;
    nc = nw = 0;
  }
  pd->nc = nc;
  pd->nw = nw;
  // the tier that takes the batch: few pairs go straight to the 64-slot tier (latency), more
  // to the fast tier and its overflow cascade (the eager launch_clip's choice)
  pd->nc_small = nc < RPD_CLIP_SMALL ? nc : 0;
  pd->nc_fast = nc < RPD_CLIP_SMALL ? 0 : nc;
}

// the batch's piece / incidence totals; the whole record, the stats, the error word, the
// removed-segment sums and the fast tier's overflow count back to the mapped mirror (the
// update's one readback)
__global__ void k_pd_final(PDyn* __restrict__ pd, PDyn* __restrict__ host,
                           const int32_t* __restrict__ p_scan, const int32_t* __restrict__ i_scan,
                           const unsigned long long* __restrict__ stats,
                           const int* __restrict__ errw, const unsigned long long* __restrict__ rm,
                           const int32_t* __restrict__ over) {
  if (threadIdx.x != 0) return;
  PDyn v = *pd;
  v.np = p_scan[v.nc];
  v.ni = i_scan[v.nc];
  for (int k = 0; k < ST_N; ++k) v.stats[k] = stats[k];
  for (int k = 0; k < 4; ++k) {
    v.removed[k] = rm[k];
    v.err[k] = errw[k];
  }
  v.n_wide = *over;
  *host = v;
  __threadfence_system();
}

// profiling marks inside a graph (event timing of captured event records is not relied on)
__global__ void k_pd_stamp(PDyn* __restrict__ pd, int k) {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  if (threadIdx.x == 0) pd->stamp[k] = t;
}

cudaError_t launch_pd_stamp(rpd_ctx* c, int k) {
  k_pd_stamp<<<1, 32, 0, c->stream>>>(c->pdd, k);
  ++c->launches;
  return cudaGetLastError();
}

cudaError_t launch_pd_init(rpd_ctx* c) {
  PdZero z{c->errw.as<int>(),
           c->stats.as<unsigned long long>(),
           c->min_epoch.as<int>(),
           c->p_over.as<int32_t>(),
           c->p_over2.as<int32_t>(),
           c->p_over3.as<int32_t>(),
           c->p_dyn.as<int>(),
           c->cand_long.as<int>(),
           c->bvh_items.as<int>(),
           c->st.long_rows.as<int>() + (c->st.long_rows.cap / sizeof(int32_t)) - 1,
           c->p_route.as<int>(),
           c->m_cnt.as<unsigned long long>(),
           c->g_scan.as<unsigned long long>(),
           (int64_t)(c->g_scan.cap / sizeof(unsigned long long))};
  k_pd_init<<<1, 256, 0, c->stream>>>(c->pdd, c->pd_hdev, z);
  ++c->launches;
  return cudaGetLastError();
}

cudaError_t launch_pd_check(rpd_ctx* c, const int32_t* c_off, const int32_t* w_off) {
  k_pd_check<<<1, 32, 0, c->stream>>>(c->pdd, c_off, w_off, c->stats.as<unsigned long long>(),
                                      c->bvh_items.as<int>(), c->errw.as<int>(), c->slab_cap);
  ++c->launches;
  return cudaGetLastError();
}

cudaError_t launch_pd_final(rpd_ctx* c) {
  k_pd_final<<<1, 32, 0, c->stream>>>(c->pdd, c->pd_hdev, c->p_scan.as<int32_t>(),
                                      c->i_scan.as<int32_t>(),
                                      c->stats.as<unsigned long long>(), c->errw.as<int>(),
                                      c->m_cnt.as<unsigned long long>(), c->p_over.as<int32_t>());
  ++c->launches;
  return cudaGetLastError();
}

// ---------------------------------------------------------------- compaction of the pools

struct PoolSrc {
  const int2 *crow, *prow;
  const int32_t* c_idx;
  const int32_t *p_sphere, *p_inc_off, *p_inc;
  const double *p_vol, *p_m1;
  const uint8_t* p_fm;
  // Euler mode (p_eu == nullptr: off)
  const long long* p_eu;
  const int32_t *p_rpf_off, *p_rpf_j;
  const long long* p_rpf_e;
  const uint8_t *p_sfm, *p_rfm;
  const unsigned long long* p_radj;
  const unsigned long long* p_rep;
};

// per-tet counts of the compacted sets: candidates, pieces, incidences, radical facets
__global__ void k_pool_counts(int64_t T, PoolSrc s, int32_t* __restrict__ cnt) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= T) return;
  const int2 cr = s.crow[t], pr = s.prow[t];
  cnt[t] = cr.y - cr.x;
  cnt[T + t] = pr.y - pr.x;
  cnt[2 * T + t] = pr.y > pr.x ? s.p_inc_off[pr.y] - s.p_inc_off[pr.x] : 0;
  if (s.p_eu) cnt[3 * T + t] = pr.y > pr.x ? s.p_rpf_off[pr.y] - s.p_rpf_off[pr.x] : 0;
}

struct PoolDst {
  const int32_t *c_off, *p_off, *i_tet, *r_tet;  // scans of the counts (new offsets)
  int32_t *c_idx, *pair_tet, *p_sphere, *p_inc_off, *p_inc;
  double *p_vol, *p_m1;
  uint8_t* p_fm;
  long long* p_eu;
  int32_t *p_rpf_off, *p_rpf_j;
  long long* p_rpf_e;
  uint8_t *p_sfm, *p_rfm;
  unsigned long long* p_radj;
  unsigned long long* p_rep;
  int32_t* c_words;  // incidence-mask words of every candidate (scanned into moff)
  const int32_t* nbr_off;
};

#ifndef RPD_MERGE_MT
#define RPD_MERGE_MT 256
#endif
constexpr int MT = RPD_MERGE_MT;  // tets per compaction tile (one block of MT threads)

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

// One block per tile of MT consecutive tets: destination offsets and source bases staged in
// shared memory, then coalesced element loops over the tile's destination ranges (an
// element's tet by binary search over the staged offsets).
__global__ void __launch_bounds__(MT) k_pool_copy(int64_t T, PoolSrc s, PoolDst D) {
  __shared__ int s_nc[MT + 1], s_np[MT + 1], s_ni[MT + 1], s_nr[MT + 1];
  __shared__ int s_sc[MT], s_sp[MT], s_si[MT], s_sr[MT];
  const bool eu = D.p_eu != nullptr;
  const int64_t t0 = (int64_t)blockIdx.x * MT;
  const int nt = (int)min((int64_t)MT, T - t0);
  for (int l = threadIdx.x; l <= nt; l += blockDim.x) {
    const int64_t t = t0 + l;
    s_nc[l] = D.c_off[t];
    s_np[l] = D.p_off[t];
    s_ni[l] = D.i_tet[t];
    if (eu) s_nr[l] = D.r_tet[t];
    if (l < nt) {
      const int2 cr = s.crow[t], pr = s.prow[t];
      s_sc[l] = cr.x;
      s_sp[l] = pr.x;
      s_si[l] = pr.y > pr.x ? s.p_inc_off[pr.x] : 0;
      if (eu) s_sr[l] = pr.y > pr.x ? s.p_rpf_off[pr.x] : 0;
    }
  }
  __syncthreads();
  for (int q = s_nc[0] + threadIdx.x; q < s_nc[nt]; q += blockDim.x) {
    const int l = tile_seg(s_nc, nt, q);
    const int i = s.c_idx[s_sc[l] + (q - s_nc[l])];
    D.c_idx[q] = i;
    D.pair_tet[q] = (int32_t)(t0 + l);
    D.c_words[q] = (__ldg(D.nbr_off + i + 1) - __ldg(D.nbr_off + i) + 31) >> 5;
  }
  for (int q = s_np[0] + threadIdx.x; q < s_np[nt]; q += blockDim.x) {
    const int l = tile_seg(s_np, nt, q);
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
  if (eu)
    for (int r = s_nr[0] + threadIdx.x; r < s_nr[nt]; r += blockDim.x) {
      const int l = tile_seg(s_nr, nt, r);
      const int src = s_sr[l] + (r - s_nr[l]);
      D.p_rpf_j[r] = s.p_rpf_j[src];
      D.p_rpf_e[r] = s.p_rpf_e[src];
      D.p_rfm[r] = s.p_rfm[src];
      D.p_radj[r] = s.p_radj[src];
      D.p_rep[r] = s.p_rep[src];
    }
  for (int r = s_ni[0] + threadIdx.x; r < s_ni[nt]; r += blockDim.x) {
    const int l = tile_seg(s_ni, nt, r);
    D.p_inc[r] = s.p_inc[s_si[l] + (r - s_ni[l])];
  }
  if (t0 + nt == T && threadIdx.x == 0) {  // terminal entries
    D.p_inc_off[s_np[nt]] = s_ni[nt];
    if (eu) D.p_rpf_off[s_np[nt]] = s_nr[nt];
  }
}

static PoolSrc pool_src(const CandSet& cs, const PieceSet& ps, bool eu) {
  return PoolSrc{cs.rows.as<int2>(),       ps.rows.as<int2>(),      cs.idx.as<int32_t>(),
                 ps.sphere.as<int32_t>(),  ps.inc_off.as<int32_t>(), ps.inc.as<int32_t>(),
                 ps.vol.as<double>(),      ps.m1.as<double>(),      ps.fm.as<uint8_t>(),
                 eu ? ps.eu.as<long long>() : nullptr, ps.rpf_off.as<int32_t>(),
                 ps.rpf_j.as<int32_t>(),   ps.rpf_e.as<long long>(), ps.sfm.as<uint8_t>(),
                 ps.rfm.as<uint8_t>(),     ps.radj.as<unsigned long long>(),
                 ps.rep.as<unsigned long long>()};
}

// phase 0: per-tet counts and their scans (cand offsets -> cn.off, piece offsets -> pn.off,
// tet-level incidence offsets -> m_off, tet-level radical-facet offsets -> m_off + 2 (T+1));
// totals at [T] of each.  phase 1: the tiled copy into cn / pn (allocated by the caller from
// the live counts), then the candidates' incidence-mask word offsets (moff) by a scan.
cudaError_t launch_compact_state(rpd_ctx* c, int64_t T, const CandSet& co, const PieceSet& po,
                                 CandSet& cn, PieceSet& pn, int phase) {
  const bool eu = c->euler != 0;
  const PoolSrc s = pool_src(co, po, eu);
  int32_t* m_off = c->m_off.as<int32_t>();
  int32_t* r_off = m_off + 2 * (T + 1);
  if (phase == 0) {
    if (T > 0) {
      k_pool_counts<<<nblk(T, 256), 256, 0, c->stream>>>(T, s, c->m_cnt.as<int32_t>());
      ++c->launches;
    }
    const int32_t* cnt = c->m_cnt.as<int32_t>();
    const int32_t* in[4] = {cnt, cnt + T, cnt + 2 * T, cnt + 3 * T};
    int32_t* out[4] = {cn.off.as<int32_t>(), pn.off.as<int32_t>(), m_off, r_off};
    return launch_scan_i32_multi(c, in, out, eu ? 4 : 3, T);
  }
  PoolDst D{cn.off.as<int32_t>(),       pn.off.as<int32_t>(),     m_off,
            r_off,                      cn.idx.as<int32_t>(),     cn.pair_tet.as<int32_t>(),
            pn.sphere.as<int32_t>(),    pn.inc_off.as<int32_t>(), pn.inc.as<int32_t>(),
            pn.vol.as<double>(),        pn.m1.as<double>(),       pn.fm.as<uint8_t>(),
            eu ? pn.eu.as<long long>() : nullptr, pn.rpf_off.as<int32_t>(),
            pn.rpf_j.as<int32_t>(),     pn.rpf_e.as<long long>(), pn.sfm.as<uint8_t>(),
            pn.rfm.as<uint8_t>(),       pn.radj.as<unsigned long long>(),
            pn.rep.as<unsigned long long>(),
            c->m_cnt.as<int32_t>(),     c->st.nbr_off.as<int32_t>()};
  if (T > 0) {
    k_pool_copy<<<nblk(T, MT), MT, 0, c->stream>>>(T, s, D);
    ++c->launches;
  } else {
    cudaError_t e = cudaMemsetAsync(pn.inc_off.p, 0, sizeof(int32_t), c->stream);
    if (e) return e;
  }
  return launch_scan_i32(c, c->m_cnt.as<int32_t>(), cn.moff.as<int32_t>(), cn.n);
}

}  // namespace rpd
