// rpd_gather.cu -- SURVEY.md §8(a) row a7 / §8(e): the multi-GPU exchange of the RPD.
//
// Every rank clips its own tet shard; the per-rank candidate and piece CSRs are all-gathered
// by NCCL (torch.distributed, plumbing) and the kernels here put them back into global tet
// order.  In partial mode only the dirty tets' segments travel, and they replace those tets'
// segments of the previous global CSR (the clean tets keep theirs byte-identically, R11).
//
// One segment-gather engine serves every case: a row map sends each output row (a tet) to
// (source, row) -- source 0 the previous global CSR or the ctx's own state, sources 1.. the
// ranks' gathered shards -- then per output row its candidate / piece / incidence counts are
// read (k_seg_count), scanned into the output offsets, and its segments copied
// (k_seg_copy_tiled: coalesced element loops per tile of output rows).  Integer work and copies only: results are byte-identical to a
// single-GPU run (per-tet outputs do not depend on the shard).
#include "rpd_ctx.h"

namespace rpd {

static inline unsigned nblk(int64_t n, int b) { return (unsigned)((n + b - 1) / b); }

__global__ void k_map_fill(int64_t n, int2* __restrict__ map) {
  const int64_t o = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (o < n) map[o] = make_int2(0, (int)o);  // row o of source 0
}

__global__ void k_map_list(const int32_t* __restrict__ list, int64_t n, int64_t T,
                           int2* __restrict__ map, int* err) {
  const int64_t o = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (o >= n) return;
  const int t = list[o];
  if (t < 0 || t >= T) {
    if (atomicCAS(err, 0, (int)RPD_EINVAL) == 0) {
      err[1] = ERR_TET_INDEX;
      err[2] = (int)o;
    }
    map[o] = make_int2(-1, 0);
    return;
  }
  map[o] = make_int2(0, t);
}

// shard r's local row a -> output row tet_ids[r][a], source 1 + r (checked: ids in [0, T))
__global__ void k_map_shards(SegShards v, int64_t T, int2* __restrict__ map, int* err) {
  const int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (x >= v.base[v.world]) return;
  int r = 0;
  while (r + 1 < v.world && v.base[r + 1] <= x) ++r;
  const int64_t a = x - v.base[r];
  const int t = v.tet_ids[r][a];
  if (t < 0 || t >= T) {
    if (atomicCAS(err, 0, (int)RPD_EINVAL) == 0) {
      err[1] = ERR_TET_INDEX;
      err[2] = (int)x;
    }
    return;
  }
  map[t] = make_int2(1 + r, (int)a);
}

// per output row: candidates, pieces, incidences of its source segment (0 for unmapped rows)
__global__ void k_seg_count(int64_t n, const int2* __restrict__ map, SegSources S,
                            int32_t* __restrict__ cc, int32_t* __restrict__ pc,
                            int32_t* __restrict__ ic) {
  const int64_t o = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (o >= n) return;
  const int2 m = map[o];
  int nc = 0, np = 0, ni = 0;
  if (m.x >= 0) {
    const SegSrc& s = S.s[m.x];
    const int64_t r = (int64_t)m.y * s.rs;
    if (s.c_beg) nc = s.c_end[r] - s.c_beg[r];
    if (s.p_beg) {
      const int p0 = s.p_beg[r], p1 = s.p_end[r];
      np = p1 - p0;
      ni = p1 > p0 ? s.i_off[p1] - s.i_off[p0] : 0;
    }
  }
  if (cc) cc[o] = nc;
  if (pc) pc[o] = np;
  if (ic) ic[o] = ni;
}

// ids_out[k] = id_map[list[k]] (or list[k]): the global ids of downloaded local tets
__global__ void k_map_ids(const int32_t* __restrict__ list, int64_t n,
                          const int32_t* __restrict__ id_map, int64_t T,
                          int32_t* __restrict__ ids_out) {
  const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (k >= n) return;
  const int t = list[k];
  ids_out[k] = id_map && t >= 0 && t < T ? id_map[t] : t;
}

cudaError_t launch_map_ids(rpd_ctx* c, const int32_t* list, int64_t n, const int32_t* id_map,
                           int64_t T, int32_t* ids_out) {
  if (n == 0) return cudaSuccess;
  k_map_ids<<<nblk(n, 256), 256, 0, c->stream>>>(list, n, id_map, T, ids_out);
  ++c->launches;
  return cudaGetLastError();
}

SegSrc seg_src_csr(const int32_t* c_off, const int32_t* c_idx, const int32_t* p_off,
                   const int32_t* p_sphere, const double* p_vol, const double* p_m1,
                   const uint8_t* p_fm, const int32_t* i_off, const int32_t* i_sph) {
  SegSrc s{};
  s.rs = 1;
  if (c_off) {
    s.c_beg = c_off;
    s.c_end = c_off + 1;
    s.c_idx = c_idx;
  }
  if (p_off) {
    s.p_beg = p_off;
    s.p_end = p_off + 1;
    s.p_sphere = p_sphere;
    s.p_vol = p_vol;
    s.p_m1 = p_m1;
    s.p_fm = p_fm;
    s.i_off = i_off;
    s.i_sph = i_sph;
  }
  return s;
}

// the ctx state: the pools addressed by their int2 rows
SegSrc seg_src_state(const CandSet& cs, const PieceSet& ps) {
  SegSrc s{};
  s.rs = 2;
  const int32_t* cr = reinterpret_cast<const int32_t*>(cs.rows.p);
  const int32_t* pr = reinterpret_cast<const int32_t*>(ps.rows.p);
  if (cr) {
    s.c_beg = cr;
    s.c_end = cr + 1;
    s.c_idx = cs.idx.as<int32_t>();
  }
  if (pr) {
    s.p_beg = pr;
    s.p_end = pr + 1;
    s.p_sphere = ps.sphere.as<int32_t>();
    s.p_vol = ps.vol.as<double>();
    s.p_m1 = ps.m1.as<double>();
    s.p_fm = ps.fm.as<uint8_t>();
    s.i_off = ps.inc_off.as<int32_t>();
    s.i_sph = ps.inc.as<int32_t>();
  }
  return s;
}

cudaError_t launch_map(rpd_ctx* c, int kind, int64_t n_out, const int32_t* list,
                       const SegShards* sh, int64_t T) {
  cudaError_t e = c->g_map.ensure(sizeof(int2) * (n_out > 0 ? n_out : 1));
  if (e) return e;
  int2* map = c->g_map.as<int2>();
  if (n_out == 0) return cudaSuccess;
  if (kind == 0 || kind == 2) {  // identity (source 0), optionally overwritten by shards
    k_map_fill<<<nblk(n_out, 256), 256, 0, c->stream>>>(n_out, map);
    ++c->launches;
  } else if (kind == 1) {  // explicit list of source-0 rows
    k_map_list<<<nblk(n_out, 256), 256, 0, c->stream>>>(list, n_out, T, map, c->errw.as<int>());
    ++c->launches;
  }
  if (kind == 3) {  // unmapped rows (no rank holds them) count zero
    if ((e = cudaMemsetAsync(map, 0xff, sizeof(int2) * n_out, c->stream))) return e;
  }
  if ((kind == 2 || kind == 3) && sh->base[sh->world] > 0) {
    k_map_shards<<<nblk(sh->base[sh->world], 256), 256, 0, c->stream>>>(*sh, T, map,
                                                                         c->errw.as<int>());
    ++c->launches;
  }
  return cudaGetLastError();
}

// counts of the mapped rows -> output offsets (cand_off / piece_off / tet-level incidence
// offsets); totals at [n_out]
cudaError_t launch_seg_counts(rpd_ctx* c, int64_t n_out, const SegSources& S, int32_t* cand_off,
                              int32_t* piece_off, int32_t** i_tet_out) {
  cudaError_t e = c->g_cnt.ensure(sizeof(int32_t) * 4 * (n_out + 1));
  if (e) return e;
  int32_t* cc = c->g_cnt.as<int32_t>();
  int32_t* pc = cc + (n_out + 1);
  int32_t* ic = pc + (n_out + 1);
  int32_t* it = ic + (n_out + 1);
  *i_tet_out = it;
  if (n_out > 0) {
    k_seg_count<<<nblk(n_out, 256), 256, 0, c->stream>>>(n_out, c->g_map.as<int2>(), S,
                                                         cand_off ? cc : nullptr,
                                                         piece_off ? pc : nullptr,
                                                         piece_off ? ic : nullptr);
    ++c->launches;
  }
  const int32_t* in[3];
  int32_t* out[3];
  int K = 0;
  if (cand_off) {
    in[K] = cc;
    out[K++] = cand_off;
  }
  if (piece_off) {
    in[K] = pc;
    out[K++] = piece_off;
    in[K] = ic;
    out[K++] = it;
  }
  return K ? launch_scan_i32_multi(c, in, out, K, n_out) : cudaSuccess;
}

// Tiled copy (one block per SEG_TILE output rows): the rows' source bases and destination
// offsets staged in shared memory, then coalesced loops over the tile's destination ranges of
// candidates, pieces and incidences (an element's row by binary search over the staged
// offsets).  Rows taken in order from one source (a gather's shard, the clean rows of a merge)
// read contiguous source memory.
constexpr int SEG_TILE = 256;

__device__ __forceinline__ int seg_of(const int* off, int n, int q) {
  int lo = 0, hi = n;  // off[lo] <= q < off[hi]
  while (hi - lo > 1) {
    const int mid = (lo + hi) >> 1;
    if (off[mid] <= q) lo = mid;
    else hi = mid;
  }
  return lo;
}

__global__ void __launch_bounds__(SEG_TILE) k_seg_copy_tiled(int64_t n, const int2* __restrict__ map,
                                                              SegSources S, SegDst D) {
  __shared__ int s_dc[SEG_TILE + 1], s_dp[SEG_TILE + 1], s_di[SEG_TILE + 1];
  __shared__ int s_src[SEG_TILE], s_sc[SEG_TILE], s_sp[SEG_TILE], s_si[SEG_TILE];
  const int64_t o0 = (int64_t)blockIdx.x * SEG_TILE;
  const int nt = (int)min((int64_t)SEG_TILE, n - o0);
  const bool cands = D.cand_idx != nullptr, pieces = D.piece_off != nullptr;
  for (int l = threadIdx.x; l <= nt; l += blockDim.x) {
    const int64_t o = o0 + l;
    s_dc[l] = cands ? D.cand_off[o] : 0;
    s_dp[l] = pieces ? D.piece_off[o] : 0;
    s_di[l] = pieces ? D.i_tet[o] : 0;
    if (l < nt) {
      const int2 m = map[o];
      s_src[l] = m.x;
      if (m.x >= 0) {
        const SegSrc& s = S.s[m.x];
        const int64_t r = (int64_t)m.y * s.rs;
        s_sc[l] = s.c_beg ? s.c_beg[r] : 0;
        const int p0 = s.p_beg ? s.p_beg[r] : 0;
        s_sp[l] = p0;
        s_si[l] = s.p_beg && s.p_end[r] > p0 ? s.i_off[p0] : 0;
      }
    }
  }
  __syncthreads();
  if (cands)
    for (int q = s_dc[0] + threadIdx.x; q < s_dc[nt]; q += blockDim.x) {
      const int l = seg_of(s_dc, nt, q);
      D.cand_idx[q] = S.s[s_src[l]].c_idx[s_sc[l] + (q - s_dc[l])];
    }
  if (pieces) {
    for (int q = s_dp[0] + threadIdx.x; q < s_dp[nt]; q += blockDim.x) {
      const int l = seg_of(s_dp, nt, q);
      const SegSrc& s = S.s[s_src[l]];
      const int p = s_sp[l] + (q - s_dp[l]);
      D.piece_sphere[q] = s.p_sphere[p];
      D.piece_vol[q] = s.p_vol[p];
      D.piece_m1[3 * (int64_t)q] = s.p_m1[3 * (int64_t)p];
      D.piece_m1[3 * (int64_t)q + 1] = s.p_m1[3 * (int64_t)p + 1];
      D.piece_m1[3 * (int64_t)q + 2] = s.p_m1[3 * (int64_t)p + 2];
      D.piece_fm[q] = s.p_fm[p];
      D.inc_off[q] = s_di[l] + (s.i_off[p] - s_si[l]);
    }
    for (int q = s_di[0] + threadIdx.x; q < s_di[nt]; q += blockDim.x) {
      const int l = seg_of(s_di, nt, q);
      D.inc_sphere[q] = S.s[s_src[l]].i_sph[s_si[l] + (q - s_di[l])];
    }
    if (o0 + nt == n && threadIdx.x == 0) D.inc_off[s_dp[nt]] = s_di[nt];  // terminal entry
  }
}

cudaError_t launch_seg_copy(rpd_ctx* c, int64_t n_out, const SegSources& S, const SegDst& D) {
  if (n_out == 0) {
    if (D.piece_off) return cudaMemsetAsync(D.inc_off, 0, sizeof(int32_t), c->stream);
    return cudaSuccess;
  }
  k_seg_copy_tiled<<<nblk(n_out, SEG_TILE), SEG_TILE, 0, c->stream>>>(n_out, c->g_map.as<int2>(),
                                                                      S, D);
  ++c->launches;
  return cudaGetLastError();
}

}  // namespace rpd
