// rpd_gather.cu -- SURVEY.md §8(a) row a7 / §8(e): the multi-GPU gather of the pieces.
//
// Every rank clips its own tet shard; the per-rank piece CSRs are all-gathered by NCCL
// (torch.distributed, plumbing) and this kernel pair puts them back into global tet order on
// every rank: per global tet its piece count and incidence count are scattered from the
// owning rank (k_g_count), scanned into the global offsets, and every rank's pieces and
// incidences copied to their global positions (k_g_copy; one thread per local tet, its few
// pieces and incidences contiguous in source and destination).  Integer work and copies: the
// result is byte-identical to a single-GPU run (per-tet outputs do not depend on the shard).
#include "rpd_ctx.h"

namespace rpd {

static inline unsigned nblk(int64_t n, int b) { return (unsigned)((n + b - 1) / b); }

struct ShardView {
  int world;
  int64_t base[RPD_MAX_RANKS + 1];  // prefix of the ranks' local tet counts
  const int32_t* tet_ids[RPD_MAX_RANKS];
  const int32_t* piece_off[RPD_MAX_RANKS];
  const int32_t* piece_sphere[RPD_MAX_RANKS];
  const double* piece_vol[RPD_MAX_RANKS];
  const double* piece_m1[RPD_MAX_RANKS];
  const uint8_t* piece_facemask[RPD_MAX_RANKS];
  const int32_t* inc_off[RPD_MAX_RANKS];
  const int32_t* inc_sphere[RPD_MAX_RANKS];
};

__device__ __forceinline__ int rank_of(const ShardView& v, int64_t x) {
  int r = 0;
  while (r + 1 < v.world && v.base[r + 1] <= x) ++r;
  return r;
}

// every rank's global tet ids in [0, T) (before any kernel writes through them)
__global__ void k_g_check(ShardView v, int64_t T, int* err) {
  const int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (x >= v.base[v.world]) return;
  const int r = rank_of(v, x);
  const int t = v.tet_ids[r][x - v.base[r]];
  if ((t < 0 || t >= T) && atomicCAS(err, 0, (int)RPD_EINVAL) == 0) {
    err[1] = ERR_TET_INDEX;
    err[2] = (int)x;
  }
}

// per global tet: pieces and incidences (from the owning rank)
__global__ void k_g_count(ShardView v, int32_t* __restrict__ pc, int32_t* __restrict__ ic) {
  const int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (x >= v.base[v.world]) return;
  const int r = rank_of(v, x);
  const int64_t a = x - v.base[r];
  const int32_t* po = v.piece_off[r];
  const int32_t* io = v.inc_off[r];
  const int t = v.tet_ids[r][a];
  const int p0 = po[a], p1 = po[a + 1];
  pc[t] = p1 - p0;
  ic[t] = io[p1] - io[p0];
}

__global__ void k_g_copy(ShardView v, const int32_t* __restrict__ goff,
                         const int32_t* __restrict__ gioff, int32_t* __restrict__ sphere,
                         double* __restrict__ vol, double* __restrict__ m1,
                         uint8_t* __restrict__ fm, int32_t* __restrict__ inc_off,
                         int32_t* __restrict__ inc, int64_t T) {
  const int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (x == 0) inc_off[goff[T]] = gioff[T];  // terminal entry
  if (x >= v.base[v.world]) return;
  const int r = rank_of(v, x);
  const int64_t a = x - v.base[r];
  const int t = v.tet_ids[r][a];
  const int32_t* po = v.piece_off[r];
  const int32_t* io = v.inc_off[r];
  const int p0 = po[a], p1 = po[a + 1];
  const int q0 = goff[t], i0 = io[p0], gi0 = gioff[t];
  for (int p = p0; p < p1; ++p) {
    const int q = q0 + (p - p0);
    sphere[q] = v.piece_sphere[r][p];
    vol[q] = v.piece_vol[r][p];
    m1[3 * (int64_t)q] = v.piece_m1[r][3 * (int64_t)p];
    m1[3 * (int64_t)q + 1] = v.piece_m1[r][3 * (int64_t)p + 1];
    m1[3 * (int64_t)q + 2] = v.piece_m1[r][3 * (int64_t)p + 2];
    fm[q] = v.piece_facemask[r][p];
    inc_off[q] = gi0 + (io[p] - i0);
  }
  for (int k = i0; k < io[p1]; ++k) inc[gi0 + (k - i0)] = v.inc_sphere[r][k];
}

static ShardView view_of(const rpd_shards* in) {
  ShardView v{};
  v.world = in->world;
  v.base[0] = 0;
  for (int r = 0; r < in->world; ++r) {
    v.base[r + 1] = v.base[r] + in->n_tets[r];
    v.tet_ids[r] = in->tet_ids[r];
    v.piece_off[r] = in->piece_off[r];
    v.piece_sphere[r] = in->piece_sphere[r];
    v.piece_vol[r] = in->piece_vol[r];
    v.piece_m1[r] = in->piece_m1[r];
    v.piece_facemask[r] = in->piece_facemask[r];
    v.inc_off[r] = in->inc_off[r];
    v.inc_sphere[r] = in->inc_sphere[r];
  }
  return v;
}

cudaError_t launch_gather_check(rpd_ctx* c, const rpd_shards* in) {
  const ShardView v = view_of(in);
  const int64_t n = v.base[in->world];
  if (n > 0) {
    k_g_check<<<nblk(n, 256), 256, 0, c->stream>>>(v, in->T, c->errw.as<int>());
    ++c->launches;
  }
  return cudaGetLastError();
}

cudaError_t launch_gather(rpd_ctx* c, const rpd_shards* in, int32_t* piece_off,
                          int32_t* piece_sphere, double* piece_vol, double* piece_m1,
                          uint8_t* piece_facemask, int32_t* inc_off, int32_t* inc_sphere) {
  const ShardView v = view_of(in);
  const int64_t T = in->T, n = v.base[in->world];
  cudaError_t e = c->g_cnt.ensure(sizeof(int32_t) * (3 * (T + 1) + 1));
  if (e) return e;
  int32_t* pc = c->g_cnt.as<int32_t>();
  int32_t* ic = pc + (T + 1);
  int32_t* gioff = ic + (T + 1);
  // tets no rank holds count zero (every tet belongs to one shard; this keeps the scan defined)
  if ((e = cudaMemsetAsync(pc, 0, sizeof(int32_t) * 2 * (T + 1), c->stream))) return e;
  if (n > 0) {
    k_g_count<<<nblk(n, 256), 256, 0, c->stream>>>(v, pc, ic);
    ++c->launches;
  }
  const int32_t* sin[2] = {pc, ic};
  int32_t* sout[2] = {piece_off, gioff};
  if ((e = launch_scan_i32_multi(c, sin, sout, 2, T))) return e;
  k_g_copy<<<nblk(n > 0 ? n : 1, 256), 256, 0, c->stream>>>(v, piece_off, gioff, piece_sphere,
                                                           piece_vol, piece_m1, piece_facemask,
                                                           inc_off, inc_sphere, T);
  ++c->launches;
  return cudaGetLastError();
}

}  // namespace rpd
