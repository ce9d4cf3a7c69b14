// rpd_api.cu -- the C ABI of librpd (include/rpd.h).  Host-side orchestration only: every
// step of the path runs in the kernels of rpd_stage.cu, rpd_filter.cu, rpd_scan.cu,
// rpd_clip.cu and rpd_partial.cu.
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include <string>
#include <vector>

#include <chrono>
#include <cmath>

#include "rpd_ctx.h"
#include "rpd_internal.cuh"

using namespace rpd;

#define RPD_VERSION "rpd-b200 0.1 (sm_100a)"

#include <mutex>
#include <set>

namespace rpd {
bool canary_on() {
  static const bool on = [] {
    const char* v = getenv("RPD_CANARY");
    return v && *v && *v != '0';
  }();
  return on;
}
static std::mutex& canary_mu() {
  static std::mutex m;
  return m;
}
static std::set<DevBuf*>& canary_set() {
  static std::set<DevBuf*>* s = new std::set<DevBuf*>();  // (never destroyed: exit order)
  return *s;
}
void canary_register(DevBuf* b) {
  std::lock_guard<std::mutex> g(canary_mu());
  canary_set().insert(b);
}
void canary_unregister(DevBuf* b) {
  std::lock_guard<std::mutex> g(canary_mu());
  canary_set().erase(b);
}
__global__ void k_canary(const unsigned char* const* __restrict__ tails, int n,
                         int* __restrict__ bad) {
  for (int q = blockIdx.x; q < n; q += gridDim.x)
    for (int k = threadIdx.x; k < (int)CANARY_BYTES; k += blockDim.x)
      if (tails[q][k] != 0xA5) atomicCAS(bad, -1, q);
}
}  // namespace rpd

namespace {

rpd_status fail(rpd_ctx* c, rpd_status s, const std::string& msg) {
  if (c) c->err = msg;
  return s;
}

rpd_status cuda_fail(rpd_ctx* c, cudaError_t e, const char* where) {
  if (e == cudaErrorMemoryAllocation) {
    cudaGetLastError();
    return fail(c, RPD_ENOMEM, std::string(where) + ": " + cudaGetErrorString(e));
  }
  return fail(c, RPD_ECUDA, std::string(where) + ": " + cudaGetErrorString(e));
}

#define CK(expr, where)                              \
  do {                                               \
    cudaError_t _e = (expr);                         \
    if (_e != cudaSuccess) return cuda_fail(c, _e, where); \
  } while (0)

bool is_host_ptr(const void* p) {
  if (!p) return false;
  cudaPointerAttributes a;
  cudaError_t e = cudaPointerGetAttributes(&a, p);
  if (e != cudaSuccess) {
    cudaGetLastError();
    return true;
  }
  return a.type == cudaMemoryTypeHost || a.type == cudaMemoryTypeUnregistered;
}

// device view of an input array (copies host arrays into ctx-owned staging memory)
template <class T>
cudaError_t resolve(rpd_ctx* c, const T* p, size_t count, DevBuf& stage, const T** out) {
  if (count == 0 || !is_host_ptr(p)) {
    *out = p;
    return cudaSuccess;
  }
  cudaError_t e = stage.ensure(sizeof(T) * count);
  if (e) return e;
  e = cudaMemcpyAsync(stage.p, p, sizeof(T) * count, cudaMemcpyHostToDevice, c->stream);
  *out = stage.as<T>();
  return e;
}

const char* err_kind_str(int k) {
  switch (k) {
    case ERR_VERT_LATTICE: return "vertex coordinate off the 2^-10 lattice or outside [0,64)";
    case ERR_VERT_NAN: return "vertex coordinate is NaN/Inf";
    case ERR_SPHERE_LATTICE: return "sphere centre/radius off the 2^-10 lattice or outside [0,64)";
    case ERR_SPHERE_NAN: return "sphere value is NaN/Inf";
    case ERR_RADIUS_NEG: return "negative radius";
    case ERR_TET_INDEX: return "tet vertex index out of range";
    case ERR_TET_ORIENT: return "tet not positively oriented";
    case ERR_NBR_INDEX: return "neighbour index out of range";
    case ERR_NBR_SELF: return "sphere lists itself as a neighbour";
    case ERR_NBR_DUP: return "duplicate neighbour";
    case ERR_NBR_SAME_CENTRE: return "neighbour with the same centre (radical plane undefined)";
    case ERR_NBR_OFF: return "bad neighbour CSR offsets";
    case ERR_SPHERE_CHANGED:
      return "partial update: an existing sphere [0, N_old) changed (only appending is allowed)";
    case ERR_NB_RECOMPUTE:
      return "neighbour lists: a long row recomputed with another length (internal error)";
    default: return "invalid input";
  }
}

// host round trips: up to 8 int32 device scalars, the stats and the error word are gathered
// by one tiny kernel straight into mapped pinned memory (no copy-engine operations)
struct Readback {
  int32_t i32[8];
  unsigned long long u64[ST_N];
  int32_t err[4];
  unsigned long long u4[4];
};

struct RbSpec {
  const int32_t* i32[8];           // nullptr -> 0
  const unsigned long long* u64;   // stats (ST_N words) or nullptr (kept)
  const int* err;                  // error word (4) or nullptr (kept)
  const unsigned long long* u4 = nullptr;  // 4 more u64 words or nullptr (kept)
};

__global__ void k_readback(RbSpec s, Readback* rb) {
  const int t = threadIdx.x;
  if (t < 8) rb->i32[t] = s.i32[t] ? *s.i32[t] : 0;
  if (s.u64 && t < ST_N) rb->u64[t] = s.u64[t];
  if (s.err && t < 4) rb->err[t] = s.err[t];
  if (s.u4 && t < 4) rb->u4[t] = s.u4[t];
  __threadfence_system();
}

cudaError_t readback(rpd_ctx* c, const RbSpec& s) {
  k_readback<<<1, 32, 0, c->stream>>>(s, (Readback*)c->pinned_dev);
  ++c->launches;
  return cudaGetLastError();
}

rpd_status check_err(rpd_ctx* c, const Readback* rb) {
  if (rb->err[0] != 0) {
    char buf[256];
    snprintf(buf, sizeof buf, "%s (element %d)", err_kind_str(rb->err[1]), rb->err[2]);
    return fail(c, (rpd_status)rb->err[0], buf);
  }
  return RPD_OK;
}

}  // namespace

static rpd_status download_rows(rpd_ctx* c, int kind, const int32_t* d_list, int64_t n,
                                rpd_csr* out);

extern "C" {

const char* rpd_version(void) { return RPD_VERSION; }

rpd_status rpd_create(rpd_ctx** out, int device, void* cuda_stream) {
  if (!out) return RPD_EINVAL;
  *out = nullptr;
  rpd_ctx* c = new rpd_ctx();
  c->device = device;
  cudaError_t e = cudaSetDevice(device);
  if (!e) e = cudaDeviceGetAttribute(&c->sms, cudaDevAttrMultiProcessorCount, device);
  if (e) {
    delete c;
    return RPD_ECUDA;
  }
  if (cuda_stream) {
    c->stream = (cudaStream_t)cuda_stream;
  } else {
    if (cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking)) {
      delete c;
      return RPD_ECUDA;
    }
    c->own_stream = true;
  }
  if (c->errw.ensure(sizeof(int) * 4) || c->stats.ensure(sizeof(unsigned long long) * ST_N) ||
      cudaHostAlloc(&c->pinned, sizeof(Readback), cudaHostAllocMapped) ||
      cudaHostGetDevicePointer(&c->pinned_dev, c->pinned, 0)) {
    rpd_destroy(c);
    return RPD_ENOMEM;
  }
  {
    const char* g = getenv("RPD_GRAPH");
    if (g && *g == '0') c->graph = 0;
    const char* n = getenv("RPD_GRAPH_NC_MAX");  // testing: a fixed batch bound
    if (n && *n) c->g_nc_fix = atoll(n);
    const char* r = getenv("RPD_CLIP_ROUTE");  // graph clip routing threshold (cut planes)
    if (r && *r) c->clip_route = atoi(r);
  }
  *out = c;
  return RPD_OK;
}

static void graph_clear(rpd_ctx* c);

void rpd_destroy(rpd_ctx* c) {
  if (!c) return;
  cudaSetDevice(c->device);
  if (c->stream) cudaStreamSynchronize(c->stream);
  DevBuf* bufs[] = {&c->h_verts, &c->h_tets, &c->h_spheres, &c->h_off, &c->h_idx, &c->h_new,
                    &c->st.tx, &c->st.sw, &c->st.nbr_off, &c->st.nbr_idx, &c->st.planes,
                    &c->st.twin, &c->st.hkey, &c->st.old_off, &c->st.old_idx, &c->st.old_planes,
                    &c->st.old_twin, &c->st.old_hkey, &c->st.old_sw, &c->errw, &c->stats, &c->scratch, &c->k_tet, &c->k_words,
                    &c->slab, &c->slab_m, &c->w_off, &c->bvh, &c->bvh_all, &c->bvh_items, &c->p_flag, &c->p_f01, &c->p_vol, &c->p_m1, &c->p_fm,
                    &c->p_ninc, &c->p_mask, &c->p_over, &c->p_over2, &c->p_over3, &c->p_dyn, &c->p_scan, &c->i_scan, &c->d_count,
                    &c->d_flag, &c->d_scan, &c->d_list, &c->m_cnt, &c->m_off, &c->c_scan, &c->c_list,
                    &c->st.repoch, &c->st.old_repoch, &c->st.htab, &c->c_flag, &c->cepoch,
                    &c->min_epoch, &c->eu_tab, &c->eu_rec, &c->eu_A, &c->eu_sum, &c->eu_Lt, &c->eu_acc, &c->eu_fin, &c->eu_den, &c->p_eu,
                    &c->p_rmask, &c->p_rval, &c->p_nrpf, &c->r_scan, &c->h_eut, &c->h_euid,
                    &c->p_sfm, &c->p_rfm, &c->eu_adj, &c->cc_par, &c->cc_out, &c->cand_long, &c->g_cnt, &c->g_map, &c->g_off, &c->g_dst, &c->g_ids, &c->h_dl, &c->h_dm, &c->env_buf, &c->env_out, &c->h_env, &c->h_env2, &c->h_env3, &c->h_env4, &c->p_radj, &c->p_rep, &c->rpe_off, &c->rpe_buf, &c->rpe_ee, &c->mm_keys, &c->mm_tmp, &c->mm_out};
  for (DevBuf* b : bufs) b->release();
  CandSet* cs[] = {&c->cand[0], &c->cand[1], &c->cand_d, &c->g_cand[0], &c->g_cand[1]};
  for (CandSet* x : cs) {
    x->off.release();
    x->idx.release();
    x->pair_tet.release();
    x->moff.release();
    x->cut.release();
    x->rows.release();
  }
  PieceSet* ps[] = {&c->pcs[0], &c->pcs[1], &c->pcs_d, &c->g_pcs[0], &c->g_pcs[1]};
  for (PieceSet* x : ps) {
    x->off.release();
    x->sphere.release();
    x->vol.release();
    x->m1.release();
    x->fm.release();
    x->inc_off.release();
    x->inc.release();
    x->eu.release();
    x->rpf_off.release();
    x->rpf_j.release();
    x->rpf_e.release();
    x->sfm.release();
    x->rfm.release();
    x->radj.release();
    x->rep.release();
    x->rows.release();
  }
  graph_clear(c);
  if (c->cap_stream) cudaStreamDestroy(c->cap_stream);
  if (c->side_stream) cudaStreamDestroy(c->side_stream);
  if (c->g_fork) cudaEventDestroy(c->g_fork);
  if (c->g_join) cudaEventDestroy(c->g_join);
  for (DevBuf* b : {&c->nb_buf, &c->nb_off, &c->nb_idx, &c->nb_tmp, &c->nb_cnt, &c->h_nb,
                    &c->nb_hits, &c->nb_prev, &c->nb_off2, &c->nb_idx2, &c->nb_flag, &c->nb_list,
                    &c->nb_len, &c->nb_misc, &c->bvh_items, &c->min_epoch,
                    &c->nb_ball, &c->eu_ids, &c->eu_g2l, &c->cc_bnd, &c->cc_gpar, &c->cc_sort,
                    &c->cc_nrec, &c->st.long_rows, &c->p_route, &c->rpe_bnd, &c->rpe_cnt,
                    &c->rk_buf, &c->rk_out})
    b->release();
  if (c->pd_host) cudaFreeHost(c->pd_host);
  for (DevBuf* b : {&c->pd_buf, &c->g_scan, &c->st.nbr_off, &c->st.nbr_idx, &c->st.planes,
                    &c->st.twin, &c->st.hkey, &c->st.old_repoch, &c->st.repoch})
    b->release();
  if (c->pinned) cudaFreeHost(c->pinned);
  for (int k = 0; k < 4; ++k)
    if (c->ev[k]) cudaEventDestroy(c->ev[k]);

  if (c->own_stream && c->stream) cudaStreamDestroy(c->stream);
  delete c;
}

const char* rpd_last_error(const rpd_ctx* c) {
  if (!c) return "null rpd_ctx";
  return c->err.c_str();
}

rpd_status rpd_set_option(rpd_ctx* c, int option, int64_t value) {
  if (!c) return RPD_EINVAL;
  switch (option) {
    case RPD_OPT_FILTER_MODE:
      if (value != RPD_FILTER_ALL_PAIRS && value != RPD_FILTER_PRUNED)
        return fail(c, RPD_EINVAL, "bad filter mode");
      c->filter_mode = (int)value;
      return RPD_OK;
    case RPD_OPT_VALIDATE:
      c->validate = value ? 1 : 0;
      return RPD_OK;
    case RPD_OPT_PROFILE:
      c->profile = value ? 1 : 0;
      if (c->profile && !c->ev[0])
        for (int k = 0; k < 4; ++k) cudaEventCreate(&c->ev[k]);
      return RPD_OK;
    case RPD_OPT_CLIP_WIDE:
      c->clip_wide = value ? 1 : 0;
      return RPD_OK;
    case RPD_OPT_CLIP_TIERS:
      c->clip_tiers = value ? 1 : 0;
      return RPD_OK;
    case RPD_OPT_GRAPH:
      c->graph = value ? 1 : 0;
      return RPD_OK;
    case RPD_OPT_STREAM:
      if (c->own_stream && c->stream) cudaStreamDestroy(c->stream);
      c->own_stream = false;
      c->stream = (cudaStream_t)(intptr_t)value;
      return RPD_OK;
    default:
      return fail(c, RPD_EINVAL, "unknown option");
  }
}

// ------------------------------------------------------------------ internal steps

// E = nbr_off[N] (host or device pointer)
static rpd_status read_E(rpd_ctx* c, const int32_t* nbr_off, int64_t N, int64_t* E) {
  if (*E >= 0 || N <= 0) {  // given by the caller (checked against nbr_off[N] on the device)
    if (N <= 0) *E = 0;
    return RPD_OK;
  }
  if (is_host_ptr(nbr_off)) {
    *E = nbr_off[N];
  } else {
    Readback* rb = (Readback*)c->pinned;
    CK(readback(c, RbSpec{{nbr_off + N}, nullptr, nullptr}), "read nbr_off[N]");
    CK(cudaStreamSynchronize(c->stream), "sync");
    *E = rb->i32[0];
  }
  if (*E < 0) return fail(c, RPD_EINVAL, "nbr_off[N] < 0");
  return RPD_OK;
}

static rpd_status stage_spheres(rpd_ctx* c, const double* spheres, int64_t N,
                                const int32_t* nbr_off, const int32_t* nbr_idx, int64_t E,
                                bool reuse_rows, int epoch) {
  rpd_status s = read_E(c, nbr_off, N, &E);
  if (s) return s;
  if (E > 0 && !nbr_idx) return fail(c, RPD_EINVAL, "nbr_idx is NULL");
  const double* d_sph = nullptr;
  const int32_t *d_off = nullptr, *d_idx = nullptr;
  CK(resolve(c, spheres, 4 * N, c->h_spheres, &d_sph), "stage spheres");
  CK(resolve(c, nbr_off, N > 0 ? N + 1 : 0, c->h_off, &d_off), "stage nbr_off");
  CK(resolve(c, nbr_idx, E, c->h_idx, &d_idx), "stage nbr_idx");
  CK(launch_stage_spheres(c, d_sph, N, d_off, d_idx, E, reuse_rows, epoch), "stage spheres");
  return RPD_OK;
}

// development trace (env RPD_TRACE_HOST=1): marks on the host clock and on the ctx stream
static void tmark(rpd_ctx* c, const char* name) {
  if (c->tr_on < 0) {
    const char* v = getenv("RPD_TRACE_HOST");
    c->tr_on = v && *v ? 1 : 0;
  }
  if (!c->tr_on || c->tr_n >= 16) return;
  if (!c->tr_ev[c->tr_n]) cudaEventCreate(&c->tr_ev[c->tr_n]);
  cudaEventRecord(c->tr_ev[c->tr_n], c->stream);
  c->tr_h[c->tr_n] = std::chrono::duration<double, std::milli>(
                         std::chrono::steady_clock::now().time_since_epoch()).count();
  c->tr_nm[c->tr_n++] = name;
}
static void tdump(rpd_ctx* c) {
  if (c->tr_on != 1 || c->tr_n == 0) return;
  cudaEventSynchronize(c->tr_ev[c->tr_n - 1]);
  fprintf(stderr, "[rpd trace]");
  for (int k = 0; k < c->tr_n; ++k) {
    float g = 0.f;
    cudaEventElapsedTime(&g, c->tr_ev[0], c->tr_ev[k]);
    fprintf(stderr, " %s h%.3f/g%.3f", c->tr_nm[k], c->tr_h[k] - c->tr_h[0], g);
  }
  fprintf(stderr, "\n");
  c->tr_n = 0;
}

// Alg. 1 over tets (tet_ids, or all ctx tets when NULL) x spheres [lo, hi) -> candidate set
// restricted re-filter of dirty tets (partial update, pruned mode): only the spheres of
// `list` (changed rows) are traversed, the old candidates with unchanged rows are kept
struct Restrict {
  const int32_t* list;
  const int* n_list_dev;  // device count of `list`
  int n_list_max;         // host upper bound
  const CandSet* old;
};

static rpd_status reserve_pools(rpd_ctx* c, int64_t add_c, int64_t add_p, int64_t add_i,
                                int64_t add_r);

// Alg. 1 + compaction of tets (tet_ids, or all) into the candidate set cs.  append: cs is
// the batch of a partial update whose candidates go to the tail of the state pool (which
// is first made large enough for them and for the batch's pieces).
static rpd_status run_filter(rpd_ctx* c, const int32_t* tet_ids, int64_t n_tets, int lo,
                             int hi, CandSet& cs, bool timed, const Restrict* rs = nullptr,
                             bool append = false) {
  Readback* rb = (Readback*)c->pinned;
  size_t nt = n_tets > 0 ? n_tets : 1;
  CK(c->k_tet.ensure(sizeof(int32_t) * nt), "alloc");
  CK(c->k_words.ensure(sizeof(int32_t) * nt), "alloc");
  CK(cs.off.ensure(sizeof(int32_t) * (n_tets + 1)), "alloc");
  CK(c->w_off.ensure(sizeof(int32_t) * (n_tets + 1)), "alloc");
  for (int attempt = 0; attempt < 3; ++attempt) {
    const int cap = c->slab_cap;
    CK(c->slab.ensure(sizeof(int32_t) * (size_t)cap * nt), "alloc slab");
    CK(c->slab_m.ensure(sizeof(uint2) * (size_t)cap * nt), "alloc slab");
    // ST_MAXK, ST_TESTED, ST_REL_TESTS
    CK(cudaMemsetAsync(c->stats.as<unsigned long long>() + ST_MAXK, 0,
                       sizeof(unsigned long long) * 3, c->stream), "memset");
    if (timed && c->profile) cudaEventRecord(c->ev[0], c->stream);
    if (rs) {
      CK(launch_filter(c, tet_ids, n_tets, cap, 0, rs->n_list_max, c->k_tet.as<int32_t>(),
                       c->slab.as<int32_t>(), c->k_words.as<int32_t>(), rs->list,
                       rs->n_list_dev), "filter");
      CK(launch_keep_old(c, tet_ids, n_tets, *rs->old, cap, c->k_tet.as<int32_t>(),
                         c->slab.as<int32_t>(), c->k_words.as<int32_t>()), "keep old");
      tmark(c, "refilter+keep");
      // the all-pairs kernel counted its own max; the BVH path recomputes it
      CK(cudaMemsetAsync(c->stats.as<unsigned long long>() + ST_MAXK, 0,
                         sizeof(unsigned long long), c->stream), "memset");
      CK(launch_max_ktet(c, n_tets, c->k_tet.as<int32_t>()), "max k");
    } else {
      CK(launch_filter(c, tet_ids, n_tets, cap, lo, hi, c->k_tet.as<int32_t>(),
                       c->slab.as<int32_t>(), c->k_words.as<int32_t>()), "filter");
    }
    if (timed && c->profile) cudaEventRecord(c->ev[1], c->stream);
    {
      const int32_t* in[2] = {c->k_tet.as<int32_t>(), c->k_words.as<int32_t>()};
      int32_t* out[2] = {cs.off.as<int32_t>(), c->w_off.as<int32_t>()};
      CK(launch_scan_i32_multi(c, in, out, 2, n_tets), "scan");
    }
    const bool bvh = c->filter_mode == RPD_FILTER_PRUNED &&
                     (rs ? rs->n_list_max > 0 : hi > lo) && n_tets > 0;
    const int32_t* nq = bvh ? c->bvh_items.as<int32_t>() : nullptr;  // queue counts
    CK(readback(c, RbSpec{{cs.off.as<int32_t>() + n_tets, c->w_off.as<int32_t>() + n_tets, nq,
                           nq ? nq + 1 : nullptr},
                          c->stats.as<unsigned long long>(), c->errw.as<int>()}),
       "readback");
    CK(cudaStreamSynchronize(c->stream), "filter");
    rpd_status s = check_err(c, rb);
    if (s) return s;
    bool retry = false;
    const int32_t need = rb->i32[2] > rb->i32[3] ? rb->i32[2] : rb->i32[3];
    if (need > c->bvh_cap_items) {  // work queue overflow: grow and redo
      c->bvh_min_items = (int64_t)need + 1024;
      retry = true;
    }
    const int maxk = (int)rb->u64[ST_MAXK];
    if (maxk > cap) {
      int ncap = 32;
      while (ncap < maxk) ncap *= 2;
      c->slab_cap = ncap;
      retry = true;
    }
    if (!retry) break;
    if (attempt == 2) return fail(c, RPD_EOVERFLOW, "filter capacity");
    continue;
  }
  const int64_t nc = rb->i32[0];
  cs.n = nc;
  cs.n_tets = n_tets;
  cs.n_words = rb->i32[1];
  cs.idx_ext = nullptr;
  if (append) {
    // the batch's candidates, and (upper bounds) its pieces, incidences and radical facets
    const int64_t nw32 = 32 * cs.n_words;
    rpd_status s = reserve_pools(c, nc, nc, nw32, c->euler ? nw32 : 0);
    if (s) return s;
    CandSet& pool = c->cand[c->cur];
    cs.idx_ext = pool.idx.as<int32_t>() + pool.fill;
  } else {
    // the state pool: room for the appends of later partial updates
    CK(cs.idx.ensure_slack(sizeof(int32_t) * (nc > 0 ? nc : 1), 2), "alloc");
  }
  CK(cs.pair_tet.ensure(sizeof(int32_t) * (nc > 0 ? nc : 1)), "alloc");
  CK(cs.moff.ensure(sizeof(int32_t) * (nc + 1)), "alloc");
  CK(cs.cut.ensure(sizeof(unsigned) * (cs.n_words > 0 ? cs.n_words : 1)), "alloc");
  CK(launch_compact_cands(c, n_tets, c->slab_cap, c->k_tet.as<int32_t>(), c->slab.as<int32_t>(),
                          cs.off.as<int32_t>(), cs.idxp(), cs.pair_tet.as<int32_t>(),
                          c->w_off.as<int32_t>(), cs.moff.as<int32_t>(), nc,
                          cs.cut.as<unsigned>()), "compact");
  c->last.max_k_tet = (int32_t)rb->u64[ST_MAXK];
  c->last.rel_tests += (int64_t)rb->u64[ST_REL_TESTS];
  c->last.pairs_tested += c->filter_mode == RPD_FILTER_PRUNED
                              ? (int64_t)rb->u64[ST_TESTED]
                              : n_tets * (int64_t)(hi - lo);
  if (timed && c->profile) {
    float ms = 0.f;
    cudaEventElapsedTime(&ms, c->ev[0], c->ev[1]);
    c->last.filter_ms += ms;
  }
  return RPD_OK;
}

static void absorb_clip_stats(rpd_ctx* c, const Readback* rb, int n_wide) {
  c->last.exact_fallbacks += (int64_t)rb->u64[ST_EXACT];
  c->last.zero_hits += (int64_t)rb->u64[ST_ZERO];
  c->last.max_vertices = max(c->last.max_vertices, (int32_t)rb->u64[ST_MAXV]);
  c->last.max_planes = max(c->last.max_planes, (int32_t)rb->u64[ST_MAXP]);
  c->last.n_wide += n_wide;
  c->last.clip_plane_evals += (int64_t)rb->u64[ST_CLIP_PLANES];
  c->last.clip_vertex_tests += (int64_t)rb->u64[ST_CLIP_TESTS];
  c->last.clip_constructions += (int64_t)rb->u64[ST_CLIP_CONSTR];
  c->last.clip_fan_triangles += (int64_t)rb->u64[ST_CLIP_FAN];
  if (getenv("RPD_DEBUG_STATS")) clip_phase_dump();
  if (getenv("RPD_DEBUG_STATS"))
    fprintf(stderr, "[rpd clip] exact sign %llu exact out-vertex %llu plane-fallback %llu\n",
            rb->u64[12], rb->u64[13], rb->u64[14]);
}

// clip every pair of cs (tets tet_ids or all) -> piece set.
// deferred: no host round trip; the piece set is sized by upper bounds (one piece per pair,
// 32 incidences per mask word) and ps.n_pieces / ps.n_inc hold those bounds until the caller
// reads the exact totals (p_scan[n], i_scan[n]), the overflow counter and the clip stats.
// deferred (partial updates): ps is the batch -- only its per-tet CSR offsets (ps.off) are
// its own, the pieces go to the tail of the state pool (reserved by run_filter's append).
static rpd_status run_clip(rpd_ctx* c, const CandSet& cs, const int32_t* tet_ids,
                           PieceSet& ps, bool deferred = false) {
  const int64_t n = cs.n, nt = cs.n_tets;
  size_t nn = n > 0 ? n : 1;
  CK(c->p_flag.ensure(nn), "alloc");
  CK(c->p_f01.ensure(sizeof(int32_t) * nn), "alloc");
  CK(c->p_fm.ensure(nn), "alloc");
  CK(c->p_vol.ensure(sizeof(double) * nn), "alloc");
  CK(c->p_m1.ensure(sizeof(double) * 3 * nn), "alloc");
  CK(c->p_ninc.ensure(sizeof(int32_t) * nn), "alloc");
  CK(c->p_over.ensure(sizeof(int32_t) * (n + 1)), "alloc");
  CK(c->p_over2.ensure(sizeof(int32_t) * (n + 1)), "alloc");
  CK(c->p_over3.ensure(sizeof(int32_t) * (n + 1)), "alloc");
  CK(c->p_mask.ensure(sizeof(unsigned) * (cs.n_words > 0 ? cs.n_words : 1)), "alloc");
  CK(c->p_scan.ensure(sizeof(int32_t) * (n + 1)), "alloc");
  CK(c->i_scan.ensure(sizeof(int32_t) * (n + 1)), "alloc");
  if (c->euler) {
    if (c->eu_T != cs.n_tets && tet_ids == nullptr)
      return fail(c, RPD_EINVAL, "Euler payloads were set for a different tet count");
    const size_t nw = cs.n_words > 0 ? cs.n_words : 1;
    CK(c->p_eu.ensure(sizeof(long long) * nn), "alloc");
    CK(c->p_nrpf.ensure(sizeof(int32_t) * nn), "alloc");
    CK(c->r_scan.ensure(sizeof(int32_t) * (n + 1)), "alloc");
    CK(c->p_rmask.ensure(sizeof(unsigned) * nw), "alloc");
    CK(c->p_rval.ensure(sizeof(long long) * 32 * nw), "alloc");
    CK(c->p_sfm.ensure(nn), "alloc");
    CK(c->p_rfm.ensure(32 * nw), "alloc");
    CK(c->p_radj.ensure(sizeof(unsigned long long) * 32 * nw), "alloc");
    CK(c->p_rep.ensure(sizeof(unsigned long long) * 32 * nw), "alloc");
  }
  const int32_t* moff = cs.moff.as<int32_t>();
  // (no memset of the incidence masks: the clip kernels write every word of non-empty pairs)
  CK(cudaMemsetAsync(c->p_over.p, 0, sizeof(int32_t), c->stream), "memset");
  CK(cudaMemsetAsync(c->p_over2.p, 0, sizeof(int32_t), c->stream), "memset");
  CK(cudaMemsetAsync(c->p_over3.p, 0, sizeof(int32_t), c->stream), "memset");
  CK(cudaMemsetAsync(c->stats.as<unsigned long long>() + ST_EXACT, 0,
                     sizeof(unsigned long long) * 5, c->stream), "memset");
  CK(cudaMemsetAsync(c->stats.as<unsigned long long>() + ST_CLIP_PLANES, 0,
                     sizeof(unsigned long long) * 8, c->stream), "memset");
  if (c->profile) cudaEventRecord(c->ev[2], c->stream);
  CK(launch_clip(c, n, cs.pair_tet.as<int32_t>(), tet_ids, cs.idxp(), moff,
                 cs.cut.as<unsigned>(), c->clip_wide),
     "clip");
  tmark(c, "clip-fast");
  if (n > 0)
    CK(launch_clip_overflow(c, cs.pair_tet.as<int32_t>(), tet_ids, cs.idxp(), moff,
                            cs.cut.as<unsigned>()),
       "clip (wide)");
  tmark(c, "clip-wide");
  if (c->profile) cudaEventRecord(c->ev[3], c->stream);
  CK(launch_piece_scans(c, n, moff), "scan");
  tmark(c, "piece-scans");
  Readback* rb = (Readback*)c->pinned;
  int64_t np = n, ni = 32 * (int64_t)cs.n_words, nr = c->euler ? ni : 0;
  if (!deferred) {
    CK(readback(c, RbSpec{{c->p_scan.as<int32_t>() + n, c->i_scan.as<int32_t>() + n,
                           c->p_over.as<int32_t>(), c->p_over2.as<int32_t>(),
                           c->euler ? c->r_scan.as<int32_t>() + n : nullptr},
                          c->stats.as<unsigned long long>(), nullptr}),
       "readback");
    CK(cudaStreamSynchronize(c->stream), "clip");
    if (rb->u64[ST_OVERFLOW])
      return fail(c, RPD_EOVERFLOW, "a piece exceeded the wide clip capacity (128 vertices/planes)");
    if (rb->u64[ST_EU_OVER])
      return fail(c, RPD_EOVERFLOW, "topology mode: a piece has more than 64 radical facets");
    np = rb->i32[0];
    ni = rb->i32[1];
    nr = rb->i32[4];
    absorb_clip_stats(c, rb, rb->i32[2]);
    if (getenv("RPD_DEBUG_STATS"))
      fprintf(stderr, "[rpd clip] pairs %lld overflow 16->32 %d 32->128 %d maxv %d maxp %d\n",
              (long long)n, rb->i32[2], rb->i32[3], c->last.max_vertices, c->last.max_planes);
  }
  CK(ps.off.ensure(sizeof(int32_t) * (nt + 1)), "alloc");
  // the destination: the state's own arrays (full clip; slack for later appends) or the tail
  // of the state pool (a partial update's batch)
  PieceSet& dst = deferred ? c->pcs[c->cur] : ps;
  const int64_t P0 = deferred ? dst.fill_p : 0, I0 = deferred ? dst.fill_i : 0,
                R0 = deferred ? dst.fill_r : 0;
  if (!deferred) {
    const size_t npp = np > 0 ? np : 1;
    CK(ps.sphere.ensure_slack(sizeof(int32_t) * npp, 2), "alloc");
    CK(ps.vol.ensure_slack(sizeof(double) * npp, 2), "alloc");
    CK(ps.m1.ensure_slack(sizeof(double) * 3 * npp, 2), "alloc");
    CK(ps.fm.ensure_slack(npp, 2), "alloc");
    CK(ps.inc_off.ensure_slack(sizeof(int32_t) * (np + 1), 2), "alloc");
    CK(ps.inc.ensure_slack(sizeof(int32_t) * (ni > 0 ? ni : 1), 2), "alloc");
    if (c->euler) {
      const size_t nrr = nr > 0 ? nr : 1;
      CK(ps.eu.ensure_slack(sizeof(long long) * npp, 2), "alloc");
      CK(ps.rpf_off.ensure_slack(sizeof(int32_t) * (np + 1), 2), "alloc");
      CK(ps.rpf_j.ensure_slack(sizeof(int32_t) * nrr, 2), "alloc");
      CK(ps.rpf_e.ensure_slack(sizeof(long long) * nrr, 2), "alloc");
      CK(ps.sfm.ensure_slack(npp, 2), "alloc");
      CK(ps.rfm.ensure_slack(nrr, 2), "alloc");
      CK(ps.radj.ensure_slack(sizeof(unsigned long long) * nrr, 2), "alloc");
      CK(ps.rep.ensure_slack(sizeof(unsigned long long) * nrr, 2), "alloc");
    }
  }
  PieceDst d{ps.off.as<int32_t>(),
             dst.sphere.as<int32_t>() + P0,
             dst.vol.as<double>() + P0,
             dst.m1.as<double>() + 3 * P0,
             dst.fm.as<uint8_t>() + P0,
             dst.inc_off.as<int32_t>() + P0,
             dst.inc.as<int32_t>() + I0,
             c->euler ? dst.eu.as<long long>() + P0 : nullptr,
             c->euler ? dst.rpf_off.as<int32_t>() + P0 : nullptr,
             c->euler ? dst.rpf_j.as<int32_t>() + R0 : nullptr,
             c->euler ? dst.rpf_e.as<long long>() + R0 : nullptr,
             c->euler ? dst.sfm.as<uint8_t>() + P0 : nullptr,
             c->euler ? dst.rfm.as<uint8_t>() + R0 : nullptr,
             c->euler ? dst.radj.as<unsigned long long>() + R0 : nullptr,
             c->euler ? dst.rep.as<unsigned long long>() + R0 : nullptr,
             (int32_t)I0,
             (int32_t)R0};
  CK(launch_compact_pieces(c, nt, n, cs.off.as<int32_t>(), cs.idxp(), moff, d),
     "compact pieces");
  ps.n_tets = nt;
  ps.n_pieces = np;
  ps.n_inc = ni;
  ps.n_rpf = nr;
  c->last.pairs_clipped += n;
  if (deferred) return RPD_OK;
  if (c->euler) CK(launch_euler_sums(c, ps), "euler sums");
  if (c->profile) {
    float ms = 0.f;
    cudaEventElapsedTime(&ms, c->ev[2], c->ev[3]);
    c->last.clip_ms += ms;
  }
  return RPD_OK;
}

// Compaction (garbage collection) of the state pools: every tet's live segments gathered by
// its rows into the other buffer set as plain CSRs (pair_tet / moff of the candidates rebuilt),
// with room for `extra` appended entries of each kind; then that set is the state.
static rpd_status compact_state(rpd_ctx* c, int64_t extra) {
  if (c->compact) return RPD_OK;
  const int64_t T = c->st.T;
  CandSet& co = c->cand[c->cur];
  PieceSet& po = c->pcs[c->cur];
  CandSet& cn = c->cand[c->cur ^ 1];
  PieceSet& pn = c->pcs[c->cur ^ 1];
  CK(c->m_cnt.ensure(sizeof(int32_t) * 4 * (T > 0 ? T : 1) + 64), "alloc");
  CK(c->m_off.ensure(sizeof(int32_t) * 3 * (T + 1)), "alloc");
  CK(cn.off.ensure(sizeof(int32_t) * (T + 1)), "alloc");
  CK(pn.off.ensure(sizeof(int32_t) * (T + 1)), "alloc");
  CK(launch_compact_state(c, T, co, po, cn, pn, 0), "compact counts");
  Readback* rb = (Readback*)c->pinned;
  const int32_t* m_off = c->m_off.as<int32_t>();
  CK(readback(c, RbSpec{{cn.off.as<int32_t>() + T, pn.off.as<int32_t>() + T, m_off + T,
                         c->euler ? m_off + 2 * (T + 1) + T : nullptr},
                        nullptr, nullptr}),
     "readback");
  CK(cudaStreamSynchronize(c->stream), "compact");
  const int64_t nc = rb->i32[0], np = rb->i32[1], ni = rb->i32[2], nr = rb->i32[3];
  auto room = [&](int64_t n) { return (size_t)((n + extra) + (n + extra) / 2 + 1); };
  CK(cn.idx.ensure(sizeof(int32_t) * room(nc)), "alloc");
  CK(cn.pair_tet.ensure(sizeof(int32_t) * (nc > 0 ? nc : 1)), "alloc");
  CK(cn.moff.ensure(sizeof(int32_t) * (nc + 1)), "alloc");
  CK(pn.sphere.ensure(sizeof(int32_t) * room(np)), "alloc");
  CK(pn.vol.ensure(sizeof(double) * room(np)), "alloc");
  CK(pn.m1.ensure(sizeof(double) * 3 * room(np)), "alloc");
  CK(pn.fm.ensure(room(np)), "alloc");
  CK(pn.inc_off.ensure(sizeof(int32_t) * (room(np) + 1)), "alloc");
  CK(pn.inc.ensure(sizeof(int32_t) * room(ni)), "alloc");
  if (c->euler) {
    CK(pn.eu.ensure(sizeof(long long) * room(np)), "alloc");
    CK(pn.rpf_off.ensure(sizeof(int32_t) * (room(np) + 1)), "alloc");
    CK(pn.rpf_j.ensure(sizeof(int32_t) * room(nr)), "alloc");
    CK(pn.rpf_e.ensure(sizeof(long long) * room(nr)), "alloc");
    CK(pn.sfm.ensure(room(np)), "alloc");
    CK(pn.rfm.ensure(room(nr)), "alloc");
    CK(pn.radj.ensure(sizeof(unsigned long long) * room(nr)), "alloc");
    CK(pn.rep.ensure(sizeof(unsigned long long) * room(nr)), "alloc");
  }
  CK(c->m_cnt.ensure(sizeof(int32_t) * 4 * (T > 0 ? T : 1) + sizeof(int32_t) * (nc + 1) + 64),
     "alloc");
  cn.n = nc;
  CK(launch_compact_state(c, T, co, po, cn, pn, 1), "compact copy");
  CK(launch_rows_from_off(c, T, &cn, &pn, &cn), "rows");
  CK(readback(c, RbSpec{{cn.moff.as<int32_t>() + nc}, nullptr, nullptr}), "readback");
  CK(cudaStreamSynchronize(c->stream), "compact");
  cn.n_tets = T;
  cn.n_words = rb->i32[0];
  // no filter values for the re-laid-out pairs: every plane is classified by the clip
  CK(cn.cut.ensure(sizeof(unsigned) * (cn.n_words > 0 ? cn.n_words : 1)), "alloc");
  CK(cudaMemsetAsync(cn.cut.p, 0xff, sizeof(unsigned) * (cn.n_words > 0 ? cn.n_words : 1),
                     c->stream), "memset");
  cn.fill = nc;
  cn.idx_ext = nullptr;
  pn.n_tets = T;
  pn.n_pieces = np;
  pn.n_inc = ni;
  pn.n_rpf = c->euler ? nr : 0;
  pn.fill_p = np;
  pn.fill_i = ni;
  pn.fill_r = pn.n_rpf;
  c->cur ^= 1;
  c->compact = true;
  ++c->n_compactions;
  return RPD_OK;
}

// make room at the pools' tails for a batch of add_* entries (compacting when they are full)
static rpd_status reserve_pools(rpd_ctx* c, int64_t add_c, int64_t add_p, int64_t add_i,
                                int64_t add_r) {
  const CandSet& pc = c->cand[c->cur];
  const PieceSet& pp = c->pcs[c->cur];
  const bool fits =
      (pc.fill + add_c) * sizeof(int32_t) <= pc.idx.cap &&
      (pp.fill_p + add_p) * sizeof(double) * 3 <= pp.m1.cap &&
      (pp.fill_p + add_p + 1) * sizeof(int32_t) <= pp.inc_off.cap &&
      (pp.fill_p + add_p) * sizeof(int32_t) <= pp.sphere.cap &&
      (pp.fill_p + add_p) * sizeof(double) <= pp.vol.cap && pp.fill_p + add_p <= (int64_t)pp.fm.cap &&
      (pp.fill_i + add_i) * sizeof(int32_t) <= pp.inc.cap &&
      (!c->euler ||
       ((pp.fill_p + add_p) * sizeof(long long) <= pp.eu.cap &&
        (pp.fill_p + add_p + 1) * sizeof(int32_t) <= pp.rpf_off.cap &&
        pp.fill_p + add_p <= (int64_t)pp.sfm.cap &&
        (pp.fill_r + add_r) * sizeof(int32_t) <= pp.rpf_j.cap &&
        (pp.fill_r + add_r) * sizeof(long long) <= pp.rpf_e.cap &&
        pp.fill_r + add_r <= (int64_t)pp.rfm.cap &&
        (pp.fill_r + add_r) * sizeof(unsigned long long) <= pp.radj.cap &&
        (pp.fill_r + add_r) * sizeof(unsigned long long) <= pp.rep.cap));
  if (fits) return RPD_OK;
  c->compact = false;  // (force: a compact pool without room is re-laid out with room)
  const int64_t extra = std::max(std::max(add_c, add_p), std::max(add_i, add_r));
  return compact_state(c, extra);
}

static void reset_last(rpd_ctx* c) {
  c->last = rpd_stats{};
  c->last.T = c->st.T;
  c->last.N = c->st.N;
}

static rpd_status fill_pieces(rpd_ctx* c, rpd_pieces* out) {
  const PieceSet& ps = c->pcs[c->cur];
  out->piece_off = c->compact ? ps.off.as<int32_t>() : nullptr;
  out->piece_rows = ps.rows.as<int32_t>();
  out->n_slots = ps.fill_p;
  out->piece_sphere = ps.sphere.as<int32_t>();
  out->piece_vol = ps.vol.as<double>();
  out->piece_m1 = ps.m1.as<double>();
  out->piece_facemask = ps.fm.as<uint8_t>();
  out->inc_off = ps.inc_off.as<int32_t>();
  out->inc_sphere = ps.inc.as<int32_t>();
  out->n_pieces = ps.n_pieces;
  out->n_inc = ps.n_inc;
  return RPD_OK;
}

// ------------------------------------------------------------------ public calls

rpd_status rpd_relations(rpd_ctx* c, const double* verts, int64_t V, const int32_t* tets,
                         int64_t T, const double* spheres, int64_t N, const int32_t* nbr_off,
                         const int32_t* nbr_idx, int64_t E, const int32_t** cand_off,
                         const int32_t** cand_idx, int64_t* n_cand) {
  if (!c) return RPD_EINVAL;
  if (V < 0 || T < 0 || N < 0 || T > 0x7fffffff || N > 0x7fffffff || (T > 0 && !tets) ||
      (V > 0 && !verts) || (N > 0 && (!spheres || !nbr_off)) || !cand_off || !cand_idx ||
      !n_cand)
    return fail(c, RPD_EINVAL, "rpd_relations: bad argument");
  CK(cudaSetDevice(c->device), "cudaSetDevice");
  c->have_rel = false;
  c->have_pieces = false;
  c->eu_valid = false;
  c->rpe_n = -1;
  const double* d_verts = nullptr;
  const int32_t* d_tets = nullptr;
  CK(resolve(c, verts, 3 * V, c->h_verts, &d_verts), "stage verts");
  CK(resolve(c, tets, 4 * T, c->h_tets, &d_tets), "stage tets");
  CK(cudaMemsetAsync(c->errw.p, 0, sizeof(int) * 4, c->stream), "memset");
  CK(cudaMemsetAsync(c->stats.p, 0, sizeof(unsigned long long) * ST_N, c->stream), "memset");
  CK(launch_stage_mesh(c, d_verts, V, d_tets, T), "stage mesh");
  c->epoch = 0;
  rpd_status s = stage_spheres(c, spheres, N, nbr_off, nbr_idx, E, false, 0);
  if (s) return s;
  CK(c->cepoch.ensure(sizeof(int32_t) * (T > 0 ? T : 1)), "alloc");
  CK(cudaMemsetAsync(c->cepoch.p, 0, sizeof(int32_t) * (T > 0 ? T : 1), c->stream), "memset");
  reset_last(c);
  c->cur = 0;
  CandSet& cs = c->cand[0];
  s = run_filter(c, nullptr, T, 0, (int)N, cs, true);
  if (s) return s;
  CK(launch_rows_from_off(c, T, &cs, nullptr, &cs), "rows");
  cs.fill = cs.n;
  c->compact = true;
  c->have_rel = true;
  c->last.n_cand = cs.n;
  c->last.pairs_filtered = T * N;
  *cand_off = cs.off.as<int32_t>();
  *cand_idx = cs.idx.as<int32_t>();
  *n_cand = cs.n;
  return RPD_OK;
}

rpd_status rpd_clip(rpd_ctx* c, rpd_pieces* out) {
  if (!c || !out) return fail(c, RPD_EINVAL, "rpd_clip: bad argument");
  if (!c->have_rel) return fail(c, RPD_ESTATE, "rpd_clip before rpd_relations");
  CK(cudaSetDevice(c->device), "cudaSetDevice");
  // after partial updates the candidate pool is re-laid out as a plain CSR first
  rpd_status s = compact_state(c, 0);
  if (s) return s;
  CandSet& cs = c->cand[c->cur];
  c->last.clip_ms = 0.0;
  c->eu_valid = false;
  c->rpe_n = -1;
  PieceSet& ps = c->pcs[c->cur];
  s = run_clip(c, cs, nullptr, ps);
  if (s) return s;
  CK(launch_rows_from_off(c, c->st.T, nullptr, &ps, nullptr), "rows");
  ps.fill_p = ps.n_pieces;
  ps.fill_i = ps.n_inc;
  ps.fill_r = ps.n_rpf;
  c->have_pieces = true;
  c->eu_valid = c->euler != 0;
  c->last.n_pieces = c->pcs[c->cur].n_pieces;
  c->last.n_inc = c->pcs[c->cur].n_inc;
  return fill_pieces(c, out);
}

static rpd_status update_partial_impl(rpd_ctx* c, const double* spheres, int64_t N_new,
                                      const int32_t* nbr_off, const int32_t* nbr_idx, int64_t E,
                                      const int32_t* new_ids, int64_t M, rpd_pieces* out,
                                      const int32_t** dirty_tets, int64_t* n_dirty,
                                      bool* mutated);
static rpd_status partial_batch(rpd_ctx* c, int64_t nd, int64_t N_new, int64_t M,
                                rpd_pieces* out, const int32_t** dirty_tets, int64_t* n_dirty);
static bool graph_eligible(const rpd_ctx* c, int64_t M);
static rpd_status partial_graph(rpd_ctx* c, const double* spheres, int64_t N_new,
                                const int32_t* nbr_off, const int32_t* nbr_idx, int64_t E,
                                const int32_t* new_ids, int64_t M, rpd_pieces* out,
                                const int32_t** dirty_tets, int64_t* n_dirty);

rpd_status rpd_update_partial(rpd_ctx* c, const double* spheres, int64_t N_new,
                              const int32_t* nbr_off, const int32_t* nbr_idx, int64_t E,
                              const int32_t* new_ids, int64_t M, rpd_pieces* out,
                              const int32_t** dirty_tets, int64_t* n_dirty) {
  if (!c) return RPD_EINVAL;
  bool mutated = false;
  rpd_status s = update_partial_impl(c, spheres, N_new, nbr_off, nbr_idx, E, new_ids, M, out,
                                     dirty_tets, n_dirty, &mutated);
  if (s != RPD_OK && mutated) {
    // the staged rows / epochs already describe the new sphere set while the candidates and
    // pieces do not: the ctx state is inconsistent, so a full rpd_relations is required
    c->have_rel = c->have_pieces = c->eu_valid = false;
    c->err += " (ctx state reset: call rpd_relations + rpd_clip again)";
  }
  return s;
}

static rpd_status update_partial_impl(rpd_ctx* c, const double* spheres, int64_t N_new,
                                      const int32_t* nbr_off, const int32_t* nbr_idx, int64_t E,
                                      const int32_t* new_ids, int64_t M, rpd_pieces* out,
                                      const int32_t** dirty_tets, int64_t* n_dirty,
                                      bool* mutated) {
  if (!out || !dirty_tets || !n_dirty || M < 0 || (M > 0 && !new_ids))
    return fail(c, RPD_EINVAL, "rpd_update_partial: bad argument");
  if (!c->have_pieces) return fail(c, RPD_ESTATE, "rpd_update_partial before rpd_clip");
  if (c->euler && !c->eu_valid)
    return fail(c, RPD_ESTATE, "Euler mode: the current pieces were clipped without payloads");
  CK(cudaSetDevice(c->device), "cudaSetDevice");
  const int64_t N_old = c->st.N, T = c->st.T;
  if (N_new != N_old + M)
    return fail(c, RPD_EINVAL, "N_new must equal N_old + M (new spheres are appended)");
  if (!spheres || (N_new > 0 && !nbr_off))
    return fail(c, RPD_EINVAL, "rpd_update_partial: bad argument");
  reset_last(c);
  CK(c->d_list.ensure(sizeof(int32_t) * (T > 0 ? T : 1)), "alloc");
  if (M == 0) {  // identity
    c->n_dirty = 0;
    *dirty_tets = c->d_list.as<int32_t>();
    *n_dirty = 0;
    c->last.n_cand = c->cand[c->cur].n;
    c->last.n_pieces = c->pcs[c->cur].n_pieces;
    c->last.n_inc = c->pcs[c->cur].n_inc;
    return fill_pieces(c, out);
  }
  if (graph_eligible(c, M)) {
    *mutated = true;
    return partial_graph(c, spheres, N_new, nbr_off, nbr_idx, E, new_ids, M, out, dirty_tets,
                         n_dirty);
  }
  const int32_t* d_new = nullptr;
  tmark(c, "start");
  CK(resolve(c, new_ids, M, c->h_new, &d_new), "stage new ids");
  CK(cudaMemsetAsync(c->errw.p, 0, sizeof(int) * 4, c->stream), "memset");
  CK(cudaMemsetAsync(c->stats.p, 0, sizeof(unsigned long long) * ST_N, c->stream), "memset");
  CK(launch_check_new_ids(c, d_new, M, N_old), "check ids");
  *mutated = true;
  c->rpe_n = -1;
  ++c->epoch;
  rpd_status s = stage_spheres(c, spheres, N_new, nbr_off, nbr_idx, E, true, c->epoch);
  if (s) return s;
  tmark(c, "staged");
  c->last.N = N_new;

  // (1) dirty tets: Alg. 1 of every tet against the new spheres only
  CK(c->d_count.ensure(sizeof(int32_t) * (T > 0 ? T : 1)), "alloc");
  CK(c->d_flag.ensure(T > 0 ? T : 1), "alloc");
  CK(c->d_scan.ensure(sizeof(int32_t) * (T + 1)), "alloc");
  if (c->profile) cudaEventRecord(c->ev[0], c->stream);
  CK(launch_filter(c, nullptr, T, 0, (int)N_old, (int)N_new, c->d_count.as<int32_t>(), nullptr,
                   nullptr), "dirty filter");
  tmark(c, "dirty-filter");
  if (c->profile) cudaEventRecord(c->ev[1], c->stream);
  CK(c->min_epoch.ensure(sizeof(int)), "alloc");
  CK(launch_dirty_list(c, T), "dirty list");
  CK(c->c_flag.ensure(N_new > 0 ? N_new : 1), "alloc");
  CK(c->c_scan.ensure(sizeof(int32_t) * (N_new + 1)), "alloc");
  CK(c->c_list.ensure(sizeof(int32_t) * (N_new > 0 ? N_new : 1)), "alloc");
  CK(launch_changed_list(c, N_new), "changed rows");
  Readback* rb = (Readback*)c->pinned;
  {
    const int32_t* nq =
        c->filter_mode == RPD_FILTER_PRUNED && T > 0 ? c->bvh_items.as<int32_t>() : nullptr;
    CK(readback(c, RbSpec{{c->d_scan.as<int32_t>() + T, nullptr, nq, nq ? nq + 1 : nullptr},
                          c->stats.as<unsigned long long>(), c->errw.as<int>()}),
       "readback");
  }
  CK(cudaStreamSynchronize(c->stream), "dirty");
  tmark(c, "dirty-sync");
  const int32_t need = rb->i32[2] > rb->i32[3] ? rb->i32[2] : rb->i32[3];
  if (need > c->bvh_cap_items) {
    // work queue overflow (never seen): grow it and redo the dirty detection
    c->bvh_min_items = (int64_t)need + 1024;
    CK(launch_filter(c, nullptr, T, 0, (int)N_old, (int)N_new, c->d_count.as<int32_t>(),
                     nullptr, nullptr), "dirty filter");
    CK(launch_dirty_list(c, T), "dirty list");
    CK(readback(c, RbSpec{{c->d_scan.as<int32_t>() + T}, nullptr, nullptr}), "readback");
    CK(cudaStreamSynchronize(c->stream), "dirty");
  }
  if (rb->err[0] != 0) {
    if (rb->err[1] == 100) return fail(c, RPD_EINVAL, "new_ids is not the appended id range");
    return check_err(c, rb);
  }
  const int64_t nd = rb->i32[0];
  c->last.rel_tests += (int64_t)rb->u64[ST_REL_TESTS];
  c->last.pairs_tested += c->filter_mode == RPD_FILTER_PRUNED ? (int64_t)rb->u64[ST_TESTED]
                                                              : T * M;
  if (c->profile) {
    float ms = 0.f;
    cudaEventElapsedTime(&ms, c->ev[0], c->ev[1]);
    c->last.filter_ms += ms;
  }
  return partial_batch(c, nd, N_new, M, out, dirty_tets, n_dirty);
}

// steps (2)-(4) of a partial update for the nd dirty tets listed in d_list (eager launches)
static rpd_status partial_batch(rpd_ctx* c, int64_t nd, int64_t N_new, int64_t M,
                                rpd_pieces* out, const int32_t** dirty_tets, int64_t* n_dirty) {
  const int64_t T = c->st.T;
  Readback* rb = (Readback*)c->pinned;
  rpd_status s;
  const int32_t* dl = c->d_list.as<int32_t>();

  // (2) re-candidate the dirty tets against all spheres -- their new candidate lists go to the
  // tail of the state pool --, (3) clip them, their pieces also appended to the pool
  CandSet& cd = c->cand_d;
  PieceSet& pd = c->pcs_d;
  if (c->filter_mode == RPD_FILTER_PRUNED) {
    Restrict rs{c->c_list.as<int32_t>(), c->c_scan.as<int>() + N_new, (int)N_new,
                &c->cand[c->cur]};
    s = run_filter(c, dl, nd, 0, (int)N_new, cd, true, &rs, /*append=*/true);
  } else {
    s = run_filter(c, dl, nd, 0, (int)N_new, cd, true, nullptr, /*append=*/true);
  }
  if (s) return s;
  tmark(c, "filter-sync");
  // (the pools may have been compacted by the reservation: take them after it)
  CandSet& pool_c = c->cand[c->cur];
  PieceSet& pool_p = c->pcs[c->cur];
  const int64_t cbase = pool_c.fill, pbase = pool_p.fill_p;
  s = run_clip(c, cd, dl, pd, /*deferred=*/true);
  if (s) return s;
  tmark(c, "clip-launched");

  // (4) re-point the dirty tets' rows at the batch (clean tets are not touched); the batch
  // totals, the removed segments' sizes, the overflow counter and the stats come back in one
  // readback at the end (the only host round trip after the re-filter)
  CK(c->m_cnt.ensure(sizeof(unsigned long long) * 4), "alloc");
  unsigned long long* rm = c->m_cnt.as<unsigned long long>();
  CK(launch_rows_update(c, dl, nd, pool_c, pool_p, cd, pd, cbase, pbase, rm), "rows");
  CK(readback(c, RbSpec{{c->p_over.as<int32_t>(), c->p_scan.as<int32_t>() + cd.n,
                         c->i_scan.as<int32_t>() + cd.n,
                         c->euler ? c->r_scan.as<int32_t>() + cd.n : nullptr},
                        c->stats.as<unsigned long long>(), nullptr, rm}),
     "readback");
  CK(cudaStreamSynchronize(c->stream), "partial update");
  tmark(c, "final-sync");
  tdump(c);
  if (rb->u64[ST_OVERFLOW])
    return fail(c, RPD_EOVERFLOW, "a piece exceeded the wide clip capacity (128 vertices/planes)");
  if (rb->u64[ST_EU_OVER])
    return fail(c, RPD_EOVERFLOW, "topology mode: a piece has more than 64 radical facets");
  absorb_clip_stats(c, rb, rb->i32[0]);
  if (c->profile) {
    float ms = 0.f;
    cudaEventElapsedTime(&ms, c->ev[2], c->ev[3]);
    c->last.clip_ms += ms;
  }
  const unsigned long long* removed = rb->u4;
  pd.n_pieces = rb->i32[1];
  pd.n_inc = rb->i32[2];
  pd.n_rpf = c->euler ? rb->i32[3] : 0;
  pd.n_tets = nd;
  pool_c.fill += cd.n;
  pool_p.fill_p += pd.n_pieces;
  pool_p.fill_i += pd.n_inc;
  pool_p.fill_r += pd.n_rpf;
  pool_c.n += cd.n - (int64_t)removed[0];
  pool_p.n_pieces += pd.n_pieces - (int64_t)removed[1];
  pool_p.n_inc += pd.n_inc - (int64_t)removed[2];
  pool_p.n_rpf += pd.n_rpf - (int64_t)removed[3];
  c->compact = false;
  c->last.n_cand_dirty = cd.n;
  c->last.n_pieces_dirty = pd.n_pieces;
  c->last.n_inc_dirty = pd.n_inc;
  if (c->euler) {  // the Euler / topology consumers read plain CSRs
    s = compact_state(c, 0);
    if (s) return s;
    CK(launch_euler_sums(c, c->pcs[c->cur]), "euler sums");
  }
  c->eu_valid = c->euler != 0;
  c->n_dirty = nd;
  c->last.n_dirty = nd;
  c->last.n_cand = c->cand[c->cur].n;
  c->last.n_pieces = c->pcs[c->cur].n_pieces;
  c->last.n_inc = c->pcs[c->cur].n_inc;
  c->last.pairs_filtered = T * M + nd * N_new;
  *dirty_tets = dl;
  *n_dirty = nd;
  return fill_pieces(c, out);
}

// ------------------------------------------------------------------ device-driven updates
//
// The latency path for few insertions ("launch latency matters, use
// CUDA Graphs"; "few (even single) spheres" per iteration).  The eager update
// reads three sizes back to the host between its ~35 launches (dirty count, candidate count,
// totals).  Here every size lives in a device record (PDyn) that the kernels read, the grids
// are sized by bounds, and the whole update -- staging, dirty detection, re-filter, clip,
// piece output, row update -- is ONE CUDA graph, captured once per buffer layout and replayed
// with one host round trip.  Checks the eager path makes on the host (slab capacity, work
// queues, pool room) are made on the device; a failed check idles the rest of the graph and
// the host redoes the batch eagerly (partial_batch), so the results are the eager path's.

#ifndef RPD_GRAPH_NC_MIN
#define RPD_GRAPH_NC_MIN (1 << 15)  // smallest batch-candidate bound of the graph's grids
#endif
#ifndef RPD_GRAPH_QUEUE_MAX
#define RPD_GRAPH_QUEUE_MAX (1 << 25)  // dirty-detection queue (worst case sized) limit, items
#endif

static inline int64_t pow2_at_least(int64_t x) {
  int64_t p = 1;
  while (p < x) p <<= 1;
  return p;
}

// new-sphere bound of a graph: M rounded up to a power of two (at least 64)
static inline int64_t graph_mb(int64_t M) { return pow2_at_least(M < 64 ? 64 : M); }

static bool graph_eligible(const rpd_ctx* c, int64_t M) {
  // (the dirty detection's work queue is sized for its worst case: every (new sphere, leaf))
  const int64_t n_leaf = (c->st.T + 31) / 32;
  return c->graph && M > 0 && graph_mb(M) * (n_leaf + 1) <= RPD_GRAPH_QUEUE_MAX &&
         c->filter_mode == RPD_FILTER_PRUNED && !c->euler && !c->clip_wide && !c->clip_tiers &&
         c->st.T > 0 && c->st.N > 0 && c->tr_on != 1;
}

static inline int64_t tiles_of(int64_t n) { return n > 0 ? (n + 4095) / 4096 : 1; }

// the launch sequence (issued once per buffer layout into a capturing stream)
static cudaError_t issue_dd(rpd_ctx* c, int64_t Nb, int64_t nc_max) {
  const int64_t T = c->st.T;
  PDyn* pd = c->pdd;
  cudaError_t e;
  unsigned long long* st = c->stats.as<unsigned long long>();
  // (k_pd_init also zeroes the error word, the stats and every small counter of the graph)
  if ((e = launch_pd_init(c))) return e;
  // (the new ids are checked by k_stage_spheres in a graph)
  if ((e = stage_launch(c, nullptr, nullptr, nullptr, true, 0))) return e;
  // (RPD_OPT_PROFILE: timer stamps around the filter and clip kernels, as the eager path's
  // events)
  auto mark = [&](int k) { return c->profile ? launch_pd_stamp(c, k) : cudaSuccess; };
  // (1) dirty tets: Alg. 1 of every tet against the new spheres only
  if ((e = mark(0))) return e;
  if ((e = launch_filter(c, nullptr, T, 0, 0, (int)c->g_mb, c->d_count.as<int32_t>(),
                         nullptr, nullptr)))
    return e;
  if ((e = mark(1))) return e;
  if ((e = launch_dirty_list(c, T))) return e;
  if ((e = launch_changed_list(c, Nb))) return e;
  // (2) re-filter of the dirty tets over the changed rows; kept old candidates
  CandSet& cd = c->cand_d;
  CandSet& pool_c = c->cand[c->cur];
  PieceSet& pool_p = c->pcs[c->cur];
  const int32_t* dl = c->d_list.as<int32_t>();
  const int cap = c->slab_cap;
  int32_t* k_tet = c->k_tet.as<int32_t>();
  int32_t* k_words = c->k_words.as<int32_t>();
  int32_t* slab = c->slab.as<int32_t>();
  if ((e = mark(2))) return e;
  if ((e = launch_filter(c, dl, T, cap, 0, (int)Nb, k_tet, slab, k_words, c->c_list.as<int32_t>(),
                         &pd->n_chg)))
    return e;
  if ((e = launch_keep_old(c, dl, T, pool_c, cap, k_tet, slab, k_words))) return e;
  if ((e = mark(3))) return e;
  if ((e = launch_max_ktet(c, T, k_tet))) return e;  // (atomicMax: no reset needed)
  {
    const int32_t* in[2] = {k_tet, k_words};
    int32_t* out[2] = {cd.off.as<int32_t>(), c->w_off.as<int32_t>()};
    if ((e = launch_scan_i32_multi(c, in, out, 2, T, &pd->nb))) return e;
  }
  if ((e = launch_pd_check(c, cd.off.as<int32_t>(), c->w_off.as<int32_t>()))) return e;
  int32_t* pool_idx = pool_c.idx.as<int32_t>();  // (the kernels add the fill level)
  if ((e = launch_compact_cands(c, T, cap, k_tet, slab, cd.off.as<int32_t>(), pool_idx,
                                cd.pair_tet.as<int32_t>(), c->w_off.as<int32_t>(),
                                cd.moff.as<int32_t>(), nc_max, cd.cut.as<unsigned>())))
    return e;
  // (3) clip the batch; its pieces to the pool's tail
  if ((e = mark(4))) return e;
  if ((e = launch_clip(c, nc_max, cd.pair_tet.as<int32_t>(), dl, pool_idx, cd.moff.as<int32_t>(),
                       cd.cut.as<unsigned>(), 0)))
    return e;
  if ((e = launch_clip_overflow(c, cd.pair_tet.as<int32_t>(), dl, pool_idx,
                                cd.moff.as<int32_t>(), cd.cut.as<unsigned>())))
    return e;
  if ((e = mark(5))) return e;
  if ((e = launch_piece_scans(c, nc_max, cd.moff.as<int32_t>()))) return e;
  PieceDst d{c->pcs_d.off.as<int32_t>(), pool_p.sphere.as<int32_t>(), pool_p.vol.as<double>(),
             pool_p.m1.as<double>(), pool_p.fm.as<uint8_t>(), pool_p.inc_off.as<int32_t>(),
             pool_p.inc.as<int32_t>(), nullptr, nullptr, nullptr, nullptr, nullptr, nullptr,
             nullptr, nullptr, 0, 0};
  if ((e = launch_compact_pieces(c, T, nc_max, cd.off.as<int32_t>(), pool_idx,
                                 cd.moff.as<int32_t>(), d)))
    return e;
  // (4) re-point the dirty tets' rows; the totals back to the host
  unsigned long long* rm = c->m_cnt.as<unsigned long long>();
  if ((e = launch_rows_update(c, dl, T, pool_c, pool_p, cd, c->pcs_d, 0, 0, rm))) return e;
  return launch_pd_final(c);  // (the one readback: into the mapped PDyn mirror)
}

static void graph_clear(rpd_ctx* c) {
  for (int k = 0; k < rpd_ctx::G_CACHE; ++k) {
    if (c->g_exec[k]) cudaGraphExecDestroy(c->g_exec[k]);
    c->g_exec[k] = nullptr;
    c->g_sig[k] = 0;
  }
}

static rpd_status partial_graph(rpd_ctx* c, const double* spheres, int64_t N_new,
                                const int32_t* nbr_off, const int32_t* nbr_idx, int64_t E,
                                const int32_t* new_ids, int64_t M, rpd_pieces* out,
                                const int32_t** dirty_tets, int64_t* n_dirty) {
  const auto h0 = std::chrono::steady_clock::now();
  const int64_t N_old = c->st.N, T = c->st.T;
  // inputs on the device (host arrays are copied on the ctx stream ahead of the graph)
  rpd_status s = read_E(c, nbr_off, N_new, &E);
  if (s) return s;
  if (E > 0 && !nbr_idx) return fail(c, RPD_EINVAL, "nbr_idx is NULL");
  const double* d_sph = nullptr;
  const int32_t *d_off = nullptr, *d_idx = nullptr, *d_new = nullptr;
  CK(resolve(c, spheres, 4 * N_new, c->h_spheres, &d_sph), "stage spheres");
  CK(resolve(c, nbr_off, N_new + 1, c->h_off, &d_off), "stage nbr_off");
  CK(resolve(c, nbr_idx, E, c->h_idx, &d_idx), "stage nbr_idx");
  CK(resolve(c, new_ids, M, c->h_new, &d_new), "stage new ids");
  // room at the pools' tails for a batch at the graph's bounds (a compaction, when the pools
  // are full, runs here -- before the new rows are staged, like every state read of the pools)
  // the batch bound: twice the last batch (never shrinking: no recapture for smaller ones)
  const int64_t nc_max =
      c->g_nc_fix > 0 ? c->g_nc_fix
                      : std::max(std::max<int64_t>(c->g_nc_max, RPD_GRAPH_NC_MIN),
                                 pow2_at_least(2 * c->g_last_nc));
  if (c->g_nc_fix <= 0) c->g_nc_max = nc_max;
  const int64_t nw_max = 4 * nc_max;
  const int64_t Mb = graph_mb(M);
  c->g_mb = Mb;
  // (the room is checked exactly on the device; the host reserves what the last batch needed
  // plus a quarter, like the eager path's exact reservation; a shortfall redoes the batch)
  {
    const int64_t ec = std::max<int64_t>(4096, c->g_last_nc + c->g_last_nc / 4);
    const int64_t ew = std::max<int64_t>(4096, c->g_last_nw + c->g_last_nw / 4);
    s = reserve_pools(c, ec, ec, 32 * ew, 0);
  }
  if (s) return s;
  c->rpe_n = -1;
  ++c->epoch;
  c->last.N = N_new;
  CK(stage_prepare(c, N_new, E), "stage");
  // every buffer sized for the graph's bounds (allocation moves buffers: a new capture)
  const int64_t Nb = (int64_t)(c->st.sw.cap / sizeof(double4));
  const int64_t n_leaf = (T + 31) / 32, n_sup = (n_leaf + 31) / 32;
  {
    const int64_t ci0 = Mb * n_leaf + 4096, cs0 = Mb * n_sup + 4096;
    int64_t ci1 = std::max<int64_t>(48 * Nb + 4 * n_leaf + 4096, c->bvh_min_items);
    int64_t cs1 = std::max<int64_t>(8 * Nb + 4 * n_sup + 4096, c->bvh_min_items);
    ci1 = std::min<int64_t>(ci1, 1 << 30);
    cs1 = std::min<int64_t>(cs1, 1 << 30);
    c->dd_cap[0][0] = ci0;
    c->dd_cap[0][1] = cs0;
    c->dd_cap[1][0] = ci1;
    c->dd_cap[1][1] = cs1;
    CK(c->bvh_items.ensure(sizeof(int2) * (std::max(ci0 + cs0, ci1 + cs1) + 1)), "alloc");
  }
  const size_t nt = (size_t)T;
  const size_t scan_words = 8 + (1 + tiles_of(T)) + (1 + tiles_of(Nb)) + (1 + 2 * tiles_of(T)) +
                            (1 + 2 * tiles_of(nc_max));
  struct {
    DevBuf* b;
    size_t bytes;
  } need[] = {
      {&c->d_count, 4 * nt},          {&c->d_flag, nt},
      {&c->d_scan, 4 * (nt + 1)},
      {&c->min_epoch, 4},             {&c->c_flag, (size_t)Nb},
      {&c->c_scan, 4 * (size_t)(Nb + 1)}, {&c->c_list, 4 * (size_t)Nb},
      {&c->k_tet, 4 * nt},            {&c->k_words, 4 * nt},
      {&c->cand_d.off, 4 * (nt + 1)}, {&c->w_off, 4 * (nt + 1)},
      {&c->slab, 4 * (size_t)c->slab_cap * nt}, {&c->slab_m, 8 * (size_t)c->slab_cap * nt},
      {&c->cand_d.pair_tet, 4 * (size_t)nc_max}, {&c->cand_d.moff, 4 * (size_t)(nc_max + 1)},
      {&c->cand_d.cut, 4 * (size_t)nw_max}, {&c->pcs_d.off, 4 * (nt + 1)},
      {&c->p_flag, (size_t)nc_max},   {&c->p_f01, 4 * (size_t)nc_max},
      {&c->p_fm, (size_t)nc_max},     {&c->p_vol, 8 * (size_t)nc_max},
      {&c->p_m1, 24 * (size_t)nc_max}, {&c->p_ninc, 4 * (size_t)nc_max},
      {&c->p_over, 4 * (size_t)(nc_max + 1)}, {&c->p_over2, 4 * (size_t)(nc_max + 1)},
      {&c->p_over3, 4 * (size_t)(nc_max + 1)}, {&c->p_mask, 4 * (size_t)nw_max},
      {&c->p_scan, 4 * (size_t)(nc_max + 1)}, {&c->i_scan, 4 * (size_t)(nc_max + 1)},
      {&c->p_dyn, 4},                 {&c->m_cnt, 32},
      {&c->cand_long, 4 * (nt + 1)},  {&c->bvh, 8 * 6 * (size_t)(n_leaf + n_sup)},
      {&c->g_scan, 8 * scan_words},   {&c->pd_buf, sizeof(PDyn)},
      {&c->p_route, 4 * (2 + 2 * (size_t)nc_max)}};
  for (auto& x : need) CK(x.b->ensure(x.bytes), "alloc");
  if (!c->pd_host) {
    void* h = nullptr;
    CK(cudaHostAlloc(&h, sizeof(PDyn), cudaHostAllocMapped), "alloc");
    c->pd_host = (PDyn*)h;
    void* hd = nullptr;
    CK(cudaHostGetDevicePointer(&hd, h, 0), "alloc");
    c->pd_hdev = (PDyn*)hd;
  }
  CandSet& pool_c = c->cand[c->cur];
  PieceSet& pool_p = c->pcs[c->cur];
  PDyn& h = *c->pd_host;
  h = PDyn{};
  h.spheres = d_sph;
  h.nbr_off = d_off;
  h.nbr_idx = d_idx;
  h.new_ids = d_new;
  h.N = (int)N_new;
  h.N_old = (int)N_old;
  h.E = (int)E;
  h.M = (int)M;
  h.epoch = c->epoch;
  h.fill_c = (int)pool_c.fill;
  h.fill_p = (int)pool_p.fill_p;
  h.fill_i = (int)pool_p.fill_i;
  h.room_c = (int)std::min<size_t>(pool_c.idx.cap / 4, INT32_MAX);
  h.room_p = (int)std::min<size_t>(
      std::min(std::min(pool_p.sphere.cap / 4, pool_p.vol.cap / 8),
               std::min(std::min(pool_p.m1.cap / 24, pool_p.fm.cap), pool_p.inc_off.cap / 4 - 1)),
      INT32_MAX);
  h.room_i = (int)std::min<size_t>(pool_p.inc.cap / 4, INT32_MAX);
  h.nc_max = (int)nc_max;
  h.nw_max = (int)nw_max;
  h.cap_items = (int)c->dd_cap[1][0];
  h.cap_sup = (int)c->dd_cap[1][1];
  // the graph of this buffer layout (captured on first use)
  // the signature: every device address and every host value the captured launches bake in
  unsigned long long sig = 1469598103934665603ull;
  auto mix = [&](unsigned long long v) { sig = (sig ^ v) * 1099511628211ull; };
  {
    const Stage& S = c->st;
    const CandSet& cd = c->cand_d;
    const DevBuf* bufs[] = {
        &c->errw, &c->stats, &c->pd_buf, &S.tx, &S.sw, &S.old_sw, &S.nbr_off, &S.old_off,
        &S.nbr_idx, &S.old_idx, &S.planes, &S.old_planes, &S.twin, &S.old_twin, &S.hkey,
        &S.old_hkey, &S.repoch, &S.old_repoch, &S.htab, &S.long_rows, &c->bvh_all, &c->bvh,
        &c->bvh_items,
        &c->d_count, &c->d_flag, &c->d_scan, &c->d_list, &c->cepoch, &c->min_epoch,
        &c->c_flag, &c->c_scan, &c->c_list, &c->g_scan, &c->k_tet, &c->k_words, &c->slab,
        &c->slab_m, &cd.off, &cd.pair_tet, &cd.moff, &cd.cut, &c->w_off, &c->cand_long,
        &pool_c.rows, &pool_c.idx, &pool_p.rows, &pool_p.sphere, &pool_p.vol, &pool_p.m1,
        &pool_p.fm, &pool_p.inc_off, &pool_p.inc, &c->pcs_d.off, &c->p_flag, &c->p_f01,
        &c->p_fm, &c->p_vol, &c->p_m1, &c->p_ninc, &c->p_mask, &c->p_over, &c->p_over2,
        &c->p_over3, &c->p_scan, &c->i_scan, &c->p_dyn, &c->m_cnt, &c->p_route};
    for (const DevBuf* b : bufs) mix((unsigned long long)(uintptr_t)b->p);
    for (unsigned long long v :
         {(unsigned long long)(S.sw.cap / sizeof(double4)), (unsigned long long)c->slab_cap,
          (unsigned long long)T, (unsigned long long)c->dd_cap[0][0],
          (unsigned long long)c->dd_cap[0][1], (unsigned long long)c->dd_cap[1][0],
          (unsigned long long)c->dd_cap[1][1], (unsigned long long)c->sms,
          (unsigned long long)nc_max, (unsigned long long)Mb, (unsigned long long)c->profile,
          (unsigned long long)c->clip_route,
          (unsigned long long)(uintptr_t)c->pinned_dev, (unsigned long long)(uintptr_t)c->pd_hdev})
      mix(v);
  }
  int slot = -1;
  for (int k = 0; k < rpd_ctx::G_CACHE; ++k)
    if (c->g_exec[k] && c->g_sig[k] == sig) slot = k;
  if (slot < 0) {
    if (!c->cap_stream) CK(cudaStreamCreateWithFlags(&c->cap_stream, cudaStreamNonBlocking), "stream");
    if (!c->side_stream) {  // (the concurrent branch: clip routing)
      CK(cudaStreamCreateWithFlags(&c->side_stream, cudaStreamNonBlocking), "stream");
      CK(cudaEventCreateWithFlags(&c->g_fork, cudaEventDisableTiming), "event");
      CK(cudaEventCreateWithFlags(&c->g_join, cudaEventDisableTiming), "event");
    }
    c->pdd_nc_max = nc_max;
    // (the capture is ordered after the work already queued on the ctx stream by the graph's
    // launch below, not by the capture itself: nothing is executed while capturing)
    cudaStream_t saved = c->stream;
    c->stream = c->cap_stream;
    c->pdd = c->pd_buf.as<PDyn>();
    c->g_scan_used = 0;
    const int64_t l0 = c->launches;
    cudaError_t e = cudaStreamBeginCapture(c->cap_stream, cudaStreamCaptureModeRelaxed);
    cudaError_t e1 = e ? e : issue_dd(c, Nb, nc_max);
    cudaGraph_t g = nullptr;
    cudaError_t e2 = e ? cudaSuccess : cudaStreamEndCapture(c->cap_stream, &g);
    c->stream = saved;
    c->pdd = nullptr;
    c->g_nodes = c->launches - l0;
    c->launches = l0;
    if (e1 || e2) {
      if (g) cudaGraphDestroy(g);
      return cuda_fail(c, e1 ? e1 : e2, "graph capture");
    }
    cudaGraphExec_t x = nullptr;
    e = cudaGraphInstantiate(&x, g, 0);
    cudaGraphDestroy(g);
    CK(e, "graph instantiate");
    slot = c->g_next;
    c->g_next = (c->g_next + 1) % rpd_ctx::G_CACHE;
    if (c->g_exec[slot]) cudaGraphExecDestroy(c->g_exec[slot]);
    c->g_exec[slot] = x;
    c->g_sig[slot] = sig;
    c->g_kernels[slot] = c->g_nodes;
    ++c->g_captures;
  }
  static const int g_time = getenv("RPD_GRAPH_TIME") ? 1 : 0;  // development: graph duration
  cudaEvent_t gt[2] = {nullptr, nullptr};
  const auto h1 = std::chrono::steady_clock::now();
  if (g_time) {
    cudaEventCreate(&gt[0]);
    cudaEventCreate(&gt[1]);
    cudaEventRecord(gt[0], c->stream);
  }
  CK(cudaGraphLaunch(c->g_exec[slot], c->stream), "graph launch");
  if (g_time) cudaEventRecord(gt[1], c->stream);
  c->launches += c->g_kernels[slot];
  ++c->g_launches;
  CK(cudaStreamSynchronize(c->stream), "partial update");
  if (g_time) {
    float ms = 0.f;
    cudaEventElapsedTime(&ms, gt[0], gt[1]);
    fprintf(stderr, "[rpd graph] %.3f ms on the device, %lld kernel nodes; host prologue %.3f ms, "
            "launch to sync %.3f ms\n", ms, (long long)c->g_kernels[slot],
            std::chrono::duration<double, std::milli>(h1 - h0).count(),
            std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - h1)
                .count());
    cudaEventDestroy(gt[0]);
    cudaEventDestroy(gt[1]);
  }
  const PDyn r = *c->pd_host;
  // the readback fields of the eager path, from the mirror
  Readback* rb = (Readback*)c->pinned;
  for (int k = 0; k < ST_N; ++k) rb->u64[k] = r.stats[k];
  for (int k = 0; k < 4; ++k) {
    rb->err[k] = r.err[k];
    rb->u4[k] = r.removed[k];
  }
  rb->i32[0] = r.n_wide;
  if (c->profile) {
    c->last.filter_ms += 1e-6 * (double)((r.stamp[1] - r.stamp[0]) + (r.stamp[3] - r.stamp[2]));
    c->last.clip_ms += 1e-6 * (double)(r.stamp[5] - r.stamp[4]);
  }
  if (rb->err[0] != 0) {
    if (rb->err[1] == 100) return fail(c, RPD_EINVAL, "new_ids is not the appended id range");
    return check_err(c, rb);
  }
  c->last.rel_tests += (int64_t)rb->u64[ST_REL_TESTS];
  c->last.pairs_tested += (int64_t)rb->u64[ST_TESTED];
  c->g_last_nc = r.nc_req;
  c->g_last_nw = r.nw_req;
  if (r.abort) {  // a device-side check failed: the batch again, eagerly (same results)
    ++c->g_fallbacks;
    return partial_batch(c, r.nd, N_new, M, out, dirty_tets, n_dirty);
  }
  if (rb->u64[ST_OVERFLOW])
    return fail(c, RPD_EOVERFLOW, "a piece exceeded the wide clip capacity (128 vertices/planes)");
  absorb_clip_stats(c, rb, rb->i32[0]);
  c->last.max_k_tet = r.maxk;
  c->last.pairs_clipped += r.nc;
  CandSet& cd = c->cand_d;
  PieceSet& pd = c->pcs_d;
  cd.n = r.nc;
  cd.n_tets = r.nd;
  cd.n_words = r.nw;
  cd.idx_ext = pool_c.idx.as<int32_t>() + pool_c.fill;
  pd.n_tets = r.nd;
  pd.n_pieces = r.np;
  pd.n_inc = r.ni;
  pd.n_rpf = 0;
  const unsigned long long* removed = rb->u4;
  pool_c.fill += r.nc;
  pool_p.fill_p += r.np;
  pool_p.fill_i += r.ni;
  pool_c.n += r.nc - (int64_t)removed[0];
  pool_p.n_pieces += r.np - (int64_t)removed[1];
  pool_p.n_inc += r.ni - (int64_t)removed[2];
  c->compact = false;
  c->eu_valid = false;
  c->last.n_cand_dirty = r.nc;
  c->last.n_pieces_dirty = r.np;
  c->last.n_inc_dirty = r.ni;
  c->n_dirty = r.nd;
  c->last.n_dirty = r.nd;
  c->last.n_cand = pool_c.n;
  c->last.n_pieces = pool_p.n_pieces;
  c->last.n_inc = pool_p.n_inc;
  c->last.pairs_filtered = T * M + (int64_t)r.nd * N_new;
  *dirty_tets = c->d_list.as<int32_t>();
  *n_dirty = r.nd;
  return fill_pieces(c, out);
}

rpd_status rpd_download_pieces(rpd_ctx* c, int32_t* piece_off, int32_t* piece_sphere,
                               double* piece_vol, double* piece_m1, uint8_t* piece_facemask,
                               int32_t* inc_off, int32_t* inc_sphere) {
  if (!c) return RPD_EINVAL;
  if (!c->have_pieces) return fail(c, RPD_ESTATE, "no pieces");
  if (!c->compact) {  // the pools after partial updates: gathered by their rows
    if (!piece_off) return fail(c, RPD_EINVAL, "rpd_download_pieces: piece_off is needed");
    CK(cudaSetDevice(c->device), "cudaSetDevice");
    rpd_csr o{nullptr, nullptr, piece_off, piece_sphere, piece_vol, piece_m1, piece_facemask,
              inc_off, inc_sphere, 0, 0, 0, 0};
    return download_rows(c, 0, nullptr, c->st.T, &o);
  }
  const PieceSet& ps = c->pcs[c->cur];
  const int64_t T = c->st.T, np = ps.n_pieces, ni = ps.n_inc;
  auto cp = [&](void* dst, const void* src, size_t bytes) -> cudaError_t {
    if (!dst || bytes == 0) return cudaSuccess;
    return cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDefault, c->stream);
  };
  CK(cp(piece_off, ps.off.p, sizeof(int32_t) * (T + 1)), "download");
  CK(cp(piece_sphere, ps.sphere.p, sizeof(int32_t) * np), "download");
  CK(cp(piece_vol, ps.vol.p, sizeof(double) * np), "download");
  CK(cp(piece_m1, ps.m1.p, sizeof(double) * 3 * np), "download");
  CK(cp(piece_facemask, ps.fm.p, np), "download");
  CK(cp(inc_off, ps.inc_off.p, sizeof(int32_t) * (np + 1)), "download");
  CK(cp(inc_sphere, ps.inc.p, sizeof(int32_t) * ni), "download");
  // host destinations are complete on return; device ones are stream-ordered
  if (is_host_ptr(piece_off) || is_host_ptr(piece_vol) || is_host_ptr(inc_sphere))
    CK(cudaStreamSynchronize(c->stream), "download");
  return RPD_OK;
}

rpd_status rpd_set_euler(rpd_ctx* c, const int32_t* tets_all, int64_t T_all, int64_t V,
                         const int32_t* local_ids, int64_t T_local, int64_t* n_primes) {
  if (!c) return RPD_EINVAL;
  c->eu_valid = false;
  if (!tets_all && T_all == 0) {  // switch off
    c->euler = 0;
    if (n_primes) *n_primes = 0;
    return RPD_OK;
  }
  if (!tets_all || T_all < 0 || T_all > 0x7fffffff || V <= 0 || V >= (1ll << 21) ||
      T_local < 0 || T_local > 0x7fffffff || (!local_ids && T_local != T_all && T_local != 0) ||
      !n_primes)
    return fail(c, RPD_EINVAL, "rpd_set_euler: bad argument (V must be in (0, 2^21))");
  CK(cudaSetDevice(c->device), "cudaSetDevice");
  const int32_t *d_tets = nullptr, *d_ids = nullptr;
  CK(resolve(c, tets_all, 4 * T_all, c->h_eut, &d_tets), "stage tets");
  CK(resolve(c, local_ids, local_ids ? T_local : 0, c->h_euid, &d_ids), "stage ids");
  CK(cudaMemsetAsync(c->errw.p, 0, sizeof(int) * 4, c->stream), "memset");
  CK(launch_euler_setup(c, d_tets, T_all, V, d_ids, T_local), "euler setup");
  const bool whole = local_ids == nullptr && T_local == T_all;
  if (!whole) {  // (sharded CC numbers: the global ids of the ctx's tets and back)
    CK(c->eu_ids.ensure(sizeof(int32_t) * (T_local > 0 ? T_local : 1)), "alloc");
    if (T_local > 0)
      CK(cudaMemcpyAsync(c->eu_ids.p, d_ids, sizeof(int32_t) * T_local, cudaMemcpyDeviceToDevice,
                         c->stream), "copy ids");
    CK(launch_g2l(c, d_ids, T_local, T_all), "id map");
  }
  long long table[129];
  CK(cudaMemcpyAsync(table, c->eu_A.p, sizeof(table), cudaMemcpyDeviceToHost, c->stream),
     "readback");
  Readback* rb = (Readback*)c->pinned;
  CK(readback(c, RbSpec{{}, nullptr, c->errw.as<int>()}), "readback");
  CK(cudaStreamSynchronize(c->stream), "euler setup");
  c->eu_tab.release();  // (hash tables: scratch of the setup only)
  if (rb->err[0] != 0) {
    if (rb->err[1] == 200)
      return fail(c, RPD_EOVERFLOW, "Euler mode: a mesh element is shared by more than 255 tets");
    if (rb->err[1] == 201)
      return fail(c, RPD_EOVERFLOW, "Euler mode: a tet's denominator (lcm of its counts) >= 2^62");
    if (rb->err[0] == RPD_ENOMEM) return fail(c, RPD_ENOMEM, "Euler mode: hash table full");
    return check_err(c, rb);
  }
  c->eu_P = (int)table[128];
  for (int j = 0; j < c->eu_P; ++j) {
    c->eu_primes[j] = (int)table[j];
    c->eu_ppow[j] = (int)table[64 + j];
  }
  c->euler = 1;
  c->eu_whole = whole;
  c->eu_T = T_local;
  *n_primes = c->eu_P;
  return RPD_OK;
}

rpd_status rpd_get_euler(rpd_ctx* c, rpd_euler* out) {
  if (!c || !out) return fail(c, RPD_EINVAL, "rpd_get_euler: bad argument");
  if (!c->euler || !c->eu_valid || !c->have_pieces)
    return fail(c, RPD_ESTATE, "no Euler data (rpd_set_euler, then rpd_clip)");
  CK(cudaSetDevice(c->device), "cudaSetDevice");
  const PieceSet& ps = c->pcs[c->cur];
  CK(launch_piece_den(c, ps), "piece denominators");
  const int64_t N = c->st.N, E = c->st.E, rows = N + E, W = 1 + c->eu_P;
  long long* vi = c->eu_fin.as<long long>();
  double* vd = reinterpret_cast<double*>(vi + rows + 1);
  uint8_t* ex = reinterpret_cast<uint8_t*>(vd + rows + 1);
  out->n_primes = c->eu_P;
  out->piece_euler = ps.eu.as<int64_t>();
  out->piece_denom = c->eu_den.as<int64_t>();
  out->rpf_off = ps.rpf_off.as<int32_t>();
  out->rpf_sphere = ps.rpf_j.as<int32_t>();
  out->rpf_euler = ps.rpf_e.as<int64_t>();
  out->rpc_sum = reinterpret_cast<const int64_t*>(vi);
  out->rpc_exact = ex;
  out->rpc_value = vd;
  out->rpf_sum = reinterpret_cast<const int64_t*>(vi + N);
  out->rpf_exact = ex + N;
  out->rpf_value = vd + N;
  out->rpc_acc = c->eu_acc.as<int64_t>();
  out->rpf_acc = c->eu_acc.as<int64_t>() + W * N;
  out->n_pieces = ps.n_pieces;
  out->n_rpf = ps.n_rpf;
  out->N = N;
  out->E = E;
  return RPD_OK;
}

rpd_status rpd_download_euler(rpd_ctx* c, int64_t* piece_euler, int64_t* piece_denom,
                              int32_t* rpf_off, int32_t* rpf_sphere, int64_t* rpf_euler,
                              int64_t* rpc_sum, uint8_t* rpc_exact, double* rpc_value,
                              int64_t* rpf_sum, uint8_t* rpf_exact, double* rpf_value,
                              int64_t* rpc_acc, int64_t* rpf_acc) {
  rpd_euler e;
  rpd_status s = rpd_get_euler(c, &e);
  if (s) return s;
  const int64_t W = 1 + e.n_primes;
  auto cp = [&](void* dst, const void* src, size_t bytes) -> cudaError_t {
    if (!dst || bytes == 0) return cudaSuccess;
    return cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDefault, c->stream);
  };
  CK(cp(piece_euler, e.piece_euler, sizeof(int64_t) * e.n_pieces), "download");
  CK(cp(piece_denom, e.piece_denom, sizeof(int64_t) * e.n_pieces), "download");
  CK(cp(rpf_off, e.rpf_off, sizeof(int32_t) * (e.n_pieces + 1)), "download");
  CK(cp(rpf_sphere, e.rpf_sphere, sizeof(int32_t) * e.n_rpf), "download");
  CK(cp(rpf_euler, e.rpf_euler, sizeof(int64_t) * e.n_rpf), "download");
  CK(cp(rpc_sum, e.rpc_sum, sizeof(int64_t) * e.N), "download");
  CK(cp(rpc_exact, e.rpc_exact, e.N), "download");
  CK(cp(rpc_value, e.rpc_value, sizeof(double) * e.N), "download");
  CK(cp(rpf_sum, e.rpf_sum, sizeof(int64_t) * e.E), "download");
  CK(cp(rpf_exact, e.rpf_exact, e.E), "download");
  CK(cp(rpf_value, e.rpf_value, sizeof(double) * e.E), "download");
  CK(cp(rpc_acc, e.rpc_acc, sizeof(int64_t) * W * e.N), "download");
  CK(cp(rpf_acc, e.rpf_acc, sizeof(int64_t) * W * e.E), "download");
  CK(cudaStreamSynchronize(c->stream), "download");
  return RPD_OK;
}

rpd_status rpd_euler_finalize(rpd_ctx* c, const int64_t* acc, int64_t n_rows, int64_t* out_sum,
                              uint8_t* out_exact, double* out_value) {
  if (!c) return RPD_EINVAL;
  if (!c->euler) return fail(c, RPD_ESTATE, "rpd_euler_finalize: Euler mode is off");
  if (n_rows < 0 || (n_rows > 0 && (!acc || !out_sum || !out_exact || !out_value)))
    return fail(c, RPD_EINVAL, "rpd_euler_finalize: bad argument");
  CK(cudaSetDevice(c->device), "cudaSetDevice");
  CK(launch_euler_final(c, reinterpret_cast<const unsigned long long*>(acc), n_rows,
                        reinterpret_cast<long long*>(out_sum), out_value, out_exact),
     "finalize");
  CK(cudaStreamSynchronize(c->stream), "finalize");
  return RPD_OK;
}

rpd_status rpd_get_topology(rpd_ctx* c, rpd_topology* out) {
  if (!c || !out) return fail(c, RPD_EINVAL, "rpd_get_topology: bad argument");
  if (!c->euler || !c->eu_valid || !c->have_pieces)
    return fail(c, RPD_ESTATE, "no topology data (rpd_set_euler, then rpd_clip)");
  if (!c->eu_whole)
    return fail(c, RPD_ESTATE, "CC numbers need the whole mesh in the ctx (local_ids == NULL)");
  CK(cudaSetDevice(c->device), "cudaSetDevice");
  const PieceSet& ps = c->pcs[c->cur];
  CK(launch_cc(c, ps), "cc");
  out->rpc_cc = c->cc_out.as<int32_t>();
  out->rpf_cc = c->cc_out.as<int32_t>() + c->st.N;
  out->piece_comp = c->cc_par.as<int32_t>();
  out->rpf_comp = c->cc_par.as<int32_t>() + ps.n_pieces;
  out->piece_sosfm = ps.sfm.as<uint8_t>();
  out->rpf_fm = ps.rfm.as<uint8_t>();
  out->rpf_adj = ps.radj.as<uint64_t>();
  out->n_pieces = ps.n_pieces;
  out->n_rpf = ps.n_rpf;
  out->N = c->st.N;
  out->E = c->st.E;
  return RPD_OK;
}

rpd_status rpd_cc_shard(rpd_ctx* c, int64_t piece_base, int64_t rpf_base, rpd_cc_records* out) {
  if (!c || !out || piece_base < 0 || rpf_base < 0)
    return fail(c, RPD_EINVAL, "rpd_cc_shard: bad argument");
  if (!c->euler || !c->eu_valid || !c->have_pieces)
    return fail(c, RPD_ESTATE, "no topology data (rpd_set_euler, then rpd_clip)");
  if (c->eu_whole)
    return fail(c, RPD_ESTATE, "rpd_cc_shard: the ctx holds the whole mesh (rpd_get_topology)");
  if (c->st.N >= (1 << 21)) return fail(c, RPD_EINVAL, "rpd_cc_shard: record keys need N < 2^21");
  CK(cudaSetDevice(c->device), "cudaSetDevice");
  const PieceSet& ps = c->pcs[c->cur];
  if (piece_base + ps.n_pieces > 0x7fffffff || rpf_base + ps.n_rpf > 0x7fffffff)
    return fail(c, RPD_EINVAL, "rpd_cc_shard: global ids beyond int32");
  CK(c->cc_nrec.ensure(sizeof(int) * 2), "alloc");
  int* n_rec = c->cc_nrec.as<int>();
  CK(launch_cc_shard(c, ps, piece_base, rpf_base, n_rec), "cc shard");
  Readback* rb = (Readback*)c->pinned;
  CK(readback(c, RbSpec{{n_rec, n_rec + 1}, nullptr, nullptr}), "readback");
  CK(cudaStreamSynchronize(c->stream), "cc shard");
  c->cc_base_c = piece_base;
  c->cc_base_f = rpf_base;
  const size_t nc = 4 * (size_t)ps.n_pieces + 1, nf = 4 * (size_t)ps.n_rpf + 1;
  const uint64_t* key_c = c->cc_bnd.as<uint64_t>();
  const uint64_t* key_f = key_c + nc;
  const int32_t* lab_c = reinterpret_cast<const int32_t*>(key_f + nf);
  const int32_t* j_f = lab_c + nc;
  const int32_t* lab_f = j_f + nf;
  *out = rpd_cc_records{key_c, lab_c, rb->i32[0], key_f, j_f, lab_f, rb->i32[1],
                        ps.n_pieces, ps.n_rpf};
  return RPD_OK;
}

rpd_status rpd_cc_merge(rpd_ctx* c, const uint64_t* key_c, const int32_t* lab_c, int64_t n_c,
                        const uint64_t* key_f, const int32_t* j_f, const int32_t* lab_f,
                        int64_t n_f, int64_t total_pieces, int64_t total_rpf, int32_t* counts) {
  if (!c || n_c < 0 || n_f < 0 || (n_c > 0 && (!key_c || !lab_c)) ||
      (n_f > 0 && (!key_f || !j_f || !lab_f)) || !counts || total_pieces < 0 || total_rpf < 0 ||
      total_pieces > 0x7ffffffe || total_rpf > 0x7ffffffe || n_c > 0x7fffffff || n_f > 0x7fffffff)
    return fail(c, RPD_EINVAL, "rpd_cc_merge: bad argument");
  if (c->cc_base_c < 0 || !c->euler || !c->eu_valid)
    return fail(c, RPD_ESTATE, "rpd_cc_merge before rpd_cc_shard");
  const PieceSet& ps = c->pcs[c->cur];
  if (c->cc_base_c + ps.n_pieces > total_pieces || c->cc_base_f + ps.n_rpf > total_rpf)
    return fail(c, RPD_EINVAL, "rpd_cc_merge: totals smaller than this rank's range");
  CK(cudaSetDevice(c->device), "cudaSetDevice");
  CK(launch_cc_merge(c, ps, reinterpret_cast<const unsigned long long*>(key_c), lab_c, n_c,
                     reinterpret_cast<const unsigned long long*>(key_f), j_f, lab_f, n_f,
                     total_pieces, total_rpf, c->cc_base_c, c->cc_base_f, counts),
     "cc merge");
  CK(cudaStreamSynchronize(c->stream), "cc merge");
  return RPD_OK;
}

rpd_status rpd_rpe_shard(rpd_ctx* c, int64_t rpe_base, rpd_rpe_records* out) {
  if (!c || !out || rpe_base < 0) return fail(c, RPD_EINVAL, "rpd_rpe_shard: bad argument");
  if (!c->euler || !c->eu_valid || !c->have_pieces)
    return fail(c, RPD_ESTATE, "no topology data (rpd_set_euler, then rpd_clip)");
  if (c->eu_whole)
    return fail(c, RPD_ESTATE, "rpd_rpe_shard: the ctx holds the whole mesh (rpd_get_rpe)");
  if (c->st.N >= (1 << 21)) return fail(c, RPD_EINVAL, "RPE keys need N < 2^21");
  CK(cudaSetDevice(c->device), "cudaSetDevice");
  CK(c->cc_nrec.ensure(sizeof(int) * 2), "alloc");
  int* n_rec = c->cc_nrec.as<int>();
  int64_t n = 0, nu = 0;
  CK(launch_rpe_shard(c, c->pcs[c->cur], rpe_base, n_rec, &n, &nu), "rpe shard");
  if (rpe_base + n > 0x7fffffff) return fail(c, RPD_EINVAL, "rpd_rpe_shard: ids beyond int32");
  Readback* rb = (Readback*)c->pinned;
  CK(readback(c, RbSpec{{n_rec}, nullptr, nullptr}), "readback");
  CK(cudaStreamSynchronize(c->stream), "rpe shard");
  c->rpe_n = n;
  c->rpe_nu = nu;
  c->rpe_base = rpe_base;
  const int64_t n1 = n > 0 ? n : 1, nb = 4 * n1;
  const unsigned long long* keys = c->rpe_buf.as<unsigned long long>();
  const unsigned long long* key_b = c->rpe_bnd.as<unsigned long long>();
  *out = rpd_rpe_records{reinterpret_cast<const uint64_t*>(keys + 4 * n1),
                         reinterpret_cast<const int64_t*>(keys + 5 * n1), nu, n,
                         reinterpret_cast<const uint64_t*>(key_b),
                         reinterpret_cast<const uint64_t*>(key_b + nb),
                         reinterpret_cast<const int32_t*>(key_b + 2 * nb), rb->i32[0]};
  return RPD_OK;
}

rpd_status rpd_rpe_merge(rpd_ctx* c, const uint64_t* key_b, const uint64_t* jk_b,
                         const int32_t* lab_b, int64_t n_b, int64_t total_rpe,
                         const uint64_t** keys, const int64_t** counts, int64_t* n) {
  if (!c || n_b < 0 || (n_b > 0 && (!key_b || !jk_b || !lab_b)) || !keys || !counts || !n ||
      total_rpe < 0 || total_rpe > 0x7ffffffe || n_b > 0x7fffffff)
    return fail(c, RPD_EINVAL, "rpd_rpe_merge: bad argument");
  if (c->rpe_base < 0 || c->rpe_n < 0)
    return fail(c, RPD_ESTATE, "rpd_rpe_merge before rpd_rpe_shard");
  if (c->rpe_base + c->rpe_n > total_rpe)
    return fail(c, RPD_EINVAL, "rpd_rpe_merge: total smaller than this rank's range");
  CK(cudaSetDevice(c->device), "cudaSetDevice");
  CK(c->cc_nrec.ensure(sizeof(int) * 2), "alloc");
  int* n_out = c->cc_nrec.as<int>();
  CK(launch_rpe_merge(c, reinterpret_cast<const unsigned long long*>(key_b),
                      reinterpret_cast<const unsigned long long*>(jk_b), lab_b, n_b, total_rpe,
                      c->rpe_base, n_out),
     "rpe merge");
  Readback* rb = (Readback*)c->pinned;
  CK(readback(c, RbSpec{{n_out}, nullptr, nullptr}), "readback");
  CK(cudaStreamSynchronize(c->stream), "rpe merge");
  const int64_t n1 = c->rpe_n > 0 ? c->rpe_n : 1;
  const unsigned long long* rk = c->rpe_cnt.as<unsigned long long>();
  *keys = reinterpret_cast<const uint64_t*>(rk + 2 * n1);
  *counts = reinterpret_cast<const int64_t*>(rk + 3 * n1);
  *n = rb->i32[0];
  return RPD_OK;
}

rpd_status rpd_reduce_by_key(rpd_ctx* c, const uint64_t* keys, const int64_t* vals, int64_t n,
                             uint64_t* out_keys, int64_t* out_vals, int64_t* n_out) {
  if (!c || n < 0 || n > 0x7fffffff || (n > 0 && (!keys || !vals || !out_keys || !out_vals)) ||
      !n_out)
    return fail(c, RPD_EINVAL, "rpd_reduce_by_key: bad argument");
  CK(cudaSetDevice(c->device), "cudaSetDevice");
  CK(c->cc_nrec.ensure(sizeof(int) * 2), "alloc");
  int* d_n = c->cc_nrec.as<int>();
  CK(launch_reduce_by_key(c, reinterpret_cast<const unsigned long long*>(keys),
                          reinterpret_cast<const long long*>(vals), n,
                          reinterpret_cast<unsigned long long*>(out_keys),
                          reinterpret_cast<long long*>(out_vals), d_n),
     "reduce by key");
  Readback* rb = (Readback*)c->pinned;
  CK(readback(c, RbSpec{{d_n}, nullptr, nullptr}), "readback");
  CK(cudaStreamSynchronize(c->stream), "reduce by key");
  *n_out = rb->i32[0];
  return RPD_OK;
}

rpd_status rpd_download_topology(rpd_ctx* c, int32_t* rpc_cc, int32_t* rpf_cc,
                                 int32_t* piece_comp, int32_t* rpf_comp, uint8_t* piece_sosfm,
                                 uint8_t* rpf_fm, uint64_t* rpf_adj) {
  rpd_topology t;
  rpd_status s = rpd_get_topology(c, &t);
  if (s) return s;
  auto cp = [&](void* dst, const void* src, size_t bytes) -> cudaError_t {
    if (!dst || bytes == 0) return cudaSuccess;
    return cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDefault, c->stream);
  };
  CK(cp(rpc_cc, t.rpc_cc, sizeof(int32_t) * t.N), "download");
  CK(cp(rpf_cc, t.rpf_cc, sizeof(int32_t) * t.E), "download");
  CK(cp(piece_comp, t.piece_comp, sizeof(int32_t) * t.n_pieces), "download");
  CK(cp(rpf_comp, t.rpf_comp, sizeof(int32_t) * t.n_rpf), "download");
  CK(cp(piece_sosfm, t.piece_sosfm, t.n_pieces), "download");
  CK(cp(rpf_fm, t.rpf_fm, t.n_rpf), "download");
  CK(cp(rpf_adj, t.rpf_adj, sizeof(uint64_t) * t.n_rpf), "download");
  CK(cudaStreamSynchronize(c->stream), "download");
  return RPD_OK;
}

static rpd_rpe rpe_view(rpd_ctx* c) {
  const int64_t n = c->rpe_n, n1 = n > 0 ? n : 1;
  unsigned long long* keys = c->rpe_buf.as<unsigned long long>();
  int32_t* ej = reinterpret_cast<int32_t*>(keys + 6 * n1);
  int32_t* ek = ej + n1;
  int32_t* cc = ek + n1;
  int32_t* tri = cc + n1;
  int32_t* par = tri + 3 * n1;
  rpd_rpe r{};
  r.denom = 2;  // tri_euler: halves
  r.rpe_off = c->rpe_off.as<int32_t>();
  r.rpe_j = ej;
  r.rpe_k = ek;
  r.rpe_euler = c->rpe_ee.as<int64_t>();
  r.rpe_fm = reinterpret_cast<uint8_t*>(par + n1);
  r.tri = tri;
  r.tri_euler = reinterpret_cast<int64_t*>(keys + 5 * n1);
  r.tri_cc = c->eu_whole ? cc : nullptr;
  r.n_pieces = c->pcs[c->cur].n_pieces;
  r.n_rpe = n;
  r.n_tri = c->rpe_nu;
  return r;
}

rpd_status rpd_get_rpe(rpd_ctx* c, rpd_rpe* out) {
  if (!c || !out) return fail(c, RPD_EINVAL, "rpd_get_rpe: bad argument");
  if (!c->euler || !c->eu_valid || !c->have_pieces)
    return fail(c, RPD_ESTATE, "no Euler data (rpd_set_euler, then rpd_clip)");
  if (c->st.N >= (1 << 21)) return fail(c, RPD_EINVAL, "RPE keys need N < 2^21");
  CK(cudaSetDevice(c->device), "cudaSetDevice");
  int64_t n = 0, nu = 0;
  CK(launch_rpe(c, c->pcs[c->cur], c->eu_whole, &n, &nu), "restricted power edges");
  CK(cudaStreamSynchronize(c->stream), "restricted power edges");
  *out = rpe_view(c);
  return RPD_OK;
}

rpd_status rpd_download_rpe(rpd_ctx* c, int32_t* rpe_off, int32_t* rpe_j, int32_t* rpe_k,
                            int64_t* rpe_euler, uint8_t* rpe_fm, int32_t* tri,
                            int64_t* tri_euler, int32_t* tri_cc) {
  if (!c) return RPD_EINVAL;
  if (c->rpe_n < 0 || !c->eu_valid) return fail(c, RPD_ESTATE, "no rpd_get_rpe results");
  const rpd_rpe r = rpe_view(c);
  auto cp = [&](void* dst, const void* src, size_t bytes) -> cudaError_t {
    if (!dst || !src || bytes == 0) return cudaSuccess;
    return cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDefault, c->stream);
  };
  CK(cp(rpe_off, r.rpe_off, sizeof(int32_t) * (r.n_pieces + 1)), "download");
  CK(cp(rpe_j, r.rpe_j, sizeof(int32_t) * r.n_rpe), "download");
  CK(cp(rpe_k, r.rpe_k, sizeof(int32_t) * r.n_rpe), "download");
  CK(cp(rpe_euler, r.rpe_euler, sizeof(int64_t) * r.n_rpe), "download");
  CK(cp(rpe_fm, r.rpe_fm, r.n_rpe), "download");
  CK(cp(tri, r.tri, sizeof(int32_t) * 3 * r.n_tri), "download");
  CK(cp(tri_euler, r.tri_euler, sizeof(int64_t) * r.n_tri), "download");
  CK(cp(tri_cc, r.tri_cc, sizeof(int32_t) * r.n_tri), "download");
  CK(cudaStreamSynchronize(c->stream), "download");
  return RPD_OK;
}

rpd_status rpd_medial_mesh(rpd_ctx* c, rpd_medial* out) {
  if (!c || !out) return fail(c, RPD_EINVAL, "rpd_medial_mesh: bad argument");
  if (!c->euler || !c->eu_valid || !c->have_pieces)
    return fail(c, RPD_ESTATE, "no topology data (rpd_set_euler, then rpd_clip)");
  if (c->st.N >= (1 << 21)) return fail(c, RPD_EINVAL, "medial mesh keys need N < 2^21");
  CK(cudaSetDevice(c->device), "cudaSetDevice");
  int64_t ne = 0, nf = 0;
  CK(launch_medial_mesh(c, c->pcs[c->cur], &ne, &nf), "medial mesh");
  out->edges = c->mm_out.as<int32_t>();
  out->faces = c->mm_out.as<int32_t>() + 2 * ne;
  out->n_edges = ne;
  out->n_faces = nf;
  c->mm_ne = ne;
  c->mm_nf = nf;
  return RPD_OK;
}

rpd_status rpd_download_medial_mesh(rpd_ctx* c, int32_t* edges, int32_t* faces) {
  if (!c) return RPD_EINVAL;
  if (c->mm_ne < 0) return fail(c, RPD_ESTATE, "no medial mesh (call rpd_medial_mesh)");
  if (edges && c->mm_ne)
    CK(cudaMemcpyAsync(edges, c->mm_out.p, sizeof(int32_t) * 2 * c->mm_ne, cudaMemcpyDefault,
                       c->stream), "download");
  if (faces && c->mm_nf)
    CK(cudaMemcpyAsync(faces, c->mm_out.as<int32_t>() + 2 * c->mm_ne,
                       sizeof(int32_t) * 3 * c->mm_nf, cudaMemcpyDefault, c->stream), "download");
  CK(cudaStreamSynchronize(c->stream), "download");
  return RPD_OK;
}

// ---- segment gather engine (rpd_gather.cu): multi-GPU gather, partial-mode merge, download
}  // extern "C"

static bool shards_ok(const rpd_shards* sh, bool pieces, bool cands) {
  if (!sh || sh->world < 1 || sh->world > RPD_MAX_RANKS || sh->T < 0 || sh->T > 0x7fffffff)
    return false;
  for (int r = 0; r < sh->world; ++r) {
    if (sh->n_tets[r] < 0) return false;
    if (sh->n_tets[r] == 0) continue;
    if (!sh->tet_ids[r]) return false;
    if (pieces && (!sh->piece_off[r] || !sh->inc_off[r])) return false;
    if (cands && !sh->cand_off[r]) return false;
  }
  return true;
}

static void shard_sources(const rpd_shards* sh, SegShards* v, SegSources* S, int first) {
  *v = SegShards{};
  v->world = sh->world;
  for (int r = 0; r < sh->world; ++r) {
    v->base[r + 1] = v->base[r] + sh->n_tets[r];
    v->tet_ids[r] = sh->tet_ids[r];
    S->s[first + r] = seg_src_csr(sh->cand_off[r], sh->cand_idx[r], sh->piece_off[r],
                                  sh->piece_sphere[r], sh->piece_vol[r], sh->piece_m1[r],
                                  sh->piece_facemask[r], sh->inc_off[r], sh->inc_sphere[r]);
    if (sh->n_tets[r] == 0) S->s[first + r] = SegSrc{};
  }
}

// map -> counts -> (sync: sizes, errors) -> copy; dst arrays sized by the caller (gather,
// download) or here (merge: ctx-owned, ensure_dst)
template <class EnsureDst>
static rpd_status seg_run(rpd_ctx* c, int kind, int64_t n_out, const int32_t* list,
                          const SegShards* v, int64_t T, const SegSources& S, SegDst D,
                          int64_t* n_cand, int64_t* n_pieces, int64_t* n_inc, bool copy,
                          EnsureDst ensure_dst) {
  CK(cudaMemsetAsync(c->errw.p, 0, sizeof(int) * 4, c->stream), "memset");
  CK(launch_map(c, kind, n_out, list, v, T), "row map");
  // the offsets go to the destination when it is known, else to scratch first
  CK(c->g_off.ensure(sizeof(int32_t) * 2 * (n_out + 1)), "alloc");
  int32_t* co = D.cand_off ? D.cand_off : (n_cand ? c->g_off.as<int32_t>() : nullptr);
  int32_t* po = D.piece_off ? D.piece_off
                            : (n_pieces ? c->g_off.as<int32_t>() + (n_out + 1) : nullptr);
  int32_t* it = nullptr;
  CK(launch_seg_counts(c, n_out, S, co, po, &it), "segment counts");
  Readback* rb = (Readback*)c->pinned;
  CK(readback(c, RbSpec{{co ? co + n_out : nullptr, po ? po + n_out : nullptr,
                         po ? it + n_out : nullptr},
                        nullptr, c->errw.as<int>()}),
     "readback");
  CK(cudaStreamSynchronize(c->stream), "segment counts");
  if (rb->err[0] != 0) return fail(c, RPD_EINVAL, "a tet id is out of range");
  if (n_cand) *n_cand = rb->i32[0];
  if (n_pieces) *n_pieces = rb->i32[1];
  if (n_inc) *n_inc = rb->i32[2];
  if (!copy) return RPD_OK;
  rpd_status s = ensure_dst(rb->i32[0], rb->i32[1], rb->i32[2], &D);
  if (s) return s;
  if (D.cand_off && D.cand_off != co && co)
    CK(cudaMemcpyAsync(D.cand_off, co, sizeof(int32_t) * (n_out + 1), cudaMemcpyDefault,
                       c->stream), "copy offsets");
  if (D.piece_off && D.piece_off != po && po)
    CK(cudaMemcpyAsync(D.piece_off, po, sizeof(int32_t) * (n_out + 1), cudaMemcpyDefault,
                       c->stream), "copy offsets");
  D.i_tet = it;
  CK(launch_seg_copy(c, n_out, S, D), "segment copy");
  // (no sync: device destinations are stream-ordered; host ones are synced by the caller)
  return RPD_OK;
}

static rpd_status no_ensure(int64_t, int64_t, int64_t, SegDst*) { return RPD_OK; }

extern "C" {

rpd_status rpd_gather_pieces(rpd_ctx* c, const rpd_shards* sh, int32_t* piece_off,
                             int32_t* piece_sphere, double* piece_vol, double* piece_m1,
                             uint8_t* piece_facemask, int32_t* inc_off, int32_t* inc_sphere) {
  if (!c) return RPD_EINVAL;
  if (!shards_ok(sh, true, false) || !piece_off || !inc_off)
    return fail(c, RPD_EINVAL, "rpd_gather_pieces: bad argument");
  CK(cudaSetDevice(c->device), "cudaSetDevice");
  rpd_shards p = *sh;
  for (int r = 0; r < p.world; ++r) p.cand_off[r] = p.cand_idx[r] = nullptr;
  SegShards v;
  SegSources S{};
  shard_sources(&p, &v, &S, 1);
  SegDst D{nullptr, nullptr, piece_off, piece_sphere, piece_vol, piece_m1, piece_facemask,
           inc_off, inc_sphere, nullptr};
  return seg_run(c, 3, sh->T, nullptr, &v, sh->T, S, D, nullptr, nullptr, nullptr, true,
                 no_ensure);
}

rpd_status rpd_gather_cands(rpd_ctx* c, const rpd_shards* sh, int32_t* cand_off,
                            int32_t* cand_idx) {
  if (!c) return RPD_EINVAL;
  if (!shards_ok(sh, false, true) || !cand_off)
    return fail(c, RPD_EINVAL, "rpd_gather_cands: bad argument");
  CK(cudaSetDevice(c->device), "cudaSetDevice");
  rpd_shards p = *sh;
  for (int r = 0; r < p.world; ++r) p.piece_off[r] = nullptr;
  SegShards v;
  SegSources S{};
  shard_sources(&p, &v, &S, 1);
  SegDst D{cand_off, cand_idx, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr,
           nullptr};
  return seg_run(c, 3, sh->T, nullptr, &v, sh->T, S, D, nullptr, nullptr, nullptr, true,
                 no_ensure);
}

static SegSrc state_source(rpd_ctx* c) {
  SegSrc s = seg_src_state(c->cand[c->cur], c->pcs[c->cur]);
  if (!c->have_pieces) {  // candidates only (after rpd_relations)
    s.p_beg = s.p_end = nullptr;
  }
  return s;
}

}  // extern "C"

// the segments of the state rows `list` (kind 1) or of all tets (kind 0, n = T) into the
// caller's arrays (host destinations through device staging and one copy per array)
static rpd_status download_rows(rpd_ctx* c, int kind, const int32_t* d_list, int64_t n,
                                rpd_csr* out) {
  SegSources S{};
  S.s[0] = state_source(c);
  const bool copy = out->cand_off || out->piece_off;
  const bool host = (out->cand_off && is_host_ptr(out->cand_off)) ||
                    (out->piece_off && is_host_ptr(out->piece_off));
  SegDst D{out->cand_off, out->cand_idx, out->piece_off, out->piece_sphere, out->piece_vol,
           out->piece_m1, out->piece_facemask, out->inc_off, out->inc_sphere, nullptr};
  int64_t nc = 0, np = 0, ni = 0;
  if (host) {
    // sizes first (the staging is laid out from them), then the copy into the staging
    rpd_status s = seg_run(c, kind, n, d_list, nullptr, c->st.T, S, SegDst{}, &nc, &np, &ni,
                           false, no_ensure);
    if (s) return s;
    size_t off = 0;
    auto take = [&](size_t bytes) { size_t o = off; off += (bytes + 15) / 16 * 16; return o; };
    const size_t o_co = take(4 * (n + 1)), o_ci = take(4 * nc), o_po = take(4 * (n + 1)),
                 o_ps = take(4 * np), o_pv = take(8 * np), o_pm = take(24 * np),
                 o_pf = take(np), o_io = take(4 * (np + 1)), o_is = take(4 * ni);
    CK(c->g_dst.ensure(off), "alloc");
    char* b = c->g_dst.as<char>();
    SegDst Dd{};
    if (out->cand_off)
      Dd.cand_off = (int32_t*)(b + o_co), Dd.cand_idx = (int32_t*)(b + o_ci);
    if (out->piece_off) {
      Dd.piece_off = (int32_t*)(b + o_po);
      Dd.piece_sphere = (int32_t*)(b + o_ps);
      Dd.piece_vol = (double*)(b + o_pv);
      Dd.piece_m1 = (double*)(b + o_pm);
      Dd.piece_fm = (uint8_t*)(b + o_pf);
      Dd.inc_off = (int32_t*)(b + o_io);
      Dd.inc_sphere = (int32_t*)(b + o_is);
    }
    s = seg_run(c, kind, n, d_list, nullptr, c->st.T, S, Dd, &nc, &np, &ni, true, no_ensure);
    if (s) return s;
    auto cp = [&](void* dst, const void* src, size_t bytes) -> cudaError_t {
      if (!dst || !src || bytes == 0) return cudaSuccess;
      return cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDefault, c->stream);
    };
    CK(cp(out->cand_off, Dd.cand_off, 4 * (n + 1)), "download");
    CK(cp(out->cand_idx, Dd.cand_idx, 4 * nc), "download");
    CK(cp(out->piece_off, Dd.piece_off, 4 * (n + 1)), "download");
    CK(cp(out->piece_sphere, Dd.piece_sphere, 4 * np), "download");
    CK(cp(out->piece_vol, Dd.piece_vol, 8 * np), "download");
    CK(cp(out->piece_m1, Dd.piece_m1, 24 * np), "download");
    CK(cp(out->piece_facemask, Dd.piece_fm, np), "download");
    CK(cp(out->inc_off, Dd.inc_off, 4 * (np + 1)), "download");
    CK(cp(out->inc_sphere, Dd.inc_sphere, 4 * ni), "download");
    CK(cudaStreamSynchronize(c->stream), "download");
  } else {
    rpd_status s = seg_run(c, kind, n, d_list, nullptr, c->st.T, S, D, &nc, &np, &ni, copy,
                           no_ensure);
    if (s) return s;
  }
  out->T = n;
  out->n_cand = nc;
  out->n_pieces = np;
  out->n_inc = ni;
  return RPD_OK;
}

extern "C" {

rpd_status rpd_sphere_volumes(rpd_ctx* c, double* out) {
  if (!c || !out) return fail(c, RPD_EINVAL, "rpd_sphere_volumes: bad argument");
  if (!c->have_pieces) return fail(c, RPD_ESTATE, "rpd_sphere_volumes before rpd_clip");
  CK(cudaSetDevice(c->device), "cudaSetDevice");
  const int64_t N = c->st.N;
  const bool host = is_host_ptr(out);
  double* d = out;
  if (host) {
    CK(c->g_dst.ensure(sizeof(double) * (N > 0 ? N : 1)), "alloc");
    d = c->g_dst.as<double>();
  }
  CK(launch_sphere_volumes(c, d), "sphere volumes");
  if (host) {
    CK(cudaMemcpyAsync(out, d, sizeof(double) * N, cudaMemcpyDeviceToHost, c->stream), "download");
    CK(cudaStreamSynchronize(c->stream), "download");
  }
  return RPD_OK;
}

rpd_status rpd_download_tets(rpd_ctx* c, const int32_t* tet_list, int64_t n,
                             const int32_t* id_map, int32_t* ids_out, rpd_csr* out) {
  if (!c) return RPD_EINVAL;
  if (!out || n < 0 || n > 0x7fffffff || (n > 0 && !tet_list))
    return fail(c, RPD_EINVAL, "rpd_download_tets: bad argument");
  if (!c->have_pieces) return fail(c, RPD_ESTATE, "rpd_download_tets before rpd_clip");
  CK(cudaSetDevice(c->device), "cudaSetDevice");
  const int32_t* d_list = nullptr;
  CK(resolve(c, tet_list, n, c->h_dl, &d_list), "stage tet list");
  if (ids_out && n > 0) {
    const int32_t* d_map = nullptr;
    CK(resolve(c, id_map, id_map ? c->st.T : 0, c->h_dm, &d_map), "stage id map");
    const bool host = is_host_ptr(ids_out);
    CK(c->g_ids.ensure(sizeof(int32_t) * n), "alloc");
    int32_t* dst = host ? c->g_ids.as<int32_t>() : ids_out;
    CK(launch_map_ids(c, d_list, n, d_map, c->st.T, dst), "ids");
    if (host)
      CK(cudaMemcpyAsync(ids_out, dst, sizeof(int32_t) * n, cudaMemcpyDefault, c->stream),
         "download ids");
  }
  return download_rows(c, 1, d_list, n, out);
}

rpd_status rpd_merge_shards(rpd_ctx* c, const rpd_shards* dirty, const rpd_csr* old,
                            rpd_csr* out) {
  if (!c) return RPD_EINVAL;
  if (!dirty || !old || !out || !shards_ok(dirty, true, true) || old->T != dirty->T ||
      !old->cand_off || !old->piece_off || !old->inc_off)
    return fail(c, RPD_EINVAL, "rpd_merge_shards: bad argument");
  CK(cudaSetDevice(c->device), "cudaSetDevice");
  const int64_t T = dirty->T;
  SegShards v;
  SegSources S{};
  S.s[0] = seg_src_csr(old->cand_off, old->cand_idx, old->piece_off, old->piece_sphere,
                       old->piece_vol, old->piece_m1, old->piece_facemask, old->inc_off,
                       old->inc_sphere);
  shard_sources(dirty, &v, &S, 1);
  // output: the ctx-owned buffer set that `old` does not live in
  int g = c->g_cur ^ 1;
  if (old->cand_off == c->g_cand[g].off.as<int32_t>()) g ^= 1;
  CandSet& cn = c->g_cand[g];
  PieceSet& pn = c->g_pcs[g];
  CK(cn.off.ensure(sizeof(int32_t) * (T + 1)), "alloc");
  CK(pn.off.ensure(sizeof(int32_t) * (T + 1)), "alloc");
  auto ensure = [&](int64_t nc, int64_t np, int64_t ni, SegDst* D) -> rpd_status {
    const size_t a = nc > 0 ? nc : 1, b = np > 0 ? np : 1, d = ni > 0 ? ni : 1;
    if (cn.idx.ensure(4 * a) || pn.sphere.ensure(4 * b) || pn.vol.ensure(8 * b) ||
        pn.m1.ensure(24 * b) || pn.fm.ensure(b) || pn.inc_off.ensure(4 * (np + 1)) ||
        pn.inc.ensure(4 * d))
      return fail(c, RPD_ENOMEM, "alloc");
    *D = SegDst{cn.off.as<int32_t>(),    cn.idx.as<int32_t>(),  pn.off.as<int32_t>(),
                pn.sphere.as<int32_t>(), pn.vol.as<double>(),   pn.m1.as<double>(),
                pn.fm.as<uint8_t>(),     pn.inc_off.as<int32_t>(), pn.inc.as<int32_t>(),
                nullptr};
    return RPD_OK;
  };
  SegDst D{cn.off.as<int32_t>(), nullptr, pn.off.as<int32_t>(), nullptr, nullptr, nullptr,
           nullptr, nullptr, nullptr, nullptr};
  int64_t nc = 0, np = 0, ni = 0;
  rpd_status s = seg_run(c, 2, T, nullptr, &v, T, S, D, &nc, &np, &ni, true, ensure);
  if (s) return s;
  c->g_cur = g;
  *out = rpd_csr{cn.off.as<int32_t>(),    cn.idx.as<int32_t>(), pn.off.as<int32_t>(),
                 pn.sphere.as<int32_t>(), pn.vol.as<double>(),  pn.m1.as<double>(),
                 pn.fm.as<uint8_t>(),     pn.inc_off.as<int32_t>(), pn.inc.as<int32_t>(),
                 T, nc, np, ni};
  return RPD_OK;
}

rpd_status rpd_envelope(rpd_ctx* c, const double* samples, int64_t S, const double* spheres,
                        int64_t N, const int32_t* edges, int64_t NE, const int32_t* faces,
                        int64_t NF, double* g_out, int32_t* prim_out, int64_t* n_eval) {
  if (!c) return RPD_EINVAL;
  if (S < 0 || N < 0 || NE < 0 || NF < 0 || S > 0x7fffffff || N + NE + NF > 0x7fffffff ||
      (S > 0 && (!samples || !g_out || !prim_out)) || (N > 0 && !spheres) ||
      (NE > 0 && !edges) || (NF > 0 && !faces) || (S > 0 && N + NE + NF == 0))
    return fail(c, RPD_EINVAL, "rpd_envelope: bad argument");
  CK(cudaSetDevice(c->device), "cudaSetDevice");
  const double *d_smp = nullptr, *d_sph = nullptr;
  const int32_t *d_e = nullptr, *d_f = nullptr;
  CK(resolve(c, samples, 3 * S, c->h_env, &d_smp), "stage samples");
  CK(resolve(c, spheres, 4 * N, c->h_env2, &d_sph), "stage spheres");
  CK(resolve(c, edges, 2 * NE, c->h_env3, &d_e), "stage edges");
  CK(resolve(c, faces, 3 * NF, c->h_env4, &d_f), "stage faces");
  const bool host_out = is_host_ptr(g_out) || is_host_ptr(prim_out);
  CK(c->env_out.ensure((sizeof(double) + sizeof(int32_t)) * (S + 1) + 16), "alloc");
  double* dg = host_out ? c->env_out.as<double>() : g_out;
  int32_t* dp = host_out ? reinterpret_cast<int32_t*>(c->env_out.as<double>() + (S + 1)) : prim_out;
  unsigned long long* ne = c->stats.as<unsigned long long>() + ST_ENV_EVAL;
  CK(cudaMemsetAsync(ne, 0, sizeof(unsigned long long), c->stream), "memset");
  if (NE + NF > 0) {  // sphere ids validated before any kernel dereferences them
    CK(cudaMemsetAsync(c->errw.p, 0, sizeof(int) * 4, c->stream), "memset");
    CK(launch_envelope_check(c, N, d_e, NE, d_f, NF), "envelope check");
    CK(readback(c, RbSpec{{}, nullptr, c->errw.as<int>()}), "readback");
    CK(cudaStreamSynchronize(c->stream), "envelope check");
    if (((Readback*)c->pinned)->err[0] != 0)
      return fail(c, RPD_EINVAL, "rpd_envelope: a cone / slab sphere id is out of range");
  }
  CK(launch_envelope(c, d_smp, S, d_sph, N, d_e, NE, d_f, NF, dg, dp, ne), "envelope");
  if (host_out && S > 0) {
    CK(cudaMemcpyAsync(g_out, dg, sizeof(double) * S, cudaMemcpyDefault, c->stream), "download");
    CK(cudaMemcpyAsync(prim_out, dp, sizeof(int32_t) * S, cudaMemcpyDefault, c->stream),
       "download");
  }
  unsigned long long h_ne = 0;
  CK(cudaMemcpyAsync(&h_ne, ne, sizeof(h_ne), cudaMemcpyDeviceToHost, c->stream), "download");
  CK(cudaStreamSynchronize(c->stream), "envelope");
  if (n_eval) *n_eval = (int64_t)h_ne;
  return RPD_OK;
}

rpd_status rpd_neighbors(rpd_ctx* c, const double* spheres, int64_t N, const double* box,
                         rpd_nbr_lists* out) {
  if (!c) return RPD_EINVAL;
  if (N < 0 || N > 0x3fffffff || (N > 0 && !spheres) || !box || !out)
    return fail(c, RPD_EINVAL, "rpd_neighbors: bad argument");
  for (int k = 0; k < 3; ++k)
    if (!std::isfinite(box[k]) || !std::isfinite(box[3 + k]) || !(box[k] <= box[3 + k]))
      return fail(c, RPD_EINVAL, "rpd_neighbors: box must be finite with lo <= hi");
  CK(cudaSetDevice(c->device), "cudaSetDevice");
  const double bx[6] = {box[0], box[1], box[2], box[3], box[4], box[5]};
  const double* d_sph = nullptr;
  CK(resolve(c, spheres, 4 * N, c->h_nb, &d_sph), "stage spheres");
  CK(c->nb_off.ensure(sizeof(int32_t) * (N + 1)), "alloc");
  CK(c->nb_cnt.ensure(sizeof(int32_t) * (N + 1)), "alloc");
  c->nb_N = -1;
  int32_t* off = c->nb_off.as<int32_t>();
  if (N == 0) {
    CK(cudaMemsetAsync(off, 0, sizeof(int32_t), c->stream), "memset");
    CK(cudaStreamSynchronize(c->stream), "neighbors");
    c->nb_N = 0;
    c->nb_E = 0;
    *out = rpd_nbr_lists{off, c->nb_idx.as<int32_t>(), 0, 0, 0, 0, 0};
    for (int k = 0; k < 6; ++k) c->nb_box[k] = bx[k];
    return RPD_OK;
  }
  CK(cudaMemsetAsync(c->errw.p, 0, sizeof(int) * 4, c->stream), "memset");
  const char* dbg_path = getenv("RPD_NB_DEBUG");  // development aid: per-sphere counters
  if (dbg_path) {
    if (c->nb_dbg) cudaFree(c->nb_dbg);
    c->nb_dbg = nullptr;
    CK(cudaMalloc(&c->nb_dbg, sizeof(long long) * 8 * N), "alloc");
    CK(cudaMemsetAsync(c->nb_dbg, 0, sizeof(long long) * 8 * N, c->stream), "memset");
  }
  CK(c->nb_ball.ensure(sizeof(double4) * 2 * N), "alloc");  // (for rpd_neighbors_update)
  CK(launch_neighbors_pass1(c, d_sph, N, bx, c->nb_cnt.as<int32_t>(), off), "neighbors");
  RbSpec rs{};
  rs.i32[0] = off + N;
  rs.i32[1] = c->nb_long;
  rs.err = c->errw.as<int>();
  CK(readback(c, rs), "readback");
  CK(cudaStreamSynchronize(c->stream), "neighbors");
  const Readback* rb = (const Readback*)c->pinned;
  if (rb->err[0] != 0) return check_err(c, rb);
  const int64_t E = rb->i32[0];
  if (dbg_path && c->nb_dbg) {
    std::vector<long long> h(8 * N);
    CK(cudaMemcpy(h.data(), c->nb_dbg, sizeof(long long) * 8 * N, cudaMemcpyDeviceToHost), "dbg");
    FILE* f = fopen(dbg_path, "wb");
    if (f) {
      fwrite(h.data(), sizeof(long long), h.size(), f);
      fclose(f);
    }
    cudaFree(c->nb_dbg);
    c->nb_dbg = nullptr;
  }
  CK(c->nb_idx.ensure(sizeof(int32_t) * (E + 1)), "alloc");
  CK(c->nb_tmp.ensure(sizeof(int32_t) * (E + 1)), "alloc");
  CK(launch_neighbors_pass2(c, d_sph, N, bx, c->nb_cnt.as<int32_t>(), off, c->nb_tmp.as<int32_t>(),
                            c->nb_idx.as<int32_t>()),
     "neighbors");
  unsigned long long h_st[4] = {0, 0, 0, 0};
  CK(cudaMemcpyAsync(h_st, c->nb_stats, sizeof(h_st), cudaMemcpyDeviceToHost, c->stream), "download");
  CK(cudaStreamSynchronize(c->stream), "neighbors");
  c->nb_N = N;
  c->nb_E = E;
  c->nb_rows = N;
  for (int k = 0; k < 6; ++k) c->nb_box[k] = bx[k];
  CK(c->nb_prev.ensure(sizeof(double) * 4 * N), "alloc");  // (for rpd_neighbors_update)
  CK(cudaMemcpyAsync(c->nb_prev.p, d_sph, sizeof(double) * 4 * N, cudaMemcpyDeviceToDevice,
                     c->stream), "copy");
  *out = rpd_nbr_lists{off, c->nb_idx.as<int32_t>(), N, E, (int64_t)h_st[1], (int64_t)h_st[0],
                       N, (int64_t)h_st[3]};
  return RPD_OK;
}

rpd_status rpd_neighbors_update(rpd_ctx* c, const double* spheres, int64_t N, int64_t M,
                                const double* box, rpd_nbr_lists* out) {
  if (!c) return RPD_EINVAL;
  if (N < 0 || N > 0x3fffffff || M < 0 || M > N || (N > 0 && !spheres) || !box || !out)
    return fail(c, RPD_EINVAL, "rpd_neighbors_update: bad argument");
  const int64_t N_old = N - M;
  if (c->nb_N < 0 || c->nb_N != N_old)
    return fail(c, RPD_ESTATE, "rpd_neighbors_update: no previous lists of N - M spheres");
  for (int k = 0; k < 6; ++k)
    if (!(box[k] == c->nb_box[k]))
      return fail(c, RPD_ESTATE, "rpd_neighbors_update: the box differs from the previous call's");
  CK(cudaSetDevice(c->device), "cudaSetDevice");
  if (M == 0) {  // the current lists
    c->nb_rows = 0;
    *out = rpd_nbr_lists{c->nb_off.as<int32_t>(), c->nb_idx.as<int32_t>(), N, c->nb_E, 0, 0, 0};
    return RPD_OK;
  }
  if (N_old == 0) return rpd_neighbors(c, spheres, N, box, out);
  const double bx[6] = {box[0], box[1], box[2], box[3], box[4], box[5]};
  const double* d_sph = nullptr;
  CK(resolve(c, spheres, 4 * N, c->h_nb, &d_sph), "stage spheres");
  // (2x on a reallocation: the sphere set grows a batch at a time)
  CK(c->nb_cnt.ensure_slack(sizeof(int32_t) * (N + 1), 2), "alloc");
  CK(c->nb_flag.ensure_slack(N, 2), "alloc");
  CK(c->nb_list.ensure_slack(sizeof(int32_t) * N, 2), "alloc");
  CK(c->nb_len.ensure_slack(sizeof(int32_t) * (N + 1), 2), "alloc");
  CK(c->nb_off2.ensure_slack(sizeof(int32_t) * (N + 1), 2), "alloc");
  CK(c->nb_misc.ensure(sizeof(int) * 8), "alloc");
  // the balls of the old rows, grown (with their content) for the new ones
  if (c->nb_ball.cap < sizeof(double4) * 2 * N) {  // (ball + vertex box per row)
    DevBuf nb;
    CK(nb.ensure(sizeof(double4) * 4 * N), "alloc");
    CK(cudaMemcpyAsync(nb.p, c->nb_ball.p, sizeof(double4) * 2 * N_old, cudaMemcpyDeviceToDevice,
                       c->stream), "copy");
    CK(cudaStreamSynchronize(c->stream), "copy");
    std::swap(c->nb_ball, nb);
    nb.release();
  }
  CK(cudaMemsetAsync(c->errw.p, 0, sizeof(int) * 4, c->stream), "memset");
  int32_t* off = c->nb_off2.as<int32_t>();
  int* misc = c->nb_misc.as<int>();
  int32_t* cnt = c->nb_cnt.as<int32_t>();
  uint8_t* flag = c->nb_flag.as<uint8_t>();
  const int32_t* o_off = c->nb_off.as<int32_t>();
  const int32_t* o_idx = c->nb_idx.as<int32_t>();
  CK(launch_nb_update1(c, d_sph, N, N_old, bx, c->nb_prev.as<double>(), cnt, flag,
                       c->nb_list.as<int32_t>(), c->nb_len.as<int32_t>(), o_off, off, misc),
     "neighbors update");
  RbSpec rs{};
  rs.i32[0] = off + N;
  rs.i32[1] = misc;
  rs.err = c->errw.as<int>();
  CK(readback(c, rs), "readback");
  CK(cudaStreamSynchronize(c->stream), "neighbors update");
  const Readback* rb = (const Readback*)c->pinned;
  if (rb->err[0] != 0) {
    c->nb_N = -1;  // (the grid scratch now describes the rejected spheres)
    return check_err(c, rb);
  }
  const int64_t E = rb->i32[0], n_rows = M + rb->i32[1];  // (new rows + changed old rows)
  CK(c->nb_idx2.ensure_slack(sizeof(int32_t) * (E + 1), 2), "alloc");
  CK(c->nb_tmp.ensure_slack(sizeof(int32_t) * (E + 1), 2), "alloc");
  CK(launch_nb_update2(c, d_sph, N, N_old, bx, cnt, c->nb_len.as<int32_t>(), o_off, o_idx, off,
                       c->nb_tmp.as<int32_t>(), c->nb_idx2.as<int32_t>()),
     "neighbors update");
  unsigned long long h_st[4] = {0, 0, 0, 0};
  CK(cudaMemcpyAsync(h_st, c->nb_stats, sizeof(h_st), cudaMemcpyDeviceToHost, c->stream), "download");
  CK(c->nb_prev.ensure_slack(sizeof(double) * 4 * N, 2), "alloc");  // (all old spheres were checked)
  CK(cudaMemcpyAsync(c->nb_prev.p, d_sph, sizeof(double) * 4 * N, cudaMemcpyDeviceToDevice,
                     c->stream), "copy");
  CK(cudaStreamSynchronize(c->stream), "neighbors update");
  std::swap(c->nb_off, c->nb_off2);
  std::swap(c->nb_idx, c->nb_idx2);
  c->nb_N = N;
  c->nb_E = E;
  c->nb_rows = n_rows;
  *out = rpd_nbr_lists{c->nb_off.as<int32_t>(), c->nb_idx.as<int32_t>(), N, E, (int64_t)h_st[1],
                       (int64_t)h_st[0], n_rows, (int64_t)h_st[3]};
  return RPD_OK;
}

rpd_status rpd_download_neighbors(rpd_ctx* c, int32_t* nbr_off, int32_t* nbr_idx) {
  if (!c) return RPD_EINVAL;
  if (c->nb_N < 0) return fail(c, RPD_ESTATE, "no neighbour lists (call rpd_neighbors)");
  if (nbr_off)
    CK(cudaMemcpyAsync(nbr_off, c->nb_off.p, sizeof(int32_t) * (c->nb_N + 1), cudaMemcpyDefault,
                       c->stream), "download");
  if (nbr_idx && c->nb_E)
    CK(cudaMemcpyAsync(nbr_idx, c->nb_idx.p, sizeof(int32_t) * c->nb_E, cudaMemcpyDefault,
                       c->stream), "download");
  CK(cudaStreamSynchronize(c->stream), "download");
  return RPD_OK;
}

rpd_status rpd_download_cands(rpd_ctx* c, int32_t* cand_off, int32_t* cand_idx) {
  if (!c) return RPD_EINVAL;
  if (!c->have_rel) return fail(c, RPD_ESTATE, "no candidates");
  if (!c->compact) {
    if (!cand_off) return fail(c, RPD_EINVAL, "rpd_download_cands: cand_off is needed");
    CK(cudaSetDevice(c->device), "cudaSetDevice");
    rpd_csr o{cand_off, cand_idx, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr,
              nullptr, 0, 0, 0, 0};
    return download_rows(c, 0, nullptr, c->st.T, &o);
  }
  const CandSet& cs = c->cand[c->cur];
  if (cand_off)
    CK(cudaMemcpyAsync(cand_off, cs.off.p, sizeof(int32_t) * (c->st.T + 1),
                       cudaMemcpyDefault, c->stream), "download");
  if (cand_idx && cs.n > 0)
    CK(cudaMemcpyAsync(cand_idx, cs.idx.p, sizeof(int32_t) * cs.n, cudaMemcpyDefault,
                       c->stream), "download");
  if (is_host_ptr(cand_off) || is_host_ptr(cand_idx))
    CK(cudaStreamSynchronize(c->stream), "download");
  return RPD_OK;
}

rpd_status rpd_debug_check(rpd_ctx* c) {
  if (!c) return RPD_EINVAL;
  if (!canary_on()) return RPD_OK;
  CK(cudaSetDevice(c->device), "cudaSetDevice");
  CK(cudaDeviceSynchronize(), "debug check");
  std::vector<const unsigned char*> tails;
  std::vector<size_t> caps;
  {
    std::lock_guard<std::mutex> g(canary_mu());
    for (DevBuf* b : canary_set())
      if (b->p) {
        tails.push_back(static_cast<const unsigned char*>(b->p) + b->cap);
        caps.push_back(b->cap);
      }
  }
  if (tails.empty()) return RPD_OK;
  const unsigned char** d_tails = nullptr;
  int* d_bad = nullptr;
  CK(cudaMalloc(&d_tails, sizeof(void*) * tails.size()), "debug check");
  CK(cudaMalloc(&d_bad, sizeof(int)), "debug check");
  CK(cudaMemcpy(d_tails, tails.data(), sizeof(void*) * tails.size(), cudaMemcpyHostToDevice),
     "debug check");
  CK(cudaMemset(d_bad, 0xff, sizeof(int)), "debug check");
  k_canary<<<256, 256>>>(d_tails, (int)tails.size(), d_bad);
  int bad = -1;
  cudaError_t e = cudaMemcpy(&bad, d_bad, sizeof(int), cudaMemcpyDeviceToHost);
  cudaFree(d_tails);
  cudaFree(d_bad);
  CK(e, "debug check");
  if (bad >= 0)
    return fail(c, RPD_ECUDA, "debug check: a write past the end of a " +
                                  std::to_string(caps[bad]) + "-byte library buffer");
  return RPD_OK;
}

rpd_status rpd_get_stats(rpd_ctx* c, rpd_stats* out) {
  if (!c || !out) return RPD_EINVAL;
  *out = c->last;
  out->kernel_launches = c->launches;
  out->graph_updates = c->g_launches;
  out->graph_captures = c->g_captures;
  out->graph_fallbacks = c->g_fallbacks;
  return RPD_OK;
}

}  // extern "C"
