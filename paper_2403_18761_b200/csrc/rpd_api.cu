// rpd_api.cu -- the C ABI of librpd (include/rpd.h).  Host-side orchestration only: every
// step of the path runs in the kernels of rpd_stage.cu, rpd_filter.cu, rpd_scan.cu,
// rpd_clip.cu and rpd_partial.cu.
#include <stdio.h>
#include <string.h>

#include <string>
#include <vector>

#include "rpd_ctx.h"
#include "rpd_internal.cuh"

using namespace rpd;

#define RPD_VERSION "rpd-b200 0.1 (sm_100a)"

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
    default: return "invalid input";
  }
}

// read k int32/int64 device scalars into the pinned buffer and synchronise
struct Readback {
  int32_t i32[8];
  unsigned long long u64[ST_N];
  int32_t err[4];
};

rpd_status check_err(rpd_ctx* c, const Readback* rb) {
  if (rb->err[0] != 0) {
    char buf[256];
    snprintf(buf, sizeof buf, "%s (element %d)", err_kind_str(rb->err[1]), rb->err[2]);
    return fail(c, (rpd_status)rb->err[0], buf);
  }
  return RPD_OK;
}

}  // namespace

extern "C" {

const char* rpd_version(void) { return RPD_VERSION; }

rpd_status rpd_create(rpd_ctx** out, int device, void* cuda_stream) {
  if (!out) return RPD_EINVAL;
  *out = nullptr;
  rpd_ctx* c = new rpd_ctx();
  c->device = device;
  cudaError_t e = cudaSetDevice(device);
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
      cudaMallocHost(&c->pinned, sizeof(Readback))) {
    rpd_destroy(c);
    return RPD_ENOMEM;
  }
  *out = c;
  return RPD_OK;
}

void rpd_destroy(rpd_ctx* c) {
  if (!c) return;
  cudaSetDevice(c->device);
  if (c->stream) cudaStreamSynchronize(c->stream);
  DevBuf* bufs[] = {&c->h_verts, &c->h_tets, &c->h_spheres, &c->h_off, &c->h_idx, &c->h_new,
                    &c->st.tx, &c->st.sw, &c->st.nbr_off, &c->st.nbr_idx, &c->st.planes,
                    &c->st.twin, &c->verts_lat, &c->tets, &c->errw, &c->stats, &c->scratch,
                    &c->k_tet, &c->slab, &c->cand_off, &c->cand_idx, &c->pair_tet, &c->p_flag,
                    &c->p_vol, &c->p_m1, &c->p_fm, &c->p_ninc, &c->p_f01, &c->p_words,
                    &c->p_moff, &c->p_mask, &c->p_over, &c->k_words, &c->w_off, &c->p_scan,
                    &c->i_scan, &c->piece_off, &c->piece_sphere, &c->piece_vol, &c->piece_m1,
                    &c->piece_fm, &c->inc_off, &c->inc_sphere, &c->dirty_flag, &c->dirty_list,
                    &c->dirty_scan};
  for (DevBuf* b : bufs) b->release();
  if (c->pinned) cudaFreeHost(c->pinned);
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
    case RPD_OPT_CLIP_WIDE:
      c->clip_wide = value ? 1 : 0;
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

rpd_status rpd_relations(rpd_ctx* c, const double* verts, int64_t V, const int32_t* tets,
                         int64_t T, const double* spheres, int64_t N, const int32_t* nbr_off,
                         const int32_t* nbr_idx, const int32_t** cand_off,
                         const int32_t** cand_idx, int64_t* n_cand) {
  if (!c) return RPD_EINVAL;
  if (V < 0 || T < 0 || N < 0 || T > 0x7fffffff || N > 0x7fffffff || (T > 0 && !tets) ||
      (V > 0 && !verts) || (N > 0 && (!spheres || !nbr_off)) || !cand_off || !cand_idx ||
      !n_cand)
    return fail(c, RPD_EINVAL, "rpd_relations: bad argument");
  CK(cudaSetDevice(c->device), "cudaSetDevice");
  c->have_rel = false;
  c->have_pieces = false;
  Readback* rb = (Readback*)c->pinned;

  // neighbour count E = nbr_off[N]
  int64_t E = 0;
  const int32_t* d_off = nullptr;
  if (N > 0) {
    if (is_host_ptr(nbr_off)) {
      E = nbr_off[N];
    } else {
      CK(cudaMemcpyAsync(&rb->i32[0], nbr_off + N, sizeof(int32_t), cudaMemcpyDeviceToHost,
                         c->stream), "read nbr_off[N]");
      CK(cudaStreamSynchronize(c->stream), "sync");
      E = rb->i32[0];
    }
    if (E < 0) return fail(c, RPD_EINVAL, "nbr_off[N] < 0");
    if (E > 0 && !nbr_idx) return fail(c, RPD_EINVAL, "nbr_idx is NULL");
  }
  const double *d_verts = nullptr, *d_sph = nullptr;
  const int32_t *d_tets = nullptr, *d_idx = nullptr;
  CK(resolve(c, verts, 3 * V, c->h_verts, &d_verts), "stage verts");
  CK(resolve(c, tets, 4 * T, c->h_tets, &d_tets), "stage tets");
  CK(resolve(c, spheres, 4 * N, c->h_spheres, &d_sph), "stage spheres");
  CK(resolve(c, nbr_off, N > 0 ? N + 1 : 0, c->h_off, &d_off), "stage nbr_off");
  CK(resolve(c, nbr_idx, E, c->h_idx, &d_idx), "stage nbr_idx");

  CK(cudaMemsetAsync(c->errw.p, 0, sizeof(int) * 4, c->stream), "memset");
  CK(cudaMemsetAsync(c->stats.p, 0, sizeof(unsigned long long) * ST_N, c->stream), "memset");
  CK(launch_stage(c, d_verts, V, d_tets, T, d_sph, N, d_off, d_idx, E), "stage");
  // keep a copy of the tets for later partial updates
  CK(c->tets.ensure(sizeof(int32_t) * 4 * (T > 0 ? T : 1)), "alloc");
  if (T > 0)
    CK(cudaMemcpyAsync(c->tets.p, d_tets, sizeof(int32_t) * 4 * T, cudaMemcpyDeviceToDevice,
                       c->stream), "copy tets");

  CK(c->k_tet.ensure(sizeof(int32_t) * (T > 0 ? T : 1)), "alloc");
  CK(c->k_words.ensure(sizeof(int32_t) * (T > 0 ? T : 1)), "alloc");
  CK(c->cand_off.ensure(sizeof(int32_t) * (T + 1)), "alloc");
  CK(c->w_off.ensure(sizeof(int32_t) * (T + 1)), "alloc");
  for (int attempt = 0; attempt < 2; ++attempt) {
    int cap = c->slab_cap;
    CK(c->slab.ensure(sizeof(int32_t) * (size_t)cap * (T > 0 ? T : 1)), "alloc slab");
    CK(launch_filter(c, nullptr, T, cap, 0, (int)N, c->k_tet.as<int32_t>(),
                     c->slab.as<int32_t>(), c->k_words.as<int32_t>()), "filter");
    CK(launch_scan_i32(c, c->k_tet.as<int32_t>(), c->cand_off.as<int32_t>(), T), "scan");
    CK(launch_scan_i32(c, c->k_words.as<int32_t>(), c->w_off.as<int32_t>(), T), "scan");
    CK(cudaMemcpyAsync(&rb->i32[0], c->cand_off.as<int32_t>() + T, sizeof(int32_t),
                       cudaMemcpyDeviceToHost, c->stream), "readback");
    CK(cudaMemcpyAsync(&rb->i32[1], c->w_off.as<int32_t>() + T, sizeof(int32_t),
                       cudaMemcpyDeviceToHost, c->stream), "readback");
    CK(cudaMemcpyAsync(rb->u64, c->stats.p, sizeof(unsigned long long) * ST_N,
                       cudaMemcpyDeviceToHost, c->stream), "readback");
    CK(cudaMemcpyAsync(rb->err, c->errw.p, sizeof(int) * 4, cudaMemcpyDeviceToHost, c->stream),
       "readback");
    CK(cudaStreamSynchronize(c->stream), "relations");
    rpd_status s = check_err(c, rb);
    if (s) return s;
    int maxk = (int)rb->u64[ST_MAXK];
    if (maxk <= cap) break;
    int nc = 32;
    while (nc < maxk) nc *= 2;
    c->slab_cap = nc;
  }
  int64_t nc = rb->i32[0];
  c->n_mask_words = rb->i32[1];
  CK(c->cand_idx.ensure(sizeof(int32_t) * (nc > 0 ? nc : 1)), "alloc");
  CK(c->pair_tet.ensure(sizeof(int32_t) * (nc > 0 ? nc : 1)), "alloc");
  CK(c->p_moff.ensure(sizeof(int32_t) * (nc + 1)), "alloc");
  CK(launch_compact_cands(c, T, c->slab_cap, c->k_tet.as<int32_t>(), c->slab.as<int32_t>(),
                          c->cand_off.as<int32_t>(), c->cand_idx.as<int32_t>(),
                          c->pair_tet.as<int32_t>(), c->w_off.as<int32_t>(),
                          c->p_moff.as<int32_t>(), nc), "compact");
  c->n_cand = nc;
  c->have_rel = true;
  c->last = rpd_stats{};
  c->last.T = T;
  c->last.N = N;
  c->last.n_cand = nc;
  c->last.pairs_filtered = T * N;
  c->last.pairs_tested = T * N;
  c->last.max_k_tet = (int32_t)rb->u64[ST_MAXK];
  *cand_off = c->cand_off.as<int32_t>();
  *cand_idx = c->cand_idx.as<int32_t>();
  *n_cand = nc;
  return RPD_OK;
}

static rpd_status fill_pieces(rpd_ctx* c, rpd_pieces* out) {
  out->piece_off = c->piece_off.as<int32_t>();
  out->piece_sphere = c->piece_sphere.as<int32_t>();
  out->piece_vol = c->piece_vol.as<double>();
  out->piece_m1 = c->piece_m1.as<double>();
  out->piece_facemask = c->piece_fm.as<uint8_t>();
  out->inc_off = c->inc_off.as<int32_t>();
  out->inc_sphere = c->inc_sphere.as<int32_t>();
  out->n_pieces = c->n_pieces;
  out->n_inc = c->n_inc;
  return RPD_OK;
}

rpd_status rpd_clip(rpd_ctx* c, rpd_pieces* out) {
  if (!c || !out) return fail(c, RPD_EINVAL, "rpd_clip: bad argument");
  if (!c->have_rel) return fail(c, RPD_ESTATE, "rpd_clip before rpd_relations");
  CK(cudaSetDevice(c->device), "cudaSetDevice");
  const int64_t n = c->n_cand, T = c->st.T;
  size_t nn = n > 0 ? n : 1;
  CK(c->p_flag.ensure(nn), "alloc");
  CK(c->p_f01.ensure(nn), "alloc");
  CK(c->p_fm.ensure(nn), "alloc");
  CK(c->p_vol.ensure(sizeof(double) * nn), "alloc");
  CK(c->p_m1.ensure(sizeof(double) * 3 * nn), "alloc");
  CK(c->p_ninc.ensure(sizeof(int32_t) * nn), "alloc");
  CK(c->p_over.ensure(sizeof(int32_t) * (n + 1)), "alloc");
  CK(c->p_mask.ensure(sizeof(unsigned) * (c->n_mask_words > 0 ? c->n_mask_words : 1)), "alloc");
  CK(c->p_scan.ensure(sizeof(int32_t) * (n + 1)), "alloc");
  CK(c->i_scan.ensure(sizeof(int32_t) * (n + 1)), "alloc");
  CK(cudaMemsetAsync(c->p_mask.p, 0, sizeof(unsigned) * c->n_mask_words, c->stream), "memset");
  CK(cudaMemsetAsync(c->p_over.p, 0, sizeof(int32_t), c->stream), "memset");
  CK(launch_clip(c, n, c->pair_tet.as<int32_t>(), nullptr, c->cand_idx.as<int32_t>(),
                 c->clip_wide), "clip");
  if (!c->clip_wide && n > 0)
    CK(launch_clip_overflow(c, c->pair_tet.as<int32_t>(), nullptr, c->cand_idx.as<int32_t>()),
       "clip (wide)");
  CK(launch_piece_scans(c, n), "scan");
  Readback* rb = (Readback*)c->pinned;
  CK(cudaMemcpyAsync(&rb->i32[0], c->p_scan.as<int32_t>() + n, sizeof(int32_t),
                     cudaMemcpyDeviceToHost, c->stream), "readback");
  CK(cudaMemcpyAsync(&rb->i32[1], c->i_scan.as<int32_t>() + n, sizeof(int32_t),
                     cudaMemcpyDeviceToHost, c->stream), "readback");
  CK(cudaMemcpyAsync(&rb->i32[2], c->p_over.p, sizeof(int32_t), cudaMemcpyDeviceToHost,
                     c->stream), "readback");
  CK(cudaMemcpyAsync(rb->u64, c->stats.p, sizeof(unsigned long long) * ST_N,
                     cudaMemcpyDeviceToHost, c->stream), "readback");
  CK(cudaStreamSynchronize(c->stream), "clip");
  if (rb->u64[ST_OVERFLOW])
    return fail(c, RPD_EOVERFLOW, "a piece exceeded the wide clip capacity (128 vertices/planes)");
  int64_t np = rb->i32[0], ni = rb->i32[1];
  size_t npp = np > 0 ? np : 1;
  CK(c->piece_off.ensure(sizeof(int32_t) * (T + 1)), "alloc");
  CK(c->piece_sphere.ensure(sizeof(int32_t) * npp), "alloc");
  CK(c->piece_vol.ensure(sizeof(double) * npp), "alloc");
  CK(c->piece_m1.ensure(sizeof(double) * 3 * npp), "alloc");
  CK(c->piece_fm.ensure(npp), "alloc");
  CK(c->inc_off.ensure(sizeof(int32_t) * (np + 1)), "alloc");
  CK(c->inc_sphere.ensure(sizeof(int32_t) * (ni > 0 ? ni : 1)), "alloc");
  PieceDst d{c->piece_off.as<int32_t>(), c->piece_sphere.as<int32_t>(), c->piece_vol.as<double>(),
             c->piece_m1.as<double>(), c->piece_fm.as<uint8_t>(), c->inc_off.as<int32_t>(),
             c->inc_sphere.as<int32_t>()};
  CK(launch_compact_pieces(c, T, n, c->cand_off.as<int32_t>(), c->cand_idx.as<int32_t>(), d),
     "compact pieces");
  c->n_pieces = np;
  c->n_inc = ni;
  c->have_pieces = true;
  c->last.n_pieces = np;
  c->last.n_inc = ni;
  c->last.exact_fallbacks = (int64_t)rb->u64[ST_EXACT];
  c->last.zero_hits = (int64_t)rb->u64[ST_ZERO];
  c->last.max_vertices = (int32_t)rb->u64[ST_MAXV];
  c->last.max_planes = (int32_t)rb->u64[ST_MAXP];
  c->last.n_wide = rb->i32[2];
  return fill_pieces(c, out);
}

rpd_status rpd_update_partial(rpd_ctx* c, const double* spheres, int64_t N_new,
                              const int32_t* nbr_off, const int32_t* nbr_idx,
                              const int32_t* new_ids, int64_t M, rpd_pieces* out,
                              const int32_t** dirty_tets, int64_t* n_dirty) {
  (void)spheres;
  (void)N_new;
  (void)nbr_off;
  (void)nbr_idx;
  (void)new_ids;
  (void)M;
  (void)out;
  (void)dirty_tets;
  (void)n_dirty;
  return fail(c, RPD_ESTATE, "rpd_update_partial: not built yet");
}

rpd_status rpd_download_pieces(rpd_ctx* c, int32_t* piece_off, int32_t* piece_sphere,
                               double* piece_vol, double* piece_m1, uint8_t* piece_facemask,
                               int32_t* inc_off, int32_t* inc_sphere) {
  if (!c) return RPD_EINVAL;
  if (!c->have_pieces) return fail(c, RPD_ESTATE, "no pieces");
  const int64_t T = c->st.T, np = c->n_pieces, ni = c->n_inc;
  auto cp = [&](void* dst, const void* src, size_t bytes) -> cudaError_t {
    if (!dst || bytes == 0) return cudaSuccess;
    return cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDefault, c->stream);
  };
  CK(cp(piece_off, c->piece_off.p, sizeof(int32_t) * (T + 1)), "download");
  CK(cp(piece_sphere, c->piece_sphere.p, sizeof(int32_t) * np), "download");
  CK(cp(piece_vol, c->piece_vol.p, sizeof(double) * np), "download");
  CK(cp(piece_m1, c->piece_m1.p, sizeof(double) * 3 * np), "download");
  CK(cp(piece_facemask, c->piece_fm.p, np), "download");
  CK(cp(inc_off, c->inc_off.p, sizeof(int32_t) * (np + 1)), "download");
  CK(cp(inc_sphere, c->inc_sphere.p, sizeof(int32_t) * ni), "download");
  CK(cudaStreamSynchronize(c->stream), "download");
  return RPD_OK;
}

rpd_status rpd_download_cands(rpd_ctx* c, int32_t* cand_off, int32_t* cand_idx) {
  if (!c) return RPD_EINVAL;
  if (!c->have_rel) return fail(c, RPD_ESTATE, "no candidates");
  if (cand_off)
    CK(cudaMemcpyAsync(cand_off, c->cand_off.p, sizeof(int32_t) * (c->st.T + 1),
                       cudaMemcpyDefault, c->stream), "download");
  if (cand_idx && c->n_cand > 0)
    CK(cudaMemcpyAsync(cand_idx, c->cand_idx.p, sizeof(int32_t) * c->n_cand,
                       cudaMemcpyDefault, c->stream), "download");
  CK(cudaStreamSynchronize(c->stream), "download");
  return RPD_OK;
}

rpd_status rpd_get_stats(rpd_ctx* c, rpd_stats* out) {
  if (!c || !out) return RPD_EINVAL;
  *out = c->last;
  out->kernel_launches = c->launches;
  return RPD_OK;
}

}  // extern "C"
