// rpd_ctx.h -- host-side context of librpd and the kernel launchers (CUDA path only).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <string>

#include "../../include/rpd.h"

namespace rpd {

// Growable ctx-owned device buffer.
struct DevBuf {
  void* p = nullptr;
  size_t cap = 0;
  cudaError_t ensure(size_t bytes) {
    if (bytes <= cap && p) return cudaSuccess;
    if (p) cudaFree(p);
    p = nullptr;
    cap = 0;
    size_t want = bytes < 256 ? 256 : bytes + bytes / 8;
    cudaError_t e = cudaMalloc(&p, want);
    if (e == cudaSuccess) cap = want;
    return e;
  }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    cap = 0;
  }
  template <class T>
  T* as() const { return reinterpret_cast<T*>(p); }
};

// device error word layout (int32[4]): [0] status (0 ok, else rpd_status), [1] kind,
// [2] index of the offending element, [3] unused
enum ErrKind {
  ERR_NONE = 0,
  ERR_VERT_LATTICE = 1,
  ERR_VERT_NAN = 2,
  ERR_SPHERE_LATTICE = 3,
  ERR_SPHERE_NAN = 4,
  ERR_RADIUS_NEG = 5,
  ERR_TET_INDEX = 6,
  ERR_TET_ORIENT = 7,
  ERR_NBR_INDEX = 8,
  ERR_NBR_SELF = 9,
  ERR_NBR_DUP = 10,
  ERR_NBR_SAME_CENTRE = 11,
  ERR_NBR_OFF = 12
};

// device statistics (uint64 counters)
enum StatIdx {
  ST_EXACT = 0,      // clip predicates decided by the exact path
  ST_ZERO = 1,       // exact-zero predicates (SoS)
  ST_MAXV = 2,       // max vertices of a piece
  ST_MAXP = 3,       // max planes of a piece
  ST_OVERFLOW = 4,   // pieces that exceeded RPD_MAXV / RPD_MAXP / RPD_INC_CAP
  ST_MAXK = 5,       // max k_tet of the last filter
  ST_TESTED = 6,     // pairs evaluated by Alg. 1 (pruned mode)
  ST_N = 8
};

struct Stage {
  // tet coordinates, SoA lattice units: tx[(3k + c) * T + t]
  DevBuf tx;
  DevBuf sw;       // double4 per sphere: (X, Y, Z, W = |Theta|^2 - R^2), lattice units
  DevBuf nbr_off;  // int32 [N+1]
  DevBuf nbr_idx;  // int32 [E], rows sorted ascending
  DevBuf planes;   // double4 per CSR entry: (n, d) of h_ij
  DevBuf twin;     // int32 per CSR entry: next entry of the row with the same oriented plane
  int64_t T = 0, N = 0, V = 0, E = 0;
};

}  // namespace rpd

struct rpd_ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  int filter_mode = RPD_FILTER_ALL_PAIRS;
  int validate = 1;
  std::string err;
  int64_t launches = 0;

  // host-input staging (used when an argument is a host pointer)
  rpd::DevBuf h_verts, h_tets, h_spheres, h_off, h_idx, h_new;

  rpd::Stage st;
  rpd::DevBuf verts_lat;   // unused placeholder for future
  rpd::DevBuf tets;        // int32 [T][4] copy (for partial updates)
  rpd::DevBuf errw;        // int32[4]
  rpd::DevBuf stats;       // uint64[ST_N]
  rpd::DevBuf scratch;     // scan block sums

  // relations
  rpd::DevBuf k_tet, slab, cand_off, cand_idx, pair_tet;
  int slab_cap = 32;
  int64_t n_cand = 0;
  bool have_rel = false;

  // clip per-pair
  rpd::DevBuf k_words, w_off;            // incidence-mask words per tet and their offsets
  rpd::DevBuf p_flag, p_f01, p_vol, p_m1, p_fm, p_ninc, p_words, p_moff, p_mask, p_over;
  rpd::DevBuf p_scan, i_scan;
  int64_t n_mask_words = 0;
  int clip_wide = 0;                     // testing: run every pair through the wide kernel
  // pieces
  rpd::DevBuf piece_off, piece_sphere, piece_vol, piece_m1, piece_fm, inc_off, inc_sphere;
  int64_t n_pieces = 0, n_inc = 0;
  bool have_pieces = false;

  // partial update
  rpd::DevBuf dirty_flag, dirty_list, dirty_scan;
  int64_t n_dirty = 0;

  rpd_stats last{};
  void* pinned = nullptr;  // small pinned host buffer for scalar readbacks
};

namespace rpd {

// launchers (all on ctx->stream; each increments ctx->launches)
cudaError_t launch_stage(rpd_ctx* c, const double* verts, int64_t V, const int32_t* tets,
                         int64_t T, const double* spheres, int64_t N, const int32_t* nbr_off,
                         const int32_t* nbr_idx, int64_t E);
cudaError_t launch_scan_i32(rpd_ctx* c, const int32_t* in, int32_t* out, int64_t n);
cudaError_t launch_scan_u8(rpd_ctx* c, const uint8_t* in, int32_t* out, int64_t n);
cudaError_t launch_filter(rpd_ctx* c, const int32_t* tet_ids, int64_t n_tets, int cap,
                          int sphere_lo, int sphere_hi, int32_t* k_tet, int32_t* slab,
                          int32_t* k_words);
cudaError_t launch_compact_cands(rpd_ctx* c, int64_t T, int cap, const int32_t* k_tet,
                                 const int32_t* slab, const int32_t* cand_off,
                                 int32_t* cand_idx, int32_t* pair_tet, const int32_t* w_off,
                                 int32_t* p_moff, int64_t n_pairs);
cudaError_t launch_clip(rpd_ctx* c, int64_t n_pairs, const int32_t* pair_tet,
                        const int32_t* tet_ids, const int32_t* cand_idx, int wide);
cudaError_t launch_clip_overflow(rpd_ctx* c, const int32_t* pair_tet, const int32_t* tet_ids,
                                 const int32_t* cand_idx);
cudaError_t launch_piece_scans(rpd_ctx* c, int64_t n_pairs);
// destination of a piece compaction
struct PieceDst {
  int32_t* off;      // [n_tets+1]
  int32_t* sphere;
  double* vol;
  double* m1;
  uint8_t* fm;
  int32_t* inc_off;  // [n_pieces+1]
  int32_t* inc;
};
cudaError_t launch_compact_pieces(rpd_ctx* c, int64_t n_tets, int64_t n_pairs,
                                  const int32_t* cand_off, const int32_t* cand_idx,
                                  const PieceDst& d);

}  // namespace rpd
