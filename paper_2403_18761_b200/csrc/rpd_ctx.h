// rpd_ctx.h -- host-side context of librpd and the kernel launchers (CUDA path only).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <string>

#include "../../include/rpd.h"

#define RPD_MAX_DEVICES 64

namespace rpd {

// Debug builds of the test runs (env RPD_CANARY=1; a stand-in for compute-sanitizer, which is
// closed on this GPU pool): every buffer gets a 256-byte canary past its capacity, and
// rpd_debug_check verifies all live canaries (a write past the end of any ctx buffer).
constexpr size_t CANARY_BYTES = 256;
bool canary_on();
struct DevBuf;
void canary_register(DevBuf* b);
void canary_unregister(DevBuf* b);

// Growable ctx-owned device buffer.
struct DevBuf {
  void* p = nullptr;
  size_t cap = 0;
  DevBuf() = default;
  DevBuf(const DevBuf&) = default;
  DevBuf& operator=(const DevBuf&) = default;
  ~DevBuf() {
    if (canary_on()) canary_unregister(this);
  }
  cudaError_t ensure(size_t bytes) {
    if (bytes <= cap && p) return cudaSuccess;
    if (p) cudaFree(p);
    p = nullptr;
    cap = 0;
    size_t want = bytes < 256 ? 256 : bytes + bytes / 8;
    const bool can = canary_on();
    cudaError_t e = cudaMalloc(&p, want + (can ? CANARY_BYTES : 0));
    if (e == cudaSuccess) {
      cap = want;
      if (can) {  // (debug only: synchronous)
        e = cudaMemset(static_cast<char*>(p) + want, 0xA5, CANARY_BYTES);
        if (!e) e = cudaDeviceSynchronize();
        canary_register(this);
      }
    }
    return e;
  }
  // like ensure, but a (re)allocation reserves `factor` x bytes (pools that grow by appends)
  cudaError_t ensure_slack(size_t bytes, int factor) {
    if (bytes <= cap && p) return cudaSuccess;
    return ensure(bytes * factor);
  }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    cap = 0;
    if (canary_on()) canary_unregister(this);
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
  ERR_NBR_OFF = 12,
  ERR_SPHERE_CHANGED = 13,
  ERR_NB_RECOMPUTE = 14  // neighbour pass 2 found another row length than pass 1 (unreachable)
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
  ST_REL_TESTS = 7,  // literal Alg. 1 vertex tests (inner break, outer early exit)
  ST_CLIP_PLANES = 8,   // (pair, plane) corner classifications in the clip
  ST_CLIP_TESTS = 9,    // vertex sign tests in the clip
  ST_CLIP_CONSTR = 10,  // vertex constructions
  ST_CLIP_FAN = 11,     // fan triangles of the volume/moment integration
  ST_EU_OVER = 15,      // pieces with more than 64 radical facets (topology mode)
  ST_ENV_EVAL = 16,     // envelope distance: (sample, primitive) evaluations
  ST_N = 17
};

struct Stage {
  // tet coordinates, SoA lattice units: tx[(3k + c) * T + t]
  DevBuf tx;
  DevBuf sw;       // double4 per sphere: (X, Y, Z, W = |Theta|^2 - R^2), lattice units
  DevBuf nbr_off;  // int32 [N+1]
  DevBuf nbr_idx;  // int32 [E], rows sorted ascending
  DevBuf planes;   // double4 per CSR entry: (n, d) of h_ij
  DevBuf twin;     // int32 per CSR entry: next entry of the row with the same oriented plane
  DevBuf hkey;     // uint64 per CSR entry: hash of the canonical plane (twin search)
  DevBuf repoch;   // int32 per sphere: epoch (update index) at which its row was last built
  DevBuf htab;     // uint64 scratch: per-row hash tables of the twin search
  // the previous rows (partial updates copy the rows whose neighbour list is unchanged)
  DevBuf old_off, old_idx, old_planes, old_twin, old_hkey, old_repoch, old_sw;
  int64_t T = 0, N = 0, V = 0, E = 0;
  int64_t N_prev = 0;  // N of the previous staging (the old rows)
  DevBuf long_rows;    // partial updates: the long rows deferred to k_stage_long (+ count)
};

}  // namespace rpd

namespace rpd {
// Candidate set over a list of tets.  As the ctx STATE (cand[cur]) it is a pool: tet t's
// candidates are idx[rows[t].x, rows[t].y); after rpd_relations the pool is compact (rows ==
// the CSR off) and a partial update appends the dirty tets' new lists at the pool's tail and
// re-points their rows (clean tets are never copied).  As a batch (cand_d: the dirty tets of an
// update) it is a CSR over the batch whose idx may live in the state pool (idx_ext).
struct CandSet {
  DevBuf off;       // int32 [n_tets+1]  CSR offsets (compact pool / batch)
  DevBuf idx;       // int32 [fill]  candidate sphere ids, ascending per tet
  DevBuf pair_tet;  // int32 [n]   local tet index of every pair (compact pool / batch)
  DevBuf moff;      // int32 [n+1] incidence-mask word offsets of every pair (compact / batch)
  DevBuf rows;      // int2 [n_tets]  state: [beg, end) of every tet's candidates in idx
  DevBuf cut;       // uint32 [n_words] per pair, incidence-mask layout: the planes of N(i)
                    // that are not positive at all 4 corners (the only ones that can cut;
                    // from the filter's Alg. 1 values; all ones where unknown)
  int32_t* idx_ext = nullptr;  // batch: candidates written here (the state pool's tail)
  int64_t n = 0, n_tets = 0, n_words = 0;
  int64_t fill = 0;            // state: pool entries in use (live + dead)
  int32_t* idxp() const { return idx_ext ? idx_ext : idx.as<int32_t>(); }
};
// Piece set over a list of tets: the same pool scheme (rows [beg, end) of piece slots per
// tet; inc_off / rpf_off are CSRs over the pool's piece slots, appended in order).
struct PieceSet {
  DevBuf off, sphere, vol, m1, fm, inc_off, inc;
  // fractional Euler characteristics (Euler mode): per piece, and per radical SoS facet
  DevBuf eu, rpf_off, rpf_j, rpf_e;
  DevBuf sfm, rfm;  // CC flags: SoS tet facets per piece, tet faces next to each radical facet
  DevBuf radj;      // per radical facet: the piece's radical facets sharing an edge (by rank)
  DevBuf rep;       // per radical facet x: for each tet face f (16 bits each) the ranks + 1 of
                    // the (at most two) radical facets y whose edge with x -- a restricted
                    // power edge -- has an endpoint on f
  DevBuf rows;      // int2 [n_tets]  state: [beg, end) of every tet's piece slots
  int64_t n_tets = 0, n_pieces = 0, n_inc = 0, n_rpf = 0;  // live counts
  int64_t fill_p = 0, fill_i = 0, fill_r = 0;              // state: pool slots in use
};
#ifndef RPD_CLIP_SMALL
#define RPD_CLIP_SMALL 2048  // below this many pairs the 64-slot tier clips all pairs directly
#endif

// Sizes of a device-driven partial update (the CUDA-graph latency path, rpd_graph.cu): the
// host writes the inputs part once per update; every size the eager path reads back to the
// host between its launches is produced and consumed on the device here instead.
enum PdAbort { PD_SLAB = 1, PD_QUEUE = 2, PD_POOL = 4, PD_BATCH = 8, PD_ERR = 16 };
struct PDyn {
  // inputs (host-written per update)
  const double* spheres;
  const int32_t* nbr_off;
  const int32_t* nbr_idx;
  const int32_t* new_ids;
  int N, N_old, E, M, epoch;
  int fill_c, fill_p, fill_i;  // state-pool fill levels (the batch is appended there)
  int room_c, room_p, room_i;  // state-pool capacities (entries)
  int nc_max, nw_max;          // batch candidate / mask-word bounds of the captured grids
  int cap_items, cap_sup;      // BVH work-queue capacities of the restricted re-filter
  // outputs (device-written)
  int nd;      // dirty tets
  int nb;      // tets of the batch: nd, or 0 once aborted (the rest of the graph idles)
  int n_chg;   // spheres whose rows changed since the dirty tets' candidate lists
  int nc, nw;  // batch candidates and incidence-mask words (0 once aborted)
  int nc_fast, nc_small;  // nc for the clip tier that takes the batch (the other gets 0)
  int nc_req, nw_req;  // the batch's candidates / mask words also when aborted (next sizes)
  int np, ni;  // batch pieces and incidences
  int maxk, need;  // largest k_tet, work-queue demand of the re-filter
  int abort;   // PdAbort bits: the eager path redoes the batch (re-filter onwards)
  unsigned long long stamp[6];  // RPD_OPT_PROFILE: %globaltimer around filter / re-filter / clip
  // copied back by the graph's last kernel (host mirror only)
  unsigned long long stats[ST_N];
  unsigned long long removed[4];  // the dirty tets' old segment sizes (cands, pieces, inc, rpf)
  int err[4];
  int n_wide;                     // pairs the fast clip tier passed on
};

}  // namespace rpd

struct rpd_ctx {
  int device = 0;
  int sms = 148;  // multiprocessor count of the device (queried at create)
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  int filter_mode = RPD_FILTER_ALL_PAIRS;
  int validate = 1;
  std::string err;
  int64_t launches = 0;

  // host-input staging (used when an argument is a host pointer)
  rpd::DevBuf h_verts, h_tets, h_spheres, h_off, h_idx, h_new;

  rpd::Stage st;
  rpd::DevBuf errw;        // int32[4]
  rpd::DevBuf stats;       // uint64[ST_N]
  rpd::DevBuf scratch;     // scan: u64 ticket counter + per-tile look-back state words
  unsigned long long scan_ticket = 0;  // tickets consumed so far (device counter value)
  unsigned scan_epoch = 0;             // call sequence number tagged into the state words

  // filter scratch
  rpd::DevBuf k_tet, k_words, slab, w_off;
  rpd::DevBuf slab_m;      // uint2 per slab entry: the candidate's 64-plane cut mask
  rpd::DevBuf cand_long;   // compaction: count + tets with more than 16 candidates
  rpd::DevBuf g_cnt;       // segment gather: per output row counts and tet-level inc offsets
  rpd::DevBuf g_map;       // segment gather: int2 (source, row) per output row
  rpd::DevBuf g_off, g_dst;  // segment gather: offsets scratch, staging of host destinations
  rpd::DevBuf g_ids, h_dl, h_dm;  // rpd_download_tets: ids staging, host list / id map
  rpd::CandSet g_cand[2];  // rpd_merge_shards outputs (alternating: the old CSR may be the
  rpd::PieceSet g_pcs[2];  // previous output)
  int g_cur = 0;
  rpd::DevBuf env_buf, env_out, h_env;  // envelope distance (NEXT-4): scratch, outputs, inputs
  rpd::DevBuf h_env2, h_env3, h_env4;
  rpd::DevBuf bvh;         // leaf and super-node boxes of the pruned filter
  rpd::DevBuf bvh_all;     // leaf + super boxes of the whole mesh (valid per staged mesh)
  bool bvh_all_valid = false;
  rpd::DevBuf bvh_items;   // (sphere, super node) work queue of the pruned filter
  int64_t bvh_cap_items = 0, bvh_min_items = 0;
  int slab_cap = 32;

  // current candidates / pieces (double-buffered for partial updates) and the dirty sets
  rpd::CandSet cand[2], cand_d;
  rpd::PieceSet pcs[2], pcs_d;
  int cur = 0;
  bool have_rel = false, have_pieces = false;
  bool compact = true;         // the state pools are plain CSRs (no partial update since)
  int64_t n_compactions = 0;   // pool compactions (garbage collection) since rpd_create

  // clip per-pair scratch
  rpd::DevBuf p_flag, p_f01, p_vol, p_m1, p_fm, p_ninc, p_mask, p_over, p_over2, p_over3, p_scan, i_scan;
  rpd::DevBuf p_dyn;  // dynamic pair counter of the fast clip kernel

  // partial update scratch
  rpd::DevBuf d_count, d_flag, d_scan, d_list, m_cnt, m_off;
  rpd::DevBuf c_flag, c_scan, c_list;  // changed-row spheres of a partial update
  rpd::DevBuf cepoch;          // int32 per tet: epoch of its candidate list
  rpd::DevBuf min_epoch;       // int32: oldest candidate-list epoch among the dirty tets
  int epoch = 0;               // 0 after rpd_relations, +1 per partial update
  int64_t n_dirty = 0;

  // device-driven partial updates captured as CUDA graphs (rpd_graph.cu)
  rpd::PDyn* pdd = nullptr;     // non-null while the device-driven sequence is being issued
  rpd::DevBuf pd_buf;           // PDyn (device)
  rpd::PDyn* pd_host = nullptr; // PDyn (mapped pinned): inputs in, outputs back
  rpd::PDyn* pd_hdev = nullptr; // its device-side address
  rpd::DevBuf g_scan;           // look-back state of the graph's scans (reset by memset nodes)
  size_t g_scan_used = 0;
  cudaStream_t cap_stream = nullptr;  // capture stream (the legacy stream cannot capture)
  static constexpr int G_CACHE = 4;
  unsigned long long g_sig[G_CACHE] = {};
  cudaGraphExec_t g_exec[G_CACHE] = {};
  int64_t g_kernels[G_CACHE] = {};  // kernel nodes per cached graph
  int64_t g_nodes = 0;
  int g_next = 0;
  int graph = 1;                // RPD_OPT_GRAPH (env RPD_GRAPH=0 turns it off)
  int64_t g_launches = 0, g_captures = 0, g_fallbacks = 0;
  int64_t dd_cap[2][2] = {};    // BVH queue capacities {items, super items}: dirty, re-filter
  int64_t g_mb = 64;            // new-sphere bound of the current graph (grid of the id check)
  int64_t g_nc_max = 0;         // batch-candidate bound of the graphs (grows, never shrinks)
  int64_t g_nc_fix = 0;         // env RPD_GRAPH_NC_MAX: a fixed bound (tests of the fallback)
  int64_t g_last_nc = 0, g_last_nw = 0;  // candidates / mask words of the last batch

  rpd_stats last{};
  int profile = 0;             // record CUDA events around the filter and clip kernels
  cudaEvent_t ev[4] = {nullptr, nullptr, nullptr, nullptr};
  // development trace of a partial update (env RPD_TRACE_HOST): host and stream timestamps
  int tr_on = -1, tr_n = 0;
  cudaEvent_t tr_ev[16] = {};
  double tr_h[16] = {};
  const char* tr_nm[16] = {};
  void* pinned = nullptr;      // small mapped pinned host buffer for scalar readbacks
  void* pinned_dev = nullptr;  // its device-side address
  int clip_wide = 0;           // testing: run every pair through the wide kernel
  int clip_small = 0;          // the last clip ran the 64-slot tier on all pairs (few pairs)
  int clip_tiers = 0;          // testing: always the fast tier + overflow cascade
  int clip_route = 0;          // graph path: pairs with more cut planes than this go straight to
                               // the 64-slot tier, concurrently with the fast tier (0: off)
  rpd::DevBuf p_route;         // routed pair lists: [small count, big count, small.., big..]
  cudaStream_t side_stream = nullptr;  // the concurrent branch of a captured graph
  cudaEvent_t g_fork = nullptr, g_join = nullptr;
  int64_t pdd_nc_max = 0;      // the batch bound of the graph being captured

  // fractional Euler characteristics (rpd_euler.cu; rpd_set_euler)
  int euler = 0;               // payloads set for the current tets
  bool eu_valid = false;       // the current pieces carry Euler data
  rpd::DevBuf h_eut, h_euid;   // host-input staging of rpd_set_euler
  int64_t eu_T = 0;            // ctx-local tet count the payloads were built for
  int eu_P = 0;                // primes p <= 255 dividing some sharing count (sum layout)
  int eu_primes[64] = {}, eu_ppow[64] = {};  // those primes and their powers p^E <= 255
  rpd::DevBuf eu_tab;          // scratch hash tables of the payload setup
  rpd::DevBuf eu_rec;          // uint4 per local tet: sharing counts of its 14 elements
  rpd::DevBuf eu_A;            // int64 [512]: primes [0, 64), p^E [64, 128), P [128],
                               // the counts-present bitmap from [257]
  rpd::DevBuf eu_Lt;           // int64 [T_local]: per tet L_t = lcm of its 14 sharing counts
  rpd::DevBuf eu_acc;          // int64 [(N + E) (1 + P)]: per-sphere / per-CSR-entry sums as an
                               // integer part + one residue per prime (exact, any mesh)
  rpd::DevBuf eu_fin;          // finalised sums: int64 [N + E], double [N + E], uint8 [N + E]
  rpd::DevBuf eu_den;          // int64 [n_pieces]: each piece's denominator (rpd_get_euler)
  rpd::DevBuf eu_sum;          // int64 [N + E + 1]: per-sphere RPC, per-CSR-entry RPF, misses
  rpd::DevBuf p_eu, p_rmask, p_rval, p_nrpf, r_scan;  // per-pair clip outputs
  rpd::DevBuf p_sfm, p_rfm, p_radj, p_rep;            // per-pair CC / medial-mesh flags
  rpd::DevBuf mm_keys, mm_tmp, mm_out;                // medial-mesh extraction scratch
  rpd::DevBuf rpe_off, rpe_buf, rpe_ee;               // restricted power edges (launch_rpe)
  int64_t rpe_n = -1, rpe_nu = -1;                     // sizes of the last rpd_get_rpe
  int64_t mm_ne = -1, mm_nf = -1;                     // sizes of the last extraction
  bool eu_whole = false;       // payloads built with the ctx holding the whole mesh in order
  rpd::DevBuf eu_adj;          // int32 [4 T_local]: face neighbour 4 t' + k' (global) or -1
  rpd::DevBuf cc_par, cc_out;  // CC numbers: union-find parents, outputs
  rpd::DevBuf eu_ids, eu_g2l;  // sharded Euler mode: local -> global tet ids and back (-1: remote)
  rpd::DevBuf cc_bnd, cc_gpar, cc_sort, cc_nrec;  // CC of a sharded job: records, global parents
  int64_t cc_base_c = -1, cc_base_f = -1;  // this rank's global id bases (rpd_cc_shard)
  rpd::DevBuf rpe_bnd, rpe_cnt, rk_buf, rk_out;  // RPEs of a sharded job; reduce-by-key
  int64_t rpe_base = -1;
  // sphere neighbours (NEXT-3): scratch (grid, pass-1 rows), outputs (off, idx), pass-2 rows
  rpd::DevBuf nb_buf, nb_off, nb_idx, nb_tmp, nb_cnt, h_nb, nb_hits;
  void* nb_grid = nullptr;
  unsigned long long* nb_stats = nullptr;
  int32_t *nb_start = nullptr, *nb_items = nullptr, *nb_long = nullptr, *nb_long_ids = nullptr,
          *nb_slab = nullptr;
  double nb_args_tol0 = 0.0;
  int nb_ball_test = 1;  // the neighbour enumeration's ball pre-test of the last nb_build (pass 2 matches it)
  void* nb_dbg = nullptr;
  void* nb_sorted = nullptr;  // double4 per sphere in cell order  // development aid: device int64 [N][8] per-sphere counters
  int64_t nb_N = -1, nb_E = 0;
  int32_t* nb_work = nullptr;   // pass-1 work counter, radius work order (nb_build)
  int32_t* nb_order = nullptr;
  double nb_box[6] = {};        // the box of the current lists
  rpd::DevBuf nb_prev;          // the spheres of the current lists (update: old ones unchanged)
  rpd::DevBuf nb_off2, nb_idx2; // the merged lists of an incremental update (swapped in)
  rpd::DevBuf nb_flag, nb_list, nb_len, nb_misc;
  int64_t nb_rows = 0;          // rows computed by the last call
  rpd::DevBuf nb_ball;          // 2 double4 per sphere: ball around its last P_K (r < 0: empty), vertex-box half extents
};

namespace rpd {

// launchers (all on ctx->stream; each increments ctx->launches)
cudaError_t launch_stage_mesh(rpd_ctx* c, const double* verts, int64_t V, const int32_t* tets,
                              int64_t T);
cudaError_t launch_stage_spheres(rpd_ctx* c, const double* spheres, int64_t N,
                                 const int32_t* nbr_off, const int32_t* nbr_idx, int64_t E,
                                 bool reuse_rows, int epoch);
// launch_stage_spheres = stage_prepare (host: buffer swap + sizes) + stage_launch (kernels)
cudaError_t stage_prepare(rpd_ctx* c, int64_t N, int64_t E);
cudaError_t stage_launch(rpd_ctx* c, const double* spheres, const int32_t* nbr_off,
                         const int32_t* nbr_idx, bool reuse_rows, int epoch);
cudaError_t launch_neighbors_pass1(rpd_ctx* c, const double* sph, int64_t N, const double box[6],
                                   int32_t* cnt, int32_t* off);
// incremental update of the lists after appending spheres [N_old, N) (rpd_neighbors_update):
// part 1 the new rows (pass 1), the old rows' lengths (old row + the new spheres whose plane
// reaches the row's P_K ball; 0 when hidden), the merged offsets (off[N] = E, misc[0] = old rows
// changed); part 2 the new long rows and the merged CSR
cudaError_t launch_nb_update1(rpd_ctx* c, const double* sph, int64_t N, int64_t N_old,
                              const double box[6], const double* prev, int32_t* cnt,
                              uint8_t* flag, int32_t* list, int32_t* len,
                              const int32_t* old_off, int32_t* off, int* misc);
cudaError_t launch_nb_update2(rpd_ctx* c, const double* sph, int64_t N, int64_t N_old,
                              const double box[6], int32_t* cnt, const int32_t* len,
                              const int32_t* old_off, const int32_t* old_idx, const int32_t* off,
                              int32_t* tmp, int32_t* idx);
cudaError_t launch_neighbors_pass2_rows(rpd_ctx* c, const double* sph, int64_t N,
                                        const double box[6], int32_t* cnt, const int32_t* off,
                                        int32_t* tmp);
// list of the flags equal to val (val < 0: non-zero; ascending) and their count (rpd_scan.cu)
cudaError_t launch_flag_list(rpd_ctx* c, const uint8_t* flag, int64_t n, int32_t* list,
                             int* count, int val = -1);
cudaError_t launch_neighbors_pass2(rpd_ctx* c, const double* sph, int64_t N, const double box[6],
                                   int32_t* cnt, const int32_t* off, int32_t* tmp, int32_t* idx);
void clip_phase_dump();  // development aid (RPD_CLIP_PHASES builds)
// n_dev (device-driven update): the length read on the device, n its bound
cudaError_t launch_scan_i32(rpd_ctx* c, const int32_t* in, int32_t* out, int64_t n,
                            const int* n_dev = nullptr);
cudaError_t launch_scan_u8(rpd_ctx* c, const uint8_t* in, int32_t* out, int64_t n,
                           const int* n_dev = nullptr);
cudaError_t launch_scan_i32_multi(rpd_ctx* c, const int32_t* const* in, int32_t* const* out,
                                  int K, int64_t n, const int* n_dev = nullptr);
cudaError_t launch_filter(rpd_ctx* c, const int32_t* tet_ids, int64_t n_tets, int cap,
                          int sphere_lo, int sphere_hi, int32_t* k_tet, int32_t* slab,
                          int32_t* k_words, const int32_t* sphere_list = nullptr,
                          const int* n_list_dev = nullptr);
// dirty tets: keep the old candidates whose neighbour row did not change (same booleans)
cudaError_t launch_keep_old(rpd_ctx* c, const int32_t* dirty, int64_t n_dirty,
                            const CandSet& co, int cap, int32_t* k_tet, int32_t* slab,
                            int32_t* k_words);
// spheres whose rows were rebuilt after the oldest candidate list of the dirty tets
cudaError_t launch_changed_list(rpd_ctx* c, int64_t N);
cudaError_t launch_max_ktet(rpd_ctx* c, int64_t n, const int32_t* k_tet);
cudaError_t launch_compact_cands(rpd_ctx* c, int64_t T, int cap, const int32_t* k_tet,
                                 int32_t* slab, const int32_t* cand_off,
                                 int32_t* cand_idx, int32_t* pair_tet, const int32_t* w_off,
                                 int32_t* p_moff, int64_t n_pairs, unsigned* p_cut);
cudaError_t launch_clip(rpd_ctx* c, int64_t n_pairs, const int32_t* pair_tet,
                        const int32_t* tet_ids, const int32_t* cand_idx, const int32_t* moff,
                        const unsigned* cut, int wide);
cudaError_t launch_clip_overflow(rpd_ctx* c, const int32_t* pair_tet, const int32_t* tet_ids,
                                 const int32_t* cand_idx, const int32_t* moff,
                                 const unsigned* cut);
cudaError_t launch_piece_scans(rpd_ctx* c, int64_t n_pairs, const int32_t* moff);
// destination of a piece compaction
struct PieceDst {
  int32_t* off;      // [n_tets+1]
  int32_t* sphere;
  double* vol;
  double* m1;
  uint8_t* fm;
  int32_t* inc_off;  // [n_pieces+1]
  int32_t* inc;
  long long* eu;      // Euler mode: [n_pieces], rpf CSR [n_pieces+1] / [n_rpf]
  int32_t* rpf_off;
  int32_t* rpf_j;
  long long* rpf_e;
  uint8_t* sfm;       // [n_pieces], [n_rpf]
  uint8_t* rfm;
  unsigned long long* radj;  // [n_rpf]
  unsigned long long* rep;   // [n_rpf]
  int32_t inc_base = 0;      // added to every inc_off / rpf_off value (appending to a pool
  int32_t rpf_base = 0;      // whose incidences / radical facets already hold this many)
};
cudaError_t launch_compact_pieces(rpd_ctx* c, int64_t n_tets, int64_t n_pairs,
                                  const int32_t* cand_off, const int32_t* cand_idx,
                                  const int32_t* moff, const PieceDst& d);
// partial update (rpd_partial.cu)
cudaError_t launch_check_new_ids(rpd_ctx* c, const int32_t* new_ids, int64_t M, int64_t N_old);
cudaError_t launch_dirty_list(rpd_ctx* c, int64_t T);
// fused scans (rpd_scan.cu): dirty tets (list, positions, epochs) and changed-row spheres
cudaError_t launch_dirty_scan(rpd_ctx* c, int64_t T);
cudaError_t launch_changed_scan(rpd_ctx* c, int64_t N);
// state rows from the compact CSRs (cand and / or piece; NULL skips)
cudaError_t launch_rows_from_off(rpd_ctx* c, int64_t T, const CandSet* cs, PieceSet* ps,
                                 CandSet* cs_rows);
// partial update: re-point the dirty tets' rows at the batch appended to the pools, and count
// the removed (old) segments' sizes into rm[0..3] = cands, pieces, incidences, radical facets
cudaError_t launch_rows_update(rpd_ctx* c, const int32_t* dirty, int64_t nd, CandSet& pool_c,
                               PieceSet& pool_p, const CandSet& cd, const PieceSet& pd,
                               int64_t cbase, int64_t pbase, unsigned long long* rm);
// device-driven partial update (rpd_graph): PDyn init from the pinned mirror, the checks
// after the re-filter (batch totals, capacities; abort), the totals back to the mirror
cudaError_t launch_pd_init(rpd_ctx* c);
// per-sphere RPC volumes of the current pieces into out [N] (device)
cudaError_t launch_sphere_volumes(rpd_ctx* c, double* out);
cudaError_t launch_pd_check(rpd_ctx* c, const int32_t* c_off, const int32_t* w_off);
cudaError_t launch_pd_final(rpd_ctx* c);
cudaError_t launch_pd_stamp(rpd_ctx* c, int k);
// compaction of the state pools (by rows) into the plain CSRs cn / pn (pair_tet and moff of
// the candidates rebuilt); phase 0: counts + scans, phase 1: copies
cudaError_t launch_compact_state(rpd_ctx* c, int64_t T, const CandSet& co, const PieceSet& po,
                                 CandSet& cn, PieceSet& pn, int phase);
// segment gather engine (rpd_gather.cu): multi-GPU gather / partial-mode merge / download
// of a tet list.  A source holds per-row candidate and piece segments [beg[r], end[r]) and a
// per-piece incidence CSR i_off (piece p: [i_off[p], i_off[p+1])); NULL parts are skipped.
struct SegSrc {
  int rs;  // row stride of the beg / end arrays: 1 (CSR offsets) or 2 (int2 rows)
  const int32_t *c_beg, *c_end, *c_idx;
  const int32_t *p_beg, *p_end, *p_sphere;
  const double *p_vol, *p_m1;
  const uint8_t* p_fm;
  const int32_t *i_off, *i_sph;
};
struct SegSources {
  SegSrc s[RPD_MAX_RANKS + 1];  // [0]: previous global CSR / the ctx state; [1 + r]: rank r
};
struct SegShards {
  int world;
  int64_t base[RPD_MAX_RANKS + 1];  // prefix of the ranks' row counts
  const int32_t* tet_ids[RPD_MAX_RANKS];
};
struct SegDst {
  int32_t *cand_off, *cand_idx;
  int32_t *piece_off, *piece_sphere;
  double *piece_vol, *piece_m1;
  uint8_t* piece_fm;
  int32_t *inc_off, *inc_sphere;
  const int32_t* i_tet;  // tet-level incidence offsets (from launch_seg_counts)
};
SegSrc seg_src_csr(const int32_t* c_off, const int32_t* c_idx, const int32_t* p_off,
                   const int32_t* p_sphere, const double* p_vol, const double* p_m1,
                   const uint8_t* p_fm, const int32_t* i_off, const int32_t* i_sph);
SegSrc seg_src_state(const CandSet& cs, const PieceSet& ps);
// kind 0: identity rows of source 0; 1: source-0 rows `list`; 2: identity overwritten by the
// shards' rows (merge); 3: only the shards' rows (gather)
cudaError_t launch_map(rpd_ctx* c, int kind, int64_t n_out, const int32_t* list,
                       const SegShards* sh, int64_t T);
cudaError_t launch_seg_counts(rpd_ctx* c, int64_t n_out, const SegSources& S, int32_t* cand_off,
                              int32_t* piece_off, int32_t** i_tet_out);
cudaError_t launch_seg_copy(rpd_ctx* c, int64_t n_out, const SegSources& S, const SegDst& D);
cudaError_t launch_map_ids(rpd_ctx* c, const int32_t* list, int64_t n, const int32_t* id_map,
                           int64_t T, int32_t* ids_out);
// envelope distance (rpd_envelope.cu)
cudaError_t launch_envelope_check(rpd_ctx* c, int64_t N, const int32_t* edges, int64_t NE,
                                  const int32_t* faces, int64_t NF);
cudaError_t launch_envelope(rpd_ctx* c, const double* smp, int64_t S, const double* sph,
                            int64_t N, const int32_t* edges, int64_t NE, const int32_t* faces,
                            int64_t NF, double* g_out, int32_t* prim_out,
                            unsigned long long* n_eval);
// fractional Euler characteristics (rpd_euler.cu)
cudaError_t launch_euler_setup(rpd_ctx* c, const int32_t* tets_all, int64_t T_all, int64_t V,
                               const int32_t* local_ids, int64_t T_local);
cudaError_t launch_euler_sums(rpd_ctx* c, const PieceSet& ps);
// accumulator rows [K, R_1 .. R_P] -> values (rpd_euler_finalize)
cudaError_t launch_euler_final(rpd_ctx* c, const unsigned long long* acc, int64_t n,
                               long long* vi, double* vd, uint8_t* ex);
cudaError_t launch_piece_den(rpd_ctx* c, const PieceSet& ps);
cudaError_t launch_cc(rpd_ctx* c, const PieceSet& ps);
// CC numbers of a tet-sharded job (distributed union-find, rpd_cc_shard / rpd_cc_merge)
cudaError_t launch_g2l(rpd_ctx* c, const int32_t* local_ids, int64_t T_local, int64_t T_all);
cudaError_t launch_cc_shard(rpd_ctx* c, const PieceSet& ps, long long base_c, long long base_f,
                            int* n_rec);
// RPEs of a sharded job (rpd_rpe_shard / rpd_rpe_merge) and the generic key reduction
cudaError_t launch_rpe_shard(rpd_ctx* c, const PieceSet& ps, long long base, int* n_rec,
                             int64_t* n_rpe, int64_t* n_tri);
cudaError_t launch_rpe_merge(rpd_ctx* c, const unsigned long long* key_b,
                             const unsigned long long* jk_b, const int32_t* lab_b, int64_t n_b,
                             int64_t total, long long base, int* n_out);
cudaError_t launch_reduce_by_key(rpd_ctx* c, const unsigned long long* keys, const long long* vals,
                                 int64_t n, unsigned long long* out_k, long long* out_v,
                                 int* n_out);
cudaError_t launch_cc_merge(rpd_ctx* c, const PieceSet& ps, const unsigned long long* key_c,
                            const int32_t* lab_c, int64_t n_c, const unsigned long long* key_f,
                            const int32_t* j_f, const int32_t* lab_f, int64_t n_f,
                            int64_t tot_c, int64_t tot_f, long long base_c, long long base_f,
                            int32_t* counts);
// restricted power edges: per-piece lists, per-(i, j, k) Euler sums, CC numbers (with_cc)
cudaError_t launch_rpe(rpd_ctx* c, const PieceSet& ps, bool with_cc, int64_t* n_rpe,
                       int64_t* n_tri);
// medial mesh: unique sorted edge keys (i << 32 | j) and face keys (i << 42 | j << 21 | k)
cudaError_t launch_medial_mesh(rpd_ctx* c, const PieceSet& ps, int64_t* n_edges,
                               int64_t* n_faces);

}  // namespace rpd
