/*
 * rpd.h -- C ABI of the B200 RPD hot path of MATTopo (arXiv 2403.18761).
 *
 * The library computes the volumetric restricted power diagram (RPD) of medial spheres over
 * a tetrahedral mesh with the paper's modified Tet-Cell strategy:
 *
 *   rpd_relations       Alg. 1 tet-sphere relation filter over every (tet, sphere) pair and
 *                       per-tet compaction into k_tet candidate lists
 *                       (PAPER.md:21-50 Supp. §1.2 Alg. 1; "every pair")
 *   rpd_clip            per (tet, candidate sphere) convex clipping of the tet by the radical
 *                       half-spaces of that sphere against all its power neighbours, giving the
 *                       restricted-power-cell pieces with volume, first moment and
 *                       face/neighbour incidences (§3.3, 488 §4.1.2)
 *   rpd_update_partial  partial update after appending M new spheres: only tets related to a
 *                       new sphere are re-filtered and re-clipped
 *   rpd_set_euler /     fractional Euler characteristics of the restricted power cells and
 *   rpd_get_euler       faces, collected on the fly by the clip (Sec. 4.1.2)
 *
 * Inputs are the paper's problem statement: tets with 4 ordered vertices,
 * medial spheres m = (theta, r) and the sphere neighbour lists k_site that the
 * paper obtains from CGAL's regular triangulation.
 *
 * Conventions:
 *  - Exact mode (default): every coordinate and radius must be a multiple of 2^-10 in
 *    [0, 64); then relation booleans, candidate lists, non-empty flags, facemasks and
 *    incidences are bit-exact (exact integer predicates + symbolic perturbation).  Inputs off
 *    that lattice fail with RPD_ENOTEXACT.
 *  - Pointers: every array argument may be a CUDA device pointer or a host pointer (pinned
 *    or pageable); host arrays are copied to ctx-owned device memory on the ctx stream.
 *    Inputs are borrowed for the duration of the call only.
 *  - Outputs are ctx-owned DEVICE arrays, valid until the next mutating call on the ctx or
 *    rpd_destroy.  Host scalars (counts) are returned by value; reading them is the only
 *    device->host synchronisation of each call.
 *  - Every call is stream-ordered on the ctx stream.  One ctx per device; a ctx is not
 *    thread-safe.  No exception crosses the ABI; every call returns an rpd_status and
 *    rpd_last_error() describes the last failure.  Asynchronous kernel faults surface as
 *    RPD_ECUDA at the next call that synchronises.
 */
#ifndef RPD_H
#define RPD_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct rpd_ctx rpd_ctx;

typedef enum {
  RPD_OK = 0,
  RPD_EINVAL = -1,     /* bad argument: tet index out of range, non-positive tet orientation,
                          r < 0, NaN/Inf, neighbour out of range / self / duplicate, neighbour
                          with the same centre, new_ids not the appended range, NULL ctx */
  RPD_ENOMEM = -2,     /* device allocation failed */
  RPD_ECUDA = -3,      /* CUDA runtime error (launch failure, fault) */
  RPD_EOVERFLOW = -4,  /* a piece exceeded even the slow-path capacity (should be unreachable) */
  RPD_ESTATE = -5,     /* call order: rpd_clip / rpd_update_partial before rpd_relations */
  RPD_ENOTEXACT = -6   /* exact mode on and an input is off the 2^-10 lattice or out of box */
} rpd_status;

/* Create a context on CUDA `device`.  `cuda_stream` is a cudaStream_t to order all work on
 * (NULL: the ctx creates its own non-blocking stream, NOT ordered with other streams; pass
 * cudaStreamLegacy to run on the legacy default stream). */
rpd_status rpd_create(rpd_ctx** out, int device, void* cuda_stream);
void rpd_destroy(rpd_ctx* ctx);
/* Human-readable description of the last failure on ctx (host string owned by ctx, valid
 * until the next call).  Safe with ctx == NULL. */
const char* rpd_last_error(const rpd_ctx* ctx);

/* Options (rpd_set_option). */
enum {
  RPD_OPT_FILTER_MODE = 1,   /* RPD_FILTER_ALL_PAIRS (literal Alg. 1 over all T*N pairs,
                                default) or RPD_FILTER_PRUNED (identical booleans; pairs that
                                provably fail Alg. 1 are skipped) */
  RPD_OPT_VALIDATE = 2,      /* 1 (default): validate inputs on device; 0: skip */
  RPD_OPT_STREAM = 3,        /* value = (intptr_t) cudaStream_t to switch the ctx stream */
  RPD_OPT_CLIP_WIDE = 4,     /* 1: clip every pair with the wide (128-vertex) kernel instead of
                                only the pairs that overflow the fast (32-vertex) one; for tests */
  RPD_OPT_PROFILE = 5,       /* 1: time the filter and clip kernels with CUDA events on the ctx
                                stream (rpd_stats.filter_ms / clip_ms) */
  RPD_OPT_CLIP_TIERS = 6,    /* 1: always the fast (16-vertex) tier and its overflow cascade, also
                                for fewer than 2048 pairs (which otherwise go straight to the
                                64-slot tier); for tests */
  RPD_OPT_GRAPH = 7          /* 1 (default; env RPD_GRAPH=0 sets 0 at rpd_create): a partial
                                update of 1..64 new spheres (pruned filter, no Euler payloads,
                                no profiling) runs as ONE device-driven CUDA graph with one host
                                round trip (DESIGN.md §8 "latency path"); 0: eager launches with
                                three round trips.  Same results either way. */
};
enum { RPD_FILTER_ALL_PAIRS = 0, RPD_FILTER_PRUNED = 1 };
rpd_status rpd_set_option(rpd_ctx* ctx, int option, int64_t value);

/* Step 1 -- Alg. 1 relation filter + per-tet compaction.
 *   verts    [V][3] double   vertex coordinates
 *   tets     [T][4] int32    vertex indices; positively oriented; face k = opposite vertex k
 *                            (this rank's tet shard; the caller keeps the local->global map)
 *   spheres  [N][4] double   (x, y, z, r), r >= 0
 *   nbr_off  [N+1]  int32    CSR offsets of the k_site neighbour lists
 *   nbr_idx  [E]    int32    neighbour sphere ids (any order; the ctx sorts a copy)
 *   E        host int64      length of nbr_idx; must equal nbr_off[N] (else RPD_EINVAL at the
 *                            call's readback); E < 0: read nbr_off[N] (one extra host round
 *                            trip when nbr_off is a device pointer)
 * Outputs (ctx-owned device arrays):
 *   *cand_off [T+1] int32    per-tet candidate offsets (k_tet(t) = cand_off[t+1]-cand_off[t])
 *   *cand_idx [n_cand] int32 candidate sphere ids, ascending per tet
 *   *n_cand   host int64
 * Relation (R1, R2, R4): for k_site(i) > 0, t relates to i iff for every neighbour
 * j some vertex v of t has PD_i(v) < PD_j(v) strictly; for k_site(i) = 0, iff N == 1. */
rpd_status rpd_relations(rpd_ctx* ctx, const double* verts, int64_t V, const int32_t* tets,
                         int64_t T, const double* spheres, int64_t N, const int32_t* nbr_off,
                         const int32_t* nbr_idx, int64_t E, const int32_t** cand_off,
                         const int32_t** cand_idx, int64_t* n_cand);

/* Pieces of the RPD restricted to the ctx's tets (device arrays owned by ctx).
 * Layout: a pool of n_slots piece slots; tet t's pieces are the slots
 * [piece_rows[2t], piece_rows[2t+1]), ascending sphere id, and piece p's incidences are
 * inc_sphere[inc_off[p], inc_off[p+1]).  After rpd_clip the pool is a plain CSR (piece_off,
 * n_slots == n_pieces); a partial update appends the dirty tets' new pieces at the pool's
 * tail and re-points their rows -- clean tets are never copied -- and piece_off is NULL
 * until the next rpd_clip (rpd_download_pieces always writes a plain CSR). */
typedef struct {
  const int32_t* piece_off;      /* [T+1] pieces of tet t: [piece_off[t], piece_off[t+1]),
                                    ascending sphere id; NULL after a partial update */
  const int32_t* piece_sphere;   /* [n_pieces] owning sphere i */
  const double* piece_vol;       /* [n_pieces] volume of P(t,i) > 0 */
  const double* piece_m1;        /* [n_pieces][3] first moment = vol * centroid */
  const uint8_t* piece_facemask; /* [n_pieces] bit k: a positive-area 2-face of P lies on tet
                                    face k (opposite vertex k) */
  const int32_t* inc_off;        /* [n_pieces+1] */
  const int32_t* inc_sphere;     /* neighbour ids j whose radical plane holds a positive-area
                                    2-face of the piece, ascending; coincident sources all
                                    listed (R7) */
  int64_t n_pieces, n_inc;       /* host values: live pieces and incidences */
  const int32_t* piece_rows;     /* [T][2] the slots of every tet's pieces (always valid) */
  int64_t n_slots;               /* pool slots in use (live + replaced) */
} rpd_pieces;

/* Step 2 -- clip every candidate of the last rpd_relations:
 *   P(t,i) = t  n  { x : PD_i(x) <= PD_j(x) for all j in N(i) }
 * Non-empty means positive volume (inward symbolic perturbation, C4, R8).
 * Returns RPD_ESTATE if rpd_relations has not run on this ctx. */
rpd_status rpd_clip(rpd_ctx* ctx, rpd_pieces* out);

/* Partial update ("only select a subset of tets ... relating to new spheres").
 * spheres [N_new][4]: the first N_old are unchanged, new sphere ids [N_old, N_new) appended;
 * nbr_off/nbr_idx/E: the new neighbour CSR over all N_new spheres (E as in rpd_relations);
 * new_ids [M] int32 must equal
 * N_old..N_new-1 (else RPD_EINVAL); M == 0 is the identity.
 * Dirty tets = { t : rel_new(t, n) for some new n } (R11); they get a full
 * re-filter + clip with the new neighbour lists; clean tets keep candidates and pieces
 * byte-identically.  Outputs: the merged pieces (as rpd_clip), the dirty tets (device int32,
 * ascending) and their count (host).  The ctx candidate CSR is updated the same way.
 * Requires a prior rpd_relations + rpd_clip (else RPD_ESTATE). */
rpd_status rpd_update_partial(rpd_ctx* ctx, const double* spheres, int64_t N_new,
                              const int32_t* nbr_off, const int32_t* nbr_idx, int64_t E,
                              const int32_t* new_ids, int64_t M, rpd_pieces* out,
                              const int32_t** dirty_tets, int64_t* n_dirty);

/* Copy the current pieces to caller-owned arrays (host or device memory) (sizes from the last rpd_pieces):
 * piece_off [T+1], piece_sphere/vol/facemask [n_pieces], piece_m1 [3 n_pieces],
 * inc_off [n_pieces+1], inc_sphere [n_inc].  Any pointer may be NULL (skipped). */
rpd_status rpd_download_pieces(rpd_ctx* ctx, int32_t* piece_off, int32_t* piece_sphere,
                               double* piece_vol, double* piece_m1, uint8_t* piece_facemask,
                               int32_t* inc_off, int32_t* inc_sphere);

/* Copy the current candidate CSR to caller-owned arrays (host or device memory): cand_off [T+1],
 * cand_idx [n_cand].  Either pointer may be NULL. */
rpd_status rpd_download_cands(rpd_ctx* ctx, int32_t* cand_off, int32_t* cand_idx);

/* ---- Fractional Euler characteristics (Sec. 4.1.2)
 *
 * "such fractional Euler characteristics are inputted together with the mesh":
 * every vertex / edge / face of the tet mesh carries 1/(number of tets sharing it) inside each
 * tet, a tet carries 1.  While clipping, a new vertex inherits the payload of the tet simplex
 * it lies on, a new edge that of the face it cuts, a new facet that of the cell; new elements
 * are not re-divided.  Per piece and per radical facet the clip then sums
 *   Euler(piece)     = sum_vertices - sum_edges + sum_facets - 1      (Eq. (1))
 *   Euler(facet j)   = sum_{vertices on it} - sum_{edges on it} + 1
 * over the symbolically perturbed (simple) polytope, and the library reduces them per sphere:
 *   Euler(RPC(m_i))      = sum over the pieces of m_i
 *   Euler(RPF(m_i, m_j)) = sum over their facets on the radical plane h_ij (seen from m_i).
 * All values are EXACT, for any mesh (R24): a piece's values are numerators over its
 * tet's denominator L_t = lcm of the tet's 14 sharing counts (< 2^62), and every per-sphere sum
 * is accumulated exactly as an integer part plus one residue modulo p^E per prime p <= 255 that
 * divides a sharing count (p^E the largest power <= 255): the sum is an integer iff every
 * residue vanishes, and then the integer is exact.  Integer adds only: identical across
 * kernels, launches and ranks; the per-sphere sums of a closed mesh are integers.
 *
 * rpd_set_euler: build the payloads of the ctx's tets (call after or before rpd_relations,
 * before rpd_clip; stays on until switched off with tets_all = NULL, T_all = 0).
 *   tets_all  [T_all][4] int32  the WHOLE mesh (sharing counts are global; a sharded rank
 *                               passes every tet, not only its own)
 *   V         host int64        vertex count, 0 < V < 2^21
 *   local_ids [T_local] int32   global index of every ctx-local tet (the tets given to
 *                               rpd_relations), or NULL when the ctx holds all tets in order
 *                               (then T_local must equal T_all)
 *   *n_primes host out          P, the number of residues of a sum's accumulator row (rows
 *                               are 1 + P int64: integer part, then the residues)
 * Errors: RPD_EINVAL (bad argument, vertex index out of range), RPD_EOVERFLOW (an element
 * shared by more than 255 tets, or some L_t >= 2^62), RPD_ENOMEM.  rpd_clip fails with
 * RPD_EINVAL if the ctx's tet count differs from T_local. */
rpd_status rpd_set_euler(rpd_ctx* ctx, const int32_t* tets_all, int64_t T_all, int64_t V,
                         const int32_t* local_ids, int64_t T_local, int64_t* n_primes);

/* Euler data of the current pieces (ctx-owned device arrays, valid until the next mutating
 * call).  RPD_ESTATE unless rpd_set_euler preceded the last rpd_clip / rpd_update_partial. */
typedef struct {
  int64_t n_primes;            /* P: accumulator rows are [integer part, P residues] */
  const int64_t* piece_euler;  /* [n_pieces] Euler of each piece, numerator ... */
  const int64_t* piece_denom;  /* [n_pieces] ... over its tet's L_t (rpd_pieces order) */
  const int32_t* rpf_off;      /* [n_pieces+1] radical facets of each piece ... */
  const int32_t* rpf_sphere;   /* [n_rpf] ... their neighbour j, ascending */
  const int64_t* rpf_euler;    /* [n_rpf] ... and the Euler of the facet (over the piece's
                                  denominator) */
  const int64_t* rpc_sum;      /* [N] Euler(RPC(m_i)) over this ctx's tets: the exact integer
                                  when rpc_exact[i], else its integer part */
  const uint8_t* rpc_exact;    /* [N] 1: the sum is an integer */
  const double* rpc_value;     /* [N] the sum as a double */
  const int64_t* rpf_sum;      /* [E] Euler(RPF(m_i, m_j)) at the CSR entry of j in row i,
                                  rows sorted ascending by neighbour id (the input order when
                                  the caller's rows are sorted); as rpc_sum */
  const uint8_t* rpf_exact;    /* [E] */
  const double* rpf_value;     /* [E] */
  const int64_t* rpc_acc;      /* [N][1+P] the raw accumulator rows (a sharded job adds them */
  const int64_t* rpf_acc;      /* [E][1+P]  over the ranks, then rpd_euler_finalize) */
  int64_t n_pieces, n_rpf, N, E;
} rpd_euler;
rpd_status rpd_get_euler(rpd_ctx* ctx, rpd_euler* out);

/* Copy the Euler data to caller-owned arrays (host or device; any pointer may be NULL; sizes as
 * in rpd_euler). */
rpd_status rpd_download_euler(rpd_ctx* ctx, int64_t* piece_euler, int64_t* piece_denom,
                              int32_t* rpf_off, int32_t* rpf_sphere, int64_t* rpf_euler,
                              int64_t* rpc_sum, uint8_t* rpc_exact, double* rpc_value,
                              int64_t* rpf_sum, uint8_t* rpf_exact, double* rpf_value,
                              int64_t* rpc_acc, int64_t* rpf_acc);

/* Accumulator rows acc [n_rows][1+P] (device; e.g. rpc_acc summed over the ranks of a sharded
 * job) -> out_sum / out_exact / out_value [n_rows] (device), with the ctx's primes. */
rpd_status rpd_euler_finalize(rpd_ctx* ctx, const int64_t* acc, int64_t n_rows,
                              int64_t* out_sum, uint8_t* out_exact, double* out_value);

/* ---- CC numbers (Sec. 4.1.1)
 *
 * "we can trace their CC numbers using a simple traversal algorithm": the
 * number of connected components of every RPC(m_i) and every RPF(m_i, m_j) (seen from m_i).
 * Two pieces of m_i in tets sharing a face f are connected when f is a facet of both; two of
 * its facets on h_ij in such tets when both have an edge on f (elements of the symbolically
 * perturbed pieces, like the Euler sums; R26-R27).  Union-find on the device over
 * the current pieces; needs rpd_set_euler with the ctx holding the whole mesh
 * (local_ids == NULL, else RPD_ESTATE: a sharded job uses rpd_cc_shard / rpd_cc_merge below)
 * before the last rpd_clip / rpd_update_partial.
 * Outputs (ctx-owned device arrays, valid until the next mutating call):
 *   rpc_cc     [N]        components of RPC(m_i) (0: no cell)
 *   rpf_cc     [E]        components of RPF(m_i, m_j) at the CSR entry of j in row i (rows
 *                         sorted ascending; 0: no face)
 *   piece_comp [n_pieces] component label of every piece (its smallest piece index) -- the
 *                         paper picks a surface point on a component other than m_i's own
 *   rpf_comp   [n_rpf]    component label of every radical facet (smallest rpf index)
 *   piece_sosfm[n_pieces] tet faces that are facets of the piece (bit k: face k)
 *   rpf_fm     [n_rpf]    tet faces the radical facet has an edge on
 *   rpf_adj    [n_rpf]    the piece's radical facets this one shares an edge with (bit b: the
 *                         piece's b-th rpf entry): its restricted power edges RPE(m_i, m_j,
 *                         m_k).  A piece with more than 64 radical facets fails the clip with
 *                         RPD_EOVERFLOW in Euler mode (never seen: pieces have <= 20 planes) */
typedef struct {
  const int32_t* rpc_cc;
  const int32_t* rpf_cc;
  const int32_t* piece_comp;
  const int32_t* rpf_comp;
  const uint8_t* piece_sosfm;
  const uint8_t* rpf_fm;
  const uint64_t* rpf_adj;
  int64_t n_pieces, n_rpf, N, E;
} rpd_topology;
rpd_status rpd_get_topology(rpd_ctx* ctx, rpd_topology* out);

/* CC numbers of a tet-SHARDED job (the tets are split over ranks, every
 * rank's ctx built with rpd_set_euler(local_ids = its tets)): a distributed union-find
 * (DESIGN.md §10 "CC numbers of a sharded job").
 * rpd_cc_shard: joins the rank's pieces / radical facets across its interior faces and
 *   returns the records of its shard-boundary faces (ctx-owned device arrays, valid until the
 *   next mutating call): RPC records key_c = (f << 21 | i) -- f the smaller 4 t + k id of the
 *   shared face (global tet ids), i the sphere -- with lab_c = the global id of the piece's
 *   local component (piece_base + its smallest local piece index); RPF records key_f, j_f (the
 *   facet's neighbour sphere), lab_f (rpf_base + ...).  piece_base / rpf_base: the sum of the
 *   lower ranks' n_pieces / n_rpf (rpd_get_euler).  N < 2^21.  RPD_ESTATE without sharded
 *   Euler data (a whole-mesh ctx uses rpd_get_topology).
 * rpd_cc_merge: the records of ALL ranks (concatenated in any order; device arrays) ->
 *   this rank's counts [N + E] (device, caller-owned): RPC components of every sphere, then
 *   RPF components of every CSR entry, counted at the components' smallest global ids that
 *   lie on this rank -- the sum over ranks (an all-reduce) gives rpd_topology's rpc_cc and
 *   rpf_cc of the whole mesh. */
typedef struct {
  const uint64_t* key_c;
  const int32_t* lab_c;
  int64_t n_c;
  const uint64_t* key_f;
  const int32_t* j_f;
  const int32_t* lab_f;
  int64_t n_f;
  int64_t n_pieces, n_rpf;
} rpd_cc_records;
rpd_status rpd_cc_shard(rpd_ctx* ctx, int64_t piece_base, int64_t rpf_base, rpd_cc_records* out);
rpd_status rpd_cc_merge(rpd_ctx* ctx, const uint64_t* key_c, const int32_t* lab_c, int64_t n_c,
                        const uint64_t* key_f, const int32_t* j_f, const int32_t* lab_f,
                        int64_t n_f, int64_t total_pieces, int64_t total_rpf, int32_t* counts);

/* Restricted power edges of a tet-SHARDED job: the per-(i, j, k) Euler
 * characteristics and CC numbers of the whole mesh from the ranks' shards, by the same
 * distributed union-find (DESIGN.md §10 "CC numbers of a sharded job").
 * rpd_rpe_shard: the rank's RPEs (as rpd_get_rpe: per-piece lists and per-key sums over its
 *   tets) joined across its interior faces; out (ctx-owned device arrays): tri_key / tri_euler
 *   [n_tri] -- the keys (i << 42 | j << 21 | k) ascending and their Euler numerators over 2 on
 *   this rank's tets -- and the records of its shard-boundary faces: key_b (f << 21 | i), jk_b
 *   (j << 21 | k), lab_b (rpe_base + the smallest local index of the part's component).
 *   rpe_base: the lower ranks' n_rpe (out->n_rpe).
 * rpd_rpe_merge: the records of ALL ranks (device) -> this rank's component counts per key at
 *   the components' smallest global ids: keys / counts [n] (ctx-owned device arrays).
 * rpd_reduce_by_key: the sums of vals per key, keys ascending (device arrays; out_* sized n
 *   by the caller; *n_out host) -- the ranks' concatenated (tri_key, tri_euler) lists give the
 *   whole mesh's Euler numerators, their (keys, counts) lists its CC numbers.  N < 2^21. */
typedef struct {
  const uint64_t* tri_key;
  const int64_t* tri_euler;
  int64_t n_tri, n_rpe;
  const uint64_t* key_b;
  const uint64_t* jk_b;
  const int32_t* lab_b;
  int64_t n_b;
} rpd_rpe_records;
rpd_status rpd_rpe_shard(rpd_ctx* ctx, int64_t rpe_base, rpd_rpe_records* out);
rpd_status rpd_rpe_merge(rpd_ctx* ctx, const uint64_t* key_b, const uint64_t* jk_b,
                         const int32_t* lab_b, int64_t n_b, int64_t total_rpe,
                         const uint64_t** keys, const int64_t** counts, int64_t* n);
rpd_status rpd_reduce_by_key(rpd_ctx* ctx, const uint64_t* keys, const int64_t* vals, int64_t n,
                             uint64_t* out_keys, int64_t* out_vals, int64_t* n_out);
/* Copy (host or device destinations; any pointer may be NULL). */
rpd_status rpd_download_topology(rpd_ctx* ctx, int32_t* rpc_cc, int32_t* rpf_cc,
                                 int32_t* piece_comp, int32_t* rpf_comp, uint8_t* piece_sosfm,
                                 uint8_t* rpf_fm, uint64_t* rpf_adj);

/* ---- Restricted power edges
 *
 * "we are expecting each restricted element (i.e., RPC, RPF, RPE) to have CC=1 and Euler=1"
 * (PAPER.md:439); "we collect the fractional Euler characteristics for all of its restricted
 * elements (RPCs, RPFs, RPEs)".  RPE(m_i, m_j, m_k) seen from m_i (j < k) is
 * the union of the edges of m_i's pieces lying on both radical planes h_ij and h_ik (elements
 * of the symbolically perturbed pieces, like rpd_get_euler).  Per piece its RPE list; per
 * (i, j, k) the fractional Euler characteristic V - E (exact: tri_euler is a numerator over
 * denom = 2 -- the endpoint payloads are 1 or 1/2; per-piece rpe_euler over the piece's L_t,
 * as rpd_get_euler) and the CC number (the parts glued across shared tet faces at their common
 * endpoint; needs the whole mesh in the ctx, else tri_cc is NULL).  Needs rpd_set_euler before
 * the last rpd_clip / rpd_update_partial (RPD_ESTATE) and N < 2^21 (RPD_EINVAL).
 * Outputs (ctx-owned device arrays, valid until the next mutating call or rpd_get_rpe):
 *   rpe_off [n_pieces+1], rpe_j / rpe_k [n_rpe] (j < k, ascending per piece), rpe_euler
 *   [n_rpe] (numerator over denom), rpe_fm [n_rpe] (bit f: an endpoint on tet face f);
 *   tri [n_tri][3] (i, j, k) ascending, tri_euler [n_tri], tri_cc [n_tri]. */
typedef struct {
  int64_t denom;
  const int32_t* rpe_off;
  const int32_t* rpe_j;
  const int32_t* rpe_k;
  const int64_t* rpe_euler;
  const uint8_t* rpe_fm;
  const int32_t* tri;
  const int64_t* tri_euler;
  const int32_t* tri_cc;
  int64_t n_pieces, n_rpe, n_tri;
} rpd_rpe;
rpd_status rpd_get_rpe(rpd_ctx* ctx, rpd_rpe* out);
/* Copy the last rpd_get_rpe outputs (host or device destinations; NULL skips); RPD_ESTATE
 * before any rpd_get_rpe. */
rpd_status rpd_download_rpe(rpd_ctx* ctx, int32_t* rpe_off, int32_t* rpe_j, int32_t* rpe_k,
                            int64_t* rpe_euler, uint8_t* rpe_fm, int32_t* tri,
                            int64_t* tri_euler, int32_t* tri_cc);

/* ---- Dual medial mesh
 * "Each sub-domain RPC(m_i) ... is dual to a vertex", "the face shared by two adjacent RPCs
 * (RPF) ... dual to an edge e_ij", "the edge shared by three RPCs (RPE) ... dual to a triangle
 * face f_ijk".  From the current pieces (Euler mode, whole mesh or shard): every radical facet
 * gives the edge (i, j), every restricted power edge of a piece of m_i on h_ij and h_ik the
 * triangle (i, j, k); keys sorted and deduplicated on the device.  Outputs (ctx-owned device
 * arrays, valid until the next mutating call): edges [n_edges][2] (i < j), faces [n_faces][3]
 * (i < j < k), both ascending lexicographically.  A sharded job concatenates the ranks' lists
 * and deduplicates.  Needs N < 2^21 (RPD_EINVAL). */
typedef struct {
  const int32_t* edges;
  const int32_t* faces;
  int64_t n_edges, n_faces;
} rpd_medial;
rpd_status rpd_medial_mesh(rpd_ctx* ctx, rpd_medial* out);
/* Copy the last extraction to caller-owned arrays (host or device; NULL skips): edges
 * [n_edges][2], faces [n_faces][3].  RPD_ESTATE before any rpd_medial_mesh. */
rpd_status rpd_download_medial_mesh(rpd_ctx* ctx, int32_t* edges, int32_t* faces);

/* ---- Multi-GPU exchange
 *
 * Each rank computes the RPD of its own tet shard (rpd_relations on its tets); the per-rank
 * candidate and piece CSRs are all-gathered by the caller (NCCL over NVLink) and the calls
 * below put them back into global tet order on the ctx's device -- byte-identical to a
 * single-GPU run of all T tets.  In partial mode only the dirty tets' segments travel
 * (rpd_download_tets of the dirty list) and rpd_merge_shards puts them into the previous
 * global CSR.  Every array is a DEVICE pointer (the gathered buffers): rank r holds n_tets[r]
 * tets (rows) whose global ids are tet_ids[r] (each global tet in at most one rank), with
 * its local CSRs piece_off[r] [n_tets[r]+1] ... inc_sphere[r] and cand_off[r] / cand_idx[r].
 * RPD_EINVAL: world outside [1, RPD_MAX_RANKS], a NULL array that the call needs, or a tet id
 * outside [0, T) (checked on the device before any copy). */
#define RPD_MAX_RANKS 16
typedef struct {
  int32_t world;
  int64_t T;
  int64_t n_tets[RPD_MAX_RANKS];
  const int32_t* tet_ids[RPD_MAX_RANKS];
  const int32_t* piece_off[RPD_MAX_RANKS];
  const int32_t* piece_sphere[RPD_MAX_RANKS];
  const double* piece_vol[RPD_MAX_RANKS];
  const double* piece_m1[RPD_MAX_RANKS];
  const uint8_t* piece_facemask[RPD_MAX_RANKS];
  const int32_t* inc_off[RPD_MAX_RANKS];
  const int32_t* inc_sphere[RPD_MAX_RANKS];
  const int32_t* cand_off[RPD_MAX_RANKS];   /* candidate CSR (rpd_gather_cands, merge) */
  const int32_t* cand_idx[RPD_MAX_RANKS];
} rpd_shards;

/* A whole candidate + piece CSR over T tets (layouts as rpd_relations / rpd_pieces). */
typedef struct {
  int32_t* cand_off;      /* [T+1] */
  int32_t* cand_idx;      /* [n_cand] */
  int32_t* piece_off;     /* [T+1] */
  int32_t* piece_sphere;  /* [n_pieces] */
  double* piece_vol;      /* [n_pieces] */
  double* piece_m1;       /* [n_pieces][3] */
  uint8_t* piece_facemask;/* [n_pieces] */
  int32_t* inc_off;       /* [n_pieces+1] */
  int32_t* inc_sphere;    /* [n_inc] */
  int64_t T, n_cand, n_pieces, n_inc;
} rpd_csr;

/* Gathered pieces in global tet order.  Outputs (caller-allocated device arrays):
 * piece_off [T+1], piece_sphere / piece_vol / piece_facemask [sum n_pieces], piece_m1
 * [3 sum n_pieces], inc_off [sum n_pieces + 1], inc_sphere [sum n_inc]. */
rpd_status rpd_gather_pieces(rpd_ctx* ctx, const rpd_shards* shards, int32_t* piece_off,
                             int32_t* piece_sphere, double* piece_vol, double* piece_m1,
                             uint8_t* piece_facemask, int32_t* inc_off, int32_t* inc_sphere);
/* Gathered candidate CSR in global tet order: cand_off [T+1], cand_idx [sum n_cand]
 * (caller-allocated device arrays). */
rpd_status rpd_gather_cands(rpd_ctx* ctx, const rpd_shards* shards, int32_t* cand_off,
                            int32_t* cand_idx);
/* Partial-mode merge: the global CSR `old` (device arrays, any owner) with the rows of the
 * dirty tets replaced by the shards' segments (shards: per rank its dirty tets' global ids
 * and their candidate + piece CSRs); every other row is copied unchanged.  The result is
 * written to ctx-owned device arrays returned in *out (valid until the next-but-one
 * rpd_merge_shards or destroy: `old` may be the previous call's output).  One host sync. */
rpd_status rpd_merge_shards(rpd_ctx* ctx, const rpd_shards* dirty, const rpd_csr* old,
                            rpd_csr* out);
/* The candidate and piece segments of the ctx's tets `tet_list` [n] (local ids, host or
 * device; e.g. the dirty tets of the last rpd_update_partial) as one CSR over the list, into
 * caller-allocated arrays in *out (host or device; cand_* or piece_* all NULL: that part is
 * skipped).  All destination pointers NULL: only the sizes are computed.  Always sets out->T
 * = n and out->n_cand / n_pieces / n_inc.  ids_out [n] (may be NULL) receives the global id
 * id_map[tet_list[k]] of every listed tet (id_map [T_local], host or device; NULL: the local
 * id).  RPD_EINVAL: a listed tet outside [0, T_local); RPD_ESTATE before rpd_clip. */
rpd_status rpd_download_tets(rpd_ctx* ctx, const int32_t* tet_list, int64_t n,
                             const int32_t* id_map, int32_t* ids_out, rpd_csr* out);
/* Validation aggregate of a sharded job (SURVEY.md §8(e) "per-sphere RPC volume ... all_reduce
 * sum"): out [N] (host or device, caller-owned) = the volume of every sphere's restricted power
 * cell over the ctx's tets, i.e. the sum of its pieces' volumes (fp64 atomics: the summation
 * order, hence the last bits, may vary between runs); a sharded job all-reduces the ranks'
 * vectors.  RPD_ESTATE before rpd_clip. */
rpd_status rpd_sphere_volumes(rpd_ctx* ctx, double* out);

/* ---- Envelope distance (Sec. 4.3)
 *
 * "For each surface sample, we compute its distance to the closest enveloping volume of the
 * medial mesh (sphere, cone, slab ...) in GPU".  A cone is the family of spheres linearly
 * interpolated between two medial spheres, a slab between three; the value of a primitive at
 * p is min over the interpolation parameters of |p - c| - r and the envelope distance is
 * max(min over primitives, 0).  Exact closed forms in fp64, brute force over
 * all primitives with exact tile culling.
 *   samples [S][3] double, spheres [N][4] double (x, y, z, r), edges [NE][2] / faces [NF][3]
 *   int32 sphere ids (e.g. the medial mesh of rpd_medial_mesh); host or device pointers
 *   g_out [S] double     the minimum value (negative inside the envelope)
 *   prim_out [S] int32   the primitive reaching it (sphere i -> i, edge e -> N + e, face f ->
 *                        N + NE + f; the smallest index among equal values)
 *   *n_eval (host, may be NULL): (sample, primitive) pairs evaluated after culling
 * No lattice requirement (geometry only; no combinatorial output). */
rpd_status rpd_envelope(rpd_ctx* ctx, const double* samples, int64_t S, const double* spheres,
                        int64_t N, const int32_t* edges, int64_t NE, const int32_t* faces,
                        int64_t NF, double* g_out, int32_t* prim_out, int64_t* n_eval);

/* ---- Sphere neighbours on the GPU
 *
 * "we use the Regular Triangulation in CGAL to compute all possible neighbors (k_site) of a
 * given sphere";
 * the neighbour lists are the k_site input of rpd_relations.  This call computes a certified
 * SUPERSET of the neighbours whose radical plane holds a positive-area facet of the power cell
 * restricted to the axis box `box` (DESIGN.md §10 "Sphere neighbours"): the RPD of any tets
 * inside the box is the same as with the regular-triangulation lists (redundant planes do not
 * change a piece), and every list may hold a few redundant spheres.
 *   spheres [N][4] double (x, y, z, r), host or device; no lattice requirement
 *   box     host double[6] = (lo_x, lo_y, lo_z, hi_x, hi_y, hi_z), e.g. the mesh's bounds
 * Outputs (ctx-owned DEVICE arrays, valid until the next rpd_neighbors or destroy; they can be
 * passed straight to rpd_relations / rpd_update_partial): nbr_off [N+1], nbr_idx [E], rows
 * ascending, no self or same-centre entries.  A sphere hidden by a same-centre sphere with a
 * larger radius (equal radius: the smaller id wins) or whose cell misses the box gets an empty
 * row; if a cell covers the whole box its row lists one redundant sphere (so that R4 does not
 * apply).  n_hidden counts the former; n_vertex_overflow counts spheres whose bounding
 * polytope overflowed the vertex buffer (their lists are computed against the whole box --
 * still a superset).  RPD_EINVAL: NULL arguments, non-finite box or lo > hi, NaN / Inf sphere
 * values or a negative radius. */
typedef struct {
  const int32_t* nbr_off;
  const int32_t* nbr_idx;
  int64_t N, E;
  int64_t n_hidden, n_vertex_overflow;
  int64_t n_rows_computed;  /* rows computed by this call (N for rpd_neighbors) */
  int64_t n_rows_block;     /* of these, rows computed by a whole block (the new rows of an
                               incremental update of at most 2048 spheres, or rows with more
                               than RPD_NB_HEAVY spheres in their first search ball; the same
                               rows as a warp would give) */
} rpd_nbr_lists;
rpd_status rpd_neighbors(rpd_ctx* ctx, const double* spheres, int64_t N, const double* box,
                         rpd_nbr_lists* out);
/* Incremental lists after appending M spheres (the paper recomputes the neighbours at every
 * insertion; its spheres are inserted a few at a time):
 * spheres [N][4] are the previous call's N - M spheres, unchanged, followed by M new ones;
 * `box` must be the previous call's.  The rows of the new spheres are computed as by
 * rpd_neighbors; every old row is kept and extended by the new spheres whose radical plane
 * reaches the ball stored around its last bounding polytope (cells only shrink when spheres
 * are added, so the new neighbours of an old sphere are old neighbours or new spheres: a
 * certified superset again, DESIGN.md §10 "Sphere neighbours", reading R34); an old sphere
 * that a new one hides (same centre, larger radius) gets an empty row.  Same outputs and
 * lifetime as rpd_neighbors (n_hidden / n_vertex_overflow / n_rows_block count the new rows
 * only; n_rows_computed = M + the old rows extended or emptied).  RPD_ESTATE: no previous lists of N - M
 * spheres or another box; RPD_EINVAL: as rpd_neighbors, or an old sphere changed. */
rpd_status rpd_neighbors_update(rpd_ctx* ctx, const double* spheres, int64_t N, int64_t M,
                                const double* box, rpd_nbr_lists* out);
/* Copy the last lists to caller-owned arrays (host or device; NULL skips).  RPD_ESTATE before
 * any rpd_neighbors. */
rpd_status rpd_download_neighbors(rpd_ctx* ctx, int32_t* nbr_off, int32_t* nbr_idx);

/* Counters of the last call (host).  Algorithmic counts are what the method computed (for
 * the roofline), kernel_launches counts this library's kernel launches since rpd_create. */
typedef struct {
  int64_t T, N, n_cand, n_pieces, n_inc, n_dirty;
  int64_t pairs_filtered;        /* (tet, sphere) pairs whose Alg. 1 boolean was decided */
  int64_t pairs_tested;          /* pairs on which Alg. 1 was actually evaluated (pruned mode) */
  int64_t pairs_clipped;         /* candidate pairs clipped by the last call */
  int64_t exact_fallbacks;       /* clip predicates decided by the int128 path */
  int64_t zero_hits;             /* exact-zero predicates resolved by symbolic perturbation */
  int64_t kernel_launches;
  int32_t max_k_tet, max_vertices, max_planes;
  int32_t n_wide;                /* pairs re-clipped by the wide kernel */
  /* algorithmic work counted by the kernels */
  int64_t rel_tests;             /* literal Alg. 1 vertex tests (inner break, outer early exit) */
  int64_t clip_plane_evals;      /* (pair, neighbour plane) corner classifications */
  int64_t clip_vertex_tests;     /* vertex sign tests of cutting candidates */
  int64_t clip_constructions;    /* new vertices */
  int64_t clip_fan_triangles;    /* fan triangles integrated for volume and first moment */
  double filter_ms, clip_ms;     /* kernel times of the last call (RPD_OPT_PROFILE only) */
  /* rpd_update_partial: sizes of the dirty tets' new segments (what a sharded job exchanges) */
  int64_t n_cand_dirty, n_pieces_dirty, n_inc_dirty;
  /* CUDA-graph partial updates since rpd_create (RPD_OPT_GRAPH): replays, captures (one per
   * buffer layout), and replays whose batch was redone eagerly (a device-side capacity check
   * failed: work queue, slab, pool room or the graph's batch bound) */
  int64_t graph_updates, graph_captures, graph_fallbacks;
} rpd_stats;
rpd_status rpd_get_stats(rpd_ctx* ctx, rpd_stats* out);

/* Library version string. */
const char* rpd_version(void);

/* Debugging aid (env RPD_CANARY=1 at the first allocation: every library buffer carries a
 * 256-byte canary past its capacity): RPD_ECUDA if any live buffer's canary was overwritten
 * (a write past its end), after synchronising the device; RPD_OK otherwise or when off. */
rpd_status rpd_debug_check(rpd_ctx* ctx);

#ifdef __cplusplus
}
#endif
#endif /* RPD_H */
