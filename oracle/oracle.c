/*
 * oracle.c -- plain, slow, obviously-correct CPU oracle of the RPD hot path of
 * MATTopo (arXiv 2403.18761).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library.  It shares no code with
 * paper_2403_18761_b200/ (the CUDA path) and neither includes the other.
 *
 * What it computes (DESIGN.md §"Oracle"):
 *
 *   PD(m, x)       = |x - theta|^2 - r^2                       PAPER.md:40 (Alg. 1)
 *   rel(t, i)      Alg. 1, prose reading (R1): for every neighbour j of i, some vertex v of t
 *                  is strictly power-closer to m_i than to m_j  (PD_i(v) < PD_j(v), R2);
 *                  rel = (d == k_site(i)).  k_site(i) = 0: rel = (N == 1) (R4).
 *                                                              PAPER.md:21-50, 26
 *   cand(t)        ascending i with rel(t, i)                  PAPER.md:28 ("k_tet")
 *   P(t, i)        = t  intersected with  { x : PD_i(x) <= PD_j(x) }  for j in N(i)
 *                  (radical half-spaces of i against its power neighbours)
 *                                                              PAPER.md:18, 380-384, 488
 *   pieces         non-empty P(t, i) (vol > 0) with volume, first moment, tet-face mask and
 *                  the ascending ids j whose radical plane holds a positive-area 2-face of P
 *                  (all coincident sources listed, R7)
 *
 * Representation (plain, checkable by eye).  All inputs are multiples of 2^-10 in [0,64)^3;
 * the oracle converts them to lattice integers X = 2^10 x, so every power distance is an
 * int64.  A piece is written in the barycentric coordinates lambda of its tet t:
 *   t            = { lambda >= 0, sum lambda = 1 }
 *   tet face k   = the half-space  e_k . lambda >= 0                (face opposite vertex k)
 *   radical j    = the half-space  g_j . lambda >= 0,  g_j[k] = PD_j(V_k) - PD_i(V_k)
 * (PD_j - PD_i is affine, so its value at a point is the lambda-weighted sum of its values at
 * the four tet vertices).  Every plane is an integer 4-vector, |entries| < 2^35.4.
 *
 * Clipping: start from the tet (4 face planes, 4 corner
 * vertices, each vertex = the triplet of planes through it); for each j in N(i), ascending:
 * sign every vertex against plane j; no '-' -> skip; no '+' -> empty; otherwise drop the '-'
 * vertices and, for each edge (two vertices sharing two planes) from '+' to '-', add the
 * vertex (shared planes) + {j}.
 *
 * Exact signs with symbolic perturbation (C4).  For vertex v = (p,q,r) and plane s:
 *   D4 = det[a_p; a_q; a_r; a_s],   D3 = det[a_p; a_q; a_r; 1]   (1 = (1,1,1,1))
 *   h_s(v) = D4 / D3  (plane value at the vertex).
 * Every plane is perturbed inward, a_k -> a_k - eps^rank(k) * 1 with rank(radical j) = j and
 * rank(face k) = N + k, so D4(eps) = D4 - sum_k eps^rank(k) C_k with C_k = det(rows, row k
 * replaced by 1).  sign = sign(D4) sign(D3) if D4 != 0, else -sign(C_k*) sign(D3) for the
 * lowest-rank k with C_k != 0 (C_s = D3 != 0 always exists).  Determinants are evaluated
 * exactly by the Leibniz formula in 256-bit integers.
 *
 * Output per non-empty piece (C1 step 7): SoS facets = planes in vertex triplets; a facet
 * has zero area iff some other plane q of its vertex triplets has D4(v, q) = 0 at every one
 * of its vertices; every positive-area facet s lists every source q of S(t,i) = {4 faces} u
 * N(i) whose plane vector is a positive multiple of a_s.  Volume and first moment: vertex
 * lambda = K / sum(K) (K = exact 3x3 cofactors), Cartesian x = V0 + sum lambda_k (V_k - V0),
 * facets walked cyclically and fan-triangulated against the vertex average.
 */
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

typedef __int128 i128;
typedef unsigned __int128 u128;

/* ------------------------------------------------------------------ 256-bit integers */

typedef struct { uint64_t w[4]; } i256;  /* two's complement, little-endian limbs */

static i256 i256_zero(void) { i256 r = {{0, 0, 0, 0}}; return r; }

static i256 i256_add(i256 a, i256 b) {
  i256 r;
  u128 c = 0;
  for (int k = 0; k < 4; ++k) {
    u128 s = (u128)a.w[k] + b.w[k] + c;
    r.w[k] = (uint64_t)s;
    c = s >> 64;
  }
  return r;
}

static i256 i256_neg(i256 a) {
  i256 r;
  for (int k = 0; k < 4; ++k) r.w[k] = ~a.w[k];
  i256 one = {{1, 0, 0, 0}};
  return i256_add(r, one);
}

static int i256_sign(i256 a) {
  if ((int64_t)a.w[3] < 0) return -1;
  if (a.w[0] | a.w[1] | a.w[2] | a.w[3]) return 1;
  return 0;
}

/* exact product of two signed 128-bit integers (|x| < 2^127) */
static i256 i256_mul(i128 x, i128 y) {
  int neg = (x < 0) != (y < 0);
  u128 a = x < 0 ? (u128)(-x) : (u128)x;
  u128 b = y < 0 ? (u128)(-y) : (u128)y;
  uint64_t a0 = (uint64_t)a, a1 = (uint64_t)(a >> 64);
  uint64_t b0 = (uint64_t)b, b1 = (uint64_t)(b >> 64);
  u128 p00 = (u128)a0 * b0, p01 = (u128)a0 * b1, p10 = (u128)a1 * b0, p11 = (u128)a1 * b1;
  i256 r = i256_zero();
  r.w[0] = (uint64_t)p00;
  u128 mid = (p00 >> 64) + (uint64_t)p01 + (uint64_t)p10;
  r.w[1] = (uint64_t)mid;
  u128 hi = (mid >> 64) + (p01 >> 64) + (p10 >> 64) + (uint64_t)p11;
  r.w[2] = (uint64_t)hi;
  r.w[3] = (uint64_t)((hi >> 64) + (p11 >> 64));
  return neg ? i256_neg(r) : r;
}

/* det of a 4x4 matrix of int64 entries (|entries| < 2^40) by the Leibniz formula */
static const int PERM4[24][4] = {
    {0, 1, 2, 3}, {0, 1, 3, 2}, {0, 2, 1, 3}, {0, 2, 3, 1}, {0, 3, 1, 2}, {0, 3, 2, 1},
    {1, 0, 2, 3}, {1, 0, 3, 2}, {1, 2, 0, 3}, {1, 2, 3, 0}, {1, 3, 0, 2}, {1, 3, 2, 0},
    {2, 0, 1, 3}, {2, 0, 3, 1}, {2, 1, 0, 3}, {2, 1, 3, 0}, {2, 3, 0, 1}, {2, 3, 1, 0},
    {3, 0, 1, 2}, {3, 0, 2, 1}, {3, 1, 0, 2}, {3, 1, 2, 0}, {3, 2, 0, 1}, {3, 2, 1, 0}};

static int perm_parity(const int* p) {
  int inv = 0;
  for (int a = 0; a < 4; ++a)
    for (int b = a + 1; b < 4; ++b)
      if (p[a] > p[b]) ++inv;
  return (inv & 1) ? -1 : 1;
}

static i256 det4(const int64_t* r0, const int64_t* r1, const int64_t* r2, const int64_t* r3) {
  i256 acc = i256_zero();
  for (int k = 0; k < 24; ++k) {
    const int* p = PERM4[k];
    i128 x = (i128)r0[p[0]] * r1[p[1]];
    i128 y = (i128)r2[p[2]] * r3[p[3]];
    i256 t = i256_mul(x, y);
    acc = i256_add(acc, perm_parity(p) > 0 ? t : i256_neg(t));
  }
  return acc;
}

/* ------------------------------------------------------------------ inputs */

typedef struct {
  int64_t V, T, N;
  const double* verts;
  const int32_t* tets;
  const double* spheres;
  const int32_t* nbr_off;
  const int32_t* nbr_idx;
  int brute; /* 1: cand(t) = all spheres and N(i) = all j != i (C1 step 8) */
  int euler; /* 1: fractional Euler characteristics of the pieces */
} oracle_input;

typedef struct {
  int64_t n_tets;
  int32_t *cand_off, *cand_idx;
  int64_t n_cand;
  int32_t *piece_off, *piece_sphere;
  double *piece_vol, *piece_m1;
  uint8_t* piece_facemask;
  int32_t *inc_off, *inc_sphere;
  int64_t n_pieces, n_inc;
  /* fractional Euler characteristics (euler = 1): exact rationals.  Every value of a piece is a
     numerator over its tet's denominator L_t = lcm of the tet's 14 sharing counts */
  int64_t euler_denom;           /* unused (0): the denominators are per tet */
  int64_t* piece_euler;          /* [n_pieces] Euler of the piece's fractional complex (num) */
  int64_t* piece_euler_den;      /* [n_pieces] its denominator L_t */
  int32_t *rpf_off, *rpf_sphere; /* [n_pieces + 1], [n_rpf]: radical facets j, ascending */
  int64_t* rpf_euler;            /* [n_rpf] Euler of the piece's facet on h_ij */
  uint8_t* piece_sosfm;          /* [n_pieces] tet faces that are facets of the piece (SoS) */
  uint8_t* rpf_fm;               /* [n_rpf] tet faces the radical facet has an edge on (SoS) */
  uint64_t* rpf_adj;             /* [n_rpf] the piece's radical facets (bit = rank by ascending
                                    j) this one shares an edge with: restricted power edges */
  int64_t n_rpf;
  /* restricted power edges RPE(m_i, m_j, m_k) of every piece: the
     piece's edge on the radical planes h_ij and h_ik, j < k, ascending (j, k) */
  int32_t *rpe_off, *rpe_j, *rpe_k; /* [n_pieces + 1], [n_rpe], [n_rpe] */
  int64_t* rpe_euler;            /* [n_rpe] its fractional Euler characteristic V - E over L */
  uint8_t* rpe_fm;               /* [n_rpe] tet faces holding an endpoint of the edge */
  int64_t n_rpe;
  /* instrumentation (C1 step 9) */
  int64_t n_rel_tests, n_clip_tests, n_constructions, n_fan_triangles, n_zero_hits;
  int status;
  char err[256];
} oracle_result;

static int64_t lat(double x) { return (int64_t)llround(x * 1024.0); }
static const int64_t ONE4[4] = {1, 1, 1, 1};

/* power distance in lattice units^2:  PD(m, x) = |x - theta|^2 - r^2 */
static int64_t pd_lat(const int64_t* X, const int64_t* S /* x,y,z,r lattice */) {
  int64_t dx = X[0] - S[0], dy = X[1] - S[1], dz = X[2] - S[2];
  return dx * dx + dy * dy + dz * dz - S[3] * S[3];
}

double oracle_power_distance(const double* sphere, const double* x) {
  double dx = x[0] - sphere[0], dy = x[1] - sphere[1], dz = x[2] - sphere[2];
  return dx * dx + dy * dy + dz * dz - sphere[3] * sphere[3];
}

static int check_input(const oracle_input* in, char* err) {
  for (int64_t v = 0; v < in->V * 3; ++v) {
    double x = in->verts[v];
    if (!(x >= 0.0 && x < 64.0) || (double)lat(x) != x * 1024.0) {
      snprintf(err, 256, "vertex coordinate %g not a multiple of 2^-10 in [0,64)", x);
      return -6;
    }
  }
  for (int64_t i = 0; i < in->N; ++i)
    for (int c = 0; c < 4; ++c) {
      double x = in->spheres[4 * i + c];
      if (!(x >= 0.0 && x < 64.0) || (double)lat(x) != x * 1024.0) {
        snprintf(err, 256, "sphere %lld value %g not a multiple of 2^-10 in [0,64)",
                 (long long)i, x);
        return -6;
      }
    }
  for (int64_t t = 0; t < in->T; ++t) {
    int64_t P[4][3];
    for (int k = 0; k < 4; ++k) {
      int32_t v = in->tets[4 * t + k];
      if (v < 0 || v >= in->V) {
        snprintf(err, 256, "tet %lld vertex index out of range", (long long)t);
        return -1;
      }
      for (int c = 0; c < 3; ++c) P[k][c] = lat(in->verts[3 * v + c]);
    }
    int64_t a[3], b[3], d[3];
    for (int c = 0; c < 3; ++c) {
      a[c] = P[1][c] - P[0][c];
      b[c] = P[2][c] - P[0][c];
      d[c] = P[3][c] - P[0][c];
    }
    i128 det = (i128)a[0] * ((i128)b[1] * d[2] - (i128)b[2] * d[1]) -
               (i128)a[1] * ((i128)b[0] * d[2] - (i128)b[2] * d[0]) +
               (i128)a[2] * ((i128)b[0] * d[1] - (i128)b[1] * d[0]);
    if (det <= 0) {
      snprintf(err, 256, "tet %lld not positively oriented", (long long)t);
      return -1;
    }
  }
  if (!in->brute) {
    for (int64_t i = 0; i < in->N; ++i)
      for (int32_t e = in->nbr_off[i]; e < in->nbr_off[i + 1]; ++e) {
        int32_t j = in->nbr_idx[e];
        if (j < 0 || j >= in->N || j == i) {
          snprintf(err, 256, "bad neighbour %d of sphere %lld", j, (long long)i);
          return -1;
        }
      }
  }
  return 0;
}

/* neighbour list of sphere i (brute mode: all j != i ascending) */
static int32_t nbr_count(const oracle_input* in, int64_t i) {
  if (in->brute) return (int32_t)(in->N - 1);
  return in->nbr_off[i + 1] - in->nbr_off[i];
}
static int32_t nbr_at(const oracle_input* in, int64_t i, int32_t e) {
  if (in->brute) return e < i ? e : e + 1;
  return in->nbr_idx[in->nbr_off[i] + e];
}

/* ------------------------------------------------------------------ Alg. 1 */

typedef struct {
  int64_t X[4][3];   /* tet vertices, lattice */
} tet_lat;

static void load_tet(const oracle_input* in, int64_t t, tet_lat* tl) {
  for (int k = 0; k < 4; ++k) {
    int32_t v = in->tets[4 * t + k];
    for (int c = 0; c < 3; ++c) tl->X[k][c] = lat(in->verts[3 * v + c]);
  }
}

static void load_sphere(const oracle_input* in, int64_t i, int64_t* S) {
  for (int c = 0; c < 4; ++c) S[c] = lat(in->spheres[4 * i + c]);
}

/* Alg. 1, prose reading R1 with strict comparison R2; hidden R4.  The outer
 * loop stops at the first neighbour with no success: d can then no longer reach k_site, so
 * the returned boolean is identical to the literal loop. */
static int relation(const oracle_input* in, const tet_lat* tl, int64_t i, int64_t* n_tests) {
  int32_t k_site = nbr_count(in, i);
  if (k_site == 0) return in->N == 1;
  int64_t Si[4], Sj[4];
  load_sphere(in, i, Si);
  int32_t d = 0;
  for (int32_t e = 0; e < k_site; ++e) {
    load_sphere(in, nbr_at(in, i, e), Sj);
    int hit = 0;
    for (int v = 0; v < 4; ++v) {
      ++*n_tests;
      if (pd_lat(tl->X[v], Si) < pd_lat(tl->X[v], Sj)) { /* closer to m_i than m_j */
        hit = 1;
        break;
      }
    }
    if (!hit) break;
    ++d;
  }
  return d == k_site;
}

/* literal relation matrix for tests: out[t * (hi-lo) + (i-lo)] */
int oracle_relation_matrix(const oracle_input* in, const int32_t* tet_ids, int64_t n_tets,
                           int64_t sphere_lo, int64_t sphere_hi, uint8_t* out, int nthreads) {
  char err[256];
  int st = check_input(in, err);
  if (st) return st;
#ifdef _OPENMP
  if (nthreads > 0) omp_set_num_threads(nthreads);
#pragma omp parallel for schedule(dynamic, 16)
#endif
  for (int64_t a = 0; a < n_tets; ++a) {
    tet_lat tl;
    int64_t dummy = 0;
    load_tet(in, tet_ids ? tet_ids[a] : a, &tl);
    for (int64_t i = sphere_lo; i < sphere_hi; ++i)
      out[a * (sphere_hi - sphere_lo) + (i - sphere_lo)] = (uint8_t)relation(in, &tl, i, &dummy);
  }
  return 0;
}

/* ------------------------------------------------------------------ fractional Euler payloads
 *
 * PAPER.md:488-491 (Sec. 4.1.2, Fig. 5): "such fractional Euler characteristics are inputted
 * together with the mesh, based on the combinatorial structure of the tetrahedral mesh" -- every
 * vertex / edge / face of the tet complex carries 1 / (number of tets sharing it) inside each
 * of those tets ("both vertex b or d are shared between A and B, so their fractional Euler
 * characteristic inside each triangle is only 1/2"), a tet carries 1.  The oracle keeps every
 * payload as an exact integer numerator over the tet's own denominator L_t = lcm of the 14
 * sharing counts of its elements: payload(element) = L_t / count (so any mesh works: no common
 * denominator of the whole mesh is formed; per-sphere sums are exact Fractions in Python).
 *
 * Per tet t, A[14 t + m]: m = 0..3 corners, 4..9 edges (corner pairs 01 02 03 12 13 23),
 * 10..13 faces (face k opposite corner k).  Counts come from sorting the keys of all
 * simplices of all tets (plain counting, no hashing). */

typedef struct { int32_t v[3]; } key3;

static int cmp_i64(const void* a, const void* b) {
  int64_t x = *(const int64_t*)a, y = *(const int64_t*)b;
  return (x > y) - (x < y);
}
static int cmp_key3(const void* a, const void* b) {
  const key3 *x = (const key3*)a, *y = (const key3*)b;
  for (int k = 0; k < 3; ++k)
    if (x->v[k] != y->v[k]) return x->v[k] < y->v[k] ? -1 : 1;
  return 0;
}
static void sort3(int32_t* a) {
  for (int p = 0; p < 3; ++p)
    for (int q = p + 1; q < 3; ++q)
      if (a[q] < a[p]) { int32_t t = a[p]; a[p] = a[q]; a[q] = t; }
}
static int64_t gcd64(int64_t a, int64_t b) {
  while (b) { int64_t t = a % b; a = b; b = t; }
  return a;
}
/* number of entries equal to the key in a sorted array */
static int64_t count_i64(const int64_t* sorted, int64_t n, int64_t key) {
  int64_t lo = 0, hi = n;  /* first >= key */
  while (lo < hi) { int64_t m = (lo + hi) / 2; if (sorted[m] < key) lo = m + 1; else hi = m; }
  int64_t c = 0;
  while (lo + c < n && sorted[lo + c] == key) ++c;
  return c;
}
static int64_t count_key3(const key3* sorted, int64_t n, const key3* key) {
  int64_t lo = 0, hi = n;
  while (lo < hi) { int64_t m = (lo + hi) / 2; if (cmp_key3(&sorted[m], key) < 0) lo = m + 1; else hi = m; }
  int64_t c = 0;
  while (lo + c < n && cmp_key3(&sorted[lo + c], key) == 0) ++c;
  return c;
}

static const int EDGE_CORNERS[6][2] = {{0, 1}, {0, 2}, {0, 3}, {1, 2}, {1, 3}, {2, 3}};

/* payload numerators of every element of every tet over the tet's denominator L_t (Lt[t]);
 * 0, or -2 if some L_t exceeds 2^62 */
static int euler_payloads(const oracle_input* in, int64_t** A_out, int64_t** Lt_out) {
  int64_t T = in->T, n = T > 0 ? T : 1;
  int64_t* cnt14 = (int64_t*)malloc(sizeof(int64_t) * 14 * n);
  int64_t* vkeys = (int64_t*)malloc(sizeof(int64_t) * 4 * n);
  int64_t* ekeys = (int64_t*)malloc(sizeof(int64_t) * 6 * n);
  key3* fkeys = (key3*)malloc(sizeof(key3) * 4 * n);
  for (int64_t t = 0; t < T; ++t) {
    const int32_t* tv = in->tets + 4 * t;
    for (int k = 0; k < 4; ++k) vkeys[4 * t + k] = tv[k];
    for (int e = 0; e < 6; ++e) {
      int64_t a = tv[EDGE_CORNERS[e][0]], b = tv[EDGE_CORNERS[e][1]];
      ekeys[6 * t + e] = a < b ? a * in->V + b : b * in->V + a;
    }
    for (int k = 0; k < 4; ++k) {
      key3 f;
      int m2 = 0;
      for (int m = 0; m < 4; ++m)
        if (m != k) f.v[m2++] = tv[m];
      sort3(f.v);
      fkeys[4 * t + k] = f;
    }
  }
  int64_t* vs = (int64_t*)malloc(sizeof(int64_t) * 4 * n);
  int64_t* es = (int64_t*)malloc(sizeof(int64_t) * 6 * n);
  key3* fs = (key3*)malloc(sizeof(key3) * 4 * n);
  memcpy(vs, vkeys, sizeof(int64_t) * 4 * T);
  memcpy(es, ekeys, sizeof(int64_t) * 6 * T);
  memcpy(fs, fkeys, sizeof(key3) * 4 * T);
  qsort(vs, 4 * T, sizeof(int64_t), cmp_i64);
  qsort(es, 6 * T, sizeof(int64_t), cmp_i64);
  qsort(fs, 4 * T, sizeof(key3), cmp_key3);
  int64_t* Lt = (int64_t*)malloc(sizeof(int64_t) * n);
  int st = 0;
  for (int64_t t = 0; t < T; ++t) {
    for (int k = 0; k < 4; ++k) cnt14[14 * t + k] = count_i64(vs, 4 * T, vkeys[4 * t + k]);
    for (int e = 0; e < 6; ++e) cnt14[14 * t + 4 + e] = count_i64(es, 6 * T, ekeys[6 * t + e]);
    for (int k = 0; k < 4; ++k) cnt14[14 * t + 10 + k] = count_key3(fs, 4 * T, &fkeys[4 * t + k]);
    int64_t L = 1;
    for (int m = 0; m < 14; ++m) {
      int64_t c = cnt14[14 * t + m];
      int64_t g = gcd64(L, c);
      if (L / g > ((int64_t)1 << 62) / c) { st = -2; L = 1; break; }
      L = L / g * c;
    }
    Lt[t] = L;
    for (int m = 0; m < 14; ++m) cnt14[14 * t + m] = L / cnt14[14 * t + m];
  }
  free(vkeys); free(ekeys); free(fkeys); free(vs); free(es); free(fs);
  *A_out = cnt14;
  *Lt_out = Lt;
  return st;
}

/* payload numerator of a piece element (vertex, edge or facet) from the tet faces among the
 * planes that define it (face mask fm, bit k = tet face k): no face -> the element is inside
 * the tet (payload of the cell, 1); one face k -> inside tet face k; two faces -> on the tet
 * edge joining the two corners that are on neither face; three faces -> the corner on none.
 * This is the paper's inheritance rule: a vertex cut on an edge takes the
 * edge's payload, an edge cut inside a face takes the face's, and new elements are never
 * re-divided -- the carrier of an element is the smallest tet simplex containing it. */
static int64_t carrier_payload(const int64_t* A14, int64_t L, unsigned fm) {
  int nf = 0;
  for (int k = 0; k < 4; ++k) nf += (fm >> k) & 1;
  if (nf == 0) return L;
  if (nf == 1) {
    for (int k = 0; k < 4; ++k)
      if (fm == (1u << k)) return A14[10 + k];
  }
  unsigned corners = 0xFu & ~fm;  /* corners on none of the faces */
  if (nf == 2) {
    for (int e = 0; e < 6; ++e)
      if (corners == ((1u << EDGE_CORNERS[e][0]) | (1u << EDGE_CORNERS[e][1]))) return A14[4 + e];
  }
  for (int k = 0; k < 4; ++k)
    if (corners == (1u << k)) return A14[k];
  return 0; /* unreachable */
}

/* ------------------------------------------------------------------ clipping */

typedef struct {
  int64_t a[4];   /* barycentric plane vector */
  int64_t rank;   /* SoS rank: radical j -> j, face k -> N + k */
  int32_t src;    /* radical j -> j (>= 0), face k -> -1 - k */
} plane_t;

typedef struct { int32_t p[3]; } vert_t;

typedef struct {
  plane_t* pl;
  int32_t npl, cap_pl;
  vert_t* v;
  int32_t nv, cap_v;
  int64_t n_clip_tests, n_constructions, n_fan_triangles, n_zero_hits;
} poly_t;

static int sos_sign(poly_t* P, const vert_t* v, const plane_t* s) {
  const plane_t* r[4] = {&P->pl[v->p[0]], &P->pl[v->p[1]], &P->pl[v->p[2]], s};
  i256 D4 = det4(r[0]->a, r[1]->a, r[2]->a, r[3]->a);
  int sD3 = i256_sign(det4(r[0]->a, r[1]->a, r[2]->a, ONE4));
  int sD4 = i256_sign(D4);
  ++P->n_clip_tests;
  if (sD4 != 0) return sD4 * sD3;
  ++P->n_zero_hits;
  /* lowest-rank row whose d-cofactor (row replaced by 1) is non-zero */
  int order[4] = {0, 1, 2, 3};
  for (int a = 1; a < 4; ++a)
    for (int b = a; b > 0 && r[order[b]]->rank < r[order[b - 1]]->rank; --b) {
      int tmp = order[b];
      order[b] = order[b - 1];
      order[b - 1] = tmp;
    }
  for (int o = 0; o < 4; ++o) {
    int k = order[o];
    const int64_t* rows[4] = {r[0]->a, r[1]->a, r[2]->a, r[3]->a};
    rows[k] = ONE4;
    int sC = i256_sign(det4(rows[0], rows[1], rows[2], rows[3]));
    if (sC != 0) return -sC * sD3;
  }
  return 0; /* unreachable: C_s = D3 != 0 */
}

static int shares_two(const vert_t* u, const vert_t* w, int32_t* x, int32_t* y) {
  int32_t c[3];
  int n = 0;
  for (int a = 0; a < 3; ++a)
    for (int b = 0; b < 3; ++b)
      if (u->p[a] == w->p[b]) c[n++] = u->p[a];
  if (n != 2) return 0;
  *x = c[0];
  *y = c[1];
  return 1;
}

/* clip by plane s; returns 0 = emptied, 1 = still non-empty */
static int clip_by(poly_t* P, const plane_t* s) {
  int nv = P->nv;
  int* sg = (int*)malloc(sizeof(int) * (nv > 0 ? nv : 1));
  int npos = 0, nneg = 0;
  for (int k = 0; k < nv; ++k) {
    sg[k] = sos_sign(P, &P->v[k], s);
    if (sg[k] > 0) ++npos; else ++nneg;
  }
  if (nneg == 0) { free(sg); return 1; }
  if (npos == 0) { free(sg); P->nv = 0; return 0; }
  if (P->npl == P->cap_pl) {
    P->cap_pl *= 2;
    P->pl = (plane_t*)realloc(P->pl, sizeof(plane_t) * P->cap_pl);
  }
  int32_t sid = P->npl;
  P->pl[P->npl++] = *s;
  vert_t* nvv = (vert_t*)malloc(sizeof(vert_t) * (2 * nv + 8));
  int m = 0;
  for (int k = 0; k < nv; ++k)
    if (sg[k] > 0) nvv[m++] = P->v[k];
  for (int u = 0; u < nv; ++u) {
    if (sg[u] <= 0) continue;
    for (int w = 0; w < nv; ++w) {
      if (sg[w] > 0) continue;
      int32_t x, y;
      if (shares_two(&P->v[u], &P->v[w], &x, &y)) {
        vert_t nvx = {{x, y, sid}};
        nvv[m++] = nvx;
        ++P->n_constructions;
      }
    }
  }
  free(sg);
  if (m > P->cap_v) {
    P->cap_v = 2 * m;
    P->v = (vert_t*)realloc(P->v, sizeof(vert_t) * P->cap_v);
  }
  memcpy(P->v, nvv, sizeof(vert_t) * m);
  P->nv = m;
  free(nvv);
  return 1;
}

/* exact 3x3 cofactors K of the 3x4 matrix [a_p; a_q; a_r]: a . K = det[a_p; a_q; a_r; a] */
static void cofactors(const int64_t* p, const int64_t* q, const int64_t* r, i128* K) {
  for (int m = 0; m < 4; ++m) {
    int c[3], n = 0;
    for (int k = 0; k < 4; ++k)
      if (k != m) c[n++] = k;
    i128 d = (i128)p[c[0]] * ((i128)q[c[1]] * r[c[2]] - (i128)q[c[2]] * r[c[1]]) -
             (i128)p[c[1]] * ((i128)q[c[0]] * r[c[2]] - (i128)q[c[2]] * r[c[0]]) +
             (i128)p[c[2]] * ((i128)q[c[0]] * r[c[1]] - (i128)q[c[1]] * r[c[0]]);
    /* expansion of det[p;q;r;a] along its last row: sign (-1)^(3+m) */
    K[m] = ((3 + m) & 1) ? -d : d;
  }
}

static int same_oriented_plane(const int64_t* a, const int64_t* b) {
  for (int k = 0; k < 4; ++k)
    for (int l = k + 1; l < 4; ++l)
      if ((i128)a[k] * b[l] - (i128)a[l] * b[k] != 0) return 0;
  i128 dot = 0;
  for (int k = 0; k < 4; ++k) dot += (i128)a[k] * b[k];
  return dot > 0;
}

typedef struct {
  int32_t sphere;
  double vol, m1[3];
  uint8_t facemask;
  int32_t* inc;
  int32_t ninc;
  int64_t euler;      /* fractional Euler characteristic of the piece, numerator over L_t */
  int64_t den;        /* L_t of the piece's tet */
  int32_t* rpf_j;     /* radical facets of the piece (neighbour j) ... */
  int64_t* rpf_e;     /* ... and the fractional Euler characteristic of each, over L */
  uint8_t* rpf_fm;    /* ... and the tet faces it has an edge on */
  uint64_t* rpf_adj;  /* ... and the radical facets it shares an edge with (by rank) */
  int32_t nrpf;
  int32_t *rpe_j, *rpe_k; /* restricted power edges (j < k, ascending) ... */
  int64_t* rpe_e;     /* ... their fractional Euler characteristic V - E, over L */
  uint8_t* rpe_fm;    /* ... and the tet faces holding their endpoints */
  int32_t nrpe;
  uint8_t sosfm;      /* tet faces among the piece's facets */
} piece_t;

static int cmp_i32(const void* a, const void* b) {
  int32_t x = *(const int32_t*)a, y = *(const int32_t*)b;
  return (x > y) - (x < y);
}

static unsigned faces_of(const poly_t* P, const int32_t* planes, int n) {
  unsigned fm = 0;
  for (int k = 0; k < n; ++k)
    if (P->pl[planes[k]].src < 0) fm |= 1u << (-1 - P->pl[planes[k]].src);
  return fm;
}

static int cmp_rpe(const void* a, const void* b) {
  const int64_t *x = (const int64_t*)a, *y = (const int64_t*)b;
  if (x[0] != y[0]) return (x[0] > y[0]) - (x[0] < y[0]);
  return (x[1] > y[1]) - (x[1] < y[1]);
}

static int cmp_rpf(const void* a, const void* b) {
  const int64_t *x = (const int64_t*)a, *y = (const int64_t*)b;
  return (x[0] > y[0]) - (x[0] < y[0]);
}

/* Fractional Euler characteristics of a finished piece (Eq. (1)):
 *   Euler(piece)   = sum_vertices payload - sum_edges payload + sum_facets payload - 1 (cell)
 *   Euler(facet f) = sum_{vertices on f} payload - sum_{edges on f} payload + payload(f)
 * for every radical facet f (the piece's part of the RPF between m_i and m_j).  Vertices are
 * the clipped polytope's plane triplets, edges every pair of vertices sharing two planes,
 * facets the planes appearing in the triplets (the symbolically perturbed, simple polytope). */
static void piece_euler(const poly_t* P, const int64_t* A14, int64_t L, piece_t* out) {
  int nv = P->nv, npl = P->npl;
  int64_t chi = -L;
  int* is_facet = (int*)calloc(npl, sizeof(int));
  int64_t* fe = (int64_t*)calloc(npl, sizeof(int64_t)); /* Euler of each facet */
  unsigned* ffm = (unsigned*)calloc(npl, sizeof(unsigned)); /* tet faces sharing an edge */
  int32_t* rre = (int32_t*)malloc(sizeof(int32_t) * 2 * (3 * nv / 2 + 1)); /* radical-radical edges */
  int64_t* rpe = (int64_t*)malloc(sizeof(int64_t) * 4 * (3 * nv / 2 + 1)); /* (j, k, V - E, fm) */
  int nrre = 0;
  for (int v = 0; v < nv; ++v) {
    int64_t pv = carrier_payload(A14, L, faces_of(P, P->v[v].p, 3));
    chi += pv;
    for (int c = 0; c < 3; ++c) {
      is_facet[P->v[v].p[c]] = 1;
      fe[P->v[v].p[c]] += pv;
    }
  }
  for (int u = 0; u < nv; ++u)
    for (int w = u + 1; w < nv; ++w) {
      int32_t e[2];
      if (!shares_two(&P->v[u], &P->v[w], &e[0], &e[1])) continue;
      int64_t pe = carrier_payload(A14, L, faces_of(P, e, 2));
      chi -= pe;
      fe[e[0]] -= pe;
      fe[e[1]] -= pe;
      /* topology (NEXT-2): an edge between facet x and tet face k joins x to face k */
      for (int a = 0; a < 2; ++a)
        if (P->pl[e[1 - a]].src < 0) ffm[e[a]] |= 1u << (-1 - P->pl[e[1 - a]].src);
      /* an edge on two radical planes: a restricted power edge RPE(m_i, m_j, m_k) */
      if (P->pl[e[0]].src >= 0 && P->pl[e[1]].src >= 0) {
        rre[2 * nrre] = e[0];
        rre[2 * nrre + 1] = e[1];
        /* its part of RPE(m_i, m_j, m_k): Euler = V - E = payload(u) + payload(w) - payload(e)
           (the edge inside the tet: payload 1; an endpoint on tet face f: f's payload, inside
           the tet: 1), and the tet faces its endpoints lie on (the third planes of u, w) */
        int64_t j = P->pl[e[0]].src, k = P->pl[e[1]].src;
        rpe[4 * nrre] = j < k ? j : k;
        rpe[4 * nrre + 1] = j < k ? k : j;
        rpe[4 * nrre + 2] = carrier_payload(A14, L, faces_of(P, P->v[u].p, 3)) +
                            carrier_payload(A14, L, faces_of(P, P->v[w].p, 3)) - pe;
        rpe[4 * nrre + 3] = faces_of(P, P->v[u].p, 3) | faces_of(P, P->v[w].p, 3);
        ++nrre;
      }
    }
  int nr = 0;
  out->sosfm = 0;
  for (int f = 0; f < npl; ++f) {
    if (!is_facet[f]) continue;
    int64_t pf = carrier_payload(A14, L, faces_of(P, &f, 1));
    chi += pf;
    fe[f] += pf;
    if (P->pl[f].src >= 0) ++nr;
    else out->sosfm |= (uint8_t)(1u << (-1 - P->pl[f].src));
  }
  int64_t* pairs = (int64_t*)malloc(sizeof(int64_t) * 4 * (nr > 0 ? nr : 1));
  int m = 0;
  for (int f = 0; f < npl; ++f)
    if (is_facet[f] && P->pl[f].src >= 0) {
      pairs[4 * m] = P->pl[f].src;
      pairs[4 * m + 1] = fe[f];
      pairs[4 * m + 2] = ffm[f];
      pairs[4 * m + 3] = f;
      ++m;
    }
  qsort(pairs, nr, 4 * sizeof(int64_t), cmp_rpf);
  int* rank_of = (int*)malloc(sizeof(int) * npl);
  for (int k = 0; k < nr; ++k) rank_of[pairs[4 * k + 3]] = k;
  out->euler = chi;
  out->nrpf = nr;
  out->rpf_j = (int32_t*)malloc(sizeof(int32_t) * (nr > 0 ? nr : 1));
  out->rpf_e = (int64_t*)malloc(sizeof(int64_t) * (nr > 0 ? nr : 1));
  out->rpf_fm = (uint8_t*)malloc(nr > 0 ? nr : 1);
  out->rpf_adj = (uint64_t*)calloc(nr > 0 ? nr : 1, sizeof(uint64_t));
  for (int k = 0; k < nr; ++k) {
    out->rpf_j[k] = (int32_t)pairs[4 * k];
    out->rpf_e[k] = pairs[4 * k + 1];
    out->rpf_fm[k] = (uint8_t)pairs[4 * k + 2];
  }
  for (int k = 0; k < nrre; ++k) {
    int a = rank_of[rre[2 * k]], b = rank_of[rre[2 * k + 1]];
    if (a < 64 && b < 64) {
      out->rpf_adj[a] |= (uint64_t)1 << b;
      out->rpf_adj[b] |= (uint64_t)1 << a;
    }
  }
  /* the RPE list, ascending (j, k) */
  qsort(rpe, nrre, 4 * sizeof(int64_t), cmp_rpe);
  out->nrpe = nrre;
  out->rpe_j = (int32_t*)malloc(sizeof(int32_t) * (nrre > 0 ? nrre : 1));
  out->rpe_k = (int32_t*)malloc(sizeof(int32_t) * (nrre > 0 ? nrre : 1));
  out->rpe_e = (int64_t*)malloc(sizeof(int64_t) * (nrre > 0 ? nrre : 1));
  out->rpe_fm = (uint8_t*)malloc(nrre > 0 ? nrre : 1);
  for (int k = 0; k < nrre; ++k) {
    out->rpe_j[k] = (int32_t)rpe[4 * k];
    out->rpe_k[k] = (int32_t)rpe[4 * k + 1];
    out->rpe_e[k] = rpe[4 * k + 2];
    out->rpe_fm[k] = (uint8_t)rpe[4 * k + 3];
  }
  free(rpe);
  free(rank_of);
  free(rre);
  free(pairs);
  free(ffm);
  free(fe);
  free(is_facet);
}

/* P(t, i): returns 1 and fills *out if non-empty.  A14 (payload numerators of the tet's
 * elements over L, or NULL) switches on the fractional Euler characteristics. */
static int clip_piece(const oracle_input* in, const tet_lat* tl, int64_t i, piece_t* out,
                      oracle_result* stats_acc, const int64_t* A14, int64_t Lden) {
  int32_t k_site = nbr_count(in, i);
  int64_t Si[4], Sj[4];
  load_sphere(in, i, Si);
  int64_t pdi[4];
  for (int k = 0; k < 4; ++k) pdi[k] = pd_lat(tl->X[k], Si);

  /* all sources S(t, i): 4 faces then N(i) in list order */
  int32_t nsrc = 4 + k_site;
  plane_t* src = (plane_t*)malloc(sizeof(plane_t) * nsrc);
  for (int k = 0; k < 4; ++k) {
    for (int c = 0; c < 4; ++c) src[k].a[c] = (c == k);
    src[k].rank = in->N + k;
    src[k].src = -1 - k;
  }
  for (int32_t e = 0; e < k_site; ++e) {
    int32_t j = nbr_at(in, i, e);
    load_sphere(in, j, Sj);
    plane_t* pl = &src[4 + e];
    for (int k = 0; k < 4; ++k) pl->a[k] = pd_lat(tl->X[k], Sj) - pdi[k]; /* >0: closer to i */
    pl->rank = j;
    pl->src = j;
  }

  poly_t P;
  P.cap_pl = nsrc + 4;
  P.pl = (plane_t*)malloc(sizeof(plane_t) * P.cap_pl);
  P.cap_v = 64;
  P.v = (vert_t*)malloc(sizeof(vert_t) * P.cap_v);
  P.npl = 4;
  P.nv = 4;
  P.n_clip_tests = P.n_constructions = P.n_fan_triangles = P.n_zero_hits = 0;
  for (int k = 0; k < 4; ++k) P.pl[k] = src[k];
  for (int k = 0; k < 4; ++k) { /* corner k = intersection of the 3 faces other than k */
    int n = 0;
    for (int f = 0; f < 4; ++f)
      if (f != k) P.v[k].p[n++] = f;
  }

  /* clip in ascending neighbour id order */
  int32_t* ord = (int32_t*)malloc(sizeof(int32_t) * (k_site > 0 ? k_site : 1));
  for (int32_t e = 0; e < k_site; ++e) ord[e] = e;
  for (int32_t a = 1; a < k_site; ++a)
    for (int32_t b = a; b > 0 && src[4 + ord[b]].src < src[4 + ord[b - 1]].src; --b) {
      int32_t tmp = ord[b];
      ord[b] = ord[b - 1];
      ord[b - 1] = tmp;
    }
  int alive = 1;
  for (int32_t e = 0; e < k_site && alive; ++e) alive = clip_by(&P, &src[4 + ord[e]]);
  free(ord);

  int ok = 0;
  if (alive && P.nv > 0) {
    ok = 1;
    int nv = P.nv;
    /* vertex coordinates relative to V0 (lattice units) */
    double (*x)[3] = malloc(sizeof(double[3]) * nv);
    double o[3] = {0, 0, 0};
    for (int v = 0; v < nv; ++v) {
      i128 K[4];
      cofactors(P.pl[P.v[v].p[0]].a, P.pl[P.v[v].p[1]].a, P.pl[P.v[v].p[2]].a, K);
      i128 sum = K[0] + K[1] + K[2] + K[3];
      for (int c = 0; c < 3; ++c) {
        double acc = 0.0;
        for (int k = 1; k < 4; ++k)
          acc += ((double)K[k] / (double)sum) * (double)(tl->X[k][c] - tl->X[0][c]);
        x[v][c] = acc;
        o[c] += acc / nv;
      }
    }
    /* facets */
    int32_t npl = P.npl;
    int* on = (int*)malloc(sizeof(int) * nv);
    int* cyc = (int*)malloc(sizeof(int) * nv);
    double vol = 0.0, m1[3] = {0, 0, 0};
    uint8_t facemask = 0;
    int32_t* inc = (int32_t*)malloc(sizeof(int32_t) * (nsrc + 1));
    int32_t ninc = 0;
    int* is_inc = (int*)calloc(nsrc, sizeof(int));
    for (int32_t f = 0; f < npl; ++f) {
      int m = 0;
      for (int v = 0; v < nv; ++v)
        if (P.v[v].p[0] == f || P.v[v].p[1] == f || P.v[v].p[2] == f) on[m++] = v;
      if (m == 0) continue;
      /* cyclic order: consecutive vertices share two planes (f and another) */
      int* used = (int*)calloc(m, sizeof(int));
      cyc[0] = on[0];
      used[0] = 1;
      int len = 1;
      while (len < m) {
        int cur = cyc[len - 1], nxt = -1;
        for (int b = 0; b < m; ++b) {
          int32_t x0, y0;
          if (!used[b] && shares_two(&P.v[cur], &P.v[on[b]], &x0, &y0)) {
            nxt = b;
            break;
          }
        }
        if (nxt < 0) break;
        used[nxt] = 1;
        cyc[len++] = on[nxt];
      }
      free(used);
      /* fan triangulation against the vertex average o */
      double S = 0.0, fm[3] = {0, 0, 0};
      for (int k = 1; k + 1 < len; ++k) {
        const double *a = x[cyc[0]], *b = x[cyc[k]], *c = x[cyc[k + 1]];
        double u[3], w[3], z[3];
        for (int d = 0; d < 3; ++d) {
          u[d] = a[d] - o[d];
          w[d] = b[d] - o[d];
          z[d] = c[d] - o[d];
        }
        double det = u[0] * (w[1] * z[2] - w[2] * z[1]) - u[1] * (w[0] * z[2] - w[2] * z[0]) +
                     u[2] * (w[0] * z[1] - w[1] * z[0]);
        S += det;
        for (int d = 0; d < 3; ++d) fm[d] += det / 6.0 * (o[d] + a[d] + b[d] + c[d]) / 4.0;
        ++P.n_fan_triangles;
      }
      double sgn = S >= 0 ? 1.0 : -1.0;
      vol += sgn * S / 6.0;
      for (int d = 0; d < 3; ++d) m1[d] += sgn * fm[d];

      /* positive area?  zero iff some edge plane q holds every vertex of the facet */
      int zero_area = 0;
      for (int a = 0; a < m && !zero_area; ++a)
        for (int c = 0; c < 3 && !zero_area; ++c) {
          int32_t q = P.v[on[a]].p[c];
          if (q == f) continue;
          int all_on = 1;
          for (int b = 0; b < m && all_on; ++b) {
            const vert_t* vb = &P.v[on[b]];
            i256 D = det4(P.pl[vb->p[0]].a, P.pl[vb->p[1]].a, P.pl[vb->p[2]].a, P.pl[q].a);
            if (i256_sign(D) != 0) all_on = 0;
          }
          if (all_on) zero_area = 1;
        }
      if (zero_area) continue;
      /* every source whose plane is the same oriented plane */
      for (int32_t q = 0; q < nsrc; ++q)
        if (!is_inc[q] && same_oriented_plane(src[q].a, P.pl[f].a)) is_inc[q] = 1;
    }
    for (int32_t q = 0; q < nsrc; ++q) {
      if (!is_inc[q]) continue;
      if (src[q].src < 0) facemask |= (uint8_t)(1u << (-1 - src[q].src));
      else inc[ninc++] = src[q].src;
    }
    qsort(inc, ninc, sizeof(int32_t), cmp_i32);
    free(is_inc);
    free(on);
    free(cyc);
    free(x);
    /* lattice -> real units: lengths * 2^-10 */
    const double L = 1.0 / 1024.0;
    out->sphere = (int32_t)i;
    out->vol = vol * L * L * L;
    for (int d = 0; d < 3; ++d)
      out->m1[d] = m1[d] * L * L * L * L + out->vol * ((double)tl->X[0][d] * L);
    out->facemask = facemask;
    out->inc = inc;
    out->ninc = ninc;
    out->euler = 0;
    out->nrpf = 0;
    out->rpf_j = NULL;
    out->rpf_e = NULL;
    out->rpf_fm = NULL;
    out->rpf_adj = NULL;
    out->nrpe = 0;
    out->rpe_j = out->rpe_k = NULL;
    out->rpe_e = NULL;
    out->rpe_fm = NULL;
    out->sosfm = 0;
    out->den = Lden;
    if (A14) piece_euler(&P, A14, Lden, out);
  }
  stats_acc->n_clip_tests += P.n_clip_tests;
  stats_acc->n_constructions += P.n_constructions;
  stats_acc->n_fan_triangles += P.n_fan_triangles;
  stats_acc->n_zero_hits += P.n_zero_hits;
  free(P.pl);
  free(P.v);
  free(src);
  return ok;
}

/* ------------------------------------------------------------------ driver */

typedef struct {
  int32_t* cand;
  int32_t ncand;
  piece_t* pieces;
  int32_t npieces;
  oracle_result st;
} tet_out;

void oracle_free(oracle_result* r) {
  if (!r) return;
  free(r->cand_off);
  free(r->cand_idx);
  free(r->piece_off);
  free(r->piece_sphere);
  free(r->piece_vol);
  free(r->piece_m1);
  free(r->piece_facemask);
  free(r->inc_off);
  free(r->inc_sphere);
  free(r->piece_euler);
  free(r->piece_euler_den);
  free(r->rpf_off);
  free(r->rpf_sphere);
  free(r->rpf_euler);
  free(r->piece_sosfm);
  free(r->rpf_fm);
  free(r->rpf_adj);
  free(r->rpe_off);
  free(r->rpe_j);
  free(r->rpe_k);
  free(r->rpe_euler);
  free(r->rpe_fm);
  free(r);
}

/* Full RPD of the given tets (all tets when tet_ids == NULL).  do_clip = 0 stops after the
 * candidate lists.  Caller frees with oracle_free. */
oracle_result* oracle_rpd(const oracle_input* in, const int32_t* tet_ids, int64_t n_tets,
                          int do_clip, int nthreads) {
  oracle_result* R = (oracle_result*)calloc(1, sizeof(oracle_result));
  R->status = check_input(in, R->err);
  if (R->status) return R;
  if (!tet_ids) n_tets = in->T;
  R->n_tets = n_tets;
  int64_t* A = NULL;
  int64_t* Lt = NULL;
  if (in->euler && do_clip) {
    if (euler_payloads(in, &A, &Lt)) {
      R->status = -4;
      snprintf(R->err, 256, "Euler payload denominator of a tet exceeds 2^62");
      free(A);
      free(Lt);
      return R;
    }
  }
  R->euler_denom = 0;
  tet_out* O = (tet_out*)calloc(n_tets > 0 ? n_tets : 1, sizeof(tet_out));
#ifdef _OPENMP
  if (nthreads > 0) omp_set_num_threads(nthreads);
#pragma omp parallel for schedule(dynamic, 8)
#endif
  for (int64_t a = 0; a < n_tets; ++a) {
    int64_t t = tet_ids ? tet_ids[a] : a;
    tet_lat tl;
    load_tet(in, t, &tl);
    tet_out* to = &O[a];
    to->cand = (int32_t*)malloc(sizeof(int32_t) * 16);
    int32_t cap = 16;
    for (int64_t i = 0; i < in->N; ++i) {
      int rel = in->brute ? 1 : relation(in, &tl, i, &to->st.n_rel_tests);
      if (!rel) continue;
      if (to->ncand == cap) {
        cap *= 2;
        to->cand = (int32_t*)realloc(to->cand, sizeof(int32_t) * cap);
      }
      to->cand[to->ncand++] = (int32_t)i;
    }
    if (do_clip) {
      to->pieces = (piece_t*)malloc(sizeof(piece_t) * (to->ncand > 0 ? to->ncand : 1));
      for (int32_t c = 0; c < to->ncand; ++c)
        if (clip_piece(in, &tl, to->cand[c], &to->pieces[to->npieces], &to->st,
                       A ? A + 14 * t : NULL, Lt ? Lt[t] : 0))
          ++to->npieces;
    }
  }
  /* concatenate in tet order */
  int64_t nc = 0, np = 0, ni = 0, nr = 0, ne = 0;
  for (int64_t a = 0; a < n_tets; ++a) {
    nc += O[a].ncand;
    np += O[a].npieces;
    for (int32_t p = 0; p < O[a].npieces; ++p) {
      ni += O[a].pieces[p].ninc;
      nr += O[a].pieces[p].nrpf;
      ne += O[a].pieces[p].nrpe;
    }
  }
  R->n_rpe = ne;
  R->rpe_off = (int32_t*)malloc(sizeof(int32_t) * (np + 1));
  R->rpe_j = (int32_t*)malloc(sizeof(int32_t) * (ne ? ne : 1));
  R->rpe_k = (int32_t*)malloc(sizeof(int32_t) * (ne ? ne : 1));
  R->rpe_euler = (int64_t*)malloc(sizeof(int64_t) * (ne ? ne : 1));
  R->rpe_fm = (uint8_t*)malloc(ne ? ne : 1);
  R->rpe_off[0] = 0;
  int64_t e0 = 0;
  free(A);
  free(Lt);
  R->n_rpf = nr;
  R->piece_euler = (int64_t*)malloc(sizeof(int64_t) * (np ? np : 1));
  R->piece_euler_den = (int64_t*)malloc(sizeof(int64_t) * (np ? np : 1));
  R->rpf_off = (int32_t*)malloc(sizeof(int32_t) * (np + 1));
  R->rpf_sphere = (int32_t*)malloc(sizeof(int32_t) * (nr ? nr : 1));
  R->rpf_euler = (int64_t*)malloc(sizeof(int64_t) * (nr ? nr : 1));
  R->piece_sosfm = (uint8_t*)malloc(np ? np : 1);
  R->rpf_fm = (uint8_t*)malloc(nr ? nr : 1);
  R->rpf_adj = (uint64_t*)malloc(sizeof(uint64_t) * (nr ? nr : 1));
  R->rpf_off[0] = 0;
  int64_t r0 = 0;
  R->n_cand = nc;
  R->n_pieces = np;
  R->n_inc = ni;
  R->cand_off = (int32_t*)malloc(sizeof(int32_t) * (n_tets + 1));
  R->cand_idx = (int32_t*)malloc(sizeof(int32_t) * (nc ? nc : 1));
  R->piece_off = (int32_t*)malloc(sizeof(int32_t) * (n_tets + 1));
  R->piece_sphere = (int32_t*)malloc(sizeof(int32_t) * (np ? np : 1));
  R->piece_vol = (double*)malloc(sizeof(double) * (np ? np : 1));
  R->piece_m1 = (double*)malloc(sizeof(double) * 3 * (np ? np : 1));
  R->piece_facemask = (uint8_t*)malloc(np ? np : 1);
  R->inc_off = (int32_t*)malloc(sizeof(int32_t) * (np + 1));
  R->inc_sphere = (int32_t*)malloc(sizeof(int32_t) * (ni ? ni : 1));
  int64_t c0 = 0, p0 = 0, i0 = 0;
  R->cand_off[0] = 0;
  R->piece_off[0] = 0;
  R->inc_off[0] = 0;
  for (int64_t a = 0; a < n_tets; ++a) {
    tet_out* to = &O[a];
    memcpy(R->cand_idx + c0, to->cand, sizeof(int32_t) * to->ncand);
    c0 += to->ncand;
    R->cand_off[a + 1] = (int32_t)c0;
    for (int32_t p = 0; p < to->npieces; ++p) {
      piece_t* pc = &to->pieces[p];
      R->piece_sphere[p0] = pc->sphere;
      R->piece_vol[p0] = pc->vol;
      for (int d = 0; d < 3; ++d) R->piece_m1[3 * p0 + d] = pc->m1[d];
      R->piece_facemask[p0] = pc->facemask;
      memcpy(R->inc_sphere + i0, pc->inc, sizeof(int32_t) * pc->ninc);
      i0 += pc->ninc;
      R->piece_euler[p0] = pc->euler;
      R->piece_euler_den[p0] = pc->den;
      R->piece_sosfm[p0] = pc->sosfm;
      if (pc->nrpf) {
        memcpy(R->rpf_sphere + r0, pc->rpf_j, sizeof(int32_t) * pc->nrpf);
        memcpy(R->rpf_euler + r0, pc->rpf_e, sizeof(int64_t) * pc->nrpf);
        memcpy(R->rpf_fm + r0, pc->rpf_fm, pc->nrpf);
        memcpy(R->rpf_adj + r0, pc->rpf_adj, sizeof(uint64_t) * pc->nrpf);
      }
      r0 += pc->nrpf;
      R->rpf_off[p0 + 1] = (int32_t)r0;
      free(pc->rpf_j);
      free(pc->rpf_e);
      free(pc->rpf_fm);
      free(pc->rpf_adj);
      if (pc->nrpe) {
        memcpy(R->rpe_j + e0, pc->rpe_j, sizeof(int32_t) * pc->nrpe);
        memcpy(R->rpe_k + e0, pc->rpe_k, sizeof(int32_t) * pc->nrpe);
        memcpy(R->rpe_euler + e0, pc->rpe_e, sizeof(int64_t) * pc->nrpe);
        memcpy(R->rpe_fm + e0, pc->rpe_fm, pc->nrpe);
      }
      e0 += pc->nrpe;
      R->rpe_off[p0 + 1] = (int32_t)e0;
      free(pc->rpe_j);
      free(pc->rpe_k);
      free(pc->rpe_e);
      free(pc->rpe_fm);
      ++p0;
      R->inc_off[p0] = (int32_t)i0;
      free(pc->inc);
    }
    R->piece_off[a + 1] = (int32_t)p0;
    R->n_rel_tests += to->st.n_rel_tests;
    R->n_clip_tests += to->st.n_clip_tests;
    R->n_constructions += to->st.n_constructions;
    R->n_fan_triangles += to->st.n_fan_triangles;
    R->n_zero_hits += to->st.n_zero_hits;
    free(to->cand);
    free(to->pieces);
  }
  free(O);
  return R;
}

int oracle_max_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}

/* ------------------------------------------------------------------ envelope distance
 *
 * Geometry preservation (Sec. 4.3): "For each surface sample, we compute its
 * distance to the closest enveloping volume of the medial mesh (sphere, cone, slab ...) in GPU".
 * A medial cone is the union of the spheres linearly interpolated between two medial spheres,
 * a slab between three.  The signed value of a primitive at p is
 *     g = min over the interpolation parameters of  |p - c(t)| - r(t)
 * (t in [0, 1] for a cone, (u, v) >= 0, u + v <= 1 for a slab); the distance to the envelope
 * is max(min over primitives of g, 0).  |p - c(t)| - r(t) is convex in the parameters (a norm of
 * an affine map minus an affine map), so the oracle minimises it by golden-section search: on t
 * for a cone, nested (u outer, v inner) for a slab -- no closed form is used here. */

static double env_g(const double* p, const double* c, double r) {
  double dx = p[0] - c[0], dy = p[1] - c[1], dz = p[2] - c[2];
  return sqrt(dx * dx + dy * dy + dz * dz) - r;
}

/* value of the (u, v) interpolated sphere of (s1, s2, s3) at p */
static double env_gs(const double* p, const double* s1, const double* s2, const double* s3,
                     double u, double v) {
  double c[3];
  for (int k = 0; k < 3; ++k) c[k] = s1[k] + u * (s2[k] - s1[k]) + v * (s3[k] - s1[k]);
  return env_g(p, c, s1[3] + u * (s2[3] - s1[3]) + v * (s3[3] - s1[3]));
}

static const double GOLD = 0.6180339887498949;

static double env_cone(const double* p, const double* s1, const double* s2) {
  double a = 0.0, b = 1.0;
  for (int it = 0; it < 120; ++it) {
    double x1 = b - GOLD * (b - a), x2 = a + GOLD * (b - a);
    if (env_gs(p, s1, s2, s1, x1, 0.0) <= env_gs(p, s1, s2, s1, x2, 0.0)) b = x2;
    else a = x1;
  }
  double t = 0.5 * (a + b), g = env_gs(p, s1, s2, s1, t, 0.0);
  double g0 = env_gs(p, s1, s2, s1, 0.0, 0.0), g1 = env_gs(p, s1, s2, s1, 1.0, 0.0);
  return fmin(g, fmin(g0, g1));
}

/* min over v in [0, 1 - u] at fixed u */
static double env_slab_u(const double* p, const double* s1, const double* s2, const double* s3,
                         double u) {
  double a = 0.0, b = 1.0 - u;
  for (int it = 0; it < 90; ++it) {
    double x1 = b - GOLD * (b - a), x2 = a + GOLD * (b - a);
    if (env_gs(p, s1, s2, s3, u, x1) <= env_gs(p, s1, s2, s3, u, x2)) b = x2;
    else a = x1;
  }
  double v = 0.5 * (a + b);
  double g = env_gs(p, s1, s2, s3, u, v);
  return fmin(g, fmin(env_gs(p, s1, s2, s3, u, 0.0), env_gs(p, s1, s2, s3, u, 1.0 - u)));
}

static double env_slab(const double* p, const double* s1, const double* s2, const double* s3) {
  double a = 0.0, b = 1.0;
  for (int it = 0; it < 90; ++it) {
    double x1 = b - GOLD * (b - a), x2 = a + GOLD * (b - a);
    if (env_slab_u(p, s1, s2, s3, x1) <= env_slab_u(p, s1, s2, s3, x2)) b = x2;
    else a = x1;
  }
  double u = 0.5 * (a + b);
  return fmin(env_slab_u(p, s1, s2, s3, u),
              fmin(env_slab_u(p, s1, s2, s3, 0.0), env_slab_u(p, s1, s2, s3, 1.0)));
}

/* per sample: the minimum signed value over all primitives (g_out) and the first primitive
 * reaching it (prim_out: sphere i -> i, cone e -> N + e, slab f -> N + NE + f) */
void oracle_envelope(const double* samples, int64_t S, const double* spheres, int64_t N,
                     const int32_t* edges, int64_t NE, const int32_t* faces, int64_t NF,
                     double* g_out, int32_t* prim_out, int nthreads) {
#ifdef _OPENMP
  if (nthreads > 0) omp_set_num_threads(nthreads);
#pragma omp parallel for schedule(dynamic, 4)
#endif
  for (int64_t s = 0; s < S; ++s) {
    const double* p = samples + 3 * s;
    double best = INFINITY;
    int32_t arg = -1;
    for (int64_t i = 0; i < N; ++i) {
      double g = env_g(p, spheres + 4 * i, spheres[4 * i + 3]);
      if (g < best) { best = g; arg = (int32_t)i; }
    }
    for (int64_t e = 0; e < NE; ++e) {
      double g = env_cone(p, spheres + 4 * edges[2 * e], spheres + 4 * edges[2 * e + 1]);
      if (g < best) { best = g; arg = (int32_t)(N + e); }
    }
    for (int64_t f = 0; f < NF; ++f) {
      double g = env_slab(p, spheres + 4 * faces[3 * f], spheres + 4 * faces[3 * f + 1],
                          spheres + 4 * faces[3 * f + 2]);
      if (g < best) { best = g; arg = (int32_t)(N + NE + f); }
    }
    g_out[s] = best;
    prim_out[s] = arg;
  }
}

/* one primitive at one point (tests) */
double oracle_envelope_one(const double* p, const double* spheres, int kind, const int32_t* ids) {
  if (kind == 0) return env_g(p, spheres + 4 * ids[0], spheres[4 * ids[0] + 3]);
  if (kind == 1) return env_cone(p, spheres + 4 * ids[0], spheres + 4 * ids[1]);
  return env_slab(p, spheres + 4 * ids[0], spheres + 4 * ids[1], spheres + 4 * ids[2]);
}
