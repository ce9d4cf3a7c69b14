// Measurement prototype (not product code): ONE THREAD PER (tet, sphere) PAIR clipping the tet
// by the pair's radical half-spaces, volume only, plain fp64 (no exact predicates, no SoS, no
// incidences / facemask / first moment).  It answers SURVEY §7 hard part 3 / VERDICT r1 weak 6:
// would a per-thread clip beat the lockstep lane groups of csrc/rpd_clip.cu on B200?
// Polytope: vertices with their 3 planes and the 3 neighbours across them (simple polytope;
// the neighbour "across plane k" is the other end of the edge leaving plane k), in local memory.
#include <cuda_runtime.h>
#include <stdint.h>

namespace {
#ifndef PROTO_MV
#define PROTO_MV 48
#endif
constexpr int MV = PROTO_MV;  // vertex slots per pair (more: flagged, not clipped further)

__global__ void __launch_bounds__(128) k_proto(
    int64_t n, const int32_t* __restrict__ pair_tet, const int32_t* __restrict__ cand,
    const double* __restrict__ verts, const int32_t* __restrict__ tets,
    const double* __restrict__ sph, const int32_t* __restrict__ off,
    const int32_t* __restrict__ idx, double* __restrict__ vol, int* __restrict__ overflow) {
  const int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (p >= n) return;
  double X[MV], Y[MV], Z[MV], S[MV];
  int pl[MV][3], nb[MV][3];
  bool alive[MV];
  const int t = pair_tet[p], i = cand[p];
  double cx = 0, cy = 0, cz = 0;
  double V0[4][3];
  for (int k = 0; k < 4; ++k) {
    const int v = tets[4 * t + k];
    V0[k][0] = verts[3 * v];
    V0[k][1] = verts[3 * v + 1];
    V0[k][2] = verts[3 * v + 2];
    cx += 0.25 * V0[k][0];
    cy += 0.25 * V0[k][1];
    cz += 0.25 * V0[k][2];
  }
  // tet: vertex k lies on the planes (faces) != k; the neighbour across plane q is vertex q
  int nv = 4;
  for (int k = 0; k < 4; ++k) {
    X[k] = V0[k][0] - cx;
    Y[k] = V0[k][1] - cy;
    Z[k] = V0[k][2] - cz;
    alive[k] = true;
    int q = 0;
    for (int f = 0; f < 4; ++f)
      if (f != k) {
        pl[k][q] = f;
        nb[k][q] = f;
        ++q;
      }
  }
  const double xi = sph[4 * i] - cx, yi = sph[4 * i + 1] - cy, zi = sph[4 * i + 2] - cz,
               ri = sph[4 * i + 3];
  const double Wi = xi * xi + yi * yi + zi * zi - ri * ri;
  bool empty = false, over = false;
  const int e0 = off[i], e1 = off[i + 1];
  for (int e = e0; e < e1 && !empty && !over; ++e) {
    const int j = idx[e];
    const double xj = sph[4 * j] - cx, yj = sph[4 * j + 1] - cy, zj = sph[4 * j + 2] - cz,
                 rj = sph[4 * j + 3];
    // h(x) = n.x + d >= 0 inside: n = 2 (theta_i - theta_j), d = W_j - W_i
    const double nx = 2.0 * (xi - xj), ny = 2.0 * (yi - yj), nz = 2.0 * (zi - zj);
    const double d = (xj * xj + yj * yj + zj * zj - rj * rj) - Wi;
    // cut test at the tet corners first (the group clip's cut mask)
    bool all_pos = true;
    for (int k = 0; k < 4 && all_pos; ++k)
      all_pos = nx * (V0[k][0] - cx) + ny * (V0[k][1] - cy) + nz * (V0[k][2] - cz) + d > 0.0;
    if (all_pos) continue;
    int n_neg = 0, n_pos = 0;
    for (int v = 0; v < nv; ++v) {
      if (!alive[v]) continue;
      S[v] = nx * X[v] + ny * Y[v] + nz * Z[v] + d;
      if (S[v] < 0.0) ++n_neg;
      else ++n_pos;
    }
    if (n_neg == 0) continue;
    if (n_pos == 0) {
      empty = true;
      break;
    }
    const int P = 4 + (e - e0);  // plane id of the cut
    int made[MV];
    int n_made = 0;
    for (int u = 0; u < nv && !over; ++u) {
      if (!alive[u] || S[u] >= 0.0) continue;
      for (int k = 0; k < 3; ++k) {
        const int w = nb[u][k];
        if (S[w] < 0.0) continue;
        // new vertex on edge (u, w): planes of the edge = u's planes but pl[u][k], plus P
        int x = -1;
        for (int s = 0; s < nv; ++s)
          if (!alive[s] && s != u) {
            bool used = false;
            for (int m = 0; m < n_made; ++m) used |= made[m] == s;
            if (!used) {
              x = s;
              break;
            }
          }
        if (x < 0) {
          if (nv >= MV) {
            over = true;
            break;
          }
          x = nv++;
        }
        const double tt = S[u] / (S[u] - S[w]);
        X[x] = X[u] + tt * (X[w] - X[u]);
        Y[x] = Y[u] + tt * (Y[w] - Y[u]);
        Z[x] = Z[u] + tt * (Z[w] - Z[u]);
        S[x] = 0.0;
        alive[x] = true;
        pl[x][0] = pl[u][(k + 1) % 3];
        pl[x][1] = pl[u][(k + 2) % 3];
        pl[x][2] = P;
        nb[x][2] = w;  // leaving P along the edge
        nb[x][0] = nb[x][1] = -1;
        for (int q = 0; q < 3; ++q)
          if (nb[w][q] == u) nb[w][q] = x;
        made[n_made++] = x;
      }
    }
    if (over) break;
    for (int u = 0; u < nv; ++u)
      if (alive[u] && S[u] < 0.0) {
        bool is_new = false;
        for (int m = 0; m < n_made; ++m) is_new |= made[m] == u;
        if (!is_new) alive[u] = false;
      }
    // link the new facet: x's neighbour leaving plane q (q one of its two old planes) is the
    // other new vertex on the old plane r != q
    for (int a = 0; a < n_made; ++a) {
      const int x = made[a];
      for (int q = 0; q < 2; ++q) {
        const int r = pl[x][1 - q];
        for (int b = 0; b < n_made; ++b) {
          const int y = made[b];
          if (y != x && (pl[y][0] == r || pl[y][1] == r)) {
            nb[x][q] = y;
            break;
          }
        }
      }
    }
  }
  if (over) {
    atomicAdd(overflow, 1);
    vol[p] = -1.0;
    return;
  }
  if (empty) {
    vol[p] = 0.0;
    return;
  }
  // volume: V = 1/3 sum_f x0_f . A_f (outward area vectors); faces walked per plane from
  // each vertex that is the face's smallest alive vertex id
  double V = 0.0, gx = 0, gy = 0, gz = 0;
  int na = 0;
  for (int v = 0; v < nv; ++v)
    if (alive[v]) {
      gx += X[v];
      gy += Y[v];
      gz += Z[v];
      ++na;
    }
  gx /= na;
  gy /= na;
  gz /= na;  // (an interior point: the face pyramids from it have positive volumes)
  for (int v = 0; v < nv; ++v) {
    if (!alive[v]) continue;
    for (int q = 0; q < 3; ++q) {
      const int f = pl[v][q];
      // is v the smallest alive vertex on plane f?  walk the face and check
      int prev = -1, cur = v, steps = 0;
      bool smallest = true;
      double ax = 0, ay = 0, az = 0;
      do {
        // the two edges of cur that stay on f leave its other two planes; take the one not
        // going back
        int qq = 0;
        while (pl[cur][qq] != f) ++qq;
        const int n1 = nb[cur][(qq + 1) % 3], n2 = nb[cur][(qq + 2) % 3];
        const int nxt = n1 != prev ? n1 : n2;
        ax += Y[cur] * Z[nxt] - Z[cur] * Y[nxt];
        ay += Z[cur] * X[nxt] - X[cur] * Z[nxt];
        az += X[cur] * Y[nxt] - Y[cur] * X[nxt];
        prev = cur;
        cur = nxt;
        if (cur < v) smallest = false;
      } while (cur != v && ++steps < MV && cur >= 0);
      if (!smallest || cur != v) continue;
      // |x0 . A| with the outward orientation: the polytope's centroid side of the plane
      const double dd = (X[v] - gx) * ax + (Y[v] - gy) * ay + (Z[v] - gz) * az;
      V += fabs(dd) / 6.0;  // ((x0 - g) . 2A) / 6
    }
  }
  vol[p] = V;
}
}  // namespace

extern "C" int proto_clip(int64_t n, const int32_t* pair_tet, const int32_t* cand,
                          const double* verts, const int32_t* tets, const double* sph,
                          const int32_t* off, const int32_t* idx, double* vol, int* overflow,
                          float* ms) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaMemset(overflow, 0, sizeof(int));
  cudaEventRecord(a);
  k_proto<<<(unsigned)((n + 127) / 128), 128>>>(n, pair_tet, cand, verts, tets, sph, off, idx,
                                                   vol, overflow);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  cudaEventElapsedTime(ms, a, b);
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  return (int)cudaGetLastError();
}
