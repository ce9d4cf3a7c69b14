"""Seeded synthetic inputs for the RPD hot path (shared by the oracle and the CUDA path).

This module holds NONE of the method's arithmetic (no power distances of tets, no Alg. 1,
no clipping).  It only builds the inputs the paper's problem statement takes
(Supp. §1: a tet mesh, medial spheres, and the sphere neighbour lists that
the paper obtains from a CGAL regular triangulation):

* tet meshes: Kuhn/Freudenthal 6-tet split of a voxelised CAD-like solid (an axis box with a
  cylindrical through-hole, genus 1, sharp edges), optional integer jitter of interior
  vertices, positive orientation enforced, tets in Morton order of their centroid;
* medial-like spheres: interior samples pushed toward the medial surface by SDF-gradient
  ascent, r = floor(SDF * f) with f drawn per radius mode, plus ~15 % zero-radius feature
  spheres on sharp edges / rims;
* sphere neighbours (k_site): edges of the lower convex hull of the lifted points
  (theta, |theta|^2 - r^2) computed by Qhull (scipy) -- the library stand-in for CGAL's
  regular triangulation.  Spheres that are not lower-hull vertices are *hidden* and get
  k_site = 0 (reading R4).

Every coordinate and radius is a multiple of 2^-10 inside the box [0, 64)^3 (C3:
the exactness budget), so every quantity the method computes on the lattice is an integer.
"""
from __future__ import annotations

import hashlib
import os
import pickle
from dataclasses import dataclass, field
from typing import Callable, List, Optional

import numpy as np

LATTICE_BITS = 10                 # coordinates are multiples of 2^-10
LATTICE = 1 << LATTICE_BITS       # lattice units per real unit
BOX = 64.0                        # [0, 64)^3  ->  16-bit lattice integers
BOX_LAT = int(BOX * LATTICE)      # 65536


@dataclass
class Workload:
    name: str
    verts: np.ndarray            # [V,3] float64, multiples of 2^-10
    tets: np.ndarray             # [T,4] int32, positively oriented
    spheres: np.ndarray          # [N,4] float64 (x, y, z, r)
    nbr_off: np.ndarray          # [N+1] int32
    nbr_idx: np.ndarray          # [sum k_site] int32, ascending per row
    meta: dict = field(default_factory=dict)
    # partial-update batches (C4): list of (spheres_after [N_k,4], nbr_off, nbr_idx)
    batches: List[tuple] = field(default_factory=list)

    @property
    def T(self):
        return int(self.tets.shape[0])

    @property
    def N(self):
        return int(self.spheres.shape[0])


# ----------------------------------------------------------------------------- lattice


def to_lattice(x):
    """Round real coordinates to the 2^-10 lattice (returns float64 multiples of 2^-10)."""
    return np.round(np.asarray(x, dtype=np.float64) * LATTICE) / LATTICE


def morton3(ix, iy, iz):
    """48-bit Morton code of three 16-bit non-negative integers."""
    def spread(v):
        v = v.astype(np.uint64) & np.uint64(0xFFFF)
        v = (v | (v << np.uint64(16))) & np.uint64(0x0000FF0000FF)
        v = (v | (v << np.uint64(8))) & np.uint64(0x00F00F00F00F)
        v = (v | (v << np.uint64(4))) & np.uint64(0x0C30C30C30C3)
        v = (v | (v << np.uint64(2))) & np.uint64(0x249249249249)
        return v
    return spread(ix) | (spread(iy) << np.uint64(1)) | (spread(iz) << np.uint64(2))


# ----------------------------------------------------------------------------- meshes

# Kuhn simplices of the unit cube: one per permutation of the axes (Freudenthal split along
# the (0,0,0)-(1,1,1) diagonal); conforming across neighbouring cubes.
_PERMS = [(0, 1, 2), (0, 2, 1), (1, 0, 2), (1, 2, 0), (2, 0, 1), (2, 1, 0)]
_PERM_SIGN = [1, -1, -1, 1, 1, -1]


def _orient_det(P):
    a = P[:, 1] - P[:, 0]
    b = P[:, 2] - P[:, 0]
    c = P[:, 3] - P[:, 0]
    return np.einsum("ij,ij->i", a, np.cross(b, c))


def kuhn_grid_mesh(n, s, origin, keep: Optional[Callable] = None, jitter: int = 0,
                   seed: int = 0, morton: bool = True):
    """Kuhn split of an n=(nx,ny,nz) voxel grid with integer voxel side ``s`` (lattice units)
    whose low corner is ``origin`` (lattice units).  ``keep(cx,cy,cz)`` (voxel centres in real
    units, arrays) selects voxels.  ``jitter`` (lattice units) perturbs interior vertices.
    Returns verts [V,3] float64 (real units, lattice multiples) and tets [T,4] int32."""
    nx, ny, nz = n
    rng = np.random.default_rng(seed)
    gi, gj, gk = np.meshgrid(np.arange(nx), np.arange(ny), np.arange(nz), indexing="ij")
    gi, gj, gk = gi.ravel(), gj.ravel(), gk.ravel()
    if keep is not None:
        cx = (origin[0] + (gi + 0.5) * s) / LATTICE
        cy = (origin[1] + (gj + 0.5) * s) / LATTICE
        cz = (origin[2] + (gk + 0.5) * s) / LATTICE
        m = keep(cx, cy, cz)
        gi, gj, gk = gi[m], gj[m], gk[m]
    nvx, nvy, nvz = nx + 1, ny + 1, nz + 1

    def vid(i, j, k):
        return (i * nvy + j) * nvz + k

    tets = []
    for p, sg in zip(_PERMS, _PERM_SIGN):
        c = [gi.copy(), gj.copy(), gk.copy()]
        v0 = vid(*c)
        c[p[0]] = c[p[0]] + 1
        v1 = vid(*c)
        c[p[1]] = c[p[1]] + 1
        v2 = vid(*c)
        c[p[2]] = c[p[2]] + 1
        v3 = vid(*c)
        if sg > 0:
            tets.append(np.stack([v0, v1, v2, v3], 1))
        else:
            tets.append(np.stack([v0, v2, v1, v3], 1))
    tets = np.concatenate(tets, 0)
    used, inv = np.unique(tets.ravel(), return_inverse=True)
    tets = inv.reshape(-1, 4).astype(np.int64)
    ii = used // (nvy * nvz)
    jj = (used // nvz) % nvy
    kk = used % nvz
    P = np.stack([origin[0] + ii * s, origin[1] + jj * s, origin[2] + kk * s], 1).astype(np.int64)
    if jitter > 0:
        # interior vertices = used by the full 24 incident tets of the Kuhn lattice
        cnt = np.bincount(tets.ravel(), minlength=len(used))
        interior = cnt == 24
        for _ in range(100):
            J = rng.integers(-jitter, jitter + 1, size=P.shape)
            J[~interior] = 0
            Q = P + J
            if np.all(_orient_det(Q[tets].astype(np.float64)) > 0):
                P = Q
                break
    assert P.min() >= 0 and P.max() < BOX_LAT, "mesh leaves the [0,64)^3 lattice box"
    det = _orient_det(P[tets].astype(np.float64))
    assert np.all(det > 0), "non-positive tet"
    if morton:
        cen = P[tets].sum(1) // 4
        order = np.argsort(morton3(cen[:, 0], cen[:, 1], cen[:, 2]), kind="stable")
        tets = tets[order]
    return P.astype(np.float64) / LATTICE, tets.astype(np.int32)


def unit_cube_6tets(scale: float = 1.0, origin=(0.0, 0.0, 0.0)):
    """The unit cube (scaled) split into its 6 Kuhn tets (BASELINE.json configs[0])."""
    s = int(round(scale * LATTICE))
    o = [int(round(v * LATTICE)) for v in origin]
    return kuhn_grid_mesh((1, 1, 1), s, o, morton=False)


def box_6tets(lo, hi):
    """The axis box [lo, hi] (lattice multiples, hi > lo per axis) split into its 6 Kuhn tets:
    the domain the NEXT-3 neighbour definition restricts power cells to."""
    v, t = kuhn_grid_mesh((1, 1, 1), 1, (0, 0, 0), morton=False)
    u = np.round(v * LATTICE)                     # unit cube corners, 0 / 1
    lo = np.asarray(lo, dtype=np.float64)
    hi = np.asarray(hi, dtype=np.float64)
    assert np.all(hi > lo)
    return lo + u * (hi - lo), t


def mesh_box(verts):
    """(lo_x, lo_y, lo_z, hi_x, hi_y, hi_z) of a mesh: the box passed to rpd_neighbors."""
    v = np.asarray(verts, dtype=np.float64)
    return np.concatenate([v.min(0), v.max(0)])


@dataclass
class BoxWithHole:
    """Axis box [lo,hi] with a cylindrical through-hole along z (genus-1 CAD-like solid)."""
    lo: np.ndarray
    hi: np.ndarray
    hole_c: np.ndarray          # (x, y) of the hole axis
    hole_r: float

    def inside(self, x, y, z):
        return ((x > self.lo[0]) & (x < self.hi[0]) & (y > self.lo[1]) & (y < self.hi[1])
                & (z > self.lo[2]) & (z < self.hi[2])
                & (np.hypot(x - self.hole_c[0], y - self.hole_c[1]) > self.hole_r))

    def sdf_grad(self, p):
        """Interior distance to the boundary (positive inside) and its gradient."""
        x, y, z = p[:, 0], p[:, 1], p[:, 2]
        rho = np.hypot(x - self.hole_c[0], y - self.hole_c[1])
        terms = np.stack([x - self.lo[0], self.hi[0] - x, y - self.lo[1], self.hi[1] - y,
                          z - self.lo[2], self.hi[2] - z, rho - self.hole_r], 1)
        k = np.argmin(terms, 1)
        d = terms[np.arange(len(p)), k]
        g = np.zeros_like(p)
        axis_dirs = [(0, 1), (0, -1), (1, 1), (1, -1), (2, 1), (2, -1)]
        for t, (ax, sg) in enumerate(axis_dirs):
            m = k == t
            g[m, ax] = sg
        m = k == 6
        rr = np.maximum(rho[m], 1e-12)
        g[m, 0] = (x[m] - self.hole_c[0]) / rr
        g[m, 1] = (y[m] - self.hole_c[1]) / rr
        return d, g

    def feature_points(self, rng, n):
        """Points on sharp edges: the 12 box edges and the two hole rims."""
        lo, hi = self.lo, self.hi
        edges = []
        for ax in range(3):
            o1, o2 = [a for a in range(3) if a != ax]
            for a in (lo[o1], hi[o1]):
                for b in (lo[o2], hi[o2]):
                    edges.append((ax, o1, a, o2, b))
        L_box = sum(hi[e[0]] - lo[e[0]] for e in edges)
        L_rim = 2 * 2 * np.pi * self.hole_r
        pts = []
        n_rim = int(round(n * L_rim / (L_box + L_rim)))
        for _ in range(n - n_rim):
            lens = np.array([hi[e[0]] - lo[e[0]] for e in edges])
            e = edges[rng.choice(len(edges), p=lens / lens.sum())]
            ax, o1, a, o2, b = e
            p = np.zeros(3)
            p[ax] = rng.uniform(lo[ax], hi[ax])
            p[o1] = a
            p[o2] = b
            pts.append(p)
        for _ in range(n_rim):
            t = rng.uniform(0, 2 * np.pi)
            z = lo[2] if rng.random() < 0.5 else hi[2]
            pts.append([self.hole_c[0] + self.hole_r * np.cos(t),
                        self.hole_c[1] + self.hole_r * np.sin(t), z])
        return np.array(pts).reshape(-1, 3)


def default_shape():
    return BoxWithHole(lo=np.array([2.0, 2.0, 2.0]), hi=np.array([62.0, 50.0, 38.0]),
                       hole_c=np.array([32.0, 26.0]), hole_r=9.0)


def shape_mesh(shape: BoxWithHole, target_tets: int, jitter_frac: float = 0.125, seed: int = 0):
    """Voxelise ``shape`` with a cubic voxel size chosen so the Kuhn mesh has ~target_tets."""
    ext = shape.hi - shape.lo
    vol = np.prod(ext) - np.pi * shape.hole_r ** 2 * ext[2]
    side = (vol / (target_tets / 6.0)) ** (1.0 / 3.0)
    s = max(2, int(round(side * LATTICE)))
    n = [int(np.ceil(e * LATTICE / s)) for e in ext]
    origin = [int(round(shape.lo[a] * LATTICE)) for a in range(3)]
    # shrink the grid so it stays in the box
    for a in range(3):
        while origin[a] + n[a] * s >= BOX_LAT:
            n[a] -= 1
    keep = lambda cx, cy, cz: shape.inside(cx, cy, cz)
    return kuhn_grid_mesh(tuple(n), s, origin, keep=keep, jitter=int(s * jitter_frac), seed=seed)


# ----------------------------------------------------------------------------- spheres


def medial_like_spheres(shape: BoxWithHole, n: int, seed: int, radius_mode: str = "uniform",
                        feature_frac: float = 0.15, region=None, existing=None):
    """Medial-like spheres: ``(1-feature_frac)`` interior spheres near the medial surface with
    r = floor(SDF * f), f ~ radius_mode, plus zero-radius feature spheres.
    ``region=(centre, radius)`` restricts interior samples to a ball (local insertions,
    PAPER.md:280, 595).  Centres are quantised to the lattice and deduplicated (also against
    ``existing`` centres)."""
    rng = np.random.default_rng(seed)
    n_feat = int(round(n * feature_frac)) if region is None else 0
    n_int = n - n_feat
    out = []
    seen = set()
    if existing is not None:
        for p in np.round(np.asarray(existing)[:, :3] * LATTICE).astype(np.int64):
            seen.add(tuple(p))
    need = n_int
    tries = 0
    while need > 0 and tries < 50:
        tries += 1
        m = max(need * 3, 64)
        if region is None:
            P = rng.uniform(shape.lo, shape.hi, size=(m, 3))
        else:
            c, rad = region
            d = rng.normal(size=(m, 3))
            d /= np.linalg.norm(d, axis=1, keepdims=True)
            P = c + d * rad * rng.random((m, 1)) ** (1 / 3)
        P = P[shape.inside(P[:, 0], P[:, 1], P[:, 2])]
        # push toward the medial surface: a few SDF-gradient ascent steps
        for it in range(3):
            d, g = shape.sdf_grad(P)
            P = P + g * (0.15 * d)[:, None]
        P = P[shape.inside(P[:, 0], P[:, 1], P[:, 2])]
        d, _ = shape.sdf_grad(P)
        if radius_mode == "uniform":
            # f ~ U(0.9, 1): near-tangent spheres; U(0.5, 1) hid ~52 % of spheres at C3
            # density (input recipe)
            f = rng.uniform(0.9, 1.0, size=len(P))
        elif radius_mode == "high_variance":
            f = np.where(rng.random(len(P)) < 0.8, rng.uniform(0.0, 0.15, len(P)),
                         rng.uniform(0.85, 1.0, len(P)))
        elif radius_mode == "equal":
            f = np.zeros(len(P))
        else:
            raise ValueError(radius_mode)
        R = np.floor(d * f * LATTICE) / LATTICE
        C = to_lattice(P)
        for c, r in zip(C, R):
            key = tuple(np.round(c * LATTICE).astype(np.int64))
            if key in seen:
                continue
            seen.add(key)
            out.append([c[0], c[1], c[2], max(r, 0.0)])
            need -= 1
            if need == 0:
                break
    F = to_lattice(shape.feature_points(rng, n_feat * 2)) if n_feat else np.zeros((0, 3))
    got = 0
    for c in F:
        if got >= n_feat:
            break
        key = tuple(np.round(c * LATTICE).astype(np.int64))
        if key in seen:
            continue
        seen.add(key)
        out.append([c[0], c[1], c[2], 0.0])
        got += 1
    S = np.array(out, dtype=np.float64).reshape(-1, 4)
    rng.shuffle(S)      # sphere ids carry no spatial order (like generated insertions)
    return S


# ----------------------------------------------------------------------------- neighbours


def power_neighbours(spheres: np.ndarray, all_pairs_below: int = 6):
    """Regular-triangulation neighbours (k_site lists) -- the input the paper gets from CGAL
    (PAPER.md:18).  Lower hull of the lifted points via Qhull; rows ascending.  Hidden spheres
    (not lower-hull vertices) get k_site = 0.  Tiny or degenerate sets fall back to all pairs
    (a superset, which is harmless: DESIGN.md C0)."""
    from scipy.spatial import ConvexHull
    N = len(spheres)
    pairs = None
    if N >= all_pairs_below:
        c = spheres[:, :3].mean(0)
        th = spheres[:, :3] - c
        lift = np.concatenate([th, (th * th).sum(1, keepdims=True) - spheres[:, 3:4] ** 2], 1)
        for opts in ("Qt", "Qt QJ"):
            try:
                h = ConvexHull(lift, qhull_options=opts)
            except Exception:
                continue
            lower = h.simplices[h.equations[:, 3] < 0]
            a = lower[:, [0, 0, 0, 1, 1, 2]].ravel()
            b = lower[:, [1, 2, 3, 2, 3, 3]].ravel()
            pairs = np.stack([np.concatenate([a, b]), np.concatenate([b, a])], 1)
            break
    if pairs is None:
        ii, jj = np.meshgrid(np.arange(N), np.arange(N), indexing="ij")
        m = ii != jj
        pairs = np.stack([ii[m], jj[m]], 1)
    pairs = np.unique(pairs, axis=0)
    pairs = pairs[pairs[:, 0] != pairs[:, 1]]
    off = np.zeros(N + 1, dtype=np.int64)
    np.add.at(off, pairs[:, 0] + 1, 1)
    off = np.cumsum(off)
    return off.astype(np.int32), pairs[:, 1].astype(np.int32)


def all_pairs_neighbours(N: int):
    """N(i) = all j != i (the brute-force mode of DESIGN.md C1 step 8)."""
    idx = [j for i in range(N) for j in range(N) if j != i]
    off = np.arange(N + 1, dtype=np.int64) * max(N - 1, 0)
    return off.astype(np.int32), np.asarray(idx, dtype=np.int32)


# ----------------------------------------------------------------------------- configs


def c1_spheres(seed: int, degenerate: bool, n: int = 16, big: bool = False):
    """16 dyadic-grid spheres for the unit cube (BASELINE.json configs[0]).
    C1a (generic): centres/radii random multiples of 2^-10.  C1b (degenerate): centres at
    multiples of 1/4, radii multiples of 1/8 so radical planes hit Kuhn faces and vertices."""
    rng = np.random.default_rng(seed)
    out, seen = [], set()
    while len(out) < n:
        if degenerate:
            c = rng.integers(0, 5, size=3) / 4.0
            r = rng.integers(0, 5 if big else 3) / 8.0
        else:
            c = rng.integers(0, LATTICE + 1, size=3) / LATTICE
            r = rng.integers(0, LATTICE // 4) / LATTICE
        key = tuple(c)
        if key in seen:
            continue
        seen.add(key)
        out.append([c[0], c[1], c[2], r])
    return np.array(out, dtype=np.float64)


def random_tiny(seed: int, n_spheres: int = 12, grid: int = 2, coarse: bool = False):
    """Tiny random configs for oracle pins: a grid^3 Kuhn cube mesh of [0,1]^3 and spheres."""
    s = LATTICE // grid
    verts, tets = kuhn_grid_mesh((grid, grid, grid), s, (0, 0, 0), morton=False)
    sph = c1_spheres(seed, degenerate=coarse, n=n_spheres)
    off, idx = power_neighbours(sph)
    return Workload(f"tiny{seed}", verts, tets, sph, off, idx, meta={"seed": seed})


def delaunay_workload(n_points: int, n_spheres: int, seed: int = 0, box: float = 16.0):
    """An unstructured tet mesh (fTetWild-like vertex valences, unlike Kuhn grids):
    the Delaunay tetrahedralisation (Qhull) of random lattice points in [1, 1 + box)^3 -- distinct
    points on the 2^-6 grid, slivers of zero volume dropped, every tet positively oriented --
    and random zero-or-small-radius spheres inside with their regular-triangulation lists."""
    from scipy.spatial import Delaunay
    rng = np.random.default_rng(seed)
    P = np.unique(rng.integers(0, int(box * 64), size=(n_points, 3)), axis=0) / 64.0 + 1.0
    tets = Delaunay(P).simplices.astype(np.int64)
    det = _orient_det(P[tets] * LATTICE)
    tets = tets[det != 0]
    det = det[det != 0]
    neg = det < 0
    tets[neg] = tets[neg][:, [0, 2, 1, 3]]
    sph = np.c_[rng.integers(0, int(box * 64), size=(n_spheres, 3)) / 64.0 + 1.0,
                rng.integers(0, 64, size=n_spheres) / 64.0]
    sph = np.unique(sph, axis=0)
    off, idx = power_neighbours(sph)
    return Workload(f"delaunay{n_points}_{seed}", P, tets.astype(np.int32), sph, off, idx,
                    meta={"seed": seed})


def make_c1(seed: int = 0, degenerate: bool = False, big: bool = False):
    verts, tets = unit_cube_6tets()
    sph = c1_spheres(seed, degenerate, big=big)
    off, idx = power_neighbours(sph)
    return Workload("C1b" if degenerate else "C1a", verts, tets, sph, off, idx,
                    meta={"seed": seed, "config": 0})


_CACHE_DIR = os.environ.get("RPD_WORKLOAD_CACHE", os.path.expanduser("~/.cache/rpd_workloads"))


def _cached(key: str, fn):
    """Memoise a deterministic generator on disk (pure speed-up: same seed -> same arrays)."""
    h = hashlib.sha1(key.encode()).hexdigest()[:16]
    path = os.path.join(_CACHE_DIR, f"{h}.pkl")
    try:
        with open(path, "rb") as f:
            return pickle.load(f)
    except Exception:
        pass
    w = fn()
    try:
        os.makedirs(_CACHE_DIR, exist_ok=True)
        tmp = path + f".{os.getpid()}.tmp"
        with open(tmp, "wb") as f:
            pickle.dump(w, f)
        os.replace(tmp, path)
    except Exception:
        pass
    return w


def make_shape_workload(name: str, target_tets: int, n_spheres: int, seed: int = 0,
                        radius_mode: str = "uniform", n_batches: int = 0, batch_m: int = 0,
                        clusters: int = 10, cache: bool = True):
    """C2/C3/C4/C5-style workload: Kuhn mesh of the box-with-hole solid + medial-like spheres,
    optional partial-update batches of ``batch_m`` spheres in ``clusters`` local regions."""
    key = f"v1|{name}|{target_tets}|{n_spheres}|{seed}|{radius_mode}|{n_batches}|{batch_m}|{clusters}"

    def build():
        shape = default_shape()
        verts, tets = shape_mesh(shape, target_tets, seed=seed)
        sph = medial_like_spheres(shape, n_spheres, seed=seed + 1, radius_mode=radius_mode)
        off, idx = power_neighbours(sph)
        w = Workload(name, verts, tets, sph, off, idx,
                     meta={"seed": seed, "radius_mode": radius_mode, "target_tets": target_tets})
        rng = np.random.default_rng(seed + 7)
        cur = sph
        for b in range(n_batches):
            per = batch_m // clusters
            new = []
            for c in range(clusters):
                m = per if c < clusters - 1 else batch_m - per * (clusters - 1)
                centre = cur[rng.integers(len(cur)), :3]
                rad = 4.0
                s = medial_like_spheres(shape, m, seed=seed * 1000 + b * 37 + c + 11,
                                        radius_mode=radius_mode, region=(centre, rad),
                                        existing=np.concatenate([cur] + new, 0))
                new.append(s)
            cur = np.concatenate([cur] + new, 0)
            o2, i2 = power_neighbours(cur)
            w.batches.append((cur, o2, i2))
        return w

    return _cached(key, build) if cache else build()


CONFIGS = {
    # name: (target_tets, n_spheres, radius_mode, n_batches, batch_m)
    "C2": (50_000, 2_000, "uniform", 0, 0),
    "C3": (200_000, 20_000, "uniform", 0, 0),
    "C4": (200_000, 20_000, "uniform", 10, 500),
    "C5": (4_000_000, 50_000, "high_variance", 0, 0),
}


def make_config(name: str, seed: int = 0, **kw):
    if name in ("C1", "C1a"):
        return make_c1(seed, degenerate=False)
    if name == "C1b":
        return make_c1(seed, degenerate=True)
    t, n, mode, nb, m = CONFIGS[name]
    return make_shape_workload(name, t, n, seed=seed, radius_mode=mode, n_batches=nb,
                               batch_m=m, **kw)


def block_cyclic_shard(T: int, world: int, rank: int, block: int = 4096):
    """Tet ids of ``rank`` under block-cyclic sharding: blocks of ``block``
    Morton-consecutive tets dealt round-robin."""
    ids = np.arange(T, dtype=np.int64)
    return ids[(ids // block) % world == rank]


def stats(w: Workload):
    k = np.diff(w.nbr_off)
    return {"T": w.T, "N": w.N, "V": int(len(w.verts)), "k_site_mean": float(k.mean()),
            "k_site_max": int(k.max()) if len(k) else 0, "hidden": int((k == 0).sum())}


def boundary_samples(verts, tets, n: int, seed: int = 0):
    """``n`` random points on the boundary surface of a tet mesh (the input shape's surface,
    PAPER.md:532 "randomly sample surface points"): boundary faces are the tet faces that
    belong to one tet; a face is drawn with probability proportional to its area and a point
    uniformly inside it.  Input generation only (no method arithmetic)."""
    t = np.asarray(tets)
    faces = np.concatenate([t[:, [1, 2, 3]], t[:, [0, 2, 3]], t[:, [0, 1, 3]], t[:, [0, 1, 2]]])
    key = np.sort(faces, axis=1)
    _, inv, cnt = np.unique(key, axis=0, return_inverse=True, return_counts=True)
    bnd = faces[cnt[inv.reshape(-1)] == 1]
    v = np.asarray(verts)
    a, b, c = v[bnd[:, 0]], v[bnd[:, 1]], v[bnd[:, 2]]
    area = 0.5 * np.linalg.norm(np.cross(b - a, c - a), axis=1)
    rng = np.random.default_rng(seed)
    pick = rng.choice(len(bnd), size=n, p=area / area.sum())
    r1, r2 = rng.random(n), rng.random(n)
    s = np.sqrt(r1)
    return (1 - s)[:, None] * a[pick] + (s * (1 - r2))[:, None] * b[pick] + \
        (s * r2)[:, None] * c[pick]
