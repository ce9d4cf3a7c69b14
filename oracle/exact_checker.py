"""Tiny exact checker -- TEST INFRASTRUCTURE ONLY (pins the C oracle).

Brute-force vertex enumeration of P(t, i) = t  n  {x : PD_i(x) <= PD_j(x), j in S} in exact
rational arithmetic, with no symbolic perturbation and no clipping order:

* half-spaces, written in Cartesian lattice coordinates X = 2^10 x:
    radical plane j   h_j(X) = PD_j(X) - PD_i(X) = 2 (Theta_i - Theta_j) . X + W_j - W_i,
                      W = |Theta|^2 - R^2
    tet face k        plane through the three vertices other than V_k, positive at V_k;
* vertices = every plane triple whose unique intersection point satisfies every half-space;
* the piece is non-empty iff the vertices span 3D (positive volume);
* a source is incident iff its plane holds >= 3 affinely independent vertices (positive-area
  2-face), so coincident sources are all listed (R7);
* volume and first moment exactly (Fractions) by fan triangulation of the facets.

Shares nothing with oracle.c (different coordinates, no SoS) or with the CUDA path.
"""
from __future__ import annotations

import functools
import itertools
from fractions import Fraction
from math import gcd

import numpy as np

L = 1024


def _lat(x):
    v = Fraction(float(x)) * L
    assert v.denominator == 1
    return int(v)


def _sub(a, b):
    return (a[0] - b[0], a[1] - b[1], a[2] - b[2])


def _cross(a, b):
    return (a[1] * b[2] - a[2] * b[1], a[2] * b[0] - a[0] * b[2], a[0] * b[1] - a[1] * b[0])


def _dot(a, b):
    return a[0] * b[0] + a[1] * b[1] + a[2] * b[2]


def _det3(a, b, c):
    return _dot(a, _cross(b, c))


def planes_for(tet_X, spheres_X, i, S):
    """Half-spaces (n, d, source) with n.X + d >= 0; sources: ('f', k) and ('r', j)."""
    out = []
    for k in range(4):
        a, b, c = [tet_X[m] for m in range(4) if m != k]
        n = _cross(_sub(b, a), _sub(c, a))
        d = -_dot(n, a)
        if _dot(n, tet_X[k]) + d < 0:
            n = (-n[0], -n[1], -n[2])
            d = -d
        out.append((n, d, ("f", k)))
    Ti, Ri = spheres_X[i][:3], spheres_X[i][3]
    Wi = _dot(Ti, Ti) - Ri * Ri
    for j in S:
        Tj, Rj = spheres_X[j][:3], spheres_X[j][3]
        Wj = _dot(Tj, Tj) - Rj * Rj
        n = (2 * (Ti[0] - Tj[0]), 2 * (Ti[1] - Tj[1]), 2 * (Ti[2] - Tj[2]))
        out.append((n, Wj - Wi, ("r", j)))
    return out


def _solve(p, q, r):
    """Homogeneous integer intersection (X, Y, Z, D), D > 0, gcd-normalised; None if singular."""
    (n1, d1, _), (n2, d2, _), (n3, d3, _) = p, q, r
    D = _det3(n1, n2, n3)
    if D == 0:
        return None
    rhs = (-d1, -d2, -d3)
    cols = list(zip(n1, n2, n3))  # columns of the 3x3 matrix with rows n1, n2, n3
    # Cramer: replace column c by rhs
    num = []
    for c in range(3):
        m = [list(n1), list(n2), list(n3)]
        for row in range(3):
            m[row][c] = rhs[row]
        num.append(_det3(tuple(m[0]), tuple(m[1]), tuple(m[2])))
    if D < 0:
        D, num = -D, [-v for v in num]
    g = gcd(gcd(gcd(abs(num[0]), abs(num[1])), abs(num[2])), D)
    return (num[0] // g, num[1] // g, num[2] // g, D // g)


def _val(pl, v):
    n, d, _ = pl
    return n[0] * v[0] + n[1] * v[1] + n[2] * v[2] + d * v[3]


def _affine_rank(pts):
    if not pts:
        return -1
    p0 = pts[0]
    vecs = [tuple(Fraction(p[c]) - Fraction(p0[c]) for c in range(3)) for p in pts[1:]]
    rank, basis = 0, []
    for v in vecs:
        if all(x == 0 for x in v):
            continue
        if rank == 0:
            basis.append(v)
            rank = 1
        elif rank == 1:
            if any(x != 0 for x in _cross(basis[0], v)):
                basis.append(v)
                rank = 2
        elif rank == 2:
            if _det3(basis[0], basis[1], v) != 0:
                return 3
    return rank


def exact_piece(tet_X, spheres_X, i, S):
    """Returns None (empty) or dict(vol, m1, facemask, inc) in lattice units, exact."""
    pls = planes_for(tet_X, spheres_X, i, S)
    verts = set()
    for a, b, c in itertools.combinations(range(len(pls)), 3):
        v = _solve(pls[a], pls[b], pls[c])
        if v is None:
            continue
        if all(_val(pl, v) >= 0 for pl in pls):
            verts.add(v)
    pts = [(Fraction(v[0], v[3]), Fraction(v[1], v[3]), Fraction(v[2], v[3])) for v in verts]
    if _affine_rank(pts) < 3:
        return None
    vlist = list(verts)
    o = tuple(sum(p[c] for p in pts) / len(pts) for c in range(3))
    facemask, inc = 0, []
    facets = {}
    for pl in pls:
        on = [k for k, v in enumerate(vlist) if _val(pl, v) == 0]
        if _affine_rank([pts[k] for k in on]) == 2:
            if pl[2][0] == "f":
                facemask |= 1 << pl[2][1]
            else:
                inc.append(pl[2][1])
            facets.setdefault(frozenset(on), pl)
    vol = Fraction(0)
    m1 = [Fraction(0)] * 3
    for on, pl in facets.items():
        P = [pts[k] for k in on]
        n = pl[0]
        ax = max(range(3), key=lambda c: abs(n[c]))
        u, w = [c for c in range(3) if c != ax]
        cu = sum(p[u] for p in P) / len(P)
        cw = sum(p[w] for p in P) / len(P)

        def cmp(p, q):
            a = (p[u] - cu, p[w] - cw)
            b = (q[u] - cu, q[w] - cw)
            ha = 0 if (a[1] > 0 or (a[1] == 0 and a[0] > 0)) else 1
            hb = 0 if (b[1] > 0 or (b[1] == 0 and b[0] > 0)) else 1
            if ha != hb:
                return ha - hb
            cr = a[0] * b[1] - a[1] * b[0]
            return -1 if cr > 0 else (1 if cr < 0 else 0)
        P.sort(key=functools.cmp_to_key(cmp))
        S6 = Fraction(0)
        fm = [Fraction(0)] * 3
        for k in range(1, len(P) - 1):
            a, b, c = P[0], P[k], P[k + 1]
            det = _det3(_sub(a, o), _sub(b, o), _sub(c, o))
            S6 += det
            for d in range(3):
                fm[d] += det * (o[d] + a[d] + b[d] + c[d]) / 24
        sg = 1 if S6 >= 0 else -1
        vol += sg * S6 / 6
        for d in range(3):
            m1[d] += sg * fm[d]
    return {"vol": vol, "m1": m1, "facemask": facemask, "inc": sorted(inc)}


def check_tet(verts, tets, spheres, t, i, S):
    """Exact piece of tet t and sphere i against sources S (list of sphere ids), converted to
    real units (Fractions): vol * 2^-30, m1 * 2^-40."""
    tet_X = [tuple(_lat(verts[v][c]) for c in range(3)) for v in tets[t]]
    sph_X = [tuple(_lat(s[c]) for c in range(4)) for s in spheres]
    r = exact_piece(tet_X, sph_X, i, S)
    if r is None:
        return None
    r["vol"] = r["vol"] / L ** 3
    r["m1"] = [m / L ** 4 for m in r["m1"]]
    return r


def exact_piece_cells(tet_X, spheres_X, i, S):
    """The piece P(t, i) as a cell complex, exactly (no SoS): None if empty, else
    (vertices, edges, facets) with vertices as exact homogeneous lattice points (X, Y, Z, D),
    edges as frozensets of two vertices that share two active planes and facets as
    (source, frozenset of vertices) for every plane holding a positive-area 2-face.
    ``generic`` is False when some vertex has more than three active planes (then the cell
    structure of the symbolically perturbed polytope may differ)."""
    pls = planes_for(tet_X, spheres_X, i, S)
    verts = set()
    for a, b, c in itertools.combinations(range(len(pls)), 3):
        v = _solve(pls[a], pls[b], pls[c])
        if v is not None and all(_val(pl, v) >= 0 for pl in pls):
            verts.add(v)
    pts = {v: (Fraction(v[0], v[3]), Fraction(v[1], v[3]), Fraction(v[2], v[3])) for v in verts}
    if _affine_rank(list(pts.values())) < 3:
        return None
    active = {v: frozenset(k for k, pl in enumerate(pls) if _val(pl, v) == 0) for v in verts}
    generic = all(len(a) == 3 for a in active.values())
    vl = list(verts)
    edges = set()
    for a in range(len(vl)):
        for b in range(a + 1, len(vl)):
            if len(active[vl[a]] & active[vl[b]]) >= 2:
                edges.add(frozenset((vl[a], vl[b])))
    facets = []
    for k, pl in enumerate(pls):
        on = [v for v in vl if k in active[v]]
        if _affine_rank([pts[v] for v in on]) == 2:
            facets.append((pl[2], frozenset(on)))
    return {"vertices": set(vl), "edges": edges, "facets": facets, "generic": generic}


def explicit_euler(verts, tets, spheres, nbr_off, nbr_idx, i):
    """Euler characteristics of the restricted elements of sphere i extracted explicitly
    ("rpc_euler equals V-E+F-C computed from an explicitly extracted ... complex"):
    the pieces of i in all tets are glued by their exact vertex coordinates into one cell
    complex; Euler(RPC) = V - E + F - C over it, and for each neighbour j Euler(RPF(i, j)) =
    V - E + F over its 2-faces on the radical plane h_ij.  Returns (rpc, {j: rpf}, generic)."""
    sph_X = [tuple(_lat(s[c]) for c in range(4)) for s in spheres]
    S = [int(j) for j in nbr_idx[nbr_off[i]:nbr_off[i + 1]]]
    if not S and len(spheres) > 1:
        return 0, {}, True  # hidden sphere (R4): no pieces
    V, E, F, C = set(), set(), set(), 0
    rpf = {}
    generic = True
    for t in range(len(tets)):
        tet_X = [tuple(_lat(verts[v][c]) for c in range(3)) for v in tets[t]]
        cell = exact_piece_cells(tet_X, sph_X, i, S)
        if cell is None:
            continue
        generic &= cell["generic"]
        C += 1
        V |= cell["vertices"]
        E |= cell["edges"]
        for src, on in cell["facets"]:
            F.add(on)
            if src[0] == "r":
                fv, fe, ff = rpf.setdefault(src[1], (set(), set(), set()))
                fv |= on
                fe |= {e for e in cell["edges"] if e <= on}
                ff.add(on)
    return (len(V) - len(E) + len(F) - C,
            {j: len(a) - len(b) + len(c) for j, (a, b, c) in rpf.items()}, generic)


def explicit_cc(verts, tets, spheres, nbr_off, nbr_idx, i):
    """CC numbers of the restricted elements of sphere i from the explicitly extracted complex
    (exact rational vertices, no SoS): pieces are connected when they share a 2-face (equal
    vertex sets), facets on the radical plane h_ij when they share an edge.  Returns
    (cc of RPC(m_i), {j: cc of RPF(m_i, m_j)}, generic)."""
    sph_X = [tuple(_lat(s[c]) for c in range(4)) for s in spheres]
    S = [int(j) for j in nbr_idx[nbr_off[i]:nbr_off[i + 1]]]
    if not S and len(spheres) > 1:
        return 0, {}, True
    cells, generic = [], True
    for t in range(len(tets)):
        tet_X = [tuple(_lat(verts[v][c]) for c in range(3)) for v in tets[t]]
        cell = exact_piece_cells(tet_X, sph_X, i, S)
        if cell is not None:
            generic &= cell["generic"]
            cells.append(cell)

    def components(items, keys):
        parent = list(range(len(items)))

        def find(x):
            while parent[x] != x:
                parent[x] = parent[parent[x]]
                x = parent[x]
            return x
        owner = {}
        for a, ks in enumerate(keys):
            for k in ks:
                if k in owner:
                    ra, rb = find(a), find(owner[k])
                    parent[max(ra, rb)] = min(ra, rb)
                else:
                    owner[k] = a
        return len({find(a) for a in range(len(items))})

    rpc = components(cells, [[on for _, on in c["facets"]] for c in cells])
    rpf = {}
    per_j = {}
    for c in cells:
        for src, on in c["facets"]:
            if src[0] == "r":
                per_j.setdefault(src[1], []).append([e for e in c["edges"] if e <= on])
    for j, facet_edges in per_j.items():
        rpf[j] = components(facet_edges, facet_edges)
    return rpc, rpf, generic


def explicit_medial_faces(verts, tets, spheres, nbr_off, nbr_idx):
    """Triangles (i, j, k) of the dual medial mesh from the exact pieces (no SoS): sphere i's
    piece has an edge of positive length on both radical planes h_ij and h_ik."""
    sph_X = [tuple(_lat(s[c]) for c in range(4)) for s in spheres]
    faces = set()
    generic = True
    for i in range(len(spheres)):
        S = [int(j) for j in nbr_idx[nbr_off[i]:nbr_off[i + 1]]]
        if not S and len(spheres) > 1:
            continue
        for t in range(len(tets)):
            tet_X = [tuple(_lat(verts[v][c]) for c in range(3)) for v in tets[t]]
            cell = exact_piece_cells(tet_X, sph_X, i, S)
            if cell is None:
                continue
            generic &= cell["generic"]
            pls = planes_for(tet_X, sph_X, i, S)
            act = {v: frozenset(k for k, pl in enumerate(pls) if _val(pl, v) == 0)
                   for v in cell["vertices"]}
            for e in cell["edges"]:
                u, w = tuple(e)
                rad = sorted(pls[k][2][1] for k in act[u] & act[w] if pls[k][2][0] == "r")
                for a in range(len(rad)):
                    for b in range(a + 1, len(rad)):
                        faces.add(tuple(sorted((i, rad[a], rad[b]))))
    return sorted(faces), generic


def explicit_rpe(verts, tets, spheres, nbr_off, nbr_idx, i):
    """Restricted power edges of sphere i extracted explicitly (exact rational vertices, no
    SoS): in every piece of i, an edge lying on the radical planes h_ij and h_ik (j < k) is
    part of RPE(m_i, m_j, m_k); the parts are glued across tets by their exact endpoints.
    Returns ({(j, k): V - E}, {(j, k): connected components}, generic)."""
    sph_X = [tuple(_lat(s[c]) for c in range(4)) for s in spheres]
    S = [int(j) for j in nbr_idx[nbr_off[i]:nbr_off[i + 1]]]
    if not S and len(spheres) > 1:
        return {}, {}, True
    per = {}  # (j, k) -> set of edges (frozensets of two exact vertices)
    generic = True
    for t in range(len(tets)):
        tet_X = [tuple(_lat(verts[v][c]) for c in range(3)) for v in tets[t]]
        cell = exact_piece_cells(tet_X, sph_X, i, S)
        if cell is None:
            continue
        generic &= cell["generic"]
        pls = planes_for(tet_X, sph_X, i, S)
        act = {v: frozenset(k for k, pl in enumerate(pls) if _val(pl, v) == 0)
               for v in cell["vertices"]}
        for e in cell["edges"]:
            u, w = tuple(e)
            rad = sorted(pls[k][2][1] for k in act[u] & act[w] if pls[k][2][0] == "r")
            for a in range(len(rad)):
                for b in range(a + 1, len(rad)):
                    per.setdefault((rad[a], rad[b]), set()).add(e)
    euler, cc = {}, {}
    for key, edges in per.items():
        vs = set().union(*edges)
        euler[key] = len(vs) - len(edges)
        parent = {v: v for v in vs}

        def find(x):
            while parent[x] != x:
                parent[x] = parent[parent[x]]
                x = parent[x]
            return x
        for e in edges:
            u, w = tuple(e)
            ru, rw = find(u), find(w)
            if ru != rw:
                parent[ru] = rw
        cc[key] = len({find(v) for v in vs})
    return euler, cc, generic
