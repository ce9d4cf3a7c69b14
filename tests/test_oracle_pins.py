"""Pins of the CPU oracle against what the paper and the mathematics fix (-m "not gpu").

Each test names the passage it follows.  None of them re-types the oracle's formulas: they
check it against the exact rational checker (brute-force vertex enumeration, no SoS), brute
force over all spheres, closed forms, SPEC.md worked examples and invariants.
"""
import json
import os
from fractions import Fraction

import numpy as np
import pytest

import oracle
import rpd_workloads as W
from oracle import exact_checker as X
from tests.helpers import compare_results, piece_tet, tet_diams, tet_volumes

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))


# ----------------------------------------------------------------------------- SPEC examples


@pytest.mark.parametrize("case", GOLD["power_distance"])
def test_power_distance_spec(case):
    """PD(m, x) = |x - theta|^2 - r^2."""
    assert oracle.power_distance(case["sphere"], case["x"]) == case["pd"]


def _cube_mesh(side):
    return W.unit_cube_6tets(scale=side)


def _axis_pair(xi, ri, xj, rj, y=1.0, z=1.0):
    sph = np.array([[xi, y, z, ri], [xj, y, z, rj]], dtype=np.float64)
    off = np.array([0, 1, 2], np.int32)
    idx = np.array([1, 0], np.int32)
    return sph, off, idx


@pytest.mark.parametrize("case", GOLD["radical_plane"])
def test_radical_plane_spec_via_volumes(case):
    """the radical plane of the two spheres is x = plane_x; cutting the
    [0,2]^3 cube (6 Kuhn tets) must give volume 4*plane_x to sphere i (x < plane_x).  Spheres
    are shifted by +1 in y,z (and x by 0) to stay in the lattice box."""
    verts, tets = _cube_mesh(2.0)
    si, sj = case["sphere_i"], case["sphere_j"]
    sph, off, idx = _axis_pair(si[0], si[3], sj[0], sj[3])
    r = oracle.rpd(verts, tets, sph, off, idx)
    vol_i = r["piece_vol"][r["piece_sphere"] == 0].sum()
    vol_j = r["piece_vol"][r["piece_sphere"] == 1].sum()
    assert abs(vol_i - 4.0 * case["plane_x"]) < 1e-12
    assert abs(vol_j - (8.0 - 4.0 * case["plane_x"])) < 1e-12
    # swapping the arguments gives the same plane with opposite orientation
    r2 = oracle.rpd(verts, tets, sph[::-1].copy(), off, idx)
    assert abs(r2["piece_vol"][r2["piece_sphere"] == 1].sum() - vol_i) < 1e-12


@pytest.mark.parametrize("case", GOLD["kuhn_axis_plane"]["cases"])
def test_kuhn_closed_forms(case):
    """per-Kuhn-tet volumes of the part x < c of the unit cube."""
    c = case["c"]
    verts, tets = _cube_mesh(1.0)
    # equal radii at x = c -/+ 1/4 (y, z = 1/2): bisector x = c
    sph = np.array([[c - 0.25, 0.5, 0.5, 0.125], [c + 0.25, 0.5, 0.5, 0.125]])
    off, idx = np.array([0, 1, 2], np.int32), np.array([1, 0], np.int32)
    r = oracle.rpd(verts, tets, sph, off, idx)
    cen = verts[tets].mean(1)
    for t in range(6):
        order = np.argsort(cen[t])
        kind = "largest" if order[2] == 0 else ("smallest" if order[0] == 0 else "middle")
        p = [k for k in range(r["piece_off"][t], r["piece_off"][t + 1])
             if r["piece_sphere"][k] == 0]
        v = r["piece_vol"][p[0]] if p else 0.0
        assert abs(v - case[kind]) < 1e-14, (t, kind, v, case[kind])
        # the bisector is a positive-area 2-face of both pieces: incidences list each other
        io = r["inc_off"]
        for k in range(r["piece_off"][t], r["piece_off"][t + 1]):
            other = 1 - r["piece_sphere"][k]
            assert r["inc_sphere"][io[k]:io[k + 1]].tolist() == [other]


# ----------------------------------------------------------------------------- special cases


def test_single_sphere_whole_tet():
    """SPEC.md:228 / north star: one sphere -> every tet relates and its cell is the whole
    mesh: piece = tet, facemask 0xF, no incidences, m1 = vol * centroid."""
    w = W.make_shape_workload("one", 600, 1, seed=2, cache=False)
    assert w.N == 1
    r = oracle.rpd_workload(w)
    assert np.array_equal(r["cand_off"], np.arange(w.T + 1))
    assert np.all(r["piece_facemask"] == 15) and len(r["inc_sphere"]) == 0
    vt = tet_volumes(w.verts, w.tets)
    assert np.allclose(r["piece_vol"], vt, rtol=1e-13, atol=0)
    cen = w.verts[w.tets].mean(1)
    assert np.allclose(r["piece_m1"], cen * vt[:, None], rtol=1e-12, atol=0)


ALG1 = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "alg1_cases.json")))


def alg1_case(case):
    """(verts, tets, spheres, nbr_off, nbr_idx) of a golden Alg. 1 case."""
    return (np.array(case["verts"], np.float64), np.array(case["tets"], np.int32),
            np.array(case["spheres"], np.float64), np.array(case["nbr_off"], np.int32),
            np.array(case["nbr_idx"], np.int32))


def check_alg1_golden(case, r):
    """Compare a result dict with the hand-derived answers of ``case`` (exact for the
    combinatorics, 1e-15 relative for the volumes and centroids, which are dyadic)."""
    verts, tets = alg1_case(case)[:2]
    for a, want in enumerate(case["cand"]):
        got = r["cand_idx"][r["cand_off"][a]:r["cand_off"][a + 1]].tolist()
        assert got == want, (case["name"], a, got, want)
    for a, want in enumerate(case["pieces"]):
        if want is None:
            continue
        ps = range(r["piece_off"][a], r["piece_off"][a + 1])
        assert [int(r["piece_sphere"][p]) for p in ps] == [w["sphere"] for w in want]
        for p, w in zip(ps, want):
            vol = float(Fraction(*w["vol"]))
            cen = np.array([float(Fraction(*x)) for x in w["centroid"]])
            assert abs(r["piece_vol"][p] - vol) <= 1e-15 * vol
            assert np.allclose(r["piece_m1"][p], vol * cen, rtol=1e-14, atol=1e-17)
            assert int(r["piece_facemask"][p]) == w["facemask"]
            inc = r["inc_sphere"][r["inc_off"][p]:r["inc_off"][p + 1]].tolist()
            assert inc == w["inc"]


@pytest.mark.parametrize("case", ALG1["cases"], ids=lambda c: c["name"])
def test_alg1_golden_cases(case):
    """PAPER.md:21-50 Alg. 1 against hand-derived answers (tests/golden/alg1_cases.json):
    a vertex exactly on h_ij does not count (strict, reading R2), a tet whose planes each have
    a positive vertex is related even though its piece is empty (the acknowledged
    over-report), and a single failing neighbour -- first or last in the list -- rejects."""
    args = alg1_case(case)
    r = oracle.rpd(*args)
    check_alg1_golden(case, r)
    R = oracle.relation_matrix(*args)
    for a, want in enumerate(case["cand"]):
        assert np.nonzero(R[a])[0].tolist() == want
    # brute force (every sphere clipped against all others) agrees on the pieces, so the
    # over-reported candidate is really empty
    rb = oracle.rpd(*args, brute=True)
    for k in ("piece_off", "piece_sphere", "piece_facemask", "inc_off", "inc_sphere"):
        assert np.array_equal(r[k], rb[k]), k


def test_relation_rejects_dominated_tet():
    """a tet whose 4 vertices are all power-closer to neighbour j than to i is
    not related to i."""
    verts, tets = _cube_mesh(1.0)
    sph = np.array([[10.0, 10.0, 10.0, 0.0], [0.5, 0.5, 0.5, 0.0]])
    off, idx = np.array([0, 1, 2], np.int32), np.array([1, 0], np.int32)
    R = oracle.relation_matrix(verts, tets, sph, off, idx)
    assert not R[:, 0].any() and R[:, 1].all()


def test_hidden_spheres_have_no_candidates():
    """DESIGN.md R4: k_site = 0 and N > 1 -> hidden -> no candidates; brute force agrees that
    the cell is empty (all N-1 planes)."""
    w = W.make_c1(5, degenerate=True, big=True)
    k = np.diff(w.nbr_off)
    hidden = np.nonzero(k == 0)[0]
    r = oracle.rpd_workload(w)
    assert not np.isin(r["cand_idx"], hidden).any()
    rb = oracle.rpd_workload(w, brute=True)
    assert not np.isin(rb["piece_sphere"], hidden).any()


# ----------------------------------------------------------------------------- exact checker


def _exact_compare(w, brute):
    r = oracle.rpd_workload(w, brute=brute)
    L = oracle.per_tet_lists(r, w.T)
    n_nonempty = 0
    for t in range(w.T):
        cands, pcs = L[t]
        pmap = {p[0]: p for p in pcs}
        for i in (range(w.N) if brute else cands):
            if brute:
                S = [j for j in range(w.N) if j != i]
            else:
                S = w.nbr_idx[w.nbr_off[i]:w.nbr_off[i + 1]].tolist()
            e = X.check_tet(w.verts, w.tets, w.spheres, t, i, S)
            p = pmap.get(i)
            if e is None:
                assert p is None, ("spurious piece", t, i)
                continue
            n_nonempty += 1
            assert p is not None, ("missing piece", t, i)
            assert p[3] == e["facemask"], (t, i, p[3], e["facemask"])
            assert list(p[4]) == e["inc"], (t, i, p[4], e["inc"])
            assert abs(p[1] - float(e["vol"])) <= 1e-13
            assert max(abs(p[2][d] - float(e["m1"][d])) for d in range(3)) <= 1e-13
    return r, n_nonempty


@pytest.mark.parametrize("seed,deg,big", [(0, False, False), (1, False, False),
                                          (0, True, False), (1, True, False), (2, True, False),
                                          (5, True, True), (6, True, True)])
def test_oracle_equals_exact_checker_c1(seed, deg, big):
    """the oracle's pieces (non-empty, facemask, incidences, vol, m1)
    equal exact rational vertex enumeration on C1a (generic) and C1b (degenerate: radical
    planes through Kuhn faces and vertices, exercising the SoS rule), k_site and brute mode."""
    w = W.make_c1(seed, degenerate=deg, big=big)
    r, n1 = _exact_compare(w, brute=False)
    rb, n2 = _exact_compare(w, brute=True)
    assert n1 == n2 > 0
    if deg:
        assert rb["stats"]["n_zero_hits"] > 0   # the degenerate configs do hit exact zeros


@pytest.mark.parametrize("seed", [0, 1, 2, 3])
def test_oracle_equals_exact_checker_tiny_grid(seed):
    """Random tiny configs on a 2^3-cube Kuhn mesh (48 tets), coarse (degenerate) spheres."""
    w = W.random_tiny(seed, n_spheres=10, grid=2, coarse=(seed % 2 == 1))
    _exact_compare(w, brute=False)


# ----------------------------------------------------------------------------- invariants


@pytest.fixture(scope="module")
def small_shape():
    return W.make_shape_workload("S", 2000, 150, seed=3, n_batches=2, batch_m=12, clusters=3,
                                 cache=False)


def test_partition(small_shape):
    """SPEC.md:251 / north star: per tet, restricted cell volumes sum to the tet volume."""
    w = small_shape
    r = oracle.rpd_workload(w)
    s = np.zeros(w.T)
    np.add.at(s, piece_tet(r), r["piece_vol"])
    vt = tet_volumes(w.verts, w.tets)
    assert np.max(np.abs(s - vt) / vt) < 1e-12
    assert np.all(r["piece_vol"] > 0)


def test_brute_force_equals_ksite(small_shape):
    """North star: on tiny inputs the oracle must agree with brute force (all N spheres as
    candidates and as clipping planes).  Incidences compared after restricting brute force
    to N(i) (they differ only if a non-neighbour plane coincides with a 2-face)."""
    w = small_shape
    ids = np.arange(0, w.T, 23, dtype=np.int32)
    r = oracle.rpd_workload(w, tet_ids=ids)
    rb = oracle.rpd_workload(w, tet_ids=ids, brute=True)
    rb = dict(rb)
    io = rb["inc_off"]
    keep_inc, new_off = [], [0]
    for p in range(len(rb["piece_sphere"])):
        i = rb["piece_sphere"][p]
        nb = set(w.nbr_idx[w.nbr_off[i]:w.nbr_off[i + 1]].tolist())
        keep_inc += [j for j in rb["inc_sphere"][io[p]:io[p + 1]] if j in nb]
        new_off.append(len(keep_inc))
    rb["inc_sphere"] = np.array(keep_inc, np.int32)
    rb["inc_off"] = np.array(new_off, np.int32)
    errs = compare_results(r, rb, w.verts, w.tets, tet_ids=ids, rel=1e-12, check_cands=False)
    assert not errs, errs
    # Alg. 1 soundness: every brute-force non-empty piece is a candidate
    for a in range(len(ids)):
        cands = set(r["cand_idx"][r["cand_off"][a]:r["cand_off"][a + 1]].tolist())
        for p in range(rb["piece_off"][a], rb["piece_off"][a + 1]):
            assert rb["piece_sphere"][p] in cands


def test_voronoi_reduction():
    """PAPER.md:347 (power diagram = Voronoi diagram for equal weights): radii all equal to c
    and radii all 0 give byte-identical outputs; the neighbour lists equal Delaunay edges."""
    from scipy.spatial import Delaunay
    w = W.make_shape_workload("V", 1500, 120, seed=4, radius_mode="equal", cache=False)
    s0 = w.spheres.copy()
    s0[:, 3] = 0.0
    sc = w.spheres.copy()
    sc[:, 3] = 0.75
    off, idx = W.power_neighbours(s0)
    d = Delaunay(s0[:, :3])
    ed = set()
    for simp in d.simplices:
        for a in range(4):
            for b in range(4):
                if a != b:
                    ed.add((simp[a], simp[b]))
    mine = {(i, j) for i in range(len(s0)) for j in idx[off[i]:off[i + 1]]}
    assert mine == ed
    r0 = oracle.rpd(w.verts, w.tets, s0, off, idx)
    rc = oracle.rpd(w.verts, w.tets, sc, off, idx)
    for k in r0:
        if k != "stats":
            assert np.array_equal(r0[k], rc[k]), k
    # Euclidean membership: each piece's centroid is nearest (Euclidean) to its sphere
    from scipy.spatial import cKDTree
    cen = r0["piece_m1"] / r0["piece_vol"][:, None]
    dist, nn = cKDTree(s0[:, :3]).query(cen, k=2)
    own = np.linalg.norm(cen - s0[r0["piece_sphere"], :3], axis=1)
    assert np.all(own <= dist[:, 0] + 1e-9)


def test_power_membership(small_shape):
    """Power-cell membership: a piece's centroid is power-nearest to its sphere; dyadic sample
    points with a unique power-nearest sphere lie in a tet whose candidates contain it."""
    w = small_shape
    r = oracle.rpd_workload(w)
    cen = r["piece_m1"] / r["piece_vol"][:, None]
    th, rad = w.spheres[:, :3], w.spheres[:, 3]
    pd = ((cen[:, None, :] - th[None]) ** 2).sum(-1) - rad[None] ** 2
    own = pd[np.arange(len(cen)), r["piece_sphere"]]
    assert np.all(own <= pd.min(1) + 1e-9 * (1 + np.abs(own)))
    rng = np.random.default_rng(0)
    pt = piece_tet(r)
    for t in rng.choice(w.T, 60, replace=False):
        P = w.verts[w.tets[t]]
        lam = rng.dirichlet(np.ones(4))
        x = W.to_lattice(lam @ P)
        pdx = ((x - th) ** 2).sum(1) - rad ** 2
        o = np.argsort(pdx)
        if pdx[o[1]] - pdx[o[0]] < 1e-6:
            continue
        # x may fall just outside t after rounding; only check interior-by-margin points
        lam_chk = np.linalg.solve(np.c_[P.T[:, 1:] - P.T[:, :1]], x - P[0])
        lam4 = np.r_[1 - lam_chk.sum(), lam_chk]
        if lam4.min() <= 1e-9:
            continue
        cands = r["cand_idx"][r["cand_off"][t]:r["cand_off"][t + 1]]
        assert o[0] in cands
        assert o[0] in r["piece_sphere"][pt == t]


def test_partial_update_equals_full(small_shape):
    """DESIGN.md R11/R12: partial update == full
    recompute (pieces) for inputs with no exact-degeneracy hits; M = 0 is the identity;
    clean tets keep their previous pieces byte-identically."""
    w = small_shape
    r = oracle.rpd_workload(w)
    n_old = w.N
    prev = r
    for (sph, off, idx) in w.batches:
        part, dirty = oracle.partial_update(prev, w.verts, w.tets, sph, off, idx, n_old)
        full = oracle.rpd(w.verts, w.tets, sph, off, idx)
        assert full["stats"]["n_zero_hits"] == 0
        errs = compare_results(part, full, w.verts, w.tets, rel=1e-12, check_cands=False)
        assert not errs, errs
        # dirty tets: candidates equal full recompute
        clean = np.setdiff1d(np.arange(w.T), dirty)
        Lp, Lf, Lprev = (oracle.per_tet_lists(x, w.T) for x in (part, full, prev))
        for t in dirty:
            assert Lp[t][0] == Lf[t][0]
        for t in clean:
            assert Lp[t] == Lprev[t]
        assert 0 < len(dirty) < w.T
        prev, n_old = part, len(sph)
    # identity
    same, dirty = oracle.partial_update(prev, w.verts, w.tets, *w.batches[-1], n_old)
    assert len(dirty) == 0
    for k in same:
        assert np.array_equal(same[k], oracle.from_per_tet_lists(
            oracle.per_tet_lists(prev, w.T))[k])


def test_csr_merge_equals_per_tet_lists(small_shape):
    """The vectorised R11 merge (CSR row selection) equals the plain per-tet-list merge."""
    w = small_shape
    prev = oracle.rpd_workload(w)
    sph, off, idx = w.batches[0]
    part, dirty = oracle.partial_update(prev, w.verts, w.tets, sph, off, idx, w.N)
    new = oracle.rpd(w.verts, w.tets, sph, off, idx, tet_ids=dirty)
    L = oracle.per_tet_lists(prev, w.T)
    Ln = oracle.per_tet_lists(new, len(dirty))
    for a, t in enumerate(dirty):
        L[t] = Ln[a]
    slow = oracle.from_per_tet_lists(L)
    for k in slow:
        assert np.array_equal(np.asarray(part[k]), slow[k]), k


# ----------------------------------------------------------------------------- fractional Euler
# "Fractional Euler Characteristic"


def _mesh_euler(tets):
    """V - E + F - T of a tet mesh, by counting its distinct simplices (plain definition)."""
    Vs, Es, Fs = set(), set(), set()
    for t in np.asarray(tets).tolist():
        Vs |= set(t)
        Es |= {frozenset((t[a], t[b])) for a in range(4) for b in range(a + 1, 4)}
        Fs |= {frozenset(t[:k] + t[k + 1:]) for k in range(4)}
    return len(Vs) - len(Es) + len(Fs) - len(tets)


@pytest.mark.parametrize("make,expect", [
    (lambda: W.unit_cube_6tets(), 1),
    (lambda: W.kuhn_grid_mesh((2, 2, 2), 512, (0, 0, 0), morton=False), 1),
    (lambda: (lambda w: (w.verts, w.tets))(
        W.make_shape_workload("one", 700, 1, seed=2, cache=False)), 0)])
def test_euler_single_sphere_is_mesh_euler(make, expect):
    """the payloads 1/(tets sharing the element) make the per-tet sums add up
    to the mesh's Euler characteristic; with one sphere every tet is one whole piece, so
    Euler(RPC) = V - E + F - T.  The box with a through-hole (genus 1) gives 0: the paper's
    Fig. 4(a) "CC = 1 but Euler = 0" for one sphere covering a torus-like solid."""
    verts, tets = make()
    sph = np.array([[0.5, 0.5, 0.5, 0.25]])
    r = oracle.rpd(verts, tets, sph, np.zeros(2, np.int32), np.zeros(0, np.int32), euler=True)
    rpc, rpf = oracle.euler_sums(r, 1, np.zeros(2, np.int32), np.zeros(0, np.int32))
    assert _mesh_euler(tets) == expect
    assert rpc[0] == expect and not rpf
    assert len(r["piece_euler"]) == len(tets)


@pytest.mark.parametrize("make", [lambda: W.make_c1(0), lambda: W.make_c1(1), lambda: W.make_c1(3),
                                  lambda: W.random_tiny(0, n_spheres=14, grid=2),
                                  lambda: W.random_tiny(2, n_spheres=14, grid=2)])
def test_euler_equals_explicit_extraction(make):
    """on small inputs the fractional sums equal V - E + F - C of the restricted
    elements extracted explicitly -- every piece of sphere i enumerated exactly (rational
    vertices, no SoS) and glued across tets by coordinates -- for every RPC and every RPF."""
    w = make()
    r = oracle.rpd_workload(w, euler=True)
    rpc, rpf = oracle.euler_sums(r, w.N, w.nbr_off, w.nbr_idx)
    for i in range(w.N):
        e_rpc, e_rpf, generic = X.explicit_euler(w.verts, w.tets, w.spheres, w.nbr_off,
                                                 w.nbr_idx, i)
        assert generic
        assert rpc[i] == e_rpc, i
        assert {j: v for (a, j), v in rpf.items() if a == i} == e_rpf, i


@pytest.mark.parametrize("make", [lambda: W.make_c1(0, degenerate=True),
                                  lambda: W.make_c1(6, degenerate=True, big=True),
                                  lambda: W.random_tiny(3, n_spheres=14, grid=2, coarse=True),
                                  lambda: W.make_shape_workload("E", 1500, 120, seed=4,
                                                                cache=False)])
def test_euler_sums_are_integers(make):
    """The fractional payloads of the elements shared between tets add up across the pieces
    of one sphere (Eq. (1): 1/2 + 1/2 = 1), so every RPC and RPF sum is an integer, also on
    degenerate inputs (symbolically perturbed complex); RPF(m_i, m_j) seen from m_i equals
    the one seen from m_j when no exact-zero predicate occurred."""
    w = make()
    r = oracle.rpd_workload(w, euler=True)
    rpc, rpf = oracle.euler_sums(r, w.N, w.nbr_off, w.nbr_idx)
    assert all(x.denominator == 1 for x in rpc)
    assert all(x.denominator == 1 for x in rpf.values())
    if r["stats"]["n_zero_hits"] == 0:
        for (i, j), v in rpf.items():
            assert rpf.get((j, i)) == v, (i, j)
    # pieces of a mesh whose spheres all have cells inside it are mostly balls (Euler 1)
    assert sum(1 for x in rpc if x == 1) >= 0.5 * sum(1 for x in rpc if x != 0)


def test_euler_unstructured_mesh():
    """an unstructured (Delaunay) mesh whose sharing counts have a common multiple
    far beyond 2^50 (valences up to ~60): the per-tet denominators keep every value exact --
    one sphere gives the mesh's Euler characteristic V - E + F - T = 1 (a convex ball), and
    with many spheres every RPC / RPF sum is an integer."""
    import math
    w = W.delaunay_workload(2000, 60, seed=1)
    L = 1  # the common denominator a global-lcm scheme would need
    r1 = oracle.rpd(w.verts, w.tets, np.array([[8.0, 8.0, 8.0, 0.5]]), np.zeros(2, np.int32),
                    np.zeros(0, np.int32), euler=True)
    rpc1, _ = oracle.euler_sums(r1, 1, np.zeros(2, np.int32), np.zeros(0, np.int32))
    assert _mesh_euler(w.tets) == 1 and rpc1 == [1]
    for d in set(r1["piece_euler_den"].tolist()):
        L = L * d // math.gcd(L, d)
    assert math.log2(L) > 60
    r = oracle.rpd_workload(w, euler=True)
    rpc, rpf = oracle.euler_sums(r, w.N, w.nbr_off, w.nbr_idx)
    assert all(x.denominator == 1 for x in rpc) and all(x.denominator == 1 for x in rpf.values())
    assert sum(1 for x in rpc if x == 1) >= 0.5 * sum(1 for x in rpc if x != 0)


def test_euler_unstructured_explicit_extraction():
    """The per-tet-denominator sums equal the explicit extraction on a small Delaunay mesh."""
    w = W.delaunay_workload(40, 8, seed=3, box=4.0)
    r = oracle.rpd_workload(w, euler=True)
    rpc, rpf = oracle.euler_sums(r, w.N, w.nbr_off, w.nbr_idx)
    for i in range(w.N):
        e_rpc, e_rpf, generic = X.explicit_euler(w.verts, w.tets, w.spheres, w.nbr_off,
                                                 w.nbr_idx, i)
        if not generic:
            continue
        assert rpc[i] == e_rpc, i
        assert {j: v for (a, j), v in rpf.items() if a == i} == e_rpf, i


@pytest.mark.parametrize("make", [lambda: W.make_c1(0), lambda: W.make_c1(1), lambda: W.make_c1(3),
                                  lambda: W.random_tiny(0, n_spheres=14, grid=2),
                                  lambda: W.random_tiny(2, n_spheres=14, grid=2)])
def test_rpe_euler_and_cc_equal_explicit_extraction(make):
    """PAPER.md:439, 497, 506 ("RPC, RPF, RPE to have CC=1 and Euler=1"; the fractional Euler
    characteristics of "all of its restricted elements (RPCs, RPFs, RPEs)"): the fractional
    sums over the pieces' edges on h_ij and h_ik and the face-glued CC numbers equal V - E and
    the components of the restricted power edges extracted explicitly (exact rational piece
    vertices, no SoS, glued across tets by coordinates)."""
    w = make()
    r = oracle.rpd_workload(w, euler=True)
    eu = oracle.rpe_sums(r)
    cc = oracle.rpe_topology(r, w.tets)
    assert eu and set(eu) == set(cc)
    for i in range(w.N):
        e_eu, e_cc, generic = X.explicit_rpe(w.verts, w.tets, w.spheres, w.nbr_off, w.nbr_idx,
                                            i)
        assert generic
        assert {(j, k): v for (a, j, k), v in eu.items() if a == i} == e_eu, i
        assert {(j, k): v for (a, j, k), v in cc.items() if a == i} == e_cc, i


def test_rpe_through_the_hole_has_two_components():
    """Three equal spheres whose centres are a right triangle in the plane x = 32 with its
    circumcentre on the hole's diameter line (y = 26, z = 20): their cells meet along that line
    (it lies on all three bisector planes), which crosses the genus-1 solid twice (x in
    [2, 23] and [41, 62]; the hole spans x in [23, 41]).  So RPE(m_0, m_1, m_2) is two segments:
    Euler 2 and CC 2, seen from each of the three spheres (the edge analogue of the paper's
    Fig. 4(b) RPF with CC = 2)."""
    w = W.make_shape_workload("one", 700, 1, seed=2, cache=False)
    sph = np.array([[32.0, 32.0, 20.0, 1.0], [32.0, 20.0, 20.0, 1.0], [32.0, 26.0, 26.0, 1.0]])
    off, idx = np.array([0, 2, 4, 6], np.int32), np.array([1, 2, 0, 2, 0, 1], np.int32)
    r = oracle.rpd(w.verts, w.tets, sph, off, idx, euler=True)
    assert oracle.rpe_sums(r) == {(0, 1, 2): 2, (1, 0, 2): 2, (2, 0, 1): 2}
    assert oracle.rpe_topology(r, w.tets) == {(0, 1, 2): 2, (1, 0, 2): 2, (2, 0, 1): 2}


@pytest.mark.parametrize("make", [lambda: W.make_c1(0, degenerate=True),
                                  lambda: W.random_tiny(3, n_spheres=14, grid=2, coarse=True),
                                  lambda: W.make_shape_workload("E", 1500, 120, seed=4,
                                                                cache=False)])
def test_rpe_sums_are_integers_and_symmetric(make):
    """Every RPE sum is an integer (shared endpoints on tet faces add 1/2 + 1/2), also on
    degenerate inputs, and RPE(m_i, m_j, m_k) is the same element seen from each of its three
    spheres when no exact-zero predicate occurred."""
    w = make()
    r = oracle.rpd_workload(w, euler=True)
    eu = oracle.rpe_sums(r)
    assert eu and all(v.denominator == 1 for v in eu.values())
    if r["stats"]["n_zero_hits"] == 0:
        for (i, j, k), v in eu.items():
            tri = sorted((i, j, k))
            for a in tri:
                b, c = [x for x in tri if x != a]
                assert eu.get((a, b, c)) == v, (i, j, k)


def test_euler_partial_update_equals_full(small_shape):
    """R11 with the Euler payloads: the partially updated pieces carry the same fractional
    Euler characteristics as a full recompute."""
    w = small_shape
    prev = oracle.rpd_workload(w, euler=True)
    n_old = w.N
    for (sph, off, idx) in w.batches:
        part, _ = oracle.partial_update(prev, w.verts, w.tets, sph, off, idx, n_old, euler=True)
        full = oracle.rpd(w.verts, w.tets, sph, off, idx, euler=True)
        assert part["euler_denom"] == full["euler_denom"]
        for k in ("piece_euler", "rpf_off", "rpf_sphere", "rpf_euler", "rpe_off", "rpe_j",
                  "rpe_k", "rpe_euler", "rpe_fm"):
            assert np.array_equal(part[k], full[k]), k
        prev, n_old = part, len(sph)


# ----------------------------------------------------------------------------- CC numbers
# "CC Number"


def _genus_one_spheres(xs, r=1.0):
    """Spheres on the hole's axis line (y = 26, z = 20) of the box-with-hole solid (hole:
    centre (32, 26), radius 9), neighbours = consecutive spheres."""
    n = len(xs)
    sph = np.array([[x, 26.0, 20.0, r] for x in xs])
    idx, off = [], [0]
    for a in range(n):
        idx += [b for b in (a - 1, a + 1) if 0 <= b < n]
        off.append(len(idx))
    return sph, np.array(off, np.int32), np.array(idx, np.int32)


def test_cc_torus_two_spheres_rpf_has_two_components():
    """PAPER.md Fig. 4(b): two spheres on a torus-like solid -- the RPF between them has
    CC = 2 (and Euler 2: two disks), each RPC is one contractible C-shaped half."""
    w = W.make_shape_workload("one", 700, 1, seed=2, cache=False)
    sph, off, idx = _genus_one_spheres([20.0, 44.0])
    r = oracle.rpd(w.verts, w.tets, sph, off, idx, euler=True)
    rpc_cc, rpf_cc = oracle.topology(r, w.tets, 2)
    rpc_eu, rpf_eu = oracle.euler_sums(r, 2, off, idx)
    assert rpc_cc == [1, 1] and rpf_cc == {(0, 1): 2, (1, 0): 2}
    assert rpc_eu == [1, 1] and rpf_eu == {(0, 1): 2, (1, 0): 2}


def test_cc_slab_cell_has_two_components():
    """PAPER.md Fig. 6(a): the RPC of the middle sphere is a slab narrower than the hole, cut
    into two components (CC = 2, Euler 2); its RPFs are two segments-wide strips each."""
    w = W.make_shape_workload("one", 700, 1, seed=2, cache=False)
    sph, off, idx = _genus_one_spheres([26.0, 32.0, 38.0])
    r = oracle.rpd(w.verts, w.tets, sph, off, idx, euler=True)
    rpc_cc, rpf_cc = oracle.topology(r, w.tets, 3)
    rpc_eu, _ = oracle.euler_sums(r, 3, off, idx)
    assert rpc_cc == [1, 2, 1] and rpc_eu == [1, 2, 1]
    assert rpf_cc == {(0, 1): 2, (1, 0): 2, (1, 2): 2, (2, 1): 2}


def test_cc_single_sphere():
    w = W.make_shape_workload("one", 700, 1, seed=2, cache=False)
    r = oracle.rpd_workload(w, euler=True)
    assert oracle.topology(r, w.tets, 1) == ([1], {})


@pytest.mark.parametrize("make", [lambda: W.make_c1(0), lambda: W.make_c1(3),
                                  lambda: W.random_tiny(0, n_spheres=14, grid=2),
                                  lambda: W.random_tiny(2, n_spheres=14, grid=2)])
def test_cc_equals_explicit_extraction(make):
    """The CC numbers from the pieces' facet / edge flags equal the components of the
    explicitly extracted complexes (pieces glued by shared exact 2-faces, RPF facets by shared
    exact edges)."""
    w = make()
    r = oracle.rpd_workload(w, euler=True)
    rpc_cc, rpf_cc = oracle.topology(r, w.tets, w.N)
    for i in range(w.N):
        e_rpc, e_rpf, generic = X.explicit_cc(w.verts, w.tets, w.spheres, w.nbr_off,
                                              w.nbr_idx, i)
        assert generic
        assert rpc_cc[i] == e_rpc, i
        assert {j: v for (a, j), v in rpf_cc.items() if a == i} == e_rpf, i


# ----------------------------------------------------------------------------- medial mesh
# the dual medial mesh


def test_medial_mesh_three_spheres_one_triangle():
    """PAPER.md:353-357 (Fig. 2): the RPD of three spheres -- three cells meeting along one
    restricted power edge inside the solid -- is dual to one triangle with its three edges."""
    verts, tets = W.kuhn_grid_mesh((2, 2, 2), 512, (0, 0, 0), morton=False)
    sph = np.array([[0.25, 0.25, 0.5, 0.0], [0.75, 0.3125, 0.5, 0.0], [0.4375, 0.75, 0.5, 0.0]])
    off = np.array([0, 2, 4, 6], np.int32)
    idx = np.array([1, 2, 0, 2, 0, 1], np.int32)
    r = oracle.rpd(verts, tets, sph, off, idx, euler=True)
    edges, faces = oracle.medial_mesh(r)
    assert edges == [(0, 1), (0, 2), (1, 2)] and faces == [(0, 1, 2)]
    rpc_cc, rpf_cc = oracle.topology(r, tets, 3)
    assert rpc_cc == [1, 1, 1] and set(rpf_cc.values()) == {1}


@pytest.mark.parametrize("make", [lambda: W.make_c1(0), lambda: W.make_c1(3),
                                  lambda: W.random_tiny(0, n_spheres=14, grid=2),
                                  lambda: W.random_tiny(2, n_spheres=14, grid=2)])
def test_medial_faces_equal_explicit_extraction(make):
    """Triangles of the medial mesh = the restricted power edges found in the exact pieces
    (edges of positive length on two radical planes), on generic inputs."""
    w = make()
    r = oracle.rpd_workload(w, euler=True)
    _, faces = oracle.medial_mesh(r)
    e_faces, generic = X.explicit_medial_faces(w.verts, w.tets, w.spheres, w.nbr_off, w.nbr_idx)
    assert generic and faces == e_faces
    # every triangle's three edges are medial edges
    edges = set(oracle.medial_mesh(r)[0])
    for (i, j, k) in faces:
        assert {(i, j), (i, k), (j, k)} <= edges


# ----------------------------------------------------------------------------- envelope distance
# distance of surface samples to the enveloping
# volume of the medial mesh (sphere / cone / slab)

ENV = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "envelope_examples.json")))


@pytest.mark.parametrize("case", ENV["cases"])
def test_envelope_spec_examples(case):
    d = oracle.envelope_one(case["p"], np.array(case["spheres"], float), case["ids"])
    assert max(d, 0.0) == pytest.approx(case["distance"], abs=1e-12)


def _seg_dist(p, a, b):
    d = b - a
    t = np.clip(np.dot(p - a, d) / np.dot(d, d), 0.0, 1.0)
    return np.linalg.norm(p - (a + t * d))


def test_envelope_equal_radii_cone_is_capsule():
    """Equal radii: the cone is a capsule -- value = distance to the segment minus r."""
    rng = np.random.default_rng(0)
    for _ in range(200):
        a, b, p = rng.normal(size=3), rng.normal(size=3), 3 * rng.normal(size=3)
        r = rng.uniform(0.1, 1.0)
        sph = np.array([[*a, r], [*b, r]])
        assert oracle.envelope_one(p, sph, [0, 1]) == pytest.approx(_seg_dist(p, a, b) - r,
                                                                    abs=1e-10)


def test_envelope_slab_vs_dense_sampling():
    """SPEC.md: a random slab at a random p matches the brute-force minimum over densely
    sampled (u, v) (10^4 samples of the triangle) within 1e-4 -- the oracle, being exact up to
    rounding, is at most the sampled minimum and within the sampling error of it."""
    rng = np.random.default_rng(1)
    n = 141
    u, v = np.meshgrid(np.linspace(0, 1, n), np.linspace(0, 1, n))
    keep = u + v <= 1.0
    u, v = u[keep], v[keep]
    for _ in range(60):
        sph = np.c_[rng.normal(size=(3, 3)), rng.uniform(0.0, 0.8, 3)]
        p = 2.5 * rng.normal(size=3)
        c = sph[0, :3] + u[:, None] * (sph[1, :3] - sph[0, :3]) + v[:, None] * (sph[2, :3] - sph[0, :3])
        r = sph[0, 3] + u * (sph[1, 3] - sph[0, 3]) + v * (sph[2, 3] - sph[0, 3])
        brute = np.min(np.linalg.norm(p - c, axis=1) - r)
        got = oracle.envelope_one(p, sph, [0, 1, 2])
        assert got <= brute + 1e-12 and brute - got < 1e-3


def test_envelope_min_over_primitives():
    """The per-sample value is the minimum over every sphere, cone and slab; a slab is never
    above its cones, a cone never above its spheres (they belong to its family)."""
    rng = np.random.default_rng(2)
    sph = np.c_[rng.uniform(0, 10, (6, 3)), rng.uniform(0, 1.5, 6)]
    edges = np.array([[0, 1], [1, 2], [0, 2], [3, 4]], np.int32)
    faces = np.array([[0, 1, 2]], np.int32)
    smp = rng.uniform(-2, 12, (40, 3))
    g, prim = oracle.envelope(smp, sph, edges, faces)
    for s in range(len(smp)):
        vals = [oracle.envelope_one(smp[s], sph, [i]) for i in range(6)] + \
               [oracle.envelope_one(smp[s], sph, list(e)) for e in edges] + \
               [oracle.envelope_one(smp[s], sph, list(f)) for f in faces]
        assert g[s] == min(vals) and vals[prim[s]] == g[s]
        assert vals[10] <= min(vals[6], vals[7], vals[8]) + 1e-12
        assert vals[6] <= min(vals[0], vals[1]) + 1e-12
