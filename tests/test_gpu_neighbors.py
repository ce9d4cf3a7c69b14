"""Sphere neighbours on the GPU through the C ABI
(-m gpu).  Several neighbour lists are correct (any superset of the box neighbours gives the
same RPD), so the tests check what is unique and that the rest is valid:
  * every GPU row contains the oracle's box-neighbour row (``oracle.box_neighbours``), and
    every extra entry is a real sphere != i with a distinct centre (rows ascending, no dups);
  * the pieces computed with the GPU lists equal the oracle's pieces with the regular-
    triangulation lists (ids, facemasks, incidences bit-exact; vol / m1 at 1e-9), and at C2 /
    C3 size the GPU pieces with either list set are equal;
  * edge cases: N = 0, N = 1, same-centre hiding, a cell covering the box, bad inputs."""
import numpy as np
import pytest

import oracle
import rpd_workloads as W
from tests.helpers import compare_results

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ctx():
    import paper_2403_18761_b200 as P
    P.build()
    c = P.RPDContext(0, filter_mode="pruned")
    yield c
    c.close()


def rows(off, idx):
    return [idx[off[i]:off[i + 1]].tolist() for i in range(len(off) - 1)]


def check_valid(sp, got):
    off, idx = np.asarray(got["nbr_off"]), np.asarray(got["nbr_idx"])
    assert off[0] == 0 and np.all(np.diff(off) >= 0) and off[-1] == len(idx)
    for i, r in enumerate(rows(off, idx)):
        assert r == sorted(set(r)), i
        for j in r:
            assert 0 <= j < len(sp) and j != i
            assert not np.array_equal(sp[i, :3], sp[j, :3])
    return off, idx


WORKLOADS = [lambda: W.make_shape_workload("nb_smoke", 1200, 100, seed=11, cache=False),
             lambda: W.make_shape_workload("nb_small", 600, 60, seed=4, cache=False),
             lambda: W.make_c1(3), lambda: W.make_c1(1, degenerate=True),
             lambda: W.random_tiny(5, n_spheres=14),
             lambda: W.random_tiny(2, n_spheres=20, coarse=True)]


@pytest.mark.parametrize("k", range(len(WORKLOADS)))
def test_neighbors_superset_and_pieces(ctx, k):
    import paper_2403_18761_b200 as P
    w = WORKLOADS[k]()
    box = W.mesh_box(w.verts)
    got = ctx.neighbors(w.spheres, box)
    off, idx = check_valid(w.spheres, got)
    roff, ridx = oracle.box_neighbours(w.spheres, box)
    g, r = rows(off, idx), rows(roff, ridx)
    for i in range(w.N):
        assert set(r[i]) <= set(g[i]), (i, sorted(set(r[i]) - set(g[i])))
    # not much looser than the definition (the bound polytope uses 16 planes)
    assert len(idx) <= 3 * max(len(ridx), 1) + 8
    a = P.rpd_full(w.verts, w.tets, w.spheres, off, idx, ctx=ctx)
    b = oracle.rpd_workload(w)
    assert compare_results(a, b, w.verts, w.tets, rel=1e-9, check_cands=False) == []


@pytest.mark.parametrize("name", ["C2", "C3", "C4-final", "C5"])
def test_neighbors_full_size_same_pieces(ctx, name):
    """Certifies the generator's Qhull neighbour lists at full size: the
    GPU lists are a certified superset of the box neighbours (R30), and every piece computed
    with them equals the piece computed with the Qhull lists -- so no missing Qhull neighbour
    changes any piece.  C4-final: the sphere set after the 10 partial-update batches."""
    import copy
    import paper_2403_18761_b200 as P
    if name == "C4-final":
        w = copy.copy(W.make_config("C4"))
        w.spheres, w.nbr_off, w.nbr_idx = w.batches[-1]
    else:
        w = W.make_config(name)
    got = ctx.neighbors(w.spheres, W.mesh_box(w.verts))
    off, idx = np.asarray(got["nbr_off"]), np.asarray(got["nbr_idx"])
    assert off[-1] == len(idx) and np.all(np.diff(off) >= 0)
    a = P.rpd_full(w.verts, w.tets, w.spheres, off, idx, ctx=ctx)
    b = P.rpd_full(w.verts, w.tets, w.spheres, w.nbr_off, w.nbr_idx, ctx=ctx)
    assert compare_results(a, b, w.verts, w.tets, rel=1e-9, check_cands=False) == []
    # the GPU rows contain every regular-triangulation neighbour that carries an incidence
    g = rows(off, idx)
    ps = np.asarray(b["piece_sphere"])
    for p in range(0, len(ps), max(1, len(ps) // 5000)):
        inc = b["inc_sphere"][b["inc_off"][p]:b["inc_off"][p + 1]]
        assert set(inc.tolist()) <= set(g[int(ps[p])])


def test_neighbors_edge_cases(ctx):
    import paper_2403_18761_b200 as P
    box = (0, 0, 0, 32, 32, 32)
    got = ctx.neighbors(np.zeros((0, 4)), box)
    assert list(got["nbr_off"]) == [0] and len(got["nbr_idx"]) == 0
    got = ctx.neighbors(np.array([[5.0, 5, 5, 1]]), box)
    assert list(got["nbr_off"]) == [0, 0]
    # same centre: the larger radius hides the smaller one; equal spheres: the smaller id wins
    sp = np.array([[8, 8, 8, 2], [8, 8, 8, 3], [20, 20, 20, 1], [20, 20, 20, 1.0]])
    got = ctx.neighbors(sp, box)
    r = rows(got["nbr_off"], got["nbr_idx"])
    assert r[0] == [] and r[3] == [] and got["n_hidden"] == 2
    assert 2 in r[1] and 1 in r[2]
    # a cell covering the whole box: one redundant entry so that R4 does not apply
    sp = np.array([[16, 16, 16, 30.0], [60, 60, 60, 0]])
    got = ctx.neighbors(sp, box)
    r = rows(got["nbr_off"], got["nbr_idx"])
    assert r == [[1], []]
    v, t = W.box_6tets((0, 0, 0), (32, 32, 32))
    a = P.rpd_full(v, t, sp, got["nbr_off"], got["nbr_idx"], ctx=ctx)
    assert list(a["piece_sphere"]) == [0] * 6
    # dominated sphere (oracle closed form in test_neighbors_oracle)
    sp = np.array([[16, 16, 16, 6], [17, 16, 16, 1], [28, 16, 16, 1]], dtype=np.float64)
    got = ctx.neighbors(sp, box)
    r = rows(got["nbr_off"], got["nbr_idx"])
    assert r[1] == [] and 2 in r[0] and 0 in r[2]


def test_neighbors_invalid(ctx):
    import paper_2403_18761_b200 as P
    sp = np.array([[1.0, 2, 3, 1], [4, 5, 6, 1]])
    for bad_box in [(0, 0, 0, -1, 1, 1), (0, 0, np.nan, 1, 1, 1)]:
        with pytest.raises(P.RPDError, match="EINVAL"):
            ctx.neighbors(sp, bad_box)
    for k, v in [(3, -1.0), (0, np.nan), (1, np.inf)]:
        s = sp.copy()
        s[1, k] = v
        with pytest.raises(P.RPDError, match="EINVAL"):
            ctx.neighbors(s, (0, 0, 0, 8, 8, 8))
    # the ctx stays usable
    got = ctx.neighbors(sp, (0, 0, 0, 8, 8, 8))
    assert rows(got["nbr_off"], got["nbr_idx"]) == [[1], [0]]
    import torch
    d = torch.tensor(sp, device="cuda")
    got = ctx.neighbors(d, (0, 0, 0, 8, 8, 8), device=True)
    assert got["nbr_idx"].is_cuda and got["nbr_idx"].tolist() == [1, 0]


def test_neighbors_partial_update(ctx):
    """C4-style: lists recomputed on the GPU after an insertion batch feed rpd_update_partial;
    the result equals a full recompute with the regular-triangulation lists."""
    import paper_2403_18761_b200 as P
    w = W.make_shape_workload("nb_part", 3000, 150, seed=6, n_batches=1, batch_m=20, cache=False)
    box = W.mesh_box(w.verts)
    g0 = ctx.neighbors(w.spheres, box)
    ctx.relations(w.verts, w.tets, w.spheres, g0["nbr_off"], g0["nbr_idx"])
    ctx.clip()
    sp1, off1, idx1 = w.batches[0]
    g1 = ctx.neighbors(sp1, box)
    n_old = w.N
    ctx.update_partial(sp1, g1["nbr_off"], g1["nbr_idx"], np.arange(n_old, len(sp1), dtype=np.int32))
    got = ctx.download_pieces()
    ref = P.rpd_full(w.verts, w.tets, sp1, off1, idx1, ctx=None, filter_mode="pruned")
    assert compare_results(got, ref, w.verts, w.tets, rel=1e-9, check_cands=False) == []


def _rows_superset(ctx_lists, sp, box):
    off, idx = check_valid(sp, ctx_lists)
    roff, ridx = oracle.box_neighbours(sp, box)
    g, r = rows(off, idx), rows(roff, ridx)
    for i in range(len(sp)):
        assert set(r[i]) <= set(g[i]), (i, sorted(set(r[i]) - set(g[i])))
    return off, idx


@pytest.mark.parametrize("m,clusters", [(1, 1), (5, 2), (20, 4)])
def test_neighbors_incremental_superset_and_pieces(ctx, m, clusters):
    """rpd_neighbors_update (reading R34): after each insertion batch the new spheres' rows are
    computed and the old rows extended by the new spheres whose plane reaches their cell's
    ball (or emptied when hidden); every row is still a certified superset of the oracle's box
    neighbours, and the pieces with the incremental lists equal the oracle's (same lists) and
    the GPU's with fully recomputed lists."""
    import paper_2403_18761_b200 as P
    w = W.make_shape_workload(f"nb_inc{m}", 1200, 100, seed=11 + m, n_batches=3, batch_m=m,
                              clusters=clusters, cache=False)
    box = W.mesh_box(w.verts)
    ctx.neighbors(w.spheres, box)
    for (sp, off1, idx1) in w.batches:
        got = ctx.neighbors_update(sp, m, box)
        assert 0 < got["n_rows"] < len(sp)
        off, idx = _rows_superset(got, sp, box)
        off, idx = off.copy(), idx.copy()
        a = P.rpd_full(w.verts, w.tets, sp, off, idx, ctx=ctx)
        # the oracle with the same lists, and the GPU with fully recomputed lists
        b = oracle.rpd(w.verts, w.tets, sp, off, idx)
        assert compare_results(a, b, w.verts, w.tets, rel=1e-9, check_cands=False) == []
        full = ctx.neighbors(sp, box)
        c = P.rpd_full(w.verts, w.tets, sp, full["nbr_off"], full["nbr_idx"], ctx=ctx)
        assert compare_results(a, c, w.verts, w.tets, rel=1e-9, check_cands=False) == []
        q = oracle.rpd(w.verts, w.tets, sp, off1, idx1)  # (the generator's Qhull lists)
        print("qhull lists give the same pieces:",
              compare_results(a, q, w.verts, w.tets, rel=1e-9, check_cands=False) == [])
        # (the full recompute replaced the ctx's lists: the chain continues from them)


def test_neighbors_incremental_c4(ctx):
    """The C4 chain at full size (10 batches of 500 spheres on the C3 set): incremental lists
    after every batch, then the final RPD with them equals the RPD with the Qhull lists."""
    import paper_2403_18761_b200 as P
    w = W.make_config("C4")
    box = W.mesh_box(w.verts)
    ctx.neighbors(w.spheres, box)
    n_rows = []
    for (sp, off1, idx1) in w.batches:
        got = ctx.neighbors_update(sp, 500, box)
        n_rows.append(got["n_rows"])
    sp, off1, idx1 = w.batches[-1]
    off, idx = np.asarray(got["nbr_off"]), np.asarray(got["nbr_idx"])
    assert off[-1] == len(idx) and np.all(np.diff(off) >= 0)
    assert max(n_rows) < len(sp) // 2
    a = P.rpd_full(w.verts, w.tets, sp, off, idx, ctx=ctx)
    b = P.rpd_full(w.verts, w.tets, sp, off1, idx1, ctx=ctx)
    assert compare_results(a, b, w.verts, w.tets, rel=1e-9, check_cands=False) == []


def test_neighbors_incremental_edge_cases(ctx):
    import paper_2403_18761_b200 as P
    box = (0, 0, 0, 32, 32, 32)
    sp = np.array([[8, 8, 8, 2], [20, 20, 20, 1], [8, 20, 8, 1.5]], dtype=np.float64)
    ctx.neighbors(sp, box)
    # a new sphere with an old one's centre and a larger radius hides it: its row empties
    sp2 = np.concatenate([sp, [[8, 8, 8, 3.0]]])
    got = ctx.neighbors_update(sp2, 1, box)
    inc = rows(got["nbr_off"], got["nbr_idx"])
    full = ctx.neighbors(sp2, box)
    assert inc[0] == []
    for r_inc, r_full in zip(inc, rows(full["nbr_off"], full["nbr_idx"])):
        assert set(r_full) <= set(r_inc) and r_inc == sorted(set(r_inc))
    # M = 0: the same lists
    same = ctx.neighbors_update(sp2, 0, box)
    assert rows(same["nbr_off"], same["nbr_idx"]) == rows(full["nbr_off"], full["nbr_idx"])
    # state errors: another box, or lists of another sphere count
    with pytest.raises(P.RPDError, match="ESTATE"):
        ctx.neighbors_update(np.concatenate([sp2, [[1, 1, 1, 1.0]]]), 1, (0, 0, 0, 33, 32, 32))
    with pytest.raises(P.RPDError, match="ESTATE"):
        ctx.neighbors_update(np.concatenate([sp2, [[1, 1, 1, 1.0]]]), 2, box)
    # an old sphere that moved
    bad = np.concatenate([sp2, [[1, 1, 1, 1.0]]])
    bad[1, 0] += 1
    with pytest.raises(P.RPDError, match="EINVAL"):
        ctx.neighbors_update(bad, 1, box)
    with pytest.raises(P.RPDError, match="ESTATE"):  # (the rejected call left no lists)
        ctx.neighbors_update(bad, 1, box)


def _lists(ctx, sp, box, mode, monkeypatch, m=None):
    monkeypatch.setenv("RPD_NB_HEAVY", str(mode))
    got = ctx.neighbors(sp, box) if m is None else ctx.neighbors_update(sp, m, box)
    return np.array(got["nbr_off"]), np.array(got["nbr_idx"]), got


@pytest.mark.parametrize("name", ["nb_smoke", "nb_small", "tiny", "C2", "C3"])
def test_neighbors_block_rows_equal_warp_rows(ctx, name, monkeypatch):
    """Heavy rows run on a whole block (k_nb_heavy): the same rows as the warp computes, entry
    for entry -- every row on a warp (RPD_NB_HEAVY=0), every row on a block (-1) and the
    default hand-off give identical CSRs."""
    if name == "nb_smoke":
        w = W.make_shape_workload("nb_smoke", 1200, 100, seed=11, cache=False)
    elif name == "nb_small":
        w = W.make_shape_workload("nb_small", 600, 60, seed=4, cache=False)
    elif name == "tiny":
        w = W.random_tiny(2, n_spheres=20, coarse=True)
    else:
        w = W.make_config(name)
    box = W.mesh_box(w.verts)
    o0, i0, g0 = _lists(ctx, w.spheres, box, 0, monkeypatch)
    o1, i1, g1 = _lists(ctx, w.spheres, box, -1, monkeypatch)
    o2, i2, g2 = _lists(ctx, w.spheres, box, 2048, monkeypatch)
    assert g0["n_rows_block"] == 0 and g1["n_rows_block"] > 0
    if name == "C3":
        assert 0 < g2["n_rows_block"] < w.N
    assert np.array_equal(o0, o1) and np.array_equal(i0, i1)
    assert np.array_equal(o0, o2) and np.array_equal(i0, i2)
    assert g0["n_vertex_overflow"] == g1["n_vertex_overflow"] == g2["n_vertex_overflow"]


def test_neighbors_block_rows_incremental(ctx, monkeypatch):
    """The incremental update's new rows on blocks equal them on warps (C4 chain, 3 batches)."""
    w = W.make_config("C4")
    box = W.mesh_box(w.verts)
    res = {}
    for mode in (0, -1):
        monkeypatch.setenv("RPD_NB_HEAVY", str(mode))
        ctx.neighbors(w.spheres, box)
        res[mode] = [_lists(ctx, sp, box, mode, monkeypatch, m=500)[:2]
                     for (sp, _, _) in w.batches[:3]]
    for (a, b), (c, d) in zip(res[0], res[-1]):
        assert np.array_equal(a, c) and np.array_equal(b, d)


def _shell(n=400, seed=0):
    """A big central sphere inside a shell of n small ones (Fibonacci directions): the central
    row lists every shell sphere (longer than the 256-entry pass-1 slab: pass 2)."""
    k = np.arange(n) + 0.5
    phi = np.arccos(1 - 2 * k / n)
    th = np.pi * (1 + 5 ** 0.5) * k
    d = np.stack([np.cos(th) * np.sin(phi), np.sin(th) * np.sin(phi), np.cos(phi)], 1)
    c = np.array([16.0, 16.0, 16.0])
    sp = np.concatenate([[[*c, 6.0]], np.c_[c + 10.0 * d, np.full(n, 0.5)]])
    return np.round(sp * 1024) / 1024, (0, 0, 0, 32, 32, 32)  # (on the oracle's lattice)


def test_neighbors_long_row_block_and_warp(ctx, monkeypatch):
    """A row longer than the pass-1 slab (pass 2 recomputes it on a warp): with every row on a
    block in pass 1 (RPD_NB_HEAVY=-1) the recomputed row has the same length (no
    ERR_NB_RECOMPUTE) and the lists equal the all-warp ones; the long row lists every shell
    sphere and contains the oracle's row."""
    sp, box = _shell()
    o0, i0, g0 = _lists(ctx, sp, box, 0, monkeypatch)
    o1, i1, g1 = _lists(ctx, sp, box, -1, monkeypatch)
    assert g1["n_rows_block"] > 0
    assert np.array_equal(o0, o1) and np.array_equal(i0, i1)
    assert o0[1] - o0[0] > 256
    assert set(range(1, len(sp))) <= set(i0[o0[0]:o0[1]].tolist())
    roff, ridx = oracle.box_neighbours(sp, box)
    assert set(ridx[roff[0]:roff[1]].tolist()) <= set(i0[o0[0]:o0[1]].tolist())


@pytest.mark.parametrize("k", range(len(WORKLOADS)))
def test_neighbors_sequential_clip_and_enumeration(ctx, k, monkeypatch):
    """The cell polytope P_K built by the sequential clip (default) and by the triple
    enumeration (RPD_NB_SEQ=0, DESIGN.md §10 "Sequential clip of P_K"): both rows contain the
    oracle's box-neighbour rows, and both give the oracle's pieces."""
    import paper_2403_18761_b200 as P
    w = WORKLOADS[k]()
    box = W.mesh_box(w.verts)
    roff, ridx = oracle.box_neighbours(w.spheres, box)
    r = rows(roff, ridx)
    b = oracle.rpd_workload(w)
    for seq in ("0", "1"):
        monkeypatch.setenv("RPD_NB_SEQ", seq)
        off, idx = check_valid(w.spheres, ctx.neighbors(w.spheres, box))
        g = rows(off, idx)
        for i in range(w.N):
            assert set(r[i]) <= set(g[i]), (seq, i, sorted(set(r[i]) - set(g[i])))
        a = P.rpd_full(w.verts, w.tets, w.spheres, off, idx, ctx=ctx)
        assert compare_results(a, b, w.verts, w.tets, rel=1e-9, check_cands=False) == []


@pytest.mark.parametrize("name", ["C2", "C3"])
def test_neighbors_sequential_clip_equals_enumeration_full_size(ctx, name, monkeypatch):
    """At C2 / C3 the two P_K constructions give the same lists (the sequential clip solves a
    subset of the enumeration's triples and loses no true vertex; measured identical)."""
    w = W.make_config(name)
    box = W.mesh_box(w.verts)
    res = {}
    for seq in ("0", "1"):
        monkeypatch.setenv("RPD_NB_SEQ", seq)
        got = ctx.neighbors(w.spheres, box)
        res[seq] = (np.array(got["nbr_off"]), np.array(got["nbr_idx"]))
    assert np.array_equal(res["0"][0], res["1"][0]) and np.array_equal(res["0"][1], res["1"][1])
