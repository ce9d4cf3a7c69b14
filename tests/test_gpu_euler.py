"""Fractional Euler characteristics: the clip
kernel's on-the-fly payload sums vs the CPU oracle, exactly (rational numerators), through the
C ABI (-m gpu)."""
from fractions import Fraction

import numpy as np
import pytest

import oracle
import rpd_workloads as W
from tests.helpers import compare_euler, piece_tet, slice_euler, slice_tets

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", params=["all_pairs", "pruned"])
def ctx(request):
    import paper_2403_18761_b200 as P
    P.build()
    c = P.RPDContext(0, filter_mode=request.param)
    yield c
    c.close()


def run_gpu_euler(ctx, w, tets=None, local_ids=None):
    tets_local = w.tets if tets is None else tets
    P = ctx.set_euler(w.tets, len(w.verts), local_ids)
    try:
        ctx.relations(w.verts, tets_local, w.spheres, w.nbr_off, w.nbr_idx)
        ctx.clip()
        out = ctx.download_cands()
        out.update(ctx.download_pieces())
        out.update(ctx.download_euler())
    finally:
        ctx.set_euler(None, 0)
    assert out["n_primes"] == P and out["rpc_acc"].shape == (w.N, 1 + P)
    return out


def check_sums(got, ref, w):
    """Per-sphere RPC and per-CSR-entry RPF sums against the oracle's sums (Fractions): the
    exact integer where the oracle's sum is an integer (flagged exact), else flagged inexact
    with the right value as a double."""
    rpc, rpf = oracle.euler_sums(ref, w.N, w.nbr_off, w.nbr_idx)
    want_rpf = [rpf.get((i, int(w.nbr_idx[e])), Fraction(0)) for i in range(w.N)
                for e in range(w.nbr_off[i], w.nbr_off[i + 1])]
    for name, want in (("rpc", rpc), ("rpf", want_rpf)):
        s, ex, val = got[name + "_sum"], got[name + "_exact"], got[name + "_value"]
        for x, f in enumerate(want):
            if f.denominator == 1:
                assert ex[x] == 1 and int(s[x]) == f, (name, x, f, s[x], ex[x])
            else:
                assert ex[x] == 0 and abs(val[x] - float(f)) < 1e-9, (name, x, f, val[x])


MAKERS = [lambda: W.make_c1(0), lambda: W.make_c1(1, degenerate=True),
          lambda: W.make_c1(6, degenerate=True, big=True),
          lambda: W.random_tiny(0, n_spheres=14, grid=2),
          lambda: W.random_tiny(3, n_spheres=14, grid=2, coarse=True),
          lambda: W.make_shape_workload("E3", 2000, 150, seed=3, cache=False),
          lambda: W.make_shape_workload("E5", 3000, 300, seed=5, radius_mode="high_variance",
                                        cache=False),
          # unstructured: a global common denominator would exceed 2^70
          lambda: W.delaunay_workload(2000, 60, seed=1)]


@pytest.mark.parametrize("make", MAKERS)
def test_euler_parity(ctx, make):
    w = make()
    got = run_gpu_euler(ctx, w)
    ref = oracle.rpd_workload(w, euler=True)
    errs = compare_euler(got, ref)
    assert not errs, errs
    check_sums(got, ref, w)


def test_euler_single_sphere_genus_one(ctx):
    """PAPER.md Fig. 4(a): one sphere covering the genus-1 solid has Euler(RPC) = 0."""
    w = W.make_shape_workload("one", 700, 1, seed=2, cache=False)
    got = run_gpu_euler(ctx, w)
    assert int(got["rpc_sum"][0]) == 0 and len(got["piece_euler"]) == w.T


@pytest.mark.parametrize("make", [lambda: W.make_c1(1, degenerate=True),
                                  lambda: W.make_shape_workload("Wd", 2500, 200, seed=9,
                                                                radius_mode="high_variance",
                                                                cache=False)])
def test_euler_wide_kernel(ctx, make):
    """The 128-vertex instantiation with Euler payloads gives the same values."""
    w = make()
    ctx.set_clip_wide(True)
    try:
        got = run_gpu_euler(ctx, w)
    finally:
        ctx.set_clip_wide(False)
    assert not compare_euler(got, oracle.rpd_workload(w, euler=True))


def test_euler_sharded_local_ids(ctx):
    """Tet shards with global payloads (rpd_set_euler local_ids): each shard's pieces match
    the oracle's, and the per-sphere sums of the shards add up to the whole mesh's."""
    w = W.make_shape_workload("Sh", 3000, 200, seed=6, cache=False)
    ref = oracle.rpd_workload(w, euler=True)
    tot_rpc, tot_rpf = 0, 0
    for rank in range(2):
        ids = W.block_cyclic_shard(w.T, 2, rank, block=256).astype(np.int32)
        got = run_gpu_euler(ctx, w, tets=w.tets[ids], local_ids=ids)
        sub = slice_tets(ref, ids)
        pidx = np.concatenate([np.arange(ref["piece_off"][t], ref["piece_off"][t + 1])
                               for t in ids])
        errs = compare_euler(got, slice_euler(ref, pidx))
        assert not errs, errs
        assert np.array_equal(got["piece_sphere"], sub["piece_sphere"])
        # the shards' accumulator rows add up (integer adds) to the whole mesh's
        tot_rpc = tot_rpc + got["rpc_acc"]
        tot_rpf = tot_rpf + got["rpf_acc"]
    full = run_gpu_euler(ctx, w)
    assert np.array_equal(tot_rpc, full["rpc_acc"]) and np.array_equal(tot_rpf, full["rpf_acc"])


def test_euler_partial_update(ctx):
    """Partial updates carry the Euler data: equal to the oracle's partial update (R11)."""
    w = W.make_shape_workload("S", 2000, 150, seed=3, n_batches=2, batch_m=12, clusters=3,
                              cache=False)
    ctx.set_euler(w.tets, len(w.verts))
    try:
        ctx.relations(w.verts, w.tets, w.spheres, w.nbr_off, w.nbr_idx)
        ctx.clip()
        prev = oracle.rpd_workload(w, euler=True)
        n_old = w.N
        for (sph, off, idx) in w.batches:
            ctx.update_partial(sph, off, idx, np.arange(n_old, len(sph), dtype=np.int32))
            got = ctx.download_pieces()
            got.update(ctx.download_euler())
            part, dirty = oracle.partial_update(prev, w.verts, w.tets, sph, off, idx, n_old,
                                                euler=True)
            assert len(dirty) == ctx.n_dirty
            errs = compare_euler(got, part)
            assert not errs, errs
            import copy
            w2 = copy.copy(w)
            w2.spheres, w2.nbr_off, w2.nbr_idx = sph, off, idx
            check_sums(got, part, w2)
            prev, n_old = part, len(sph)
    finally:
        ctx.set_euler(None, 0)


def test_euler_errors(ctx):
    import paper_2403_18761_b200 as P
    w = W.make_c1(0)
    with pytest.raises(P.RPDError) as e:   # V beyond the face-key range
        ctx.set_euler(w.tets, 1 << 21)
    assert e.value.status == -1
    ctx.relations(w.verts, w.tets, w.spheres, w.nbr_off, w.nbr_idx)
    ctx.clip()
    with pytest.raises(P.RPDError) as e:   # no Euler data for these pieces
        ctx.download_euler()
    assert e.value.status == -5
    ctx.set_euler(w.tets[:3], len(w.verts))  # payloads for 3 tets, ctx holds 6
    try:
        with pytest.raises(P.RPDError) as e:
            ctx.clip()
        assert e.value.status == -1
    finally:
        ctx.set_euler(None, 0)


def test_euler_c3_sampled(ctx):
    """BASELINE.json configs[2] at full size: sampled pieces vs the oracle, every RPC / RPF
    sum an integer (the fractional payloads of shared elements add up)."""
    w = W.make_config("C3")
    got = run_gpu_euler(ctx, w)
    rng = np.random.default_rng(3)
    ids = np.sort(rng.choice(w.T, 40, replace=False)).astype(np.int32)
    ref = oracle.rpd_workload(w, tet_ids=ids, euler=True)
    pidx = np.concatenate([np.arange(got["piece_off"][t], got["piece_off"][t + 1]) for t in ids])
    errs = compare_euler(slice_euler(got, pidx), ref)
    assert not errs, errs
    assert np.all(got["rpc_exact"] == 1) and np.all(got["rpf_exact"] == 1)
    chi = got["rpc_sum"]
    assert np.sum(chi == 1) > 0.5 * np.sum(chi != 0)


# ----------------------------------------------------------------------------- CC numbers
# SURVEY.md §8(f) NEXT-2


def run_gpu_topology(ctx, w):
    ctx.set_euler(w.tets, len(w.verts))
    try:
        ctx.relations(w.verts, w.tets, w.spheres, w.nbr_off, w.nbr_idx)
        ctx.clip()
        out = ctx.download_pieces()
        out.update(ctx.download_euler())
        out.update(ctx.download_topology())
    finally:
        ctx.set_euler(None, 0)
    return out


def check_topology(got, ref, w):
    assert np.array_equal(got["piece_sosfm"], ref["piece_sosfm"])
    assert np.array_equal(got["rpf_fm"], ref["rpf_fm"])
    assert np.array_equal(got["rpf_adj"].astype(np.uint64), ref["rpf_adj"])
    rpc_cc, rpf_cc = oracle.topology(ref, w.tets, w.N)
    assert got["rpc_cc"].tolist() == rpc_cc
    for i in range(w.N):
        for e in range(w.nbr_off[i], w.nbr_off[i + 1]):
            assert got["rpf_cc"][e] == rpf_cc.get((i, int(w.nbr_idx[e])), 0)
    # component labels: one root per component, labels are roots of the same sphere's pieces
    roots = got["piece_comp"] == np.arange(len(got["piece_comp"]))
    assert roots.sum() == sum(rpc_cc)
    assert np.array_equal(got["piece_sphere"][got["piece_comp"]], got["piece_sphere"])


@pytest.mark.parametrize("make", MAKERS)
def test_topology_parity(ctx, make):
    w = make()
    got = run_gpu_topology(ctx, w)
    check_topology(got, oracle.rpd_workload(w, euler=True), w)


@pytest.mark.parametrize("xs,rpc,rpf", [([20.0, 44.0], [1, 1], 2),
                                        ([26.0, 32.0, 38.0], [1, 2, 1], 2)])
def test_topology_paper_figures(ctx, xs, rpc, rpf):
    """PAPER.md Fig. 4(b) (torus, two spheres: RPF CC = 2) and Fig. 6(a) (the middle sphere's
    RPC cut by the hole: CC = 2) on the genus-1 box with a hole."""
    import copy
    w = copy.copy(W.make_shape_workload("one", 700, 1, seed=2, cache=False))
    n = len(xs)
    w.spheres = np.array([[x, 26.0, 20.0, 1.0] for x in xs])
    idx, off = [], [0]
    for a in range(n):
        idx += [b for b in (a - 1, a + 1) if 0 <= b < n]
        off.append(len(idx))
    w.nbr_off, w.nbr_idx = np.array(off, np.int32), np.array(idx, np.int32)
    got = run_gpu_topology(ctx, w)
    assert got["rpc_cc"].tolist() == rpc
    assert np.all(got["rpf_cc"] == rpf)
    assert got["rpc_sum"].tolist() == rpc  # contractible components


def test_topology_after_partial_update(ctx):
    w = W.make_shape_workload("S", 2000, 150, seed=3, n_batches=2, batch_m=12, clusters=3,
                              cache=False)
    ctx.set_euler(w.tets, len(w.verts))
    try:
        ctx.relations(w.verts, w.tets, w.spheres, w.nbr_off, w.nbr_idx)
        ctx.clip()
        prev = oracle.rpd_workload(w, euler=True)
        n_old = w.N
        import copy
        for (sph, off, idx) in w.batches:
            ctx.update_partial(sph, off, idx, np.arange(n_old, len(sph), dtype=np.int32))
            got = ctx.download_pieces()
            got.update(ctx.download_topology())
            part, _ = oracle.partial_update(prev, w.verts, w.tets, sph, off, idx, n_old,
                                            euler=True)
            w2 = copy.copy(w)
            w2.spheres, w2.nbr_off, w2.nbr_idx = sph, off, idx
            check_topology(got, part, w2)
            prev, n_old = part, len(sph)
    finally:
        ctx.set_euler(None, 0)


def test_topology_needs_whole_mesh(ctx):
    import paper_2403_18761_b200 as P
    w = W.make_c1(0)
    ids = np.arange(3, dtype=np.int32)
    ctx.set_euler(w.tets, len(w.verts), ids)
    try:
        ctx.relations(w.verts, w.tets[ids], w.spheres, w.nbr_off, w.nbr_idx)
        ctx.clip()
        with pytest.raises(P.RPDError) as e:
            ctx.download_topology()
        assert e.value.status == -5
    finally:
        ctx.set_euler(None, 0)


def test_topology_c3(ctx):
    """At full C3 size: every sphere with pieces has >= 1 component, labels consistent, and
    most cells are connected (CC = 1)."""
    w = W.make_config("C3")
    got = run_gpu_topology(ctx, w)
    has = np.bincount(got["piece_sphere"], minlength=w.N) > 0
    assert np.all((got["rpc_cc"] > 0) == has)
    roots = got["piece_comp"] == np.arange(len(got["piece_comp"]))
    assert roots.sum() == got["rpc_cc"].sum()
    assert np.mean(got["rpc_cc"][has] == 1) > 0.9



# ----------------------------------------------------------------------------- medial mesh
# the dual medial mesh


def gpu_medial(ctx, w, tets=None, local_ids=None):
    ctx.set_euler(w.tets, len(w.verts), local_ids)
    try:
        ctx.relations(w.verts, w.tets if tets is None else tets, w.spheres, w.nbr_off, w.nbr_idx)
        ctx.clip()
        return ctx.medial_mesh()
    finally:
        ctx.set_euler(None, 0)


@pytest.mark.parametrize("make", MAKERS)
def test_medial_mesh_parity(ctx, make):
    w = make()
    got = gpu_medial(ctx, w)
    edges, faces = oracle.medial_mesh(oracle.rpd_workload(w, euler=True))
    assert [tuple(e) for e in got["edges"].tolist()] == edges
    assert [tuple(f) for f in got["faces"].tolist()] == faces


def test_medial_mesh_three_spheres(ctx):
    """three cells meeting along one RPE -> one triangle, three edges."""
    import copy
    verts, tets = W.kuhn_grid_mesh((2, 2, 2), 512, (0, 0, 0), morton=False)
    w = copy.copy(W.make_c1(0))
    w.verts, w.tets = verts, tets
    w.spheres = np.array([[0.25, 0.25, 0.5, 0.0], [0.75, 0.3125, 0.5, 0.0],
                          [0.4375, 0.75, 0.5, 0.0]])
    w.nbr_off = np.array([0, 2, 4, 6], np.int32)
    w.nbr_idx = np.array([1, 2, 0, 2, 0, 1], np.int32)
    got = gpu_medial(ctx, w)
    assert got["edges"].tolist() == [[0, 1], [0, 2], [1, 2]]
    assert got["faces"].tolist() == [[0, 1, 2]]


def test_medial_mesh_shards_union(ctx):
    """Tet shards: the union of the shards' medial meshes is the whole mesh's."""
    w = W.make_shape_workload("Sh", 3000, 200, seed=6, cache=False)
    full = gpu_medial(ctx, w)
    E, F = set(), set()
    for rank in range(2):
        ids = W.block_cyclic_shard(w.T, 2, rank, block=256).astype(np.int32)
        part = gpu_medial(ctx, w, tets=w.tets[ids], local_ids=ids)
        E |= {tuple(e) for e in part["edges"].tolist()}
        F |= {tuple(f) for f in part["faces"].tolist()}
    assert sorted(E) == [tuple(e) for e in full["edges"].tolist()]
    assert sorted(F) == [tuple(f) for f in full["faces"].tolist()]


def test_medial_mesh_c3(ctx):
    """Full C3 size: every triangle's edges are medial edges; the mesh is non-trivial."""
    w = W.make_config("C3")
    got = gpu_medial(ctx, w)
    E = {tuple(e) for e in got["edges"].tolist()}
    assert len(got["faces"]) > 1000
    for (i, j, k) in got["faces"][:: max(1, len(got["faces"]) // 2000)].tolist():
        assert (i, j) in E and (i, k) in E and (j, k) in E


def test_euler_topology_c4_partial_equals_full(ctx):
    """BASELINE.json configs[3] at full size with the Euler / topology data on: after the 10
    partial updates (M = 500 each) the per-sphere Euler sums, CC numbers and the medial mesh
    equal those of a full recompute on the final sphere set (R11/R12: pieces of dirty tets are
    recomputed, clean ones kept)."""
    w = W.make_config("C4")
    ctx.set_euler(w.tets, len(w.verts))
    try:
        ctx.relations(w.verts, w.tets, w.spheres, w.nbr_off, w.nbr_idx)
        ctx.clip()
        n_old = w.N
        for (sph, off, idx) in w.batches:
            ctx.update_partial(sph, off, idx, np.arange(n_old, len(sph), dtype=np.int32))
            n_old = len(sph)
        zero_hits = ctx.stats()["zero_hits"]
        part = ctx.download_euler()
        part.update(ctx.download_topology())
        part_mm = ctx.medial_mesh()
        part_rpe = ctx.rpe()
        sph, off, idx = w.batches[-1]
        ctx.relations(w.verts, w.tets, sph, off, idx)
        ctx.clip()
        full = ctx.download_euler()
        full.update(ctx.download_topology())
        full_mm = ctx.medial_mesh()
        full_rpe = ctx.rpe()
    finally:
        ctx.set_euler(None, 0)
    for k in ("rpc_sum", "rpf_sum", "rpc_cc", "rpf_cc"):
        assert np.array_equal(part[k], full[k]), (k, zero_hits)
    for k in ("tri", "tri_euler", "tri_cc"):
        assert np.array_equal(part_rpe[k], full_rpe[k]), k
    assert np.array_equal(part_mm["edges"], full_mm["edges"])
    assert np.array_equal(part_mm["faces"], full_mm["faces"])


# ---------------------------------------------------------------- restricted power edges


def run_gpu_rpe(ctx, w, tets=None, local_ids=None):
    ctx.set_euler(w.tets, len(w.verts), local_ids)
    try:
        ctx.relations(w.verts, w.tets if tets is None else tets, w.spheres, w.nbr_off,
                      w.nbr_idx)
        ctx.clip()
        out = ctx.rpe()
    finally:
        ctx.set_euler(None, 0)
    return out


def check_rpe(got, ref, w):
    """Per-piece RPE lists exactly (ids, endpoint faces, Euler as exact rationals) and the
    per-(i, j, k) Euler sums and CC numbers against the oracle."""
    for k in ("rpe_off", "rpe_j", "rpe_k", "rpe_fm"):
        assert np.array_equal(got[k], ref[k]), k
    # per-piece values over the piece's denominator (the same L_t on both sides: both are the
    # lcm of the tet's sharing counts)
    assert np.array_equal(got["rpe_euler"], ref["rpe_euler"])
    sums = oracle.rpe_sums(ref)
    keys = sorted(sums)
    assert [tuple(x) for x in got["tri"].tolist()] == keys
    assert [Fraction(int(v), got["euler_denom"]) for v in got["tri_euler"]] == \
        [sums[k] for k in keys]
    if got["tri_cc"] is not None:
        cc = oracle.rpe_topology(ref, w.tets)
        assert got["tri_cc"].tolist() == [cc[k] for k in keys]


@pytest.mark.parametrize("make", MAKERS)
def test_rpe_parity(ctx, make):
    """NEXT-1 / PAPER.md:439, 497, 506: the restricted power edges of every piece, their
    fractional Euler characteristics and the per-(i, j, k) Euler sums and CC numbers equal the
    oracle's (pinned by explicit exact extraction in test_oracle_pins)."""
    w = make()
    got = run_gpu_rpe(ctx, w)
    check_rpe(got, oracle.rpd_workload(w, euler=True), w)


def test_rpe_through_the_hole(ctx):
    """The RPE of three spheres whose common line crosses the genus-1 solid twice: Euler 2 and
    CC 2 seen from each sphere (tests/test_oracle_pins.py derives it by hand)."""
    import copy
    w = copy.copy(W.make_shape_workload("one", 700, 1, seed=2, cache=False))
    w.spheres = np.array([[32.0, 32.0, 20.0, 1.0], [32.0, 20.0, 20.0, 1.0],
                          [32.0, 26.0, 26.0, 1.0]])
    w.nbr_off = np.array([0, 2, 4, 6], np.int32)
    w.nbr_idx = np.array([1, 2, 0, 2, 0, 1], np.int32)
    got = run_gpu_rpe(ctx, w)
    assert got["tri"].tolist() == [[0, 1, 2], [1, 0, 2], [2, 0, 1]]
    assert [Fraction(int(v), got["euler_denom"]) for v in got["tri_euler"]] == [2, 2, 2]
    assert got["tri_cc"].tolist() == [2, 2, 2]


def test_rpe_c3_sampled(ctx):
    """At C3 size (BASELINE.json configs[2]): every per-(i, j, k) RPE Euler sum is an integer
    and RPE(m_i, m_j, m_k) has the same Euler and CC seen from each of its spheres; the pieces
    of sampled tets carry the oracle's RPE lists."""
    w = W.make_config("C3")
    ctx.set_euler(w.tets, len(w.verts))
    try:
        ctx.relations(w.verts, w.tets, w.spheres, w.nbr_off, w.nbr_idx)
        ctx.clip()
        got = ctx.rpe()
        pcs = ctx.download_pieces()
        zh = ctx.stats()["zero_hits"]
    finally:
        ctx.set_euler(None, 0)
    L = got["euler_denom"]  # 2: RPE values are halves
    assert len(got["tri"]) > 1000
    assert np.all(got["tri_euler"] % L == 0)
    if zh == 0:
        val = {tuple(k): (int(e), int(c)) for k, e, c in zip(got["tri"].tolist(),
                                                            got["tri_euler"], got["tri_cc"])}
        for (i, j, k), v in val.items():
            a, b, c = sorted((i, j, k))
            assert val.get((a, b, c)) == v and val.get((b, a, c)) == v and val.get((c, a, b)) == v
    rng = np.random.default_rng(2)
    ids = np.sort(rng.choice(w.T, 32, replace=False)).astype(np.int32)
    ref = oracle.rpd_workload(w, tet_ids=ids, euler=True)
    po, eo = pcs["piece_off"], got["rpe_off"]
    for a, t in enumerate(ids):
        for q, qr in zip(range(po[t], po[t + 1]), range(ref["piece_off"][a], ref["piece_off"][a + 1])):
            g = list(zip(got["rpe_j"][eo[q]:eo[q + 1]].tolist(), got["rpe_k"][eo[q]:eo[q + 1]].tolist(),
                         got["rpe_fm"][eo[q]:eo[q + 1]].tolist()))
            ro = ref["rpe_off"]
            r = list(zip(ref["rpe_j"][ro[qr]:ro[qr + 1]].tolist(), ref["rpe_k"][ro[qr]:ro[qr + 1]].tolist(),
                         ref["rpe_fm"][ro[qr]:ro[qr + 1]].tolist()))
            assert g == r, (t, q)
