"""CUDA path vs the CPU oracle, element by element, through the C ABI (-m gpu).

Bar: candidate CSR, non-empty set, facemasks and incidences bit-exact;
|dvol| <= 1e-9 vol(t), |dm1| <= 1e-9 vol(t) diam(t) (north star tolerance, R10).
"""
import json
import os

import numpy as np
import pytest

import oracle
import rpd_workloads as W
from tests.helpers import compare_results, piece_tet, slice_tets, tet_volumes

pytestmark = pytest.mark.gpu

REL = 1e-9


@pytest.fixture(scope="module")
def ctx():
    import paper_2403_18761_b200 as P
    P.build()
    c = P.RPDContext(0)
    yield c
    c.close()


def run_gpu(ctx, w, device_inputs=True):
    import torch
    args = [w.verts, w.tets, w.spheres, w.nbr_off, w.nbr_idx]
    if device_inputs:
        args = [torch.as_tensor(np.asarray(a)).cuda() for a in args]
    ctx.relations(*args)
    ctx.clip()
    out = ctx.download_cands()
    out.update(ctx.download_pieces())
    out["stats"] = ctx.stats()
    return out


def check(ctx, w, **kw):
    got = run_gpu(ctx, w, **kw)
    ref = oracle.rpd_workload(w)
    errs = compare_results(got, ref, w.verts, w.tets, rel=REL)
    assert not errs, errs[:5]
    return got, ref


@pytest.mark.parametrize("seed,deg,big", [(0, False, False), (1, False, False), (2, False, False),
                                          (0, True, False), (1, True, False), (2, True, False),
                                          (5, True, True), (6, True, True)])
def test_c1_unit_cube(ctx, seed, deg, big):
    """BASELINE.json configs[0]: unit cube, 6 Kuhn tets, 16 dyadic spheres; C1b is degenerate
    (radical planes through Kuhn faces/vertices) and exercises the exact SoS path."""
    got, ref = check(ctx, W.make_c1(seed, degenerate=deg, big=big))
    if deg:
        assert got["stats"]["zero_hits"] > 0


@pytest.mark.parametrize("seed", range(6))
def test_tiny_grids(ctx, seed):
    check(ctx, W.random_tiny(seed, n_spheres=14, grid=2, coarse=(seed % 2 == 1)))


@pytest.mark.parametrize("seed,tets,sph,mode", [(3, 2000, 150, "uniform"),
                                                (4, 5000, 400, "uniform"),
                                                (5, 3000, 300, "high_variance"),
                                                (6, 4000, 60, "uniform")])
def test_shape_workloads(ctx, seed, tets, sph, mode):
    """Several tiles (256-tet filter blocks, 8-pair clip blocks) and a ragged tail."""
    w = W.make_shape_workload(f"P{seed}", tets, sph, seed=seed, radius_mode=mode, cache=False)
    assert w.T % 256 != 0
    got, ref = check(ctx, w)
    # the kernel's algorithmic-work counter equals the oracle's literal Alg. 1 test count
    assert got["stats"]["rel_tests"] == ref["stats"]["n_rel_tests"]
    vt = tet_volumes(w.verts, w.tets)
    s = np.zeros(w.T)
    np.add.at(s, piece_tet(got), got["piece_vol"])
    assert np.max(np.abs(s - vt) / vt) < 1e-9


def test_host_inputs_equal_device_inputs(ctx):
    w = W.make_shape_workload("H", 1500, 120, seed=8, cache=False)
    a = run_gpu(ctx, w, device_inputs=True)
    b = run_gpu(ctx, w, device_inputs=False)
    for k in a:
        if k != "stats":
            assert np.array_equal(np.asarray(a[k]), np.asarray(b[k])), k


def test_torch_inputs_other_dtypes_are_stream_ordered(ctx):
    """Inputs made by torch kernels just before the call (float32 -> float64 and int64 ->
    int32 conversions inside the binding, all on torch's default stream) are read by the
    library in stream order (the ctx runs on the legacy default stream)."""
    import torch
    w = W.make_shape_workload("Hd", 3000, 250, seed=21, cache=False)
    for _ in range(3):
        args = [torch.as_tensor(w.verts).cuda().float(), torch.as_tensor(w.tets).cuda().long(),
                torch.as_tensor(w.spheres).cuda().float(),
                torch.as_tensor(w.nbr_off).cuda().long(), torch.as_tensor(w.nbr_idx).cuda().long()]
        ctx.relations(*args)
        ctx.clip()
        got = ctx.download_cands()
        got.update(ctx.download_pieces())
        errs = compare_results(got, oracle.rpd_workload(w), w.verts, w.tets, rel=REL)
        assert not errs, errs[:5]


def _shell_workload(n_shell=100):
    """One big tet; a sphere at c = (12.5, 12.5, 12.5) surrounded by n_shell spheres on a shell
    of radius 6 (Fibonacci points on the 2^-10 lattice), all radii 0, all-pairs neighbour lists
    (a superset): the inner sphere's piece is its whole Voronoi cell, a
    polytope with ~n_shell facets and ~2 n_shell vertices."""
    import types
    verts = np.array([[0.0, 0.0, 0.0], [60.0, 0.0, 0.0], [0.0, 60.0, 0.0], [0.0, 0.0, 60.0]])
    tets = np.array([[0, 1, 2, 3]], np.int32)
    k = np.arange(n_shell) + 0.5
    phi = np.arccos(1 - 2 * k / n_shell)
    th = np.pi * (1 + 5 ** 0.5) * k
    pts = 12.5 + 6.0 * np.c_[np.cos(th) * np.sin(phi), np.sin(th) * np.sin(phi), np.cos(phi)]
    pts = np.round(pts * 1024) / 1024
    sph = np.vstack([[12.5, 12.5, 12.5, 0.0], np.c_[pts, np.zeros(n_shell)]])
    N = len(sph)
    off = np.arange(N + 1, dtype=np.int32) * (N - 1)
    idx = np.array([j for i in range(N) for j in range(N) if j != i], np.int32)
    return types.SimpleNamespace(verts=verts, tets=tets, spheres=sph, nbr_off=off, nbr_idx=idx,
                                 T=1, N=N)


@pytest.mark.parametrize("tiers", [False, True])
def test_slow_path_large_piece(ctx, tiers):
    """a piece beyond the 128-slot tier (here ~200 vertices, 104 planes) is
    clipped by the 256-slot slow path, not dropped: parity with the oracle, and the stats show
    the large piece."""
    w = _shell_workload()
    ctx.set_clip_tiers(tiers)
    try:
        got, ref = check(ctx, w)
    finally:
        ctx.set_clip_tiers(False)
    assert got["stats"]["max_vertices"] > 128
    inner = [p for p in range(len(got["piece_sphere"])) if got["piece_sphere"][p] == 0]
    assert len(inner) == 1 and len(got["inc_sphere"][got["inc_off"][inner[0]]:
                                                     got["inc_off"][inner[0] + 1]]) > 90


def test_single_sphere(ctx):
    w = W.make_shape_workload("one", 700, 1, seed=2, cache=False)
    got, _ = check(ctx, w)
    assert np.all(got["piece_facemask"] == 15) and len(got["inc_sphere"]) == 0


def test_equal_radii_vs_zero_radii(ctx):
    """equal weights -> Voronoi; r = c and r = 0 give byte-identical output."""
    w = W.make_shape_workload("V", 1500, 120, seed=4, radius_mode="equal", cache=False)
    s0 = w.spheres.copy()
    s0[:, 3] = 0.0
    sc = w.spheres.copy()
    sc[:, 3] = 0.75
    off, idx = W.power_neighbours(s0)
    import copy
    w0 = copy.copy(w)
    w0.spheres, w0.nbr_off, w0.nbr_idx = s0, off, idx
    wc = copy.copy(w0)
    wc.spheres = sc
    a = run_gpu(ctx, w0)
    b = run_gpu(ctx, wc)
    for k in a:
        if k != "stats":
            assert np.array_equal(np.asarray(a[k]), np.asarray(b[k])), k


def test_empty_inputs(ctx):
    w = W.make_c1(0)
    n = ctx.relations(w.verts, np.zeros((0, 4), np.int32), w.spheres, w.nbr_off, w.nbr_idx)
    assert n == 0
    c = ctx.clip()
    assert c.n_pieces == 0
    n = ctx.relations(w.verts, w.tets, np.zeros((0, 4)), np.zeros(1, np.int32),
                      np.zeros(0, np.int32))
    assert n == 0


def test_input_errors(ctx):
    import paper_2403_18761_b200 as P
    w = W.make_c1(0)
    bad = w.verts.copy()
    bad[0, 0] = 1.0 / 3.0
    with pytest.raises(P.RPDError) as e:
        ctx.relations(bad, w.tets, w.spheres, w.nbr_off, w.nbr_idx)
    assert e.value.status == -6
    flipped = w.tets.copy()
    flipped[0, [1, 2]] = flipped[0, [2, 1]]
    with pytest.raises(P.RPDError) as e:
        ctx.relations(w.verts, flipped, w.spheres, w.nbr_off, w.nbr_idx)
    assert e.value.status == -1
    idx = w.nbr_idx.copy()
    idx[0] = 0  # sphere 0 lists itself
    with pytest.raises(P.RPDError) as e:
        ctx.relations(w.verts, w.tets, w.spheres, w.nbr_off, idx)
    assert e.value.status == -1
    sph = w.spheres.copy()
    sph[3, 3] = -1.0 / 1024
    with pytest.raises(P.RPDError) as e:
        ctx.relations(w.verts, w.tets, sph, w.nbr_off, w.nbr_idx)
    assert e.value.status == -1
    # clip after a failed relations call is a state error
    with pytest.raises(P.RPDError) as e:
        ctx.clip()
    assert e.value.status == -5


@pytest.mark.parametrize("mode", ["all_pairs", "pruned"])
def test_bench_config_every_tet(ctx, ctx_pruned, c4_workload, oracle_c4_chain, mode):
    """At BASELINE.json's full size (C3: ~200k tets, 20k spheres), in the launch configuration
    bench.py times: EVERY tet's candidates and pieces compared with the oracle's full RPD
    (Alg. 1 over all 20k spheres), plus the partition of every tet."""
    w = c4_workload
    got = run_gpu(ctx if mode == "all_pairs" else ctx_pruned, w)
    ref = oracle_c4_chain[0][0]
    errs = compare_results(got, ref, w.verts, w.tets, rel=REL)
    assert not errs, errs[:5]
    assert got["stats"]["n_cand"] == len(ref["cand_idx"])
    if mode == "all_pairs":
        assert got["stats"]["rel_tests"] == ref["stats"]["n_rel_tests"]
    vt = tet_volumes(w.verts, w.tets)
    s = np.zeros(w.T)
    np.add.at(s, piece_tet(got), got["piece_vol"])
    assert np.max(np.abs(s - vt) / vt) < 1e-9


ALG1 = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "alg1_cases.json")))


@pytest.mark.parametrize("case", ALG1["cases"], ids=lambda c: c["name"])
@pytest.mark.parametrize("mode", ["all_pairs", "pruned"])
def test_alg1_golden_cases_gpu(ctx, ctx_pruned, case, mode):
    """The hand-derived Alg. 1 answers (strict tie, over-report, first/last neighbour
    rejection; tests/golden/alg1_cases.json) through the C ABI, both filter modes."""
    from tests.test_oracle_pins import alg1_case, check_alg1_golden
    c = ctx if mode == "all_pairs" else ctx_pruned
    args = alg1_case(case)
    c.relations(*args)
    c.clip()
    r = c.download_cands()
    r.update(c.download_pieces())
    check_alg1_golden(case, r)


@pytest.mark.parametrize("make", [lambda: W.make_c1(1, degenerate=True),
                                  lambda: W.make_c1(6, degenerate=True, big=True),
                                  lambda: W.make_shape_workload("Wd", 2500, 200, seed=9,
                                                                radius_mode="high_variance",
                                                                cache=False)])
def test_wide_kernel_parity(ctx, make):
    """The 128-vertex clip instantiation (used for pairs that overflow the fast 32-vertex
    kernel) run on every pair gives the same results."""
    ctx.set_clip_wide(True)
    try:
        check(ctx, make())
    finally:
        ctx.set_clip_wide(False)


@pytest.fixture(scope="module")
def ctx_pruned():
    import paper_2403_18761_b200 as P
    P.build()
    c = P.RPDContext(0, filter_mode="pruned")
    yield c
    c.close()


@pytest.mark.parametrize("make", [lambda: W.make_c1(0), lambda: W.make_c1(1, degenerate=True),
                                  lambda: W.make_c1(6, degenerate=True, big=True),
                                  lambda: W.random_tiny(3, n_spheres=14, grid=2, coarse=True),
                                  lambda: W.make_shape_workload("P3", 2000, 150, seed=3,
                                                                cache=False),
                                  lambda: W.make_shape_workload("P5", 3000, 300, seed=5,
                                                                radius_mode="high_variance",
                                                                cache=False),
                                  lambda: W.make_shape_workload("one", 700, 1, seed=2,
                                                                cache=False)])
def test_pruned_filter_parity(ctx_pruned, make):
    """the pruned filter gives the same candidate lists (and pieces) as the
    literal all-pairs Alg. 1 / the oracle, while evaluating fewer pairs."""
    w = make()
    got, ref = check(ctx_pruned, w)
    st = got["stats"]
    assert st["pairs_tested"] <= st["pairs_filtered"]


def test_pruned_equals_allpairs_c3(ctx, ctx_pruned):
    w = W.make_config("C3")
    a = run_gpu(ctx, w)
    b = run_gpu(ctx_pruned, w)
    for k in ("cand_off", "cand_idx", "piece_off", "piece_sphere", "piece_vol", "piece_m1",
              "piece_facemask", "inc_off", "inc_sphere"):
        assert np.array_equal(np.asarray(a[k]), np.asarray(b[k])), k
    assert b["stats"]["pairs_tested"] < a["stats"]["pairs_tested"] / 20


def test_c5_sampled(ctx_pruned):
    """BASELINE.json configs[4] at full size (C5: ~4M tets, 50k spheres, high radius variance,
    k_site tails of 1000+), pruned filter as bench.py --config C5 runs it: ~8k sampled tets
    (random + one whole Morton block) compared one by one with the oracle (Alg. 1 over all 50k
    spheres), partition on every tet."""
    w = W.make_config("C5")
    got = run_gpu(ctx_pruned, w)
    rng = np.random.default_rng(5)
    # 4096 random tets + one whole 4096-tet Morton block (a rank's shard unit, spatially
    # contiguous: shared faces, the same spheres' cells) in the middle of the mesh
    blk = (w.T // 2) // 4096 * 4096
    ids = np.union1d(rng.choice(w.T, 4096, replace=False),
                     np.arange(blk, min(blk + 4096, w.T))).astype(np.int32)
    ref = oracle.rpd_workload(w, tet_ids=ids)
    errs = compare_results(slice_tets(got, ids), ref, w.verts, w.tets, tet_ids=ids, rel=REL)
    assert not errs, errs[:5]
    vt = tet_volumes(w.verts, w.tets)
    s = np.zeros(w.T)
    np.add.at(s, piece_tet(got), got["piece_vol"])
    assert np.max(np.abs(s - vt) / vt) < 1e-9


@pytest.mark.parametrize("make", [lambda: W.make_c1(0), lambda: W.make_c1(1, degenerate=True),
                                  lambda: W.make_c1(6, degenerate=True, big=True),
                                  lambda: W.random_tiny(3, n_spheres=14, grid=2, coarse=True),
                                  lambda: W.make_shape_workload("T3", 2000, 150, seed=3,
                                                                cache=False)])
def test_fast_tier_parity_small_inputs(ctx, make):
    """Fewer than 2048 pairs normally go straight to the 64-slot tier; the fast 16-slot tier
    and its overflow cascade, forced on the same small (and degenerate) inputs, agree."""
    ctx.set_clip_tiers(True)
    try:
        check(ctx, make())
    finally:
        ctx.set_clip_tiers(False)
