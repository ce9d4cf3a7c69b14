"""Partial RPD update on the GPU vs the oracle (-m gpu).  DESIGN.md R11/R12: dirty tets =
tets related (Alg. 1) to a new sphere, re-filtered and re-clipped; clean tets keep their
pieces byte-identically; pieces equal a full recompute (inputs without exact-zero hits)."""
import numpy as np
import pytest

import oracle
import rpd_workloads as W
from tests.helpers import compare_results, slice_tets

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", params=["all_pairs", "pruned"])
def ctx(request):
    import paper_2403_18761_b200 as P
    P.build()
    c = P.RPDContext(0, filter_mode=request.param)
    yield c
    c.close()


def gpu_state(ctx):
    out = ctx.download_cands()
    out.update(ctx.download_pieces())
    return out


@pytest.mark.parametrize("seed", [3, 7])
def test_partial_equals_oracle_partial(ctx, seed):
    w = W.make_shape_workload("S", 2000, 150, seed=seed, n_batches=3, batch_m=12, clusters=3,
                              cache=False)
    ctx.relations(w.verts, w.tets, w.spheres, w.nbr_off, w.nbr_idx)
    ctx.clip()
    prev = oracle.rpd_workload(w)
    n_old = w.N
    for (sph, off, idx) in w.batches:
        new = np.arange(n_old, len(sph), dtype=np.int32)
        counts, nd = ctx.update_partial(sph, off, idx, new)
        got = gpu_state(ctx)
        ref, dirty = oracle.partial_update(prev, w.verts, w.tets, sph, off, idx, n_old)
        assert nd == len(dirty) and nd > 0
        errs = compare_results(got, ref, w.verts, w.tets, rel=1e-9)
        assert not errs, errs[:5]
        # pieces also equal a full recompute (no exact-zero hits on this generic input)
        full = oracle.rpd(w.verts, w.tets, sph, off, idx)
        errs = compare_results(got, full, w.verts, w.tets, rel=1e-9, check_cands=False)
        assert not errs, errs[:5]
        prev, n_old = ref, len(sph)


def test_partial_identity_and_errors(ctx):
    import paper_2403_18761_b200 as P
    w = W.make_shape_workload("S", 2000, 150, seed=3, n_batches=1, batch_m=12, clusters=3,
                              cache=False)
    ctx.relations(w.verts, w.tets, w.spheres, w.nbr_off, w.nbr_idx)
    ctx.clip()
    before = gpu_state(ctx)
    counts, nd = ctx.update_partial(w.spheres, w.nbr_off, w.nbr_idx, np.zeros(0, np.int32))
    assert nd == 0
    after = gpu_state(ctx)
    for k in before:
        assert np.array_equal(before[k], after[k]), k
    sph, off, idx = w.batches[0]
    bad = np.arange(w.N, len(sph), dtype=np.int32)[::-1].copy()
    with pytest.raises(P.RPDError) as e:
        ctx.update_partial(sph, off, idx, bad)
    assert e.value.status == -1


def test_partial_error_leaves_ctx_usable(ctx):
    """A failed update (a changed old sphere, or new ids that are not the appended range)
    resets the ctx instead of leaving it half-updated: the next rpd_clip / update is a state
    error, and a fresh rpd_relations + rpd_clip gives the oracle's result again."""
    import paper_2403_18761_b200 as P
    w = W.make_shape_workload("S", 2000, 150, seed=3, n_batches=1, batch_m=12, clusters=3,
                              cache=False)
    sph, off, idx = w.batches[0]
    new = np.arange(w.N, len(sph), dtype=np.int32)
    for bad_case in ("moved", "ids"):
        ctx.relations(w.verts, w.tets, w.spheres, w.nbr_off, w.nbr_idx)
        ctx.clip()
        s2, ids = sph.copy(), new
        if bad_case == "moved":
            s2[5, 3] += 1.0 / 1024  # an existing sphere's radius changes
        else:
            ids = new[::-1].copy()
        with pytest.raises(P.RPDError) as e:
            ctx.update_partial(s2, off, idx, ids)
        assert e.value.status == -1
        with pytest.raises(P.RPDError) as e:
            ctx.clip()
        assert e.value.status == -5
        with pytest.raises(P.RPDError) as e:
            ctx.update_partial(sph, off, idx, new)
        assert e.value.status == -5
    ctx.relations(w.verts, w.tets, sph, off, idx)
    ctx.clip()
    errs = compare_results(gpu_state(ctx), oracle.rpd(w.verts, w.tets, sph, off, idx),
                           w.verts, w.tets, rel=1e-9)
    assert not errs, errs[:5]


def test_partial_before_clip_is_state_error():
    import paper_2403_18761_b200 as P
    c = P.RPDContext(0)
    w = W.make_c1(0)
    with pytest.raises(P.RPDError) as e:
        c.update_partial(w.spheres, w.nbr_off, w.nbr_idx, np.zeros(0, np.int32))
    assert e.value.status == -5
    c.close()


def test_c4_chain_every_tet(ctx, c4_workload, oracle_c4_chain):
    """BASELINE.json configs[3] at full size, as bench.py runs it: the C3 full RPD, then 10
    iterations x M = 500 on the 200k-tet mesh.  After EVERY iteration, the dirty-tet list, the
    candidate CSR and the pieces of EVERY tet equal the oracle's R11 partial-update chain
    (oracle.partial_update from the oracle's own full RPD)."""
    w = c4_workload
    ctx.relations(w.verts, w.tets, w.spheres, w.nbr_off, w.nbr_idx)
    ctx.clip()
    errs = compare_results(gpu_state(ctx), oracle_c4_chain[0][0], w.verts, w.tets, rel=1e-9)
    assert not errs, errs[:5]
    n_old = w.N
    for it, (sph, off, idx) in enumerate(w.batches):
        new = np.arange(n_old, len(sph), dtype=np.int32)
        counts, nd = ctx.update_partial(sph, off, idx, new)
        ref, dirty = oracle_c4_chain[it + 1]
        assert nd == len(dirty) and 0 < nd < w.T
        assert np.array_equal(ctx.dirty_tets().cpu().numpy(), dirty), it
        errs = compare_results(gpu_state(ctx), ref, w.verts, w.tets, rel=1e-9,
                               label=f"iteration {it}: ")
        assert not errs, errs[:5]
        n_old = len(sph)


@pytest.mark.parametrize("seed", [1, 2])
def test_c4_chain_every_tet_other_seeds(seed):
    """The C4 workload of seeds 1 and 2 (seeds 0, 1, 2 per config; bench.py
    --seed, tools/seeds.py) as the bench runs it (pruned filter, graph updates): the C3 full
    RPD and the 10 x 500 chain equal the oracle's on every tet after every iteration."""
    import paper_2403_18761_b200 as P
    P.build()
    w = W.make_config("C4", seed=seed)
    c = P.RPDContext(0, filter_mode="pruned")
    try:
        c.relations(w.verts, w.tets, w.spheres, w.nbr_off, w.nbr_idx)
        c.clip()
        prev = oracle.rpd_workload(w)
        errs = compare_results(gpu_state(c), prev, w.verts, w.tets, rel=1e-9)
        assert not errs, errs[:5]
        n_old = w.N
        for it, (sph, off, idx) in enumerate(w.batches):
            new = np.arange(n_old, len(sph), dtype=np.int32)
            counts, nd = c.update_partial(sph, off, idx, new)
            prev, dirty = oracle.partial_update(prev, w.verts, w.tets, sph, off, idx, n_old)
            assert nd == len(dirty)
            assert np.array_equal(c.dirty_tets().cpu().numpy(), dirty), it
            errs = compare_results(gpu_state(c), prev, w.verts, w.tets, rel=1e-9,
                                   label=f"seed {seed} iteration {it}: ")
            assert not errs, errs[:5]
            n_old = len(sph)
        assert c.stats()["graph_updates"] == len(w.batches)
    finally:
        c.close()
