"""The CUDA-graph latency path of partial updates (RPD_OPT_GRAPH; DESIGN.md §8 "latency
path"; SURVEY §8(a) a6 / (d) C4 "use CUDA Graphs"; "few (even single) spheres").
A device-driven update of 1..64 new spheres replayed as one graph must leave the ctx in the
same state as the eager launches, byte for byte (candidates, dirty lists, pieces), and equal
the oracle's R11 partial-update chain; a failed device-side capacity check falls back to the
eager batch with the same result."""
import numpy as np
import pytest

import oracle
import rpd_workloads as W
from tests.helpers import compare_results

pytestmark = pytest.mark.gpu


def _state(ctx):
    out = ctx.download_cands()
    out.update(ctx.download_pieces())
    out["dirty"] = ctx.dirty_tets().cpu().numpy()
    return out


def _chain(ctx, w, graph, device_inputs=False):
    """relations + clip, then every batch of w as a partial update; the state after each."""
    import torch
    to = (lambda a: torch.as_tensor(np.ascontiguousarray(a)).cuda()) if device_inputs \
        else (lambda a: a)
    ctx.set_graph(graph)
    ctx.relations(to(w.verts), to(w.tets), to(w.spheres), to(w.nbr_off), to(w.nbr_idx))
    ctx.clip()
    states, n_old = [], w.N
    for (sph, off, idx) in w.batches:
        ctx.update_partial(to(sph), to(off), to(idx),
                           to(np.arange(n_old, len(sph), dtype=np.int32)))
        states.append(_state(ctx))
        n_old = len(sph)
    return states


def _same(a, b):
    for k in a:
        assert np.array_equal(np.asarray(a[k]), np.asarray(b[k])), k


@pytest.mark.parametrize("m,clusters", [(1, 1), (3, 3), (10, 5), (40, 8)])
def test_graph_equals_eager_and_oracle(m, clusters):
    import paper_2403_18761_b200 as P
    P.build()
    w = W.make_shape_workload(f"G{m}", 3000, 250, seed=5 + m, n_batches=5, batch_m=m,
                              clusters=clusters, cache=False)
    ctx = P.RPDContext(0, filter_mode="pruned")
    try:
        st0 = ctx.stats()
        eager = _chain(ctx, w, graph=False)
        st1 = ctx.stats()
        assert st1["graph_updates"] == st0["graph_updates"]
        graph = _chain(ctx, w, graph=True)
        st2 = ctx.stats()
        assert st2["graph_updates"] - st1["graph_updates"] == len(w.batches)
        # one capture per buffer layout: the stage buffers alternate, the pools may compact once
        assert st2["graph_captures"] - st1["graph_captures"] <= 4
        for g, e in zip(graph, eager):
            _same(g, e)
        # and the oracle's chain (every tet)
        ref, n_old = oracle.rpd_workload(w), w.N
        for (sph, off, idx), g in zip(w.batches, graph):
            ref, dirty = oracle.partial_update(ref, w.verts, w.tets, sph, off, idx, n_old)
            assert np.array_equal(g["dirty"], dirty)
            errs = compare_results(g, ref, w.verts, w.tets, rel=1e-9)
            assert not errs, errs[:5]
            n_old = len(sph)
    finally:
        ctx.close()


def test_graph_device_inputs_and_replays():
    """Device-tensor inputs (pointers differ per update: read from the device record, not baked
    into the graph) and many replays of the same captured graphs."""
    import paper_2403_18761_b200 as P
    w = W.make_shape_workload("Gd", 3000, 250, seed=21, n_batches=12, batch_m=2, clusters=2,
                              cache=False)
    ctx = P.RPDContext(0, filter_mode="pruned")
    try:
        eager = _chain(ctx, w, graph=False, device_inputs=True)
        c0 = ctx.stats()["graph_captures"]
        graph = _chain(ctx, w, graph=True, device_inputs=True)
        st = ctx.stats()
        assert st["graph_captures"] - c0 <= 4 < len(w.batches)
        assert st["graph_fallbacks"] == 0
        for g, e in zip(graph, eager):
            _same(g, e)
    finally:
        ctx.close()


def test_graph_fallback_large_batch(monkeypatch):
    """A batch beyond the graph's candidate bound (here fixed at 1024 by the testing knob
    RPD_GRAPH_NC_MAX, read at ctx creation) aborts on the device and is redone by the eager
    launches: same state as the eager chain, and the fallback is counted."""
    import paper_2403_18761_b200 as P
    w = W.make_shape_workload("Gf", 3000, 250, seed=2, n_batches=3, batch_m=30, clusters=6,
                              cache=False)
    ctx = P.RPDContext(0, filter_mode="pruned")
    try:
        eager = _chain(ctx, w, graph=False)
    finally:
        ctx.close()
    monkeypatch.setenv("RPD_GRAPH_NC_MAX", "1024")
    ctx = P.RPDContext(0, filter_mode="pruned")
    try:
        graph = _chain(ctx, w, graph=True)
        st = ctx.stats()
        for g, e in zip(graph, eager):
            _same(g, e)
        assert st["n_cand_dirty"] > 1024 and st["graph_fallbacks"] >= 1
        assert st["graph_updates"] == len(w.batches)
    finally:
        ctx.close()


def test_graph_bench_sized_batches():
    """Large batches (M = 200, the bench's regime) also run as graphs (fast clip tier and its
    overflow cascade; the batch bound grows with the batches): equal to the eager chain."""
    import paper_2403_18761_b200 as P
    w = W.make_shape_workload("Gb", 20000, 1500, seed=4, n_batches=4, batch_m=200, clusters=10,
                              cache=False)
    ctx = P.RPDContext(0, filter_mode="pruned")
    ctx.set_profile(True)  # (bench.py's setting: timer stamps inside the graph)
    try:
        eager = _chain(ctx, w, graph=False)
        f0 = ctx.stats()["graph_fallbacks"]
        graph = _chain(ctx, w, graph=True)
        st = ctx.stats()
        for g, e in zip(graph, eager):
            _same(g, e)
        assert st["n_cand_dirty"] >= 2048  # (the fast tier took the batch)
        assert st["filter_ms"] > 0 and st["clip_ms"] > 0 and st["graph_updates"] > 0
        print("graph fallbacks", st["graph_fallbacks"] - f0, "captures", st["graph_captures"])
    finally:
        ctx.close()


@pytest.mark.parametrize("route", [4, 10])
def test_graph_clip_routing(monkeypatch, route):
    """RPD_CLIP_ROUTE: the graph sends the pairs with more cut planes than the threshold to the
    64-slot tier in a concurrent branch; same state as the eager chain."""
    import paper_2403_18761_b200 as P
    w = W.make_shape_workload("Gr", 20000, 1500, seed=4, n_batches=3, batch_m=200, clusters=10,
                              cache=False)
    ctx = P.RPDContext(0, filter_mode="pruned")
    try:
        eager = _chain(ctx, w, graph=False)
    finally:
        ctx.close()
    monkeypatch.setenv("RPD_CLIP_ROUTE", str(route))
    ctx = P.RPDContext(0, filter_mode="pruned")
    try:
        graph = _chain(ctx, w, graph=True)
        for g, e in zip(graph, eager):
            _same(g, e)
        assert ctx.stats()["graph_updates"] == len(w.batches)
    finally:
        ctx.close()


def test_graph_errors_reset_ctx():
    """Input errors found inside the graph (new ids not the appended range, a moved old
    sphere) fail the call like the eager path and reset the ctx."""
    import paper_2403_18761_b200 as P
    w = W.make_shape_workload("Ge", 2000, 150, seed=3, n_batches=1, batch_m=4, clusters=2,
                              cache=False)
    sph, off, idx = w.batches[0]
    ctx = P.RPDContext(0, filter_mode="pruned")
    try:
        for case in ("ids", "moved"):
            ctx.relations(w.verts, w.tets, w.spheres, w.nbr_off, w.nbr_idx)
            ctx.clip()
            new = np.arange(w.N, len(sph), dtype=np.int32)
            s2 = sph.copy()
            if case == "ids":
                new = new[::-1].copy()
            else:
                s2[0, 0] += 2.0 ** -10
            with pytest.raises(P.RPDError) as e:
                ctx.update_partial(s2, off, idx, new)
            assert e.value.status == -1
            with pytest.raises(P.RPDError):
                ctx.clip()
        # usable again after a fresh relations + clip
        ctx.relations(w.verts, w.tets, w.spheres, w.nbr_off, w.nbr_idx)
        ctx.clip()
        ctx.update_partial(sph, off, idx, np.arange(w.N, len(sph), dtype=np.int32))
        ref, _ = oracle.partial_update(oracle.rpd_workload(w), w.verts, w.tets, sph, off, idx,
                                       w.N)
        errs = compare_results(_state(ctx), ref, w.verts, w.tets, rel=1e-9)
        assert not errs, errs[:5]
    finally:
        ctx.close()
