"""Envelope distance: the CUDA closed forms with
tile culling vs the oracle's golden-section minimisation, through the C ABI (-m gpu).
Tolerance: |dg| <= 1e-9 * (box diagonal) (fp64 closed forms vs a converged convex search)."""
import numpy as np
import pytest

import oracle
import rpd_workloads as W

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ctx():
    import paper_2403_18761_b200 as P
    P.build()
    c = P.RPDContext(0, filter_mode="pruned")
    yield c
    c.close()


def check(ctx, smp, sph, edges, faces, diag):
    g, prim, n_eval = ctx.envelope(smp, sph, edges, faces)
    g_ref, _ = oracle.envelope(smp, sph, edges, faces)
    assert np.max(np.abs(g - g_ref)) <= 1e-9 * diag
    # the reported primitive reaches the minimum
    N, NE = len(sph), len(edges)
    for s in range(0, len(smp), max(1, len(smp) // 40)):
        p = prim[s]
        ids = [p] if p < N else (list(edges[p - N]) if p < N + NE else list(faces[p - N - NE]))
        assert abs(oracle.envelope_one(smp[s], sph, ids) - g_ref[s]) <= 1e-9 * diag
    return g, n_eval


@pytest.mark.parametrize("seed", range(4))
def test_envelope_random(ctx, seed):
    rng = np.random.default_rng(seed)
    sph = np.c_[rng.uniform(0, 10, (30, 3)), rng.uniform(0, 1.5, 30)]
    sph[:3, 3] = [2.5, 0.0, 0.1]  # a big sphere, a zero-radius one
    edges = np.array([[i, (i * 7 + 3) % 30] for i in range(30) if i != (i * 7 + 3) % 30],
                     np.int32)
    faces = np.array([[i, (i + 1) % 30, (i + 5) % 30] for i in range(0, 30, 2)], np.int32)
    smp = rng.uniform(-3, 13, (300, 3))
    check(ctx, smp, sph, edges, faces, 16 * np.sqrt(3))


def test_envelope_degenerate_primitives(ctx):
    """Nested end spheres (|dr| >= L), collinear slab centres, equal radii (capsule)."""
    sph = np.array([[0, 0, 0, 3.0], [1, 0, 0, 0.5], [2, 0, 0, 1.0], [4, 0, 0, 1.0],
                    [0, 4, 0, 1.0], [6, 1, 0, 0.0]])
    edges = np.array([[0, 1], [2, 3], [3, 5]], np.int32)
    faces = np.array([[1, 2, 3], [2, 3, 4], [0, 4, 5]], np.int32)
    rng = np.random.default_rng(9)
    smp = rng.uniform(-4, 8, (400, 3))
    check(ctx, smp, sph, edges, faces, 12 * np.sqrt(3))


def test_envelope_medial_mesh_c2(ctx):
    """The medial mesh of a C2-style RPD (our own pipeline) against boundary samples of its
    mesh, the paper's use."""
    w = W.make_shape_workload("Env", 8000, 300, seed=21, cache=False)
    ctx.set_euler(w.tets, len(w.verts))
    try:
        ctx.relations(w.verts, w.tets, w.spheres, w.nbr_off, w.nbr_idx)
        ctx.clip()
        mm = ctx.medial_mesh()
    finally:
        ctx.set_euler(None, 0)
    smp = W.boundary_samples(w.verts, w.tets, 64, seed=3)
    g, n_eval = check(ctx, smp, w.spheres, mm["edges"], mm["faces"], 100.0)
    P = len(w.spheres) + len(mm["edges"]) + len(mm["faces"])
    assert n_eval < len(smp) * P  # the tile culling skipped work


def test_envelope_c3_sampled(ctx):
    """At the bench size (C3 medial mesh: 20k spheres, ~56k cones, ~80k slabs; 100k boundary
    samples): sampled samples against the oracle; every distance finite, the culling
    effective."""
    w = W.make_config("C3")
    ctx.set_euler(w.tets, len(w.verts))
    try:
        ctx.relations(w.verts, w.tets, w.spheres, w.nbr_off, w.nbr_idx)
        ctx.clip()
        mm = ctx.medial_mesh()
    finally:
        ctx.set_euler(None, 0)
    smp = W.boundary_samples(w.verts, w.tets, 100_000, seed=5)
    g, prim, n_eval = ctx.envelope(smp, w.spheres, mm["edges"], mm["faces"])
    assert np.all(np.isfinite(g))
    P = len(w.spheres) + len(mm["edges"]) + len(mm["faces"])
    assert n_eval < 0.1 * len(smp) * P
    ids = np.random.default_rng(0).choice(len(smp), 6, replace=False)
    g_ref, _ = oracle.envelope(smp[ids], w.spheres, mm["edges"], mm["faces"])
    assert np.max(np.abs(g[ids] - g_ref)) <= 1e-9 * 100.0


def test_envelope_bad_ids(ctx):
    import paper_2403_18761_b200 as P
    sph = np.array([[0, 0, 0, 1.0], [3, 0, 0, 1.0]])
    with pytest.raises(P.RPDError) as e:
        ctx.envelope(np.zeros((4, 3)), sph, np.array([[0, 2]], np.int32), np.zeros((0, 3), np.int32))
    assert e.value.status == -1
    g, _, _ = ctx.envelope(np.array([[1.5, 2.0, 0.0]]), sph, np.array([[0, 1]], np.int32),
                           np.zeros((0, 3), np.int32))  # the ctx still works
    assert g[0] == pytest.approx(1.0, abs=1e-12)
