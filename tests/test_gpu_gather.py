"""Multi-GPU exchange kernels against the ORACLE: block-cyclic tet shards
clipped one after another on one GPU (no kernel waits on another rank), their packed payloads
put back in global tet order by rpd_gather_cands / rpd_gather_pieces, and in partial mode the
dirty segments merged by rpd_merge_shards -- equal to the oracle's single-rank full RPD and its
R11 partial-update chain (P8).  The collective itself (counts all-gather + padded payload
all-gather, dist.exchange) runs on gloo in tests/test_dist_gloo.py and on NCCL (world 1) here."""
import numpy as np
import pytest

import oracle
import rpd_workloads as W
from tests.helpers import compare_results

pytestmark = pytest.mark.gpu


def _pack(ctx, counts, fill, with_ids=False):
    """One rank's packed payload (the bytes dist.exchange would all-gather), as typed views."""
    import torch
    from paper_2403_18761_b200 import dist as D
    secs, nb = D.layout(counts, with_ids)
    buf = torch.empty(nb, dtype=torch.uint8, device="cuda")
    v = D.views(buf, secs)
    fill(v)
    return v


def _host(d):
    return {k: v.cpu().numpy() for k, v in d.items()}


@pytest.mark.parametrize("world,block", [(2, 256), (3, 512), (8, 128)])
def test_gather_and_merge_equal_oracle(world, block):
    import torch
    import paper_2403_18761_b200 as P
    from paper_2403_18761_b200.dist import shard_tets
    P.build()
    ctxs = [P.RPDContext(0, filter_mode="pruned") for _ in range(world)]
    try:
        w = W.make_shape_workload("Gg", 4000, 300, seed=13, n_batches=2, batch_m=15,
                                  clusters=3, cache=False)
        ids = [shard_tets(w.T, world, r, block) for r in range(world)]
        ids_dev = [torch.as_tensor(i, device="cuda") for i in ids]
        shards = []
        for r, ctx in enumerate(ctxs):  # one ctx per simulated rank (each keeps its shard)
            ctx.relations(w.verts, w.tets[ids[r]], w.spheres, w.nbr_off, w.nbr_idx)
            ctx.clip()
            counts = (len(ids[r]), ctx.n_cand, ctx.counts.n_pieces, ctx.counts.n_inc)
            shards.append(_pack(ctx, counts, lambda v, c=ctx: (c.download_cands(out=v),
                                                               c.download_pieces(out=v))))
        nc = sum(int(s["cand_idx"].numel()) for s in shards)
        npc = sum(int(s["piece_sphere"].numel()) for s in shards)
        ni = sum(int(s["inc_sphere"].numel()) for s in shards)
        glob = ctxs[0].gather_all(shards, ids_dev, w.T, nc, npc, ni)
        ref = oracle.rpd_workload(w)
        errs = compare_results(_host(glob), ref, w.verts, w.tets, rel=1e-9)
        assert not errs, errs[:5]
        # partial updates: only the dirty segments (with global ids) are exchanged and merged
        n_old = w.N
        for (sph, off, idx) in w.batches:
            new = np.arange(n_old, len(sph), dtype=np.int32)
            dshards = []
            for r, ctx in enumerate(ctxs):
                _, nd = ctx.update_partial(sph, off, idx, new)
                st = ctx.stats()
                counts = (nd, st["n_cand_dirty"], st["n_pieces_dirty"], st["n_inc_dirty"])
                dshards.append(_pack(ctx, counts, lambda v, c=ctx, n=nd, r=r: c.download_tets(
                    c.dirty_ptr(), n, v, id_map=ids_dev[r]), with_ids=True))
            glob = ctxs[0].merge_shards(dshards, glob, w.T)
            ref, dirty = oracle.partial_update(ref, w.verts, w.tets, sph, off, idx, n_old)
            got_dirty = np.sort(np.concatenate([s["tet_ids"].cpu().numpy() for s in dshards]))
            assert np.array_equal(got_dirty, dirty)
            errs = compare_results(_host(glob), ref, w.verts, w.tets, rel=1e-9)
            assert not errs, errs[:5]
            n_old = len(sph)
    finally:
        for c in ctxs:
            c.close()


def test_download_tets_host_and_device():
    """rpd_download_tets of a tet list equals the slices of the full download, to host
    (pinned / pageable) and device destinations, with and without an id map."""
    import torch
    import paper_2403_18761_b200 as P
    from tests.helpers import slice_tets
    ctx = P.RPDContext(0)
    try:
        w = W.make_shape_workload("Dt", 2500, 200, seed=15, cache=False)
        ctx.relations(w.verts, w.tets, w.spheres, w.nbr_off, w.nbr_idx)
        ctx.clip()
        full = ctx.download_cands()
        full.update(ctx.download_pieces())
        lst = np.sort(np.random.default_rng(3).choice(w.T, 300, replace=False)).astype(np.int32)
        want = slice_tets(full, lst)
        nc, npc, ni = ctx.download_tets(lst, len(lst), {})
        assert (nc, npc, ni) == (len(want["cand_idx"]), len(want["piece_vol"]),
                                 len(want["inc_sphere"]))
        idmap = (np.arange(w.T, dtype=np.int32) * 7 + 3)
        for device in (False, True):
            out = {"cand_off": np.empty(len(lst) + 1, np.int32), "cand_idx": np.empty(nc, np.int32),
                   "piece_off": np.empty(len(lst) + 1, np.int32),
                   "piece_sphere": np.empty(npc, np.int32), "piece_vol": np.empty(npc),
                   "piece_m1": np.empty((npc, 3)), "piece_facemask": np.empty(npc, np.uint8),
                   "inc_off": np.empty(npc + 1, np.int32), "inc_sphere": np.empty(ni, np.int32),
                   "tet_ids": np.empty(len(lst), np.int32)}
            if device:
                out = {k: torch.as_tensor(v).cuda() for k, v in out.items()}
            ctx.download_tets(torch.as_tensor(lst).cuda() if device else lst, len(lst), out,
                              id_map=idmap)
            got = {k: (v.cpu().numpy() if device else v) for k, v in out.items()}
            assert np.array_equal(got["tet_ids"], idmap[lst])
            for k in want:
                assert np.array_equal(np.asarray(got[k]).reshape(np.asarray(want[k]).shape),
                                      np.asarray(want[k])), k
    finally:
        ctx.close()


def test_sharded_rpd_nccl_world1():
    """The bench's sharded path end to end on one GPU: NCCL process group of size 1,
    ShardedRPD.full (counts + payload all-gather, gather kernels) and .partial (dirty segments,
    merge) equal the oracle."""
    import os
    import torch
    import torch.distributed as dist
    import paper_2403_18761_b200 as P
    from paper_2403_18761_b200.dist import ShardedRPD, free_port
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(free_port()))
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    ctx = P.RPDContext(0, filter_mode="pruned")
    try:
        w = W.make_shape_workload("Gn", 2500, 200, seed=14, n_batches=2, batch_m=10,
                                  clusters=2, cache=False)
        S = ShardedRPD(ctx, w.T)
        glob = S.full(w.verts, S.local_tets(w.tets), w.spheres, w.nbr_off, w.nbr_idx)
        ref = oracle.rpd_workload(w)
        errs = compare_results(_host(glob), ref, w.verts, w.tets, rel=1e-9)
        assert not errs, errs[:5]
        n_old = w.N
        for (sph, off, idx) in w.batches:
            glob, nd = S.partial(sph, off, idx, np.arange(n_old, len(sph), dtype=np.int32))
            ref, dirty = oracle.partial_update(ref, w.verts, w.tets, sph, off, idx, n_old)
            assert nd == len(dirty)
            errs = compare_results(_host(glob), ref, w.verts, w.tets, rel=1e-9)
            assert not errs, errs[:5]
            n_old = len(sph)
    finally:
        ctx.close()
        dist.destroy_process_group()


def test_gather_bad_tet_id():
    import torch
    import paper_2403_18761_b200 as P
    ctx = P.RPDContext(0)
    try:
        w = W.make_c1(0)
        ctx.relations(w.verts, w.tets, w.spheres, w.nbr_off, w.nbr_idx)
        ctx.clip()
        loc = {k: v.clone() for k, v in ctx.download_pieces(device=True).items()}
        ids = torch.arange(6, dtype=torch.int32, device="cuda")
        ids[5] = 99
        with pytest.raises(P.RPDError) as e:
            ctx.gather_pieces([loc], [ids], 6)
        assert e.value.status == -1
    finally:
        ctx.close()


def test_gather_c5_two_ranks_equals_single_gpu():
    """a world-2 gather at C5 size (4M tets, 50k spheres, pruned filter): the two
    block-cyclic shards, clipped by two ctxs and put back in global order by the gather kernels,
    are byte-identical to the single-ctx RPD of all tets (candidates and pieces)."""
    import torch
    import paper_2403_18761_b200 as P
    from paper_2403_18761_b200.dist import shard_tets
    w = W.make_config("C5")
    ctx = P.RPDContext(0, filter_mode="pruned")
    try:
        ctx.relations(w.verts, w.tets, w.spheres, w.nbr_off, w.nbr_idx)
        ctx.clip()
        ref = ctx.download_cands(device=True)
        ref.update(ctx.download_pieces(device=True))
        ref = {k: v.clone() for k, v in ref.items()}
        shards, ids = [], []
        for r in range(2):
            tid = shard_tets(w.T, 2, r)
            ctx.relations(w.verts, w.tets[tid], w.spheres, w.nbr_off, w.nbr_idx)
            ctx.clip()
            counts = (len(tid), ctx.n_cand, ctx.counts.n_pieces, ctx.counts.n_inc)
            shards.append(_pack(ctx, counts, lambda v: (ctx.download_cands(out=v),
                                                        ctx.download_pieces(out=v))))
            ids.append(torch.as_tensor(tid, device="cuda"))
        nc = sum(int(s["cand_idx"].numel()) for s in shards)
        npc = sum(int(s["piece_sphere"].numel()) for s in shards)
        ni = sum(int(s["inc_sphere"].numel()) for s in shards)
        got = ctx.gather_all(shards, ids, w.T, nc, npc, ni)
        for k in ref:
            assert torch.equal(got[k].reshape(ref[k].shape), ref[k]), k
    finally:
        ctx.close()


def test_sphere_volumes_shards_sum_to_whole():
    """The validation aggregate of a sharded job: per-sphere RPC volumes of
    the shards (rpd_sphere_volumes) add up to the single ctx's and to the oracle's piece
    volumes summed per sphere (to 1e-12 of the mesh volume: fp64 sums in another order); also
    after partial updates (state pools) and through dist.sphere_volumes on NCCL world 1."""
    import os
    import torch
    import torch.distributed as dist
    import paper_2403_18761_b200 as P
    from paper_2403_18761_b200.dist import free_port, shard_tets, sphere_volumes
    w = W.make_shape_workload("Sv", 3000, 250, seed=9, n_batches=2, batch_m=20, clusters=4,
                              cache=False)
    ref = oracle.rpd_workload(w)
    want = np.bincount(np.asarray(ref["piece_sphere"]), weights=np.asarray(ref["piece_vol"]),
                       minlength=w.N)
    Vt = w.verts[w.tets]
    tol = 1e-12 * np.abs(np.linalg.det(np.stack([Vt[:, k] - Vt[:, 0] for k in (1, 2, 3)],
                                                axis=1))).sum() / 6
    ctxs = [P.RPDContext(0, filter_mode="pruned") for _ in range(3)]
    try:
        whole = ctxs[0]
        whole.relations(w.verts, w.tets, w.spheres, w.nbr_off, w.nbr_idx)
        whole.clip()
        got = whole.sphere_volumes()
        assert np.max(np.abs(got - want)) <= tol
        parts = []
        for r, c in enumerate(ctxs[1:]):
            ids = shard_tets(w.T, 2, r, 256)
            c.relations(w.verts, w.tets[ids], w.spheres, w.nbr_off, w.nbr_idx)
            c.clip()
            parts.append(c.sphere_volumes())
        assert np.max(np.abs(parts[0] + parts[1] - want)) <= tol
        # after the partial updates (pools): still the whole mesh's per-sphere volumes
        n_old, prev = w.N, ref
        for (sph, off, idx) in w.batches:
            new = np.arange(n_old, len(sph), dtype=np.int32)
            whole.update_partial(sph, off, idx, new)
            prev, _ = oracle.partial_update(prev, w.verts, w.tets, sph, off, idx, n_old)
            n_old = len(sph)
        want2 = np.bincount(np.asarray(prev["piece_sphere"]),
                            weights=np.asarray(prev["piece_vol"]), minlength=n_old)
        assert np.max(np.abs(whole.sphere_volumes() - want2)) <= tol
    finally:
        for c in ctxs:
            c.close()
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(free_port()))
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    c = P.RPDContext(0, filter_mode="pruned")
    try:
        c.relations(w.verts, w.tets, w.spheres, w.nbr_off, w.nbr_idx)
        c.clip()
        v = sphere_volumes(c)
        assert np.max(np.abs(v.cpu().numpy() - want)) <= tol
    finally:
        c.close()
        dist.destroy_process_group()
