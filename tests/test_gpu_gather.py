"""rpd_gather_pieces: per-rank piece CSRs of block-cyclic tet shards,
put back in global tet order by the CUDA kernels, are byte-identical to a single-GPU run
(P8).  The ranks are run one after another on one GPU (no kernel waits on another rank)."""
import numpy as np
import pytest

import rpd_workloads as W

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("world,block", [(2, 256), (3, 512), (8, 128)])
def test_gather_equals_single_gpu(world, block):
    import torch
    import paper_2403_18761_b200 as P
    from paper_2403_18761_b200.dist import shard_tets
    P.build()
    ctx = P.RPDContext(0, filter_mode="pruned")
    try:
        w = W.make_shape_workload("Gg", 4000, 300, seed=13, cache=False)
        ctx.relations(w.verts, w.tets, w.spheres, w.nbr_off, w.nbr_idx)
        ctx.clip()
        ref = ctx.download_pieces()
        shards, ids = [], []
        for r in range(world):
            tid = shard_tets(w.T, world, r, block)
            ctx.relations(w.verts, w.tets[tid], w.spheres, w.nbr_off, w.nbr_idx)
            ctx.clip()
            shards.append({k: v.clone() for k, v in ctx.download_pieces(device=True).items()})
            ids.append(torch.as_tensor(tid, device="cuda"))
        got = ctx.gather_pieces(shards, ids, w.T)
        for k in ref:
            assert np.array_equal(got[k].cpu().numpy().reshape(np.asarray(ref[k]).shape),
                                  np.asarray(ref[k])), k
    finally:
        ctx.close()


def test_dist_gather_pieces_nccl_world1():
    """The bench's gather path end to end on one GPU: NCCL process group of size 1,
    dist.gather_pieces (all-gather + rpd_gather_pieces) returns the rank's own pieces."""
    import os
    import socket
    import torch
    import torch.distributed as dist
    import paper_2403_18761_b200 as P
    from paper_2403_18761_b200.dist import gather_pieces, shard_tets
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    ctx = P.RPDContext(0, filter_mode="pruned")
    try:
        w = W.make_shape_workload("Gn", 2500, 200, seed=14, cache=False)
        ids = shard_tets(w.T, 1, 0)
        ctx.relations(w.verts, w.tets[ids], w.spheres, w.nbr_off, w.nbr_idx)
        ctx.clip()
        loc = ctx.download_pieces(device=True)
        got = gather_pieces(loc, ids, w.T, ctx)
        for k in loc:
            assert torch.equal(got[k].reshape(loc[k].shape), loc[k]), k
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
