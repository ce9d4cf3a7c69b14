"""Multi-rank path on CPU (gloo, world_size 2), started through bench.py's launcher: block-cyclic
tet shards of the oracle's results exchanged by dist.exchange (the collective of the gather:
counts all-gather + padded payload all-gather) and reordered equal the single-rank result byte
for byte, also for the dirty-segment exchange of partial updates.  The
CUDA reorder / merge kernels (rpd_gather_*, rpd_merge_shards) are tested against the oracle in
tests/test_gpu_gather.py."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
import rpd_workloads as W


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _reorder(shards, ids, T):
    """Test-side reorder of all-gathered per-rank CSRs into global tet order (the product path
    does this in rpd_gather_cands / rpd_gather_pieces, tested against the oracle in -m gpu)."""
    L = [None] * T
    for d, tid in zip(shards, ids):
        for a, row in enumerate(oracle.per_tet_lists(d, len(tid))):
            L[int(tid[a])] = row
    return oracle.from_per_tet_lists(L)


def test_launcher_two_gloo_ranks(tmp_path):
    """bench.py's launcher (dist.launch_ranks: torch.distributed.run, 127.0.0.1) starts 2 gloo
    ranks; through dist.exchange (one counts all-gather + one padded payload all-gather per
    exchange) every rank receives every shard, and the shards reordered into global tet order
    equal the single-rank oracle -- for the full RPD and, after each partial update, with only
    the dirty segments (and their global ids) exchanged and merged."""
    import pickle
    from paper_2403_18761_b200.dist import launch_ranks, shard_tets
    out = tmp_path / "rounds.pkl"
    rc = launch_ranks(2, os.path.join(os.path.dirname(__file__), "dist_worker.py"), [str(out)])
    assert rc == 0
    rounds = pickle.load(open(out, "rb"))
    w = W.make_shape_workload("G", 3000, 200, seed=12, n_batches=2, batch_m=12, clusters=3,
                              cache=False)
    ids = [shard_tets(w.T, 2, r, block=256) for r in range(2)]
    ref = oracle.rpd_workload(w)
    got = _reorder(rounds[0]["full"], ids, w.T)
    for k in got:
        assert np.array_equal(np.asarray(got[k]), np.asarray(ref[k])), k
    n_old = w.N
    for rd, (sph, off, idx) in zip(rounds[1:], w.batches):
        ref, dirty = oracle.partial_update(ref, w.verts, w.tets, sph, off, idx, n_old)
        shards = rd["dirty"]
        gids = np.concatenate([s["tet_ids"] for s in shards])
        assert np.array_equal(np.sort(gids), dirty)
        L = oracle.per_tet_lists(got, w.T)
        for s in shards:
            for a, row in enumerate(oracle.per_tet_lists(s, len(s["tet_ids"]))):
                L[int(s["tet_ids"][a])] = row
        got = oracle.from_per_tet_lists(L)
        for k in got:
            assert np.array_equal(np.asarray(got[k]), np.asarray(ref[k])), k
        n_old = len(sph)


def test_shards_partition_the_tets():
    from paper_2403_18761_b200.dist import shard_tets
    T = 100_003
    for world in (1, 2, 4, 8):
        ids = np.concatenate([shard_tets(T, world, r) for r in range(world)])
        assert np.array_equal(np.sort(ids), np.arange(T))
        sizes = [len(shard_tets(T, world, r)) for r in range(world)]
        assert max(sizes) - min(sizes) <= 4096


def _euler_csr(r, w):
    """Oracle per-piece Euler numerators summed per sphere (rpc [N]) and per CSR entry of its
    neighbour row (rpf [E]) as int64 -- the layout of rpd_download_euler."""
    rpc = np.zeros(w.N, np.int64)
    rpf = np.zeros(len(w.nbr_idx), np.int64)
    ro = r["rpf_off"]
    for p, i in enumerate(r["piece_sphere"].tolist()):
        rpc[i] += r["piece_euler"][p]
        row = w.nbr_idx[w.nbr_off[i]:w.nbr_off[i + 1]]
        for k in range(ro[p], ro[p + 1]):
            e = w.nbr_off[i] + int(np.nonzero(row == r["rpf_sphere"][k])[0][0])
            rpf[e] += r["rpf_euler"][k]
    return rpc, rpf


def _euler_worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2403_18761_b200.dist import allreduce_euler, shard_tets
        w = W.make_shape_workload("G", 3000, 200, seed=12, cache=False)
        ids = shard_tets(w.T, world, rank, block=256)
        r = oracle.rpd_workload(w, tet_ids=ids, euler=True)
        rpc, rpf = _euler_csr(r, w)
        out = allreduce_euler({"rpc_sum": torch.as_tensor(rpc), "rpf_sum": torch.as_tensor(rpf)})
        if rank == 0:
            q.put({k: v.numpy() for k, v in out.items()} | {"L": r["euler_denom"]})
    finally:
        dist.destroy_process_group()


def test_euler_allreduce_equals_single_rank():
    """NEXT-1 on the sharded path: the per-rank RPC / RPF sums of the tet shards, all-reduced,
    equal the single-rank sums (payloads built from the whole mesh on every rank)."""
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_euler_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = q.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    w = W.make_shape_workload("G", 3000, 200, seed=12, cache=False)
    ref = oracle.rpd_workload(w, euler=True)
    rpc, rpf = _euler_csr(ref, w)
    assert got["L"] == ref["euler_denom"]
    assert np.array_equal(got["rpc_sum"], rpc) and np.array_equal(got["rpf_sum"], rpf)
