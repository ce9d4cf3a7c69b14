"""Multi-rank path on CPU (gloo, world_size 2): block-cyclic tet shards of the oracle's
results all-gathered (dist.all_gather_pieces, the collective of the gather) and reordered
equal the single-rank result byte for byte.  The CUDA kernels are
per-tet independent, so the same holds on NCCL; the reorder kernel (rpd_gather_pieces) is
tested against a single-GPU run in tests/test_gpu_gather.py."""
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


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2403_18761_b200.dist import all_gather_pieces, shard_tets
        w = W.make_shape_workload("G", 3000, 200, seed=12, cache=False)
        ids = shard_tets(w.T, world, rank, block=256)
        r = oracle.rpd_workload(w, tet_ids=ids)
        local = {k: torch.as_tensor(np.asarray(v)) for k, v in r.items() if k != "stats"}
        local["piece_m1"] = local["piece_m1"].reshape(-1, 3)
        shards = all_gather_pieces(local)
        if rank == 0:
            q.put(_reorder([{k: v.numpy() for k, v in d.items()} for d in shards],
                           [shard_tets(w.T, world, s, block=256) for s in range(world)], w.T))
    finally:
        dist.destroy_process_group()


def _reorder(shards, ids, T):
    """Test-side reorder of all-gathered per-rank CSRs into global tet order (the product path
    does this in rpd_gather_pieces, tested against the single-GPU result in -m gpu)."""
    per_tet = [None] * T
    for d, tid in zip(shards, ids):
        po, io = d["piece_off"], d["inc_off"]
        for a, t in enumerate(tid):
            pcs = []
            for p in range(po[a], po[a + 1]):
                pcs.append((d["piece_sphere"][p], d["piece_vol"][p], tuple(d["piece_m1"][p]),
                            d["piece_facemask"][p], list(d["inc_sphere"][io[p]:io[p + 1]])))
            per_tet[t] = pcs
    out = {k: [] for k in ("piece_sphere", "piece_vol", "piece_m1", "piece_facemask",
                           "inc_sphere")}
    off, ioff = [0], [0]
    for pcs in per_tet:
        for (s, v, m, f, inc) in pcs:
            out["piece_sphere"].append(s)
            out["piece_vol"].append(v)
            out["piece_m1"].append(m)
            out["piece_facemask"].append(f)
            out["inc_sphere"] += inc
            ioff.append(len(out["inc_sphere"]))
        off.append(len(out["piece_sphere"]))
    out = {k: np.array(v) for k, v in out.items()}
    out["piece_off"], out["inc_off"] = np.array(off, np.int32), np.array(ioff, np.int32)
    return out


def test_gather_equals_single_rank():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = q.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    w = W.make_shape_workload("G", 3000, 200, seed=12, cache=False)
    ref = oracle.rpd_workload(w)
    for k in ("piece_off", "piece_sphere", "piece_vol", "piece_facemask", "inc_off",
              "inc_sphere"):
        assert np.array_equal(np.asarray(got[k]), np.asarray(ref[k])), k
    assert np.array_equal(got["piece_m1"].reshape(-1, 3), ref["piece_m1"])


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
