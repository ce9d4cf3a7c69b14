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


PRIMES = [p for p in range(2, 256) if all(p % d for d in range(2, int(p ** 0.5) + 1))]
PPOW = [max(p ** e for e in range(1, 9) if p ** e <= 255) for p in PRIMES]


def _acc_row(fr):
    """A Fraction as the library's accumulator row [K, R_1 .. R_P] over PRIMES (test side:
    partial fractions by Python integers; residues scaled to p^E)."""
    from fractions import Fraction
    num, L = fr.numerator, fr.denominator
    row = [0] * (1 + len(PRIMES))
    rest = Fraction(num, L)
    for j, p in enumerate(PRIMES):
        if L % p:
            continue
        q = p
        while L % (q * p) == 0:
            q *= p
        a = num * pow(L // q, -1, q) % q
        row[1 + j] = a * (PPOW[j] // q)
        rest -= Fraction(a, q)
    assert rest.denominator == 1
    row[0] = int(rest)
    return row


def _euler_csr(r, w):
    """Oracle per-piece Euler values summed per sphere (rpc [N, 1+P]) and per CSR entry of
    its neighbour row (rpf [E, 1+P]) as accumulator rows -- the layout of rpd_download_euler."""
    from fractions import Fraction
    rpc = np.zeros((w.N, 1 + len(PRIMES)), np.int64)
    rpf = np.zeros((len(w.nbr_idx), 1 + len(PRIMES)), np.int64)
    ro = r["rpf_off"]
    for p, i in enumerate(r["piece_sphere"].tolist()):
        L = int(r["piece_euler_den"][p])
        rpc[i] += _acc_row(Fraction(int(r["piece_euler"][p]), L))
        row = w.nbr_idx[w.nbr_off[i]:w.nbr_off[i + 1]]
        for k in range(ro[p], ro[p + 1]):
            e = w.nbr_off[i] + int(np.nonzero(row == r["rpf_sphere"][k])[0][0])
            rpf[e] += _acc_row(Fraction(int(r["rpf_euler"][k]), L))
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
        out = allreduce_euler({"rpc_acc": torch.as_tensor(rpc), "rpf_acc": torch.as_tensor(rpf)},
                              None)
        if rank == 0:
            q.put({k: v.numpy() for k, v in out.items()})
    finally:
        dist.destroy_process_group()


def test_euler_allreduce_equals_single_rank():
    """NEXT-1 on the sharded path: the per-rank exact accumulator rows of the RPC / RPF sums
    (integer part + one residue per prime, R24), all-reduced, equal the single-rank
    rows, and decode to the oracle's exact sums (payloads built from the whole mesh on every
    rank)."""
    from fractions import Fraction
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
    assert np.array_equal(got["rpc_acc"], rpc) and np.array_equal(got["rpf_acc"], rpf)
    want, _ = oracle.euler_sums(ref, w.N, w.nbr_off, w.nbr_idx)
    dec = [int(row[0]) + sum(Fraction(int(x), q) for x, q in zip(row[1:], PPOW)) for row in rpc]
    assert dec == want


def _records_worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2403_18761_b200.dist import gather_records
        rng = np.random.default_rng(rank)
        n = [5, 0, 37][rank]  # (ragged, one rank empty)
        parts = {"key_c": torch.as_tensor(rng.integers(0, 1 << 50, n), dtype=torch.int64),
                 "lab_c": torch.arange(n, dtype=torch.int32) + 1000 * rank,
                 "j_f": torch.as_tensor(rng.integers(0, 99, 2 * n), dtype=torch.int32)}
        out = gather_records(parts, torch.device("cpu"))
        if rank == 0:
            q.put({k: v.numpy() for k, v in out.items()})
    finally:
        dist.destroy_process_group()


def test_gather_records_three_gloo_ranks():
    """The record exchange of the sharded CC numbers (dist.gather_records: one counts
    all-gather + one padded byte all-gather) concatenates the ranks' ragged arrays in rank
    order, every dtype intact."""
    world = 3
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_records_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = q.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    want = {"key_c": [], "lab_c": [], "j_f": []}
    for r in range(world):
        rng = np.random.default_rng(r)
        n = [5, 0, 37][r]
        want["key_c"].append(rng.integers(0, 1 << 50, n))
        want["lab_c"].append(np.arange(n, dtype=np.int32) + 1000 * r)
        want["j_f"].append(rng.integers(0, 99, 2 * n))
    for k in want:
        assert np.array_equal(got[k], np.concatenate(want[k]).astype(got[k].dtype)), k
