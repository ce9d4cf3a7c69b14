"""CC numbers of every RPC and RPF of a tet-SHARDED job ("we can trace their
CC numbers using a simple traversal algorithm"; VERDICT r1 missing item 6): a distributed
union-find -- each rank joins its pieces across its interior faces and exports records of its
shard-boundary faces (rpd_cc_shard), the records of all ranks are joined on every rank and
each rank counts the components whose smallest global id it holds (rpd_cc_merge); the sums
over the ranks must equal the whole mesh's CC numbers from the oracle (oracle.topology) and
from a ctx holding the whole mesh.  Ranks are simulated by one ctx each on one GPU (no kernel
waits on another rank); the collective (dist.cc_sharded) runs on NCCL with world size 1 and,
for its record exchange, on gloo in tests/test_dist_gloo.py."""
import copy

import numpy as np
import pytest

import oracle
import rpd_workloads as W

pytestmark = pytest.mark.gpu

KEYS = ("key_c", "lab_c", "key_f", "j_f", "lab_f")


def sharded_cc(w, world, block, filter_mode="pruned"):
    """The sharded job on `world` simulated ranks: (rpc_cc [N], rpf_cc [E]) as numpy."""
    import torch
    import paper_2403_18761_b200 as P
    ctxs = [P.RPDContext(0, filter_mode=filter_mode) for _ in range(world)]
    try:
        for r, c in enumerate(ctxs):
            ids = W.block_cyclic_shard(w.T, world, r, block=block).astype(np.int32)
            c.set_euler(w.tets, len(w.verts), ids)
            c.relations(w.verts, w.tets[ids], w.spheres, w.nbr_off, w.nbr_idx)
            c.clip()
        sizes = np.array([c.euler_sizes()[:2] for c in ctxs])
        recs = []
        for r, c in enumerate(ctxs):
            rec = c.cc_shard(int(sizes[:r, 0].sum()), int(sizes[:r, 1].sum()))
            recs.append({k: rec[k].clone() for k in KEYS})
        allrec = {k: torch.cat([x[k] for x in recs]) for k in KEYS}
        counts = sum(c.cc_merge(allrec, int(sizes[:, 0].sum()), int(sizes[:, 1].sum()))
                     for c in ctxs)
        N = w.N
        out = counts.cpu().numpy()
        return out[:N], out[N:], sum(int(x["key_c"].numel()) for x in recs)
    finally:
        for c in ctxs:
            c.close()


def whole_cc(w):
    import paper_2403_18761_b200 as P
    c = P.RPDContext(0, filter_mode="pruned")
    try:
        c.set_euler(w.tets, len(w.verts))
        c.relations(w.verts, w.tets, w.spheres, w.nbr_off, w.nbr_idx)
        c.clip()
        t = c.download_topology()
        return np.asarray(t["rpc_cc"]), np.asarray(t["rpf_cc"])
    finally:
        c.close()


def hole_spheres(xs):
    """PAPER.md Fig. 4(b) / 6(a) on the genus-1 box with a hole (components split by it)."""
    w = copy.copy(W.make_shape_workload("one", 700, 1, seed=2, cache=False))
    n = len(xs)
    w.spheres = np.array([[x, 26.0, 20.0, 1.0] for x in xs])
    idx, off = [], [0]
    for a in range(n):
        idx += [b for b in (a - 1, a + 1) if 0 <= b < n]
        off.append(len(idx))
    w.nbr_off, w.nbr_idx = np.array(off, np.int32), np.array(idx, np.int32)
    return w


MAKERS = [lambda: W.make_c1(0), lambda: W.make_c1(1, degenerate=True),
          lambda: W.make_shape_workload("E3", 2000, 150, seed=3, cache=False),
          lambda: W.make_shape_workload("E5", 3000, 300, seed=5, radius_mode="high_variance",
                                        cache=False),
          lambda: W.delaunay_workload(2000, 60, seed=1),
          lambda: hole_spheres([20.0, 44.0]), lambda: hole_spheres([26.0, 32.0, 38.0])]


@pytest.mark.parametrize("k", range(len(MAKERS)))
@pytest.mark.parametrize("world,block", [(2, 64), (3, 256), (8, 32)])
def test_cc_sharded_equals_oracle(k, world, block):
    w = MAKERS[k]()
    rpc, rpf, n_bnd = sharded_cc(w, world, block)
    ref = oracle.rpd_workload(w, euler=True)
    rpc_ref, rpf_ref = oracle.topology(ref, w.tets, w.N)
    assert rpc.tolist() == rpc_ref
    for i in range(w.N):
        for e in range(w.nbr_off[i], w.nbr_off[i + 1]):
            assert rpf[e] == rpf_ref.get((i, int(w.nbr_idx[e])), 0), (i, e)
    if w.T > world * block:
        assert n_bnd > 0  # (the shards do share faces)


@pytest.mark.parametrize("world", [2, 8])
def test_cc_sharded_c3_equals_whole(world):
    """At full C3 size (195 k tets, 20 k spheres, 4096-tet blocks as bench.py shards them)."""
    w = W.make_config("C3")
    rpc, rpf, _ = sharded_cc(w, world, 4096)
    rpc_w, rpf_w = whole_cc(w)
    assert np.array_equal(rpc, rpc_w) and np.array_equal(rpf, rpf_w)


def test_cc_sharded_nccl_world1():
    """dist.cc_sharded through a size-1 NCCL group equals the whole-mesh ctx."""
    import os
    import torch
    import torch.distributed as dist
    import paper_2403_18761_b200 as P
    from paper_2403_18761_b200.dist import cc_sharded, free_port
    w = W.make_shape_workload("E3", 2000, 150, seed=3, cache=False)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(free_port()))
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    c = P.RPDContext(0, filter_mode="pruned")
    try:
        ids = np.arange(w.T, dtype=np.int32)
        c.set_euler(w.tets, len(w.verts), ids)
        c.relations(w.verts, w.tets, w.spheres, w.nbr_off, w.nbr_idx)
        c.clip()
        got = cc_sharded(c)
        rpc_w, rpf_w = whole_cc(w)
        assert np.array_equal(got["rpc_cc"].cpu().numpy(), rpc_w)
        assert np.array_equal(got["rpf_cc"].cpu().numpy(), rpf_w)
    finally:
        c.close()
        dist.destroy_process_group()


def test_cc_shard_state_errors():
    import paper_2403_18761_b200 as P
    w = W.make_c1(0)
    c = P.RPDContext(0)
    try:
        c.set_euler(w.tets, len(w.verts))  # whole mesh: rpd_get_topology, not the shard path
        c.relations(w.verts, w.tets, w.spheres, w.nbr_off, w.nbr_idx)
        c.clip()
        with pytest.raises(P.RPDError) as e:
            c.cc_shard(0, 0)
        assert e.value.status == -5
    finally:
        c.close()


RPE_KEYS = ("key_b", "jk_b", "lab_b")


def sharded_rpe(w, world, block):
    """RPEs of the sharded job on simulated ranks (dist.rpe_sharded's protocol without the
    collectives): (tri [n][3], tri_euler [n], tri_cc [n]) as numpy."""
    import torch
    import paper_2403_18761_b200 as P
    ctxs = [P.RPDContext(0, filter_mode="pruned") for _ in range(world)]
    try:
        for r, c in enumerate(ctxs):
            ids = W.block_cyclic_shard(w.T, world, r, block=block).astype(np.int32)
            c.set_euler(w.tets, len(w.verts), ids)
            c.relations(w.verts, w.tets[ids], w.spheres, w.nbr_off, w.nbr_idx)
            c.clip()
        n_rpe = [c.rpe_shard(0)["n_rpe"] for c in ctxs]
        recs = []
        for r, c in enumerate(ctxs):
            rec = c.rpe_shard(int(sum(n_rpe[:r])))
            recs.append({k: v.clone() if torch.is_tensor(v) else v for k, v in rec.items()})
        cat = lambda k: torch.cat([x[k] for x in recs])
        keys, euler = ctxs[0].reduce_by_key(cat("tri_key"), cat("tri_euler"))
        allb = {k: cat(k) for k in RPE_KEYS}
        parts = [tuple(t.clone() for t in c.rpe_merge(allb, sum(n_rpe))) for c in ctxs]
        ck, cc = ctxs[0].reduce_by_key(torch.cat([p[0] for p in parts]),
                                       torch.cat([p[1] for p in parts]))
        assert torch.equal(ck, keys)
        k = keys.cpu().numpy()
        tri = np.stack([k >> 42, (k >> 21) & 0x1FFFFF, k & 0x1FFFFF], 1).astype(np.int32)
        return tri, euler.cpu().numpy(), cc.cpu().numpy(), sum(int(x["key_b"].numel())
                                                               for x in recs)
    finally:
        for c in ctxs:
            c.close()


def whole_rpe(w):
    import paper_2403_18761_b200 as P
    c = P.RPDContext(0, filter_mode="pruned")
    try:
        c.set_euler(w.tets, len(w.verts))
        c.relations(w.verts, w.tets, w.spheres, w.nbr_off, w.nbr_idx)
        c.clip()
        return c.rpe()
    finally:
        c.close()


def rpe_crossing_the_hole():
    """Three spheres whose common line crosses the genus-1 solid twice (Euler 2, CC 2)."""
    w = copy.copy(W.make_shape_workload("one", 700, 1, seed=2, cache=False))
    w.spheres = np.array([[32.0, 32.0, 20.0, 1.0], [32.0, 20.0, 20.0, 1.0],
                          [32.0, 26.0, 26.0, 1.0]])
    w.nbr_off = np.array([0, 2, 4, 6], np.int32)
    w.nbr_idx = np.array([1, 2, 0, 2, 0, 1], np.int32)
    return w


RPE_MAKERS = [lambda: W.make_shape_workload("E3", 2000, 150, seed=3, cache=False),
              lambda: W.make_shape_workload("E5", 3000, 300, seed=5,
                                            radius_mode="high_variance", cache=False),
              lambda: W.delaunay_workload(2000, 60, seed=1), rpe_crossing_the_hole]


@pytest.mark.parametrize("k", range(len(RPE_MAKERS)))
@pytest.mark.parametrize("world,block", [(2, 64), (3, 32)])
def test_rpe_sharded_equals_whole(k, world, block):
    """Per-(i, j, k) RPE Euler characteristics and CC numbers of a sharded job equal those of
    the ctx holding the whole mesh (whose RPEs are pinned against the oracle's explicit
    extraction in tests/test_gpu_euler.py)."""
    w = RPE_MAKERS[k]()
    tri, euler, cc, n_bnd = sharded_rpe(w, world, block)
    ref = whole_rpe(w)
    assert np.array_equal(tri, ref["tri"])
    assert np.array_equal(euler, ref["tri_euler"])
    assert np.array_equal(cc, ref["tri_cc"])
    if k == len(RPE_MAKERS) - 1:
        assert cc.tolist() == [2, 2, 2] and n_bnd > 0


def test_rpe_sharded_nccl_world1():
    import os
    import torch
    import torch.distributed as dist
    import paper_2403_18761_b200 as P
    from paper_2403_18761_b200.dist import free_port, rpe_sharded
    w = W.make_shape_workload("E3", 2000, 150, seed=3, cache=False)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(free_port()))
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    c = P.RPDContext(0, filter_mode="pruned")
    try:
        ids = np.arange(w.T, dtype=np.int32)
        c.set_euler(w.tets, len(w.verts), ids)
        c.relations(w.verts, w.tets, w.spheres, w.nbr_off, w.nbr_idx)
        c.clip()
        got = rpe_sharded(c)
        ref = whole_rpe(w)
        assert np.array_equal(got["tri"].cpu().numpy(), ref["tri"])
        assert np.array_equal(got["tri_euler"].cpu().numpy(), ref["tri_euler"])
        assert np.array_equal(got["tri_cc"].cpu().numpy(), ref["tri_cc"])
    finally:
        c.close()
        dist.destroy_process_group()


def test_medial_mesh_sharded_nccl_world1():
    """dist.medial_mesh_sharded (keys all-gathered, deduplicated by rpd_reduce_by_key) through
    a size-1 NCCL group, and the library dedupe of two shards' keys, equal the whole mesh's."""
    import os
    import torch
    import torch.distributed as dist
    import paper_2403_18761_b200 as P
    from paper_2403_18761_b200.dist import free_port, medial_mesh_sharded
    w = W.make_shape_workload("Sh", 3000, 200, seed=6, cache=False)
    c = P.RPDContext(0, filter_mode="pruned")
    try:
        c.set_euler(w.tets, len(w.verts))
        c.relations(w.verts, w.tets, w.spheres, w.nbr_off, w.nbr_idx)
        c.clip()
        full = c.medial_mesh()
        keys = []
        for r in range(2):  # two shards' face keys, deduplicated by the library
            ids = W.block_cyclic_shard(w.T, 2, r, block=256).astype(np.int32)
            c.set_euler(w.tets, len(w.verts), ids)
            c.relations(w.verts, w.tets[ids], w.spheres, w.nbr_off, w.nbr_idx)
            c.clip()
            f = torch.as_tensor(c.medial_mesh()["faces"].astype(np.int64)).cuda()
            keys.append((f[:, 0] << 42) | (f[:, 1] << 21) | f[:, 2])
        fk, _ = c.reduce_by_key(torch.cat(keys), torch.zeros(sum(len(k) for k in keys),
                                                             dtype=torch.int64, device="cuda"))
        got = torch.stack([fk >> 42, (fk >> 21) & 0x1FFFFF, fk & 0x1FFFFF], 1).cpu().numpy()
        assert np.array_equal(got, full["faces"])
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(free_port()))
        dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
        try:
            c.set_euler(w.tets, len(w.verts), np.arange(w.T, dtype=np.int32))
            c.relations(w.verts, w.tets, w.spheres, w.nbr_off, w.nbr_idx)
            c.clip()
            mm = medial_mesh_sharded(c)
            assert np.array_equal(mm["edges"].cpu().numpy(), full["edges"])
            assert np.array_equal(mm["faces"].cpu().numpy(), full["faces"])
        finally:
            dist.destroy_process_group()
    finally:
        c.close()
