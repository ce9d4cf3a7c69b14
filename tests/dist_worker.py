"""One rank of the CPU multi-rank test (tests/test_dist_gloo.py::test_launcher_*), started by
paper_2403_18761_b200.dist.launch_ranks (torch.distributed.run, gloo): the rank's block-cyclic
shard of the oracle's results goes through dist.exchange -- the same counts + padded payload
all-gathers the NCCL path runs -- first the full candidate + piece CSRs, then per partial update
only the dirty tets' segments with their global ids.  Rank 0 saves every rank's received
payloads to argv[1] (npz); the test reorders / merges them and compares with the single-rank
oracle.  (Packing here is a host copy: there is no GPU on the CPU box.)"""
import os
import pickle
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
import rpd_workloads as W  # noqa: E402
from paper_2403_18761_b200 import dist as D  # noqa: E402


def fill_from(res, ids=None):
    def fill(v):
        for k, t in v.items():
            src = np.asarray(ids if k == "tet_ids" else res[k]).reshape(-1)
            t.reshape(-1).copy_(torch.as_tensor(src))
    return fill


def main():
    out_path = sys.argv[1]
    dist.init_process_group("gloo")
    rank, world = dist.get_rank(), dist.get_world_size()
    w = W.make_shape_workload("G", 3000, 200, seed=12, n_batches=2, batch_m=12, clusters=3,
                              cache=False)
    ids = D.shard_tets(w.T, world, rank, block=256)
    r = oracle.rpd_workload(w, tet_ids=ids)
    counts = (len(ids), len(r["cand_idx"]), len(r["piece_vol"]), len(r["inc_sphere"]))
    got, cnt = D.exchange(counts, fill_from(r), torch.device("cpu"))
    rounds = [{"full": [{k: v.numpy().copy() for k, v in g.items()} for g in got]}]
    n_old = w.N
    for (sph, off, idx) in w.batches:
        r, dirty_local = oracle.partial_update(r, w.verts, w.tets[ids], sph, off, idx, n_old)
        sub = oracle.rpd(w.verts, w.tets[ids], sph, off, idx, tet_ids=dirty_local) \
            if len(dirty_local) else None
        if sub is None:
            sub = {k: np.zeros(0) for k in ("cand_idx", "piece_vol", "inc_sphere")}
            sub.update(cand_off=np.zeros(1, np.int32), piece_off=np.zeros(1, np.int32),
                       inc_off=np.zeros(1, np.int32))
        counts = (len(dirty_local), len(sub["cand_idx"]), len(sub["piece_vol"]),
                  len(sub["inc_sphere"]))
        got, cnt = D.exchange(counts, fill_from(sub, ids[dirty_local]), torch.device("cpu"),
                              with_ids=True)
        rounds.append({"dirty": [{k: v.numpy().copy() for k, v in g.items()} for g in got]})
        n_old = len(sph)
    if rank == 0:
        with open(out_path, "wb") as f:
            pickle.dump(rounds, f)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
