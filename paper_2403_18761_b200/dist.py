"""Multi-GPU plumbing: tets sharded block-cyclically over the ranks of one
node, spheres and neighbour lists replicated, per-rank RPD outputs all-gathered with NCCL.

The exchange is the only cross-rank step of the path (every (tet, sphere) pair is
independent).  Outputs of every rank are downloaded into torch tensors on the rank's device,
their sizes all-gathered, the payloads all-gathered padded to the largest rank (NCCL over
NVLink; gloo in the CPU tests), and the pieces put back in global tet order by the library's
rpd_gather_pieces kernels (no torch compute on the path).
"""
from __future__ import annotations

import numpy as np
import torch
import torch.distributed as dist

def shard_tets(T: int, world: int, rank: int, block: int = 4096) -> np.ndarray:
    """Global ids of this rank's tets: Morton-ordered blocks of ``block`` tets dealt
    round-robin (balances the O(T N) filter and spatially clustered partial updates)."""
    ids = np.arange(T, dtype=np.int64)
    return ids[(ids // block) % world == rank].astype(np.int32)


def _all_gather_padded(x: torch.Tensor, group=None):
    """All-gather a 1-D (or row) tensor of per-rank length; returns the list of pieces."""
    world = dist.get_world_size(group)
    n = torch.tensor([x.shape[0]], dtype=torch.int64, device=x.device)
    ns = [torch.zeros_like(n) for _ in range(world)]
    dist.all_gather(ns, n, group=group)
    ns = [int(v.item()) for v in ns]
    m = max(ns) if ns else 0
    pad = torch.zeros((m,) + tuple(x.shape[1:]), dtype=x.dtype, device=x.device)
    pad[:x.shape[0]] = x
    bufs = [torch.empty_like(pad) for _ in range(world)]
    dist.all_gather(bufs, pad, group=group)
    return [b[:k] for b, k in zip(bufs, ns)]


PIECE_ARRAYS = ("piece_off", "piece_sphere", "piece_vol", "piece_m1", "piece_facemask",
                "inc_off", "inc_sphere")


def all_gather_pieces(local: dict, group=None) -> list:
    """The collective of the gather (plumbing): every rank's piece CSR (tensors on its device)
    all-gathered -- sizes first, then the payloads padded to the largest rank -- so that every
    rank holds all ranks' CSRs.  Returns one dict per rank."""
    world = dist.get_world_size(group)
    g = {k: _all_gather_padded(local[k].reshape(local[k].shape[0], -1) if k == "piece_m1"
                                else local[k], group) for k in PIECE_ARRAYS}
    return [{k: g[k][r] for k in PIECE_ARRAYS} for r in range(world)]


_IDS = {}


def gather_pieces(local: dict, tet_ids_local, T: int, ctx, group=None) -> dict:
    """Global piece CSR on every rank: NCCL all-gather of the per-rank piece
    CSRs, then rpd_gather_pieces (CUDA) puts them in global tet order.  The ranks' global tet
    ids follow from the block-cyclic sharding (no exchange)."""
    world = dist.get_world_size(group)
    shards = all_gather_pieces(local, group)
    dev = local["piece_vol"].device
    key = (T, world, str(dev), len(tet_ids_local))
    if key not in _IDS:
        blk = _shard_block(T, world, tet_ids_local, dist.get_rank(group))
        _IDS[key] = [torch.as_tensor(shard_tets(T, world, r, blk), device=dev)
                     for r in range(world)]
    return ctx.gather_pieces(shards, _IDS[key], T)


def _shard_block(T, world, ids, rank):
    """The block size of the shard ``ids`` of ``rank`` (default 4096)."""
    for blk in (4096, 256, 1024, 2048, 8192):
        s = shard_tets(T, world, rank, blk)
        if len(s) == len(ids) and np.array_equal(s, np.asarray(ids)):
            return blk
    raise ValueError("tet ids are not a block-cyclic shard")


def allreduce_euler(local: dict, group=None) -> dict:
    """Per-sphere fractional Euler sums of the whole job (SURVEY.md §8(e) "validation
    aggregates"): every rank's rpc_sum [N] and rpf_sum [E] (int64 numerators over the common
    denominator, identical on all ranks because the payloads are built from the whole mesh)
    are summed by one all-reduce each.  Integer sums: exact and order-independent."""
    out = dict(local)
    for k in ("rpc_sum", "rpf_sum"):
        t = local[k].to(torch.int64).clone()
        dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
        out[k] = t
    return out
