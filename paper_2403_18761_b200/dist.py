"""Multi-GPU plumbing: tets sharded block-cyclically over the ranks of one
node, spheres and neighbour lists replicated, per-rank RPD outputs all-gathered with NCCL.

The exchange is the only cross-rank step of the path (every (tet, sphere) pair is
independent).  Outputs of every rank are downloaded into torch tensors on the rank's device,
their sizes all-gathered, the payloads all-gathered padded to the largest rank, and the
pieces put back in global tet order.  Works with any torch.distributed backend (NCCL on the
GPUs, gloo for the CPU tests).
"""
from __future__ import annotations

import numpy as np
import torch
import torch.distributed as dist

PIECE_KEYS = ("piece_sphere", "piece_vol", "piece_m1", "piece_facemask")


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


def gather_pieces(local: dict, tet_ids_local, T: int, group=None) -> dict:
    """All-gather the per-rank piece CSRs (keys piece_off, piece_sphere, piece_vol, piece_m1,
    piece_facemask, inc_off, inc_sphere; tensors on the rank's device) and reorder them to
    global tet order.  Returns the global CSR on every rank."""
    world = dist.get_world_size(group)
    dev = local["piece_vol"].device
    tid = torch.as_tensor(np.asarray(tet_ids_local), dtype=torch.int64, device=dev)
    po = local["piece_off"].to(torch.int64)
    counts = po[1:] - po[:-1]
    io = local["inc_off"].to(torch.int64)
    ninc = io[1:] - io[:-1]
    g_tid = _all_gather_padded(tid, group)
    g_cnt = _all_gather_padded(counts, group)
    g = {k: _all_gather_padded(local[k], group) for k in PIECE_KEYS}
    g_ninc = _all_gather_padded(ninc, group)
    g_inc = _all_gather_padded(local["inc_sphere"], group)
    # global per-tet piece counts -> offsets
    cnt = torch.zeros(T, dtype=torch.int64, device=dev)
    for r in range(world):
        cnt[g_tid[r].long()] = g_cnt[r]
    off = torch.zeros(T + 1, dtype=torch.int64, device=dev)
    off[1:] = torch.cumsum(cnt, 0)
    n_pieces = int(off[-1].item())
    out = {"piece_off": off.to(torch.int32)}
    # destination index of every piece of every rank
    dest = []
    for r in range(world):
        c = g_cnt[r]
        start = off[g_tid[r].long()]
        local_off = torch.cumsum(c, 0) - c            # first piece of each tet (local)
        rep_start = torch.repeat_interleave(start - local_off, c)
        dest.append(rep_start + torch.arange(int(c.sum().item()), device=dev))
    for k in PIECE_KEYS:
        shape = (n_pieces,) + tuple(g[k][0].shape[1:])
        buf = torch.empty(shape, dtype=g[k][0].dtype, device=dev)
        for r in range(world):
            buf[dest[r]] = g[k][r]
        out[k] = buf
    ninc_all = torch.zeros(n_pieces, dtype=torch.int64, device=dev)
    for r in range(world):
        ninc_all[dest[r]] = g_ninc[r]
    inc_off = torch.zeros(n_pieces + 1, dtype=torch.int64, device=dev)
    inc_off[1:] = torch.cumsum(ninc_all, 0)
    inc = torch.empty(int(inc_off[-1].item()), dtype=torch.int32, device=dev)
    for r in range(world):
        n_r = g_ninc[r]
        src_start = torch.cumsum(n_r, 0) - n_r
        d_start = inc_off[dest[r]]
        rep = torch.repeat_interleave(d_start - src_start, n_r)
        inc[rep + torch.arange(int(n_r.sum().item()), device=dev)] = g_inc[r]
    out["inc_off"] = inc_off.to(torch.int32)
    out["inc_sphere"] = inc
    out["piece_m1"] = out["piece_m1"].reshape(-1, 3)
    return out


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
