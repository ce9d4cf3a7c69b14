"""Multi-GPU plumbing: tets sharded block-cyclically over the ranks of one
node, spheres and neighbour lists replicated, and the per-rank RPD outputs exchanged with NCCL.

The exchange is the only cross-rank step of the path (every (tet, sphere) pair is
independent).  Per exchange there is ONE counts all-gather (4 int64 per rank, one host sync)
and ONE payload all-gather: every rank packs its segments into one byte buffer (the library
copies them in, ``rpd_download_*`` / ``rpd_download_tets``), the buffers are all-gathered
padded to the largest rank (NCCL over NVLink/NVSwitch; gloo in the CPU tests), and the library
puts them into global tet order on every rank:

* full RPD: the candidate and piece CSRs of every shard -> ``rpd_gather_cands`` +
  ``rpd_gather_pieces``;
* partial update: only the dirty tets' segments and their global ids -> ``rpd_merge_shards``
  replaces those rows of the previous global CSR (SURVEY.md §8(e) "all-gathers only the
  changed segments plus the dirty-tet ids").

No torch compute runs on the path: torch provides the buffers and the collectives.
"""
from __future__ import annotations

import os
import socket
import subprocess
import sys

import numpy as np
import torch
import torch.distributed as dist

BLOCK = 4096


def shard_tets(T: int, world: int, rank: int, block: int = BLOCK) -> np.ndarray:
    """Global ids of this rank's tets: Morton-ordered blocks of ``block`` tets dealt
    round-robin (balances the O(T N) filter and spatially clustered partial updates)."""
    ids = np.arange(T, dtype=np.int64)
    return ids[(ids // block) % world == rank].astype(np.int32)


# ------------------------------------------------------------------ packed payload layout

# (key, dtype, length as a function of the counts (rows, n_cand, n_pieces, n_inc))
SECTIONS = {
    "ids": ("tet_ids", np.int32, lambda n, c, p, i: n),
    "cands": [("cand_off", np.int32, lambda n, c, p, i: n + 1),
              ("cand_idx", np.int32, lambda n, c, p, i: c)],
    "pieces": [("piece_off", np.int32, lambda n, c, p, i: n + 1),
               ("piece_sphere", np.int32, lambda n, c, p, i: p),
               ("piece_vol", np.float64, lambda n, c, p, i: p),
               ("piece_m1", np.float64, lambda n, c, p, i: 3 * p),
               ("piece_facemask", np.uint8, lambda n, c, p, i: p),
               ("inc_off", np.int32, lambda n, c, p, i: p + 1),
               ("inc_sphere", np.int32, lambda n, c, p, i: i)],
}


def layout(counts, with_ids: bool):
    """Byte layout of one rank's packed payload: [(key, dtype, length, byte offset)], each
    section 16-byte aligned; returns (sections, total bytes)."""
    n, c, p, i = (int(x) for x in counts)
    secs = ([SECTIONS["ids"]] if with_ids else []) + SECTIONS["cands"] + SECTIONS["pieces"]
    out, off = [], 0
    for key, dt, f in secs:
        ln = int(f(n, c, p, i))
        out.append((key, dt, ln, off))
        off += (ln * np.dtype(dt).itemsize + 15) // 16 * 16
    return out, off


_TDT = {np.int32: torch.int32, np.float64: torch.float64, np.uint8: torch.uint8}


def views(buf: torch.Tensor, secs) -> dict:
    """Typed views of the sections of a packed byte buffer."""
    out = {}
    for key, dt, ln, off in secs:
        nb = ln * np.dtype(dt).itemsize
        out[key] = buf[off:off + nb].view(_TDT[dt])
    out["piece_m1"] = out["piece_m1"].reshape(-1, 3)
    return out


def exchange(counts_local, fill, device, group=None, with_ids=False):
    """The collective of one exchange: counts all-gathered (one host sync), every rank's
    payload packed by ``fill(views)`` into one buffer, all-gathered padded to the largest rank.
    Returns (per-rank typed views of the gathered payloads, per-rank counts [world, 4])."""
    world = dist.get_world_size(group)
    cl = torch.tensor([int(x) for x in counts_local], dtype=torch.int64, device=device)
    ca = torch.empty(world * 4, dtype=torch.int64, device=device)
    dist.all_gather_into_tensor(ca, cl, group=group)
    counts = ca.view(world, 4).cpu().numpy()                       # the one host sync
    lay = [layout(counts[r], with_ids) for r in range(world)]
    maxb = max(b for _, b in lay)
    rank = dist.get_rank(group)
    buf = torch.empty(maxb, dtype=torch.uint8, device=device)
    fill(views(buf, lay[rank][0]))
    big = torch.empty(world * maxb, dtype=torch.uint8, device=device)
    dist.all_gather_into_tensor(big, buf, group=group)
    return [views(big[r * maxb:(r + 1) * maxb], lay[r][0]) for r in range(world)], counts


# ------------------------------------------------------------------ the sharded RPD


class ShardedRPD:
    """The RPD of all T tets on every rank of ``group``: each rank clips its block-cyclic
    shard with its own librpd ctx, and the exchanges above assemble the global candidate and
    piece CSRs (torch CUDA tensors / ctx-owned arrays) on every rank."""

    def __init__(self, ctx, T: int, group=None, block: int = BLOCK):
        self.ctx, self.T, self.group, self.block = ctx, int(T), group, block
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self.dev = torch.device("cuda", ctx.device)
        self.ids = shard_tets(self.T, self.world, self.rank, block)
        self.ids_dev = torch.as_tensor(self.ids, device=self.dev)
        self.all_ids = [torch.as_tensor(shard_tets(self.T, self.world, r, block),
                                        device=self.dev) for r in range(self.world)]
        self.glob = None      # the global CSR: dict of device tensors (views of ctx arrays)
        self.bytes_sent = 0

    def local_tets(self, tets):
        return tets[self.ids]

    def full(self, verts, tets_local, spheres, nbr_off, nbr_idx):
        """rpd_relations + rpd_clip of this rank's shard, then the gather of every shard."""
        self.ctx.relations(verts, tets_local, spheres, nbr_off, nbr_idx)
        self.ctx.clip()
        return self.gather_full()

    def gather_full(self):
        """The exchange after a full RPD of every shard: all candidate + piece CSRs."""
        ctx = self.ctx
        counts = (len(self.ids), ctx.n_cand, ctx.counts.n_pieces, ctx.counts.n_inc)

        def fill(v):
            ctx.download_cands(out=v)
            ctx.download_pieces(out=v)
        shards, cnt = exchange(counts, fill, self.dev, self.group)
        self.bytes_sent = int(sum(layout(cnt[r], False)[1] for r in range(self.world)))
        nc, npc, ni = (int(cnt[:, k].sum()) for k in (1, 2, 3))
        self.glob = ctx.gather_all(shards, self.all_ids, self.T, nc, npc, ni)
        return self.glob

    def partial(self, spheres, nbr_off, nbr_idx, new_ids):
        """rpd_update_partial of this rank's shard, then the exchange of the dirty tets'
        segments and their global ids, merged into the global CSR (rpd_merge_shards)."""
        _, nd = self.ctx.update_partial(spheres, nbr_off, nbr_idx, new_ids)
        return self.exchange_partial(nd)

    def exchange_partial(self, nd: int):
        """The exchange after a partial update of every shard: the dirty tets' segments with
        their global ids, merged into the global CSR; returns (global CSR, total dirty)."""
        ctx = self.ctx
        st = ctx.stats_struct()  # (a ctypes struct: no dict on the timed path)
        counts = (nd, st.n_cand_dirty, st.n_pieces_dirty, st.n_inc_dirty)

        def fill(v):
            ctx.download_tets(ctx.dirty_ptr(), nd, v, id_map=self.ids_dev)
        shards, cnt = exchange(counts, fill, self.dev, self.group, with_ids=True)
        self.bytes_sent = int(sum(layout(cnt[r], True)[1] for r in range(self.world)))
        self.glob = ctx.merge_shards(shards, self.glob, self.T)
        return self.glob, int(cnt[:, 0].sum())


def gather_records(parts: dict, device, group=None) -> dict:
    """All-gather variable-length 1-D tensors (the same keys and dtypes on every rank): one
    counts all-gather (one host sync) and one all-gather of a packed byte buffer padded to the
    largest rank; returns, per key, the concatenation over the ranks in rank order."""
    world = dist.get_world_size(group)
    keys = sorted(parts)
    K = len(keys)
    cl = torch.tensor([int(parts[k].numel()) for k in keys], dtype=torch.int64, device=device)
    ca = torch.empty(world * K, dtype=torch.int64, device=device)
    dist.all_gather_into_tensor(ca, cl, group=group)
    counts = ca.view(world, K).cpu().numpy()                       # the one host sync
    isz = [parts[k].element_size() for k in keys]
    def lay(r):
        offs, off = [], 0
        for q in range(K):
            offs.append(off)
            off += (int(counts[r, q]) * isz[q] + 15) // 16 * 16
        return offs, off
    lays = [lay(r) for r in range(world)]
    maxb = max(max(b for _, b in lays), 16)
    rank = dist.get_rank(group)
    buf = torch.zeros(maxb, dtype=torch.uint8, device=device)
    for q, k in enumerate(keys):
        nb = int(counts[rank, q]) * isz[q]
        if nb:
            buf[lays[rank][0][q]:lays[rank][0][q] + nb] = parts[k].contiguous().view(torch.uint8)
    big = torch.empty(world * maxb, dtype=torch.uint8, device=device)
    dist.all_gather_into_tensor(big, buf, group=group)
    out = {}
    for q, k in enumerate(keys):
        segs = []
        for r in range(world):
            o = r * maxb + lays[r][0][q]
            segs.append(big[o:o + int(counts[r, q]) * isz[q]].view(parts[k].dtype))
        out[k] = torch.cat(segs)
    return out


def cc_sharded(ctx, group=None) -> dict:
    """CC numbers of every RPC and RPF of a tet-sharded job (DESIGN.md §10
    "CC numbers of a sharded job"): the ranks' piece / radical-facet counts all-gathered into
    global id bases, each rank's local union-find and shard-boundary records (rpd_cc_shard),
    the records all-gathered (one packed all-gather), the global union-find and this rank's
    counts (rpd_cc_merge), summed by one all-reduce.  Returns rpc_cc [N], rpf_cc [E] (int32
    CUDA tensors, identical on every rank)."""
    world, rank = dist.get_world_size(group), dist.get_rank(group)
    dev = torch.device("cuda", ctx.device)
    npc, nrf, N, E = ctx.euler_sizes()
    sz = torch.empty(world * 2, dtype=torch.int64, device=dev)
    dist.all_gather_into_tensor(sz, torch.tensor([npc, nrf], dtype=torch.int64, device=dev),
                                group=group)
    sz = sz.view(world, 2).cpu().numpy()
    base_c, base_f = int(sz[:rank, 0].sum()), int(sz[:rank, 1].sum())
    rec = ctx.cc_shard(base_c, base_f)
    allrec = gather_records({k: rec[k] for k in ("key_c", "lab_c", "key_f", "j_f", "lab_f")},
                            dev, group)
    counts = ctx.cc_merge(allrec, int(sz[:, 0].sum()), int(sz[:, 1].sum()))
    dist.all_reduce(counts, op=dist.ReduceOp.SUM, group=group)
    return {"rpc_cc": counts[:N], "rpf_cc": counts[N:N + E]}


def rpe_sharded(ctx, group=None) -> dict:
    """Restricted power edges of a tet-sharded job: every (i, j, k)
    with its Euler characteristic (numerator over 2) and CC number over the whole mesh.  The
    ranks' n_rpe give global id bases; each rank's per-key Euler numerators and shard-boundary
    records (rpd_rpe_shard) are all-gathered (one packed all-gather each); the Euler numerators
    and the ranks' component counts (rpd_rpe_merge over all records) are summed per key
    (rpd_reduce_by_key).  Returns tri [n][3], tri_euler [n], tri_cc [n] (CUDA tensors, keys
    ascending, identical on every rank)."""
    world, rank = dist.get_world_size(group), dist.get_rank(group)
    dev = torch.device("cuda", ctx.device)
    rec = ctx.rpe_shard(0)  # (sizes first; the base is applied by a second call below)
    n = torch.tensor([rec["n_rpe"]], dtype=torch.int64, device=dev)
    alln = torch.empty(world, dtype=torch.int64, device=dev)
    dist.all_gather_into_tensor(alln, n, group=group)
    alln = alln.cpu().numpy()
    base = int(alln[:rank].sum())
    if base:
        rec = ctx.rpe_shard(base)
    eu = gather_records({"k": rec["tri_key"], "v": rec["tri_euler"]}, dev, group)
    keys, euler = ctx.reduce_by_key(eu["k"], eu["v"])
    allb = gather_records({k: rec[k] for k in ("key_b", "jk_b", "lab_b")}, dev, group)
    ck, cv = ctx.rpe_merge(allb, int(alln.sum()))
    cc = gather_records({"k": ck.clone(), "v": cv.clone()}, dev, group)
    ckeys, counts = ctx.reduce_by_key(cc["k"], cc["v"])
    assert torch.equal(ckeys, keys), "every (i, j, k) has one component root"
    tri = torch.stack([keys >> 42, (keys >> 21) & 0x1FFFFF, keys & 0x1FFFFF], 1).to(torch.int32)
    return {"tri": tri, "tri_euler": euler, "tri_cc": counts}


def medial_mesh_sharded(ctx, group=None) -> dict:
    """The dual medial mesh of a tet-sharded job: every rank's edges and
    triangles (rpd_medial_mesh over its tets) as keys, all-gathered (one packed all-gather) and
    deduplicated by the library (rpd_reduce_by_key).  Returns edges [n, 2], faces [n, 3]
    (int32 CUDA tensors, ascending, identical on every rank)."""
    dev = torch.device("cuda", ctx.device)
    mm = ctx.medial_mesh(device=True)
    e, f = mm["edges"].to(torch.int64), mm["faces"].to(torch.int64)
    parts = {"e": (e[:, 0] << 21) | e[:, 1], "f": (f[:, 0] << 42) | (f[:, 1] << 21) | f[:, 2]}
    allk = gather_records(parts, dev, group)
    ek, _ = ctx.reduce_by_key(allk["e"], torch.zeros_like(allk["e"]))
    fk, _ = ctx.reduce_by_key(allk["f"], torch.zeros_like(allk["f"]))
    edges = torch.stack([ek >> 21, ek & 0x1FFFFF], 1).to(torch.int32)
    faces = torch.stack([fk >> 42, (fk >> 21) & 0x1FFFFF, fk & 0x1FFFFF], 1).to(torch.int32)
    return {"edges": edges, "faces": faces}


def sphere_volumes(ctx, group=None):
    """Per-sphere RPC volume of the whole job (SURVEY.md §8(e) validation aggregate): every
    rank's vector (rpd_sphere_volumes over its tets) summed by one all-reduce."""
    v = ctx.sphere_volumes(device=True)
    dist.all_reduce(v, op=dist.ReduceOp.SUM, group=group)
    return v


def allreduce_euler(local: dict, ctx, group=None) -> dict:
    """Per-sphere fractional Euler sums of the whole job (SURVEY.md §8(e) "validation
    aggregates"): every rank's exact accumulator rows rpc_acc [N, 1+P] and rpf_acc [E, 1+P]
    (integer part + one residue per prime, identical layouts on all ranks because the payloads
    are built from the whole mesh) are summed by one all-reduce each, then finalised by the
    library (rpd_euler_finalize).  Integer sums: exact and order-independent."""
    out = dict(local)
    for k in ("rpc", "rpf"):
        acc = local[k + "_acc"].to(torch.int64).clone()
        dist.all_reduce(acc, op=dist.ReduceOp.SUM, group=group)
        out[k + "_acc"] = acc
        if ctx is not None:
            out[k + "_sum"], out[k + "_exact"], out[k + "_value"] = ctx.euler_finalize(acc)
    return out


# ------------------------------------------------------------------ launcher


def free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def launch_ranks(n: int, script: str, argv) -> int:
    """Run ``script argv`` as n ranks of one node through torch.distributed.run (rendezvous on
    127.0.0.1); returns the launcher's exit code.  Rank 0's stdout passes through."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={n}", "--master-addr=127.0.0.1", f"--master-port={free_port()}",
           script, *argv]
    env = dict(os.environ)
    env.setdefault("OMP_NUM_THREADS", "1")
    return subprocess.call(cmd, env=env)
