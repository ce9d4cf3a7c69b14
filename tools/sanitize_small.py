"""Small end-to-end run for compute-sanitizer (memcheck / racecheck / synccheck / initcheck):
the hot path (both filters, all clip tiers, partial updates) and the widened rows (Euler and
topology flags, CC numbers, medial mesh, envelope distance, gather kernels)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2403_18761_b200 as P
import rpd_workloads as W
for mode in ("all_pairs", "pruned"):
    ctx = P.RPDContext(0, filter_mode=mode)
    for w in (W.make_c1(0), W.make_c1(1, degenerate=True),
              W.make_shape_workload("S", 2000, 150, seed=3, n_batches=2, batch_m=12, clusters=3,
                                    cache=False)):
        for wide, euler, tiers in ((False, False, False), (True, False, False),
                                   (False, True, False), (False, True, True)):
            ctx.set_clip_wide(wide)
            ctx.set_clip_tiers(tiers)
            ctx.set_euler(w.tets if euler else None, len(w.verts))
            ctx.relations(w.verts, w.tets, w.spheres, w.nbr_off, w.nbr_idx)
            ctx.clip()
            n_old = w.N
            for (s, o, i) in w.batches:
                ctx.update_partial(s, o, i, np.arange(n_old, len(s), dtype=np.int32))
                n_old = len(s)
            ctx.download_pieces()
            ctx.download_cands()
            if ctx.n_dirty if hasattr(ctx, "n_dirty") else 0:
                ctx.download_tets(ctx.dirty_ptr(), ctx.n_dirty, {})
            if euler:
                ctx.download_euler()
                ctx.download_topology()
                ctx.rpe()
                mm = ctx.medial_mesh()
                smp = W.boundary_samples(w.verts, w.tets, 200, seed=1)
                sph = w.batches[-1][0] if w.batches else w.spheres
                ctx.envelope(smp, sph, mm["edges"], mm["faces"])
        ctx.set_euler(None, 0)
    # gather kernels: two shards of the last workload
    from paper_2403_18761_b200.dist import shard_tets
    shards, ids = [], []
    for r in range(2):
        tid = shard_tets(w.T, 2, r, 256)
        ctx.relations(w.verts, w.tets[tid], w.spheres, w.nbr_off, w.nbr_idx)
        ctx.clip()
        shards.append({k: v.clone() for k, v in ctx.download_pieces(device=True).items()})
        ids.append(torch.as_tensor(tid, device="cuda"))
    ctx.gather_pieces(shards, ids, w.T)
    # the 256-slot slow path: one tet, a sphere inside a shell of 100 spheres
    from tests.test_gpu_parity import _shell_workload
    ws = _shell_workload()
    ctx.relations(ws.verts, ws.tets, ws.spheres, ws.nbr_off, ws.nbr_idx)
    ctx.clip()
    ctx.download_pieces()
    # sphere neighbours (NEXT-3) of a small set
    ctx.neighbors(w.spheres, W.mesh_box(w.verts))
    ctx.close()
print("sanitize run ok")
