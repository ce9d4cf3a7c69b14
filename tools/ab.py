"""A/B timing of librpd build variants (development aid; bench.py is the contract).

usage: python tools/ab.py CONFIG tag1:"-DFOO=1" tag2:"..." tag3:@path/to/librpd.so ...
Builds each variant (extra nvcc flags), runs full RPD (relations + clip) 5x and, when the
config has partial batches, the partial updates; prints median filter / clip / full ms, mean
partial ms, and whether the outputs are byte-identical to the first variant's.
"""
import importlib
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import rpd_workloads as W

cfg = sys.argv[1]
w = W.make_config(cfg)
dev = torch.device("cuda", 0)
to = lambda a: torch.as_tensor(np.ascontiguousarray(a)).to(dev)
base = [to(a) for a in (w.verts, w.tets, w.spheres, w.nbr_off, w.nbr_idx)]
bat = []
n_prev = w.N
for (s, o, i) in getattr(w, "batches", []) or []:
    bat.append((to(s), to(o), to(i), to(np.arange(n_prev, len(s), dtype=np.int32))))
    n_prev = len(s)
ref_full = ref_part = None
KEYS = ("piece_off", "piece_sphere", "piece_vol", "piece_m1", "piece_facemask", "inc_off",
        "inc_sphere")
for spec in sys.argv[2:]:
    tag, flags = spec.split(":", 1)
    import paper_2403_18761_b200._build as B
    import paper_2403_18761_b200.rpd as R
    B = importlib.reload(B)
    if flags.startswith("@"):   # a prebuilt library (e.g. of another commit)
        B.LIB = flags[1:]
    else:
        B.NVCC_FLAGS += flags.split()
        B.LIB = B.LIB.replace("librpd.so", f"librpd_{tag}.so")
        B.build(force=True)
    R._lib = None
    R.load_library(B.LIB)
    ctx = R.RPDContext(0, filter_mode="pruned")
    ctx.set_profile(True)
    fs, cs, tot, parts = [], [], [], []
    for it in range(6):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        ctx.relations(*base)
        ctx.clip()
        e1.record()
        torch.cuda.synchronize()
        st = ctx.stats()
        if it:
            fs.append(st["filter_ms"]); cs.append(st["clip_ms"]); tot.append(e0.elapsed_time(e1))
    full = ctx.download_pieces()
    for b in bat:
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        ctx.update_partial(*b)
        e1.record()
        torch.cuda.synchronize()
        parts.append(e0.elapsed_time(e1))
    for rnd in range(2 if bat else 0):   # later rounds (the first allocates / captures)
        parts = []
        ctx.relations(*base)
        ctx.clip()
        for b in bat:
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            ctx.update_partial(*b)
            e1.record()
            torch.cuda.synchronize()
            parts.append(e0.elapsed_time(e1))
    part = ctx.download_pieces() if bat else None
    same = "ref"
    if ref_full is None:
        ref_full, ref_part = full, part
    else:
        bad = [k for k in KEYS if not np.array_equal(np.asarray(full[k]), np.asarray(ref_full[k]))]
        if part is not None:
            bad += ["partial:" + k for k in KEYS
                    if not np.array_equal(np.asarray(part[k]), np.asarray(ref_part[k]))]
        same = "SAME" if not bad else "DIFF " + ",".join(bad)
    ps = f" partial {np.median(parts):.3f} ms (median)" if parts else ""
    print(f"{tag:12s} filter {np.median(fs):.3f} clip {np.median(cs):.3f} full {np.median(tot):.3f} ms"
          f"{ps}  pieces {len(full['piece_vol'])}  {same}", flush=True)
    ctx.close()
