"""Time relations + clip of prebuilt librpd variants on one config, in one process.
usage: python tools/lib_time.py CONFIG MODE path/to/libA.so path/to/libB.so ...  (repeats twice)"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import rpd_workloads as W
import paper_2403_18761_b200.rpd as R
cfg, mode, libs = sys.argv[1], sys.argv[2], sys.argv[3:]
w = W.make_config(cfg)
args = [torch.as_tensor(np.asarray(a)).cuda() for a in (w.verts, w.tets, w.spheres, w.nbr_off, w.nbr_idx)]
for rep in range(2):
    for lib in libs:
        R._lib = None
        R.load_library(lib)
        ctx = R.RPDContext(0, filter_mode=mode)
        ctx.set_profile(True)
        fs, cs = [], []
        for it in range(6):
            ctx.relations(*args); ctx.clip()
            st = ctx.stats()
            fs.append(st["filter_ms"]); cs.append(st["clip_ms"])
        print(f"{os.path.basename(lib):22s} filter {np.median(fs[1:]):.3f} ms  clip {np.median(cs[1:]):.3f} ms"
              f"  pieces {st['n_pieces']} inc {st['n_inc']}", flush=True)
        ctx.close()
