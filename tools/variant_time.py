"""Build librpd variants with extra nvcc flags and time relations+clip on a config.
usage: python tools/variant_time.py CONFIG MODE tag1:"-DFOO=1" tag2:"..." ..."""
import sys, os, importlib
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import rpd_workloads as W
cfg, mode = sys.argv[1], sys.argv[2]
w = W.make_config(cfg)
args = None
for spec in sys.argv[3:]:
    tag, flags = spec.split(":", 1)
    import paper_2403_18761_b200._build as B
    import paper_2403_18761_b200.rpd as R
    B = importlib.reload(B)
    B.NVCC_FLAGS += flags.split()
    B.LIB = B.LIB.replace("librpd.so", f"librpd_{tag}.so")
    B.build(force=True)
    R._lib = None
    R.load_library(B.LIB)
    ctx = R.RPDContext(0, filter_mode=mode)
    ctx.set_profile(True)
    if args is None:
        args = [torch.as_tensor(np.asarray(a)).cuda() for a in (w.verts, w.tets, w.spheres, w.nbr_off, w.nbr_idx)]
    fs, cs = [], []
    for it in range(5):
        ctx.relations(*args); ctx.clip()
        st = ctx.stats()
        fs.append(st["filter_ms"]); cs.append(st["clip_ms"])
    print(f"{tag:12s} filter {np.median(fs[1:]):.3f} ms  clip {np.median(cs[1:]):.3f} ms  n_cand {st['n_cand']} pieces {st['n_pieces']}", flush=True)
    ctx.close()
