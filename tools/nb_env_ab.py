"""A/B of a neighbour-kernel knob read per rpd_neighbors call.  Usage:
    nb_env_ab.py [VAR[=v0,v1,...]] C3 C5        (default RPD_NB_SEQ=0,1)
Times (interleaved, median of 5), list sizes, whether each variant's CSR equals the first
variant's and, where rows differ, in how many rows the variant's row is a subset."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2403_18761_b200 as P  # noqa: E402
import rpd_workloads as W  # noqa: E402


def run(ctx, sp, box, var, val):
    os.environ[var] = str(val)
    torch.cuda.synchronize()
    t = time.perf_counter()
    g = ctx.neighbors(sp, box, device=True)
    torch.cuda.synchronize()
    return (time.perf_counter() - t) * 1e3, g


def main():
    args = sys.argv[1:]
    var, vals = "RPD_NB_SEQ", ["0", "1"]
    if args and args[0].startswith("RPD_"):
        spec = args.pop(0)
        var, _, v = spec.partition("=")
        if v:
            vals = v.split(",")
    P.build()
    ctx = P.RPDContext(0, filter_mode="pruned")
    for name in args or ["C3", "C5"]:
        w = W.make_config(name)
        box = W.mesh_box(w.verts)
        sp = torch.tensor(w.spheres, device="cuda")
        ts = {v: [] for v in vals}
        gs = {}
        for rep in range(6):
            for v in vals:
                t, g = run(ctx, sp, box, var, v)
                if rep >= 1:
                    ts[v].append(t)
                gs[v] = {k: g[k].cpu().numpy().copy() for k in ("nbr_off", "nbr_idx")}
        ref = gs[vals[0]]
        for v in vals:
            same = all(np.array_equal(ref[k], gs[v][k]) for k in ("nbr_off", "nbr_idx"))
            r0, r1 = np.diff(ref["nbr_off"]), np.diff(gs[v]["nbr_off"])
            n_sub = 0
            for i in np.nonzero(r0 != r1)[0][:2000]:
                a = set(ref["nbr_idx"][ref["nbr_off"][i]:ref["nbr_off"][i + 1]].tolist())
                b = set(gs[v]["nbr_idx"][gs[v]["nbr_off"][i]:gs[v]["nbr_off"][i + 1]].tolist())
                n_sub += b <= a
            print(f"{name}: {var}={v} median {np.median(ts[v]):.3f} ms; E {len(gs[v]['nbr_idx'])};"
                  f" CSR equal to {var}={vals[0]}: {same}; rows differing {(r0 != r1).sum()}"
                  f" (subset in {n_sub})", flush=True)


if __name__ == "__main__":
    main()
