"""A/B of a neighbour-kernel knob read per rpd_neighbors call (default RPD_NB_SEQ=0/1; usage:
nb_env_ab.py [VAR] C3 C5): times (interleaved), list sizes, whether the CSRs are identical and,
where rows differ, whether the variant-1 row is a subset of the variant-0 row."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2403_18761_b200 as P  # noqa: E402
import rpd_workloads as W  # noqa: E402


def run(ctx, sp, box, edge):
    os.environ[VAR] = str(edge)
    torch.cuda.synchronize()
    t = time.perf_counter()
    g = ctx.neighbors(sp, box, device=True)
    torch.cuda.synchronize()
    return (time.perf_counter() - t) * 1e3, g


VAR = "RPD_NB_SEQ"


def main():
    global VAR
    args = sys.argv[1:]
    if args and args[0].startswith("RPD_"):
        VAR = args.pop(0)
    P.build()
    ctx = P.RPDContext(0, filter_mode="pruned")
    for name in args or ["C3", "C5"]:
        w = W.make_config(name)
        box = W.mesh_box(w.verts)
        sp = torch.tensor(w.spheres, device="cuda")
        ts = {0: [], 1: []}
        gs = {}
        for rep in range(6):
            for e in (0, 1):
                t, g = run(ctx, sp, box, e)
                if rep >= 1:
                    ts[e].append(t)
                gs[e] = {k: g[k].cpu().numpy().copy() for k in ("nbr_off", "nbr_idx")}
        same = all(np.array_equal(gs[0][k], gs[1][k]) for k in ("nbr_off", "nbr_idx"))
        r0 = np.diff(gs[0]["nbr_off"])
        r1 = np.diff(gs[1]["nbr_off"])
        n_sub = 0
        for i in np.nonzero(r0 != r1)[0][:2000]:
            a = set(gs[0]["nbr_idx"][gs[0]["nbr_off"][i]:gs[0]["nbr_off"][i + 1]].tolist())
            b = set(gs[1]["nbr_idx"][gs[1]["nbr_off"][i]:gs[1]["nbr_off"][i + 1]].tolist())
            n_sub += b <= a
        print(f"{name}: {VAR}=0 median {np.median(ts[0]):.3f} ms, =1 median {np.median(ts[1]):.3f} ms;"
              f" E {len(gs[0]['nbr_idx'])} -> {len(gs[1]['nbr_idx'])}; identical CSR {same};"
              f" rows differing {(r0 != r1).sum()} (=1 row a subset in {n_sub})", flush=True)


if __name__ == "__main__":
    main()
