"""NEXT-3 timing: rpd_neighbors at C3 / C5 (device inputs, host-timed around the call, which
syncs), list sizes against the regular-triangulation lists, and the full RPD (relations +
clip) with either list set."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2403_18761_b200 as P  # noqa: E402
import rpd_workloads as W  # noqa: E402


def main():
    P.build()
    ctx = P.RPDContext(0, filter_mode="pruned")
    for name in sys.argv[1:] or ["C3", "C5"]:
        w = W.make_config(name)
        box = W.mesh_box(w.verts)
        sp = torch.tensor(w.spheres, device="cuda")
        for _ in range(3):
            g = ctx.neighbors(sp, box, device=True)
        ts = []
        for _ in range(10):
            torch.cuda.synchronize()
            t = time.perf_counter()
            g = ctx.neighbors(sp, box, device=True)
            torch.cuda.synchronize()
            ts.append((time.perf_counter() - t) * 1e3)
        E = int(g["nbr_idx"].numel())
        dv = {k: torch.tensor(getattr(w, k), device="cuda") for k in ("verts", "tets", "nbr_off", "nbr_idx")}

        def full(off, idx):
            for _ in range(2):
                ctx.relations(dv["verts"], dv["tets"], sp, off, idx)
                ctx.clip()
            torch.cuda.synchronize()
            t = time.perf_counter()
            ctx.relations(dv["verts"], dv["tets"], sp, off, idx)
            c = ctx.clip()
            torch.cuda.synchronize()
            return (time.perf_counter() - t) * 1e3, c.n_pieces

        t_rt, np_rt = full(dv["nbr_off"], dv["nbr_idx"])
        t_nb, np_nb = full(g["nbr_off"], g["nbr_idx"])
        print(f"{name}: N={w.N} neighbors median {np.median(ts):.3f} ms min {min(ts):.3f} ms; "
              f"E_gpu={E} E_rt={len(w.nbr_idx)} hidden={g['n_hidden']} "
              f"vover={g['n_vertex_overflow']}; full RPD rt {t_rt:.3f} ms ({np_rt} pieces) "
              f"gpu-lists {t_nb:.3f} ms ({np_nb} pieces)", flush=True)


if __name__ == "__main__":
    main()
