"""Development aid: rpd_neighbors at a config with the heavy-row hand-off threshold of
RPD_NB_HEAVY; prints the rows computed on blocks (run under ncu for the pass-1 / heavy-kernel
split)."""
import os
import sys

import torch

sys.path.insert(0, ".")
import paper_2403_18761_b200 as P  # noqa: E402
import rpd_workloads as W  # noqa: E402

w = W.make_config(sys.argv[1] if len(sys.argv) > 1 else "C3")
ctx = P.RPDContext(0, filter_mode="pruned")
sp = torch.tensor(w.spheres, device="cuda")
for _ in range(2):
    g = ctx.neighbors(sp, W.mesh_box(w.verts), device=True)
print("RPD_NB_HEAVY", os.environ.get("RPD_NB_HEAVY"), "rows on blocks", g["n_rows_block"],
      "of", w.N, "E", int(g["nbr_off"][-1]))
