"""Algorithmic work of the bench step counted by the ORACLE: the literal
Alg. 1 vertex tests and the clip's vertex-plane tests, constructions and fan triangles of the
C3 full RPD and of the dirty tets of each C4 partial update (oracle.partial_update's re-clip).
Calls only oracle/ and the seeded generator; writes profiles/oracle_work.json, which bench.py
reads for the roofline's algorithmic flops:
    filter: 7 flop per vertex test (3 FMA + compare)
    clip:   6 per vertex-plane test + 40 per vertex construction + 30 per fan triangle
Usage: python tools/oracle_work.py [--config C4]"""
import argparse
import json
import os
import platform
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import oracle  # noqa: E402
import rpd_workloads as W  # noqa: E402

KEYS = ("n_rel_tests", "n_clip_tests", "n_constructions", "n_fan_triangles", "n_zero_hits")


def flops(st):
    return {"filter_flops": 7 * st["n_rel_tests"],
            "clip_flops": 6 * st["n_clip_tests"] + 40 * st["n_constructions"] +
            30 * st["n_fan_triangles"]}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C4")
    a = ap.parse_args()
    w = W.make_config(a.config)
    t0 = time.time()
    r = oracle.rpd_workload(w)
    full = {k: r["stats"][k] for k in KEYS}
    full.update(n_cand=int(len(r["cand_idx"])), n_pieces=int(len(r["piece_vol"])),
                T=int(w.T), N=int(w.N), **flops(full))
    parts = []
    n_old = w.N
    for (sph, off, idx) in w.batches:
        # the re-clip of the dirty tets, exactly as oracle.partial_update computes it
        R = oracle.relation_matrix(w.verts, w.tets, sph, off, idx, sphere_lo=n_old,
                                   sphere_hi=len(sph))
        dirty = np.nonzero(R.any(1))[0].astype(np.int32)
        rd = oracle.rpd(w.verts, w.tets, sph, off, idx, tet_ids=dirty)
        st = {k: rd["stats"][k] for k in KEYS}
        st.update(n_dirty=int(len(dirty)), n_cand=int(len(rd["cand_idx"])), **flops(st))
        parts.append(st)
        n_old = len(sph)
    out = {"config": a.config, "full": full, "partial": parts,
           "partial_total": {k: int(sum(p[k] for p in parts)) for k in parts[0]},
           "how": "tools/oracle_work.py (oracle counters; SURVEY.md §8(d) per-op constants)",
           "oracle_seconds": round(time.time() - t0, 1), "host": platform.processor() or
           platform.machine()}
    os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
    with open(os.path.join(ROOT, "profiles", "oracle_work.json"), "w") as f:
        json.dump(out, f, indent=1)
    print(json.dumps(out["full"]), json.dumps(out["partial_total"]))


if __name__ == "__main__":
    main()
