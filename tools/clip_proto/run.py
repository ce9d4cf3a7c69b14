"""Per-thread clip prototype vs the library's lane-group clip on the C3 candidate pairs
(measurement only; see proto.cu).  Prints the volume agreement and the kernel times."""
import ctypes as C, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch
import paper_2403_18761_b200 as P
import rpd_workloads as W
cfg = sys.argv[1] if len(sys.argv) > 1 else "C3"
w = W.make_config(cfg)
dev = torch.device("cuda", 0)
to = lambda a: torch.as_tensor(np.ascontiguousarray(a)).to(dev)
ctx = P.RPDContext(0, filter_mode="pruned")
ctx.set_profile(True)
ctx.relations(to(w.verts), to(w.tets), to(w.spheres), to(w.nbr_off), to(w.nbr_idx))
clip_ms = []
for r in range(5):
    ctx.relations(to(w.verts), to(w.tets), to(w.spheres), to(w.nbr_off), to(w.nbr_idx))
    ctx.clip()
    clip_ms.append(ctx.stats()["clip_ms"])
cands = ctx.download_cands()
pcs = ctx.download_pieces()
off, idx = cands["cand_off"], cands["cand_idx"]
n = len(idx)
pair_tet = np.repeat(np.arange(w.T, dtype=np.int32), np.diff(off))
# rows sorted ascending like the library's staging
roff, ridx = w.nbr_off, w.nbr_idx.copy()
for i in range(w.N):
    ridx[roff[i]:roff[i + 1]].sort()
L = C.CDLL(os.path.join(os.path.dirname(os.path.abspath(__file__)),
                        sys.argv[2] if len(sys.argv) > 2 else "libproto.so"))
d = {k: to(v) for k, v in dict(pt=pair_tet, ci=idx, verts=w.verts, tets=w.tets, sph=w.spheres,
                                off=roff, idx=ridx).items()}
vol = torch.empty(n, dtype=torch.float64, device=dev)
ov = torch.zeros(1, dtype=torch.int32, device=dev)
ms = C.c_float()
p_ = lambda t: C.c_void_p(t.data_ptr())
times = []
for r in range(5):
    st = L.proto_clip(C.c_int64(n), p_(d["pt"]), p_(d["ci"]), p_(d["verts"]), p_(d["tets"]),
                      p_(d["sph"]), p_(d["off"]), p_(d["idx"]), p_(vol), p_(ov), C.byref(ms))
    assert st == 0, st
    times.append(ms.value)
v = vol.cpu().numpy()
# library volumes per pair (0 for empty pairs): pieces keyed (tet, sphere) like the pairs
lib = np.zeros(n)
poff, ps, pv = pcs["piece_off"], pcs["piece_sphere"], pcs["piece_vol"]
ptet = np.repeat(np.arange(w.T, dtype=np.int64), np.diff(poff))
pair_key = pair_tet.astype(np.int64) * w.N + idx
lib[np.searchsorted(pair_key, ptet * w.N + ps)] = pv
ok = v >= 0
Vt = w.verts[w.tets]
tv = np.abs(np.linalg.det(np.stack([Vt[:, k] - Vt[:, 0] for k in (1, 2, 3)], axis=1))) / 6
rel = np.abs(v[ok] - lib[ok]) / tv[pair_tet[ok]]
print(f"{cfg}: pairs {n}, overflow {int(ov.item())}, max |dvol|/vol(t) {rel.max():.2e}, "
      f"p99.9 {np.quantile(rel, 0.999):.2e}")
print(f"library clip (all tiers, volume + m1 + incidences + facemasks, exact predicates) "
      f"median {np.median(clip_ms):.3f} ms; per-thread prototype (volume only, fp64) median "
      f"{np.median(times):.3f} ms  {times}")
