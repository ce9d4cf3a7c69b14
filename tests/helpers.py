"""Shared test helpers: comparing RPD results element by element (no method arithmetic)."""
import numpy as np


def tet_volumes(verts, tets):
    P = np.asarray(verts)[np.asarray(tets)]
    a, b, c = P[:, 1] - P[:, 0], P[:, 2] - P[:, 0], P[:, 3] - P[:, 0]
    return np.einsum("ij,ij->i", a, np.cross(b, c)) / 6.0


def tet_diams(verts, tets):
    P = np.asarray(verts)[np.asarray(tets)]
    d = 0
    for a in range(4):
        for b in range(a + 1, 4):
            d = np.maximum(d, np.linalg.norm(P[:, a] - P[:, b], axis=1))
    return d


def piece_tet(res):
    """tet index (local) of every piece"""
    po = np.asarray(res["piece_off"])
    return np.repeat(np.arange(len(po) - 1), np.diff(po))


def compare_results(a, b, verts, tets, tet_ids=None, rel=1e-9, check_cands=True, label=""):
    """Parity bar: candidate CSR, piece set, facemask and incidence CSR
    bit-exact; |dvol| <= rel*vol(t); |dm1| <= rel*vol(t)*diam(t).  Returns a list of
    human-readable mismatches (empty = pass)."""
    errs = []
    ids = np.arange(len(tets)) if tet_ids is None else np.asarray(tet_ids)
    vt = tet_volumes(verts, np.asarray(tets)[ids])
    dt = tet_diams(verts, np.asarray(tets)[ids])
    if check_cands:
        for k in ("cand_off", "cand_idx"):
            if not np.array_equal(np.asarray(a[k]), np.asarray(b[k])):
                errs.append(f"{label}{k} differs")
    for k in ("piece_off", "piece_sphere", "piece_facemask", "inc_off", "inc_sphere"):
        x, y = np.asarray(a[k]), np.asarray(b[k])
        if x.shape != y.shape or not np.array_equal(x, y):
            if x.shape == y.shape:
                bad = np.nonzero(x != y)[0][:5]
                errs.append(f"{label}{k} differs at {bad.tolist()}")
            else:
                errs.append(f"{label}{k} shape {x.shape} vs {y.shape}")
    if errs:
        return errs
    pt = piece_tet(a)
    dv = np.abs(np.asarray(a["piece_vol"]) - np.asarray(b["piece_vol"]))
    if len(dv) and np.any(dv > rel * vt[pt]):
        k = int(np.argmax(dv / (rel * vt[pt])))
        errs.append(f"{label}vol piece {k}: {a['piece_vol'][k]} vs {b['piece_vol'][k]}")
    dm = np.linalg.norm(np.asarray(a["piece_m1"]) - np.asarray(b["piece_m1"]), axis=1)
    if len(dm) and np.any(dm > rel * vt[pt] * dt[pt]):
        k = int(np.argmax(dm / (rel * vt[pt] * dt[pt])))
        errs.append(f"{label}m1 piece {k}: {a['piece_m1'][k]} vs {b['piece_m1'][k]}")
    return errs


def slice_tets(res, ids):
    """Sub-result of the tets ``ids`` (CSR slicing with numpy)."""
    ids = np.asarray(ids)
    co, po, io = (np.asarray(res[k]) for k in ("cand_off", "piece_off", "inc_off"))
    out = {}
    cs = [np.arange(co[t], co[t + 1]) for t in ids]
    ps = [np.arange(po[t], po[t + 1]) for t in ids]
    cidx = np.concatenate(cs) if cs else np.zeros(0, int)
    pidx = np.concatenate(ps) if ps else np.zeros(0, int)
    out["cand_off"] = np.r_[0, np.cumsum([len(c) for c in cs])].astype(np.int32)
    out["cand_idx"] = np.asarray(res["cand_idx"])[cidx]
    out["piece_off"] = np.r_[0, np.cumsum([len(p) for p in ps])].astype(np.int32)
    for k in ("piece_sphere", "piece_vol", "piece_m1", "piece_facemask"):
        out[k] = np.asarray(res[k])[pidx]
    incs = [np.arange(io[p], io[p + 1]) for p in pidx]
    out["inc_off"] = np.r_[0, np.cumsum([len(x) for x in incs])].astype(np.int32)
    out["inc_sphere"] = np.asarray(res["inc_sphere"])[np.concatenate(incs) if incs else
                                                      np.zeros(0, int)]
    return out


def piece_dens(res):
    """Per-piece Euler denominators (library: piece_denom; oracle: piece_euler_den)."""
    return np.asarray(res["piece_denom"] if "piece_denom" in res else res["piece_euler_den"])


def slice_euler(res, piece_ids):
    """Euler arrays of the pieces ``piece_ids`` (per-piece value and radical-facet CSR)."""
    ro = np.asarray(res["rpf_off"])
    rs = [np.arange(ro[p], ro[p + 1]) for p in piece_ids]
    ridx = np.concatenate(rs) if rs else np.zeros(0, int)
    pid = np.asarray(piece_ids, int)
    return {"piece_euler": np.asarray(res["piece_euler"])[pid],
            "piece_euler_den": piece_dens(res)[pid],
            "rpf_off": np.r_[0, np.cumsum([len(r) for r in rs])].astype(np.int32),
            "rpf_sphere": np.asarray(res["rpf_sphere"])[ridx],
            "rpf_euler": np.asarray(res["rpf_euler"])[ridx]}


def compare_euler(a, b):
    """Exact comparison of two Euler results: every piece value and radical-facet value
    num / den (each over its piece's denominator) compared as rationals, x_a / L_a == x_b / L_b
    <=> x_a L_b == x_b L_a (Python integers)."""
    errs = []
    for k in ("rpf_off", "rpf_sphere"):
        if not np.array_equal(np.asarray(a[k]), np.asarray(b[k])):
            errs.append(f"{k} differs")
            return errs
    da, db = piece_dens(a).tolist(), piece_dens(b).tolist()
    if len(da) != len(db):
        return [f"piece counts {len(da)} vs {len(db)}"]
    nr = np.diff(np.asarray(a["rpf_off"]))
    ra, rb = np.repeat(da, nr).tolist(), np.repeat(db, nr).tolist()
    for k, (La, Lb) in (("piece_euler", (da, db)), ("rpf_euler", (ra, rb))):
        x = [int(v) * int(L) for v, L in zip(np.asarray(a[k]).tolist(), Lb)]
        y = [int(v) * int(L) for v, L in zip(np.asarray(b[k]).tolist(), La)]
        bad = [i for i in range(len(x)) if x[i] != y[i]]
        if len(x) != len(y) or bad:
            errs.append(f"{k}: {len(bad)} of {len(x)} differ (first {bad[:3]})")
    return errs
