"""CPU oracle of the RPD hot path -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (cpu_baseline leg and
``--impl reference``) may import this package.  It shares no code with
``paper_2403_18761_b200`` (the CUDA path); the only common module is ``rpd_workloads``, the
seeded input generator, which holds none of the method's arithmetic.

``oracle.c`` is the plain C implementation (see its header for the definitions and the
PAPER.md passages they follow); this file compiles it with gcc and marshals numpy arrays.
``exact_checker.py`` is the independent brute-force rational checker that pins it.

Parity status of each function (DESIGN.md §Oracle pins):
  relation / candidate lists ... pinned (brute-force soundness, single sphere, SPEC examples)
  pieces: non-empty, facemask, incidences, vol, m1 ... pinned (exact checker, brute force,
          Kuhn closed forms, partition, Voronoi reduction, power membership)
  partial update (R11) ... pinned (partial == full recompute, M = 0 identity)
  box neighbours (NEXT-3) ... pinned (subset of the Qhull regular-triangulation edges, two-sphere
          closed form, sufficiency: same pieces as with the regular-triangulation lists)
  fractional Euler characteristics (NEXT-1) ... pinned (mesh Euler by V-E+F-T, a single
          sphere gives the mesh's Euler, explicit extraction of every RPC / RPF complex by
          exact rational vertex enumeration, RPF symmetry on generic inputs)
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lock = threading.Lock()
_lib = None


def build(force: bool = False) -> str:
    """Compile liboracle.so (gcc, -O2, OpenMP) if missing or stale."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".{os.getpid()}.tmp"
        cmd = ["gcc", "-O2", "-march=x86-64-v2", "-fopenmp", "-shared", "-fPIC", "-std=gnu11",
               "-o", tmp, _SRC, "-lm"]
        subprocess.check_call(cmd)
        os.replace(tmp, _LIB)
    return _LIB


class _Input(C.Structure):
    _fields_ = [("V", C.c_int64), ("T", C.c_int64), ("N", C.c_int64),
                ("verts", C.c_void_p), ("tets", C.c_void_p), ("spheres", C.c_void_p),
                ("nbr_off", C.c_void_p), ("nbr_idx", C.c_void_p), ("brute", C.c_int),
                ("euler", C.c_int)]


class _Result(C.Structure):
    _fields_ = [("n_tets", C.c_int64),
                ("cand_off", C.POINTER(C.c_int32)), ("cand_idx", C.POINTER(C.c_int32)),
                ("n_cand", C.c_int64),
                ("piece_off", C.POINTER(C.c_int32)), ("piece_sphere", C.POINTER(C.c_int32)),
                ("piece_vol", C.POINTER(C.c_double)), ("piece_m1", C.POINTER(C.c_double)),
                ("piece_facemask", C.POINTER(C.c_uint8)),
                ("inc_off", C.POINTER(C.c_int32)), ("inc_sphere", C.POINTER(C.c_int32)),
                ("n_pieces", C.c_int64), ("n_inc", C.c_int64),
                ("euler_denom", C.c_int64), ("piece_euler", C.POINTER(C.c_int64)),
                ("piece_euler_den", C.POINTER(C.c_int64)),
                ("rpf_off", C.POINTER(C.c_int32)), ("rpf_sphere", C.POINTER(C.c_int32)),
                ("rpf_euler", C.POINTER(C.c_int64)),
                ("piece_sosfm", C.POINTER(C.c_uint8)), ("rpf_fm", C.POINTER(C.c_uint8)),
                ("rpf_adj", C.POINTER(C.c_uint64)),
                ("n_rpf", C.c_int64),
                ("rpe_off", C.POINTER(C.c_int32)), ("rpe_j", C.POINTER(C.c_int32)),
                ("rpe_k", C.POINTER(C.c_int32)), ("rpe_euler", C.POINTER(C.c_int64)),
                ("rpe_fm", C.POINTER(C.c_uint8)), ("n_rpe", C.c_int64),
                ("n_rel_tests", C.c_int64), ("n_clip_tests", C.c_int64),
                ("n_constructions", C.c_int64), ("n_fan_triangles", C.c_int64),
                ("n_zero_hits", C.c_int64),
                ("status", C.c_int), ("err", C.c_char * 256)]


def lib():
    global _lib
    with _lock:
        if _lib is None:
            L = C.CDLL(build())
            L.oracle_rpd.restype = C.POINTER(_Result)
            L.oracle_rpd.argtypes = [C.POINTER(_Input), C.c_void_p, C.c_int64, C.c_int, C.c_int]
            L.oracle_free.argtypes = [C.POINTER(_Result)]
            L.oracle_relation_matrix.restype = C.c_int
            L.oracle_relation_matrix.argtypes = [C.POINTER(_Input), C.c_void_p, C.c_int64,
                                                 C.c_int64, C.c_int64, C.c_void_p, C.c_int]
            L.oracle_power_distance.restype = C.c_double
            L.oracle_power_distance.argtypes = [C.c_void_p, C.c_void_p]
            L.oracle_max_threads.restype = C.c_int
            L.oracle_envelope.restype = None
            L.oracle_envelope.argtypes = [C.c_void_p, C.c_int64, C.c_void_p, C.c_int64,
                                          C.c_void_p, C.c_int64, C.c_void_p, C.c_int64,
                                          C.c_void_p, C.c_void_p, C.c_int]
            L.oracle_envelope_one.restype = C.c_double
            L.oracle_envelope_one.argtypes = [C.c_void_p, C.c_void_p, C.c_int, C.c_void_p]
            _lib = L
    return _lib


class OracleError(RuntimeError):
    pass


def _prep(verts, tets, spheres, nbr_off, nbr_idx, brute, euler=False):
    keep = [np.ascontiguousarray(verts, dtype=np.float64),
            np.ascontiguousarray(tets, dtype=np.int32),
            np.ascontiguousarray(spheres, dtype=np.float64).reshape(-1, 4),
            np.ascontiguousarray(nbr_off, dtype=np.int32),
            np.ascontiguousarray(nbr_idx if len(nbr_idx) else np.zeros(1), dtype=np.int32)]
    inp = _Input(len(keep[0]), len(keep[1]), len(keep[2]), keep[0].ctypes.data,
                 keep[1].ctypes.data, keep[2].ctypes.data, keep[3].ctypes.data,
                 keep[4].ctypes.data, int(brute), int(euler))
    return inp, keep


def power_distance(sphere, x) -> float:
    """PD(m, x) = |x - theta|^2 - r^2."""
    s = np.ascontiguousarray(sphere, dtype=np.float64)
    p = np.ascontiguousarray(x, dtype=np.float64)
    return lib().oracle_power_distance(s.ctypes.data, p.ctypes.data)


def rpd(verts, tets, spheres, nbr_off, nbr_idx, tet_ids=None, brute=False, clip=True,
        nthreads=0, euler=False):
    """Oracle RPD of ``tet_ids`` (all tets when None).  Returns a dict of numpy arrays in the
    boundary's layout (cand CSR, piece CSR, incidence CSR) plus instrumentation counters.
    ``euler``: also the fractional Euler characteristics -- per piece
    ``piece_euler`` and per radical facet ``rpf_off/rpf_sphere/rpf_euler``, exact numerators
    over ``euler_denom`` (payloads from the whole mesh, even when ``tet_ids`` is a subset)."""
    inp, keep = _prep(verts, tets, spheres, nbr_off, nbr_idx, brute, euler)
    if tet_ids is None:
        ids_p, n = None, len(keep[1])
    else:
        ids = np.ascontiguousarray(tet_ids, dtype=np.int32)
        keep.append(ids)
        ids_p, n = ids.ctypes.data, len(ids)
    L = lib()
    rp = L.oracle_rpd(C.byref(inp), ids_p, n, int(clip), int(nthreads))
    try:
        r = rp.contents
        if r.status != 0:
            raise OracleError(f"oracle status {r.status}: {r.err.decode()}")

        def arr(p, n, dt):
            if n == 0:
                return np.zeros(0, dtype=dt)
            return np.ctypeslib.as_array(p, shape=(n,)).copy()
        out = {
            "cand_off": arr(r.cand_off, r.n_tets + 1, np.int32),
            "cand_idx": arr(r.cand_idx, r.n_cand, np.int32),
            "piece_off": arr(r.piece_off, r.n_tets + 1, np.int32),
            "piece_sphere": arr(r.piece_sphere, r.n_pieces, np.int32),
            "piece_vol": arr(r.piece_vol, r.n_pieces, np.float64),
            "piece_m1": arr(r.piece_m1, 3 * r.n_pieces, np.float64).reshape(-1, 3),
            "piece_facemask": arr(r.piece_facemask, r.n_pieces, np.uint8),
            "inc_off": arr(r.inc_off, r.n_pieces + 1, np.int32),
            "inc_sphere": arr(r.inc_sphere, r.n_inc, np.int32),
            "stats": {k: int(getattr(r, k)) for k in ("n_rel_tests", "n_clip_tests",
                                                      "n_constructions", "n_fan_triangles",
                                                      "n_zero_hits")},
        }
        if euler and clip:
            out.update({"euler_denom": int(r.euler_denom),
                        "piece_euler": arr(r.piece_euler, r.n_pieces, np.int64),
                        "piece_euler_den": arr(r.piece_euler_den, r.n_pieces, np.int64),
                        "rpf_off": arr(r.rpf_off, r.n_pieces + 1, np.int32),
                        "rpf_sphere": arr(r.rpf_sphere, r.n_rpf, np.int32),
                        "rpf_euler": arr(r.rpf_euler, r.n_rpf, np.int64),
                        "piece_sosfm": arr(r.piece_sosfm, r.n_pieces, np.uint8),
                        "rpf_fm": arr(r.rpf_fm, r.n_rpf, np.uint8),
                        "rpf_adj": arr(r.rpf_adj, r.n_rpf, np.uint64),
                        "rpe_off": arr(r.rpe_off, r.n_pieces + 1, np.int32),
                        "rpe_j": arr(r.rpe_j, r.n_rpe, np.int32),
                        "rpe_k": arr(r.rpe_k, r.n_rpe, np.int32),
                        "rpe_euler": arr(r.rpe_euler, r.n_rpe, np.int64),
                        "rpe_fm": arr(r.rpe_fm, r.n_rpe, np.uint8)})
    finally:
        L.oracle_free(rp)
    return out


def box_neighbours(spheres, box, nthreads=0):
    """NEXT-3 definition (DESIGN.md §10 "Sphere neighbours"): j is a box
    neighbour of i iff the radical plane h_ij holds a positive-area 2-face of C_i ∩ B, B the
    axis box ``box`` = (lo, hi).  Computed literally: B split into its 6 Kuhn tets, every piece
    P(t, i) clipped in brute-force mode (N(i) = all j != i), and the
    incidences (geometric, positive-area faces: C1 step 7) of i's pieces united.  Returns the
    CSR (off [N+1], idx ascending)."""
    import rpd_workloads as W
    sp = np.ascontiguousarray(spheres, dtype=np.float64).reshape(-1, 4)
    N = len(sp)
    bx = np.asarray(box, dtype=np.float64).reshape(6)
    bv, bt = W.box_6tets(bx[:3], bx[3:])
    z = np.zeros(N + 1, dtype=np.int32)
    r = rpd(bv, bt, sp, z, np.zeros(0, dtype=np.int32), brute=True, nthreads=nthreads)
    rows = [set() for _ in range(N)]
    for p, i in enumerate(r["piece_sphere"]):
        rows[int(i)].update(r["inc_sphere"][r["inc_off"][p]:r["inc_off"][p + 1]].tolist())
    off = np.zeros(N + 1, dtype=np.int32)
    off[1:] = np.cumsum([len(x) for x in rows])
    idx = np.array([j for x in rows for j in sorted(x)], dtype=np.int32)
    return off, idx


def relation_matrix(verts, tets, spheres, nbr_off, nbr_idx, tet_ids=None, sphere_lo=0,
                    sphere_hi=None, nthreads=0):
    """Literal Alg. 1 booleans rel(t, i) for t in tet_ids, i in [sphere_lo, sphere_hi)."""
    inp, keep = _prep(verts, tets, spheres, nbr_off, nbr_idx, False)
    N = len(keep[2])
    hi = N if sphere_hi is None else sphere_hi
    if tet_ids is None:
        ids_p, n = None, len(keep[1])
    else:
        ids = np.ascontiguousarray(tet_ids, dtype=np.int32)
        keep.append(ids)
        ids_p, n = ids.ctypes.data, len(ids)
    out = np.zeros((n, max(hi - sphere_lo, 0)), dtype=np.uint8)
    st = lib().oracle_relation_matrix(C.byref(inp), ids_p, n, sphere_lo, hi, out.ctypes.data,
                                      int(nthreads))
    if st:
        raise OracleError(f"oracle status {st}")
    return out.astype(bool)


def rpd_workload(w, **kw):
    return rpd(w.verts, w.tets, w.spheres, w.nbr_off, w.nbr_idx, **kw)


def partial_update(old, verts, tets, spheres_new, nbr_off_new, nbr_idx_new, n_old,
                   nthreads=0, euler=False):
    """Partial RPD update, reading R11: spheres [n_old, N_new) are new; dirty tets =
    {t : exists new n with rel_new(t, n)}; dirty tets get a full re-candidate + clip with the
    new neighbour lists; clean tets keep ``old``'s candidates and pieces.  Returns
    (merged result dict, dirty tet ids ascending)."""
    N_new = len(spheres_new)
    T = len(tets)
    if N_new > n_old:
        R = relation_matrix(verts, tets, spheres_new, nbr_off_new, nbr_idx_new,
                            sphere_lo=n_old, sphere_hi=N_new, nthreads=nthreads)
        dirty = np.nonzero(R.any(1))[0].astype(np.int32)
    else:
        dirty = np.zeros(0, dtype=np.int32)
    new = rpd(verts, tets, spheres_new, nbr_off_new, nbr_idx_new, tet_ids=dirty,
              nthreads=nthreads, euler=euler) if len(dirty) else None
    return merge_per_tet(old, new, dirty, T), dirty


def per_tet_lists(res, T):
    """Split a result dict into per-tet python lists (used to merge and compare)."""
    out = []
    co, ci = res["cand_off"], res["cand_idx"]
    po = res["piece_off"]
    io = res["inc_off"]
    ro = res.get("rpf_off")
    for a in range(T):
        cands = ci[co[a]:co[a + 1]].tolist()
        pcs = []
        for p in range(po[a], po[a + 1]):
            eu = None
            if ro is not None and len(ro) == len(res["piece_sphere"]) + 1:
                eo = res["rpe_off"]
                eu = ((int(res["piece_euler"][p]), int(res["piece_euler_den"][p])),
                      tuple(res["rpf_sphere"][ro[p]:ro[p + 1]].tolist()),
                      tuple(res["rpf_euler"][ro[p]:ro[p + 1]].tolist()),
                      int(res["piece_sosfm"][p]),
                      tuple(res["rpf_fm"][ro[p]:ro[p + 1]].tolist()),
                      tuple(res["rpf_adj"][ro[p]:ro[p + 1]].tolist()),
                      tuple(zip(res["rpe_j"][eo[p]:eo[p + 1]].tolist(),
                                res["rpe_k"][eo[p]:eo[p + 1]].tolist(),
                                res["rpe_euler"][eo[p]:eo[p + 1]].tolist(),
                                res["rpe_fm"][eo[p]:eo[p + 1]].tolist())))
            pcs.append((int(res["piece_sphere"][p]), float(res["piece_vol"][p]),
                        tuple(res["piece_m1"][p].tolist()), int(res["piece_facemask"][p]),
                        tuple(res["inc_sphere"][io[p]:io[p + 1]].tolist()), eu))
        out.append((cands, pcs))
    return out


def from_per_tet_lists(L):
    cand_off = [0]
    cand_idx, piece_off, ps, pv, pm, pf, inc_off, inc = [], [0], [], [], [], [], [0], []
    pe, rpf_off, rpf_j, rpf_e, sfm, rfm, radj = [], [0], [], [], [], [], []
    pden = []
    rpe_off, rpe = [0], []
    for cands, pcs in L:
        cand_idx += cands
        cand_off.append(len(cand_idx))
        for (s, v, m, f, ii, eu) in pcs:
            ps.append(s)
            pv.append(v)
            pm.append(m)
            pf.append(f)
            inc += list(ii)
            inc_off.append(len(inc))
            if eu is not None:
                pe.append(eu[0][0])
                pden.append(eu[0][1])
                rpf_j += list(eu[1])
                rpf_e += list(eu[2])
                sfm.append(eu[3])
                rfm += list(eu[4])
                radj += list(eu[5])
                rpf_off.append(len(rpf_j))
                rpe += list(eu[6])
                rpe_off.append(len(rpe))
        piece_off.append(len(ps))
    eul = {}
    if len(pe) == len(ps) and len(rpf_off) == len(ps) + 1:
        eul = {"piece_euler": np.array(pe, np.int64),
               "piece_euler_den": np.array(pden, np.int64),
               "rpf_off": np.array(rpf_off, np.int32),
               "rpf_sphere": np.array(rpf_j, np.int32), "rpf_euler": np.array(rpf_e, np.int64),
               "piece_sosfm": np.array(sfm, np.uint8), "rpf_fm": np.array(rfm, np.uint8),
               "rpf_adj": np.array(radj, np.uint64),
               "rpe_off": np.array(rpe_off, np.int32),
               "rpe_j": np.array([x[0] for x in rpe], np.int32),
               "rpe_k": np.array([x[1] for x in rpe], np.int32),
               "rpe_euler": np.array([x[2] for x in rpe], np.int64),
               "rpe_fm": np.array([x[3] for x in rpe], np.uint8)}
    return {**eul, "cand_off": np.array(cand_off, np.int32), "cand_idx": np.array(cand_idx, np.int32),
            "piece_off": np.array(piece_off, np.int32), "piece_sphere": np.array(ps, np.int32),
            "piece_vol": np.array(pv, np.float64),
            "piece_m1": np.array(pm, np.float64).reshape(-1, 3),
            "piece_facemask": np.array(pf, np.uint8), "inc_off": np.array(inc_off, np.int32),
            "inc_sphere": np.array(inc, np.int32)}


def _segments(off, sel):
    """Element indices of the CSR segments ``sel`` (in that order) of offsets ``off``."""
    off = np.asarray(off, np.int64)
    sel = np.asarray(sel, np.int64)
    lens = off[sel + 1] - off[sel]
    if lens.sum() == 0:
        return np.zeros(0, np.int64)
    first = np.repeat(off[sel] - np.concatenate(([0], np.cumsum(lens)[:-1])), lens)
    return first + np.arange(lens.sum())


def _csr_of(lens):
    return np.concatenate(([0], np.cumsum(lens))).astype(np.int32)


def merge_per_tet(old, new, dirty, T):
    """Tet t's candidates and pieces from ``new`` (row a) when t = dirty[a], else from
    ``old`` (row t) -- the R11 merge.  Plain CSR row selection; Euler results go through
    the per-tet lists."""
    if "rpf_off" not in old:
        dirty = np.asarray(dirty, np.int64)
        src_new = np.zeros(T, bool)
        src_new[dirty] = True
        row = np.arange(T, dtype=np.int64)
        row[dirty] = T + np.arange(len(dirty))       # rows T.. are new's rows
        nn = new if new is not None else {k: old[k][:0] for k in old if k != "stats"}
        if new is None:
            nn["cand_off"] = nn["piece_off"] = np.zeros(1, np.int32)
            nn["inc_off"] = np.zeros(1, np.int32)

        def cat_off(a, b):  # offsets of the concatenated segment lists a then b
            a, b = np.asarray(a, np.int64), np.asarray(b, np.int64)
            return np.concatenate((a, a[-1] + b[1:]))
        c_off = cat_off(old["cand_off"], nn["cand_off"])
        c_idx = np.concatenate((old["cand_idx"], nn["cand_idx"]))
        p_off = cat_off(old["piece_off"], nn["piece_off"])
        i_off = cat_off(old["inc_off"], nn["inc_off"])
        cs = _segments(c_off, row)
        ps = _segments(p_off, row)
        out = {"cand_off": _csr_of(c_off[row + 1] - c_off[row]),
               "cand_idx": c_idx[cs].astype(np.int32),
               "piece_off": _csr_of(p_off[row + 1] - p_off[row])}
        for k in ("piece_sphere", "piece_vol", "piece_m1", "piece_facemask"):
            out[k] = np.concatenate((old[k], nn[k]))[ps]
        out["inc_off"] = _csr_of(i_off[ps + 1] - i_off[ps])
        out["inc_sphere"] = np.concatenate((old["inc_sphere"], nn["inc_sphere"]))[
            _segments(i_off, ps)].astype(np.int32)
        return out
    L = per_tet_lists(old, T)
    if new is not None:
        Ln = per_tet_lists(new, len(dirty))
        for a, t in enumerate(dirty):
            L[t] = Ln[a]
    out = from_per_tet_lists(L)
    if "euler_denom" in old:
        out["euler_denom"] = old["euler_denom"]
        if new is not None and new.get("euler_denom", 0) != old["euler_denom"]:
            raise OracleError("partial update: Euler denominators differ")
    return out


def euler_sums(res, N, nbr_off, nbr_idx):
    """Per-sphere fractional Euler sums ("For each medial sphere, we collect
    the fractional Euler characteristics for all of its restricted elements"), as exact Python
    Fractions: rpc[i] = Euler(RPC(m_i)) = sum over the pieces of m_i; rpf[(i, j)] =
    Euler(RPF(m_i, m_j)) seen from m_i = sum over its pieces' facets on h_ij."""
    from fractions import Fraction
    rpc = [Fraction(0)] * N
    rpf = {}
    po, ro = res["piece_off"], res["rpf_off"]
    for p, i in enumerate(res["piece_sphere"].tolist()):
        L = int(res["piece_euler_den"][p])  # the piece's tet denominator L_t
        rpc[i] += Fraction(int(res["piece_euler"][p]), L)
        for r in range(ro[p], ro[p + 1]):
            key = (i, int(res["rpf_sphere"][r]))
            rpf[key] = rpf.get(key, Fraction(0)) + Fraction(int(res["rpf_euler"][r]), L)
    return rpc, rpf


def rpe_sums(res):
    """Per-sphere fractional Euler sums of the restricted power edges ("the
    fractional Euler characteristic of all restricted elements (RPCs, RPFs, RPEs)"): rpe[(i,
    j, k)] = Euler(RPE(m_i, m_j, m_k)) seen from m_i (j < k) = sum over m_i's pieces of their
    edge on h_ij and h_ik, as exact Fractions."""
    from fractions import Fraction
    eo = res["rpe_off"]
    out = {}
    for p, i in enumerate(res["piece_sphere"].tolist()):
        L = int(res["piece_euler_den"][p])
        for r in range(eo[p], eo[p + 1]):
            key = (i, int(res["rpe_j"][r]), int(res["rpe_k"][r]))
            out[key] = out.get(key, Fraction(0)) + Fraction(int(res["rpe_euler"][r]), L)
    return out


def rpe_topology(res, tets):
    """CC numbers of the restricted power edges: RPE(m_i, m_j, m_k) seen from
    m_i is the union of the edges of m_i's pieces on h_ij and h_ik; two of them in tets sharing
    face f are connected when both have an endpoint on f (a line meets the face plane once, so
    those endpoints are the same point).  Plain union-find.  Returns {(i, j, k): cc}."""
    parent = {}

    def find(x):
        while parent[x] != x:
            parent[x] = parent[parent[x]]
            x = parent[x]
        return x

    adj = face_adjacency(tets)
    po, eo = res["piece_off"], res["rpe_off"]
    ps = res["piece_sphere"].tolist()
    items = {}  # (t, i, j, k) -> endpoint tet-face mask
    for t in range(len(tets)):
        for q in range(po[t], po[t + 1]):
            for r in range(eo[q], eo[q + 1]):
                key = (t, ps[q], int(res["rpe_j"][r]), int(res["rpe_k"][r]))
                items[key] = int(res["rpe_fm"][r])
                parent[key] = key
    for (t, i, j, k), fm in items.items():
        for f in range(4):
            if not (fm >> f) & 1 or adj[t][f] is None:
                continue
            t2, f2 = adj[t][f]
            o = (t2, i, j, k)
            if o in items and (items[o] >> f2) & 1:
                ra, rb = find((t, i, j, k)), find(o)
                if ra != rb:
                    parent[max(ra, rb)] = min(ra, rb)
    cc = {}
    for x in parent:
        if find(x) == x:
            cc[x[1:]] = cc.get(x[1:], 0) + 1
    return cc


def face_adjacency(tets):
    """adj[t][k] = (t', k'): the tet sharing face k of t (face k = opposite vertex k), or None
    (boundary).  Plain dictionary of sorted vertex triples."""
    owners = {}
    for t, tv in enumerate(np.asarray(tets).tolist()):
        for k in range(4):
            owners.setdefault(tuple(sorted(tv[:k] + tv[k + 1:])), []).append((t, k))
    adj = [[None] * 4 for _ in range(len(tets))]
    for own in owners.values():
        if len(own) == 2:
            (a, ka), (b, kb) = own
            adj[a][ka] = (b, kb)
            adj[b][kb] = (a, ka)
    return adj


def topology(res, tets, N):
    """CC numbers ("trace their CC numbers using a simple traversal"):
    components of every RPC(m_i) -- the pieces of m_i, two pieces in tets sharing face f
    connected when f is a facet of both -- and of every RPF(m_i, m_j) seen from m_i -- the
    facets of m_i's pieces on h_ij, connected across a shared tet face f when both have an
    edge on f.  Elements of the symbolically perturbed pieces (R26-R27), so they
    match the Euler sums.  Plain union-find over Python objects.  Returns (rpc_cc [N],
    {(i, j): cc})."""
    parent = {}

    def find(x):
        while parent[x] != x:
            parent[x] = parent[parent[x]]
            x = parent[x]
        return x

    def union(a, b):
        ra, rb = find(a), find(b)
        if ra != rb:
            parent[max(ra, rb)] = min(ra, rb)

    adj = face_adjacency(tets)
    po, ro = res["piece_off"], res["rpf_off"]
    ps = res["piece_sphere"].tolist()
    piece_of = {}          # (t, i) -> piece index
    for t in range(len(tets)):
        for q in range(po[t], po[t + 1]):
            piece_of[(t, ps[q])] = q
            parent[("c", q)] = ("c", q)
            for r in range(ro[q], ro[q + 1]):
                parent[("f", ps[q], int(res["rpf_sphere"][r]), t)] = \
                    ("f", ps[q], int(res["rpf_sphere"][r]), t)
    for t in range(len(tets)):
        for q in range(po[t], po[t + 1]):
            i = ps[q]
            for k in range(4):
                nb = adj[t][k]
                if nb is None:
                    continue
                t2, k2 = nb
                q2 = piece_of.get((t2, i))
                if q2 is None:
                    continue
                if (res["piece_sosfm"][q] >> k) & 1 and (res["piece_sosfm"][q2] >> k2) & 1:
                    union(("c", q), ("c", q2))
                f2 = {int(res["rpf_sphere"][r]): int(res["rpf_fm"][r])
                      for r in range(ro[q2], ro[q2 + 1])}
                for r in range(ro[q], ro[q + 1]):
                    j = int(res["rpf_sphere"][r])
                    if (res["rpf_fm"][r] >> k) & 1 and j in f2 and (f2[j] >> k2) & 1:
                        union(("f", i, j, t), ("f", i, j, t2))
    rpc_cc = [0] * N
    rpf_cc = {}
    for x in parent:
        if find(x) == x:
            if x[0] == "c":
                rpc_cc[ps[x[1]]] += 1
            else:
                rpf_cc[(x[1], x[2])] = rpf_cc.get((x[1], x[2]), 0) + 1
    return rpc_cc, rpf_cc


def medial_mesh(res):
    """The dual medial mesh of the RPD: a vertex per sphere with a cell, an
    edge e_ij per restricted power face RPF(m_i, m_j) and a triangle f_ijk per restricted power
    edge RPE(m_i, m_j, m_k) -- an edge of a piece of m_i lying on the radical planes of m_j and
    m_k (symbolically perturbed pieces).  Seen from every sphere's pieces and merged: sorted
    unique (i, j) with i < j and (i, j, k) with i < j < k."""
    edges, faces = set(), set()
    ro = res["rpf_off"]
    for q, i in enumerate(res["piece_sphere"].tolist()):
        js = res["rpf_sphere"][ro[q]:ro[q + 1]].tolist()
        adj = res["rpf_adj"][ro[q]:ro[q + 1]].tolist()
        for a, j in enumerate(js):
            edges.add((min(i, j), max(i, j)))
            for b in range(a + 1, len(js)):
                if (int(adj[a]) >> b) & 1:
                    faces.add(tuple(sorted((i, j, js[b]))))
    return sorted(edges), sorted(faces)


def envelope(samples, spheres, edges, faces, nthreads=0):
    """Geometry preservation: per surface sample the minimum over the medial
    mesh's spheres, cones (edges) and slabs (faces) of min_params |p - c| - r (golden-section
    search on the convex interpolation parameters, see oracle.c); returns (g [S], prim [S]);
    the envelope distance is max(g, 0)."""
    smp = np.ascontiguousarray(samples, dtype=np.float64).reshape(-1, 3)
    sph = np.ascontiguousarray(spheres, dtype=np.float64).reshape(-1, 4)
    e = np.ascontiguousarray(edges, dtype=np.int32).reshape(-1, 2)
    f = np.ascontiguousarray(faces, dtype=np.int32).reshape(-1, 3)
    g = np.zeros(len(smp))
    prim = np.zeros(len(smp), np.int32)
    lib().oracle_envelope(smp.ctypes.data, len(smp), sph.ctypes.data, len(sph),
                          e.ctypes.data if len(e) else None, len(e),
                          f.ctypes.data if len(f) else None, len(f), g.ctypes.data,
                          prim.ctypes.data, int(nthreads))
    return g, prim


def envelope_one(p, spheres, ids):
    """Signed value of one primitive (1 id: sphere, 2: cone, 3: slab) at p."""
    pp = np.ascontiguousarray(p, dtype=np.float64)
    sph = np.ascontiguousarray(spheres, dtype=np.float64).reshape(-1, 4)
    ii = np.ascontiguousarray(ids, dtype=np.int32)
    return lib().oracle_envelope_one(pp.ctypes.data, sph.ctypes.data, len(ii) - 1, ii.ctypes.data)


def max_threads() -> int:
    return int(lib().oracle_max_threads())
