"""Thin Python binding of librpd (include/rpd.h) -- argument marshalling only.

Every step of the RPD path runs in librpd's CUDA kernels; this module passes pointers of
torch tensors (device or host) or numpy arrays to the C ABI and wraps the results.  There is
no CPU fallback: if librpd.so is missing or no CUDA device is present the calls raise.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "librpd.so")

RPD_OK, RPD_EINVAL, RPD_ENOMEM, RPD_ECUDA, RPD_EOVERFLOW, RPD_ESTATE, RPD_ENOTEXACT = \
    0, -1, -2, -3, -4, -5, -6
STATUS_NAMES = {0: "RPD_OK", -1: "RPD_EINVAL", -2: "RPD_ENOMEM", -3: "RPD_ECUDA",
                -4: "RPD_EOVERFLOW", -5: "RPD_ESTATE", -6: "RPD_ENOTEXACT"}
OPT_FILTER_MODE, OPT_VALIDATE, OPT_STREAM, OPT_CLIP_WIDE, OPT_PROFILE = 1, 2, 3, 4, 5
OPT_CLIP_TIERS, OPT_GRAPH = 6, 7
FILTER_ALL_PAIRS, FILTER_PRUNED = 0, 1
CUDA_STREAM_LEGACY = 0x1  # cudaStreamLegacy

EXPORTED = ["rpd_create", "rpd_destroy", "rpd_last_error", "rpd_set_option", "rpd_relations",
            "rpd_clip", "rpd_update_partial", "rpd_download_pieces", "rpd_download_cands",
            "rpd_get_stats", "rpd_version", "rpd_set_euler", "rpd_get_euler",
            "rpd_download_euler", "rpd_get_topology", "rpd_download_topology",
            "rpd_medial_mesh", "rpd_download_medial_mesh", "rpd_gather_pieces", "rpd_envelope",
            "rpd_neighbors", "rpd_download_neighbors", "rpd_gather_cands", "rpd_merge_shards",
            "rpd_download_tets", "rpd_get_rpe", "rpd_download_rpe", "rpd_euler_finalize",
            "rpd_neighbors_update", "rpd_cc_shard", "rpd_cc_merge", "rpd_sphere_volumes",
            "rpd_debug_check", "rpd_rpe_shard", "rpd_rpe_merge", "rpd_reduce_by_key"]


class RPDError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"{STATUS_NAMES.get(status, status)}: {msg}")
        self.status = status


class _Pieces(C.Structure):
    _fields_ = [("piece_off", C.c_void_p), ("piece_sphere", C.c_void_p),
                ("piece_vol", C.c_void_p), ("piece_m1", C.c_void_p),
                ("piece_facemask", C.c_void_p), ("inc_off", C.c_void_p),
                ("inc_sphere", C.c_void_p), ("n_pieces", C.c_int64), ("n_inc", C.c_int64),
                ("piece_rows", C.c_void_p), ("n_slots", C.c_int64)]


EULER_KEYS = ("piece_euler", "piece_denom", "rpf_off", "rpf_sphere", "rpf_euler", "rpc_sum",
              "rpc_exact", "rpc_value", "rpf_sum", "rpf_exact", "rpf_value", "rpc_acc",
              "rpf_acc")


class _Euler(C.Structure):
    _fields_ = [("n_primes", C.c_int64)] + [(k, C.c_void_p) for k in EULER_KEYS] + \
        [("n_pieces", C.c_int64), ("n_rpf", C.c_int64), ("N", C.c_int64), ("E", C.c_int64)]


class _Topology(C.Structure):
    _fields_ = [("rpc_cc", C.c_void_p), ("rpf_cc", C.c_void_p), ("piece_comp", C.c_void_p),
                ("rpf_comp", C.c_void_p), ("piece_sosfm", C.c_void_p), ("rpf_fm", C.c_void_p),
                ("rpf_adj", C.c_void_p), ("n_pieces", C.c_int64), ("n_rpf", C.c_int64), ("N", C.c_int64),
                ("E", C.c_int64)]


class _CcRecords(C.Structure):
    _fields_ = [("key_c", C.c_void_p), ("lab_c", C.c_void_p), ("n_c", C.c_int64),
                ("key_f", C.c_void_p), ("j_f", C.c_void_p), ("lab_f", C.c_void_p),
                ("n_f", C.c_int64), ("n_pieces", C.c_int64), ("n_rpf", C.c_int64)]


class _RpeRecords(C.Structure):
    _fields_ = [("tri_key", C.c_void_p), ("tri_euler", C.c_void_p), ("n_tri", C.c_int64),
                ("n_rpe", C.c_int64), ("key_b", C.c_void_p), ("jk_b", C.c_void_p),
                ("lab_b", C.c_void_p), ("n_b", C.c_int64)]


class _Rpe(C.Structure):
    _fields_ = [("denom", C.c_int64)] + [(k, C.c_void_p) for k in (
        "rpe_off", "rpe_j", "rpe_k", "rpe_euler", "rpe_fm", "tri", "tri_euler", "tri_cc")] + \
        [("n_pieces", C.c_int64), ("n_rpe", C.c_int64), ("n_tri", C.c_int64)]


class _NbrLists(C.Structure):
    _fields_ = [("nbr_off", C.c_void_p), ("nbr_idx", C.c_void_p), ("N", C.c_int64),
                ("E", C.c_int64), ("n_hidden", C.c_int64), ("n_vertex_overflow", C.c_int64),
                ("n_rows_computed", C.c_int64), ("n_rows_block", C.c_int64)]


class _Medial(C.Structure):
    _fields_ = [("edges", C.c_void_p), ("faces", C.c_void_p), ("n_edges", C.c_int64),
                ("n_faces", C.c_int64)]


MAX_RANKS = 16


SHARD_KEYS = ("tet_ids", "piece_off", "piece_sphere", "piece_vol", "piece_m1",
              "piece_facemask", "inc_off", "inc_sphere", "cand_off", "cand_idx")
CSR_KEYS = ("cand_off", "cand_idx", "piece_off", "piece_sphere", "piece_vol", "piece_m1",
            "piece_facemask", "inc_off", "inc_sphere")


class _Shards(C.Structure):
    _fields_ = [("world", C.c_int32), ("T", C.c_int64), ("n_tets", C.c_int64 * MAX_RANKS)] + \
               [(k, C.c_void_p * MAX_RANKS) for k in SHARD_KEYS]


class _Csr(C.Structure):
    _fields_ = [(k, C.c_void_p) for k in CSR_KEYS] + \
               [(k, C.c_int64) for k in ("T", "n_cand", "n_pieces", "n_inc")]


class _Stats(C.Structure):
    _fields_ = [("T", C.c_int64), ("N", C.c_int64), ("n_cand", C.c_int64),
                ("n_pieces", C.c_int64), ("n_inc", C.c_int64), ("n_dirty", C.c_int64),
                ("pairs_filtered", C.c_int64), ("pairs_tested", C.c_int64),
                ("pairs_clipped", C.c_int64),
                ("exact_fallbacks", C.c_int64), ("zero_hits", C.c_int64),
                ("kernel_launches", C.c_int64), ("max_k_tet", C.c_int32),
                ("max_vertices", C.c_int32), ("max_planes", C.c_int32), ("n_wide", C.c_int32),
                ("rel_tests", C.c_int64), ("clip_plane_evals", C.c_int64),
                ("clip_vertex_tests", C.c_int64), ("clip_constructions", C.c_int64),
                ("clip_fan_triangles", C.c_int64), ("filter_ms", C.c_double),
                ("clip_ms", C.c_double), ("n_cand_dirty", C.c_int64),
                ("n_pieces_dirty", C.c_int64), ("n_inc_dirty", C.c_int64),
                ("graph_updates", C.c_int64), ("graph_captures", C.c_int64),
                ("graph_fallbacks", C.c_int64)]


_lib = None


def load_library(path: str = LIB_PATH):
    """Load librpd.so (fails loudly if it has not been built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise ImportError(f"librpd.so not built at {path}: run __graft_entry__.build()")
    L = C.CDLL(path)
    vp, i64, i32 = C.c_void_p, C.c_int64, C.c_int
    L.rpd_create.argtypes = [C.POINTER(vp), i32, vp]
    L.rpd_destroy.argtypes = [vp]
    L.rpd_destroy.restype = None
    L.rpd_last_error.argtypes = [vp]
    L.rpd_last_error.restype = C.c_char_p
    L.rpd_set_option.argtypes = [vp, i32, i64]
    L.rpd_relations.argtypes = [vp, vp, i64, vp, i64, vp, i64, vp, vp, i64, C.POINTER(vp),
                                C.POINTER(vp), C.POINTER(i64)]
    L.rpd_clip.argtypes = [vp, C.POINTER(_Pieces)]
    L.rpd_update_partial.argtypes = [vp, vp, i64, vp, vp, i64, vp, i64, C.POINTER(_Pieces),
                                     C.POINTER(vp), C.POINTER(i64)]
    L.rpd_download_pieces.argtypes = [vp] * 8
    L.rpd_download_cands.argtypes = [vp, vp, vp]
    L.rpd_get_stats.argtypes = [vp, C.POINTER(_Stats)]
    L.rpd_set_euler.argtypes = [vp, vp, i64, i64, vp, i64, C.POINTER(i64)]
    L.rpd_get_euler.argtypes = [vp, C.POINTER(_Euler)]
    L.rpd_download_euler.argtypes = [vp] * 14
    L.rpd_euler_finalize.argtypes = [vp, vp, i64, vp, vp, vp]
    L.rpd_get_topology.argtypes = [vp, C.POINTER(_Topology)]
    L.rpd_download_topology.argtypes = [vp] * 8
    L.rpd_medial_mesh.argtypes = [vp, C.POINTER(_Medial)]
    L.rpd_download_medial_mesh.argtypes = [vp, vp, vp]
    L.rpd_neighbors.argtypes = [vp, vp, i64, vp, C.POINTER(_NbrLists)]
    L.rpd_neighbors_update.argtypes = [vp, vp, i64, i64, vp, C.POINTER(_NbrLists)]
    L.rpd_cc_shard.argtypes = [vp, i64, i64, C.POINTER(_CcRecords)]
    L.rpd_sphere_volumes.argtypes = [vp, vp]
    L.rpd_debug_check.argtypes = [vp]
    L.rpd_rpe_shard.argtypes = [vp, i64, C.POINTER(_RpeRecords)]
    L.rpd_rpe_merge.argtypes = [vp, vp, vp, vp, i64, i64, C.POINTER(C.c_void_p),
                                C.POINTER(C.c_void_p), C.POINTER(i64)]
    L.rpd_reduce_by_key.argtypes = [vp, vp, vp, i64, vp, vp, C.POINTER(i64)]
    L.rpd_cc_merge.argtypes = [vp, vp, vp, i64, vp, vp, vp, i64, i64, i64, vp]
    L.rpd_download_neighbors.argtypes = [vp, vp, vp]
    L.rpd_gather_pieces.argtypes = [vp, C.POINTER(_Shards)] + [vp] * 7
    L.rpd_gather_cands.argtypes = [vp, C.POINTER(_Shards), vp, vp]
    L.rpd_merge_shards.argtypes = [vp, C.POINTER(_Shards), C.POINTER(_Csr), C.POINTER(_Csr)]
    L.rpd_download_tets.argtypes = [vp, vp, i64, vp, vp, C.POINTER(_Csr)]
    L.rpd_get_rpe.argtypes = [vp, C.POINTER(_Rpe)]
    L.rpd_download_rpe.argtypes = [vp] * 9
    L.rpd_envelope.argtypes = [vp, vp, i64, vp, i64, vp, i64, vp, i64, vp, vp, C.POINTER(i64)]
    L.rpd_version.restype = C.c_char_p
    for f in ("rpd_create", "rpd_set_option", "rpd_relations", "rpd_clip", "rpd_update_partial",
              "rpd_download_pieces", "rpd_download_cands", "rpd_get_stats", "rpd_set_euler",
              "rpd_get_euler", "rpd_download_euler", "rpd_get_topology",
              "rpd_download_topology", "rpd_medial_mesh", "rpd_download_medial_mesh",
              "rpd_gather_pieces", "rpd_envelope", "rpd_neighbors",
              "rpd_download_neighbors", "rpd_gather_cands", "rpd_merge_shards",
              "rpd_download_tets", "rpd_get_rpe", "rpd_download_rpe", "rpd_euler_finalize",
              "rpd_neighbors_update", "rpd_cc_shard", "rpd_cc_merge", "rpd_sphere_volumes",
              "rpd_debug_check", "rpd_rpe_shard", "rpd_rpe_merge", "rpd_reduce_by_key"):
        getattr(L, f).restype = C.c_int
    _lib = L
    return L


def _numel(a) -> int:
    """Element count of a torch tensor or numpy array (no numpy reduction on the timed path)."""
    n = a.numel() if callable(getattr(a, "numel", None)) else a.size
    return int(n)


def _ptr(x, dtype):
    """(pointer, keepalive) of a torch tensor (CUDA or CPU) or array-like, C-contiguous."""
    try:
        import torch
        if isinstance(x, torch.Tensor):
            tdt = torch.float64 if dtype is np.float64 else torch.int32
            if x.dtype is not tdt or not x.is_contiguous():  # (fast path: no torch dispatch)
                x = x.to(tdt).contiguous()
            return (x.data_ptr() if x.numel() else None), x
    except ImportError:
        pass
    a = np.ascontiguousarray(x, dtype=dtype)
    return (a.ctypes.data if a.size else None), a


@dataclass
class PieceCounts:
    n_pieces: int
    n_inc: int


class RPDContext:
    """One librpd context on one CUDA device (stream-ordered on ``stream``; default: the
    current torch stream of that device)."""

    def __init__(self, device: int = 0, stream=None, filter_mode: str = "all_pairs",
                 validate: bool = True):
        import torch
        if not torch.cuda.is_available():
            raise RuntimeError("RPDContext needs a CUDA device (no CPU fallback)")
        self.L = load_library()
        self.device = device
        if stream is None:
            stream = torch.cuda.current_stream(device)
        self._stream = stream
        h = C.c_void_p()
        # torch's default stream has handle 0, which rpd_create would read as "make a private
        # non-blocking stream" -- unordered with torch / NCCL work.  Bind the ctx to the legacy
        # default stream (cudaStreamLegacy) instead, so every call is ordered after the work
        # torch queued before it (dtype conversions in _ptr, NCCL all-gathers, ...).
        handle = stream.cuda_stream or CUDA_STREAM_LEGACY
        st = self.L.rpd_create(C.byref(h), device, C.c_void_p(handle))
        if st != 0:
            raise RPDError(st, "rpd_create failed")
        self.h = h
        self.set_filter_mode(filter_mode)
        self.L.rpd_set_option(self.h, OPT_VALIDATE, int(bool(validate)))
        self.T = 0
        self.N = 0
        self.n_cand = 0
        self.counts = None

    _CANARY = os.environ.get("RPD_CANARY", "0") not in ("", "0")

    def _check(self, st):
        if st != 0:
            raise RPDError(st, self.L.rpd_last_error(self.h).decode())
        if self._CANARY and self.h:  # debugging: every buffer's canary after every call
            st = self.L.rpd_debug_check(self.h)
            if st != 0:
                raise RPDError(st, self.L.rpd_last_error(self.h).decode())

    def set_filter_mode(self, mode: str):
        m = {"all_pairs": FILTER_ALL_PAIRS, "pruned": FILTER_PRUNED}[mode]
        self._check(self.L.rpd_set_option(self.h, OPT_FILTER_MODE, m))

    def set_clip_wide(self, on: bool):
        """Testing: route every pair through the wide (128-vertex) clip kernel."""
        self._check(self.L.rpd_set_option(self.h, OPT_CLIP_WIDE, int(bool(on))))

    def set_clip_tiers(self, on: bool):
        """Testing: the fast clip tier and its overflow cascade also for < 2048 pairs."""
        self._check(self.L.rpd_set_option(self.h, OPT_CLIP_TIERS, int(bool(on))))

    def set_graph(self, on: bool):
        """Partial updates of 1..64 spheres as one device-driven CUDA graph (default on)."""
        self._check(self.L.rpd_set_option(self.h, OPT_GRAPH, int(bool(on))))

    def set_profile(self, on: bool):
        """Time the filter and clip kernels with CUDA events (stats filter_ms / clip_ms)."""
        self._check(self.L.rpd_set_option(self.h, OPT_PROFILE, int(bool(on))))

    def close(self):
        if getattr(self, "h", None):
            self.L.rpd_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ------------------------------------------------------------------ calls
    def relations(self, verts, tets, spheres, nbr_off, nbr_idx) -> int:
        """Alg. 1 + k_tet compaction; returns n_cand (candidates stay on the device)."""
        pv, kv = _ptr(verts, np.float64)
        pt, kt = _ptr(tets, np.int32)
        ps, ks = _ptr(spheres, np.float64)
        po, ko = _ptr(nbr_off, np.int32)
        pi, ki = _ptr(nbr_idx, np.int32)
        V = _numel(kv) // 3
        T = _numel(kt) // 4
        N = _numel(ks) // 4
        co, ci, nc = C.c_void_p(), C.c_void_p(), C.c_int64()
        E = _numel(ki)  # length of nbr_idx (no device read of nbr_off[N])
        self._check(self.L.rpd_relations(self.h, pv, V, pt, T, ps, N, po, pi, E, C.byref(co),
                                         C.byref(ci), C.byref(nc)))
        self.T, self.N, self.n_cand = T, N, nc.value
        self._keep = (kv, kt, ks, ko, ki)
        return nc.value

    def clip(self) -> PieceCounts:
        P = _Pieces()
        self._check(self.L.rpd_clip(self.h, C.byref(P)))
        self.counts = PieceCounts(P.n_pieces, P.n_inc)
        return self.counts

    def update_partial(self, spheres, nbr_off, nbr_idx, new_ids):
        ps, ks = _ptr(spheres, np.float64)
        po, ko = _ptr(nbr_off, np.int32)
        pi, ki = _ptr(nbr_idx, np.int32)
        pn, kn = _ptr(new_ids, np.int32)
        N_new = _numel(ks) // 4
        M = _numel(kn)
        P = _Pieces()
        dt, nd = C.c_void_p(), C.c_int64()
        E = _numel(ki)
        self._check(self.L.rpd_update_partial(self.h, ps, N_new, po, pi, E, pn, M, C.byref(P),
                                              C.byref(dt), C.byref(nd)))
        self.N = N_new
        self.counts = PieceCounts(P.n_pieces, P.n_inc)
        sb = self._sbuf = getattr(self, "_sbuf", None) or _Stats()
        self._check(self.L.rpd_get_stats(self.h, C.byref(sb)))  # (no dict: on the timed path)
        self.n_cand = sb.n_cand
        self.n_dirty = nd.value
        self._dirty_ptr = dt.value
        self._keep_p = (ks, ko, ki, kn)
        return self.counts, nd.value

    # ------------------------------------------------------------------ outputs
    def dirty_tets(self):
        """The dirty tets of the last update_partial (ascending) as a torch CUDA int32 tensor
        (a copy of the ctx-owned device array)."""
        return _device_view(self.dirty_ptr(), int(getattr(self, "n_dirty", 0)), "<i4").clone()

    def download_cands(self, device=False, out=None):
        """Candidate CSR as numpy (host) or torch CUDA tensors (device=True); ``out``: optional
        preallocated destinations (numpy or torch, host or device) keyed like the result."""
        T, n = self.T, self.n_cand
        specs = [(T + 1, np.int32), (n, np.int32)]
        keys = ["cand_off", "cand_idx"]
        arrs = self._alloc(specs, device) if out is None else self._outs(out, keys, specs)
        self._check(self.L.rpd_download_cands(self.h, self._p(arrs[0]), self._p(arrs[1])))
        return dict(zip(keys, arrs))

    @staticmethod
    def _outs(out, keys, specs):
        """Views [:n] of caller destinations, checked for dtype and length."""
        arrs = []
        for k, (n, dt) in zip(keys, specs):
            a = out[k].reshape(-1)
            adt = np.dtype(dt)
            ok = (a.dtype == adt) if isinstance(a, np.ndarray) else \
                (a.element_size() == adt.itemsize and str(a.dtype).endswith(adt.name))
            if not ok or (a.size if isinstance(a, np.ndarray) else a.numel()) < n:
                raise ValueError(f"out[{k!r}] needs {n} x {adt}")
            arrs.append(a[:n])
        return arrs

    def download_pieces(self, device=False, out=None):
        """Piece CSR as numpy (host) or torch CUDA tensors (device=True).  `out`: optional
        preallocated destinations (e.g. pinned host arrays), a dict with the returned keys,
        each at least as long as the current piece set needs; views of them are returned."""
        T = self.T
        npc, ni = self.counts.n_pieces, self.counts.n_inc
        specs = [(T + 1, np.int32), (npc, np.int32), (npc, np.float64),
                 (3 * npc, np.float64), (npc, np.uint8), (npc + 1, np.int32), (ni, np.int32)]
        keys = ["piece_off", "piece_sphere", "piece_vol", "piece_m1", "piece_facemask",
                "inc_off", "inc_sphere"]
        arrs = self._alloc(specs, device) if out is None else self._outs(out, keys, specs)
        self._check(self.L.rpd_download_pieces(self.h, *[self._p(a) for a in arrs]))
        out = dict(zip(keys, arrs))
        out["piece_m1"] = out["piece_m1"].reshape(-1, 3)
        return out

    def set_euler(self, tets_all, V: int, local_ids=None) -> int:
        """Fractional Euler payloads of the ctx's tets from the whole mesh ``tets_all``
        (PAPER.md:491); ``local_ids``: global index of every ctx-local tet (None: the ctx holds
        all tets in order).  Returns P, the number of prime residues of a sum's accumulator
        row (R24).  ``tets_all=None`` switches Euler mode off."""
        L = C.c_int64()
        if tets_all is None:
            self._check(self.L.rpd_set_euler(self.h, None, 0, 0, None, 0, C.byref(L)))
            return 0
        pt, kt = _ptr(tets_all, np.int32)
        T_all = _numel(kt) // 4
        if local_ids is None:
            pl, kl, T_local = None, None, T_all
        else:
            pl, kl = _ptr(local_ids, np.int32)
            T_local = _numel(kl)
        self._check(self.L.rpd_set_euler(self.h, pt, T_all, int(V), pl, T_local, C.byref(L)))
        self._keep_eu = (kt, kl)
        return L.value

    def download_euler(self, device=False) -> dict:
        """Euler data of the current pieces (exact, R24): piece_euler numerators over
        piece_denom (the tet's L_t), rpf_off / rpf_sphere / rpf_euler (radical facets of each
        piece, over the piece's denominator), per sphere rpc_sum / rpc_exact / rpc_value and
        per CSR entry of the row-sorted CSR rpf_sum / rpf_exact / rpf_value (the integer sum,
        whether it is exact, the value as a double), and the raw accumulator rows rpc_acc
        [N, 1+P] / rpf_acc [E, 1+P] (summed over the ranks of a sharded job, then
        euler_finalize)."""
        e = _Euler()
        self._check(self.L.rpd_get_euler(self.h, C.byref(e)))
        W = 1 + e.n_primes
        specs = [(e.n_pieces, np.int64), (e.n_pieces, np.int64), (e.n_pieces + 1, np.int32),
                 (e.n_rpf, np.int32), (e.n_rpf, np.int64), (e.N, np.int64), (e.N, np.uint8),
                 (e.N, np.float64), (e.E, np.int64), (e.E, np.uint8), (e.E, np.float64),
                 (W * e.N, np.int64), (W * e.E, np.int64)]
        arrs = self._alloc(specs, device)
        self._check(self.L.rpd_download_euler(self.h, *[self._p(a) for a in arrs]))
        out = dict(zip(EULER_KEYS, arrs))
        out["rpc_acc"] = out["rpc_acc"].reshape(-1, W)
        out["rpf_acc"] = out["rpf_acc"].reshape(-1, W)
        out["n_primes"] = int(e.n_primes)
        return out

    def euler_finalize(self, acc):
        """Accumulator rows acc [n, 1+P] (torch CUDA int64, e.g. all-reduced over the ranks) ->
        (sum int64 [n], exact uint8 [n], value float64 [n]) as CUDA tensors."""
        import torch
        acc = acc.to(torch.int64).contiguous()
        n = int(acc.shape[0])
        dev = acc.device
        out = (torch.empty(n, dtype=torch.int64, device=dev),
               torch.empty(n, dtype=torch.uint8, device=dev),
               torch.empty(n, dtype=torch.float64, device=dev))
        self._check(self.L.rpd_euler_finalize(self.h, self._p(acc), n, self._p(out[0]),
                                              self._p(out[1]), self._p(out[2])))
        return out

    def sphere_volumes(self, device=False):
        """Per-sphere RPC volume over the ctx's tets (fp64 [N]; rpd_sphere_volumes)."""
        (out,) = self._alloc([(int(self.N), np.float64)], device)
        self._check(self.L.rpd_sphere_volumes(self.h, self._p(out)))
        return out

    def rpe_shard(self, rpe_base: int) -> dict:
        """RPEs of a sharded job, step 1 (rpd_rpe_shard): this rank's per-key Euler numerators
        (tri_key, tri_euler; over 2) and its shard-boundary records, as torch CUDA views of
        ctx-owned arrays (uint64 keys as int64); n_rpe sizes the next rank's base."""
        r = _RpeRecords()
        self._check(self.L.rpd_rpe_shard(self.h, int(rpe_base), C.byref(r)))
        return {"tri_key": _device_view(r.tri_key, r.n_tri, "<i8"),
                "tri_euler": _device_view(r.tri_euler, r.n_tri, "<i8"),
                "key_b": _device_view(r.key_b, r.n_b, "<i8"),
                "jk_b": _device_view(r.jk_b, r.n_b, "<i8"),
                "lab_b": _device_view(r.lab_b, r.n_b, "<i4"), "n_rpe": int(r.n_rpe)}

    def rpe_merge(self, rec: dict, total_rpe: int):
        """Step 2 (rpd_rpe_merge): all ranks' boundary records -> this rank's (keys, counts)
        of RPE components at their smallest global ids (torch CUDA views)."""
        kb, jb, lb = (rec[k].contiguous() for k in ("key_b", "jk_b", "lab_b"))
        pk, pc, n = C.c_void_p(), C.c_void_p(), C.c_int64()
        self._check(self.L.rpd_rpe_merge(self.h, self._p(kb), self._p(jb), self._p(lb),
                                         int(kb.numel()), int(total_rpe), C.byref(pk),
                                         C.byref(pc), C.byref(n)))
        return _device_view(pk.value, n.value, "<i8"), _device_view(pc.value, n.value, "<i8")

    def reduce_by_key(self, keys, vals):
        """Sums of vals per key, keys ascending (rpd_reduce_by_key; int64 CUDA tensors)."""
        import torch
        keys, vals = keys.contiguous(), vals.to(torch.int64).contiguous()
        n = int(keys.numel())
        ok = torch.empty(max(n, 1), dtype=torch.int64, device=keys.device)
        ov = torch.empty(max(n, 1), dtype=torch.int64, device=keys.device)
        m = C.c_int64()
        self._check(self.L.rpd_reduce_by_key(self.h, self._p(keys), self._p(vals), n,
                                             self._p(ok), self._p(ov), C.byref(m)))
        return ok[:m.value], ov[:m.value]

    def euler_sizes(self):
        """(n_pieces, n_rpf, N, E) of the current pieces in Euler mode."""
        e = _Euler()
        self._check(self.L.rpd_get_euler(self.h, C.byref(e)))
        return int(e.n_pieces), int(e.n_rpf), int(e.N), int(e.E)

    def cc_shard(self, piece_base: int, rpf_base: int) -> dict:
        """CC numbers of a sharded job, step 1 (rpd_cc_shard): local union-find and the records
        of the shard-boundary faces as torch CUDA views of ctx-owned arrays (key_c / key_f are
        int64 views of the uint64 keys)."""
        r = _CcRecords()
        self._check(self.L.rpd_cc_shard(self.h, int(piece_base), int(rpf_base), C.byref(r)))
        return {"key_c": _device_view(r.key_c, r.n_c, "<i8"), "lab_c": _device_view(r.lab_c, r.n_c, "<i4"),
                "key_f": _device_view(r.key_f, r.n_f, "<i8"), "j_f": _device_view(r.j_f, r.n_f, "<i4"),
                "lab_f": _device_view(r.lab_f, r.n_f, "<i4"), "n_pieces": int(r.n_pieces),
                "n_rpf": int(r.n_rpf)}

    def cc_merge(self, rec: dict, total_pieces: int, total_rpf: int):
        """Step 2 (rpd_cc_merge): the records of all ranks (dict of CUDA tensors, as cc_shard
        returns, concatenated) -> this rank's counts, an int32 CUDA tensor [N + E] (rpc then rpf
        components; sum over the ranks)."""
        import torch
        rec = {k: v.contiguous() for k, v in rec.items() if torch.is_tensor(v)}
        nc, nf = int(rec["key_c"].numel()), int(rec["key_f"].numel())
        e = _Euler()
        self._check(self.L.rpd_get_euler(self.h, C.byref(e)))
        out = torch.empty(int(e.N) + int(e.E), dtype=torch.int32, device=rec["key_c"].device)
        self._check(self.L.rpd_cc_merge(self.h, self._p(rec["key_c"]), self._p(rec["lab_c"]), nc,
                                        self._p(rec["key_f"]), self._p(rec["j_f"]),
                                        self._p(rec["lab_f"]), nf, int(total_pieces),
                                        int(total_rpf), self._p(out)))
        return out

    def topology(self):
        """Run the CC-number kernels on the current pieces (results stay on the device)."""
        t = _Topology()
        self._check(self.L.rpd_get_topology(self.h, C.byref(t)))
        return t

    def download_topology(self, device=False) -> dict:
        """CC numbers of the current pieces: rpc_cc [N], rpf_cc [E]
        (row-sorted CSR), component labels piece_comp / rpf_comp and the SoS facet flags
        piece_sosfm / rpf_fm.  Needs Euler mode with the whole mesh in the ctx."""
        t = _Topology()
        self._check(self.L.rpd_get_topology(self.h, C.byref(t)))
        specs = [(t.N, np.int32), (t.E, np.int32), (t.n_pieces, np.int32), (t.n_rpf, np.int32),
                 (t.n_pieces, np.uint8), (t.n_rpf, np.uint8), (t.n_rpf, np.uint64)]
        arrs = self._alloc(specs, device)
        self._check(self.L.rpd_download_topology(self.h, *[self._p(a) for a in arrs]))
        return dict(zip(["rpc_cc", "rpf_cc", "piece_comp", "rpf_comp", "piece_sosfm", "rpf_fm",
                         "rpf_adj"], arrs))

    def rpe(self, device=False) -> dict:
        """Restricted power edges of the current pieces: per piece
        its RPEs (rpe_off, rpe_j < rpe_k, rpe_euler numerators, rpe_fm endpoint tet faces) and
        per (i, j, k) seen from m_i (tri [n, 3]) the Euler characteristic (tri_euler over
        euler_denom) and the CC number (tri_cc; None unless the ctx holds the whole mesh)."""
        r = _Rpe()
        self._check(self.L.rpd_get_rpe(self.h, C.byref(r)))
        specs = [(r.n_pieces + 1, np.int32), (r.n_rpe, np.int32), (r.n_rpe, np.int32),
                 (r.n_rpe, np.int64), (r.n_rpe, np.uint8), (3 * r.n_tri, np.int32),
                 (r.n_tri, np.int64), (r.n_tri, np.int32)]
        arrs = self._alloc(specs, device)
        if not r.tri_cc:
            arrs[-1] = None
        self._check(self.L.rpd_download_rpe(self.h, *[self._p(a) if a is not None else None
                                                       for a in arrs]))
        out = dict(zip(["rpe_off", "rpe_j", "rpe_k", "rpe_euler", "rpe_fm", "tri", "tri_euler",
                        "tri_cc"], arrs))
        out["tri"] = out["tri"].reshape(-1, 3)
        out["euler_denom"] = int(r.denom)
        return out

    def medial_mesh(self, device=False) -> dict:
        """The dual medial mesh of the current pieces: unique sorted edges
        [n, 2] (i < j) and triangles [n, 3] (i < j < k)."""
        m = _Medial()
        self._check(self.L.rpd_medial_mesh(self.h, C.byref(m)))
        e, f = self._alloc([(2 * m.n_edges, np.int32), (3 * m.n_faces, np.int32)], device)
        self._check(self.L.rpd_download_medial_mesh(self.h, self._p(e), self._p(f)))
        return {"edges": e.reshape(-1, 2), "faces": f.reshape(-1, 3)}

    def neighbors(self, spheres, box, device=False) -> dict:
        """Sphere neighbour lists on the GPU (NEXT-3): a certified superset of
        the power-cell neighbours inside the axis box ``box`` = (lo_x, lo_y, lo_z, hi_x, hi_y,
        hi_z); returns nbr_off [N+1], nbr_idx [E] (rows ascending) and counters."""
        ps, ks = _ptr(spheres, np.float64)
        bx = np.ascontiguousarray(np.asarray(box, dtype=np.float64).reshape(6))
        n = _NbrLists()
        N = _numel(ks) // 4
        self._check(self.L.rpd_neighbors(self.h, ps, N, bx.ctypes.data, C.byref(n)))
        off, idx = self._alloc([(n.N + 1, np.int32), (n.E, np.int32)], device)
        self._check(self.L.rpd_download_neighbors(self.h, self._p(off), self._p(idx)))
        return {"nbr_off": off, "nbr_idx": idx, "n_hidden": n.n_hidden,
                "n_vertex_overflow": n.n_vertex_overflow, "n_rows": n.n_rows_computed,
                "n_rows_block": n.n_rows_block}

    def neighbors_update(self, spheres, M: int, box, device=False) -> dict:
        """Incremental lists after appending the last M of ``spheres`` (the previous call's
        spheres unchanged, same box): the new spheres' rows are computed, the old rows
        extended by the new spheres that reach their cell's ball (rpd_neighbors_update)."""
        ps, ks = _ptr(spheres, np.float64)
        bx = np.ascontiguousarray(np.asarray(box, dtype=np.float64).reshape(6))
        n = _NbrLists()
        N = _numel(ks) // 4
        self._check(self.L.rpd_neighbors_update(self.h, ps, N, int(M), bx.ctypes.data,
                                                C.byref(n)))
        off, idx = self._alloc([(n.N + 1, np.int32), (n.E, np.int32)], device)
        self._check(self.L.rpd_download_neighbors(self.h, self._p(off), self._p(idx)))
        return {"nbr_off": off, "nbr_idx": idx, "n_hidden": n.n_hidden,
                "n_vertex_overflow": n.n_vertex_overflow, "n_rows": n.n_rows_computed,
                "n_rows_block": n.n_rows_block}

    def dirty_ptr(self):
        """Device address of the ctx-owned dirty-tet list of the last update_partial."""
        return getattr(self, "_dirty_ptr", None)

    def download_tets(self, tet_list, n: int, out: dict, id_map=None):
        """Candidate + piece segments of the ctx's tets ``tet_list`` (a device address or an
        array of local ids) as one CSR over the list into the destinations ``out`` (numpy or
        torch, keyed like download_cands / download_pieces, plus ``tet_ids`` for the global
        ids ``id_map[tet_list]``); returns the sizes (n_cand, n_pieces, n_inc)."""
        keep = []
        if isinstance(tet_list, int) or tet_list is None:
            pl = tet_list
        else:
            pl, kl = _ptr(tet_list, np.int32)
            keep.append(kl)
        pm = None
        if id_map is not None:
            pm, km = _ptr(id_map, np.int32)
            keep.append(km)
        cs = _Csr()
        for k in CSR_KEYS:
            if k in out:
                setattr(cs, k, self._p(out[k]))
        ids = out.get("tet_ids")
        self._check(self.L.rpd_download_tets(self.h, pl, int(n), pm,
                                             self._p(ids) if ids is not None else None,
                                             C.byref(cs)))
        return cs.n_cand, cs.n_pieces, cs.n_inc

    def _shards(self, shards, T, tet_ids=None):
        world = len(shards)
        if world > MAX_RANKS:
            raise ValueError("too many ranks")
        sh = _Shards()
        sh.world, sh.T = world, int(T)
        keep = []
        for r, d in enumerate(shards):
            ids = d["tet_ids"] if tet_ids is None else tet_ids[r]
            sh.n_tets[r] = int(ids.numel())
            for k in SHARD_KEYS:
                t = ids if k == "tet_ids" else d.get(k)
                if t is None:
                    continue
                t = t.contiguous()
                keep.append(t)
                getattr(sh, k)[r] = t.data_ptr() if t.numel() else None
        return sh, keep

    def gather_all(self, shards, tet_ids, T: int, n_cand: int, n_pieces: int,
                   n_inc: int) -> dict:
        """Global candidate + piece CSRs (torch CUDA tensors) from the per-rank CSRs
        ``shards`` (dicts of CUDA tensors, e.g. views of the all-gathered payload) of the
        ranks' tets ``tet_ids`` (global ids): rpd_gather_cands + rpd_gather_pieces."""
        import torch
        sh, keep = self._shards(shards, T, tet_ids)
        dev = torch.device("cuda", self.device)
        e = lambda n, dt: torch.empty(max(n, 0), dtype=dt, device=dev)
        out = {"cand_off": e(T + 1, torch.int32), "cand_idx": e(n_cand, torch.int32),
               "piece_off": e(T + 1, torch.int32), "piece_sphere": e(n_pieces, torch.int32),
               "piece_vol": e(n_pieces, torch.float64),
               "piece_m1": e(3 * n_pieces, torch.float64).reshape(-1, 3),
               "piece_facemask": e(n_pieces, torch.uint8), "inc_off": e(n_pieces + 1, torch.int32),
               "inc_sphere": e(n_inc, torch.int32)}
        self._check(self.L.rpd_gather_cands(self.h, C.byref(sh), self._p(out["cand_off"]),
                                            self._p(out["cand_idx"])))
        self._check(self.L.rpd_gather_pieces(self.h, C.byref(sh), *[
            self._p(out[k]) for k in ("piece_off", "piece_sphere", "piece_vol", "piece_m1",
                                      "piece_facemask", "inc_off", "inc_sphere")]))
        return out

    def merge_shards(self, shards, glob, T: int) -> "GlobalCSR":
        """Partial-mode merge (rpd_merge_shards): the global CSR ``glob`` (a dict of tensors or
        the GlobalCSR of the previous merge) with the dirty rows replaced by the shards'
        segments (each shard dict holds ``tet_ids``, the global ids of its dirty tets, and
        their candidate + piece CSRs).  Returns a GlobalCSR over the ctx-owned result (valid
        until the next-but-one merge); it behaves as a dict of torch tensors, made on demand."""
        sh, keep = self._shards(shards, T)
        if isinstance(glob, GlobalCSR):
            old = glob.raw
        else:
            old = _Csr()
            for k in CSR_KEYS:
                setattr(old, k, self._p(glob[k]))
            old.T = int(T)
        res = _Csr()
        self._check(self.L.rpd_merge_shards(self.h, C.byref(sh), C.byref(old), C.byref(res)))
        return GlobalCSR(res, T)

    def gather_pieces(self, shards, tet_ids, T: int) -> dict:
        """Global piece CSR (torch CUDA tensors) from per-rank piece CSRs (``shards``: one dict
        per rank of CUDA tensors piece_off, piece_sphere, piece_vol, piece_m1, piece_facemask,
        inc_off, inc_sphere; ``tet_ids``: per rank the CUDA int32 global ids of its tets), put
        in global tet order by rpd_gather_pieces."""
        import torch
        tet_ids = [ids.to(torch.int32) for ids in tet_ids]
        shards = [{k: v for k, v in d.items() if not k.startswith("cand")} for d in shards]
        sh, keep = self._shards(shards, T, tet_ids)
        npc = sum(int(d["piece_sphere"].numel()) for d in shards)
        ninc = sum(int(d["inc_sphere"].numel()) for d in shards)
        dev = shards[0]["piece_vol"].device
        out = {"piece_off": torch.empty(T + 1, dtype=torch.int32, device=dev),
               "piece_sphere": torch.empty(npc, dtype=torch.int32, device=dev),
               "piece_vol": torch.empty(npc, dtype=torch.float64, device=dev),
               "piece_m1": torch.empty((npc, 3), dtype=torch.float64, device=dev),
               "piece_facemask": torch.empty(npc, dtype=torch.uint8, device=dev),
               "inc_off": torch.empty(npc + 1, dtype=torch.int32, device=dev),
               "inc_sphere": torch.empty(ninc, dtype=torch.int32, device=dev)}
        self._check(self.L.rpd_gather_pieces(self.h, C.byref(sh), *[
            self._p(out[k]) for k in ("piece_off", "piece_sphere", "piece_vol", "piece_m1",
                                      "piece_facemask", "inc_off", "inc_sphere")]))
        return out

    def envelope(self, samples, spheres, edges, faces, device=False):
        """Envelope distance of surface samples to the medial mesh's spheres / cones / slabs
        (PAPER.md:520-542): returns (g [S], prim [S], evaluated pairs); distance = max(g, 0)."""
        ps, ks = _ptr(samples, np.float64)
        pp, kp = _ptr(spheres, np.float64)
        pe, ke = _ptr(edges, np.int32)
        pf, kf = _ptr(faces, np.int32)
        S = _numel(ks) // 3
        g, prim = self._alloc([(S, np.float64), (S, np.int32)], device)
        ne = C.c_int64()
        self._check(self.L.rpd_envelope(self.h, ps, S, pp, _numel(kp) // 4, pe,
                                        _numel(ke) // 2, pf,
                                        _numel(kf) // 3, self._p(g), self._p(prim),
                                        C.byref(ne)))
        return g, prim, ne.value

    def stats_struct(self):
        """The raw rpd_stats struct (a fresh ctypes copy; cheaper than stats() on timed paths)."""
        st = _Stats()
        self._check(self.L.rpd_get_stats(self.h, C.byref(st)))
        return st

    def stats(self) -> dict:
        s = _Stats()
        self._check(self.L.rpd_get_stats(self.h, C.byref(s)))
        return {k: getattr(s, k) for k, _ in _Stats._fields_}

    @staticmethod
    def _alloc(specs, device):
        if device:
            import torch
            tdt = {np.int32: torch.int32, np.float64: torch.float64, np.uint8: torch.uint8,
                   np.int64: torch.int64, np.uint64: torch.int64}
            return [torch.empty(max(n, 0), dtype=tdt[dt], device="cuda") for n, dt in specs]
        return [np.empty(max(n, 0), dtype=dt) for n, dt in specs]

    @staticmethod
    def _p(a):
        try:
            import torch
            if isinstance(a, torch.Tensor):
                return a.data_ptr() if a.numel() else None
        except ImportError:
            pass
        return a.ctypes.data if a.size else None


class GlobalCSR:
    """A whole candidate + piece CSR in ctx-owned device arrays (rpd_merge_shards output): the
    raw pointers are kept (the next merge reads them directly); the torch views of the arrays
    are made on first access, dict-style (keys as rpd_csr)."""

    SPEC = {"cand_off": "<i4", "cand_idx": "<i4", "piece_off": "<i4", "piece_sphere": "<i4",
            "piece_vol": "<f8", "piece_m1": "<f8", "piece_facemask": "|u1", "inc_off": "<i4",
            "inc_sphere": "<i4"}

    def __init__(self, raw, T):
        self.raw, self.T, self._v = raw, int(T), {}

    def _len(self, k):
        r, T = self.raw, self.T
        return {"cand_off": T + 1, "cand_idx": r.n_cand, "piece_off": T + 1,
                "piece_sphere": r.n_pieces, "piece_vol": r.n_pieces, "piece_m1": 3 * r.n_pieces,
                "piece_facemask": r.n_pieces, "inc_off": r.n_pieces + 1,
                "inc_sphere": r.n_inc}[k]

    def __getitem__(self, k):
        if k not in self._v:
            v = _device_view(getattr(self.raw, k), self._len(k), self.SPEC[k])
            self._v[k] = v.reshape(-1, 3) if k == "piece_m1" else v
        return self._v[k]

    def keys(self):
        return list(self.SPEC)

    def items(self):
        return [(k, self[k]) for k in self.SPEC]

    def values(self):
        return [self[k] for k in self.SPEC]

    def __iter__(self):
        return iter(self.SPEC)


class _View:
    """__cuda_array_interface__ over a device array owned by librpd (no copy)."""

    def __init__(self, ptr, n, typestr):
        self.__cuda_array_interface__ = {"shape": (int(n),), "typestr": typestr,
                                         "data": (ptr or 0, False), "version": 3,
                                         "stream": None}


def _device_view(ptr, n, typestr):
    import torch
    if n <= 0 or not ptr:
        tdt = {"<i4": torch.int32, "<f8": torch.float64, "|u1": torch.uint8,
               "<i8": torch.int64}[typestr]
        return torch.zeros(0, dtype=tdt, device="cuda")
    return torch.as_tensor(_View(ptr, n, typestr), device="cuda")


def rpd_full(verts, tets, spheres, nbr_off, nbr_idx, ctx: RPDContext = None, **kw):
    """Convenience: relations + clip, results as numpy dicts (host)."""
    own = ctx is None
    ctx = ctx or RPDContext(**kw)
    try:
        ctx.relations(verts, tets, spheres, nbr_off, nbr_idx)
        ctx.clip()
        out = ctx.download_cands()
        out.update(ctx.download_pieces())
        out["stats"] = ctx.stats()
        return out
    finally:
        if own:
            ctx.close()
