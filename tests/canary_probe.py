"""Subprocess of tests/test_gpu_canary.py (RPD_CANARY=1 must be set before the library's first
allocation): one byte written just past the end of a library buffer (the candidate offsets,
whose size the probe recomputes as DevBuf::ensure sizes it) must be reported by
rpd_debug_check, and nothing before that write."""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
assert os.environ.get("RPD_CANARY") == "1"
import numpy as np
import torch

import paper_2403_18761_b200 as P
import rpd_workloads as W

w = W.make_c1(0)
ctx = P.RPDContext(0)
ctx.relations(w.verts, w.tets, w.spheres, w.nbr_off, w.nbr_idx)  # (checked after the call)
L = ctx.L
co, ci, nc = C.c_void_p(), C.c_void_p(), C.c_int64()
vp = lambda a: np.ascontiguousarray(a)
arrs = [vp(w.verts), vp(w.tets.astype(np.int32)), vp(w.spheres), vp(w.nbr_off.astype(np.int32)),
        vp(w.nbr_idx.astype(np.int32))]
st = L.rpd_relations(ctx.h, arrs[0].ctypes.data, len(w.verts), arrs[1].ctypes.data, w.T,
                     arrs[2].ctypes.data, w.N, arrs[3].ctypes.data, arrs[4].ctypes.data,
                     len(w.nbr_idx), C.byref(co), C.byref(ci), C.byref(nc))
assert st == 0 and L.rpd_debug_check(ctx.h) == 0
nbytes = 4 * (w.T + 1)  # the candidate offsets: DevBuf::ensure(4 (T + 1))
cap = 256 if nbytes < 256 else nbytes + nbytes // 8
torch.cuda.synchronize()
from paper_2403_18761_b200.rpd import _View
past_end = torch.as_tensor(_View(co.value + cap, 1, "|u1"), device="cuda")  # no copy
past_end.fill_(0)  # one byte written just past the buffer's capacity (its canary starts there)
torch.cuda.synchronize()
st = L.rpd_debug_check(ctx.h)
print("canary after the overrun:", st, L.rpd_last_error(ctx.h).decode())
sys.exit(0 if st == -3 else 1)
