"""The CUDA path's exact predicates (rpd_internal.cuh) against their definition evaluated in
Python integers: det[a_p; a_q; a_r; a_s] of barycentric plane vectors and the inward
symbolic-perturbation rule (C4).  Host build runs here (-m "not gpu"); the same
cases are evaluated inside a kernel on the GPU (-m gpu)."""
import itertools
import os
import random
import subprocess

import numpy as np
import pytest

import rpd_workloads as W

HERE = os.path.dirname(os.path.abspath(__file__))
NVCC = "/usr/local/cuda/bin/nvcc"


def det(M):
    n = len(M)
    tot = 0
    for perm in itertools.permutations(range(n)):
        s = 1
        for a in range(n):
            for b in range(a + 1, n):
                if perm[a] > perm[b]:
                    s = -s
        prod = 1
        for a in range(n):
            prod *= M[a][perm[a]]
        tot += s * prod
    return tot


def sgn(x):
    return (x > 0) - (x < 0)


ONE = [1, 1, 1, 1]


def sos(rows, ranks):
    D4 = det(rows)
    D3 = det(rows[:3] + [ONE])
    if D4:
        return sgn(D4) * sgn(D3)
    for k in sorted(range(4), key=lambda k: ranks[k]):
        R = [list(r) for r in rows]
        R[k] = ONE
        C = det(R)
        if C:
            return -sgn(C) * sgn(D3)
    return 0


def cases(n_per_pair=12, seeds=(0, 1, 2)):
    """Random plane quadruples from degenerate C1b configs (exact zeros are frequent)."""
    rng = random.Random(0)
    lines, expect = [], []
    for seed in seeds:
        for big in (False, True):
            w = W.make_c1(seed, degenerate=True, big=big)
            S = [[int(round(c * 1024)) for c in s] for s in w.spheres]
            for t in range(w.T):
                X = [[int(round(c * 1024)) for c in w.verts[v]] for v in w.tets[t]]
                for i in range(w.N):
                    def pd(s, x):
                        return sum((x[c] - s[c]) ** 2 for c in range(3)) - s[3] ** 2
                    planes = [(0, [int(c == k) for c in range(4)], [0, 0, 0], w.N + k)
                              for k in range(4)]
                    for j in w.nbr_idx[w.nbr_off[i]:w.nbr_off[i + 1]]:
                        g = [pd(S[j], x) - pd(S[i], x) for x in X]
                        n = [2 * (S[i][c] - S[j][c]) for c in range(3)]
                        planes.append((1, g, n, int(j)))
                    for _ in range(n_per_pair):
                        q = rng.sample(range(len(planes)), 4)
                        rows = [planes[k][1] for k in q]
                        if det(rows[:3] + [ONE]) == 0:
                            continue
                        lines.append(" ".join(" ".join(map(str, [planes[k][0]] + planes[k][1] +
                                                             planes[k][2] + [planes[k][3]]))
                                              for k in q))
                        expect.append((sgn(det(rows)), sos(rows, [planes[k][3] for k in q]),
                                       int(det(rows) == 0)))
    return lines, expect


def run(exe, lines):
    out = subprocess.run([exe], input="\n".join(lines) + "\n", capture_output=True, text=True,
                         check=True).stdout.split()
    return [tuple(map(int, out[3 * k:3 * k + 3])) for k in range(len(out) // 3)]


def build(src, exe, device):
    flags = ["-gencode", "arch=compute_100a,code=sm_100a"] if device else []
    subprocess.check_call([NVCC, "-O3", "-std=c++17", *flags, "-o", exe, src],
                          stderr=subprocess.DEVNULL)


def test_host_predicates_match_definition(tmp_path):
    exe = str(tmp_path / "pred_host")
    build(os.path.join(HERE, "native", "pred_harness.cu"), exe, device=False)
    lines, expect = cases()
    got = run(exe, lines)
    assert len(got) == len(expect)
    assert sum(e[2] for e in expect) > 30           # many exact zeros (SoS exercised)
    bad = [(l, e, g) for l, e, g in zip(lines, expect, got) if e != g]
    assert not bad, bad[:3]


@pytest.mark.gpu
def test_device_predicates_match_definition(tmp_path):
    exe = str(tmp_path / "pred_dev")
    build(os.path.join(HERE, "native", "pred_device.cu"), exe, device=True)
    lines, expect = cases()
    got = run(exe, lines)
    bad = [(l, e, g) for l, e, g in zip(lines, expect, got) if e != g]
    assert not bad, bad[:3]
