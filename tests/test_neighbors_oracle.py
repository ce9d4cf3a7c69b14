"""NEXT-3 oracle pins (DESIGN.md §10 "Sphere neighbours"): the box-restricted
power-cell neighbours ``oracle.box_neighbours`` against what does not come from the oracle's
own clip -- the regular triangulation edges Qhull computes (a box facet is a triangulation
edge), closed forms on collinear spheres, and sufficiency (the pieces of the mesh are the same
with the box lists as with the regular-triangulation lists)."""
import numpy as np
import pytest

import oracle
import rpd_workloads as W
from tests.helpers import compare_results


def rows(off, idx):
    return [set(idx[off[i]:off[i + 1]].tolist()) for i in range(len(off) - 1)]


WORKLOADS = [lambda: W.make_shape_workload("nb_smoke", 1200, 100, seed=11, cache=False),
             lambda: W.make_c1(3), lambda: W.random_tiny(5, n_spheres=14),
             lambda: W.make_shape_workload("nb_small", 600, 60, seed=4, cache=False)]


@pytest.mark.parametrize("k", range(len(WORKLOADS)))
def test_box_neighbours_in_regular_triangulation(k):
    w = WORKLOADS[k]()
    off, idx = oracle.box_neighbours(w.spheres, W.mesh_box(w.verts))
    rt = rows(w.nbr_off, w.nbr_idx)
    for i, r in enumerate(rows(off, idx)):
        assert r <= rt[i], (i, sorted(r - rt[i]))
        assert i not in r
    # symmetric: a positive-area facet of C_i ∩ B on h_ij is one of C_j ∩ B on h_ji
    R = rows(off, idx)
    for i, r in enumerate(R):
        for j in r:
            assert i in R[j]


@pytest.mark.parametrize("k", range(len(WORKLOADS)))
def test_box_neighbours_sufficient(k):
    w = WORKLOADS[k]()
    off, idx = oracle.box_neighbours(w.spheres, W.mesh_box(w.verts))
    a = oracle.rpd(w.verts, w.tets, w.spheres, off, idx)
    b = oracle.rpd_workload(w)
    assert compare_results(a, b, w.verts, w.tets, check_cands=False) == []


def test_box_neighbours_collinear_closed_form():
    # centres on the x axis at 8, 16, 24 (equal radii): bisector planes x = 12, x = 20 cut the
    # box [0, 32]^3 -> chain 0 - 1 - 2; with r_1 = 0 and r_0 = r_2 = 5 the planes move to
    # x = 12 + 25/16 and x = 20 - 25/16 (PD_0 = PD_1: 16 x = 217) and stay inside.  A box
    # [0, 14] x ... keeps only the first plane, [0, 13] none.
    sp = np.array([[8, 16, 16, 1], [16, 16, 16, 1], [24, 16, 16, 1]], dtype=np.float64)
    off, idx = oracle.box_neighbours(sp, (0, 0, 0, 32, 32, 32))
    assert rows(off, idx) == [{1}, {0, 2}, {1}]
    sp[:, 3] = [5, 0, 5]
    off, idx = oracle.box_neighbours(sp, (0, 0, 0, 32, 32, 32))
    assert rows(off, idx) == [{1}, {0, 2}, {1}]
    off, idx = oracle.box_neighbours(sp, (0, 0, 0, 14, 32, 32))
    assert rows(off, idx) == [{1}, {0}, set()]
    off, idx = oracle.box_neighbours(sp, (0, 0, 0, 13, 32, 32))
    assert rows(off, idx) == [set(), set(), set()]
    # a plane outside the box: no neighbours at all (sphere 1's cell misses the box)
    off, idx = oracle.box_neighbours(sp[:2], (0, 0, 0, 4, 32, 32))
    assert rows(off, idx) == [set(), set()]


def test_box_neighbours_dominated_sphere():
    # sphere 1 (small, off-centre inside sphere 0's power cell region) has an empty cell when
    # the power distance of 0 is below 1's everywhere: r_0^2 - r_1^2 >= |c_0 - c_1|^2
    sp = np.array([[16, 16, 16, 6], [17, 16, 16, 1], [28, 16, 16, 1]], dtype=np.float64)
    off, idx = oracle.box_neighbours(sp, (0, 0, 0, 32, 32, 32))
    assert rows(off, idx) == [{2}, set(), {0}]
