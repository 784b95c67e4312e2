"""Pins of oracle/geometry.py and oracle/assembly.py classification
(readings C6-C8, C17)."""
import itertools

import numpy as np
import pytest

import sc_inputs
from oracle.geometry import (is_physical, build_tree, lattice_coord, UNCUT, CUT, EMPTY,
                             leaf_gauss_points)
from oracle.assembly import classify, make_grid
from oracle.basis import gauss_rule


def test_membership_closed_domain():
    circ = [{"kind": "ellipsoid", "c": [0.0, 0.0, 0.0], "A": [1.0, 1.0, 0.0, 0.0, 0.0, 0.0]}]
    X = np.array([[0, 0, 0], [1, 0, 0], [0.5, 0.5, 0], [2, 0, 0], [0, -1, 0]], dtype=float)
    # centre: void; on the circle (q == 1): physical (closed Omega_p); outside: physical
    assert list(is_physical(X, circ)) == [False, True, False, True, True]
    hs = [{"kind": "halfspace", "n": [0.0, 1.0, 0.0], "b": 0.5}]
    X = np.array([[0, 0.5, 0], [0, 0.5000001, 0], [0, 0.2, 0]])
    assert list(is_physical(X, hs)) == [True, False, True]
    # rotated ellipse: A from R diag(1/a^2, 1/b^2) R^T, point on the major axis
    th = 0.3
    R = np.array([[np.cos(th), -np.sin(th)], [np.sin(th), np.cos(th)]])
    A = R @ np.diag([1 / 0.04, 1 / 0.01]) @ R.T
    v = [{"kind": "ellipsoid", "c": [0.5, 0.5, 0], "A": [A[0, 0], A[1, 1], 0, A[0, 1], 0, 0]}]
    on_major_in = 0.5 + 0.19 * np.array([np.cos(th), np.sin(th)])
    on_major_out = 0.5 + 0.21 * np.array([np.cos(th), np.sin(th)])
    on_minor_out = 0.5 + 0.11 * np.array([-np.sin(th), np.cos(th)])
    X = np.array([[*on_major_in, 0], [*on_major_out, 0], [*on_minor_out, 0]])
    assert list(is_physical(X, v)) == [False, True, True]


def test_lattice_coordinate_dyadic_consistency():
    # same rational at two levels -> identical double (one rounding of m/den)
    for m in range(0, 257):
        a = lattice_coord(0.0, 1.0, m, 256)
        b = lattice_coord(0.0, 1.0, 2 * m, 512)
        assert a == b


def _grid1():
    return {"dim": 2, "cells": [1, 1], "lo": [0.0, 0.0], "hi": [1.0, 1.0], "s": 4}


def test_tree_uncut_and_halfcut_by_hand():
    g = _grid1()
    lv, a, root = build_tree(g, [], (0, 0), 3)
    assert root == "phys" and len(lv) == 1 and lv[0] == 0
    # void y > 0.3: lattice spacing 1/4 at level 0 -> mixed; level-1 nodes with
    # y-range [0,0.5] are mixed (0.3 strictly inside), [0.5,1] fictitious
    hs = [{"kind": "halfspace", "n": [0.0, 1.0, 0.0], "b": 0.3}]
    lv, a, root = build_tree(g, hs, (0, 0), 2)
    assert root == "mixed"
    # level 1: 2 fictitious leaves (top row), 2 mixed -> level 2: each mixed
    # level-1 node y in [0,0.5] has 4 children: y in [0,0.25] phys, [0.25,0.5] mixed
    # -> at depth D=2 mixed nodes are leaves: 2 + 2*4 = 10 leaves
    assert len(lv) == 10
    assert np.sum(lv == 1) == 2 and np.sum(lv == 2) == 8
    # leaves tile the cell exactly
    assert abs(np.sum(0.25 ** lv) - 1.0) < 1e-15


@pytest.mark.parametrize("depth", [2, 4, 6, 8])
def test_fill_ratio_converges(depth):
    # fraction of physical Gauss weight of a half-plane cut at y = 0.3141 -> 0.3141
    g = _grid1()
    hs = [{"kind": "halfspace", "n": [0.0, 1.0, 0.0], "b": 0.3141}]
    lv, a, _ = build_tree(g, hs, (0, 0), depth)
    gx, gw = gauss_rule(4)
    X = leaf_gauss_points(g, (0, 0), lv, a, gx)
    ph = is_physical(X, hs).reshape(len(lv), 16)
    wq = np.kron(gw, gw) / 4.0
    eta = np.sum(ph * wq[None, :] * (0.25 ** lv)[:, None])
    assert abs(eta - 0.3141) <= 0.5 ** depth / 2 + 1e-12


def _brute_force_partition(cfg, cl):
    """Independent support scan: for each lattice node, visit every
    cell in the box and test whether the node lies on that cell."""
    d, p = cfg["dim"], cfg["p"]
    N = cfg["cells"]
    n = [N[k] * p + 1 for k in range(d)]
    retained, is_c = [], []
    for lat in range(int(np.prod(n))):
        ijk, rem = [], lat
        for k in range(d):
            ijk.append(rem % n[k])
            rem //= n[k]
        ne, cut = False, False
        for cell in itertools.product(*[range(N[k]) for k in range(d)]):
            if all(cell[k] * p <= ijk[k] <= cell[k] * p + p for k in range(d)):
                ci = sum(cell[k] * int(np.prod(N[:k])) for k in range(d))
                ne |= cl.cell_class[ci] != EMPTY
                cut |= cl.cell_class[ci] == CUT
        retained.append(ne)
        is_c.append(cut)
    return np.array(retained), np.array(is_c)


@pytest.mark.parametrize("case", ["circle2d", "halfspace_face", "config1", "sphere3d"])
def test_partition_brute_force(case):
    if case == "circle2d":
        cfg = sc_inputs.small_config(2, [6, 5], 2, voids=[{"kind": "ellipsoid", "c": [0.45, 0.5, 0],
                                     "A": [1 / 0.09, 1 / 0.09, 0, 0, 0, 0]}], depth=2)
    elif case == "halfspace_face":
        # void boundary exactly on a cell face: the empty cells' neighbours
        cfg = sc_inputs.small_config(2, [4, 3], 2, voids=[{"kind": "halfspace", "n": [1.0, 0, 0],
                                     "b": 0.75}], depth=2)
    elif case == "config1":
        cfg = sc_inputs.get_config(1)
    else:
        cfg = sc_inputs.small_config(3, [3, 3, 2], 2, voids=[{"kind": "ellipsoid", "c": [0.5, 0.5, 0.5],
                                     "A": [1 / 0.1, 1 / 0.1, 1 / 0.1, 0, 0, 0]}], depth=1)
    cl = classify(cfg)
    ret, isc = _brute_force_partition(cfg, cl)
    assert np.array_equal(np.nonzero(ret)[0], cl.lattice_index)
    assert np.array_equal(isc[cl.lattice_index], cl.is_c)
    assert cl.n_dof == ret.sum()


def test_config1_counts():
    # reading C8: x = 0.937 lies in cell 29 (cut); cells 30-31 are empty and
    # discarded: n_dof = 121, n_c = 5, n_d = 116
    cl = classify(sc_inputs.get_config(1))
    assert list(cl.cell_class[28:]) == [UNCUT, CUT, EMPTY, EMPTY]
    assert cl.n_dof == 121 and cl.is_c.sum() == 5 and (~cl.is_c).sum() == 116


def test_dof_counts_tiny_meshes():
    # 2x1 cells p=1 -> 6 DOFs; 1x1 cell p=3 -> 16 DOFs
    assert classify(sc_inputs.small_config(2, [2, 1], 1)).n_dof == 6
    assert classify(sc_inputs.small_config(2, [1, 1], 3)).n_dof == 16


def test_config2_counts():
    # cross-check (prototype; all coordinates dyadic)
    cl = classify(sc_inputs.get_config(2))
    assert list(np.bincount(cl.cell_class, minlength=3)) == [3536, 92, 468]
    assert cl.n_dof == 58752 and cl.is_c.sum() == 1872


def test_empty_cell_threshold_reading():
    # C7: at the configs' depths a cell with >= 1 physical Gauss point has eta >> 1e-10,
    # so "eta < 1e-10" <=> "no physical Gauss point".  Smallest possible eta:
    # one Gauss weight of one depth-D leaf.
    for d, p, D in [(1, 4, 3), (2, 4, 3), (3, 3, 2), (3, 4, 2)]:
        _, w = gauss_rule(p + 1)
        eta_min = (w.min() / 2.0) ** d / (2 ** D) ** d
        assert eta_min > 1e-10
