"""Pins of oracle/elements.py and oracle/assembly.py (PAPER.md P:444-463,
P:466-543; Fig. 2; reading C5)."""
import os

import numpy as np
import numpy.polynomial.polynomial as P
import pytest

import sc_inputs
from oracle.basis import gll_rule, lagrange
from oracle.elements import uncut_element, cut_element
from oracle.geometry import build_tree
from oracle.assembly import classify, build_system, dense_brute_force, K_apply
from oracle.spectra import fill_ratio_cell_omega

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def test_uncut_1d_p1_hand():
    # M_e = diag(h/2, h/2), K_e = (1/h)[[1,-1],[-1,1]]
    h = 0.3
    Me, Ke = uncut_element(1, [h], 1.0, 1.0)
    assert np.allclose(Me, [h / 2, h / 2], rtol=1e-15)
    assert np.allclose(Ke, np.array([[1, -1], [-1, 1]]) / h, rtol=1e-14)


@pytest.mark.parametrize("d,p", [(1, 4), (2, 2), (2, 4), (3, 2), (3, 3)])
def test_uncut_properties(d, p):
    h = [0.1 * (k + 1) for k in range(d)]
    rho, c = 2.0, 3.0
    Me, Ke = uncut_element(p, h, rho, c)
    assert abs(Me.sum() - rho * np.prod(h)) < 1e-13        # mass = rho * volume
    assert np.allclose(Ke.sum(axis=1), 0, atol=1e-10 * abs(Ke).max())  # K 1 = 0
    assert np.allclose(Ke, Ke.T)
    # energy of the linear field u = x: int rho c^2 |grad u|^2 = rho c^2 vol
    nodes, _ = gll_rule(p)
    loc = (nodes + 1) / 2 * h[0]
    u = np.kron(np.ones((p + 1) ** (d - 1)), loc) if d > 1 else loc
    assert abs(u @ Ke @ u - rho * c * c * np.prod(h)) < 1e-11


def _poly_int_matrix(nodes, a, b):
    """Exact int_a^b l_i l_j dxi and int_a^b l_i' l_j' dxi by polynomial
    algebra (numpy.polynomial), independent of the quadrature routines."""
    n = len(nodes)
    polys = []
    for i in range(n):
        c = np.array([1.0])
        for j in range(n):
            if j != i:
                c = P.polymul(c, np.array([-nodes[j], 1.0]) / (nodes[i] - nodes[j]))
        polys.append(c)
    M = np.zeros((n, n))
    K = np.zeros((n, n))
    for i in range(n):
        for j in range(n):
            m = P.polyint(P.polymul(polys[i], polys[j]))
            k = P.polyint(P.polymul(P.polyder(polys[i]), P.polyder(polys[j])))
            M[i, j] = P.polyval(b, m) - P.polyval(a, m)
            K[i, j] = P.polyval(b, k) - P.polyval(a, k)
    return M, K


@pytest.mark.parametrize("p", [1, 2, 3])
def test_cut_element_half_split_exact(p):
    # unit square cut at y = 0.5 (a leaf boundary): the spacetree integral is
    # exact and equals M_low + alpha M_up with polynomial integrals over the
    # reference halves xi_y in [-1,0] and [0,1].
    g = {"dim": 2, "cells": [1, 1], "lo": [0.0, 0.0], "hi": [1.0, 1.0], "s": 4}
    voids = [{"kind": "halfspace", "n": [0.0, 1.0, 0.0], "b": 0.5}]
    lv, a, _ = build_tree(g, voids, (0, 0), 3)
    alpha = 1e-3
    Me, Ke = cut_element(g, voids, (0, 0), lv, a, p, alpha, 1.0, 1.0)
    nodes, _ = gll_rule(p)
    Mf, Kf = _poly_int_matrix(nodes, -1.0, 1.0)
    Ml, Kl = _poly_int_matrix(nodes, -1.0, 0.0)
    Mu, Ku = _poly_int_matrix(nodes, 0.0, 1.0)
    J = 0.25      # (h/2)^2 with h = 1
    Me_ref = J * (np.kron(Ml, Mf) + alpha * np.kron(Mu, Mf))
    # grad in physical coords: (2/h)^2 J = 1
    Ke_ref = np.kron(Ml, Kf) + np.kron(Kl, Mf) + alpha * (np.kron(Mu, Kf) + np.kron(Ku, Mf))
    assert np.allclose(Me, Me_ref, rtol=1e-12, atol=1e-15)
    assert np.allclose(Ke, Ke_ref, rtol=1e-12, atol=1e-14)


@pytest.mark.parametrize("d,p", [(2, 2), (3, 2)])
def test_cut_element_alpha_one_equals_consistent(d, p):
    # with alpha = 1 the spacetree Gauss rule integrates the polynomial
    # integrands exactly -> consistent full-cell matrices; K equals the uncut K
    cells = [1] * d
    g = {"dim": d, "cells": cells, "lo": [0.0] * d, "hi": [0.5] * d, "s": 4}
    voids = [{"kind": "ellipsoid", "c": [0.2, 0.3, 0.25 if d == 3 else 0.0], "A": [1 / 0.01] * 3 + [0, 0, 0]}]
    lv, a, root = build_tree(g, voids, (0,) * d, 2)
    assert root == "mixed"
    Me, Ke = cut_element(g, voids, (0,) * d, lv, a, p, 1.0, 1.0, 1.0)
    _, Ke_u = uncut_element(p, [0.5] * d, 1.0, 1.0)
    nodes, _ = gll_rule(p)
    Mf, _ = _poly_int_matrix(nodes, -1.0, 1.0)
    Mref = Mf * 0.25
    for _ in range(d - 1):
        Mref = np.kron(Mf * 0.25, Mref)
    assert np.allclose(Me, Mref, rtol=1e-12)
    assert np.allclose(Ke, Ke_u, rtol=1e-11, atol=1e-13)


def _fig2_rows():
    rows = []
    for line in open(os.path.join(GOLD, "fig2_fill_ratio.txt")):
        if line.startswith("#") or not line.strip():
            continue
        p, eta, om = line.split()[:3]
        rows.append((int(p), float(eta), float(om)))
    return rows


@pytest.mark.parametrize("p", [1, 2, 3])
def test_fig2_fill_ratio_table(p):
    """P3: all 33 (eta, omega) points of Fig. 2 for order p, depth 13."""
    rows = [r for r in _fig2_rows() if r[0] == p]
    assert len(rows) == 33
    tol = {1: 1e-11, 2: 1e-9, 3: 1e-9}[p]
    worst = 0.0
    for _, eta, om in rows:
        w = fill_ratio_cell_omega(eta, p, depth=13)
        worst = max(worst, abs(w - om) / om)
    assert worst < tol, worst


@pytest.mark.parametrize("case", ["circle", "halfspace_face", "sphere3d", "config1"])
def test_assembly_vs_dense_brute_force(case):
    """P4: sparse assembly == brute-force dense assembly; K symmetric, K 1 = 0,
    M^dc = 0, M^dd diagonal; ebe K application == sparse K."""
    if case == "circle":
        cfg = sc_inputs.small_config(2, [4, 4], 3, voids=[{"kind": "ellipsoid", "c": [0.55, 0.45, 0],
                                     "A": [1 / 0.06, 1 / 0.06, 0, 0, 0, 0]}], depth=2, alpha=1e-4)
    elif case == "halfspace_face":
        cfg = sc_inputs.small_config(2, [4, 2], 2, voids=[{"kind": "halfspace", "n": [1.0, 0, 0], "b": 0.75}])
    elif case == "sphere3d":
        cfg = sc_inputs.small_config(3, [3, 2, 2], 2, voids=[{"kind": "ellipsoid", "c": [0.5, 0.5, 0.5],
                                     "A": [1 / 0.08, 1 / 0.08, 1 / 0.08, 0, 0, 0]}], depth=1)
    else:
        cfg = sc_inputs.get_config(1)
    cl = classify(cfg)
    s = build_system(cfg, "sparse", cl=cl)
    M, K = dense_brute_force(cfg, cl=cl)
    assert np.allclose(s.K.toarray(), K, rtol=1e-13, atol=1e-13 * abs(K).max())
    assert np.allclose(s.M.toarray(), M, rtol=1e-13, atol=1e-16)
    assert np.allclose(K, K.T, atol=1e-12 * abs(K).max())
    assert np.allclose(K @ np.ones(len(K)), 0, atol=1e-10 * abs(K).max())
    Id, Ic = s.I_d, s.I_c
    assert np.all(M[np.ix_(Id, Ic)] == 0)
    Mdd = M[np.ix_(Id, Id)]
    assert np.all(Mdd[~np.eye(len(Id), dtype=bool)] == 0)
    assert np.allclose(s.M_dd, np.diag(Mdd), rtol=1e-14)
    assert np.allclose(s.M_cc.toarray(), M[np.ix_(Ic, Ic)], rtol=1e-13, atol=1e-16)
    assert np.allclose(s.K_cc.toarray(), K[np.ix_(Ic, Ic)], rtol=1e-13, atol=1e-13 * abs(K).max())
    e = build_system(cfg, "ebe", cl=cl)
    u = np.random.default_rng(0).standard_normal(s.n_dof)
    assert np.allclose(K_apply(e, u), K @ u, rtol=1e-12, atol=1e-12 * abs(K @ u).max())


def test_mass_conservation_config2():
    # sum M = int alpha rho; quadtree-resolved circle: 1 - pi 0.04 (1 - 1e-5)
    s = build_system(sc_inputs.get_config(2), "sparse")
    exact = 1 - np.pi * 0.04 * (1 - 1e-5)
    assert abs(s.M.sum() - exact) < 2e-6
