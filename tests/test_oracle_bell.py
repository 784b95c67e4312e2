"""Pins of the oracle's Gaussian-bell load (oracle.assembly.bell_load, Eq.
eq:fx, f_x = amp exp(-|x - x_s|^2 / (2 sigma^2)), assembled as f_i = int alpha f_x N_i):
* partition of unity: sum_i f_i = int alpha f_x over the non-empty cells; on an all-uncut box
  with the bell well inside, that is the closed form amp (2 pi sigma^2)^(d/2) up to the
  quadrature error of the resolved bell (tight for sigma of a few cells);
* brute force: every f_i against an independent tensor quadrature of N_i f_x on each incident
  cell with 3x more Gauss points (scipy-free, numpy.polynomial Gauss rule);
* alpha scaling inside a void (a half-space void over half the box scales that half by alpha)."""
import numpy as np

import sc_inputs
from oracle.assembly import build_system, node_coords


def _cfg(voids, sigma=0.12, xs=(0.5, 0.5), cells=(8, 8), p=3):
    cfg = sc_inputs.small_config(2, list(cells), p, voids=voids, depth=3, alpha=1e-6, steps=1,
                                 source={"kind": "bell", "x": [xs[0], xs[1], 0.0], "sigma": sigma, "amp": 10.0})
    cfg["dt"] = 1e-3
    return cfg


def test_bell_total_is_closed_form():
    import math
    sig = 0.12
    sysm = build_system(_cfg([], sigma=sig, cells=(16, 16)), "sparse")
    total = sysm.f_x.sum()
    # int over [0,1]^2 of the bell = amp 2 pi sigma^2 prod_k [Phi((1 - x_k)/sigma) - Phi(-x_k/sigma)]
    Phi = lambda z: 0.5 * math.erfc(-z / math.sqrt(2.0))   # noqa: E731
    exact = 10.0 * 2.0 * math.pi * sig ** 2 * (Phi(0.5 / sig) - Phi(-0.5 / sig)) ** 2
    assert abs(total - exact) / exact < 1e-7, (total, exact)


def test_bell_entries_brute_force():
    cfg = _cfg([], sigma=0.15, xs=(0.42, 0.55), cells=(5, 4), p=2)
    sysm = build_system(cfg, "sparse")
    from oracle.basis import gll_rule, lagrange
    nodes, _ = gll_rule(2)
    xg, wg = np.polynomial.legendre.leggauss(12)
    h = [1.0 / 5, 1.0 / 4]
    f = np.zeros(sysm.n_dof)
    for cy in range(4):
        for cx in range(5):
            X0 = cx * h[0] + (xg + 1) * 0.5 * h[0]
            Y0 = cy * h[1] + (xg + 1) * 0.5 * h[1]
            vx, _ = lagrange(nodes, xg)
            vy, _ = lagrange(nodes, xg)
            F = 10.0 * np.exp(-((X0[None, :] - 0.42) ** 2 + (Y0[:, None] - 0.55) ** 2) / (2 * 0.15 ** 2))
            W = np.outer(wg, wg) * h[0] * h[1] / 4.0
            for j in range(3):
                for i in range(3):
                    val = np.sum(W * F * np.outer(vy[:, j], vx[:, i]))
                    lat = (cx * 2 + i) + 11 * (cy * 2 + j)
                    f[sysm.cl.dof_of_lattice[lat]] += val
    # (p+1)-point Gauss vs 12-point: the quadrature error of a smooth bell at sigma = 0.75 h
    assert np.max(np.abs(sysm.f_x - f)) / np.max(np.abs(f)) < 2e-3
    assert np.linalg.norm(sysm.f_x - f) / np.linalg.norm(f) < 2e-3


def test_bell_alpha_scaling_in_void():
    # half-space void x > 0.5 on a cell face: the nodes strictly inside it are scaled by alpha
    cfg0 = _cfg([], xs=(0.5, 0.5))
    cfg1 = _cfg([{"kind": "halfspace", "n": [1.0, 0.0, 0.0], "b": 0.5}], xs=(0.5, 0.5))
    s0, s1 = build_system(cfg0, "sparse"), build_system(cfg1, "sparse")
    X0 = node_coords(cfg0, s0.cl.lattice_index)
    X1 = node_coords(cfg1, s1.cl.lattice_index)
    left0 = s0.f_x[X0[:, 0] < 0.5 - 1e-12]
    left1 = s1.f_x[X1[:, 0] < 0.5 - 1e-12]
    assert np.allclose(left0, left1, rtol=1e-13, atol=0)
