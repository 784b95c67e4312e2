"""Critical time steps and the single-cut-cell study (ORACLE - test infra only).

PAPER.md P:63-71 (§Critical time step analysis): dt_crit = 2 / omega_max,
omega_max = sqrt(lambda_max(K, M)) of the generalized eigenproblem.
P:869: the cell-wise critical step of the uncut cells is a cheap, good
estimate of the IMEX critical step (Table tab:criticaltimestepsizes,
P:872-890).  P:73-90 + Fig. fig:fillRatioHZ: one unit cell cut by
a horizontal line at height eta, rho_p = c_p = 1, rho_f = 1e-6, c_f = 1,
p = 1..3, quadtree depth 13; the plotted quantity is omega = sqrt(lambda_max)
(reading C18: the axis label says Hz, the values are rad/s; eta = 1 for
p = 1 gives exactly 2).
"""
import numpy as np
import scipy.linalg as sla

from .elements import uncut_element, cut_element
from .geometry import build_tree, classify_cell, UNCUT
from .basis import gauss_rule


def lambda_max(K, M):
    """Largest generalized eigenvalue of (K, M) (dense; library eigh)."""
    K = np.asarray(K.todense() if hasattr(K, "todense") else K)
    M = np.asarray(M.todense() if hasattr(M, "todense") else M)
    if M.ndim == 1:
        M = np.diag(M)
    w = sla.eigh(K, M, eigvals_only=True)
    return float(w[-1])


def dt_crit(K, M):
    return 2.0 / np.sqrt(lambda_max(K, M))


def dt_crit_uncut(dim, p, h, rho=1.0, c=1.0):
    """Cell-wise critical step of an uncut cell."""
    Me, Ke = uncut_element(p, [h] * dim, rho, c)
    return dt_crit(Ke, Me)


def fill_ratio_cell_omega(eta, p, depth=13, rho_f=1e-6, s=4):
    """omega_max of the unit square [0,1]^2 cut by the line y = eta
    (physical below, fictitious above), Fig. 2."""
    grid = {"dim": 2, "cells": [1, 1], "lo": [0.0, 0.0], "hi": [1.0, 1.0], "s": s}
    voids = [{"kind": "halfspace", "n": [0.0, 1.0, 0.0], "b": float(eta)}]
    g, _ = gauss_rule(p + 1)
    cls, levels, a, ph = classify_cell(grid, voids, (0, 0), depth, g)
    if cls == UNCUT:
        Me, Ke = uncut_element(p, [1.0, 1.0], 1.0, 1.0)
        return float(np.sqrt(lambda_max(Ke, Me)))
    Me, Ke = cut_element(grid, voids, (0, 0), levels, a, p, rho_f, 1.0, 1.0, phys=ph)
    return float(np.sqrt(lambda_max(Ke, Me)))


__all__ = ["lambda_max", "dt_crit", "dt_crit_uncut", "fill_ratio_cell_omega", "build_tree"]


def cell_dt_map(sysm, which="consistent"):
    """Cell-wise critical time steps (Fig. fig:tCritsCircles, Table
    tab:criticaltimestepsizes): dt_e = 2 / sqrt(lambda_max(K_e, M_e)) per cell, cells x
    fastest; uncut cells with their GLL-lumped mass, cut cells with the consistent mass
    (which="consistent") or the HRZ-lumped mass (which="hrz"); empty cells 0."""
    from .assembly import hrz_element
    from .geometry import UNCUT, CUT
    cl = sysm.cl
    out = np.zeros(len(cl.cell_class))
    out[cl.cell_class == UNCUT] = dt_crit(sysm.Ke_uncut, sysm.Me_uncut)
    cut = np.nonzero(cl.cell_class == CUT)[0]
    for k, ci in enumerate(cut):
        Me = sysm.cut_M[k]
        if which == "hrz":
            Me = hrz_element(Me)
        out[ci] = dt_crit(sysm.cut_K[k], Me)
    return out
