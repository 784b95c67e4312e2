"""DOF map, partition, global M and K, point-source load (ORACLE - test infra only).

PAPER.md P:401-416 (C0 spectral basis on the GLL lattice)
(M u'' + K u = f_t(t) f_x), P:466-543 (§Partitioning of the Degrees of
Freedom: a DOF is 'd' iff all its supporting cells are uncut, else 'c';
M = diag(M^dd, M^cc) with M^dd diagonal; K = [[K^dd, K^dc],[K^cd, K^cc]]),
P:866 (empty cells are discarded: the DOF set is the lattice nodes of the
non-empty cells).

Canonical DOF order: retained lattice nodes, lexicographic, x fastest;
lattice index = i + n0*(j + n1*k), n_k = N_k*p + 1.

Two assembly modes with identical arithmetic meaning:
* ``mode="sparse"``: global scipy CSR M and K assembled explicitly
  (configs 1-3, brute-force tests);
* ``mode="ebe"``: element-by-element K application (dense K_e per element,
  batched), for grids whose global K is too large to store (configs 4-5).
In both modes the c-blocks M^cc, K^cc (and S) are assembled explicitly.
"""
import numpy as np
import scipy.sparse as sp

from .basis import gll_rule, gauss_rule
from .geometry import (UNCUT, CUT, EMPTY, root_all_physical, classify_cell,
                       is_physical)
from .elements import uncut_element, cut_element, eval_basis_at, cell_bounds


def make_grid(cfg):
    return {"dim": cfg["dim"], "cells": list(cfg["cells"]), "lo": list(cfg["lo"]),
            "hi": list(cfg["hi"]), "s": cfg["lattice_s"]}


def cell_index_array(grid):
    d = grid["dim"]
    N = grid["cells"]
    n_cells = int(np.prod(N))
    idx = np.arange(n_cells)
    out = np.zeros((n_cells, d), dtype=np.int64)
    for k in range(d):
        out[:, k] = idx % N[k]
        idx = idx // N[k]
    return out


def element_nodes(grid, p, cell_idx):
    """Lattice indices of the (p+1)^d local nodes (x fastest) of each cell."""
    d = grid["dim"]
    n = [grid["cells"][k] * p + 1 for k in range(d)]
    loc = np.arange(p + 1)
    stride = [1, n[0], n[0] * (n[1] if d > 1 else 1)]
    out = np.zeros((len(cell_idx),) + (p + 1,) * d, dtype=np.int64)
    for k in range(d):
        shp = [1] * (d + 1)
        shp[0] = len(cell_idx)
        shp[d - k] = p + 1
        comp = ((cell_idx[:, k] * p)[:, None] + loc[None, :]) * stride[k]
        out = out + comp.reshape([len(cell_idx)] + [p + 1 if j == d - 1 - k else 1 for j in range(d)])
    return out.reshape(len(cell_idx), -1)


class Classification:
    pass


def classify(cfg):
    """Cell classes (UNCUT/CUT/EMPTY, int8, cells x fastest), spacetree leaves
    of the non-uncut cells, DOF map and d/c partition (C6-C8)."""
    grid = make_grid(cfg)
    p = cfg["p"]
    g, _ = gauss_rule(p + 1)
    allphys, cidx = root_all_physical(grid, cfg["voids"])
    cls = np.full(len(allphys), UNCUT, dtype=np.int8)
    trees = {}
    for ci in np.nonzero(~allphys)[0]:
        c, levels, a, ph = classify_cell(grid, cfg["voids"], cidx[ci], cfg["tree_depth"], g)
        cls[ci] = c
        trees[int(ci)] = (levels, a, ph)
    out = Classification()
    out.grid = grid
    out.cell_class = cls
    out.cell_idx = cidx
    out.trees = trees
    out.enodes = element_nodes(grid, p, cidx)
    n_lat = int(np.prod([grid["cells"][k] * p + 1 for k in range(grid["dim"])]))
    retained = np.zeros(n_lat, dtype=bool)
    retained[out.enodes[cls != EMPTY].ravel()] = True
    is_c_lat = np.zeros(n_lat, dtype=bool)
    is_c_lat[out.enodes[cls == CUT].ravel()] = True
    out.lattice_index = np.nonzero(retained)[0]
    out.n_dof = len(out.lattice_index)
    dof_of = np.full(n_lat, -1, dtype=np.int64)
    dof_of[out.lattice_index] = np.arange(out.n_dof)
    out.dof_of_lattice = dof_of
    out.is_c = is_c_lat[out.lattice_index]
    out.n_lattice = n_lat
    return out


class System:
    pass


def node_coords(cfg, lattice_index):
    """Physical coordinates of lattice nodes (for nodal interpolation, C16)."""
    d = cfg["dim"]
    p = cfg["p"]
    nodes, _ = gll_rule(p)
    n = [cfg["cells"][k] * p + 1 for k in range(d)]
    X = np.zeros((len(lattice_index), 3))
    rem = np.asarray(lattice_index).copy()
    for k in range(d):
        ik = rem % n[k]
        rem //= n[k]
        e = np.minimum(ik // p, cfg["cells"][k] - 1)
        loc = ik - e * p
        h = (cfg["hi"][k] - cfg["lo"][k]) / cfg["cells"][k]
        X[:, k] = cfg["lo"][k] + h * (e + (nodes[loc] + 1.0) * 0.5)
    return X


def point_load(cfg, cl, x):
    """f_x,i = alpha(x_s) N_i(x_s), evaluated in the lowest-index non-empty
    cell containing x_s (P:456-459 separable load, reading C11)."""
    d = cfg["dim"]
    grid = cl.grid
    cand = []
    for k in range(d):
        ks = []
        for e in range(grid["cells"][k]):
            lo_e = grid["lo"][k] + (grid["hi"][k] - grid["lo"][k]) * (np.float64(e) / grid["cells"][k])
            hi_e = grid["lo"][k] + (grid["hi"][k] - grid["lo"][k]) * (np.float64(e + 1) / grid["cells"][k])
            if lo_e <= x[k] <= hi_e:
                ks.append(e)
        cand.append(ks)
    cells = [()]
    for k in range(d):
        cells = [c + (e,) for c in cells for e in cand[k]]
    N = grid["cells"]

    def lin(c):
        s, m = 0, 1
        for k in range(d):
            s += c[k] * m
            m *= N[k]
        return s
    cells.sort(key=lin)
    f = np.zeros(cl.n_dof)
    for c in cells:
        ci = lin(c)
        if cl.cell_class[ci] == EMPTY:
            continue
        X = np.zeros((1, 3))
        X[0, :d] = x[:d]
        alpha_s = 1.0 if is_physical(X, cfg["voids"])[0] else cfg["alpha"]
        vals = eval_basis_at(grid, c, np.asarray(x[:d], dtype=np.float64), cfg["p"])
        f[cl.dof_of_lattice[cl.enodes[ci]]] += alpha_s * vals
        return f
    raise ValueError("source point is outside every non-empty cell")


def bell_load(cfg, cl):
    """f_x,i = int alpha f_x N_i for the Gaussian bell f_x of PAPER.md P:851-853 (Eq. eq:fx),
    amp exp(-|x - x_s|^2 / (2 sigma^2)), assembled over every non-empty cell (Gauss points on
    the spacetree leaves of cut cells)."""
    from .elements import cell_load, gaussian_bell
    src = cfg["source"]
    d = cfg["dim"]
    xs = np.asarray(src["x"][:d], dtype=np.float64)
    fx = lambda X: gaussian_bell(X, xs, src["sigma"], src["amp"])   # noqa: E731
    grid = cl.grid
    f = np.zeros(cl.n_dof)
    root = (np.zeros((1,), dtype=np.int64), np.zeros((1, d), dtype=np.int64))
    for ci in range(len(cl.cell_class)):
        if cl.cell_class[ci] == EMPTY:
            continue
        cell = cl.cell_idx[ci]
        if cl.cell_class[ci] == UNCUT:
            fe = cell_load(grid, cfg["voids"], cell, root[0], root[1], cfg["p"], cfg["alpha"], fx,
                           phys=np.ones((cfg["p"] + 1) ** d, dtype=bool))
        else:
            levels, a, ph = cl.trees[int(ci)]
            fe = cell_load(grid, cfg["voids"], cell, levels, a, cfg["p"], cfg["alpha"], fx, phys=ph)
        np.add.at(f, cl.dof_of_lattice[cl.enodes[ci]], fe)
    return f


def point_values(cfg, cl, x):
    """Receiver weights: u(x) = sum_i N_i(x) u_i with the basis of the lowest-index
    non-empty cell containing x (the evaluation point_load uses, without alpha; SURVEY
    NEXT-3, the paper's receiver traces P:1758-1765)."""
    d = cfg["dim"]
    grid = cl.grid
    cand = []
    for k in range(d):
        ks = []
        for e in range(grid["cells"][k]):
            lo_e = grid["lo"][k] + (grid["hi"][k] - grid["lo"][k]) * (np.float64(e) / grid["cells"][k])
            hi_e = grid["lo"][k] + (grid["hi"][k] - grid["lo"][k]) * (np.float64(e + 1) / grid["cells"][k])
            if lo_e <= x[k] <= hi_e:
                ks.append(e)
        cand.append(ks)
    cells = [()]
    for k in range(d):
        cells = [c + (e,) for c in cells for e in cand[k]]
    N = grid["cells"]
    cells.sort(key=lambda c: sum(c[k] * int(np.prod(N[:k])) for k in range(d)))
    for c in cells:
        ci = sum(c[k] * int(np.prod(N[:k])) for k in range(d))
        if cl.cell_class[ci] == EMPTY:
            continue
        w = np.zeros(cl.n_dof)
        w[cl.dof_of_lattice[cl.enodes[ci]]] += eval_basis_at(grid, c, np.asarray(x[:d], dtype=np.float64), cfg["p"])
        return w
    raise ValueError("point outside every non-empty cell")


def build_system(cfg, mode="sparse", cl=None):
    """Assemble the partitioned system of P:449-543 for the input dict."""
    if cl is None:
        cl = classify(cfg)
    d = cfg["dim"]
    p = cfg["p"]
    rho, c, alpha = cfg["rho"], cfg["c"], cfg["alpha"]
    grid = cl.grid
    h = [(grid["hi"][k] - grid["lo"][k]) / grid["cells"][k] for k in range(d)]
    Me_u, Ke_u = uncut_element(p, h, rho, c)
    nb = (p + 1) ** d
    sysm = System()
    sysm.cfg = cfg
    sysm.cl = cl
    sysm.n_dof = cl.n_dof
    sysm.I_c = np.nonzero(cl.is_c)[0]
    sysm.I_d = np.nonzero(~cl.is_c)[0]
    sysm.Ke_uncut = Ke_u
    sysm.Me_uncut = Me_u
    uncut = np.nonzero(cl.cell_class == UNCUT)[0]
    cut = np.nonzero(cl.cell_class == CUT)[0]
    sysm.uncut_dofs = cl.dof_of_lattice[cl.enodes[uncut]]
    sysm.cut_dofs = cl.dof_of_lattice[cl.enodes[cut]]
    cut_M, cut_K = [], []
    for ci in cut:
        levels, a, ph = cl.trees[int(ci)]
        Me, Ke = cut_element(grid, cfg["voids"], cl.cell_idx[ci], levels, a, p, alpha, rho, c, phys=ph)
        cut_M.append(Me)
        cut_K.append(Ke)
    sysm.cut_M = np.array(cut_M).reshape(len(cut), nb, nb)
    sysm.cut_K = np.array(cut_K).reshape(len(cut), nb, nb)
    n = cl.n_dof
    # diagonal of the mass from uncut cells (nodal lumping) + consistent cut mass
    mdiag = np.bincount(sysm.uncut_dofs.ravel(), weights=np.tile(Me_u, len(uncut)), minlength=n)
    sysm.M_dd = mdiag[sysm.I_d]
    # explicit c-blocks
    pos_c = np.full(n, -1, dtype=np.int64)
    pos_c[sysm.I_c] = np.arange(len(sysm.I_c))
    sysm.pos_c = pos_c
    nc = len(sysm.I_c)
    rows, cols, mv, kv = [], [], [], []
    # uncut elements touching c nodes: lumped mass diag + stiffness c-c entries
    tc = np.nonzero((pos_c[sysm.uncut_dofs] >= 0).any(axis=1))[0]
    for e in tc:
        dofs = sysm.uncut_dofs[e]
        pc = pos_c[dofs]
        m = pc >= 0
        ii, jj = np.meshgrid(pc[m], pc[m], indexing="ij")
        rows.append(ii.ravel())
        cols.append(jj.ravel())
        kv.append(Ke_u[np.ix_(m, m)].ravel())
        mv.append(np.diag(Me_u[m]).ravel())
    for e in range(len(cut)):
        pc = pos_c[sysm.cut_dofs[e]]
        ii, jj = np.meshgrid(pc, pc, indexing="ij")
        rows.append(ii.ravel())
        cols.append(jj.ravel())
        kv.append(sysm.cut_K[e].ravel())
        mv.append(sysm.cut_M[e].ravel())
    if nc:
        rows = np.concatenate(rows)
        cols = np.concatenate(cols)
        sysm.M_cc = sp.csr_matrix((np.concatenate(mv), (rows, cols)), shape=(nc, nc))
        sysm.K_cc = sp.csr_matrix((np.concatenate(kv), (rows, cols)), shape=(nc, nc))
    else:
        sysm.M_cc = sp.csr_matrix((0, 0))
        sysm.K_cc = sp.csr_matrix((0, 0))
    sysm.mode = mode
    if mode == "sparse":
        r = [np.repeat(sysm.uncut_dofs, nb, axis=1).ravel()]
        cc = [np.tile(sysm.uncut_dofs, (1, nb)).ravel()]
        v = [np.tile(Ke_u.ravel(), len(uncut))]
        if len(cut):
            r.append(np.repeat(sysm.cut_dofs, nb, axis=1).ravel())
            cc.append(np.tile(sysm.cut_dofs, (1, nb)).ravel())
            v.append(sysm.cut_K.ravel())
        sysm.K = sp.csr_matrix((np.concatenate(v), (np.concatenate(r), np.concatenate(cc))), shape=(n, n))
        mr = [sysm.uncut_dofs.ravel()]
        mc = [sysm.uncut_dofs.ravel()]
        mvv = [np.tile(Me_u, len(uncut))]
        if len(cut):
            mr.append(np.repeat(sysm.cut_dofs, nb, axis=1).ravel())
            mc.append(np.tile(sysm.cut_dofs, (1, nb)).ravel())
            mvv.append(sysm.cut_M.ravel())
        sysm.M = sp.csr_matrix((np.concatenate(mvv), (np.concatenate(mr), np.concatenate(mc))), shape=(n, n))
    else:
        sysm.K = None
        sysm.M = None
    # load vector: point load (reading C11) or the paper's Gaussian bell (Eq. eq:fx)
    if cfg.get("source") is not None and cfg["source"].get("kind", "point") == "bell":
        sysm.f_x = bell_load(cfg, cl)
    elif cfg.get("source") is not None:
        sysm.f_x = point_load(cfg, cl, cfg["source"]["x"])
    else:
        sysm.f_x = np.zeros(n)
    return sysm


def hrz_element(Me):
    """HRZ lumping of a consistent element mass (§Lumping of Cut Cells):
    M~_ii = m_e / (sum_k M_kk) * M_ii with m_e = sum_ij M_ij (the element's total mass),
    M~_ij = 0 for i != j.  Returns the diagonal."""
    Me = np.asarray(Me, dtype=np.float64)
    d = np.diag(Me)
    return Me.sum() / d.sum() * d


def hrz_mass(sysm):
    """Global diagonal mass of the HRZ-lumped SCM: nodally lumped uncut cells plus
    HRZ-lumped cut cells."""
    n = sysm.n_dof
    m = np.bincount(sysm.uncut_dofs.ravel(), weights=np.tile(sysm.Me_uncut, len(sysm.uncut_dofs)), minlength=n)
    for e in range(len(sysm.cut_dofs)):
        m += np.bincount(sysm.cut_dofs[e], weights=hrz_element(sysm.cut_M[e]), minlength=n)
    return m


def K_apply(sysm, u):
    """K u over all DOFs (sparse mode: CSR product; ebe mode: batched dense
    element products scattered with bincount)."""
    if sysm.K is not None:
        return sysm.K @ u
    n = sysm.n_dof
    out = np.zeros(n)
    chunk = 200000
    for st in range(0, len(sysm.uncut_dofs), chunk):
        dofs = sysm.uncut_dofs[st:st + chunk]
        Y = u[dofs] @ sysm.Ke_uncut.T
        out += np.bincount(dofs.ravel(), weights=Y.ravel(), minlength=n)
    if len(sysm.cut_dofs):
        Y = np.einsum("eij,ej->ei", sysm.cut_K, u[sysm.cut_dofs])
        out += np.bincount(sysm.cut_dofs.ravel(), weights=Y.ravel(), minlength=n)
    return out


def dense_brute_force(cfg, cl=None):
    """Brute-force dense global M and K: loop over every non-empty cell and
    add its element matrix into dense n x n arrays (tiny grids only; pin P4)."""
    if cl is None:
        cl = classify(cfg)
    d = cfg["dim"]
    p = cfg["p"]
    grid = cl.grid
    h = [(grid["hi"][k] - grid["lo"][k]) / grid["cells"][k] for k in range(d)]
    Me_u, Ke_u = uncut_element(p, h, cfg["rho"], cfg["c"])
    n = cl.n_dof
    M = np.zeros((n, n))
    K = np.zeros((n, n))
    for ci in range(len(cl.cell_class)):
        if cl.cell_class[ci] == EMPTY:
            continue
        dofs = cl.dof_of_lattice[cl.enodes[ci]]
        if cl.cell_class[ci] == UNCUT:
            Me, Ke = np.diag(Me_u), Ke_u
        else:
            levels, a, ph = cl.trees[ci]
            Me, Ke = cut_element(grid, cfg["voids"], cl.cell_idx[ci], levels, a, p,
                                 cfg["alpha"], cfg["rho"], cfg["c"], phys=ph)
        for i in range(len(dofs)):
            for j in range(len(dofs)):
                M[dofs[i], dofs[j]] += Me[i, j]
                K[dofs[i], dofs[j]] += Ke[i, j]
    return M, K


__all__ = ["classify", "build_system", "K_apply", "node_coords", "dense_brute_force",
           "cell_bounds", "UNCUT", "CUT", "EMPTY"]
