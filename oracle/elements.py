"""Element matrices (ORACLE - test infrastructure only).

PAPER.md P:444-448 (Eqs. eq:Mglobal, eq:K): M_ij = int alpha rho N_i N_j,
K_ij = int alpha rho c^2 grad N_i . grad N_j, with rho* = alpha rho.
P:463: uncut cells integrate the mass with GLL points (diagonal, nodal
lumping) and the stiffness with Gauss-Legendre points; cut cells integrate
both with Gauss-Legendre points on the spacetree leaves.  Reading C5
(pinned by Fig. 2's eta = 1 points): uncut = GLL-lumped mass + (p+1)-point
Gauss stiffness.

Local node order: tensor product, x fastest (i = i0 + (p+1) i1 + (p+1)^2 i2).
"""
import numpy as np

from .basis import gll_rule, gauss_rule, lagrange, reference_matrices
from .geometry import leaf_gauss_points, is_physical


def _kron_chain(factors):
    """factors[k] acts on axis k (axis 0 = x, fastest)."""
    out = factors[0]
    for f in factors[1:]:
        out = np.kron(f, out)
    return out


def uncut_element(p, h, rho, c):
    """(Me_diag, Ke) of an uncut cell with edge lengths h (len d)."""
    Mc, Kh, W = reference_matrices(p)
    d = len(h)
    Ke = 0.0
    for k in range(d):
        fac = [((2.0 / h[j]) * Kh if j == k else (h[j] / 2.0) * Mc) for j in range(d)]
        Ke = Ke + _kron_chain(fac)
    Ke = rho * c * c * Ke
    Wd = _kron_chain([np.diag((h[j] / 2.0) * W) for j in range(d)])
    return rho * np.diag(Wd).copy(), Ke


def cell_bounds(grid, cell):
    """Physical bounds of a cell (lattice coordinates at level 0, C17)."""
    d = grid["dim"]
    lo = np.zeros(d)
    hi = np.zeros(d)
    for k in range(d):
        den = np.float64(grid["cells"][k])
        lo[k] = grid["lo"][k] + (grid["hi"][k] - grid["lo"][k]) * (np.float64(cell[k]) / den)
        hi[k] = grid["lo"][k] + (grid["hi"][k] - grid["lo"][k]) * (np.float64(cell[k] + 1) / den)
    return lo, hi


def cut_element(grid, voids, cell, levels, a, p, alpha, rho, c, phys=None):
    """Consistent (Me, Ke) of a cut cell from its spacetree leaves: (p+1)^d
    Gauss points per leaf, pointwise alpha in {1, alpha}.

    ``h`` is the cell edge from the grid spacing (hi-lo)/N (uniform grid)."""
    d = grid["dim"]
    nodes, _ = gll_rule(p)
    g, wg = gauss_rule(p + 1)
    n = p + 1
    h = [(grid["hi"][k] - grid["lo"][k]) / grid["cells"][k] for k in range(d)]
    if phys is None:
        X = leaf_gauss_points(grid, cell, levels, a, g)
        phys = is_physical(X, voids)
    a_q = np.where(phys, 1.0, alpha)
    L = len(levels)
    scale = 1.0 / (2.0 ** levels)                      # leaf size in reference units / 2
    V = []
    D = []
    Wk = []
    for k in range(d):
        # reference coordinate in the cell: xi = -1 + 2*(a + (g+1)/2)/2^l
        xi = -1.0 + 2.0 * (a[:, k][:, None] + (g[None, :] + 1.0) * 0.5) * scale[:, None]
        v, dv = lagrange(nodes, xi.reshape(-1))
        V.append(v.reshape(L, n, n))                  # (leaf, gauss pt, basis)
        D.append(dv.reshape(L, n, n))
        Wk.append(wg[None, :] * scale[:, None] * (h[k] / 2.0))   # (leaf, gauss pt)

    def tens(mats, leaf_w=False):
        # tensor over axes, x fastest for both point and basis index
        if d == 1:
            return mats[0].reshape(L * n, n) if not leaf_w else mats[0].reshape(L * n)
        if d == 2:
            if leaf_w:
                return np.einsum("lb,la->lba", mats[1], mats[0]).reshape(L * n * n)
            return np.einsum("lqj,lpi->lqpji", mats[1], mats[0]).reshape(L * n * n, n * n)
        if leaf_w:
            return np.einsum("lc,lb,la->lcba", mats[2], mats[1], mats[0]).reshape(L * n ** 3)
        return np.einsum("lrk,lqj,lpi->lrqpkji", mats[2], mats[1], mats[0]).reshape(L * n ** 3, n ** 3)

    w = tens(Wk, leaf_w=True) * a_q
    N = tens(V)
    Me = rho * (N * w[:, None]).T @ N
    Ke = 0.0
    for k in range(d):
        mats = [(D[j] * (2.0 / h[j])) if j == k else V[j] for j in range(d)]
        G = tens(mats)
        Ke = Ke + (G * w[:, None]).T @ G
    Ke = rho * c * c * Ke
    return Me, Ke


def eval_basis_at(grid, cell, x, p):
    """Values of the (p+1)^d cell basis functions at physical point x."""
    d = grid["dim"]
    nodes, _ = gll_rule(p)
    lo, hi = cell_bounds(grid, cell)
    vals = []
    for k in range(d):
        xi = -1.0 + 2.0 * (x[k] - lo[k]) / (hi[k] - lo[k])
        v, _ = lagrange(nodes, np.array([xi]))
        vals.append(v[0])
    out = vals[0]
    for k in range(1, d):
        out = np.kron(vals[k], out)
    return out


def gaussian_bell(X, xs, sigma, amp):
    """f_x(x) = amp exp(-|x - x_s|^2 / (2 sigma^2)) (Eq. eq:fx; the paper
    has amp = 10, sigma_s = 6e-2 m)."""
    d = len(xs)
    r2 = np.sum((X[:, :d] - np.asarray(xs, dtype=np.float64)[None, :]) ** 2, axis=1)
    return amp * np.exp(-r2 / (2.0 * sigma * sigma))


def cell_load(grid, voids, cell, levels, a, p, alpha, fx, phys=None):
    """Element load vector f_i = int alpha f_x N_i (Eq. eq:f) with (p+1)^d Gauss
    points per spacetree leaf (the load is Gauss-integrated in cut and uncut cells; an
    uncut cell is the single leaf (levels [0], a [0...]) with alpha = 1).  fx(X) -> values."""
    d = grid["dim"]
    nodes, _ = gll_rule(p)
    g, wg = gauss_rule(p + 1)
    n = p + 1
    h = [(grid["hi"][k] - grid["lo"][k]) / grid["cells"][k] for k in range(d)]
    X = leaf_gauss_points(grid, cell, levels, a, g)
    if phys is None:
        phys = is_physical(X, voids)
    a_q = np.where(phys, 1.0, alpha)
    L = len(levels)
    scale = 1.0 / (2.0 ** levels)
    V, Wk = [], []
    for k in range(d):
        xi = -1.0 + 2.0 * (a[:, k][:, None] + (g[None, :] + 1.0) * 0.5) * scale[:, None]
        v, _ = lagrange(nodes, xi.reshape(-1))
        V.append(v.reshape(L, n, n))
        Wk.append(wg[None, :] * scale[:, None] * (h[k] / 2.0))
    if d == 1:
        N, w = V[0].reshape(L * n, n), Wk[0].reshape(L * n)
    elif d == 2:
        N = np.einsum("lqj,lpi->lqpji", V[1], V[0]).reshape(L * n * n, n * n)
        w = np.einsum("lb,la->lba", Wk[1], Wk[0]).reshape(L * n * n)
    else:
        N = np.einsum("lrk,lqj,lpi->lrqpkji", V[2], V[1], V[0]).reshape(L * n ** 3, n ** 3)
        w = np.einsum("lc,lb,la->lcba", Wk[2], Wk[1], Wk[0]).reshape(L * n ** 3)
    return N.T @ (w * a_q * fx(X))
