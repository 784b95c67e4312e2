"""1D rules and Lagrange basis (ORACLE - test infrastructure only).

PAPER.md P:405-416 (§Spatial Discretization): N_i^{Lag,p}(xi) is the product
formula over the p+1 GLL points; the GLL points are -1, +1 and the roots of
the Lobatto polynomial of order p-1 (= roots of P'_p, the derivative of the
Legendre polynomial of degree p).  GLL weights w_j = 2 / (p(p+1) P_p(xi_j)^2)
(standard).  Gauss-Legendre rule with p+1 points for the
stiffness, the load and the cut cells.
"""
import numpy as np


def legendre(n, x):
    """P_n(x) and P_n'(x) by the three-term (Bonnet) recurrence."""
    x = np.asarray(x, dtype=np.float64)
    p0 = np.ones_like(x)
    if n == 0:
        return p0, np.zeros_like(x)
    p1 = x.copy()
    for k in range(2, n + 1):
        p0, p1 = p1, ((2 * k - 1) * x * p1 - (k - 1) * p0) / k
    # derivative: (1-x^2) P_n' = n (P_{n-1} - x P_n); valid away from +-1
    with np.errstate(divide="ignore", invalid="ignore"):
        dp = n * (p0 - x * p1) / (1.0 - x * x)
    end = np.abs(x) == 1.0
    if np.any(end):
        dp = np.where(end, 0.5 * n * (n + 1) * np.power(x, n + 1), dp)
    return p1, dp


def gll_rule(p):
    """p+1 GLL points (ascending) and weights."""
    if p < 1:
        raise ValueError("p >= 1")
    # interior points: roots of P_p'; Newton on P_p' starting from the
    # Chebyshev-Gauss-Lobatto guess.  P_p'' from the Legendre ODE:
    # (1-x^2) P'' = 2x P' - p(p+1) P.
    x = -np.cos(np.pi * np.arange(1, p) / p)
    for _ in range(100):
        P, dP = legendre(p, x)
        ddP = (2.0 * x * dP - p * (p + 1) * P) / (1.0 - x * x)
        dx = dP / ddP
        x = x - dx
        if np.all(np.abs(dx) < 1e-16):
            break
    nodes = np.concatenate([[-1.0], np.sort(x), [1.0]])
    P, _ = legendre(p, nodes)
    weights = 2.0 / (p * (p + 1) * P * P)
    return nodes, weights


def gauss_rule(n):
    """n-point Gauss-Legendre rule (library primitive, numpy leggauss)."""
    x, w = np.polynomial.legendre.leggauss(n)
    return x, w


def lagrange(nodes, xi):
    """Values and derivatives of the Lagrange polynomials on ``nodes`` at
    points ``xi``; P:407 product formula, derivative by the product rule.

    Returns (V, D) with shape (len(xi), len(nodes)).
    """
    nodes = np.asarray(nodes, dtype=np.float64)
    xi = np.atleast_1d(np.asarray(xi, dtype=np.float64))
    n = len(nodes)
    V = np.ones((len(xi), n))
    D = np.zeros((len(xi), n))
    for i in range(n):
        for j in range(n):
            if j == i:
                continue
            V[:, i] *= (xi - nodes[j]) / (nodes[i] - nodes[j])
        for m in range(n):
            if m == i:
                continue
            term = np.full(len(xi), 1.0 / (nodes[i] - nodes[m]))
            for j in range(n):
                if j == i or j == m:
                    continue
                term *= (xi - nodes[j]) / (nodes[i] - nodes[j])
            D[:, i] += term
    return V, D


def reference_matrices(p):
    """1D reference matrices on [-1,1] (P:444-448 with P:463):

    Mc  = sum_q w_q l(g_q) l(g_q)^T   (Gauss, p+1 points: exact, consistent)
    Kh  = sum_q w_q l'(g_q) l'(g_q)^T (Gauss, p+1 points: exact)
    W   = GLL weights (nodal lumping of the uncut mass)
    """
    nodes, wgll = gll_rule(p)
    g, wg = gauss_rule(p + 1)
    V, D = lagrange(nodes, g)
    Mc = (V * wg[:, None]).T @ V
    Kh = (D * wg[:, None]).T @ D
    return Mc, Kh, wgll
