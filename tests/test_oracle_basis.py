"""Pins of oracle/basis.py against closed forms."""
import numpy as np
import pytest

from oracle.basis import gll_rule, gauss_rule, lagrange, reference_matrices, legendre


def test_gll_closed_forms():
    # p=1: {-1,1}, w = {1,1}; p=2: {-1,0,1}, w = {1/3,4/3,1/3}
    x, w = gll_rule(1)
    assert np.allclose(x, [-1, 1], atol=0) and np.allclose(w, [1, 1], atol=1e-15)
    x, w = gll_rule(2)
    assert np.allclose(x, [-1, 0, 1], atol=1e-16)
    assert np.allclose(w, [1 / 3, 4 / 3, 1 / 3], rtol=1e-15)
    # p=4: +-1, +-sqrt(3/7), 0; weights 1/10, 49/90, 32/45
    x, w = gll_rule(4)
    r = np.sqrt(3.0 / 7.0)
    assert np.allclose(x, [-1, -r, 0, r, 1], atol=2e-16)
    assert np.allclose(w, [0.1, 49 / 90, 32 / 45, 49 / 90, 0.1], rtol=1e-14)


@pytest.mark.parametrize("p", range(1, 11))
def test_gll_exactness(p):
    x, w = gll_rule(p)
    assert abs(w.sum() - 2.0) < 1e-14
    for k in range(2 * p):           # exact to degree 2p-1
        exact = 0.0 if k % 2 else 2.0 / (k + 1)
        assert abs(np.dot(w, x ** k) - exact) < 1e-13
    # interior points are roots of P_p'
    _, dP = legendre(p, x[1:-1])
    assert np.all(np.abs(dP) < 1e-11 * p * p)


@pytest.mark.parametrize("n", range(1, 10))
def test_gauss_exactness(n):
    x, w = gauss_rule(n)
    for k in range(2 * n):
        exact = 0.0 if k % 2 else 2.0 / (k + 1)
        assert abs(np.dot(w, x ** k) - exact) < 1e-13
    # and not exact at degree 2n
    assert abs(np.dot(w, x ** (2 * n)) - 2.0 / (2 * n + 1)) > 1e-6


@pytest.mark.parametrize("p", [1, 2, 3, 4, 6])
def test_lagrange_kronecker_partition_derivative(p):
    nodes, _ = gll_rule(p)
    V, D = lagrange(nodes, nodes)
    assert np.allclose(V, np.eye(p + 1), atol=1e-14)
    xi = np.linspace(-1, 1, 37)
    V, D = lagrange(nodes, xi)
    assert np.allclose(V.sum(axis=1), 1.0, atol=1e-13)
    assert np.allclose(D.sum(axis=1), 0.0, atol=1e-11)
    eps = 1e-6
    Vp, _ = lagrange(nodes, xi + eps)
    Vm, _ = lagrange(nodes, xi - eps)
    assert np.allclose((Vp - Vm) / (2 * eps), D, atol=1e-6 * (p + 1) ** 2)
    # reproduces polynomials of degree p exactly: interpolate x^p
    assert np.allclose(V @ nodes ** p, xi ** p, atol=1e-13)


def test_reference_matrices_p1_hand():
    Mc, Kh, W = reference_matrices(1)
    assert np.allclose(Mc, [[2 / 3, 1 / 3], [1 / 3, 2 / 3]], atol=1e-15)
    assert np.allclose(Kh, [[0.5, -0.5], [-0.5, 0.5]], atol=1e-15)
    assert np.allclose(W, [1, 1])


@pytest.mark.parametrize("p", [2, 3, 4, 5])
def test_reference_matrices_properties(p):
    Mc, Kh, W = reference_matrices(p)
    # int 1 = 2; constants in the kernel of the derivative; symmetric; the
    # consistent mass integrates x*x exactly: sum_ij x_i x_j Mc_ij = int x^2 = 2/3
    nodes, _ = gll_rule(p)
    assert abs(Mc.sum() - 2.0) < 1e-14
    assert np.allclose(Kh.sum(axis=1), 0.0, atol=1e-12)
    assert np.allclose(Mc, Mc.T) and np.allclose(Kh, Kh.T)
    assert abs(nodes @ Mc @ nodes - 2.0 / 3.0) < 1e-13
    # int (x')^2 for x -> 2 ; int (x^2)'^2 = int 4x^2 = 8/3
    assert abs(nodes @ Kh @ nodes - 2.0) < 1e-12
    assert abs((nodes ** 2) @ Kh @ (nodes ** 2) - 8.0 / 3.0) < 1e-12
    # GLL lumping preserves the total mass
    assert abs(W.sum() - 2.0) < 1e-14
