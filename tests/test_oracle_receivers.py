"""Pins of oracle.assembly.point_values (receiver weights): the Lagrange
basis of the evaluating cell sums to one (partition of unity), reproduces the
nodal value at a lattice node (Kronecker property) and reproduces a degree-p field
exactly (the GLL nodes carry the degree-p interpolant)."""
import numpy as np

import sc_inputs
from oracle.assembly import classify, node_coords, point_values


def _cfg():
    return sc_inputs.small_config(2, [5, 4], 3, voids=[
        {"kind": "ellipsoid", "c": [0.55, 0.45, 0.0], "A": [40.0, 60.0, 0.0, 5.0, 0.0, 0.0]}], depth=2)


def test_partition_of_unity_and_kronecker():
    cfg = _cfg()
    cl = classify(cfg)
    for x in ([0.13, 0.77], [0.5, 0.5], [0.91, 0.08]):
        w = point_values(cfg, cl, np.array(x))
        assert abs(w.sum() - 1.0) < 1e-13
    X = node_coords(cfg, cl.lattice_index)
    for i in (0, 7, len(X) // 2):
        w = point_values(cfg, cl, X[i, :2])
        assert abs(w[i] - 1.0) < 1e-12 and np.abs(np.delete(w, i)).max() < 1e-12


def test_reproduces_polynomial_field():
    cfg = _cfg()
    cl = classify(cfg)
    X = node_coords(cfg, cl.lattice_index)
    f = lambda x, y: 1.0 + 2.0 * x - 3.0 * y + x ** 3 * y ** 2 - 0.5 * x * y ** 3
    u = f(X[:, 0], X[:, 1])
    for x in ([0.13, 0.77], [0.21, 0.33], [0.66, 0.94]):
        assert abs(point_values(cfg, cl, np.array(x)) @ u - f(*x)) < 1e-12
