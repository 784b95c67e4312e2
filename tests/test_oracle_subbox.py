"""Pins the sub-box parity harness (tests/subbox.py) oracle against oracle on the CPU: from a
compactly supported u0 near voids with no load, the oracle's IMEX run on the full domain,
restricted to closure_box(), equals the oracle's run on that box alone (same arithmetic up to
the summation order of K u and the per-box factorisation), and is EXACTLY zero outside it.
The box must really truncate the domain and the c DOFs must carry a non-negligible share of
u, so that the GPU tests built on this harness check the implicit (c) path.

Measured floor (2D case): the d DOFs agree to ~3e-15, the c DOFs to ~3e-12 from the first
implicit solve on - the box computes its cut-cell quadrature points from its own lo, which
moves them by ulps, and S amplifies that by its condition number (kappa(S)
~1e4-1e5).  A missing dependency would show as an O(1) difference, so the bar here is the
north_star parity bar 1e-10 plus exact zeros outside the box."""
import numpy as np
import pytest

import sc_inputs
from oracle.assembly import build_system, node_coords
from oracle.integrators import from_system, imex
from oracle.spectra import dt_crit_uncut
from subbox import box_config, box_to_full_lattice, closure_box


def _voids2d():
    return [{"kind": "ellipsoid", "c": [0.30, 0.42, 0.0], "A": [1 / 0.045 ** 2, 1 / 0.03 ** 2, 0, 20.0, 0, 0]},
            {"kind": "ellipsoid", "c": [0.40, 0.47, 0.0], "A": [1 / 0.03 ** 2, 1 / 0.03 ** 2, 0, 0, 0, 0]},
            {"kind": "ellipsoid", "c": [0.80, 0.80, 0.0], "A": [1 / 0.04 ** 2, 1 / 0.04 ** 2, 0, 0, 0, 0]},
            {"kind": "ellipsoid", "c": [0.15, 0.85, 0.0], "A": [1 / 0.03 ** 2, 1 / 0.05 ** 2, 0, 0, 0, 0]}]


def _voids3d():
    return [{"kind": "ellipsoid", "c": [0.30, 0.34, 0.36], "A": [1 / 0.06 ** 2, 1 / 0.05 ** 2, 1 / 0.07 ** 2, 10, 0, 5]},
            {"kind": "ellipsoid", "c": [0.85, 0.80, 0.75], "A": [1 / 0.06 ** 2, 1 / 0.06 ** 2, 1 / 0.06 ** 2, 0, 0, 0]}]


def _run(cfg, x0, R, steps):
    sysm = build_system(cfg, "sparse")
    u0 = sc_inputs.compact_bump(node_coords(cfg, sysm.cl.lattice_index), x0, R)
    u = imex(from_system(sysm), cfg["dt"], steps, None, u0, None)
    return u, sysm


@pytest.mark.parametrize("dim", [2, 3])
def test_full_domain_equals_closure_box(dim):
    if dim == 2:
        cfg = sc_inputs.small_config(2, [48, 48], 3, voids=_voids2d(), depth=3, alpha=1e-5)
        x0, R, steps = [0.33, 0.40], 0.06, 10
    else:
        cfg = sc_inputs.small_config(3, [28, 28, 28], 2, voids=_voids3d(), depth=2, alpha=1e-5)
        x0, R, steps = [0.30, 0.36, 0.37], 0.07, 3
    cfg["dt"] = 0.9 * dt_crit_uncut(dim, cfg["p"], 1.0 / cfg["cells"][0])
    lo, hi, used = closure_box(cfg, x0, R, steps)
    # the box truncates the domain and holds the touched voids only
    assert any(hi[k] - lo[k] < cfg["cells"][k] for k in range(dim))
    assert 0 < len(used) < len(cfg["voids"])
    bcfg = box_config(cfg, lo, hi)
    u_full, sf = _run(cfg, x0, R, steps)
    u_box, sb = _run(bcfg, x0, R, steps)
    # map the box DOFs into the full DOF numbering
    lat_full = box_to_full_lattice(cfg, lo, sb.cl.lattice_index, bcfg["cells"])
    idx = sf.cl.dof_of_lattice[lat_full]
    assert np.all(idx >= 0)
    ref = u_full[idx]
    err = np.linalg.norm(u_box - ref) / np.linalg.norm(ref)
    assert err < 1e-10, err
    # c DOFs inside the box: separate bar, and a non-negligible share of u
    c = sb.cl.is_c
    assert np.linalg.norm(u_box[c]) / np.linalg.norm(u_box) > 1e-2
    err_c = np.linalg.norm(u_box[c] - ref[c]) / np.linalg.norm(ref[c])
    assert err_c < 1e-10, err_c
    # exactly zero outside the box in the full run
    outside = np.ones(sf.n_dof, dtype=bool)
    outside[idx] = False
    assert np.all(u_full[outside] == 0.0)
    # the d DOFs (no implicit solve) agree to roundoff of the explicit update
    err_d = np.linalg.norm(u_box[~c] - ref[~c]) / np.linalg.norm(ref[~c])
    assert err_d < 1e-13, err_d
