"""NEXT-2: device Lanczos iteration for the critical time step of the explicit
subsystem, dt = 2 / sqrt(lambda_max(K_dd, M_dd)), against the oracle's
dense generalized eigenvalue of the same (K_dd, M_dd); and the paper's relation that the
IMEX critical step is governed by the uncut cells (Table tab:criticaltimestepsizes)."""
import numpy as np
import pytest
import scipy.sparse as sp

import sc_inputs
from oracle.assembly import build_system
from oracle.spectra import dt_crit_uncut, lambda_max

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def pkg():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2310_14712_b200.build import build
    build()
    import paper_2310_14712_b200 as p
    p.load_library()
    return p


def _oracle_lambda(cfg):
    s = build_system(cfg, "sparse")
    Id = s.I_d
    Kdd = sp.csr_matrix(s.K)[Id][:, Id]
    return lambda_max(Kdd, s.M_dd)


@pytest.mark.parametrize("dim,cells,p", [(2, [9, 8], 3), (3, [4, 5, 4], 2), (1, [12], 4)])
def test_power_iteration_matches_dense_eigenvalue(pkg, dim, cells, p):
    voids = {1: [{"kind": "halfspace", "n": [1.0, 0.0, 0.0], "b": 0.81}],
             2: [{"kind": "ellipsoid", "c": [0.45, 0.55, 0.0], "A": [40.0, 60.0, 0.0, 5.0, 0.0, 0.0]}],
             3: [{"kind": "ellipsoid", "c": [0.5, 0.45, 0.5], "A": [30.0, 40.0, 35.0, 2.0, 1.0, 0.0]}]}[dim]
    cfg = sc_inputs.small_config(dim, cells, p, voids=voids, depth=2, steps=1,
                                 source={"x": [0.3, 0.3, 0.3][:3], "f0": 3.0})
    cfg["dt"] = 0.9 * dt_crit_uncut(dim, p, 1.0 / max(cells))
    ref = _oracle_lambda(cfg)
    s = pkg.from_config(cfg)
    lam, dt = s.estimate_dt(3000)                # Lanczos (M inner product), converged well before
    s.close()
    assert lam <= ref * (1 + 1e-12)              # Ritz values approach from below
    assert abs(lam - ref) / ref < 1e-10, (lam, ref)
    assert abs(dt - 2.0 / np.sqrt(lam)) < 1e-15 * dt


def test_config2_imex_step_governed_by_uncut_cells(pkg):
    # P:869 / Table tab:criticaltimestepsizes: the explicit subsystem's critical step is at
    # least the uncut cell-wise one (Irons) and close to it (18.14 vs 18.13 ms in the paper)
    cfg = sc_inputs.get_config(2)
    s = pkg.from_config(cfg)
    lam, dt = s.estimate_dt(4000)
    s.close()
    dtu = dt_crit_uncut(2, cfg["p"], 1.0 / cfg["cells"][0])
    assert dt >= dtu * (1 - 1e-9)
    assert dt < dtu * 1.01
