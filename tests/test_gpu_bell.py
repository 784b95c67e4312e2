"""NEXT-3: the paper's own excitation pair - Gaussian-bell spatial load f_x
(Eq. eq:fx; source kind 2, assembled on the host of the library from Gauss
points of cells and spacetree leaves) with the Gaussian-derivative f_t (Eq. eq:ft) -
through the device step, against the oracle (oracle.assembly.bell_load, pinned in
tests/test_oracle_bell.py): the load reaches tensor-d nodes (k_load_d), irregular d nodes and
c nodes, so the bell is placed across a void."""
import numpy as np
import pytest

import sc_inputs
from oracle.run import run_config
from oracle.spectra import dt_crit_uncut

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


CASES = [(2, [16, 12], 4, {"kind": "ellipsoid", "c": [0.55, 0.45, 0.0], "A": [40.0, 60.0, 0.0, 5.0, 0.0, 0.0]},
          [0.42, 0.45, 0.0], 0.06),
         (3, [6, 5, 7], 3, {"kind": "ellipsoid", "c": [0.5, 0.45, 0.5], "A": [30.0, 40.0, 35.0, 2.0, 1.0, 0.0]},
          [0.4, 0.5, 0.45], 0.09)]


@pytest.mark.parametrize("dim,cells,p,void,xs,sigma", CASES)
def test_bell_source_matches_oracle(pkg, dim, cells, p, void, xs, sigma):
    steps = 120
    cfg = sc_inputs.small_config(dim, cells, p, voids=[void], depth=2, steps=steps,
                                 source={"kind": "bell", "x": xs, "sigma": sigma, "amp": 10.0,
                                         "signal": "gauss_deriv", "f0": 4.0})
    cfg["dt"] = 0.9 * dt_crit_uncut(dim, p, 1.0 / max(cells))
    s = pkg.from_config(cfg)
    s.step(steps)
    u = s.read()
    s.close()
    ref, sysm = run_config(cfg, steps=steps, mode="sparse")
    assert (sysm.f_x != 0).sum() > sysm.cl.enodes.shape[1]   # a distributed load
    assert np.abs(sysm.f_x[sysm.I_c]).max() > 0             # reaching c nodes too
    err = np.linalg.norm(u - ref) / np.linalg.norm(ref)
    assert np.abs(ref).max() > 0 and err < 1e-10, err
