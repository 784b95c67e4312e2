"""NEXT-1(1b): the high-cut-fraction stress case, config 6 (2D, 128^2 cells, p = 4,
400 voids, 31% of the DOFs c — the regime of the paper's 51%-cut pillar, where the c part
dominates the step), at FULL size against the oracle: bit-exact classification and the IMEX
state after 10 steps within rel L2 1e-10."""
import numpy as np
import pytest

import sc_inputs
from oracle.assembly import build_system
from oracle.run import run_config

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


def test_config6_stress_full_size_parity(pkg):
    steps = 10
    cfg = sc_inputs.get_config(6, steps=steps)
    s = pkg.from_config(cfg, f_t=sc_inputs.source_signal(cfg, steps + 2))
    s.step(steps)
    u = s.read()
    cc, isc, lat = s.classification()
    s.close()
    sysm = build_system(cfg, "sparse")
    assert np.array_equal(cc, sysm.cl.cell_class)
    assert np.array_equal(isc, sysm.cl.is_c) and np.array_equal(lat, sysm.cl.lattice_index)
    assert isc.mean() > 0.25                      # the stress regime: >= a quarter of the DOFs c
    ref, _ = run_config(cfg, sysm=sysm)
    err = np.linalg.norm(u - ref) / np.linalg.norm(ref)
    assert np.linalg.norm(ref) > 0 and err < 1e-10, err
