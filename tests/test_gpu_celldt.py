"""Cell-wise critical time steps on the device (sc_cell_dt, PAPER.md
P:857-890) against the oracle's per-cell generalized eigenvalues (oracle.spectra.cell_dt_map:
scipy eigh per cell), with the consistent and the HRZ-lumped cut-cell mass; a single cut cell
against the Fig. 2 single-cell study (oracle.spectra.fill_ratio_cell_omega, pinned to the
paper's printed values); config 5 (the bench workload): the paper's Table 1 relation, cut-cell
minimum below the uncut cell-wise value."""
import numpy as np
import pytest

import sc_inputs
from oracle.assembly import build_system
from oracle.spectra import cell_dt_map, fill_ratio_cell_omega

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


def test_config2_cell_dt_vs_oracle(pkg):
    cfg = sc_inputs.get_config(2)
    s = pkg.from_config(cfg)
    g_cons, g_hrz = s.cell_dt(0), s.cell_dt(1)
    s.close()
    sysm = build_system(cfg, "sparse")
    o_cons, o_hrz = cell_dt_map(sysm, "consistent"), cell_dt_map(sysm, "hrz")
    cls = sysm.cl.cell_class
    for g, o in ((g_cons, o_cons), (g_hrz, o_hrz)):
        assert np.array_equal(g == 0.0, o == 0.0)
        nz = o > 0
        assert np.max(np.abs(g[nz] - o[nz]) / o[nz]) <= 1e-9
    # Table 1: the cut-cell minimum lies far below the uncut cell-wise value
    assert g_cons[cls == 1].min() < 0.5 * g_cons[cls == 0][0]


@pytest.mark.parametrize("p,eta", [(1, 0.5), (1, 0.05), (2, 0.3), (3, 0.1), (3, 0.7)])
def test_single_cut_cell_fig2(pkg, p, eta):
    cfg = sc_inputs.small_config(2, [1, 1], p, voids=[{"kind": "halfspace", "n": [0.0, 1.0, 0.0], "b": eta}],
                                 depth=6, alpha=1e-6, steps=1)
    cfg["dt"] = 1e-3
    s = pkg.from_config(cfg)
    m = s.cell_dt(0)
    s.close()
    omega = fill_ratio_cell_omega(eta, p, depth=6)
    assert abs(2.0 / m[0] - omega) <= 1e-9 * omega, (2.0 / m[0], omega)


def test_config5_cell_dt_relation(pkg):
    cfg = sc_inputs.get_config(5)
    s = pkg.from_config(cfg)
    m = s.cell_dt(0)
    unc = s.info["dt_crit_uncut"]
    cls, _, _ = s.classification()
    s.close()
    assert np.all(m[cls == 0] == unc) and np.all(m[cls == 2] == 0.0)
    cut = m[cls == 1]
    assert np.all(cut > 0) and cut.min() < unc
