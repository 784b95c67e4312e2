"""Pins of the oracle's cell-wise critical time steps (oracle.spectra.cell_dt_map; PAPER.md
P:857-890): uncut cells carry the uncut cell-wise value; a single cut cell reproduces the
single-cell study of Fig. 2 (fig:fillRatioHZ), which tests/test_oracle_basis pins to
the paper's printed values; HRZ lumping of an uncut (already lumped) cell changes nothing;
the paper's ordering: the cut-cell minimum lies below the uncut value (Table 1)."""
import numpy as np

import sc_inputs
from oracle.assembly import build_system
from oracle.spectra import cell_dt_map, dt_crit_uncut, fill_ratio_cell_omega


def test_uncut_cells_and_ordering():
    cfg = sc_inputs.small_config(2, [6, 6], 3, voids=[{"kind": "ellipsoid", "c": [0.52, 0.47, 0.0],
                                 "A": [1 / 0.04, 1 / 0.05, 0.0, 5.0, 0.0, 0.0]}], depth=3, alpha=1e-5)
    sysm = build_system(cfg, "sparse")
    m = cell_dt_map(sysm)
    cls = sysm.cl.cell_class
    unc = dt_crit_uncut(2, 3, 1.0 / 6)
    assert np.all(m[cls == 2] == 0.0)
    assert np.all(m[cls == 0] == unc)
    assert (cls == 1).sum() > 0 and m[cls == 1].min() < m[cls == 0][0]
    h = cell_dt_map(sysm, "hrz")
    assert np.array_equal(h[cls == 0], m[cls == 0])


def test_single_cut_cell_is_fig2():
    for p, eta in ((1, 0.5), (2, 0.3), (3, 0.1)):
        cfg = sc_inputs.small_config(2, [1, 1], p, voids=[{"kind": "halfspace", "n": [0.0, 1.0, 0.0], "b": eta}],
                                     depth=6, alpha=1e-6)
        sysm = build_system(cfg, "sparse")
        m = cell_dt_map(sysm)
        assert sysm.cl.cell_class[0] == 1
        omega = fill_ratio_cell_omega(eta, p, depth=6)
        assert abs(2.0 / m[0] - omega) <= 1e-10 * omega, (p, eta, 2.0 / m[0], omega)
