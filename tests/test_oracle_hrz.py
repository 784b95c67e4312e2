"""Pins of the HRZ-lumped SCM (oracle.assembly.hrz_element / hrz_mass; NEXT-1(c) of SURVEY
§8(f)), §Lumping of Cut Cells:
* each element's total mass is preserved (the defining property);
* HRZ diagonals are positive even where row-summing gives negative masses;
* an uncut element is returned unchanged (its mass is already nodally lumped);
* explicit treatment of the cut cells restricts the step (Table tab:criticaltimestepsizes,
  P:869): the HRZ-lumped and the consistent global critical steps both lie far
  below the uncut cell-wise step that governs Newmark IMEX.  (Their mutual order depends on
  the cut geometry: the paper's plate has HRZ < consistent, this small case the reverse.)"""
import numpy as np
import scipy.sparse as sp

import sc_inputs
from oracle.assembly import build_system, hrz_element, hrz_mass
from oracle.elements import uncut_element
from oracle.spectra import dt_crit, dt_crit_uncut

CFG = sc_inputs.small_config(2, [8, 8], 3, voids=[
    {"kind": "ellipsoid", "c": [0.5, 0.5, 0.0], "A": [1 / 0.06, 1 / 0.06, 0.0, 0.0, 0.0, 0.0]}], depth=3,
    alpha=1e-5)


def test_element_mass_preserved_and_positive():
    s = build_system(CFG, "sparse")
    assert len(s.cut_M) > 0
    neg_rowsum = 0
    for Me in s.cut_M:
        d = hrz_element(Me)
        assert abs(d.sum() - Me.sum()) <= 1e-14 * abs(Me.sum())
        assert (d > 0).all()
        neg_rowsum += int((Me.sum(axis=1) < 0).any())
    assert neg_rowsum > 0          # row-summing would produce negative masses here


def test_uncut_element_unchanged_and_global_mass():
    Me, _ = uncut_element(3, [0.125, 0.125], 1.0, 1.0)
    assert np.allclose(hrz_element(np.diag(Me)), Me, rtol=1e-15, atol=0)
    s = build_system(CFG, "sparse")
    m = hrz_mass(s)
    assert abs(m.sum() - s.M.sum()) <= 1e-13 * s.M.sum()
    assert (m > 0).all()


def test_critical_step_ordering():
    s = build_system(CFG, "sparse")
    K = s.K.toarray()
    dt_hrz = dt_crit(K, hrz_mass(s))
    dt_cons = dt_crit(K, s.M.toarray())
    dt_unc = dt_crit_uncut(2, 3, 0.125)
    assert dt_hrz < 0.5 * dt_unc and dt_cons < 0.5 * dt_unc
