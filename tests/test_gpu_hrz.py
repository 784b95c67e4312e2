"""NEXT-1(c): the paper's explicit comparison scheme — CDM on the HRZ-lumped
SCM (§Lumping of Cut Cells; CDM P:577-583) — on the same kernels
(integrator 1), against the oracle's CDM with the HRZ-lumped global mass (oracle.assembly.
hrz_mass, pinned in tests/test_oracle_hrz.py), at half its critical step."""
import numpy as np
import pytest
import scipy.sparse as sp

import sc_inputs
from oracle.assembly import build_system, hrz_mass
from oracle.integrators import Problem, cdm
from oracle.spectra import dt_crit, lambda_max

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


CASES = [(2, [10, 9], 3, {"kind": "ellipsoid", "c": [0.55, 0.45, 0.0], "A": [40.0, 60.0, 0.0, 5.0, 0.0, 0.0]}),
         (3, [5, 4, 6], 2, {"kind": "ellipsoid", "c": [0.5, 0.45, 0.5], "A": [30.0, 40.0, 35.0, 2.0, 1.0, 0.0]}),
         (1, [14], 4, {"kind": "halfspace", "n": [1.0, 0.0, 0.0], "b": 0.83})]


@pytest.mark.parametrize("dim,cells,p,void", CASES)
def test_cdm_hrz_matches_oracle(pkg, dim, cells, p, void):
    steps = 150
    cfg = sc_inputs.small_config(dim, cells, p, voids=[void], depth=2, steps=steps,
                                 source={"x": [0.25, 0.3, 0.3], "f0": 5.0})
    sysm = build_system(cfg, "sparse")
    m = hrz_mass(sysm)
    K = sysm.K.toarray()
    lam = lambda_max(K, m)
    cfg["dt"] = 0.5 * 2.0 / np.sqrt(lam)
    cfg["integrator"] = "cdm_hrz"
    s = pkg.from_config(cfg)
    s.step(steps)
    u = s.read()
    lam_gpu, _ = s.estimate_dt(6000)
    s.close()
    pr = Problem(sp.diags(m), sysm.K, sysm.f_x, sysm.I_d, sysm.I_c)
    ref = cdm(pr, cfg["dt"], steps, sc_inputs.source_signal(cfg, steps + 1), np.zeros(sysm.n_dof))
    err = np.linalg.norm(u - ref) / np.linalg.norm(ref)
    assert np.abs(ref).max() > 0 and err < 1e-10, err
    # Lanczos in the HRZ mass inner product (sc_estimate_dt): converged to rounding
    assert lam_gpu <= lam * (1 + 1e-12) and abs(lam_gpu - lam) / lam < 1e-10, (lam_gpu, lam)


def test_hrz_step_is_restricted_by_cut_cells(pkg):
    # the point of the method: the explicit HRZ scheme's critical step on config 2
    # is far below the IMEX step, which the uncut cells alone set
    cfg = dict(sc_inputs.get_config(2))
    cfg["integrator"] = "cdm_hrz"
    s = pkg.from_config(cfg)
    _, dt_hrz = s.estimate_dt(3000)
    s.close()
    assert dt_hrz < 0.5 * cfg["dt"]


@pytest.mark.parametrize("dim,cells,p,void", CASES[:2])
def test_trapezoidal_and_consistent_cdm_match_oracle(pkg, dim, cells, p, void):
    """NEXT-1(a, b): CDM on the consistent SCM (integrator 3) and trapezoidal Newmark on all DOFs
    (integrator 2) on the same kernels, against oracle.integrators.cdm_consistent / trapezoidal
    (pinned in tests/test_oracle_integrators.py)."""
    from oracle.integrators import cdm_consistent, from_system, trapezoidal
    steps = 80
    cfg = sc_inputs.small_config(dim, cells, p, voids=[void], depth=2, steps=steps,
                                 source={"x": [0.25, 0.3, 0.3], "f0": 5.0})
    sysm = build_system(cfg, "sparse")
    pr = from_system(sysm)
    # consistent CDM at half its critical step (device estimate vs the dense eigenvalue)
    lam = lambda_max(sysm.K.toarray(), sysm.M.toarray())
    c3 = dict(cfg, dt=0.5 * 2.0 / np.sqrt(lam), integrator="cdm_consistent")
    s = pkg.from_config(c3)
    s.step(steps)
    u = s.read()
    lam_gpu, _ = s.estimate_dt(6000)
    s.close()
    ref = cdm_consistent(pr, c3["dt"], steps, sc_inputs.source_signal(c3, steps + 1), np.zeros(sysm.n_dof))
    assert np.linalg.norm(u - ref) / np.linalg.norm(ref) < 1e-10
    assert abs(lam_gpu - lam) / lam < 1e-3
    # trapezoidal Newmark on all DOFs at 3x the IMEX step (unconditionally stable)
    from oracle.spectra import dt_crit_uncut
    c2 = dict(cfg, dt=3.0 * 0.9 * dt_crit_uncut(dim, p, 1.0 / max(cells)), integrator="trapezoidal")
    s = pkg.from_config(c2)
    assert s.info["n_d"] == 0 and s.info["n_c"] == sysm.n_dof
    s.step(steps)
    u = s.read()
    s.close()
    M = sysm.M
    prt = Problem(M, sysm.K, sysm.f_x, np.array([], dtype=int), np.arange(sysm.n_dof))
    ref = trapezoidal(prt, c2["dt"], steps, sc_inputs.source_signal(c2, steps + 1), np.zeros(sysm.n_dof))
    assert np.linalg.norm(u - ref) / np.linalg.norm(ref) < 1e-10
