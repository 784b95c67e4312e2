"""NEXT-4: leap-frog substepping of the cut DOFs on the same
kernels (integrator 4: the explicit d update with dt, then m CDM substeps of dt/m of the c DOFs
on the consistent M^cc through its factor), both readings of the unstated coupling rule (LF3:
interpolated / frozen d values during the substeps), against the oracle's leapfrog (pinned in
tests/test_oracle_leapfrog.py) at the IMEX step of each case, with m chosen so that dt/m is half
the critical step of the cut block (K^cc, M^cc)."""
import numpy as np
import pytest

import sc_inputs
from oracle.assembly import build_system
from oracle.integrators import from_system, leapfrog
from oracle.spectra import dt_crit, dt_crit_uncut

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
         (3, [5, 4, 6], 2, {"kind": "ellipsoid", "c": [0.5, 0.45, 0.5], "A": [30.0, 40.0, 35.0, 2.0, 1.0, 0.0]})]


@pytest.mark.parametrize("coupling", ["interpolated", "frozen"])
@pytest.mark.parametrize("dim,cells,p,void", CASES)
def test_leapfrog_matches_oracle(pkg, dim, cells, p, void, coupling):
    steps = 60
    cfg = sc_inputs.small_config(dim, cells, p, voids=[void], depth=2, steps=steps,
                                 source={"x": [0.25, 0.3, 0.3], "f0": 5.0})
    cfg["dt"] = 0.5 * dt_crit_uncut(dim, p, 1.0 / max(cells))
    sysm = build_system(cfg, "sparse")
    Ic = sysm.I_c
    Kcc = sysm.K[Ic][:, Ic].toarray()
    dtc = dt_crit(Kcc, sysm.M_cc.toarray())
    m = int(np.ceil(cfg["dt"] / (0.5 * dtc)))
    assert 1 < m <= 64
    cfg.update(integrator="leapfrog", lf_m=m, lf_coupling=coupling)
    s = pkg.from_config(cfg)
    s.step(steps)
    u = s.read()
    s.close()
    f_t = sc_inputs.source_signal(cfg, steps + 2)
    ref = leapfrog(from_system(sysm), cfg["dt"], steps, f_t, np.zeros(sysm.n_dof), m, coupling)
    err = np.linalg.norm(u - ref) / np.linalg.norm(ref)
    assert np.abs(ref).max() > 0 and err < 1e-10, (err, m)


def test_leapfrog_config_errors(pkg):
    cfg = sc_inputs.small_config(2, [4, 4], 2, voids=[], steps=1)
    cfg["dt"] = 1e-3
    cfg.update(integrator="leapfrog", lf_m=0)
    with pytest.raises(pkg.ScError) as e:
        pkg.from_config(cfg)
    assert e.value.status == pkg.SC_ERR_CONFIG
