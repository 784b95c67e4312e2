"""NEXT-3: the elastic-energy observer E = 1/2 u^T K u computed on
the device (sc_elastic_energy) against the oracle's assembled K (oracle.integrators.Problem.Ku)
applied to the same state, across the node classes that route through different kernels
(tensor-d far/near, irregular d next to empty cells, c rows through the c-element products)."""
import numpy as np
import pytest

import sc_inputs
from oracle.assembly import build_system
from oracle.integrators import from_system, imex
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


def _cfg(dim, integrator="imex"):
    if dim == 1:
        cfg = sc_inputs.get_config(1, steps=30)
    elif dim == 2:
        cfg = sc_inputs.small_config(2, [10, 9], 3, depth=2, steps=30,
                                     voids=[{"kind": "ellipsoid", "c": [0.55, 0.45, 0.0],
                                             "A": [40.0, 60.0, 0.0, 5.0, 0.0, 0.0]}],
                                     source={"x": [0.25, 0.3, 0.3], "f0": 5.0})
        cfg["dt"] = 0.9 * dt_crit_uncut(2, 3, 1.0 / 10)
    else:
        cfg = sc_inputs.small_config(3, [5, 4, 6], 2, depth=2, steps=30,
                                     voids=[{"kind": "ellipsoid", "c": [0.5, 0.45, 0.5],
                                             "A": [30.0, 40.0, 35.0, 2.0, 1.0, 0.0]}],
                                     source={"x": [0.25, 0.3, 0.3], "f0": 5.0})
        cfg["dt"] = 0.9 * dt_crit_uncut(3, 2, 1.0 / 6)
    cfg["integrator"] = integrator
    return cfg


def _bound(u, Ku):
    # rounding bound of a length-n dot product, relative to sum |u_i (K u)_i|
    return 1e-11 * 0.5 * np.abs(u * Ku).sum() + 1e-300


@pytest.mark.parametrize("dim,integrator", [(1, "imex"), (2, "imex"), (3, "imex"), (2, "trapezoidal")])
def test_energy_matches_oracle_on_the_same_state(pkg, dim, integrator):
    cfg = _cfg(dim, integrator)
    sysm = build_system(cfg, "sparse")
    pr = from_system(sysm)
    steps = 25
    s = pkg.from_config(cfg, f_t=sc_inputs.source_signal(cfg, steps + 1) if cfg.get("source") else None)
    s.step(steps)
    u = s.read()
    e_gpu = s.elastic_energy()
    u_after = s.read()
    e_again = s.elastic_energy()
    s.close()
    Ku = pr.Ku(u)
    e_ref = 0.5 * float(u @ Ku)
    assert e_ref > 0.0
    assert abs(e_gpu - e_ref) <= _bound(u, Ku), (e_gpu, e_ref)
    assert np.array_equal(u, u_after)      # the observer does not touch the state
    assert e_again == e_gpu                # fixed-order reduction: bit-reproducible


def test_energy_follows_the_oracle_trajectory(pkg):
    # the device energy after n steps vs the oracle's own IMEX state after n steps
    cfg = _cfg(2)
    sysm = build_system(cfg, "sparse")
    pr = from_system(sysm)
    steps = 30
    f_t = sc_inputs.source_signal(cfg, steps + 1)
    s = pkg.from_config(cfg, f_t=f_t)
    got = []
    for _ in range(3):
        s.step(10)
        got.append(s.elastic_energy())
    s.close()
    ref = []
    imex(pr, cfg["dt"], steps, f_t, np.zeros(sysm.n_dof),
         observer=lambda k, u: ref.append(0.5 * float(u @ pr.Ku(u))) if k % 10 == 0 else None)
    assert len(ref) == 3
    np.testing.assert_allclose(got, ref, rtol=1e-9, atol=0.0)


def test_energy_of_a_constant_field_is_zero(pkg):
    # homogeneous Neumann boundaries: constants are in the kernel of K, so E(1) = 0
    cfg = _cfg(3)
    sysm = build_system(cfg, "sparse")
    s = pkg.from_config(cfg)
    n = s.info["n_dof"]
    s.set_state(np.ones(n), np.zeros(n))
    e1 = s.elastic_energy()
    rng = np.random.default_rng(7)
    s.set_state(rng.standard_normal(n), np.zeros(n))
    e_rand = s.elastic_energy()
    s.close()
    assert e_rand > 0.0
    assert abs(e1) <= 1e-12 * e_rand
