"""NEXT-3: receiver traces u(x_r, t_n) recorded on the device after every step
(sc_set_receivers / sc_read_traces) against the oracle's IMEX run observed at the same
points (basis of the lowest-index non-empty cell containing x_r)."""
import numpy as np
import pytest

import sc_inputs
from oracle.assembly import build_system, point_values
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


@pytest.mark.parametrize("dim,cells,p,recv", [
    (2, [10, 9], 3, [[0.15, 0.8, 0.0], [0.3, 1.0 / 3.0, 0.0], [0.85, 0.15, 0.0], [0.7, 0.62, 0.0]]),
    (3, [5, 4, 6], 2, [[0.5, 0.5, 0.75], [0.1, 0.9, 0.2], [0.4, 0.25, 0.5]])])
def test_receiver_traces_match_oracle(pkg, dim, cells, p, recv):
    void = {"kind": "ellipsoid", "c": [0.5, 0.45, 0.5], "A": [30.0, 40.0, 35.0, 2.0, 1.0, 0.0]}
    if dim == 2:
        void = {"kind": "ellipsoid", "c": [0.55, 0.45, 0.0], "A": [40.0, 60.0, 0.0, 5.0, 0.0, 0.0]}
    steps = 40
    cfg = sc_inputs.small_config(dim, cells, p, voids=[void], depth=2, steps=steps,
                                 source={"x": [0.25, 0.3, 0.3], "f0": 5.0})
    cfg["dt"] = 0.9 * dt_crit_uncut(dim, p, 1.0 / max(cells))
    s = pkg.from_config(cfg)
    s.set_receivers(recv, capacity=steps + 5)
    s.step(steps)
    tr = s.traces()
    s.close()
    assert tr.shape == (steps, len(recv))
    sysm = build_system(cfg, "sparse")
    W = np.stack([point_values(cfg, sysm.cl, np.asarray(x[:dim])) for x in recv])
    ref = []
    imex(from_system(sysm), cfg["dt"], steps, sc_inputs.source_signal(cfg, steps + 1), np.zeros(sysm.n_dof),
         observer=lambda k, u: ref.append(W @ u))
    ref = np.array(ref)
    err = np.linalg.norm(tr - ref) / np.linalg.norm(ref)
    assert np.abs(ref).max() > 0 and err < 1e-10, err


def test_paper_excitations_match_oracle(pkg):
    """The paper's own temporal signals (Gaussian derivative; two-cycle sine burst,
    P:1759-1764) through the same path: device state after 40 steps vs the oracle's IMEX."""
    from oracle.run import run_config
    for sig, f0 in (("gauss_deriv", 6.0), ("sine_burst", 12.0)):
        steps = 40
        cfg = sc_inputs.small_config(2, [10, 9], 3, depth=2, steps=steps,
                                     voids=[{"kind": "ellipsoid", "c": [0.55, 0.45, 0.0],
                                             "A": [40.0, 60.0, 0.0, 5.0, 0.0, 0.0]}],
                                     source={"x": [0.25, 0.3, 0.3], "f0": f0, "signal": sig})
        cfg["dt"] = 0.9 * dt_crit_uncut(2, 3, 1.0 / 10)
        f_t = sc_inputs.source_signal(cfg, steps + 2)
        assert np.abs(f_t).max() > 0
        s = pkg.from_config(cfg, f_t=f_t)
        s.step(steps)
        u = s.read()
        s.close()
        ref, _ = run_config(cfg, sysm=build_system(cfg, "sparse"), f_t=f_t)
        err = np.linalg.norm(u - ref) / np.linalg.norm(ref)
        assert np.linalg.norm(ref) > 0 and err < 1e-10, (sig, err)
