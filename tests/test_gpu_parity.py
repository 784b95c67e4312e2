"""GPU parity: the CUDA path (through the C ABI) vs the CPU oracle on the same seeded
inputs.  Bars (BASELINE.json north_star): bit-exact cell classification and d/c DOF
partition; relative L2 <= 1e-10 in u after the stated step count."""
import numpy as np
import pytest

import sc_inputs
from oracle.assembly import build_system, classify
from oracle.run import run_config
from oracle.spectra import dt_crit_uncut

pytestmark = pytest.mark.gpu

TOL = 1e-10


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


def _rel(a, b):
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


def _check(pkg, cfg, steps, mode="sparse", tol=TOL):
    cfg = dict(cfg)
    cfg["steps"] = steps
    s = pkg.from_config(cfg)
    s.step(steps)
    u = s.read()
    sysm = build_system(cfg, mode)
    ref, _ = run_config(cfg, steps=steps, sysm=sysm)
    cc, isc, lat = s.classification()
    assert np.array_equal(cc, sysm.cl.cell_class)
    assert np.array_equal(lat, sysm.cl.lattice_index)
    assert np.array_equal(isc, sysm.cl.is_c)
    err = _rel(u, ref)
    info = s.info
    s.close()
    assert np.all(np.isfinite(u))
    assert err <= tol, (err, info)
    return err, info


def _small(dim, cells, p, voids, steps=30, depth=2, alpha=1e-5, source=None, frac=0.9):
    cfg = sc_inputs.small_config(dim, cells, p, voids=voids, depth=depth, alpha=alpha, steps=steps,
                                 source=source)
    h = 1.0 / max(cells)
    cfg["dt"] = frac * dt_crit_uncut(dim, p, h)
    return cfg


CIRCLE = {"kind": "ellipsoid", "c": [0.47, 0.53, 0.0], "A": [1 / 0.06, 1 / 0.05, 0.0, 3.0, 0.0, 0.0]}
SPHERE = {"kind": "ellipsoid", "c": [0.52, 0.45, 0.5], "A": [1 / 0.05, 1 / 0.06, 1 / 0.07, 2.0, 1.0, 0.5]}


@pytest.mark.parametrize("p", [1, 2, 3, 4, 5, 6])
def test_2d_ragged_all_orders(pkg, p):
    # 13 x 11 cells: several tiles with ragged tails in x and y
    cfg = _small(2, [13, 11], p, [CIRCLE], steps=25, depth=3,
                 source={"x": [0.2, 0.3, 0.0], "f0": 5.0})
    _check(pkg, cfg, 25)


@pytest.mark.parametrize("p", [2, 3, 4])
def test_3d_ragged(pkg, p):
    cfg = _small(3, [7, 6, 9], p, [SPHERE], steps=15, depth=2,
                 source={"x": [0.21, 0.33, 0.4], "f0": 4.0})
    _check(pkg, cfg, 15)


# 3D explicit kernel layouts (explicit3w.cuh): several x-warps per plane group (named-barrier
# exchange of the element-boundary partials), several x segments (halo lane), y chunks with a
# warm-up element, the domain-end x node, non-cubic cells (s0 != s1 != s2), voids on x-warp
# boundaries (non-clean blocks).  cells, p, hi, void centre
LAYOUTS = [
    ([40, 3, 4], 2, [1.0, 0.15, 0.2], [0.80, 0.075, 0.1]),      # 2 x-warps, non-cubic
    ([70, 2, 3], 4, [1.0, 0.04, 0.06], [0.457, 0.02, 0.03]),    # 3 x-warps (one partly idle)
    ([64, 3, 2], 3, [1.0, 0.05, 0.03], [0.5, 0.025, 0.015]),    # exactly 2 full x-warps: end lane = lane 31
    ([170, 2, 2], 4, [1.0, 0.0118, 0.0118], [0.75, 0.006, 0.006]),   # 2 x segments (halo lane)
]


@pytest.mark.parametrize("cells,p,hi,vc", LAYOUTS)
def test_3d_kernel_layouts(pkg, cells, p, hi, vc):
    h = min(hi[k] / cells[k] for k in range(3))
    r = 1.6 * h
    void = {"kind": "ellipsoid", "c": vc, "A": [1 / r ** 2, 1 / r ** 2, 1 / r ** 2, 0.0, 0.0, 0.0]}
    cfg = sc_inputs.small_config(3, cells, p, voids=[void], depth=2, alpha=1e-5, steps=12, hi=hi,
                                 source={"x": [0.31, hi[1] * 0.4, hi[2] * 0.6], "f0": 6.0})
    cfg["dt"] = 0.9 * dt_crit_uncut(3, p, h)
    _check(pkg, cfg, 12, mode="ebe")


def test_1d_config1_full(pkg):
    # BASELINE configs[0] at its full 2000 steps
    _check(pkg, sc_inputs.get_config(1), 2000)


def test_all_uncut_box_is_cdm(pkg):
    # I_c empty: IMEX reduces to CDM; source inside a cell -> irregular nodes
    cfg = _small(2, [9, 10], 4, [], steps=200, source={"x": [0.41, 0.37, 0.0], "f0": 3.0})
    err, info = _check(pkg, cfg, 200)
    assert info["n_c"] == 0


def test_all_cut_is_trapezoidal(pkg):
    # every cell cut: I_d empty -> pure trapezoidal Newmark on all DOFs
    cfg = _small(2, [2, 2], 3, [{"kind": "ellipsoid", "c": [0.5, 0.5, 0.0],
                                 "A": [1 / 0.09, 1 / 0.09, 0.0, 0.0, 0.0, 0.0]}], steps=50)
    cfg["dt"] *= 3.0   # implicit: no explicit limit applies
    err, info = _check(pkg, cfg, 50)
    assert info["n_d"] == 0


def test_void_boundary_on_cell_face_irregular(pkg):
    # half-space void exactly on a cell face: d nodes next to empty cells (irregular path)
    cfg = _small(2, [8, 6], 3, [{"kind": "halfspace", "n": [1.0, 0.0, 0.0], "b": 0.75}], steps=80,
                 source={"x": [0.3, 0.5, 0.0], "f0": 4.0})
    err, info = _check(pkg, cfg, 80)
    assert info["n_irregular"] > 1


def test_3d_face_halfspace(pkg):
    cfg = _small(3, [4, 4, 6], 2, [{"kind": "halfspace", "n": [0.0, 0.0, 1.0], "b": 0.5},
                                   {"kind": "ellipsoid", "c": [0.5, 0.5, 0.25], "A": [40, 40, 40, 0, 0, 0]}],
                 steps=20, source={"x": [0.25, 0.25, 0.125], "f0": 3.0})
    _check(pkg, cfg, 20)


def test_config2_full(pkg):
    # BASELINE configs[1] at its full 5000 steps
    err, info = _check(pkg, sc_inputs.get_config(2), 5000)
    assert info["n_dof"] == 58752 and info["n_c"] == 1872


def test_config3_prefix(pkg):
    # BASELINE configs[2] at full size, 150-step prefix (oracle time bound)
    _check(pkg, sc_inputs.get_config(3), 150)


def test_config4_classification_and_prefix(pkg):
    # BASELINE configs[3] at full size: bit-exact classification + 6-step prefix (ebe oracle)
    _check(pkg, sc_inputs.get_config(4), 6, mode="ebe")


def test_determinism(pkg):
    cfg = sc_inputs.get_config(2)
    a = pkg.from_config(cfg)
    b = pkg.from_config(cfg)
    a.step(300)
    b.step(300)
    ua, ub = a.read(), b.read()
    a.close()
    b.close()
    assert np.array_equal(ua, ub)


def test_set_state_restart(pkg):
    cfg = sc_inputs.get_config(2)
    s = pkg.from_config(cfg)
    s.step(100)
    u100 = s.read()
    s.set_state(None, None)
    s.step(100)
    assert np.array_equal(s.read(), u100)
    s.close()


def test_numeric_failure_flagged(pkg):
    # 3x the explicit limit: the explicit subsystem blows up -> SC_ERR_NUMERIC
    cfg = _small(2, [6, 6], 2, [CIRCLE], steps=400, source={"x": [0.2, 0.3, 0.0], "f0": 5.0}, frac=3.0)
    s = pkg.from_config(cfg)
    s.step(400)
    with pytest.raises(pkg.ScError) as e:
        s.sync()
    assert e.value.status == pkg.SC_ERR_NUMERIC
    s.close()


def test_config_errors(pkg):
    cfg = _small(2, [4, 4], 2, [])
    with pytest.raises(pkg.ScError) as e:
        pkg.Solver(cfg, 0, 1e-5, {"voids": []}, cfg["dt"])
    assert e.value.status == pkg.SC_ERR_CONFIG
    with pytest.raises(pkg.ScError):
        pkg.Solver(cfg, 2, 1e-5, {"voids": []}, -1.0)
