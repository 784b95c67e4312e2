"""Multi-rank slab decomposition validated on ONE GPU: world ranks live in
one process (sc_dist with world > 1 and no NCCL id) and exchange through device copies
(sc_exchange_local) after every step.  The ranks' owned DOFs must reproduce the single-rank
run bit for bit (same per-node arithmetic on every rank), hence the oracle within 1e-10."""
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


def _run_group(pkg, cfg, world, steps):
    ranks = [pkg.from_config(cfg, rank=r, world=world) for r in range(world)]
    for _ in range(steps):
        for s in ranks:
            s.step(1)
        pkg.exchange_local(ranks)
    u = pkg.read_group(ranks)
    infos = [s.info for s in ranks]
    for s in ranks:
        s.sync()
        s.close()
    return u, infos


def _single(pkg, cfg, steps):
    s = pkg.from_config(cfg)
    s.step(steps)
    u = s.read()
    s.close()
    return u


def _small(dim, cells, p, voids, steps, depth=2, source=None):
    cfg = sc_inputs.small_config(dim, cells, p, voids=voids, depth=depth, steps=steps, source=source)
    cfg["dt"] = 0.9 * dt_crit_uncut(dim, p, 1.0 / max(cells))
    return cfg


# voids placed so that c components straddle the slab boundaries of 2-4 ranks
SPHERES = [{"kind": "ellipsoid", "c": [0.5, 0.45, 0.5], "A": [1 / 0.02, 1 / 0.03, 1 / 0.025, 2.0, 1.0, 0.5]},
           {"kind": "ellipsoid", "c": [0.3, 0.6, 0.26], "A": [60.0, 60.0, 60.0, 0.0, 0.0, 0.0]},
           {"kind": "ellipsoid", "c": [0.7, 0.3, 0.76], "A": [80.0, 50.0, 70.0, 0.0, 0.0, 0.0]}]


@pytest.mark.parametrize("world", [2, 3, 4])
def test_3d_slabs_match_single_rank_bitwise(pkg, world):
    cfg = _small(3, [8, 7, 12], 3, SPHERES, 25, source={"x": [0.2, 0.5, 0.5], "f0": 4.0})
    ref = _single(pkg, cfg, 25)
    u, infos = _run_group(pkg, cfg, world, 25)
    assert sum(i["n_owned"] for i in infos) == infos[0]["n_dof"]
    assert sum(i["n_c_local"] for i in infos) == infos[0]["n_c"]
    assert np.array_equal(u, ref), np.abs(u - ref).max()


def test_2d_config2_two_and_four_ranks_vs_oracle(pkg):
    cfg = sc_inputs.get_config(2)
    steps = 400
    for world in (2, 4):
        u, infos = _run_group(pkg, cfg, world, steps)
        assert all(i["halo_recv"] > 0 for i in infos)
        if world == 2:
            ref, _ = run_config(cfg, steps=steps)
            err = np.linalg.norm(u - ref) / np.linalg.norm(ref)
            assert err < 1e-10, err
            u2 = u
        else:
            assert np.array_equal(u, u2)


def test_1d_config1_three_ranks(pkg):
    cfg = sc_inputs.get_config(1)
    ref = _single(pkg, cfg, 500)
    u, _ = _run_group(pkg, cfg, 3, 500)
    assert np.array_equal(u, ref)
