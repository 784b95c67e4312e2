"""BASELINE configs[4] (160^3 cells, p = 4, 200 voids; the bench workload) at FULL size in the
launch configuration bench.py times.  The oracle cannot step 2.6e8 DOFs in test time, so:
* cell classification is local to a cell: the GPU's classes on the corner 20^3-cell block
  must equal, bit for bit, the oracle's classification of that sub-box (same h, same voids);
* properties that hold at any size: two runs are bit-identical (determinism), the in-process
  2-rank slab decomposition reproduces the single-rank state bit for bit, the state stays
  finite and the DOF counts are consistent."""
import os
import sys

import numpy as np
import pytest

import sc_inputs
from oracle.assembly import classify

pytestmark = [pytest.mark.gpu]

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


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


@pytest.fixture(scope="module")
def cfg():
    return sc_inputs.get_config(5)


def test_config5_corner_classification_bit_exact(pkg, cfg):
    sys.path.insert(0, ROOT)
    from bench import sub_box
    s = pkg.from_config(cfg)
    cc, isc, lat = s.classification()
    info = s.info
    s.close()
    N = cfg["cells"][0]
    assert info["n_dof"] == len(lat) and info["n_c"] == int(isc.sum())
    assert info["cells_uncut"] + info["cells_cut"] + info["cells_empty"] == N ** 3
    sub = sub_box(cfg, 0.125)
    n = sub["cells"][0]
    ref = classify(sub).cell_class.reshape(n, n, n)
    mine = cc.reshape(N, N, N)[:n, :n, :n]
    assert np.array_equal(mine, ref)
    assert (ref == 1).sum() > 0          # the block holds cut cells


def test_config5_determinism_and_two_rank_decomposition(pkg, cfg):
    steps = 12
    a = pkg.from_config(cfg)
    a.step(steps)
    ua = a.read()
    a.close()
    b = pkg.from_config(cfg)
    b.step(steps)
    ub = b.read()
    b.close()
    assert np.all(np.isfinite(ua)) and np.abs(ua).max() > 0
    assert np.array_equal(ua, ub)
    ranks = [pkg.from_config(cfg, rank=r, world=2) for r in range(2)]
    for _ in range(steps):
        for s in ranks:
            s.step(1)
        pkg.exchange_local(ranks)
    ug = pkg.read_group(ranks)
    for s in ranks:
        s.close()
    assert np.array_equal(ug, ua)
