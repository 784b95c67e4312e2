"""The five BASELINE.json configurations as explicit input dictionaries.

Restated from BASELINE.json ``configs`` with the readings of DESIGN.md §3
(SURVEY.md §8(c) C8-C15, §8(d) table):

1. 1D, [0,1], 32 cells, p=4, half-space void x > 0.937, alpha=1e-5, D=3
   (C9), u0 = exp(-(x-0.3)^2/0.002), v0 = 0, no source, 2000 steps.
2. 2D, [0,1]^2, 64^2 cells, p=4, circle r=0.2 at (0.5,0.5), D=3,
   alpha=1e-5, Ricker f0=10 at (0.25,0.25), 5000 steps.
3. 2D porous plate, 256^2 cells, p=4, 40 seeded ellipses (semi-axes
   U[0.01,0.04]), D=3, alpha=1e-6, Ricker f0=20 at (0, 0.5) (C15), 10000 steps.
4. 3D, 64^3 cells, p=3, 12 seeded spheres r ~ U[0.03,0.08], D=2,
   alpha=1e-5, Ricker f0=8 at (0.1,0.5,0.5), 2000 steps.
5. 3D, 160^3 cells, p=4, 200 seeded ellipsoids (semi-axes U[0.01,0.03]),
   D=2, alpha=1e-6, Ricker f0=15 at (0.1,0.5,0.5) (C14), 1000 steps.

Config 6 is NOT a BASELINE config: the high-cut-fraction stress case of SURVEY NEXT-1(1b)
(the paper's pillar has 51% cut DOFs; configs 2-5 have 1-4%): 2D, 128^2 cells, p=4,
400 seeded ellipses (semi-axes U[0.006,0.015]) -> 31% c DOFs, D=3, alpha=1e-6, Ricker f0=20
at (0, 0.5), 5000 steps.

rho = c = 1 (C10); homogeneous Neumann on the box; lattice_s = 4 (C6);
fill_eps = 1e-10.  dt = 0.9 x the uncut cell-wise critical step
(C12), written here as full-precision literals produced by
``scripts/gen_dt_literals.py`` (which calls only oracle/); the oracle test
``test_config_dt`` re-checks each literal (this module does no eigen-analysis).
"""
import numpy as np

from .voids import generate_voids
from .signals import ricker_series, signal_series

CONFIG_IDS = (1, 2, 3, 4, 5)   # BASELINE configs; 6 = NEXT-1(1b) stress case

# dt literals (reading C12): 0.9 * Delta t_crit^uncut (scripts/gen_dt_literals.py).
_DT = {1: 0.004154166182068483, 2: 0.0015247322583105771, 3: 0.0003811830645776443,
       4: 0.002096313728906055, 5: 0.0004979754702963185, 6: 0.0007623661291552886}


def _base(cid, dim, n, p, alpha, depth, steps):
    return {
        "id": cid, "dim": dim, "cells": [n] * dim, "lo": [0.0] * dim, "hi": [1.0] * dim,
        "p": p, "alpha": alpha, "tree_depth": depth, "lattice_s": 4, "fill_eps": 1e-10,
        "rho": 1.0, "c": 1.0, "voids": [], "source": None, "u0": None,
        "dt": _DT[cid], "steps": steps,
    }


def get_config(cid, steps=None):
    """Return the explicit input dict of BASELINE config ``cid`` (1..5) or the stress case 6."""
    if cid == 1:
        cfg = _base(1, 1, 32, 4, 1e-5, 3, 2000)
        cfg["voids"] = [{"kind": "halfspace", "n": [1.0, 0.0, 0.0], "b": 0.937}]
        cfg["u0"] = "gaussian_pulse"
        cfg["name"] = "1D-cut-bar-32xp4"
    elif cid == 2:
        cfg = _base(2, 2, 64, 4, 1e-5, 3, 5000)
        cfg["voids"] = [{"kind": "ellipsoid", "c": [0.5, 0.5, 0.0],
                         "A": [25.0, 25.0, 0.0, 0.0, 0.0, 0.0]}]
        cfg["source"] = {"x": [0.25, 0.25, 0.0], "f0": 10.0}
        cfg["name"] = "2D-circle-64x64xp4"
    elif cid == 3:
        cfg = _base(3, 2, 256, 4, 1e-6, 3, 10000)
        src = [0.0, 0.5, 0.0]
        cfg["voids"] = generate_voids(3, 2, 40, 0.01, 0.04, "ellipse", 1.0 / 256, src)
        cfg["source"] = {"x": src, "f0": 20.0}
        cfg["name"] = "2D-porous-plate-256x256xp4"
    elif cid == 4:
        cfg = _base(4, 3, 64, 3, 1e-5, 2, 2000)
        src = [0.1, 0.5, 0.5]
        cfg["voids"] = generate_voids(4, 3, 12, 0.03, 0.08, "sphere", 1.0 / 64, src)
        cfg["source"] = {"x": src, "f0": 8.0}
        cfg["name"] = "3D-spheres-64^3xp3"
    elif cid == 5:
        cfg = _base(5, 3, 160, 4, 1e-6, 2, 1000)
        src = [0.1, 0.5, 0.5]
        cfg["voids"] = generate_voids(5, 3, 200, 0.01, 0.03, "ellipsoid", 1.0 / 160, src)
        cfg["source"] = {"x": src, "f0": 15.0}
        cfg["name"] = "3D-ellipsoids-160^3xp4"
    elif cid == 6:
        cfg = _base(6, 2, 128, 4, 1e-6, 3, 5000)
        src = [0.0, 0.5, 0.0]
        cfg["voids"] = generate_voids(6, 2, 400, 0.006, 0.015, "ellipse", 1.0 / 128, src)
        cfg["source"] = {"x": src, "f0": 20.0}
        cfg["name"] = "2D-dense-voids-128x128xp4 (stress, 31% c DOFs)"
    else:
        raise ValueError(f"unknown config {cid}")
    if steps is not None:
        cfg["steps"] = int(steps)
    return cfg


def small_config(dim, cells, p, voids=(), alpha=1e-5, depth=2, dt=None, steps=10,
                 source=None, u0=None, lo=None, hi=None, rho=1.0, c=1.0):
    """A custom (test-sized) input dict with the same schema."""
    cells = list(cells)
    assert len(cells) == dim
    return {
        "id": 0, "name": "custom", "dim": dim, "cells": cells,
        "lo": list(lo) if lo is not None else [0.0] * dim,
        "hi": list(hi) if hi is not None else [1.0] * dim,
        "p": p, "alpha": alpha, "tree_depth": depth, "lattice_s": 4, "fill_eps": 1e-10,
        "rho": rho, "c": c, "voids": list(voids), "source": source, "u0": u0,
        "dt": dt, "steps": steps,
    }


def source_signal(cfg, n_values=None):
    """f_t(k*dt), k = 0..n_values-1 (default steps+1), or None without source."""
    if cfg["source"] is None:
        return None
    if n_values is None:
        n_values = cfg["steps"] + 1
    kind = cfg["source"].get("signal", "ricker")
    if kind == "ricker":
        return ricker_series(cfg["source"]["f0"], cfg["dt"], n_values)
    return signal_series(kind, cfg["source"]["f0"], cfg["dt"], n_values)


def describe(cfg):
    return {k: cfg[k] for k in ("id", "name", "dim", "cells", "p", "alpha", "tree_depth",
                                "dt", "steps")} | {"n_voids": len(cfg["voids"])}


__all__ = ["get_config", "small_config", "source_signal", "describe", "CONFIG_IDS", "np"]
