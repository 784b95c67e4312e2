"""Config dict -> assembled system -> Newmark IMEX run (ORACLE - test infra only).

Composes assembly and integrators.imex for the input
dictionaries of ``sc_inputs``: u0 by nodal interpolation (reading C16),
v0 = 0, f_t(t_k) from ``sc_inputs.source_signal`` (reading C11).
"""
import numpy as np

from sc_inputs import source_signal, gaussian_pulse
from .assembly import build_system, node_coords
from .integrators import from_system, imex


def initial_field(cfg, sysm):
    if cfg.get("u0") is None:
        return np.zeros(sysm.n_dof)
    if cfg["u0"] == "gaussian_pulse":
        X = node_coords(cfg, sysm.cl.lattice_index)
        return gaussian_pulse(X[:, 0])
    raise ValueError(cfg["u0"])


def run_config(cfg, steps=None, mode=None, sysm=None, observer=None, f_t=None):
    """Returns (u_N in canonical DOF order, system)."""
    if steps is None:
        steps = cfg["steps"]
    if sysm is None:
        if mode is None:
            mode = "sparse" if np.prod(cfg["cells"]) * (cfg["p"] + 1) ** (2 * cfg["dim"]) < 1.2e8 else "ebe"
        sysm = build_system(cfg, mode=mode)
    if f_t is None:
        f_t = source_signal(cfg, steps + 1)
    pr = from_system(sysm)
    u0 = initial_field(cfg, sysm)
    u = imex(pr, cfg["dt"], steps, f_t, u0, None, observer=observer)
    return u, sysm
