"""Writes the dt literals of sc_inputs/configs.py (reading C12).

dt = 0.9 * Delta t_crit^uncut, the cell-wise critical step of an uncut cell
(PAPER.md P:869), computed by the ORACLE (oracle.spectra.dt_crit_uncut).
This script calls only oracle/ and prints the dict to paste into
sc_inputs/configs.py; tests/test_oracle_integrators.py::test_config_dt
re-checks every literal.
"""
import sys
import os
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
from oracle.spectra import dt_crit_uncut  # noqa: E402

SPEC = {1: (1, 4, 1 / 32), 2: (2, 4, 1 / 64), 3: (2, 4, 1 / 256), 4: (3, 3, 1 / 64), 5: (3, 4, 1 / 160),
        6: (2, 4, 1 / 128)}
if __name__ == "__main__":
    out = {cid: 0.9 * dt_crit_uncut(d, p, h) for cid, (d, p, h) in SPEC.items()}
    print("_DT = {" + ", ".join(f"{k}: {v!r}" for k, v in out.items()) + "}")
