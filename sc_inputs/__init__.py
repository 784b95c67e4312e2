"""Seeded synthetic input generators shared by the oracle and the CUDA path.

This module holds NONE of the method's arithmetic (no basis, quadrature,
classification, assembly or time stepping).  It only produces the *inputs*
of the problem statement (§Spatial Discretization: domain,
material, alpha, initial conditions, separable source f = f_t(t) f_x,
P:456-459):

* ``configs``  - the five BASELINE.json configurations, restated concretely
                 (readings C8-C15 in DESIGN.md);
* ``voids``    - seeded void (ellipse / sphere / ellipsoid) generation
                 (reading C13);
* ``signals``  - the Ricker wavelet f_t(t_k) (reading C11, NOT in the paper)
                 and the config-1 Gaussian initial field u0(x).

Both the oracle (``oracle/``) and the product path
(``paper_2310_14712_b200``) consume exactly the dictionaries built here, so
"same seeded inputs" holds by construction.
"""
from .configs import get_config, CONFIG_IDS, small_config, source_signal, describe  # noqa: F401
from .signals import ricker, gaussian_pulse, gaussian_derivative, sine_burst, compact_bump  # noqa: F401
