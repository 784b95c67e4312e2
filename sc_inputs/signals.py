"""Temporal signals and initial fields (inputs only, no method arithmetic).

* Ricker wavelet: NOT in the paper (the paper uses a Gaussian-derivative
  f_t, PAPER.md P:847-850 Eq. ``eq:ft``, and a two-cycle sine burst,
  P:1758-1765).  BASELINE.json's configs name a point Ricker source, so we
  use R(t) = (1 - 2 pi^2 f0^2 (t-t0)^2) exp(-pi^2 f0^2 (t-t0)^2) with
  t0 = 1.5/f0 (reading C11; |R(0)| ~ 1e-8, following the paper's
  convention of centring the pulse so it starts from ~0).
  f_t(t_k) is precomputed here on the host for every t_k = k*dt and handed
  to BOTH sides, so no CPU/GPU ``exp`` ulp difference can enter.
* Config-1 initial field u0(x) = exp(-(x-0.3)^2/0.002) (BASELINE.json
  configs[0]); both sides interpolate it nodally at their own node
  coordinates (reading C16).
"""
import numpy as np


def ricker(t, f0):
    t = np.asarray(t, dtype=np.float64)
    t0 = 1.5 / f0
    a = (np.pi * f0 * (t - t0)) ** 2
    return (1.0 - 2.0 * a) * np.exp(-a)


def gaussian_pulse(x):
    x = np.asarray(x, dtype=np.float64)
    return np.exp(-((x - 0.3) ** 2) / 0.002)


def ricker_series(f0, dt, n_values):
    """f_t(k*dt) for k = 0 .. n_values-1."""
    return ricker(np.arange(n_values, dtype=np.float64) * dt, f0)
