"""Temporal signals and initial fields (inputs only, no method arithmetic).

* Ricker wavelet: NOT in the paper (the paper uses a Gaussian-derivative
  f_t, PAPER.md P:847-850 Eq. ``eq:ft``, and a two-cycle sine burst,
  P:1758-1765).  BASELINE.json's configs name a point Ricker source, so we
  use R(t) = (1 - 2 pi^2 f0^2 (t-t0)^2) exp(-pi^2 f0^2 (t-t0)^2) with
  t0 = 1.5/f0 (reading C11; |R(0)| ~ 1e-8, following the paper's
  convention of centring the pulse so it starts from ~0).
  f_t(t_k) is precomputed here on the host for every t_k = k*dt and handed
  to BOTH sides, so no CPU/GPU ``exp`` ulp difference can enter.
* The paper's own temporal signals (inputs like the Ricker series): the derivative of a
  Gaussian, PAPER.md P:847-850 Eq. ``eq:ft``, f_t(t) = -(t - t0) / (sqrt(2 pi) sigma^3)
  exp(-(t - t0)^2 / (2 sigma^2)), t0 = 1/f_s, sigma = 1/(2 pi f_s); and the n_c-cycle sine
  burst, f_t(t) = sin(2 pi f_s t) sin^2(pi f_s t / n_c) for t <= n_c/f_s, else 0.
  Select with cfg["source"]["signal"] = "ricker" (default) | "gauss_deriv" | "sine_burst".
* Config-1 initial field u0(x) = exp(-(x-0.3)^2/0.002) (BASELINE.json
  configs[0]); both sides interpolate it nodally at their own node
  coordinates (reading C16).
* Compactly supported initial displacement u0(x) = (1 - |x - x0|^2 / R^2)^4 for
  |x - x0| < R, else 0 (a C^3 bump; P:752 gives the initial displacement as an input).  Its
  exact zero outside the ball bounds the dependency region of a finite number of steps, so
  a full-size run can be checked against the oracle on a sub-box (tests/subbox.py).
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


def gaussian_derivative(t, fs):
    """PAPER.md P:847-850 Eq. eq:ft: t0 = 1/fs, sigma_t = 1/(2 pi fs)."""
    t = np.asarray(t, dtype=np.float64)
    t0 = 1.0 / fs
    sig = 1.0 / (2.0 * np.pi * fs)
    return -(t - t0) / (np.sqrt(2.0 * np.pi) * sig ** 3) * np.exp(-((t - t0) ** 2) / (2.0 * sig ** 2))


def sine_burst(t, fs, n_cycles=2):
    """n_c-cycle sine burst (n_c = 2 in the paper)."""
    t = np.asarray(t, dtype=np.float64)
    v = np.sin(2.0 * np.pi * fs * t) * np.sin(np.pi * fs * t / n_cycles) ** 2
    return np.where(t <= n_cycles / fs, v, 0.0)


def signal_series(kind, f0, dt, n_values):
    """f_t(k*dt) for k = 0 .. n_values-1 of the named signal."""
    t = np.arange(n_values, dtype=np.float64) * dt
    if kind == "ricker":
        return ricker(t, f0)
    if kind == "gauss_deriv":
        return gaussian_derivative(t, f0)
    if kind == "sine_burst":
        return sine_burst(t, f0)
    raise ValueError(f"unknown signal {kind!r}")


def compact_bump(X, x0, R):
    """u0 at the points X (n x 3): (1 - r^2/R^2)^4 for r = |X - x0| < R, else exactly 0."""
    X = np.asarray(X, dtype=np.float64)
    x0 = np.asarray(x0, dtype=np.float64)
    r2 = np.sum((X[:, :len(x0)] - x0[None, :]) ** 2, axis=1)
    q = 1.0 - r2 / (R * R)
    return np.where(q > 0.0, q ** 4, 0.0)
