"""The paper's temporal excitations as inputs (sc_inputs.signals), pinned to properties their
definitions fix: the Gaussian derivative of PAPER.md P:847-850 (Eq. eq:ft) and the two-cycle
sine burst of P:1759-1764.  (Inputs only: both the oracle and the CUDA path receive the same
host-computed series.)"""
import numpy as np

from sc_inputs.signals import gaussian_derivative, sine_burst, signal_series


def test_gaussian_derivative_shape():
    fs = 2.0                                    # the paper's plate example
    t0, sig = 1.0 / fs, 1.0 / (2.0 * np.pi * fs)
    assert gaussian_derivative(t0, fs) == 0.0   # centred at t0
    # odd about t0
    for d in (0.01, 0.05, 0.2):
        assert np.isclose(gaussian_derivative(t0 - d, fs), -gaussian_derivative(t0 + d, fs), rtol=1e-14)
    # extrema at t0 -/+ sigma with value +/- e^{-1/2} / (sqrt(2 pi) sigma^2)
    peak = np.exp(-0.5) / (np.sqrt(2 * np.pi) * sig ** 2)
    assert np.isclose(gaussian_derivative(t0 - sig, fs), peak, rtol=1e-14)
    tt = np.linspace(0.0, 2.0 * t0, 200001)
    g = gaussian_derivative(tt, fs)
    assert np.isclose(tt[np.argmax(g)], t0 - sig, atol=2e-5)
    # it is d/dt of the unit-mass Gaussian: its integral over [0, 2 t0] ~ 0, and its first
    # moment -int (t - t0) g dt = 1 (the Gaussian's mass) up to the truncated tails
    dt = tt[1] - tt[0]
    assert abs(np.trapezoid(g, dx=dt)) < 1e-9 * peak
    assert np.isclose(-np.trapezoid((tt - t0) * g, dx=dt), 1.0, atol=1e-6)
    # starts from ~0 (t0 = 2 pi sigma: the pulse is 6.3 sigma from t = 0)
    assert abs(gaussian_derivative(0.0, fs)) < 1e-7 * peak


def test_sine_burst_shape():
    fs, nc = 20e3, 2                            # the pillar example
    T = nc / fs
    assert sine_burst(0.0, fs) == 0.0
    assert np.all(sine_burst(np.array([T * 1.0001, 2 * T, 10 * T]), fs) == 0.0)
    assert abs(sine_burst(T, fs)) < 1e-12      # continuous at the end of the burst
    t = np.linspace(0.0, T, 100001)
    v = sine_burst(t, fs)
    assert 0.0 < np.abs(v).max() <= 1.0
    # at fs t = 1/4 the carrier is sin(pi/2) = 1 and the window sin^2(pi/8)
    assert np.isclose(sine_burst(0.25 / fs, fs), np.sin(np.pi / 8) ** 2, rtol=1e-14)
    # the window sin^2(pi fs t / nc) is symmetric about T/2 and the carrier odd about it: the
    # burst is odd about T/2
    assert np.allclose(v, -v[::-1], atol=1e-12)


def test_signal_series_sampling():
    dt, n = 1e-3, 50
    assert np.array_equal(signal_series("sine_burst", 100.0, dt, n), sine_burst(np.arange(n) * dt, 100.0))
    assert np.array_equal(signal_series("gauss_deriv", 2.0, dt, n), gaussian_derivative(np.arange(n) * dt, 2.0))
