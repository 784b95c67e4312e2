"""Pins of the oracle's leap-frog substepping (oracle.integrators.leapfrog; PAPER.md P:585-589,
readings LF1-LF4 of DESIGN.md: the coupling rule is not in the paper, so both the "frozen" and
the "interpolated" reading are built and pinned):
* m = 1 with the frozen coupling is CDM on the consistent SCM (cdm_consistent) bit for bit
  (the same arithmetic: every DOF advanced by one CDM step reading u_n);
* I_c empty: the leap-frog step is the diagonal CDM bit for bit, for any m;
* the spring chain of P:740-754 (the two light "cut" masses): at the coarse step of the
  explicit subsystem (0.9 dt_crit^explicit) plain CDM blows up, while leap-frog with the
  interpolated coupling and dt / m below the cut block's own critical step stays bounded -
  the point of substepping ("only dt_fine must satisfy the highly restrictive
  stability constraints"); the frozen coupling loses stability at such coarse steps
  (measured: unbounded for dt >= 0.5 dt_crit^explicit, bounded at 0.3);
* second-order convergence of the interpolated coupling at fixed m (slope 2 in dt)."""
import numpy as np
import pytest
import scipy.sparse as sp

from oracle.integrators import Problem, cdm, cdm_consistent, leapfrog
from oracle.spectra import dt_crit
from test_oracle_integrators import _random_system, _spring_problem, _golden_spring


@pytest.mark.parametrize("seed", range(4))
def test_m1_frozen_is_consistent_cdm(seed):
    rng = np.random.default_rng(300 + seed)
    n = int(rng.integers(5, 12))
    M, K = _random_system(rng, n, True)
    nd = n // 2
    Mc = rng.standard_normal((n - nd, n - nd)) * 0.2
    Mfull = np.zeros((n, n))
    Mfull[:nd, :nd] = np.diag(rng.uniform(0.5, 2.0, nd))
    Mfull[nd:, nd:] = np.eye(n - nd) + Mc @ Mc.T
    f = rng.standard_normal(n)
    f_t = rng.standard_normal(60)
    u0, v0 = rng.standard_normal(n), rng.standard_normal(n)
    pr = Problem(sp.csr_matrix(Mfull), K, f, np.arange(nd), np.arange(nd, n))
    dt = 0.5 * dt_crit(K.toarray(), Mfull)
    a = leapfrog(pr, dt, 50, f_t, u0, 1, "frozen", v0)
    b = cdm_consistent(pr, dt, 50, f_t, u0, v0)
    assert np.array_equal(a, b)


@pytest.mark.parametrize("m", [1, 3])
def test_no_cut_dofs_is_cdm(m):
    rng = np.random.default_rng(7)
    n = 8
    M, K = _random_system(rng, n, True)
    f, f_t = rng.standard_normal(n), rng.standard_normal(40)
    u0, v0 = rng.standard_normal(n), rng.standard_normal(n)
    pr = Problem(M, K, f, np.arange(n), np.array([], dtype=int))
    dt = 0.5 * dt_crit(K.toarray(), M.toarray())
    assert np.array_equal(leapfrog(pr, dt, 30, f_t, u0, m, "interpolated", v0), cdm(pr, dt, 30, f_t, u0, v0))


def _spring_run(coupling, dt, m, T):
    pr, A, w, g, K = _spring_problem()
    N = int(round(T / dt))
    f_t = np.sin(w * dt * np.arange(N + 2))
    E = []
    leapfrog(pr, dt, N, f_t, np.zeros(10), m, coupling, A * w,
             observer=lambda k, u: E.append(0.5 * u @ K @ u))
    return np.array(E)


def test_spring_chain_substepping_stability():
    pr, A, w, g, K = _spring_problem()
    dtc = dt_crit(K[8:, 8:], pr.M.toarray()[8:, 8:])   # the light (cut) block alone
    # interpolated coupling: substeps below the cut block's limit keep the chain stable at the
    # coarse step of the explicit subsystem; without substepping CDM on the cut block blows up
    dt = 0.9 * g["dt_crit_explicit"]
    m_ok = int(np.ceil(dt / (0.5 * dtc)))
    E_ok = _spring_run("interpolated", dt, m_ok, g["T"])
    assert np.all(np.isfinite(E_ok)) and E_ok.max() < 20.0
    E_bad = _spring_run("interpolated", dt, 1, g["T"])
    assert not np.all(np.isfinite(E_bad)) or E_bad.max() > 1e6
    # frozen coupling (u^d held at t_n during the substeps): measured to lose stability for
    # coarse steps >= 0.5 dt_crit^explicit whatever m (the non-symmetric time coupling), while
    # it is stable well below; the coupling rule the paper leaves to [meineMA] matters
    E_fz = _spring_run("frozen", dt, m_ok, g["T"])
    assert E_fz.max() > 100 * E_ok.max()
    dt3 = 0.3 * g["dt_crit_explicit"]
    E_fz3 = _spring_run("frozen", dt3, int(np.ceil(dt3 / (0.5 * dtc))), g["T"])
    assert np.all(np.isfinite(E_fz3)) and E_fz3.max() < 20.0


def test_interpolated_second_order():
    pr, A, w, g, K = _spring_problem()
    T = g["T"]
    errs = []
    for N in (2000, 4000, 8000):
        dt = T / N
        f_t = np.sin(w * dt * np.arange(N + 2))
        u = leapfrog(pr, dt, N, f_t, np.zeros(10), 2, "interpolated", A * w)
        errs.append(np.linalg.norm(u - A * np.sin(w * T)))
    s1, s2 = np.log2(errs[0] / errs[1]), np.log2(errs[1] / errs[2])
    assert 1.8 < s1 < 2.2 and 1.8 < s2 < 2.2, (errs, s1, s2)
