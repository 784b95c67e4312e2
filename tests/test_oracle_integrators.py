"""Pins of oracle/integrators.py and oracle/run.py (PAPER.md P:564-595,
§Spring-coupled masses P:740-758; readings C1-C4, C12)."""
import os

import numpy as np
import pytest
import scipy.sparse as sp

import sc_inputs
from oracle.integrators import Problem, imex, cdm, trapezoidal, from_system
from oracle.spectra import dt_crit, dt_crit_uncut
from oracle.assembly import build_system, node_coords
from oracle.run import run_config

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _golden_spring():
    vals = {}
    for line in open(os.path.join(GOLD, "spring_chain.txt")):
        if line.startswith("#") or not line.strip():
            continue
        k, v = line.split()[:2]
        vals[k] = float(v)
    return vals


def spring_chain():
    """Ten masses, wall spring at mass 1, mass 10 free (the topology
    is fixed by the two critical steps of P:678/P:682)."""
    g = _golden_spring()
    n = 10
    m = np.array([g["m1"]] * 8 + [g["m2"]] * 2)
    k = g["k"]
    K = np.zeros((n, n))
    for i in range(n):
        K[i, i] = 2 * k
        if i + 1 < n:
            K[i, i + 1] = K[i + 1, i] = -k
    K[n - 1, n - 1] = k
    f = np.zeros(n)
    f[n - 3] = 1.0                      # "third last mass"
    return np.diag(m), K, f, g


def test_spring_chain_critical_steps():
    M, K, f, g = spring_chain()
    assert abs(dt_crit(K, M) - g["dt_crit_global"]) < 5e-9
    # explicit subsystem = the eight 'uncut' masses (K^dd, M^dd)
    de = dt_crit(K[:8, :8], M[:8, :8])
    assert abs(de - g["dt_crit_explicit"]) < 5e-9
    assert abs(de - 2 / np.sqrt(2 + 2 * np.cos(np.pi / 9))) < 1e-14


def _spring_problem():
    M, K, f, g = spring_chain()
    pr = Problem(sp.csr_matrix(M), sp.csr_matrix(K), f, np.arange(8), np.arange(8, 10))
    w = 2 * np.pi * g["f_s"]
    A = np.linalg.solve(K - w * w * M, f)          # Helmholtz amplitude
    return pr, A, w, g, K


def _run_spring(method, N):
    pr, A, w, g, K = _spring_problem()
    T = g["T"]
    dt = T / N
    f_t = np.sin(w * dt * np.arange(N + 2))
    u0 = np.zeros(10)
    v0 = A * w
    if method == "imex":
        u = imex(pr, dt, N, f_t, u0, v0)
    elif method == "cdm":
        u = cdm(pr, dt, N, f_t, u0, v0)
    else:
        u = trapezoidal(pr, dt, N, f_t, u0, v0)
    return np.linalg.norm(u - A * np.sin(w * T))


@pytest.mark.parametrize("method", ["cdm", "trap", "imex"])
def test_spring_chain_second_order(method):
    # Fig. fig:springCoupledMassesConvergence: slope 2, final-time l2 (C21)
    e = [_run_spring(method, N) for N in (2000, 4000, 8000)]
    s1 = np.log2(e[0] / e[1])
    s2 = np.log2(e[1] / e[2])
    assert 1.85 < s1 < 2.15 and 1.85 < s2 < 2.15, (e, s1, s2)


def _energy_run(method, factor, dt_ref):
    pr, A, w, g, K = _spring_problem()
    dt = factor * dt_ref
    N = int(g["T"] / dt)
    f_t = np.sin(w * dt * np.arange(N + 2))
    E = []
    obs = (lambda k, u, *rest: E.append(0.5 * u @ K @ u))
    u0, v0 = np.zeros(10), A * w
    if method == "imex":
        imex(pr, dt, N, f_t, u0, v0, observer=obs)
    else:
        cdm(pr, dt, N, f_t, u0, v0, observer=obs)
    return np.array(E)


def test_imex_stability_bracket():
    # Fig. fig:springCoupledMassesElastic: bounded at 0.99 dt_explicit,
    # unbounded growth at 1.01 dt_explicit
    g = _golden_spring()
    Es = _energy_run("imex", 0.99, g["dt_crit_explicit"])
    Eu = _energy_run("imex", 1.01, g["dt_crit_explicit"])
    assert np.all(np.isfinite(Es)) and Es.max() < 20.0
    assert Eu.max() > 1e3 and Eu.max() > 100 * Es.max()


def test_cdm_global_bracket():
    # CDM is bound by dt_crit^global
    g = _golden_spring()
    Es = _energy_run("cdm", 0.99, g["dt_crit_global"])
    Eu = _energy_run("cdm", 1.01, g["dt_crit_global"])
    assert Es.max() < 20.0
    assert not np.all(np.isfinite(Eu)) or Eu.max() > 1e6


def _random_system(rng, n, diag_mass):
    B = rng.standard_normal((n, n))
    K = B @ B.T / n
    if diag_mass:
        M = np.diag(rng.uniform(0.5, 2.0, n))
    else:
        C = rng.standard_normal((n, n)) * 0.1
        M = np.eye(n) + C @ C.T
    return sp.csr_matrix(M), sp.csr_matrix(K)


@pytest.mark.parametrize("seed", range(20))
def test_degenerate_splits(seed):
    """I_c = {} -> IMEX == CDM bit for bit;
    I_d = {} -> IMEX == trapezoidal within 1e-12."""
    rng = np.random.default_rng(seed)
    n = int(rng.integers(3, 12))
    M, K = _random_system(rng, n, True)
    f = rng.standard_normal(n)
    f_t = rng.standard_normal(60)
    u0, v0 = rng.standard_normal(n), rng.standard_normal(n)
    dt = 0.5 * dt_crit(K.toarray(), M.toarray())
    pr = Problem(M, K, f, np.arange(n), np.array([], dtype=int))
    a = imex(pr, dt, 50, f_t, u0, v0)
    b = cdm(pr, dt, 50, f_t, u0, v0)
    assert np.array_equal(a, b)
    M2, K2 = _random_system(rng, n, False)
    pr2 = Problem(M2, K2, f, np.array([], dtype=int), np.arange(n))
    dt2 = 3.0 * dt_crit(K2.toarray(), M2.toarray())     # implicit: any dt
    a = imex(pr2, dt2, 50, f_t, u0, v0)
    b = trapezoidal(pr2, dt2, 50, f_t, u0, v0)
    assert np.max(np.abs(a - b)) <= 1e-12 * max(1.0, np.max(np.abs(b)))


def test_energy_trapezoidal_and_cdm_modified():
    """P7: unforced trapezoidal conserves 1/2 v'Mv + 1/2 u'Ku; CDM conserves
    1/2 v_{n+1/2}'M v_{n+1/2} + 1/2 u_{n+1}'K u_n."""
    rng = np.random.default_rng(7)
    n = 12
    M2, K2 = _random_system(rng, n, False)
    pr = Problem(M2, K2, np.zeros(n), np.array([], dtype=int), np.arange(n))
    u0, v0 = rng.standard_normal(n), rng.standard_normal(n)
    Md, Kd = M2.toarray(), K2.toarray()
    E = []
    trapezoidal(pr, 0.37, 20000, None, u0, v0,
                observer=lambda k, u, v: E.append(0.5 * v @ Md @ v + 0.5 * u @ Kd @ u))
    E = np.array(E)
    assert np.max(np.abs(E - E[0])) / E[0] < 1e-12
    Mdiag, Kc = _random_system(rng, n, True)
    prc = Problem(Mdiag, Kc, np.zeros(n), np.arange(n), np.array([], dtype=int))
    dt = 0.7 * dt_crit(Kc.toarray(), Mdiag.toarray())
    us = [u0.copy()]
    cdm(prc, dt, 20000, None, u0, v0, observer=lambda k, u: us.append(u.copy()))
    Md, Kd = Mdiag.toarray(), Kc.toarray()
    Em = []
    for i in range(len(us) - 1):
        vh = (us[i + 1] - us[i]) / dt
        Em.append(0.5 * vh @ Md @ vh + 0.5 * us[i + 1] @ Kd @ us[i])
    Em = np.array(Em)
    assert np.max(np.abs(Em - Em[0])) / Em[0] < 1e-12


def _dalembert_error(p, frac=0.02, T=1.0, cells=32):
    cfg = sc_inputs.small_config(1, [cells], p, voids=[], u0="gaussian_pulse")
    s = build_system(cfg, "sparse")
    dtc = dt_crit_uncut(1, p, 1.0 / cells)
    N = int(np.ceil(T / (frac * dtc)))
    dt = T / N
    X = node_coords(cfg, s.cl.lattice_index)[:, 0]
    u0 = sc_inputs.gaussian_pulse(X)
    u = imex(from_system(s), dt, N, None, u0, None)

    def ext(y):
        y = np.mod(y, 2.0)
        return sc_inputs.gaussian_pulse(np.where(y > 1.0, 2.0 - y, y))
    ue = 0.5 * (ext(X - T) + ext(X + T))
    return np.linalg.norm(u - ue) / np.linalg.norm(ue)


def test_dalembert_and_p_convergence():
    """P8/P9: uncut 1D bar with Neumann ends vs the d'Alembert solution
    (even 2-periodic extension); error falls >= 10x per +1 in p (p <= 5)."""
    errs = {p: _dalembert_error(p) for p in (2, 3, 4, 5, 6)}
    assert errs[4] < 5e-5
    for p in (2, 3, 4):
        assert errs[p + 1] < errs[p] / 10.0, errs
    # p = 6 approaches the O(dt^2) temporal floor at dt = 0.02 dt_crit
    assert errs[6] < errs[5] / 8.0, errs


def test_config_dt():
    """C12: each config's dt literal equals 0.9 x the oracle's uncut
    cell-wise critical step."""
    spec = {1: (1, 4, 32), 2: (2, 4, 64), 3: (2, 4, 256), 4: (3, 3, 64), 5: (3, 4, 160), 6: (2, 4, 128)}
    for cid, (d, p, n) in spec.items():
        dt = sc_inputs.get_config(cid)["dt"]
        ref = 0.9 * dt_crit_uncut(d, p, 1.0 / n)
        assert abs(dt - ref) <= 1e-14 * ref


def test_config1_runs_bounded_and_stable():
    """P10 on config 1: IMEX at 0.9 x the uncut cell-wise limit stays bounded
    despite the cut cell (eta = 0.984 here), and the explicit-subsystem critical
    step is >= the uncut cell-wise estimate (Irons bound)."""
    cfg = sc_inputs.get_config(1)
    E = []
    u, s = run_config(cfg, observer=lambda k, u: E.append(np.max(np.abs(u))))
    assert np.all(np.isfinite(E)) and max(E) < 1.5
    Kdd = s.K[s.I_d][:, s.I_d].toarray()
    assert dt_crit(Kdd, s.M_dd) >= dt_crit_uncut(1, 4, 1 / 32) * (1 - 1e-12)


def test_config2_crosscheck_p15():
    """SURVEY P15 (non-authoritative cross-check from an independent
    prototype under the same readings): config 2 after 5000 steps."""
    u, s = run_config(sc_inputs.get_config(2))
    src = s.cl.dof_of_lattice[64 + 257 * 64]
    assert abs(np.linalg.norm(u) - 2.973550776199) < 1e-9
    assert abs(u[src] - 5.586249111673e-2) < 1e-11


@pytest.mark.parametrize("seed", range(6))
def test_cdm_consistent_pins(seed):
    """CDM on the consistent SCM (oracle.integrators.cdm_consistent, NEXT-1(a)): with I_c empty
    it is the diagonal CDM bit for bit; with a non-diagonal M^cc the modified energy
    1/2 v_{n+1/2}'M v_{n+1/2} + 1/2 u_{n+1}'K u_n is conserved (unforced, dt below critical)."""
    from oracle.integrators import cdm_consistent
    rng = np.random.default_rng(100 + seed)
    n = int(rng.integers(4, 12))
    M, K = _random_system(rng, n, True)
    f = rng.standard_normal(n)
    f_t = rng.standard_normal(80)
    u0, v0 = rng.standard_normal(n), rng.standard_normal(n)
    dt = 0.5 * dt_crit(K.toarray(), M.toarray())
    pr = Problem(M, K, f, np.arange(n), np.array([], dtype=int))
    assert np.array_equal(cdm_consistent(pr, dt, 60, f_t, u0, v0), cdm(pr, dt, 60, f_t, u0, v0))
    # block mass: diagonal d block, SPD c block
    nd = n // 2
    Mc = rng.standard_normal((n - nd, n - nd)) * 0.2
    Mfull = np.zeros((n, n))
    Mfull[:nd, :nd] = np.diag(rng.uniform(0.5, 2.0, nd))
    Mfull[nd:, nd:] = np.eye(n - nd) + Mc @ Mc.T
    prc = Problem(sp.csr_matrix(Mfull), K, np.zeros(n), np.arange(nd), np.arange(nd, n))
    dtc = 0.6 * dt_crit(K.toarray(), Mfull)
    us = [u0.copy()]
    cdm_consistent(prc, dtc, 5000, None, u0, v0, observer=lambda k, u: us.append(u.copy()))
    Kd = K.toarray()
    Em = []
    for i in range(len(us) - 1):
        vh = (us[i + 1] - us[i]) / dtc
        Em.append(0.5 * vh @ Mfull @ vh + 0.5 * us[i + 1] @ Kd @ us[i])
    Em = np.array(Em)
    assert np.max(np.abs(Em - Em[0])) / Em[0] < 1e-11
