"""Time integrators (ORACLE - test infrastructure only).

PAPER.md §Time Integration, P:564-595:
* Newmark formulas (Eqs. eq:Newmark1, eq:Newmark2).
* CDM two-step form u_{n+1} = 2u_n - u_{n-1} + dt^2 a_n (Eq. eq:CDMstep,
  P:577) with M a_n = f_t(t_n) f_x - K u_n (Eq. eq:CDMacc).
* Trapezoidal Newmark, beta = 1/4, gamma = 1/2, predictor-corrector
  (flowchart fig:implicitNewmark is missing -> reading C2):
  predict u~ = u_n + dt v_n + dt^2/4 a_n, v~ = v_n + dt/2 a_n;
  solve S a_{n+1} = f_t(t_{n+1}) f_x - K u~, S = M + dt^2/4 K (factored once);
  correct u_{n+1} = u~ + dt^2/4 a_{n+1}, v_{n+1} = v~ + dt/2 a_{n+1}.
* Newmark IMEX (flowchart fig:TrapCDMIMEX is missing -> reading C1):
  (a1) r^d = f_t(t_n) f_x^d - K^d u_n
  (a2) u^d_{n+1} = 2u^d_n - u^d_{n-1} + dt^2 r^d / M^dd
  (a3) u~^c = u^c_n + dt v^c_n + dt^2/4 a^c_n ; v~^c = v^c_n + dt/2 a^c_n
  (a4) r^c = f_t(t_{n+1}) f_x^c - K^c w,  w = [u^d_{n+1}; u~^c]
  (a5) S a^c_{n+1} = r^c,  S = M^cc + dt^2/4 K^cc (factored once)
  (a6) u^c_{n+1} = u~^c + dt^2/4 a^c_{n+1} ; v^c_{n+1} = v~^c + dt/2 a^c_{n+1}
* Startup (reading C3): a_0 from M a_0 = f_t(0) f_x - K u_0 (blockwise);
  u^d_{-1} = u^d_0 - dt v^d_0 + dt^2/2 a^d_0.

f_t is passed as the array f_t[k] = f_t(k dt) (inputs, sc_inputs); beyond
its end f_t is taken as 0.

The integrators are generic: they take a "problem" with n, M (diagonal
vector or sparse), K (sparse, or a function u -> K u), f_x and the index sets.
"""
import numpy as np
import scipy.sparse as sp
import scipy.sparse.linalg as spla


def _ft(f_t, k):
    if f_t is None or k >= len(f_t):
        return 0.0
    return float(f_t[k])


# Fill-reducing column ordering of the sparse LU (scipy/SuperLU permc_spec).  A library
# parameter, not arithmetic of the method: the parity tests run the oracle with two orderings
# to measure its own rounding floor on ill-conditioned S (reading C24).
PERMC_SPEC = "COLAMD"


def _factor(A):
    A = sp.csc_matrix(A)
    if A.shape[0] == 0:
        return lambda b: b.copy()
    lu = spla.splu(A, permc_spec=PERMC_SPEC)
    return lu.solve


class Problem:
    """Generic second-order system M u'' + K u = f_t(t) f_x partitioned into
    I_d (diagonal mass block) and I_c."""

    def __init__(self, M, K, f_x, I_d, I_c, K_apply=None):
        self.n = len(f_x)
        self.M = M                       # sparse n x n (or None when blocks given)
        self.K = K                       # sparse n x n or None
        self._Kapply = K_apply
        self.f_x = np.asarray(f_x, dtype=np.float64)
        self.I_d = np.asarray(I_d, dtype=np.int64)
        self.I_c = np.asarray(I_c, dtype=np.int64)
        self.M_dd = None
        self.M_cc = None
        self.K_cc = None
        if M is not None:
            M = sp.csr_matrix(M)
            self.M_dd = M[self.I_d][:, self.I_d].diagonal()
            self.M_cc = M[self.I_c][:, self.I_c]
            # M^dc = 0 structurally and M^dd diagonal
            assert M[self.I_d][:, self.I_c].nnz == 0 or abs(M[self.I_d][:, self.I_c]).max() == 0
            Mdd = M[self.I_d][:, self.I_d]
            off = Mdd - sp.diags(Mdd.diagonal())
            assert off.nnz == 0 or abs(off).max() == 0
        if K is not None:
            self.K_cc = sp.csr_matrix(K)[self.I_c][:, self.I_c]

    def Ku(self, u):
        if self.K is not None:
            return self.K @ u
        return self._Kapply(u)


def from_system(sysm):
    """Wrap an assembled oracle System (assembly.build_system) as a Problem."""
    from .assembly import K_apply
    pr = Problem(None, sysm.K, sysm.f_x, sysm.I_d, sysm.I_c,
                 K_apply=lambda u: K_apply(sysm, u))
    pr.M_dd = sysm.M_dd
    pr.M_cc = sysm.M_cc
    pr.K_cc = sysm.K_cc
    pr.M = sysm.M
    return pr


def startup(pr, dt, f_t, u0, v0):
    """Consistent initial acceleration (reading C3), blockwise solve."""
    r = _ft(f_t, 0) * pr.f_x - pr.Ku(u0)
    a0 = np.zeros(pr.n)
    a0[pr.I_d] = r[pr.I_d] / pr.M_dd
    if len(pr.I_c):
        a0[pr.I_c] = _factor(pr.M_cc)(r[pr.I_c])
    return a0


def imex(pr, dt, n_steps, f_t, u0, v0=None, observer=None):
    """Newmark IMEX, steps (a1)-(a6) of the module docstring (C1)."""
    n = pr.n
    u = np.array(u0, dtype=np.float64, copy=True)
    v0 = np.zeros(n) if v0 is None else np.asarray(v0, dtype=np.float64)
    a0 = startup(pr, dt, f_t, u, v0)
    Id, Ic = pr.I_d, pr.I_c
    u_prev_d = u[Id] - dt * v0[Id] + 0.5 * dt * dt * a0[Id]
    v_c = v0[Ic].copy()
    a_c = a0[Ic].copy()
    solve_S = _factor(pr.M_cc + 0.25 * dt * dt * pr.K_cc) if len(Ic) else None
    for k in range(n_steps):
        # (a1) r^d = f_t(t_n) f_x^d - K^d u_n
        r_d = _ft(f_t, k) * pr.f_x[Id] - pr.Ku(u)[Id]
        # (a2) CDM sum step with the diagonal mass
        u_d_new = 2.0 * u[Id] - u_prev_d + dt * dt * r_d / pr.M_dd
        # (a3) predictor
        ut_c = u[Ic] + dt * v_c + 0.25 * dt * dt * a_c
        vt_c = v_c + 0.5 * dt * a_c
        # (a4) w = [u^d_{n+1}; u~^c], r^c = f_t(t_{n+1}) f_x^c - K^c w
        w = np.empty(n)
        w[Id] = u_d_new
        w[Ic] = ut_c
        if len(Ic):
            r_c = _ft(f_t, k + 1) * pr.f_x[Ic] - pr.Ku(w)[Ic]
            # (a5) implicit solve with the factor computed once
            a_c = solve_S(r_c)
            # (a6) corrector
            u_c_new = ut_c + 0.25 * dt * dt * a_c
            v_c = vt_c + 0.5 * dt * a_c
        u_prev_d = u[Id].copy()
        u[Id] = u_d_new
        if len(Ic):
            u[Ic] = u_c_new
        if observer is not None:
            observer(k + 1, u)
    return u


def cdm(pr, dt, n_steps, f_t, u0, v0=None, observer=None):
    """Explicit CDM on all DOFs with diagonal M (Eqs. eq:CDMstep, eq:CDMacc)."""
    n = pr.n
    u = np.array(u0, dtype=np.float64, copy=True)
    v0 = np.zeros(n) if v0 is None else np.asarray(v0, dtype=np.float64)
    mdiag = np.zeros(n)
    if pr.M is not None:
        M = sp.csr_matrix(pr.M)
        off = M - sp.diags(M.diagonal())
        assert off.nnz == 0 or abs(off).max() == 0, "cdm() needs a diagonal mass"
        mdiag = M.diagonal()
    else:
        mdiag[pr.I_d] = pr.M_dd
    a0 = (_ft(f_t, 0) * pr.f_x - pr.Ku(u)) / mdiag
    u_prev = u - dt * v0 + 0.5 * dt * dt * a0
    for k in range(n_steps):
        r = _ft(f_t, k) * pr.f_x - pr.Ku(u)
        u_new = 2.0 * u - u_prev + dt * dt * r / mdiag
        u_prev = u
        u = u_new
        if observer is not None:
            observer(k + 1, u)
    return u


def cdm_consistent(pr, dt, n_steps, f_t, u0, v0=None, observer=None):
    """CDM on the consistent SCM (the paper's "CDM, consistent SCM", Table
    tab:times3D): u_{n+1} = 2u_n - u_{n-1} + dt^2 a_n with M a_n = f_t(t_n) f_x - K u_n solved
    blockwise (M^dd diagonal, M^cc factored once; M^dc = 0).  Same start as imex."""
    n = pr.n
    u = np.array(u0, dtype=np.float64, copy=True)
    v0 = np.zeros(n) if v0 is None else np.asarray(v0, dtype=np.float64)
    a0 = startup(pr, dt, f_t, u, v0)
    Id, Ic = pr.I_d, pr.I_c
    u_prev = u - dt * v0 + 0.5 * dt * dt * a0
    solve_M = _factor(pr.M_cc) if len(Ic) else None
    for k in range(n_steps):
        r = _ft(f_t, k) * pr.f_x - pr.Ku(u)
        step = np.empty(n)                       # dt^2 a_n, a_n = M^{-1} r blockwise
        step[Id] = dt * dt * r[Id] / pr.M_dd
        if len(Ic):
            step[Ic] = dt * dt * solve_M(r[Ic])
        u_new = 2.0 * u - u_prev + step
        u_prev = u
        u = u_new
        if observer is not None:
            observer(k + 1, u)
    return u


def _ft_frac(f_t, k, theta):
    """f_t at t_k + theta dt from the supplied samples f_t(k dt): linear interpolation
    (reading LF4; theta = 0 is the sample itself)."""
    if theta == 0.0:
        return _ft(f_t, k)
    return (1.0 - theta) * _ft(f_t, k) + theta * _ft(f_t, k + 1)


def leapfrog(pr, dt, n_steps, f_t, u0, m, coupling="interpolated", v0=None, observer=None):
    """Leap-frog substepping of the cut DOFs ("the cut cells are integrated
    in time with a finer time step size dt_fine = dt_coarse / m"; the details are deferred to
    [NAC22, meineMA], not available - DESIGN.md readings LF1-LF4):
    * LF1: the d DOFs take the CDM step of the IMEX method with dt (diagonal M^dd),
      reading u_n (including u^c_n);
    * LF2: the c DOFs take m CDM steps with dt_f = dt/m on the consistent M^cc (factored once,
      P:583): u^c_{k+1} = 2u^c_k - u^c_{k-1} + dt_f^2 (M^cc)^-1 (f_t(t_k) f^c - (K w_k)_c),
      w_k = [u^d(t_k); u^c_k];
    * LF3 (the coupling rule, unstated): u^d(t_k) = u^d_n ("frozen") or the linear
      interpolation u^d_n + (k/m)(u^d_{n+1} - u^d_n) ("interpolated");
    * LF4: f_t at the fine times by linear interpolation of the supplied samples f_t(k dt).
    Start: a_0 blockwise as imex (reading C3); u^d_{-1} with dt, u^c_{-1} with dt_f."""
    n = pr.n
    u = np.array(u0, dtype=np.float64, copy=True)
    v0 = np.zeros(n) if v0 is None else np.asarray(v0, dtype=np.float64)
    a0 = startup(pr, dt, f_t, u, v0)
    Id, Ic = pr.I_d, pr.I_c
    dtf = dt / m
    u_prev_d = u[Id] - dt * v0[Id] + 0.5 * dt * dt * a0[Id]
    uc = u[Ic].copy()
    uc_prev = u[Ic] - dtf * v0[Ic] + 0.5 * dtf * dtf * a0[Ic]
    solve_M = _factor(pr.M_cc) if len(Ic) else None
    interp = coupling == "interpolated"
    if coupling not in ("interpolated", "frozen"):
        raise ValueError(coupling)
    for k in range(n_steps):
        # LF1: the d CDM step
        r_d = _ft(f_t, k) * pr.f_x[Id] - pr.Ku(u)[Id]
        u_d_new = 2.0 * u[Id] - u_prev_d + dt * dt * r_d / pr.M_dd
        # LF2/LF3: m fine CDM steps of the c DOFs
        if len(Ic):
            w = np.empty(n)
            for j in range(m):
                th = j / m
                w[Id] = u[Id] + th * (u_d_new - u[Id]) if interp else u[Id]
                w[Ic] = uc
                r_c = _ft_frac(f_t, k, th) * pr.f_x[Ic] - pr.Ku(w)[Ic]
                uc_new = 2.0 * uc - uc_prev + dtf * dtf * solve_M(r_c)
                uc_prev = uc
                uc = uc_new
        u_prev_d = u[Id].copy()
        u[Id] = u_d_new
        if len(Ic):
            u[Ic] = uc
        if observer is not None:
            observer(k + 1, u)
    return u


def trapezoidal(pr, dt, n_steps, f_t, u0, v0=None, observer=None, return_v=False):
    """Implicit trapezoidal Newmark on all DOFs (reading C2)."""
    n = pr.n
    u = np.array(u0, dtype=np.float64, copy=True)
    v = np.zeros(n) if v0 is None else np.array(v0, dtype=np.float64, copy=True)
    M = sp.csc_matrix(pr.M)
    a = _factor(M)(_ft(f_t, 0) * pr.f_x - pr.Ku(u))
    solve_S = _factor(M + 0.25 * dt * dt * sp.csc_matrix(pr.K))
    for k in range(n_steps):
        ut = u + dt * v + 0.25 * dt * dt * a
        vt = v + 0.5 * dt * a
        a = solve_S(_ft(f_t, k + 1) * pr.f_x - pr.Ku(ut))
        u = ut + 0.25 * dt * dt * a
        v = vt + 0.5 * dt * a
        if observer is not None:
            observer(k + 1, u, v)
    return (u, v) if return_v else u
