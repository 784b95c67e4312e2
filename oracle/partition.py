"""Partitioned Newmark IMEX (ORACLE - test infrastructure only, pin P13).

The IMEX step of integrators.imex (reading C1) run by `world` ranks that each own a
part of the DOFs and exchange values after every step (torch.distributed, any backend):

* d DOFs are owned by the rank whose slab holds their lattice plane along the last axis
  (slabs = equal ranges of element layers);
* c DOFs are owned per connected component of the c-graph (the blocks of S): the
  component goes to the rank whose slab holds its mean lattice plane, so (a3)-(a6) of a
  component run on one rank and the implicit solve needs no communication;
* each rank applies (a1)-(a2) to its d rows and (a3)-(a6) to its components using its copy
  of u_n, then all ranks exchange their owned entries of u_{n+1} (all_gather).

Independent of the CUDA path's decomposition (which exchanges only region boundaries); the
pin is that any ownership split reproduces the single-process oracle: the d rows by the same arithmetic (to the last bit), the c rows
up to the factorisation of S per rank instead of over all components (rounding only).
"""
import numpy as np
import scipy.sparse as sp
import scipy.sparse.csgraph as csg

from .integrators import _factor, _ft, startup


def owners(pr, lattice_index, nl, p, n_layers, world):
    """Owner rank of every DOF (see module docstring)."""
    plane = lattice_index // int(np.prod(nl[:-1]))
    layer = np.minimum(plane // p, n_layers - 1)
    bounds = [(n_layers * r) // world for r in range(world + 1)]
    own = np.searchsorted(bounds, layer, side="right") - 1
    Ic = pr.I_c
    if len(Ic):
        Kcc = sp.csr_matrix(pr.K_cc) if pr.K_cc is not None else None
        G = (abs(Kcc) + abs(sp.csr_matrix(pr.M_cc))) if Kcc is not None else sp.csr_matrix(pr.M_cc)
        ncomp, lab = csg.connected_components(G, directed=False)
        for k in range(ncomp):
            members = Ic[lab == k]
            zc = plane[members].mean() / p
            own[members] = np.searchsorted(bounds, min(int(zc), n_layers - 1), side="right") - 1
    return own


def imex_partitioned(pr, dt, n_steps, f_t, u0, own, rank, world, allgather):
    """integrators.imex with rank `rank` updating only the DOFs it owns; `allgather(vec)`
    returns the list of every rank's vector (the exchange)."""
    n = pr.n
    u = np.array(u0, dtype=np.float64, copy=True)
    v0 = np.zeros(n)
    a0 = startup(pr, dt, f_t, u, v0)
    Id, Ic = pr.I_d, pr.I_c
    md = own[Id] == rank            # owned d rows
    mc = own[Ic] == rank            # owned c rows (whole components)
    Id_o, Ic_o = Id[md], Ic[mc]
    Mdd_o = pr.M_dd[md]
    u_prev = u[Id_o] - dt * v0[Id_o] + 0.5 * dt * dt * a0[Id_o]
    v_c = np.zeros(len(Ic_o))
    a_c = a0[Ic_o].copy()
    solve = None
    if len(Ic_o):
        sub = np.nonzero(mc)[0]
        S = sp.csr_matrix(pr.M_cc + 0.25 * dt * dt * pr.K_cc)[sub][:, sub]
        solve = _factor(S)
    for k in range(n_steps):
        Ku = pr.Ku(u)
        r_d = _ft(f_t, k) * pr.f_x[Id_o] - Ku[Id_o]
        u_d_new = 2.0 * u[Id_o] - u_prev + dt * dt * r_d / Mdd_o
        new = np.zeros(n)
        new[Id_o] = u_d_new
        if len(Ic_o):
            ut_c = u[Ic_o] + dt * v_c + 0.25 * dt * dt * a_c
            vt_c = v_c + 0.5 * dt * a_c
        # w needs u^d_{n+1} on the rows of the own components: exchange the d part first
        d_parts = allgather(new)
        w = np.sum(d_parts, axis=0)
        if len(Ic_o):
            w[Ic_o] = ut_c
            r_c = _ft(f_t, k + 1) * pr.f_x[Ic_o] - pr.Ku(w)[Ic_o]
            a_c = solve(r_c)
            u_c_new = ut_c + 0.25 * dt * dt * a_c
            v_c = vt_c + 0.5 * dt * a_c
            cvec = np.zeros(n)
            cvec[Ic_o] = u_c_new
        else:
            cvec = np.zeros(n)
        c_parts = allgather(cvec)
        u_prev = u[Id_o].copy()
        u = w
        u[Ic] = np.sum(c_parts, axis=0)[Ic]
    return u
