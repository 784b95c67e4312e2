/*
 * sc.h - C ABI of the B200-native immersed Newmark IMEX spectral cell solver.
 *
 * The problem statement these calls take follows PAPER.md (arXiv 2310.14712):
 *   rho u'' - div(rho c^2 grad u) = f on the extended box Omega = Omega_p U Omega_f
 *   (Eq. eq:scalarWaveEq), homogeneous Neumann on the box,
 *   FCM indicator alpha = 1 in Omega_p, alpha_f in Omega_f,
 *   order-p GLL spectral cells on a Cartesian grid,
 *   separable load f = f_t(t) f_x,
 *   Newmark IMEX time stepping: explicit CDM on the 'd' DOFs
 *   (supported only by uncut cells), implicit trapezoidal Newmark on the
 *   'c' DOFs (supported by >= 1 cut cell).
 *
 * Conventions (all functions):
 *  - Every pointer argument is a HOST pointer unless stated otherwise; the
 *    caller owns it; inputs are copied during the call and may be freed after.
 *  - The context owns all device memory, the factors, the CUDA graphs and (for
 *    world > 1) the NCCL communicator.  sc_destroy releases everything.
 *  - Errors are returned as sc_status; a human-readable message is available
 *    from sc_last_error(ctx).  No function aborts the process.
 *  - Canonical DOF order: retained lattice nodes (nodes of non-empty cells,
 *    P:866) in lexicographic order, x fastest; lattice index
 *    = i + n0*(j + n1*k) with n_k = cells[k]*p + 1.
 *  - All floating point is IEEE fp64.
 */
#ifndef SC_H
#define SC_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct sc_ctx sc_ctx; /* opaque */

typedef enum {
  SC_OK = 0,
  SC_ERR_CONFIG = 2,  /* invalid argument / unsupported configuration (SPEC exit code 2) */
  SC_ERR_NUMERIC = 3, /* non-finite state or non-positive pivot (SPEC exit code 3) */
  SC_ERR_CUDA = 4,    /* CUDA runtime error */
  SC_ERR_NCCL = 5,    /* NCCL error (world > 1) */
  SC_ERR_OOM = 6,     /* device or host allocation failed */
  SC_ERR_STATE = 7    /* call not valid in the current state (e.g. NULL ctx) */
} sc_status;

/* Uniform Cartesian grid of the extended domain Omega (Fig. fig:FCM).
 * dim in {1,2,3}; cells[k] >= 1 and lo[k] < hi[k] for k < dim (entries k >= dim ignored). */
typedef struct {
  int32_t dim;
  int32_t cells[3];
  double lo[3];
  double hi[3];
} sc_grid;

/* One void (part of the fictitious domain Omega_f).
 *  kind SC_VOID_ELLIPSOID: void = {x : (x-c)^T A (x-c) < 1} (strict: Omega_p is closed),
 *       A symmetric positive definite, packed A00,A11,A22,A01,A02,A12 (unused dims 0);
 *  kind SC_VOID_HALFSPACE: void = {x : n.x > b}.
 * Membership is evaluated exactly as DESIGN.md reading C17 (no FMA). */
enum { SC_VOID_ELLIPSOID = 1, SC_VOID_HALFSPACE = 2 };
typedef struct {
  int32_t kind;
  double c[3];
  double A[6];
  double n[3];
  double b;
} sc_void;

/* Geometry and material.  tree_depth = spacetree depth D; lattice_s = s of the
 * cut-test lattice (reading C6, default 4); fill_eps = empty-cell threshold (P:866-868,
 * default 1e-10; reading C7: a cell is empty iff none of its Gauss points is physical, which
 * equals eta < fill_eps because sc_setup rejects (SC_ERR_CONFIG) any dim/p/tree_depth whose
 * smallest nonzero fill ratio (2^-D w_min/2)^dim is below fill_eps); rho, c constant (P:846,
 * reading C10); integrator below. */
typedef struct {
  int32_t n_voids;
  const sc_void* voids;
  int32_t tree_depth;
  int32_t lattice_s;
  double fill_eps;
  double rho;
  double c;
  int32_t integrator; /* the paper's schemes on the same kernels (Table tab:times3D):
                         0 Newmark IMEX (the method);
                         1 CDM on the HRZ-lumped SCM (every DOF explicit, cut cells
                           HRZ-lumped; dt below its much smaller critical step);
                         2 trapezoidal Newmark on all DOFs (every DOF implicit, S
                           factored over the whole mesh: small problems);
                         3 CDM on the consistent SCM (M^cc solved each step
                           with its factor; dt below the consistent critical step);
                         4 leap-frog substepping: the d DOFs as in 0 (CDM, dt), the c
                           DOFs lf_m CDM steps of dt/lf_m on the consistent M^cc per step
                           (readings LF1-LF4) */
  int32_t lf_m;        /* integrator 4: substeps m >= 1 (ignored otherwise) */
  int32_t lf_coupling; /* integrator 4: d values during the substeps, 0 = linear interpolation
                          between u^d_n and u^d_{n+1}, 1 = frozen at u^d_n (reading LF3) */
} sc_geometry;

/* Separable source f(x,t) = f_t(t) f_x(x), f_t[k] = f_t(k*dt) for k < n_t (host
 * array, copied), f_t = 0 beyond n_t.  kind 0 = no source (f_t ignored);
 * kind 1 = point source at x (reading C11): f_x,i = alpha(x_s) N_i(x_s) in the lowest-index
 *   non-empty cell containing x_s;
 * kind 2 = the paper's Gaussian bell (Eq. eq:fx): f_x(x) = amp exp(-|x - x|^2 /
 *   (2 sigma^2)), f_x,i = int alpha f_x N_i with (p+1)^d Gauss points per cell / spacetree leaf
 *   (P:461-463), assembled in ascending cell order (deterministic); sigma > 0. */
typedef struct {
  int32_t kind;
  double x[3];
  int64_t n_t;
  const double* f_t;
  double sigma; /* kind 2 */
  double amp;   /* kind 2 */
} sc_source;

/* Distribution: NULL => one GPU (current device, current stream semantics below).
 * rank/world: slab decomposition over world ranks (z-slabs of whole element
 * layers, cost-weighted; each c component owned by one rank; one point-to-point exchange per
 * step); device: CUDA device ordinal; nccl_unique_id: 128-byte ncclUniqueId shared by all
 * ranks (sc_nccl_unique_id on one rank, broadcast by the caller) -> one process per GPU, the
 * exchange runs inside sc_step over NCCL (NVLink/NVSwitch); NULL with world > 1 => ranks
 * living in ONE process (validation on one GPU): the caller alternates sc_step(ctx_r, 1) on
 * every rank with sc_exchange_local; cuda_stream: cudaStream_t to enqueue on (NULL => the
 * context creates its own). */
typedef struct {
  int32_t rank;
  int32_t world;
  int32_t device;
  const void* nccl_unique_id;
  void* cuda_stream;
} sc_dist;

typedef struct {
  int64_t n_dof, n_d, n_c;          /* retained DOFs; |I_d|; |I_c| */
  int64_t n_irregular;              /* d DOFs updated off the tensor kernel (touching an
                                       empty cell, or carrying the point load) */
  int64_t cells_uncut, cells_cut, cells_empty;
  int64_t n_components;             /* connected components of the c-graph (blocks of S) */
  int64_t n_supernodes;
  int64_t nnz_factor;               /* stored entries of the S factor (Linv + L panels) */
  int32_t factor_height;            /* supernodal elimination-tree height */
  double dt;
  double dt_crit_uncut;             /* 2/sqrt(lambda_max(K_e, M_e)) of an uncut cell */
  int64_t step;                     /* steps taken since the last (re)start */
  double bytes_per_step;            /* algorithmic HBM bytes per step */
  double bytes_explicit_per_step;   /* ... of the fused explicit (a1)+(a2) kernel on the
                                       tensor-d DOFs (sc_profile which = 0) */
  int32_t kernels_per_step;         /* kernel launches per step */
  int64_t lattice_nodes;            /* prod(cells*p+1) */
  double setup_seconds;
  int64_t n_near;                   /* tensor-d DOFs sharing an element with a c DOF (updated
                                       after the c part of the step; the rest of the tensor-d
                                       DOFs overlap it) */
  double bytes_solve_per_step;      /* algorithmic HBM bytes of the implicit solve (a5) */
  double bytes_celem_per_step;      /* ... of the c-element products (a3)+(a4) */
  int32_t rank, world;              /* this context's rank in the slab decomposition */
  int64_t n_c_local;                /* c DOFs of this rank's components (its implicit solve) */
  int64_t halo_send, halo_recv;     /* values sent / received per step by the exchange */
  int64_t n_owned;                  /* DOFs owned by this rank (sc_read_owned writes these) */
} sc_info;

/* Build the discretisation, classify cells and DOFs, integrate the cut cells, factor
 * S = M^cc + dt^2/4 K^cc once and compute the consistent start
 * (reading C3).  u0, v0: nullable host arrays of length n_dof in canonical order (NULL =>
 * zero); since n_dof is only known after classification, callers with a nonzero initial
 * field pass NULL here and then call sc_set_state.  dt is fixed for the context (S depends
 * on dt).  On success *out receives the new context; on failure *out is NULL and the
 * message is available from sc_last_error(NULL) (thread-local). */
sc_status sc_setup(const sc_grid* grid, int32_t p, double alpha, const sc_geometry* geom,
                   double dt, const sc_source* src, const double* u0, const double* v0,
                   const sc_dist* dist, sc_ctx** out);

/* Reset the state to (u0, v0) at t = 0 (host arrays of len entries in canonical order; NULL
 * => zero) and recompute the start a_0 = M^-1 (f_t(0) f_x - K u0), u^d_-1 (reading C3;
 * P:752 gives the initial displacement and velocity).  len must equal n_dof whenever u0 or v0
 * is non-NULL (SC_ERR_CONFIG otherwise, nothing read).  The arrays are staged through
 * context-owned device buffers (no allocation per call after the first v0); pinned host
 * memory makes the copies asynchronous.  Synchronises the context stream. */
sc_status sc_set_state(sc_ctx* ctx, const double* u0, const double* v0, int64_t len);

/* Enqueue n >= 0 Newmark IMEX steps (steps (a1)-(a6) of DESIGN.md §2) on the
 * context stream.  Asynchronous: returns after enqueueing.  Blow-up (non-finite u) sets a
 * device flag that sc_sync / sc_read report as SC_ERR_NUMERIC. */
sc_status sc_step(sc_ctx* ctx, int64_t n);

/* Wait for all enqueued work; SC_ERR_NUMERIC if a non-finite value was produced. */
sc_status sc_sync(sc_ctx* ctx);

/* Copy u_n (canonical order) to the host array u of length len >= n_dof.  Synchronises.
 * world > 1 over NCCL: collective, every rank receives the whole field. */
sc_status sc_read(sc_ctx* ctx, double* u, int64_t len);

/* Write the DOFs THIS rank owns (canonical order positions) into the host array u (len >=
 * n_dof); other entries are left untouched.  With world == 1 this is sc_read.  The owned sets
 * of all ranks partition the DOFs, so the ranks' outputs combined give u_n. */
sc_status sc_read_owned(sc_ctx* ctx, double* u, int64_t len);

/* In-process ranks (world > 1, no NCCL id): after every rank's sc_step(ctx_r, 1), copy each
 * rank's packed values to its peers and unpack them (device copies; synchronises all ranks'
 * streams).  ctxs[r] must be rank r. */
sc_status sc_exchange_local(sc_ctx* const* ctxs, int32_t world);

/* Critical time step of the explicit subsystem:
 * lambda_max of M_dd^{-1} K_dd on the device (c DOFs held at zero; integrators 1 and 3: of
 * M^{-1} K over all DOFs with their mass), dt_crit = 2 / sqrt(lambda_max); not for integrator 2
 * (unconditionally stable).  Integrators 0 and 1 (diagonal mass): Lanczos in the M inner
 * product, at most `iters` steps, stopped once the largest Ritz value changes by less than
 * 1e-14 relative over 10 steps; integrator 3 (consistent M^cc): `iters` power-iteration steps
 * (Rayleigh quotient).  Both approach lambda_max from below.
 * Clobbers the state: call sc_set_state before stepping again.  One rank only. */
sc_status sc_estimate_dt(sc_ctx* ctx, int32_t iters, double* lambda_max, double* dt_crit);

/* Cell-wise critical time steps (Fig. fig:tCritsCircles,
 * Table tab:criticaltimestepsizes): dt_cell[i] = 2 / sqrt(lambda_max(K_e, M_e)) of cell i (cells x
 * fastest, len >= prod(cells)); uncut cells: the uncut cell-wise value (GLL-lumped mass,
 * = sc_info.dt_crit_uncut); cut cells: which = 0 with the consistent cut-cell mass (the
 * "consistent SCM"), which = 1 with the HRZ-lumped mass; empty cells: 0.  Computed
 * on the device at setup (per cut cell: Cholesky of M_e and power iteration on
 * L^-1 K_e L^-T to a 1e-15 relative Rayleigh-quotient change).  Host output; synchronises. */
sc_status sc_cell_dt(sc_ctx* ctx, int32_t which, double* dt_cell, int64_t len);

/* Elastic energy E = 1/2 u_n^T K u_n of the current state (PAPER.md P:758,
 * the quantity of fig:springCoupledMassesElastic) into *energy (host).  Computed by the step
 * kernels with zero CDM coefficients (M^{-1} K u on the d rows, K u on the c rows through the
 * c-element products) and a fixed-order reduction: bit-reproducible.  Does not change the
 * state; synchronises.  One rank only (SC_ERR_CONFIG otherwise). */
sc_status sc_elastic_energy(sc_ctx* ctx, double* energy);

/* Receivers (the paper's receiver traces, fig:solutions3D):
 * record u(x_r, t_{n+1}) = sum_i N_i(x_r) u_i (basis of the lowest-index non-empty cell
 * containing x_r) after every step; xyz: n points (x, y, z) each (unused dims ignored);
 * capacity: rows kept (steps after the last sc_set_state / setup; later rows dropped).
 * Replaces any previous set; n = 0 removes the receivers.  One rank only. */
sc_status sc_set_receivers(sc_ctx* ctx, const double* xyz, int32_t n, int64_t capacity);

/* Copy the recorded rows (row k = after step k+1, n_rec values each) to out (host,
 * max_rows x n_rec); *rows receives the number of rows copied.  Synchronises. */
sc_status sc_read_traces(sc_ctx* ctx, double* out, int64_t max_rows, int64_t* rows);

/* A new 128-byte ncclUniqueId (world > 1 over NCCL; call on one rank and broadcast). */
sc_status sc_nccl_unique_id(void* out128);

/* Copy v^c_n and a^c_n of the c DOFs (canonical order of I_c) to host arrays (nullable). */
sc_status sc_read_c_state(sc_ctx* ctx, double* v_c, double* a_c, int64_t len);

/* Counters and sizes; see sc_info. */
sc_status sc_query(sc_ctx* ctx, sc_info* out);

/* Classification readback: cell_class[prod(cells)] (0 uncut, 1 cut, 2 empty; cells x
 * fastest), dof_is_c[n_dof] (1 = c DOF), dof_lattice_index[n_dof].  Each nullable. */
sc_status sc_read_classification(sc_ctx* ctx, int8_t* cell_class, uint8_t* dof_is_c,
                                 int64_t* dof_lattice_index);

/* Physical coordinates of the DOFs (GLL node positions): xyz[3*i + k], len >= 3*n_dof. */
sc_status sc_dof_coords(sc_ctx* ctx, double* xyz, int64_t len);

/* Instrumentation: enqueue n launches of ONE sub-kernel of the step on the context stream
 * so that a caller can time it with events: which = 0 fused explicit (a1)+(a2) tensor
 * kernel on all tensor-d DOFs, 1 c-element products (a4), 2 supernodal solve of S (a5),
 * 3 the explicit kernel on the near tensor-d DOFs alone (the pipelined mode's second launch).  Clobbers the state: call sc_set_state
 * before stepping again. */
sc_status sc_profile(sc_ctx* ctx, int32_t which, int64_t n);

/* Last error message of ctx (or of the calling thread's last failed sc_setup if NULL). */
const char* sc_last_error(const sc_ctx* ctx);

/* Release the context and everything it owns.  NULL is a no-op. */
void sc_destroy(sc_ctx* ctx);

#ifdef __cplusplus
}
#endif

#endif /* SC_H */
