"""B200-native immersed Newmark IMEX spectral cell solver (arXiv 2310.14712).

Thin Python binding over the C ABI of ``libsc.so`` (``include/sc.h``): argument
marshalling only - every step of the method runs in the library's CUDA kernels.
There is no CPU fallback: if the library is missing or cannot be loaded every
call raises ``RuntimeError``.
"""
import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("SC_LIB", os.path.join(_HERE, "libsc.so"))   # SC_LIB: variant builds (experiments)

SC_OK, SC_ERR_CONFIG, SC_ERR_NUMERIC = 0, 2, 3
SC_VOID_ELLIPSOID, SC_VOID_HALFSPACE = 1, 2


class sc_grid(ctypes.Structure):
    _fields_ = [("dim", ctypes.c_int32), ("cells", ctypes.c_int32 * 3),
                ("lo", ctypes.c_double * 3), ("hi", ctypes.c_double * 3)]


class sc_void(ctypes.Structure):
    _fields_ = [("kind", ctypes.c_int32), ("c", ctypes.c_double * 3), ("A", ctypes.c_double * 6),
                ("n", ctypes.c_double * 3), ("b", ctypes.c_double)]


class sc_geometry(ctypes.Structure):
    _fields_ = [("n_voids", ctypes.c_int32), ("voids", ctypes.POINTER(sc_void)),
                ("tree_depth", ctypes.c_int32), ("lattice_s", ctypes.c_int32),
                ("fill_eps", ctypes.c_double), ("rho", ctypes.c_double), ("c", ctypes.c_double),
                ("integrator", ctypes.c_int32), ("lf_m", ctypes.c_int32), ("lf_coupling", ctypes.c_int32)]


class sc_source(ctypes.Structure):
    _fields_ = [("kind", ctypes.c_int32), ("x", ctypes.c_double * 3), ("n_t", ctypes.c_int64),
                ("f_t", ctypes.POINTER(ctypes.c_double)), ("sigma", ctypes.c_double), ("amp", ctypes.c_double)]


class sc_dist(ctypes.Structure):
    _fields_ = [("rank", ctypes.c_int32), ("world", ctypes.c_int32), ("device", ctypes.c_int32),
                ("nccl_unique_id", ctypes.c_void_p), ("cuda_stream", ctypes.c_void_p)]


class sc_info(ctypes.Structure):
    _fields_ = [("n_dof", ctypes.c_int64), ("n_d", ctypes.c_int64), ("n_c", ctypes.c_int64),
                ("n_irregular", ctypes.c_int64), ("cells_uncut", ctypes.c_int64),
                ("cells_cut", ctypes.c_int64), ("cells_empty", ctypes.c_int64),
                ("n_components", ctypes.c_int64), ("n_supernodes", ctypes.c_int64),
                ("nnz_factor", ctypes.c_int64), ("factor_height", ctypes.c_int32),
                ("dt", ctypes.c_double), ("dt_crit_uncut", ctypes.c_double), ("step", ctypes.c_int64),
                ("bytes_per_step", ctypes.c_double), ("bytes_explicit_per_step", ctypes.c_double),
                ("kernels_per_step", ctypes.c_int32), ("lattice_nodes", ctypes.c_int64),
                ("setup_seconds", ctypes.c_double), ("n_near", ctypes.c_int64),
                ("bytes_solve_per_step", ctypes.c_double), ("bytes_celem_per_step", ctypes.c_double),
                ("rank", ctypes.c_int32), ("world", ctypes.c_int32), ("n_c_local", ctypes.c_int64),
                ("halo_send", ctypes.c_int64), ("halo_recv", ctypes.c_int64), ("n_owned", ctypes.c_int64)]


EXPORTS = ("sc_setup", "sc_set_state", "sc_step", "sc_sync", "sc_read", "sc_read_owned", "sc_read_c_state",
           "sc_query", "sc_read_classification", "sc_dof_coords", "sc_profile", "sc_exchange_local",
           "sc_nccl_unique_id", "sc_estimate_dt", "sc_cell_dt", "sc_elastic_energy", "sc_set_receivers", "sc_read_traces", "sc_last_error",
           "sc_destroy")

_lib = None


def load_library(path=LIB_PATH):
    """Load libsc.so (raises RuntimeError if it is missing: no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise RuntimeError(f"libsc.so not built at {path}; run __graft_entry__.build()")
    lib = ctypes.CDLL(path)
    P = ctypes.POINTER
    lib.sc_setup.argtypes = [P(sc_grid), ctypes.c_int32, ctypes.c_double, P(sc_geometry), ctypes.c_double,
                             P(sc_source), P(ctypes.c_double), P(ctypes.c_double), P(sc_dist),
                             P(ctypes.c_void_p)]
    lib.sc_set_state.argtypes = [ctypes.c_void_p, P(ctypes.c_double), P(ctypes.c_double), ctypes.c_int64]
    lib.sc_step.argtypes = [ctypes.c_void_p, ctypes.c_int64]
    lib.sc_sync.argtypes = [ctypes.c_void_p]
    lib.sc_read.argtypes = [ctypes.c_void_p, P(ctypes.c_double), ctypes.c_int64]
    lib.sc_read_owned.argtypes = [ctypes.c_void_p, P(ctypes.c_double), ctypes.c_int64]
    lib.sc_exchange_local.argtypes = [P(ctypes.c_void_p), ctypes.c_int32]
    lib.sc_nccl_unique_id.argtypes = [ctypes.c_void_p]
    lib.sc_estimate_dt.argtypes = [ctypes.c_void_p, ctypes.c_int32, P(ctypes.c_double), P(ctypes.c_double)]
    lib.sc_elastic_energy.argtypes = [ctypes.c_void_p, P(ctypes.c_double)]
    lib.sc_cell_dt.argtypes = [ctypes.c_void_p, ctypes.c_int32, P(ctypes.c_double), ctypes.c_int64]
    lib.sc_set_receivers.argtypes = [ctypes.c_void_p, P(ctypes.c_double), ctypes.c_int32, ctypes.c_int64]
    lib.sc_read_traces.argtypes = [ctypes.c_void_p, P(ctypes.c_double), ctypes.c_int64, P(ctypes.c_int64)]
    lib.sc_read_c_state.argtypes = [ctypes.c_void_p, P(ctypes.c_double), P(ctypes.c_double), ctypes.c_int64]
    lib.sc_query.argtypes = [ctypes.c_void_p, P(sc_info)]
    lib.sc_read_classification.argtypes = [ctypes.c_void_p, P(ctypes.c_int8), P(ctypes.c_uint8),
                                           P(ctypes.c_int64)]
    lib.sc_dof_coords.argtypes = [ctypes.c_void_p, P(ctypes.c_double), ctypes.c_int64]
    lib.sc_profile.argtypes = [ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64]
    lib.sc_last_error.argtypes = [ctypes.c_void_p]
    lib.sc_last_error.restype = ctypes.c_char_p
    lib.sc_destroy.argtypes = [ctypes.c_void_p]
    lib.sc_destroy.restype = None
    for name in EXPORTS:
        if name not in ("sc_last_error", "sc_destroy"):
            getattr(lib, name).restype = ctypes.c_int
    _lib = lib
    return lib


class ScError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"sc status {status}: {msg}")
        self.status = status


def _dptr(a):
    return None if a is None else a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


class Solver:
    """One context of the library (sc_setup ... sc_destroy)."""

    def __init__(self, grid, p, alpha, geometry, dt, source=None, u0=None, v0=None, stream=None, device=None,
                 rank=0, world=1, nccl_id=None):
        lib = load_library()
        self._lib = lib
        dim = grid["dim"]
        g = sc_grid()
        g.dim = dim
        for k in range(3):
            g.cells[k] = grid["cells"][k] if k < dim else 1
            g.lo[k] = grid["lo"][k] if k < dim else 0.0
            g.hi[k] = grid["hi"][k] if k < dim else 0.0
        vs = geometry.get("voids", [])
        arr = (sc_void * max(1, len(vs)))()
        for i, v in enumerate(vs):
            if v["kind"] == "ellipsoid":
                arr[i].kind = SC_VOID_ELLIPSOID
                for k in range(3):
                    arr[i].c[k] = v["c"][k]
                for k in range(6):
                    arr[i].A[k] = v["A"][k]
            else:
                arr[i].kind = SC_VOID_HALFSPACE
                for k in range(3):
                    arr[i].n[k] = v["n"][k]
                arr[i].b = v["b"]
        geo = sc_geometry(len(vs), arr, geometry.get("tree_depth", 2), geometry.get("lattice_s", 4),
                          geometry.get("fill_eps", 1e-10), geometry.get("rho", 1.0), geometry.get("c", 1.0),
                          {"imex": 0, "cdm_hrz": 1, "trapezoidal": 2, "cdm_consistent": 3, "leapfrog": 4}[
                              geometry.get("integrator", "imex")], int(geometry.get("lf_m", 1)),
                          {"interpolated": 0, "frozen": 1}[geometry.get("lf_coupling", "interpolated")])
        src = None
        self._ft = None
        if source is not None:
            ft = np.ascontiguousarray(source["f_t"], dtype=np.float64)
            self._ft = ft
            src = sc_source()
            src.kind = 2 if source.get("kind", "point") == "bell" else 1
            src.sigma = float(source.get("sigma", 0.0))
            src.amp = float(source.get("amp", 0.0))
            for k in range(3):
                src.x[k] = source["x"][k] if k < len(source["x"]) else 0.0
            src.n_t = len(ft)
            src.f_t = _dptr(ft)
        dist = None
        self._nccl_id = None
        if stream is not None or device is not None or world > 1:
            if nccl_id is not None:
                self._nccl_id = ctypes.create_string_buffer(bytes(nccl_id), 128)
            dist = sc_dist(int(rank), int(world), -1 if device is None else int(device),
                           ctypes.cast(self._nccl_id, ctypes.c_void_p) if self._nccl_id is not None else None,
                           ctypes.c_void_p(stream) if stream is not None else None)
        ctx = ctypes.c_void_p()
        u0a = None if u0 is None else np.ascontiguousarray(u0, dtype=np.float64)
        v0a = None if v0 is None else np.ascontiguousarray(v0, dtype=np.float64)
        st = lib.sc_setup(ctypes.byref(g), int(p), float(alpha), ctypes.byref(geo), float(dt),
                          ctypes.byref(src) if src is not None else None, _dptr(u0a), _dptr(v0a),
                          ctypes.byref(dist) if dist is not None else None, ctypes.byref(ctx))
        if st != SC_OK:
            raise ScError(st, lib.sc_last_error(None).decode())
        self.ctx = ctx
        self.info = self.query()

    # -- ABI mirrors -------------------------------------------------------------
    def _check(self, st):
        if st != SC_OK:
            raise ScError(st, self._lib.sc_last_error(self.ctx).decode())

    def query(self):
        inf = sc_info()
        self._check(self._lib.sc_query(self.ctx, ctypes.byref(inf)))
        return {k: getattr(inf, k) for k, _ in sc_info._fields_}

    def set_state(self, u0=None, v0=None):
        n = self.info["n_dof"]
        u0a = None if u0 is None else np.ascontiguousarray(u0, dtype=np.float64)
        v0a = None if v0 is None else np.ascontiguousarray(v0, dtype=np.float64)
        for name, a in (("u0", u0a), ("v0", v0a)):
            if a is not None and a.shape != (n,):
                raise ValueError(f"set_state: {name} must have shape ({n},), got {a.shape}")
        self._check(self._lib.sc_set_state(self.ctx, _dptr(u0a), _dptr(v0a), n))

    def step(self, n):
        self._check(self._lib.sc_step(self.ctx, int(n)))

    def sync(self):
        self._check(self._lib.sc_sync(self.ctx))

    def read(self, out=None):
        n = self.info["n_dof"]
        if out is None:
            out = np.empty(n, dtype=np.float64)
        self._check(self._lib.sc_read(self.ctx, _dptr(out), len(out)))
        return out

    def read_owned(self, out):
        """Write the DOFs this rank owns into ``out`` (length n_dof; other entries untouched)."""
        self._check(self._lib.sc_read_owned(self.ctx, _dptr(out), len(out)))
        return out

    def set_receivers(self, xyz, capacity):
        """Record u at the points xyz (n x 3) after every step (at most `capacity` rows)."""
        X = np.ascontiguousarray(np.asarray(xyz, dtype=np.float64).reshape(-1, 3))
        self._n_rec = len(X)
        self._check(self._lib.sc_set_receivers(self.ctx, _dptr(X), len(X), int(capacity)))

    def traces(self, max_rows=None):
        """Recorded receiver rows (rows x n_rec): row k is u after step k+1."""
        n = getattr(self, "_n_rec", 0)
        cap = max_rows if max_rows is not None else self.query()["step"]
        out = np.zeros((max(cap, 1), max(n, 1)))
        rows = ctypes.c_int64()
        self._check(self._lib.sc_read_traces(self.ctx, _dptr(out), int(cap), ctypes.byref(rows)))
        return out[:rows.value, :n]

    def estimate_dt(self, iters=2000):
        """(lambda_max, dt_crit) of the explicit subsystem by device power iteration
        (clobbers the state: call set_state before stepping again)."""
        lam, dt = ctypes.c_double(), ctypes.c_double()
        self._check(self._lib.sc_estimate_dt(self.ctx, int(iters), ctypes.byref(lam), ctypes.byref(dt)))
        return lam.value, dt.value

    def cell_dt(self, which=0):
        """Cell-wise critical time steps (cells x fastest): uncut cells the uncut cell-wise
        value, cut cells with the consistent (which=0) or HRZ-lumped (which=1) mass, 0 if empty."""
        out = np.empty(self._n_cells)
        self._check(self._lib.sc_cell_dt(self.ctx, int(which), _dptr(out), len(out)))
        return out

    def elastic_energy(self):
        """E = 1/2 u_n^T K u_n of the current state (device; state unchanged)."""
        e = ctypes.c_double()
        self._check(self._lib.sc_elastic_energy(self.ctx, ctypes.byref(e)))
        return e.value

    def read_c_state(self):
        n = self.info["n_c"]
        v = np.empty(max(n, 1))
        a = np.empty(max(n, 1))
        self._check(self._lib.sc_read_c_state(self.ctx, _dptr(v), _dptr(a), n))
        return v[:n], a[:n]

    def classification(self):
        n_cells = 1
        # cell count from the lattice: product of cells; keep it from construction
        cc = np.empty(self._n_cells, dtype=np.int8)
        isc = np.empty(self.info["n_dof"], dtype=np.uint8)
        lat = np.empty(self.info["n_dof"], dtype=np.int64)
        del n_cells
        self._check(self._lib.sc_read_classification(
            self.ctx, cc.ctypes.data_as(ctypes.POINTER(ctypes.c_int8)),
            isc.ctypes.data_as(ctypes.POINTER(ctypes.c_uint8)),
            lat.ctypes.data_as(ctypes.POINTER(ctypes.c_int64))))
        return cc, isc.astype(bool), lat

    def dof_coords(self):
        n = self.info["n_dof"]
        X = np.empty(3 * n)
        self._check(self._lib.sc_dof_coords(self.ctx, _dptr(X), len(X)))
        return X.reshape(n, 3)

    def profile(self, which, n):
        """Instrumentation: n launches of one sub-kernel (clobbers the state)."""
        self._check(self._lib.sc_profile(self.ctx, int(which), int(n)))

    def close(self):
        if getattr(self, "ctx", None) is not None and self.ctx.value:
            self._lib.sc_destroy(self.ctx)
            self.ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def nccl_unique_id():
    """A new ncclUniqueId (128 bytes) for a world > 1 group; broadcast it to every rank."""
    lib = load_library()
    buf = ctypes.create_string_buffer(128)
    st = lib.sc_nccl_unique_id(ctypes.cast(buf, ctypes.c_void_p))
    if st != SC_OK:
        raise ScError(st, lib.sc_last_error(None).decode())
    return buf.raw


def exchange_local(solvers):
    """In-process ranks: sc_exchange_local over the contexts (solvers[r] is rank r)."""
    lib = load_library()
    arr = (ctypes.c_void_p * len(solvers))(*[s.ctx.value for s in solvers])
    st = lib.sc_exchange_local(arr, len(solvers))
    if st != SC_OK:
        raise ScError(st, lib.sc_last_error(solvers[0].ctx).decode())


def read_group(solvers):
    """In-process ranks: u_n assembled from every rank's owned DOFs."""
    u = np.zeros(solvers[0].info["n_dof"])
    for s in solvers:
        s.read_owned(u)
    return u


def from_config(cfg, f_t=None, stream=None, device=None, set_initial=True, rank=0, world=1, nccl_id=None):
    """Build a Solver from an ``sc_inputs`` config dict (marshalling only)."""
    src = None
    if cfg.get("source") is not None:
        if f_t is None:
            from sc_inputs import source_signal
            f_t = source_signal(cfg)
        src = {"x": cfg["source"]["x"], "f_t": f_t}
        for k in ("kind", "sigma", "amp"):
            if k in cfg["source"]:
                src[k] = cfg["source"][k]
    geo = {k: cfg[k] for k in ("voids", "tree_depth", "lattice_s", "fill_eps", "rho", "c")}
    geo["integrator"] = cfg.get("integrator", "imex")
    geo["lf_m"] = cfg.get("lf_m", 1)
    geo["lf_coupling"] = cfg.get("lf_coupling", "interpolated")
    s = Solver(cfg, cfg["p"], cfg["alpha"], geo, cfg["dt"], source=src, stream=stream, device=device,
               rank=rank, world=world, nccl_id=nccl_id)
    s._n_cells = int(np.prod(cfg["cells"]))
    if set_initial and cfg.get("u0") == "gaussian_pulse":
        from sc_inputs import gaussian_pulse
        s.set_state(gaussian_pulse(s.dof_coords()[:, 0]), None)
    return s
