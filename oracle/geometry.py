"""Geometry, cut detection, spacetree and cell classes (ORACLE - test infra only).

Follows PAPER.md P:417-442 (FCM embedding, indicator alpha)
(spacetree refined towards the boundary, Gauss points on leaves)
(quadrature by cell class) and P:866-868 (cells with fill ratio below
eps = 1e-10 are empty and discarded).  The paper does not state its cut test
nor its refinement rule; DESIGN.md readings:

C6  lattice rule: a tree node (cell or sub-cell) is tested at an (s+1)^d
    uniform lattice including its corners (s = 4).  All points physical ->
    physical leaf; none -> fictitious leaf; otherwise mixed: split into 2^d
    children while depth < D, a mixed node at depth D is a leaf.  Every leaf
    carries (p+1)^d Gauss points with POINTWISE alpha.  Cell class: UNCUT iff
    the root lattice is all physical; EMPTY iff none of its Gauss points is
    physical; else CUT.  Physical = not strictly inside any void (closed
    Omega_p).
C7  "eta < 1e-10" <=> "zero physical Gauss points" at the configs' depths.
C17 bit-exact arithmetic: lattice coordinate x = lo + (hi-lo)*(m/den) with m,
    den integers and ONE correctly rounded division; ellipsoid predicate
    q = (A00 d0)d0 + (A11 d1)d1 + (A22 d2)d2 + 2((A01 d0)d1 + (A02 d0)d2 + (A12 d1)d2)
    left to right, no FMA, void iff q < 1; half-space void iff
    (n0 x0 + n1 x1) + n2 x2 > b.
Gauss point of a leaf: x = leaf_lo + (leaf_hi - leaf_lo) * ((g + 1) * 0.5),
leaf_lo / leaf_hi being lattice coordinates of the leaf corners.
"""
import numpy as np

UNCUT, CUT, EMPTY = 0, 1, 2


def lattice_coord(lo, hi, m, den):
    """x = lo + (hi - lo) * (m / den)  (reading C17)."""
    m = np.asarray(m, dtype=np.float64)
    return lo + (hi - lo) * (m / np.float64(den))


def is_physical(X, voids):
    """X: (n, 3) float64 points (unused dims = 0).  True where the point is
    not strictly inside any void (P:432-438 alpha = 1 on Omega_p)."""
    X = np.asarray(X, dtype=np.float64)
    inside = np.zeros(len(X), dtype=bool)
    for v in voids:
        if v["kind"] == "ellipsoid":
            c = v["c"]
            A = v["A"]
            d0 = X[:, 0] - c[0]
            d1 = X[:, 1] - c[1]
            d2 = X[:, 2] - c[2]
            q = (A[0] * d0) * d0
            q = q + (A[1] * d1) * d1
            q = q + (A[2] * d2) * d2
            t = (A[3] * d0) * d1
            t = t + (A[4] * d0) * d2
            t = t + (A[5] * d1) * d2
            q = q + 2.0 * t
            inside |= q < 1.0
        elif v["kind"] == "halfspace":
            n = v["n"]
            s = n[0] * X[:, 0] + n[1] * X[:, 1]
            s = s + n[2] * X[:, 2]
            inside |= s > v["b"]
        else:
            raise ValueError(v["kind"])
    return ~inside


def _axis_coords(grid, k, m, level):
    s_den = grid["cells"][k] * grid["s"] * (2 ** level)
    return lattice_coord(grid["lo"][k], grid["hi"][k], m, s_den)


def _tensor_points(per_axis):
    """per_axis: list over axes of (n_nodes, n_pts_k) arrays -> (n_nodes*prod, 3)
    with x fastest inside each node."""
    dim = len(per_axis)
    n_nodes = per_axis[0].shape[0]
    cols = []
    shape = [a.shape[1] for a in per_axis]
    for k in range(dim):
        # broadcast axis k over the tensor grid (x fastest -> axis 0 varies fastest)
        idx_shape = [1] * dim
        idx_shape[dim - 1 - k] = shape[k]
        arr = per_axis[k].reshape((n_nodes, *idx_shape))
        arr = np.broadcast_to(arr, (n_nodes, *shape[::-1]))
        cols.append(arr.reshape(n_nodes, -1))
    X = np.zeros((n_nodes * cols[0].shape[1], 3))
    for k in range(dim):
        X[:, k] = cols[k].reshape(-1)
    return X


def node_lattice_points(grid, cell, levels, a):
    """Lattice test points of tree nodes (level l, integer offsets a in
    [0,2^l)^d) of cell ``cell``: (n_nodes*(s+1)^d, 3)."""
    s = grid["s"]
    dim = grid["dim"]
    per_axis = []
    t = np.arange(s + 1)
    for k in range(dim):
        m = (cell[k] * s * (2 ** levels) + a[:, k] * s)[:, None] + t[None, :]
        per_axis.append(_axis_coords_levels(grid, k, m, levels))
    return _tensor_points(per_axis)


def _axis_coords_levels(grid, k, m, levels):
    den = (grid["cells"][k] * grid["s"] * (2 ** levels)).astype(np.float64)[:, None]
    m = np.asarray(m, dtype=np.float64)
    return grid["lo"][k] + (grid["hi"][k] - grid["lo"][k]) * (m / den)


def build_tree(grid, voids, cell, depth):
    """Spacetree of one cell by the lattice rule C6.  Returns leaf levels
    (L,) and offsets (L, d) (int64) and the root test result
    ('phys' | 'fict' | 'mixed')."""
    dim = grid["dim"]
    npts = (grid["s"] + 1) ** dim
    levels = np.zeros(1, dtype=np.int64)
    a = np.zeros((1, dim), dtype=np.int64)
    leaf_l, leaf_a = [], []
    root = None
    for lev in range(depth + 1):
        X = node_lattice_points(grid, cell, levels, a)
        ph = is_physical(X, voids).reshape(len(levels), npts)
        allp = ph.all(axis=1)
        nonep = ~ph.any(axis=1)
        mixed = ~(allp | nonep)
        if lev == 0:
            root = "phys" if allp[0] else ("fict" if nonep[0] else "mixed")
        if lev == depth:
            leaf_l.append(levels)
            leaf_a.append(a)
            break
        done = ~mixed
        leaf_l.append(levels[done])
        leaf_a.append(a[done])
        am = a[mixed]
        if len(am) == 0:
            break
        kids = []
        for off in range(2 ** dim):
            bits = np.array([(off >> k) & 1 for k in range(dim)], dtype=np.int64)
            kids.append(2 * am + bits[None, :])
        a = np.concatenate(kids, axis=0)
        levels = np.full(len(a), lev + 1, dtype=np.int64)
    return np.concatenate(leaf_l), np.concatenate(leaf_a, axis=0), root


def leaf_gauss_points(grid, cell, levels, a, g):
    """Gauss points (x fastest) of every leaf: coordinates (L*n^d, 3) and the
    leaf-local reference coordinates are implied by (levels, a, g)."""
    dim = grid["dim"]
    s = grid["s"]
    tq = (g + 1.0) * 0.5
    per_axis = []
    for k in range(dim):
        m0 = cell[k] * s * (2 ** levels) + a[:, k] * s
        lo_k = _axis_coords_levels(grid, k, m0[:, None], levels)
        hi_k = _axis_coords_levels(grid, k, (m0 + s)[:, None], levels)
        per_axis.append(lo_k + (hi_k - lo_k) * tq[None, :])
    return _tensor_points(per_axis)


def classify_cell(grid, voids, cell, depth, gauss_nodes):
    """Returns (class, levels, a, phys_mask) for one cell (C6/C7)."""
    levels, a, root = build_tree(grid, voids, cell, depth)
    if root == "phys":
        return UNCUT, levels, a, None
    X = leaf_gauss_points(grid, cell, levels, a, gauss_nodes)
    ph = is_physical(X, voids)
    cls = CUT if ph.any() else EMPTY
    return cls, levels, a, ph


def root_all_physical(grid, voids):
    """Vectorised root-lattice test of every cell: bool array (n_cells,),
    cells in lexicographic order (x fastest)."""
    dim = grid["dim"]
    N = grid["cells"]
    s = grid["s"]
    n_cells = int(np.prod(N))
    out = np.zeros(n_cells, dtype=bool)
    idx = np.arange(n_cells)
    cell_idx = np.zeros((n_cells, dim), dtype=np.int64)
    rem = idx.copy()
    for k in range(dim):
        cell_idx[:, k] = rem % N[k]
        rem //= N[k]
    npts = (s + 1) ** dim
    chunk = max(1, 4_000_000 // npts)
    t = np.arange(s + 1)
    for st in range(0, n_cells, chunk):
        ci = cell_idx[st:st + chunk]
        per_axis = []
        for k in range(dim):
            m = (ci[:, k] * s)[:, None] + t[None, :]
            per_axis.append(grid["lo"][k] + (grid["hi"][k] - grid["lo"][k]) * (m / np.float64(N[k] * s)))
        X = _tensor_points(per_axis)
        out[st:st + chunk] = is_physical(X, voids).reshape(len(ci), npts).all(axis=1)
    return out, cell_idx
