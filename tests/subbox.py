"""Sub-box parity harness (test infrastructure; no method arithmetic).

A full-size run started from a compactly supported u0 (sc_inputs.compact_bump) with no load
can be checked against the oracle on a sub-box, because the IMEX step has a bounded
dependency region (steps (a1)-(a6) of DESIGN.md §2):

* (a1)+(a2): a d DOF reads only the DOFs of its incident elements, so the support of u grows
  by at most one element per step (the start a_0 = M^-1 (-K u_0), reading C3, is one more);
* (a4)+(a5): the implicit solve couples every c DOF of a connected c component at once
  (S is block diagonal by component), so a component touched anywhere becomes nonzero
  everywhere at that step; components are unions of the c shells of voids, each inside the
  cell bounding box of its void(s).

closure_box() tracks the cells that may hold a nonzero value step by step (one layer of
neighbouring cells per step, plus the whole cell box of every void whose box is reached).  Outside that box u stays EXACTLY zero for `steps` steps in the full domain, and the
box's own boundary (homogeneous Neumann in the sub-box oracle) only ever sees zeros, so the
oracle run on the box equals the full run restricted to it.  tests/test_oracle_subbox.py pins
this claim oracle-against-oracle on the CPU (full domain vs box) before any GPU test uses it.
"""
import copy
import math

import numpy as np


def void_radius(v, dim):
    """Bounding-sphere radius of an ellipsoid void (1/sqrt of the smallest eigenvalue of A)."""
    A = np.array([[v["A"][0], v["A"][3], v["A"][4]], [v["A"][3], v["A"][1], v["A"][5]],
                  [v["A"][4], v["A"][5], v["A"][2]]])[:dim, :dim]
    return 1.0 / math.sqrt(np.linalg.eigvalsh(A).min())


def _cell_box(cfg, lo_x, hi_x):
    d = cfg["dim"]
    lo, hi = [], []
    for k in range(d):
        h = (cfg["hi"][k] - cfg["lo"][k]) / cfg["cells"][k]
        lo.append(int(math.floor((lo_x[k] - cfg["lo"][k]) / h)) - 1)
        hi.append(int(math.ceil((hi_x[k] - cfg["lo"][k]) / h)) + 1)
    return lo, hi


def closure_box(cfg, x0, R, steps, margin=2):
    """Cell box [lo, hi) (per axis) that contains every DOF a run of `steps` steps from a u0
    supported in the ball (x0, R) can touch, plus `margin` cells; and the voids touched.

    Cell-level reachability: A_0 = cells holding a node of the ball; every step (and the start,
    which applies K once) A <- cells sharing a node with A (3^d dilation), then every void whose
    cell bounding box meets A adds that whole box (its c component is solved at once; merged
    shells follow because their boxes intersect), repeated to a fixed point."""
    from scipy import ndimage
    d = cfg["dim"]
    N = cfg["cells"]
    lo0, hi0 = _cell_box(cfg, [x0[k] - R for k in range(d)], [x0[k] + R for k in range(d)])
    act = np.zeros(N[::-1], dtype=bool)          # [z][y][x]
    sl = tuple(slice(max(0, lo0[k]), min(N[k], hi0[k])) for k in reversed(range(d)))
    act[sl] = True
    vbox = []
    for v in cfg["voids"]:
        if v["kind"] != "ellipsoid":
            raise ValueError("closure_box handles ellipsoid voids only")
        r = void_radius(v, d)
        vl, vh = _cell_box(cfg, [v["c"][k] - r for k in range(d)], [v["c"][k] + r for k in range(d)])
        vbox.append(tuple(slice(max(0, vl[k]), min(N[k], vh[k])) for k in reversed(range(d))))
    used = set()
    st = np.ones((3,) * d, dtype=bool)

    def absorb():
        changed = True
        while changed:
            changed = False
            for i, b in enumerate(vbox):
                if i not in used and act[b].any():
                    used.add(i)
                    act[b] = True
                    changed = True

    absorb()
    for _ in range(steps + 1):      # the start + each step
        act = ndimage.binary_dilation(act, structure=st)
        absorb()
    idx = np.nonzero(act)
    lo = [max(0, int(idx[d - 1 - k].min()) - margin) for k in range(d)]
    hi = [min(N[k], int(idx[d - 1 - k].max()) + 1 + margin) for k in range(d)]
    return lo, hi, sorted(used)


def box_config(cfg, lo, hi):
    """The same problem restricted to the cell box [lo, hi): same h, p, alpha, depth, dt; the
    voids whose bounding sphere meets the box; no source."""
    d = cfg["dim"]
    c = copy.deepcopy(cfg)
    c["cells"] = [hi[k] - lo[k] for k in range(d)]
    c["lo"] = [cfg["lo"][k] + (cfg["hi"][k] - cfg["lo"][k]) * (lo[k] / cfg["cells"][k]) for k in range(d)]
    c["hi"] = [cfg["lo"][k] + (cfg["hi"][k] - cfg["lo"][k]) * (hi[k] / cfg["cells"][k]) for k in range(d)]
    keep = []
    for v in cfg["voids"]:
        r = void_radius(v, d)
        ctr = np.array(v["c"][:d])
        near = np.clip(ctr, c["lo"], c["hi"])
        if np.linalg.norm(near - ctr) <= r:
            keep.append(v)
    c["voids"] = keep
    c["source"] = None
    c["u0"] = None
    c["name"] = f"{cfg.get('name', 'cfg')}-box{lo}-{hi}"
    return c


def box_to_full_lattice(cfg, lo, lattice_index_box, box_cells):
    """Lattice indices of the box's lattice nodes in the full grid's (canonical, unpadded)
    lattice numbering."""
    d = cfg["dim"]
    p = cfg["p"]
    nb = [box_cells[k] * p + 1 for k in range(d)]
    nf = [cfg["cells"][k] * p + 1 for k in range(d)]
    rem = np.asarray(lattice_index_box, dtype=np.int64).copy()
    out = np.zeros_like(rem)
    stride = 1
    for k in range(d):
        ik = rem % nb[k]
        rem //= nb[k]
        out += (ik + lo[k] * p) * stride
        stride *= nf[k]
    return out


def interior_cells(cfg, lo, hi, box_cells, pad=1):
    """(full-grid cell indices, box cell indices) of the box cells at least `pad` cells away
    from the box faces (their classification cannot depend on the box truncation)."""
    d = cfg["dim"]
    rng = [np.arange(pad, box_cells[k] - pad) for k in range(d)]
    grids = np.meshgrid(*rng, indexing="ij")
    local = [g.ravel() for g in grids]
    bidx = np.zeros(len(local[0]), dtype=np.int64)
    fidx = np.zeros(len(local[0]), dtype=np.int64)
    bs, fs = 1, 1
    for k in range(d):
        bidx += local[k] * bs
        fidx += (local[k] + lo[k]) * fs
        bs *= box_cells[k]
        fs *= cfg["cells"][k]
    return fidx, bidx
