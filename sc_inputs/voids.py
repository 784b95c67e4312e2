"""Seeded void generation (reading C13).

BASELINE.json only says "seeded ... non-overlapping" voids.  Reading C13:
``numpy.random.Generator(PCG64(seed))`` with seed = config index; per
attempt draw the semi-axes, then the orientation (2D: theta ~ U[0, pi);
3D ellipsoid: uniform rotation from a normalised Gaussian quaternion;
spheres: none), then the centre ~ U[R+h, 1-R-h]^d with R the largest
semi-axis.  Reject if the bounding sphere comes within h of an accepted
void's bounding sphere, or within h of the source point.

The output is the explicit quadratic form of each void,
void = {x : (x-c)^T A (x-c) < 1}, stored as A00, A11, A22, A01, A02, A12
(full double precision).  These doubles ARE the input to both sides.
"""
import numpy as np


def _rot2(theta):
    c, s = np.cos(theta), np.sin(theta)
    return np.array([[c, -s], [s, c]])


def _rot3_from_quat(q):
    q = q / np.linalg.norm(q)
    w, x, y, z = q
    return np.array([
        [1 - 2 * (y * y + z * z), 2 * (x * y - z * w), 2 * (x * z + y * w)],
        [2 * (x * y + z * w), 1 - 2 * (x * x + z * z), 2 * (y * z - x * w)],
        [2 * (x * z - y * w), 2 * (y * z + x * w), 1 - 2 * (x * x + y * y)],
    ])


def _pack(A, dim):
    if dim == 2:
        return [float(A[0, 0]), float(A[1, 1]), 0.0, float(A[0, 1]), 0.0, 0.0]
    return [float(A[0, 0]), float(A[1, 1]), float(A[2, 2]),
            float(A[0, 1]), float(A[0, 2]), float(A[1, 2])]


def generate_voids(seed, dim, n_voids, semi_lo, semi_hi, kind, h, source,
                   max_attempts=200000):
    """kind: 'ellipse' (2D), 'sphere' (3D) or 'ellipsoid' (3D)."""
    rng = np.random.Generator(np.random.PCG64(seed))
    accepted = []  # (centre, R)
    out = []
    src = None if source is None else np.asarray(source[:dim], dtype=np.float64)
    attempts = 0
    while len(out) < n_voids:
        attempts += 1
        if attempts > max_attempts:
            raise RuntimeError("void generation did not converge")
        if kind == "sphere":
            semi = np.repeat(rng.uniform(semi_lo, semi_hi), dim)
            rot = np.eye(dim)
        else:
            semi = rng.uniform(semi_lo, semi_hi, size=dim)
            if dim == 2:
                rot = _rot2(rng.uniform(0.0, np.pi))
            else:
                rot = _rot3_from_quat(rng.standard_normal(4))
        R = float(np.max(semi))
        centre = rng.uniform(R + h, 1.0 - R - h, size=dim)
        ok = all(np.linalg.norm(centre - c2) >= R + R2 + h for c2, R2 in accepted)
        if ok and src is not None:
            ok = np.linalg.norm(centre - src) >= R + h
        if not ok:
            continue
        accepted.append((centre, R))
        A = rot @ np.diag(1.0 / semi ** 2) @ rot.T
        A = 0.5 * (A + A.T)
        c3 = [0.0, 0.0, 0.0]
        c3[:dim] = [float(v) for v in centre]
        out.append({"kind": "ellipsoid", "c": c3, "A": _pack(A, dim)})
    return out
