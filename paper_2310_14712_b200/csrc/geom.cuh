// Device geometry helpers: exact (FMA-free) lattice coordinates and void membership.
//
// PAPER.md P:417-442 (FCM embedding, alpha = 1 in Omega_p, alpha_f in Omega_f);
// DESIGN.md reading C17: x = lo + (hi-lo)*(m/den) with ONE correctly rounded division,
// q = (A00 d0)d0 + (A11 d1)d1 + (A22 d2)d2 + 2((A01 d0)d1 + (A02 d0)d2 + (A12 d1)d2)
// evaluated left to right without contraction, void iff q < 1 (Omega_p closed);
// half-space void iff (n0 x0 + n1 x1) + n2 x2 > b.  The intrinsics __dmul_rn/__dadd_rn
// are never contracted into FMAs, so the decisions are bit-identical to any IEEE
// implementation that evaluates the same expression in the same order.
#pragma once
#include "sc_internal.h"

__device__ __forceinline__ double lat_coord(double lo, double hi, long long m, long long den) {
  return __dadd_rn(lo, __dmul_rn(__dadd_rn(hi, -lo), __ddiv_rn((double)m, (double)den)));
}

__device__ __forceinline__ bool void_contains(const DVoid& v, double x0, double x1, double x2) {
  if (v.kind == SC_VOID_ELLIPSOID) {
    // exact-safe culling: outside the inflated bounding box q >= (1+1e-6)^2 > 1
    if (x0 < v.bblo[0] || x0 > v.bbhi[0] || x1 < v.bblo[1] || x1 > v.bbhi[1] ||
        x2 < v.bblo[2] || x2 > v.bbhi[2])
      return false;
    const double d0 = __dadd_rn(x0, -v.c[0]);
    const double d1 = __dadd_rn(x1, -v.c[1]);
    const double d2 = __dadd_rn(x2, -v.c[2]);
    double q = __dmul_rn(__dmul_rn(v.A[0], d0), d0);
    q = __dadd_rn(q, __dmul_rn(__dmul_rn(v.A[1], d1), d1));
    q = __dadd_rn(q, __dmul_rn(__dmul_rn(v.A[2], d2), d2));
    double t = __dmul_rn(__dmul_rn(v.A[3], d0), d1);
    t = __dadd_rn(t, __dmul_rn(__dmul_rn(v.A[4], d0), d2));
    t = __dadd_rn(t, __dmul_rn(__dmul_rn(v.A[5], d1), d2));
    q = __dadd_rn(q, __dmul_rn(2.0, t));
    return q < 1.0;
  } else {
    double s = __dadd_rn(__dmul_rn(v.n[0], x0), __dmul_rn(v.n[1], x1));
    s = __dadd_rn(s, __dmul_rn(v.n[2], x2));
    return s > v.b;
  }
}

// candidate voids of an axis-aligned box [blo, bhi] (superset: bbox overlap)
__device__ __forceinline__ int box_candidates(const DVoid* __restrict__ V, int nv, const double* blo,
                                              const double* bhi, int* cand, int maxc) {
  int nc = 0;
  for (int i = 0; i < nv; ++i) {
    const DVoid& v = V[i];
    bool hit = true;
    if (v.kind == SC_VOID_ELLIPSOID) {
      for (int k = 0; k < 3; ++k)
        if (bhi[k] < v.bblo[k] || blo[k] > v.bbhi[k]) hit = false;
    }
    if (hit) {
      if (nc >= maxc) return -1;
      cand[nc++] = i;
    }
  }
  return nc;
}

__device__ __forceinline__ bool phys_cand(const DVoid* __restrict__ V, int nv, const int* cand, int nc,
                                          double x0, double x1, double x2) {
  if (nc < 0) {
    for (int i = 0; i < nv; ++i)
      if (void_contains(V[i], x0, x1, x2)) return false;
    return true;
  }
  for (int i = 0; i < nc; ++i)
    if (void_contains(V[cand[i]], x0, x1, x2)) return false;
  return true;
}
