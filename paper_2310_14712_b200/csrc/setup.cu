// Setup kernels of libsc: cell classification (lattice cut test + spacetree, reading C6),
// node classification (d / c partition), cut-cell element matrices
// (spacetree Gauss quadrature with pointwise alpha).
#include <cmath>
#include <cstring>
#include <numeric>

#include "geom.cuh"
#include "sc_internal.h"

#define MAXCAND 24

namespace {

__device__ __forceinline__ void cell_coords(const GridP& g, long long cell, int* ci) {
  long long t = cell;
  for (int k = 0; k < 3; ++k) {
    if (k < g.dim) {
      ci[k] = (int)(t % g.N[k]);
      t /= g.N[k];
    } else {
      ci[k] = 0;
    }
  }
}

__device__ __forceinline__ void cell_box(const GridP& g, const int* ci, double* blo, double* bhi) {
  for (int k = 0; k < 3; ++k) {
    if (k < g.dim) {
      blo[k] = lat_coord(g.lo[k], g.hi[k], ci[k], g.N[k]);
      bhi[k] = lat_coord(g.lo[k], g.hi[k], ci[k] + 1, g.N[k]);
    } else {
      blo[k] = 0.0;
      bhi[k] = 0.0;
    }
  }
}

// lattice test of tree node (level l, offsets a) of cell ci: returns 0 all phys, 1 all fict, 2 mixed
__device__ int node_test(const GridP& g, const DVoid* V, int nv, const int* cand, int nc, const int* ci,
                         int l, const int* a) {
  const int s = g.s;
  bool anyp = false, anyf = false;
  const int n0 = s + 1, n1 = g.dim > 1 ? s + 1 : 1, n2 = g.dim > 2 ? s + 1 : 1;
  double xs[3][17];
  for (int k = 0; k < 3; ++k) {
    if (k < g.dim) {
      const long long den = (long long)g.N[k] * s << l;
      const long long m0 = ((long long)ci[k] * s << l) + (long long)a[k] * s;
      for (int t = 0; t <= s; ++t) xs[k][t] = lat_coord(g.lo[k], g.hi[k], m0 + t, den);
    } else {
      xs[k][0] = 0.0;
    }
  }
  for (int t2 = 0; t2 < n2; ++t2)
    for (int t1 = 0; t1 < n1; ++t1)
      for (int t0 = 0; t0 < n0; ++t0) {
        bool ph = phys_cand(V, nv, cand, nc, xs[0][t0], xs[1][t1], xs[2][t2]);
        anyp |= ph;
        anyf |= !ph;
        if (anyp && anyf) return 2;
      }
  return anyp ? 0 : 1;
}

__global__ void k_root_classify(GridP g, const DVoid* __restrict__ V, int nv, long long n_cells,
                                uint8_t* __restrict__ root) {
  long long cell = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (cell >= n_cells) return;
  int ci[3];
  cell_coords(g, cell, ci);
  double blo[3], bhi[3];
  cell_box(g, ci, blo, bhi);
  int cand[MAXCAND];
  int nc = box_candidates(V, nv, blo, bhi, cand, MAXCAND);
  if (nc == 0) {
    root[cell] = 0;
    return;
  }
  int a[3] = {0, 0, 0};
  root[cell] = (uint8_t)node_test(g, V, nv, cand, nc, ci, 0, a);
}

// One thread per candidate cell (root not all-physical): depth-first spacetree by the
// lattice rule; leaves stored packed; physical Gauss points counted -> CUT / EMPTY.
__global__ void k_tree(GridP g, const DVoid* __restrict__ V, int nv, const long long* __restrict__ cells,
                       int n, int cap, const double* __restrict__ tq, unsigned long long* __restrict__ leaves,
                       int* __restrict__ nleaves, int8_t* __restrict__ cls, int* __restrict__ err) {
  int idx = blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= n) return;
  long long cell = cells[idx];
  int ci[3];
  cell_coords(g, cell, ci);
  double blo[3], bhi[3];
  cell_box(g, ci, blo, bhi);
  int cand[MAXCAND];
  int nc = box_candidates(V, nv, blo, bhi, cand, MAXCAND);
  const int d = g.dim, nch = 1 << d;
  // explicit DFS stack
  int st_l[64];
  int st_a[64][3];
  int sp = 0;
  st_l[0] = 0;
  st_a[0][0] = st_a[0][1] = st_a[0][2] = 0;
  sp = 1;
  int nl = 0;
  long long nphys = 0;
  const int P1 = g.p + 1;
  const int npk1 = g.dim > 1 ? P1 : 1, npk2 = g.dim > 2 ? P1 : 1;
  while (sp > 0) {
    --sp;
    const int l = st_l[sp];
    int a[3] = {st_a[sp][0], st_a[sp][1], st_a[sp][2]};
    int t = node_test(g, V, nv, cand, nc, ci, l, a);
    if (t == 2 && l < g.depth) {
      if (sp + nch > 64) {
        atomicExch(err, 1);
        return;
      }
      for (int o = nch - 1; o >= 0; --o) {
        st_l[sp] = l + 1;
        for (int k = 0; k < 3; ++k) st_a[sp][k] = (k < d) ? 2 * a[k] + ((o >> k) & 1) : 0;
        ++sp;
      }
      continue;
    }
    if (nl >= cap) {
      atomicExch(err, 2);
      return;
    }
    leaves[(long long)idx * cap + nl] = ((unsigned long long)l << 48) | ((unsigned long long)a[2] << 32) |
                                        ((unsigned long long)a[1] << 16) | (unsigned long long)a[0];
    ++nl;
    // physical Gauss points of this leaf (pointwise alpha, C6)
    double lo_[3], span[3];
    for (int k = 0; k < 3; ++k) {
      if (k < d) {
        const long long den = (long long)g.N[k] * g.s << l;
        const long long m0 = ((long long)ci[k] * g.s << l) + (long long)a[k] * g.s;
        double xlo = lat_coord(g.lo[k], g.hi[k], m0, den);
        double xhi = lat_coord(g.lo[k], g.hi[k], m0 + g.s, den);
        lo_[k] = xlo;
        span[k] = __dadd_rn(xhi, -xlo);
      } else {
        lo_[k] = 0.0;
        span[k] = 0.0;
      }
    }
    for (int q2 = 0; q2 < npk2; ++q2)
      for (int q1 = 0; q1 < npk1; ++q1)
        for (int q0 = 0; q0 < P1; ++q0) {
          double x0 = __dadd_rn(lo_[0], __dmul_rn(span[0], tq[q0]));
          double x1 = d > 1 ? __dadd_rn(lo_[1], __dmul_rn(span[1], tq[q1])) : 0.0;
          double x2 = d > 2 ? __dadd_rn(lo_[2], __dmul_rn(span[2], tq[q2])) : 0.0;
          nphys += phys_cand(V, nv, cand, nc, x0, x1, x2) ? 1 : 0;
        }
  }
  nleaves[idx] = nl;
  cls[cell] = nphys > 0 ? 1 : 2;  // CUT : EMPTY
}

// node types: 0 hole, 1 tensor-d (all incident in-box cells uncut), 2 irregular-d
// (no cut incident cell, some empty one), 3 c (>= 1 cut incident cell)
__global__ void k_node_type(GridP g, const int8_t* __restrict__ cls, long long n_lat, uint8_t* __restrict__ nt) {
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= n_lat) return;
  long long t = i;
  int e0[3], e1[3];
  for (int k = 0; k < 3; ++k) {
    if (k < g.dim) {
      long long j = t % g.nl[k];
      t /= g.nl[k];
      if (j % g.p == 0) {
        e0[k] = (int)(j / g.p) - 1;
        e1[k] = (int)(j / g.p);
      } else {
        e0[k] = e1[k] = (int)(j / g.p);
      }
      if (e0[k] < 0) e0[k] = e1[k];
      if (e1[k] >= g.N[k]) e1[k] = e0[k];
    } else {
      e0[k] = e1[k] = 0;
    }
  }
  bool anycut = false, anyempty = false, anyne = false;
  for (int c2 = e0[2]; c2 <= e1[2]; ++c2)
    for (int c1 = e0[1]; c1 <= e1[1]; ++c1)
      for (int c0 = e0[0]; c0 <= e1[0]; ++c0) {
        long long ci = c0 + (long long)g.N[0] * (c1 + (long long)(g.dim > 1 ? g.N[1] : 1) * c2);
        int8_t c = cls[ci];
        anycut |= (c == 1);
        anyempty |= (c == 2);
        anyne |= (c != 2);
      }
  nt[i] = !anyne ? 0 : (anycut ? 3 : (anyempty ? 2 : 1));
}

__device__ double d_lagr(const double* nodes, int n, int i, double xi, double* der) {
  double val = 1.0, dv = 0.0;
  for (int j = 0; j < n; ++j) {
    if (j == i) continue;
    double inv = 1.0 / (nodes[i] - nodes[j]);
    double f = (xi - nodes[j]) * inv;
    dv = dv * f + val * inv;
    val *= f;
  }
  *der = dv;
  return val;
}

// s + c += x*y with an error-free product (fma) and Neumaier's compensated addition; the
// _rn intrinsics keep the compiler from contracting the error terms into FMAs.
__device__ __forceinline__ void comp_add(double& s, double& c, double x, double y) {
  const double p = __dmul_rn(x, y);
  const double e = fma(x, y, -p);
  const double t = __dadd_rn(s, p);
  const double z = fabs(s) >= fabs(p) ? __dadd_rn(__dadd_rn(s, -t), p) : __dadd_rn(__dadd_rn(p, -t), s);
  c = __dadd_rn(c, __dadd_rn(z, e));
  s = t;
}

// Cut-cell element matrices: one CTA per CUT cell; each thread owns a 4x4 tile of both M_e
// and K_e (tiles on and above the diagonal only: M_e and K_e are symmetric, the lower tiles are
// written as mirror images); quadrature points are staged in chunks of QC points in shared
// memory and replayed once per group of blockDim.x tiles.
#define QC 8
__global__ void __launch_bounds__(256) k_cut_matrices(GridP g, const DVoid* __restrict__ V, int nv, const long long* __restrict__ cells,
                               const int* __restrict__ slot, const unsigned long long* __restrict__ leaves,
                               const int* __restrict__ nleaves, int cap, const double* __restrict__ gll,
                               const double* __restrict__ gx, const double* __restrict__ gw,
                               const double* __restrict__ tq, double alpha, double rho, double c2, int nb,
                               int nbp, double* __restrict__ Kout, double* __restrict__ Mout) {
  extern __shared__ double sm[];
  double* sN = sm;                    // [QC][nbp]
  double* sG = sN + QC * nbp;         // [3][QC][nbp]
  double* sphi = sG + 3 * QC * nbp;   // [QC][3][SC_MAXP1]
  double* sdph = sphi + QC * 3 * SC_MAXP1;
  double* sw = sdph + QC * 3 * SC_MAXP1;  // [QC] weight incl alpha
  __shared__ int cand[MAXCAND];
  __shared__ int s_nc;
  const int e = blockIdx.x;
  const long long cell = cells[e];
  const int sl = slot[e];
  const int d = g.dim, P1 = g.p + 1;
  int ci[3];
  cell_coords(g, cell, ci);
  if (threadIdx.x == 0) {
    double blo[3], bhi[3];
    cell_box(g, ci, blo, bhi);
    s_nc = box_candidates(V, nv, blo, bhi, cand, MAXCAND);
  }
  __syncthreads();
  const int nc = s_nc;
  const int T = nbp / 4;
  const int ntiles = T * (T + 1) / 2;   // upper-triangular tiles (ti <= tj)
  const int npts = (d == 1) ? P1 : (d == 2 ? P1 * P1 : P1 * P1 * P1);
  const int nl = nleaves[sl];
  const long long total = (long long)nl * npts;
  double hk[3] = {g.h[0], g.h[1], g.h[2]};
  // tile groups: each thread owns one 4x4 tile per group; the quadrature is replayed per group
  for (int tg = 0; tg * (int)blockDim.x < ntiles; ++tg) {
  const int tile = tg * blockDim.x + threadIdx.x;
  int ti = 0, rem = tile;   // tile -> (ti, tj), ti <= tj, row-major over the upper triangle
  while (ti < T && rem >= T - ti) {
    rem -= T - ti;
    ++ti;
  }
  const int i0 = ti * 4, j0 = (ti + rem) * 4;
  const bool active = tile < ntiles;
  // compensated (Neumaier + exact-product) accumulation: the quadrature sums have up to
  // (2^D)^d (p+1)^d terms with cancellation; plain accumulation loses ~sqrt(n) ulps, which
  // the IMEX recursion amplifies over thousands of steps (reading C23)
  double accM[4][4], accK[4][4], cmpM[4][4], cmpK[4][4];
  for (int a = 0; a < 4; ++a)
    for (int b = 0; b < 4; ++b) accM[a][b] = accK[a][b] = cmpM[a][b] = cmpK[a][b] = 0.0;
  for (long long q0 = 0; q0 < total; q0 += QC) {
    const int nq = (int)min((long long)QC, total - q0);
    // per point, per axis, per basis function: the 1D value/derivative, one thread each;
    // the alpha-weighted quadrature weight of each point on the threads after those
    const int nbas = nq * 3 * P1;
    for (int t = threadIdx.x; t < nbas + nq; t += blockDim.x) {
      if (t < nbas) {
        const int i = t % P1, qk = t / P1, qq = qk / 3, k = qk % 3;
        if (k >= d) continue;
        const long long q = q0 + qq;
        const unsigned long long lf = leaves[(long long)sl * cap + q / npts];
        const int l = (int)(lf >> 48);
        const int a = (int)((lf >> (16 * k)) & 0xFFFF);
        const int loc = (int)(q % npts);
        const int gk = (k == 0) ? loc % P1 : (k == 1 ? (loc / P1) % P1 : loc / (P1 * P1));
        const double xi = -1.0 + (2.0 * a + 1.0 + gx[gk]) * ldexp(1.0, -l);
        double dd;
        sphi[(qq * 3 + k) * SC_MAXP1 + i] = d_lagr(gll, P1, i, xi, &dd);
        sdph[(qq * 3 + k) * SC_MAXP1 + i] = dd * (2.0 / hk[k]);
      } else {
        const int qq = t - nbas;
        const long long q = q0 + qq;
        const unsigned long long lf = leaves[(long long)sl * cap + q / npts];
        const int l = (int)(lf >> 48);
        const int loc = (int)(q % npts);
        // alpha at the physical Gauss point (same arithmetic as the classifier)
        double x[3] = {0.0, 0.0, 0.0};
        double w = 1.0;
        int gg[3] = {loc % P1, (loc / P1) % P1, loc / (P1 * P1)};
        for (int kk = 0; kk < d; ++kk) {
          const int ak = (int)((lf >> (16 * kk)) & 0xFFFF);
          const long long den = (long long)g.N[kk] * g.s << l;
          const long long m0 = ((long long)ci[kk] * g.s << l) + (long long)ak * g.s;
          double xlo = lat_coord(g.lo[kk], g.hi[kk], m0, den);
          double xhi = lat_coord(g.lo[kk], g.hi[kk], m0 + g.s, den);
          x[kk] = __dadd_rn(xlo, __dmul_rn(__dadd_rn(xhi, -xlo), tq[gg[kk]]));
          w *= gw[gg[kk]] * 0.5 * hk[kk] * ldexp(1.0, -l);
        }
        const bool ph = phys_cand(V, nv, cand, nc, x[0], x[1], x[2]);
        sw[qq] = w * (ph ? 1.0 : alpha);
      }
    }
    __syncthreads();
    for (int t = threadIdx.x; t < nq * nbp; t += blockDim.x) {
      const int qq = t / nbp, i = t % nbp;
      double N = 0.0, G0 = 0.0, G1 = 0.0, G2 = 0.0;
      if (i < nb) {
        const int a0 = i % P1, a1 = (i / P1) % P1, a2 = i / (P1 * P1);
        const double* ph = &sphi[qq * 3 * SC_MAXP1];
        const double* dp = &sdph[qq * 3 * SC_MAXP1];
        if (d == 1) {
          N = ph[a0];
          G0 = dp[a0];
        } else if (d == 2) {
          N = ph[a0] * ph[SC_MAXP1 + a1];
          G0 = dp[a0] * ph[SC_MAXP1 + a1];
          G1 = ph[a0] * dp[SC_MAXP1 + a1];
        } else {
          const double f0 = ph[a0], f1 = ph[SC_MAXP1 + a1], f2 = ph[2 * SC_MAXP1 + a2];
          N = f0 * f1 * f2;
          G0 = dp[a0] * f1 * f2;
          G1 = f0 * dp[SC_MAXP1 + a1] * f2;
          G2 = f0 * f1 * dp[2 * SC_MAXP1 + a2];
        }
      }
      sN[qq * nbp + i] = N;
      sG[(0 * QC + qq) * nbp + i] = G0;
      sG[(1 * QC + qq) * nbp + i] = G1;
      sG[(2 * QC + qq) * nbp + i] = G2;
    }
    __syncthreads();
    if (active) {
      for (int qq = 0; qq < nq; ++qq) {
        const double w = sw[qq];
        double ni[4], nj[4];
        for (int a = 0; a < 4; ++a) {
          ni[a] = w * sN[qq * nbp + i0 + a];
          nj[a] = sN[qq * nbp + j0 + a];
        }
        for (int a = 0; a < 4; ++a)
          for (int b = 0; b < 4; ++b) comp_add(accM[a][b], cmpM[a][b], ni[a], nj[b]);
        for (int k = 0; k < d; ++k) {
          const double* G = &sG[(k * QC + qq) * nbp];
          for (int a = 0; a < 4; ++a) {
            ni[a] = w * G[i0 + a];
            nj[a] = G[j0 + a];
          }
          for (int a = 0; a < 4; ++a)
            for (int b = 0; b < 4; ++b) comp_add(accK[a][b], cmpK[a][b], ni[a], nj[b]);
        }
      }
    }
    __syncthreads();
  }
  if (active) {
    for (int a = 0; a < 4; ++a)
      for (int b = 0; b < 4; ++b) {
        const int i = i0 + a, j = j0 + b;
        if (i < nb && j < nb && i <= j) {   // (i, j) and its mirror (j, i): exactly symmetric
          const double kv = rho * c2 * (accK[a][b] + cmpK[a][b]), mv = rho * (accM[a][b] + cmpM[a][b]);
          Kout[(long long)e * nb * nb + (long long)i * nb + j] = kv;
          Mout[(long long)e * nb * nb + (long long)i * nb + j] = mv;
          Kout[(long long)e * nb * nb + (long long)j * nb + i] = kv;
          Mout[(long long)e * nb * nb + (long long)j * nb + i] = mv;
        }
      }
  }
  __syncthreads();
  }
}

}  // namespace

static void upload_voids(sc_ctx* c) {
  for (DVoid& v : c->voids) {
    for (int k = 0; k < 3; ++k) {
      v.bblo[k] = -INFINITY;
      v.bbhi[k] = INFINITY;
    }
    if (v.kind != SC_VOID_ELLIPSOID) continue;
    const int d = c->g.dim;
    // inverse of the leading d x d block of A: half-extents sqrt((A^-1)_kk)
    double A[3][3] = {{v.A[0], v.A[3], v.A[4]}, {v.A[3], v.A[1], v.A[5]}, {v.A[4], v.A[5], v.A[2]}};
    double inv[3] = {0, 0, 0};
    if (d == 1) {
      inv[0] = 1.0 / A[0][0];
    } else if (d == 2) {
      double det = A[0][0] * A[1][1] - A[0][1] * A[1][0];
      inv[0] = A[1][1] / det;
      inv[1] = A[0][0] / det;
    } else {
      double c00 = A[1][1] * A[2][2] - A[1][2] * A[2][1];
      double c11 = A[0][0] * A[2][2] - A[0][2] * A[2][0];
      double c22 = A[0][0] * A[1][1] - A[0][1] * A[1][0];
      double det = A[0][0] * c00 - A[0][1] * (A[1][0] * A[2][2] - A[1][2] * A[2][0]) +
                   A[0][2] * (A[1][0] * A[2][1] - A[1][1] * A[2][0]);
      inv[0] = c00 / det;
      inv[1] = c11 / det;
      inv[2] = c22 / det;
    }
    for (int k = 0; k < d; ++k) {
      if (!(inv[k] > 0.0) || !std::isfinite(inv[k]))
        throw ScError(SC_ERR_CONFIG, "void quadratic form is not positive definite");
      double ext = std::sqrt(inv[k]) * (1.0 + 1e-6) + 1e-12;
      v.bblo[k] = v.c[k] - ext;
      v.bbhi[k] = v.c[k] + ext;
    }
  }
  if (!c->voids.empty()) {
    SC_CUDA(cudaMalloc(&c->d_voids, sizeof(DVoid) * c->voids.size()));
    SC_CUDA(cudaMemcpy(c->d_voids, c->voids.data(), sizeof(DVoid) * c->voids.size(), cudaMemcpyHostToDevice));
  }
}

// Classification, DOF partition, cut-cell matrices.  Fills host vectors in c and returns
// the cut-cell mass matrices (host) for the factorisation.
// ---- NEXT-2: cell-wise critical time steps (Fig.
// fig:tCritsCircles, Table tab:criticaltimestepsizes): dt_e = 2 / sqrt(lambda_max(K_e, M_e))
// of every cut cell, with its consistent mass (the "consistent SCM") and with its HRZ-lumped
// mass (M~_ii = m_e / sum_k M_kk M_ii).  One CTA per cut cell, everything in
// shared memory: HRZ: power iteration on D^-1/2 K D^-1/2; consistent: Cholesky M = L L^T
// (packed), C = L^-1 K L^-T (two substitution sweeps), power iteration on C; the Rayleigh
// quotient is iterated until it changes by <= 1e-15 relative for 8 consecutive iterations
// (at most 20000).  out[2 e] = consistent, out[2 e + 1] = HRZ (0 if a pivot is not positive).
__device__ double block_sum(double v, double* red) {
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) red[w] = v;
  __syncthreads();
  double s = 0.0;
  for (int k = 0; k < (int)(blockDim.x >> 5); ++k) s += red[k];
  return s;
}

// power iteration on the symmetric nb x nb matrix S (shared, row-major): lambda_max
__device__ double power_max(const double* S, int nb, double* x, double* y, double* red) {
  const int t = threadIdx.x;
  for (int i = t; i < nb; i += blockDim.x) x[i] = 1.0 + 0.25 * (double)((i * 7919) % 97) / 97.0;
  __syncthreads();
  double lam = 0.0;
  int stable = 0;
  for (int it = 0; it < 20000 && stable < 8; ++it) {
    double xy = 0.0, xx = 0.0, yy = 0.0;
    for (int i = t; i < nb; i += blockDim.x) {
      double a = 0.0;
      for (int j = 0; j < nb; ++j) a = fma(S[i * nb + j], x[j], a);
      y[i] = a;
      xy += x[i] * a;
      xx += x[i] * x[i];
      yy += a * a;
    }
    xy = block_sum(xy, red);
    xx = block_sum(xx, red + 8);
    yy = block_sum(yy, red + 16);
    const double l2 = xy / xx, sc = yy > 0.0 ? 1.0 / sqrt(yy) : 0.0;
    stable = (fabs(l2 - lam) <= 1e-15 * fabs(l2)) ? stable + 1 : 0;
    lam = l2;
    for (int i = t; i < nb; i += blockDim.x) x[i] = y[i] * sc;
    __syncthreads();
  }
  return lam;
}

__global__ void k_cell_dt(const double* __restrict__ Kfull, const double* __restrict__ Mfull, int nb, double* out) {
  extern __shared__ double sh[];
  const int np = nb * (nb + 1) / 2;
  double* L = sh;                 // packed lower Cholesky factor, row i at i (i + 1) / 2
  double* S = L + np;             // nb x nb
  double* x = S + nb * nb;
  double* y = x + nb;
  double* d = y + nb;             // HRZ diagonal
  double* red = d + nb;           // [24] reductions
  const int e = blockIdx.x, t = threadIdx.x, nt = blockDim.x;
  const double* K = Kfull + (size_t)e * nb * nb;
  const double* M = Mfull + (size_t)e * nb * nb;
  // ---- HRZ-lumped mass: m_e = sum_ij M_ij, trace = sum_k M_kk
  double me = 0.0, tr = 0.0;
  for (int q = t; q < nb * nb; q += nt) me += M[q];
  for (int i = t; i < nb; i += nt) tr += M[(size_t)i * nb + i];
  me = block_sum(me, red);
  tr = block_sum(tr, red + 8);
  for (int i = t; i < nb; i += nt) d[i] = 1.0 / sqrt(me / tr * M[(size_t)i * nb + i]);
  __syncthreads();
  for (int q = t; q < nb * nb; q += nt) S[q] = d[q / nb] * K[q] * d[q % nb];
  __syncthreads();
  const double lh = power_max(S, nb, x, y, red);
  // ---- consistent mass: Cholesky of M (lower, packed), right-looking
  for (int q = t; q < np; q += nt) {
    int i = (int)((sqrt(8.0 * q + 1.0) - 1.0) * 0.5);
    while (i * (i + 1) / 2 > q) --i;
    while ((i + 1) * (i + 2) / 2 <= q) ++i;
    const int j = q - i * (i + 1) / 2;
    L[q] = M[(size_t)i * nb + j];
  }
  __syncthreads();
  bool ok = true;
  for (int k = 0; k < nb; ++k) {
    const double pk = L[k * (k + 1) / 2 + k];
    if (!(pk > 0.0)) ok = false;
    const double lkk = sqrt(pk);
    __syncthreads();
    for (int i = k + 1 + t; i < nb; i += nt) L[i * (i + 1) / 2 + k] /= lkk;
    if (t == 0) L[k * (k + 1) / 2 + k] = lkk;
    __syncthreads();
    // trailing update L_ij -= L_ik L_jk, k < j <= i
    const int m = nb - k - 1;
    for (int q = t; q < m * (m + 1) / 2; q += nt) {
      int a = (int)((sqrt(8.0 * q + 1.0) - 1.0) * 0.5);
      while (a * (a + 1) / 2 > q) --a;
      while ((a + 1) * (a + 2) / 2 <= q) ++a;
      const int b = q - a * (a + 1) / 2;
      const int i = k + 1 + a, j = k + 1 + b;
      L[i * (i + 1) / 2 + j] -= L[i * (i + 1) / 2 + k] * L[j * (j + 1) / 2 + k];
    }
    __syncthreads();
  }
  double lc = 0.0;
  if (ok) {
    for (int q = t; q < nb * nb; q += nt) S[q] = K[q];
    __syncthreads();
    // S <- L^-1 S (forward substitution, one column per thread)
    for (int j = t; j < nb; j += nt)
      for (int i = 0; i < nb; ++i) {
        double a = S[i * nb + j];
        for (int k = 0; k < i; ++k) a -= L[i * (i + 1) / 2 + k] * S[k * nb + j];
        S[i * nb + j] = a / L[i * (i + 1) / 2 + i];
      }
    __syncthreads();
    // S <- S L^-T (forward substitution on the rows, one row per thread)
    for (int i = t; i < nb; i += nt)
      for (int j = 0; j < nb; ++j) {
        double a = S[i * nb + j];
        for (int k = 0; k < j; ++k) a -= S[i * nb + k] * L[j * (j + 1) / 2 + k];
        S[i * nb + j] = a / L[j * (j + 1) / 2 + j];
      }
    __syncthreads();
    // symmetrise (rounding) and iterate
    for (int q = t; q < nb * nb; q += nt) {
      const int i = q / nb, j = q % nb;
      if (i < j) {
        const double a = 0.5 * (S[i * nb + j] + S[j * nb + i]);
        S[i * nb + j] = a;
        S[j * nb + i] = a;
      }
    }
    __syncthreads();
    lc = power_max(S, nb, x, y, red);
  }
  if (t == 0) {
    out[2 * (size_t)e] = (ok && lc > 0.0) ? 2.0 / sqrt(lc) : 0.0;
    out[2 * (size_t)e + 1] = lh > 0.0 ? 2.0 / sqrt(lh) : 0.0;
  }
}

void setup_device_geometry(sc_ctx* c) {
  upload_voids(c);
  const GridP& g = c->g;
  const int nv = (int)c->voids.size();
  const long long n_cells = c->n_cells;
  uint8_t* d_root = nullptr;
  SC_CUDA(cudaMalloc(&d_root, n_cells));
  SC_CUDA(cudaMalloc(&c->d_cell_class, n_cells));
  k_root_classify<<<(unsigned)((n_cells + 255) / 256), 256, 0, c->stream>>>(g, c->d_voids, nv, n_cells, d_root);
  SC_CUDA(cudaGetLastError());
  std::vector<uint8_t> root(n_cells);
  SC_CUDA(cudaMemcpyAsync(root.data(), d_root, n_cells, cudaMemcpyDeviceToHost, c->stream));
  SC_CUDA(cudaStreamSynchronize(c->stream));
  cudaFree(d_root);
  c->cell_class.assign(n_cells, 0);
  std::vector<long long> cand;
  for (long long i = 0; i < n_cells; ++i)
    if (root[i] != 0) cand.push_back(i);
  // spacetree of candidate cells
  int cap = 1;
  for (int l = 0; l < g.depth; ++l) cap *= (1 << g.dim);
  if (cap > 4096) throw ScError(SC_ERR_CONFIG, "tree_depth too large (more than 4096 leaves per cell)");
  const int n_cand = (int)cand.size();
  long long* d_cand = nullptr;
  unsigned long long* d_leaves = nullptr;
  int *d_nleaves = nullptr, *d_err = nullptr;
  double* d_tq = nullptr;
  std::vector<double> tq(g.p + 1);
  for (int i = 0; i <= g.p; ++i) tq[i] = (c->gau_x[i] + 1.0) * 0.5;
  SC_CUDA(cudaMalloc(&d_tq, sizeof(double) * tq.size()));
  SC_CUDA(cudaMemcpy(d_tq, tq.data(), sizeof(double) * tq.size(), cudaMemcpyHostToDevice));
  SC_CUDA(cudaMalloc(&d_err, sizeof(int)));
  SC_CUDA(cudaMemset(d_err, 0, sizeof(int)));
  SC_CUDA(cudaMemsetAsync(c->d_cell_class, 0, n_cells, c->stream));
  if (n_cand > 0) {
    SC_CUDA(cudaMalloc(&d_cand, sizeof(long long) * n_cand));
    SC_CUDA(cudaMalloc(&d_leaves, sizeof(unsigned long long) * (size_t)n_cand * cap));
    SC_CUDA(cudaMalloc(&d_nleaves, sizeof(int) * n_cand));
    SC_CUDA(cudaMemcpyAsync(d_cand, cand.data(), sizeof(long long) * n_cand, cudaMemcpyHostToDevice, c->stream));
    k_tree<<<(n_cand + 127) / 128, 128, 0, c->stream>>>(g, c->d_voids, nv, d_cand, n_cand, cap, d_tq, d_leaves,
                                                          d_nleaves, c->d_cell_class, d_err);
    SC_CUDA(cudaGetLastError());
  }
  int herr = 0;
  SC_CUDA(cudaMemcpyAsync(&herr, d_err, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
  SC_CUDA(cudaMemcpyAsync(c->cell_class.data(), c->d_cell_class, n_cells, cudaMemcpyDeviceToHost, c->stream));
  SC_CUDA(cudaStreamSynchronize(c->stream));
  if (herr) throw ScError(SC_ERR_CONFIG, "spacetree capacity exceeded");
  c->cells_uncut = c->cells_cut = c->cells_empty = 0;
  for (long long i = 0; i < n_cells; ++i) {
    int8_t k = c->cell_class[i];
    if (k == 0) ++c->cells_uncut;
    else if (k == 1) ++c->cells_cut;
    else ++c->cells_empty;
  }
  // node types
  SC_CUDA(cudaMalloc(&c->d_ntype, c->n_lat));
  k_node_type<<<(unsigned)((c->n_lat + 255) / 256), 256, 0, c->stream>>>(g, c->d_cell_class, c->n_lat, c->d_ntype);
  SC_CUDA(cudaGetLastError());
  c->ntype.resize(c->n_lat);
  SC_CUDA(cudaMemcpyAsync(c->ntype.data(), c->d_ntype, c->n_lat, cudaMemcpyDeviceToHost, c->stream));
  SC_CUDA(cudaStreamSynchronize(c->stream));
  // cut-cell element matrices (cut cells in ascending cell order)
  std::vector<long long> cutcells;
  std::vector<int> slots;
  for (int i = 0; i < n_cand; ++i)
    if (c->cell_class[cand[i]] == 1) {
      cutcells.push_back(cand[i]);
      slots.push_back(i);
    }
  c->n_cut = (int64_t)cutcells.size();
  const int nb = c->nb;
  if (c->n_cut > 0) {
    long long* d_cc = nullptr;
    int* d_slots = nullptr;
    double *d_gll = nullptr, *d_gx = nullptr, *d_gw = nullptr, *d_M = nullptr;
    SC_CUDA(cudaMalloc(&d_cc, sizeof(long long) * c->n_cut));
    SC_CUDA(cudaMalloc(&d_slots, sizeof(int) * c->n_cut));
    SC_CUDA(cudaMemcpy(d_cc, cutcells.data(), sizeof(long long) * c->n_cut, cudaMemcpyHostToDevice));
    SC_CUDA(cudaMemcpy(d_slots, slots.data(), sizeof(int) * c->n_cut, cudaMemcpyHostToDevice));
    SC_CUDA(cudaMalloc(&d_gll, sizeof(double) * (g.p + 1)));
    SC_CUDA(cudaMalloc(&d_gx, sizeof(double) * (g.p + 1)));
    SC_CUDA(cudaMalloc(&d_gw, sizeof(double) * (g.p + 1)));
    SC_CUDA(cudaMemcpy(d_gll, c->gll_x.data(), sizeof(double) * (g.p + 1), cudaMemcpyHostToDevice));
    SC_CUDA(cudaMemcpy(d_gx, c->gau_x.data(), sizeof(double) * (g.p + 1), cudaMemcpyHostToDevice));
    SC_CUDA(cudaMemcpy(d_gw, c->gau_w.data(), sizeof(double) * (g.p + 1), cudaMemcpyHostToDevice));
    const size_t mat = (size_t)c->n_cut * nb * nb;
    SC_CUDA(cudaMalloc(&c->d_Kcut, sizeof(double) * mat));
    SC_CUDA(cudaMalloc(&d_M, sizeof(double) * mat));
    const int nbp = ((nb + 15) / 16) * 16;
    if (nbp > 128) throw ScError(SC_ERR_CONFIG, "(p+1)^dim > 128 not supported by the cut-cell kernel");
    // threads: one upper-triangular 4x4 tile each per replay of the quadrature (nbp = 128: 528
    // tiles, 3 replays of 256; 256 threads keep the 202-register accumulators unspilled)
    const int ntile = (nbp / 4) * (nbp / 4 + 1) / 2;
    const int threads = std::min(256, std::max(32, (ntile + 31) / 32 * 32));
    const size_t smem = sizeof(double) * (4 * QC * nbp + 2 * QC * 3 * SC_MAXP1 + QC);
    SC_CUDA(cudaFuncSetAttribute(k_cut_matrices, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    k_cut_matrices<<<(unsigned)c->n_cut, threads, smem, c->stream>>>(
        g, c->d_voids, nv, d_cc, d_slots, d_leaves, d_nleaves, cap, d_gll, d_gx, d_gw, d_tq, c->alpha, c->rho,
        c->c * c->c, nb, nbp, c->d_Kcut, d_M);
    SC_CUDA(cudaGetLastError());
    // cell-wise critical steps of the cut cells (consistent, HRZ), 2 per cut cell
    {
      SC_CUDA(cudaMalloc(&c->d_cut_dt, sizeof(double) * 2 * c->n_cut));
      const size_t sm = sizeof(double) * ((size_t)nb * (nb + 1) / 2 + (size_t)nb * nb + 3 * (size_t)nb + 24);
      SC_CUDA(cudaFuncSetAttribute(k_cell_dt, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
      k_cell_dt<<<(unsigned)c->n_cut, 128, sm, c->stream>>>(c->d_Kcut, d_M, nb, c->d_cut_dt);
      SC_CUDA(cudaGetLastError());
    }
    c->Kcut_host.resize(mat);
    c->Mcut_host.resize(mat);
    SC_CUDA(cudaMemcpyAsync(c->Kcut_host.data(), c->d_Kcut, sizeof(double) * mat, cudaMemcpyDeviceToHost, c->stream));
    SC_CUDA(cudaMemcpyAsync(c->Mcut_host.data(), d_M, sizeof(double) * mat, cudaMemcpyDeviceToHost, c->stream));
    // the Gaussian-bell load (source kind 2) integrates over the same leaves on the host
    if (c->src_kind == 2) {
      std::vector<unsigned long long> lv((size_t)n_cand * cap);
      std::vector<int> nl(n_cand);
      SC_CUDA(cudaMemcpy(lv.data(), d_leaves, sizeof(unsigned long long) * lv.size(), cudaMemcpyDeviceToHost));
      SC_CUDA(cudaMemcpy(nl.data(), d_nleaves, sizeof(int) * n_cand, cudaMemcpyDeviceToHost));
      c->cut_leaves.assign(c->n_cut, {});
      for (int64_t k = 0; k < c->n_cut; ++k) {
        const int sl = slots[k];
        c->cut_leaves[k].assign(lv.begin() + (size_t)sl * cap, lv.begin() + (size_t)sl * cap + nl[sl]);
      }
    }
    SC_CUDA(cudaStreamSynchronize(c->stream));
    cudaFree(d_cc);
    cudaFree(d_slots);
    cudaFree(d_gll);
    cudaFree(d_gx);
    cudaFree(d_gw);
    cudaFree(d_M);
  }
  c->cut_cells = cutcells;
  if (d_cand) cudaFree(d_cand);
  if (d_leaves) cudaFree(d_leaves);
  if (d_nleaves) cudaFree(d_nleaves);
  cudaFree(d_tq);
  cudaFree(d_err);
}
