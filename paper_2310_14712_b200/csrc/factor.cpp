// Host-side setup of the implicit cut-DOF solve (a5) and of the c-part data structures.
//
// PAPER.md P:583 / P:1425 / P:1767: the system matrix S = M^cc + beta dt^2 K^cc
// (beta = 1/4) is "factorized once outside the time integration loop"; each step
// performs forward and backward substitution.  B200 design:
//  * S is block diagonal by connected component of the c-graph (voids are disjoint);
//  * each component is ordered by geometric nested dissection on the integer lattice
//    coordinates: planes x_k = m*p (element boundaries) are exact separators of the
//    element graph;
//  * every ND tree node is one dense supernode; the numeric factorisation is multifrontal
//    (dense fronts, partial Cholesky, extend-add);
//  * for the device solve each supernode stores L_ss^{-1} (so the per-step TRSV becomes a
//    GEMV) and the panel L_{R_s,s}; both column-major.
// Also builds: irregular-d list (d DOFs touching an empty cell or carrying the point
// load), the c-element list (cut cells + uncut cells touching a c DOF) with their local
// c-index maps, and the CSR that gathers element products into r^c.
#include <omp.h>

#include <chrono>
#include <cstdio>

#include <algorithm>
#include <map>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <numeric>

#include "sc_internal.h"

namespace {

struct SNode {
  int comp;
  int c0 = 0, w = 0;
  std::vector<int> cols;      // ND indices are c0..c0+w-1; cols holds local node ids before numbering
  std::vector<int> R;         // sorted ND indices > c0+w-1
  std::vector<int> children;
  int parent = -1;
  int height = 0;
};

struct Builder {
  sc_ctx* c;
  int d, p, n1, nb;
  // c nodes in canonical (lattice) order
  std::vector<int64_t> clat;                 // canonical c index -> lattice
  std::vector<int> nd_of_canon;              // canonical -> ND
  std::vector<int> canon_of_nd;
  std::vector<int64_t> celem_cell;
  std::vector<int> celem_kidx;
  std::vector<int> celem_cidx;               // [e*nb+loc] canonical c index or -1 (converted to ND later)
  std::vector<int> node_eptr, node_eidx;     // canonical c node -> list of (e*nb+loc)
  std::vector<SNode> sn;
  std::vector<int> comp_roots;
  std::vector<int> comp_of;                  // canonical c -> component
};

inline void lat_ijk(const GridP& g, int64_t lat, int64_t* ijk) {
  for (int k = 0; k < 3; ++k) {
    if (k < g.dim) {
      ijk[k] = lat % g.nl[k];
      lat /= g.nl[k];
    } else {
      ijk[k] = 0;
    }
  }
}

inline int64_t cell_lin(const GridP& g, const int64_t* ci) {
  return ci[0] + (int64_t)g.N[0] * (ci[1] + (int64_t)(g.dim > 1 ? g.N[1] : 1) * ci[2]);
}

// lattice index of local node loc of cell (ci)
inline int64_t elem_node(const GridP& g, const int64_t* ci, int loc, int n1) {
  int64_t l[3] = {loc % n1, (loc / n1) % n1, loc / (n1 * n1)};
  int64_t lat = 0, stride = 1;
  for (int k = 0; k < g.dim; ++k) {
    lat += (ci[k] * g.p + l[k]) * stride;
    stride *= g.nl[k];
  }
  return lat;
}

struct UF {
  std::vector<int> p;
  explicit UF(int n) : p(n) { std::iota(p.begin(), p.end(), 0); }
  int f(int x) {
    while (p[x] != x) x = p[x] = p[p[x]];
    return x;
  }
  void u(int a, int b) {
    a = f(a);
    b = f(b);
    if (a != b) p[std::max(a, b)] = std::min(a, b);
  }
};

// ---------------------------------------------------------------- dense kernels
// Partial Cholesky of the (n x n, lower, column-major, ld) front on its first w columns,
// then the Schur update of the trailing (n-w) block.  Returns the failing column or -1.
// The dense host kernels are compiled twice (AVX2 and baseline x86-64, selected at load time
// by the CPU): their inner loops are independent element updates, so the vector versions give
// the same bits (no reassociation, no contraction: -ffp-contract=off).
#define SC_HOST_SIMD __attribute__((target_clones("avx2", "default")))
SC_HOST_SIMD int front_factor(double* F, int n, int w) {
  for (int j = 0; j < w; ++j) {
    double* Fj = F + (size_t)j * n;
    for (int k = 0; k < j; ++k) {
      const double* Fk = F + (size_t)k * n;
      const double f = Fk[j];
      if (f == 0.0) continue;
      for (int i = j; i < n; ++i) Fj[i] -= Fk[i] * f;
    }
    if (!(Fj[j] > 0.0) || !std::isfinite(Fj[j])) return j;
    const double dgn = std::sqrt(Fj[j]);
    const double inv = 1.0 / dgn;
    Fj[j] = dgn;
    for (int i = j + 1; i < n; ++i) Fj[i] *= inv;
  }
  // U = F22 - L21 L21^T (lower part), blocked over k for cache reuse
  const int r = n - w;
  const int KB = 64;
  for (int k0 = 0; k0 < w; k0 += KB) {
    const int k1 = std::min(w, k0 + KB);
    for (int jj = 0; jj < r; ++jj) {
      const int j = w + jj;
      double* Fj = F + (size_t)j * n;
      for (int k = k0; k < k1; ++k) {
        const double* Fk = F + (size_t)k * n;
        const double f = Fk[j];
        if (f == 0.0) continue;
        for (int i = j; i < n; ++i) Fj[i] -= Fk[i] * f;
      }
    }
  }
  return -1;
}

// inverse of the lower-triangular w x w block L (column-major, ld n) into X (w x w, col-major)
SC_HOST_SIMD void tri_inverse(const double* L, int n, int w, double* X) {
  std::fill(X, X + (size_t)w * w, 0.0);
  for (int col = 0; col < w; ++col) {
    double* x = X + (size_t)col * w;
    x[col] = 1.0 / L[(size_t)col * n + col];
    // forward substitution for rows > col: x_i = -(sum_{k=col}^{i-1} L_ik x_k) / L_ii
    for (int k = col; k < w; ++k) {
      if (k > col) x[k] /= L[(size_t)k * n + k];
      const double xk = x[k];
      const double* Lk = L + (size_t)k * n;
      for (int i = k + 1; i < w; ++i) x[i] -= Lk[i] * xk;
    }
    // note: x[k] for k>col accumulated -(sum) then divided above
  }
}

// Stacked device panel of one supernode from its factored front F (n x n, ld n, lower;
// columns 0..w-1 hold L_ss over L_Rs):  rows [0, w) = D_s = L_ss^{-T} L_ss^{-1} (full),
// rows [wp, wp + r) = G_s = L_Rs L_ss^{-1}, zero padding rows in between / below, with
// wp = w rounded up to even and ld = wp + (r rounded up to even) (panel_ld): every column
// segment the device copies with bulk (TMA) copies is then 16-byte aligned.  Column-major.
int panel_wp(int w) { return (w + 1) & ~1; }
int panel_ld(int w, int r) { return panel_wp(w) + ((r + 1) & ~1); }

SC_HOST_SIMD void make_panel(const double* F, int n, int w, double* P) {
  const int r = n - w, wp = panel_wp(w), ld = panel_ld(w, r);
  std::fill(P, P + (size_t)ld * w, 0.0);
  std::vector<double> X((size_t)w * w);
  tri_inverse(F, n, w, X.data());   // X = L_ss^{-1}, lower, column-major (ld w)
  for (int j = 0; j < w; ++j) {
    const double* xj = X.data() + (size_t)j * w;
    for (int i = j; i < w; ++i) {
      const double* xi = X.data() + (size_t)i * w;
      double s = 0.0;
      for (int k = i; k < w; ++k) s += xi[k] * xj[k];   // (X^T X)_{ij}, k >= max(i, j) = i
      P[(size_t)j * ld + i] = s;
      P[(size_t)i * ld + j] = s;
    }
  }
  for (int j = 0; j < w; ++j) {
    double* g = P + (size_t)j * ld + wp;
    const double* xj = X.data() + (size_t)j * w;
    for (int k = j; k < w; ++k) {
      const double f = xj[k];
      if (f == 0.0) continue;
      const double* lk = F + (size_t)k * n + w;   // column k of L_Rs
      for (int i = 0; i < r; ++i) g[i] += lk[i] * f;
    }
  }
}

}  // namespace

// Nested dissection of one component (local node ids into b.clat, canonical indices).
static void nested_dissection(Builder& b, int comp, std::vector<int>& nodes, std::vector<int>& roots,
                              int& next_col, std::vector<int>& order_out) {
  const GridP& g = b.c->g;
  static const int LEAF = sc_knob("SC_ND_LEAF") ? atoi(sc_knob("SC_ND_LEAF")) : 32;   // max nodes of an ND leaf (r1_solve_variants.txt)
  std::function<void(std::vector<int>&, std::vector<int>&)> rec = [&](std::vector<int>& nd,
                                                                      std::vector<int>& out_roots) {
    if (nd.empty()) return;
    int axis = -1;
    int64_t plane = 0;
    if ((int)nd.size() > LEAF) {
      int64_t lo[3] = {INT64_MAX, INT64_MAX, INT64_MAX}, hi[3] = {INT64_MIN, INT64_MIN, INT64_MIN};
      for (int v : nd) {
        int64_t ijk[3];
        lat_ijk(g, b.clat[v], ijk);
        for (int k = 0; k < g.dim; ++k) {
          lo[k] = std::min(lo[k], ijk[k]);
          hi[k] = std::max(hi[k], ijk[k]);
        }
      }
      // axes by decreasing extent; first with an interior element-boundary plane
      int ax[3] = {0, 1, 2};
      std::sort(ax, ax + g.dim, [&](int a1, int a2) { return hi[a1] - lo[a1] > hi[a2] - lo[a2]; });
      for (int t = 0; t < g.dim && axis < 0; ++t) {
        const int k = ax[t];
        // median coordinate
        std::vector<int64_t> cs;
        cs.reserve(nd.size());
        for (int v : nd) {
          int64_t ijk[3];
          lat_ijk(g, b.clat[v], ijk);
          cs.push_back(ijk[k]);
        }
        std::nth_element(cs.begin(), cs.begin() + cs.size() / 2, cs.end());
        const int64_t med = cs[cs.size() / 2];
        int64_t best = -1;
        int64_t bestd = INT64_MAX;
        for (int64_t m = (lo[k] / g.p) * g.p; m <= hi[k]; m += g.p) {
          if (m <= lo[k] || m >= hi[k]) continue;
          int64_t dd = std::llabs(m - med);
          if (dd < bestd) {
            bestd = dd;
            best = m;
          }
        }
        if (best >= 0) {
          axis = k;
          plane = best;
        }
      }
    }
    if (axis < 0) {
      SNode s;
      s.comp = comp;
      s.cols = nd;
      std::sort(s.cols.begin(), s.cols.end());
      s.c0 = next_col;
      s.w = (int)nd.size();
      for (int v : s.cols) order_out.push_back(v);
      next_col += s.w;
      b.sn.push_back(std::move(s));
      out_roots.push_back((int)b.sn.size() - 1);
      return;
    }
    std::vector<int> left, right, sep;
    for (int v : nd) {
      int64_t ijk[3];
      lat_ijk(g, b.clat[v], ijk);
      if (ijk[axis] < plane) left.push_back(v);
      else if (ijk[axis] > plane) right.push_back(v);
      else sep.push_back(v);
    }
    nd.clear();
    nd.shrink_to_fit();
    std::vector<int> sub;
    rec(left, sub);
    rec(right, sub);
    if (sep.empty()) {
      for (int r : sub) out_roots.push_back(r);
      return;
    }
    SNode s;
    s.comp = comp;
    s.cols = sep;
    std::sort(s.cols.begin(), s.cols.end());
    s.c0 = next_col;
    s.w = (int)sep.size();
    for (int v : s.cols) order_out.push_back(v);
    next_col += s.w;
    s.children = sub;
    b.sn.push_back(std::move(s));
    const int id = (int)b.sn.size() - 1;
    for (int ch : sub) b.sn[ch].parent = id;
    out_roots.push_back(id);
  };
  rec(nodes, roots);
}

// Basis functions of the lowest-index non-empty cell containing x at x (P:456-459 for the
// point load, reading C11): out = (lattice index, [alpha(x)] N_i(x)) for the nonzero N_i.
void point_weights(const sc_ctx* c, const double* x, bool with_alpha,
                   std::vector<std::pair<int64_t, double>>& out) {
  const GridP& g = c->g;
  const int n1 = g.p + 1, nb = c->nb;
  out.clear();
  int64_t cand[3][2];
  int nc[3] = {1, 1, 1};
  for (int k = 0; k < 3; ++k) {
    cand[k][0] = 0;
    if (k >= g.dim) continue;
    nc[k] = 0;
    for (int64_t e = 0; e < g.N[k]; ++e) {
      double lo = host_lattice(g.lo[k], g.hi[k], e, g.N[k]);
      double hi = host_lattice(g.lo[k], g.hi[k], e + 1, g.N[k]);
      if (lo <= x[k] && x[k] <= hi && nc[k] < 2) cand[k][nc[k]++] = e;
    }
    if (nc[k] == 0) throw ScError(SC_ERR_CONFIG, "point outside the grid");
  }
  // lowest linear index first: iterate z, y, x ascending
  for (int a2 = 0; a2 < nc[2]; ++a2)
    for (int a1 = 0; a1 < nc[1]; ++a1)
      for (int a0 = 0; a0 < nc[0]; ++a0) {
        int64_t ci[3] = {cand[0][a0], cand[1][a1], cand[2][a2]};
        int64_t cl = cell_lin(g, ci);
        if (c->cell_class[cl] == 2) continue;
        double xs[3] = {x[0], g.dim > 1 ? x[1] : 0.0, g.dim > 2 ? x[2] : 0.0};
        const double al = (!with_alpha || host_phys(c->voids, xs)) ? 1.0 : c->alpha;
        double v[3][SC_MAXP1];
        for (int k = 0; k < 3; ++k) {
          if (k < g.dim) {
            double lo = host_lattice(g.lo[k], g.hi[k], ci[k], g.N[k]);
            double hi = host_lattice(g.lo[k], g.hi[k], ci[k] + 1, g.N[k]);
            double xi = -1.0 + 2.0 * (xs[k] - lo) / (hi - lo);
            host_lagrange(c->gll_x, xi, v[k], nullptr);
          } else {
            for (int i = 0; i < n1; ++i) v[k][i] = (i == 0) ? 1.0 : 0.0;
          }
        }
        for (int loc = 0; loc < nb; ++loc) {
          int l0 = loc % n1, l1 = (loc / n1) % n1, l2 = loc / (n1 * n1);
          double val = al * v[0][l0] * v[1][l1] * v[2][l2];
          if (val != 0.0) out.push_back({elem_node(g, ci, loc, n1), val});
        }
        return;
      }
  throw ScError(SC_ERR_CONFIG, "point lies only in empty cells");
}

// Gaussian-bell load (source kind 2, Eq. eq:fx, P:444-448 Eq. eq:f):
// f_x,i = int alpha f_x N_i, f_x = amp exp(-|x - x_s|^2 / (2 sigma^2)), with (p+1)^d Gauss
// points per uncut cell (alpha = 1) and per spacetree leaf of a cut cell (the leaves the device
// built; pointwise alpha with the classifier's arithmetic, C17), accumulated in ascending cell
// order (deterministic).  Cells farther than 40 sigma from x_s contribute exact zeros
// (exp(-800) underflows) and are skipped.  out = (lattice index, value), ascending lattice.
void bell_weights(const sc_ctx* c, std::vector<std::pair<int64_t, double>>& out) {
  const GridP& g = c->g;
  const int d = g.dim, n1 = g.p + 1, nb = c->nb;
  const double sig = c->src_sigma, amp = c->src_amp;
  const double rcut = 40.0 * sig;
  std::vector<double> tq(n1);
  for (int i = 0; i < n1; ++i) tq[i] = (c->gau_x[i] + 1.0) * 0.5;
  std::map<int64_t, double> acc;
  std::vector<double> fe(nb);
  int64_t kcut = 0;   // running index into the ascending cut-cell list
  for (int64_t cl = 0; cl < c->n_cells; ++cl) {
    const int8_t cls = c->cell_class[cl];
    const bool is_cut = cls == 1;
    const int64_t my_cut = is_cut ? kcut++ : -1;
    if (cls == 2) continue;
    int64_t ci[3] = {cl % g.N[0], d > 1 ? (cl / g.N[0]) % g.N[1] : 0, d > 2 ? cl / ((int64_t)g.N[0] * g.N[1]) : 0};
    // distance of the cell box to x_s
    double dist2 = 0.0;
    for (int k = 0; k < d; ++k) {
      const double lo = host_lattice(g.lo[k], g.hi[k], ci[k], g.N[k]);
      const double hi = host_lattice(g.lo[k], g.hi[k], ci[k] + 1, g.N[k]);
      const double q = c->src_x[k] < lo ? lo - c->src_x[k] : (c->src_x[k] > hi ? c->src_x[k] - hi : 0.0);
      dist2 += q * q;
    }
    if (dist2 > rcut * rcut) continue;
    std::fill(fe.begin(), fe.end(), 0.0);
    // leaves: the whole cell (level 0) for an uncut cell
    std::vector<unsigned long long> one(1, 0ull);
    const std::vector<unsigned long long>& leaves = is_cut ? c->cut_leaves[my_cut] : one;
    for (unsigned long long lf : leaves) {
      const int l = (int)(lf >> 48);
      int a[3];
      for (int k = 0; k < 3; ++k) a[k] = (int)((lf >> (16 * k)) & 0xFFFF);
      double xlo[3] = {0, 0, 0}, span[3] = {0, 0, 0};
      for (int k = 0; k < d; ++k) {
        const int64_t den = (int64_t)g.N[k] * g.s << l;
        const int64_t m0 = ((int64_t)ci[k] * g.s << l) + (int64_t)a[k] * g.s;
        xlo[k] = host_lattice(g.lo[k], g.hi[k], m0, den);
        span[k] = host_lattice(g.lo[k], g.hi[k], m0 + g.s, den) - xlo[k];
      }
      const double sc = std::ldexp(1.0, -l);
      // basis values at the leaf's Gauss points per axis
      double v[3][SC_MAXP1][SC_MAXP1];
      for (int k = 0; k < 3; ++k)
        for (int q = 0; q < n1; ++q) {
          if (k < d) {
            const double xi = -1.0 + (2.0 * a[k] + 1.0 + c->gau_x[q]) * sc;
            host_lagrange(c->gll_x, xi, v[k][q], nullptr);
          } else {
            for (int i = 0; i < n1; ++i) v[k][q][i] = (q == 0 && i == 0) ? 1.0 : 0.0;
          }
        }
      const int nq1 = d > 1 ? n1 : 1, nq2 = d > 2 ? n1 : 1;
      for (int q2 = 0; q2 < nq2; ++q2)
        for (int q1 = 0; q1 < nq1; ++q1)
          for (int q0 = 0; q0 < n1; ++q0) {
            const int qq[3] = {q0, q1, q2};
            double x[3] = {0, 0, 0}, w = 1.0, r2 = 0.0;
            for (int k = 0; k < d; ++k) {
              x[k] = xlo[k] + span[k] * tq[qq[k]];
              w *= c->gau_w[qq[k]] * 0.5 * g.h[k] * sc;
              const double dx = x[k] - c->src_x[k];
              r2 += dx * dx;
            }
            const double al = (!is_cut || host_phys(c->voids, x)) ? 1.0 : c->alpha;
            const double f = al * w * amp * std::exp(-r2 / (2.0 * sig * sig));
            if (f == 0.0) continue;
            for (int loc = 0; loc < nb; ++loc) {
              const int l0 = loc % n1, l1 = (loc / n1) % n1, l2 = loc / (n1 * n1);
              fe[loc] += f * v[0][q0][l0] * (d > 1 ? v[1][q1][l1] : 1.0) * (d > 2 ? v[2][q2][l2] : 1.0);
            }
          }
    }
    for (int loc = 0; loc < nb; ++loc)
      if (fe[loc] != 0.0) acc[elem_node(g, ci, loc, n1)] += fe[loc];
  }
  out.assign(acc.begin(), acc.end());
}

void setup_factor(sc_ctx* c, const std::vector<double>& /*unused*/) {
  // SC_SETUP_TIMES (diagnostics): phase times on stderr
  auto flap = [tl = std::chrono::steady_clock::now()](const char* what) mutable {
    const auto now = std::chrono::steady_clock::now();
    if (getenv("SC_SETUP_TIMES"))
      fprintf(stderr, "sc_setup   factor: %-34s %8.3f s\n", what, std::chrono::duration<double>(now - tl).count());
    tl = now;
  };
  Builder b;
  b.c = c;
  const GridP& g = c->g;
  b.d = g.dim;
  b.p = g.p;
  b.n1 = g.p + 1;
  b.nb = c->nb;
  const int nb = c->nb, n1 = b.n1;
  // ---------------- source, DOF lists, irregular nodes
  std::vector<std::pair<int64_t, double>> src;  // (lattice, f_x value), ascending lattice
  if (c->src_kind == 1) {
    point_weights(c, c->src_x, true, src);
    for (auto& sv : src)
      if (c->ntype[sv.first] == 1) c->ntype[sv.first] = 2;  // point-load d nodes -> irregular path
    std::sort(src.begin(), src.end());
  } else if (c->src_kind == 2) {
    bell_weights(c, src);   // tensor-d nodes keep the tensor kernel; their load is added after it
  }
  // integrator 2 (trapezoidal Newmark on all DOFs): every DOF is treated implicitly
  if (c->integrator == 2)
    for (int64_t L = 0; L < c->n_lat; ++L)
      if (c->ntype[L] == 1 || c->ntype[L] == 2 || c->ntype[L] == 4) c->ntype[L] = 3;
  c->dof_lat.clear();
  c->n_d = c->n_c = c->n_irr = 0;
  {
    int64_t nd = 0, ncc = 0;
#pragma omp parallel for reduction(+ : nd, ncc)
    for (int64_t i = 0; i < c->n_lat; ++i) {
      nd += c->ntype[i] != 0;
      ncc += c->ntype[i] == 3;
    }
    c->dof_lat.reserve((size_t)nd);
    b.clat.reserve((size_t)ncc);
  }
  for (int64_t i = 0; i < c->n_lat; ++i) {
    const uint8_t t = c->ntype[i];
    if (!t) continue;
    c->dof_lat.push_back(i);
    if (t == 3) {
      b.clat.push_back(i);
      ++c->n_c;
    } else {
      ++c->n_d;
      if (t == 2) ++c->n_irr;
    }
  }
  c->n_dof = (int64_t)c->dof_lat.size();
  // irregular d nodes: lattice index, 1/M_i (lumped, non-empty incident cells), f_x
  // (uploaded after the partition plan: each rank keeps the ones it updates)
  std::vector<int32_t> ilat;
  std::vector<double> iinv, ifx;
  {
    std::vector<std::pair<int64_t, double>> srcs = src;
    std::sort(srcs.begin(), srcs.end());
    for (int64_t i = 0; i < c->n_lat; ++i) {
      if (c->ntype[i] != 2) continue;
      int64_t ijk[3];
      lat_ijk(g, i, ijk);
      int64_t e0[3], e1[3];
      for (int k = 0; k < 3; ++k) {
        if (k < g.dim) {
          if (ijk[k] % g.p == 0) {
            e0[k] = ijk[k] / g.p - 1;
            e1[k] = ijk[k] / g.p;
          } else {
            e0[k] = e1[k] = ijk[k] / g.p;
          }
          if (e0[k] < 0) e0[k] = e1[k];
          if (e1[k] >= g.N[k]) e1[k] = e0[k];
        } else {
          e0[k] = e1[k] = 0;
        }
      }
      double m = 0.0;
      for (int64_t a2 = e0[2]; a2 <= e1[2]; ++a2)
        for (int64_t a1 = e0[1]; a1 <= e1[1]; ++a1)
          for (int64_t a0 = e0[0]; a0 <= e1[0]; ++a0) {
            int64_t ci[3] = {a0, a1, a2};
            if (c->cell_class[cell_lin(g, ci)] == 2) continue;
            double mm = c->rho;
            for (int k = 0; k < g.dim; ++k) mm *= 0.5 * g.h[k] * c->gll_w[ijk[k] - ci[k] * g.p];
            m += mm;
          }
      ilat.push_back((int32_t)i);
      iinv.push_back(1.0 / m);
      auto it = std::lower_bound(srcs.begin(), srcs.end(), i,
                                 [](const std::pair<int64_t, double>& a, int64_t v) { return a.first < v; });
      ifx.push_back((it != srcs.end() && it->first == i) ? it->second : 0.0);
    }
  }
  int nc = (int)c->n_c;
  int ne = 0;
  std::vector<int> comp_id;
  std::vector<std::vector<int>> comps;
  // canonical c index of a lattice node (binary search in clat)
  auto cidx_of = [&](int64_t lat) -> int {
    auto it = std::lower_bound(b.clat.begin(), b.clat.end(), lat);
    return (it != b.clat.end() && *it == lat) ? (int)(it - b.clat.begin()) : -1;
  };
  // c elements, node -> element lists and components of the current c set b.clat
  auto build_c = [&](bool first) {
    // ---------------- c elements: cut cells + uncut cells with >= 1 c node
    std::vector<uint8_t> mark;
    {
      std::vector<int64_t> cells;
      for (int64_t lat : b.clat) {
        int64_t ijk[3];
        lat_ijk(g, lat, ijk);
        int64_t e0[3], e1[3];
        for (int k = 0; k < 3; ++k) {
          if (k < g.dim) {
            if (ijk[k] % g.p == 0) {
              e0[k] = ijk[k] / g.p - 1;
              e1[k] = ijk[k] / g.p;
            } else {
              e0[k] = e1[k] = ijk[k] / g.p;
            }
            if (e0[k] < 0) e0[k] = e1[k];
            if (e1[k] >= g.N[k]) e1[k] = e0[k];
          } else {
            e0[k] = e1[k] = 0;
          }
        }
        for (int64_t a2 = e0[2]; a2 <= e1[2]; ++a2)
          for (int64_t a1 = e0[1]; a1 <= e1[1]; ++a1)
            for (int64_t a0 = e0[0]; a0 <= e1[0]; ++a0) {
              int64_t ci[3] = {a0, a1, a2};
              int64_t cl = cell_lin(g, ci);
              if (c->cell_class[cl] != 2) cells.push_back(cl);
            }
      }
      std::sort(cells.begin(), cells.end());
      cells.erase(std::unique(cells.begin(), cells.end()), cells.end());
      b.celem_cell = cells;
    }
    ne = (int)b.celem_cell.size();
    c->n_celem = ne;
    b.celem_kidx.assign(ne, -1);
    b.celem_cidx.assign((size_t)ne * nb, -1);
    for (int e = 0; e < ne; ++e) {
      const int64_t cl = b.celem_cell[e];
      if (c->cell_class[cl] == 1) {
        auto it = std::lower_bound(c->cut_cells.begin(), c->cut_cells.end(), (long long)cl);
        b.celem_kidx[e] = (int)(it - c->cut_cells.begin());
      }
      int64_t ci[3];
      int64_t t = cl;
      for (int k = 0; k < 3; ++k) {
        if (k < g.dim) {
          ci[k] = t % g.N[k];
          t /= g.N[k];
        } else {
          ci[k] = 0;
        }
      }
      for (int loc = 0; loc < nb; ++loc) b.celem_cidx[(size_t)e * nb + loc] = cidx_of(elem_node(g, ci, loc, n1));
    }
    // near-d nodes (type 4): tensor-d nodes of uncut c elements, i.e. d nodes whose residual
    // reads a c value; the step pipeline updates them after the c part (step.cu)
    if (first) c->n_near = 0;
    for (int e = 0; e < ne && first; ++e) {
      if (b.celem_kidx[e] >= 0) continue;   // cut cell: all its nodes are c
      int64_t ci[3];
      int64_t t = b.celem_cell[e];
      for (int k = 0; k < 3; ++k) {
        if (k < g.dim) {
          ci[k] = t % g.N[k];
          t /= g.N[k];
        } else {
          ci[k] = 0;
        }
      }
      for (int loc = 0; loc < nb; ++loc) {
        const int64_t L = elem_node(g, ci, loc, n1);
        if (c->ntype[L] == 1) {
          c->ntype[L] = 4;
          ++c->n_near;
        }
      }
    }
    // node -> (e, loc) lists, canonical order
    b.node_eptr.assign(nc + 1, 0);
    for (size_t q = 0; q < b.celem_cidx.size(); ++q)
      if (b.celem_cidx[q] >= 0) ++b.node_eptr[b.celem_cidx[q] + 1];
    for (int i = 0; i < nc; ++i) b.node_eptr[i + 1] += b.node_eptr[i];
    b.node_eidx.resize(b.node_eptr[nc]);
    {
      std::vector<int> fill(b.node_eptr.begin(), b.node_eptr.end() - 1);
      for (size_t q = 0; q < b.celem_cidx.size(); ++q)
        if (b.celem_cidx[q] >= 0) b.node_eidx[fill[b.celem_cidx[q]]++] = (int)q;
    }
    // ---------------- components (union-find over c elements)
    UF uf(std::max(nc, 1));
    for (int e = 0; e < ne; ++e) {
      int first = -1;
      for (int loc = 0; loc < nb; ++loc) {
        int ci = b.celem_cidx[(size_t)e * nb + loc];
        if (ci < 0) continue;
        if (first < 0) first = ci;
        else uf.u(first, ci);
      }
    }
    comp_id.assign(nc, -1);
    comps.clear();
    for (int i = 0; i < nc; ++i) {
      int r = uf.f(i);
      if (comp_id[r] < 0) {
        comp_id[r] = (int)comps.size();
        comps.emplace_back();
      }
      comps[comp_id[r]].push_back(i);
    }
  };
  build_c(true);
  flap("DOF lists, c elements, components");
  // ---------------- partition plan (world > 1; partition.cpp): component owners, regions
  const std::vector<int64_t> clat_global = b.clat;
  std::vector<int> c_owner(nc, 0);
  {
    const int ax = g.dim - 1;
    int64_t plane = 1, per_layer = 1;
    for (int k = 0; k < ax; ++k) {
      plane *= g.nl[k];
      per_layer *= g.N[k];
    }
    std::vector<CompSpan> spans(comps.size());
    for (size_t k = 0; k < comps.size(); ++k) {
      CompSpan sp{INT32_MAX, -1, 0, 0.0};
      double zsum = 0.0;
      for (int v : comps[k]) {
        zsum += (double)(b.clat[v] / plane);
        for (int q = b.node_eptr[v]; q < b.node_eptr[v + 1]; ++q) {
          const int L = (int)(b.celem_cell[b.node_eidx[q] / nb] / per_layer);
          sp.lmin = std::min(sp.lmin, L);
          sp.lmax = std::max(sp.lmax, L);
        }
      }
      sp.centroid = (int)(zsum / (double)comps[k].size() / g.p);
      sp.cost = 4500.0 * (double)comps[k].size();   // ~2 sweeps x ~280 panel entries per c DOF
      spans[k] = sp;
    }
    std::vector<int> owner;
    plan_partition(c, spans, owner);
    for (size_t k = 0; k < comps.size(); ++k)
      for (int v : comps[k]) c_owner[v] = owner[k];
    c->n_components = (int64_t)comps.size();
    // node types this rank updates: d nodes of planes whose incident elements lie in its region
    c->ntype_rank = c->ntype;
    if (c->world > 1)
      for (int64_t L = 0; L < c->n_lat; ++L) {
        const uint8_t t = c->ntype[L];
        if ((t == 1 || t == 2 || t == 4) && !region_computes_plane(c, c->rank, L / plane)) c->ntype_rank[L] = 0;
      }
    SC_CUDA(cudaMemcpy(c->d_ntype, c->ntype_rank.data(), c->n_lat, cudaMemcpyHostToDevice));
    // irregular d nodes this rank updates
    std::vector<int32_t> il;
    std::vector<double> im, ifv;
    for (size_t i = 0; i < ilat.size(); ++i)
      if (c->ntype_rank[ilat[i]] == 2) {
        il.push_back(ilat[i]);
        im.push_back(iinv[i]);
        ifv.push_back(ifx[i]);
      }
    c->n_irr = (int64_t)il.size();
    // tensor-d nodes this rank updates that carry a distributed load: f_x / M_ii with the
    // lumped mass rho prod_k (h_k/2) wt_k (the mass the explicit kernel divides by)
    {
      std::vector<int32_t> ll;
      std::vector<double> lf;
      for (auto& sv : src) {
        const uint8_t t = c->ntype_rank[sv.first];
        if (t != 1 && t != 4) continue;
        int64_t ijk[3];
        lat_ijk(g, sv.first, ijk);
        double m = c->rho;
        for (int k = 0; k < g.dim; ++k) {
          const int64_t l = ijk[k] % g.p, e = ijk[k] / g.p;
          const double wt = l ? c->gll_w[l] : ((e > 0 ? c->gll_w[g.p] : 0.0) + (e < g.N[k] ? c->gll_w[0] : 0.0));
          m *= 0.5 * g.h[k] * wt;
        }
        ll.push_back((int32_t)sv.first);
        lf.push_back(sv.second / m);
      }
      c->n_load = (int64_t)ll.size();
      if (c->n_load) {
        SC_CUDA(cudaMalloc(&c->d_load_lat, sizeof(int32_t) * c->n_load));
        SC_CUDA(cudaMalloc(&c->d_load_fxm, sizeof(double) * c->n_load));
        SC_CUDA(cudaMemcpy(c->d_load_lat, ll.data(), sizeof(int32_t) * c->n_load, cudaMemcpyHostToDevice));
        SC_CUDA(cudaMemcpy(c->d_load_fxm, lf.data(), sizeof(double) * c->n_load, cudaMemcpyHostToDevice));
      }
    }
    if (c->n_irr) {
      SC_CUDA(cudaMalloc(&c->d_irr_lat, sizeof(int32_t) * c->n_irr));
      SC_CUDA(cudaMalloc(&c->d_irr_invm, sizeof(double) * c->n_irr));
      SC_CUDA(cudaMalloc(&c->d_irr_fx, sizeof(double) * c->n_irr));
      SC_CUDA(cudaMemcpy(c->d_irr_lat, il.data(), sizeof(int32_t) * c->n_irr, cudaMemcpyHostToDevice));
      SC_CUDA(cudaMemcpy(c->d_irr_invm, im.data(), sizeof(double) * c->n_irr, cudaMemcpyHostToDevice));
      SC_CUDA(cudaMemcpy(c->d_irr_fx, ifv.data(), sizeof(double) * c->n_irr, cudaMemcpyHostToDevice));
    }
  }
  // this rank's c set: the c nodes of its own components (all of them when world == 1)
  std::vector<int> glob_of_own;   // own canonical index -> global canonical c index
  if (c->world > 1) {
    std::vector<int64_t> own;
    for (int i = 0; i < nc; ++i)
      if (c_owner[i] == c->rank) {
        own.push_back(clat_global[i]);
        glob_of_own.push_back(i);
      }
    b.clat = own;
    nc = (int)own.size();
    build_c(false);
  } else {
    glob_of_own.resize(nc);
    std::iota(glob_of_own.begin(), glob_of_own.end(), 0);
  }
  c->n_cl = nc;

  flap("partition plan");
  // ---------------- nested dissection -> ND order and supernodes
  std::vector<int> order;  // ND index -> canonical
  order.reserve(nc);
  int next_col = 0;
  for (int k = 0; k < (int)comps.size(); ++k) {
    std::vector<int> roots;
    nested_dissection(b, k, comps[k], roots, next_col, order);
  }
  b.canon_of_nd = order;
  b.nd_of_canon.assign(nc, -1);
  for (int i = 0; i < nc; ++i) b.nd_of_canon[order[i]] = i;
  c->c_lat.resize(nc);
  c->c_canon.resize(nc);
  for (int i = 0; i < nc; ++i) {
    c->c_lat[i] = b.clat[order[i]];
    c->c_canon[i] = glob_of_own[order[i]];
  }
  // convert element maps to ND indices
  for (auto& v : b.celem_cidx)
    if (v >= 0) v = b.nd_of_canon[v];
  flap("nested dissection");
  // ---------------- symbolic: R_s = (adj(cols) U struct(children)) above the supernode
  const int nsn = (int)b.sn.size();
  std::vector<int> sn_of(nc);
  for (int s = 0; s < nsn; ++s)
    for (int j = 0; j < b.sn[s].w; ++j) sn_of[b.sn[s].c0 + j] = s;
  // supernodes of each component form a contiguous postorder range; components are
  // independent, so the symbolic and numeric phases run one component per OpenMP task
  std::vector<std::vector<int>> comp_sn(comps.size());
  for (int s = 0; s < nsn; ++s) comp_sn[b.sn[s].comp].push_back(s);
#pragma omp parallel
  {
    std::vector<int> stamp(std::max(ne, 1), -1);   // element already scanned for supernode s
#pragma omp for schedule(dynamic, 1)
    for (int k = 0; k < (int)comps.size(); ++k) {
      for (int s : comp_sn[k]) {  // postorder: children first
        SNode& S = b.sn[s];
        const int last = S.c0 + S.w - 1;
        std::vector<int> R;
        for (int v : S.cols) {  // canonical ids
          for (int q = b.node_eptr[v]; q < b.node_eptr[v + 1]; ++q) {
            const int e = b.node_eidx[q] / nb;
            if (stamp[e] == s) continue;
            stamp[e] = s;
            for (int loc = 0; loc < nb; ++loc) {
              int j = b.celem_cidx[(size_t)e * nb + loc];
              if (j > last) R.push_back(j);
            }
          }
        }
        for (int ch : S.children)
          for (int j : b.sn[ch].R)
            if (j > last) R.push_back(j);
        std::sort(R.begin(), R.end());
        R.erase(std::unique(R.begin(), R.end()), R.end());
        S.R = std::move(R);
        int h = 0;
        for (int ch : S.children) h = std::max(h, b.sn[ch].height + 1);
        S.height = h;
      }
    }
  }
  flap("symbolic");
  // ---------------- numeric multifrontal factorisation of S and M^cc
  const double beta_dt2 = 0.25 * c->dt * c->dt;
  // symmetric Jacobi scaling D A D (unit diagonal): the fictitious-region rows of S are
  // ~1/alpha smaller than the physical ones; scaling keeps L_ss^{-1} well conditioned so
  // the inverse-based device sweeps stay as accurate as substitution.
  std::vector<double> dS(nc, 0.0), dM(nc, 0.0);
  for (int e = 0; e < ne; ++e) {
    const int kidx = b.celem_kidx[e];
    for (int l = 0; l < nb; ++l) {
      const int i = b.celem_cidx[(size_t)e * nb + l];
      if (i < 0) continue;
      const double m = kidx >= 0 ? c->Mcut_host[(size_t)kidx * nb * nb + (size_t)l * nb + l] : c->Mref[l];
      const double k = kidx >= 0 ? c->Kcut_host[(size_t)kidx * nb * nb + (size_t)l * nb + l]
                                 : c->Kref[(size_t)l * nb + l];
      dS[i] += m + beta_dt2 * k;
      dM[i] += m;
    }
  }
  // CDM with HRZ-lumped cut cells (integrator 1): the c DOFs are explicit
  // with the diagonal mass sum_e M~_ii, M~_ii = m_e / (sum_k M_kk) M_ii on cut cells
  if (c->integrator == 1) {
    std::vector<double> mc(nc, 0.0);
    for (int e = 0; e < ne; ++e) {
      const int kidx = b.celem_kidx[e];
      double scale = 1.0;
      if (kidx >= 0) {
        const double* Me = &c->Mcut_host[(size_t)kidx * nb * nb];
        double tot = 0.0, dia = 0.0;
        for (size_t q = 0; q < (size_t)nb * nb; ++q) tot += Me[q];
        for (int l = 0; l < nb; ++l) dia += Me[(size_t)l * nb + l];
        scale = tot / dia;
      }
      for (int l = 0; l < nb; ++l) {
        const int i = b.celem_cidx[(size_t)e * nb + l];
        if (i < 0) continue;
        mc[i] += kidx >= 0 ? scale * c->Mcut_host[(size_t)kidx * nb * nb + (size_t)l * nb + l] : c->Mref[l];
      }
    }
    for (int i = 0; i < nc; ++i)
      if (!(mc[i] > 0.0)) throw ScError(SC_ERR_NUMERIC, "non-positive HRZ mass at c DOF " + std::to_string(i));
    SC_CUDA(cudaMalloc(&c->d_mc, sizeof(double) * std::max(1, nc)));
    SC_CUDA(cudaMemcpy(c->d_mc, mc.data(), sizeof(double) * nc, cudaMemcpyHostToDevice));
  }
  for (int i = 0; i < nc; ++i) {
    if (!(dS[i] > 0.0) || !(dM[i] > 0.0))
      throw ScError(SC_ERR_NUMERIC, "non-positive diagonal of S or M^cc at c DOF " + std::to_string(i));
    dS[i] = 1.0 / std::sqrt(dS[i]);
    dM[i] = 1.0 / std::sqrt(dM[i]);
  }
  std::vector<int64_t> a_off(nsn + 1, 0);
  for (int s = 0; s < nsn; ++s)
    a_off[s + 1] = a_off[s] + (int64_t)b.sn[s].w * panel_ld(b.sn[s].w, (int)b.sn[s].R.size());
  c->nnz_factor = 0;
  c->nnz_G = 0;
  c->sum_r = 0;
  for (int s = 0; s < nsn; ++s) {
    c->nnz_factor += (int64_t)b.sn[s].w * (b.sn[s].w + (int64_t)b.sn[s].R.size());
    c->nnz_G += (int64_t)b.sn[s].w * (int64_t)b.sn[s].R.size();
    c->sum_r += (int64_t)b.sn[s].R.size();
  }
  std::vector<double> hAS(a_off[nsn]), hAM(a_off[nsn]);
  int fail_comp = -1, fail_row = -1, fail_which = 0;
  const double* Kref = c->Kref.data();
  const double* Mref = c->Mref.data();
  // (no factor for the explicit HRZ integrator: the panels stay zero and the solve never runs)
  const int n_fact = c->integrator == 1 ? 0 : (int)comps.size();
  // tasks (component, matrix) in decreasing order of their dense work (sum of front sizes
  // cubed): the two factorisations of a component are independent, and the largest
  // components start first (they bound the wall time)
  std::vector<std::pair<double, int>> tasks;
  for (int k = 0; k < n_fact; ++k) {
    double cost = 0.0;
    for (int sn : comp_sn[k]) {
      const double nn = (double)b.sn[sn].w + (double)b.sn[sn].R.size();
      cost += nn * nn * nn;
    }
    tasks.push_back({cost, 2 * k});
    tasks.push_back({cost, 2 * k + 1});
  }
  std::stable_sort(tasks.begin(), tasks.end(), [](const std::pair<double, int>& a, const std::pair<double, int>& b) {
    return a.first > b.first;
  });
#pragma omp parallel for schedule(dynamic, 1)
  for (int tk = 0; tk < (int)tasks.size(); ++tk) {
    const int k = tasks[tk].second / 2;
    {
      const int which = tasks[tk].second % 2;     // 0: S, 1: M^cc
      std::vector<std::vector<double>> upd(nsn);  // update matrices (sparse by sn id; only this comp used)
      for (int s : comp_sn[k]) {
        const SNode& S = b.sn[s];
        const int w = S.w, r = (int)S.R.size(), n = w + r;
        std::vector<double> F((size_t)n * n, 0.0);
        auto pos = [&](int j) -> int {
          if (j >= S.c0 && j < S.c0 + w) return j - S.c0;
          auto it = std::lower_bound(S.R.begin(), S.R.end(), j);
          return w + (int)(it - S.R.begin());
        };
        // original entries of columns C_s
        for (int jj = 0; jj < w; ++jj) {
          const int jnd = S.c0 + jj;
          const int v = b.canon_of_nd[jnd];
          for (int q = b.node_eptr[v]; q < b.node_eptr[v + 1]; ++q) {
            const int e = b.node_eidx[q] / nb, lj = b.node_eidx[q] % nb;
            const int kidx = b.celem_kidx[e];
            const double* Ke = kidx >= 0 ? &c->Kcut_host[(size_t)kidx * nb * nb] : Kref;
            const double* Me = kidx >= 0 ? &c->Mcut_host[(size_t)kidx * nb * nb] : nullptr;
            for (int li = 0; li < nb; ++li) {
              const int i = b.celem_cidx[(size_t)e * nb + li];
              if (i < jnd) continue;
              double m = Me ? Me[(size_t)li * nb + lj] : (li == lj ? Mref[li] : 0.0);
              double val = which == 0 ? m + beta_dt2 * Ke[(size_t)li * nb + lj] : m;
              const std::vector<double>& dd = which == 0 ? dS : dM;
              F[(size_t)jj * n + pos(i)] += val * dd[i] * dd[jnd];
            }
          }
        }
        // extend-add of the children's update matrices
        for (int ch : S.children) {
          const SNode& C = b.sn[ch];
          const int rc = (int)C.R.size();
          std::vector<int> pm(rc);
          for (int a = 0; a < rc; ++a) pm[a] = pos(C.R[a]);
          const std::vector<double>& U = upd[ch];
          for (int bb = 0; bb < rc; ++bb)
            for (int a = bb; a < rc; ++a) F[(size_t)pm[bb] * n + pm[a]] += U[(size_t)bb * rc + a];
          upd[ch].clear();
          upd[ch].shrink_to_fit();
        }
        const int bad = front_factor(F.data(), n, w);
        if (bad >= 0) {
#pragma omp critical
          {
            fail_comp = k;
            fail_row = S.c0 + bad;
            fail_which = which;
          }
          break;
        }
        make_panel(F.data(), n, w, (which == 0 ? hAS.data() : hAM.data()) + a_off[s]);
        std::vector<double> U((size_t)r * r);
        for (int j = 0; j < r; ++j)
          for (int i = j; i < r; ++i) U[(size_t)j * r + i] = F[(size_t)(w + j) * n + w + i];
        upd[s] = std::move(U);
      }
    }
  }
  if (fail_comp >= 0)
    throw ScError(SC_ERR_NUMERIC, std::string("non-positive pivot in the factorisation of ") +
                                      (fail_which == 0 ? "S" : "M^cc") + " (component " +
                                      std::to_string(fail_comp) + ", row " + std::to_string(fail_row) + ")");
  flap("numeric");
  // ---------------- device structures
  c->n_sn = nsn;
  int H = 0;
  for (auto& S : b.sn) H = std::max(H, S.height);
  c->height = nsn ? H + 1 : 0;
  std::vector<int32_t> c0(nsn), wv(nsn), rv(nsn), roff(nsn + 1, 0), uoff(nsn + 1, 0), goff(nsn + 1, 0);
  std::vector<int64_t> ao(nsn);
  for (int s = 0; s < nsn; ++s) {
    c0[s] = b.sn[s].c0;
    wv[s] = b.sn[s].w;
    rv[s] = (int)b.sn[s].R.size();
    ao[s] = a_off[s];
    roff[s + 1] = roff[s] + rv[s];
    uoff[s + 1] = uoff[s] + rv[s];
    goff[s + 1] = goff[s] + wv[s] + rv[s];
    if (wv[s] > 4096) throw ScError(SC_ERR_CONFIG, "supernode wider than 4096 columns");
    c->max_w = std::max(c->max_w, wv[s]);
  }
  std::vector<int32_t> Rall(roff[nsn]);
  for (int s = 0; s < nsn; ++s) std::copy(b.sn[s].R.begin(), b.sn[s].R.end(), Rall.begin() + roff[s]);
  // front gather lists: position t of supernode s <- update entries of its children
  std::vector<std::vector<int32_t>> gl((size_t)goff[nsn]);
  for (int s = 0; s < nsn; ++s) {
    const SNode& S = b.sn[s];
    for (int ch : S.children) {
      const SNode& C = b.sn[ch];
      for (int a = 0; a < (int)C.R.size(); ++a) {
        const int j = C.R[a];
        int pos;
        if (j >= S.c0 && j < S.c0 + S.w) pos = j - S.c0;
        else pos = S.w + (int)(std::lower_bound(S.R.begin(), S.R.end(), j) - S.R.begin());
        gl[goff[s] + pos].push_back(uoff[ch] + a);
      }
    }
  }
  std::vector<int32_t> gptr(goff[nsn] + 1, 0), gidx;
  for (int32_t t = 0; t < goff[nsn]; ++t) {
    gptr[t + 1] = gptr[t] + (int32_t)gl[t].size();
    gidx.insert(gidx.end(), gl[t].begin(), gl[t].end());
  }
  // the same lists with the (usual) <= 2 entries inline: (i0, i1), -1 = none; longer lists
  // are flagged (-2 - first CSR position) and read through gptr/gidx
  std::vector<int32_t> g2(2 * (size_t)goff[nsn], -1);
  for (int32_t t = 0; t < goff[nsn]; ++t) {
    if (gl[t].size() > 2) {
      g2[2 * (size_t)t] = -2 - gptr[t];
    } else {
      if (gl[t].size() > 0) g2[2 * (size_t)t] = gl[t][0];
      if (gl[t].size() > 1) g2[2 * (size_t)t + 1] = gl[t][1];
    }
  }
  // persistent-solve work list (solve.cu).  Items of a phase cover the supernode's panel in
  // tiles that fill one staging buffer of `stage` doubles (SOLVE_STAGE = 32 KB: 5 CTAs per
  // SM; measured 8 K / 16 K doubles slower on configs 4 and 5 — fewer resident CTAs):
  //  forward  F: panel rows [r0, r0 + nr) x columns [c0, c0 + nc); C = min(w, SOLVE_TILE)
  //              columns per tile, R = 32 * 2^k rows (as many as fit, >= 32)
  //  backward B: G_s columns [c0, c0 + nc) (nc <= 32) x G_s rows [r0, r0 + nr), rows as
  //              many as fit (<= SOLVE_BROWS)
  // A tile group (same rows for F / same columns for B) whose reduction spans ntb > 1 tiles
  // writes partials (slot pslot, ticket bctr).  Per item 20 int32 (everything the item
  // needs, one load): (type, s, t, ntb) (pslot, bctr, r0, nr) (col0, nc, dof0, w)
  // (r, goff, uoff, roff) (aoff lo, aoff hi, ld, wp).
  const int TILE = SOLVE_TILE;
  int stage = SOLVE_STAGE;
  if (const char* v = sc_knob("SC_SOLVE_STAGE")) stage = std::max(1024, std::min(4 * SOLVE_STAGE, atoi(v)));
  c->solve_stage = stage;
  std::vector<int32_t> items;
  std::vector<int32_t> nblk(2 * (size_t)nsn, 0);
  std::vector<std::vector<int>> by_h(c->height);
  for (int s = 0; s < nsn; ++s) by_h[b.sn[s].height].push_back(s);
  int64_t pslot = 0;
  int n_bctr = 0;
  auto group = [&](int ph, int s, int ntb, int outs, auto&& geom) {   // one output group
    for (int t = 0; t < ntb; ++t) {
      int r0, nr, c0_, nc;
      geom(t, r0, nr, c0_, nc);
      const int64_t ao = a_off[s];
      items.insert(items.end(), {ph, s, t, ntb, (int32_t)pslot, ntb > 1 ? n_bctr : 0, r0, nr, c0_, nc,
                                 c0[s], wv[s], rv[s], goff[s], uoff[s], roff[s], (int32_t)(ao & 0xffffffff),
                                 (int32_t)(ao >> 32), panel_ld(wv[s], rv[s]), panel_wp(wv[s])});
    }
    if (ntb > 1) {
      if (pslot + (int64_t)ntb * outs > INT32_MAX) throw ScError(SC_ERR_CONFIG, "solve partial buffer too large");
      pslot += (int64_t)ntb * outs;
      ++n_bctr;
    }
    ++nblk[(size_t)ph * nsn + s];
  };
  auto fwd_items = [&](int s) {
    const int w = wv[s], ld = panel_ld(w, rv[s]);
    const int C = std::min({w, TILE, stage / 32});
    int R = 32;
    while (2 * R * C <= stage && R < ((ld + 31) / 32) * 32) R *= 2;
    const int ntb = (w + C - 1) / C;
    for (int r0 = 0; r0 < ld; r0 += R)
      group(0, s, ntb, R, [&](int t, int& rr, int& nr, int& cc, int& nc) {
        rr = r0;
        nr = std::min(R, ld - r0);
        cc = t * C;
        nc = std::min(C, w - t * C);
      });
  };
  auto bwd_items = [&](int s) {
    const int w = wv[s], rp = (rv[s] + 1) & ~1;
    const int NC = std::min(32, w);
    int RR = std::min(SOLVE_BROWS, (stage / NC) & ~1);
    RR = std::max(2, std::min(RR, std::max(rp, 2)));
    const int ntb = std::max(1, (rp + RR - 1) / RR);
    for (int o0 = 0; o0 < w; o0 += 32)
      group(1, s, ntb, 32, [&](int t, int& rr, int& nr, int& cc, int& nc) {
        rr = t * RR;
        nr = std::max(0, std::min(RR, rp - t * RR));
        cc = o0;
        nc = std::min(32, w - o0);
      });
  };
  // items of one phase of one supernode are contiguous: [item_first, item_first + item_cnt)
  std::vector<int32_t> item_first(2 * (size_t)nsn, 0), item_cnt(2 * (size_t)nsn, 0);
  for (int h = 0; h < c->height; ++h)
    for (int s : by_h[h]) {
      item_first[s] = (int32_t)(items.size() / 20);
      fwd_items(s);
      item_cnt[s] = (int32_t)(items.size() / 20) - item_first[s];
    }
  for (int h = c->height - 1; h >= 0; --h)
    for (int s : by_h[h]) {
      item_first[nsn + s] = (int32_t)(items.size() / 20);
      bwd_items(s);
      item_cnt[nsn + s] = (int32_t)(items.size() / 20) - item_first[nsn + s];
    }
  c->n_items = (int)(items.size() / 20);
  // ready-queue metadata (solve.cu): the forward items of the leaves are ready at launch;
  // every other phase is pushed by the CTA that completes its last dependency
  std::vector<int32_t> qmeta;
  qmeta.insert(qmeta.end(), item_first.begin(), item_first.end());
  qmeta.insert(qmeta.end(), item_cnt.begin(), item_cnt.end());
  for (int s = 0; s < nsn; ++s) qmeta.push_back((int32_t)b.sn[s].children.size());
  c->n_init = 0;
  for (int s = 0; s < nsn; ++s)
    if (b.sn[s].children.empty())
      for (int k = 0; k < item_cnt[s]; ++k) {
        qmeta.push_back(item_first[s] + k);
        ++c->n_init;
      }
  if (getenv("SC_DEBUG")) {
    int64_t maxw = 0, maxr = 0;
    for (int s = 0; s < nsn; ++s) {
      maxw = std::max<int64_t>(maxw, wv[s]);
      maxr = std::max<int64_t>(maxr, rv[s]);
    }
    fprintf(stderr, "[sc] supernodes %d max w %lld max r %lld height %d items %d components %lld\n", nsn,
            (long long)maxw, (long long)maxr, c->height, c->n_items, (long long)c->n_components);
  }
  // per-launch counters (zeroed by launch_solve): phase block counts [2 nsn], finished
  // children [nsn], tile tickets [n_bctr], ready slots [n_items], head, tail
  c->n_counters = 3 * (size_t)nsn + n_bctr + (size_t)c->n_items + 2;
  c->h_items = items;
  std::vector<int32_t> chptr(nsn + 1, 0), chidx, parent(nsn, -1);
  for (int s = 0; s < nsn; ++s) {
    for (int ch : b.sn[s].children) chidx.push_back(ch);
    chptr[s + 1] = (int32_t)chidx.size();
    parent[s] = b.sn[s].parent;
  }
  auto up32 = [&](int32_t** dst, const std::vector<int32_t>& v) {
    SC_CUDA(cudaMalloc(dst, sizeof(int32_t) * std::max<size_t>(1, v.size())));
    if (!v.empty()) SC_CUDA(cudaMemcpy(*dst, v.data(), sizeof(int32_t) * v.size(), cudaMemcpyHostToDevice));
  };
  auto up64 = [&](int64_t** dst, const std::vector<int64_t>& v) {
    SC_CUDA(cudaMalloc(dst, sizeof(int64_t) * std::max<size_t>(1, v.size())));
    if (!v.empty()) SC_CUDA(cudaMemcpy(*dst, v.data(), sizeof(int64_t) * v.size(), cudaMemcpyHostToDevice));
  };
  auto upd_ = [&](double** dst, const std::vector<double>& v) {
    SC_CUDA(cudaMalloc(dst, sizeof(double) * std::max<size_t>(1, v.size())));
    if (!v.empty()) SC_CUDA(cudaMemcpy(*dst, v.data(), sizeof(double) * v.size(), cudaMemcpyHostToDevice));
  };
  up32(&c->d_sn_c0, c0);
  up32(&c->d_sn_w, wv);
  up32(&c->d_sn_r, rv);
  up64(&c->d_sn_aoff, ao);
  up32(&c->d_sn_roff, roff);
  up32(&c->d_sn_uoff, uoff);
  up32(&c->d_sn_goff, goff);
  up32(&c->d_R, Rall);
  up32(&c->d_gptr, gptr);
  up32(&c->d_gidx, gidx);
  up32(&c->d_g2, g2);
  up32(&c->d_items, items);
  up32(&c->d_nitem, nblk);
  up32(&c->d_qmeta, qmeta);
  SC_CUDA(cudaMalloc(&c->d_part, sizeof(double) * std::max<int64_t>(1, pslot)));
  up32(&c->d_chptr, chptr);
  up32(&c->d_chidx, chidx);
  up32(&c->d_parent, parent);
  SC_CUDA(cudaMalloc(&c->d_solve_cnt, sizeof(int) * c->n_counters));
  upd_(&c->fS.A, hAS);
  upd_(&c->fM.A, hAM);
  SC_CUDA(cudaMalloc(&c->d_U, sizeof(double) * std::max<int32_t>(1, uoff[nsn])));
  // c element tables
  std::vector<int32_t> cell32(ne), kidx32(ne);
  for (int e = 0; e < ne; ++e) {
    cell32[e] = (int32_t)b.celem_cell[e];
    kidx32[e] = b.celem_kidx[e];
  }
  up32(&c->d_celem_cell, cell32);
  up32(&c->d_celem_kidx, kidx32);
  up32(&c->d_celem_cidx, b.celem_cidx);
  // element id lists: cut elements (dense K_e streamed, k_celem) and uncut ones (the reference
  // K_e shared by all: one batched product, k_celem_ref)
  {
    std::vector<int32_t> ids_cut, ids_ref;
    for (int e = 0; e < ne; ++e) (kidx32[e] >= 0 ? ids_cut : ids_ref).push_back(e);
    c->n_celem_cut = (int64_t)ids_cut.size();
    c->n_celem_ref = (int64_t)ids_ref.size();
    up32(&c->d_celem_cut_ids, ids_cut);
    up32(&c->d_celem_ref_ids, ids_ref);
  }
  // r^c gather CSR in ND order
  std::vector<int32_t> rptr(nc + 1, 0), ridx;
  ridx.reserve(b.node_eidx.size());
  for (int i = 0; i < nc; ++i) {
    const int v = b.canon_of_nd[i];
    for (int q = b.node_eptr[v]; q < b.node_eptr[v + 1]; ++q) ridx.push_back(b.node_eidx[q]);
    rptr[i + 1] = (int32_t)ridx.size();
  }
  up32(&c->d_rhs_ptr, rptr);
  up32(&c->d_rhs_idx, ridx);
  // c-node lattice indices (ND order), f_x^c
  std::vector<int32_t> clat32(nc);
  std::vector<double> fxc(nc, 0.0);
  for (int i = 0; i < nc; ++i) clat32[i] = (int32_t)c->c_lat[i];
  for (auto& sv : src) {
    int ci = cidx_of(sv.first);
    if (ci >= 0) fxc[b.nd_of_canon[ci]] = sv.second;
  }
  up32(&c->d_c_lat, clat32);
  upd_(&c->d_fxc, fxc);
  upd_(&c->fS.d, dS);
  upd_(&c->fM.d, dM);
  const size_t ncs = std::max(1, nc);
  SC_CUDA(cudaMalloc(&c->d_vc, sizeof(double) * ncs));
  SC_CUDA(cudaMalloc(&c->d_ac, sizeof(double) * ncs));
  SC_CUDA(cudaMalloc(&c->d_b, sizeof(double) * ncs));
  SC_CUDA(cudaMalloc(&c->d_q, sizeof(double) * ncs));
  SC_CUDA(cudaMalloc(&c->d_x, sizeof(double) * ncs));
  SC_CUDA(cudaMalloc(&c->d_Y, sizeof(double) * std::max<size_t>(1, (size_t)ne * nb)));
  SolveDev& sd = c->solve_dev;
  sd.items = reinterpret_cast<const int4*>(c->d_items);
  sd.n_items = c->n_items;
  sd.n_sn = nsn;
  sd.w = c->d_sn_w;
  sd.r = c->d_sn_r;
  sd.c0 = c->d_sn_c0;
  sd.goff = c->d_sn_goff;
  sd.gptr = c->d_gptr;
  sd.gidx = c->d_gidx;
  sd.g2 = reinterpret_cast<const int2*>(c->d_g2);
  sd.uoff = c->d_sn_uoff;
  sd.roff = c->d_sn_roff;
  sd.R = c->d_R;
  sd.aoff = c->d_sn_aoff;
  sd.nblk = c->d_nitem;
  sd.part = c->d_part;
  sd.chptr = c->d_chptr;
  sd.chidx = c->d_chidx;
  sd.parent = c->d_parent;
  sd.U = c->d_U;
  sd.b = c->d_b;
  sd.q = c->d_q;
  sd.x = c->d_x;
  sd.cnt = c->d_solve_cnt;
  sd.done_ch = c->d_solve_cnt + 2 * (size_t)nsn;
  sd.bcnt = c->d_solve_cnt + 3 * (size_t)nsn;
  sd.ready = sd.bcnt + n_bctr;
  sd.head = c->d_solve_cnt + c->n_counters - 2;
  sd.tail = c->d_solve_cnt + c->n_counters - 1;
  sd.item_first = c->d_qmeta;
  sd.item_cnt = c->d_qmeta + 2 * (size_t)nsn;
  sd.nch = c->d_qmeta + 4 * (size_t)nsn;
  sd.init = c->d_qmeta + 5 * (size_t)nsn;
  sd.n_init = c->n_init;
  sd.tile = TILE;
  sd.trace = nullptr;
  if (getenv("SC_TRACE")) {
    SC_CUDA(cudaMalloc(&c->d_trace, sizeof(unsigned long long) * 5 * std::max(1, c->n_items)));
    sd.trace = c->d_trace;
  }
  if (c->world > 1) build_exchange(c, c_owner, clat_global);
  c->Kcut_host.clear();
  c->Kcut_host.shrink_to_fit();
  c->Mcut_host.clear();
  c->Mcut_host.shrink_to_fit();
  flap("device structures");
}
