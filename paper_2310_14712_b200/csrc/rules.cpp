// Host-side quadrature rules, Lagrange basis and uncut reference matrices of libsc.
//
// Lagrange polynomials on the p+1 GLL points (-1, +1 and the roots
// of P_p'): GLL quadrature for the uncut mass (nodal lumping), Gauss-Legendre with
// p+1 points for the stiffness (and on the leaves of cut cells).
// Independent implementation (C++, product path); the oracle has its own.
#include <cmath>
#include <stdexcept>

#include "sc_internal.h"

namespace {
// Legendre P_n and derivative by the three-term recurrence
void legendre_pd(int n, double x, double& P, double& dP) {
  double p0 = 1.0, p1 = x;
  if (n == 0) {
    P = 1.0;
    dP = 0.0;
    return;
  }
  double dp0 = 0.0, dp1 = 1.0;
  for (int k = 2; k <= n; ++k) {
    double p2 = ((2.0 * k - 1.0) * x * p1 - (k - 1.0) * p0) / k;
    double dp2 = dp0 + (2.0 * k - 1.0) * p1;  // P_k' = P_{k-2}' + (2k-1) P_{k-1}
    p0 = p1;
    p1 = p2;
    dp0 = dp1;
    dp1 = dp2;
  }
  P = p1;
  dP = dp1;
}
}  // namespace

void host_gauss(int n, std::vector<double>& x, std::vector<double>& w) {
  x.assign(n, 0.0);
  w.assign(n, 0.0);
  for (int i = 0; i < n; ++i) {
    double t = -std::cos(M_PI * (i + 0.75) / (n + 0.5));  // ascending initial guess
    for (int it = 0; it < 100; ++it) {
      double P, dP;
      legendre_pd(n, t, P, dP);
      double d = P / dP;
      t -= d;
      if (std::fabs(d) < 1e-17) break;
    }
    double P, dP;
    legendre_pd(n, t, P, dP);
    x[i] = t;
    w[i] = 2.0 / ((1.0 - t * t) * dP * dP);
  }
  if (n % 2 == 1) x[n / 2] = 0.0;
}

void host_gll(int p, std::vector<double>& x, std::vector<double>& w) {
  x.assign(p + 1, 0.0);
  w.assign(p + 1, 0.0);
  x[0] = -1.0;
  x[p] = 1.0;
  for (int i = 1; i < p; ++i) {
    double t = -std::cos(M_PI * i / p);
    for (int it = 0; it < 100; ++it) {
      double P, dP;
      legendre_pd(p, t, P, dP);
      // Legendre ODE: (1-t^2) P'' = 2t P' - p(p+1) P
      double ddP = (2.0 * t * dP - p * (p + 1.0) * P) / (1.0 - t * t);
      double d = dP / ddP;
      t -= d;
      if (std::fabs(d) < 1e-17) break;
    }
    x[i] = t;
  }
  if (p % 2 == 0) x[p / 2] = 0.0;
  for (int i = 0; i <= p; ++i) {
    double P, dP;
    legendre_pd(p, x[i], P, dP);
    w[i] = 2.0 / (p * (p + 1.0) * P * P);
  }
}

void host_lagrange(const std::vector<double>& nodes, double xi, double* v, double* dv) {
  const int n = (int)nodes.size();
  for (int i = 0; i < n; ++i) {
    double val = 1.0, der = 0.0;
    for (int j = 0; j < n; ++j) {
      if (j == i) continue;
      double f = (xi - nodes[j]) / (nodes[i] - nodes[j]);
      der = der * f + val / (nodes[i] - nodes[j]);  // product rule, running
      val *= f;
    }
    v[i] = val;
    if (dv) dv[i] = der;
  }
}

double host_lattice(double lo, double hi, int64_t m, int64_t den) {
  volatile double q = (double)m / (double)den;
  volatile double span = hi - lo;
  volatile double t = span * q;
  return lo + t;
}

bool host_phys(const std::vector<DVoid>& voids, const double x[3]) {
  for (const DVoid& v : voids) {
    if (v.kind == SC_VOID_ELLIPSOID) {
      volatile double d0 = x[0] - v.c[0], d1 = x[1] - v.c[1], d2 = x[2] - v.c[2];
      volatile double q = (v.A[0] * d0) * d0;
      volatile double t1 = (v.A[1] * d1) * d1;
      q = q + t1;
      t1 = (v.A[2] * d2) * d2;
      q = q + t1;
      volatile double t = (v.A[3] * d0) * d1;
      volatile double t2 = (v.A[4] * d0) * d2;
      t = t + t2;
      t2 = (v.A[5] * d1) * d2;
      t = t + t2;
      volatile double tt = 2.0 * t;
      q = q + tt;
      if (q < 1.0) return false;
    } else {
      volatile double s = v.n[0] * x[0];
      volatile double s1 = v.n[1] * x[1];
      s = s + s1;
      s1 = v.n[2] * x[2];
      s = s + s1;
      if (s > v.b) return false;
    }
  }
  return true;
}

// 1D reference matrices, uncut element K_e (dense, tensor sum) and lumped M_e diagonal.
void host_reference(sc_ctx* c) {
  const int p = c->g.p, n = p + 1, d = c->g.dim;
  host_gll(p, c->gll_x, c->gll_w);
  host_gauss(n, c->gau_x, c->gau_w);
  c->Mhat.assign(n * n, 0.0);
  c->Khat.assign(n * n, 0.0);
  std::vector<double> v(n), dv(n);
  for (int q = 0; q < n; ++q) {
    host_lagrange(c->gll_x, c->gau_x[q], v.data(), dv.data());
    for (int i = 0; i < n; ++i)
      for (int j = 0; j < n; ++j) {
        c->Mhat[i * n + j] += c->gau_w[q] * v[i] * v[j];
        c->Khat[i * n + j] += c->gau_w[q] * dv[i] * dv[j];
      }
  }
  // K_e = rho c^2 sum_k prod_j (k==j ? (2/h_j) Khat : (h_j/2) Mhat)  (tensor, x fastest)
  const int nb = c->nb;
  c->Kref.assign((size_t)nb * nb, 0.0);
  c->Mref.assign(nb, 0.0);
  int li[3], lj[3];
  for (int a = 0; a < nb; ++a) {
    int t = a;
    for (int k = 0; k < d; ++k) { li[k] = t % n; t /= n; }
    double m = c->rho;
    for (int k = 0; k < d; ++k) m *= 0.5 * c->g.h[k] * c->gll_w[li[k]];
    c->Mref[a] = m;
    for (int b = 0; b < nb; ++b) {
      int u = b;
      for (int k = 0; k < d; ++k) { lj[k] = u % n; u /= n; }
      double s = 0.0;
      for (int k = 0; k < d; ++k) {
        double prod = 1.0;
        for (int j = 0; j < d; ++j) {
          if (j == k) prod *= (2.0 / c->g.h[j]) * c->Khat[li[j] * n + lj[j]];
          else prod *= 0.5 * c->g.h[j] * c->Mhat[li[j] * n + lj[j]];
        }
        s += prod;
      }
      c->Kref[(size_t)a * nb + b] = c->rho * c->c * c->c * s;
    }
  }
  // dt_crit of the uncut cell: power iteration on M^-1/2 K M^-1/2 (symmetric)
  std::vector<double> x(nb), y(nb);
  for (int i = 0; i < nb; ++i) x[i] = 1.0 + 0.37 * std::sin(1.0 + i);
  double lam = 0.0;
  for (int it = 0; it < 5000; ++it) {
    double nrm = 0.0;
    for (int i = 0; i < nb; ++i) {
      double s = 0.0;
      for (int j = 0; j < nb; ++j) s += c->Kref[(size_t)i * nb + j] * x[j] / std::sqrt(c->Mref[j]);
      y[i] = s / std::sqrt(c->Mref[i]);
      nrm += y[i] * y[i];
    }
    nrm = std::sqrt(nrm);
    double num = 0.0, den = 0.0;
    for (int i = 0; i < nb; ++i) { num += x[i] * y[i]; den += x[i] * x[i]; }
    double l2 = num / den;
    for (int i = 0; i < nb; ++i) x[i] = y[i] / nrm;
    if (it > 10 && std::fabs(l2 - lam) <= 1e-15 * std::fabs(l2)) { lam = l2; break; }
    lam = l2;
  }
  c->dt_crit_uncut = 2.0 / std::sqrt(lam);
}
