// Reference tables (step a0): Gauss-Legendre rule, equispaced Lagrange basis,
// tensorised values / reference gradients.  PAPER.md: basis expansion Eq. fe1
// (P:346-349), 'u.bf' / 'u.bfg' operands (Tab. 4), quadrature on
// the reference cell.  Readings: [0,1]^3, equispaced
// nodes, x-fastest lexicographic order.
#include "tables.h"

#include <cmath>

namespace feb200 {

void gauss_legendre01(int n, std::vector<double>& x, std::vector<double>& w) {
  x.assign(n, 0.0);
  w.assign(n, 0.0);
  const double pi = 3.141592653589793238462643383279502884;
  for (int i = 0; i < (n + 1) / 2; ++i) {
    // Tricomi-style initial guess for the i-th largest root of P_n on [-1,1]
    double r = std::cos(pi * (4.0 * i + 3.0) / (4.0 * n + 2.0)) *
               (1.0 - (n - 1.0) / (8.0 * n * n * n));
    double dP = 1.0;
    for (int it = 0; it < 60; ++it) {
      // Bonnet recursion for P_n(r) and P_{n-1}(r)
      double Pm1 = 1.0, P = r;
      for (int k = 2; k <= n; ++k) {
        double Pn = ((2.0 * k - 1.0) * r * P - (k - 1.0) * Pm1) / k;
        Pm1 = P;
        P = Pn;
      }
      if (n == 1) { Pm1 = 1.0; P = r; }
      dP = n * (Pm1 - r * P) / (1.0 - r * r);
      double step = P / dP;
      r -= step;
      if (std::fabs(step) <= 1e-17) break;
    }
    {
      double Pm1 = 1.0, P = r;
      for (int k = 2; k <= n; ++k) {
        double Pn = ((2.0 * k - 1.0) * r * P - (k - 1.0) * Pm1) / k;
        Pm1 = P;
        P = Pn;
      }
      dP = n * (Pm1 - r * P) / (1.0 - r * r);
    }
    double wt = 2.0 / ((1.0 - r * r) * dP * dP);
    // symmetric pair +-r on [-1,1] -> (1 +- r)/2 on [0,1]
    x[n - 1 - i] = 0.5 * (1.0 + r);
    x[i] = 0.5 * (1.0 - r);
    w[n - 1 - i] = 0.5 * wt;
    w[i] = 0.5 * wt;
  }
  if (n % 2 == 1) x[n / 2] = 0.5;
}

void lagrange_equispaced(int p, double t, double* val, double* der) {
  // barycentric-free direct form: l_i(t) = prod_{j!=i} (t - t_j)/(t_i - t_j);
  // l_i'(t) = l_i(t) * sum_{j!=i} 1/(t - t_j) is singular at nodes, so use the
  // product-rule sum instead.
  for (int i = 0; i <= p; ++i) {
    double ti = double(i) / p;
    double denom = 1.0;
    for (int j = 0; j <= p; ++j)
      if (j != i) denom *= (ti - double(j) / p);
    double num = 1.0;
    for (int j = 0; j <= p; ++j)
      if (j != i) num *= (t - double(j) / p);
    val[i] = num / denom;
    double dsum = 0.0;
    for (int m = 0; m <= p; ++m) {
      if (m == i) continue;
      double prod = 1.0;
      for (int j = 0; j <= p; ++j)
        if (j != i && j != m) prod *= (t - double(j) / p);
      dsum += prod;
    }
    der[i] = dsum / denom;
  }
}

HostTables build_tables(int p, int q1d) {
  HostTables T;
  T.p = p;
  T.q1d = q1d;
  const int n1 = p + 1;
  T.nb = n1 * n1 * n1;
  T.nq = q1d * q1d * q1d;
  gauss_legendre01(q1d, T.x1, T.w1);
  T.b1.assign(q1d * n1, 0.0);
  T.d1.assign(q1d * n1, 0.0);
  for (int a = 0; a < q1d; ++a) lagrange_equispaced(p, T.x1[a], &T.b1[a * n1], &T.d1[a * n1]);
  T.xi.assign(3 * T.nq, 0.0);
  T.w.assign(T.nq, 0.0);
  T.phi.assign(size_t(T.nq) * T.nb, 0.0);
  T.dphi.assign(size_t(T.nq) * 3 * T.nb, 0.0);
  for (int qz = 0; qz < q1d; ++qz)
    for (int qy = 0; qy < q1d; ++qy)
      for (int qx = 0; qx < q1d; ++qx) {
        const int q = qx + q1d * (qy + q1d * qz);
        T.xi[3 * q + 0] = T.x1[qx];
        T.xi[3 * q + 1] = T.x1[qy];
        T.xi[3 * q + 2] = T.x1[qz];
        T.w[q] = T.w1[qx] * T.w1[qy] * T.w1[qz];
        for (int kz = 0; kz < n1; ++kz)
          for (int ky = 0; ky < n1; ++ky)
            for (int kx = 0; kx < n1; ++kx) {
              const int k = kx + n1 * (ky + n1 * kz);
              const double bx = T.b1[qx * n1 + kx], by = T.b1[qy * n1 + ky], bz = T.b1[qz * n1 + kz];
              const double dx = T.d1[qx * n1 + kx], dy = T.d1[qy * n1 + ky], dz = T.d1[qz * n1 + kz];
              T.phi[size_t(q) * T.nb + k] = bx * by * bz;
              T.dphi[(size_t(q) * 3 + 0) * T.nb + k] = dx * by * bz;
              T.dphi[(size_t(q) * 3 + 1) * T.nb + k] = bx * dy * bz;
              T.dphi[(size_t(q) * 3 + 2) * T.nb + k] = bx * by * dz;
            }
      }
  const int M = 4 * T.nq;
  T.fwd.assign(size_t(T.nb) * M, 0.0);
  T.bwd.assign(size_t(M) * T.nb, 0.0);
  for (int q = 0; q < T.nq; ++q)
    for (int k = 0; k < T.nb; ++k) {
      double v[4] = {T.phi[size_t(q) * T.nb + k], T.dphi[(size_t(q) * 3 + 0) * T.nb + k],
                     T.dphi[(size_t(q) * 3 + 1) * T.nb + k], T.dphi[(size_t(q) * 3 + 2) * T.nb + k]};
      for (int c = 0; c < 4; ++c) {
        T.fwd[size_t(k) * M + 4 * q + c] = v[c];
        T.bwd[size_t(4 * q + c) * T.nb + k] = v[c];
      }
    }
  return T;
}

}  // namespace feb200
