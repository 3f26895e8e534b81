// Host reference tables of the product library (csrc/tables.cpp, hot-path step a0) checked
// against what the mathematics fixes; built with -fsanitize=address,undefined by
// tests/test_host_tables.py.  No oracle code is involved.
#include <cmath>
#include <cstdio>
#include <vector>

#include "tables.h"

using namespace feb200;

static int fails = 0;
#define CHECK(c, ...) do { if (!(c)) { ++fails; std::printf("FAIL %s:%d: ", __FILE__, __LINE__); std::printf(__VA_ARGS__); std::printf("\n"); } } while (0)

int main() {
  // Gauss-Legendre on [0,1]: n points integrate t^k exactly for k <= 2n-1; degree 2n has the
  // textbook error term
  for (int n = 1; n <= 8; ++n) {
    std::vector<double> x, w;
    gauss_legendre01(n, x, w);
    CHECK((int)x.size() == n && (int)w.size() == n, "sizes n=%d", n);
    for (int i = 0; i < n; ++i) {
      CHECK(x[i] > 0 && x[i] < 1 && w[i] > 0, "range n=%d i=%d", n, i);
      if (i) CHECK(x[i] > x[i - 1], "ascending n=%d", n);
      CHECK(std::fabs(x[i] + x[n - 1 - i] - 1.0) < 1e-15 && std::fabs(w[i] - w[n - 1 - i]) < 1e-15, "symmetry n=%d", n);
    }
    for (int k = 0; k <= 2 * n; ++k) {
      double s = 0;
      for (int i = 0; i < n; ++i) s += w[i] * std::pow(x[i], k);
      const double err = std::fabs(s - 1.0 / (k + 1));
      if (k < 2 * n) CHECK(err < 2e-15, "exactness n=%d k=%d err=%g", n, k, err);
      else if (n <= 5) {
        // degree 2n: the n-point rule on [0,1] misses int t^2n by (n!)^4 / ((2n+1) ((2n)!)^2)
        double f = 1, f2 = 1;
        for (int i = 2; i <= n; ++i) f *= i;
        for (int i = 2; i <= 2 * n; ++i) f2 *= i;
        const double e = f * f * f * f / ((2 * n + 1) * f2 * f2);
        CHECK(std::fabs(err - e) < 0.01 * e, "degree 2n error n=%d: %g vs %g", n, err, e);
      }
    }
  }
  // Lagrange basis on t_i = i/p: Kronecker at the nodes, partition of unity, sum of derivatives
  // 0, reproduces t (sum_i t_i phi_i = t, sum_i t_i phi_i' = 1), derivative vs central difference
  for (int p = 1; p <= 4; ++p) {
    std::vector<double> v(p + 1), d(p + 1), vp(p + 1), vm(p + 1), dd(p + 1);
    for (int i = 0; i <= p; ++i) {
      lagrange_equispaced(p, double(i) / p, v.data(), d.data());
      for (int j = 0; j <= p; ++j) CHECK(std::fabs(v[j] - (i == j)) < 1e-14, "kronecker p=%d", p);
    }
    for (double t : {0.0, 0.137, 0.5, 0.81, 1.0}) {
      lagrange_equispaced(p, t, v.data(), d.data());
      double s = 0, sd = 0, st = 0, std_ = 0;
      for (int i = 0; i <= p; ++i) { s += v[i]; sd += d[i]; st += v[i] * i / p; std_ += d[i] * i / p; }
      CHECK(std::fabs(s - 1) < 1e-13 && std::fabs(sd) < 1e-12, "unity p=%d t=%g", p, t);
      CHECK(std::fabs(st - t) < 1e-13 && std::fabs(std_ - 1) < 1e-12, "linear p=%d t=%g", p, t);
      const double h = 1e-6;
      lagrange_equispaced(p, t + h, vp.data(), dd.data());
      lagrange_equispaced(p, t - h, vm.data(), dd.data());
      for (int i = 0; i <= p; ++i) CHECK(std::fabs((vp[i] - vm[i]) / (2 * h) - d[i]) < 1e-7, "derivative p=%d i=%d", p, i);
    }
  }
  // 3D tables: sizes, tensor-product structure (x fastest), weights, fwd / bwd transposes
  for (int p = 1; p <= 4; ++p)
    for (int q1d = p; q1d <= p + 2 && q1d <= 6; ++q1d) {
      if (q1d < 1) continue;
      const HostTables T = build_tables(p, q1d);
      const int n1 = p + 1, nb = n1 * n1 * n1, nq = q1d * q1d * q1d;
      CHECK(T.p == p && T.q1d == q1d && T.nb == nb && T.nq == nq, "header p=%d", p);
      CHECK((int)T.xi.size() == 3 * nq && (int)T.w.size() == nq && (int)T.phi.size() == nq * nb &&
            (int)T.dphi.size() == 3 * nq * nb && (int)T.fwd.size() == 4 * nq * nb &&
            (int)T.bwd.size() == 4 * nq * nb && (int)T.b1.size() == q1d * n1 && (int)T.d1.size() == q1d * n1,
            "sizes p=%d q1d=%d", p, q1d);
      double ws = 0;
      for (int q = 0; q < nq; ++q) ws += T.w[q];
      CHECK(std::fabs(ws - 1) < 1e-14, "weights p=%d", p);
      for (int q = 0; q < nq; ++q) {
        const int a = q % q1d, b = (q / q1d) % q1d, c = q / (q1d * q1d);
        CHECK(T.xi[3 * q] == T.x1[a] && T.xi[3 * q + 1] == T.x1[b] && T.xi[3 * q + 2] == T.x1[c], "xi order");
        CHECK(std::fabs(T.w[q] - T.w1[a] * T.w1[b] * T.w1[c]) < 1e-16, "w product");
        double s = 0, g[3] = {0, 0, 0}, gx[3] = {0, 0, 0};
        for (int k = 0; k < nb; ++k) {
          const int i = k % n1, j = (k / n1) % n1, l = k / (n1 * n1);
          const double ph = T.b1[a * n1 + i] * T.b1[b * n1 + j] * T.b1[c * n1 + l];
          CHECK(std::fabs(T.phi[q * nb + k] - ph) < 1e-15, "phi tensor p=%d q=%d k=%d", p, q, k);
          const double dr[3] = {T.d1[a * n1 + i] * T.b1[b * n1 + j] * T.b1[c * n1 + l],
                                T.b1[a * n1 + i] * T.d1[b * n1 + j] * T.b1[c * n1 + l],
                                T.b1[a * n1 + i] * T.b1[b * n1 + j] * T.d1[c * n1 + l]};
          const double xn[3] = {double(i) / p, double(j) / p, double(l) / p};
          s += T.phi[q * nb + k];
          for (int m = 0; m < 3; ++m) {
            CHECK(std::fabs(T.dphi[(q * 3 + m) * nb + k] - dr[m]) < 1e-13, "dphi tensor p=%d m=%d", p, m);
            g[m] += T.dphi[(q * 3 + m) * nb + k];
            gx[m] += T.dphi[(q * 3 + m) * nb + k] * xn[m];   // d x_m / d xi_m of the identity map
            CHECK(T.bwd[(q * 4 + 1 + m) * nb + k] == T.dphi[(q * 3 + m) * nb + k], "bwd grad");
            CHECK(T.fwd[k * 4 * nq + q * 4 + 1 + m] == T.dphi[(q * 3 + m) * nb + k], "fwd grad");
          }
          CHECK(T.bwd[(q * 4) * nb + k] == T.phi[q * nb + k] && T.fwd[k * 4 * nq + q * 4] == T.phi[q * nb + k], "fwd / bwd values");
        }
        CHECK(std::fabs(s - 1) < 1e-13, "partition of unity p=%d q=%d", p, q);
        for (int m = 0; m < 3; ++m) CHECK(std::fabs(g[m]) < 1e-11 && std::fabs(gx[m] - 1) < 1e-11, "gradient sums p=%d q=%d m=%d", p, q, m);
      }
    }
  std::printf(fails ? "FAILED %d\n" : "tables ok\n", fails);
  return fails ? 1 : 0;
}
