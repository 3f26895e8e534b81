// Host-side reference tables of the product library (step a0 of the hot path).
// Independent of oracle/: written from the definitions, not shared.
#pragma once
#include <vector>

namespace feb200 {

// Gauss-Legendre rule with n points on [0,1] (weights sum to 1).
void gauss_legendre01(int n, std::vector<double>& x, std::vector<double>& w);

// 1D Lagrange basis of order p on equispaced nodes t_i = i/p: values and
// derivatives of all p+1 functions at t.
void lagrange_equispaced(int p, double t, double* val, double* der);

struct HostTables {
  int p = 0, q1d = 0, nb = 0, nq = 0;
  std::vector<double> x1, w1;          // 1D rule [q1d]
  std::vector<double> b1, d1;          // 1D basis at 1D points [q1d][p+1]
  std::vector<double> xi;              // [nq][3]
  std::vector<double> w;               // [nq]
  std::vector<double> phi;             // [nq][nb]
  std::vector<double> dphi;            // [nq][3][nb]
  std::vector<double> fwd;             // [nb][4 nq]: fwd[k][(q,c)] = T[(q,c)][k]
  std::vector<double> bwd;             // [4 nq][nb]: bwd[(q,c)][k] = T[(q,c)][k]
};

// T[(q,0)][k] = phi_k(xi_q), T[(q,1+m)][k] = d phi_k / d xi_m (xi_q);
// lexicographic x-fastest qp and node order.
HostTables build_tables(int p, int q1d);

}  // namespace feb200
