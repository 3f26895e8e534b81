/*
 * fe_oracle.c -- CPU oracle for batched finite-element weak-form evaluation.
 *
 * TEST INFRASTRUCTURE ONLY.  Nothing on the product path (the CUDA library
 * under paper_2107_04121_b200/) may include, link or call this file.  Only
 * tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
 * reference legs use it.  It shares no code, header, table or constant with
 * the CUDA path.
 *
 * What it computes: the plain definition of the paper's method, i.e. the
 * quadrature-evaluated element integrals of arXiv 2107.04121:
 *   - Alg. 1 "eval_residual": for each cell, for each qp,
 *       r[c] += detw(q) * F(c, q, v, u, d)
 *   - Alg. 2 "eval_matrix": for each cell, for each qp,
 *       M[c] += detw(q) * dF/du(c, q, v, u, d)
 * with the quadrature weight folded into the mapping determinant
 * ("The quadrature weights are incorporated in the element reference mapping
 * Jacobian"; Tab. 4 "v.det").
 *
 * Integrands (element-local DOF index a*n_b + k, component-major, Eq. fe1b
 * P:491-526 and the reshape (j,k)->J of P:589):
 *   diffusion     int kappa grad v . grad u          (weak Laplacian, Tab. 2)
 *   mass          int rho v u                        (dot product, Tab. 2)
 *   vector mass   int rho v_i u_i, D=3               (Eq. fe2a-fe3c)
 *   mass+diff     int rho v u + kappa grad v.grad u  (BASELINE config 4)
 *   elasticity    int e(v)^T D e(u), Voigt via Psg   (Tab. 2, einsum P:1033)
 *   convective    int v_i (du_i/dx_j) u_j            (Eq. fe2)
 *                 tangent = both terms of Eq. fe4
 *
 * Readings of points the paper leaves open are listed in DESIGN.md
 * ("Readings"): reference cell [0,1]^3, equispaced Lagrange nodes, x-fastest
 * lexicographic node/vertex/qp order, trilinear geometry from 8 vertices,
 * Psg with 9 ones (engineering shears), Newton tangent for the convective term.
 *
 * Style: deliberately plain.  No blocking, no fusion, no reordering beyond the
 * loops the definitions state; every table is built from the formula.
 * IEEE fp64, compiled without -ffast-math.
 * OpenMP parallelises only the outer cell loop (for the timed CPU baseline);
 * every cell writes only its own output slice, and the scatter-add
 * (oracle_assemble) is serial in ascending (cell, component, node) order, so
 * results do not depend on the thread count.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define OR_OK 0
#define OR_ERR_ARG (-1)
#define OR_ERR_DEGENERATE (-3)

enum {
  OR_DIFFUSION = 0,
  OR_MASS = 1,
  OR_VECTOR_MASS = 2,
  OR_MASS_DIFFUSION = 3,
  OR_ELASTICITY = 4,
  OR_CONVECTIVE = 5,
  OR_WEIGHTED_DOT = 6, /* Tab. 2 'ij,i,j': int v_i M_ij u_j, M per qp [E][nq][3][3] */
  OR_DIVERGENCE = 7    /* Tab. 2 'i.i': int dv_i/dx_i (linear form, no trial) */
};
#define OR_LAST_FORM OR_DIVERGENCE

/* material kinds for the elasticity form */
enum { OR_MAT_PER_QP = 0, OR_MAT_PER_ELEM = 1, OR_MAT_FULL_D = 2 };

static int64_t g_bad_elem = -1;
int64_t oracle_bad_element(void) { return g_bad_elem; }

/* ------------------------------------------------------------------ */
/* 1D Gauss-Legendre rule on [0,1]: Newton iteration on P_n in long double,
 * started from the Chebyshev-like guesses cos(pi (i + 3/4) / (n + 1/2)),
 * then mapped x = (t + 1)/2, w = w_t / 2 (weights sum to 1, the volume of the
 * reference cell [0,1]).  Points returned in ascending order. */
int oracle_gauss_legendre(int n, double *x, double *w) {
  if (n < 1 || n > 64) return OR_ERR_ARG;
  for (int i = 0; i < n; ++i) {
    long double t = cosl(3.14159265358979323846264338327950288L * (i + 0.75L) / (n + 0.5L));
    long double dp = 0.0L;
    for (int it = 0; it < 100; ++it) {
      /* three-term recurrence: (k+1) P_{k+1} = (2k+1) t P_k - k P_{k-1} */
      long double p0 = 1.0L, p1 = t;
      for (int k = 1; k < n; ++k) {
        long double p2 = ((2.0L * k + 1.0L) * t * p1 - k * p0) / (k + 1.0L);
        p0 = p1;
        p1 = p2;
      }
      /* p1 = P_n(t), p0 = P_{n-1}(t);  P_n'(t) = n (t P_n - P_{n-1}) / (t^2 - 1) */
      dp = n * (t * p1 - p0) / (t * t - 1.0L);
      long double dt = p1 / dp;
      t -= dt;
      if (fabsl(dt) < 1e-19L) break;
    }
    /* recompute derivative at the converged root */
    long double p0 = 1.0L, p1 = t;
    for (int k = 1; k < n; ++k) {
      long double p2 = ((2.0L * k + 1.0L) * t * p1 - k * p0) / (k + 1.0L);
      p0 = p1;
      p1 = p2;
    }
    dp = n * (t * p1 - p0) / (t * t - 1.0L);
    long double wt = 2.0L / ((1.0L - t * t) * dp * dp);
    /* roots come out descending in t; store ascending in x */
    x[n - 1 - i] = (double)((t + 1.0L) * 0.5L);
    w[n - 1 - i] = (double)(wt * 0.5L);
  }
  return OR_OK;
}

/* 1D Lagrange basis of order p on equispaced nodes t_i = i/p:
 *   phi_i(t)  = prod_{j != i} (t - t_j) / (t_i - t_j)
 *   phi_i'(t) = sum_{m != i} 1/(t_i - t_m) prod_{j != i, m} (t - t_j)/(t_i - t_j) */
int oracle_lagrange_1d(int p, double t, double *phi, double *dphi) {
  if (p < 1 || p > 8) return OR_ERR_ARG;
  for (int i = 0; i <= p; ++i) {
    double ti = (double)i / p;
    double v = 1.0;
    for (int j = 0; j <= p; ++j) {
      if (j == i) continue;
      double tj = (double)j / p;
      v *= (t - tj) / (ti - tj);
    }
    phi[i] = v;
    double d = 0.0;
    for (int m = 0; m <= p; ++m) {
      if (m == i) continue;
      double tm = (double)m / p;
      double prod = 1.0 / (ti - tm);
      for (int j = 0; j <= p; ++j) {
        if (j == i || j == m) continue;
        double tj = (double)j / p;
        prod *= (t - tj) / (ti - tj);
      }
      d += prod;
    }
    dphi[i] = d;
  }
  return OR_OK;
}

/* Reference tables on the tensor-product rule with q1d points per axis.
 * qp index q = a + q1d (b + q1d c) (x fastest); node index
 * k = i + (p+1)(j + (p+1) l) (x fastest).
 *   xi[q][3], w[q], Phi[q][k] = phi_i(x_a) phi_j(x_b) phi_l(x_c),
 *   dPhi[q][m][k] = d Phi_k / d xi_m. */
int oracle_tables(int p, int q1d, double *xi, double *w, double *Phi, double *dPhi) {
  if (p < 1 || p > 8 || q1d < 1 || q1d > 16) return OR_ERR_ARG;
  int n1 = p + 1, nb = n1 * n1 * n1;
  double gx[16], gw[16];
  oracle_gauss_legendre(q1d, gx, gw);
  for (int c = 0; c < q1d; ++c)
    for (int b = 0; b < q1d; ++b)
      for (int a = 0; a < q1d; ++a) {
        int q = a + q1d * (b + q1d * c);
        double pa[9], da[9], pb[9], db[9], pc[9], dc[9];
        oracle_lagrange_1d(p, gx[a], pa, da);
        oracle_lagrange_1d(p, gx[b], pb, db);
        oracle_lagrange_1d(p, gx[c], pc, dc);
        if (xi) { xi[3 * q + 0] = gx[a]; xi[3 * q + 1] = gx[b]; xi[3 * q + 2] = gx[c]; }
        if (w) w[q] = gw[a] * gw[b] * gw[c];
        for (int l = 0; l < n1; ++l)
          for (int j = 0; j < n1; ++j)
            for (int i = 0; i < n1; ++i) {
              int k = i + n1 * (j + n1 * l);
              if (Phi) Phi[(int64_t)q * nb + k] = pa[i] * pb[j] * pc[l];
              if (dPhi) {
                dPhi[((int64_t)q * 3 + 0) * nb + k] = da[i] * pb[j] * pc[l];
                dPhi[((int64_t)q * 3 + 1) * nb + k] = pa[i] * db[j] * pc[l];
                dPhi[((int64_t)q * 3 + 2) * nb + k] = pa[i] * pb[j] * dc[l];
              }
            }
      }
  return OR_OK;
}

/* ------------------------------------------------------------------ */
/* Reference mapping of one cell at reference point xi:
 *   x(xi) = sum_v x_v psi_v(xi),  psi_v trilinear, v = a + 2b + 4c,
 *   J_ij = d x_i / d xi_j = sum_v x_{v,i} d psi_v / d xi_j.
 * Returns det J; fills Jinv (row-major, Jinv[m][j]) by cofactors / det. */
static double cell_jacobian(const double *coords, const int32_t *cv, const double *xi,
                            double J[3][3], double Jinv[3][3]) {
  double l[3][2], dl[3][2];
  for (int d = 0; d < 3; ++d) oracle_lagrange_1d(1, xi[d], l[d], dl[d]);
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) J[i][j] = 0.0;
  for (int c = 0; c < 2; ++c)
    for (int b = 0; b < 2; ++b)
      for (int a = 0; a < 2; ++a) {
        int v = a + 2 * b + 4 * c;
        double dpsi[3] = {dl[0][a] * l[1][b] * l[2][c], l[0][a] * dl[1][b] * l[2][c],
                          l[0][a] * l[1][b] * dl[2][c]};
        const double *xv = coords + 3 * (int64_t)cv[v];
        for (int i = 0; i < 3; ++i)
          for (int j = 0; j < 3; ++j) J[i][j] += xv[i] * dpsi[j];
      }
  double cof[3][3];
  cof[0][0] = J[1][1] * J[2][2] - J[1][2] * J[2][1];
  cof[0][1] = -(J[1][0] * J[2][2] - J[1][2] * J[2][0]);
  cof[0][2] = J[1][0] * J[2][1] - J[1][1] * J[2][0];
  cof[1][0] = -(J[0][1] * J[2][2] - J[0][2] * J[2][1]);
  cof[1][1] = J[0][0] * J[2][2] - J[0][2] * J[2][0];
  cof[1][2] = -(J[0][0] * J[2][1] - J[0][1] * J[2][0]);
  cof[2][0] = J[0][1] * J[1][2] - J[0][2] * J[1][1];
  cof[2][1] = -(J[0][0] * J[1][2] - J[0][2] * J[1][0]);
  cof[2][2] = J[0][0] * J[1][1] - J[0][1] * J[1][0];
  double det = J[0][0] * cof[0][0] + J[0][1] * cof[0][1] + J[0][2] * cof[0][2];
  /* inverse = adjugate / det, adjugate = cofactor^T */
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) Jinv[i][j] = cof[j][i] / det;
  return det;
}

/* Geometry of all cells (steps a1 and b of the hot path), materialised:
 *   detw[e][q] = w_q det J,  Jinv[e][q][3][3].
 * Fails with OR_ERR_DEGENERATE (cell index via oracle_bad_element) when
 * det J <= 0 anywhere (|J| > 0 required). */
int oracle_geometry(int q1d, int64_t n_elems, const double *coords, const int32_t *conn,
                    double *detw, double *Jinv_out) {
  int nq = q1d * q1d * q1d;
  double *xi = malloc(sizeof(double) * 3 * nq), *w = malloc(sizeof(double) * nq);
  oracle_tables(1, q1d, xi, w, NULL, NULL);
  int status = OR_OK;
  g_bad_elem = -1;
  for (int64_t e = 0; e < n_elems && status == OR_OK; ++e)
    for (int q = 0; q < nq; ++q) {
      double J[3][3], Ji[3][3];
      double det = cell_jacobian(coords, conn + 8 * e, xi + 3 * q, J, Ji);
      if (!(det > 0.0)) { status = OR_ERR_DEGENERATE; g_bad_elem = e; break; }
      if (detw) detw[e * nq + q] = w[q] * det;
      if (Jinv_out)
        for (int i = 0; i < 3; ++i)
          for (int j = 0; j < 3; ++j) Jinv_out[(e * nq + q) * 9 + 3 * i + j] = Ji[i][j];
    }
  free(xi);
  free(w);
  return status;
}

/* Psg[r][j][I]: vector storage of the symmetric gradient (Tab. 4),
 * Voigt order I = (xx, yy, zz, xy, xz, yz), engineering shears:
 * e_I(u) = sum_{r,j} Psg[r][j][I] du_r/dx_j.  9 ones (reading 7). */
static void build_psg(double Psg[3][3][6]) {
  memset(Psg, 0, sizeof(double) * 54);
  Psg[0][0][0] = 1.0;
  Psg[1][1][1] = 1.0;
  Psg[2][2][2] = 1.0;
  Psg[0][1][3] = 1.0; Psg[1][0][3] = 1.0;
  Psg[0][2][4] = 1.0; Psg[2][0][4] = 1.0;
  Psg[1][2][5] = 1.0; Psg[2][1][5] = 1.0;
}

/* isotropic Voigt elasticity matrix D = lambda 1_3 1_3^T (+) 0 + diag(2mu,2mu,2mu,mu,mu,mu) */
void oracle_isotropic_D(double lam, double mu, double *D) {
  for (int I = 0; I < 6; ++I)
    for (int K = 0; K < 6; ++K) D[6 * I + K] = 0.0;
  for (int I = 0; I < 3; ++I)
    for (int K = 0; K < 3; ++K) D[6 * I + K] = lam;
  for (int I = 0; I < 3; ++I) D[6 * I + I] += 2.0 * mu;
  for (int I = 3; I < 6; ++I) D[6 * I + I] = mu;
}

static int form_ncomp(int form) {
  return (form == OR_VECTOR_MASS || form == OR_ELASTICITY || form == OR_CONVECTIVE ||
          form == OR_WEIGHTED_DOT || form == OR_DIVERGENCE) ? 3 : 1;
}

/* Elastic matrix at (e, q) from the material description. */
static void material_D(int mat_kind, const double *a, const double *b, int64_t e, int q, int nq,
                       double D[36]) {
  if (mat_kind == OR_MAT_FULL_D) {
    for (int i = 0; i < 36; ++i) D[i] = a[(e * nq + q) * 36 + i];
  } else if (mat_kind == OR_MAT_PER_ELEM) {
    oracle_isotropic_D(a[e], b[e], D);
  } else {
    oracle_isotropic_D(a[e * nq + q], b[e * nq + q], D);
  }
}

/* scalar per-qp material value, or 0 when absent */
static double qp_value(const double *arr, int64_t e, int q, int nq) {
  return arr ? arr[e * nq + q] : 0.0;
}

/* ------------------------------------------------------------------ */
/* Alg. 2 eval_matrix: K[e][ndof][ndof], row = test (a, k),
 * column = trial (b, l), local index a*n_b + k.
 *   mat_a / mat_b: see DESIGN.md (kappa | rho | rho,kappa | lambda,mu | unused)
 *   u_state: convective state, global node-major [n_nodes][3] (NULL otherwise)
 *   dof_conn: [E][n_b] global node of each element node (NULL => conn, p == 1) */
int oracle_eval_matrix(int form, int p, int q1d, int64_t n_elems, const double *coords,
                       const int32_t *conn, const int32_t *dof_conn, int mat_kind,
                       const double *mat_a, const double *mat_b, const double *u_state,
                       double *K) {
  if (p < 1 || p > 8 || q1d < 1 || q1d > 16 || n_elems < 0) return OR_ERR_ARG;
  if (form < 0 || form > OR_WEIGHTED_DOT) return OR_ERR_ARG; /* divergence: no trial variable */
  if (form == OR_CONVECTIVE && !u_state) return OR_ERR_ARG;
  if (form == OR_WEIGHTED_DOT && !mat_a) return OR_ERR_ARG;
  const int n1 = p + 1, nb = n1 * n1 * n1, nq = q1d * q1d * q1d;
  const int D = form_ncomp(form), ndof = D * nb;
  if (!dof_conn) {
    if (p != 1) return OR_ERR_ARG;
    dof_conn = conn;
  }
  double *xi = malloc(sizeof(double) * 3 * nq), *w = malloc(sizeof(double) * nq);
  double *Phi = malloc(sizeof(double) * nq * nb), *dPhi = malloc(sizeof(double) * nq * 3 * nb);
  oracle_tables(p, q1d, xi, w, Phi, dPhi);
  double Psg[3][3][6];
  build_psg(Psg);
  int status = OR_OK;
  g_bad_elem = -1;

#pragma omp parallel for schedule(static)
  for (int64_t e = 0; e < n_elems; ++e) {
    double *Ke = K + e * (int64_t)ndof * ndof;
    double *G = malloc(sizeof(double) * 3 * nb);   /* physical gradients G[j][k] */
    double *Bv = malloc(sizeof(double) * 6 * ndof); /* Voigt B[I][(r,e)] */
    for (int64_t i = 0; i < (int64_t)ndof * ndof; ++i) Ke[i] = 0.0;
    for (int q = 0; q < nq; ++q) {
      double J[3][3], Ji[3][3];
      double det = cell_jacobian(coords, conn + 8 * e, xi + 3 * q, J, Ji);
      if (!(det > 0.0)) {
#pragma omp critical
        { status = OR_ERR_DEGENERATE; if (g_bad_elem < 0 || e < g_bad_elem) g_bad_elem = e; }
        break;
      }
      const double detw = w[q] * det;
      const double *phi = Phi + (int64_t)q * nb;
      /* step b: G = J^-T grad_xi phi, i.e. dphi/dx_j = sum_m dphi/dxi_m Jinv[m][j] */
      for (int j = 0; j < 3; ++j)
        for (int k = 0; k < nb; ++k) {
          double s = 0.0;
          for (int m = 0; m < 3; ++m) s += dPhi[((int64_t)q * 3 + m) * nb + k] * Ji[m][j];
          G[j * nb + k] = s;
        }
      if (form == OR_DIFFUSION || form == OR_MASS || form == OR_MASS_DIFFUSION) {
        double kappa = (form == OR_DIFFUSION) ? qp_value(mat_a, e, q, nq)
                       : (form == OR_MASS_DIFFUSION) ? qp_value(mat_b, e, q, nq) : 0.0;
        double rho = (form == OR_MASS || form == OR_MASS_DIFFUSION) ? qp_value(mat_a, e, q, nq) : 0.0;
        for (int i = 0; i < nb; ++i)
          for (int j = 0; j < nb; ++j) {
            double f = 0.0;
            if (form != OR_MASS)
              f += kappa * (G[0 * nb + i] * G[0 * nb + j] + G[1 * nb + i] * G[1 * nb + j] +
                            G[2 * nb + i] * G[2 * nb + j]);
            if (form != OR_DIFFUSION) f += rho * phi[i] * phi[j];
            Ke[(int64_t)i * ndof + j] += detw * f;
          }
      } else if (form == OR_VECTOR_MASS) {
        /* einsum('cq,qd,ir,qe,is->crdse'): delta_ir delta_is phi_d phi_e */
        double rho = qp_value(mat_a, e, q, nq);
        for (int r = 0; r < 3; ++r)
          for (int d = 0; d < nb; ++d)
            for (int s = 0; s < 3; ++s)
              for (int ee = 0; ee < nb; ++ee) {
                double f = 0.0;
                for (int i = 0; i < 3; ++i) f += (i == r) * (i == s) * phi[d] * phi[ee];
                Ke[(int64_t)(r * nb + d) * ndof + s * nb + ee] += detw * rho * f;
              }
      } else if (form == OR_ELASTICITY) {
        /* einsum('cq,cqje,rjI,cqIK,cqlf,slK->cresf'):
         * B[I][(r,e)] = sum_j Psg[r][j][I] G[j][e];  K += detw B^T D B */
        double Dm[36];
        material_D(mat_kind, mat_a, mat_b, e, q, nq, Dm);
        for (int I = 0; I < 6; ++I)
          for (int r = 0; r < 3; ++r)
            for (int k = 0; k < nb; ++k) {
              double s = 0.0;
              for (int j = 0; j < 3; ++j) s += Psg[r][j][I] * G[j * nb + k];
              Bv[I * ndof + r * nb + k] = s;
            }
        for (int a = 0; a < ndof; ++a)
          for (int b = 0; b < ndof; ++b) {
            double f = 0.0;
            for (int I = 0; I < 6; ++I)
              for (int Kk = 0; Kk < 6; ++Kk) f += Bv[I * ndof + a] * Dm[6 * I + Kk] * Bv[Kk * ndof + b];
            Ke[(int64_t)a * ndof + b] += detw * f;
          }
      } else if (form == OR_WEIGHTED_DOT) {
        /* 'ij,i,j': K[(a,k),(b,l)] += detw M_ab phi_k phi_l */
        const double *M = mat_a + (e * nq + q) * 9;
        for (int a = 0; a < 3; ++a)
          for (int k = 0; k < nb; ++k)
            for (int b = 0; b < 3; ++b)
              for (int l = 0; l < nb; ++l)
                Ke[(int64_t)(a * nb + k) * ndof + b * nb + l] += detw * M[3 * a + b] * phi[k] * phi[l];
      } else { /* OR_CONVECTIVE, Eq. fe4 */
        /* state at the qp: u_j(q) = sum_m u^m_j phi_m,  du_i/dx_j = sum_l u^l_i G[j][l] */
        double uq[3] = {0, 0, 0}, gu[3][3] = {{0}};
        for (int m = 0; m < nb; ++m) {
          const double *um = u_state + 3 * (int64_t)dof_conn[e * nb + m];
          for (int i = 0; i < 3; ++i) {
            uq[i] += um[i] * phi[m];
            for (int j = 0; j < 3; ++j) gu[i][j] += um[i] * G[j * nb + m];
          }
        }
        for (int a = 0; a < 3; ++a)
          for (int k = 0; k < nb; ++k)
            for (int b = 0; b < 3; ++b)
              for (int l = 0; l < nb; ++l) {
                /* term 1: phi_k delta_ab dphi_l/dx_j u_j ; term 2: phi_k du_a/dx_b phi_l */
                double adv = 0.0;
                for (int j = 0; j < 3; ++j) adv += G[j * nb + l] * uq[j];
                double f = phi[k] * ((a == b) * adv + gu[a][b] * phi[l]);
                Ke[(int64_t)(a * nb + k) * ndof + b * nb + l] += detw * f;
              }
      }
    }
    free(G);
    free(Bv);
  }
  free(xi); free(w); free(Phi); free(dPhi);
  return status;
}

/* ------------------------------------------------------------------ */
/* Alg. 1 eval_residual over cells [elem_begin, elem_end):
 * r_elem[e - elem_begin][ndof] (overwritten).  u is the global node-major
 * DOF vector [n_nodes][D] (Eq. fe1c), gathered per cell through dof_conn
 * ("the mesh cell connectivity is used to index the DOF vector").
 * The integrand is evaluated at each qp from u_h(q) and grad u_h(q), then
 * tested against v = phi_k e_a. */
int oracle_eval_residual(int form, int p, int q1d, int64_t n_elems, const double *coords,
                         const int32_t *conn, const int32_t *dof_conn, int mat_kind,
                         const double *mat_a, const double *mat_b, const double *u,
                         int64_t elem_begin, int64_t elem_end, double *r_elem) {
  if (p < 1 || p > 8 || q1d < 1 || q1d > 16 || n_elems < 0) return OR_ERR_ARG;
  if (form < 0 || form > OR_LAST_FORM || !u) return OR_ERR_ARG;
  if (form == OR_WEIGHTED_DOT && !mat_a) return OR_ERR_ARG;
  if (elem_begin < 0 || elem_end > n_elems || elem_begin > elem_end) return OR_ERR_ARG;
  const int n1 = p + 1, nb = n1 * n1 * n1, nq = q1d * q1d * q1d;
  const int D = form_ncomp(form), ndof = D * nb;
  if (!dof_conn) {
    if (p != 1) return OR_ERR_ARG;
    dof_conn = conn;
  }
  double *xi = malloc(sizeof(double) * 3 * nq), *w = malloc(sizeof(double) * nq);
  double *Phi = malloc(sizeof(double) * nq * nb), *dPhi = malloc(sizeof(double) * nq * 3 * nb);
  oracle_tables(p, q1d, xi, w, Phi, dPhi);
  double Psg[3][3][6];
  build_psg(Psg);
  int status = OR_OK;
  g_bad_elem = -1;

#pragma omp parallel for schedule(static)
  for (int64_t e = elem_begin; e < elem_end; ++e) {
    double *re = r_elem + (e - elem_begin) * (int64_t)ndof;
    double *G = malloc(sizeof(double) * 3 * nb);
    double *ue = malloc(sizeof(double) * ndof);
    for (int a = 0; a < D; ++a)
      for (int k = 0; k < nb; ++k) ue[a * nb + k] = u[(int64_t)dof_conn[e * nb + k] * D + a];
    for (int i = 0; i < ndof; ++i) re[i] = 0.0;
    for (int q = 0; q < nq; ++q) {
      double J[3][3], Ji[3][3];
      double det = cell_jacobian(coords, conn + 8 * e, xi + 3 * q, J, Ji);
      if (!(det > 0.0)) {
#pragma omp critical
        { status = OR_ERR_DEGENERATE; if (g_bad_elem < 0 || e < g_bad_elem) g_bad_elem = e; }
        break;
      }
      const double detw = w[q] * det;
      const double *phi = Phi + (int64_t)q * nb;
      for (int j = 0; j < 3; ++j)
        for (int k = 0; k < nb; ++k) {
          double s = 0.0;
          for (int m = 0; m < 3; ++m) s += dPhi[((int64_t)q * 3 + m) * nb + k] * Ji[m][j];
          G[j * nb + k] = s;
        }
      /* u_h and grad u_h at the qp (Eq. fe1c; du_i/dx_j = sum_k u^k_i dphi_k/dx_j) */
      double uq[3] = {0, 0, 0}, gu[3][3] = {{0}};
      for (int a = 0; a < D; ++a)
        for (int k = 0; k < nb; ++k) {
          uq[a] += ue[a * nb + k] * phi[k];
          for (int j = 0; j < 3; ++j) gu[a][j] += ue[a * nb + k] * G[j * nb + k];
        }
      if (form == OR_DIFFUSION || form == OR_MASS || form == OR_MASS_DIFFUSION) {
        double kappa = (form == OR_DIFFUSION) ? qp_value(mat_a, e, q, nq)
                       : (form == OR_MASS_DIFFUSION) ? qp_value(mat_b, e, q, nq) : 0.0;
        double rho = (form == OR_MASS || form == OR_MASS_DIFFUSION) ? qp_value(mat_a, e, q, nq) : 0.0;
        for (int k = 0; k < nb; ++k) {
          double f = 0.0;
          if (form != OR_MASS)
            f += kappa * (G[0 * nb + k] * gu[0][0] + G[1 * nb + k] * gu[0][1] + G[2 * nb + k] * gu[0][2]);
          if (form != OR_DIFFUSION) f += rho * phi[k] * uq[0];
          re[k] += detw * f;
        }
      } else if (form == OR_VECTOR_MASS) {
        double rho = qp_value(mat_a, e, q, nq);
        for (int a = 0; a < 3; ++a)
          for (int k = 0; k < nb; ++k) re[a * nb + k] += detw * rho * phi[k] * uq[a];
      } else if (form == OR_ELASTICITY) {
        /* e(u)_K = sum_{s,l} Psg[s][l][K] du_s/dx_l ; sigma_I = sum_K D_IK e_K ;
         * r[(r,e)] += detw sum_I (sum_j Psg[r][j][I] G[j][e]) sigma_I */
        double Dm[36], eps[6], sig[6];
        material_D(mat_kind, mat_a, mat_b, e, q, nq, Dm);
        for (int Kk = 0; Kk < 6; ++Kk) {
          double s = 0.0;
          for (int s_ = 0; s_ < 3; ++s_)
            for (int l = 0; l < 3; ++l) s += Psg[s_][l][Kk] * gu[s_][l];
          eps[Kk] = s;
        }
        for (int I = 0; I < 6; ++I) {
          double s = 0.0;
          for (int Kk = 0; Kk < 6; ++Kk) s += Dm[6 * I + Kk] * eps[Kk];
          sig[I] = s;
        }
        for (int r = 0; r < 3; ++r)
          for (int k = 0; k < nb; ++k) {
            double f = 0.0;
            for (int I = 0; I < 6; ++I) {
              double bv = 0.0;
              for (int j = 0; j < 3; ++j) bv += Psg[r][j][I] * G[j * nb + k];
              f += bv * sig[I];
            }
            re[r * nb + k] += detw * f;
          }
      } else if (form == OR_WEIGHTED_DOT) {
        /* int v_a M_ab u_b: tested against v = phi_k e_a */
        const double *M = mat_a + (e * nq + q) * 9;
        for (int a = 0; a < 3; ++a) {
          double f0 = 0.0;
          for (int b = 0; b < 3; ++b) f0 += M[3 * a + b] * uq[b];
          for (int k = 0; k < nb; ++k) re[a * nb + k] += detw * phi[k] * f0;
        }
      } else if (form == OR_DIVERGENCE) {
        /* int dv_a/dx_a with v = phi_k e_a: r[(a,k)] = int dphi_k/dx_a (u is not used) */
        for (int a = 0; a < 3; ++a)
          for (int k = 0; k < nb; ++k) re[a * nb + k] += detw * G[a * nb + k];
      } else { /* OR_CONVECTIVE: c(v,u,u) = int v_i du_i/dx_j u_j (Eq. fe2) */
        for (int a = 0; a < 3; ++a) {
          double f0 = 0.0;
          for (int j = 0; j < 3; ++j) f0 += gu[a][j] * uq[j];
          for (int k = 0; k < nb; ++k) re[a * nb + k] += detw * phi[k] * f0;
        }
      }
    }
    free(G);
    free(ue);
  }
  free(xi); free(w); free(Phi); free(dPhi);
  return status;
}

/* Scatter-add of element residuals into the global node-major vector
 * (the assembly step the paper leaves to SfePy):
 *   r_global[dof_conn[e][k] * D + a] += r_elem[e][a * n_b + k]
 * Serial, ascending (e, a, k): deterministic. */
int oracle_assemble(int64_t n_elems, int nb, int D, const int32_t *dof_conn,
                    const double *r_elem, double *r_global) {
  if (n_elems < 0 || nb < 1 || D < 1) return OR_ERR_ARG;
  for (int64_t e = 0; e < n_elems; ++e)
    for (int a = 0; a < D; ++a)
      for (int k = 0; k < nb; ++k)
        r_global[(int64_t)dof_conn[e * nb + k] * D + a] += r_elem[e * (int64_t)D * nb + a * nb + k];
  return OR_OK;
}

/* ------------------------------------------------------------------ */
/* 'eval' mode ("returning the integral value in case all variables
 * passed to the evaluation function have associated DOFs"): the form with the
 * test function replaced by the field itself, summed over cells [elem_begin, elem_end):
 *   diffusion    int kappa grad u . grad u
 *   mass         int rho u u              vector mass  int rho u_i u_i
 *   mass+diff    int rho u u + kappa grad u . grad u
 *   elasticity   int e(u)^T D e(u)
 *   convective   int u_i (du_i/dx_j) u_j  (c(u, u, u), Eq. fe2)
 * Plain quadrature sum, Alg. 1's loop with F evaluated at v = u. */
int oracle_eval_scalar(int form, int p, int q1d, int64_t n_elems, const double *coords,
                       const int32_t *conn, const int32_t *dof_conn, int mat_kind,
                       const double *mat_a, const double *mat_b, const double *u,
                       int64_t elem_begin, int64_t elem_end, double *value) {
  if (p < 1 || p > 8 || q1d < 1 || q1d > 16 || n_elems < 0) return OR_ERR_ARG;
  if (form < 0 || form > OR_LAST_FORM || !u || !value) return OR_ERR_ARG;
  if (form == OR_WEIGHTED_DOT && !mat_a) return OR_ERR_ARG;
  if (elem_begin < 0 || elem_end > n_elems || elem_begin > elem_end) return OR_ERR_ARG;
  const int n1 = p + 1, nb = n1 * n1 * n1, nq = q1d * q1d * q1d;
  const int D = form_ncomp(form);
  if (!dof_conn) {
    if (p != 1) return OR_ERR_ARG;
    dof_conn = conn;
  }
  double *xi = malloc(sizeof(double) * 3 * nq), *w = malloc(sizeof(double) * nq);
  double *Phi = malloc(sizeof(double) * nq * nb), *dPhi = malloc(sizeof(double) * nq * 3 * nb);
  oracle_tables(p, q1d, xi, w, Phi, dPhi);
  double Psg[3][3][6];
  build_psg(Psg);
  int status = OR_OK;
  double total = 0.0;
  for (int64_t e = elem_begin; e < elem_end && status == OR_OK; ++e) {
    for (int q = 0; q < nq; ++q) {
      double J[3][3], Ji[3][3];
      double det = cell_jacobian(coords, conn + 8 * e, xi + 3 * q, J, Ji);
      if (!(det > 0.0)) { status = OR_ERR_DEGENERATE; g_bad_elem = e; break; }
      const double detw = w[q] * det;
      const double *phi = Phi + (int64_t)q * nb;
      double uq[3] = {0, 0, 0}, gu[3][3] = {{0}};
      for (int k = 0; k < nb; ++k) {
        double g[3];
        for (int j = 0; j < 3; ++j) {
          g[j] = 0.0;
          for (int m = 0; m < 3; ++m) g[j] += dPhi[((int64_t)q * 3 + m) * nb + k] * Ji[m][j];
        }
        for (int a = 0; a < D; ++a) {
          const double ua = u[(int64_t)dof_conn[e * nb + k] * D + a];
          uq[a] += ua * phi[k];
          for (int j = 0; j < 3; ++j) gu[a][j] += ua * g[j];
        }
      }
      double f = 0.0;
      if (form == OR_DIFFUSION || form == OR_MASS || form == OR_MASS_DIFFUSION) {
        double kappa = (form == OR_DIFFUSION) ? qp_value(mat_a, e, q, nq)
                       : (form == OR_MASS_DIFFUSION) ? qp_value(mat_b, e, q, nq) : 0.0;
        double rho = (form == OR_MASS || form == OR_MASS_DIFFUSION) ? qp_value(mat_a, e, q, nq) : 0.0;
        f = kappa * (gu[0][0] * gu[0][0] + gu[0][1] * gu[0][1] + gu[0][2] * gu[0][2]) + rho * uq[0] * uq[0];
      } else if (form == OR_VECTOR_MASS) {
        double rho = qp_value(mat_a, e, q, nq);
        f = rho * (uq[0] * uq[0] + uq[1] * uq[1] + uq[2] * uq[2]);
      } else if (form == OR_ELASTICITY) {
        double Dm[36], eps[6];
        material_D(mat_kind, mat_a, mat_b, e, q, nq, Dm);
        for (int I = 0; I < 6; ++I) {
          eps[I] = 0.0;
          for (int r = 0; r < 3; ++r)
            for (int l = 0; l < 3; ++l) eps[I] += Psg[r][l][I] * gu[r][l];
        }
        for (int I = 0; I < 6; ++I)
          for (int K = 0; K < 6; ++K) f += eps[I] * Dm[6 * I + K] * eps[K];
      } else if (form == OR_WEIGHTED_DOT) {
        const double *M = mat_a + (e * nq + q) * 9;
        for (int a = 0; a < 3; ++a)
          for (int b = 0; b < 3; ++b) f += uq[a] * M[3 * a + b] * uq[b];
      } else if (form == OR_DIVERGENCE) {
        f = gu[0][0] + gu[1][1] + gu[2][2]; /* int div u */
      } else {
        for (int i = 0; i < 3; ++i)
          for (int j = 0; j < 3; ++j) f += uq[i] * gu[i][j] * uq[j];
      }
      total += detw * f;
    }
  }
  free(xi); free(w); free(Phi); free(dPhi);
  if (status == OR_OK) *value = total;
  return status;
}

/* Thread count of the cell-parallel loops (timing only; results do not depend on it). */
int oracle_set_threads(int n) {
#ifdef _OPENMP
  if (n > 0) omp_set_num_threads(n);
  return omp_get_max_threads();
#else
  (void)n;
  return 1;
#endif
}

/* Cauchy stress (Tab. 2 'IK,s(k:l)->K'): sigma = D e(u) at every quadrature
 * point of cells [elem_begin, elem_end), Voigt order (xx, yy, zz, xy, xz, yz), engineering
 * shear strains (reading 7); "evaluated only" (no test variable):
 *   sigma[e - elem_begin][q][6]. */
static int stress_impl(int p, int q1d, int64_t n_elems, const double *coords, const int32_t *conn,
                       const int32_t *dof_conn, int mat_kind, const double *mat_a,
                       const double *mat_b, const double *u, int64_t elem_begin, int64_t elem_end,
                       double *sigma, int integ) {
  if (p < 1 || p > 8 || q1d < 1 || q1d > 16 || n_elems < 0 || !u || !sigma) return OR_ERR_ARG;
  if (elem_begin < 0 || elem_end > n_elems || elem_begin > elem_end) return OR_ERR_ARG;
  const int n1 = p + 1, nb = n1 * n1 * n1, nq = q1d * q1d * q1d;
  if (!dof_conn) {
    if (p != 1) return OR_ERR_ARG;
    dof_conn = conn;
  }
  double *xi = malloc(sizeof(double) * 3 * nq), *w = malloc(sizeof(double) * nq);
  double *Phi = malloc(sizeof(double) * nq * nb), *dPhi = malloc(sizeof(double) * nq * 3 * nb);
  oracle_tables(p, q1d, xi, w, Phi, dPhi);
  double Psg[3][3][6];
  build_psg(Psg);
  int status = OR_OK;
  for (int64_t e = elem_begin; e < elem_end && status == OR_OK; ++e) {
    for (int q = 0; q < nq; ++q) {
      double J[3][3], Ji[3][3];
      double det = cell_jacobian(coords, conn + 8 * e, xi + 3 * q, J, Ji);
      if (!(det > 0.0)) { status = OR_ERR_DEGENERATE; g_bad_elem = e; break; }
      double gu[3][3] = {{0}};
      for (int k = 0; k < nb; ++k)
        for (int j = 0; j < 3; ++j) {
          double g = 0.0;
          for (int m = 0; m < 3; ++m) g += dPhi[((int64_t)q * 3 + m) * nb + k] * Ji[m][j];
          for (int a = 0; a < 3; ++a) gu[a][j] += u[(int64_t)dof_conn[e * nb + k] * 3 + a] * g;
        }
      double Dm[36], eps[6];
      material_D(mat_kind, mat_a, mat_b, e, q, nq, Dm);
      for (int I = 0; I < 6; ++I) {
        eps[I] = 0.0;
        for (int r = 0; r < 3; ++r)
          for (int l = 0; l < 3; ++l) eps[I] += Psg[r][l][I] * gu[r][l];
      }
      for (int I = 0; I < 6; ++I) {
        double sI = 0.0;
        for (int K = 0; K < 6; ++K) sI += Dm[6 * I + K] * eps[K];
        if (integ)  /* 'eval' mode: int_e sigma = sum_q w_q det J sigma */
          sigma[(e - elem_begin) * 6 + I] += w[q] * det * sI;
        else
          sigma[((e - elem_begin) * nq + q) * 6 + I] = sI;
      }
    }
  }
  free(xi); free(w); free(Phi); free(dPhi);
  return status;
}

/* Cauchy stress at every qp: sigma[e - elem_begin][q][6]. */
int oracle_eval_stress(int p, int q1d, int64_t n_elems, const double *coords, const int32_t *conn,
                       const int32_t *dof_conn, int mat_kind, const double *mat_a,
                       const double *mat_b, const double *u, int64_t elem_begin, int64_t elem_end,
                       double *sigma) {
  return stress_impl(p, q1d, n_elems, coords, conn, dof_conn, mat_kind, mat_a, mat_b, u,
                     elem_begin, elem_end, sigma, 0);
}

/* The Cauchy stress in 'eval' mode ("the integral value"): per cell
 * sigma_int[e - elem_begin][6] = int_e sigma dx (quadrature as everywhere: w_q det J). */
int oracle_eval_stress_integral(int p, int q1d, int64_t n_elems, const double *coords,
                                const int32_t *conn, const int32_t *dof_conn, int mat_kind,
                                const double *mat_a, const double *mat_b, const double *u,
                                int64_t elem_begin, int64_t elem_end, double *sigma_int) {
  if (sigma_int && elem_end > elem_begin && elem_begin >= 0)
    memset(sigma_int, 0, sizeof(double) * 6 * (size_t)(elem_end - elem_begin));
  return stress_impl(p, q1d, n_elems, coords, conn, dof_conn, mat_kind, mat_a, mat_b, u,
                     elem_begin, elem_end, sigma_int, 1);
}

/* ------------------------------------------------------------------ */
/* Mixed velocity-pressure forms (Tab. 2): velocity space Q_pv (vector, D = 3,
 * tables Phi / dPhi), pressure space Q_pp (scalar, tables Psi), one quadrature rule q1d
 * shared by both (reading 19).
 *   Stokes coupling            ('i.i,0', v, p): int (dv_i/dx_i) p
 *       matrix  B[e'][a*nbv + k][l] = int dphi_k/dx_a psi_l      (test v, trial p)
 *       residual r[e'][a*nbv + k]   = int dphi_k/dx_a p_h        (p_h = sum_l psi_l p_l)
 *   transposed Stokes coupling ('i.i,0', u, q): int q (du_i/dx_i)
 *       matrix  C[e'][l][a*nbv + k] = int psi_l dphi_k/dx_a      (test q, trial u)
 *       residual r[e'][l]           = int psi_l div u_h
 *   eval (both):  int p_h div u_h
 * u: [n_v][3] node-major (Eq. fe1c), p: [n_p].  transposed selects the second form. */
static int coupling_common(int pv, int pp, int q1d, int64_t n_elems, int64_t e0, int64_t e1) {
  if (pv < 1 || pv > 8 || pp < 1 || pp > 8 || q1d < 1 || q1d > 16 || n_elems < 0) return OR_ERR_ARG;
  if (e0 < 0 || e1 > n_elems || e0 > e1) return OR_ERR_ARG;
  return OR_OK;
}

/* mode 0: matrix (out = B or C); mode 1: residual (in = p or u, out = r); mode 2: eval */
static int coupling_run(int mode, int transposed, int pv, int pp, int q1d, int64_t n_elems,
                        const double *coords, const int32_t *conn, const int32_t *dof_v,
                        const int32_t *dof_p, const double *u, const double *p, int64_t e0,
                        int64_t e1, double *out, double *value) {
  int st = coupling_common(pv, pp, q1d, n_elems, e0, e1);
  if (st != OR_OK) return st;
  const int nv1 = pv + 1, nbv = nv1 * nv1 * nv1, np1 = pp + 1, nbp = np1 * np1 * np1;
  const int nq = q1d * q1d * q1d;
  double *xi = malloc(sizeof(double) * 3 * nq), *w = malloc(sizeof(double) * nq);
  double *Phi = malloc(sizeof(double) * nq * nbv), *dPhi = malloc(sizeof(double) * nq * 3 * nbv);
  double *xi2 = malloc(sizeof(double) * 3 * nq), *w2 = malloc(sizeof(double) * nq);
  double *Psi = malloc(sizeof(double) * nq * nbp), *dPsi = malloc(sizeof(double) * nq * 3 * nbp);
  oracle_tables(pv, q1d, xi, w, Phi, dPhi);
  oracle_tables(pp, q1d, xi2, w2, Psi, dPsi); /* same points: the shared rule */
  const int64_t osz = mode == 0 ? (int64_t)3 * nbv * nbp : (transposed ? nbp : 3 * nbv);
  int status = OR_OK;
  double total = 0.0;
  double *G = malloc(sizeof(double) * 3 * nbv);
  for (int64_t e = e0; e < e1 && status == OR_OK; ++e) {
    double *oe = out ? out + (e - e0) * osz : NULL;
    if (oe)
      for (int64_t i = 0; i < osz; ++i) oe[i] = 0.0;
    for (int q = 0; q < nq; ++q) {
      double J[3][3], Ji[3][3];
      double det = cell_jacobian(coords, conn + 8 * e, xi + 3 * q, J, Ji);
      if (!(det > 0.0)) { status = OR_ERR_DEGENERATE; g_bad_elem = e; break; }
      const double detw = w[q] * det;
      const double *psi = Psi + (int64_t)q * nbp;
      /* G[a][k] = dphi_k/dx_a = sum_m dPhi_m,k Jinv[m][a] */
      for (int a = 0; a < 3; ++a)
        for (int k = 0; k < nbv; ++k) {
          double s = 0.0;
          for (int m = 0; m < 3; ++m) s += dPhi[((int64_t)q * 3 + m) * nbv + k] * Ji[m][a];
          G[a * nbv + k] = s;
        }
      double ph = 0.0, divu = 0.0;
      if ((mode == 1 && !transposed) || mode == 2)
        for (int l = 0; l < nbp; ++l) ph += psi[l] * p[dof_p[e * nbp + l]];
      if ((mode == 1 && transposed) || mode == 2)
        for (int a = 0; a < 3; ++a)
          for (int k = 0; k < nbv; ++k) divu += G[a * nbv + k] * u[(int64_t)dof_v[e * nbv + k] * 3 + a];
      if (mode == 0) {
        for (int a = 0; a < 3; ++a)
          for (int k = 0; k < nbv; ++k)
            for (int l = 0; l < nbp; ++l) {
              const double v = detw * G[a * nbv + k] * psi[l];
              if (transposed) oe[(int64_t)l * 3 * nbv + a * nbv + k] += v;
              else oe[((int64_t)a * nbv + k) * nbp + l] += v;
            }
      } else if (mode == 1) {
        if (transposed)
          for (int l = 0; l < nbp; ++l) oe[l] += detw * psi[l] * divu;
        else
          for (int i = 0; i < 3 * nbv; ++i) oe[i] += detw * G[i] * ph;
      } else {
        total += detw * ph * divu;
      }
    }
  }
  free(G); free(xi); free(w); free(Phi); free(dPhi); free(xi2); free(w2); free(Psi); free(dPsi);
  if (status == OR_OK && mode == 2) *value = total;
  return status;
}

int oracle_coupling_matrix(int transposed, int pv, int pp, int q1d, int64_t n_elems,
                           const double *coords, const int32_t *conn, int64_t elem_begin,
                           int64_t elem_end, double *out) {
  if (!out) return OR_ERR_ARG;
  return coupling_run(0, transposed, pv, pp, q1d, n_elems, coords, conn, NULL, NULL, NULL, NULL,
                      elem_begin, elem_end, out, NULL);
}

int oracle_coupling_residual(int transposed, int pv, int pp, int q1d, int64_t n_elems,
                             const double *coords, const int32_t *conn, const int32_t *dof_v,
                             const int32_t *dof_p, const double *u, const double *p,
                             int64_t elem_begin, int64_t elem_end, double *r_elem) {
  if (!r_elem || (transposed ? (!u || !dof_v) : (!p || !dof_p))) return OR_ERR_ARG;
  return coupling_run(1, transposed, pv, pp, q1d, n_elems, coords, conn, dof_v, dof_p, u, p,
                      elem_begin, elem_end, r_elem, NULL);
}

int oracle_coupling_eval(int pv, int pp, int q1d, int64_t n_elems, const double *coords,
                         const int32_t *conn, const int32_t *dof_v, const int32_t *dof_p,
                         const double *u, const double *p, int64_t elem_begin, int64_t elem_end,
                         double *value) {
  if (!value || !u || !p || !dof_v || !dof_p) return OR_ERR_ARG;
  return coupling_run(2, 0, pv, pp, q1d, n_elems, coords, conn, dof_v, dof_p, u, p, elem_begin,
                      elem_end, NULL, value);
}
