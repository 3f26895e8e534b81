// Cauchy stress at the quadrature points (Tab. 2 'IK,s(k:l)->K'):
//   sigma[e][q][I] = sum_K D_IK(e, q) eps_K(u)(q),
//   eps = (du0/dx0, du1/dx1, du2/dx2, du0/dx1 + du1/dx0, du0/dx2 + du2/dx0, du1/dx2 + du2/dx1)
// (Voigt, engineering shears: DESIGN.md reading 7).  An "evaluated only" form (no test
// variable): no contraction against basis functions, one output per (cell, qp).
//
// One thread per (cell, qp).  A CTA stages CB cells at a time: the 8 vertex coordinates and
// the gathered nodal values u_e[3][NB] go to shared memory (each is read by all NQ threads
// of the cell); the reference-gradient table dphi[q][m][k] is read through L1 (shared by
// all cells).  Output rows of 6 doubles are contiguous in (cell, qp) order, so the stores
// of a warp cover one contiguous 48 B-per-thread range.
//
// INTEG: the paper's only mode for this form is 'eval', "returning the integral value"
// (P:806-813): sigma_int[e][I] = sum_q w_q det J_q sigma[e][q][I] (the integral of sigma over
// cell e; the domain integral is their sum).  The weighted per-qp values are staged in shared
// memory and summed over q in ascending order by one thread per (cell, I): deterministic.
#include "fe_device.cuh"
#include "fe_internal.h"

namespace feb200 {

template <int NB, int NQ>
struct StressL {
  static constexpr int THREADS = 128;
  static constexpr int CB = NQ >= THREADS ? 1 : THREADS / NQ;  // cells per CTA batch
  static constexpr int NT = (CB * NQ + 31) / 32 * 32;           // threads used
};

template <int NB, int NQ, bool INTEG>
__global__ void __launch_bounds__(128)
    k_stress(MeshView mv, int mat_kind, const double* __restrict__ ma, const double* __restrict__ mb,
             const double* __restrict__ u, int64_t e0, int64_t e1, double* __restrict__ sigma) {
  using L = StressL<NB, NQ>;
  constexpr int CB = L::CB;
  __shared__ double xv[CB][24];
  __shared__ double ue[CB][3][NB];
  __shared__ double acc[INTEG ? L::NT : 1][6];
  const int tid = threadIdx.x;
  for (int64_t eb = e0 + (int64_t)blockIdx.x * CB; eb < e1; eb += (int64_t)gridDim.x * CB) {
    const int ne = (int)((e1 - eb) < CB ? (e1 - eb) : CB);
    __syncthreads();
    for (int i = tid; i < ne * 24; i += blockDim.x) {
      const int c = i / 24, r = i - 24 * c;
      xv[c][r] = mv.coords[3 * (int64_t)mv.conn[8 * (eb + c) + r / 3] + r % 3];
    }
    for (int i = tid; i < ne * NB; i += blockDim.x) {
      const int c = i / NB, k = i - NB * c;
      const int64_t n = mv.dof_conn[(eb + c) * NB + k];
      ue[c][0][k] = u[3 * n];
      ue[c][1][k] = u[3 * n + 1];
      ue[c][2][k] = u[3 * n + 2];
    }
    __syncthreads();
    const int c = tid / NQ, q = tid - c * NQ;
    if (c < ne) {
    const int64_t e = eb + c;
    double Ji[9];
    const double det = hex_geometry(xv[c], mv.xi[3 * q], mv.xi[3 * q + 1], mv.xi[3 * q + 2], Ji);
    // reference gradient r[a][m] = sum_k dphi[q][m][k] u_e[a][k]
    double r[3][3] = {{0, 0, 0}, {0, 0, 0}, {0, 0, 0}};
    const double* dp = mv.dphi + (int64_t)q * 3 * NB;
#pragma unroll 3
    for (int k = 0; k < NB; ++k) {
      const double g0 = __ldg(dp + k), g1 = __ldg(dp + NB + k), g2 = __ldg(dp + 2 * NB + k);
#pragma unroll
      for (int a = 0; a < 3; ++a) {
        const double v = ue[c][a][k];
        r[a][0] = fma(g0, v, r[a][0]);
        r[a][1] = fma(g1, v, r[a][1]);
        r[a][2] = fma(g2, v, r[a][2]);
      }
    }
    // physical gradient gu[a][j] = sum_m r[a][m] Jinv[m][j]
    double gu[3][3];
#pragma unroll
    for (int a = 0; a < 3; ++a)
#pragma unroll
      for (int j = 0; j < 3; ++j) gu[a][j] = r[a][0] * Ji[j] + r[a][1] * Ji[3 + j] + r[a][2] * Ji[6 + j];
    const double eps[6] = {gu[0][0], gu[1][1], gu[2][2], gu[0][1] + gu[1][0], gu[0][2] + gu[2][0],
                           gu[1][2] + gu[2][1]};
    double s[6];
    if (mat_kind == FE_MAT_FULL_D) {
      const double* Dm = ma + (e * NQ + q) * 36;
#pragma unroll
      for (int I = 0; I < 6; ++I) {
        double t = 0.0;
#pragma unroll
        for (int K = 0; K < 6; ++K) t = fma(Dm[6 * I + K], eps[K], t);
        s[I] = t;
      }
    } else {
      const int64_t mi = mat_kind == FE_MAT_PER_ELEM ? e : e * NQ + q;
      const double lam = ma[mi], mu = mb[mi];
      const double tr = lam * (eps[0] + eps[1] + eps[2]);
      s[0] = tr + 2.0 * mu * eps[0];
      s[1] = tr + 2.0 * mu * eps[1];
      s[2] = tr + 2.0 * mu * eps[2];
      s[3] = mu * eps[3];
      s[4] = mu * eps[4];
      s[5] = mu * eps[5];
    }
    if constexpr (INTEG) {
      const double dw = mv.w[q] * det;
#pragma unroll
      for (int I = 0; I < 6; ++I) acc[tid][I] = dw * s[I];
    } else {
      double* o = sigma + ((e - e0) * NQ + q) * 6;
#pragma unroll
      for (int I = 0; I < 6; ++I) o[I] = s[I];
    }
    }  // c < ne
    if constexpr (INTEG) {
      __syncthreads();
      for (int i = tid; i < ne * 6; i += blockDim.x) {
        const int cc = i / 6, I = i - 6 * cc;
        double t = 0.0;
        for (int qq = 0; qq < NQ; ++qq) t += acc[cc * NQ + qq][I];
        sigma[(eb + cc - e0) * 6 + I] = t;
      }
    }
  }
}

template <int P, int Q>
static cudaError_t launch_stress_t(const fe_mesh* mh, MatArgs mat, const double* u, int64_t e0,
                                   int64_t e1, double* sigma, bool integ, cudaStream_t st) {
  constexpr int NB = (P + 1) * (P + 1) * (P + 1), NQ = Q * Q * Q;
  using L = StressL<NB, NQ>;
  auto kern = integ ? k_stress<NB, NQ, true> : k_stress<NB, NQ, false>;
  const LaunchFacts lf = launch_facts((const void*)kern, L::NT, 0);
  if (lf.err != cudaSuccess) return lf.err;
  const int nsm = lf.nsm, per_sm = lf.per_sm;
  const int64_t nb = (e1 - e0 + L::CB - 1) / L::CB;
  int grid = (int)(nb < (int64_t)nsm * per_sm ? nb : (int64_t)nsm * per_sm);
  grid = grid_cap(grid);
  if (grid <= 0) return cudaSuccess;
  kern<<<grid, L::NT, 0, st>>>(view_of(mh), mat.kind, (const double*)mat.a, (const double*)mat.b, u,
                               e0, e1, sigma);
  count_launch();
  return cudaGetLastError();
}

cudaError_t launch_stress(const fe_mesh* mh, MatArgs mat, const double* u, int64_t e0, int64_t e1,
                          double* sigma, bool integ, cudaStream_t st) {
  // the mesh's own quadrature (meshes are built with q1d = order + 1)
#define ST_CASE(P) \
  if (mh->order == P && mh->q1d == P + 1) return launch_stress_t<P, P + 1>(mh, mat, u, e0, e1, sigma, integ, st);
  ST_CASE(1) ST_CASE(2) ST_CASE(3) ST_CASE(4)
#undef ST_CASE
  return cudaErrorNotSupported;
}

}  // namespace feb200
