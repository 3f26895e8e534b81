// Matrix mode (Alg. 2): K_e = sum_q detw(q) dF/du for
// every cell of a range, one CTA per cell at a time (persistent grid).
//
// Per cell:
//   a1  geometry at every qp from the 8 vertices (J, det J, J^-1)
//   b   physical gradients G[q][j][k] = sum_m dphi[q][m][k] J^-1[m][j]
//   c1  the form's contraction as FP64 tensor-core GEMMs (mma.sync m8n8k4 ->
//       DMMA) with the contraction index running over (qp, component):
//         diffusion    K = sum_{q,j} (detw kappa G_j)^T G_j          ('cq,cqjd,cqje->cde' P:955)
//         mass         K = sum_q (detw rho phi)^T phi
//         vector mass  scalar mass on the D diagonal blocks
//         elasticity   K_ab = sum_{q,j} G_j^T H^ab_j,  H^ab_j = sum_l C_ajbl G_l,
//                      C_ajbl = detw D[I(a,j)][I(b,l)]  (Psg contracted analytically,
//                      'cq,cqje,rjI,cqIK,cqlf,slK->cresf' P:1033)
//         convective   K_ab = sum_q phi^T detw (delta_ab (u.G) + d_b u_a phi)  (Eq. fe4)
// Output K[e - e0][a*nb + k][b*nb + l] written straight from the MMA fragments.
#include <algorithm>
#include <cstdlib>
#include <cstring>

#include "fe_device.cuh"
#include "fe_internal.h"

namespace feb200 {

__device__ __forceinline__ int voigt_index(int a, int j) {
  // (xx, yy, zz, xy, xz, yz)
  return a == j ? a : (a + j == 1 ? 3 : (a + j == 2 ? 4 : 5));
}

template <int FORM>
struct FormInfo {
  static constexpr int D = (FORM == FE_FORM_VECTOR_MASS || FORM == FE_FORM_ELASTICITY ||
                            FORM == FE_FORM_CONVECTIVE || FORM == FE_FORM_WEIGHTED_DOT) ? 3 : 1;
};

template <int P, int FORM>
struct MatLayout {
  static constexpr int Q = P + 1, NB = (P + 1) * (P + 1) * (P + 1), NQ = Q * Q * Q;
  static constexpr int D = FormInfo<FORM>::D, NDOF = D * NB;
  static constexpr bool NEED_G = FORM != FE_FORM_MASS && FORM != FE_FORM_VECTOR_MASS &&
                                 FORM != FE_FORM_WEIGHTED_DOT;
  // offsets in doubles
  static constexpr int XV = 0;
  static constexpr int JINV = XV + 24;
  static constexpr int DETW = JINV + 9 * NQ;
  static constexpr int WT = DETW + NQ;                      // row weights, 4 NQ
  static constexpr int G = WT + 4 * NQ;                     // [NQ][3][NB]
  static constexpr int X1 = G + (NEED_G ? 3 * NQ * NB : 0); // form scratch 1
  // elasticity: the C_ajbl of one block (a, b) at a time, [NQ][9]
  static constexpr int X1_SIZE = FORM == FE_FORM_ELASTICITY ? 9 * NQ
                                 : FORM == FE_FORM_CONVECTIVE ? (3 * NB + 12 * NQ + NQ * NB) : 0;
  static constexpr int X2 = X1 + X1_SIZE;                   // form scratch 2
  static constexpr int X2_SIZE = FORM == FE_FORM_ELASTICITY ? 3 * NQ * NB
                                 : FORM == FE_FORM_CONVECTIVE ? NQ * NB : 0;
  static constexpr int TOTAL = X2 + X2_SIZE;
  static constexpr size_t BYTES = size_t(TOTAL) * sizeof(double);
};

template <int P, int FORM>
__global__ void __launch_bounds__(256) k_matrix(MeshView m, int mat_kind, const double* __restrict__ ma,
                                                const double* __restrict__ mb,
                                                const double* __restrict__ state_u, int64_t e0,
                                                int64_t e1, double* __restrict__ K) {
  using L = MatLayout<P, FORM>;
  constexpr int NB = L::NB, NQ = L::NQ, NDOF = L::NDOF;
  extern __shared__ double smem[];
  double* xv = smem + L::XV;
  double* jinv = smem + L::JINV;
  double* detw = smem + L::DETW;
  double* wt = smem + L::WT;
  double* G = smem + L::G;
  double* X1 = smem + L::X1;
  double* X2 = smem + L::X2;
  const int tid = threadIdx.x, nthr = blockDim.x;
  const int lane = tid & 31, warp = tid >> 5, nwarps = nthr >> 5;

  for (int64_t e = e0 + blockIdx.x; e < e1; e += gridDim.x) {
    double* Ke = K + (e - e0) * (int64_t)NDOF * NDOF;
    if (tid < 24) xv[tid] = m.coords[3 * (int64_t)m.conn[8 * e + tid / 3] + tid % 3];
    __syncthreads();
    for (int q = tid; q < NQ; q += nthr) {
      double Ji[9];
      const double det = hex_geometry(xv, m.xi[3 * q], m.xi[3 * q + 1], m.xi[3 * q + 2], Ji);
#pragma unroll
      for (int i = 0; i < 9; ++i) jinv[9 * q + i] = Ji[i];
      detw[q] = m.w[q] * det;
    }
    __syncthreads();
    if constexpr (L::NEED_G) {
      for (int idx = tid; idx < NQ * NB; idx += nthr) {
        const int q = idx / NB, k = idx - q * NB;
        const double g0 = m.dphi[(3 * q + 0) * NB + k], g1 = m.dphi[(3 * q + 1) * NB + k],
                     g2 = m.dphi[(3 * q + 2) * NB + k];
        const double* Ji = jinv + 9 * q;
#pragma unroll
        for (int j = 0; j < 3; ++j) G[(3 * q + j) * NB + k] = g0 * Ji[j] + g1 * Ji[3 + j] + g2 * Ji[6 + j];
      }
    }

    if constexpr (FORM == FE_FORM_DIFFUSION || FORM == FE_FORM_MASS ||
                  FORM == FE_FORM_MASS_DIFFUSION || FORM == FE_FORM_VECTOR_MASS) {
      for (int q = tid; q < NQ; q += nthr) {
        const double a = ma[e * NQ + q] * detw[q];
        if constexpr (FORM == FE_FORM_DIFFUSION) {
          wt[3 * q] = a; wt[3 * q + 1] = a; wt[3 * q + 2] = a;
        } else if constexpr (FORM == FE_FORM_MASS_DIFFUSION) {
          const double b = mb[e * NQ + q] * detw[q];
          wt[q] = a;
          wt[NQ + 3 * q] = b; wt[NQ + 3 * q + 1] = b; wt[NQ + 3 * q + 2] = b;
        } else {
          wt[q] = a;
        }
      }
      __syncthreads();
      Seg segs[2];
      int nseg = 0;
      if constexpr (FORM == FE_FORM_DIFFUSION) {
        segs[nseg++] = Seg{G, G, wt, NB, NB, 3 * NQ};
      } else if constexpr (FORM == FE_FORM_MASS_DIFFUSION) {
        segs[nseg++] = Seg{m.phi, m.phi, wt, NB, NB, NQ};
        segs[nseg++] = Seg{G, G, wt + NQ, NB, NB, 3 * NQ};
      } else {
        segs[nseg++] = Seg{m.phi, m.phi, wt, NB, NB, NQ};
      }
      if constexpr (FORM == FE_FORM_VECTOR_MASS) {
        seg_gemm<2>(segs, nseg, NB, NB, warp, nwarps, lane, [&](int r, int c, double v) {
#pragma unroll
          for (int a = 0; a < 3; ++a) Ke[(int64_t)(a * NB + r) * NDOF + a * NB + c] = v;
        });
        for (int idx = tid; idx < 6 * NB * NB; idx += nthr) {
          const int blk = idx / (NB * NB), rem = idx - blk * NB * NB;
          const int a = blk / 2, b = (blk % 2 == 0) ? (a + 1) % 3 : (a + 2) % 3;
          const int r = rem / NB, c = rem - r * NB;
          Ke[(int64_t)(a * NB + r) * NDOF + b * NB + c] = 0.0;
        }
      } else {
        seg_gemm<2>(segs, nseg, NB, NB, warp, nwarps, lane,
                    [&](int r, int c, double v) { Ke[(int64_t)r * NDOF + c] = v; });
      }
      __syncthreads();
    } else if constexpr (FORM == FE_FORM_WEIGHTED_DOT) {
      // K_ab = sum_q detw M_ab(q) phi phi^T ('ij,i,j'): nine weighted mass blocks
      for (int a = 0; a < 3; ++a)
        for (int b = 0; b < 3; ++b) {
          for (int q = tid; q < NQ; q += nthr) wt[q] = detw[q] * ma[(e * NQ + q) * 9 + 3 * a + b];
          __syncthreads();
          Seg s{m.phi, m.phi, wt, NB, NB, NQ};
          seg_gemm<2>(&s, 1, NB, NB, warp, nwarps, lane, [&](int r, int c, double v) {
            Ke[(int64_t)(a * NB + r) * NDOF + b * NB + c] = v;
          });
          __syncthreads();
        }
    } else if constexpr (FORM == FE_FORM_ELASTICITY) {
      double* Cab = X1;  // [NQ][9]: C[a][j][b][l] = detw D[I(a,j)][I(b,l)] of the current (a, b)
      double* H = X2;    // [NQ][3][NB]
      for (int a = 0; a < 3; ++a)
        for (int b = 0; b < 3; ++b) {
          for (int idx = tid; idx < NQ * 9; idx += nthr) {
            const int q = idx / 9, j = (idx / 3) % 3, l = idx % 3;
            const int I = voigt_index(a, j), Kv = voigt_index(b, l);
            double dik;
            if (mat_kind == FE_MAT_FULL_D) {
              dik = ma[(e * NQ + q) * 36 + 6 * I + Kv];
            } else {
              const double lam = mat_kind == FE_MAT_PER_ELEM ? ma[e] : ma[e * NQ + q];
              const double mu = mat_kind == FE_MAT_PER_ELEM ? mb[e] : mb[e * NQ + q];
              dik = (I < 3 && Kv < 3 ? lam : 0.0) + (I == Kv ? (I < 3 ? 2.0 * mu : mu) : 0.0);
            }
            Cab[idx] = detw[q] * dik;
          }
          __syncthreads();
          for (int idx = tid; idx < NQ * 3 * NB; idx += nthr) {
            const int q = idx / (3 * NB), r = idx - q * 3 * NB;
            const int j = r / NB, k = r - j * NB;
            const double* C = Cab + q * 9 + j * 3;
            const double* Gq = G + 3 * q * NB + k;
            H[idx] = C[0] * Gq[0] + C[1] * Gq[NB] + C[2] * Gq[2 * NB];
          }
          __syncthreads();
          Seg s{G, H, nullptr, NB, NB, 3 * NQ};
          seg_gemm<2>(&s, 1, NB, NB, warp, nwarps, lane, [&](int r, int c, double v) {
            Ke[(int64_t)(a * NB + r) * NDOF + b * NB + c] = v;
          });
          __syncthreads();
        }
    } else {  // FE_FORM_CONVECTIVE, Eq. fe4
      double* ue = X1;                  // [3][NB]
      double* uq = ue + 3 * NB;         // [NQ][3]
      double* gu = uq + 3 * NQ;         // [NQ][9], gu[a][j] = du_a/dx_j
      double* UG = gu + 9 * NQ;         // [NQ][NB], (u . G)_l
      double* Bab = X2;                 // [NQ][NB]
      for (int idx = tid; idx < 3 * NB; idx += nthr) {
        const int a = idx / NB, k = idx - a * NB;
        ue[idx] = state_u[3 * (int64_t)m.dof_conn[e * NB + k] + a];
      }
      __syncthreads();
      for (int idx = tid; idx < NQ * 12; idx += nthr) {
        const int q = idx / 12, r = idx - q * 12;
        double s = 0.0;
        if (r < 3) {
          for (int k = 0; k < NB; ++k) s += ue[r * NB + k] * m.phi[q * NB + k];
          uq[3 * q + r] = s;
        } else {
          const int a = (r - 3) / 3, j = (r - 3) % 3;
          for (int k = 0; k < NB; ++k) s += ue[a * NB + k] * G[(3 * q + j) * NB + k];
          gu[9 * q + 3 * a + j] = s;
        }
      }
      __syncthreads();
      for (int idx = tid; idx < NQ * NB; idx += nthr) {
        const int q = idx / NB, l = idx - q * NB;
        UG[idx] = uq[3 * q] * G[(3 * q) * NB + l] + uq[3 * q + 1] * G[(3 * q + 1) * NB + l] +
                  uq[3 * q + 2] * G[(3 * q + 2) * NB + l];
      }
      __syncthreads();
      for (int a = 0; a < 3; ++a)
        for (int b = 0; b < 3; ++b) {
          for (int idx = tid; idx < NQ * NB; idx += nthr) {
            const int q = idx / NB, l = idx - q * NB;
            double v = gu[9 * q + 3 * a + b] * m.phi[idx];
            if (a == b) v += UG[idx];
            Bab[idx] = detw[q] * v;
          }
          __syncthreads();
          Seg s{m.phi, Bab, nullptr, NB, NB, NQ};
          seg_gemm<2>(&s, 1, NB, NB, warp, nwarps, lane, [&](int r, int c, double v) {
            Ke[(int64_t)(a * NB + r) * NDOF + b * NB + c] = v;
          });
          __syncthreads();
        }
    }
    __syncthreads();
  }
}

template <int P, int FORM>
static cudaError_t launch_matrix_t(const fe_mesh* mh, MatArgs mat, const double* state_u,
                                   int64_t e0, int64_t e1, double* K, cudaStream_t st) {
  using L = MatLayout<P, FORM>;
  if (L::BYTES > 227 * 1024) return cudaErrorNotSupported;
  auto kern = k_matrix<P, FORM>;
  const LaunchFacts lf = launch_facts((const void*)kern, 256, L::BYTES);
  if (lf.err != cudaSuccess) return lf.err;
  const int nsm = lf.nsm, per_sm = lf.per_sm;
  const int64_t n = e1 - e0;
  int grid = (int)std::min<int64_t>(n, (int64_t)nsm * per_sm);
  grid = grid_cap(grid);
  if (grid <= 0) return cudaSuccess;
  kern<<<grid, 256, L::BYTES, st>>>(view_of(mh), mat.kind, (const double*)mat.a,
                                    (const double*)mat.b, state_u, e0, e1, K);
  count_launch();
  return cudaGetLastError();
}

template <int P>
static cudaError_t dispatch_form(const fe_mesh* mh, int form, MatArgs mat, const double* state_u,
                                 int64_t e0, int64_t e1, double* K, cudaStream_t st) {
  switch (form) {
    case FE_FORM_DIFFUSION: return launch_matrix_t<P, FE_FORM_DIFFUSION>(mh, mat, state_u, e0, e1, K, st);
    case FE_FORM_MASS: return launch_matrix_t<P, FE_FORM_MASS>(mh, mat, state_u, e0, e1, K, st);
    case FE_FORM_VECTOR_MASS: return launch_matrix_t<P, FE_FORM_VECTOR_MASS>(mh, mat, state_u, e0, e1, K, st);
    case FE_FORM_MASS_DIFFUSION: return launch_matrix_t<P, FE_FORM_MASS_DIFFUSION>(mh, mat, state_u, e0, e1, K, st);
    case FE_FORM_ELASTICITY: return launch_matrix_t<P, FE_FORM_ELASTICITY>(mh, mat, state_u, e0, e1, K, st);
    case FE_FORM_CONVECTIVE: return launch_matrix_t<P, FE_FORM_CONVECTIVE>(mh, mat, state_u, e0, e1, K, st);
    case FE_FORM_WEIGHTED_DOT: return launch_matrix_t<P, FE_FORM_WEIGHTED_DOT>(mh, mat, state_u, e0, e1, K, st);
  }
  return cudaErrorNotSupported;
}

cudaError_t launch_matrix(const fe_mesh* mh, int form, MatArgs mat, const double* state_u,
                          int64_t e0, int64_t e1, double* K, cudaStream_t st) {
  if (mh->q1d != mh->order + 1) return cudaErrorNotSupported;
  // sum-factorised kernels first; FE_OPT_MATRIX_IMPL = dense selects the dense DMMA kernels
  if (option(FE_OPT_MATRIX_IMPL) != MATRIX_DENSE) {
    cudaError_t e = launch_matrix_sf(mh, form, mat, e0, e1, K, st);
    if (e != cudaErrorNotSupported) return e;
    e = launch_matrix_vp(mh, form, mat, state_u, e0, e1, K, st);
    if (e != cudaErrorNotSupported) return e;
    e = launch_matrix_sfv(mh, form, mat, state_u, e0, e1, K, st);
    if (e != cudaErrorNotSupported) return e;
  }
  switch (mh->order) {
    case 1: return dispatch_form<1>(mh, form, mat, state_u, e0, e1, K, st);
    case 2: return dispatch_form<2>(mh, form, mat, state_u, e0, e1, K, st);
    case 3: return dispatch_form<3>(mh, form, mat, state_u, e0, e1, K, st);
  }
  return cudaErrorNotSupported;
}

}  // namespace feb200
