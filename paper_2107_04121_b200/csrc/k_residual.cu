// Residual mode (Alg. 1) with the gather of cell DOFs
// and the fused scatter-add into the global vector.
//
// One CTA per batch of NE cells (persistent grid).  With T the stacked table
// T[(q,0)][k] = phi_k(xi_q), T[(q,1+m)][k] = d phi_k/d xi_m (xi_q):
//   1. gather   U[k][(e,a)] = u[dof_conn[e][k]][a]                     (u.dofs 'cie')
//   2. forward  V = T U   -> u_h and reference gradients at every qp   (shared-A GEMM, N = batch)
//   3. pointwise, per (qp, cell): geometry (a1), physical gradient
//      du/dx = (du/dxi) J^-1, flux of the form, pulled back:
//        F[(q,0)] = detw f0,  F[(q,1+m)] = detw sum_j J^-1[m][j] f1_j
//   4. backward r_e = T^T F                                             (shared-A GEMM)
//   5. scatter  r_global[dof_conn[e][k]][a] += r_e[a][k]  (fp atomics), and/or r_elem.
// Fluxes: diffusion f1 = kappa grad u; mass f0 = rho u; mass+diffusion both;
// vector mass f0_a = rho u_a; elasticity f1 = sigma = D e(u) (Voigt,
// engineering shears, Psg of P:942); convective f0_a = (du_a/dx_j) u_j (Eq. fe2).
// fp64 GEMMs run on the FP64 tensor cores (DMMA); the fp32 variant uses FFMA
// with geometry still computed from the fp64 coordinates.
#include <algorithm>
#include <cstdlib>
#include <cstring>

#include "fe_device.cuh"
#include "fe_flux.cuh"
#include "fe_internal.h"

namespace feb200 {

template <int FORM>
struct RForm {
  static constexpr int D = FormD<FORM>::D;
};

template <int P, int FORM>
struct ResLayout {
  static constexpr int Q = P + 1, NB = (P + 1) * (P + 1) * (P + 1), NQ = Q * Q * Q;
  static constexpr int D = RForm<FORM>::D;
  static constexpr int NE = D == 1 ? (P >= 4 ? 8 : 32) : (P >= 4 ? 4 : 16);
  static constexpr int NCOL = D * NE;
  static constexpr int M4 = 4 * NQ;
};

template <int P, int FORM, typename T>
__global__ void __launch_bounds__(256) k_residual(MeshView m, int mat_kind, const T* __restrict__ ma,
                                                  const T* __restrict__ mb, const T* __restrict__ u,
                                                  int64_t e0, int64_t e1, T* __restrict__ r_elem,
                                                  T* __restrict__ r_global) {
  using L = ResLayout<P, FORM>;
  constexpr int NB = L::NB, NQ = L::NQ, D = L::D, NE = L::NE, NCOL = L::NCOL, M4 = L::M4;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double* xv = reinterpret_cast<double*>(smem_raw);                 // [NE][24]
  int32_t* dc = reinterpret_cast<int32_t*>(xv + NE * 24);           // [NE][NB]
  T* U = reinterpret_cast<T*>(smem_raw + ((NE * 24 * 8 + NE * NB * 4 + 15) & ~15));  // [NB][NCOL]
  T* V = U + NB * NCOL;                                             // [M4][NCOL]
  const T* fwd;
  const T* bwd;
  if constexpr (sizeof(T) == 8) { fwd = (const T*)m.fwd; bwd = (const T*)m.bwd; }
  else { fwd = (const T*)m.fwd_f; bwd = (const T*)m.bwd_f; }
  const int tid = threadIdx.x, nthr = blockDim.x;
  const int lane = tid & 31, warp = tid >> 5, nwarps = nthr >> 5;
  const int64_t nbatch = (e1 - e0 + NE - 1) / NE;

  for (int64_t bidx = blockIdx.x; bidx < nbatch; bidx += gridDim.x) {
    const int64_t eb = e0 + bidx * NE;
    const int ne = (int)((e1 - eb) < NE ? (e1 - eb) : NE);
    for (int idx = tid; idx < NE * NB; idx += nthr) {
      const int el = idx / NB;
      dc[idx] = el < ne ? m.dof_conn[(eb + el) * NB + (idx - el * NB)] : 0;
    }
    for (int idx = tid; idx < NE * 24; idx += nthr) {
      const int el = idx / 24, r = idx - el * 24;
      xv[idx] = el < ne ? m.coords[3 * (int64_t)m.conn[8 * (eb + el) + r / 3] + r % 3] : 0.0;
    }
    __syncthreads();
    for (int idx = tid; idx < NB * NCOL; idx += nthr) {
      const int k = idx / NCOL, n = idx - k * NCOL;
      const int el = n / D, a = n - el * D;
      U[idx] = el < ne ? u[(int64_t)dc[el * NB + k] * D + a] : T(0);
    }
    __syncthreads();
    // forward: V[(q,c)][n] = sum_k T[(q,c)][k] U[k][n]
    if constexpr (sizeof(T) == 8) {
      Seg s{(const double*)fwd, (const double*)U, nullptr, M4, NCOL, NB};
      seg_gemm<4>(&s, 1, M4, NCOL, warp, nwarps, lane,
                  [&](int r, int c, double v) { V[r * NCOL + c] = v; });
    } else {
      const T* As[1] = {fwd};
      const T* Bs[1] = {U};
      const int ar[1] = {M4}, br[1] = {NCOL}, cn[1] = {NB};
      seg_gemm_simt<T>(As, Bs, ar, br, cn, 1, M4, NCOL, tid, nthr,
                       [&](int r, int c, T v) { V[r * NCOL + c] = v; });
    }
    __syncthreads();
    // pointwise flux at every (qp, cell)
    for (int idx = tid; idx < NQ * NE; idx += nthr) {
      const int el = idx / NQ, q = idx - el * NQ;
      if (el >= ne) {
        for (int c = 0; c < 4; ++c)
          for (int a = 0; a < D; ++a) V[(4 * q + c) * NCOL + el * D + a] = T(0);
        continue;
      }
      const int64_t e = eb + el;
      double Ji[9];
      const double det = hex_geometry(xv + 24 * el, m.xi[3 * q], m.xi[3 * q + 1], m.xi[3 * q + 2], Ji);
      const double dw = m.w[q] * det;
      double uq[D], gr[D][3];  // value and reference gradient
#pragma unroll
      for (int a = 0; a < D; ++a) {
        uq[a] = (double)V[(4 * q) * NCOL + el * D + a];
#pragma unroll
        for (int mm = 0; mm < 3; ++mm) gr[a][mm] = (double)V[(4 * q + 1 + mm) * NCOL + el * D + a];
      }
      double gu[D][3];  // du_a/dx_j = sum_m gr[a][m] Jinv[m][j]
#pragma unroll
      for (int a = 0; a < D; ++a)
#pragma unroll
        for (int j = 0; j < 3; ++j) gu[a][j] = gr[a][0] * Ji[j] + gr[a][1] * Ji[3 + j] + gr[a][2] * Ji[6 + j];
      double f0[D], f1[D][3];
      qp_flux<FORM, T>(uq, gu, e, q, NQ, mat_kind, ma, mb, f0, f1);
#pragma unroll
      for (int a = 0; a < D; ++a) {
        V[(4 * q) * NCOL + el * D + a] = (T)(dw * f0[a]);
#pragma unroll
        for (int mm = 0; mm < 3; ++mm)
          V[(4 * q + 1 + mm) * NCOL + el * D + a] =
              (T)(dw * (Ji[3 * mm] * f1[a][0] + Ji[3 * mm + 1] * f1[a][1] + Ji[3 * mm + 2] * f1[a][2]));
      }
    }
    __syncthreads();
    // backward: r[k][n] = sum_{(q,c)} T[(q,c)][k] F[(q,c)][n]; fused scatter
    auto epi = [&](int k, int n, T v) {
      const int el = n / D, a = n - el * D;
      if (el < ne) {
        if (r_elem) r_elem[(eb + el - e0) * (int64_t)(D * NB) + a * NB + k] = v;
        if (r_global) atomic_add(r_global + (int64_t)dc[el * NB + k] * D + a, v);
      }
    };
    if constexpr (sizeof(T) == 8) {
      Seg s{(const double*)bwd, (const double*)V, nullptr, NB, NCOL, M4};
      seg_gemm<2>(&s, 1, NB, NCOL, warp, nwarps, lane, epi);
    } else {
      const T* As[1] = {bwd};
      const T* Bs[1] = {V};
      const int ar[1] = {NB}, br[1] = {NCOL}, cn[1] = {M4};
      seg_gemm_simt<T>(As, Bs, ar, br, cn, 1, NB, NCOL, tid, nthr, epi);
    }
    __syncthreads();
  }
}

template <int P, int FORM, typename T>
static cudaError_t launch_res_t(const fe_mesh* mh, MatArgs mat, const T* u, int64_t e0, int64_t e1,
                                T* r_elem, T* r_global, cudaStream_t st) {
  using L = ResLayout<P, FORM>;
  const size_t head = (L::NE * 24 * 8 + L::NE * L::NB * 4 + 15) & ~size_t(15);
  const size_t bytes = head + sizeof(T) * size_t(L::NB + L::M4) * L::NCOL;
  if (bytes > 227 * 1024) return cudaErrorNotSupported;
  auto kern = k_residual<P, FORM, T>;
  const LaunchFacts lf = launch_facts((const void*)kern, 256, bytes);
  if (lf.err != cudaSuccess) return lf.err;
  const int nsm = lf.nsm, per_sm = lf.per_sm;
  const int64_t nbatch = (e1 - e0 + L::NE - 1) / L::NE;
  int grid = (int)std::min<int64_t>(nbatch, (int64_t)nsm * per_sm);
  grid = grid_cap(grid);
  if (grid <= 0) return cudaSuccess;
  kern<<<grid, 256, bytes, st>>>(view_of(mh), mat.kind, (const T*)mat.a, (const T*)mat.b, u, e0, e1,
                                 r_elem, r_global);
  count_launch();
  return cudaGetLastError();
}

template <int P, typename T>
static cudaError_t res_form(const fe_mesh* mh, int form, MatArgs mat, const T* u, int64_t e0,
                            int64_t e1, T* re, T* rg, cudaStream_t st) {
  switch (form) {
    case FE_FORM_DIFFUSION: return launch_res_t<P, FE_FORM_DIFFUSION, T>(mh, mat, u, e0, e1, re, rg, st);
    case FE_FORM_MASS: return launch_res_t<P, FE_FORM_MASS, T>(mh, mat, u, e0, e1, re, rg, st);
    case FE_FORM_MASS_DIFFUSION: return launch_res_t<P, FE_FORM_MASS_DIFFUSION, T>(mh, mat, u, e0, e1, re, rg, st);
    default: break;
  }
  if constexpr (sizeof(T) == 8) {
    switch (form) {
      case FE_FORM_VECTOR_MASS: return launch_res_t<P, FE_FORM_VECTOR_MASS, T>(mh, mat, u, e0, e1, re, rg, st);
      case FE_FORM_ELASTICITY: return launch_res_t<P, FE_FORM_ELASTICITY, T>(mh, mat, u, e0, e1, re, rg, st);
      case FE_FORM_CONVECTIVE: return launch_res_t<P, FE_FORM_CONVECTIVE, T>(mh, mat, u, e0, e1, re, rg, st);
      case FE_FORM_WEIGHTED_DOT: return launch_res_t<P, FE_FORM_WEIGHTED_DOT, T>(mh, mat, u, e0, e1, re, rg, st);
      case FE_FORM_DIVERGENCE: return launch_res_t<P, FE_FORM_DIVERGENCE, T>(mh, mat, u, e0, e1, re, rg, st);
      default: break;
    }
  }
  return cudaErrorNotSupported;
}

template <typename T>
static cudaError_t res_dispatch(const fe_mesh* mh, int form, MatArgs mat, const T* u, int64_t e0,
                                int64_t e1, T* re, T* rg, cudaStream_t st) {
  if (mh->q1d != mh->order + 1) return cudaErrorNotSupported;
  switch (mh->order) {
    case 1: return res_form<1, T>(mh, form, mat, u, e0, e1, re, rg, st);
    case 2: return res_form<2, T>(mh, form, mat, u, e0, e1, re, rg, st);
    case 3: return res_form<3, T>(mh, form, mat, u, e0, e1, re, rg, st);
    case 4: return res_form<4, T>(mh, form, mat, u, e0, e1, re, rg, st);
  }
  return cudaErrorNotSupported;
}

// sum-factorised kernels first; FE_OPT_RESIDUAL_IMPL = dense selects the dense DMMA kernels
static bool want_dense_residual() { return option(FE_OPT_RESIDUAL_IMPL) == RESIDUAL_DENSE; }

// FE_OPT_RESIDUAL_IMPL = sf keeps the shared-memory sum-factorised kernel for every form
bool want_residual_t3() { return option(FE_OPT_RESIDUAL_IMPL) == RESIDUAL_DEFAULT; }

cudaError_t launch_residual_f64(const fe_mesh* m, int form, MatArgs mat, const double* u,
                                int64_t e0, int64_t e1, double* r_elem, double* r_global,
                                cudaStream_t st) {
  if (!want_dense_residual()) {
    cudaError_t e = cudaErrorNotSupported;
    if (want_residual_t3()) e = launch_residual_t3(m, form, mat, u, e0, e1, r_elem, r_global, st);
    if (e != cudaErrorNotSupported) return e;
    e = launch_residual_sf<double>(m, form, mat, u, e0, e1, r_elem, r_global, st);
    if (e != cudaErrorNotSupported) return e;
  }
  return res_dispatch<double>(m, form, mat, u, e0, e1, r_elem, r_global, st);
}

cudaError_t launch_residual_f32(const fe_mesh* m, int form, MatArgs mat, const float* u,
                                int64_t e0, int64_t e1, float* r_elem, float* r_global,
                                cudaStream_t st) {
  if (!want_dense_residual()) {
    cudaError_t e = launch_residual_sf<float>(m, form, mat, u, e0, e1, r_elem, r_global, st);
    if (e != cudaErrorNotSupported) return e;
  }
  return res_dispatch<float>(m, form, mat, u, e0, e1, r_elem, r_global, st);
}

}  // namespace feb200
