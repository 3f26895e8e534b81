// Mixed velocity-pressure forms (Tab. 2) on a Q_PV x Q_PP pair sharing
// the mesh's quadrature (reading 19):
//   Stokes coupling            ('i.i,0', v, p):  int (dv_i/dx_i) p
//   transposed Stokes coupling ('i.i,0', u, q):  int q (du_i/dx_i)
// Every entry is a sum over qps of W_{ma}(q) D^m_k(q) psi_l(q) with the per-qp weights
// W_{ma} = detw Jinv[m][a] (the physical gradient dphi_k/dx_a = sum_m Jinv[m][a] dphi_k/dxi_m,
// P:655-658, with the quadrature weight folded into the determinant).
//
// Organisation: a CTA takes CB cells (CB * NQ <= 256).  Phase 1, one thread per (cell, qp):
// geometry -> W[q][9] and detw in shared memory, plus the interpolated fields the mode needs
// (p_h(q) from the gathered pressure, div u_h(q) from the gathered velocity).  Phase 2, one
// thread per (cell, output entry): the qp sum against the reference tables (dphi of the
// velocity space, psi of the pressure space; read through L1, shared by all cells), written
// contiguously per cell; residuals are scatter-added into the global vector with fp atomics.
// These kernels are outside the BASELINE.json configs; they are the plain batched form of the
// operation (no sum factorisation).
#include "fe_device.cuh"
#include "fe_internal.h"

namespace feb200 {

enum { CPL_MATRIX = 0, CPL_RESIDUAL = 1, CPL_EVAL = 2 };

template <int PV, int PP>
struct CplL {
  static constexpr int NBV = (PV + 1) * (PV + 1) * (PV + 1), NBP = (PP + 1) * (PP + 1) * (PP + 1);
  static constexpr int NQ = (PV + 1) * (PV + 1) * (PV + 1);
  static constexpr int THREADS = 256;
  static constexpr int CB = NQ >= THREADS ? 1 : THREADS / NQ;
};

template <int PV, int PP, int MODE, bool TRANS>
__global__ void __launch_bounds__(256)
    k_coupling(MeshView mv, const int32_t* __restrict__ pdof, const double* __restrict__ psi,
               const double* __restrict__ u, const double* __restrict__ p, int64_t e0, int64_t e1,
               double* __restrict__ out, double* __restrict__ r_global, double* __restrict__ value) {
  using L = CplL<PV, PP>;
  constexpr int NBV = L::NBV, NBP = L::NBP, NQ = L::NQ, CB = L::CB;
  constexpr bool NEED_P = MODE == CPL_EVAL || (MODE == CPL_RESIDUAL && !TRANS);
  constexpr bool NEED_U = MODE == CPL_EVAL || (MODE == CPL_RESIDUAL && TRANS);
  constexpr int NOUT = MODE == CPL_MATRIX ? 3 * NBV * NBP : (TRANS ? NBP : 3 * NBV);
  __shared__ double xv[CB][24];
  __shared__ double W[CB][NQ][10];  // detw Jinv[m][a] at 3m + a, detw at 9
  __shared__ double fq[CB][NQ];     // p_h(q) (Stokes residual) or detw div u_h(q) (transposed)
  __shared__ double ue[NEED_U ? CB : 1][3][NBV];
  __shared__ double pe[NEED_P ? CB : 1][NBP];
  const int tid = threadIdx.x;
  double ev = 0.0;
  for (int64_t eb = e0 + (int64_t)blockIdx.x * CB; eb < e1; eb += (int64_t)gridDim.x * CB) {
    const int ne = (int)((e1 - eb) < CB ? (e1 - eb) : CB);
    __syncthreads();
    for (int i = tid; i < ne * 24; i += blockDim.x) {
      const int c = i / 24, r = i - 24 * c;
      xv[c][r] = mv.coords[3 * (int64_t)mv.conn[8 * (eb + c) + r / 3] + r % 3];
    }
    if constexpr (NEED_U) {
      for (int i = tid; i < ne * NBV; i += blockDim.x) {
        const int c = i / NBV, k = i - NBV * c;
        const int64_t n = mv.dof_conn[(eb + c) * NBV + k];
        ue[c][0][k] = u[3 * n];
        ue[c][1][k] = u[3 * n + 1];
        ue[c][2][k] = u[3 * n + 2];
      }
    }
    if constexpr (NEED_P) {
      for (int i = tid; i < ne * NBP; i += blockDim.x) {
        const int c = i / NBP, l = i - NBP * c;
        pe[c][l] = p[pdof[(eb + c) * NBP + l]];
      }
    }
    __syncthreads();
    // ---- phase 1: one thread per (cell, qp)
    for (int i = tid; i < ne * NQ; i += blockDim.x) {
      const int c = i / NQ, q = i - NQ * c;
      double Ji[9];
      const double det = hex_geometry(xv[c], mv.xi[3 * q], mv.xi[3 * q + 1], mv.xi[3 * q + 2], Ji);
      const double dw = mv.w[q] * det;
#pragma unroll
      for (int j = 0; j < 9; ++j) W[c][q][j] = dw * Ji[j];
      W[c][q][9] = dw;
      double ph = 0.0, du = 0.0;
      if constexpr (NEED_P) {
        const double* ps = psi + (int64_t)q * NBP;
        for (int l = 0; l < NBP; ++l) ph = fma(__ldg(ps + l), pe[c][l], ph);
      }
      if constexpr (NEED_U) {
        // div u = sum_a sum_m Jinv[m][a] (d u_a / d xi_m)
        const double* dp = mv.dphi + (int64_t)q * 3 * NBV;
        double r[3][3] = {{0, 0, 0}, {0, 0, 0}, {0, 0, 0}};
        for (int k = 0; k < NBV; ++k) {
          const double g0 = __ldg(dp + k), g1 = __ldg(dp + NBV + k), g2 = __ldg(dp + 2 * NBV + k);
#pragma unroll
          for (int a = 0; a < 3; ++a) {
            const double v = ue[c][a][k];
            r[a][0] = fma(g0, v, r[a][0]);
            r[a][1] = fma(g1, v, r[a][1]);
            r[a][2] = fma(g2, v, r[a][2]);
          }
        }
#pragma unroll
        for (int a = 0; a < 3; ++a) du += r[a][0] * Ji[a] + r[a][1] * Ji[3 + a] + r[a][2] * Ji[6 + a];
      }
      if constexpr (MODE == CPL_EVAL) ev = fma(dw * ph, du, ev);
      else if constexpr (MODE == CPL_RESIDUAL) fq[c][q] = TRANS ? dw * du : ph;
    }
    if constexpr (MODE == CPL_EVAL) continue;
    __syncthreads();
    // ---- phase 2: one thread per (cell, output entry)
    for (int i = tid; i < ne * NOUT; i += blockDim.x) {
      const int c = i / NOUT, o = i - NOUT * c;
      const int64_t e = eb + c;
      double s = 0.0;
      if constexpr (MODE == CPL_RESIDUAL && TRANS) {  // r_q[l] = sum_q psi_l(q) detw div u_h(q)
        const int l = o;
        for (int q = 0; q < NQ; ++q) s = fma(__ldg(psi + (int64_t)q * NBP + l), fq[c][q], s);
      } else {
        int a, k, l = 0;
        if constexpr (MODE == CPL_RESIDUAL) {  // o = a * NBV + k
          a = o / NBV; k = o - a * NBV;
        } else if constexpr (TRANS) {  // o = l * 3 NBV + a * NBV + k
          l = o / (3 * NBV);
          const int r = o - l * 3 * NBV;
          a = r / NBV; k = r - a * NBV;
        } else {  // o = (a * NBV + k) * NBP + l
          const int r = o / NBP;
          l = o - r * NBP;
          a = r / NBV; k = r - a * NBV;
        }
        for (int q = 0; q < NQ; ++q) {
          const double* dp = mv.dphi + (int64_t)q * 3 * NBV + k;
          const double g = W[c][q][a] * __ldg(dp) + W[c][q][3 + a] * __ldg(dp + NBV) +
                           W[c][q][6 + a] * __ldg(dp + 2 * NBV);
          const double f = MODE == CPL_MATRIX ? __ldg(psi + (int64_t)q * NBP + l) : fq[c][q];
          s = fma(g, f, s);
        }
      }
      if (out) out[(e - e0) * (int64_t)NOUT + o] = s;
      if constexpr (MODE == CPL_RESIDUAL) {
        if (r_global) {
          if constexpr (TRANS) atomicAdd(r_global + pdof[e * NBP + o], s);
          else atomicAdd(r_global + 3 * (int64_t)mv.dof_conn[e * NBV + o % NBV] + o / NBV, s);
        }
      }
    }
  }
  if constexpr (MODE == CPL_EVAL) {
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) ev += __shfl_xor_sync(0xffffffffu, ev, off);
    if ((tid & 31) == 0 && ev != 0.0) atomicAdd(value, ev);
  }
}

template <int PV, int PP, int MODE, bool TRANS>
static cudaError_t launch_cpl_t(const fe_mesh* mh, const fe_field* f, const double* u, const double* p,
                                int64_t e0, int64_t e1, double* out, double* rg, double* val,
                                cudaStream_t st) {
  using L = CplL<PV, PP>;
  auto kern = k_coupling<PV, PP, MODE, TRANS>;
  int nsm = 148, per_sm = 1, dev = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, L::THREADS, 0);
  if (per_sm < 1) per_sm = 1;
  const int64_t nb = (e1 - e0 + L::CB - 1) / L::CB;
  int grid = (int)(nb < (int64_t)nsm * per_sm ? nb : (int64_t)nsm * per_sm);
  grid = grid_cap(grid);
  if (grid <= 0) return cudaSuccess;
  kern<<<grid, L::THREADS, 0, st>>>(view_of(mh), f->dof_conn, f->psi, u, p, e0, e1, out, rg, val);
  count_launch();
  return cudaGetLastError();
}

template <int PV, int PP>
static cudaError_t cpl_mode(const fe_mesh* mh, const fe_field* f, int mode, bool trans, const double* u,
                            const double* p, int64_t e0, int64_t e1, double* out, double* rg,
                            double* val, cudaStream_t st) {
  if (mode == CPL_MATRIX)
    return trans ? launch_cpl_t<PV, PP, CPL_MATRIX, true>(mh, f, u, p, e0, e1, out, rg, val, st)
                 : launch_cpl_t<PV, PP, CPL_MATRIX, false>(mh, f, u, p, e0, e1, out, rg, val, st);
  if (mode == CPL_RESIDUAL)
    return trans ? launch_cpl_t<PV, PP, CPL_RESIDUAL, true>(mh, f, u, p, e0, e1, out, rg, val, st)
                 : launch_cpl_t<PV, PP, CPL_RESIDUAL, false>(mh, f, u, p, e0, e1, out, rg, val, st);
  return launch_cpl_t<PV, PP, CPL_EVAL, false>(mh, f, u, p, e0, e1, out, rg, val, st);
}

cudaError_t launch_coupling(const fe_mesh* mh, const fe_field* f, int mode, bool trans,
                            const double* u, const double* p, int64_t e0, int64_t e1, double* out,
                            double* rg, double* val, cudaStream_t st) {
  if (mh->q1d != mh->order + 1) return cudaErrorNotSupported;
#define CPL_CASE(PV, PP)                    \
  if (mh->order == PV && f->order == PP) \
    return cpl_mode<PV, PP>(mh, f, mode, trans, u, p, e0, e1, out, rg, val, st);
  CPL_CASE(1, 1) CPL_CASE(2, 1) CPL_CASE(2, 2) CPL_CASE(3, 2) CPL_CASE(3, 3) CPL_CASE(4, 3)
  CPL_CASE(4, 4)
#undef CPL_CASE
  return cudaErrorNotSupported;
}

}  // namespace feb200
