// Pointwise integrands of residual mode (Alg. 1's F) at one
// quadrature point: given u_h(q) and its physical gradient du_a/dx_j, return the
// coefficients f0[a] (tested against v = phi e_a) and f1[a][j] (tested against
// dv_a/dx_j) of
//   diffusion        f1 = kappa grad u                     ('0.i,0.i')
//   mass             f0 = rho u
//   vector mass      f0_a = rho u_a                        ('i,i')
//   mass+diffusion   f0 = rho u, f1 = kappa grad u         (BASELINE config 4)
//   elasticity       f1 = sigma = D e(u), Voigt with engineering shears
//                    (Psg of P:942, reading 7)   ('IK,s(i:j)->I,s(k:l)->K')
//   convective       f0_a = (du_a/dx_j) u_j                (Eq. fe2)
//   weighted dot     f0_a = M_ab u_b, M per qp             ('ij,i,j')
//   divergence       f1_aj = delta_aj (u does not enter)   ('i.i')
#pragma once
#include "fe_device.cuh"
#include "feb200.h"
#ifndef FEB200_FLUX_V4
#define FEB200_FLUX_V4 1
#endif

namespace feb200 {

template <int FORM>
struct FormD {
  static constexpr int D = (FORM == FE_FORM_VECTOR_MASS || FORM == FE_FORM_ELASTICITY ||
                            FORM == FE_FORM_CONVECTIVE || FORM == FE_FORM_WEIGHTED_DOT ||
                            FORM == FE_FORM_DIVERGENCE) ? 3 : 1;
};

// Material values at one (cell, qp), loaded ahead of use so the global-load
// latency overlaps the interpolation (FULL_D keeps a pointer to its 6x6 block).
template <typename T>
struct MatQ {
  double a, b;
  const T* Dm;
};

template <int FORM, typename T>
__device__ __forceinline__ MatQ<T> load_matq(int64_t e, int q, int nq, int mat_kind,
                                             const T* __restrict__ ma, const T* __restrict__ mb) {
  MatQ<T> m{0.0, 0.0, nullptr};
  if constexpr (FORM == FE_FORM_CONVECTIVE || FORM == FE_FORM_DIVERGENCE) return m;
  if constexpr (FORM == FE_FORM_WEIGHTED_DOT) {
    m.Dm = ma + (e * nq + q) * 9;
    return m;
  }
  if constexpr (FORM == FE_FORM_ELASTICITY) {
    if (mat_kind == FE_MAT_FULL_D) {
      m.Dm = ma + (e * nq + q) * 36;
    } else if (mat_kind == FE_MAT_PER_ELEM) {
      m.a = (double)ma[e];
      m.b = (double)mb[e];
    } else {
      m.a = (double)ma[e * nq + q];
      m.b = (double)mb[e * nq + q];
    }
    return m;
  }
  m.a = (double)ma[e * nq + q];
  if constexpr (FORM == FE_FORM_MASS_DIFFUSION) m.b = (double)mb[e * nq + q];
  return m;
}

template <int FORM, typename T>
__device__ __forceinline__ void qp_flux_m(const double (&uq)[FormD<FORM>::D],
                                          const double (&gu)[FormD<FORM>::D][3], const MatQ<T>& mq,
                                          int mat_kind, double (&f0)[FormD<FORM>::D],
                                          double (&f1)[FormD<FORM>::D][3]) {
  constexpr int D = FormD<FORM>::D;
#pragma unroll
  for (int a = 0; a < D; ++a) {
    f0[a] = 0.0;
    f1[a][0] = f1[a][1] = f1[a][2] = 0.0;
  }
  if constexpr (FORM == FE_FORM_DIFFUSION) {
    const double kap = mq.a;
    f1[0][0] = kap * gu[0][0]; f1[0][1] = kap * gu[0][1]; f1[0][2] = kap * gu[0][2];
  } else if constexpr (FORM == FE_FORM_MASS || FORM == FE_FORM_VECTOR_MASS) {
    const double rho = mq.a;
#pragma unroll
    for (int a = 0; a < D; ++a) f0[a] = rho * uq[a];
  } else if constexpr (FORM == FE_FORM_MASS_DIFFUSION) {
    const double rho = mq.a, kap = mq.b;
    f0[0] = rho * uq[0];
    f1[0][0] = kap * gu[0][0]; f1[0][1] = kap * gu[0][1]; f1[0][2] = kap * gu[0][2];
  } else if constexpr (FORM == FE_FORM_ELASTICITY) {
    // engineering strain (xx, yy, zz, xy, xz, yz)
    const double eps[6] = {gu[0][0], gu[1 % D][1], gu[2 % D][2], gu[0][1] + gu[1 % D][0],
                           gu[0][2] + gu[2 % D][0], gu[1 % D][2] + gu[2 % D][1]};
    double sig[6];
    if (mat_kind == FE_MAT_FULL_D) {
      const T* Dm = mq.Dm;
      if (sizeof(T) == 8 && FEB200_FLUX_V4 && (reinterpret_cast<uintptr_t>(Dm) & 31u) == 0) {
        // 32-byte loads: one full sector per lane and instruction (the 288-B block of a qp is
        // nine of them), so no sector is fetched twice through L1
        const double* D8 = reinterpret_cast<const double*>(Dm);
        double dv[36];
#pragma unroll
        for (int h = 0; h < 9; ++h) ld_nc_v4(D8 + 4 * h, dv[4 * h], dv[4 * h + 1], dv[4 * h + 2], dv[4 * h + 3]);
#pragma unroll
        for (int I = 0; I < 6; ++I) {
          double s = 0.0;
#pragma unroll
          for (int K = 0; K < 6; ++K) s = fma(dv[6 * I + K], eps[K], s);
          sig[I] = s;
        }
      } else if (sizeof(T) == 8 && (reinterpret_cast<uintptr_t>(Dm) & 15u) == 0) {
        // 16-byte loads: a warp's 36 scalar loads of 288-byte-strided blocks would each touch
        // 32 sectors for 8 useful bytes; pairs halve the sector re-fetches through L1
        const double2* D2 = reinterpret_cast<const double2*>(Dm);
#pragma unroll
        for (int I = 0; I < 6; ++I) {
          double s = 0.0;
#pragma unroll
          for (int K2 = 0; K2 < 3; ++K2) {
            const double2 d = __ldg(D2 + 3 * I + K2);
            s += d.x * eps[2 * K2] + d.y * eps[2 * K2 + 1];
          }
          sig[I] = s;
        }
      } else {
#pragma unroll
        for (int I = 0; I < 6; ++I) {
          double s = 0.0;
#pragma unroll
          for (int K = 0; K < 6; ++K) s += (double)Dm[6 * I + K] * eps[K];
          sig[I] = s;
        }
      }
    } else {
      const double lam = mq.a, mu = mq.b;
      const double tr = eps[0] + eps[1] + eps[2];
      sig[0] = lam * tr + 2.0 * mu * eps[0];
      sig[1] = lam * tr + 2.0 * mu * eps[1];
      sig[2] = lam * tr + 2.0 * mu * eps[2];
      sig[3] = mu * eps[3];
      sig[4] = mu * eps[4];
      sig[5] = mu * eps[5];
    }
    // f1[a][j] = sum_I Psg[a][j][I] sig_I (the symmetric stress tensor)
    const double st[3][3] = {{sig[0], sig[3], sig[4]}, {sig[3], sig[1], sig[5]}, {sig[4], sig[5], sig[2]}};
#pragma unroll
    for (int a = 0; a < D; ++a)
#pragma unroll
      for (int j = 0; j < 3; ++j) f1[a][j] = st[a][j];
  } else if constexpr (FORM == FE_FORM_WEIGHTED_DOT) {  // f0_a = M_ab u_b ('ij,i,j')
    const T* M = mq.Dm;
#pragma unroll
    for (int a = 0; a < D; ++a)
      f0[a] = (double)M[3 * a] * uq[0] + (double)M[3 * a + 1] * uq[1 % D] + (double)M[3 * a + 2] * uq[2 % D];
  } else if constexpr (FORM == FE_FORM_DIVERGENCE) {  // f1_aj = delta_aj ('i.i')
#pragma unroll
    for (int a = 0; a < D; ++a) f1[a][a] = 1.0;
  } else {  // CONVECTIVE
#pragma unroll
    for (int a = 0; a < D; ++a) f0[a] = gu[a][0] * uq[0] + gu[a][1] * uq[1 % D] + gu[a][2] * uq[2 % D];
  }
}

template <int FORM, typename T>
__device__ __forceinline__ void qp_flux(const double (&uq)[FormD<FORM>::D],
                                        const double (&gu)[FormD<FORM>::D][3], int64_t e, int q,
                                        int nq, int mat_kind, const T* __restrict__ ma,
                                        const T* __restrict__ mb, double (&f0)[FormD<FORM>::D],
                                        double (&f1)[FormD<FORM>::D][3]) {
  const MatQ<T> mq = load_matq<FORM, T>(e, q, nq, mat_kind, ma, mb);
  qp_flux_m<FORM, T>(uq, gu, mq, mat_kind, f0, f1);
}

}  // namespace feb200
