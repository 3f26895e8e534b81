// Register-resident residual mode for the scalar forms at p = 2 (Alg. 1, PAPER.md P:392-429,
// with the gather and fused scatter-add of P:1093-1095): three threads per cell, thread j
// owning the z-plane j of the cell -- its 3 x 3 nodes (kz = j) on the way in and its 3 x 3
// quadrature points (qz = j) at the flux.  The x- and y-contractions of the sum
// factorisation (Eq. fe1) run in registers; the z-contraction is the only
// exchange and goes through warp shuffles between the three lanes of a cell (forward: the
// other planes' partial sums; backward: each plane's contribution to the other node planes).
// Shared memory is not used at all: the shared-memory data pipe that binds the column-per-
// thread kernel (k_residual_sf.cu, four exchanges through smem) is bypassed.
//   forward   u(kx,ky,kz=j) -> [x] -> [y] -> c00, c01, c10 at (qx,qy,kz=j)
//             -> [z, shuffles] -> u, du/dxi at (qx,qy,qz=j)
//   flux      geometry at the 9 qps (trilinear map), f0 = rho u, f1 = kappa grad u
//             pulled back: F = detw J^-1 f1
//   backward  [z^T, shuffles] -> [y^T] -> [x^T] -> r(kx,ky,kz=j) -> atomic scatter
// 10 cells per warp (lanes 30, 31 idle).
#include "fe_const.cuh"
#include "fe_device.cuh"
#include "fe_internal.h"

#ifndef FEB200_T3_THREADS
#define FEB200_T3_THREADS 64
#endif
#ifndef FEB200_T3_SEPGEO
#define FEB200_T3_SEPGEO 1
#endif
#ifndef FEB200_T3C
#define FEB200_T3C 1
#endif
// t3c flux: v = w C u (C the cofactors of J) is the same for the three components of a qp, so
// component lane a forms it at the qps qx = a of its plane only and the others fetch it by
// shuffle (a third of the per-qp geometry per lane, about as many shuffles as fetching u)
#ifndef FEB200_T3C_VSHARE
#define FEB200_T3C_VSHARE 1
#endif
#ifndef FEB200_T3E
#define FEB200_T3E 1  // register-resident elasticity residual (p = 2, isotropic)
#endif
#ifndef FEB200_T3E_MINB
#define FEB200_T3E_MINB 4
#endif
#ifndef FEB200_T3C_MINB
#define FEB200_T3C_MINB 4
#endif
#ifndef FEB200_T3_MINB
#define FEB200_T3_MINB 4
#endif

namespace feb200 {

namespace {
__device__ __forceinline__ void t3_cp8(void* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(static_cast<uint32_t>(__cvta_generic_to_shared(dst))),
               "l"(src) : "memory");
}
__device__ __forceinline__ void t3_cp4(void* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(static_cast<uint32_t>(__cvta_generic_to_shared(dst))),
               "l"(src) : "memory");
}
__device__ __forceinline__ void t3_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void t3_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }
}  // namespace

cudaError_t upload_const_tables_residual_t3(int order, const double* b1, const double* d1,
                                           const double* x1, const double* w1, cudaStream_t st) {
  return upload_tables_this_tu(order, b1, d1, x1, w1, st);
}

template <int FORM, bool EVAL, bool PEER = false>
__global__ void __launch_bounds__(FEB200_T3_THREADS, FEB200_T3_MINB)
    k_residual_t3(MeshView mv, const double* __restrict__ ma, const double* __restrict__ mb,
                  const double* __restrict__ u, int64_t e0, int64_t e1, double* __restrict__ r_elem,
                  double* __restrict__ r_global, double* __restrict__ eval_out, PeerWin pw) {
  constexpr int P = 2, N = 3, NB = 27, NQ = 27;
  constexpr bool VAL = FORM == FE_FORM_MASS || FORM == FE_FORM_MASS_DIFFUSION;
  constexpr bool GRAD = FORM != FE_FORM_MASS;
#define B0(q, k) c_tab1d[P][0][q][k]
#define B1(q, k) c_tab1d[P][1][q][k]
  const int lane = threadIdx.x & 31;
  const int cl = lane / 3, j = lane - 3 * cl;  // cell in the warp, plane
  const bool lane_ok = lane < 30;
  const int base = 3 * cl;
  // per-lane coefficients B^a[qz = j][kz = (j + s) % 3] and the partner lanes
  double f0[3], f1[3];
  int srcf[3], srcb[3];
#pragma unroll
  for (int s = 0; s < 3; ++s) {
    const int k = (j + s) % 3;
    f0[s] = lane_ok ? c_tab1d[P][0][j][k] : 0.0;
    f1[s] = lane_ok ? c_tab1d[P][1][j][k] : 0.0;
    srcf[s] = lane_ok ? base + k : lane;                  // forward: plane (j + s) % 3
    srcb[s] = lane_ok ? base + (j - s + 3) % 3 : lane;    // backward: plane (j - s) % 3
  }
  const double tZ = lane_ok ? c_x1d[P][j] : 0.5, wz = lane_ok ? c_w1d[P][j] : 0.0;
  const int64_t nloc = e1 - e0;
  const int wpb = blockDim.x >> 5;
  const int64_t gw = (int64_t)blockIdx.x * wpb + (threadIdx.x >> 5), nw = (int64_t)gridDim.x * wpb;
  constexpr int NCOEF = FORM == FE_FORM_MASS_DIFFUSION ? 2 : 1;
  // cp.async prefetch rings in shared memory, lane-interleaved ([slot][element][thread]):
  // S1 (3 slots, two groups ahead): dof ids, conn, material of the lane's cell plane;
  // S2 (2 slots, one group ahead): u at the dofs, 8 of the cell's 24 vertex coordinates
  constexpr int TH = FEB200_T3_THREADS;
  extern __shared__ __align__(16) unsigned char t3s[];
  double* s1m = reinterpret_cast<double*>(t3s);                 // [3][NCOEF * 9][TH]
  double* s2u = s1m + 3 * NCOEF * 9 * TH;                       // [2][9][TH]
  double* s2x = s2u + 2 * 9 * TH;                               // [2][8][TH]
  int32_t* s1d = reinterpret_cast<int32_t*>(s2x + 2 * 8 * TH);  // [3][9][TH]
  int32_t* s1c = s1d + 3 * 9 * TH;                              // [3][8][TH]
  const int tid = threadIdx.x;
  auto group_cell = [&](int64_t g, int64_t& le, bool& ok) {
    le = (gw + g * nw) * 10 + cl;
    ok = lane_ok && le < nloc;
  };
  auto issue_s1 = [&](int64_t g) {
    int64_t le;
    bool ok;
    group_cell(g, le, ok);
    if (ok) {
      const int sl = (int)(g % 3);
      const int64_t e = e0 + le;
#pragma unroll
      for (int k = 0; k < 9; ++k) t3_cp4(&s1d[(sl * 9 + k) * TH + tid], mv.dof_conn + e * NB + N * N * j + k);
#pragma unroll
      for (int v = 0; v < 8; ++v) t3_cp4(&s1c[(sl * 8 + v) * TH + tid], mv.conn + 8 * e + v);
#pragma unroll
      for (int k = 0; k < 9; ++k) {
        t3_cp8(&s1m[(sl * NCOEF * 9 + k) * TH + tid], ma + e * NQ + N * N * j + k);
        if (NCOEF == 2) t3_cp8(&s1m[(sl * NCOEF * 9 + 9 + k) * TH + tid], mb + e * NQ + N * N * j + k);
      }
    }
    t3_commit();
  };
  auto issue_s2 = [&](int64_t g) {  // needs S1(g) in shared memory
    int64_t le;
    bool ok;
    group_cell(g, le, ok);
    if (ok) {
      const int s1 = (int)(g % 3), s2 = (int)(g & 1);
      // all staged indices first (the copies' asm memory clobbers would otherwise serialise
      // each index load behind the previous copy), then the copies
      int dd[9], vv[8];
#pragma unroll
      for (int k = 0; k < 9; ++k) dd[k] = s1d[(s1 * 9 + k) * TH + tid];
#pragma unroll
      for (int h = 0; h < 8; ++h) vv[h] = s1c[(s1 * 8 + (8 * j + h) / 3) * TH + tid];
#pragma unroll
      for (int k = 0; k < 9; ++k) t3_cp8(&s2u[(s2 * 9 + k) * TH + tid], u + dd[k]);
#pragma unroll
      for (int h = 0; h < 8; ++h) {  // coordinate p = 8 j + h of the cell: vertex p / 3, component p % 3
        const int pidx = 8 * j + h, v = pidx / 3, i = pidx - 3 * v;
        t3_cp8(&s2x[(s2 * 8 + h) * TH + tid], mv.coords + 3 * (int64_t)vv[h] + i);
        (void)v;
      }
    }
    t3_commit();
  };
  issue_s1(0);
  issue_s1(1);
  t3_wait<1>();
  issue_s2(0);
  for (int64_t g = 0;; ++g) {
    int64_t le;
    bool valid;
    group_cell(g, le, valid);
    if ((gw + g * nw) * 10 >= nloc) break;
    t3_wait<0>();  // S2(g) and S1(g + 1)
    __syncwarp();
    issue_s2(g + 1);
    issue_s1(g + 2);
    const int64_t e = e0 + (valid ? le : 0);
    const int s1 = (int)(g % 3), s2 = (int)(g & 1);
    // ---- u at the nodes (kx, ky, kz = j), gathered by cp.async
    int dof[N][N];
    double uv[N][N];
#pragma unroll
    for (int ky = 0; ky < N; ++ky)
#pragma unroll
      for (int kx = 0; kx < N; ++kx) {
        dof[ky][kx] = s1d[(s1 * 9 + kx + N * ky) * TH + tid];
        uv[ky][kx] = valid ? s2u[(s2 * 9 + kx + N * ky) * TH + tid] : 0.0;
      }
    // ---- x- and y-contractions in registers
    double c00[N][N], c01[N][N], c10[N][N];  // [qy][qx] at kz = j
    {
      double a0[N][N], a1[N][N];  // [ky][qx]
#pragma unroll
      for (int ky = 0; ky < N; ++ky)
#pragma unroll
        for (int qx = 0; qx < N; ++qx) {
          double s0 = 0.0, s1 = 0.0;
#pragma unroll
          for (int kx = 0; kx < N; ++kx) {
            s0 = fma(B0(qx, kx), uv[ky][kx], s0);
            if (GRAD) s1 = fma(B1(qx, kx), uv[ky][kx], s1);
          }
          a0[ky][qx] = s0;
          a1[ky][qx] = s1;
        }
#pragma unroll
      for (int qy = 0; qy < N; ++qy)
#pragma unroll
        for (int qx = 0; qx < N; ++qx) {
          double s00 = 0.0, s01 = 0.0, s10 = 0.0;
#pragma unroll
          for (int ky = 0; ky < N; ++ky) {
            s00 = fma(B0(qy, ky), a0[ky][qx], s00);
            if (GRAD) {
              s01 = fma(B1(qy, ky), a0[ky][qx], s01);
              s10 = fma(B0(qy, ky), a1[ky][qx], s10);
            }
          }
          c00[qy][qx] = s00;
          c01[qy][qx] = s01;
          c10[qy][qx] = s10;
        }
    }
    // ---- z-contraction through the cell's three lanes: value / reference gradient at qz = j
    double Uq[N][N], Gx[N][N], Gy[N][N], Gz[N][N];
#pragma unroll
    for (int qy = 0; qy < N; ++qy)
#pragma unroll
      for (int qx = 0; qx < N; ++qx) {
        double v00 = c00[qy][qx], v01 = c01[qy][qx], v10 = c10[qy][qx];
        double uq = f0[0] * v00, gz = f1[0] * v00, gy = f0[0] * v01, gx = f0[0] * v10;
#pragma unroll
        for (int s = 1; s < 3; ++s) {
          const double w00 = __shfl_sync(0xffffffffu, v00, srcf[s]);
          uq = fma(f0[s], w00, uq);
          if (GRAD) {
            const double w01 = __shfl_sync(0xffffffffu, v01, srcf[s]);
            const double w10 = __shfl_sync(0xffffffffu, v10, srcf[s]);
            gz = fma(f1[s], w00, gz);
            gy = fma(f0[s], w01, gy);
            gx = fma(f0[s], w10, gx);
          }
        }
        Uq[qy][qx] = uq;
        Gx[qy][qx] = gx;
        Gy[qy][qx] = gy;
        Gz[qy][qx] = gz;
      }
    // ---- geometry and flux at the 9 qps (qx, qy, qz = j); F = detw J^-1 f1 (reference)
    double X[8][3];  // the cell's vertices, fetched by its three lanes (8 values each)
    const int wb = tid - lane;
#pragma unroll
    for (int pidx = 0; pidx < 24; ++pidx)
      X[pidx / 3][pidx % 3] = valid ? s2x[(s2 * 8 + pidx % 8) * TH + wb + base + pidx / 8] : 0.0;
    // separable trilinear Jacobian on this lane's plane (t2 = tZ fixed): column 0 is linear in
    // t1, column 1 linear in t0, column 2 bilinear; the t2 interpolation is done once per cell
    double gE0[3], gdE[3], gF0[3], gdF[3], gH0[N][3], gdH[N][3];
#pragma unroll
    for (int i = 0; i < 3; ++i) {
      const double e0 = (1 - tZ) * (X[1][i] - X[0][i]) + tZ * (X[5][i] - X[4][i]);
      const double e1 = (1 - tZ) * (X[3][i] - X[2][i]) + tZ * (X[7][i] - X[6][i]);
      const double f0_ = (1 - tZ) * (X[2][i] - X[0][i]) + tZ * (X[6][i] - X[4][i]);
      const double f1_ = (1 - tZ) * (X[3][i] - X[1][i]) + tZ * (X[7][i] - X[5][i]);
      gE0[i] = e0; gdE[i] = e1 - e0; gF0[i] = f0_; gdF[i] = f1_ - f0_;
#pragma unroll
      for (int qx = 0; qx < N; ++qx) {
        const double t0 = c_x1d[P][qx];
        const double h0 = (1 - t0) * (X[4][i] - X[0][i]) + t0 * (X[5][i] - X[1][i]);
        const double h1 = (1 - t0) * (X[6][i] - X[2][i]) + t0 * (X[7][i] - X[3][i]);
        gH0[qx][i] = h0;
        gdH[qx][i] = h1 - h0;
      }
    }
    double Fv[N][N], Fx[N][N], Fy[N][N], Fz[N][N];
#pragma unroll
    for (int qy = 0; qy < N; ++qy)
#pragma unroll
      for (int qx = 0; qx < N; ++qx) {
        const double t0 = c_x1d[P][qx], t1 = c_x1d[P][qy];
        double J[3][3];
#pragma unroll
        for (int i = 0; i < 3; ++i) {
          if (FEB200_T3_SEPGEO) {
            J[i][0] = fma(t1, gdE[i], gE0[i]);
            J[i][1] = fma(t0, gdF[i], gF0[i]);
            J[i][2] = fma(t1, gdH[qx][i], gH0[qx][i]);
          } else {
            const double t2 = tZ;
            J[i][0] = (1 - t1) * (1 - t2) * (X[1][i] - X[0][i]) + t1 * (1 - t2) * (X[3][i] - X[2][i]) +
                      (1 - t1) * t2 * (X[5][i] - X[4][i]) + t1 * t2 * (X[7][i] - X[6][i]);
            J[i][1] = (1 - t0) * (1 - t2) * (X[2][i] - X[0][i]) + t0 * (1 - t2) * (X[3][i] - X[1][i]) +
                      (1 - t0) * t2 * (X[6][i] - X[4][i]) + t0 * t2 * (X[7][i] - X[5][i]);
            J[i][2] = (1 - t0) * (1 - t1) * (X[4][i] - X[0][i]) + t0 * (1 - t1) * (X[5][i] - X[1][i]) +
                      (1 - t0) * t1 * (X[6][i] - X[2][i]) + t0 * t1 * (X[7][i] - X[3][i]);
          }
        }
        // cofactors C[r][c] of J; J^-1[m][r] = C[r][m] / det
        const double C00 = J[1][1] * J[2][2] - J[1][2] * J[2][1], C01 = J[1][2] * J[2][0] - J[1][0] * J[2][2],
                     C02 = J[1][0] * J[2][1] - J[1][1] * J[2][0], C10 = J[0][2] * J[2][1] - J[0][1] * J[2][2],
                     C11 = J[0][0] * J[2][2] - J[0][2] * J[2][0], C12 = J[0][1] * J[2][0] - J[0][0] * J[2][1],
                     C20 = J[0][1] * J[1][2] - J[0][2] * J[1][1], C21 = J[0][2] * J[1][0] - J[0][0] * J[1][2],
                     C22 = J[0][0] * J[1][1] - J[0][1] * J[1][0];
        const double det = J[0][0] * C00 + J[0][1] * C01 + J[0][2] * C02;
        const double wq = c_w1d[P][qx] * c_w1d[P][qy] * wz;
        const int q = qx + N * qy + N * N * j;
        double fv = 0.0, fx = 0.0, fy = 0.0, fz = 0.0;
        if (valid) {
          if constexpr (VAL) {
            const double rho = s1m[(s1 * NCOEF * 9 + qx + N * qy) * TH + tid];
            fv = wq * det * rho * Uq[qy][qx];
          }
          if constexpr (GRAD) {
            const double kap = s1m[(s1 * NCOEF * 9 + (NCOEF - 1) * 9 + qx + N * qy) * TH + tid];
            // grad u = J^-T grad_ref u: t_r = sum_m C[r][m] g_m (= det * (grad u)_r);
            // F_m = detw kappa sum_r J^-1[m][r] (grad u)_r = (w kappa / det) sum_r C[r][m] t_r
            const double g0 = Gx[qy][qx], g1 = Gy[qy][qx], g2 = Gz[qy][qx];
            const double tr0 = C00 * g0 + C01 * g1 + C02 * g2;
            const double tr1 = C10 * g0 + C11 * g1 + C12 * g2;
            const double tr2 = C20 * g0 + C21 * g1 + C22 * g2;
            const double sc = wq * kap * rcp_nr(det);
            fx = sc * (C00 * tr0 + C10 * tr1 + C20 * tr2);
            fy = sc * (C01 * tr0 + C11 * tr1 + C21 * tr2);
            fz = sc * (C02 * tr0 + C12 * tr1 + C22 * tr2);
          }
        }
        Fv[qy][qx] = fv;
        Fx[qy][qx] = fx;
        Fy[qy][qx] = fy;
        Fz[qy][qx] = fz;
      }
    // ---- z^T through the cell's lanes: node plane j collects the contributions
    //      B^a[qz][kz = j] F(qz) of the three qp planes
    double Hv[N][N], Hx[N][N], Hy[N][N];  // [qy][qx] at kz = j
#pragma unroll
    for (int qy = 0; qy < N; ++qy)
#pragma unroll
      for (int qx = 0; qx < N; ++qx) {
        const double fv = Fv[qy][qx], fx = Fx[qy][qx], fy = Fy[qy][qx], fz = Fz[qy][qx];
        double hv = 0.0, hx = 0.0, hy = 0.0;
        if (VAL) hv = f0[0] * fv;
        if (GRAD) {
          hv = fma(f1[0], fz, hv);
          hx = f0[0] * fx;
          hy = f0[0] * fy;
        }
#pragma unroll
        for (int s = 1; s < 3; ++s) {
          // this lane's contribution to node plane (j + s) % 3; pulled by that plane's lane
          double cv = 0.0, cx = 0.0, cy = 0.0;
          if (VAL) cv = f0[s] * fv;
          if (GRAD) {
            cv = fma(f1[s], fz, cv);
            cx = f0[s] * fx;
            cy = f0[s] * fy;
          }
          hv += __shfl_sync(0xffffffffu, cv, srcb[s]);
          if (GRAD) {
            hx += __shfl_sync(0xffffffffu, cx, srcb[s]);
            hy += __shfl_sync(0xffffffffu, cy, srcb[s]);
          }
        }
        Hv[qy][qx] = hv;
        Hx[qy][qx] = hx;
        Hy[qy][qx] = hy;
      }
    // ---- y^T and x^T in registers, scatter
    double ev = 0.0;
#pragma unroll
    for (int ky = 0; ky < N; ++ky) {
      double Iv[N], Ix[N];  // [qx]
#pragma unroll
      for (int qx = 0; qx < N; ++qx) {
        double sv = 0.0, sx = 0.0;
#pragma unroll
        for (int qy = 0; qy < N; ++qy) {
          sv = fma(B0(qy, ky), Hv[qy][qx], sv);
          if (GRAD) {
            sv = fma(B1(qy, ky), Hy[qy][qx], sv);
            sx = fma(B0(qy, ky), Hx[qy][qx], sx);
          }
        }
        Iv[qx] = sv;
        Ix[qx] = sx;
      }
#pragma unroll
      for (int kx = 0; kx < N; ++kx) {
        double rr = 0.0;
#pragma unroll
        for (int qx = 0; qx < N; ++qx) {
          rr = fma(B0(qx, kx), Iv[qx], rr);
          if (GRAD) rr = fma(B1(qx, kx), Ix[qx], rr);
        }
        if (valid) {
          if (r_elem) r_elem[le * NB + kx + N * ky + N * N * j] = rr;
          if (r_global) atomicAdd(r_global + dof[ky][kx], rr);
          if constexpr (PEER) peer_scatter<1>(pw, dof[ky][kx], 0, rr);
          if (EVAL) ev = fma(rr, u[dof[ky][kx]], ev);
        }
      }
    }
    if (EVAL) {
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) ev += __shfl_xor_sync(0xffffffffu, ev, o);
      if (lane == 0 && ev != 0.0) atomicAdd(eval_out, ev);
    }
  }
  t3_wait<0>();
#undef B0
#undef B1
}

template <int FORM>
static cudaError_t launch_t3_t(const fe_mesh* mh, MatArgs mat, const double* u, int64_t e0, int64_t e1,
                               double* r_elem, double* r_global, double* eval_out, cudaStream_t st) {
  const PeerWin pw = g_peer;
  auto kern = eval_out ? k_residual_t3<FORM, true> : (pw.n > 0 ? k_residual_t3<FORM, false, true>
                                                                : k_residual_t3<FORM, false>);
  constexpr int NCOEF = FORM == FE_FORM_MASS_DIFFUSION ? 2 : 1;
  const size_t smem = (size_t)FEB200_T3_THREADS * (8 * (3 * NCOEF * 9 + 2 * 9 + 2 * 8) + 4 * (3 * 9 + 3 * 8));
  const LaunchFacts lf = launch_facts((const void*)kern, FEB200_T3_THREADS, smem);
  if (lf.err != cudaSuccess) return lf.err;
  const int nsm = lf.nsm, per_sm = lf.per_sm;
  const int64_t ncg = (e1 - e0 + 9) / 10;                       // 10 cells per warp
  const int64_t nblk = (ncg + FEB200_T3_THREADS / 32 - 1) / (FEB200_T3_THREADS / 32);
  int grid = (int)(nblk < (int64_t)nsm * per_sm ? nblk : (int64_t)nsm * per_sm);
  grid = grid_cap(grid);
  if (grid <= 0) return cudaSuccess;
  kern<<<grid, FEB200_T3_THREADS, smem, st>>>(view_of(mh), (const double*)mat.a, (const double*)mat.b, u,
                                              e0, e1, r_elem, r_global, eval_out, pw);
  count_launch();
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------------------
// Convective residual r_(a,k) = int phi_k sum_j (du_a/dx_j) u_j (Eq. fe2) at p = 2,
// fp64, register-resident: NINE lanes per cell, lane (a, j) owning component a on z-plane j
// (3 cells per warp, lanes 27-31 idle).  Each component runs the scalar forward pass of the
// kernel above (x, y in registers, z by shuffles among the component's three plane lanes);
// at the flux the velocity components u_b(q) come from the cell's other component lanes by
// shuffle.  With t = C^T grad_ref u_a = det grad u_a (C the cofactors of J),
//   detw f0_a = w det (1/det) sum_r t_r u_r = w sum_r t_r u_r      (det cancels).
// The backward pass tests against v only (values), as in the shared-memory kernel.
template <bool EVAL, bool PEER = false>
__global__ void __launch_bounds__(FEB200_T3_THREADS, FEB200_T3C_MINB)
    k_residual_t3c(MeshView mv, const double* __restrict__ u, int64_t e0, int64_t e1,
                   double* __restrict__ r_elem, double* __restrict__ r_global,
                   double* __restrict__ eval_out, PeerWin pw) {
  constexpr int P = 2, N = 3, NB = 27;
#define B0(q, k) c_tab1d[P][0][q][k]
#define B1(q, k) c_tab1d[P][1][q][k]
  const int lane = threadIdx.x & 31;
  const int cl = lane / 9, rem = lane - 9 * cl, a = rem / 3, j = rem - 3 * a;
  const bool lane_ok = lane < 27;
  const int base = 9 * cl + 3 * a;  // the three plane lanes of (cell, component)
  double f0[3], f1[3];
  int srcf[3], srcb[3];
#pragma unroll
  for (int s = 0; s < 3; ++s) {
    const int k = (j + s) % 3;
    f0[s] = lane_ok ? c_tab1d[P][0][j][k] : 0.0;
    f1[s] = lane_ok ? c_tab1d[P][1][j][k] : 0.0;
    srcf[s] = lane_ok ? base + k : lane;
    srcb[s] = lane_ok ? base + (j - s + 3) % 3 : lane;
  }
  const int srcu0 = lane_ok ? 9 * cl + j : lane, srcu1 = lane_ok ? 9 * cl + 3 + j : lane,
            srcu2 = lane_ok ? 9 * cl + 6 + j : lane;  // component lanes of the same plane
  const double tZ = lane_ok ? c_x1d[P][j] : 0.5, wz = lane_ok ? c_w1d[P][j] : 0.0;
  // VSHARE: this lane's qx = a (point, weight) and the lanes of component (a + s) % 3
  const double tXa = lane_ok ? c_x1d[P][a] : 0.5, wXa = lane_ok ? c_w1d[P][a] : 0.0;
  int srcc[3], srcv[3];
#pragma unroll
  for (int s = 0; s < 3; ++s) {
    srcc[s] = lane_ok ? 9 * cl + 3 * ((a + s) % 3) + j : lane;
    srcv[s] = lane_ok ? 9 * cl + 3 * s + j : lane;  // component lane s holds v at qx = s
  }
  const int64_t nloc = e1 - e0;
  const int wpb = blockDim.x >> 5;
  const int64_t gw = (int64_t)blockIdx.x * wpb + (threadIdx.x >> 5), nw = (int64_t)gridDim.x * wpb;
  constexpr int TH = FEB200_T3_THREADS;
  extern __shared__ __align__(16) unsigned char t3s[];
  double* s2u = reinterpret_cast<double*>(t3s);                 // [2][9][TH]
  double* s2x = s2u + 2 * 9 * TH;                               // [2][8][TH]
  int32_t* s1d = reinterpret_cast<int32_t*>(s2x + 2 * 8 * TH);  // [3][9][TH]
  int32_t* s1c = s1d + 3 * 9 * TH;                              // [3][8][TH]
  const int tid = threadIdx.x;
  auto group_cell = [&](int64_t g, int64_t& le, bool& ok) {
    le = (gw + g * nw) * 3 + cl;
    ok = lane_ok && le < nloc;
  };
  auto issue_s1 = [&](int64_t g) {
    int64_t le;
    bool ok;
    group_cell(g, le, ok);
    if (ok) {
      const int sl = (int)(g % 3);
      const int64_t e = e0 + le;
#pragma unroll
      for (int k = 0; k < 9; ++k) t3_cp4(&s1d[(sl * 9 + k) * TH + tid], mv.dof_conn + e * NB + N * N * j + k);
      if (a == 0) {
#pragma unroll
        for (int v = 0; v < 8; ++v) t3_cp4(&s1c[(sl * 8 + v) * TH + tid], mv.conn + 8 * e + v);
      }
    }
    t3_commit();
  };
  auto issue_s2 = [&](int64_t g) {
    int64_t le;
    bool ok;
    group_cell(g, le, ok);
    if (ok) {
      const int s1 = (int)(g % 3), s2 = (int)(g & 1);
      // staged indices first, then the copies (see the scalar kernel)
      int dd[9];
#pragma unroll
      for (int k = 0; k < 9; ++k) dd[k] = s1d[(s1 * 9 + k) * TH + tid];
#pragma unroll
      for (int k = 0; k < 9; ++k) t3_cp8(&s2u[(s2 * 9 + k) * TH + tid], u + 3 * (int64_t)dd[k] + a);
      if (a == 0) {
        int vv[8];
#pragma unroll
        for (int h = 0; h < 8; ++h) vv[h] = s1c[(s1 * 8 + (8 * j + h) / 3) * TH + tid];
#pragma unroll
        for (int h = 0; h < 8; ++h) {
          const int pidx = 8 * j + h, i = pidx % 3;
          t3_cp8(&s2x[(s2 * 8 + h) * TH + tid], mv.coords + 3 * (int64_t)vv[h] + i);
        }
      }
    }
    t3_commit();
  };
  issue_s1(0);
  issue_s1(1);
  t3_wait<1>();
  issue_s2(0);
  for (int64_t g = 0;; ++g) {
    int64_t le;
    bool valid;
    group_cell(g, le, valid);
    if ((gw + g * nw) * 3 >= nloc) break;
    t3_wait<0>();
    __syncwarp();
    issue_s2(g + 1);
    issue_s1(g + 2);
    const int s1 = (int)(g % 3), s2 = (int)(g & 1);
    int dof[N][N];
    double uv[N][N];
#pragma unroll
    for (int ky = 0; ky < N; ++ky)
#pragma unroll
      for (int kx = 0; kx < N; ++kx) {
        dof[ky][kx] = s1d[(s1 * 9 + kx + N * ky) * TH + tid];
        uv[ky][kx] = valid ? s2u[(s2 * 9 + kx + N * ky) * TH + tid] : 0.0;
      }
    double c00[N][N], c01[N][N], c10[N][N];
    {
      double a0[N][N], a1[N][N];
#pragma unroll
      for (int ky = 0; ky < N; ++ky)
#pragma unroll
        for (int qx = 0; qx < N; ++qx) {
          double s0 = 0.0, sd = 0.0;
#pragma unroll
          for (int kx = 0; kx < N; ++kx) {
            s0 = fma(B0(qx, kx), uv[ky][kx], s0);
            sd = fma(B1(qx, kx), uv[ky][kx], sd);
          }
          a0[ky][qx] = s0;
          a1[ky][qx] = sd;
        }
#pragma unroll
      for (int qy = 0; qy < N; ++qy)
#pragma unroll
        for (int qx = 0; qx < N; ++qx) {
          double s00 = 0.0, s01 = 0.0, s10 = 0.0;
#pragma unroll
          for (int ky = 0; ky < N; ++ky) {
            s00 = fma(B0(qy, ky), a0[ky][qx], s00);
            s01 = fma(B1(qy, ky), a0[ky][qx], s01);
            s10 = fma(B0(qy, ky), a1[ky][qx], s10);
          }
          c00[qy][qx] = s00;
          c01[qy][qx] = s01;
          c10[qy][qx] = s10;
        }
    }
    double Uq[N][N], Gx[N][N], Gy[N][N], Gz[N][N];
#pragma unroll
    for (int qy = 0; qy < N; ++qy)
#pragma unroll
      for (int qx = 0; qx < N; ++qx) {
        const double v00 = c00[qy][qx], v01 = c01[qy][qx], v10 = c10[qy][qx];
        double uq = f0[0] * v00, gz = f1[0] * v00, gy = f0[0] * v01, gx = f0[0] * v10;
#pragma unroll
        for (int s = 1; s < 3; ++s) {
          const double w00 = __shfl_sync(0xffffffffu, v00, srcf[s]);
          const double w01 = __shfl_sync(0xffffffffu, v01, srcf[s]);
          const double w10 = __shfl_sync(0xffffffffu, v10, srcf[s]);
          uq = fma(f0[s], w00, uq);
          gz = fma(f1[s], w00, gz);
          gy = fma(f0[s], w01, gy);
          gx = fma(f0[s], w10, gx);
        }
        Uq[qy][qx] = uq;
        Gx[qy][qx] = gx;
        Gy[qy][qx] = gy;
        Gz[qy][qx] = gz;
      }
    double X[8][3];
    const int wb = tid - lane;
#pragma unroll
    for (int pidx = 0; pidx < 24; ++pidx)
      X[pidx / 3][pidx % 3] = valid ? s2x[(s2 * 8 + pidx % 8) * TH + wb + 9 * cl + pidx / 8] : 0.0;
    // separable trilinear Jacobian on this lane's plane (t2 = tZ fixed): column 0 is linear in
    // t1, column 1 linear in t0, column 2 bilinear; the t2 interpolation is done once per cell
    double gE0[3], gdE[3], gF0[3], gdF[3], gH0[N][3], gdH[N][3];
#pragma unroll
    for (int i = 0; i < 3; ++i) {
      const double e0 = (1 - tZ) * (X[1][i] - X[0][i]) + tZ * (X[5][i] - X[4][i]);
      const double e1 = (1 - tZ) * (X[3][i] - X[2][i]) + tZ * (X[7][i] - X[6][i]);
      const double f0_ = (1 - tZ) * (X[2][i] - X[0][i]) + tZ * (X[6][i] - X[4][i]);
      const double f1_ = (1 - tZ) * (X[3][i] - X[1][i]) + tZ * (X[7][i] - X[5][i]);
      gE0[i] = e0; gdE[i] = e1 - e0; gF0[i] = f0_; gdF[i] = f1_ - f0_;
#pragma unroll
      for (int qx = 0; qx < N; ++qx) {
        const double t0 = c_x1d[P][qx];
        const double h0 = (1 - t0) * (X[4][i] - X[0][i]) + t0 * (X[5][i] - X[1][i]);
        const double h1 = (1 - t0) * (X[6][i] - X[2][i]) + t0 * (X[7][i] - X[3][i]);
        gH0[qx][i] = h0;
        gdH[qx][i] = h1 - h0;
      }
    }
    double Fv[N][N];
    if constexpr (FEB200_T3C_VSHARE) {
      // u_b at the qps (qx = a, qy) of this plane: own component by select, the others from the
      // component lanes b = (a + s) % 3, which send their value at qx = a = (b - s) % 3
      double U3[N][3];
#pragma unroll
      for (int s = 0; s < 3; ++s) {
        const int xs = (a - s + 3) % 3;  // the qx the lane of component a - s asks this lane for
#pragma unroll
        for (int qy = 0; qy < N; ++qy) {
          const double snd = xs == 0 ? Uq[qy][0] : (xs == 1 ? Uq[qy][1] : Uq[qy][2]);
          U3[qy][s] = s == 0 ? snd : __shfl_sync(0xffffffffu, snd, srcc[s]);
        }
      }
      // v = w C u at (qx = a, qy):  v_m = sum_r C_rm u_r
      double V[N][3];
#pragma unroll
      for (int qy = 0; qy < N; ++qy) {
        const double t1 = c_x1d[P][qy];
        double J[3][3];
#pragma unroll
        for (int i = 0; i < 3; ++i) {
          const double h0 = (1 - tXa) * (X[4][i] - X[0][i]) + tXa * (X[5][i] - X[1][i]);
          const double h1 = (1 - tXa) * (X[6][i] - X[2][i]) + tXa * (X[7][i] - X[3][i]);
          J[i][0] = fma(t1, gdE[i], gE0[i]);
          J[i][1] = fma(tXa, gdF[i], gF0[i]);
          J[i][2] = fma(t1, h1 - h0, h0);
        }
        const double C00 = J[1][1] * J[2][2] - J[1][2] * J[2][1], C01 = J[1][2] * J[2][0] - J[1][0] * J[2][2],
                     C02 = J[1][0] * J[2][1] - J[1][1] * J[2][0], C10 = J[0][2] * J[2][1] - J[0][1] * J[2][2],
                     C11 = J[0][0] * J[2][2] - J[0][2] * J[2][0], C12 = J[0][1] * J[2][0] - J[0][0] * J[2][1],
                     C20 = J[0][1] * J[1][2] - J[0][2] * J[1][1], C21 = J[0][2] * J[1][0] - J[0][0] * J[1][2],
                     C22 = J[0][0] * J[1][1] - J[0][1] * J[1][0];
        // U3[qy][s] = u_{(a + s) % 3}: back to component order
        const double u0 = a == 0 ? U3[qy][0] : (a == 1 ? U3[qy][2] : U3[qy][1]);
        const double u1 = a == 0 ? U3[qy][1] : (a == 1 ? U3[qy][0] : U3[qy][2]);
        const double u2 = a == 0 ? U3[qy][2] : (a == 1 ? U3[qy][1] : U3[qy][0]);
        const double wq = wXa * c_w1d[P][qy] * wz;
        V[qy][0] = wq * (C00 * u0 + C10 * u1 + C20 * u2);
        V[qy][1] = wq * (C01 * u0 + C11 * u1 + C21 * u2);
        V[qy][2] = wq * (C02 * u0 + C12 * u1 + C22 * u2);
      }
      // detw f0_a = w sum_r t_r u_r = grad_ref u_a . v  (t = C^T grad_ref u_a)
#pragma unroll
      for (int qy = 0; qy < N; ++qy)
#pragma unroll
        for (int qx = 0; qx < N; ++qx) {
          const double v0 = __shfl_sync(0xffffffffu, V[qy][0], srcv[qx]);
          const double v1 = __shfl_sync(0xffffffffu, V[qy][1], srcv[qx]);
          const double v2 = __shfl_sync(0xffffffffu, V[qy][2], srcv[qx]);
          Fv[qy][qx] = valid ? (Gx[qy][qx] * v0 + Gy[qy][qx] * v1 + Gz[qy][qx] * v2) : 0.0;
        }
    } else {
#pragma unroll
    for (int qy = 0; qy < N; ++qy)
#pragma unroll
      for (int qx = 0; qx < N; ++qx) {
        const double t0 = c_x1d[P][qx], t1 = c_x1d[P][qy];
        double J[3][3];
#pragma unroll
        for (int i = 0; i < 3; ++i) {
          if (FEB200_T3_SEPGEO) {
            J[i][0] = fma(t1, gdE[i], gE0[i]);
            J[i][1] = fma(t0, gdF[i], gF0[i]);
            J[i][2] = fma(t1, gdH[qx][i], gH0[qx][i]);
          } else {
            const double t2 = tZ;
            J[i][0] = (1 - t1) * (1 - t2) * (X[1][i] - X[0][i]) + t1 * (1 - t2) * (X[3][i] - X[2][i]) +
                      (1 - t1) * t2 * (X[5][i] - X[4][i]) + t1 * t2 * (X[7][i] - X[6][i]);
            J[i][1] = (1 - t0) * (1 - t2) * (X[2][i] - X[0][i]) + t0 * (1 - t2) * (X[3][i] - X[1][i]) +
                      (1 - t0) * t2 * (X[6][i] - X[4][i]) + t0 * t2 * (X[7][i] - X[5][i]);
            J[i][2] = (1 - t0) * (1 - t1) * (X[4][i] - X[0][i]) + t0 * (1 - t1) * (X[5][i] - X[1][i]) +
                      (1 - t0) * t1 * (X[6][i] - X[2][i]) + t0 * t1 * (X[7][i] - X[3][i]);
          }
        }
        const double C00 = J[1][1] * J[2][2] - J[1][2] * J[2][1], C01 = J[1][2] * J[2][0] - J[1][0] * J[2][2],
                     C02 = J[1][0] * J[2][1] - J[1][1] * J[2][0], C10 = J[0][2] * J[2][1] - J[0][1] * J[2][2],
                     C11 = J[0][0] * J[2][2] - J[0][2] * J[2][0], C12 = J[0][1] * J[2][0] - J[0][0] * J[2][1],
                     C20 = J[0][1] * J[1][2] - J[0][2] * J[1][1], C21 = J[0][2] * J[1][0] - J[0][0] * J[1][2],
                     C22 = J[0][0] * J[1][1] - J[0][1] * J[1][0];
        const double g0 = Gx[qy][qx], g1 = Gy[qy][qx], g2 = Gz[qy][qx];
        const double tr0 = C00 * g0 + C01 * g1 + C02 * g2;  // det (grad u_a)_r
        const double tr1 = C10 * g0 + C11 * g1 + C12 * g2;
        const double tr2 = C20 * g0 + C21 * g1 + C22 * g2;
        const double uq = Uq[qy][qx];
        const double w0 = __shfl_sync(0xffffffffu, uq, srcu0);  // u_0, u_1, u_2 at the qp
        const double w1 = __shfl_sync(0xffffffffu, uq, srcu1);
        const double w2 = __shfl_sync(0xffffffffu, uq, srcu2);
        const double wq = c_w1d[P][qx] * c_w1d[P][qy] * wz;
        Fv[qy][qx] = valid ? wq * (tr0 * w0 + tr1 * w1 + tr2 * w2) : 0.0;
      }
    }
    double Hv[N][N];
#pragma unroll
    for (int qy = 0; qy < N; ++qy)
#pragma unroll
      for (int qx = 0; qx < N; ++qx) {
        const double fv = Fv[qy][qx];
        double hv = f0[0] * fv;
#pragma unroll
        for (int s = 1; s < 3; ++s) hv += __shfl_sync(0xffffffffu, f0[s] * fv, srcb[s]);
        Hv[qy][qx] = hv;
      }
    double ev = 0.0;
#pragma unroll
    for (int ky = 0; ky < N; ++ky) {
      double Iv[N];
#pragma unroll
      for (int qx = 0; qx < N; ++qx) {
        double sv = 0.0;
#pragma unroll
        for (int qy = 0; qy < N; ++qy) sv = fma(B0(qy, ky), Hv[qy][qx], sv);
        Iv[qx] = sv;
      }
#pragma unroll
      for (int kx = 0; kx < N; ++kx) {
        double rr = 0.0;
#pragma unroll
        for (int qx = 0; qx < N; ++qx) rr = fma(B0(qx, kx), Iv[qx], rr);
        if (valid) {
          if (r_elem) r_elem[le * 3 * NB + a * NB + kx + N * ky + N * N * j] = rr;
          if (r_global) atomicAdd(r_global + 3 * (int64_t)dof[ky][kx] + a, rr);
          if constexpr (PEER) peer_scatter<3>(pw, dof[ky][kx], a, rr);
          if (EVAL) ev = fma(rr, uv[ky][kx], ev);
        }
      }
    }
    if (EVAL) {
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) ev += __shfl_xor_sync(0xffffffffu, ev, o);
      if (lane == 0 && ev != 0.0) atomicAdd(eval_out, ev);
    }
  }
  t3_wait<0>();
#undef B0
#undef B1
}

static cudaError_t launch_t3c(const fe_mesh* mh, const double* u, int64_t e0, int64_t e1,
                              double* r_elem, double* r_global, double* eval_out, cudaStream_t st) {
  const PeerWin pw = g_peer;
  auto kern = eval_out ? k_residual_t3c<true> : (pw.n > 0 ? k_residual_t3c<false, true>
                                                            : k_residual_t3c<false>);
  const size_t smem = (size_t)FEB200_T3_THREADS * (8 * (2 * 9 + 2 * 8) + 4 * (3 * 9 + 3 * 8));
  const LaunchFacts lf = launch_facts((const void*)kern, FEB200_T3_THREADS, smem);
  if (lf.err != cudaSuccess) return lf.err;
  const int nsm = lf.nsm, per_sm = lf.per_sm;
  const int64_t ncg = (e1 - e0 + 2) / 3;                        // 3 cells per warp
  const int64_t nblk = (ncg + FEB200_T3_THREADS / 32 - 1) / (FEB200_T3_THREADS / 32);
  int grid = (int)(nblk < (int64_t)nsm * per_sm ? nblk : (int64_t)nsm * per_sm);
  grid = grid_cap(grid);
  if (grid <= 0) return cudaSuccess;
  kern<<<grid, FEB200_T3_THREADS, smem, st>>>(view_of(mh), u, e0, e1, r_elem, r_global, eval_out, pw);
  count_launch();
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------------------
// Isotropic linear elasticity residual r_(a,k) = int sum_r sigma_ar(u) d phi_k / dx_r (P:1033,
// Voigt D = lambda m m^T + mu (2 I_3 (+) I_3), contracted analytically) at p = 2, fp64,
// register-resident with the lane layout of k_residual_t3c: NINE lanes per cell, lane (a, j)
// owning component a on z-plane j.  Forward pass per component (x, y in registers, z by
// shuffles among the plane lanes) gives the reference gradient g of u_a at the lane's 9 qps;
// t = C g = det grad u_a (C the cofactors of J).  The stress needs, from the other component
// lanes b of the same plane, t_b[b] (the trace) and t_b[a] (the symmetric part): four shuffles
// per qp.  With S_r = det sigma_ar = lambda delta_ar sum_b t_b[b] + mu (t_a[r] + t_r[a]),
//   F_m = detw sum_r sigma_ar J^-1[m][r] = (w / det) sum_r C[r][m] S_r,
// and the backward pass is that of the scalar diffusion kernel (z^T by shuffles, y^T, x^T in
// registers, fused scatter).  PERQP: lambda, mu per quadrature point, else per cell.
template <bool PERQP, bool EVAL, bool PEER = false>
__global__ void __launch_bounds__(FEB200_T3_THREADS, FEB200_T3E_MINB)
    k_residual_t3e(MeshView mv, const double* __restrict__ ma, const double* __restrict__ mb,
                   const double* __restrict__ u, int64_t e0, int64_t e1, double* __restrict__ r_elem,
                   double* __restrict__ r_global, double* __restrict__ eval_out, PeerWin pw) {
  constexpr int P = 2, N = 3, NB = 27, NQ = 27;
  constexpr int NM = PERQP ? 18 : 2;  // staged material values per lane (lambda, mu)
#define B0(q, k) c_tab1d[P][0][q][k]
#define B1(q, k) c_tab1d[P][1][q][k]
  const int lane = threadIdx.x & 31;
  const int cl = lane / 9, rem = lane - 9 * cl, a = rem / 3, j = rem - 3 * a;
  const bool lane_ok = lane < 27;
  const int base = 9 * cl + 3 * a;  // the three plane lanes of (cell, component)
  double f0[3], f1[3];
  int srcf[3], srcb[3], srcc[3];
#pragma unroll
  for (int s = 0; s < 3; ++s) {
    const int k = (j + s) % 3;
    f0[s] = lane_ok ? c_tab1d[P][0][j][k] : 0.0;
    f1[s] = lane_ok ? c_tab1d[P][1][j][k] : 0.0;
    srcf[s] = lane_ok ? base + k : lane;
    srcb[s] = lane_ok ? base + (j - s + 3) % 3 : lane;
    srcc[s] = lane_ok ? 9 * cl + 3 * ((a + s) % 3) + j : lane;  // component (a + s) % 3, same plane
  }
  const double tZ = lane_ok ? c_x1d[P][j] : 0.5, wz = lane_ok ? c_w1d[P][j] : 0.0;
  const int64_t nloc = e1 - e0;
  const int wpb = blockDim.x >> 5;
  const int64_t gw = (int64_t)blockIdx.x * wpb + (threadIdx.x >> 5), nw = (int64_t)gridDim.x * wpb;
  constexpr int TH = FEB200_T3_THREADS;
  extern __shared__ __align__(16) unsigned char t3s[];
  double* s1m = reinterpret_cast<double*>(t3s);                 // [3][NM][TH]
  double* s2u = s1m + 3 * NM * TH;                              // [2][9][TH]
  double* s2x = s2u + 2 * 9 * TH;                               // [2][8][TH]
  int32_t* s1d = reinterpret_cast<int32_t*>(s2x + 2 * 8 * TH);  // [3][9][TH]
  int32_t* s1c = s1d + 3 * 9 * TH;                              // [3][8][TH]
  const int tid = threadIdx.x;
  auto group_cell = [&](int64_t g, int64_t& le, bool& ok) {
    le = (gw + g * nw) * 3 + cl;
    ok = lane_ok && le < nloc;
  };
  auto issue_s1 = [&](int64_t g) {
    int64_t le;
    bool ok;
    group_cell(g, le, ok);
    if (ok) {
      const int sl = (int)(g % 3);
      const int64_t e = e0 + le;
#pragma unroll
      for (int k = 0; k < 9; ++k) t3_cp4(&s1d[(sl * 9 + k) * TH + tid], mv.dof_conn + e * NB + N * N * j + k);
      if (a == 0) {
#pragma unroll
        for (int v = 0; v < 8; ++v) t3_cp4(&s1c[(sl * 8 + v) * TH + tid], mv.conn + 8 * e + v);
      }
      if constexpr (PERQP) {
#pragma unroll
        for (int k = 0; k < 9; ++k) {
          t3_cp8(&s1m[(sl * NM + k) * TH + tid], ma + e * NQ + N * N * j + k);
          t3_cp8(&s1m[(sl * NM + 9 + k) * TH + tid], mb + e * NQ + N * N * j + k);
        }
      } else {
        t3_cp8(&s1m[(sl * NM + 0) * TH + tid], ma + e);
        t3_cp8(&s1m[(sl * NM + 1) * TH + tid], mb + e);
      }
    }
    t3_commit();
  };
  auto issue_s2 = [&](int64_t g) {
    int64_t le;
    bool ok;
    group_cell(g, le, ok);
    if (ok) {
      const int s1 = (int)(g % 3), s2 = (int)(g & 1);
      int dd[9];
#pragma unroll
      for (int k = 0; k < 9; ++k) dd[k] = s1d[(s1 * 9 + k) * TH + tid];
#pragma unroll
      for (int k = 0; k < 9; ++k) t3_cp8(&s2u[(s2 * 9 + k) * TH + tid], u + 3 * (int64_t)dd[k] + a);
      if (a == 0) {
        int vv[8];
#pragma unroll
        for (int h = 0; h < 8; ++h) vv[h] = s1c[(s1 * 8 + (8 * j + h) / 3) * TH + tid];
#pragma unroll
        for (int h = 0; h < 8; ++h) {
          const int pidx = 8 * j + h, i = pidx % 3;
          t3_cp8(&s2x[(s2 * 8 + h) * TH + tid], mv.coords + 3 * (int64_t)vv[h] + i);
        }
      }
    }
    t3_commit();
  };
  issue_s1(0);
  issue_s1(1);
  t3_wait<1>();
  issue_s2(0);
  for (int64_t g = 0;; ++g) {
    int64_t le;
    bool valid;
    group_cell(g, le, valid);
    if ((gw + g * nw) * 3 >= nloc) break;
    t3_wait<0>();
    __syncwarp();
    issue_s2(g + 1);
    issue_s1(g + 2);
    const int s1 = (int)(g % 3), s2 = (int)(g & 1);
    int dof[N][N];
    double uv[N][N];
#pragma unroll
    for (int ky = 0; ky < N; ++ky)
#pragma unroll
      for (int kx = 0; kx < N; ++kx) {
        dof[ky][kx] = s1d[(s1 * 9 + kx + N * ky) * TH + tid];
        uv[ky][kx] = valid ? s2u[(s2 * 9 + kx + N * ky) * TH + tid] : 0.0;
      }
    // ---- forward: reference gradient of u_a at the qps (qx, qy, qz = j)
    double c01[N][N], c10[N][N], c00[N][N];
    {
      double a0[N][N], a1[N][N];
#pragma unroll
      for (int ky = 0; ky < N; ++ky)
#pragma unroll
        for (int qx = 0; qx < N; ++qx) {
          double s0 = 0.0, sd = 0.0;
#pragma unroll
          for (int kx = 0; kx < N; ++kx) {
            s0 = fma(B0(qx, kx), uv[ky][kx], s0);
            sd = fma(B1(qx, kx), uv[ky][kx], sd);
          }
          a0[ky][qx] = s0;
          a1[ky][qx] = sd;
        }
#pragma unroll
      for (int qy = 0; qy < N; ++qy)
#pragma unroll
        for (int qx = 0; qx < N; ++qx) {
          double s00 = 0.0, s01 = 0.0, s10 = 0.0;
#pragma unroll
          for (int ky = 0; ky < N; ++ky) {
            s00 = fma(B0(qy, ky), a0[ky][qx], s00);
            s01 = fma(B1(qy, ky), a0[ky][qx], s01);
            s10 = fma(B0(qy, ky), a1[ky][qx], s10);
          }
          c00[qy][qx] = s00;
          c01[qy][qx] = s01;
          c10[qy][qx] = s10;
        }
    }
    double Gx[N][N], Gy[N][N], Gz[N][N];
#pragma unroll
    for (int qy = 0; qy < N; ++qy)
#pragma unroll
      for (int qx = 0; qx < N; ++qx) {
        const double v00 = c00[qy][qx], v01 = c01[qy][qx], v10 = c10[qy][qx];
        double gz = f1[0] * v00, gy = f0[0] * v01, gx = f0[0] * v10;
#pragma unroll
        for (int s = 1; s < 3; ++s) {
          const double w00 = __shfl_sync(0xffffffffu, v00, srcf[s]);
          const double w01 = __shfl_sync(0xffffffffu, v01, srcf[s]);
          const double w10 = __shfl_sync(0xffffffffu, v10, srcf[s]);
          gz = fma(f1[s], w00, gz);
          gy = fma(f0[s], w01, gy);
          gx = fma(f0[s], w10, gx);
        }
        Gx[qy][qx] = gx;
        Gy[qy][qx] = gy;
        Gz[qy][qx] = gz;
      }
    double X[8][3];
    const int wb = tid - lane;
#pragma unroll
    for (int pidx = 0; pidx < 24; ++pidx)
      X[pidx / 3][pidx % 3] = valid ? s2x[(s2 * 8 + pidx % 8) * TH + wb + 9 * cl + pidx / 8] : 0.0;
    double gE0[3], gdE[3], gF0[3], gdF[3], gH0[N][3], gdH[N][3];
#pragma unroll
    for (int i = 0; i < 3; ++i) {
      const double e0_ = (1 - tZ) * (X[1][i] - X[0][i]) + tZ * (X[5][i] - X[4][i]);
      const double e1_ = (1 - tZ) * (X[3][i] - X[2][i]) + tZ * (X[7][i] - X[6][i]);
      const double f0_ = (1 - tZ) * (X[2][i] - X[0][i]) + tZ * (X[6][i] - X[4][i]);
      const double f1_ = (1 - tZ) * (X[3][i] - X[1][i]) + tZ * (X[7][i] - X[5][i]);
      gE0[i] = e0_; gdE[i] = e1_ - e0_; gF0[i] = f0_; gdF[i] = f1_ - f0_;
#pragma unroll
      for (int qx = 0; qx < N; ++qx) {
        const double t0 = c_x1d[P][qx];
        const double h0 = (1 - t0) * (X[4][i] - X[0][i]) + t0 * (X[5][i] - X[1][i]);
        const double h1 = (1 - t0) * (X[6][i] - X[2][i]) + t0 * (X[7][i] - X[3][i]);
        gH0[qx][i] = h0;
        gdH[qx][i] = h1 - h0;
      }
    }
    double lamE = 0.0, muE = 0.0;
    if constexpr (!PERQP) {
      lamE = s1m[(s1 * NM + 0) * TH + tid];
      muE = s1m[(s1 * NM + 1) * TH + tid];
    }
    // ---- flux F_m = (w / det) sum_r C[r][m] S_r at the 9 qps, the backward z^T pulled after
    double Fx[N][N], Fy[N][N], Fz[N][N];
#pragma unroll
    for (int qy = 0; qy < N; ++qy)
#pragma unroll
      for (int qx = 0; qx < N; ++qx) {
        const double t0 = c_x1d[P][qx], t1 = c_x1d[P][qy];
        double J[3][3];
#pragma unroll
        for (int i = 0; i < 3; ++i) {
          J[i][0] = fma(t1, gdE[i], gE0[i]);
          J[i][1] = fma(t0, gdF[i], gF0[i]);
          J[i][2] = fma(t1, gdH[qx][i], gH0[qx][i]);
        }
        const double C00 = J[1][1] * J[2][2] - J[1][2] * J[2][1], C01 = J[1][2] * J[2][0] - J[1][0] * J[2][2],
                     C02 = J[1][0] * J[2][1] - J[1][1] * J[2][0], C10 = J[0][2] * J[2][1] - J[0][1] * J[2][2],
                     C11 = J[0][0] * J[2][2] - J[0][2] * J[2][0], C12 = J[0][1] * J[2][0] - J[0][0] * J[2][1],
                     C20 = J[0][1] * J[1][2] - J[0][2] * J[1][1], C21 = J[0][2] * J[1][0] - J[0][0] * J[1][2],
                     C22 = J[0][0] * J[1][1] - J[0][1] * J[1][0];
        const double det = J[0][0] * C00 + J[0][1] * C01 + J[0][2] * C02;
        const double g0 = Gx[qy][qx], g1 = Gy[qy][qx], g2 = Gz[qy][qx];
        // t_r = det (grad u_a)_r
        const double ta0 = C00 * g0 + C01 * g1 + C02 * g2;
        const double ta1 = C10 * g0 + C11 * g1 + C12 * g2;
        const double ta2 = C20 * g0 + C21 * g1 + C22 * g2;
        // own diagonal t_a[a]; for the lane of component a - s: t_a[(a - s) % 3]
        const double dg = a == 0 ? ta0 : (a == 1 ? ta1 : ta2);
        const double sn1 = a == 0 ? ta2 : (a == 1 ? ta0 : ta1);  // (a - 1) % 3
        const double sn2 = a == 0 ? ta1 : (a == 1 ? ta2 : ta0);  // (a - 2) % 3
        const double rd1 = __shfl_sync(0xffffffffu, dg, srcc[1]);   // t_b[b], b = (a + 1) % 3
        const double ro1 = __shfl_sync(0xffffffffu, sn1, srcc[1]);  // t_b[a]
        const double rd2 = __shfl_sync(0xffffffffu, dg, srcc[2]);   // b = (a + 2) % 3
        const double ro2 = __shfl_sync(0xffffffffu, sn2, srcc[2]);
        double lam = lamE, mu = muE;
        if constexpr (PERQP) {
          lam = s1m[(s1 * NM + qx + N * qy) * TH + tid];
          mu = s1m[(s1 * NM + 9 + qx + N * qy) * TH + tid];
        }
        const double T = dg + rd1 + rd2;  // det tr(grad u)
        // S_r in rotated order: r = a, (a + 1) % 3, (a + 2) % 3
        const double S0r = fma(lam, T, 2.0 * mu * dg);
        const double t_a1 = a == 0 ? ta1 : (a == 1 ? ta2 : ta0);  // t_a[(a + 1) % 3]
        const double t_a2 = a == 0 ? ta2 : (a == 1 ? ta0 : ta1);  // t_a[(a + 2) % 3]
        const double S1r = mu * (t_a1 + ro1);
        const double S2r = mu * (t_a2 + ro2);
        const double S0 = a == 0 ? S0r : (a == 1 ? S2r : S1r);
        const double S1 = a == 0 ? S1r : (a == 1 ? S0r : S2r);
        const double S2 = a == 0 ? S2r : (a == 1 ? S1r : S0r);
        const double sc = valid ? c_w1d[P][qx] * c_w1d[P][qy] * wz * rcp_nr(det) : 0.0;
        Fx[qy][qx] = sc * (C00 * S0 + C10 * S1 + C20 * S2);
        Fy[qy][qx] = sc * (C01 * S0 + C11 * S1 + C21 * S2);
        Fz[qy][qx] = sc * (C02 * S0 + C12 * S1 + C22 * S2);
      }
    // ---- z^T through the component's plane lanes
    double Hv[N][N], Hx[N][N], Hy[N][N];
#pragma unroll
    for (int qy = 0; qy < N; ++qy)
#pragma unroll
      for (int qx = 0; qx < N; ++qx) {
        const double fx = Fx[qy][qx], fy = Fy[qy][qx], fz = Fz[qy][qx];
        double hv = f1[0] * fz, hx = f0[0] * fx, hy = f0[0] * fy;
#pragma unroll
        for (int s = 1; s < 3; ++s) {
          hv += __shfl_sync(0xffffffffu, f1[s] * fz, srcb[s]);
          hx += __shfl_sync(0xffffffffu, f0[s] * fx, srcb[s]);
          hy += __shfl_sync(0xffffffffu, f0[s] * fy, srcb[s]);
        }
        Hv[qy][qx] = hv;
        Hx[qy][qx] = hx;
        Hy[qy][qx] = hy;
      }
    double ev = 0.0;
#pragma unroll
    for (int ky = 0; ky < N; ++ky) {
      double Iv[N], Ix[N];
#pragma unroll
      for (int qx = 0; qx < N; ++qx) {
        double sv = 0.0, sx = 0.0;
#pragma unroll
        for (int qy = 0; qy < N; ++qy) {
          sv = fma(B0(qy, ky), Hv[qy][qx], sv);
          sv = fma(B1(qy, ky), Hy[qy][qx], sv);
          sx = fma(B0(qy, ky), Hx[qy][qx], sx);
        }
        Iv[qx] = sv;
        Ix[qx] = sx;
      }
#pragma unroll
      for (int kx = 0; kx < N; ++kx) {
        double rr = 0.0;
#pragma unroll
        for (int qx = 0; qx < N; ++qx) {
          rr = fma(B0(qx, kx), Iv[qx], rr);
          rr = fma(B1(qx, kx), Ix[qx], rr);
        }
        if (valid) {
          if (r_elem) r_elem[le * 3 * NB + a * NB + kx + N * ky + N * N * j] = rr;
          if (r_global) atomicAdd(r_global + 3 * (int64_t)dof[ky][kx] + a, rr);
          if constexpr (PEER) peer_scatter<3>(pw, dof[ky][kx], a, rr);
          if (EVAL) ev = fma(rr, uv[ky][kx], ev);
        }
      }
    }
    if (EVAL) {
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) ev += __shfl_xor_sync(0xffffffffu, ev, o);
      if (lane == 0 && ev != 0.0) atomicAdd(eval_out, ev);
    }
  }
  t3_wait<0>();
#undef B0
#undef B1
}

template <bool PERQP>
static cudaError_t launch_t3e_t(const fe_mesh* mh, MatArgs mat, const double* u, int64_t e0, int64_t e1,
                                double* r_elem, double* r_global, double* eval_out, cudaStream_t st) {
  const PeerWin pw = g_peer;
  auto kern = eval_out ? k_residual_t3e<PERQP, true>
                       : (pw.n > 0 ? k_residual_t3e<PERQP, false, true> : k_residual_t3e<PERQP, false>);
  constexpr int NM = PERQP ? 18 : 2;
  const size_t smem = (size_t)FEB200_T3_THREADS * (8 * (3 * NM + 2 * 9 + 2 * 8) + 4 * (3 * 9 + 3 * 8));
  const LaunchFacts lf = launch_facts((const void*)kern, FEB200_T3_THREADS, smem);
  if (lf.err != cudaSuccess) return lf.err;
  const int nsm = lf.nsm, per_sm = lf.per_sm;
  const int64_t ncg = (e1 - e0 + 2) / 3;  // 3 cells per warp
  const int64_t nblk = (ncg + FEB200_T3_THREADS / 32 - 1) / (FEB200_T3_THREADS / 32);
  int grid = (int)(nblk < (int64_t)nsm * per_sm ? nblk : (int64_t)nsm * per_sm);
  grid = grid_cap(grid);
  if (grid <= 0) return cudaSuccess;
  kern<<<grid, FEB200_T3_THREADS, smem, st>>>(view_of(mh), (const double*)mat.a, (const double*)mat.b, u,
                                              e0, e1, r_elem, r_global, eval_out, pw);
  count_launch();
  return cudaGetLastError();
}

// Scalar forms at p = 2 in fp64; cudaErrorNotSupported otherwise (the smem kernel runs).
cudaError_t launch_residual_t3(const fe_mesh* mh, int form, MatArgs mat, const double* u, int64_t e0,
                               int64_t e1, double* r_elem, double* r_global, cudaStream_t st,
                               double* eval_out) {
  if (mh->order != 2 || mh->q1d != 3) return cudaErrorNotSupported;
  switch (form) {
    case FE_FORM_DIFFUSION: return launch_t3_t<FE_FORM_DIFFUSION>(mh, mat, u, e0, e1, r_elem, r_global, eval_out, st);
    case FE_FORM_MASS: return launch_t3_t<FE_FORM_MASS>(mh, mat, u, e0, e1, r_elem, r_global, eval_out, st);
    case FE_FORM_MASS_DIFFUSION:
      return launch_t3_t<FE_FORM_MASS_DIFFUSION>(mh, mat, u, e0, e1, r_elem, r_global, eval_out, st);
    case FE_FORM_CONVECTIVE:
      if (FEB200_T3C) return launch_t3c(mh, u, e0, e1, r_elem, r_global, eval_out, st);
      return cudaErrorNotSupported;
    case FE_FORM_ELASTICITY:  // isotropic lambda, mu per cell or per qp (general D: the smem kernel)
      if (!FEB200_T3E) return cudaErrorNotSupported;
      if (mat.kind == FE_MAT_PER_ELEM) return launch_t3e_t<false>(mh, mat, u, e0, e1, r_elem, r_global, eval_out, st);
      if (mat.kind == FE_MAT_PER_QP) return launch_t3e_t<true>(mh, mat, u, e0, e1, r_elem, r_global, eval_out, st);
      return cudaErrorNotSupported;
    default: return cudaErrorNotSupported;
  }
}

}  // namespace feb200
