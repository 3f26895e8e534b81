// Sum-factorised element matrices for the symmetric scalar forms (diffusion,
// mass, mass + diffusion) -- SURVEY 8(f) N1, applied to matrix mode.
//
// Same integral as Alg. 2 and the einsum
// 'cq,cqjd,cqje->cde', reorganised with the tensor-product structure
// of the Lagrange basis (Eq. fe1) and of the Gauss rule:
//
//   K[i][j] = sum_{m,n} sum_q W^{mn}(q) D^m_i(q) D^n_j(q),
//   W^{mn}(q) = detw(q) kappa(q) sum_k Jinv[m][k] Jinv[n][k]   (m, n < 3)
//   W^{33}(q) = detw(q) rho(q)                                   (value-value)
//   D^m_i(q)  = prod_d B^{[m == d]}[q_d][i_d]   (B^0 values, B^1 derivatives, 1D)
//
// contracted one axis at a time:
//   stage z: T1^{mn}[qx,qy][iz,jz]   = sum_qz B^{mz}[qz][iz] B^{nz}[qz][jz] W^{mn}[qx,qy,qz]
//   stage y: S_c[qx][(iy,iz),(jy,jz)] = sum_{(m,n) in class c} sum_qy B^{my}B^{ny} T1^{mn}
//   stage x: K[(ix,.),(jx,.)]         = sum_qx sum_{a,b} B^a[qx][ix] B^b[qx][jx] S_{(a,b)}[qx]
// where class c = ([m==0], [n==0]).  W symmetric => only m <= n is formed and
// K is symmetric => only z-pairs iz <= jz are computed and mirrored.
// Q2: ~12k FMA per cell instead of ~66k for the dense form; the 5.8 KB K_e
// write then dominates, so K is staged in shared memory and written with TMA
// bulk stores (cp.async.bulk) that overlap the next batch.
#ifndef FEB200_SF_E2
#define FEB200_SF_E2 2
#endif
#ifndef FEB200_SFP_E2
#define FEB200_SFP_E2 8
#endif
#ifndef FEB200_SFP
#define FEB200_SFP 1
#endif
#ifndef FEB200_SFP_T1PAD
#define FEB200_SFP_T1PAD 13
#endif
#ifndef FEB200_SFP_NOSTORE
#define FEB200_SFP_NOSTORE 0
#endif
#ifndef FEB200_SFP_NOX
#define FEB200_SFP_NOX 0
#endif
#ifndef FEB200_SFP_NOG
#define FEB200_SFP_NOG 0  // experiment: G skips geometry and stage z (X reads stale T1)
#endif
#ifndef FEB200_SFP_GH
#define FEB200_SFP_GH 1
#endif
#ifndef FEB200_SFP_YB
#define FEB200_SFP_YB 3  // y pairs per X thread at p = 2 (1 or 3)
#endif
#ifndef FEB200_SFP_ZTRI
#define FEB200_SFP_ZTRI 1  // stage z: only z pairs iz <= jz for the pairs m == n
#endif
#ifndef FEB200_SFP_MAP
#define FEB200_SFP_MAP 1  // YB = 3: generated lane -> task permutation (sfp_tasks.h)
#endif
#ifndef FEB200_SF_MINB
#define FEB200_SF_MINB 1
#endif
#ifndef FEB200_SFP_EVF
#define FEB200_SFP_EVF 0  // experiment: L2 evict_first hint on the K bulk stores (C2 +0.3 %: off)
#endif
#include "fe_const.cuh"
#include "fe_device.cuh"
#include "fe_internal.h"
#include "sfp_tasks.h"
#include <cstdlib>
#include <cstring>
#include <type_traits>

namespace feb200 {

template <int P, bool DIFF, bool MASS>
struct SFM {
  static constexpr int N1 = P + 1, Q1 = P + 1, NB = N1 * N1 * N1, NQ = Q1 * Q1 * Q1;
  static constexpr int NUP = (DIFF ? 6 : 0) + (MASS ? 1 : 0);   // unique (m <= n) pairs
  static constexpr int NOP = (DIFF ? 9 : 0) + (MASS ? 1 : 0);   // ordered pairs
  static constexpr int YP = N1 * N1, YPS = N1 * (N1 + 1) / 2;
  // stage-y/x threads per cell: z-pairs iz < jz with every y-pair, and iz == jz
  // with y-pairs iy <= jy (the rest of K follows by symmetry)
  static constexpr int TOFF = YP * (N1 * (N1 - 1) / 2);
  static constexpr int TPE = TOFF + N1 * YPS;
  static constexpr int E = P == 1 ? 8 : (P == 2 ? FEB200_SF_E2 : 1);  // cells per CTA iteration
  static constexpr int T_GEO = E * NQ, T_Z = E * NUP * Q1 * Q1, T_YX = E * TPE, T_EDGE = E * 36;
  static constexpr int M1 = T_GEO > T_Z ? T_GEO : T_Z, M2 = T_YX > T_EDGE ? T_YX : T_EDGE;
  static constexpr int THREADS = ((M1 > M2 ? M1 : M2) + 31) / 32 * 32;
  // shared memory (doubles)
  static constexpr int KST = E * NB * NB;                       // one staging buffer
  // K staging buffers: two (the TMA store of batch it overlaps batch it + 1), one at p = 4
  // (K_e alone is 125 KB there)
  static constexpr int NKB = P >= 4 ? 1 : 2;
  static constexpr int QQP = (Q1 * Q1 + 1) / 2 * 2;             // (qx,qy) padded for LDS.128
  static constexpr int OFF_K = 0;                               // 2 x KST (16-B aligned)
  static constexpr int OFF_EDGE = OFF_K + NKB * KST;            // [E][3 dirs][4][3]
  static constexpr int OFF_COEF = OFF_EDGE + E * 36;            // [E][2][NQ] kappa, rho
  static constexpr int OFF_W = OFF_COEF + E * 2 * NQ;           // [E][NUP][NQ]
  static constexpr int OFF_T1 = (OFF_W + E * NUP * NQ + 1) / 2 * 2;  // [E][NUP][N1*N1][QQP]
  static constexpr int OFF_XW = OFF_T1 + E * NUP * N1 * N1 * QQP;  // [2][Q1] 1D points, weights
  static constexpr int TOTAL = OFF_XW + 2 * Q1;
  static constexpr size_t BYTES = size_t(TOTAL) * 8;
};

// stage-z outer products c_zz[p][az][bz][qz][a][b] = B^az[qz][a] B^bz[qz][b] (p <= 3), so the
// pipelined kernel's stage z is one constant-operand FMA per term
__constant__ double c_zz[4][2][2][4][4][4];

cudaError_t upload_const_tables_matrix(int order, const double* b1, const double* d1,
                                      const double* x1, const double* w1, cudaStream_t st) {
  cudaError_t e = upload_tables_this_tu(order, b1, d1, x1, w1, st);
  if (e != cudaSuccess || order < 1 || order > 3) return e;
  double h[2][2][4][4][4] = {};  // per call (stack): concurrent mesh creation is safe
  const int n1 = order + 1, q1 = order + 1;
  for (int az = 0; az < 2; ++az)
    for (int bz = 0; bz < 2; ++bz)
      for (int q = 0; q < q1; ++q)
        for (int a = 0; a < n1; ++a)
          for (int b = 0; b < n1; ++b)
            h[az][bz][q][a][b] = (az ? d1 : b1)[q * n1 + a] * (bz ? d1 : b1)[q * n1 + b];
  e = cudaMemcpyToSymbolAsync(c_zz, h, sizeof(h), sizeof(h) * order, cudaMemcpyHostToDevice, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  return e;
}

// unique pair u -> (m, n), m <= n; index 6 is the value-value pair (3,3)
__device__ __forceinline__ void upair(int u, int& m, int& n) {
  // m = {0,0,0,1,1,2,3}[u], n = {0,1,2,1,2,2,3}[u] as packed nibbles (no local memory)
  m = (0x3211000 >> (4 * u)) & 0xF;
  n = (0x3221210 >> (4 * u)) & 0xF;
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// edge e (0..11) of a hex: direction d = e / 4, the other two bits k = e % 4;
// returns the two vertex ids (v = a + 2b + 4c) of the edge.
__device__ __forceinline__ void hex_edge(int e, int& v0, int& v1) {
  const int d = e >> 2, k = e & 3;
  const int lo = k & 1, hi = k >> 1;
  int a0, b0, c0;
  if (d == 0) { a0 = 0; b0 = lo; c0 = hi; }
  else if (d == 1) { a0 = lo; b0 = 0; c0 = hi; }
  else { a0 = lo; b0 = hi; c0 = 0; }
  v0 = a0 + 2 * b0 + 4 * c0;
  v1 = v0 + (1 << d);
}

template <int P, int FORM>
__global__ void __launch_bounds__(SFM<P, FORM != FE_FORM_MASS, FORM != FE_FORM_DIFFUSION>::THREADS, FEB200_SF_MINB)
    k_matrix_sf(MeshView mv, const double* __restrict__ ma, const double* __restrict__ mb,
                int64_t e0, int64_t e1, double* __restrict__ K) {
  constexpr bool DIFF = FORM != FE_FORM_MASS, MASS = FORM != FE_FORM_DIFFUSION;
  using L = SFM<P, DIFF, MASS>;
  constexpr int N1 = L::N1, Q1 = L::Q1, NB = L::NB, NQ = L::NQ, NUP = L::NUP, E = L::E;
  constexpr int QQP = L::QQP;
  constexpr int UBASE = DIFF ? 0 : 6;  // first unique-pair id
  extern __shared__ __align__(128) double sm[];
  double* edge = sm + L::OFF_EDGE;
  double* coef = sm + L::OFF_COEF;
  double* W = sm + L::OFF_W;
  double* T1 = sm + L::OFF_T1;
  const int tid = threadIdx.x;

  // 1D tables B^a[q][i] (a = 0 values, 1 derivatives) from constant memory
#define Bt(a, q, i) c_tab1d[P][a][q][i]

  // ---- thread-constant stage-z task (one per thread)
  const int z_el = tid / (NUP * Q1 * Q1), z_r = tid - z_el * (NUP * Q1 * Q1);
  const int z_ul = z_r / (Q1 * Q1), z_qxy = z_r - z_ul * (Q1 * Q1);
  const int z_qx = z_qxy / Q1, z_qy = z_qxy - z_qx * Q1;
  double Bza[Q1][N1], Bzb[Q1][N1];
  {
    int m, n;
    upair(UBASE + (z_ul < NUP ? z_ul : 0), m, n);
#pragma unroll
    for (int q = 0; q < Q1; ++q)
#pragma unroll
      for (int i = 0; i < N1; ++i) {
        Bza[q][i] = m == 2 ? Bt(1, q, i) : Bt(0, q, i);
        Bzb[q][i] = n == 2 ? Bt(1, q, i) : Bt(0, q, i);
      }
  }

  // ---- thread-constant stage-y/x task
  const int yx_el = tid / L::TPE, yx_r = tid - yx_el * L::TPE;
  int iz, jz, iy, jy;
  if (yx_r < L::TOFF) {  // off-diagonal z pair, any y pair
    int c = yx_r / L::YP;
    const int yp = yx_r - c * L::YP;
    iy = yp / N1;
    jy = yp - iy * N1;
    iz = 0;
    jz = 1;
    for (int a = 0; a < N1; ++a) {
      if (c < N1 - 1 - a) { iz = a; jz = a + 1 + c; break; }
      c -= N1 - 1 - a;
    }
  } else {               // diagonal z pair, y pairs iy <= jy
    const int r = yx_r - L::TOFF;
    iz = jz = r / L::YPS;
    int c = r - iz * L::YPS;
    iy = 0;
    jy = 0;
    for (int a = 0; a < N1; ++a) {
      if (c < N1 - a) { iy = a; jy = a + c; break; }
      c -= N1 - a;
    }
  }
  const bool mirror = (iz < jz) || (iy < jy);
  double Byp[4][Q1];  // Byp[ay*2+by][qy] = B^ay[qy][iy] B^by[qy][jy]
#pragma unroll
  for (int q = 0; q < Q1; ++q)
#pragma unroll
    for (int a = 0; a < 2; ++a)
#pragma unroll
      for (int b = 0; b < 2; ++b) Byp[a * 2 + b][q] = Bt(a, q, iy) * Bt(b, q, jy);

  // ---- software pipeline of the global reads: conn two batches ahead,
  // edge vectors and coefficients one batch ahead, held in registers.
  const int64_t nloc = e1 - e0;
  const int64_t nbatch = (nloc + E - 1) / E;
  static_assert(E * 36 <= L::THREADS && E * NQ <= L::THREADS, "one prefetch slot per thread");
  const int pe_el = tid / 36, pe_r = tid - pe_el * 36;       // edge slot: edge pe_r/3, comp pe_r%3
  int pe_v0, pe_v1;
  hex_edge(pe_r / 3, pe_v0, pe_v1);
  const int pe_c = pe_r % 3;
  const int pk_el = tid / NQ, pk_q = tid - pk_el * NQ;       // coefficient slot
  const bool pe_on = tid < E * 36, pk_on = tid < E * NQ;
  auto ld_conn2 = [&](int64_t b, int& c0, int& c1) {
    const int64_t le = b * E + pe_el;
    if (pe_on && b < nbatch && le < nloc) {
      const int32_t* cn = mv.conn + 8 * (e0 + le);
      c0 = cn[pe_v0];
      c1 = cn[pe_v1];
    } else {
      c0 = c1 = -1;
    }
  };
  // the two end-point coordinates stay in registers until the next batch: subtracting
  // them right away would wait for the loads here instead of overlapping them
  auto ld_edge = [&](int c0, int c1, double& xa, double& xb) {
    xa = c0 >= 0 ? mv.coords[3 * (int64_t)c0 + pe_c] : 0.0;
    xb = c0 >= 0 ? mv.coords[3 * (int64_t)c1 + pe_c] : 0.0;
  };
  auto ld_k = [&](int64_t b, double& kap, double& rho) {
    kap = rho = 0.0;
    const int64_t le = b * E + pk_el;
    if (pk_on && b < nbatch && le < nloc) {
      const int64_t g = (e0 + le) * NQ + pk_q;
      if constexpr (FORM == FE_FORM_DIFFUSION) kap = ma[g];
      if constexpr (FORM == FE_FORM_MASS) rho = ma[g];
      if constexpr (FORM == FE_FORM_MASS_DIFFUSION) { rho = ma[g]; kap = mb[g]; }
    }
  };
  int cn0, cn1;
  ld_conn2(blockIdx.x, cn0, cn1);
  double xa_cur, xb_cur, k_cur, r_cur;
  ld_edge(cn0, cn1, xa_cur, xb_cur);
  ld_k(blockIdx.x, k_cur, r_cur);
  ld_conn2(blockIdx.x + gridDim.x, cn0, cn1);

  int it = 0;
  for (int64_t bidx = blockIdx.x; bidx < nbatch; bidx += gridDim.x, ++it) {
    const int64_t lb = bidx * E;                 // local index of the first cell
    const int ne = (int)((nloc - lb) < E ? (nloc - lb) : E);
    double* Kst = sm + L::OFF_K + (L::NKB == 2 ? (it & 1) * L::KST : 0);
    // A. this batch's data from the prefetch registers; issue the next reads
    if (pe_on) edge[tid] = xb_cur - xa_cur;
    if (pk_on) {
      coef[(pk_el * 2) * NQ + pk_q] = k_cur;
      coef[(pk_el * 2 + 1) * NQ + pk_q] = r_cur;
    }
    ld_edge(cn0, cn1, xa_cur, xb_cur);
    ld_k(bidx + gridDim.x, k_cur, r_cur);
    ld_conn2(bidx + 2 * (int64_t)gridDim.x, cn0, cn1);
    // the TMA store issued two batches ago (one with a single buffer) read this staging
    // buffer: wait for it
    if (tid == 0) {
      if constexpr (L::NKB == 2) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
      else asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
    }
    __syncthreads();
    // B. geometry from the 12 edge vectors -> W^{mn}[q]
    if (tid < E * NQ) {
      const int el = tid / NQ, q = tid - el * NQ;
      const double t0 = mv.xi[3 * q], t1 = mv.xi[3 * q + 1], t2 = mv.xi[3 * q + 2];
      const double* ed = edge + el * 36;
      // J[:,d] = sum_k w_k e_d[k], bilinear weights of the two other coordinates
      double J[3][3];
      const double wA[4] = {(1 - t1) * (1 - t2), t1 * (1 - t2), (1 - t1) * t2, t1 * t2};
      const double wB[4] = {(1 - t0) * (1 - t2), t0 * (1 - t2), (1 - t0) * t2, t0 * t2};
      const double wC[4] = {(1 - t0) * (1 - t1), t0 * (1 - t1), (1 - t0) * t1, t0 * t1};
#pragma unroll
      for (int i = 0; i < 3; ++i) {
        J[i][0] = wA[0] * ed[0 * 3 + i] + wA[1] * ed[1 * 3 + i] + wA[2] * ed[2 * 3 + i] + wA[3] * ed[3 * 3 + i];
        J[i][1] = wB[0] * ed[4 * 3 + i] + wB[1] * ed[5 * 3 + i] + wB[2] * ed[6 * 3 + i] + wB[3] * ed[7 * 3 + i];
        J[i][2] = wC[0] * ed[8 * 3 + i] + wC[1] * ed[9 * 3 + i] + wC[2] * ed[10 * 3 + i] + wC[3] * ed[11 * 3 + i];
      }
      // cofactors; J^-1[m][k] = cof[k][m] / det
      const double c00 = J[1][1] * J[2][2] - J[1][2] * J[2][1];
      const double c01 = J[1][2] * J[2][0] - J[1][0] * J[2][2];
      const double c02 = J[1][0] * J[2][1] - J[1][1] * J[2][0];
      const double c10 = J[0][2] * J[2][1] - J[0][1] * J[2][2];
      const double c11 = J[0][0] * J[2][2] - J[0][2] * J[2][0];
      const double c12 = J[0][1] * J[2][0] - J[0][0] * J[2][1];
      const double c20 = J[0][1] * J[1][2] - J[0][2] * J[1][1];
      const double c21 = J[0][2] * J[1][0] - J[0][0] * J[1][2];
      const double c22 = J[0][0] * J[1][1] - J[0][1] * J[1][0];
      const double det = J[0][0] * c00 + J[0][1] * c01 + J[0][2] * c02;
      const double wq = mv.w[q];
      double* Wel = W + el * NUP * NQ;
      if constexpr (DIFF) {
        // W^{mn} = detw kappa sum_k Jinv[m][k] Jinv[n][k] = w kappa / det * sum_k cof[k][m] cof[k][n]
        const double s = wq * coef[(el * 2) * NQ + q] * rcp_nr(det);
        const double C[3][3] = {{c00, c01, c02}, {c10, c11, c12}, {c20, c21, c22}};
#pragma unroll
        for (int u = 0; u < 6; ++u) {
          int m, n;
          upair(u, m, n);
          Wel[u * NQ + q] = s * (C[0][m] * C[0][n] + C[1][m] * C[1][n] + C[2][m] * C[2][n]);
        }
      }
      if constexpr (MASS) Wel[(NUP - 1) * NQ + q] = wq * det * coef[(el * 2 + 1) * NQ + q];
    }
    __syncthreads();
    // C. stage z: T1^{u}[iz,jz][qx,qy] = sum_qz B^{mz}[qz][iz] B^{nz}[qz][jz] W^u[qx,qy,qz]
    if (tid < L::T_Z) {
      const double* w = W + (z_el * NUP + z_ul) * NQ + z_qx + Q1 * z_qy;
      double t[Q1][N1];
#pragma unroll
      for (int qz = 0; qz < Q1; ++qz) {
        const double c = w[Q1 * Q1 * qz];
#pragma unroll
        for (int a = 0; a < N1; ++a) t[qz][a] = c * Bza[qz][a];
      }
      double* out = T1 + (z_el * NUP + z_ul) * N1 * N1 * QQP + z_qxy;
#pragma unroll
      for (int a = 0; a < N1; ++a)
#pragma unroll
        for (int b = 0; b < N1; ++b) {
          double s = 0.0;
#pragma unroll
          for (int qz = 0; qz < Q1; ++qz) s = fma(t[qz][a], Bzb[qz][b], s);
          out[(a * N1 + b) * QQP] = s;
        }
    }
    __syncthreads();
    // D. stage y + stage x, one (z-pair, y-pair) per thread
    if (tid < L::T_YX && yx_el < ne) {
      double S[4][Q1];
#pragma unroll
      for (int c = 0; c < 4; ++c)
#pragma unroll
        for (int q = 0; q < Q1; ++q) S[c][q] = 0.0;
      const double* T1e = T1 + yx_el * NUP * N1 * N1 * QQP;
#pragma unroll
      for (int op = 0; op < L::NOP; ++op) {
        int m, n;
        if (DIFF && op < 9) { m = op / 3; n = op % 3; } else { m = 3; n = 3; }
        const int mm = m < n ? m : n, nn = m < n ? n : m;
        const int ul = (mm == 3) ? NUP - 1 : (mm == 0 ? nn : (mm == 1 ? 2 + nn : 5));
        const int zidx = (m > n) ? (jz * N1 + iz) : (iz * N1 + jz);
        const int ay = m == 1, by = n == 1, cls = (m == 0) * 2 + (n == 0);
        const double2* src = reinterpret_cast<const double2*>(T1e + (ul * N1 * N1 + zidx) * QQP);
        double tv[QQP];
#pragma unroll
        for (int h = 0; h < QQP / 2; ++h) {
          const double2 v = src[h];
          tv[2 * h] = v.x;
          tv[2 * h + 1] = v.y;
        }
#pragma unroll
        for (int qx = 0; qx < Q1; ++qx)
#pragma unroll
          for (int qy = 0; qy < Q1; ++qy)
            S[cls][qx] = fma(Byp[ay * 2 + by][qy], tv[qx * Q1 + qy], S[cls][qx]);
      }
      double acc[N1][N1];
#pragma unroll
      for (int a = 0; a < N1; ++a)
#pragma unroll
        for (int b = 0; b < N1; ++b) acc[a][b] = 0.0;
#pragma unroll
      for (int qx = 0; qx < Q1; ++qx)
#pragma unroll
        for (int ax = 0; ax < 2; ++ax) {
          double u[N1];
#pragma unroll
          for (int b = 0; b < N1; ++b) u[b] = Bt(0, qx, b) * S[ax * 2 + 0][qx] + Bt(1, qx, b) * S[ax * 2 + 1][qx];
#pragma unroll
          for (int a = 0; a < N1; ++a)
#pragma unroll
            for (int b = 0; b < N1; ++b) acc[a][b] = fma(Bt(ax, qx, a), u[b], acc[a][b]);
        }
      double* Ke = Kst + yx_el * NB * NB;
      const int ib = N1 * (iy + N1 * iz), jb = N1 * (jy + N1 * jz);
#pragma unroll
      for (int a = 0; a < N1; ++a)
#pragma unroll
        for (int b = 0; b < N1; ++b) {
          Ke[(ib + a) * NB + jb + b] = acc[a][b];
          if (mirror) Ke[(jb + b) * NB + ib + a] = acc[a][b];
        }
    }
    // E. write the batch: one TMA bulk store of ne * NB^2 doubles (contiguous in K)
    const uint32_t bytes = (uint32_t)ne * NB * NB * 8;
    double* gdst = K + lb * NB * NB;
    if (((reinterpret_cast<uintptr_t>(gdst) | bytes) & 15u) == 0) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncthreads();
      if (tid == 0) {
        if (FEB200_SFP_EVF) {
          uint64_t pol_;
          asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol_));
          asm volatile("cp.async.bulk.global.shared::cta.bulk_group.L2::cache_hint [%0], [%1], %2, %3;"
                     :: "l"(gdst), "r"(smem_u32(Kst)), "r"(bytes), "l"(pol_) : "memory");
        } else asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;"
                     :: "l"(gdst), "r"(smem_u32(Kst)), "r"(bytes) : "memory");
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      }
    } else {
      __syncthreads();
      for (int i = tid; i < ne * NB * NB; i += blockDim.x) gdst[i] = Kst[i];
    }
  }
  if (tid == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
#undef Bt
}

// ---------------------------------------------------------------------------
// Warp-specialised pipelined variant (P = 1, 2): the same three contraction
// stages, but run by three groups of warps on different cell batches at once,
// handing data over through shared-memory rings guarded by mbarriers instead
// of CTA-wide barriers (one persistent CTA per SM):
//   L (1 warp)   : gathers the batch's vertex coordinates and coefficients
//                  into ring slot L[it % 2]                     (loads)
//   G (NG warps) : one thread per (cell, qx, qy) column: geometry at its Q1
//                  qps (a1) -> W^{mn} in registers -> stage z
//                  for all unique pairs -> T1 ring slot [it % 2]
//   X (NX warps) : one thread per (cell, z-pair, y-pair): stages y and x
//                  (b, c1) -> K staging slot [it % 2] -> one TMA bulk store
// The geometry + stage-z thread uses compile-time pair indices, so every 1D
// table operand is a constant-bank operand.
template <int P, int NUPMAX, bool RES = false, int KB = 8>
struct SFP {
  static constexpr int N1 = P + 1, Q1 = P + 1, NB = N1 * N1 * N1, NQ = Q1 * Q1 * Q1, Q2 = Q1 * Q1;
  static constexpr int YP = N1 * N1, YPS = N1 * (N1 + 1) / 2;
  // YB: y pairs per X thread.  YB = 1: one task per (z pair, y pair), every T1 value a thread
  // loads feeds one FMA.  YB = 3 (p = 2): one task per (z pair iz < jz, iy) over jy = 0..2,
  // and two per diagonal z pair (y pairs (0,0),(0,1),(0,2) and (1,1),(1,2),(2,2)) -- each
  // loaded T1 value feeds three FMAs, a third of the shared-memory load wavefronts per cell
  static constexpr int YB = P == 2 ? FEB200_SFP_YB : 1;
  static constexpr int TOFF = YB == 1 ? YP * (N1 * (N1 - 1) / 2) : N1 * (N1 * (N1 - 1) / 2);
  static constexpr int TPE = YB == 1 ? TOFF + N1 * YPS : TOFF + 2 * N1;  // X tasks per cell
  static constexpr int E = P == 1 ? 16 : FEB200_SFP_E2;   // cells per batch (even: TMA size)
  static constexpr int GH = FEB200_SFP_GH;                // G thread groups per column
  static constexpr int NGW = (E * Q2 + 31) / 32;          // G warps per group
  static constexpr int NG = GH * NGW;                     // G warps
  static constexpr int NX = (E * TPE + 31) / 32;           // X warps
  static constexpr int THREADS = 32 * (1 + NG + NX);
  static constexpr int QQP = (Q2 + 1) / 2 * 2;
  // shared memory (bytes)
  static constexpr size_t LSLOT = size_t(E) * (24 + (NUPMAX == 7 ? 2 : 1) * NQ) * 8;  // coords, coef a[, b]
  // per-cell T1 stride padded by T1PAD doubles (an odd pad makes the G threads' column stores
  // of consecutive cells hit disjoint banks; X then reads the vectors with 8-B loads)
  static constexpr int T1PAD = FEB200_SFP_T1PAD;
  static constexpr int T1CELL = NUPMAX * N1 * N1 * QQP + T1PAD;
  static constexpr size_t T1SLOT = size_t(E) * T1CELL * 8;
  static constexpr size_t KSLOT = size_t(E) * NB * NB * KB;  // K staging in the output type
  static constexpr size_t OFF_K = 0;                                  // [2][KSLOT]
  static constexpr size_t OFF_T1 = OFF_K + 2 * KSLOT;                 // [2][T1SLOT]
  static constexpr size_t OFF_L = OFF_T1 + 2 * T1SLOT;                // [2][LSLOT]
  static constexpr size_t OFF_CONN = OFF_L + 2 * LSLOT;               // [3][E * 8] int32
  // fused residual (RES): u_e [SU][E][NB] and dof ids [SU][E][NB] in a ring the L warp fills
  // SU - 1 batches ahead; row-group partial sums [E][NB][N1^2] (written and scattered by X
  // within one batch)
  static constexpr int SU = 4;
  static constexpr size_t OFF_U = (OFF_CONN + 3 * E * 8 * 4 + 15) / 16 * 16;
  static constexpr size_t OFF_R = OFF_U + (RES ? SU * size_t(E) * NB * 8 : 0);
  static constexpr size_t OFF_DC = OFF_R + (RES ? size_t(E) * NB * N1 * N1 * 8 : 0);
  static constexpr size_t OFF_BAR = (OFF_DC + (RES ? SU * size_t(E) * NB * 4 : 0) + 15) / 16 * 16;
  static constexpr size_t BYTES = OFF_BAR + 24 * 8;  // 11 + 2 SU mbarriers
};

__device__ __forceinline__ void sfp_bar_init(uint64_t* bar, int count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void sfp_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void sfp_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tWAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)), "r"(parity) : "memory");
}
__device__ __forceinline__ void sfp_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.expect_tx.relaxed.cta.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void sfp_expect_arrive(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
// TMA bulk copy global -> shared (16-B aligned, size % 16 == 0), completion on an mbarrier
__device__ __forceinline__ void sfp_tma_load(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)) : "memory");
}
#ifdef FEB200_SFP_PROF
// per-role wait-cycle counters (A/B builds only): sum over warps of clock64 deltas
__device__ unsigned long long g_sfp_prof[16];
#define SFP_T(k, stmt)                                  \
  do {                                                  \
    const long long t0_ = clock64();                    \
    stmt;                                               \
    prof_[k] += (unsigned long long)(clock64() - t0_);  \
  } while (0)
#else
#define SFP_T(k, stmt) stmt
#endif
__device__ __forceinline__ void sfp_named_bar(int id, int nthreads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

// KT: element type of the material arrays and of K (double, or float for the FE_F32 matrix
// path: the contraction runs in fp64 on the fp32 inputs and K is rounded to fp32 when staged)
template <int P, int FORM, bool RES, typename KT = double>
__global__ void __launch_bounds__(SFP<P, (FORM != FE_FORM_MASS ? 6 : 0) + (FORM != FE_FORM_DIFFUSION ? 1 : 0), RES, (int)sizeof(KT)>::THREADS, 1)
    k_matrix_sfp(MeshView mv, const KT* __restrict__ ma, const KT* __restrict__ mb,
                 int64_t e0, int64_t e1, KT* __restrict__ K, const double* __restrict__ u,
                 double* __restrict__ r_elem, double* __restrict__ r_global) {
  static_assert(!RES || sizeof(KT) == 8, "the fused matrix + residual kernel is fp64");
  constexpr bool DIFF = FORM != FE_FORM_MASS, MASS = FORM != FE_FORM_DIFFUSION;
  constexpr int NUP = (DIFF ? 6 : 0) + (MASS ? 1 : 0);
  using L = SFP<P, NUP, RES, (int)sizeof(KT)>;
  constexpr int N1 = L::N1, Q1 = L::Q1, NB = L::NB, NQ = L::NQ, Q2 = L::Q2, E = L::E;
  constexpr int QQP = L::QQP;
  constexpr int NOP = (DIFF ? 9 : 0) + (MASS ? 1 : 0);
  constexpr int UBASE = DIFF ? 0 : 6;
  constexpr int NCOEF = MASS && DIFF ? 2 : 1;
  extern __shared__ __align__(128) unsigned char smp[];
  uint64_t* bars = reinterpret_cast<uint64_t*>(smp + L::OFF_BAR);
  uint64_t* fullL = bars + 0;   // [2] L -> G
  uint64_t* emptyL = bars + 2;  // [2] G -> L
  uint64_t* fullT = bars + 4;   // [2] G -> X
  uint64_t* emptyT = bars + 6;  // [2] X -> G
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int64_t nloc = e1 - e0;
  const int64_t nbatch = (nloc + E - 1) / E;
#ifdef FEB200_SFP_PROF
  unsigned long long prof_[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  const long long tstart_ = clock64();
#endif
  if (tid == 0) {
    sfp_bar_init(&fullL[0], 32);
    sfp_bar_init(&fullL[1], 32);
    sfp_bar_init(&emptyL[0], 32 * L::NG);
    sfp_bar_init(&emptyL[1], 32 * L::NG);
    sfp_bar_init(&fullT[0], 32 * L::NG);
    sfp_bar_init(&fullT[1], 32 * L::NG);
    sfp_bar_init(&emptyT[0], 32 * L::NX);
    sfp_bar_init(&emptyT[1], 32 * L::NX);
    sfp_bar_init(&bars[8], 1);
    sfp_bar_init(&bars[9], 1);
    sfp_bar_init(&bars[10], 1);
    if (RES) {
      for (int k = 0; k < L::SU; ++k) {
        sfp_bar_init(&bars[11 + k], 32);                 // fullU[SU]: L -> X (u_e, dof ids)
        sfp_bar_init(&bars[11 + L::SU + k], 32 * L::NX);  // doneR[SU]: X -> L (slot free)
      }
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  uint64_t* fullU = bars + 11;
  uint64_t* doneR = bars + 11 + L::SU;
  double* Ub = reinterpret_cast<double*>(smp + L::OFF_U);    // [2][E][NB] gathered u_e
  double* Rb = reinterpret_cast<double*>(smp + L::OFF_R);    // [2][E][NB] r_e accumulators
  int32_t* DCb = reinterpret_cast<int32_t*>(smp + L::OFF_DC); // [2][E][NB] dof ids
  (void)fullU; (void)doneR; (void)Ub; (void)Rb; (void)DCb;
#define Bt(a, q, i) c_tab1d[P][a][q][i]

  if (warp == 0) {
    // ======================= L: loader warp =======================
    // conn blocks arrive by TMA two batches ahead (3-deep ring, own mbarriers); the vertex
    // coordinates of batch it + 1 are gathered into registers while batch it is handed
    // over; coefficient blocks go by TMA straight into the slot (tx-counted on fullL).
    int32_t* connb = reinterpret_cast<int32_t*>(smp + L::OFF_CONN);
    uint64_t* connbar = bars + 8;  // [3]
    auto batch_of = [&](int64_t j, int64_t& lb, int& ne) {
      const int64_t b = blockIdx.x + j * (int64_t)gridDim.x;
      lb = b * E;
      ne = b < nbatch ? (int)((nloc - lb) < E ? (nloc - lb) : E) : 0;
    };
    auto conn_issue = [&](int64_t j) {  // lane 0
      int64_t lb;
      int ne;
      batch_of(j, lb, ne);
      if (ne <= 0) return;
      const int k = (int)(j % 3);
      sfp_expect_arrive(&connbar[k], (uint32_t)ne * 32u);
      sfp_tma_load(connb + k * E * 8, mv.conn + 8 * (e0 + lb), (uint32_t)ne * 32u, &connbar[k]);
    };
    constexpr int XPL = (E * 24 + 31) / 32, KPL = (E * NQ + 31) / 32;
    double xr[XPL];
    auto coords_issue = [&](int64_t j) {
      int64_t lb;
      int ne;
      batch_of(j, lb, ne);
      if (ne <= 0) return;
      const int k = (int)(j % 3);
      SFP_T(0, sfp_wait(&connbar[k], (uint32_t)((j / 3) & 1)));
      const int32_t* cb = connb + k * E * 8;
#pragma unroll
      for (int h = 0; h < XPL; ++h) {
        const int i = lane + 32 * h, c = i / 24, r = i - c * 24;
        xr[h] = (i < E * 24 && c < ne) ? mv.coords[3 * (int64_t)cb[c * 8 + r / 3] + r % 3] : 0.0;
      }
    };
    if (lane == 0) {
      conn_issue(0);
      conn_issue(1);
    }
    coords_issue(0);
    constexpr int UPL = RES ? (E * NB + 31) / 32 : 1;
    int32_t dnext[UPL];
    auto load_dof = [&](int64_t j) {  // dof ids of the j-th batch (fused residual)
      int64_t lbj;
      int nej;
      batch_of(j, lbj, nej);
#pragma unroll
      for (int h = 0; h < UPL; ++h) {
        const int i = lane + 32 * h;
        dnext[h] = (RES && i < nej * NB) ? mv.dof_conn[(e0 + lbj) * NB + i] : 0;
      }
    };
    // fused residual: u_e of batch j into slot j % 2 (dof ids loaded one call ahead)
    // fused residual, software-pipelined gathers: uvn / dcn hold u_e and the dof ids of the
    // next batch to publish (their loads were issued one call earlier), dnext the dof ids
    // of the batch after it
    double uvn[UPL];
    int32_t dcn[UPL];
    auto issue_u = [&](int64_t j) {  // dcn = dof(j) (from dnext), uvn = u[dcn], dnext = dof(j+1)
      int64_t lbj;
      int nej;
      batch_of(j, lbj, nej);
#pragma unroll
      for (int h = 0; h < UPL; ++h) {
        const int i = lane + 32 * h;
        dcn[h] = dnext[h];
        uvn[h] = i < nej * NB ? u[dcn[h]] : 0.0;
      }
      load_dof(j + 1);
    };
    auto publish_u = [&](int64_t j) {  // u_e / dof ids of batch j (in uvn / dcn) -> slot j % SU
      int64_t lbj;
      int nej;
      batch_of(j, lbj, nej);
      if (nej <= 0) return;
      const int sj = (int)(j % L::SU);
      if (j >= L::SU)  // X released this slot (batch j - SU)
        SFP_T(0, sfp_wait(&doneR[sj], (uint32_t)(((j - L::SU) / L::SU) & 1)));
#pragma unroll
      for (int h = 0; h < UPL; ++h) {
        const int i = lane + 32 * h;
        if (i < E * NB) {
          DCb[sj * E * NB + i] = dcn[h];
          Ub[sj * E * NB + i] = uvn[h];
        }
      }
      sfp_arrive(&fullU[sj]);
    };
    if constexpr (RES) {
      load_dof(0);
      issue_u(0);
      publish_u(0);
      issue_u(1);
    }
    for (int64_t it = 0;; ++it) {
      int64_t lb;
      int ne;
      batch_of(it, lb, ne);
      if (ne <= 0) break;
      const int sl = (int)(it & 1);
      __syncwarp();
      if (lane == 0) conn_issue(it + 2);  // ring slot (it+2)%3 was last read in iteration it-2
      SFP_T(1, sfp_wait(&emptyL[sl], (uint32_t)(((it >> 1) & 1) ^ 1)));
      double* slot = reinterpret_cast<double*>(smp + L::OFF_L + sl * L::LSLOT);
      const KT* ga = ma + (e0 + lb) * NQ;
      const KT* gb = NCOEF == 2 ? mb + (e0 + lb) * NQ : nullptr;
      const uint32_t kbytes = (uint32_t)ne * NQ * (uint32_t)sizeof(KT);
      const bool tma_ok = (((reinterpret_cast<uintptr_t>(ga) | (NCOEF == 2 ? reinterpret_cast<uintptr_t>(gb) : 0) |
                             kbytes) & 15u) == 0);
      if (tma_ok) {
        if (lane == 0) {
          sfp_expect_tx(&fullL[sl], kbytes * NCOEF);
          sfp_tma_load(slot + E * 24, ga, kbytes, &fullL[sl]);
          if (NCOEF == 2) sfp_tma_load(slot + E * 24 + E * NQ, gb, kbytes, &fullL[sl]);
        }
      } else {
#pragma unroll
        for (int h = 0; h < KPL; ++h) {
          const int i = lane + 32 * h;
          if (i < ne * NQ) {  // the coefficient blocks keep the input type (as the TMA copy)
            reinterpret_cast<KT*>(slot + E * 24)[i] = ga[i];
            if (NCOEF == 2) reinterpret_cast<KT*>(slot + E * 24 + E * NQ)[i] = gb[i];
          }
        }
      }
#pragma unroll
      for (int h = 0; h < XPL; ++h) {
        const int i = lane + 32 * h;
        if (i < E * 24) slot[i] = xr[h];
      }
      sfp_arrive(&fullL[sl]);
      coords_issue(it + 1);
      if constexpr (RES) {
        // fused residual: scatter batch it-1 once X is done with it, then refill its u slot
        // with batch it+1 (u_e of batch 0 was filled before the loop)
        publish_u(it + 1);
        issue_u(it + 2);
      }
    }
  } else if (warp <= L::NG) {
    // ======================= G: geometry + stage z =======================
    // GH warp-uniform groups per column; group h forms the unique pairs [ulo, uhi)
    const int gtid0 = tid - 32;
    const int h = gtid0 / (32 * L::NGW), gtid = gtid0 - h * 32 * L::NGW;
    constexpr int UPH = (NUP + L::GH - 1) / L::GH;
    const int ulo = h * UPH, uhi = (h + 1) * UPH < NUP ? (h + 1) * UPH : NUP;
    const int el = gtid / Q2, qxy = gtid - el * Q2;
    const int tx = qxy / Q1, ty = qxy - tx * Q1;  // T1's inner index is qx * Q1 + qy
    const bool gact = gtid < E * Q2 && ulo < uhi;
    const double tX = c_x1d[P][tx], tY = c_x1d[P][ty];
    const double wxy = c_w1d[P][tx] * c_w1d[P][ty];
    for (int64_t it = 0;; ++it) {
      const int64_t b = blockIdx.x + it * (int64_t)gridDim.x;
      if (b >= nbatch) break;
      const int64_t lb = b * E;
      const int ne = (int)((nloc - lb) < E ? (nloc - lb) : E);
      const int sl = (int)(it & 1);
      const uint32_t par = (uint32_t)((it >> 1) & 1);
      SFP_T(2, sfp_wait(&fullL[sl], par));
      const double* slot = reinterpret_cast<const double*>(smp + L::OFF_L + sl * L::LSLOT);
      const bool on = gact && el < ne;
      // edge-vector combinations of this column: J[:,0] = (1-tZ) e0y[0] + tZ e0y[1],
      // J[:,1] = (1-tZ) e1x[0] + tZ e1x[1], J[:,2] = col2 (trilinear map, vertex v = a + 2b + 4c)
      double e0y[2][3], e1x[2][3], col2[3], ca[Q1], cb[Q1];
      {
        const double* X = slot + (on ? el : 0) * 24;
#pragma unroll
        for (int i = 0; i < 3; ++i) {
#pragma unroll
          for (int c = 0; c < 2; ++c) {
            // x-edges at (b, c): X[1+2b+4c] - X[2b+4c];  y-edges at (a, c): X[a+2+4c] - X[a+4c]
            e0y[c][i] = (1 - tY) * (X[3 * (1 + 4 * c) + i] - X[3 * (4 * c) + i]) +
                        tY * (X[3 * (3 + 4 * c) + i] - X[3 * (2 + 4 * c) + i]);
            e1x[c][i] = (1 - tX) * (X[3 * (2 + 4 * c) + i] - X[3 * (4 * c) + i]) +
                        tX * (X[3 * (3 + 4 * c) + i] - X[3 * (1 + 4 * c) + i]);
          }
          // z-edges at (a, b): X[a+2b+4] - X[a+2b]
          col2[i] = (1 - tX) * (1 - tY) * (X[3 * 4 + i] - X[3 * 0 + i]) +
                    tX * (1 - tY) * (X[3 * 5 + i] - X[3 * 1 + i]) +
                    (1 - tX) * tY * (X[3 * 6 + i] - X[3 * 2 + i]) + tX * tY * (X[3 * 7 + i] - X[3 * 3 + i]);
        }
#pragma unroll
        for (int qz = 0; qz < Q1; ++qz) {
          const int q = tx + Q1 * ty + Q2 * qz;
          ca[qz] = on ? (double)reinterpret_cast<const KT*>(slot + E * 24)[el * NQ + q] : 0.0;
          cb[qz] = (on && NCOEF == 2) ? (double)reinterpret_cast<const KT*>(slot + E * 24 + E * NQ)[el * NQ + q] : 0.0;
        }
      }
      sfp_arrive(&emptyL[sl]);
      // W^{u}[qz] for the unique pairs u (m <= n), value-value pair last
      double Wr[NUP][Q1];
#pragma unroll
      for (int qz = 0; qz < Q1; ++qz) {
        const double tZ = c_x1d[P][qz];
        double J[3][3];
#pragma unroll
        for (int i = 0; i < 3; ++i) {
          J[i][0] = (1 - tZ) * e0y[0][i] + tZ * e0y[1][i];
          J[i][1] = (1 - tZ) * e1x[0][i] + tZ * e1x[1][i];
          J[i][2] = col2[i];
        }
        const double C[3][3] = {{J[1][1] * J[2][2] - J[1][2] * J[2][1], J[1][2] * J[2][0] - J[1][0] * J[2][2],
                                 J[1][0] * J[2][1] - J[1][1] * J[2][0]},
                                {J[0][2] * J[2][1] - J[0][1] * J[2][2], J[0][0] * J[2][2] - J[0][2] * J[2][0],
                                 J[0][1] * J[2][0] - J[0][0] * J[2][1]},
                                {J[0][1] * J[1][2] - J[0][2] * J[1][1], J[0][2] * J[1][0] - J[0][0] * J[1][2],
                                 J[0][0] * J[1][1] - J[0][1] * J[1][0]}};
        const double det = J[0][0] * C[0][0] + J[0][1] * C[0][1] + J[0][2] * C[0][2];
        const double wq = wxy * c_w1d[P][qz];
        if constexpr (DIFF) {
          const double kap = MASS ? cb[qz] : ca[qz];
          // 1/det: rcp.approx + two Newton steps (relative error ~1 ulp; det > 0 checked at create)
          double rd;
          asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(rd) : "d"(det));
          double er = fma(-det, rd, 1.0);
          rd = fma(rd, er, rd);
          er = fma(-det, rd, 1.0);
          rd = fma(rd, er, rd);
          const double sc = on ? wq * kap * rd : 0.0;
#pragma unroll
          for (int u = 0; u < 6; ++u) {
            if (L::GH > 1 && (u < ulo || u >= uhi)) continue;
            int m, n;
            upair(u, m, n);
            Wr[u][qz] = sc * (C[0][m] * C[0][n] + C[1][m] * C[1][n] + C[2][m] * C[2][n]);
          }
        }
        if constexpr (MASS) Wr[NUP - 1][qz] = wq * det * ca[qz];
      }
      // stage z into T1 slot it % 2 once X has released it
      SFP_T(3, sfp_wait(&emptyT[sl], par ^ 1u));
      double* T1 = reinterpret_cast<double*>(smp + L::OFF_T1 + sl * L::T1SLOT);
      if (gact && !FEB200_SFP_NOG) {
#pragma unroll
        for (int ul = 0; ul < NUP; ++ul) {
          if (L::GH > 1 && (ul < ulo || ul >= uhi)) continue;
          int m, n;
          upair(UBASE + ul, m, n);
          const int az = m == 2, bz = n == 2;
          double* out = T1 + el * L::T1CELL + ul * N1 * N1 * QQP + qxy;
#pragma unroll
          for (int a = 0; a < N1; ++a)
#pragma unroll
            for (int bb = 0; bb < N1; ++bb) {
              // pairs m == n: X reads T1 only at z pairs iz <= jz (the unique pair's vector
              // serves both orders), so the lower entries are not formed
              if (FEB200_SFP_ZTRI && m == n && a > bb) continue;
              double sacc = 0.0;
#pragma unroll
              for (int qz = 0; qz < Q1; ++qz) sacc = fma(Wr[ul][qz], c_zz[P][az][bz][qz][a][bb], sacc);
              out[(a * N1 + bb) * QQP] = sacc;
            }
        }
      }
      sfp_arrive(&fullT[sl]);
    }
  } else if constexpr (L::YB == 3) {
    // ============ X, register-blocked: one z pair, three y pairs per thread ============
    static_assert(P == 2, "YB = 3 is the p = 2 task map");
    const int xtid = tid - 32 * (1 + L::NG);
    constexpr int NXT = 32 * L::NX;
    // lane -> task: the generated bank-conflict-optimised permutation (sfp_tasks.h) for the
    // default batch of 8 cells, natural order otherwise
    int task = xtid;
#if FEB200_SFP_MAP
    if constexpr (E == 8) {
      static_assert(32 * L::NX == 128 && E * L::TPE == 120, "sfp_tasks.h is the E = 8 map");
      task = sfp_tasks_yb3[xtid];
    }
#endif
    const bool xact = task >= 0 && task < E * L::TPE;
    if (!xact) task = 0;
    int yx_el, iz, jz, yi[3], yj[3];
    if (task < E * L::TOFF) {  // z pair iz < jz (zp 0, 1, 2 = (0,1), (0,2), (1,2)), row iy
      yx_el = task / L::TOFF;
      const int r = task - yx_el * L::TOFF, zp = r / N1, iy = r - zp * N1;
      iz = zp >> 1;
      jz = zp == 0 ? 1 : 2;
#pragma unroll
      for (int k = 0; k < 3; ++k) { yi[k] = iy; yj[k] = k; }
    } else {  // diagonal z pair iz == jz, upper-triangle y pairs in two groups of three
      const int t = task - E * L::TOFF;
      yx_el = t / (L::TPE - L::TOFF);
      const int r = t - yx_el * (L::TPE - L::TOFF), hf = r & 1;
      iz = jz = (r >> 1) < N1 ? (r >> 1) : N1 - 1;
      yi[0] = hf; yj[0] = hf;        // (0,0) | (1,1)
      yi[1] = hf; yj[1] = hf + 1;    // (0,1) | (1,2)
      yi[2] = 2 * hf; yj[2] = 2;     // (0,2) | (2,2)
    }
    double Byp[3][4][Q1];
#pragma unroll
    for (int k = 0; k < 3; ++k)
#pragma unroll
      for (int q = 0; q < Q1; ++q)
#pragma unroll
        for (int a = 0; a < 2; ++a)
#pragma unroll
          for (int bb = 0; bb < 2; ++bb) Byp[k][a * 2 + bb][q] = Bt(a, q, yi[k]) * Bt(bb, q, yj[k]);
    for (int64_t it = 0;; ++it) {
      const int64_t b = blockIdx.x + it * (int64_t)gridDim.x;
      if (b >= nbatch) break;
      const int64_t lb = b * E;
      const int ne = (int)((nloc - lb) < E ? (nloc - lb) : E);
      const int sl = (int)(it & 1);
      SFP_T(5, sfp_named_bar(1, NXT));
      SFP_T(4, sfp_wait(&fullT[sl], (uint32_t)((it >> 1) & 1)));
      const double* T1e = reinterpret_cast<const double*>(smp + L::OFF_T1 + sl * L::T1SLOT) +
                          yx_el * L::T1CELL;
      double S[3][4][Q1];
#pragma unroll
      for (int k = 0; k < 3; ++k)
#pragma unroll
        for (int c = 0; c < 4; ++c)
#pragma unroll
          for (int q = 0; q < Q1; ++q) S[k][c][q] = 0.0;
      if (xact && !FEB200_SFP_NOX) {
        // ordered pairs (m, n): the unique pair first, its transpose (n, m) right after -- on a
        // diagonal z pair that is the same T1 vector, kept in registers (no second load)
        const bool zdiag = iz == jz;
        double tv[Q2];
#pragma unroll
        for (int op = 0; op < NOP; ++op) {
          int m, n;
          // DIFF order: (0,0) (0,1) (1,0) (0,2) (2,0) (1,1) (1,2) (2,1) (2,2) [(3,3)]
          if (DIFF && op < 9) {
            m = (0x221120100 >> (4 * op)) & 0xF;
            n = (0x212102010 >> (4 * op)) & 0xF;
          } else { m = 3; n = 3; }
          const int mm = m < n ? m : n, nn = m < n ? n : m;
          const int ul = (mm == 3) ? NUP - 1 : (mm == 0 ? nn : (mm == 1 ? 2 + nn : 5));
          const int zidx = (m > n) ? (jz * N1 + iz) : (iz * N1 + jz);
          const double* src = T1e + (ul * N1 * N1 + zidx) * QQP;
          if (m <= n || !zdiag) {
#pragma unroll
            for (int h = 0; h < Q2; ++h) tv[h] = src[h];
          }
          const int ay = m == 1, by = n == 1, cls = (m == 0) * 2 + (n == 0);
#pragma unroll
          for (int k = 0; k < 3; ++k)
#pragma unroll
            for (int qx = 0; qx < Q1; ++qx)
#pragma unroll
              for (int qy = 0; qy < Q1; ++qy)
                S[k][cls][qx] = fma(Byp[k][ay * 2 + by][qy], tv[qx * Q1 + qy], S[k][cls][qx]);
        }
      }
      sfp_arrive(&emptyT[sl]);
      KT* Kst = reinterpret_cast<KT*>(smp + L::OFF_K + sl * L::KSLOT);
      const int su = (int)(it % L::SU);
      if constexpr (RES) SFP_T(7, sfp_wait(&fullU[su], (uint32_t)((it / L::SU) & 1)));
      if (xact && yx_el < ne) {
        KT* Ke = Kst + yx_el * NB * NB;
#pragma unroll
        for (int k = 0; k < 3; ++k) {
          double acc[N1][N1];
#pragma unroll
          for (int a = 0; a < N1; ++a)
#pragma unroll
            for (int bb = 0; bb < N1; ++bb) acc[a][bb] = 0.0;
#pragma unroll
          for (int qx = 0; qx < Q1; ++qx)
#pragma unroll
            for (int ax = 0; ax < 2; ++ax) {
              double u[N1];
#pragma unroll
              for (int bb = 0; bb < N1; ++bb)
                u[bb] = Bt(0, qx, bb) * S[k][ax * 2 + 0][qx] + Bt(1, qx, bb) * S[k][ax * 2 + 1][qx];
#pragma unroll
              for (int a = 0; a < N1; ++a)
#pragma unroll
                for (int bb = 0; bb < N1; ++bb) acc[a][bb] = fma(Bt(ax, qx, a), u[bb], acc[a][bb]);
            }
          const bool mirror = (iz < jz) || (yi[k] < yj[k]);
          const int ib = N1 * (yi[k] + N1 * iz), jb = N1 * (yj[k] + N1 * jz);
#pragma unroll
          for (int a = 0; a < N1; ++a)
#pragma unroll
            for (int bb = 0; bb < N1; ++bb) {
              Ke[(ib + a) * NB + jb + bb] = (KT)acc[a][bb];
              if (mirror) Ke[(jb + bb) * NB + ib + a] = (KT)acc[a][bb];
            }
          if constexpr (RES) {  // fixed (row, column-group) slots, as in the YB = 1 path
            const double* ue = Ub + (su * E + yx_el) * NB;
            double* re = Rb + yx_el * NB * N1 * N1;
            const int gj = yj[k] + N1 * jz, gi = yi[k] + N1 * iz;
#pragma unroll
            for (int a = 0; a < N1; ++a) {
              double t = 0.0;
#pragma unroll
              for (int bb = 0; bb < N1; ++bb) t = fma(acc[a][bb], ue[jb + bb], t);
              re[(ib + a) * N1 * N1 + gj] = t;
            }
            if (mirror) {
#pragma unroll
              for (int bb = 0; bb < N1; ++bb) {
                double t = 0.0;
#pragma unroll
                for (int a = 0; a < N1; ++a) t = fma(acc[a][bb], ue[ib + a], t);
                re[(jb + bb) * N1 * N1 + gi] = t;
              }
            }
          }
        }
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      SFP_T(6, sfp_named_bar(2, NXT));
      if constexpr (RES) {
        for (int i = xtid; i < ne * NB; i += NXT) {
          const double* rg = Rb + (size_t)i * N1 * N1;
          double v = 0.0;
#pragma unroll
          for (int g = 0; g < N1 * N1; ++g) v += rg[g];
          if (r_elem) r_elem[lb * NB + i] = v;
          if (r_global) atomicAdd(r_global + DCb[su * E * NB + i], v);
        }
        sfp_arrive(&doneR[su]);
      }
      const uint32_t bytes = (uint32_t)ne * NB * NB * (uint32_t)sizeof(KT);
      KT* gdst = K + lb * NB * NB;
      if (FEB200_SFP_NOSTORE) {
      } else if (((reinterpret_cast<uintptr_t>(gdst) | bytes) & 15u) == 0) {
        if (xtid == 0) {
          if (FEB200_SFP_EVF) {
          uint64_t pol_;
          asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol_));
          asm volatile("cp.async.bulk.global.shared::cta.bulk_group.L2::cache_hint [%0], [%1], %2, %3;"
                       :: "l"(gdst), "r"(smem_u32(Kst)), "r"(bytes), "l"(pol_) : "memory");
        } else asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;"
                       :: "l"(gdst), "r"(smem_u32(Kst)), "r"(bytes) : "memory");
          asm volatile("cp.async.bulk.commit_group;" ::: "memory");
          asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
        }
      } else {
        for (int i = xtid; i < ne * NB * NB; i += NXT) gdst[i] = Kst[i];
      }
    }
    if (xtid == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  } else {
    // ======================= X: stages y and x, K store =======================
    const int xtid = tid - 32 * (1 + L::NG);
    // task order: all off-diagonal z-pair tasks of the batch, then all diagonal ones, so that
    // most warps are uniform and the diagonal warps can share T1 vectors between the two
    // orders (m, n), (n, m) of a pair (same vector when iz == jz)
    int yx_el, yx_r;
    if (xtid < E * L::TOFF) {
      yx_el = xtid / L::TOFF;
      yx_r = xtid - yx_el * L::TOFF;
    } else {
      const int t = xtid - E * L::TOFF;
      yx_el = t / (L::TPE - L::TOFF);
      yx_r = L::TOFF + (t - yx_el * (L::TPE - L::TOFF));
    }
    const bool xact = xtid < E * L::TPE;
    int iz = 0, jz = 0, iy = 0, jy = 0;
    if (yx_r < L::TOFF) {
      int c = yx_r / L::YP;
      const int yp = yx_r - c * L::YP;
      iy = yp / N1;
      jy = yp - iy * N1;
      for (int a = 0; a < N1; ++a) {
        if (c < N1 - 1 - a) { iz = a; jz = a + 1 + c; break; }
        c -= N1 - 1 - a;
      }
    } else {
      const int r = yx_r - L::TOFF;
      iz = jz = r / L::YPS;
      int c = r - iz * L::YPS;
      for (int a = 0; a < N1; ++a) {
        if (c < N1 - a) { iy = a; jy = a + c; break; }
        c -= N1 - a;
      }
    }
    const bool mirror = (iz < jz) || (iy < jy);
    const bool diag_warp = __all_sync(0xffffffffu, !xact || iz == jz);  // all lanes vote
    double Byp[4][Q1];
#pragma unroll
    for (int q = 0; q < Q1; ++q)
#pragma unroll
      for (int a = 0; a < 2; ++a)
#pragma unroll
        for (int bb = 0; bb < 2; ++bb) Byp[a * 2 + bb][q] = Bt(a, q, iy) * Bt(bb, q, jy);
    constexpr int NXT = 32 * L::NX;
    for (int64_t it = 0;; ++it) {
      const int64_t b = blockIdx.x + it * (int64_t)gridDim.x;
      if (b >= nbatch) break;
      const int64_t lb = b * E;
      const int ne = (int)((nloc - lb) < E ? (nloc - lb) : E);
      const int sl = (int)(it & 1);
      // the elected thread waited (end of iteration it - 1) for the store that last read
      // K slot it % 2; this barrier publishes that to the group
      SFP_T(5, sfp_named_bar(1, NXT));
      SFP_T(4, sfp_wait(&fullT[sl], (uint32_t)((it >> 1) & 1)));
      const double* T1e = reinterpret_cast<const double*>(smp + L::OFF_T1 + sl * L::T1SLOT) +
                          yx_el * L::T1CELL;
      double acc[N1][N1];
      if (FEB200_SFP_NOX) {
#pragma unroll
        for (int a = 0; a < N1; ++a)
#pragma unroll
          for (int bb = 0; bb < N1; ++bb) acc[a][bb] = (double)(a + bb);
        sfp_arrive(&emptyT[sl]);
      } else if (xact) {
        double S[4][Q1];
#pragma unroll
        for (int c = 0; c < 4; ++c)
#pragma unroll
          for (int q = 0; q < Q1; ++q) S[c][q] = 0.0;
        auto load_tv = [&](int ul, int zidx, double (&tv)[QQP]) {
          const double* src1 = T1e + (ul * N1 * N1 + zidx) * QQP;
          if constexpr (L::T1PAD % 2 == 1) {  // 8-B aligned vectors: LDS.64 (same wavefronts)
#pragma unroll
            for (int h = 0; h < Q2; ++h) tv[h] = src1[h];
          } else {
            const double2* src = reinterpret_cast<const double2*>(src1);
#pragma unroll
            for (int h = 0; h < Q2 / 2; ++h) {  // Q2 of the QQP values: the odd one by LDS.64
              const double2 v = src[h];
              tv[2 * h] = v.x;
              tv[2 * h + 1] = v.y;
            }
            if (Q2 & 1) tv[Q2 - 1] = src1[Q2 - 1];
          }
        };
        auto add_pair = [&](int m, int n, const double (&tv)[QQP]) {
          const int ay = m == 1, by = n == 1, cls = (m == 0) * 2 + (n == 0);
#pragma unroll
          for (int qx = 0; qx < Q1; ++qx)
#pragma unroll
            for (int qy = 0; qy < Q1; ++qy)
              S[cls][qx] = fma(Byp[ay * 2 + by][qy], tv[qx * Q1 + qy], S[cls][qx]);
        };
        if (diag_warp) {
          // diagonal z pair: T1^{u}[iz,iz] serves both orders of the unique pair u
#pragma unroll
          for (int ul = 0; ul < NUP; ++ul) {
            int m, n;
            upair(UBASE + ul, m, n);
            double tv[QQP];
            load_tv(ul, iz * N1 + iz, tv);
            add_pair(m, n, tv);
            if (m != n) add_pair(n, m, tv);
          }
        } else {
#pragma unroll
          for (int op = 0; op < NOP; ++op) {
            int m, n;
            if (DIFF && op < 9) { m = op / 3; n = op % 3; } else { m = 3; n = 3; }
            const int mm = m < n ? m : n, nn = m < n ? n : m;
            const int ul = (mm == 3) ? NUP - 1 : (mm == 0 ? nn : (mm == 1 ? 2 + nn : 5));
            const int zidx = (m > n) ? (jz * N1 + iz) : (iz * N1 + jz);
            double tv[QQP];
            load_tv(ul, zidx, tv);
            add_pair(m, n, tv);
          }
        }
        sfp_arrive(&emptyT[sl]);
#pragma unroll
        for (int a = 0; a < N1; ++a)
#pragma unroll
          for (int bb = 0; bb < N1; ++bb) acc[a][bb] = 0.0;
#pragma unroll
        for (int qx = 0; qx < Q1; ++qx)
#pragma unroll
          for (int ax = 0; ax < 2; ++ax) {
            double u[N1];
#pragma unroll
            for (int bb = 0; bb < N1; ++bb) u[bb] = Bt(0, qx, bb) * S[ax * 2 + 0][qx] + Bt(1, qx, bb) * S[ax * 2 + 1][qx];
#pragma unroll
            for (int a = 0; a < N1; ++a)
#pragma unroll
              for (int bb = 0; bb < N1; ++bb) acc[a][bb] = fma(Bt(ax, qx, a), u[bb], acc[a][bb]);
          }
      } else {
        sfp_arrive(&emptyT[sl]);
      }
      KT* Kst = reinterpret_cast<KT*>(smp + L::OFF_K + sl * L::KSLOT);
      const int su = (int)(it % L::SU);
      if constexpr (RES) SFP_T(7, sfp_wait(&fullU[su], (uint32_t)((it / L::SU) & 1)));
      if (xact && yx_el < ne) {
        KT* Ke = Kst + yx_el * NB * NB;
        const int ib = N1 * (iy + N1 * iz), jb = N1 * (jy + N1 * jz);
#pragma unroll
        for (int a = 0; a < N1; ++a)
#pragma unroll
          for (int bb = 0; bb < N1; ++bb) {
            Ke[(ib + a) * NB + jb + bb] = (KT)acc[a][bb];
            if (mirror) Ke[(jb + bb) * NB + ib + a] = (KT)acc[a][bb];
          }
        if constexpr (RES) {
          // r_e = K_e u_e (Alg. 1 for a linear form, pin P8).  Row (ix, iy, iz) of K_e is
          // split into N1^2 column groups (jy, jz) of N1 entries; exactly one task (direct
          // or mirrored) owns each (row, group), so the partial sums go to fixed slots
          // R[row][group] without atomics and are summed in a fixed order below.
          const double* ue = Ub + (su * E + yx_el) * NB;
          double* re = Rb + yx_el * NB * N1 * N1;
          const int gj = jy + N1 * jz, gi = iy + N1 * iz;
#pragma unroll
          for (int a = 0; a < N1; ++a) {
            double t = 0.0;
#pragma unroll
            for (int bb = 0; bb < N1; ++bb) t = fma(acc[a][bb], ue[jb + bb], t);
            re[(ib + a) * N1 * N1 + gj] = t;
          }
          if (mirror) {
#pragma unroll
            for (int bb = 0; bb < N1; ++bb) {
              double t = 0.0;
#pragma unroll
              for (int a = 0; a < N1; ++a) t = fma(acc[a][bb], ue[ib + a], t);
              re[(jb + bb) * N1 * N1 + gi] = t;
            }
          }
        }
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      SFP_T(6, sfp_named_bar(2, NXT));
      if constexpr (RES) {
        // sum the row groups, scatter r_e (fused assembly)
        for (int i = xtid; i < ne * NB; i += NXT) {
          const double* rg = Rb + (size_t)i * N1 * N1;
          double v = 0.0;
#pragma unroll
          for (int g = 0; g < N1 * N1; ++g) v += rg[g];
          if (r_elem) r_elem[lb * NB + i] = v;
          if (r_global) atomicAdd(r_global + DCb[su * E * NB + i], v);
        }
        sfp_arrive(&doneR[su]);
      }
      const uint32_t bytes = (uint32_t)ne * NB * NB * (uint32_t)sizeof(KT);
      KT* gdst = K + lb * NB * NB;
      if (FEB200_SFP_NOSTORE) {
      } else if (((reinterpret_cast<uintptr_t>(gdst) | bytes) & 15u) == 0) {
        if (xtid == 0) {
          if (FEB200_SFP_EVF) {
          uint64_t pol_;
          asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol_));
          asm volatile("cp.async.bulk.global.shared::cta.bulk_group.L2::cache_hint [%0], [%1], %2, %3;"
                       :: "l"(gdst), "r"(smem_u32(Kst)), "r"(bytes), "l"(pol_) : "memory");
        } else asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;"
                       :: "l"(gdst), "r"(smem_u32(Kst)), "r"(bytes) : "memory");
          asm volatile("cp.async.bulk.commit_group;" ::: "memory");
          asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
        }
      } else {
        for (int i = xtid; i < ne * NB * NB; i += NXT) gdst[i] = Kst[i];
      }
    }
    if (xtid == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  }
#ifdef FEB200_SFP_PROF
  if (lane == 0) {
    for (int k = 0; k < 8; ++k) if (prof_[k]) atomicAdd(&g_sfp_prof[k], prof_[k]);
    const int role = warp == 0 ? 0 : (warp <= L::NG ? 1 : 2);
    atomicAdd(&g_sfp_prof[8 + role], (unsigned long long)(clock64() - tstart_));
    atomicAdd(&g_sfp_prof[12 + role], 1ull);
  }
#endif
#undef Bt
}

template <int P, int FORM, bool RES = false, typename KT = double>
static cudaError_t launch_sfp_t(const fe_mesh* mh, MatArgs mat, int64_t e0, int64_t e1, KT* K,
                                cudaStream_t st, const double* u = nullptr, double* r_elem = nullptr,
                                double* r_global = nullptr) {
  using L = SFP<P, (FORM != FE_FORM_MASS ? 6 : 0) + (FORM != FE_FORM_DIFFUSION ? 1 : 0), RES, (int)sizeof(KT)>;
  auto kern = k_matrix_sfp<P, FORM, RES, KT>;
  const LaunchFacts lf = launch_facts((const void*)kern, L::THREADS, L::BYTES);
  if (lf.err != cudaSuccess) return lf.err;
  const int nsm = lf.nsm;
  const int64_t nbatch = (e1 - e0 + L::E - 1) / L::E;
  int grid = (int)(nbatch < nsm ? nbatch : nsm);
  grid = grid_cap(grid);
  if (grid <= 0) return cudaSuccess;
  kern<<<grid, L::THREADS, L::BYTES, st>>>(view_of(mh), (const KT*)mat.a, (const KT*)mat.b,
                                           e0, e1, K, u, r_elem, r_global);
  count_launch();
  return cudaGetLastError();
}

// Matrix mode plus the residual of the same linear scalar form from the element matrices
// (r_e = K_e u_e, scatter-added) in one pass of the pipelined kernel (p = 1, 2).
cudaError_t launch_matrix_residual_sf(const fe_mesh* mh, int form, MatArgs mat, const double* u,
                                      int64_t e0, int64_t e1, double* K, double* r_elem,
                                      double* r_global, cudaStream_t st) {
  if (mh->q1d != mh->order + 1 || (mh->order != 1 && mh->order != 2)) return cudaErrorNotSupported;
#define SFPR_CASE(P)                                                                                     \
  if (mh->order == P) switch (form) {                                                                    \
      case FE_FORM_DIFFUSION:                                                                            \
        return launch_sfp_t<P, FE_FORM_DIFFUSION, true>(mh, mat, e0, e1, K, st, u, r_elem, r_global);    \
      case FE_FORM_MASS:                                                                                 \
        return launch_sfp_t<P, FE_FORM_MASS, true>(mh, mat, e0, e1, K, st, u, r_elem, r_global);         \
      case FE_FORM_MASS_DIFFUSION:                                                                       \
        return launch_sfp_t<P, FE_FORM_MASS_DIFFUSION, true>(mh, mat, e0, e1, K, st, u, r_elem, r_global); \
      default: return cudaErrorNotSupported;                                                             \
    }
  SFPR_CASE(1)
  SFPR_CASE(2)
#undef SFPR_CASE
  return cudaErrorNotSupported;
}

template <int P, int FORM>
static cudaError_t launch_sf_t(const fe_mesh* mh, MatArgs mat, int64_t e0, int64_t e1, double* K,
                               cudaStream_t st) {
  constexpr bool DIFF = FORM != FE_FORM_MASS, MASS = FORM != FE_FORM_DIFFUSION;
  using L = SFM<P, DIFF, MASS>;
  auto kern = k_matrix_sf<P, FORM>;
  const LaunchFacts lf = launch_facts((const void*)kern, L::THREADS, L::BYTES);
  if (lf.err != cudaSuccess) return lf.err;
  const int nsm = lf.nsm, per_sm = lf.per_sm;
  const int64_t nbatch = (e1 - e0 + L::E - 1) / L::E;
  int grid = (int)((nbatch < (int64_t)nsm * per_sm) ? nbatch : (int64_t)nsm * per_sm);
  grid = grid_cap(grid);
  if (grid <= 0) return cudaSuccess;
  kern<<<grid, L::THREADS, L::BYTES, st>>>(view_of(mh), (const double*)mat.a, (const double*)mat.b,
                                          e0, e1, K);
  count_launch();
  return cudaGetLastError();
}

// fp32 element matrices of the scalar forms (FE_F32: fp32 coefficients and K, contraction in
// fp64) through the pipelined kernel, p = 1, 2; cudaErrorNotSupported otherwise.
cudaError_t launch_matrix_sf_f32(const fe_mesh* mh, int form, MatArgs mat, int64_t e0, int64_t e1,
                                 float* K, cudaStream_t st) {
  if (mh->q1d != mh->order + 1 || !FEB200_SFP) return cudaErrorNotSupported;
#define SFP32_CASE(P)                                                                                          \
  if (mh->order == P) switch (form) {                                                                          \
      case FE_FORM_DIFFUSION: return launch_sfp_t<P, FE_FORM_DIFFUSION, false, float>(mh, mat, e0, e1, K, st); \
      case FE_FORM_MASS: return launch_sfp_t<P, FE_FORM_MASS, false, float>(mh, mat, e0, e1, K, st);           \
      case FE_FORM_MASS_DIFFUSION:                                                                             \
        return launch_sfp_t<P, FE_FORM_MASS_DIFFUSION, false, float>(mh, mat, e0, e1, K, st);                  \
      default: return cudaErrorNotSupported;                                                                   \
    }
  SFP32_CASE(1)
  SFP32_CASE(2)
#undef SFP32_CASE
  return cudaErrorNotSupported;
}

// Returns cudaErrorNotSupported when the combination has no sum-factorised kernel.
cudaError_t launch_matrix_sf(const fe_mesh* mh, int form, MatArgs mat, int64_t e0, int64_t e1,
                             double* K, cudaStream_t st) {
  if (mh->q1d != mh->order + 1) return cudaErrorNotSupported;
  const bool pipelined = FEB200_SFP && option(FE_OPT_MATRIX_IMPL) != MATRIX_SF1;
  if (pipelined && (mh->order == 1 || mh->order == 2)) {
#define SFP_CASE(P)                                                                                \
  if (mh->order == P) switch (form) {                                                              \
      case FE_FORM_DIFFUSION: return launch_sfp_t<P, FE_FORM_DIFFUSION>(mh, mat, e0, e1, K, st);   \
      case FE_FORM_MASS: return launch_sfp_t<P, FE_FORM_MASS>(mh, mat, e0, e1, K, st);             \
      case FE_FORM_MASS_DIFFUSION: return launch_sfp_t<P, FE_FORM_MASS_DIFFUSION>(mh, mat, e0, e1, K, st); \
      default: return cudaErrorNotSupported;                                                       \
    }
    SFP_CASE(1)
    SFP_CASE(2)
#undef SFP_CASE
  }
#define SF_CASE(P)                                                                              \
  case P:                                                                                       \
    switch (form) {                                                                             \
      case FE_FORM_DIFFUSION: return launch_sf_t<P, FE_FORM_DIFFUSION>(mh, mat, e0, e1, K, st); \
      case FE_FORM_MASS: return launch_sf_t<P, FE_FORM_MASS>(mh, mat, e0, e1, K, st);           \
      case FE_FORM_MASS_DIFFUSION:                                                              \
        return launch_sf_t<P, FE_FORM_MASS_DIFFUSION>(mh, mat, e0, e1, K, st);                  \
      default: return cudaErrorNotSupported;                                                    \
    }
  switch (mh->order) {
    SF_CASE(1)
    SF_CASE(2)
    SF_CASE(3)
    SF_CASE(4)
  }
#undef SF_CASE
  return cudaErrorNotSupported;
}

}  // namespace feb200

#ifdef FEB200_SFP_PROF
extern "C" int fe_debug_sfp_prof(unsigned long long* out, int reset) {
  cudaDeviceSynchronize();
  cudaMemcpyFromSymbol(out, feb200::g_sfp_prof, sizeof(unsigned long long) * 16);
  if (reset) {
    unsigned long long z[16] = {};
    cudaMemcpyToSymbol(feb200::g_sfp_prof, z, sizeof(z));
  }
  return 0;
}
#endif
