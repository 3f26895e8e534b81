// Sum-factorised element matrices for the vector forms (elasticity, convective
// tangent, vector mass): Alg. 2 organised in D x D blocks
//   K_ab[k][l] = sum_q sum_{(m,n)} W^{ab}_{mn}(q) D^m_k(q) D^n_l(q),
//   D^m_k(q) = prod_d B^{[m == d]}[q_d][k_d]  (m = 0,1,2 reference derivative, 3 = value)
// with per-block, per-qp weights
//   elasticity  W^{ab}_{mn} = detw sum_{j,l} Jinv[m][j] C_{ajbl} Jinv[n][l],
//               C_{ajbl} = D[I(a,j)][I(b,l)]  (Voigt D with engineering shears; the Psg
//               of 'cq,cqje,rjI,cqIK,cqlf,slK->cresf', contracted analytically);
//               isotropic: C = lam d_aj d_bl + mu (d_ab d_jl + d_al d_jb)
//   convective  W^{ab}_{3n} = d_ab detw (Jinv u)_n,  W^{ab}_{33} = detw du_a/dx_b   (Eq. fe4)
//   vector mass W^{aa}_{33} = detw rho, off-diagonal blocks zero
//   weighted dot W^{ab}_{33} = detw M_ab(q)                                       ('ij,i,j')
// Each block is contracted axis by axis exactly as in k_matrix_sf.cu (stage z in
// smem, stages y and x in registers, one (z-pair, y-pair) per thread).  Elasticity
// blocks satisfy K_ba = K_ab^T, so only a <= b is computed; diagonal blocks are
// symmetric and use the symmetric thread set.  One cell per CTA iteration; the
// 81 x 81 K_e is staged in shared memory and written with coalesced stores.
#include "fe_const.cuh"
#include "fe_device.cuh"
#include "fe_internal.h"

namespace feb200 {

cudaError_t upload_const_tables_matrix_v(int order, const double* b1, const double* d1,
                                        const double* x1, const double* w1, cudaStream_t st) {
  return upload_tables_this_tu(order, b1, d1, x1, w1, st);
}

__device__ __forceinline__ int voigt(int a, int j) {
  return a == j ? a : (a + j == 1 ? 3 : (a + j == 2 ? 4 : 5));
}

// Block structure per form (all blocks of a cell are processed concurrently):
//   elasticity, isotropic: (0,0) (1,1) (2,2) symmetric + (0,1) (0,2) (1,2) mirrored; 9 pairs each
//   elasticity, FULL_D:    all 9 blocks, 9 pairs each, no symmetry assumed
//   convective:            diagonal blocks pairs (3,0) (3,1) (3,2) (3,3); off-diagonal (3,3), symmetric
//   vector mass:           3 diagonal blocks, pair (3,3), symmetric
//   weighted dot:          all 9 blocks, pair (3,3); each block symmetric in (k, l), M need not be
template <int FORM, bool FULLD>
struct BlockSet {
  static constexpr int NBLK = FORM == FE_FORM_VECTOR_MASS ? 3
                              : ((FORM == FE_FORM_CONVECTIVE || FORM == FE_FORM_WEIGHTED_DOT || FULLD) ? 9 : 6);
  static constexpr int NPAIR = FORM == FE_FORM_ELASTICITY ? 9 * NBLK
                               : (FORM == FE_FORM_CONVECTIVE ? 3 * 4 + 6 : (FORM == FE_FORM_WEIGHTED_DOT ? 9 : 3));
  __host__ __device__ static constexpr void info(int blk, int& a, int& b, bool& sym, bool& mirror, int& np,
                                                 int& pbase) {
    if (FORM == FE_FORM_VECTOR_MASS) {
      a = b = blk; sym = true; mirror = false; np = 1; pbase = blk;
    } else if (FORM == FE_FORM_WEIGHTED_DOT) {
      a = blk / 3; b = blk % 3; sym = true; mirror = false; np = 1; pbase = blk;
    } else if (FORM == FE_FORM_CONVECTIVE) {
      a = blk / 3; b = blk % 3; sym = a != b; mirror = false; np = a == b ? 4 : 1;
      pbase = 0;
      for (int i = 0; i < blk; ++i) pbase += (i / 3 == i % 3) ? 4 : 1;
    } else if (FULLD) {
      a = blk / 3; b = blk % 3; sym = false; mirror = false; np = 9; pbase = 9 * blk;
    } else {
      a = (0x100210 >> (4 * blk)) & 0xF;  // (0,0) (1,1) (2,2) (0,1) (0,2) (1,2)
      b = (0x221210 >> (4 * blk)) & 0xF;
      sym = a == b; mirror = a != b; np = 9; pbase = 9 * blk;
    }
  }
  // ordered pair p of a block -> (m, n); 3 = value
  __host__ __device__ static constexpr void pair(int a, int b, int p, int& m, int& n) {
    if (FORM == FE_FORM_ELASTICITY) { m = p / 3; n = p % 3; }
    else if (FORM == FE_FORM_CONVECTIVE) { m = 3; n = (a == b && p < 3) ? p : 3; }
    else { m = 3; n = 3; }
  }
};

template <int P, int FORM, bool FULLD = false>
struct SFV {
  using BS = BlockSet<FORM, FULLD>;
  static constexpr int N1 = P + 1, Q1 = P + 1, NB = N1 * N1 * N1, NQ = Q1 * Q1 * Q1;
  static constexpr int NDOF = 3 * NB;
  static constexpr int NPMAX = BS::NPAIR;  // pairs over all blocks
  static constexpr int QQP = (Q1 * Q1 + 1) / 2 * 2;
  static constexpr int T_YX = BS::NBLK * N1 * N1 * N1 * N1;  // upper bound of stage-y/x tasks
  static constexpr int THREADS = FORM == FE_FORM_VECTOR_MASS ? 128 : (FORM == FE_FORM_CONVECTIVE ? 512 : 384);
  // (weighted dot: 9 symmetric blocks, 384 threads)
  // per-qp data: Jinv (9), detw, lam, mu  | convective: Jinv, detw, u (3), grad u (9)
  static constexpr int QD = FORM == FE_FORM_CONVECTIVE ? 23 : 13;  // odd stride: no bank conflicts
  static constexpr int OFF_K = 0;                        // [NDOF][NDOF]
  static constexpr int OFF_EDGE = OFF_K + NDOF * NDOF;   // [36]
  static constexpr int OFF_QD = OFF_EDGE + 36;           // [NQ][QD]
  static constexpr int OFF_UE = OFF_QD + NQ * QD;        // [3][NB] state (convective)
  static constexpr int OFF_REF = OFF_UE + 3 * NB;        // [NQ][3][4] reference value/gradients of the state
  static constexpr int OFF_W = OFF_REF + (FORM == FE_FORM_CONVECTIVE ? 12 * NQ : 0);  // [NPMAX][NQ]
  static constexpr int OFF_T1 = (OFF_W + NPMAX * NQ + 1) / 2 * 2;  // [NPMAX][N1*N1][QQP]
  static constexpr int OFF_TAB = OFF_T1 + NPMAX * N1 * N1 * QQP;  // int tables: pair info, y/x tasks
  static constexpr int NTASK = T_YX;
  static constexpr int TOTAL = OFF_TAB + (NPMAX + NTASK + 2) / 2;
  static constexpr size_t BYTES = size_t(TOTAL) * 8;
};

template <int P, int FORM, bool FULLD>
__global__ void __launch_bounds__(SFV<P, FORM, FULLD>::THREADS)
    k_matrix_sfv(MeshView mv, int mat_kind, const double* __restrict__ ma,
                 const double* __restrict__ mb, const double* __restrict__ state_u, int64_t e0,
                 int64_t e1, double* __restrict__ K, const int* __restrict__ run_if) {
  // device-side dispatch (general D at p = 2, launch_matrix_vp): runs only when the symmetry
  // check flagged a non-symmetric D
  if (run_if != nullptr && *run_if == 0) return;
  using L = SFV<P, FORM, FULLD>;
  using BS = typename L::BS;
  constexpr int N1 = L::N1, Q1 = L::Q1, NB = L::NB, NQ = L::NQ, NDOF = L::NDOF, QQP = L::QQP;
  constexpr int QD = L::QD;
  extern __shared__ __align__(128) double sm[];
  double* Kst = sm + L::OFF_K;
  double* edge = sm + L::OFF_EDGE;
  double* qd = sm + L::OFF_QD;
  double* ue = sm + L::OFF_UE;
  double* ref = sm + L::OFF_REF;
  double* W = sm + L::OFF_W;
  double* T1 = sm + L::OFF_T1;
  int* pinfo = reinterpret_cast<int*>(sm + L::OFF_TAB);   // [NPMAX] ba | bb << 4 | m << 8 | n << 12 | pb << 16
  int* tinfo = pinfo + L::NPMAX;                           // [NTASK] blk | iz | jz | iy | jy (4 bits each), -1 = idle
  const int tid = threadIdx.x;
#define Bt(a, q, i) c_tab1d[P][a][q][i]
  constexpr int FULLT = N1 * N1 * N1 * N1;
  constexpr int SYMT = N1 * N1 * (N1 * (N1 - 1) / 2) + N1 * (N1 * (N1 + 1) / 2);
  // element-independent task tables
  for (int gp = tid; gp < L::NPMAX; gp += blockDim.x) {
    int blk = 0, ba = 0, bb = 0, np = 0, pb = 0;
    bool sym = false, mir = false;
    for (; blk < BS::NBLK; ++blk) {
      BS::info(blk, ba, bb, sym, mir, np, pb);
      if (gp < pb + np) break;
    }
    int m, n;
    BS::pair(ba, bb, gp - pb, m, n);
    pinfo[gp] = ba | (bb << 4) | (m << 8) | (n << 12) | (pb << 16);
  }
  for (int i = tid; i < L::NTASK; i += blockDim.x) {
    int blk = 0, ba = 0, bb = 0, np = 0, pb = 0, base = 0;
    bool sym = false, mir = false;
    for (; blk < BS::NBLK; ++blk) {
      BS::info(blk, ba, bb, sym, mir, np, pb);
      const int cnt = sym ? SYMT : FULLT;
      if (i < base + cnt) break;
      base += cnt;
    }
    if (blk == BS::NBLK) { tinfo[i] = -1; continue; }
    const int r = i - base;
    int iz, jz, iy, jy;
    if (!sym) {
      const int zp = r / (N1 * N1), yp = r % (N1 * N1);
      iz = zp / N1; jz = zp % N1; iy = yp / N1; jy = yp % N1;
    } else if (r < N1 * N1 * (N1 * (N1 - 1) / 2)) {  // off-diagonal z pair, any y pair
      int c = r / (N1 * N1);
      const int yp = r % (N1 * N1);
      iy = yp / N1; jy = yp % N1;
      iz = 0; jz = 1;
      for (int a = 0; a < N1; ++a) {
        if (c < N1 - 1 - a) { iz = a; jz = a + 1 + c; break; }
        c -= N1 - 1 - a;
      }
    } else {  // diagonal z pair, y pairs iy <= jy
      const int rr = r - N1 * N1 * (N1 * (N1 - 1) / 2);
      iz = jz = rr / (N1 * (N1 + 1) / 2);
      int c = rr % (N1 * (N1 + 1) / 2);
      iy = 0; jy = 0;
      for (int a = 0; a < N1; ++a) {
        if (c < N1 - a) { iy = a; jy = a + c; break; }
        c -= N1 - a;
      }
    }
    tinfo[i] = blk | (iz << 4) | (jz << 8) | (iy << 12) | (jy << 16);
  }
  __syncthreads();

  for (int64_t e = e0 + blockIdx.x; e < e1; e += gridDim.x) {
    // ---- A. edge vectors, state gather
    for (int i = tid; i < 36; i += blockDim.x) {
      const int ed = i / 3, comp = i % 3;
      const int d = ed >> 2, k = ed & 3, lo = k & 1, hi = k >> 1;
      const int v0 = d == 0 ? (2 * lo + 4 * hi) : (d == 1 ? (lo + 4 * hi) : (lo + 2 * hi));
      const int32_t* cn = mv.conn + 8 * e;
      edge[i] = mv.coords[3 * (int64_t)cn[v0 + (1 << d)] + comp] - mv.coords[3 * (int64_t)cn[v0] + comp];
    }
    if constexpr (FORM == FE_FORM_CONVECTIVE) {
      for (int i = tid; i < 3 * NB; i += blockDim.x) {
        const int a = i / NB, k = i % NB;
        ue[i] = state_u[3 * (int64_t)mv.dof_conn[e * NB + k] + a];
      }
    }
    __syncthreads();
    // ---- B. per-qp geometry (+ material / state)
    for (int q = tid; q < NQ; q += blockDim.x) {
      const double t0 = mv.xi[3 * q], t1 = mv.xi[3 * q + 1], t2 = mv.xi[3 * q + 2];
      double J[3][3];
#pragma unroll
      for (int i = 0; i < 3; ++i) {
        J[i][0] = (1 - t1) * (1 - t2) * edge[0 * 3 + i] + t1 * (1 - t2) * edge[1 * 3 + i] +
                  (1 - t1) * t2 * edge[2 * 3 + i] + t1 * t2 * edge[3 * 3 + i];
        J[i][1] = (1 - t0) * (1 - t2) * edge[4 * 3 + i] + t0 * (1 - t2) * edge[5 * 3 + i] +
                  (1 - t0) * t2 * edge[6 * 3 + i] + t0 * t2 * edge[7 * 3 + i];
        J[i][2] = (1 - t0) * (1 - t1) * edge[8 * 3 + i] + t0 * (1 - t1) * edge[9 * 3 + i] +
                  (1 - t0) * t1 * edge[10 * 3 + i] + t0 * t1 * edge[11 * 3 + i];
      }
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
      const double id = rcp_nr(det);
      double* o = qd + q * QD;
      // Jinv[m][j] = cof[j][m] / det
      o[0] = c00 * id; o[1] = c10 * id; o[2] = c20 * id;
      o[3] = c01 * id; o[4] = c11 * id; o[5] = c21 * id;
      o[6] = c02 * id; o[7] = c12 * id; o[8] = c22 * id;
      o[9] = mv.w[q] * det;
      if constexpr (FORM == FE_FORM_ELASTICITY) {
        if (mat_kind == FE_MAT_PER_ELEM) { o[10] = ma[e]; o[11] = mb[e]; }
        else if (mat_kind == FE_MAT_PER_QP) { o[10] = ma[e * NQ + q]; o[11] = mb[e * NQ + q]; }
      } else if constexpr (FORM == FE_FORM_VECTOR_MASS) {
        o[10] = ma[e * NQ + q];
      }
    }
    if constexpr (FORM == FE_FORM_CONVECTIVE) {
      // state at the qps: ref[q][a][c] = sum_k T[(q,c)][k] u_e[a][k], c = value, d/dxi_0..2
      for (int i = tid; i < NQ * 12; i += blockDim.x) {
        const int q = i / 12, a = (i / 4) % 3, c = i % 4;
        const double* tb = c == 0 ? mv.phi + q * NB : mv.dphi + (3 * q + c - 1) * NB;
        const double* uu = ue + a * NB;
        double sacc = 0.0;
        for (int k = 0; k < NB; ++k) sacc = fma(tb[k], uu[k], sacc);
        ref[i] = sacc;
      }
      __syncthreads();
      for (int q = tid; q < NQ; q += blockDim.x) {
        double* o = qd + q * QD;
        const double* rq = ref + q * 12;
#pragma unroll
        for (int a = 0; a < 3; ++a) {
          o[10 + a] = rq[4 * a];
#pragma unroll
          for (int j = 0; j < 3; ++j)
            o[13 + 3 * a + j] = rq[4 * a + 1] * o[j] + rq[4 * a + 2] * o[3 + j] + rq[4 * a + 3] * o[6 + j];
        }
      }
    }
    __syncthreads();
    // ---- C1. weights of every (block, pair) at every qp
    for (int i = tid; i < L::NPMAX * NQ; i += blockDim.x) {
      const int gp = i / NQ, q = i - gp * NQ;
      const int pi = pinfo[gp];
      const int ba = pi & 15, bb = (pi >> 4) & 15, m = (pi >> 8) & 15, n = (pi >> 12) & 15;
      const double* o = qd + q * QD;
      const double dw = o[9];
      double wv;
      if constexpr (FORM == FE_FORM_ELASTICITY) {
        if constexpr (FULLD) {
          const double* Dm = ma + (e * NQ + q) * 36;
          double sacc = 0.0;
#pragma unroll
          for (int j = 0; j < 3; ++j)
#pragma unroll
            for (int l = 0; l < 3; ++l)
              sacc += o[3 * m + j] * Dm[6 * voigt(ba, j) + voigt(bb, l)] * o[3 * n + l];
          wv = dw * sacc;
        } else {
          // sum_{j,l} Jinv[m][j] C_{a j b l} Jinv[n][l], C isotropic
          const double lam = o[10], mu = o[11];
          const double jj = o[3 * m] * o[3 * n] + o[3 * m + 1] * o[3 * n + 1] + o[3 * m + 2] * o[3 * n + 2];
          wv = dw * (lam * o[3 * m + ba] * o[3 * n + bb] + mu * ((ba == bb ? jj : 0.0) + o[3 * m + bb] * o[3 * n + ba]));
        }
      } else if constexpr (FORM == FE_FORM_WEIGHTED_DOT) {
        wv = dw * ma[(e * NQ + q) * 9 + 3 * ba + bb];
      } else if constexpr (FORM == FE_FORM_CONVECTIVE) {
        if (n == 3) wv = dw * o[13 + 3 * ba + bb];  // du_a/dx_b
        else wv = dw * (o[3 * n] * o[10] + o[3 * n + 1] * o[11] + o[3 * n + 2] * o[12]);  // (Jinv u)_n
      } else {
        wv = dw * o[10];
      }
      W[i] = wv;
    }
    __syncthreads();
    // ---- C2. stage z for every (block, pair): T1^gp[iz,jz][qx,qy]
    for (int i = tid; i < L::NPMAX * Q1 * Q1; i += blockDim.x) {
      const int gp = i / (Q1 * Q1), qxy = i - gp * Q1 * Q1;
      const int qx = qxy / Q1, qy = qxy - qx * Q1;
      const int pi = pinfo[gp];
      const int m = (pi >> 8) & 15, n = (pi >> 12) & 15;
      const int az = m == 2, bz = n == 2;
      const double* w = W + gp * NQ + qx + Q1 * qy;
      double t[Q1][N1];
#pragma unroll
      for (int qz = 0; qz < Q1; ++qz) {
        const double c = w[Q1 * Q1 * qz];
#pragma unroll
        for (int a = 0; a < N1; ++a) t[qz][a] = c * (az ? Bt(1, qz, a) : Bt(0, qz, a));
      }
      double* out = T1 + gp * N1 * N1 * QQP + qxy;
#pragma unroll
      for (int a = 0; a < N1; ++a)
#pragma unroll
        for (int b = 0; b < N1; ++b) {
          double sacc = 0.0;
#pragma unroll
          for (int qz = 0; qz < Q1; ++qz) sacc = fma(t[qz][a], bz ? Bt(1, qz, b) : Bt(0, qz, b), sacc);
          out[(a * N1 + b) * QQP] = sacc;
        }
    }
    __syncthreads();
    // ---- C3. stage y + x: one (block, z-pair, y-pair) per task
    for (int i = tid; i < L::NTASK; i += blockDim.x) {
      const int ti = tinfo[i];
      if (ti < 0) break;
      const int blk = ti & 15, iz = (ti >> 4) & 15, jz = (ti >> 8) & 15, iy = (ti >> 12) & 15, jy = (ti >> 16) & 15;
      int ba, bb, np, pb;
      bool sym, mir;
      BS::info(blk, ba, bb, sym, mir, np, pb);
      double S[4][Q1];
#pragma unroll
      for (int c = 0; c < 4; ++c)
#pragma unroll
        for (int q = 0; q < Q1; ++q) S[c][q] = 0.0;
      // pairs of the block; convective off-diagonal blocks have only (3,3) = slot 3
      constexpr int NPB = FORM == FE_FORM_ELASTICITY ? 9 : (FORM == FE_FORM_CONVECTIVE ? 4 : 1);
#pragma unroll
      for (int pp = 0; pp < NPB; ++pp) {
        int m, n;
        if (FORM == FE_FORM_ELASTICITY) { m = pp / 3; n = pp % 3; }
        else if (FORM == FE_FORM_CONVECTIVE) { m = 3; n = pp < 3 ? pp : 3; }
        else { m = 3; n = 3; }
        const bool on = (FORM == FE_FORM_CONVECTIVE && np == 1) ? (pp == 3) : true;
        if (!on) continue;
        const int p = (FORM == FE_FORM_CONVECTIVE && np == 1) ? 0 : pp;
        const int ay = m == 1, by = n == 1, cls = (m == 0) * 2 + (n == 0);
        const double2* src = reinterpret_cast<const double2*>(T1 + ((pb + p) * N1 * N1 + iz * N1 + jz) * QQP);
        double tv[QQP];
#pragma unroll
        for (int h = 0; h < QQP / 2; ++h) {
          const double2 v = src[h];
          tv[2 * h] = v.x;
          tv[2 * h + 1] = v.y;
        }
#pragma unroll
        for (int qx = 0; qx < Q1; ++qx) {
          double sq = 0.0;
#pragma unroll
          for (int qy = 0; qy < Q1; ++qy)
            sq = fma((ay ? Bt(1, qy, iy) : Bt(0, qy, iy)) * (by ? Bt(1, qy, jy) : Bt(0, qy, jy)),
                     tv[qx * Q1 + qy], sq);
          S[cls][qx] += sq;
        }
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
          double uu[N1];
#pragma unroll
          for (int b = 0; b < N1; ++b) uu[b] = Bt(0, qx, b) * S[ax * 2 + 0][qx] + Bt(1, qx, b) * S[ax * 2 + 1][qx];
#pragma unroll
          for (int a = 0; a < N1; ++a)
#pragma unroll
            for (int b = 0; b < N1; ++b) acc[a][b] = fma(Bt(ax, qx, a), uu[b], acc[a][b]);
        }
      const int ib = N1 * (iy + N1 * iz), jb = N1 * (jy + N1 * jz);
      const bool mirror_in = sym && (iz < jz || iy < jy);
#pragma unroll
      for (int a = 0; a < N1; ++a)
#pragma unroll
        for (int b = 0; b < N1; ++b) {
          const int rr = ba * NB + ib + a, cc = bb * NB + jb + b;
          Kst[rr * NDOF + cc] = acc[a][b];
          if (mirror_in) Kst[(ba * NB + jb + b) * NDOF + bb * NB + ib + a] = acc[a][b];
          if (mir) Kst[cc * NDOF + rr] = acc[a][b];
        }
    }
    __syncthreads();
    // ---- D. coalesced store (vector mass: off-diagonal blocks are zero)
    double* Ke = K + (e - e0) * (int64_t)NDOF * NDOF;
    for (int i = tid; i < NDOF * NDOF; i += blockDim.x) {
      double v = Kst[i];
      if constexpr (FORM == FE_FORM_VECTOR_MASS) {
        const int r = i / NDOF, c = i - r * NDOF;
        if (r / NB != c / NB) v = 0.0;
      }
      Ke[i] = v;
    }
    __syncthreads();
  }
#undef Bt
}

template <int P, int FORM, bool FULLD = false>
static cudaError_t launch_sfv_t(const fe_mesh* mh, MatArgs mat, const double* state_u, int64_t e0,
                                int64_t e1, double* K, cudaStream_t st, const int* run_if = nullptr) {
  if constexpr (FORM == FE_FORM_ELASTICITY && !FULLD) {
    if (mat.kind == FE_MAT_FULL_D) return launch_sfv_t<P, FORM, true>(mh, mat, state_u, e0, e1, K, st, run_if);
  }
  using L = SFV<P, FORM, FULLD>;
  if (L::BYTES > 227 * 1024) return cudaErrorNotSupported;
  auto kern = k_matrix_sfv<P, FORM, FULLD>;
  const LaunchFacts lf = launch_facts((const void*)kern, L::THREADS, L::BYTES);
  if (lf.err != cudaSuccess) return lf.err;
  const int nsm = lf.nsm, per_sm = lf.per_sm;
  const int64_t n = e1 - e0;
  int grid = (int)((n < (int64_t)nsm * per_sm) ? n : (int64_t)nsm * per_sm);
  grid = grid_cap(grid);
  if (grid <= 0) return cudaSuccess;
  kern<<<grid, L::THREADS, L::BYTES, st>>>(view_of(mh), mat.kind, (const double*)mat.a,
                                           (const double*)mat.b, state_u, e0, e1, K, run_if);
  count_launch();
  return cudaGetLastError();
}

cudaError_t launch_matrix_sfv_gated(const fe_mesh* mh, int form, MatArgs mat, const double* state_u,
                                    int64_t e0, int64_t e1, double* K, cudaStream_t st,
                                    const int* run_if) {
  if (mh->q1d != mh->order + 1 || mh->order != 2 || form != FE_FORM_ELASTICITY ||
      mat.kind != FE_MAT_FULL_D)
    return cudaErrorNotSupported;
  return launch_sfv_t<2, FE_FORM_ELASTICITY, true>(mh, mat, state_u, e0, e1, K, st, run_if);
}

cudaError_t launch_matrix_sfv(const fe_mesh* mh, int form, MatArgs mat, const double* state_u,
                              int64_t e0, int64_t e1, double* K, cudaStream_t st) {
  if (mh->q1d != mh->order + 1) return cudaErrorNotSupported;
#define SFV_CASE(P)                                                                                       \
  case P:                                                                                                 \
    switch (form) {                                                                                       \
      case FE_FORM_ELASTICITY: return launch_sfv_t<P, FE_FORM_ELASTICITY>(mh, mat, state_u, e0, e1, K, st); \
      case FE_FORM_CONVECTIVE: return launch_sfv_t<P, FE_FORM_CONVECTIVE>(mh, mat, state_u, e0, e1, K, st); \
      case FE_FORM_VECTOR_MASS: return launch_sfv_t<P, FE_FORM_VECTOR_MASS>(mh, mat, state_u, e0, e1, K, st); \
      case FE_FORM_WEIGHTED_DOT: return launch_sfv_t<P, FE_FORM_WEIGHTED_DOT>(mh, mat, state_u, e0, e1, K, st); \
      default: return cudaErrorNotSupported;                                                              \
    }
  switch (mh->order) {
    SFV_CASE(1)
    SFV_CASE(2)
  }
#undef SFV_CASE
  return cudaErrorNotSupported;
}

}  // namespace feb200
