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
#include "fe_device.cuh"
#include "fe_internal.h"

namespace feb200 {

template <int P, bool DIFF, bool MASS>
struct SFM {
  static constexpr int N1 = P + 1, Q1 = P + 1, NB = N1 * N1 * N1, NQ = Q1 * Q1 * Q1;
  static constexpr int NUP = (DIFF ? 6 : 0) + (MASS ? 1 : 0);   // unique (m <= n) pairs
  static constexpr int NOP = (DIFF ? 9 : 0) + (MASS ? 1 : 0);   // ordered pairs
  static constexpr int ZP = N1 * (N1 + 1) / 2, YP = N1 * N1;
  static constexpr int TPE = ZP * YP;                          // stage-y/x threads per cell
  static constexpr int E = P == 1 ? 16 : (P == 2 ? 4 : 1);      // cells per CTA iteration
  static constexpr int T_GEO = E * NQ, T_Z = E * NUP * Q1 * Q1, T_YX = E * TPE;
  static constexpr int TMAX = T_GEO > T_Z ? (T_GEO > T_YX ? T_GEO : T_YX) : (T_Z > T_YX ? T_Z : T_YX);
  static constexpr int THREADS = (TMAX + 31) / 32 * 32;
  // shared memory (doubles)
  static constexpr int KST = E * NB * NB;                       // one staging buffer
  static constexpr int OFF_K = 0;                               // 2 x KST (16-B aligned)
  static constexpr int OFF_XV = OFF_K + 2 * KST;
  static constexpr int OFF_COEF = OFF_XV + E * 24;              // [E][2][NQ] kappa, rho
  static constexpr int OFF_W = OFF_COEF + E * 2 * NQ;           // [E][NUP][NQ]
  static constexpr int OFF_T1 = OFF_W + E * NUP * NQ;           // [E][NUP][Q1*Q1][N1*N1]
  static constexpr int OFF_B = OFF_T1 + E * NUP * Q1 * Q1 * N1 * N1;  // [2][Q1][N1]
  static constexpr int TOTAL = OFF_B + 2 * Q1 * N1;
  static constexpr size_t BYTES = size_t(TOTAL) * 8;
};

// unique pair u -> (m, n), m <= n; index 6 is the value-value pair (3,3)
__device__ __forceinline__ void upair(int u, int& m, int& n) {
  // m = {0,0,0,1,1,2,3}[u], n = {0,1,2,1,2,2,3}[u] as packed nibbles (no local memory)
  m = (0x3211000 >> (4 * u)) & 0xF;
  n = (0x3221210 >> (4 * u)) & 0xF;
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

template <int P, int FORM>
__global__ void __launch_bounds__(SFM<P, FORM != FE_FORM_MASS, FORM != FE_FORM_DIFFUSION>::THREADS)
    k_matrix_sf(MeshView mv, const double* __restrict__ ma, const double* __restrict__ mb,
                int64_t e0, int64_t e1, double* __restrict__ K) {
  constexpr bool DIFF = FORM != FE_FORM_MASS, MASS = FORM != FE_FORM_DIFFUSION;
  using L = SFM<P, DIFF, MASS>;
  constexpr int N1 = L::N1, Q1 = L::Q1, NB = L::NB, NQ = L::NQ, NUP = L::NUP, E = L::E;
  constexpr int UBASE = DIFF ? 0 : 6;  // first unique-pair id
  extern __shared__ __align__(128) double sm[];
  double* xv = sm + L::OFF_XV;
  double* coef = sm + L::OFF_COEF;
  double* W = sm + L::OFF_W;
  double* T1 = sm + L::OFF_T1;
  double* Bt = sm + L::OFF_B;
  const int tid = threadIdx.x;

  for (int i = tid; i < 2 * Q1 * N1; i += blockDim.x) Bt[i] = (i < Q1 * N1) ? mv.b1[i] : mv.d1[i - Q1 * N1];
  __syncthreads();

  // thread-constant stage-y/x data
  const int yx_el = tid / L::TPE, yx_r = tid - yx_el * L::TPE;
  const int zp = yx_r / L::YP, yp = yx_r - zp * L::YP;
  int iz = 0, jz = 0;
  {
    int c = zp;
    for (int a = 0; a < N1; ++a) {
      if (c < N1 - a) { iz = a; jz = a + c; break; }
      c -= N1 - a;
    }
  }
  const int iy = yp / N1, jy = yp - iy * N1;
  double Byp[4][Q1];  // Byp[ay*2+by][qy] = B^ay[qy][iy] B^by[qy][jy]
  double Bx[2][Q1][N1];
#pragma unroll
  for (int q = 0; q < Q1; ++q) {
#pragma unroll
    for (int a = 0; a < 2; ++a)
#pragma unroll
      for (int b = 0; b < 2; ++b) Byp[a * 2 + b][q] = Bt[(a * Q1 + q) * N1 + iy] * Bt[(b * Q1 + q) * N1 + jy];
#pragma unroll
    for (int a = 0; a < 2; ++a)
#pragma unroll
      for (int i = 0; i < N1; ++i) Bx[a][q][i] = Bt[(a * Q1 + q) * N1 + i];
  }

  const int64_t nloc = e1 - e0;
  const int64_t nbatch = (nloc + E - 1) / E;
  int it = 0;
  for (int64_t bidx = blockIdx.x; bidx < nbatch; bidx += gridDim.x, ++it) {
    const int64_t lb = bidx * E;                 // local index of the first cell
    const int ne = (int)((nloc - lb) < E ? (nloc - lb) : E);
    double* Kst = sm + L::OFF_K + (it & 1) * L::KST;
    // A. cell data: vertices and per-qp coefficients
    for (int i = tid; i < E * 24; i += blockDim.x) {
      const int el = i / 24, r = i - el * 24;
      xv[i] = el < ne ? mv.coords[3 * (int64_t)mv.conn[8 * (e0 + lb + el) + r / 3] + r % 3] : 0.0;
    }
    for (int i = tid; i < E * NQ; i += blockDim.x) {
      const int el = i / NQ, q = i - el * NQ;
      const int64_t g = (e0 + lb + el) * NQ + q;
      double kap = 0.0, rho = 0.0;
      if (el < ne) {
        if constexpr (FORM == FE_FORM_DIFFUSION) kap = ma[g];
        if constexpr (FORM == FE_FORM_MASS) rho = ma[g];
        if constexpr (FORM == FE_FORM_MASS_DIFFUSION) { rho = ma[g]; kap = mb[g]; }
      }
      coef[(el * 2) * NQ + q] = kap;
      coef[(el * 2 + 1) * NQ + q] = rho;
    }
    // the TMA store issued two batches ago read this staging buffer: wait for it
    if (tid == 0) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
    __syncthreads();
    // B. geometry -> W^{mn}[q]
    for (int i = tid; i < E * NQ; i += blockDim.x) {
      const int el = i / NQ, q = i - el * NQ;
      double Ji[9];
      const double det = hex_geometry(xv + 24 * el, mv.xi[3 * q], mv.xi[3 * q + 1], mv.xi[3 * q + 2], Ji);
      const double dw = det * mv.w[q];
      double* Wel = W + el * NUP * NQ;
      if constexpr (DIFF) {
        const double s = dw * coef[(el * 2) * NQ + q];
#pragma unroll
        for (int u = 0; u < 6; ++u) {
          int m, n;
          upair(u, m, n);
          Wel[u * NQ + q] = s * (Ji[3 * m] * Ji[3 * n] + Ji[3 * m + 1] * Ji[3 * n + 1] + Ji[3 * m + 2] * Ji[3 * n + 2]);
        }
      }
      if constexpr (MASS) Wel[(NUP - 1) * NQ + q] = dw * coef[(el * 2 + 1) * NQ + q];
    }
    __syncthreads();
    // C. stage z
    for (int i = tid; i < L::T_Z; i += blockDim.x) {
      const int el = i / (NUP * Q1 * Q1), r = i - el * NUP * Q1 * Q1;
      const int ul = r / (Q1 * Q1), qxy = r - ul * Q1 * Q1;  // qxy = qx * Q1 + qy
      const int qx = qxy / Q1, qy = qxy - qx * Q1;
      int m, n;
      upair(UBASE + ul, m, n);
      const int az = m == 2, bz = n == 2;
      const double* w = W + (el * NUP + ul) * NQ + qx + Q1 * qy;
      double t[Q1][N1];
#pragma unroll
      for (int qz = 0; qz < Q1; ++qz) {
        const double c = w[Q1 * Q1 * qz];
#pragma unroll
        for (int a = 0; a < N1; ++a) t[qz][a] = c * Bt[(az * Q1 + qz) * N1 + a];
      }
      double* out = T1 + ((el * NUP + ul) * Q1 * Q1 + qxy) * N1 * N1;
#pragma unroll
      for (int a = 0; a < N1; ++a)
#pragma unroll
        for (int b = 0; b < N1; ++b) {
          double s = 0.0;
#pragma unroll
          for (int qz = 0; qz < Q1; ++qz) s = fma(t[qz][a], Bt[(bz * Q1 + qz) * N1 + b], s);
          out[a * N1 + b] = s;
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
      const double* T1e = T1 + yx_el * NUP * Q1 * Q1 * N1 * N1;
#pragma unroll
      for (int op = 0; op < L::NOP; ++op) {
        int m, n;
        if (DIFF && op < 9) { m = op / 3; n = op % 3; } else { m = 3; n = 3; }
        const int mm = m < n ? m : n, nn = m < n ? n : m;
        const int ul = (mm == 3) ? NUP - 1 : (mm == 0 ? nn : (mm == 1 ? 2 + nn : 5));
        const int zidx = (m > n) ? (jz * N1 + iz) : (iz * N1 + jz);
        const int ay = m == 1, by = n == 1, cls = (m == 0) * 2 + (n == 0);
        const double* src = T1e + ul * Q1 * Q1 * N1 * N1 + zidx;
#pragma unroll
        for (int qx = 0; qx < Q1; ++qx)
#pragma unroll
          for (int qy = 0; qy < Q1; ++qy)
            S[cls][qx] = fma(Byp[ay * 2 + by][qy], src[(qx * Q1 + qy) * N1 * N1], S[cls][qx]);
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
          for (int b = 0; b < N1; ++b) u[b] = Bx[0][qx][b] * S[ax * 2 + 0][qx] + Bx[1][qx][b] * S[ax * 2 + 1][qx];
#pragma unroll
          for (int a = 0; a < N1; ++a)
#pragma unroll
            for (int b = 0; b < N1; ++b) acc[a][b] = fma(Bx[ax][qx][a], u[b], acc[a][b]);
        }
      double* Ke = Kst + yx_el * NB * NB;
      const int ib = N1 * (iy + N1 * iz), jb = N1 * (jy + N1 * jz);
#pragma unroll
      for (int a = 0; a < N1; ++a)
#pragma unroll
        for (int b = 0; b < N1; ++b) {
          Ke[(ib + a) * NB + jb + b] = acc[a][b];
          if (iz < jz) Ke[(jb + b) * NB + ib + a] = acc[a][b];
        }
    }
    // E. write the batch: one TMA bulk store of ne * NB^2 doubles (contiguous in K)
    const uint32_t bytes = (uint32_t)ne * NB * NB * 8;
    double* gdst = K + lb * NB * NB;
    if ((bytes & 15u) == 0) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncthreads();
      if (tid == 0) {
        asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;"
                     :: "l"(gdst), "r"(smem_u32(Kst)), "r"(bytes) : "memory");
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      }
    } else {
      __syncthreads();
      for (int i = tid; i < ne * NB * NB; i += blockDim.x) gdst[i] = Kst[i];
    }
  }
  if (tid == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

template <int P, int FORM>
static cudaError_t launch_sf_t(const fe_mesh* mh, MatArgs mat, int64_t e0, int64_t e1, double* K,
                               cudaStream_t st) {
  constexpr bool DIFF = FORM != FE_FORM_MASS, MASS = FORM != FE_FORM_DIFFUSION;
  using L = SFM<P, DIFF, MASS>;
  auto kern = k_matrix_sf<P, FORM>;
  cudaError_t err = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)L::BYTES);
  if (err != cudaSuccess) return err;
  int nsm = 148, per_sm = 1, dev = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, L::THREADS, L::BYTES);
  if (per_sm < 1) per_sm = 1;
  const int64_t nbatch = (e1 - e0 + L::E - 1) / L::E;
  const int grid = (int)((nbatch < (int64_t)nsm * per_sm) ? nbatch : (int64_t)nsm * per_sm);
  if (grid <= 0) return cudaSuccess;
  kern<<<grid, L::THREADS, L::BYTES, st>>>(view_of(mh), (const double*)mat.a, (const double*)mat.b,
                                          e0, e1, K);
  count_launch();
  return cudaGetLastError();
}

// Returns cudaErrorNotSupported when the combination has no sum-factorised kernel.
cudaError_t launch_matrix_sf(const fe_mesh* mh, int form, MatArgs mat, int64_t e0, int64_t e1,
                             double* K, cudaStream_t st) {
  if (mh->q1d != mh->order + 1) return cudaErrorNotSupported;
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
  }
#undef SF_CASE
  return cudaErrorNotSupported;
}

}  // namespace feb200
