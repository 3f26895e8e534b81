// Device-side building blocks of the B200 hot path.
//   - dmma_884: FP64 tensor-core MMA (mma.sync m8n8k4 f64 -> SASS DMMA),
//     the only FP64 tensor path on sm_100a (tcgen05 has no f64 kind).
//   - seg_gemm: warp-tiled  C[m][n] = sum_seg sum_kk wt[kk] A[kk][m] B[kk][n]
//     over "segments" of rows, with predicated (zero) padding to 8x8x4 tiles.
//   - hex_geometry: J, det J, J^-1 of the trilinear map at a reference point
//     (J_ij = dx_i/dxi_j; du/dx_j = du/dxi_k J^-1_kj P:657).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace feb200 {

struct Seg {
  const double* A;   // A[kk * a_rs + m]
  const double* B;   // B[kk * b_rs + n]
  const double* wt;  // optional row weight wt[kk] applied to A (nullable)
  int a_rs, b_rs, count;
};

__device__ __forceinline__ void dmma_884(double c[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(c[0]), "+d"(c[1])
               : "d"(a), "d"(b));
}

// Warp-cooperative GEMM over segments; each warp owns groups of 1 x NTG tiles
// of 8x8 outputs.  Fragment layouts (PTX ISA mma.m8n8k4 .f64):
//   A: a0 = A[m = lane/4][k = lane%4];  B: b0 = B[k = lane%4][n = lane/4];
//   C: c_i = C[m = lane/4][n = 2 (lane%4) + i].
// epi(m, n, value) is called once for every valid output (m < M, n < N).
template <int NTG, class Epi>
__device__ __forceinline__ void seg_gemm(const Seg* segs, int nseg, int M, int N, int warp,
                                         int nwarps, int lane, Epi&& epi) {
  const int mt = (M + 7) >> 3, nt = (N + 7) >> 3;
  const int ngn = (nt + NTG - 1) / NTG;
  const int lr = lane >> 2, lc = lane & 3;
  for (int g = warp; g < mt * ngn; g += nwarps) {
    const int tm = g / ngn, tn0 = (g - tm * ngn) * NTG;
    double c[NTG][2];
#pragma unroll
    for (int t = 0; t < NTG; ++t) c[t][0] = c[t][1] = 0.0;
    const int am = tm * 8 + lr;
    const bool am_ok = am < M;
    for (int s = 0; s < nseg; ++s) {
      const Seg sg = segs[s];
      for (int k0 = 0; k0 < sg.count; k0 += 4) {
        const int kk = k0 + lc;
        const bool kv = kk < sg.count;
        double a = 0.0;
        if (kv && am_ok) {
          a = sg.A[(int64_t)kk * sg.a_rs + am];
          if (sg.wt) a *= sg.wt[kk];
        }
#pragma unroll
        for (int t = 0; t < NTG; ++t) {
          const int bn = (tn0 + t) * 8 + lr;
          const double b = (kv && bn < N) ? sg.B[(int64_t)kk * sg.b_rs + bn] : 0.0;
          dmma_884(c[t], a, b);
        }
      }
    }
    const int row = tm * 8 + lr;
#pragma unroll
    for (int t = 0; t < NTG; ++t) {
      const int col = (tn0 + t) * 8 + 2 * lc;
      if (row < M) {
        if (col < N) epi(row, col, c[t][0]);
        if (col + 1 < N) epi(row, col + 1, c[t][1]);
      }
    }
  }
}

// SIMT fallback of the same contraction for non-fp64 element types (fp32 path).
template <typename T, class Epi>
__device__ __forceinline__ void seg_gemm_simt(const T* const* As, const T* const* Bs,
                                              const int* a_rs, const int* b_rs, const int* counts,
                                              int nseg, int M, int N, int tid, int nthreads,
                                              Epi&& epi) {
  for (int o = tid; o < M * N; o += nthreads) {
    const int m = o / N, n = o - m * N;
    T acc = T(0);
    for (int s = 0; s < nseg; ++s) {
      const T* A = As[s];
      const T* B = Bs[s];
      for (int kk = 0; kk < counts[s]; ++kk) acc = fma(A[(int64_t)kk * a_rs[s] + m], B[(int64_t)kk * b_rs[s] + n], acc);
    }
    epi(m, n, acc);
  }
}

// Jacobian of the trilinear map x(xi) = sum_v x_v psi_v(xi) at xi, vertices
// xv[v][3] with v = a + 2b + 4c.  Returns det J; Jinv row-major Jinv[m][j].
// 1/x for x > 0 (det J): rcp.approx + two Newton steps, within ~1 ulp of the IEEE quotient
// and a few instructions instead of the division's slow-path-guarded sequence
__device__ __forceinline__ double rcp_nr(double x) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  double e = fma(-x, r, 1.0);
  r = fma(r, e, r);
  e = fma(-x, r, 1.0);
  return fma(r, e, r);
}

__device__ __forceinline__ double hex_geometry(const double* __restrict__ xv, double x0, double x1,
                                               double x2, double Jinv[9]) {
  double J[9];
#pragma unroll
  for (int i = 0; i < 9; ++i) J[i] = 0.0;
#pragma unroll
  for (int v = 0; v < 8; ++v) {
    const int a = v & 1, b = (v >> 1) & 1, c = v >> 2;
    const double la = a ? x0 : 1.0 - x0, lb = b ? x1 : 1.0 - x1, lc = c ? x2 : 1.0 - x2;
    const double da = a ? 1.0 : -1.0, db = b ? 1.0 : -1.0, dc = c ? 1.0 : -1.0;
    const double g0 = da * lb * lc, g1 = la * db * lc, g2 = la * lb * dc;
#pragma unroll
    for (int i = 0; i < 3; ++i) {
      const double x = xv[3 * v + i];
      J[3 * i + 0] = fma(x, g0, J[3 * i + 0]);
      J[3 * i + 1] = fma(x, g1, J[3 * i + 1]);
      J[3 * i + 2] = fma(x, g2, J[3 * i + 2]);
    }
  }
  const double c00 = J[4] * J[8] - J[5] * J[7];
  const double c01 = J[5] * J[6] - J[3] * J[8];
  const double c02 = J[3] * J[7] - J[4] * J[6];
  const double c10 = J[2] * J[7] - J[1] * J[8];
  const double c11 = J[0] * J[8] - J[2] * J[6];
  const double c12 = J[1] * J[6] - J[0] * J[7];
  const double c20 = J[1] * J[5] - J[2] * J[4];
  const double c21 = J[2] * J[3] - J[0] * J[5];
  const double c22 = J[0] * J[4] - J[1] * J[3];
  const double det = J[0] * c00 + J[1] * c01 + J[2] * c02;
  const double id = 1.0 / det;
  // inverse = adjugate / det = cofactor^T / det
  Jinv[0] = c00 * id; Jinv[1] = c10 * id; Jinv[2] = c20 * id;
  Jinv[3] = c01 * id; Jinv[4] = c11 * id; Jinv[5] = c21 * id;
  Jinv[6] = c02 * id; Jinv[7] = c12 * id; Jinv[8] = c22 * id;
  return det;
}

// 32-byte read-only load (LDG.256 on sm_100): four consecutive doubles, 32-B aligned address
__device__ __forceinline__ void ld_nc_v4(const double* p, double& x, double& y, double& z, double& w) {
  asm("ld.global.nc.v4.f64 {%0,%1,%2,%3}, [%4];" : "=d"(x), "=d"(y), "=d"(z), "=d"(w) : "l"(p));
}

// Bulk prefetch of a contiguous global range into L2 (TMA engine; one instruction, no
// completion tracking).  p and bytes must be 16-byte multiples; the caller checks.
__device__ __forceinline__ void l2_prefetch_bulk(const void* p, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}

template <typename T>
__device__ __forceinline__ void atomic_add(T* p, T v) {
  atomicAdd(p, v);
}

}  // namespace feb200
