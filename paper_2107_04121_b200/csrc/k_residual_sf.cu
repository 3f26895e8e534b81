// Sum-factorised residual mode (Alg. 1) with
// the gather of the cell DOFs and the fused scatter-add.
//
// Same integral as k_residual.cu, with the dense stacked table T = [Phi; grad Phi]
// replaced by its tensor-product factors (Eq. fe1):
//   Phi_k(q) = B0[qx][kx] B0[qy][ky] B0[qz][kz],  d Phi_k/d xi_x = B1[qx][kx] B0 B0, ...
// so interpolation and testing are sequences of 1D contractions of length p+1.
// One thread per (x, y) column of a cell holds its z-column in registers:
//   gather  -> stage x (smem exchange) -> stage y (smem exchange) -> stage z (registers)
//   -> per-qp geometry (edge vectors) + flux (fe_flux.cuh), pulled back to reference
//   -> z^T (registers) -> y^T (smem) -> x^T (smem) -> fused atomic scatter.
// Q2: ~1.5k FMA per cell and component for the contractions instead of ~4.4k
// (dense); Q4: ~11k instead of ~125k.
#include "fe_const.cuh"
#include "fe_device.cuh"
#include "fe_flux.cuh"
#include "fe_internal.h"

namespace feb200 {

cudaError_t upload_const_tables_residual(int order, const double* b1, const double* d1,
                                        const double* x1, const double* w1, cudaStream_t st) {
  return upload_tables_this_tu(order, b1, d1, x1, w1, st);
}

__device__ __forceinline__ uint32_t saddr(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, int count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(saddr(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(saddr(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(saddr(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tWAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n\t}" ::"r"(saddr(bar)), "r"(parity) : "memory");
}
// TMA bulk copy global -> shared, completion counted on an mbarrier (16-B aligned, size % 16 == 0)
__device__ __forceinline__ void tma_load(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               ::"r"(saddr(dst)), "l"(src), "r"(bytes), "r"(saddr(bar)) : "memory");
}

#ifndef FEB200_RSF_PADT
#define FEB200_RSF_PADT 0
#endif
#ifndef FEB200_RSF_PAD
#define FEB200_RSF_PAD 1
#endif
#ifndef FEB200_RSF_EB3
#define FEB200_RSF_EB3 14  // 126 of 128 lanes busy (aligned-superset fetch)
#endif
#ifndef FEB200_RSF_EB2
#define FEB200_RSF_EB2 20
#endif
#ifndef FEB200_RSF_MINB2
#define FEB200_RSF_MINB2 2
#endif
#ifndef FEB200_RSF_EB4
#define FEB200_RSF_EB4 5  // 125 of 128 lanes busy (needs the aligned-superset fetch: 5 cells are not 16-B multiples)
#endif
#ifndef FEB200_RSF_MINB4
#define FEB200_RSF_MINB4 3
#endif
#ifndef FEB200_RSF_MINB3
#define FEB200_RSF_MINB3 2
#endif
#ifndef FEB200_RSF_PADB
#define FEB200_RSF_PADB (sizeof(T) == 8 ? 96 : 32)
#endif
#ifndef FEB200_RSF_L2PF
#define FEB200_RSF_L2PF 0  // measured: 0.383 ms with, 0.360 ms without (C3d residual)
#endif
#ifndef FEB200_RSF_PADP
#define FEB200_RSF_PADP 4
#endif
// PENCIL (scalar forms, p >= 3): each stage runs on pencils along its own direction -- the
// thread of a cell's (p0, p1) slot is the x-pencil (y, z) = (p0, p1) for stages x / x^T, the
// y-pencil (x, z) for y / y^T and the z-column (x, y) for z / flux / z^T -- with the tensors
// transposed through two shared-memory buffers in between: every exchanged value is stored
// once and loaded once (5 + 5 per value and stage instead of 1 + p + 1 loads), one barrier
// per stage
#ifndef FEB200_RSF_PENCIL
#define FEB200_RSF_PENCIL 1
#endif
#ifndef FEB200_RSF_COF
#define FEB200_RSF_COF 1
#endif
template <int P, int FORM, typename T>
struct RSF {
  static constexpr int N1 = P + 1, Q1 = P + 1, NB = N1 * N1 * N1, NQ = Q1 * Q1 * Q1;
  static constexpr int D = FormD<FORM>::D;
  static constexpr int TPE = Q1 * Q1;  // threads per cell
  static constexpr int EB0 = P == 1 ? 32 : (P == 2 ? 28 : (P == 3 ? 16 : 8));  // multiples of 4 (TMA alignment)
  // cells per CTA iteration; vector forms at p = 2 use smaller batches so that the three
  // components' register arrays fit without spilling (fewer, fatter threads per SM)
  static constexpr int EB = (D == 3 && P >= 3) ? EB0 / 2
                           : ((D == 3 && P == 2) ? FEB200_RSF_EB3
                              : (P == 2 ? FEB200_RSF_EB2 : (P == 4 ? FEB200_RSF_EB4 : EB0)));
  // PENCIL at p = 4: fp64 two CTAs per SM (204 registers, no spills; three: 168 with spills,
  // 0.200 vs 0.181 ms on C4), fp32 three
  static constexpr int MINB = (D == 3 && P == 2) ? FEB200_RSF_MINB3
                              : (D == 1 && P == 2 ? FEB200_RSF_MINB2
                                 : (D == 1 && P == 4 ? ((FEB200_RSF_PENCIL && sizeof(T) == 8) ? 2 : FEB200_RSF_MINB4) : 2));
  static constexpr int THREADS = (EB * TPE + 31) / 32 * 32;
  static constexpr int THREADS_ = THREADS;
  // exchange buffer per cell (elements of T), padded so that consecutive cells start PADB
  // bytes apart modulo 128 B (fp64: 96 B, chosen with a half-warp bank model of the column
  // stores and the x- / y-direction reads of the stages; fp32: 32 B)
  static constexpr int XS0 = 3 * D * NQ;
  // FEB200_RSF_PADT: per-cell stride congruent to the threads per cell (mod one 128-B row), so
  // that the column stores of consecutive cells continue each other's bank sequence
  static constexpr int XSB = (int)(128 / sizeof(T));
  // (measured: P = 4 gains 1.3 % (C4 f64) / 1.1 % (f32) with it; P <= 3 keep the 96 / 32-B pad)
  static constexpr int XSQ = (FEB200_RSF_PADT || P == 4) ? (TPE % XSB) : (int)(FEB200_RSF_PADB / sizeof(T));
  static constexpr int XS = (FEB200_RSF_PAD && (P <= FEB200_RSF_PADP)) ? XS0 + ((XSQ - XS0 % XSB) % XSB + XSB) % XSB : XS0;
  // prefetch slots (x2): conn [EB][8], dof_conn [EB][NB] (int32), material a, b [EB][NQ] (T),
  // vertex coordinates [EB][24]; plus two mbarriers
  static constexpr size_t SL_CONN = 0;
  static constexpr size_t SL_DOF = SL_CONN + size_t(EB) * 8 * 4;
  // dof / material regions carry 16 B of slack: a batch whose block does not start on a 16-B
  // boundary is fetched as the enclosing 16-B-aligned range and read at its offset
  static constexpr size_t SL_MA = (SL_DOF + size_t(EB) * NB * 4 + 16 + 15) / 16 * 16;
  static constexpr size_t SL_MB = (SL_MA + size_t(EB) * NQ * sizeof(T) + 16 + 15) / 16 * 16;
  static constexpr size_t SL_SIZE = (SL_MB + size_t(EB) * NQ * sizeof(T) + 16 + 15) / 16 * 16;
  static constexpr size_t OFF_X = (2 * Q1 * N1 * 8 + 15) / 16 * 16;
  static constexpr bool PENCIL = FEB200_RSF_PENCIL && D == 1 && P >= 3;
  // PENCIL transpose layouts (element offset x sx + y sy + z sz + cell * CS), chosen with a
  // bank model of the stage accesses at p = 4, 5 cells per CTA: XY for the tensors written and
  // read along x and y (stage x -> y, y^T -> x^T), YZ for those along y and z (stage y -> z,
  // z^T -> y^T); at p = 3 the same strides are injective too
  static constexpr int PSX = sizeof(T) == 8 ? 5 : 1, PSY = sizeof(T) == 8 ? 11 : 5, PSZ = 25;
  static constexpr int CSXY = sizeof(T) == 8 ? 509 : 381;
  static constexpr int PZY = 37, CSYZ = 569, PTS = 185;  // YZ: x + 5 y + 37 z, tensor stride
  static constexpr int PTSXY = sizeof(T) == 8 ? 165 : 125;
  static constexpr int PXS = CSXY > CSYZ ? CSXY : CSYZ;  // per-cell footprint of a buffer
  static constexpr size_t OFF_XV = (OFF_X + size_t(EB) * (PENCIL ? 2 * PXS : XS) * sizeof(T) + 15) / 16 * 16;
  static constexpr int XVS = 28;  // per-cell stride of the staged vertex coordinates (bank spread)
  static constexpr size_t OFF_SLOT = OFF_XV + size_t(EB) * XVS * 8;
  static constexpr int NSLOT = 3;  // index/material ring: TMA two batches ahead
  static constexpr size_t OFF_BAR = OFF_SLOT + NSLOT * SL_SIZE;
  static constexpr size_t BYTES = OFF_BAR + 8 * NSLOT;
  static constexpr int PX = (EB * 24 + THREADS_ - 1) / THREADS_;  // vertex coordinates per thread
  static constexpr bool VAL = FORM == FE_FORM_MASS || FORM == FE_FORM_VECTOR_MASS ||
                              FORM == FE_FORM_MASS_DIFFUSION || FORM == FE_FORM_CONVECTIVE ||
                              FORM == FE_FORM_WEIGHTED_DOT;
  // GRAD: the flux reads grad u (forward gradient stages); BGRAD: the flux has an f1 part
  // (tested against grad v: backward gradient stages)
  static constexpr bool GRAD = FORM == FE_FORM_DIFFUSION || FORM == FE_FORM_MASS_DIFFUSION ||
                               FORM == FE_FORM_ELASTICITY || FORM == FE_FORM_CONVECTIVE;
  static constexpr bool BGRAD = FORM == FE_FORM_DIFFUSION || FORM == FE_FORM_MASS_DIFFUSION ||
                                FORM == FE_FORM_ELASTICITY || FORM == FE_FORM_DIVERGENCE;
};

template <int P, int FORM, typename T, bool PEER = false>
__global__ void __launch_bounds__(RSF<P, FORM, T>::THREADS, RSF<P, FORM, T>::MINB)
    k_residual_sf(MeshView mv, int mat_kind, const T* __restrict__ ma, const T* __restrict__ mb,
                  const T* __restrict__ u, int64_t e0, int64_t e1, T* __restrict__ r_elem,
                  T* __restrict__ r_global, double* __restrict__ eval_out, PeerWin pw) {
  using L = RSF<P, FORM, T>;
  constexpr int N1 = L::N1, Q1 = L::Q1, NB = L::NB, NQ = L::NQ, D = L::D, EB = L::EB;
  constexpr int Q2 = Q1 * Q1;
  constexpr bool VAL = L::VAL, GRAD = L::GRAD;
  // the backward pass tests against grad v only where the flux has an f1 part
  // (the convective residual v . (grad u) u has f0 only, Eq. fe2)
  constexpr bool BGRAD = L::BGRAD;
  // scalar per-qp forms: the flux in cofactor form (FEB200_RSF_COF)
  constexpr bool SCALARF = FEB200_RSF_COF && D == 1 &&
                           (FORM == FE_FORM_DIFFUSION || FORM == FE_FORM_MASS || FORM == FE_FORM_MASS_DIFFUSION);
  // forms whose flux is linear in grad u (f0 of the convective form, f1 of elasticity): the
  // flux evaluated at det grad u in cofactor form (FEB200_RSF_COF)
  constexpr bool COFV = FEB200_RSF_COF && (FORM == FE_FORM_ELASTICITY || FORM == FE_FORM_CONVECTIVE);
  constexpr bool PENCIL = L::PENCIL;
  using A = T;  // contraction arithmetic in the call's precision (geometry and flux stay fp64)
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T* Bs = reinterpret_cast<T*>(smem_raw);  // [2][Q1][N1] in the arithmetic type
  T* X = reinterpret_cast<T*>(smem_raw + L::OFF_X);  // [EB][D][3][Q1^3]
  double* xvs = reinterpret_cast<double*>(smem_raw + L::OFF_XV);  // [EB][24] vertex coordinates
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem_raw + L::OFF_BAR);
  auto slot_base = [&](int s_) { return smem_raw + L::OFF_SLOT + s_ * L::SL_SIZE; };
  const int tid = threadIdx.x;
  const int el = tid / L::TPE, tt = tid - el * L::TPE;
  const int tx = tt % Q1, ty = tt / Q1;
  const bool active = tid < EB * L::TPE;
#define B(a, q, i) ((A)c_tab1d[P][a][q][i])
  // 1D tables in smem for the thread-dependent rows / columns (stages x, y, y^T, x^T);
  // stage z and z^T use the warp-uniform constant copy.
  for (int i = tid; i < 2 * Q1 * N1; i += blockDim.x) Bs[i] = (&c_tab1d[P][0][0][0])[(i / (Q1 * N1)) * 25 + ((i / N1) % Q1) * 5 + i % N1];
#define Rx(a, i) Bs[((a) * Q1 + tx) * N1 + (i)]
#define Ry(a, i) Bs[((a) * Q1 + ty) * N1 + (i)]
#define Cx(a, q) Bs[((a) * Q1 + (q)) * N1 + tx]
#define Cy(a, q) Bs[((a) * Q1 + (q)) * N1 + ty]
  __syncthreads();

  const int64_t nloc = e1 - e0;
  const int64_t nbatch = (nloc + EB - 1) / EB;
  const int64_t G = gridDim.x;
  // material blocks fetched with the indices: per-qp arrays of the scalar forms / elasticity
  constexpr bool MAT_QP = FORM == FE_FORM_DIFFUSION || FORM == FE_FORM_MASS ||
                          FORM == FE_FORM_VECTOR_MASS || FORM == FE_FORM_MASS_DIFFUSION;
  const int nma = MAT_QP ? NQ : ((FORM == FE_FORM_ELASTICITY && mat_kind == FE_MAT_PER_QP) ? NQ
                                 : (FORM == FE_FORM_ELASTICITY && mat_kind == FE_MAT_PER_ELEM) ? 1 : 0);
  const bool has_mb = FORM == FE_FORM_MASS_DIFFUSION || (FORM == FE_FORM_ELASTICITY && nma > 0);
  if (tid == 0) {
    for (int k = 0; k < L::NSLOT; ++k) mbar_init(&bars[k], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  // byte offset of a block start within its 16-B line (the fetch and the readers agree on it)
  auto misal = [](const void* p_) { return (uint32_t)(reinterpret_cast<uintptr_t>(p_) & 15u); };
  // TMA bulk loads of the contiguous per-batch blocks (conn, dof_conn, material) into slot j % NSLOT
  auto fetch_idx = [&](int64_t j) {
    const int64_t b = blockIdx.x + j * G;
    if (b >= nbatch) return;
    const int sl = (int)(j % L::NSLOT);
    unsigned char* base = slot_base(sl);
    const int64_t eb = e0 + b * EB;
    const int ne = (int)((e1 - eb) < EB ? (e1 - eb) : EB);
    const uint32_t bc = ne * 32u, bd = ne * NB * 4u, bm = ne * nma * (uint32_t)sizeof(T);
    const void* gc = mv.conn + 8 * eb;
    const void* gd = mv.dof_conn + eb * NB;
    const void* ga = ma + eb * nma;
    const void* gb = has_mb ? (const void*)(mb + eb * nma) : nullptr;
    auto al = [](const void* p, uint32_t n) { return ((reinterpret_cast<uintptr_t>(p) | n) & 15u) == 0; };
    if constexpr (FORM == FE_FORM_ELASTICITY) {
      // general D (7.8 KB per Q2 cell, read per qp through L1 by the flux): pull this batch's
      // block into L2 two batches ahead
      if (FEB200_RSF_L2PF && mat_kind == FE_MAT_FULL_D && tid == 0) {
        const void* gD = ma + eb * NQ * 36;
        const uint32_t bD = (uint32_t)ne * NQ * 36u * (uint32_t)sizeof(T);
        if (al(gD, bD)) l2_prefetch_bulk(gD, bD);
      }
    }
    // 16-B-aligned enclosing ranges (the data lands at offset o* in the slot region)
    const uint32_t od = misal(gd), oa = nma ? misal(ga) : 0u, ob = has_mb ? misal(gb) : 0u;
    const uint32_t bd2 = (od + bd + 15u) & ~15u, ba2 = (oa + bm + 15u) & ~15u, bb2 = (ob + bm + 15u) & ~15u;
    const char* dend = reinterpret_cast<const char*>(mv.dof_conn + mv.n_elems * NB);
    const char* aend = reinterpret_cast<const char*>(ma + mv.n_elems * nma);
    const char* bend = has_mb ? reinterpret_cast<const char*>(mb + mv.n_elems * nma) : nullptr;
    const bool ok = al(gc, bc) && reinterpret_cast<const char*>(gd) - od + bd2 <= dend &&
                    (nma == 0 || (reinterpret_cast<const char*>(ga) - oa + ba2 <= aend &&
                                  (!has_mb || reinterpret_cast<const char*>(gb) - ob + bb2 <= bend)));
    if (ok) {
      if (tid == 0) {
        mbar_expect_tx(&bars[sl], bc + bd2 + (nma ? ba2 + (has_mb ? bb2 : 0u) : 0u));
        tma_load(base + L::SL_CONN, gc, bc, &bars[sl]);
        tma_load(base + L::SL_DOF, reinterpret_cast<const char*>(gd) - od, bd2, &bars[sl]);
        if (nma) {
          tma_load(base + L::SL_MA, reinterpret_cast<const char*>(ga) - oa, ba2, &bars[sl]);
          if (has_mb) tma_load(base + L::SL_MB, reinterpret_cast<const char*>(gb) - ob, bb2, &bars[sl]);
        }
      }
    } else {  // range at the end of an array: plain copies (same offsets), then a plain arrival
      int32_t* cs = reinterpret_cast<int32_t*>(base + L::SL_CONN);
      int32_t* ds = reinterpret_cast<int32_t*>(base + L::SL_DOF + od);
      T* as_ = reinterpret_cast<T*>(base + L::SL_MA + oa);
      T* bs_ = reinterpret_cast<T*>(base + L::SL_MB + ob);
      for (int i = tid; i < ne * 8; i += blockDim.x) cs[i] = mv.conn[8 * eb + i];
      for (int i = tid; i < ne * NB; i += blockDim.x) ds[i] = mv.dof_conn[eb * NB + i];
      for (int i = tid; i < ne * nma; i += blockDim.x) {
        as_[i] = ma[eb * nma + i];
        if (has_mb) bs_[i] = mb[eb * nma + i];
      }
      __syncthreads();
      if (tid == 0) mbar_arrive(&bars[sl]);
    }
  };
  // register prefetch of the dependent gathers (u at the column's nodes, vertex coordinates)
  A u_next[D][N1];
  double x_next[L::PX];
  auto gather_next = [&](int64_t j) {
    const int64_t b = blockIdx.x + j * G;
    const int sl = (int)(j % L::NSLOT);
    const unsigned char* base = slot_base(sl);
    const int32_t* cs = reinterpret_cast<const int32_t*>(base + L::SL_CONN);
    const int64_t eb = e0 + b * EB;
    const int32_t* ds = reinterpret_cast<const int32_t*>(base + L::SL_DOF + misal(mv.dof_conn + eb * NB));
    const int ne = b < nbatch ? (int)((e1 - eb) < EB ? (e1 - eb) : EB) : 0;
    if (ne > 0) mbar_wait(&bars[sl], (uint32_t)((j / L::NSLOT) & 1));
    const bool v = active && el < ne;
#pragma unroll
    for (int kz = 0; kz < N1; ++kz) {
      // z-column (tx, ty, kz); PENCIL: x-pencil (kx = kz, y = tx, z = ty)
      const int nidx = PENCIL ? kz + N1 * tx + N1 * N1 * ty : tx + N1 * ty + N1 * N1 * kz;
      const int dof = v ? ds[el * NB + nidx] : 0;
#pragma unroll
      for (int a = 0; a < D; ++a) u_next[a][kz] = v ? (A)u[(int64_t)dof * D + a] : A(0);
    }
#pragma unroll
    for (int h = 0; h < L::PX; ++h) {
      const int i = tid + h * blockDim.x;
      const int c = i / 24, r = i - c * 24;
      x_next[h] = (i < EB * 24 && c < ne) ? mv.coords[3 * (int64_t)cs[c * 8 + r / 3] + r % 3] : 0.0;
    }
  };
  fetch_idx(0);
  fetch_idx(1);
  gather_next(0);
  int64_t it = 0;
  for (int64_t bidx = blockIdx.x; bidx < nbatch; bidx += G, ++it) {
    const int64_t eb = e0 + bidx * EB;
    const int ne = (int)((e1 - eb) < EB ? (e1 - eb) : EB);
    const bool valid = active && el < ne;
    const int64_t e = eb + el;
    const int sl = (int)(it % L::NSLOT);
    const unsigned char* base = slot_base(sl);
    fetch_idx(it + 2);  // slot (it+2)%3 was last read by batch it-1 (done)
    // this batch's vertex coordinates and column values from the prefetch registers
#pragma unroll
    for (int h = 0; h < L::PX; ++h) {
      const int i = tid + h * blockDim.x;
      if (i < EB * 24) xvs[(i / 24) * L::XVS + i % 24] = x_next[h];
    }
    const int32_t* ds = reinterpret_cast<const int32_t*>(base + L::SL_DOF + misal(mv.dof_conn + eb * NB)) + el * NB;
    const T* msa = reinterpret_cast<const T*>(base + L::SL_MA + (nma ? misal(ma + eb * nma) : 0u)) + el * nma;
    const T* msb = reinterpret_cast<const T*>(base + L::SL_MB + (has_mb ? misal(mb + eb * nma) : 0u)) + el * nma;
    int dcol[N1];
    A uc[D][N1];
#pragma unroll
    for (int kz = 0; kz < N1; ++kz) {
      dcol[kz] = valid ? ds[PENCIL ? kz + N1 * tx + N1 * N1 * ty : tx + N1 * ty + N1 * N1 * kz] : 0;
#pragma unroll
      for (int a = 0; a < D; ++a) uc[a][kz] = u_next[a][kz];
    }
    // gathers of the next batch now, so that their latency overlaps this whole batch
    gather_next(it + 1);
    MatQ<T> mq[Q1];
    auto load_mq = [&]() {
#pragma unroll
    for (int qz = 0; qz < Q1; ++qz) {
      const int q = tx + Q1 * ty + Q1 * Q1 * qz;
      MatQ<T> m{0.0, 0.0, nullptr};
      if (valid) {
        if constexpr (FORM == FE_FORM_ELASTICITY) {
          if (mat_kind == FE_MAT_FULL_D) m.Dm = ma + (e * NQ + q) * 36;
          else if (mat_kind == FE_MAT_PER_ELEM) { m.a = (double)msa[0]; m.b = (double)msb[0]; }
          else { m.a = (double)msa[q]; m.b = (double)msb[q]; }
        } else if constexpr (FORM == FE_FORM_WEIGHTED_DOT) {
          m.Dm = ma + (e * NQ + q) * 9;  // 3x3 block read through L1 like FULL_D
        } else if constexpr (MAT_QP) {
          m.a = (double)msa[q];
          if constexpr (FORM == FE_FORM_MASS_DIFFUSION) m.b = (double)msb[q];
        }
      }
      mq[qz] = m;
    }
    };
    if constexpr (!PENCIL) load_mq();  // PENCIL: loaded after the transposes (register pressure)
    T* Xe = X + el * L::XS;
    // PENCIL: buffers A (X) and B (X + EB PXS), each in layout XY or YZ per use
    T* XaXY = X + el * L::CSXY;
    T* XaYZ = X + el * L::CSYZ;
    T* XbXY = X + (size_t)EB * L::PXS + el * L::CSXY;
    T* XbYZ = X + (size_t)EB * L::PXS + el * L::CSYZ;
    auto oXY = [](int x, int y, int z) { return x * L::PSX + y * L::PSY + z * L::PSZ; };
    auto oYZ = [](int x, int y, int z) { return x + 5 * y + L::PZY * z; };
    (void)XaXY; (void)XaYZ; (void)XbXY; (void)XbYZ; (void)oXY; (void)oYZ;
    A c00[D][N1], c01[D][N1], c10[D][N1];  // [kz] at (qx = tx, qy = ty)
    if constexpr (PENCIL) {
      // ---- stage x on the x-pencil (y, z) = (tx, ty): kx -> qx, into buffer A (layout XY)
      if (active) {
#pragma unroll
        for (int qx = 0; qx < Q1; ++qx) {
          A s0 = A(0), s1 = A(0);
#pragma unroll
          for (int kx = 0; kx < N1; ++kx) {
            s0 = fma(B(0, qx, kx), uc[0][kx], s0);
            if (GRAD) s1 = fma(B(1, qx, kx), uc[0][kx], s1);
          }
          XaXY[oXY(qx, tx, ty)] = (T)s0;
          if (GRAD) XaXY[L::PTSXY + oXY(qx, tx, ty)] = (T)s1;
        }
      }
      __syncthreads();
      // ---- stage y on the y-pencil (x, z) = (tx, ty): ky -> qy, into buffer B (layout YZ)
      if (active) {
        A v0[N1], v1[N1];
#pragma unroll
        for (int ky = 0; ky < N1; ++ky) {
          v0[ky] = (A)XaXY[oXY(tx, ky, ty)];
          v1[ky] = GRAD ? (A)XaXY[L::PTSXY + oXY(tx, ky, ty)] : A(0);
        }
#pragma unroll
        for (int qy = 0; qy < Q1; ++qy) {
          A s00 = A(0), s01 = A(0), s10 = A(0);
#pragma unroll
          for (int ky = 0; ky < N1; ++ky) {
            s00 = fma(B(0, qy, ky), v0[ky], s00);
            if (GRAD) {
              s01 = fma(B(1, qy, ky), v0[ky], s01);
              s10 = fma(B(0, qy, ky), v1[ky], s10);
            }
          }
          const int o = oYZ(tx, qy, ty);
          XbYZ[o] = (T)s00;
          if (GRAD) {
            XbYZ[L::PTS + o] = (T)s01;
            XbYZ[2 * L::PTS + o] = (T)s10;
          }
        }
      }
      __syncthreads();
      // ---- the z-column (x, y) = (tx, ty) of the three tensors
#pragma unroll
      for (int kz = 0; kz < N1; ++kz) {
        const int o = oYZ(tx, ty, kz);
        c00[0][kz] = active ? (A)XbYZ[o] : A(0);
        c01[0][kz] = (active && GRAD) ? (A)XbYZ[L::PTS + o] : A(0);
        c10[0][kz] = (active && GRAD) ? (A)XbYZ[2 * L::PTS + o] : A(0);
      }
    } else {
    // ---- stage x: contract kx -> qx
    if (active) {
#pragma unroll
      for (int a = 0; a < D; ++a)
#pragma unroll
        for (int kz = 0; kz < N1; ++kz) Xe[(a * 3) * NQ + kz * Q2 + ty * Q1 + tx] = (T)uc[a][kz];
    }
    __syncthreads();
    A a0[D][N1], a1[D][N1];  // [kz] at (qx = tx, ky = ty)
#pragma unroll
    for (int a = 0; a < D; ++a)
#pragma unroll
      for (int kz = 0; kz < N1; ++kz) {
        A s0 = A(0), s1 = A(0);
        const T* src = Xe + (a * 3) * NQ + kz * Q2 + ty * Q1;
#pragma unroll
        for (int kx = 0; kx < N1; ++kx) {
          const A v = active ? (A)src[kx] : A(0);
          s0 = fma(Rx(0, kx), v, s0);
          if (GRAD) s1 = fma(Rx(1, kx), v, s1);
        }
        a0[a][kz] = s0;
        a1[a][kz] = s1;
      }
    __syncthreads();
    // ---- stage y: contract ky -> qy
    if (active) {
#pragma unroll
      for (int a = 0; a < D; ++a)
#pragma unroll
        for (int kz = 0; kz < N1; ++kz) {
          Xe[(a * 3 + 0) * NQ + kz * Q2 + ty * Q1 + tx] = (T)a0[a][kz];
          if (GRAD) Xe[(a * 3 + 1) * NQ + kz * Q2 + ty * Q1 + tx] = (T)a1[a][kz];
        }
    }
    __syncthreads();
#pragma unroll
    for (int a = 0; a < D; ++a)
#pragma unroll
      for (int kz = 0; kz < N1; ++kz) {
        A s00 = A(0), s01 = A(0), s10 = A(0);
#pragma unroll
        for (int ky = 0; ky < N1; ++ky) {
          const A v0 = active ? (A)Xe[(a * 3 + 0) * NQ + kz * Q2 + ky * Q1 + tx] : A(0);
          s00 = fma(Ry(0, ky), v0, s00);
          if (GRAD) {
            const A v1 = active ? (A)Xe[(a * 3 + 1) * NQ + kz * Q2 + ky * Q1 + tx] : A(0);
            s01 = fma(Ry(1, ky), v0, s01);
            s10 = fma(Ry(0, ky), v1, s10);
          }
        }
        c00[a][kz] = s00;
        c01[a][kz] = s01;
        c10[a][kz] = s10;
      }
    }
    if constexpr (PENCIL) load_mq();
    // ---- geometry constants of this column from the cell's vertex coordinates (staged in
    // smem before the first sync; vertex v = a + 2b + 4c at X[3 v + i]):
    // J[:,0] = (1-tZ) e0y[0] + tZ e0y[1], J[:,1] = (1-tZ) e1x[0] + tZ e1x[1], J[:,2] = col2
    const double* X = xvs + el * L::XVS;
    const double tX = mv.xi[3 * tx], tY = mv.xi[3 * Q1 * ty + 1];
    double col2[3], e0y[2][3], e1x[2][3];
#pragma unroll
    for (int i = 0; i < 3; ++i) {
      col2[i] = (1 - tX) * (1 - tY) * (X[12 + i] - X[i]) + tX * (1 - tY) * (X[15 + i] - X[3 + i]) +
                (1 - tX) * tY * (X[18 + i] - X[6 + i]) + tX * tY * (X[21 + i] - X[9 + i]);
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        e0y[c][i] = (1 - tY) * (X[3 * (1 + 4 * c) + i] - X[3 * (4 * c) + i]) +
                    tY * (X[3 * (3 + 4 * c) + i] - X[3 * (2 + 4 * c) + i]);
        e1x[c][i] = (1 - tX) * (X[3 * (2 + 4 * c) + i] - X[3 * (4 * c) + i]) +
                    tX * (X[3 * (3 + 4 * c) + i] - X[3 * (1 + 4 * c) + i]);
      }
    }
    // ---- stage z (registers) + pointwise flux + z^T (registers)
    A Hv[D][N1], Hx[D][N1], Hy[D][N1];
#pragma unroll
    for (int a = 0; a < D; ++a)
#pragma unroll
      for (int kz = 0; kz < N1; ++kz) Hv[a][kz] = Hx[a][kz] = Hy[a][kz] = 0.0;
#pragma unroll
    for (int qz = 0; qz < Q1; ++qz) {
      double uq[D], gr[D][3];
#pragma unroll
      for (int a = 0; a < D; ++a) {
        A su = A(0), sx = A(0), sy = A(0), sz = A(0);
#pragma unroll
        for (int kz = 0; kz < N1; ++kz) {
          su = fma(B(0, qz, kz), c00[a][kz], su);
          if (GRAD) {
            sz = fma(B(1, qz, kz), c00[a][kz], sz);
            sy = fma(B(0, qz, kz), c01[a][kz], sy);
            sx = fma(B(0, qz, kz), c10[a][kz], sx);
          }
        }
        uq[a] = su;
        gr[a][0] = sx;
        gr[a][1] = sy;
        gr[a][2] = sz;
      }
      // geometry at (tx, ty, qz)
      const double tZ = mv.xi[3 * Q2 * qz + 2];
      double J[3][3];
#pragma unroll
      for (int i = 0; i < 3; ++i) {
        J[i][0] = (1 - tZ) * e0y[0][i] + tZ * e0y[1][i];
        J[i][1] = (1 - tZ) * e1x[0][i] + tZ * e1x[1][i];
        J[i][2] = col2[i];
      }
      const double c00g = J[1][1] * J[2][2] - J[1][2] * J[2][1];
      const double c01g = J[1][2] * J[2][0] - J[1][0] * J[2][2];
      const double c02g = J[1][0] * J[2][1] - J[1][1] * J[2][0];
      const double c10g = J[0][2] * J[2][1] - J[0][1] * J[2][2];
      const double c11g = J[0][0] * J[2][2] - J[0][2] * J[2][0];
      const double c12g = J[0][1] * J[2][0] - J[0][0] * J[2][1];
      const double c20g = J[0][1] * J[1][2] - J[0][2] * J[1][1];
      const double c21g = J[0][2] * J[1][0] - J[0][0] * J[1][2];
      const double c22g = J[0][0] * J[1][1] - J[0][1] * J[1][0];
      const double det = J[0][0] * c00g + J[0][1] * c01g + J[0][2] * c02g;
      if constexpr (SCALARF) {
        // scalar forms in cofactor form (as k_residual_t3): with t = C g (C the cofactors,
        // t = det grad u), F = detw J^-1 kappa grad u = (w kappa / det) C^T t and
        // F0 = w det rho u -- no J^-1, and 1/det by rcp.approx + two Newton steps (~1 ulp)
        const int q = tx + Q1 * ty + Q2 * qz;
        const double w = mv.w[q];
        double F0d = 0.0, Fxd = 0.0, Fyd = 0.0, Fzd = 0.0;
        if (valid) {
          if constexpr (VAL) F0d = w * det * mq[qz].a * uq[0];
          if constexpr (GRAD) {
            const double kap = FORM == FE_FORM_MASS_DIFFUSION ? mq[qz].b : mq[qz].a;
            const double g0 = gr[0][0], g1 = gr[0][1], g2 = gr[0][2];
            const double t0 = c00g * g0 + c01g * g1 + c02g * g2;
            const double t1 = c10g * g0 + c11g * g1 + c12g * g2;
            const double t2 = c20g * g0 + c21g * g1 + c22g * g2;
            const double sc = w * kap * rcp_nr(det);
            Fxd = sc * (c00g * t0 + c10g * t1 + c20g * t2);
            Fyd = sc * (c01g * t0 + c11g * t1 + c21g * t2);
            Fzd = sc * (c02g * t0 + c12g * t1 + c22g * t2);
          }
        }
        const A F0 = (A)F0d, Fx = (A)Fxd, Fy = (A)Fyd, Fz = (A)Fzd;
#pragma unroll
        for (int kz = 0; kz < N1; ++kz) {
          A hv = A(0);
          if (VAL) hv = B(0, qz, kz) * F0;
          if (BGRAD) {
            hv = fma(B(1, qz, kz), Fz, hv);
            Hx[0][kz] = fma(B(0, qz, kz), Fx, Hx[0][kz]);
            Hy[0][kz] = fma(B(0, qz, kz), Fy, Hy[0][kz]);
          }
          Hv[0][kz] += hv;
        }
        continue;
      }
      if constexpr (COFV) {
        // elasticity / convective: the flux is linear in grad u, so it is evaluated at
        // t = det grad u (t[a][j] = sum_m C[j][m] g[a][m], C the cofactors) and scaled back:
        // F1[a][m] = (w / det) sum_j C[j][m] f1(t)[a][j], F0[a] = w f0(t)[a] -- no J^-1
        const int q = tx + Q1 * ty + Q2 * qz;
        const double w = mv.w[q];
        const double C[3][3] = {{c00g, c01g, c02g}, {c10g, c11g, c12g}, {c20g, c21g, c22g}};
        double tg[D][3];
#pragma unroll
        for (int a = 0; a < D; ++a)
#pragma unroll
          for (int j = 0; j < 3; ++j) tg[a][j] = C[j][0] * gr[a][0] + C[j][1] * gr[a][1] + C[j][2] * gr[a][2];
        double f0[D], f1[D][3];
        if (valid) {
          qp_flux_m<FORM, T>(uq, tg, mq[qz], mat_kind, f0, f1);
        } else {
#pragma unroll
          for (int a = 0; a < D; ++a) f0[a] = f1[a][0] = f1[a][1] = f1[a][2] = 0.0;
        }
        const double sw = BGRAD ? w * rcp_nr(det) : 0.0;
#pragma unroll
        for (int a = 0; a < D; ++a) {
          const A F0 = (A)(w * f0[a]);
          A Fx = A(0), Fy = A(0), Fz = A(0);
          if (BGRAD) {
            Fx = (A)(sw * (C[0][0] * f1[a][0] + C[1][0] * f1[a][1] + C[2][0] * f1[a][2]));
            Fy = (A)(sw * (C[0][1] * f1[a][0] + C[1][1] * f1[a][1] + C[2][1] * f1[a][2]));
            Fz = (A)(sw * (C[0][2] * f1[a][0] + C[1][2] * f1[a][1] + C[2][2] * f1[a][2]));
          }
#pragma unroll
          for (int kz = 0; kz < N1; ++kz) {
            A hv = A(0);
            if (VAL) hv = B(0, qz, kz) * F0;
            if (BGRAD) {
              hv = fma(B(1, qz, kz), Fz, hv);
              Hx[a][kz] = fma(B(0, qz, kz), Fx, Hx[a][kz]);
              Hy[a][kz] = fma(B(0, qz, kz), Fy, Hy[a][kz]);
            }
            Hv[a][kz] += hv;
          }
        }
        continue;
      }
      const double id = rcp_nr(det);
      // Jinv[m][j] = cof[j][m] / det
      const double Ji[9] = {c00g * id, c10g * id, c20g * id, c01g * id, c11g * id,
                            c21g * id, c02g * id, c12g * id, c22g * id};
      const int q = tx + Q1 * ty + Q2 * qz;
      const double dw = mv.w[q] * det;
      double gu[D][3];
#pragma unroll
      for (int a = 0; a < D; ++a)
#pragma unroll
        for (int j = 0; j < 3; ++j) gu[a][j] = gr[a][0] * Ji[j] + gr[a][1] * Ji[3 + j] + gr[a][2] * Ji[6 + j];
      double f0[D], f1[D][3];
      if (valid) {
        qp_flux_m<FORM, T>(uq, gu, mq[qz], mat_kind, f0, f1);
      } else {
#pragma unroll
        for (int a = 0; a < D; ++a) f0[a] = f1[a][0] = f1[a][1] = f1[a][2] = 0.0;
      }
      // pull back and test along z
#pragma unroll
      for (int a = 0; a < D; ++a) {
        const A F0 = (A)(dw * f0[a]);
        const A Fx = (A)(dw * (Ji[0] * f1[a][0] + Ji[1] * f1[a][1] + Ji[2] * f1[a][2]));
        const A Fy = (A)(dw * (Ji[3] * f1[a][0] + Ji[4] * f1[a][1] + Ji[5] * f1[a][2]));
        const A Fz = (A)(dw * (Ji[6] * f1[a][0] + Ji[7] * f1[a][1] + Ji[8] * f1[a][2]));
#pragma unroll
        for (int kz = 0; kz < N1; ++kz) {
          A hv = A(0);
          if (VAL) hv = B(0, qz, kz) * F0;
          if (BGRAD) {
            hv = fma(B(1, qz, kz), Fz, hv);
            Hx[a][kz] = fma(B(0, qz, kz), Fx, Hx[a][kz]);
            Hy[a][kz] = fma(B(0, qz, kz), Fy, Hy[a][kz]);
          }
          Hv[a][kz] += hv;
        }
      }
    }
    double ev = 0.0;  // eval mode: sum_k u_k r_k(u) of this column
    if constexpr (PENCIL) {
      // ---- H (z-column) into buffer A (layout YZ); A was last read by stage y (before a barrier)
      if (active) {
#pragma unroll
        for (int kz = 0; kz < N1; ++kz) {
          const int o = oYZ(tx, ty, kz);
          XaYZ[o] = (T)Hv[0][kz];
          if (BGRAD) {
            XaYZ[L::PTS + o] = (T)Hx[0][kz];
            XaYZ[2 * L::PTS + o] = (T)Hy[0][kz];
          }
        }
      }
      __syncthreads();
      // ---- y^T on the y-pencil (x, kz) = (tx, ty): qy -> ky, into buffer B (layout XY)
      if (active) {
        A hv[Q1], hx[Q1], hy[Q1];
#pragma unroll
        for (int qy = 0; qy < Q1; ++qy) {
          const int o = oYZ(tx, qy, ty);
          hv[qy] = (A)XaYZ[o];
          hx[qy] = BGRAD ? (A)XaYZ[L::PTS + o] : A(0);
          hy[qy] = BGRAD ? (A)XaYZ[2 * L::PTS + o] : A(0);
        }
#pragma unroll
        for (int ky = 0; ky < N1; ++ky) {
          A sv = A(0), sx = A(0);
#pragma unroll
          for (int qy = 0; qy < Q1; ++qy) {
            sv = fma(B(0, qy, ky), hv[qy], sv);
            if (BGRAD) {
              sv = fma(B(1, qy, ky), hy[qy], sv);
              sx = fma(B(0, qy, ky), hx[qy], sx);
            }
          }
          const int o = oXY(tx, ky, ty);
          XbXY[o] = (T)sv;
          if (BGRAD) XbXY[L::PTSXY + o] = (T)sx;
        }
      }
      __syncthreads();
      // ---- x^T on the x-pencil (ky, kz) = (tx, ty): qx -> kx, scatter
      if (valid) {
        A iv[Q1], ix[Q1];
#pragma unroll
        for (int qx = 0; qx < Q1; ++qx) {
          const int o = oXY(qx, tx, ty);
          iv[qx] = (A)XbXY[o];
          ix[qx] = BGRAD ? (A)XbXY[L::PTSXY + o] : A(0);
        }
#pragma unroll
        for (int kx = 0; kx < N1; ++kx) {
          A sr = A(0);
#pragma unroll
          for (int qx = 0; qx < Q1; ++qx) {
            sr = fma(B(0, qx, kx), iv[qx], sr);
            if (BGRAD) sr = fma(B(1, qx, kx), ix[qx], sr);
          }
          const T v = (T)sr;
          const int k = kx + N1 * tx + N1 * N1 * ty;
          if (r_elem) r_elem[(e - e0) * (int64_t)NB + k] = v;
          if (r_global) atomicAdd(r_global + (int64_t)dcol[kx], v);
          if constexpr (PEER) peer_scatter<D>(pw, dcol[kx], 0, (double)v);
          if (eval_out) ev = fma((double)sr, (double)u[dcol[kx]], ev);  // u re-read: uc is dead after stage x
        }
      }
    } else {
    __syncthreads();  // everyone is done reading Xe (stage y)
    // ---- y^T: contract qy -> ky
    if (active) {
#pragma unroll
      for (int a = 0; a < D; ++a)
#pragma unroll
        for (int kz = 0; kz < N1; ++kz) {
          Xe[(a * 3 + 0) * NQ + kz * Q2 + ty * Q1 + tx] = (T)Hv[a][kz];
          if (BGRAD) {
            Xe[(a * 3 + 1) * NQ + kz * Q2 + ty * Q1 + tx] = (T)Hx[a][kz];
            Xe[(a * 3 + 2) * NQ + kz * Q2 + ty * Q1 + tx] = (T)Hy[a][kz];
          }
        }
    }
    __syncthreads();
    A Iv[D][N1], Ix[D][N1];  // [kz] at (qx = tx, ky = ty)
#pragma unroll
    for (int a = 0; a < D; ++a)
#pragma unroll
      for (int kz = 0; kz < N1; ++kz) {
        A sv = A(0), sx = A(0);
#pragma unroll
        for (int qy = 0; qy < Q1; ++qy) {
          const int o = kz * Q2 + qy * Q1 + tx;
          const A hv = active ? (A)Xe[(a * 3 + 0) * NQ + o] : A(0);
          sv = fma(Cy(0, qy), hv, sv);
          if (BGRAD) {
            sv = fma(Cy(1, qy), active ? (A)Xe[(a * 3 + 2) * NQ + o] : A(0), sv);
            sx = fma(Cy(0, qy), active ? (A)Xe[(a * 3 + 1) * NQ + o] : A(0), sx);
          }
        }
        Iv[a][kz] = sv;
        Ix[a][kz] = sx;
      }
    __syncthreads();
    // ---- x^T: contract qx -> kx
    if (active) {
#pragma unroll
      for (int a = 0; a < D; ++a)
#pragma unroll
        for (int kz = 0; kz < N1; ++kz) {
          Xe[(a * 3 + 0) * NQ + kz * Q2 + ty * Q1 + tx] = (T)Iv[a][kz];
          if (BGRAD) Xe[(a * 3 + 1) * NQ + kz * Q2 + ty * Q1 + tx] = (T)Ix[a][kz];
        }
    }
    __syncthreads();
    if (valid) {
#pragma unroll
      for (int a = 0; a < D; ++a)
#pragma unroll
        for (int kz = 0; kz < N1; ++kz) {
          A s = A(0);
#pragma unroll
          for (int qx = 0; qx < Q1; ++qx) {
            const int o = kz * Q2 + ty * Q1 + qx;
            s = fma(Cx(0, qx), (A)Xe[(a * 3 + 0) * NQ + o], s);
            if (BGRAD) s = fma(Cx(1, qx), (A)Xe[(a * 3 + 1) * NQ + o], s);
          }
          const T v = (T)s;
          const int k = tx + N1 * ty + N1 * N1 * kz;
          if (r_elem) r_elem[(e - e0) * (int64_t)(D * NB) + a * NB + k] = v;
          if (r_global) atomicAdd(r_global + (int64_t)dcol[kz] * D + a, v);
          if constexpr (PEER) peer_scatter<D>(pw, dcol[kz], a, (double)v);
          if (eval_out) ev = fma((double)s, (double)uc[a][kz], ev);
        }
    }
    }
    if (eval_out) {
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) ev += __shfl_xor_sync(0xffffffffu, ev, o);
      if ((tid & 31) == 0 && ev != 0.0) atomicAdd(eval_out, ev);
    }
    __syncthreads();
  }
#undef B
#undef Rx
#undef Ry
#undef Cx
#undef Cy
}

template <int P, int FORM, typename T>
static cudaError_t launch_rsf_t(const fe_mesh* mh, MatArgs mat, const T* u, int64_t e0, int64_t e1,
                                T* r_elem, T* r_global, double* eval_out, cudaStream_t st) {
  using L = RSF<P, FORM, T>;
  const PeerWin pw = g_peer;
  auto kern = k_residual_sf<P, FORM, T>;
  if constexpr (sizeof(T) == 8) {
    if (pw.n > 0) kern = k_residual_sf<P, FORM, T, true>;
  }
  const LaunchFacts lf = launch_facts((const void*)kern, L::THREADS, L::BYTES);
  if (lf.err != cudaSuccess) return lf.err;
  const int nsm = lf.nsm, per_sm = lf.per_sm;
  const int64_t nbatch = (e1 - e0 + L::EB - 1) / L::EB;
  int grid = (int)((nbatch < (int64_t)nsm * per_sm) ? nbatch : (int64_t)nsm * per_sm);
  grid = grid_cap(grid);
  if (grid <= 0) return cudaSuccess;
  kern<<<grid, L::THREADS, L::BYTES, st>>>(view_of(mh), mat.kind, (const T*)mat.a, (const T*)mat.b,
                                           u, e0, e1, r_elem, r_global, eval_out, pw);
  count_launch();
  return cudaGetLastError();
}

template <int P, typename T>
static cudaError_t rsf_form(const fe_mesh* mh, int form, MatArgs mat, const T* u, int64_t e0,
                            int64_t e1, T* re, T* rg, double* ev, cudaStream_t st) {
  switch (form) {
    case FE_FORM_DIFFUSION: return launch_rsf_t<P, FE_FORM_DIFFUSION, T>(mh, mat, u, e0, e1, re, rg, ev, st);
    case FE_FORM_MASS: return launch_rsf_t<P, FE_FORM_MASS, T>(mh, mat, u, e0, e1, re, rg, ev, st);
    case FE_FORM_MASS_DIFFUSION: return launch_rsf_t<P, FE_FORM_MASS_DIFFUSION, T>(mh, mat, u, e0, e1, re, rg, ev, st);
    default: break;
  }
  if constexpr (sizeof(T) == 8) {
    switch (form) {
      case FE_FORM_VECTOR_MASS: return launch_rsf_t<P, FE_FORM_VECTOR_MASS, T>(mh, mat, u, e0, e1, re, rg, ev, st);
      case FE_FORM_ELASTICITY: return launch_rsf_t<P, FE_FORM_ELASTICITY, T>(mh, mat, u, e0, e1, re, rg, ev, st);
      case FE_FORM_CONVECTIVE: return launch_rsf_t<P, FE_FORM_CONVECTIVE, T>(mh, mat, u, e0, e1, re, rg, ev, st);
      case FE_FORM_WEIGHTED_DOT: return launch_rsf_t<P, FE_FORM_WEIGHTED_DOT, T>(mh, mat, u, e0, e1, re, rg, ev, st);
      case FE_FORM_DIVERGENCE: return launch_rsf_t<P, FE_FORM_DIVERGENCE, T>(mh, mat, u, e0, e1, re, rg, ev, st);
      default: break;
    }
  }
  return cudaErrorNotSupported;
}

template <typename T>
cudaError_t launch_residual_sf(const fe_mesh* mh, int form, MatArgs mat, const T* u, int64_t e0,
                               int64_t e1, T* re, T* rg, cudaStream_t st, double* ev) {
  if (mh->q1d != mh->order + 1) return cudaErrorNotSupported;
  switch (mh->order) {
    case 1: return rsf_form<1, T>(mh, form, mat, u, e0, e1, re, rg, ev, st);
    case 2: return rsf_form<2, T>(mh, form, mat, u, e0, e1, re, rg, ev, st);
    case 3: return rsf_form<3, T>(mh, form, mat, u, e0, e1, re, rg, ev, st);
    case 4: return rsf_form<4, T>(mh, form, mat, u, e0, e1, re, rg, ev, st);
  }
  return cudaErrorNotSupported;
}

template cudaError_t launch_residual_sf<double>(const fe_mesh*, int, MatArgs, const double*, int64_t,
                                                int64_t, double*, double*, cudaStream_t, double*);
template cudaError_t launch_residual_sf<float>(const fe_mesh*, int, MatArgs, const float*, int64_t,
                                               int64_t, float*, float*, cudaStream_t, double*);

}  // namespace feb200
