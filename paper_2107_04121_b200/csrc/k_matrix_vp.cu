// Warp-specialised, pipelined, sum-factorised element matrices for the vector forms
// (isotropic elasticity, convective Newton tangent) -- Alg. 2 with
// the integrands of 'cq,cqje,rjI,cqIK,cqlf,slK->cresf' and Eq. fe4.
//
// The 3 x 3 block structure K_ab[k][l] = sum_q sum_{(m,n)} W^{ab}_{mn}(q) D^m_k(q) D^n_l(q)
// (D^m_k = prod_d B^{[m == d]}[q_d][k_d], m = 3 the value) is processed one block ("item")
// at a time through the same three-role pipeline as the scalar kernel (k_matrix_sf.cu):
//   L (1 warp)    gathers vertex coordinates, material (lambda, mu per cell or per qp)
//                 or the state u_e of the convective tangent into a 2-deep ring;
//   G (NG warps)  phase 1 per batch: per-qp geometry J^-1, detw
//                 and the per-qp data of the form (lambda, mu | u, grad u, J^-1 u);
//                 phase 2 per item: the block's pair weights W^{ab}_{mn} and stage z
//                 -> T1 ring slot (3 deep, mbarrier full/empty handshake with X);
//   X (NX warps)  per item: stages y and x of one (z pair, y pair) per thread -> K_e
//                 staged in shared memory; one TMA bulk store per batch.
// Items (blocks) per form:
//   elasticity  (0,0) (1,1) (2,2): symmetric, 6 unique pairs m <= n,
//               W^{aa}_{mn} = detw ((lam + mu) Ji[m][a] Ji[n][a] + mu (Ji Ji^T)_{mn});
//               (0,1) (0,2) (1,2): 9 pairs, W^{ab}_{mn} = detw (lam Ji[m][a] Ji[n][b] +
//               mu Ji[m][b] Ji[n][a]), mirrored into K_ba = K_ab^T.  (Psg contracted
//               analytically, reading 7.)
//   convective  (a,a): pairs (3,n) with detw (Ji u)_n (advection) and (3,3) with detw du_a/dx_a;
//               (a,b), a != b: pair (3,3) with detw du_a/dx_b (reaction; symmetric block).
#ifndef FEB200_VP_EVF
#define FEB200_VP_EVF 1  // L2 evict_first hint on the K bulk stores (C5t 3.66 -> 3.56 ms, C3 equal)
#endif
#include "fe_const.cuh"
#include "fe_device.cuh"
#include "fe_internal.h"
#include "vp_tasks.h"
#include "vp_yb3_tasks.h"
#ifndef FEB200_VP_L2PF
#define FEB200_VP_L2PF 1
#endif
#include <cstdlib>
#include <cstring>
#include <type_traits>

#ifndef FEB200_VP_E
#define FEB200_VP_E 2
#endif
#ifndef FEB200_VP_TASKMAP
#define FEB200_VP_TASKMAP 1
#endif
#ifndef FEB200_VP_GMAP
#define FEB200_VP_GMAP 1
#endif
// per-form role sizes (elasticity / convective): X groups, G pair groups, T1 ring depth.
// Measured (B200, C3 / C5t): 4 G groups for elasticity (1.96 vs 2.10 ms with 3; 17 warps at
// 96 registers), 2 for the convective tangent (3.69 vs 3.71 ms).  An X role with register
// reuse (one thread per (cell, z pair, iy) over the three jy: a third of the T1 loads) was
// 20-70 % slower in every X / G split tried -- the role becomes latency-bound.
#ifndef FEB200_VP_XG_EL
#define FEB200_VP_XG_EL (FEB200_VP_E == 1 ? 1 : 2)
#endif
// YB3: the register-blocked X role of the scalar kernel (k_matrix_sf.cu) for the elasticity
// items -- measured slower here (B200, C3 matrix: 2.29 ms natural lane map, 2.14 ms with the
// annealed map of tools/gen_vp_yb3_tasks.c, vs 1.86 ms): the X shared-memory wavefronts halve
// (data pipe 78 % -> 43 %) but with 6 X warps at 168 registers the role turns latency-bound and
// waits on the single K staging buffer's store (kfree); off by default, kept for A/B
#ifndef FEB200_VP_YB3
#define FEB200_VP_YB3 0
#endif
#ifndef FEB200_VP_NOSTORE
#define FEB200_VP_NOSTORE 0
#endif
#ifndef FEB200_VP_YB3MAP
#define FEB200_VP_YB3MAP 1
#endif
#ifndef FEB200_VP_XG_CV
#define FEB200_VP_XG_CV (FEB200_VP_E == 1 ? 1 : 2)
#endif
#ifndef FEB200_VP_GH_EL
#define FEB200_VP_GH_EL 4
#endif
#ifndef FEB200_VP_GH_ELD
#define FEB200_VP_GH_ELD 3
#endif
#ifndef FEB200_VP_GH_CV
#define FEB200_VP_GH_CV 2
#endif
#ifndef FEB200_VP_S_EL
#define FEB200_VP_S_EL 4
#endif
#ifndef FEB200_VP_S_CV
#define FEB200_VP_S_CV 4
#endif
// G split (warps of a dedicated phase-1 sub-role, 0 = one G role doing both phases): with a
// split, G1 warps compute the pair weights of batch it+1 into the second half of a double-
// buffered Wsm while the G2 warps run stage z of batch it.  Measured (B200): general D
// elasticity (C3d) 2.24 ms with 2 G1 warps vs 2.58 without (its phase 1 -- 36 D loads and the
// 9 blocks J^-T C J^-1 per qp -- stalled stage z; 2.20 with 3 stage-z groups instead of 4);
// convective tangent (C5t) 3.69 vs 3.75 with 1
// (2: 17 warps at 96 registers, 3.87); isotropic elasticity (C3) 1.873 with 1, 1.877 without,
// 1.96 with 2 or 3
#ifndef FEB200_VP_G1W_EL
#define FEB200_VP_G1W_EL 1
#endif
#ifndef FEB200_VP_G1W_ELD
#define FEB200_VP_G1W_ELD 2
#endif
#ifndef FEB200_VP_G1W_CV
#define FEB200_VP_G1W_CV 1
#endif

namespace feb200 {

namespace {
// c_zzv[p][az][bz][q][a][b] = B^az[q][a] B^bz[q][b]: stage-z (and stage-y) coefficients
__constant__ double c_zzv[4][2][2][4][4][4];

__device__ __forceinline__ uint32_t vp_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void vp_bar_init(uint64_t* bar, int count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(vp_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void vp_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(vp_u32(bar)) : "memory");
}
__device__ __forceinline__ void vp_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tWAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n\t}" ::"r"(vp_u32(bar)), "r"(parity) : "memory");
}
#ifdef FEB200_VP_PROF
__device__ unsigned long long g_vp_prof[16];
#define VP_T(k, stmt)                                   \
  do {                                                  \
    const long long t0_ = clock64();                    \
    stmt;                                               \
    prof_[k] += (unsigned long long)(clock64() - t0_);  \
  } while (0)
#else
#define VP_T(k, stmt) stmt
#endif
__device__ __forceinline__ void vp_named_bar(int id, int nthreads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}
// unique pair u -> (m, n), m <= n; index 6 is the value-value pair (3,3)
__host__ __device__ constexpr int vp_voigt(int a, int j) {
  return a == j ? a : (a + j == 1 ? 3 : (a + j == 2 ? 4 : 5));
}
__host__ __device__ constexpr int vp_um(int u) { return (0x3211000 >> (4 * u)) & 0xF; }
__host__ __device__ constexpr int vp_un(int u) { return (0x3221210 >> (4 * u)) & 0xF; }
// YB3 symmetric items: on a diagonal z pair the y pairs iy > jy are not stored (the (jy, iy)
// task's mirror writes them)
__device__ __forceinline__ bool zdiag_skip(bool sym, int iz, int jz, int iy, int jy) {
  return sym && iz == jz && iy > jy;
}
template <int I, int N, class F>
__device__ __forceinline__ void vp_static_for(F&& f) {
  if constexpr (I < N) {
    f(std::integral_constant<int, I>{});
    vp_static_for<I + 1, N>(f);
  }
}
}  // namespace

cudaError_t upload_const_tables_matrix_vp(int order, const double* b1, const double* d1,
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
  e = cudaMemcpyToSymbolAsync(c_zzv, h, sizeof(h), sizeof(h) * order, cudaMemcpyHostToDevice, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  return e;
}

// ---------------------------------------------------------------------------------------
// Item (block) tables.  SYM items list unique pairs (m <= n) and are consumed with the
// transposition trick of the scalar kernel; FULL items list ordered pairs.
template <int FORM>
struct VItems;

template <>
struct VItems<FE_FORM_ELASTICITY> {
  static constexpr int NITEM = 6, NPMAX = 9, QD = 12;
  __host__ __device__ static constexpr int a(int i) { return i < 3 ? i : (i == 5 ? 1 : 0); }
  __host__ __device__ static constexpr int b(int i) { return i < 3 ? i : (i == 3 ? 1 : 2); }
  __host__ __device__ static constexpr bool sym(int i) { return i < 3; }
  __host__ __device__ static constexpr bool mirror(int i) { return i >= 3; }
  __host__ __device__ static constexpr int np(int i) { return i < 3 ? 6 : 9; }
  __host__ __device__ static constexpr int pm(int i, int p) { return i < 3 ? vp_um(p) : p / 3; }
  __host__ __device__ static constexpr int pn(int i, int p) { return i < 3 ? vp_un(p) : p % 3; }
  __host__ __device__ static constexpr int pbase(int i) { return i < 3 ? 6 * i : 18 + 9 * (i - 3); }
  static constexpr int NWP = 45;
};

template <>
struct VItems<FE_FORM_CONVECTIVE> {
  // item 0: the three diagonal blocks together -- the advection part A (pairs (3,n), n < 3,
  // weight detw (Ji u)_n) is the same for every (a,a) and is contracted once, plus the three
  // reaction parts R_aa (pair (3,3), weight detw du_a/dx_a); K_aa = A + R_aa.
  // items 1..6: off-diagonal reaction blocks (0,1) (0,2) (1,0) (1,2) (2,0) (2,1), pair (3,3)
  // with weight detw du_a/dx_b (symmetric 27 x 27 blocks).
  static constexpr int NITEM = 7, NPMAX = 6, QD = 22;
  __host__ __device__ static constexpr int a(int i) { return i < 1 ? 0 : (i - 1) / 2; }
  __host__ __device__ static constexpr int b(int i) {
    return i < 1 ? 0 : ((i - 1) % 2 == 0 ? ((i - 1) / 2 == 0 ? 1 : 0) : ((i - 1) / 2 == 2 ? 1 : 2));
  }
  __host__ __device__ static constexpr bool sym(int i) { return i >= 1; }
  __host__ __device__ static constexpr bool mirror(int) { return false; }
  __host__ __device__ static constexpr int np(int i) { return i < 1 ? 6 : 1; }
  __host__ __device__ static constexpr int pm(int, int) { return 3; }
  __host__ __device__ static constexpr int pn(int i, int p) { return (i < 1 && p < 3) ? p : 3; }
  __host__ __device__ static constexpr int pbase(int i) { return i < 1 ? 0 : 6 + (i - 1); }
  static constexpr int NWP = 12;
};

template <int P, int FORM, bool FD>
struct VPL {
  using IT = VItems<FORM>;
  static constexpr int N1 = P + 1, Q1 = P + 1, NB = N1 * N1 * N1, NQ = Q1 * Q1 * Q1, Q2 = Q1 * Q1;
  static constexpr int NDOF = 3 * NB;
  static constexpr bool EL = FORM == FE_FORM_ELASTICITY;
  static constexpr int E = FEB200_VP_E;                  // cells per batch
  static constexpr int GH = EL ? (FD ? FEB200_VP_GH_ELD : FEB200_VP_GH_EL) : FEB200_VP_GH_CV;  // G pair groups
  static constexpr int QQP = (Q2 + 1) / 2 * 2;
  static constexpr int NWP = IT::NWP;                    // pair weights per qp (all items)
  static constexpr int G1T = E * NQ;                     // phase-1 tasks (per qp)
  static constexpr int G2W = (E * Q2 + 31) / 32;         // warps per pair group (warp-uniform group)
  // phase-1 warps (0: no split); FD: the general-D (FE_MAT_FULL_D) elasticity instantiation
  static constexpr int NG1 = EL ? (FD ? FEB200_VP_G1W_ELD : FEB200_VP_G1W_EL) : FEB200_VP_G1W_CV;
  static constexpr bool SPLIT = NG1 > 0;
  static constexpr int NG = SPLIT ? NG1 + GH * G2W
                                  : (((G1T + 31) / 32 > GH * G2W) ? (G1T + 31) / 32 : GH * G2W);
  static constexpr int NG2 = SPLIT ? NG - NG1 : NG;      // warps that run stage z
  static constexpr int NFULL = N1 * N1 * N1 * N1;        // (z pair, y pair) tasks, ordered
  static constexpr int NSYM = N1 * N1 * (N1 * (N1 - 1) / 2) + N1 * (N1 * (N1 + 1) / 2);
  // YB3 (elasticity, E = 2): register-blocked X -- one thread per (z pair, iy) over jy = 0..2
  // (a third of the T1 loads per output), every lane keeping one iy for all items so that its
  // y-pair factors stay in registers; 3 X groups of 2 warps, each group one symmetric and one
  // full item per batch
  static constexpr bool YB3 = FEB200_VP_YB3 && EL && P == 2 && E == 2;
  static constexpr int XG = YB3 ? 3 : (EL ? FEB200_VP_XG_EL : FEB200_VP_XG_CV);  // X groups (alternate items)
  static constexpr int NXW = YB3 ? 2 : (E * NFULL + 31) / 32;  // warps per X group
  static constexpr int NX = XG * NXW;
  static constexpr int THREADS = 32 * (1 + NG + NX);
  static constexpr int S = EL ? FEB200_VP_S_EL : FEB200_VP_S_CV;  // T1 ring depth (items)
  static constexpr bool TASKMAP = FEB200_VP_TASKMAP && P == 2 && E == 2 && NXW == 6 && !YB3;
  static constexpr bool CONV = FORM == FE_FORM_CONVECTIVE;
  // L slot (doubles): coords [E][24], material a/b [E][NQ] | state [E][3][NB]
  static constexpr int LS_X = 0, LS_A = E * 24, LS_B = LS_A + E * NQ, LS_U = LS_B + E * NQ;
  static constexpr int LSLOT = CONV ? LS_A + E * 3 * NB : LS_B + E * NQ;
  static constexpr size_t KBYTES = size_t(E) * NDOF * NDOF * 8;
  static constexpr size_t T1SLOT = size_t(E) * IT::NPMAX * N1 * N1 * QQP * 8;
  static constexpr size_t OFF_K = 0;
  static constexpr size_t OFF_T1 = (OFF_K + KBYTES + 127) / 128 * 128;
  static constexpr size_t OFF_QD = OFF_T1 + S * T1SLOT;
  static constexpr size_t WSZ = size_t(E) * IT::NWP * NQ;  // doubles per Wsm buffer
  static constexpr size_t OFF_L = OFF_QD + (SPLIT ? 2 : 1) * WSZ * 8;
  static constexpr size_t OFF_IDX = OFF_L + 2 * size_t(LSLOT) * 8;       // [2][E][8 + NB] int32
  static constexpr size_t OFF_BAR = (OFF_IDX + 2 * size_t(E) * (8 + NB) * 4 + 15) / 16 * 16;
  static constexpr size_t BYTES = OFF_BAR + (10 + 2 * S) * 8;
  // E = 1: two CTAs per SM (each ~100 KB), so that one CTA's K store drains while the other
  // computes (the single K staging buffer of a CTA otherwise stalls X on kfree)
  static constexpr int MINB = E == 1 ? 2 : 1;
};

template <int P, int FORM, bool FD>
__global__ void __launch_bounds__(VPL<P, FORM, FD>::THREADS, VPL<P, FORM, FD>::MINB)
    k_matrix_vp(MeshView mv, int mat_kind, const double* __restrict__ ma, const double* __restrict__ mb,
                const double* __restrict__ state_u, int64_t e0, int64_t e1, double* __restrict__ K,
                int* __restrict__ nonsym) {
  // general D (FD): the kernel reads the upper triangle of each 6x6 block and sets *nonsym when
  // a block is not symmetric; the general 9-block kernel k_matrix_sfv, launched next and gated
  // on the flag, then recomputes K (reading 23)
  using L = VPL<P, FORM, FD>;
  using IT = typename L::IT;
  constexpr int N1 = L::N1, Q1 = L::Q1, NB = L::NB, NQ = L::NQ, Q2 = L::Q2, E = L::E, QQP = L::QQP;
  constexpr int NDOF = L::NDOF, NITEM = IT::NITEM, S = L::S, GH = L::GH;
  extern __shared__ __align__(128) unsigned char smv[];
  uint64_t* bars = reinterpret_cast<uint64_t*>(smv + L::OFF_BAR);
  uint64_t* fullL = bars + 0;   // [2]
  uint64_t* emptyL = bars + 2;  // [2]
  uint64_t* fullT = bars + 4;          // [S]
  uint64_t* emptyT = bars + 4 + L::S;  // [S]
  // K staging handshake (single buffer): every X thread arrives on kfull after its last K
  // write of a batch; the L warp then issues the TMA bulk store and arrives on kfree once the
  // store has read the buffer; X threads wait on kfree before their first K write of the next
  // batch (no CTA-wide barrier couples the two X groups or the store to the X warps)
  uint64_t* kfull = bars + 4 + 2 * L::S;
  uint64_t* kfree = bars + 5 + 2 * L::S;
  uint64_t* fullW = bars + 6 + 2 * L::S;   // [2] (G split only) G1 -> G2: Wsm buffer written
  uint64_t* emptyW = bars + 8 + 2 * L::S;  // [2] G2 -> G1: Wsm buffer read
  double* Kst = reinterpret_cast<double*>(smv + L::OFF_K);
  double* Wsm = reinterpret_cast<double*>(smv + L::OFF_QD);  // [E][NWP][NQ] pair weights
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int64_t nloc = e1 - e0;
  const int64_t nbatch = (nloc + E - 1) / E;
#ifdef FEB200_VP_PROF
  unsigned long long prof_[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  const long long tstart_ = clock64();
#endif
  if (tid == 0) {
    vp_bar_init(&fullL[0], 32);
    vp_bar_init(&fullL[1], 32);
    vp_bar_init(&emptyL[0], 32 * (L::SPLIT ? L::NG1 : L::NG));
    vp_bar_init(&emptyL[1], 32 * (L::SPLIT ? L::NG1 : L::NG));
    for (int b = 0; b < 2; ++b) {
      vp_bar_init(&fullW[b], 32 * (L::SPLIT ? L::NG1 : 1));
      vp_bar_init(&emptyW[b], 32 * L::NG2);
    }
    for (int s = 0; s < S; ++s) {
      vp_bar_init(&fullT[s], 32 * L::NG2);
      vp_bar_init(&emptyT[s], 32 * L::NXW);
    }
    vp_bar_init(kfull, 32 * L::NX);
    vp_bar_init(kfree, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
#define Bt(a, q, i) c_tab1d[P][a][q][i]
  auto batch_of = [&](int64_t j, int64_t& lb, int& ne) {
    const int64_t b = blockIdx.x + j * (int64_t)gridDim.x;
    lb = b * E;
    ne = b < nbatch ? (int)((nloc - lb) < E ? (nloc - lb) : E) : 0;
  };

  if (warp == 0) {
    // ======================= L: loader warp =======================
    int32_t* idxb = reinterpret_cast<int32_t*>(smv + L::OFF_IDX);  // [2][E][8 + NB]
    constexpr int IDXN = E * (8 + (L::CONV ? NB : 0));
    auto load_idx = [&](int64_t j) {
      int64_t lb;
      int ne;
      batch_of(j, lb, ne);
      if (ne <= 0) return;
      int32_t* ib = idxb + (j & 1) * E * (8 + NB);
      if (FEB200_VP_L2PF && !L::CONV && (FD || mat_kind == FE_MAT_FULL_D) && lane == 0) {  // D block of batch j -> L2
        const double* gD = ma + (e0 + lb) * NQ * 36;
        const uint32_t bD = (uint32_t)ne * NQ * 36u * 8u;
        if (((reinterpret_cast<uintptr_t>(gD) | bD) & 15u) == 0) l2_prefetch_bulk(gD, bD);
      }
      for (int i = lane; i < IDXN; i += 32) {
        const int c = i < E * 8 ? i / 8 : (i - E * 8) / NB;
        int v = 0;
        if (c < ne) v = i < E * 8 ? mv.conn[8 * (e0 + lb) + i] : mv.dof_conn[(e0 + lb) * NB + (i - E * 8)];
        ib[i] = v;
      }
    };
    constexpr int XPL = (E * 24 + 31) / 32;
    constexpr int MPL = L::CONV ? 0 : (E * NQ + 31) / 32;
    constexpr int UPL = L::CONV ? (E * 3 * NB + 31) / 32 : 0;
    // K store of batch j (after every X thread's last K write of it), then kfree
    auto store_batch = [&](int64_t j) {
      int64_t lbj;
      int nej;
      batch_of(j, lbj, nej);
      if (nej <= 0) return;
      VP_T(6, vp_wait(kfull, (uint32_t)(j & 1)));
      const uint32_t bytes = (uint32_t)((size_t)nej * NDOF * NDOF * 8);
      double* gdst = K + lbj * NDOF * NDOF;
      if (FEB200_VP_NOSTORE) {  // experiment: K is not stored (the cost of the store path)
      } else if (((reinterpret_cast<uintptr_t>(gdst) | bytes) & 15u) == 0) {
        if (lane == 0) {
          if (FEB200_VP_EVF) {
          uint64_t pol_;
          asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol_));
          asm volatile("cp.async.bulk.global.shared::cta.bulk_group.L2::cache_hint [%0], [%1], %2, %3;"
                       :: "l"(gdst), "r"(vp_u32(Kst)), "r"(bytes), "l"(pol_) : "memory");
        } else asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;"
                       :: "l"(gdst), "r"(vp_u32(Kst)), "r"(bytes) : "memory");
          asm volatile("cp.async.bulk.commit_group;" ::: "memory");
          asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
        }
      } else {
        for (int i = lane; i < nej * NDOF * NDOF; i += 32) gdst[i] = Kst[i];
      }
      __syncwarp();
      if (lane == 0) vp_arrive(kfree);
    };
    load_idx(0);
    __syncwarp();
    int64_t nit = 0;  // batches of this CTA
    for (int64_t it = 0;; ++it) {
      int64_t lb;
      int ne;
      batch_of(it, lb, ne);
      if (ne <= 0) {
        nit = it;
        break;
      }
      const int sl = (int)(it & 1);
      const int32_t* ib = idxb + sl * E * (8 + NB);
      double xr[XPL], mra[MPL > 0 ? MPL : 1], mrb[MPL > 0 ? MPL : 1], ur[UPL > 0 ? UPL : 1];
#pragma unroll
      for (int h = 0; h < XPL; ++h) {
        const int i = lane + 32 * h, c = i / 24, r = i - c * 24;
        xr[h] = (i < E * 24 && c < ne) ? mv.coords[3 * (int64_t)ib[c * 8 + r / 3] + r % 3] : 0.0;
      }
      if constexpr (!L::CONV) {
#pragma unroll
        for (int h = 0; h < MPL; ++h) {
          const int i = lane + 32 * h, c = i / NQ, q = i - c * NQ;
          double va = 0.0, vb = 0.0;
          if (i < E * NQ && c < ne && mat_kind != FE_MAT_FULL_D) {
            if (mat_kind == FE_MAT_PER_ELEM) {
              va = ma[e0 + lb + c];
              vb = mb[e0 + lb + c];
            } else {
              va = ma[(e0 + lb + c) * NQ + q];
              vb = mb[(e0 + lb + c) * NQ + q];
            }
          }
          mra[h] = va;
          mrb[h] = vb;
        }
      } else {
#pragma unroll
        for (int h = 0; h < UPL; ++h) {
          const int i = lane + 32 * h, c = i / (3 * NB), r = i - c * 3 * NB;
          const int a = r / NB, k = r - a * NB;
          ur[h] = (i < E * 3 * NB && c < ne) ? state_u[3 * (int64_t)ib[E * 8 + c * NB + k] + a] : 0.0;
        }
      }
      __syncwarp();
      load_idx(it + 1);  // other half of the index ring (read in iteration it - 1)
      if (it >= 2) store_batch(it - 2);  // overlaps the latency of the gathers above
      VP_T(1, vp_wait(&emptyL[sl], (uint32_t)(((it >> 1) & 1) ^ 1)));
      double* slot = reinterpret_cast<double*>(smv + L::OFF_L) + sl * L::LSLOT;
#pragma unroll
      for (int h = 0; h < XPL; ++h) {
        const int i = lane + 32 * h;
        if (i < E * 24) slot[L::LS_X + i] = xr[h];
      }
      if constexpr (!L::CONV) {
#pragma unroll
        for (int h = 0; h < MPL; ++h) {
          const int i = lane + 32 * h;
          if (i < E * NQ) {
            slot[L::LS_A + i] = mra[h];
            slot[L::LS_B + i] = mrb[h];
          }
        }
      } else {
#pragma unroll
        for (int h = 0; h < UPL; ++h) {
          const int i = lane + 32 * h;
          if (i < E * 3 * NB) slot[L::LS_A + i] = ur[h];
        }
      }
      __syncwarp();
      vp_arrive(&fullL[sl]);
    }
    if (nit >= 2) store_batch(nit - 2);
    if (nit >= 1) store_batch(nit - 1);
    if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  } else if (warp <= L::NG) {
    // ======================= G: per-qp data, pair weights, stage z =======================
    const int gtid = tid - 32;
    constexpr int NGT = 32 * L::NG;
    // G split: warps 1..NG1 run phase 1 only (G1), the rest phase 2 only (G2)
    const bool g1 = !L::SPLIT || warp <= L::NG1, g2 = !L::SPLIT || warp > L::NG1;
    constexpr int NGT1 = L::SPLIT ? 32 * L::NG1 : NGT;
    const int gtid2 = L::SPLIT ? gtid - 32 * L::NG1 : gtid;
    // phase-2 mapping: warp-uniform pair group h (pairs p with p % GH == h), column (el, qxy)
    const int h2 = gtid2 / (32 * L::G2W), r2 = gtid2 - h2 * (32 * L::G2W);
    // column of this lane.  E = 2: the second cell's columns whose T1 stores would share a bank
    // with the first cell's in half-warp 0 (per-cell T1 stride S mod 16: banks (S + qxy) mod 16
    // against 0..8) move to half-warp 1, behind idle lanes -- 2 instead of 3 wavefronts per store
    constexpr int S16 = (IT::NPMAX * N1 * N1 * QQP) % 16;
    constexpr int KOK = (S16 >= 9 && FEB200_VP_GMAP) ? 16 - S16 : Q2;  // second-cell columns in half-warp 0
    int col2 = r2;
    if (E == 2 && Q2 == 9 && KOK < Q2) col2 = r2 < Q2 + KOK ? r2 : (r2 < 16 ? -1 : r2 - 16 + Q2 + KOK);
    const int el2 = col2 >= 0 ? col2 / Q2 : 0, qxy = col2 >= 0 ? col2 - el2 * Q2 : 0;
    const int tx = qxy / Q1, ty = qxy - tx * Q1;  // T1's inner index is qx * Q1 + qy
    const bool act2 = h2 < GH && col2 >= 0 && col2 < E * Q2;
    int64_t gi = 0;  // global item counter (T1 ring position)
    for (int64_t it = 0;; ++it) {
      int64_t lb;
      int ne;
      batch_of(it, lb, ne);
      if (ne <= 0) break;
      const int sl = (int)(it & 1);
      const int wb = L::SPLIT ? (int)(it & 1) : 0;
      double* const Wb_ = Wsm + wb * L::WSZ;
      if (g1) {
      VP_T(2, vp_wait(&fullL[sl], (uint32_t)((it >> 1) & 1)));
      const double* slot = reinterpret_cast<const double*>(smv + L::OFF_L) + sl * L::LSLOT;
      // ---- phase 1: pair weights of the batch (Wsm is free once every G thread left phase 2 of
      // it-1, or -- G split -- once the G2 warps released this buffer after batch it-2)
      if constexpr (L::SPLIT) {
        VP_T(0, vp_wait(&emptyW[wb], (uint32_t)(((it >> 1) & 1) ^ 1)));
      } else {
        VP_T(0, vp_named_bar(1, NGT));
      }
      for (int t = gtid; t < L::G1T; t += NGT1) {
        const int el = t / NQ, q = t - el * NQ;
        const int qx = q % Q1, qy = (q / Q1) % Q1, qz = q / Q2;
        const double t0 = c_x1d[P][qx], t1 = c_x1d[P][qy], t2 = c_x1d[P][qz];
        const double* X = slot + L::LS_X + el * 24;
        double J[3][3];
#pragma unroll
        for (int i = 0; i < 3; ++i) {
          // edges: x at (b,c): X[1+2b+4c]-X[2b+4c]; y at (a,c): X[a+2+4c]-X[a+4c]; z at (a,b): X[a+2b+4]-X[a+2b]
          J[i][0] = (1 - t1) * (1 - t2) * (X[3 * 1 + i] - X[3 * 0 + i]) + t1 * (1 - t2) * (X[3 * 3 + i] - X[3 * 2 + i]) +
                    (1 - t1) * t2 * (X[3 * 5 + i] - X[3 * 4 + i]) + t1 * t2 * (X[3 * 7 + i] - X[3 * 6 + i]);
          J[i][1] = (1 - t0) * (1 - t2) * (X[3 * 2 + i] - X[3 * 0 + i]) + t0 * (1 - t2) * (X[3 * 3 + i] - X[3 * 1 + i]) +
                    (1 - t0) * t2 * (X[3 * 6 + i] - X[3 * 4 + i]) + t0 * t2 * (X[3 * 7 + i] - X[3 * 5 + i]);
          J[i][2] = (1 - t0) * (1 - t1) * (X[3 * 4 + i] - X[3 * 0 + i]) + t0 * (1 - t1) * (X[3 * 5 + i] - X[3 * 1 + i]) +
                    (1 - t0) * t1 * (X[3 * 6 + i] - X[3 * 2 + i]) + t0 * t1 * (X[3 * 7 + i] - X[3 * 3 + i]);
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
        const bool on = el < ne;
        const double id = on ? rcp_nr(det) : 0.0;
        // Ji[m][j] = cof[j][m] / det
        const double Ji[9] = {c00 * id, c10 * id, c20 * id, c01 * id, c11 * id, c21 * id, c02 * id, c12 * id, c22 * id};
        const double dw = on ? c_w1d[P][qx] * c_w1d[P][qy] * c_w1d[P][qz] * det : 0.0;
        // all pair weights W^{ab}_{mn}(q) of the batch, item-major: Wsm[el][PB(i) + p][q]
        double* Wq = Wb_ + el * L::NWP * NQ + q;
        // the isotropic elasticity instantiation keeps the (there unused) general-D branch:
        // without it ptxas allocated the isotropic path differently (1.93 vs 1.88 ms on C3)
        if (!L::CONV && (FD || mat_kind == FE_MAT_FULL_D)) {
          // general Voigt D, the upper triangle read (symmetry checked below, reading 23):
          // W^{ab}_{mn} = dw sum_{j,l} Ji[m][j] D[v(a,j)][v(b,l)] Ji[n][l]
          double Dm[36];
          const double* Dg = ma + ((e0 + lb + el) * NQ + q) * 36;
          if (on && (reinterpret_cast<uintptr_t>(Dg) & 31u) == 0) {  // nine 32-B loads
#pragma unroll
            for (int h = 0; h < 9; ++h) ld_nc_v4(Dg + 4 * h, Dm[4 * h], Dm[4 * h + 1], Dm[4 * h + 2], Dm[4 * h + 3]);
          } else {
#pragma unroll
            for (int i = 0; i < 36; ++i) Dm[i] = on ? __ldg(Dg + i) : 0.0;
          }
          if constexpr (FD) {
            // |D_IK - D_KI| > 8 eps max(|D_IK|, |D_KI|) (or NaN): not symmetric (a D formed as
            // A A^T in floating point may differ from its transpose in the last bits)
            bool ns = false;
#pragma unroll
            for (int I = 0; I < 6; ++I)
#pragma unroll
              for (int Kk = I + 1; Kk < 6; ++Kk) {
                const double a = Dm[6 * I + Kk], b = Dm[6 * Kk + I];
                ns |= !(fabs(a - b) <= 8.0 * 2.220446049250313e-16 * fmax(fabs(a), fabs(b)));
              }
            if (ns && nonsym != nullptr) *nonsym = 1;
          }
          auto Dv = [&](int a, int j, int b, int l) {
            const int I = vp_voigt(a, j), Kk = vp_voigt(b, l);
            return I <= Kk ? Dm[6 * I + Kk] : Dm[6 * Kk + I];
          };
          auto wblk = [&](int a, int b, double (&Wb)[3][3]) {
            double R[3][3];  // R[j][n] = sum_l C_{ajbl} Ji[n][l]
#pragma unroll
            for (int j = 0; j < 3; ++j)
#pragma unroll
              for (int n = 0; n < 3; ++n)
                R[j][n] = Dv(a, j, b, 0) * Ji[3 * n] + Dv(a, j, b, 1) * Ji[3 * n + 1] + Dv(a, j, b, 2) * Ji[3 * n + 2];
#pragma unroll
            for (int m = 0; m < 3; ++m)
#pragma unroll
              for (int n = 0; n < 3; ++n)
                Wb[m][n] = dw * (Ji[3 * m] * R[0][n] + Ji[3 * m + 1] * R[1][n] + Ji[3 * m + 2] * R[2][n]);
          };
#pragma unroll
          for (int a2 = 0; a2 < 3; ++a2) {
            double Wb[3][3];
            wblk(a2, a2, Wb);
#pragma unroll
            for (int u = 0; u < 6; ++u) Wq[(6 * a2 + u) * NQ] = Wb[vp_um(u)][vp_un(u)];
          }
#pragma unroll
          for (int ob = 0; ob < 3; ++ob) {
            const int a2 = ob == 2 ? 1 : 0, b2 = ob == 0 ? 1 : 2;
            double Wb[3][3];
            wblk(a2, b2, Wb);
#pragma unroll
            for (int pp = 0; pp < 9; ++pp) Wq[(18 + 9 * ob + pp) * NQ] = Wb[pp / 3][pp % 3];
          }
        } else if constexpr (!L::CONV) {
          const double lam = slot[L::LS_A + el * NQ + q];  // per-cell material replicated per qp by L
          const double mu = slot[L::LS_B + el * NQ + q];
          // pre-scaled factors: Lm = dw lam Ji, Mu = dw mu Ji, Sd = Lm + Mu, Q = dw mu Ji Ji^T
          double Lm[9], Mu[9];
          const double dl = dw * lam, dm = dw * mu;
#pragma unroll
          for (int k = 0; k < 9; ++k) {
            Lm[k] = dl * Ji[k];
            Mu[k] = dm * Ji[k];
          }
          // diagonal blocks (a,a), unique pairs m <= n: dw ((lam + mu) Ji[m][a] Ji[n][a] + mu (Ji Ji^T)_mn)
#pragma unroll
          for (int u = 0; u < 6; ++u) {
            const int m = vp_um(u), n = vp_un(u);
            const double g = Mu[3 * m] * Ji[3 * n] + Mu[3 * m + 1] * Ji[3 * n + 1] + Mu[3 * m + 2] * Ji[3 * n + 2];
#pragma unroll
            for (int a2 = 0; a2 < 3; ++a2)
              Wq[(6 * a2 + u) * NQ] = fma(Lm[3 * m + a2] + Mu[3 * m + a2], Ji[3 * n + a2], g);
          }
          // off-diagonal blocks (0,1) (0,2) (1,2): dw (lam Ji[m][a] Ji[n][b] + mu Ji[m][b] Ji[n][a])
#pragma unroll
          for (int ob = 0; ob < 3; ++ob) {
            const int a2 = ob == 2 ? 1 : 0, b2 = ob == 0 ? 1 : 2;
#pragma unroll
            for (int pp = 0; pp < 9; ++pp) {
              const int m = pp / 3, n = pp % 3;
              Wq[(18 + 9 * ob + pp) * NQ] = fma(Lm[3 * m + a2], Ji[3 * n + b2], Mu[3 * m + b2] * Ji[3 * n + a2]);
            }
          }
        } else {
          // state at the qp: u_a and reference gradient du_a/dxi_m, 1D factors of Phi (Eq. fe1)
          const double* U = slot + L::LS_A + el * 3 * NB;
          double b0x[N1], b1x[N1], b0y[N1], b1y[N1], b0z[N1], b1z[N1];
#pragma unroll
          for (int i = 0; i < N1; ++i) {
            b0x[i] = Bt(0, qx, i); b1x[i] = Bt(1, qx, i);
            b0y[i] = Bt(0, qy, i); b1y[i] = Bt(1, qy, i);
            b0z[i] = Bt(0, qz, i); b1z[i] = Bt(1, qz, i);
          }
          double uq[3], du[3][3];
#pragma unroll
          for (int a = 0; a < 3; ++a) {
            double s0 = 0, sx = 0, sy = 0, sz = 0;
#pragma unroll
            for (int kz = 0; kz < N1; ++kz) {
              double y00 = 0, y01 = 0, y10 = 0;
#pragma unroll
              for (int ky = 0; ky < N1; ++ky) {
                double x0 = 0, x1 = 0;
#pragma unroll
                for (int kx = 0; kx < N1; ++kx) {
                  const double v = U[a * NB + kx + N1 * (ky + N1 * kz)];
                  x0 = fma(b0x[kx], v, x0);
                  x1 = fma(b1x[kx], v, x1);
                }
                y00 = fma(b0y[ky], x0, y00);
                y01 = fma(b1y[ky], x0, y01);
                y10 = fma(b0y[ky], x1, y10);
              }
              s0 = fma(b0z[kz], y00, s0);
              sz = fma(b1z[kz], y00, sz);
              sy = fma(b0z[kz], y01, sy);
              sx = fma(b0z[kz], y10, sx);
            }
            uq[a] = s0;
            du[a][0] = sx;
            du[a][1] = sy;
            du[a][2] = sz;
          }
          // item 0: (3,n) advection dw (Ji u)_n (shared by the diagonal blocks), then the
          // reactions dw du_a/dx_a of the diagonal blocks
#pragma unroll
          for (int n = 0; n < 3; ++n)
            Wq[n * NQ] = dw * (Ji[3 * n] * uq[0] + Ji[3 * n + 1] * uq[1] + Ji[3 * n + 2] * uq[2]);
          // du_a/dx_b = sum_m du_a/dxi_m Ji[m][b]
#pragma unroll
          for (int a2 = 0; a2 < 3; ++a2)
#pragma unroll
            for (int b2 = 0; b2 < 3; ++b2) {
              const double g = dw * (du[a2][0] * Ji[b2] + du[a2][1] * Ji[3 + b2] + du[a2][2] * Ji[6 + b2]);
              // diagonal -> pair 3 + a of item 0; off-diagonal -> the single pair of item 1..6
              const int slotw = a2 == b2 ? 3 + a2 : 6 + (2 * a2 + (b2 > a2 ? b2 - 1 : b2));
              Wq[slotw * NQ] = g;
            }
        }
      }
      vp_arrive(&emptyL[sl]);
      if constexpr (L::SPLIT) vp_arrive(&fullW[wb]);
      }  // g1
      if constexpr (L::SPLIT) {
        if (!g2) continue;
        VP_T(2, vp_wait(&fullW[wb], (uint32_t)((it >> 1) & 1)));
      } else {
        VP_T(0, vp_named_bar(1, NGT));
      }
      // ---- phase 2: stage z of every item, one compiled body per item kind (symmetric /
      // full pair set) inside a runtime item loop, so the code stays in the instruction cache
      auto g_item = [&](auto SYMc, int i) {
        constexpr bool SYMI = decltype(SYMc)::value;
        constexpr int NP = SYMI ? (L::CONV ? 1 : 6) : (L::CONV ? 6 : 9);
        const int s = (int)(gi % S);
        const double* Wi = Wb_ + (act2 ? el2 : 0) * L::NWP * NQ + IT::pbase(i) * NQ + tx + Q1 * ty;
        VP_T(3, vp_wait(&emptyT[s], (uint32_t)(((gi / S) & 1) ^ 1)));
        double* T1 = reinterpret_cast<double*>(smv + L::OFF_T1 + s * L::T1SLOT);
        if (act2) {
#pragma unroll
          for (int p = 0; p < NP; ++p) {
            if (p % GH != h2) continue;
            const int m = L::CONV ? 3 : (SYMI ? vp_um(p) : p / 3);
            const int n = L::CONV ? ((SYMI || p >= 3) ? 3 : p) : (SYMI ? vp_un(p) : p % 3);
            double Wq[Q1];
#pragma unroll
            for (int qz = 0; qz < Q1; ++qz) Wq[qz] = Wi[p * NQ + Q2 * qz];
            const int az = m == 2, bz = n == 2;
            double* out = T1 + (el2 * IT::NPMAX + p) * N1 * N1 * QQP + qxy;
#pragma unroll
            for (int a = 0; a < N1; ++a)
#pragma unroll
              for (int bb = 0; bb < N1; ++bb) {
                double sacc = 0.0;
#pragma unroll
                for (int qz = 0; qz < Q1; ++qz) sacc = fma(Wq[qz], c_zzv[P][az][bz][qz][a][bb], sacc);
                out[(a * N1 + bb) * QQP] = sacc;
              }
          }
        }
        vp_arrive(&fullT[s]);
        ++gi;
      };
#pragma unroll 1
      for (int i = 0; i < NITEM; ++i) {
        if (IT::sym(i)) g_item(std::true_type{}, i);
        else g_item(std::false_type{}, i);
      }
      if constexpr (L::SPLIT) vp_arrive(&emptyW[wb]);
    }
  } else if constexpr (L::YB3) {
    // ============ X, register-blocked (YB3): one (z pair, iy) per thread over jy = 0..2 ============
    const int xall = tid - 32 * (1 + L::NG);
    const int xg = xall / (32 * L::NXW), xtid = xall - xg * 32 * L::NXW;  // group, thread in group
    // lane -> (iy; full task; symmetric task).  Full items: every ordered z pair (iz, jz);
    // symmetric items: z pairs iz < jz and iz == jz -- the diagonal ones over all three iy
    // (the y pairs iy > jy of those are computed and not stored: the (jy, iy) task's mirror
    // writes them), so that every task has the form (z pair, iy; jy = 0..2)
    int f_el = -1, f_iz = 0, f_jz = 0, s_el = -1, s_iz = 0, s_jz = 0, iy = 0;
    if (FEB200_VP_YB3MAP) {  // generated bank-conflict-optimised map (tools/gen_vp_yb3_tasks.c)
      const unsigned v = vp_yb3_tasks[xg][xtid];
      iy = v & 3;
      if (iy < 3) {
        f_el = (v >> 2) & 3;
        f_iz = (v >> 4) & 3;
        f_jz = (v >> 6) & 3;
        s_el = (v >> 8) & 3;
        s_iz = (v >> 10) & 3;
        s_jz = (v >> 12) & 3;
        if (f_el == 3) f_el = -1;
        if (s_el == 3) s_el = -1;
      } else {
        iy = 0;
      }
    } else {
      const int cls = xtid / 21, j = xtid - cls * 21;
      if (cls < 3) {
        iy = cls;
        if (j < E * 9) { f_el = j / 9; f_iz = (j % 9) / 3; f_jz = j % 3; }
        if (j < E * 6) {
          s_el = j / 6;
          const int z6 = j % 6;
          s_iz = z6 < 3 ? (z6 >> 1) : z6 - 3;
          s_jz = z6 < 3 ? (z6 == 0 ? 1 : 2) : z6 - 3;
        }
      }
    }
    double Byp[3][4][Q1];  // Byp[jy][ay * 2 + by][qy] = B^ay[qy][iy] B^by[qy][jy]
#pragma unroll
    for (int k = 0; k < 3; ++k)
#pragma unroll
      for (int q = 0; q < Q1; ++q)
#pragma unroll
        for (int a2 = 0; a2 < 2; ++a2)
#pragma unroll
          for (int b2 = 0; b2 < 2; ++b2) Byp[k][a2 * 2 + b2][q] = Bt(a2, q, iy) * Bt(b2, q, k);
    for (int64_t it = 0;; ++it) {
      int64_t lb;
      int ne;
      batch_of(it, lb, ne);
      if (ne <= 0) break;
      auto item = [&](auto SYMc, int I, int ia, int ib_) {
        constexpr bool SYM = decltype(SYMc)::value;
        const bool MIR = IT::mirror(I);
        const int el = SYM ? s_el : f_el, iz = SYM ? s_iz : f_iz, jz = SYM ? s_jz : f_jz;
        const bool xact = el >= 0;
        const int64_t gi = it * NITEM + I;
        const int s = (int)(gi % S);
        VP_T(4, vp_wait(&fullT[s], (uint32_t)((gi / S) & 1)));
        const double* T1e = reinterpret_cast<const double*>(smv + L::OFF_T1 + s * L::T1SLOT) +
                            (xact ? el : 0) * IT::NPMAX * N1 * N1 * QQP;
        double Sx[3][4][Q1];
#pragma unroll
        for (int k = 0; k < 3; ++k)
#pragma unroll
          for (int c = 0; c < 4; ++c)
#pragma unroll
            for (int q = 0; q < Q1; ++q) Sx[k][c][q] = 0.0;
        if (xact) {
          const bool zdiag = SYM && iz == jz;
          double tv[Q2];
#pragma unroll
          for (int op = 0; op < 9; ++op) {
            int m, n, pidx, zidx;
            if constexpr (SYM) {
              // (0,0) (0,1) (1,0) (0,2) (2,0) (1,1) (1,2) (2,1) (2,2): a unique pair, then its
              // transpose -- the same T1 vector on a diagonal z pair (kept, not reloaded)
              m = (0x221120100 >> (4 * op)) & 0xF;
              n = (0x212102010 >> (4 * op)) & 0xF;
              const int mm = m < n ? m : n, nn = m < n ? n : m;
              pidx = mm == 0 ? nn : (mm == 1 ? 2 + nn : 5);
              zidx = (m > n) ? (jz * N1 + iz) : (iz * N1 + jz);
            } else {
              m = op / 3;
              n = op % 3;
              pidx = op;
              zidx = iz * N1 + jz;
            }
            const double* src = T1e + (pidx * N1 * N1 + zidx) * QQP;
            if (!SYM || m <= n || !zdiag) {
#pragma unroll
              for (int hh = 0; hh < Q2; ++hh) tv[hh] = src[hh];
            }
            const int ay = m == 1, by = n == 1, cls = (m == 0) * 2 + (n == 0);
#pragma unroll
            for (int k = 0; k < 3; ++k)
#pragma unroll
              for (int qx = 0; qx < Q1; ++qx)
#pragma unroll
                for (int qy = 0; qy < Q1; ++qy)
                  Sx[k][cls][qx] = fma(Byp[k][ay * 2 + by][qy], tv[qx * Q1 + qy], Sx[k][cls][qx]);
          }
        }
        vp_arrive(&emptyT[s]);
        if (I == xg && it > 0) {
          // first K write of this thread in the batch: the store of batch it-1 has read the
          // staging buffer
          VP_T(5, vp_wait(kfree, (uint32_t)((it - 1) & 1)));
        }
        if (xact && el < ne) {
          double* Kc = Kst + el * NDOF * NDOF;
#pragma unroll
          for (int k = 0; k < 3; ++k) {
            if (zdiag_skip(SYM, iz, jz, iy, k)) continue;
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
                  u[bb] = Bt(0, qx, bb) * Sx[k][ax * 2 + 0][qx] + Bt(1, qx, bb) * Sx[k][ax * 2 + 1][qx];
#pragma unroll
                for (int a = 0; a < N1; ++a)
#pragma unroll
                  for (int bb = 0; bb < N1; ++bb) acc[a][bb] = fma(Bt(ax, qx, a), u[bb], acc[a][bb]);
              }
            const int ib = N1 * (iy + N1 * iz), jb = N1 * (k + N1 * jz);
            const bool mir_in = SYM && (iz < jz || iy < k);
#pragma unroll
            for (int a = 0; a < N1; ++a)
#pragma unroll
              for (int bb = 0; bb < N1; ++bb) {
                const double v = acc[a][bb];
                Kc[(ia * NB + ib + a) * NDOF + ib_ * NB + jb + bb] = v;
                if (mir_in) Kc[(ia * NB + jb + bb) * NDOF + ib_ * NB + ib + a] = v;
                if (MIR) Kc[(ib_ * NB + jb + bb) * NDOF + ia * NB + ib + a] = v;
              }
          }
        }
      };
#pragma unroll 1
      for (int i = xg; i < NITEM; i += L::XG) {
        if (IT::sym(i)) item(std::true_type{}, i, IT::a(i), IT::b(i));
        else item(std::false_type{}, i, IT::a(i), IT::b(i));
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      vp_arrive(kfull);
    }
  } else {
    // ======================= X: stages y and x per item, K staging, TMA store =======================
    const int xall = tid - 32 * (1 + L::NG);
    const int xg = xall / (32 * L::NXW), xtid = xall - xg * 32 * L::NXW;  // group, thread in group
    int task_full = -1, task_sym = -1;
    if constexpr (L::TASKMAP) {
      task_full = vp_tasks_full[xtid];
      task_sym = vp_tasks_sym[xtid];
    }
    for (int64_t it = 0;; ++it) {
      int64_t lb;
      int ne;
      batch_of(it, lb, ne);
      if (ne <= 0) break;
      auto item = [&](auto SYMc, int I, int ia, int ib_) {
        constexpr bool SYM = decltype(SYMc)::value;
        constexpr int NP = SYM ? (L::CONV ? 1 : 6) : (L::CONV ? 6 : 9);
        constexpr bool ADV = L::CONV && !SYM;  // convective item 0: A + R_aa for the 3 diagonal blocks
        const bool MIR = IT::mirror(I);
        constexpr int TPE = SYM ? L::NSYM : L::NFULL;
        int el = xtid / TPE;
        const int r = xtid - el * TPE;
        bool xact = xtid < E * TPE;
        int iz = 0, jz = 0, iy = 0, jy = 0;
        if constexpr (L::TASKMAP) {
          // bank-conflict-optimised lane -> task permutation (tools/gen_vp_tasks.py)
          const int tk = SYM ? task_sym : task_full;
          xact = tk >= 0;
          el = tk & 15;
          iz = (tk >> 4) & 15;
          jz = (tk >> 8) & 15;
          iy = (tk >> 12) & 15;
          jy = (tk >> 16) & 15;
        } else if constexpr (SYM) {
          constexpr int YP = N1 * N1, YPS = N1 * (N1 + 1) / 2, TOFF = YP * (N1 * (N1 - 1) / 2);
          if (r < TOFF) {
            int c = r / YP;
            const int yp = r - c * YP;
            iy = yp / N1;
            jy = yp - iy * N1;
            for (int a = 0; a < N1; ++a) {
              if (c < N1 - 1 - a) { iz = a; jz = a + 1 + c; break; }
              c -= N1 - 1 - a;
            }
          } else {
            const int rr = r - TOFF;
            iz = jz = rr / YPS;
            int c = rr - iz * YPS;
            for (int a = 0; a < N1; ++a) {
              if (c < N1 - a) { iy = a; jy = a + c; break; }
              c -= N1 - a;
            }
          }
        } else {
          const int zp = r / (N1 * N1), yp = r - zp * (N1 * N1);
          iz = zp / N1; jz = zp - iz * N1;
          iy = yp / N1; jy = yp - iy * N1;
        }
        const int64_t gi = it * NITEM + I;
        const int s = (int)(gi % S);
        VP_T(4, vp_wait(&fullT[s], (uint32_t)((gi / S) & 1)));
        const double* T1e = reinterpret_cast<const double*>(smv + L::OFF_T1 + s * L::T1SLOT) +
                            (xact ? el : 0) * IT::NPMAX * N1 * N1 * QQP;
        double acc[N1][N1];
        double accr[ADV ? 3 : 1][N1][N1];  // ADV: K_aa = A + R_aa
        if (xact) {
          double Byp[4][Q1];
#pragma unroll
          for (int q = 0; q < Q1; ++q)
#pragma unroll
            for (int a2 = 0; a2 < 2; ++a2)
#pragma unroll
              for (int b2 = 0; b2 < 2; ++b2) Byp[a2 * 2 + b2][q] = Bt(a2, q, iy) * Bt(b2, q, jy);
          double Sx[4][Q1];
#pragma unroll
          for (int c = 0; c < 4; ++c)
#pragma unroll
            for (int q = 0; q < Q1; ++q) Sx[c][q] = 0.0;
          constexpr int NOPS = SYM ? (NP == 1 ? 1 : 9) : (ADV ? 3 : NP);
          double Sr[3][Q1];  // ADV: reaction accumulators of the three diagonal blocks (class (3,3))
#pragma unroll
          for (int a2 = 0; a2 < 3; ++a2)
#pragma unroll
            for (int q = 0; q < Q1; ++q) Sr[a2][q] = 0.0;
          if constexpr (ADV) {
#pragma unroll
            for (int a2 = 0; a2 < 3; ++a2) {
              const double* src = T1e + ((3 + a2) * N1 * N1 + iz * N1 + jz) * QQP;
#pragma unroll
              for (int qx = 0; qx < Q1; ++qx)
#pragma unroll
                for (int qy = 0; qy < Q1; ++qy) Sr[a2][qx] = fma(Byp[0][qy], src[qx * Q1 + qy], Sr[a2][qx]);
            }
          }
#pragma unroll
          for (int op = 0; op < NOPS; ++op) {
            int m, n, pidx, zidx;
            if constexpr (SYM) {
              if constexpr (NP == 1) {
                m = 3; n = 3; pidx = 0; zidx = iz * N1 + jz;
              } else {
                m = op / 3; n = op % 3;
                const int mm = m < n ? m : n, nn = m < n ? n : m;
                pidx = mm == 0 ? nn : (mm == 1 ? 2 + nn : 5);
                zidx = (m > n) ? (jz * N1 + iz) : (iz * N1 + jz);
              }
            } else {
              m = L::CONV ? 3 : op / 3;
              n = L::CONV ? op : op % 3;  // ADV: the advection pairs (3, 0..2)
              pidx = op;
              zidx = iz * N1 + jz;
            }
            const int ay = m == 1, by = n == 1, cls = (m == 0) * 2 + (n == 0);
            const double* src = T1e + (pidx * N1 * N1 + zidx) * QQP;
            double tv[QQP];
#pragma unroll
            for (int hh = 0; hh < Q2 / 2; ++hh) {
              const double2 v = reinterpret_cast<const double2*>(src)[hh];
              tv[2 * hh] = v.x;
              tv[2 * hh + 1] = v.y;
            }
            if (Q2 & 1) tv[Q2 - 1] = src[Q2 - 1];
#pragma unroll
            for (int qx = 0; qx < Q1; ++qx)
#pragma unroll
              for (int qy = 0; qy < Q1; ++qy)
                Sx[cls][qx] = fma(Byp[ay * 2 + by][qy], tv[qx * Q1 + qy], Sx[cls][qx]);
          }
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
              for (int bb = 0; bb < N1; ++bb) u[bb] = Bt(0, qx, bb) * Sx[ax * 2 + 0][qx] + Bt(1, qx, bb) * Sx[ax * 2 + 1][qx];
#pragma unroll
              for (int a = 0; a < N1; ++a)
#pragma unroll
                for (int bb = 0; bb < N1; ++bb) acc[a][bb] = fma(Bt(ax, qx, a), u[bb], acc[a][bb]);
            }
          if constexpr (ADV) {  // stage x of the reaction parts (value x value, class 0)
#pragma unroll
            for (int a2 = 0; a2 < 3; ++a2) {
#pragma unroll
              for (int a = 0; a < N1; ++a)
#pragma unroll
                for (int bb = 0; bb < N1; ++bb) accr[a2][a][bb] = acc[a][bb];
#pragma unroll
              for (int qx = 0; qx < Q1; ++qx) {
                double u[N1];
#pragma unroll
                for (int bb = 0; bb < N1; ++bb) u[bb] = Bt(0, qx, bb) * Sr[a2][qx];
#pragma unroll
                for (int a = 0; a < N1; ++a)
#pragma unroll
                  for (int bb = 0; bb < N1; ++bb) accr[a2][a][bb] = fma(Bt(0, qx, a), u[bb], accr[a2][a][bb]);
              }
            }
          }
        }
        vp_arrive(&emptyT[s]);
        if (I == xg && it > 0) {
          // first K write of this thread in the batch: the store of batch it-1 has read the
          // staging buffer
          VP_T(5, vp_wait(kfree, (uint32_t)((it - 1) & 1)));
        }
        if (ADV && xact && el < ne) {  // K_aa = A + R_aa for a = 0, 1, 2
          double* Kc = Kst + el * NDOF * NDOF;
          const int ib = N1 * (iy + N1 * iz), jb = N1 * (jy + N1 * jz);
#pragma unroll
          for (int a2 = 0; a2 < 3; ++a2)
#pragma unroll
            for (int a = 0; a < N1; ++a)
#pragma unroll
              for (int bb = 0; bb < N1; ++bb)
                Kc[(a2 * NB + ib + a) * NDOF + a2 * NB + jb + bb] = accr[a2][a][bb];
        } else if (xact && el < ne) {
          double* Kc = Kst + el * NDOF * NDOF;
          const int ib = N1 * (iy + N1 * iz), jb = N1 * (jy + N1 * jz);
          const bool mir_in = SYM && (iz < jz || iy < jy);
#pragma unroll
          for (int a = 0; a < N1; ++a)
#pragma unroll
            for (int bb = 0; bb < N1; ++bb) {
              const double v = acc[a][bb];
              Kc[(ia * NB + ib + a) * NDOF + ib_ * NB + jb + bb] = v;
              if (mir_in) Kc[(ia * NB + jb + bb) * NDOF + ib_ * NB + ib + a] = v;
              if (MIR) Kc[(ib_ * NB + jb + bb) * NDOF + ia * NB + ib + a] = v;
            }
        }
      };
#pragma unroll 1
      for (int i = xg; i < NITEM; i += L::XG) {
        if (IT::sym(i)) item(std::true_type{}, i, IT::a(i), IT::b(i));
        else item(std::false_type{}, i, IT::a(i), IT::b(i));
      }
      // ---- hand the batch's K staging to the store (L warp)
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      vp_arrive(kfull);
    }
  }
#ifdef FEB200_VP_PROF
  if (lane == 0) {
    for (int k = 0; k < 7; ++k) if (prof_[k]) atomicAdd(&g_vp_prof[k], prof_[k]);
    const int role = warp == 0 ? 0 : (warp <= L::NG ? 1 : 2);
    atomicAdd(&g_vp_prof[8 + role], (unsigned long long)(clock64() - tstart_));
    atomicAdd(&g_vp_prof[12 + role], 1ull);
  }
#endif
#undef Bt
}

template <int P, int FORM, bool FD>
static cudaError_t launch_vp_t(const fe_mesh* mh, MatArgs mat, const double* state_u, int64_t e0,
                               int64_t e1, double* K, cudaStream_t st, int* nonsym = nullptr) {
  using L = VPL<P, FORM, FD>;
  if (L::BYTES > 227 * 1024) return cudaErrorNotSupported;
  auto kern = k_matrix_vp<P, FORM, FD>;
  const LaunchFacts lf = launch_facts((const void*)kern, L::THREADS, L::BYTES);
  if (lf.err != cudaSuccess) return lf.err;
  const int64_t nsm = (int64_t)lf.nsm * (lf.per_sm < L::MINB ? lf.per_sm : L::MINB);
  const int64_t nbatch = (e1 - e0 + L::E - 1) / L::E;
  int grid = (int)(nbatch < nsm ? nbatch : nsm);
  grid = grid_cap(grid);
  if (grid <= 0) return cudaSuccess;
  kern<<<grid, L::THREADS, L::BYTES, st>>>(view_of(mh), mat.kind, (const double*)mat.a,
                                           (const double*)mat.b, state_u, e0, e1, K, nonsym);
  count_launch();
  return cudaGetLastError();
}

// Returns cudaErrorNotSupported when the combination has no pipelined vector kernel
// (vector mass, weighted dot, p != 2: the single-stage k_matrix_sfv handles those; with
// FEB200_MATRIX_IMPL=sf1 the general non-symmetric FULL_D path of k_matrix_sfv is used).
// General D (FE_MAT_FULL_D) is read as given by every path: the pipelined kernel, which
// derives K_ba = K_ab^T, is exact only for a symmetric D; it flags a non-symmetric block on
// the device, and the general kernel launched after it recomputes K when the flag is set and
// returns at once otherwise (no host synchronisation, so the call stays asynchronous and
// graph-capturable; the symmetric case costs one empty launch, not a second read of D).
cudaError_t launch_matrix_vp(const fe_mesh* mh, int form, MatArgs mat, const double* state_u,
                             int64_t e0, int64_t e1, double* K, cudaStream_t st) {
  if (mh->q1d != mh->order + 1 || mh->order != 2) return cudaErrorNotSupported;
  if (option(FE_OPT_MATRIX_IMPL) == MATRIX_SF1) return cudaErrorNotSupported;
  if (form == FE_FORM_ELASTICITY && mat.kind == FE_MAT_FULL_D) {
    if (e1 <= e0) return cudaSuccess;
    int* flag = nullptr;
    cudaError_t e = cudaMallocAsync((void**)&flag, sizeof(int), st);
    if (e != cudaSuccess) return e;
    e = cudaMemsetAsync(flag, 0, sizeof(int), st);
    if (e == cudaSuccess) e = launch_vp_t<2, FE_FORM_ELASTICITY, true>(mh, mat, state_u, e0, e1, K, st, flag);
    if (e == cudaSuccess) e = launch_matrix_sfv_gated(mh, form, mat, state_u, e0, e1, K, st, flag);
    cudaError_t ef = cudaFreeAsync(flag, st);
    return e != cudaSuccess ? e : ef;
  }
  if (form == FE_FORM_ELASTICITY)
    return launch_vp_t<2, FE_FORM_ELASTICITY, false>(mh, mat, state_u, e0, e1, K, st);
  if (form == FE_FORM_CONVECTIVE)
    return launch_vp_t<2, FE_FORM_CONVECTIVE, false>(mh, mat, state_u, e0, e1, K, st);
  return cudaErrorNotSupported;
}

}  // namespace feb200

#ifdef FEB200_VP_PROF
extern "C" int fe_debug_vp_prof(unsigned long long* out, int reset) {
  cudaDeviceSynchronize();
  cudaMemcpyFromSymbol(out, feb200::g_vp_prof, sizeof(unsigned long long) * 16);
  if (reset) {
    unsigned long long z[16] = {};
    cudaMemcpyToSymbol(feb200::g_vp_prof, z, sizeof(z));
  }
  return 0;
}
#endif
