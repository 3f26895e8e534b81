// Internal (non-ABI) declarations shared by the host API and the kernel units.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>

#include "feb200.h"

struct fe_mesh {
  int32_t order = 0, q1d = 0, nb = 0, nq = 0;
  int64_t n_vertices = 0, n_elems = 0, n_nodes = 0;
  double min_det = 0.0;
  int device = 0;
  // library-owned device copies
  double* coords = nullptr;    // [V][3]
  int32_t* conn = nullptr;     // [E][8]
  int32_t* dof_conn = nullptr; // [E][nb]  (== conn copy when order == 1)
  // reference tables (device), fp64 and fp32 copies
  double *xi = nullptr, *w = nullptr, *phi = nullptr, *dphi = nullptr, *fwd = nullptr, *bwd = nullptr;
  float *phi_f = nullptr, *dphi_f = nullptr, *fwd_f = nullptr, *bwd_f = nullptr;
  double *b1 = nullptr, *d1 = nullptr, *x1 = nullptr, *w1 = nullptr;  // 1D tables
};

// A second (scalar) Lagrange space on the cells of a mesh (the pressure space of the Stokes
// coupling forms): its own connectivity and its basis values at the mesh's quadrature points.
struct fe_field {
  int32_t order = 0, nb = 0;
  int64_t n_elems = 0, n_nodes = 0;
  const fe_mesh* mesh = nullptr;
  int32_t* dof_conn = nullptr;  // [E][nb] device
  double* psi = nullptr;        // [nq][nb] device
};

namespace feb200 {

// NVTX range around every ABI entry point that queues or performs work (visible in nsys /
// ncu --nvtx timelines; header-only NVTX3: a no-op branch when no tool is attached).
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};
#define FE_NVTX_RANGE(name) ::feb200::NvtxRange fe_nvtx_range_(name)

// Read-only view passed to kernels by value.
struct MeshView {
  const double* coords;
  const int32_t* conn;
  const int32_t* dof_conn;
  int64_t n_elems;
  const double* xi;
  const double* w;
  const double* phi;
  const double* dphi;
  const double* fwd;
  const double* bwd;
  const float* fwd_f;
  const float* bwd_f;
  const double* b1;
  const double* d1;
};

inline MeshView view_of(const fe_mesh* m) {
  return MeshView{m->coords, m->conn, m->dof_conn, m->n_elems, m->xi, m->w, m->phi, m->dphi,
                  m->fwd, m->bwd, m->fwd_f, m->bwd_f, m->b1, m->d1};
}

// Peer scatter windows of the fused residual + interface exchange (fe_eval_residual_peer,
// DESIGN.md 9): a scattered node n in [lo, hi) is also added (system-scope fp64 atomics,
// NVLink peer memory or any device pointer) at dst[(n - lo + off) * D + a].
struct PeerWin {
  int n;
  int64_t lo[2], hi[2], off[2];
  double* dst[2];
};
// set by fe_eval_residual_peer around the launch (per host thread)
extern thread_local PeerWin g_peer;

template <int D>
__device__ __forceinline__ void peer_scatter(const PeerWin& pw, int64_t n, int a, double v) {
#pragma unroll
  for (int w = 0; w < 2; ++w)
    if (w < pw.n && n >= pw.lo[w] && n < pw.hi[w])
      atomicAdd_system(pw.dst[w] + (n - pw.lo[w] + pw.off[w]) * D + a, v);
}

struct MatArgs {
  int kind;
  const void* a;
  const void* b;
};

// Launchers (return cudaError_t of the launch; cudaErrorNotSupported when the
// (form, order, dtype) combination is not built).
cudaError_t launch_matrix(const fe_mesh* m, int form, MatArgs mat, const double* state_u,
                          int64_t e0, int64_t e1, double* K, cudaStream_t st);
cudaError_t launch_matrix_sf(const fe_mesh* m, int form, MatArgs mat, int64_t e0, int64_t e1,
                             double* K, cudaStream_t st);
cudaError_t launch_matrix_sf_f32(const fe_mesh* m, int form, MatArgs mat, int64_t e0, int64_t e1,
                                 float* K, cudaStream_t st);
cudaError_t launch_matrix_residual_sf(const fe_mesh* m, int form, MatArgs mat, const double* u,
                                      int64_t e0, int64_t e1, double* K, double* r_elem,
                                      double* r_global, cudaStream_t st);
template <typename T>
cudaError_t launch_residual_sf(const fe_mesh* m, int form, MatArgs mat, const T* u, int64_t e0,
                               int64_t e1, T* r_elem, T* r_global, cudaStream_t st,
                               double* eval_out = nullptr);
cudaError_t launch_residual_t3(const fe_mesh* m, int form, MatArgs mat, const double* u, int64_t e0,
                               int64_t e1, double* r_elem, double* r_global, cudaStream_t st,
                               double* eval_out = nullptr);
cudaError_t upload_const_tables_residual_t3(int order, const double* b1, const double* d1,
                                           const double* x1, const double* w1, cudaStream_t st);
bool want_residual_t3();
cudaError_t launch_matrix_sfv(const fe_mesh* m, int form, MatArgs mat, const double* state_u,
                              int64_t e0, int64_t e1, double* K, cudaStream_t st);
cudaError_t launch_matrix_vp(const fe_mesh* m, int form, MatArgs mat, const double* state_u,
                             int64_t e0, int64_t e1, double* K, cudaStream_t st);
// general-D elasticity at p = 2 through k_matrix_sfv, executed only when *run_if != 0 (set on
// the device by the symmetry check of launch_matrix_vp)
cudaError_t launch_matrix_sfv_gated(const fe_mesh* m, int form, MatArgs mat, const double* state_u,
                                    int64_t e0, int64_t e1, double* K, cudaStream_t st,
                                    const int* run_if);
cudaError_t upload_const_tables_matrix_vp(int order, const double* b1, const double* d1,
                                         const double* x1, const double* w1, cudaStream_t st);
cudaError_t upload_const_tables_matrix_v(int order, const double* b1, const double* d1,
                                        const double* x1, const double* w1, cudaStream_t st);
cudaError_t launch_residual_f64(const fe_mesh* m, int form, MatArgs mat, const double* u,
                                int64_t e0, int64_t e1, double* r_elem, double* r_global,
                                cudaStream_t st);
cudaError_t launch_residual_f32(const fe_mesh* m, int form, MatArgs mat, const float* u,
                                int64_t e0, int64_t e1, float* r_elem, float* r_global,
                                cudaStream_t st);
cudaError_t launch_assemble(const fe_mesh* m, int dtype, int ncomp, int64_t e0, int64_t e1,
                            const void* r_elem, void* r_global, cudaStream_t st);
cudaError_t launch_geometry_check(const fe_mesh* m, double* block_min, unsigned long long* bad,
                                  int64_t nblocks, cudaStream_t st);
int64_t geometry_check_blocks(const fe_mesh* m);
cudaError_t launch_conn_check(const int32_t* idx, int64_t count, int64_t bound, int* flag,
                              cudaStream_t st);
cudaError_t launch_geometry_materialize(const fe_mesh* m, double* detw, double* jinv,
                                        cudaStream_t st);

void count_launch();
// Per-(kernel, device) launch facts, computed on the first launch on each device and cached:
// the max-dynamic-shared-memory attribute is set, the SM count and the resident CTAs per SM
// queried (keeps the per-call host overhead of small launches low).
struct LaunchFacts {
  int nsm, per_sm;
  cudaError_t err;
};
LaunchFacts launch_facts(const void* kern, int threads, size_t smem);
cudaError_t launch_coupling(const fe_mesh* mh, const fe_field* f, int mode, bool trans,
                            const double* u, const double* p, int64_t e0, int64_t e1, double* out,
                            double* rg, double* val, cudaStream_t st);
cudaError_t launch_stress(const fe_mesh* m, MatArgs mat, const double* u, int64_t e0, int64_t e1,
                          double* sigma, bool integrated, cudaStream_t st);
// Implementation options (fe_set_option; defaults from the environment, read once at load).
int64_t option(int opt);
bool set_option(int opt, int64_t value);
enum { MATRIX_DEFAULT = 0, MATRIX_SF1 = 1, MATRIX_DENSE = 2 };
enum { RESIDUAL_DEFAULT = 0, RESIDUAL_SF = 1, RESIDUAL_DENSE = 2 };
// Test hook: FE_OPT_MAX_CTAS caps the grid of the persistent kernels so that small meshes
// still run many batches per CTA (ring-buffer phases wrap several times in the parity tests).
int grid_cap(int grid);
cudaError_t upload_const_tables_matrix(int order, const double* b1, const double* d1,
                                      const double* x1, const double* w1, cudaStream_t st);
cudaError_t upload_const_tables_residual(int order, const double* b1, const double* d1,
                                        const double* x1, const double* w1, cudaStream_t st);

}  // namespace feb200
