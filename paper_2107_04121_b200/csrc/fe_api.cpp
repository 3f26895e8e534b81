// C ABI of libfeb200.so (include/feb200.h): validation, table set-up, handle
// ownership and dispatch.  No exception crosses the ABI; errors are fe_status
// codes with a thread-local message.
#include <algorithm>
#include <cstdio>
#include <new>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "fe_internal.h"
#include "tables.h"

namespace feb200 {
int64_t launch_count_value();
}

namespace {

thread_local std::string g_err;
thread_local int64_t g_err_elem = -1;

fe_status fail(fe_status s, const std::string& msg, int64_t elem = -1) {
  g_err = msg;
  g_err_elem = elem;
  return s;
}

fe_status cuda_fail(cudaError_t e, const char* where) {
  if (e == cudaErrorMemoryAllocation)
    return fail(FE_ERR_OOM, std::string(where) + ": " + cudaGetErrorString(e));
  return fail(FE_ERR_CUDA, std::string(where) + ": " + cudaGetErrorString(e));
}

fe_status ok() {
  g_err.clear();
  g_err_elem = -1;
  return FE_OK;
}

template <typename T>
cudaError_t upload(T** dst, const std::vector<T>& src, cudaStream_t st) {
  cudaError_t e = cudaMallocAsync((void**)dst, src.size() * sizeof(T) + 16, st);
  if (e != cudaSuccess) return e;
  return cudaMemcpyAsync(*dst, src.data(), src.size() * sizeof(T), cudaMemcpyHostToDevice, st);
}

// Device memory of the handles comes from the stream-ordered allocator (cudaMallocAsync on the
// create stream) and is returned with cudaFreeAsync on the destroy stream: no device-wide
// synchronisation, other streams keep running.
cudaError_t free_mesh(fe_mesh* m, cudaStream_t st) {
  if (!m) return cudaSuccess;
  void* ptrs[] = {m->coords, m->conn, m->dof_conn, m->xi, m->w, m->phi, m->dphi, m->fwd, m->bwd,
                  m->phi_f, m->dphi_f, m->fwd_f, m->bwd_f, m->b1, m->d1, m->x1, m->w1};
  cudaError_t e = cudaSuccess;
  for (void* p : ptrs)
    if (p) {
      const cudaError_t ee = cudaFreeAsync(p, st);
      if (e == cudaSuccess) e = ee;
    }
  delete m;
  return e;
}

int form_ncomp(int form) {
  return (form == FE_FORM_VECTOR_MASS || form == FE_FORM_ELASTICITY || form == FE_FORM_CONVECTIVE ||
          form == FE_FORM_WEIGHTED_DOT || form == FE_FORM_DIVERGENCE) ? 3 : 1;
}

fe_status check_common(const fe_mesh* mesh, int form, int64_t e0, int64_t e1) {
  if (!mesh) return fail(FE_ERR_INVALID_ARG, "mesh is NULL");
  if (form < FE_FORM_DIFFUSION || form > FE_FORM_DIVERGENCE)
    return fail(FE_ERR_INVALID_ARG, "unknown form " + std::to_string(form));
  if (e0 < 0 || e1 > mesh->n_elems || e0 > e1)
    return fail(FE_ERR_INVALID_ARG, "element range [" + std::to_string(e0) + ", " +
                                        std::to_string(e1) + ") outside [0, " +
                                        std::to_string(mesh->n_elems) + ")");
  return FE_OK;
}

fe_status check_material(int form, const fe_material* mat) {
  if (form == FE_FORM_CONVECTIVE || form == FE_FORM_DIVERGENCE) return FE_OK;
  if (!mat) return fail(FE_ERR_INVALID_ARG, "material is NULL");
  if (!mat->a) return fail(FE_ERR_INVALID_ARG, "material array a is NULL");
  if (form == FE_FORM_ELASTICITY) {
    if (mat->kind != FE_MAT_PER_QP && mat->kind != FE_MAT_PER_ELEM && mat->kind != FE_MAT_FULL_D)
      return fail(FE_ERR_INVALID_ARG, "unknown material kind");
    if (mat->kind != FE_MAT_FULL_D && !mat->b)
      return fail(FE_ERR_INVALID_ARG, "elasticity needs lambda (a) and mu (b)");
  } else {
    if (mat->kind != FE_MAT_PER_QP)
      return fail(FE_ERR_UNSUPPORTED, "this form takes per-quadrature-point material only");
    if (form == FE_FORM_MASS_DIFFUSION && !mat->b)
      return fail(FE_ERR_INVALID_ARG, "mass+diffusion needs rho (a) and kappa (b)");
  }
  return FE_OK;
}

}  // namespace

namespace feb200 {
thread_local PeerWin g_peer{};
// error setter shared with the other ABI units (k_csr.cu)
fe_status set_error(fe_status s, const char* msg) {
  if (s == FE_OK) return ok();
  return fail(s, msg);
}
}  // namespace feb200

extern "C" {

const char* fe_last_error(void) { return g_err.c_str(); }
int64_t fe_last_error_element(void) { return g_err_elem; }
int64_t fe_launch_count(void) { return feb200::launch_count_value(); }

fe_status fe_set_option(int32_t option, int64_t value) {
  if (!feb200::set_option(option, value))
    return fail(FE_ERR_INVALID_ARG, "fe_set_option: unknown option or value out of range");
  return ok();
}

fe_status fe_get_option(int32_t option, int64_t* value) {
  if (!value || option < 0 || option >= FE_OPT_COUNT)
    return fail(FE_ERR_INVALID_ARG, "fe_get_option: unknown option or NULL value");
  *value = feb200::option(option);
  return ok();
}

fe_status fe_create_mesh_geometry(int64_t n_vertices, const double* coords, int64_t n_elems,
                                  const int32_t* conn, int32_t order, int32_t q1d, int64_t n_nodes,
                                  const int32_t* dof_conn, void* stream, fe_mesh** out) {
  FE_NVTX_RANGE("fe_create_mesh_geometry");
  if (!out) return fail(FE_ERR_INVALID_ARG, "out is NULL");
  *out = nullptr;
  if (n_vertices < 8 || n_elems < 0) return fail(FE_ERR_INVALID_ARG, "bad sizes");
  if (!coords || (n_elems > 0 && !conn)) return fail(FE_ERR_INVALID_ARG, "coords/conn is NULL");
  if (order < 1 || order > 8 || q1d < 1 || q1d > 16)
    return fail(FE_ERR_INVALID_ARG, "order must be 1..8 and q1d 1..16");
  if (order > 4 || q1d != order + 1)
    return fail(FE_ERR_UNSUPPORTED, "GPU path built for order 1..4 with q1d = order + 1");
  if (order == 1 && !dof_conn) n_nodes = n_vertices;
  if (order > 1 && !dof_conn) return fail(FE_ERR_INVALID_ARG, "dof_conn required for order > 1");
  if (n_nodes < 1 || n_nodes >= (int64_t(1) << 31)) return fail(FE_ERR_INVALID_ARG, "bad n_nodes");
  cudaStream_t st = (cudaStream_t)stream;
  fe_mesh* m = new (std::nothrow) fe_mesh();
  if (!m) return fail(FE_ERR_OOM, "host allocation failed");
  cudaGetDevice(&m->device);
  m->order = order;
  m->q1d = q1d;
  m->nb = (order + 1) * (order + 1) * (order + 1);
  m->nq = q1d * q1d * q1d;
  m->n_vertices = n_vertices;
  m->n_elems = n_elems;
  m->n_nodes = n_nodes;
  cudaError_t e;
#define CK(x, where)                     \
  do {                                   \
    e = (x);                             \
    if (e != cudaSuccess) {              \
      free_mesh(m, st);                  \
      return cuda_fail(e, where);        \
    }                                    \
  } while (0)
  CK(cudaMallocAsync((void**)&m->coords, sizeof(double) * 3 * n_vertices, st), "alloc coords");
  CK(cudaMemcpyAsync(m->coords, coords, sizeof(double) * 3 * n_vertices, cudaMemcpyDefault, st), "copy coords");
  CK(cudaMallocAsync((void**)&m->conn, sizeof(int32_t) * 8 * std::max<int64_t>(n_elems, 1), st), "alloc conn");
  if (n_elems > 0)
    CK(cudaMemcpyAsync(m->conn, conn, sizeof(int32_t) * 8 * n_elems, cudaMemcpyDefault, st), "copy conn");
  const int64_t ndc = int64_t(m->nb) * std::max<int64_t>(n_elems, 1);
  CK(cudaMallocAsync((void**)&m->dof_conn, sizeof(int32_t) * ndc, st), "alloc dof_conn");
  if (n_elems > 0)
    CK(cudaMemcpyAsync(m->dof_conn, dof_conn ? dof_conn : conn, sizeof(int32_t) * m->nb * n_elems,
                       cudaMemcpyDefault, st), "copy dof_conn");
  // tables (step a0)
  feb200::HostTables T = feb200::build_tables(order, q1d);
  CK(upload(&m->xi, T.xi, st), "tables");
  CK(upload(&m->w, T.w, st), "tables");
  CK(upload(&m->phi, T.phi, st), "tables");
  CK(upload(&m->dphi, T.dphi, st), "tables");
  CK(upload(&m->fwd, T.fwd, st), "tables");
  CK(upload(&m->bwd, T.bwd, st), "tables");
  CK(upload(&m->b1, T.b1, st), "tables");
  CK(upload(&m->d1, T.d1, st), "tables");
  CK(upload(&m->x1, T.x1, st), "tables");
  CK(upload(&m->w1, T.w1, st), "tables");
  CK(feb200::upload_const_tables_matrix(order, T.b1.data(), T.d1.data(), T.x1.data(), T.w1.data(), st),
     "constant tables");
  CK(feb200::upload_const_tables_matrix_v(order, T.b1.data(), T.d1.data(), T.x1.data(), T.w1.data(), st),
     "constant tables");
  CK(feb200::upload_const_tables_matrix_vp(order, T.b1.data(), T.d1.data(), T.x1.data(), T.w1.data(), st),
     "constant tables");
  CK(feb200::upload_const_tables_residual(order, T.b1.data(), T.d1.data(), T.x1.data(), T.w1.data(), st),
     "constant tables");
  CK(feb200::upload_const_tables_residual_t3(order, T.b1.data(), T.d1.data(), T.x1.data(), T.w1.data(), st),
     "constant tables");
  std::vector<float> tmp;
  auto upf = [&](float** dst, const std::vector<double>& src) {
    tmp.assign(src.begin(), src.end());
    cudaError_t ee = upload(dst, tmp, st);
    if (ee == cudaSuccess) ee = cudaStreamSynchronize(st);  // tmp is reused
    return ee;
  };
  CK(upf(&m->phi_f, T.phi), "tables");
  CK(upf(&m->dphi_f, T.dphi), "tables");
  CK(upf(&m->fwd_f, T.fwd), "tables");
  CK(upf(&m->bwd_f, T.bwd), "tables");
  // connectivity range checks
  int* flag = nullptr;
  CK(cudaMallocAsync((void**)&flag, sizeof(int) * 2, st), "alloc flag");
  CK(cudaMemsetAsync(flag, 0, sizeof(int) * 2, st), "memset");
  CK(feb200::launch_conn_check(m->conn, 8 * n_elems, n_vertices, flag, st), "conn check");
  CK(feb200::launch_conn_check(m->dof_conn, int64_t(m->nb) * n_elems, n_nodes, flag + 1, st), "dof check");
  int hflag[2] = {0, 0};
  CK(cudaMemcpyAsync(hflag, flag, sizeof(hflag), cudaMemcpyDeviceToHost, st), "copy flag");
  cudaFreeAsync(flag, st);
  CK(cudaStreamSynchronize(st), "sync");
  if (hflag[0] || hflag[1]) {
    free_mesh(m, st);
    return fail(FE_ERR_INVALID_ARG, hflag[0] ? "conn entry out of [0, n_vertices)"
                                             : "dof_conn entry out of [0, n_nodes)");
  }
  // det J > 0 at every (cell, qp)
  const int64_t nblk = feb200::geometry_check_blocks(m);
  m->min_det = 1e300;
  if (nblk > 0) {
    double* bmin = nullptr;
    unsigned long long* bad = nullptr;
    CK(cudaMallocAsync((void**)&bmin, sizeof(double) * nblk, st), "alloc");
    CK(cudaMallocAsync((void**)&bad, sizeof(unsigned long long), st), "alloc");
    CK(cudaMemsetAsync(bad, 0xff, sizeof(unsigned long long), st), "memset");
    CK(feb200::launch_geometry_check(m, bmin, bad, nblk, st), "geometry check");
    std::vector<double> hmin(nblk);
    unsigned long long hbad = ~0ull;
    CK(cudaMemcpyAsync(hmin.data(), bmin, sizeof(double) * nblk, cudaMemcpyDeviceToHost, st), "copy");
    CK(cudaMemcpyAsync(&hbad, bad, sizeof(hbad), cudaMemcpyDeviceToHost, st), "copy");
    cudaFreeAsync(bmin, st);
    cudaFreeAsync(bad, st);
    CK(cudaStreamSynchronize(st), "sync");
    for (double v : hmin) m->min_det = std::min(m->min_det, v);
    if (hbad != ~0ull) {
      free_mesh(m, st);
      return fail(FE_ERR_DEGENERATE,
                  "det J <= 0 in cell " + std::to_string((long long)hbad), (int64_t)hbad);
    }
  }
#undef CK
  *out = m;
  return ok();
}

fe_status fe_destroy_mesh(fe_mesh* mesh, void* stream) {
  FE_NVTX_RANGE("fe_destroy_mesh");
  if (!mesh) return ok();
  int cur = 0;
  cudaGetDevice(&cur);
  const int dev = mesh->device;
  if (cur != dev) cudaSetDevice(dev);
  const cudaError_t e = free_mesh(mesh, (cudaStream_t)stream);
  if (cur != dev) cudaSetDevice(cur);
  if (e != cudaSuccess) return cuda_fail(e, "fe_destroy_mesh");
  return ok();
}

fe_status fe_mesh_info(const fe_mesh* mesh, fe_info* info) {
  if (!mesh || !info) return fail(FE_ERR_INVALID_ARG, "NULL argument");
  info->order = mesh->order;
  info->q1d = mesh->q1d;
  info->nb = mesh->nb;
  info->nq = mesh->nq;
  info->n_vertices = mesh->n_vertices;
  info->n_elems = mesh->n_elems;
  info->n_nodes = mesh->n_nodes;
  info->min_det_j = mesh->min_det;
  return ok();
}

fe_status fe_eval_element_matrices(const fe_mesh* mesh, int32_t form, int32_t dtype,
                                   const fe_material* mat, const void* state_u, int64_t elem_begin,
                                   int64_t elem_end, void* K, void* stream) {
  FE_NVTX_RANGE("fe_eval_element_matrices");
  fe_status s = check_common(mesh, form, elem_begin, elem_end);
  if (s != FE_OK) return s;
  if (dtype != FE_F64 && dtype != FE_F32) return fail(FE_ERR_INVALID_ARG, "unknown dtype");
  if ((s = check_material(form, mat)) != FE_OK) return s;
  if (dtype == FE_F32) {
    if (elem_end > elem_begin && !K) return fail(FE_ERR_INVALID_ARG, "K is NULL");
    if (feb200::option(FE_OPT_MATRIX_IMPL) != feb200::MATRIX_DEFAULT)
      return fail(FE_ERR_UNSUPPORTED, "FE_F32 element matrices: the pipelined kernels only");
    feb200::MatArgs ma{mat->kind, mat->a, mat->b};
    cudaError_t e = feb200::launch_matrix_sf_f32(mesh, form, ma, elem_begin, elem_end, (float*)K,
                                                 (cudaStream_t)stream);
    if (e == cudaErrorNotSupported)
      return fail(FE_ERR_UNSUPPORTED, "FE_F32 element matrices are built for the scalar forms "
                                      "(diffusion, mass, mass + diffusion) at order 1 and 2");
    if (e != cudaSuccess) return cuda_fail(e, "fe_eval_element_matrices");
    return ok();
  }
  if (form == FE_FORM_CONVECTIVE && !state_u)
    return fail(FE_ERR_INVALID_ARG, "convective tangent needs state_u");
  if (form == FE_FORM_DIVERGENCE)
    return fail(FE_ERR_UNSUPPORTED, "the divergence operator has no trial variable: no matrix mode");
  if (elem_end > elem_begin && !K) return fail(FE_ERR_INVALID_ARG, "K is NULL");
  feb200::MatArgs ma{mat ? mat->kind : 0, mat ? mat->a : nullptr, mat ? mat->b : nullptr};
  cudaError_t e = feb200::launch_matrix(mesh, form, ma, (const double*)state_u, elem_begin,
                                        elem_end, (double*)K, (cudaStream_t)stream);
  if (e == cudaErrorNotSupported)
    return fail(FE_ERR_UNSUPPORTED, "matrix mode not built for form " + std::to_string(form) +
                                        " at order " + std::to_string(mesh->order));
  if (e != cudaSuccess) return cuda_fail(e, "fe_eval_element_matrices");
  return ok();
}

fe_status fe_eval_residual(const fe_mesh* mesh, int32_t form, int32_t dtype, const fe_material* mat,
                           const void* u, int64_t elem_begin, int64_t elem_end, void* r_elem,
                           void* r_global, void* stream) {
  FE_NVTX_RANGE("fe_eval_residual");
  fe_status s = check_common(mesh, form, elem_begin, elem_end);
  if (s != FE_OK) return s;
  if ((s = check_material(form, mat)) != FE_OK) return s;
  if (!u) return fail(FE_ERR_INVALID_ARG, "u is NULL");
  if (dtype != FE_F64 && dtype != FE_F32) return fail(FE_ERR_INVALID_ARG, "unknown dtype");
  feb200::MatArgs ma{mat ? mat->kind : 0, mat ? mat->a : nullptr, mat ? mat->b : nullptr};
  cudaError_t e;
  if (dtype == FE_F64)
    e = feb200::launch_residual_f64(mesh, form, ma, (const double*)u, elem_begin, elem_end,
                                    (double*)r_elem, (double*)r_global, (cudaStream_t)stream);
  else
    e = feb200::launch_residual_f32(mesh, form, ma, (const float*)u, elem_begin, elem_end,
                                    (float*)r_elem, (float*)r_global, (cudaStream_t)stream);
  if (e == cudaErrorNotSupported)
    return fail(FE_ERR_UNSUPPORTED, "residual mode not built for form " + std::to_string(form) +
                                        " / dtype " + std::to_string(dtype) + " at order " +
                                        std::to_string(mesh->order));
  if (e != cudaSuccess) return cuda_fail(e, "fe_eval_residual");
  return ok();
}

fe_status fe_eval_residual_peer(const fe_mesh* mesh, int32_t form, const fe_material* mat,
                                const double* u, int64_t elem_begin, int64_t elem_end,
                                double* r_elem, double* r_global, const fe_peer_window* windows,
                                int32_t n_windows, void* stream) {
  FE_NVTX_RANGE("fe_eval_residual_peer");
  if (n_windows < 0 || n_windows > 2 || (n_windows > 0 && !windows))
    return fail(FE_ERR_INVALID_ARG, "fe_eval_residual_peer: 0..2 windows");
  if (feb200::option(FE_OPT_RESIDUAL_IMPL) == feb200::RESIDUAL_DENSE)
    return fail(FE_ERR_UNSUPPORTED, "fe_eval_residual_peer: not built for the dense residual kernels");
  feb200::PeerWin pw{};
  pw.n = n_windows;
  for (int w = 0; w < n_windows; ++w) {
    const fe_peer_window& x = windows[w];
    if (!x.dst || x.node_begin < 0 || x.node_end < x.node_begin || x.dst_node_offset < 0)
      return fail(FE_ERR_INVALID_ARG, "fe_eval_residual_peer: bad window");
    pw.lo[w] = x.node_begin;
    pw.hi[w] = x.node_end;
    pw.off[w] = x.dst_node_offset;
    pw.dst[w] = x.dst;
  }
  feb200::g_peer = pw;
  const fe_status s = fe_eval_residual(mesh, form, FE_F64, mat, u, elem_begin, elem_end, r_elem,
                                       r_global, stream);
  feb200::g_peer = feb200::PeerWin{};
  return s;
}

fe_status fe_ipc_alloc(int64_t bytes, void** dev_ptr, unsigned char handle[64]) {
  FE_NVTX_RANGE("fe_ipc_alloc");
  if (!dev_ptr || !handle || bytes <= 0) return fail(FE_ERR_INVALID_ARG, "fe_ipc_alloc: bad argument");
  *dev_ptr = nullptr;
  cudaError_t e = cudaMalloc(dev_ptr, (size_t)bytes);
  if (e != cudaSuccess) return cuda_fail(e, "fe_ipc_alloc");
  cudaIpcMemHandle_t h;
  e = cudaIpcGetMemHandle(&h, *dev_ptr);
  if (e != cudaSuccess) {
    cudaFree(*dev_ptr);
    *dev_ptr = nullptr;
    return cuda_fail(e, "fe_ipc_alloc: cudaIpcGetMemHandle");
  }
  static_assert(sizeof(h) == 64, "IPC handle size");
  std::memcpy(handle, &h, 64);
  return ok();
}

fe_status fe_ipc_free(void* dev_ptr) {
  FE_NVTX_RANGE("fe_ipc_free");
  if (dev_ptr) cudaFree(dev_ptr);
  return ok();
}

fe_status fe_ipc_open(const unsigned char handle[64], void** dev_ptr) {
  FE_NVTX_RANGE("fe_ipc_open");
  if (!handle || !dev_ptr) return fail(FE_ERR_INVALID_ARG, "fe_ipc_open: bad argument");
  cudaIpcMemHandle_t h;
  std::memcpy(&h, handle, 64);
  cudaError_t e = cudaIpcOpenMemHandle(dev_ptr, h, cudaIpcMemLazyEnablePeerAccess);
  if (e != cudaSuccess) return cuda_fail(e, "fe_ipc_open");
  return ok();
}

fe_status fe_ipc_close(void* dev_ptr) {
  FE_NVTX_RANGE("fe_ipc_close");
  if (dev_ptr) {
    cudaError_t e = cudaIpcCloseMemHandle(dev_ptr);
    if (e != cudaSuccess) return cuda_fail(e, "fe_ipc_close");
  }
  return ok();
}

fe_status fe_eval_matrix_residual(const fe_mesh* mesh, int32_t form, int32_t dtype,
                                  const fe_material* mat, const void* u, int64_t elem_begin,
                                  int64_t elem_end, void* K, void* r_elem, void* r_global,
                                  void* stream) {
  FE_NVTX_RANGE("fe_eval_matrix_residual");
  fe_status s = check_common(mesh, form, elem_begin, elem_end);
  if (s != FE_OK) return s;
  if (dtype != FE_F64) return fail(FE_ERR_UNSUPPORTED, "fe_eval_matrix_residual is built for FE_F64 only");
  if ((s = check_material(form, mat)) != FE_OK) return s;
  if (form != FE_FORM_DIFFUSION && form != FE_FORM_MASS && form != FE_FORM_MASS_DIFFUSION)
    return fail(FE_ERR_UNSUPPORTED, "fe_eval_matrix_residual: linear scalar forms only");
  if (elem_end > elem_begin && (!K || !u)) return fail(FE_ERR_INVALID_ARG, "K / u is NULL");
  feb200::MatArgs ma{mat ? mat->kind : 0, mat ? mat->a : nullptr, mat ? mat->b : nullptr};
  cudaError_t e = feb200::launch_matrix_residual_sf(mesh, form, ma, (const double*)u, elem_begin,
                                                    elem_end, (double*)K, (double*)r_elem,
                                                    (double*)r_global, (cudaStream_t)stream);
  if (e == cudaErrorNotSupported)
    return fail(FE_ERR_UNSUPPORTED, "fe_eval_matrix_residual: order " + std::to_string(mesh->order) +
                                        " not built (orders 1, 2)");
  if (e != cudaSuccess) return cuda_fail(e, "fe_eval_matrix_residual");
  return ok();
}

fe_status fe_eval_scalar(const fe_mesh* mesh, int32_t form, int32_t dtype, const fe_material* mat,
                         const void* u, int64_t elem_begin, int64_t elem_end, double* value,
                         void* stream) {
  FE_NVTX_RANGE("fe_eval_scalar");
  fe_status s = check_common(mesh, form, elem_begin, elem_end);
  if (s != FE_OK) return s;
  if ((s = check_material(form, mat)) != FE_OK) return s;
  if (!u || !value) return fail(FE_ERR_INVALID_ARG, "u / value is NULL");
  if (dtype != FE_F64 && dtype != FE_F32) return fail(FE_ERR_INVALID_ARG, "unknown dtype");
  feb200::MatArgs ma{mat ? mat->kind : 0, mat ? mat->a : nullptr, mat ? mat->b : nullptr};
  cudaError_t e;
  e = cudaErrorNotSupported;
  if (dtype == FE_F64 && feb200::want_residual_t3())
    e = feb200::launch_residual_t3(mesh, form, ma, (const double*)u, elem_begin, elem_end, nullptr,
                                   nullptr, (cudaStream_t)stream, value);
  if (e != cudaErrorNotSupported) {
  } else if (dtype == FE_F64)
    e = feb200::launch_residual_sf<double>(mesh, form, ma, (const double*)u, elem_begin, elem_end,
                                           nullptr, nullptr, (cudaStream_t)stream, value);
  else
    e = feb200::launch_residual_sf<float>(mesh, form, ma, (const float*)u, elem_begin, elem_end,
                                          nullptr, nullptr, (cudaStream_t)stream, value);
  if (e == cudaErrorNotSupported)
    return fail(FE_ERR_UNSUPPORTED, "eval mode not built for this form / order / dtype");
  if (e != cudaSuccess) return cuda_fail(e, "fe_eval_scalar");
  return ok();
}

static fe_status eval_stress_impl(const fe_mesh* mesh, const fe_material* mat, const double* u,
                                  int64_t elem_begin, int64_t elem_end, double* sigma, bool integ,
                                  void* stream, const char* name) {
  fe_status s = check_common(mesh, FE_FORM_ELASTICITY, elem_begin, elem_end);
  if (s != FE_OK) return s;
  if ((s = check_material(FE_FORM_ELASTICITY, mat)) != FE_OK) return s;
  if (elem_end > elem_begin && (!u || !sigma)) return fail(FE_ERR_INVALID_ARG, "u / sigma is NULL");
  feb200::MatArgs ma{mat->kind, mat->a, mat->b};
  cudaError_t e = feb200::launch_stress(mesh, ma, u, elem_begin, elem_end, sigma, integ,
                                        (cudaStream_t)stream);
  if (e == cudaErrorNotSupported)
    return fail(FE_ERR_UNSUPPORTED, std::string(name) + ": q1d " + std::to_string(mesh->q1d) +
                                        " not built for order " + std::to_string(mesh->order));
  if (e != cudaSuccess) return cuda_fail(e, name);
  return ok();
}

fe_status fe_eval_stress(const fe_mesh* mesh, const fe_material* mat, const double* u,
                         int64_t elem_begin, int64_t elem_end, double* sigma, void* stream) {
  FE_NVTX_RANGE("fe_eval_stress");
  return eval_stress_impl(mesh, mat, u, elem_begin, elem_end, sigma, false, stream, "fe_eval_stress");
}

fe_status fe_eval_stress_integral(const fe_mesh* mesh, const fe_material* mat, const double* u,
                                  int64_t elem_begin, int64_t elem_end, double* sigma_int,
                                  void* stream) {
  FE_NVTX_RANGE("fe_eval_stress_integral");
  return eval_stress_impl(mesh, mat, u, elem_begin, elem_end, sigma_int, true, stream,
                          "fe_eval_stress_integral");
}

fe_status fe_create_field(const fe_mesh* mesh, int32_t order, int64_t n_nodes,
                          const int32_t* dof_conn, void* stream, fe_field** out) {
  FE_NVTX_RANGE("fe_create_field");
  if (!out) return fail(FE_ERR_INVALID_ARG, "out is NULL");
  *out = nullptr;
  if (!mesh) return fail(FE_ERR_INVALID_ARG, "mesh is NULL");
  if (order < 1 || order > mesh->order)
    return fail(FE_ERR_INVALID_ARG, "pressure order must be 1..mesh order");
  if (n_nodes < 1 || n_nodes >= (int64_t(1) << 31)) return fail(FE_ERR_INVALID_ARG, "bad n_nodes");
  if (mesh->n_elems > 0 && !dof_conn) return fail(FE_ERR_INVALID_ARG, "dof_conn is NULL");
  cudaStream_t st = (cudaStream_t)stream;
  fe_field* f = new (std::nothrow) fe_field();
  if (!f) return fail(FE_ERR_OOM, "host allocation failed");
  f->order = order;
  f->nb = (order + 1) * (order + 1) * (order + 1);
  f->n_elems = mesh->n_elems;
  f->n_nodes = n_nodes;
  f->mesh = mesh;
  auto bail = [&](cudaError_t e, const char* where) {
    if (f->dof_conn) cudaFreeAsync(f->dof_conn, st);
    if (f->psi) cudaFreeAsync(f->psi, st);
    delete f;
    return cuda_fail(e, where);
  };
  cudaError_t e;
  const int64_t n = int64_t(f->nb) * mesh->n_elems;
  if ((e = cudaMallocAsync((void**)&f->dof_conn, sizeof(int32_t) * std::max<int64_t>(n, 1), st)) != cudaSuccess)
    return bail(e, "alloc dof_conn");
  if (n > 0 && (e = cudaMemcpyAsync(f->dof_conn, dof_conn, sizeof(int32_t) * n, cudaMemcpyDefault, st)) != cudaSuccess)
    return bail(e, "copy dof_conn");
  // pressure basis at the mesh's quadrature points (the same Gauss rule, step a0)
  feb200::HostTables T = feb200::build_tables(order, mesh->q1d);
  if ((e = upload(&f->psi, T.phi, st)) != cudaSuccess) return bail(e, "tables");
  int* flag = nullptr;
  int hflag = 0;
  if ((e = cudaMallocAsync((void**)&flag, sizeof(int), st)) != cudaSuccess) return bail(e, "alloc flag");
  e = cudaMemsetAsync(flag, 0, sizeof(int), st);
  if (e == cudaSuccess) e = feb200::launch_conn_check(f->dof_conn, n, n_nodes, flag, st);
  if (e == cudaSuccess) e = cudaMemcpyAsync(&hflag, flag, sizeof(int), cudaMemcpyDeviceToHost, st);
  cudaFreeAsync(flag, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  if (e != cudaSuccess) return bail(e, "dof check");
  if (hflag) {
    cudaFreeAsync(f->dof_conn, st);
    cudaFreeAsync(f->psi, st);
    delete f;
    return fail(FE_ERR_INVALID_ARG, "pressure dof_conn entry out of [0, n_nodes)");
  }
  *out = f;
  return ok();
}

fe_status fe_destroy_field(fe_field* field, void* stream) {
  FE_NVTX_RANGE("fe_destroy_field");
  if (!field) return ok();
  cudaStream_t st = (cudaStream_t)stream;
  cudaError_t e = cudaSuccess, e2 = cudaSuccess;
  if (field->dof_conn) e = cudaFreeAsync(field->dof_conn, st);
  if (field->psi) e2 = cudaFreeAsync(field->psi, st);
  delete field;
  if (e == cudaSuccess) e = e2;
  if (e != cudaSuccess) return cuda_fail(e, "fe_destroy_field");
  return ok();
}

static fe_status check_coupling(const fe_mesh* mesh, const fe_field* f, int64_t e0, int64_t e1) {
  fe_status s = check_common(mesh, FE_FORM_DIVERGENCE, e0, e1);
  if (s != FE_OK) return s;
  if (!f) return fail(FE_ERR_INVALID_ARG, "pressure field is NULL");
  if (f->mesh != mesh) return fail(FE_ERR_INVALID_ARG, "pressure field belongs to another mesh");
  return FE_OK;
}

static fe_status coupling_status(cudaError_t e, const fe_mesh* mesh, const fe_field* f, const char* what) {
  if (e == cudaErrorNotSupported)
    return fail(FE_ERR_UNSUPPORTED, std::string(what) + ": pair (" + std::to_string(mesh->order) +
                                        ", " + std::to_string(f->order) + ") not built");
  if (e != cudaSuccess) return cuda_fail(e, what);
  return ok();
}

fe_status fe_eval_coupling_matrices(const fe_mesh* mesh, const fe_field* pressure, int32_t transposed,
                                    int64_t elem_begin, int64_t elem_end, double* out, void* stream) {
  FE_NVTX_RANGE("fe_eval_coupling_matrices");
  fe_status s = check_coupling(mesh, pressure, elem_begin, elem_end);
  if (s != FE_OK) return s;
  if (elem_end > elem_begin && !out) return fail(FE_ERR_INVALID_ARG, "out is NULL");
  return coupling_status(feb200::launch_coupling(mesh, pressure, 0, transposed != 0, nullptr, nullptr,
                                                 elem_begin, elem_end, out, nullptr, nullptr,
                                                 (cudaStream_t)stream),
                         mesh, pressure, "fe_eval_coupling_matrices");
}

fe_status fe_eval_coupling_residual(const fe_mesh* mesh, const fe_field* pressure, int32_t transposed,
                                    const double* x, int64_t elem_begin, int64_t elem_end,
                                    double* r_elem, double* r_global, void* stream) {
  FE_NVTX_RANGE("fe_eval_coupling_residual");
  fe_status s = check_coupling(mesh, pressure, elem_begin, elem_end);
  if (s != FE_OK) return s;
  if (!x) return fail(FE_ERR_INVALID_ARG, "input vector is NULL");
  const bool tr = transposed != 0;
  return coupling_status(feb200::launch_coupling(mesh, pressure, 1, tr, tr ? x : nullptr, tr ? nullptr : x,
                                                 elem_begin, elem_end, r_elem, r_global, nullptr,
                                                 (cudaStream_t)stream),
                         mesh, pressure, "fe_eval_coupling_residual");
}

fe_status fe_eval_coupling_scalar(const fe_mesh* mesh, const fe_field* pressure, const double* u,
                                  const double* p, int64_t elem_begin, int64_t elem_end,
                                  double* value, void* stream) {
  FE_NVTX_RANGE("fe_eval_coupling_scalar");
  fe_status s = check_coupling(mesh, pressure, elem_begin, elem_end);
  if (s != FE_OK) return s;
  if (!u || !p || !value) return fail(FE_ERR_INVALID_ARG, "u / p / value is NULL");
  return coupling_status(feb200::launch_coupling(mesh, pressure, 2, false, u, p, elem_begin, elem_end,
                                                 nullptr, nullptr, value, (cudaStream_t)stream),
                         mesh, pressure, "fe_eval_coupling_scalar");
}

fe_status fe_assemble_vector(const fe_mesh* mesh, int32_t dtype, int32_t ncomp, int64_t elem_begin,
                             int64_t elem_end, const void* r_elem, void* r_global, void* stream) {
  FE_NVTX_RANGE("fe_assemble_vector");
  fe_status s = check_common(mesh, FE_FORM_DIFFUSION, elem_begin, elem_end);
  if (s != FE_OK) return s;
  if (ncomp != 1 && ncomp != 3) return fail(FE_ERR_INVALID_ARG, "ncomp must be 1 or 3");
  if (dtype != FE_F64 && dtype != FE_F32) return fail(FE_ERR_INVALID_ARG, "unknown dtype");
  if (elem_end > elem_begin && (!r_elem || !r_global))
    return fail(FE_ERR_INVALID_ARG, "r_elem / r_global is NULL");
  cudaError_t e = feb200::launch_assemble(mesh, dtype, ncomp, elem_begin, elem_end, r_elem,
                                          r_global, (cudaStream_t)stream);
  if (e != cudaSuccess) return cuda_fail(e, "fe_assemble_vector");
  return ok();
}

fe_status fe_geometry(const fe_mesh* mesh, double* detw, double* jinv, void* stream) {
  FE_NVTX_RANGE("fe_geometry");
  if (!mesh) return fail(FE_ERR_INVALID_ARG, "mesh is NULL");
  cudaError_t e = feb200::launch_geometry_materialize(mesh, detw, jinv, (cudaStream_t)stream);
  if (e != cudaSuccess) return cuda_fail(e, "fe_geometry");
  return ok();
}

}  // extern "C"
