// Global sparse (CSR) matrix assembly from element matrices -- SURVEY 8(f) N2,
// "the step after matrix mode" (the paper leaves it to SfePy and times it only
// in the FEniCS comparison).
//
// Pattern (setup, once per mesh and component count): every (cell, k, l) node
// pair becomes a key row * n_nodes + col; sort + unique on the GPU gives the
// scalar node-to-node pattern, row pointers come from a vectorised lower_bound,
// and a per-(cell, k, l) map stores the column's index inside its row.  Vector
// fields (D = 3) use the interleaved global numbering of Eq. fe1c (dof = node D +
// a), so every node pair expands to a D x D block laid out row by row:
//   row (r, a) starts at D^2 rowptr_node[r] + a D n_r,  column (c, b) is at
//   idx_in_row(r, c) D + b.
// Assembly: values[pos(e, a k, b l)] += K_e[a k][b l] with fp64 atomics
// (atomic order is the only run-to-run difference, as for the residual).
#include <algorithm>
#ifndef FEB200_CSR_CONST
#define FEB200_CSR_CONST 1
#endif
#include <cstdlib>
#include <cstring>
#include <exception>
#include <new>
#include <string>
#include <type_traits>

#include <thrust/binary_search.h>
#include <thrust/iterator/counting_iterator.h>
#include <thrust/iterator/transform_iterator.h>
#include <thrust/device_ptr.h>
#include <thrust/execution_policy.h>
#include <thrust/sequence.h>
#include <thrust/copy.h>
#include <thrust/sort.h>
#include <thrust/unique.h>

#include "fe_internal.h"

struct fe_csr {
  const fe_mesh* mesh = nullptr;
  int32_t ncomp = 1;
  int64_t n_nodes = 0, nnz_node = 0;
  int64_t* rowptr_node = nullptr;   // [n_nodes + 1] scalar node pattern
  int32_t* col_node = nullptr;      // [nnz_node]
  void* pos_in_row = nullptr;       // [E][nb][nb] index of column node l inside row node k
  int pos_bytes = 4;                // 1, 2 or 4: narrowest type holding every row length
  int64_t* n2c_ptr = nullptr;       // [n_nodes + 1] node -> incident (cell, local node) list
  int32_t* n2c = nullptr;           // [E nb] entries e nb + k, sorted by (node, e)
  int hmax = 0;                     // longest node row of the scalar pattern
  int64_t* rowptr = nullptr;        // [n_nodes D + 1] expanded pattern
  int32_t* col = nullptr;           // [nnz_node D^2]
};

namespace feb200 {

struct RowKey {
  int64_t n;
  __host__ __device__ int64_t operator()(int64_t r) const { return r * n; }
};

__global__ void k_pair_keys(const int32_t* __restrict__ dc, int nb, int64_t E, int64_t n_nodes,
                            int64_t* __restrict__ keys) {
  const int64_t n = E * nb * nb;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t e = i / (nb * nb);
    const int r = (int)(i - e * nb * nb), k = r / nb, l = r - k * nb;
    keys[i] = (int64_t)dc[e * nb + k] * n_nodes + dc[e * nb + l];
  }
}

__global__ void k_cols(const int64_t* __restrict__ keys, int64_t nnz, int64_t n_nodes, int32_t* __restrict__ col) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nnz; i += (int64_t)gridDim.x * blockDim.x)
    col[i] = (int32_t)(keys[i] % n_nodes);
}

template <typename PT>
__global__ void k_pos_map(const int32_t* __restrict__ dc, int nb, int64_t E, const int64_t* __restrict__ rowptr,
                          const int32_t* __restrict__ col, PT* __restrict__ pos) {
  const int64_t n = E * nb * nb;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t e = i / (nb * nb);
    const int r = (int)(i - e * nb * nb), k = r / nb, l = r - k * nb;
    const int32_t row = dc[e * nb + k], c = dc[e * nb + l];
    int64_t lo = rowptr[row], hi = rowptr[row + 1];
    const int64_t base = lo;
    while (lo < hi) {  // binary search of c in the sorted row
      const int64_t mid = (lo + hi) >> 1;
      if (col[mid] < c) lo = mid + 1; else hi = mid;
    }
    pos[i] = (PT)(lo - base);
  }
}

// expanded (vector) pattern: rowptr[r D + a] = D^2 rowptr_node[r] + a D n_r
__global__ void k_expand(const int64_t* __restrict__ rpn, const int32_t* __restrict__ cn, int64_t n_nodes, int D,
                         int64_t* __restrict__ rowptr, int32_t* __restrict__ col) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n_nodes; r += (int64_t)gridDim.x * blockDim.x) {
    const int64_t b0 = rpn[r], nr = rpn[r + 1] - b0;
    for (int a = 0; a < D; ++a) {
      const int64_t rs = (int64_t)D * D * b0 + (int64_t)a * D * nr;
      rowptr[r * D + a] = rs;
      for (int64_t j = 0; j < nr; ++j)
        for (int b = 0; b < D; ++b) col[rs + j * D + b] = cn[b0 + j] * D + b;
    }
    if (r == n_nodes - 1) rowptr[n_nodes * D] = (int64_t)D * D * rpn[n_nodes];
  }
}

__global__ void k_max_row(const int64_t* __restrict__ rpn, int64_t n, unsigned long long* __restrict__ mx) {
  unsigned long long m = 0;
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n; r += (int64_t)gridDim.x * blockDim.x) {
    const unsigned long long len = (unsigned long long)(rpn[r + 1] - rpn[r]);
    m = len > m ? len : m;
  }
  for (int o = 16; o > 0; o >>= 1) {
    const unsigned long long v = __shfl_xor_sync(0xffffffffu, m, o);
    m = v > m ? v : m;
  }
  if ((threadIdx.x & 31) == 0) atomicMax(mx, m);
}

// values[pos] += K[e - e0][a nb + k][b nb + l]; the position map is stored in the narrowest
// integer type that holds every row length (uint8 for the Q2 lattice: 4x less map traffic)
template <typename PT>
__global__ void __launch_bounds__(256) k_assemble_matrix(const int32_t* __restrict__ dc, int nb, int D,
                                                         int64_t e0, int64_t e1,
                                                         const int64_t* __restrict__ rpn,
                                                         const PT* __restrict__ pos,
                                                         const double* __restrict__ K,
                                                         double* __restrict__ values) {
  const int nd = D * nb;
  const int64_t n = (e1 - e0) * nd * nd;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t el = i / (nd * nd);
    const int rr = (int)(i - el * nd * nd), row = rr / nd, cl = rr - row * nd;
    const int a = row / nb, k = row - a * nb, b = cl / nb, l = cl - b * nb;
    const int64_t e = e0 + el;
    const int32_t rn = dc[e * nb + k];
    const int64_t b0 = rpn[rn], nr = rpn[rn + 1] - b0;
    const int64_t p = (int64_t)D * D * b0 + (int64_t)a * D * nr +
                      (int64_t)pos[(e * nb + k) * nb + l] * D + b;
    atomicAdd(values + p, K[i]);
  }
}


// Same, with compile-time sizes and 32-bit index arithmetic (divisions by constants become
// multiply-shifts; the generic kernel divides 64-bit indices per entry)
template <typename PT, int NB, int D>
__global__ void __launch_bounds__(256) k_assemble_matrix_c(const int32_t* __restrict__ dc, int64_t e0,
                                                           uint32_t n, const int64_t* __restrict__ rpn,
                                                           const PT* __restrict__ pos,
                                                           const double* __restrict__ K,
                                                           double* __restrict__ values) {
  constexpr uint32_t ND = D * NB, NE = ND * ND;
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const uint32_t el = i / NE, rr = i - el * NE, row = rr / ND, j = rr - row * ND;
    // D = 3: the column component b runs fastest over the lanes, so consecutive lanes add to
    // consecutive CSR values (node-major interleaved columns) -- 4 lanes per 32-B sector
    // instead of one -- while the K reads stay three runs of consecutive doubles
    const uint32_t l = D == 1 ? j : j / D, b = D == 1 ? 0 : j - l * D;
    const uint32_t a = row / NB, k = row - a * NB;
    const int64_t e = e0 + el;
    const int32_t rn = dc[e * NB + k];
    const int64_t b0 = rpn[rn], nr = rpn[rn + 1] - b0;
    const int64_t p = (int64_t)D * D * b0 + (int64_t)a * D * nr + (int64_t)pos[(e * NB + k) * NB + l] * D + b;
    atomicAdd(values + p, K[(uint64_t)el * NE + row * ND + b * NB + l]);
  }
}

// Gather ("row-owner") assembly, no atomics: one warp owns one node row r of the pattern,
// accumulates in shared memory the rows k of every incident cell's K_e (node-to-cell list,
// ascending cell order) at the positions of the cell's column nodes, then adds the D rows
// (r, a) to values with coalesced read-modify-writes.  Every K_e row is read exactly once,
// every value is written once, and the summation order is fixed (bitwise reproducible).
template <typename PT, int D>
__global__ void __launch_bounds__(256) k_assemble_gather(const int64_t* __restrict__ rpn,
                                                         const int64_t* __restrict__ n2c_ptr,
                                                         const int32_t* __restrict__ n2c, int nb,
                                                         int64_t N, const PT* __restrict__ pos,
                                                         const double* __restrict__ K, int64_t e0,
                                                         int64_t e1, int hmax,
                                                         double* __restrict__ values) {
  extern __shared__ double acc_all[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  double* acc = acc_all + (size_t)warp * D * D * hmax;
  const int nd = D * nb;
  constexpr int CH = 8;  // incident cells whose K rows are loaded together
  for (int64_t r = (int64_t)blockIdx.x * nw + warp; r < N; r += (int64_t)gridDim.x * nw) {
    const int64_t b0 = rpn[r];
    const int nr = (int)(rpn[r + 1] - b0);
    for (int t = lane; t < D * D * nr; t += 32) acc[t] = 0.0;
    __syncwarp();
    const int64_t j0 = n2c_ptr[r], j1 = n2c_ptr[r + 1];
    for (int64_t jc = j0; jc < j1; jc += CH) {
      constexpr int TPL = (D * 27 + 31) / 32;  // (b, l) entries per lane for nb <= 27
      double v[CH][D][TPL];
      int jj[CH][TPL];
#pragma unroll
      for (int u = 0; u < CH; ++u) {
        const int64_t j = jc + u;
        int64_t c = -1;
        int k = 0;
        if (j < j1) {
          const int32_t ik = n2c[j];
          c = ik / nb;
          k = ik - (int)c * nb;
          if (c < e0 || c >= e1) c = -1;
        }
#pragma unroll
        for (int h = 0; h < TPL; ++h) {
          const int t = lane + 32 * h;  // t = b nb + l
          const bool on = c >= 0 && t < nd;
          const int b = t / nb, l = t - b * nb;
          jj[u][h] = on ? (int)pos[((int64_t)c * nb + k) * nb + l] * D + b : -1;
#pragma unroll
          for (int a = 0; a < D; ++a)
            v[u][a][h] = on ? K[(c - e0) * nd * nd + (int64_t)(a * nb + k) * nd + t] : 0.0;
        }
      }
#pragma unroll
      for (int u = 0; u < CH; ++u) {
#pragma unroll
        for (int h = 0; h < TPL; ++h)
          if (jj[u][h] >= 0)
#pragma unroll
            for (int a = 0; a < D; ++a) acc[a * D * nr + jj[u][h]] += v[u][a][h];
        __syncwarp();
      }
    }
    double* out = values + (int64_t)D * D * b0;
    for (int t = lane; t < D * D * nr; t += 32) out[t] += acc[t];
    __syncwarp();
  }
}

}  // namespace feb200

namespace feb200 {
fe_status set_error(fe_status s, const char* msg);
}

extern "C" {

// The CSR object's arrays come from the stream-ordered allocator and are released with
// cudaFreeAsync (no device-wide synchronisation).
static cudaError_t free_csr(fe_csr* c, cudaStream_t st = 0) {
  if (!c) return cudaSuccess;
  void* p[] = {c->rowptr_node, c->col_node, c->pos_in_row, c->n2c_ptr, c->n2c, c->rowptr, c->col};
  cudaError_t e = cudaSuccess;
  for (void* q : p)
    if (q) {
      const cudaError_t ee = cudaFreeAsync(q, st);
      if (e == cudaSuccess) e = ee;
    }
  delete c;
  return e;
}

static fe_status create_csr_impl(const fe_mesh* mesh, int32_t ncomp, void* stream, fe_csr** out);

fe_status fe_create_csr(const fe_mesh* mesh, int32_t ncomp, void* stream, fe_csr** out) {
  FE_NVTX_RANGE("fe_create_csr");
  try {  // thrust reports failures with exceptions; none may cross the ABI
    return create_csr_impl(mesh, ncomp, stream, out);
  } catch (const std::bad_alloc&) {
    return feb200::set_error(FE_ERR_OOM, "fe_create_csr: out of memory in sort");
  } catch (const std::exception& ex) {
    return feb200::set_error(FE_ERR_CUDA, ex.what());
  } catch (...) {
    return feb200::set_error(FE_ERR_CUDA, "fe_create_csr: unknown failure");
  }
}

static fe_status create_csr_impl(const fe_mesh* mesh, int32_t ncomp, void* stream, fe_csr** out) {
  if (!mesh || !out || (ncomp != 1 && ncomp != 3))
    return feb200::set_error(FE_ERR_INVALID_ARG, "fe_create_csr: NULL argument or ncomp not in {1, 3}");
  *out = nullptr;
  cudaStream_t st = (cudaStream_t)stream;
  const int nb = mesh->nb;
  const int64_t E = mesh->n_elems, N = mesh->n_nodes, npairs = E * nb * nb;
  if (N * ncomp >= (int64_t(1) << 31) || npairs <= 0)
    return feb200::set_error(FE_ERR_UNSUPPORTED, "fe_create_csr: empty mesh or > 2^31 rows");
  fe_csr* c = new fe_csr();
  c->mesh = mesh;
  c->ncomp = ncomp;
  c->n_nodes = N;
  int64_t* keys = nullptr;
  cudaError_t e = cudaMalloc(&keys, sizeof(int64_t) * npairs);
  if (e != cudaSuccess) { free_csr(c, st); return feb200::set_error(FE_ERR_OOM, "fe_create_csr: keys"); }
  const int grid = 148 * 16;
  feb200::k_pair_keys<<<grid, 256, 0, st>>>(mesh->dof_conn, nb, E, N, keys);
  feb200::count_launch();
  auto pol = thrust::cuda::par.on(st);
  thrust::device_ptr<int64_t> kp(keys);
  thrust::sort(pol, kp, kp + npairs);
  const int64_t nnz = thrust::unique(pol, kp, kp + npairs) - kp;
  c->nnz_node = nnz;
  e = cudaMallocAsync((void**)&c->rowptr_node, sizeof(int64_t) * (N + 1), st);
  if (e == cudaSuccess) e = cudaMallocAsync((void**)&c->col_node, sizeof(int32_t) * nnz, st);
  if (e != cudaSuccess) { cudaFree(keys); free_csr(c, st); return feb200::set_error(FE_ERR_OOM, "fe_create_csr: pattern"); }
  // rowptr_node[r] = first key >= r * N
  thrust::device_ptr<int64_t> rp(c->rowptr_node);
  auto row_keys = thrust::make_transform_iterator(thrust::make_counting_iterator<int64_t>(0),
                                                  feb200::RowKey{N});
  thrust::lower_bound(pol, kp, kp + nnz, row_keys, row_keys + N + 1, rp);
  feb200::k_cols<<<grid, 256, 0, st>>>(keys, nnz, N, c->col_node);
  feb200::count_launch();
  unsigned long long* dmax = nullptr;
  unsigned long long hmax = 0;
  e = cudaMalloc(&dmax, sizeof(unsigned long long));
  if (e == cudaSuccess) e = cudaMemsetAsync(dmax, 0, sizeof(unsigned long long), st);
  if (e == cudaSuccess) {
    feb200::k_max_row<<<grid, 256, 0, st>>>(c->rowptr_node, N, dmax);
    feb200::count_launch();
    e = cudaMemcpyAsync(&hmax, dmax, sizeof(hmax), cudaMemcpyDeviceToHost, st);
  }
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  if (dmax) cudaFree(dmax);
  c->pos_bytes = hmax <= 256 ? 1 : (hmax <= 65536 ? 2 : 4);
  if (e == cudaSuccess) e = cudaMallocAsync((void**)&c->pos_in_row, (size_t)c->pos_bytes * npairs, st);
  if (e != cudaSuccess) { cudaFree(keys); free_csr(c, st); return feb200::set_error(FE_ERR_OOM, "fe_create_csr: position map"); }
  if (c->pos_bytes == 1)
    feb200::k_pos_map<uint8_t><<<grid, 256, 0, st>>>(mesh->dof_conn, nb, E, c->rowptr_node, c->col_node, (uint8_t*)c->pos_in_row);
  else if (c->pos_bytes == 2)
    feb200::k_pos_map<uint16_t><<<grid, 256, 0, st>>>(mesh->dof_conn, nb, E, c->rowptr_node, c->col_node, (uint16_t*)c->pos_in_row);
  else
    feb200::k_pos_map<int32_t><<<grid, 256, 0, st>>>(mesh->dof_conn, nb, E, c->rowptr_node, c->col_node, (int32_t*)c->pos_in_row);
  feb200::count_launch();
  c->hmax = (int)hmax;
  // node -> (cell, local node) list: stable key sort of the dof_conn entries by node
  {
    const int64_t ne = E * nb;
    int32_t* nkeys = nullptr;
    e = cudaMalloc(&nkeys, sizeof(int32_t) * ne);
    if (e == cudaSuccess) e = cudaMallocAsync((void**)&c->n2c, sizeof(int32_t) * ne, st);
    if (e == cudaSuccess) e = cudaMallocAsync((void**)&c->n2c_ptr, sizeof(int64_t) * (N + 1), st);
    if (e != cudaSuccess) {
      if (nkeys) cudaFree(nkeys);
      cudaFree(keys);
      free_csr(c, st);
      return feb200::set_error(FE_ERR_OOM, "fe_create_csr: node-to-cell list");
    }
    thrust::device_ptr<int32_t> nk(nkeys), nv(c->n2c);
    thrust::copy(pol, thrust::device_ptr<const int32_t>(mesh->dof_conn),
                 thrust::device_ptr<const int32_t>(mesh->dof_conn) + ne, nk);
    thrust::sequence(pol, nv, nv + ne);
    thrust::stable_sort_by_key(pol, nk, nk + ne, nv);
    thrust::lower_bound(pol, nk, nk + ne, thrust::make_counting_iterator<int32_t>(0),
                        thrust::make_counting_iterator<int32_t>((int32_t)N + 1),
                        thrust::device_ptr<int64_t>(c->n2c_ptr));
    cudaStreamSynchronize(st);
    cudaFree(nkeys);
  }
  e = cudaMallocAsync((void**)&c->rowptr, sizeof(int64_t) * (N * ncomp + 1), st);
  if (e == cudaSuccess) e = cudaMallocAsync((void**)&c->col, sizeof(int32_t) * nnz * ncomp * ncomp, st);
  if (e != cudaSuccess) { cudaFree(keys); free_csr(c, st); return feb200::set_error(FE_ERR_OOM, "fe_create_csr: expanded pattern"); }
  feb200::k_expand<<<grid, 256, 0, st>>>(c->rowptr_node, c->col_node, N, ncomp, c->rowptr, c->col);
  feb200::count_launch();
  e = cudaStreamSynchronize(st);
  cudaFree(keys);
  if (e != cudaSuccess) { free_csr(c, st); return feb200::set_error(FE_ERR_CUDA, cudaGetErrorString(e)); }
  *out = c;
  return feb200::set_error(FE_OK, "");
}

fe_status fe_csr_info(const fe_csr* csr, int64_t* n_rows, int64_t* nnz) {
  if (!csr) return feb200::set_error(FE_ERR_INVALID_ARG, "csr is NULL");
  if (n_rows) *n_rows = csr->n_nodes * csr->ncomp;
  if (nnz) *nnz = csr->nnz_node * csr->ncomp * csr->ncomp;
  return FE_OK;
}

fe_status fe_csr_arrays(const fe_csr* csr, const int64_t** row_ptr, const int32_t** col_idx) {
  if (!csr) return feb200::set_error(FE_ERR_INVALID_ARG, "csr is NULL");
  if (row_ptr) *row_ptr = csr->rowptr;
  if (col_idx) *col_idx = csr->col;
  return FE_OK;
}

fe_status fe_csr_copy_arrays(const fe_csr* csr, int64_t* row_ptr, int32_t* col_idx, void* stream) {
  FE_NVTX_RANGE("fe_csr_copy_arrays");
  if (!csr) return feb200::set_error(FE_ERR_INVALID_ARG, "csr is NULL");
  cudaStream_t st = (cudaStream_t)stream;
  cudaError_t e = cudaSuccess;
  const int64_t nr = csr->n_nodes * csr->ncomp, nz = csr->nnz_node * csr->ncomp * csr->ncomp;
  if (row_ptr) e = cudaMemcpyAsync(row_ptr, csr->rowptr, sizeof(int64_t) * (nr + 1), cudaMemcpyDefault, st);
  if (e == cudaSuccess && col_idx) e = cudaMemcpyAsync(col_idx, csr->col, sizeof(int32_t) * nz, cudaMemcpyDefault, st);
  return e == cudaSuccess ? feb200::set_error(FE_OK, "") : feb200::set_error(FE_ERR_CUDA, cudaGetErrorString(e));
}

fe_status fe_assemble_matrix(const fe_csr* csr, const double* K, int64_t elem_begin, int64_t elem_end,
                             double* values, void* stream) {
  FE_NVTX_RANGE("fe_assemble_matrix");
  if (!csr || (!K && elem_end > elem_begin) || !values)
    return feb200::set_error(FE_ERR_INVALID_ARG, "fe_assemble_matrix: NULL argument");
  if (elem_begin < 0 || elem_end > csr->mesh->n_elems || elem_begin > elem_end)
    return feb200::set_error(FE_ERR_INVALID_ARG, "fe_assemble_matrix: bad element range");
  const int nd = csr->ncomp * csr->mesh->nb;
  const int64_t n = (elem_end - elem_begin) * nd * nd;
  if (n == 0) return FE_OK;
  const int grid = (int)((n + 255) / 256 < 148 * 32 ? (n + 255) / 256 : 148 * 32);
  // default: fp64 atomics (fastest on B200); FE_OPT_CSR_IMPL = 1 (gather) selects the
  // atomic-free row-owner kernel (fixed summation order, bitwise reproducible; nb <= 27)
  const bool atomic = feb200::option(FE_OPT_CSR_IMPL) == 0 || csr->mesh->nb > 27;
  const int D = csr->ncomp;
  const size_t smem = (size_t)8 * D * D * csr->hmax * 8;  // 8 warps per block
  auto launch = [&](auto* pos) {
    // 32-bit loop index: i + gridDim*blockDim must not wrap past 2^32 on the last stride
    if (atomic && csr->mesh->nb == 27 && n <= int64_t(UINT32_MAX) - int64_t(grid) * 256 &&
        FEB200_CSR_CONST) {
      using PT = std::remove_const_t<std::remove_pointer_t<decltype(pos)>>;
      if (D == 1)
        feb200::k_assemble_matrix_c<PT, 27, 1><<<grid, 256, 0, (cudaStream_t)stream>>>(
            csr->mesh->dof_conn, elem_begin, (uint32_t)n, csr->rowptr_node, pos, K, values);
      else
        feb200::k_assemble_matrix_c<PT, 27, 3><<<grid, 256, 0, (cudaStream_t)stream>>>(
            csr->mesh->dof_conn, elem_begin, (uint32_t)n, csr->rowptr_node, pos, K, values);
      return;
    }
    if (atomic) {
      feb200::k_assemble_matrix<<<grid, 256, 0, (cudaStream_t)stream>>>(
          csr->mesh->dof_conn, csr->mesh->nb, csr->ncomp, elem_begin, elem_end, csr->rowptr_node, pos, K,
          values);
      return;
    }
    using PT = std::remove_const_t<std::remove_pointer_t<decltype(pos)>>;
    auto kern = D == 1 ? feb200::k_assemble_gather<PT, 1> : feb200::k_assemble_gather<PT, 3>;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    const int64_t rows = csr->n_nodes;
    const int g = (int)std::min<int64_t>((rows + 7) / 8, 148 * 64);
    kern<<<g, 256, smem, (cudaStream_t)stream>>>(csr->rowptr_node, csr->n2c_ptr, csr->n2c, csr->mesh->nb,
                                                 rows, pos, K, elem_begin, elem_end, csr->hmax, values);
  };
  if (csr->pos_bytes == 1) launch((const uint8_t*)csr->pos_in_row);
  else if (csr->pos_bytes == 2) launch((const uint16_t*)csr->pos_in_row);
  else launch((const int32_t*)csr->pos_in_row);
  feb200::count_launch();
  const cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? feb200::set_error(FE_OK, "") : feb200::set_error(FE_ERR_CUDA, cudaGetErrorString(e));
}

fe_status fe_destroy_csr(fe_csr* csr, void* stream) {
  FE_NVTX_RANGE("fe_destroy_csr");
  if (!csr) return feb200::set_error(FE_OK, "");
  const cudaError_t e = free_csr(csr, (cudaStream_t)stream);
  return e == cudaSuccess ? feb200::set_error(FE_OK, "")
                          : feb200::set_error(FE_ERR_CUDA, cudaGetErrorString(e));
}

}  // extern "C"
