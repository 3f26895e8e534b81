// Element-kind grouping (a rectangular einsum call covers cells
// "of the same shape and approximation order"; p- / hp-adaptive meshes "would require an
// additional sorting/grouping of the same element kinds together").
//
// fe_group_cells: a stable sort of the cell ids by kind on the GPU (thrust stable key sort of
// (kind, id) pairs), then the group boundaries by binary search of the sorted kinds.
// fe_gather_rows_*: dense [n][width] blocks gathered from a (possibly ragged, CSR-addressed)
// per-cell array in grouped order -- the connectivity, DOF and material rows of each group,
// which then go through the single-kind kernels unchanged.
#include <thrust/binary_search.h>
#include <thrust/device_ptr.h>
#include <thrust/execution_policy.h>
#include <thrust/iterator/counting_iterator.h>
#include <thrust/sequence.h>
#include <thrust/sort.h>

#include <new>
#include <vector>

#include "fe_internal.h"

namespace feb200 {
fe_status set_error(fe_status s, const char* msg);

template <typename T>
__global__ void k_gather_rows(const T* __restrict__ in, const int64_t* __restrict__ row_ptr, int width,
                              const int64_t* __restrict__ perm, int64_t n, T* __restrict__ out) {
  const int64_t total = n * width;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / width, j = i - r * width;
    const int64_t src = perm[r];
    out[i] = in[(row_ptr ? row_ptr[src] : src * width) + j];
  }
}

template <typename T>
static fe_status gather_rows(const T* in, const int64_t* row_ptr, int32_t width, const int64_t* perm,
                             int64_t n, T* out, void* stream) {
  if (n < 0 || width < 0) return set_error(FE_ERR_INVALID_ARG, "fe_gather_rows: negative size");
  if (n == 0 || width == 0) return set_error(FE_OK, "");
  if (!in || !perm || !out) return set_error(FE_ERR_INVALID_ARG, "fe_gather_rows: NULL argument");
  const int64_t total = n * width;
  const int64_t want = (total + 255) / 256;
  const int grid = (int)(want < 148 * 16 ? want : 148 * 16);
  k_gather_rows<T><<<grid, 256, 0, (cudaStream_t)stream>>>(in, row_ptr, width, perm, n, out);
  count_launch();
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return set_error(FE_ERR_CUDA, cudaGetErrorString(e));
  return set_error(FE_OK, "");
}

static fe_status group_cells_impl(const int32_t* kind, int64_t n, int32_t n_kinds, int64_t* perm,
                                  int64_t* offsets, void* stream) {
  if (n < 0 || n_kinds < 1 || !offsets || (n > 0 && (!kind || !perm)))
    return set_error(FE_ERR_INVALID_ARG, "fe_group_cells: bad argument");
  if (n == 0) {
    for (int k = 0; k <= n_kinds; ++k) offsets[k] = 0;
    return set_error(FE_OK, "");
  }
  cudaStream_t st = (cudaStream_t)stream;
  int32_t* keys = nullptr;
  cudaError_t e = cudaMalloc(&keys, sizeof(int32_t) * n);
  if (e != cudaSuccess) return set_error(FE_ERR_OOM, "fe_group_cells: keys");
  int64_t* dofs = nullptr;
  e = cudaMalloc(&dofs, sizeof(int64_t) * (n_kinds + 1));
  if (e != cudaSuccess) {
    cudaFree(keys);
    return set_error(FE_ERR_OOM, "fe_group_cells: offsets");
  }
  cudaMemcpyAsync(keys, kind, sizeof(int32_t) * n, cudaMemcpyDefault, st);
  auto pol = thrust::cuda::par.on(st);
  thrust::device_ptr<int32_t> kp(keys);
  thrust::device_ptr<int64_t> pp(perm);
  thrust::sequence(pol, pp, pp + n);
  thrust::stable_sort_by_key(pol, kp, kp + n, pp);  // stable: ascending ids within a kind
  thrust::lower_bound(pol, kp, kp + n, thrust::counting_iterator<int32_t>(0),
                      thrust::counting_iterator<int32_t>(n_kinds + 1), thrust::device_ptr<int64_t>(dofs));
  int32_t lohi[2] = {0, 0};
  cudaMemcpyAsync(&lohi[0], keys, sizeof(int32_t), cudaMemcpyDeviceToHost, st);
  cudaMemcpyAsync(&lohi[1], keys + n - 1, sizeof(int32_t), cudaMemcpyDeviceToHost, st);
  cudaMemcpyAsync(offsets, dofs, sizeof(int64_t) * (n_kinds + 1), cudaMemcpyDeviceToHost, st);
  e = cudaStreamSynchronize(st);
  cudaFree(keys);
  cudaFree(dofs);
  if (e != cudaSuccess) return set_error(FE_ERR_CUDA, cudaGetErrorString(e));
  if (lohi[0] < 0 || lohi[1] >= n_kinds)
    return set_error(FE_ERR_INVALID_ARG, "fe_group_cells: kind outside [0, n_kinds)");
  offsets[n_kinds] = n;
  return set_error(FE_OK, "");
}

}  // namespace feb200

extern "C" {

fe_status fe_group_cells(const int32_t* kind, int64_t n_cells, int32_t n_kinds, int64_t* perm,
                         int64_t* offsets, void* stream) {
  FE_NVTX_RANGE("fe_group_cells");
  try {  // thrust reports failures with exceptions; none may cross the ABI
    return feb200::group_cells_impl(kind, n_cells, n_kinds, perm, offsets, stream);
  } catch (const std::bad_alloc&) {
    return feb200::set_error(FE_ERR_OOM, "fe_group_cells: out of memory in sort");
  } catch (const std::exception& ex) {
    return feb200::set_error(FE_ERR_CUDA, ex.what());
  } catch (...) {
    return feb200::set_error(FE_ERR_CUDA, "fe_group_cells: unknown failure");
  }
}

fe_status fe_gather_rows_i32(const int32_t* in, const int64_t* row_ptr, int32_t width,
                             const int64_t* perm, int64_t n, int32_t* out, void* stream) {
  FE_NVTX_RANGE("fe_gather_rows_i32");
  return feb200::gather_rows<int32_t>(in, row_ptr, width, perm, n, out, stream);
}

fe_status fe_gather_rows_f64(const double* in, const int64_t* row_ptr, int32_t width,
                             const int64_t* perm, int64_t n, double* out, void* stream) {
  FE_NVTX_RANGE("fe_gather_rows_f64");
  return feb200::gather_rows<double>(in, row_ptr, width, perm, n, out, stream);
}

}  // extern "C"
