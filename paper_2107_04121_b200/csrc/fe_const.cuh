// 1D reference tables in __constant__ memory, one copy per translation unit
// (whole-program compilation: a __constant__ symbol is private to its TU, so every
// kernel unit that reads it exposes its own upload function, called at mesh creation).
// c_tab1d[p][a][q][i] = B^a[q][i]: a = 0 values, 1 derivatives of the 1D Lagrange
// basis of order p at the q1d = p+1 Gauss points; the values depend only on p.
#pragma once
#include <cuda_runtime.h>

namespace feb200 {
namespace {
__constant__ double c_tab1d[5][2][5][5];
__constant__ double c_x1d[5][5];  // 1D Gauss points on [0,1]
__constant__ double c_w1d[5][5];  // 1D Gauss weights

cudaError_t upload_tables_this_tu(int order, const double* b1, const double* d1, const double* x1,
                                  const double* w1, cudaStream_t st) {
  if (order < 1 || order > 4) return cudaSuccess;
  double h[2][5][5] = {}, hx[5] = {}, hw[5] = {};
  const int n1 = order + 1, q1 = order + 1;
  for (int q = 0; q < q1; ++q) {
    hx[q] = x1[q];
    hw[q] = w1[q];
    for (int i = 0; i < n1; ++i) {
      h[0][q][i] = b1[q * n1 + i];
      h[1][q][i] = d1[q * n1 + i];
    }
  }
  cudaError_t e = cudaMemcpyToSymbolAsync(c_tab1d, h, sizeof(h), sizeof(h) * order,
                                          cudaMemcpyHostToDevice, st);
  if (e == cudaSuccess)
    e = cudaMemcpyToSymbolAsync(c_x1d, hx, sizeof(hx), sizeof(hx) * order, cudaMemcpyHostToDevice, st);
  if (e == cudaSuccess)
    e = cudaMemcpyToSymbolAsync(c_w1d, hw, sizeof(hw), sizeof(hw) * order, cudaMemcpyHostToDevice, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  return e;
}
}  // namespace
}  // namespace feb200
