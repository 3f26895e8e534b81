// Micro-benchmark of per-SM issue rates that bound the FE kernels: warp shuffles vs shared
// loads (both go through the MIO path) and FP64 FMA latency / throughput.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/mb tools/mb_pipes.cu && /tmp/mb
#include <cstdio>
#include <cuda_runtime.h>

constexpr int ITERS = 4096;

__global__ void k_shfl(double* out, int seed) {
  double a0 = threadIdx.x + seed, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3;
  const int l = threadIdx.x & 31;
#pragma unroll 4
  for (int i = 0; i < ITERS; ++i) {
    a0 = __shfl_sync(0xffffffffu, a0, (l + 1) & 31);
    a1 = __shfl_sync(0xffffffffu, a1, (l + 3) & 31);
    a2 = __shfl_sync(0xffffffffu, a2, (l + 5) & 31);
    a3 = __shfl_sync(0xffffffffu, a3, (l + 7) & 31);
  }
  if (a0 + a1 + a2 + a3 == -1.0) out[0] = a0;
}
__global__ void k_lds64(double* out, int seed) {
  __shared__ double s[1024];
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) s[i] = i + seed;
  __syncthreads();
  double acc = 0;
  int idx = threadIdx.x & 31;
#pragma unroll 4
  for (int i = 0; i < ITERS; ++i) {
    double v0 = s[idx], v1 = s[idx + 32], v2 = s[idx + 64], v3 = s[idx + 96];
    acc += v0 + v1 + v2 + v3;
    idx = (idx + 128 + (int)v0 * 0) & 511;
  }
  if (acc == -1.0) out[0] = acc;
}
__global__ void k_lds64_bcast(double* out, int seed) {
  __shared__ double s[1024];
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) s[i] = i + seed;
  __syncthreads();
  double acc = 0;
  int idx = (threadIdx.x >> 5) * 4;
#pragma unroll 4
  for (int i = 0; i < ITERS; ++i) {
    double v0 = s[idx], v1 = s[idx + 1], v2 = s[idx + 2], v3 = s[idx + 3];
    acc += v0 + v1 + v2 + v3;
    idx = (idx + 64 + (int)v0 * 0) & 511;
  }
  if (acc == -1.0) out[0] = acc;
}
// LDS.128 with `ndist` distinct 16-B addresses per warp (lanes grouped), dependent chain
template <int NDIST>
__global__ void k_lds128(double* out, int seed) {
  __shared__ double2 s[2048];
  for (int i = threadIdx.x; i < 2048; i += blockDim.x) s[i] = make_double2(i + seed, 0.0);
  __syncthreads();
  double acc = 0;
  const int l = threadIdx.x & 31;
  int idx = (l * NDIST / 32) * 1 + (threadIdx.x >> 5) * 64;
#pragma unroll 4
  for (int i = 0; i < ITERS; ++i) {
    double2 v0 = s[idx], v1 = s[idx + 8], v2 = s[idx + 16], v3 = s[idx + 24];
    acc += v0.x + v1.y + v2.x + v3.y;
    idx = (idx + 32 + (int)(v0.y + v1.y + v2.y + v3.y)) & 2047;
  }
  if (acc == -1.0) out[0] = acc;
}
__global__ void k_dfma_thru(double* out, int seed) {
  double a[8];
  for (int k = 0; k < 8; ++k) a[k] = threadIdx.x + k + seed;
  const double b = 1.0000001, c = 1e-9;
#pragma unroll 4
  for (int i = 0; i < ITERS; ++i)
#pragma unroll
    for (int k = 0; k < 8; ++k) a[k] = fma(a[k], b, c);
  double s = 0;
  for (int k = 0; k < 8; ++k) s += a[k];
  if (s == -1.0) out[0] = s;
}
__global__ void k_dfma_lat(double* out, long long* cyc, int seed) {
  double a = threadIdx.x + seed;
  const double b = 1.0000001, c = 1e-9;
  long long t0 = clock64();
#pragma unroll 8
  for (int i = 0; i < ITERS; ++i) a = fma(a, b, c);
  long long t1 = clock64();
  if (threadIdx.x == 0 && blockIdx.x == 0) cyc[0] = t1 - t0;
  if (a == -1.0) out[0] = a;
}

int main() {
  double* out;
  long long* cyc;
  cudaMalloc(&out, 8);
  cudaMalloc(&cyc, 8);
  int dev = 0, clk = 0, nsm = 0;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  auto timeit = [&](const char* name, auto launch, double ops_per_thread, int threads) {
    for (int w = 0; w < 3; ++w) launch();
    cudaEventRecord(e0);
    for (int r = 0; r < 10; ++r) launch();
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double s = ms * 1e-3 / 10;
    const double warp_ops = ops_per_thread * threads / 32.0 * nsm;
    printf("%-14s %8.3f ms  %7.3f warp-instr/clk/SM (clk %.0f MHz nominal)\n", name, ms / 10,
           warp_ops / s / nsm / (clk * 1e3), clk / 1e3);
  };
  const int T = 512;
  timeit("shfl.f64", [&] { k_shfl<<<nsm * 2, T>>>(out, 1); }, 4.0 * 2 * ITERS, T * 2);
  timeit("lds.64", [&] { k_lds64<<<nsm * 2, T>>>(out, 1); }, 4.0 * ITERS, T * 2);
  timeit("lds.64 bcast", [&] { k_lds64_bcast<<<nsm * 2, T>>>(out, 1); }, 4.0 * ITERS, T * 2);
  timeit("lds.128 d1", [&] { k_lds128<1><<<nsm * 2, T>>>(out, 1); }, 4.0 * ITERS, T * 2);
  timeit("lds.128 d4", [&] { k_lds128<4><<<nsm * 2, T>>>(out, 1); }, 4.0 * ITERS, T * 2);
  timeit("lds.128 d8", [&] { k_lds128<8><<<nsm * 2, T>>>(out, 1); }, 4.0 * ITERS, T * 2);
  timeit("lds.128 d32", [&] { k_lds128<32><<<nsm * 2, T>>>(out, 1); }, 4.0 * ITERS, T * 2);
  timeit("dfma", [&] { k_dfma_thru<<<nsm * 2, T>>>(out, 1); }, 8.0 * ITERS, T * 2);
  k_dfma_lat<<<1, 32>>>(out, cyc, 1);
  long long c;
  cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
  printf("dfma dependent latency: %.2f cycles\n", (double)c / ITERS);
  return 0;
}
