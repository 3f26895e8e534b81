// FP64 peak microbenchmark for B200 (sm_100a): sustained DFMA and DMMA
// (mma.sync f64) throughput. Produces the FP64 roofline denominator that
// MEASURED_PEAKS.json does not carry. Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3
#include <cstdio>
#include <cuda_runtime.h>
#include <chrono>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

template <int CHAINS>
__global__ void dfma_loop(double* out, long iters, double a, double b) {
  double acc[CHAINS];
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) acc[c] = threadIdx.x * 1e-9 + c;
  for (long i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) acc[c] = fma(acc[c], a, b);
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) s += acc[c];
  if (s == 12345.678) out[0] = s;
}

// m8n8k4 f64: A 1 reg, B 1 reg, C/D 2 regs per thread; 256 FMA per warp-instr
__global__ void dmma_m8n8k4(double* out, long iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 - threadIdx.x * 1e-4;
  double c[4][2];
#pragma unroll
  for (int t = 0; t < 4; ++t) { c[t][0] = 0; c[t][1] = 0; }
  for (long i = 0; i < iters; ++i) {
#pragma unroll
    for (int t = 0; t < 4; ++t)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(c[t][0]), "+d"(c[t][1]) : "d"(a), "d"(b));
  }
  double s = 0;
#pragma unroll
  for (int t = 0; t < 4; ++t) s += c[t][0] + c[t][1];
  if (s == 12345.678) out[0] = s;
}

// m16n8k4 f64: A 2, B 1, C 4 ; 512 FMA
__global__ void dmma_m16n8k4(double* out, long iters) {
  double a0 = threadIdx.x * 1e-3, a1 = a0 + 1, b = 1.0 - threadIdx.x * 1e-4;
  double c[4][4];
#pragma unroll
  for (int t = 0; t < 4; ++t) for (int r = 0; r < 4; ++r) c[t][r] = 0;
  for (long i = 0; i < iters; ++i) {
#pragma unroll
    for (int t = 0; t < 4; ++t)
      asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};"
                   : "+d"(c[t][0]), "+d"(c[t][1]), "+d"(c[t][2]), "+d"(c[t][3]) : "d"(a0), "d"(a1), "d"(b));
  }
  double s = 0;
#pragma unroll
  for (int t = 0; t < 4; ++t) s += c[t][0] + c[t][1] + c[t][2] + c[t][3];
  if (s == 12345.678) out[0] = s;
}

// m16n8k16 f64: A 8, B 4, C 4 ; 2048 FMA
__global__ void dmma_m16n8k16(double* out, long iters) {
  double a[8], b[4];
#pragma unroll
  for (int r = 0; r < 8; ++r) a[r] = threadIdx.x * 1e-3 + r;
#pragma unroll
  for (int r = 0; r < 4; ++r) b[r] = 1.0 - threadIdx.x * 1e-4 * r;
  double c[2][4];
#pragma unroll
  for (int t = 0; t < 2; ++t) for (int r = 0; r < 4; ++r) c[t][r] = 0;
  for (long i = 0; i < iters; ++i) {
#pragma unroll
    for (int t = 0; t < 2; ++t)
      asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};"
                   : "+d"(c[t][0]), "+d"(c[t][1]), "+d"(c[t][2]), "+d"(c[t][3])
                   : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]),
                     "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
  }
  double s = 0;
#pragma unroll
  for (int t = 0; t < 2; ++t) s += c[t][0] + c[t][1] + c[t][2] + c[t][3];
  if (s == 12345.678) out[0] = s;
}

template <typename F>
static double time_kernel(F launch, int reps) {
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  launch();  // warm
  cudaDeviceSynchronize();
  cudaEventRecord(e0);
  for (int r = 0; r < reps; ++r) launch();
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  return ms / reps;
}

int main(int argc, char** argv) {
  double sustain_s = argc > 1 ? atof(argv[1]) : 4.0;
  int nsm; cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  double* out; CK(cudaMalloc(&out, 8));
  printf("{\"sms\": %d", nsm);
  for (int bpsm : {1, 2, 4, 8}) {
    int threads = 256; long iters = 1 << 16; int grid = nsm * bpsm;
    double ms = time_kernel([&] { dfma_loop<8><<<grid, threads>>>(out, iters, 1.0000001, 1e-9); }, 5);
    double tf = 2.0 * 8 * iters * (double)grid * threads / (ms * 1e-3) / 1e12;
    printf(", \"dfma_tflops_bpsm%d\": %.2f", bpsm, tf);
  }
  CK(cudaGetLastError());
  for (int bpsm : {1, 2, 4, 8}) {
    int threads = 256; long iters = 1 << 14; int grid = nsm * bpsm;
    double ms = time_kernel([&] { dmma_m8n8k4<<<grid, threads>>>(out, iters); }, 5);
    double tf = 2.0 * 256 * 4 * iters * (double)grid * (threads / 32) / (ms * 1e-3) / 1e12;
    printf(", \"dmma_m8n8k4_tflops_bpsm%d\": %.2f", bpsm, tf);
    ms = time_kernel([&] { dmma_m16n8k4<<<grid, threads>>>(out, iters); }, 5);
    tf = 2.0 * 512 * 4 * iters * (double)grid * (threads / 32) / (ms * 1e-3) / 1e12;
    printf(", \"dmma_m16n8k4_tflops_bpsm%d\": %.2f", bpsm, tf);
    ms = time_kernel([&] { dmma_m16n8k16<<<grid, threads>>>(out, iters / 4); }, 5);
    tf = 2.0 * 2048 * 2 * (iters / 4) * (double)grid * (threads / 32) / (ms * 1e-3) / 1e12;
    printf(", \"dmma_m16n8k16_tflops_bpsm%d\": %.2f", bpsm, tf);
  }
  CK(cudaGetLastError());
  // sustained: back-to-back DFMA for sustain_s seconds
  {
    int threads = 256, grid = nsm * 4; long iters = 1 << 16;
    double ms1 = time_kernel([&] { dfma_loop<8><<<grid, threads>>>(out, iters, 1.0000001, 1e-9); }, 3);
    int reps = (int)(sustain_s * 1e3 / ms1) + 1;
    double ms = time_kernel([&] { dfma_loop<8><<<grid, threads>>>(out, iters, 1.0000001, 1e-9); }, reps);
    double tf = 2.0 * 8 * iters * (double)grid * threads / (ms * 1e-3) / 1e12;
    printf(", \"dfma_tflops_sustained\": %.2f, \"sustained_s\": %.2f", tf, ms * reps * 1e-3);
    ms1 = time_kernel([&] { dmma_m16n8k4<<<grid, threads>>>(out, iters / 4); }, 3);
    reps = (int)(sustain_s * 1e3 / ms1) + 1;
    ms = time_kernel([&] { dmma_m16n8k4<<<grid, threads>>>(out, iters / 4); }, reps);
    tf = 2.0 * 512 * 4 * (iters / 4) * (double)grid * (threads / 32) / (ms * 1e-3) / 1e12;
    printf(", \"dmma_m16n8k4_tflops_sustained\": %.2f", tf);
  }
  CK(cudaGetLastError());
  printf("}\n");
  return 0;
}
