// FP64 peak probe for B200 (sm_100a): DFMA vector pipe, DMMA (mma.sync m8n8k4 f64)
// and both interleaved in one warp.  Used to pick the Legendre-stage inner loop
// (SURVEY.md §7 "FP64 rate"); results go to profiles/fp64_peak_*.txt.
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); return 1; } } while (0)

constexpr int ITERS = 4096;

__global__ void k_dfma(double* out, double a, double b) {
  double x[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) x[k] = threadIdx.x * 1e-3 + k;
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int k = 0; k < 8; ++k) x[k] = fma(x[k], a, b);
  }
  double s = 0;
#pragma unroll
  for (int k = 0; k < 8; ++k) s += x[k];
  if (s == 12345.678) out[threadIdx.x] = s;
}

__device__ __forceinline__ void dmma(double (&d)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d[0]), "+d"(d[1]) : "d"(a), "d"(b));
}

__global__ void k_dmma(double* out, double a, double b) {
  double acc[8][2];
#pragma unroll
  for (int k = 0; k < 8; ++k) { acc[k][0] = k; acc[k][1] = -k; }
  double av = a + threadIdx.x * 1e-9, bv = b - threadIdx.x * 1e-9;
  for (int it = 0; it < ITERS / 8; ++it) {
#pragma unroll
    for (int k = 0; k < 8; ++k) dmma(acc[k], av, bv);
  }
  double s = 0;
#pragma unroll
  for (int k = 0; k < 8; ++k) s += acc[k][0] + acc[k][1];
  if (s == 12345.678) out[threadIdx.x] = s;
}

// the analysis k-step's operand pattern: 16 accumulators acc[p][mt][n],
// A changes every 4 DMMAs (p, mt), B differs per (p, n) -- all in registers
__global__ void k_dmma_ana(double* out, double a, double b) {
  double acc[2][2][4][2];
  double av[2][2], bv[2][4];
#pragma unroll
  for (int p = 0; p < 2; ++p) {
#pragma unroll
    for (int m = 0; m < 2; ++m) av[p][m] = a + (p * 2 + m + threadIdx.x) * 1e-9;
#pragma unroll
    for (int n = 0; n < 4; ++n) bv[p][n] = b - (p * 4 + n + threadIdx.x) * 1e-9;
#pragma unroll
    for (int m = 0; m < 2; ++m)
#pragma unroll
      for (int n = 0; n < 4; ++n) { acc[p][m][n][0] = n; acc[p][m][n][1] = -n; }
  }
  for (int it = 0; it < ITERS / 16; ++it) {
#pragma unroll
    for (int p = 0; p < 2; ++p)
#pragma unroll
      for (int m = 0; m < 2; ++m)
#pragma unroll
        for (int n = 0; n < 4; ++n) dmma(acc[p][m][n], av[p][m], bv[p][n]);
  }
  double s = 0;
#pragma unroll
  for (int p = 0; p < 2; ++p)
#pragma unroll
    for (int m = 0; m < 2; ++m)
#pragma unroll
      for (int n = 0; n < 4; ++n) s += acc[p][m][n][0] + acc[p][m][n][1];
  if (s == 12345.678) out[threadIdx.x] = s;
}

// interleave: per iteration 1 DMMA (256 FMA/warp) + NF DFMA per thread
template <int NF>
__global__ void k_mixed(double* out, double a, double b) {
  double acc[8][2];
  double x[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) { acc[k][0] = k; acc[k][1] = -k; x[k] = threadIdx.x * 1e-3 + k; }
  double av = a + threadIdx.x * 1e-9, bv = b - threadIdx.x * 1e-9;
  for (int it = 0; it < ITERS / 8; ++it) {
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      dmma(acc[k], av, bv);
#pragma unroll
      for (int f = 0; f < NF; ++f) x[(k + f) & 7] = fma(x[(k + f) & 7], a, b);
    }
  }
  double s = 0;
#pragma unroll
  for (int k = 0; k < 8; ++k) s += acc[k][0] + acc[k][1] + x[k];
  if (s == 12345.678) out[threadIdx.x] = s;
}

template <typename K>
float timeit(K kern, int blocks, int threads, double* out) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int w = 0; w < 3; ++w) kern<<<blocks, threads>>>(out, 0.999999, 1e-7);
  cudaEventRecord(e0);
  for (int w = 0; w < 10; ++w) kern<<<blocks, threads>>>(out, 0.999999, 1e-7);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  return ms / 10;
}

int main() {
  double* out; CK(cudaMalloc(&out, 1 << 20));
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  printf("SMs %d\n", sms);
  for (int occ : {1, 2, 3, 4, 8, 16}) {
    int blocks = sms * occ, threads = 128;
    float ms = timeit(k_dfma, blocks, threads, out);
    double fl = 2.0 * 8 * ITERS * (double)blocks * threads;
    printf("DFMA  warps/SM=%2d : %.3f ms  %.2f TFLOP/s\n", occ * 4, ms, fl / ms / 1e9);
    ms = timeit(k_dmma, blocks, threads, out);
    fl = 2.0 * 256 * ITERS * (double)blocks * threads / 32;
    printf("DMMA  warps/SM=%2d : %.3f ms  %.2f TFLOP/s\n", occ * 4, ms, fl / ms / 1e9);
    ms = timeit(k_dmma_ana, blocks, threads, out);
    fl = 2.0 * 256 * ITERS * (double)blocks * threads / 32;
    printf("DMMA-ana warps/SM=%2d : %.3f ms  %.2f TFLOP/s\n", occ * 4, ms, fl / ms / 1e9);
    ms = timeit(k_mixed<2>, blocks, threads, out);
    fl = 2.0 * 256 * ITERS * (double)blocks * threads / 32 + 2.0 * 2 * ITERS * (double)blocks * threads;
    printf("MIX2  warps/SM=%2d : %.3f ms  %.2f TFLOP/s\n", occ * 4, ms, fl / ms / 1e9);
    ms = timeit(k_mixed<4>, blocks, threads, out);
    fl = 2.0 * 256 * ITERS * (double)blocks * threads / 32 + 2.0 * 4 * ITERS * (double)blocks * threads;
    printf("MIX4  warps/SM=%2d : %.3f ms  %.2f TFLOP/s\n", occ * 4, ms, fl / ms / 1e9);
    ms = timeit(k_mixed<8>, blocks, threads, out);
    fl = 2.0 * 256 * ITERS * (double)blocks * threads / 32 + 2.0 * 8 * ITERS * (double)blocks * threads;
    printf("MIX8  warps/SM=%2d : %.3f ms  %.2f TFLOP/s\n", occ * 4, ms, fl / ms / 1e9);
  }
  CK(cudaGetLastError());
  return 0;
}
