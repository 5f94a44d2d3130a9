// FP64 peak microbenchmarks for the roofline denominator (no GPU-specific
// numbers are given in MEASURED_PEAKS.json for FP64): DFMA pipe, DMMA
// (mma.sync m8n8k4 f64) tensor path, and both at once.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void dfma_kernel(double* out, int iters, double a, double b) {
  double x[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) x[i] = threadIdx.x * 1e-3 + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int r = 0; r < 16; ++r)
#pragma unroll
      for (int i = 0; i < 8; ++i) x[i] = fma(x[i], a, b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += x[i];
  if (s == 123.456) out[0] = s;
}

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}

__global__ void dmma_kernel(double* out, int iters, double a, double b) {
  double acc[16][2];
#pragma unroll
  for (int i = 0; i < 16; ++i) { acc[i][0] = 0; acc[i][1] = 0; }
  double av = a + threadIdx.x * 1e-9, bv = b;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int r = 0; r < 2; ++r)
#pragma unroll
      for (int i = 0; i < 16; ++i) dmma(acc[i][0], acc[i][1], av, bv);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 16; ++i) s += acc[i][0] + acc[i][1];
  if (s == 123.456) out[0] = s;
}

__global__ void mixed_kernel(double* out, int iters, double a, double b) {
  // warps with even id run DMMA, odd run DFMA
  int w = threadIdx.x >> 5;
  if (w & 1) {
    double x[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] = threadIdx.x * 1e-3 + i;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int r = 0; r < 16; ++r)
#pragma unroll
        for (int i = 0; i < 8; ++i) x[i] = fma(x[i], a, b);
    }
    double s = 0;
    for (int i = 0; i < 8; ++i) s += x[i];
    if (s == 123.456) out[0] = s;
  } else {
    double acc[16][2];
#pragma unroll
    for (int i = 0; i < 16; ++i) { acc[i][0] = 0; acc[i][1] = 0; }
    double av = a + threadIdx.x * 1e-9, bv = b;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int r = 0; r < 2; ++r)
#pragma unroll
        for (int i = 0; i < 16; ++i) dmma(acc[i][0], acc[i][1], av, bv);
    }
    double s = 0;
    for (int i = 0; i < 16; ++i) s += acc[i][0] + acc[i][1];
    if (s == 123.456) out[0] = s;
  }
}

int main() {
  double* out;
  cudaMalloc(&out, 8);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int threads : {128, 256, 512}) {
    for (int cpsm : {1, 2, 4}) {
      int grid = sms * cpsm;
      // DFMA: flops per thread per iter = 16*8*2
      int iters = 4000;
      dfma_kernel<<<grid, threads>>>(out, 10, 1.0000001, 1e-9);
      cudaEventRecord(e0);
      dfma_kernel<<<grid, threads>>>(out, iters, 1.0000001, 1e-9);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      double fl = (double)grid * threads * iters * 16 * 8 * 2;
      printf("DFMA  threads=%d ctas/sm=%d : %.2f TFLOP/s (%.3f ms)\n", threads, cpsm, fl / ms / 1e9, ms);
      // DMMA: per warp per iter 32 dmma * 512 flop
      int it2 = 2000;
      dmma_kernel<<<grid, threads>>>(out, 10, 1.0, 1e-9);
      cudaEventRecord(e0);
      dmma_kernel<<<grid, threads>>>(out, it2, 1.0, 1e-9);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      cudaEventElapsedTime(&ms, e0, e1);
      fl = (double)grid * (threads / 32) * it2 * 32 * 512;
      printf("DMMA  threads=%d ctas/sm=%d : %.2f TFLOP/s (%.3f ms)\n", threads, cpsm, fl / ms / 1e9, ms);
      // mixed
      mixed_kernel<<<grid, threads>>>(out, 10, 1.0, 1e-9);
      cudaEventRecord(e0);
      mixed_kernel<<<grid, threads>>>(out, 2000, 1.0, 1e-9);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      cudaEventElapsedTime(&ms, e0, e1);
      double fl_m = (double)grid * (threads / 64) * 2000 * 32 * 512 + (double)grid * (threads / 2) * 2000 * 16 * 8 * 2;
      printf("MIXED threads=%d ctas/sm=%d : %.2f TFLOP/s (%.3f ms)\n", threads, cpsm, fl_m / ms / 1e9, ms);
    }
  }
  cudaError_t e = cudaGetLastError();
  printf("status %s\n", cudaGetErrorString(e));
  return 0;
}
