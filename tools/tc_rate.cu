// tcgen05.mma issue-rate microbenchmark (development tool): cycles per
// kind::tf32 / kind::f16 MMA with both operands in shared memory (SS), M=128,
// cta_group::1, for N = 64/128/256, alone and with 8 other warps streaming
// LDS.128 from shared memory at the same time (is the tensor core's operand
// read path the same 128 B/clk shared-memory bandwidth?).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/tc_rate tools/tc_rate.cu
#include <cstdio>
#include <cuda_runtime.h>
#include <stdint.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((saddr & 0x3FFFFu) >> 4) | ((uint64_t)((lbo >> 4) & 0x3FFFu) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFFu) << 32) | (1ull << 46) | (2ull << 61);
}

template <int KIND>  // 0 tf32, 1 f16
__device__ __forceinline__ void mma(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  if (KIND == 0)
    asm volatile("{.reg .pred p; setp.ne.b32 p, %4, 0; tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;}"
                 ::"r"(d), "l"(a), "l"(b), "r"(idesc), "r"(acc) : "memory");
  else
    asm volatile("{.reg .pred p; setp.ne.b32 p, %4, 0; tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;}"
                 ::"r"(d), "l"(a), "l"(b), "r"(idesc), "r"(acc) : "memory");
}

template <int KIND>
__global__ void __launch_bounds__(288, 1) rate(int N, int iters, int hammer, unsigned long long* out,
                                               float* sink) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* base = (uint8_t*)(((uintptr_t)sm + 1023) & ~(uintptr_t)1023);
  // A: 128 rows x 128 B (SW128 K-major), B: N rows x 128 B, hammer region after them
  uint8_t* sA = base;
  uint8_t* sB = base + 16384;
  uint8_t* sH = base + 16384 + 32768;
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  __shared__ volatile int stop;
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int i = tid; i < (16384 + 32768 + 65536) / 16; i += blockDim.x)
    reinterpret_cast<float4*>(base)[i] = make_float4(0.f, 0.f, 0.f, 0.f);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (tid == 0) {
    stop = 0;
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&bar)), "r"(1));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tbase)),
                 "r"(256)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tm = tbase;
  if (warp == 0) {
    if (tid == 0) {
      // kind::tf32: D f32, A/B tf32 (2); kind::f16: A/B bf16 (1); both K-major
      const uint32_t ab = KIND == 0 ? 2u : 1u;
      const uint32_t idesc = (1u << 4) | (ab << 7) | (ab << 10) | ((uint32_t)(N >> 3) << 17) | ((128u >> 4) << 24);
      const uint32_t a0 = smem_u32(sA), b0 = smem_u32(sB);
      long long t0 = clock64();
      for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int j = 0; j < 4; ++j)
          mma<KIND>(tm, sdesc(a0 + 32u * j, 16, 1024), sdesc(b0 + 32u * j, 16, 1024), idesc, (it | j) ? 1u : 0u);
      }
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar))
                   : "memory");
      asm volatile("{.reg .pred p; W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0; @!p bra W;}" ::"r"(
                       smem_u32(&bar))
                   : "memory");
      long long t1 = clock64();
      stop = 1;
      if (blockIdx.x == 0) out[0] = (unsigned long long)(t1 - t0);
    }
    __syncwarp();
  } else if (hammer) {
    // hammer 1: LDS.128 stream over a 64 KiB region; 2: STS.128 stream;
    // 3: the split-warp mix (1 LDS.128 + 2 STS.128)
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    float4* h = reinterpret_cast<float4*>(sH);
    int i = (tid - 32) & 4095;
    long long n = 0;
    while (!stop) {
#pragma unroll
      for (int u = 0; u < 16; ++u) {
        const int x = (i + u * 256) & 4095;
        if (hammer == 1) {
          float4 v = h[x];
          acc.x += v.x;
          acc.y += v.y;
        } else if (hammer == 2) {
          h[x] = acc;
          acc.x += 1.f;
        } else {
          float4 v = h[x];
          h[x ^ 2048] = v;
          h[x ^ 1024] = acc;
          acc.x += v.x;
        }
      }
      n += 16;
      i = (i + 32) & 4095;
    }
    if (acc.x == 1234.f) sink[0] = acc.y;
    if (blockIdx.x == 0 && (tid & 31) == 0) atomicAdd(&out[1], (unsigned long long)n * 512ull * (hammer == 3 ? 3 : 1));
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tm), "r"(256) : "memory");
  }
}

int main() {
  unsigned long long* out;
  float* sink;
  cudaMalloc(&out, 16);
  cudaMalloc(&sink, 8);
  const int smem = 1024 + 16384 + 32768 + 65536;
  cudaFuncSetAttribute(rate<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(rate<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int iters = 2000;
  for (int kind = 0; kind < 1; ++kind)
    for (int N : {64, 128, 256})
      for (int hammer = 0; hammer < 4; ++hammer) {
        cudaMemset(out, 0, 16);
        if (kind == 0) rate<0><<<148, 288, smem>>>(N, iters, hammer, out, sink);
        else rate<1><<<148, 288, smem>>>(N, iters, hammer, out, sink);
        cudaError_t e = cudaDeviceSynchronize();
        unsigned long long o2[2] = {0, 0};
        cudaMemcpy(o2, out, 16, cudaMemcpyDeviceToHost);
        const unsigned long long cyc = o2[0];
        const double per = (double)cyc / (iters * 4.0);
        const int K = kind == 0 ? 8 : 16;
        const double opbytes = (128.0 * K + (double)N * K) * (kind == 0 ? 4 : 2);
        printf("%s N=%3d hammer=%d: %.1f cycles/MMA (floor %.0f), %.0f MAC/clk/SM, operand bytes %.0f B/clk, hammer %.0f B/clk  [%s]\n",
               kind == 0 ? "tf32" : "bf16", N, hammer, per, 128.0 * N / 256.0, 128.0 * N * K / per, opbytes / per,
               (double)o2[1] / (double)cyc, cudaGetErrorString(e));
      }
  return 0;
}
