// TS tcgen05.mma (kind::tf32, A in TMEM, B in smem, M=128 N=128) issue rate with
// concurrent traffic from 8 other warps (development tool):
//   0 none, 1 LDS.128 stream, 2 STS.128 stream, 3 tcgen05.st.32x32b.x32 stream
//   (other TMEM columns), 4 tcgen05.ld stream, 5 LDS+STS mix.
#include <cstdio>
#include <cuda_runtime.h>
#include <stdint.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo, uint64_t lt) {
  return (uint64_t)((saddr & 0x3FFFFu) >> 4) | ((uint64_t)((lbo >> 4) & 0x3FFFu) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFFu) << 32) | (1ull << 46) | (lt << 61);
}

__global__ void __launch_bounds__(288, 1) rate(int iters, int mode, unsigned long long* out, float* sink,
                                               int commit_every, int ncommit, int altd) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* base = (uint8_t*)(((uintptr_t)sm + 1023) & ~(uintptr_t)1023);
  uint8_t* sB = base;            // 16 KiB B (K-major SW128, N=128 rows)
  uint8_t* sH = base + 16384;    // 64 KiB hammer region
  __shared__ uint64_t bar, cbar[2];
  __shared__ uint32_t tbase;
  __shared__ volatile int stop;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  for (int i = tid; i < (16384 + 65536) / 16; i += blockDim.x)
    reinterpret_cast<float4*>(base)[i] = make_float4(0.f, 0.f, 0.f, 0.f);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (tid == 0) {
    stop = 0;
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&bar)), "r"(1));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&cbar[0])), "r"(1));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&cbar[1])), "r"(1));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tbase)), "r"(512)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tm = tbase;
  if (warp == 0) {
    if (tid == 0) {
      const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((128u >> 3) << 17) | ((128u >> 4) << 24);
      const uint32_t b0 = smem_u32(sB);
      long long t0 = clock64();
      for (int it = 0; it < iters; ++it)
        for (int j = 0; j < 4; ++j) {
          const uint32_t acc = (it | j) > 0;
          asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n}\n" ::"r"(tm + (altd ? 256u * (j & 1) : 0u)),
                       "r"(tm + 128 + 8 * j), "l"(sdesc(b0 + 32 * j, 16, 1024, 2)), "r"(idesc), "r"(acc)
                       : "memory");
          if (commit_every && ((it * 4 + j + 1) % commit_every) == 0) {
            asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                             smem_u32(&cbar[0]))
                         : "memory");
            if (ncommit > 1)
              asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                               smem_u32(&cbar[1]))
                           : "memory");
          }
        }
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar))
                   : "memory");
      asm volatile("{\n.reg .pred p;\nW:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n@!p bra W;\n}\n" ::"r"(
                       smem_u32(&bar))
                   : "memory");
      out[0] = clock64() - t0;
      stop = 1;
    }
    __syncwarp();
  } else if (mode) {
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    float4* h = reinterpret_cast<float4*>(sH);
    int i = (tid - 32) & 4095;
    long long n = 0;
    const uint32_t q = (uint32_t)(warp & 3);
    const uint32_t tcol = tm + 256 + 32 * ((warp - 1) >> 2) + ((32 * q) << 16);  // other columns
    uint32_t v[32];
    for (int c = 0; c < 32; ++c) v[c] = c;
    while (!stop) {
      if (mode == 1 || mode == 2 || mode == 5) {
#pragma unroll
        for (int u = 0; u < 16; ++u) {
          const int x = (i + u * 256) & 4095;
          if (mode == 1) {
            float4 y = h[x];
            acc.x += y.x;
          } else if (mode == 2) {
            h[x] = acc;
            acc.x += 1.f;
          } else {
            float4 y = h[x];
            h[x ^ 2048] = y;
            acc.x += y.x;
          }
        }
        n += 16 * 512 * (mode == 5 ? 2 : 1);
        i = (i + 32) & 4095;
      } else if (mode == 3) {
        asm volatile(
            "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,"
            "%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(tcol),
            "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]), "r"(v[9]),
            "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]), "r"(v[16]), "r"(v[17]), "r"(v[18]),
            "r"(v[19]), "r"(v[20]), "r"(v[21]), "r"(v[22]), "r"(v[23]), "r"(v[24]), "r"(v[25]), "r"(v[26]), "r"(v[27]),
            "r"(v[28]), "r"(v[29]), "r"(v[30]), "r"(v[31])
            : "memory");
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
        n += 4096;
      } else {
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,"
            "%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
            : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]), "=r"(v[8]),
              "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]), "=r"(v[16]),
              "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]),
              "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
            : "r"(tcol));
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        acc.x += __uint_as_float(v[lane]);
        n += 4096;
      }
    }
    if (acc.x == 1234.f) sink[0] = acc.y;
    if (blockIdx.x == 0 && lane == 0) atomicAdd(&out[1], (unsigned long long)n);
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tm), "r"(512) : "memory");
  }
}

template <int COMMITS, int ROT>  // commits after every group of 4 MMAs; ROT: rotate A slot / B stage per group
__global__ void __launch_bounds__(128, 1) rate_commit(int iters, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* base = (uint8_t*)(((uintptr_t)sm + 1023) & ~(uintptr_t)1023);
  __shared__ uint64_t bar, cbar[2];
  __shared__ uint32_t tbase;
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int i = tid; i < 4 * 16384 / 16; i += blockDim.x) reinterpret_cast<float4*>(base)[i] = make_float4(0.f, 0.f, 0.f, 0.f);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&bar)), "r"(1));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&cbar[0])), "r"(1));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&cbar[1])), "r"(1));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tbase)), "r"(512)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tm = tbase;
  if (warp == 0) {
    const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((128u >> 3) << 17) | ((128u >> 4) << 24);
    const uint32_t b0 = smem_u32(base);
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
      if (tid == 0) {
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const uint32_t acc = (it | j) > 0;
          const uint32_t rot = ROT ? (uint32_t)(it & 3) : 0u;
          asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n}\n" ::"r"(tm),
                       "r"(tm + 256 + 64 * rot + 8 * j), "l"(sdesc(b0 + 16384 * rot + 32 * j, 16, 1024, 2)), "r"(idesc), "r"(acc)
                       : "memory");
        }
#pragma unroll
        for (int c = 0; c < COMMITS; ++c)
          asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                           smem_u32(&cbar[c & 1]))
                       : "memory");
      }
      __syncwarp();
    }
    if (tid == 0) {
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar))
                   : "memory");
      asm volatile("{\n.reg .pred p;\nW:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n@!p bra W;\n}\n" ::"r"(
                       smem_u32(&bar))
                   : "memory");
      out[0] = clock64() - t0;
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tm), "r"(512) : "memory");
  }
}

// The FP32 kernel's exact per-step MMA sequence: 4 K-slices x (cross += a_lo.b_hi,
// cross += a_hi.b_lo, main += a_hi.b_hi), B hi/lo MN-major (32-byte-atom SW128),
// A hi/lo in a rotating TMEM slot, B in a rotating smem stage, COMMITS commits per step.
template <int COMMITS, int FENCE = 0, int RANDOM = 0>
__global__ void __launch_bounds__(128, 1) rate_step(int steps, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* base = (uint8_t*)(((uintptr_t)sm + 1023) & ~(uintptr_t)1023);
  __shared__ uint64_t bar, cbar[2];
  __shared__ uint32_t tbase;
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int i = tid; i < 4 * 32768 / 4; i += blockDim.x) {
    float x = 0.f;
    if (RANDOM) {
      unsigned h = (unsigned)i * 2654435761u + 12345u;
      h ^= h >> 13; h *= 0x5bd1e995u; h ^= h >> 15;
      x = (float)(h & 0xffffff) * (1.0f / 16777216.0f) - 0.5f;
    }
    reinterpret_cast<float*>(base)[i] = x;
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&bar)), "r"(1));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&cbar[0])), "r"(1));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&cbar[1])), "r"(1));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tbase)), "r"(512)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tm = tbase;
  if (RANDOM) {
    uint32_t v[32];
    for (int c = 0; c < 32; ++c) {
      unsigned h = (unsigned)(tid * 131 + c) * 2654435761u;
      h ^= h >> 15;
      v[c] = __float_as_uint((float)(h & 0xffff) * (1.0f / 65536.0f) - 0.5f);
    }
    for (int col = 384; col < 512; col += 32)
      asm volatile(
          "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,"
          "%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(tm + col + ((uint32_t)(warp * 32) << 16)),
          "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]), "r"(v[9]),
          "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]), "r"(v[16]), "r"(v[17]), "r"(v[18]),
          "r"(v[19]), "r"(v[20]), "r"(v[21]), "r"(v[22]), "r"(v[23]), "r"(v[24]), "r"(v[25]), "r"(v[26]), "r"(v[27]),
          "r"(v[28]), "r"(v[29]), "r"(v[30]), "r"(v[31])
          : "memory");
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  }
  if (warp == 0) {
    // idesc: D f32, A/B tf32, A K-major (TMEM), B MN-major
    const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | (1u << 16) | ((128u >> 3) << 17) | ((128u >> 4) << 24);
    const uint32_t b0 = smem_u32(base);
    long long t0 = clock64();
    for (int s = 0; s < steps; ++s) {
      if (FENCE == 1) asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      if (FENCE == 2) {
        asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
        __syncwarp();
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      }
      if (tid == 0) {
        const uint32_t st = b0 + 32768u * (uint32_t)(s & 3);
        const uint32_t stB = st, loB = st + 16384u;
        const uint32_t d_main = tm, d_cross = tm + 256;
        const uint32_t a_slot = tm + 384 + 64u * (uint32_t)(s & 1);
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const uint64_t b_hi = sdesc(stB + 1024u * j, 4096, 512, 1);
          const uint64_t b_lo = sdesc(loB + 1024u * j, 4096, 512, 1);
          const uint32_t a_hi = a_slot + 8u * j, a_lo = a_hi + 32u;
          const uint32_t acc = (s | j) > 0;
          asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n}\n" ::"r"(d_cross),
                       "r"(a_lo), "l"(b_hi), "r"(idesc), "r"(acc) : "memory");
          asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n}\n" ::"r"(d_cross),
                       "r"(a_hi), "l"(b_lo), "r"(idesc), "r"(1u) : "memory");
          asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n}\n" ::"r"(d_main),
                       "r"(a_hi), "l"(b_hi), "r"(idesc), "r"(acc) : "memory");
        }
#pragma unroll
        for (int c = 0; c < COMMITS; ++c)
          asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                           smem_u32(&cbar[c & 1]))
                       : "memory");
      }
      __syncwarp();
    }
    if (tid == 0) {
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar))
                   : "memory");
      asm volatile("{\n.reg .pred p;\nW:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n@!p bra W;\n}\n" ::"r"(
                       smem_u32(&bar))
                   : "memory");
      out[0] = clock64() - t0;
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tm), "r"(512) : "memory");
  }
}

int main() {
  unsigned long long* out;
  float* sink;
  cudaMalloc(&out, 16);
  cudaMalloc(&sink, 8);
  const int smem = 1024 + 16384 + 65536;
  cudaFuncSetAttribute(rate, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const char* names[] = {"none", "LDS.128", "STS.128", "tcgen05.st", "tcgen05.ld", "LDS+STS"};
  for (int c = 0; c < 6; ++c) {
    auto k = c == 0 ? rate_step<0> : c == 1 ? rate_step<1> : c == 2 ? rate_step<2> : c == 3 ? rate_step<2, 1> : c == 4 ? rate_step<2, 2> : rate_step<2, 0, 1>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 140000);
    cudaMemset(out, 0, 16);
    k<<<148, 128, 140000>>>(1000, out);
    cudaError_t e = cudaDeviceSynchronize();
    unsigned long long o[2];
    cudaMemcpy(o, out, 16, cudaMemcpyDeviceToHost);
    printf("FP32 kernel step sequence (12 MMAs), %d commit(s) per step%s: %.1f cycles/step (floor 768) [%s]\n",
           c < 3 ? c : 2, c == 3 ? " + fence::after_thread_sync" : c == 4 ? " + before/syncwarp/after fences" : c == 5 ? ", RANDOM operands" : "",
           (double)o[0] / 1000.0, cudaGetErrorString(e));
  }
  cudaFuncSetAttribute(rate_commit<0, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, 70000);
  cudaFuncSetAttribute(rate_commit<1, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, 70000);
  cudaFuncSetAttribute(rate_commit<2, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, 70000);
  cudaFuncSetAttribute(rate_commit<0, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 70000);
  cudaFuncSetAttribute(rate_commit<1, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 70000);
  cudaFuncSetAttribute(rate_commit<2, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 70000);
  for (int c = 0; c < 6; ++c) {
    cudaMemset(out, 0, 16);
    if (c == 0) rate_commit<0, 0><<<148, 128, 70000>>>(2000, out);
    if (c == 1) rate_commit<1, 0><<<148, 128, 70000>>>(2000, out);
    if (c == 2) rate_commit<2, 0><<<148, 128, 70000>>>(2000, out);
    if (c == 3) rate_commit<0, 1><<<148, 128, 70000>>>(2000, out);
    if (c == 4) rate_commit<1, 1><<<148, 128, 70000>>>(2000, out);
    if (c == 5) rate_commit<2, 1><<<148, 128, 70000>>>(2000, out);
    cudaError_t e = cudaDeviceSynchronize();
    unsigned long long o[2];
    cudaMemcpy(o, out, 16, cudaMemcpyDeviceToHost);
    printf("template loop, %d commit(s) per 4 MMAs, %s: %.1f cycles/MMA [%s]\n", c % 3,
           c >= 3 ? "A slot / B stage rotating" : "same A / B", (double)o[0] / 8000.0, cudaGetErrorString(e));
  }
  for (int altd = 0; altd < 2; ++altd)
    for (int nc = 1; nc <= 2; ++nc)
      for (int ce : {4, 12, 48}) {
        cudaMemset(out, 0, 16);
        rate<<<148, 288, smem>>>(2000, 0, out, sink, ce, nc, altd);
        cudaDeviceSynchronize();
        unsigned long long o[2];
        cudaMemcpy(o, out, 16, cudaMemcpyDeviceToHost);
        printf("TS tf32 M=128 N=128, %d commit(s) every %2d MMAs, %s D: %.1f cycles/MMA\n", nc, ce,
               altd ? "alternating" : "one", (double)o[0] / 8000.0);
      }
  for (int mode = 0; mode < 6; ++mode) {
    cudaMemset(out, 0, 16);
    rate<<<148, 288, smem>>>(2000, mode, out, sink, 0, 0, 0);
    cudaError_t e = cudaDeviceSynchronize();
    unsigned long long o[2];
    cudaMemcpy(o, out, 16, cudaMemcpyDeviceToHost);
    printf("TS tf32 M=128 N=128 with %-10s: %.1f cycles/MMA (floor 64), concurrent traffic %.0f B/clk [%s]\n", names[mode],
           (double)o[0] / 8000.0, (double)o[1] / (double)o[0], cudaGetErrorString(e));
  }
  return 0;
}
