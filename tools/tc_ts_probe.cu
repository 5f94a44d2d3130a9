// Probe of tcgen05.mma kind::tf32 with the A operand in tensor memory
// ("TS": D[tmem] = A[tmem] * B[smem]; development tool).  A (128x32) is
// written to TMEM with tcgen05.st.32x32b (lane = row, one 32-bit column per K
// element), B (32x128) sits in shared memory as in the FP32 kernel (K-major
// SW128, or MN-major 32-byte-atom SW128).  Checks D bit-exactly on integer
// data, then times back-to-back TS MMAs (M=128, N=128).
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>
#include <stdint.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo, uint64_t lt) {
  return (uint64_t)((saddr & 0x3FFFFu) >> 4) | ((uint64_t)((lbo >> 4) & 0x3FFFu) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFFu) << 32) | (1ull << 46) | (lt << 61);
}

__global__ void probe(const float* A, const float* B, float* D, int variant, int iters, unsigned long long* cyc) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* base = (uint8_t*)(((uintptr_t)sm + 1023) & ~(uintptr_t)1023);
  float* sB = (float*)base;  // 16 KB
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  for (int e = tid; e < 32 * 128; e += blockDim.x) {
    int k = e / 128, n = e % 128;
    if (variant == 0) {  // K-major: rows n, 32 k per row, SW128
      int r = n, c = k;
      sB[r * 32 + ((((c >> 2) ^ (r & 7)) << 2) | (c & 3))] = B[e];
    } else {  // MN-major, 32-byte-atom SW128: block jb at jb*4096 B, row k of 32 n
      int jb = n / 32, r = k, c = n % 32;
      sB[jb * 1024 + r * 32 + ((((c >> 3) ^ (r & 3)) << 3) | (c & 7))] = B[e];
    }
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&bar)), "r"(1));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tbase)), "r"(256)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tm = tbase, ta = tbase + 128;
  // A rows 32w..32w+31 -> TMEM lanes of warp w, columns ta..ta+31
  {
    const int row = warp * 32 + lane;
    uint32_t v[32];
    for (int c = 0; c < 32; ++c) v[c] = __float_as_uint(A[row * 32 + c]);
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,"
        "%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(ta + ((uint32_t)(warp * 32) << 16)),
        "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]), "r"(v[9]),
        "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]), "r"(v[16]), "r"(v[17]), "r"(v[18]),
        "r"(v[19]), "r"(v[20]), "r"(v[21]), "r"(v[22]), "r"(v[23]), "r"(v[24]), "r"(v[25]), "r"(v[26]), "r"(v[27]),
        "r"(v[28]), "r"(v[29]), "r"(v[30]), "r"(v[31])
        : "memory");
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  // D f32, A/B tf32, A K-major (TMEM), B major per variant
  const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(variant == 1) << 16) | ((128u >> 3) << 17) |
                         ((128u >> 4) << 24);
  if (tid == 0) {
    const uint32_t b0 = smem_u32(sB);
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it)
      for (int j = 0; j < 4; ++j) {
        const uint64_t bd = variant == 0 ? sdesc(b0 + 32 * j, 16, 1024, 2) : sdesc(b0 + 1024 * j, 4096, 512, 1);
        const uint32_t acc = (it | j) > 0;
        asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n}\n" ::"r"(tm),
                     "r"(ta + 8 * j), "l"(bd), "r"(idesc), "r"(acc)
                     : "memory");
      }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar))
                 : "memory");
    asm volatile("{\n.reg .pred p;\nW:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n@!p bra W;\n}\n" ::"r"(
                     smem_u32(&bar))
                 : "memory");
    cyc[0] = clock64() - t0;
  }
  asm volatile("{\n.reg .pred p;\nW2:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n@!p bra W2;\n}\n" ::"r"(
                   smem_u32(&bar))
               : "memory");
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  for (int j = 0; j < 4; ++j) {
    uint32_t v[32];
    uint32_t tl = tm + ((uint32_t)(warp * 32) << 16) + 32 * j;
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,"
        "%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]), "=r"(v[8]),
          "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]), "=r"(v[16]),
          "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]),
          "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
        : "r"(tl));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    int row = warp * 32 + lane;
    for (int c = 0; c < 32; ++c) D[row * 128 + j * 32 + c] = __uint_as_float(v[c]);
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tm), "r"(256) : "memory");
}

int main() {
  const int M = 128, N = 128, K = 32;
  float *hA = (float*)malloc(M * K * 4), *hB = (float*)malloc(K * N * 4), *hD = (float*)malloc(M * N * 4);
  for (int i = 0; i < M * K; ++i) hA[i] = (float)((i * 7) % 9 - 4);
  for (int i = 0; i < K * N; ++i) hB[i] = (float)((i * 5) % 9 - 4);
  double* ref = (double*)malloc(M * N * 8);
  for (int m = 0; m < M; ++m)
    for (int n = 0; n < N; ++n) {
      double s = 0;
      for (int k = 0; k < K; ++k) s += (double)hA[m * K + k] * hB[k * N + n];
      ref[m * N + n] = s;
    }
  float *dA, *dB, *dD;
  unsigned long long* dc;
  cudaMalloc(&dA, M * K * 4);
  cudaMalloc(&dB, K * N * 4);
  cudaMalloc(&dD, M * N * 4);
  cudaMalloc(&dc, 8);
  cudaMemcpy(dA, hA, M * K * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, hB, K * N * 4, cudaMemcpyHostToDevice);
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 40000);
  for (int variant = 0; variant < 2; ++variant) {
    for (int iters : {1, 2000}) {
      cudaMemset(dD, 0, M * N * 4);
      probe<<<1, 128, 40000>>>(dA, dB, dD, variant, iters, dc);
      cudaError_t e = cudaDeviceSynchronize();
      unsigned long long cyc = 0;
      cudaMemcpy(hD, dD, M * N * 4, cudaMemcpyDeviceToHost);
      cudaMemcpy(&cyc, dc, 8, cudaMemcpyDeviceToHost);
      int bad = 0;
      double maxerr = 0;
      for (int i = 0; i < M * N; ++i) {
        const double want = ref[i] * iters;
        maxerr = fmax(maxerr, fabs(hD[i] - want));
        if (hD[i] != (float)want) ++bad;
      }
      printf("TS variant %d (%s B) iters %d: %s mismatches %d maxerr %g D[0..1]=%g %g ref %g %g | %.1f cycles/MMA\n", variant,
             variant == 0 ? "K-major" : "MN-major 32B-atom", iters, cudaGetErrorString(e), bad, maxerr, hD[0], hD[1],
             ref[0] * iters, ref[1] * iters, (double)cyc / (iters * 4.0));
      if (e != cudaSuccess) return 1;
    }
  }
  return 0;
}
