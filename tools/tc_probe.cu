// Probe of tcgen05.mma kind::tf32 descriptor conventions (development tool):
// D(128x128) = A(128x32) * B(32x128), A K-major SW128, B either K-major SW128
// (variant 0) or MN-major SW128 with 32-wide N atoms LBO-strided (variant 1).
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <cuda_runtime.h>
#include <stdint.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo, int ver, uint64_t lt = 2) {
  return (uint64_t)((saddr & 0x3FFFFu) >> 4) | ((uint64_t)((lbo >> 4) & 0x3FFFu) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFFu) << 32) | ((uint64_t)ver << 46) | (lt << 61);
}

__global__ void probe(const float* A, const float* B, float* D, int variant, int ver, int lbo_a,
                      int lbo_b, int sbo_b) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* base = (uint8_t*)(((uintptr_t)sm + 1023) & ~(uintptr_t)1023);
  float* sA = (float*)base;            // 128 x 32, K-major rows of 128 B, SW128
  float* sB = (float*)(base + 16384);  // 16 KB
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  // A[m][k] row-major 128x32 -> swizzled
  for (int e = tid; e < 128 * 32; e += blockDim.x) {
    int r = e / 32, c = e % 32;
    sA[r * 32 + ((((c >> 2) ^ (r & 7)) << 2) | (c & 3))] = A[e];
  }
  // B[k][n] row-major 32x128
  for (int e = tid; e < 32 * 128; e += blockDim.x) {
    int k = e / 128, n = e % 128;
    if (variant == 0) {
      // K-major: B^T rows n (128 rows), 32 k per row
      int r = n, c = k;
      sB[r * 32 + ((((c >> 2) ^ (r & 7)) << 2) | (c & 3))] = B[e];
    } else if (variant == 1) {
      // MN-major: block jb = n/32 at jb*4096 B, row k of 32 n
      int jb = n / 32, r = k, c = n % 32;
      sB[jb * 1024 + r * 32 + ((((c >> 2) ^ (r & 7)) << 2) | (c & 3))] = B[e];
    } else {
      // MN-major, 128B swizzle with 32-byte atoms: 32B chunk (c>>3) ^ (r & 3)
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
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tbase)), "r"(128) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  uint32_t tm = tbase;
  const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | (0u << 15) | ((uint32_t)(variant >= 1) << 16) |
                         ((128u >> 3) << 17) | ((128u >> 4) << 24);
  if (tid == 0) {
    uint32_t a0 = smem_u32(sA), b0 = smem_u32(sB);
    for (int j = 0; j < 4; ++j) {
      uint64_t ad = sdesc(a0 + 32 * j, lbo_a, 1024, ver);
      uint64_t bd = variant == 0 ? sdesc(b0 + 32 * j, lbo_a, 1024, ver)
                  : variant == 1 ? sdesc(b0 + 1024 * j, lbo_b, sbo_b, ver)
                                 : sdesc(b0 + 1024 * j, lbo_b, sbo_b, ver, 1);
      uint32_t acc = j > 0;
      asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n"
                   ::"r"(tm), "l"(ad), "l"(bd), "r"(idesc), "r"(acc) : "memory");
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)) : "memory");
  }
  asm volatile("{\n.reg .pred p;\nW:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n@!p bra W;\n}\n" ::"r"(smem_u32(&bar)) : "memory");
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  for (int j = 0; j < 4; ++j) {
    uint32_t v[32];
    uint32_t ta = tm + ((uint32_t)(warp * 32) << 16) + 32 * j;
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
                 : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
                 : "r"(ta));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    int row = warp * 32 + lane;
    for (int c = 0; c < 32; ++c) D[row * 128 + j * 32 + c] = __uint_as_float(v[c]);
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tm), "r"(128) : "memory");
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
  cudaMalloc(&dA, M * K * 4); cudaMalloc(&dB, K * N * 4); cudaMalloc(&dD, M * N * 4);
  cudaMemcpy(dA, hA, M * K * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, hB, K * N * 4, cudaMemcpyHostToDevice);
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 40000);
  struct V { int variant, ver, lbo_a, lbo_b, sbo_b; } vs[] = {
      {0, 1, 16, 0, 0}, {1, 1, 16, 4096, 1024}, {2, 1, 16, 4096, 512}, {2, 1, 16, 512, 4096}, {2, 1, 16, 4096, 1024}};
  for (auto v : vs) {
    cudaMemset(dD, 0, M * N * 4);
    probe<<<1, 128, 40000>>>(dA, dB, dD, v.variant, v.ver, v.lbo_a, v.lbo_b, v.sbo_b);
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(hD, dD, M * N * 4, cudaMemcpyDeviceToHost);
    double maxerr = 0, maxref = 0;
    int bad = 0;
    for (int i = 0; i < M * N; ++i) {
      maxerr = fmax(maxerr, fabs(hD[i] - ref[i]));
      maxref = fmax(maxref, fabs(ref[i]));
      if (hD[i] != (float)ref[i]) ++bad;
    }
    printf("variant %d ver %d lbo_a %d lbo_b %d sbo_b %d : %s maxerr %g (maxref %g) mismatches %d  D[0..3]=%g %g %g %g ref %g %g\n",
           v.variant, v.ver, v.lbo_a, v.lbo_b, v.sbo_b, cudaGetErrorString(e), maxerr, maxref, bad, hD[0], hD[1], hD[2],
           hD[3], ref[0], ref[1]);
    if (e != cudaSuccess) return 1;
  }
  return 0;
}
