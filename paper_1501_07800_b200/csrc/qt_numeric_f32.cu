// FP32 numeric block-sparse multiply on the 5th-generation tensor cores
// (tcgen05.mma kind::tf32, accumulators in TMEM) with the 3xTF32 split.
//
// Paper: the leaf multiply of §4.1 in single precision (the paper
// benchmarks both precisions).  Reading C-9: inputs are FP32, the
// result must be within 1e-5 relative Frobenius of the double product of the
// FP32 inputs; one TF32 product per term is ~2.5e-4 off, so each product is
// a_hi*b_hi + a_hi*b_lo + a_lo*b_hi with x_hi = x truncated to TF32 and
// x_lo = x - x_hi (error ~2^-21 per term, FP32 accumulation in TMEM).
//
// Work item ("tile") = one C node at level L-2: 4x4 C blocks = a 128x128 FP32
// accumulator in TMEM (128 lanes x 128 columns).  A step of the tile is one
// inner block index k: the A column A(I0..I3, k) (128x32) and the B row
// B(k, J0..J3) (32x128) — absent blocks are copied from a zero block — staged
// by eight 4 KiB cp.async.bulk copies (A into the A ring, B into the B ring,
// see below).  The pool stores every
// FP32 block in the canonical 128-byte swizzle (qt_common.cuh swz32).  Per
// step: 4 K-slices x 3 MMAs (M=128, N=128, K=8).
//
// Data path (measured with tools/tc_rate and tools/tc_ts_probe): the tensor
// core's shared-memory operand reads and LDS share the SM's 128 B/clk
// shared-memory read bandwidth, tensor core first — back-to-back M=128 N=128
// tf32 MMAs with both operands in shared memory read exactly 128 B/clk and
// leave an LDS stream 6 B/clk, so an in-SM hi/lo split that reads the landed
// stage starves.  Here the A operand lives in TENSOR MEMORY ("TS" MMAs): the
// split warps of A read the landed A column once (LDS), split each row into
// hi/lo in registers and write them to TMEM with tcgen05.st (lane = row, one
// 32-bit column per K element); the MMAs then read only B from shared memory
// (64 B/clk), which leaves room for the split warps' LDS.
//
// Warp roles (448 threads, one CTA per SM, persistent over tiles):
//   warps 0-3  epilogue  TMEM -> registers (tcgen05.ld 32x32b) -> C pool
//   warps 4-7  split A   block q: rows -> (hi, lo) -> tcgen05.st into TMEM
//   warps 8-11 split B   block q: fp32 -> (tf32 hi in place, lo copy) in smem
//   warp 12    producer  task metadata + TMA bulk copies (eight lanes issue a step's copies)
//   warp 13    MMA       lane 0 alone waits, issues tcgen05.mma / commit
// Each C block is written once by one thread row-set: no atomics; summation
// order per element is fixed (ascending k, and within a k the fixed K-slice
// and hi/lo order), so results are run-to-run deterministic.
#include <atomic>

#include <cuda_runtime.h>

#include "qt_common.cuh"
#include "qt_internal.h"

namespace qt {

namespace {

// smem: two rings advanced once per step.  The B ring (5 stages): B[4]
// (landed, then hi in place) | B lo[4] = 32 KiB, released by the MMAs'
// commit.  The A ring (3 stages): A raw[4] = 16 KiB, read once by the A split
// warps and released by them as soon as A is in TMEM — so an A landing slot
// turns over in TMA latency + split time, without waiting for the MMAs, and
// the B ring gets five stages in the same shared memory (the kernel's
// throughput is bounded by ring depth / stage round-trip time).
constexpr int kStages = 5;
constexpr int kAStages = 3;
constexpr int kBlkBytes = 4096;                 // 32x32 fp32
constexpr int kBloOff = 4 * kBlkBytes;          // B lo after B
constexpr int kStageBytes = 8 * kBlkBytes;
constexpr int kAStageBytes = 4 * kBlkBytes;
constexpr int kARingOff = kStages * kStageBytes;
constexpr int kSplitWarps = 8;
constexpr int kProducerWarp = 4 + kSplitWarps;
constexpr int kMmaWarp = kProducerWarp + 1;
constexpr int kThreads = (kMmaWarp + 1) * 32;
// TMEM (512 columns): two hi*hi accumulators (double-buffered tiles, columns
// 0 and 128), one cross-term accumulator (256), and two A slots of 64 columns
// (hi 32 + lo 32, K along columns) at 384 and 448.  The hi*hi products go to
// one accumulator, the two cross terms (2^-11 smaller) to the other; the
// epilogue adds them with a round-to-nearest FADD.  The tensor core's own
// accumulation into D is not round-to-nearest, so its error grows with the
// number of MMAs that add into one large accumulator: measured on config 5
// (65 k-steps), one accumulator for all 12 MMAs per step gave 1.02e-5
// relative Frobenius error, even/odd k-step accumulators 5.1e-6; the hi*hi /
// cross split leaves 4 MMAs per step on the large accumulator.  The cross
// accumulator is single-buffered: a tile's first MMAs wait until the
// epilogue has drained the previous tile.
constexpr int kTmemCols = 512;
constexpr uint32_t kColCross = 256;
constexpr uint32_t kColA = 384;

enum : int { F_FIRST = 1, F_END = 2, F_DONE = 4 };

struct __align__(16) Hdr {
  int tile;
  int flags;
  int pad[2];
};

struct Smem {
  Hdr hdr[kStages];
  Hdr ahdr[kAStages];       // flags of the A ring's steps
  int acc_tile[2];
  uint32_t tmem_base;
  uint32_t pad;
  uint64_t full[kStages];   // TMA landed (1 arrival + tx)
  uint64_t conv[kStages];   // A in TMEM and B hi/lo in smem (one arrival per split warp)
  uint64_t empty[kStages];  // MMAs that read the stage done (tcgen05.commit)
  uint64_t afull[kAStages];   // A landed (1 arrival + tx)
  uint64_t aempty[kAStages];  // A split into TMEM (one arrival per A split warp)
  uint64_t afree[2];        // MMAs that read the A slot done (tcgen05.commit)
  uint64_t tfull[2];        // accumulator ready (commit + MMA-lane arrive)
  uint64_t tempty[2];       // epilogue drained the hi*hi accumulator (4 warp arrivals)
  uint64_t cfree;           // epilogue drained the cross accumulator (4 warp arrivals)
  // producer: the current batch's block references, row = task lane: A(x, kk)
  // at 4x+kk, B(kk, x) at 16+4kk+x, and at 32 the mask of k-steps with an A
  // and a B block
  int refs[32][33];
};
constexpr size_t kSmemBytes =
    1024 /*align slack*/ + (size_t)kStages * kStageBytes + (size_t)kAStages * kAStageBytes + sizeof(Smem);

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, int count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   smem_u32(bar))
               : "memory");
}
// D[tmem] (+)= A[tmem] * B[smem], kind::tf32 (A: lane = row, column = K element)
__device__ __forceinline__ void tc_mma_ts(uint32_t tmem_d, uint32_t tmem_a, uint64_t bdesc,
                                          uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n"
      "}\n" ::"r"(tmem_d),
      "r"(tmem_a), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
// 32 consecutive 32-bit TMEM columns of this warp's 32 lanes
__device__ __forceinline__ void tmem_st32(uint32_t taddr, const uint32_t (&v)[32]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,"
      "%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
      "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]),
      "r"(v[8]), "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]),
      "r"(v[16]), "r"(v[17]), "r"(v[18]), "r"(v[19]), "r"(v[20]), "r"(v[21]), "r"(v[22]), "r"(v[23]),
      "r"(v[24]), "r"(v[25]), "r"(v[26]), "r"(v[27]), "r"(v[28]), "r"(v[29]), "r"(v[30]), "r"(v[31])
      : "memory");
}
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&v)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,"
      "%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
        "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]),
        "=r"(v[14]), "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]),
        "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]), "=r"(v[25]),
        "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
      : "r"(taddr));
}
// x_hi: the top 19 bits of x (a TF32 value); x - x_hi is exact in FP32 and
// has at most 13 significant bits, of which the tensor core reads 11, so
// x_hi + tf32(x - x_hi) represents x to ~2^-22 relative.
__device__ __forceinline__ float tf32_trunc(float x) {
  return __uint_as_float(__float_as_uint(x) & 0xffffe000u);
}

// Shared-memory matrix descriptor (tcgen05): start >> 4 in [0,14), leading
// byte offset >> 4 in [16,30), stride byte offset >> 4 in [32,46), version 1
// at [46,48), layout type at [61,64).  (Measured with tools/tc_probe.cu: an
// MN-major tf32 operand in the plain SWIZZLE_128B layout reads as zeros; the
// 32-byte-atom variant SWIZZLE_128B_BASE32B with 4-row K atoms is exact.)
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo,
                                          uint64_t layout) {
  return (uint64_t)((saddr & 0x3FFFFu) >> 4) | ((uint64_t)((lbo >> 4) & 0x3FFFu) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFFu) << 32) | (1ull << 46) | (layout << 61);
}
constexpr uint64_t kSW128 = 2;         // K-major A: 16-byte chunks ^ (row & 7)
constexpr uint64_t kSW128_32B = 1;     // MN-major B (32-bit types): 32-byte chunks ^ (row & 3)

// Instruction descriptor: D f32 (bits 4-5 = 1), A tf32 (7-9 = 2), B tf32
// (10-12 = 2), A major (15: 0 = K), B major (16: 1 = MN), N>>3 at 17, M>>4 at 24.
// A stored row-major block is K-major as an A operand and MN-major as a B
// operand; a transposed operand (C = A^T B, A B^T) flips that.

// TS form: A comes from TMEM in the M-lanes x K-columns layout (K-major)
template <bool kTB>
__host__ __device__ constexpr uint32_t idesc_tf32_ts() {
  return (1u << 4) | (2u << 7) | (2u << 10) | (0u << 15) | ((kTB ? 0u : 1u) << 16) |
         ((128u >> 3) << 17) | ((128u >> 4) << 24);
}

template <bool kTA, bool kTB, bool kSym>
__global__ void __launch_bounds__(kThreads, 1) k_numeric_f32(NumericArgs32 a) {
  extern __shared__ uint8_t smem_raw[];
  // 1024-byte aligned start (kept as an offset from the shared array so the
  // compiler still emits shared-space LDS/STS for the split warps)
  uint8_t* data = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  Smem& S = *reinterpret_cast<Smem*>(data + (size_t)kARingOff + (size_t)kAStages * kAStageBytes);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&S.full[s], 1);
      mbar_init(&S.conv[s], kSplitWarps);
      mbar_init(&S.empty[s], 1);
    }
    for (int s = 0; s < kAStages; ++s) {
      mbar_init(&S.afull[s], 1);
      mbar_init(&S.aempty[s], 4);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&S.afree[b], 1);
      mbar_init(&S.tfull[b], 2);
      mbar_init(&S.tempty[b], 4);
    }
    mbar_init(&S.cfree, 4);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(&S.tmem_base)),
                 "r"(kTmemCols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = S.tmem_base;

  if (warp == kProducerWarp) {
    // ------------------------------------------------------------ producer
    const float* poolA = static_cast<const float*>(a.poolA);
    const float* poolB = static_cast<const float*>(a.poolB);
    const float* poolB2 = static_cast<const float*>(a.poolB2);
    const float* zeros = static_cast<const float*>(a.zeros);
    int stage = 0, ast = 0;
    uint32_t phase = 0, aphase = 0;
    auto next_stage = [&]() {
      if (++stage == kStages) {
        stage = 0;
        phase ^= 1;
      }
      if (++ast == kAStages) {
        ast = 0;
        aphase ^= 1;
      }
    };
    // a step without data (end-of-tile / done marker) on both rings
    auto post_marker = [&](int tile, int flags) {
      mbar_wait(&S.empty[stage], phase ^ 1);
      mbar_wait(&S.aempty[ast], aphase ^ 1);
      if (lane == 0) {
        S.hdr[stage].tile = tile;
        S.hdr[stage].flags = flags;
        S.ahdr[ast].flags = flags;
        mbar_arrive(&S.full[stage]);
        mbar_arrive(&S.afull[ast]);
      }
      __syncwarp();
      next_stage();
    };
    // phase launches of the multi-rank overlap: tiles map[t_off + i]
    int ntiles = (int)a.ntiles, t_off = 0;
    if (a.ntiles_dev) ntiles = *a.ntiles_dev;  // sync-free product: the BFS's count (a.ntiles: its bound)
    if (a.phase) {
      const int ns = *a.nsel;
      t_off = a.phase == 1 ? 0 : ns;
      ntiles = a.phase == 1 ? ns : (int)a.ntiles - ns;
    }
    for (;;) {
      int t = 0;
      if (lane == 0) t = atomicAdd(a.counter, 1);
      t = __shfl_sync(0xffffffffu, t, 0);
      if (t >= ntiles) {
        post_marker(-1, F_DONE);
        break;
      }
      if (a.tile_map) t = a.tile_map[t_off + t];
      const int p0 = a.tile_start[t], p1 = a.tile_start[t + 1];
      bool first = true;
      for (int pb0 = p0; pb0 < p1; pb0 += 32) {
        const int p = pb0 + lane;
        // this lane's task: A blocks A(i, kk) and B blocks B(kk, j), i, kk, j in 0..3
        int ab[4][4], bb[4][4];
#pragma unroll
        for (int x = 0; x < 4; ++x)
#pragma unroll
          for (int y = 0; y < 4; ++y) ab[x][y] = bb[x][y] = -1;
        if (p < p1) {
          // op(A) quads (i', k') in slot 2i'+k' and op(B) quads (k', j') in slot
          // 2k'+j'; symmetric square: references into U (index, diagonal,
          // transposed bits), block references idx*4 + diag*2 + t
          const int4 qa = op_children(a.childA2, a.pa[p], kTA, kSym);
          const int4 qb = op_children(a.childB2, a.pb[p], kTB, kSym);
          const int qa_[4] = {qa.x, qa.y, qa.z, qa.w};
          const int qb_[4] = {qb.x, qb.y, qb.z, qb.w};
#pragma unroll
          for (int s = 0; s < 4; ++s) {
            const int hi = s >> 1, lo = s & 1;
            if (qa_[s] >= 0) {
              const int4 c = op_children(a.childA1, qa_[s], kTA, kSym);  // (i'', k'') in slot 2i''+k''
              ab[2 * hi + 0][2 * lo + 0] = c.x;
              ab[2 * hi + 0][2 * lo + 1] = c.y;
              ab[2 * hi + 1][2 * lo + 0] = c.z;
              ab[2 * hi + 1][2 * lo + 1] = c.w;
            }
            if (qb_[s] >= 0) {
              const int4 c = op_children(a.childB1, qb_[s], kTB, kSym);  // (k'', j'') in slot 2k''+j''
              bb[2 * hi + 0][2 * lo + 0] = c.x;
              bb[2 * hi + 0][2 * lo + 1] = c.y;
              bb[2 * hi + 1][2 * lo + 0] = c.z;
              bb[2 * hi + 1][2 * lo + 1] = c.w;
            }
          }
        }
        __syncwarp();  // (every lane is done with the previous batch's table)
        {
          int vm = 0;
#pragma unroll
          for (int kk = 0; kk < 4; ++kk) {
            bool anyA = false, anyB = false;
#pragma unroll
            for (int x = 0; x < 4; ++x) {
              S.refs[lane][4 * x + kk] = ab[x][kk];
              S.refs[lane][16 + 4 * kk + x] = bb[kk][x];
              anyA |= ab[x][kk] >= 0;
              anyB |= bb[kk][x] >= 0;
            }
            vm |= (anyA && anyB ? 1 : 0) << kk;
          }
          S.refs[lane][32] = vm;
        }
        __syncwarp();
        const int nloc = min(32, p1 - pb0);
        for (int u = 0; u < nloc; ++u) {
          const int vm = S.refs[u][32];
#pragma unroll
          for (int kk = 0; kk < 4; ++kk) {
            if (!((vm >> kk) & 1)) continue;
            mbar_wait(&S.empty[stage], phase ^ 1);
            mbar_wait(&S.aempty[ast], aphase ^ 1);
            if (lane == 0) {
              S.hdr[stage].tile = t;
              S.hdr[stage].flags = first ? F_FIRST : 0;
              S.ahdr[ast].flags = first ? F_FIRST : 0;
              mbar_arrive_expect_tx(&S.full[stage], 4u * kBlkBytes);
              mbar_arrive_expect_tx(&S.afull[ast], 4u * kBlkBytes);
            }
            __syncwarp();
            // eight lanes issue the eight 4 KiB copies at once (lane x < 4: A
            // block x, lane 4 + x: B block x)
            if (lane < 8) {
              const int ref = S.refs[u][lane < 4 ? 4 * lane + kk : 16 + 4 * kk + (lane - 4)];
              const float* src;
              if (kSym) {
                // symmetric square: a block of U read transposed comes from the
                // transposed copy of the pool, so the split warps read blocks as stored
                const float* poolT = static_cast<const float*>(a.poolT);
                src = ref < 0 ? zeros : ((ref & 1) ? poolT : poolA) + (size_t)(ref >> 2) * 1024;
              } else if (lane < 4) {
                src = ref >= 0 ? poolA + (size_t)ref * 1024 : zeros;
              } else {
                src = ref < 0 ? zeros
                              : (ref < a.splitB ? poolB + (size_t)ref * 1024 : poolB2 + (size_t)(ref - a.splitB) * 1024);
              }
              if (lane < 4)
                bulk_g2s(data + kARingOff + (size_t)ast * kAStageBytes + lane * kBlkBytes, src, kBlkBytes, &S.afull[ast]);
              else
                bulk_g2s(data + (size_t)stage * kStageBytes + (lane - 4) * kBlkBytes, src, kBlkBytes, &S.full[stage]);
            }
            __syncwarp();
            first = false;
            next_stage();
          }
        }
      }
      post_marker(t, F_END);  // end-of-tile marker (no data)
    }
  } else if (warp >= 4 && warp < 8) {
    // ------------------------------------------------------------ split A -> TMEM
    // Warp 4+q owns A block q = rows 32q..32q+31 of the 128-row A column,
    // i.e. exactly its own TMEM lane quarter; lane r holds row r.  The row's
    // 32 fp32 (K) are read once from the landed stage, split into hi (TF32
    // truncation) and lo (exact remainder) and written to the A slot's hi and
    // lo columns.  A transposed A (C = A^T B) is read by columns instead.
    const int q = warp - 4;
    int stage = 0, ast = 0;
    uint32_t phase = 0, aphase = 0;
    int as = 0;
    uint32_t aph = 0;
    for (;;) {
      mbar_wait(&S.afull[ast], aphase);
      const int flags = S.ahdr[ast].flags;
      if (!(flags & (F_END | F_DONE))) {
        mbar_wait(&S.afree[as], aph ^ 1);
        const float* blk =
            reinterpret_cast<const float*>(data + kARingOff + (size_t)ast * kAStageBytes + q * kBlkBytes);
        uint32_t hv[32], lv[32];
        const int r = lane;
        if (!kTA) {
#pragma unroll
          for (int c = 0; c < 8; ++c) {  // 16-byte chunk c of row r (SW128: chunk c ^ (r & 7))
            const float4 x = *reinterpret_cast<const float4*>(blk + r * 32 + ((c ^ (r & 7)) << 2));
            const float xs[4] = {x.x, x.y, x.z, x.w};
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              const float h = tf32_trunc(xs[e]);
              hv[4 * c + e] = __float_as_uint(h);
              lv[4 * c + e] = __float_as_uint(xs[e] - h);  // exact: at most 13 significant bits
            }
          }
        } else {
          // op(A)(r, k) = stored(k, r): column r of the stored block
#pragma unroll
          for (int k = 0; k < 32; ++k) {
            const float x = blk[k * 32 + ((((r >> 2) ^ (k & 7)) << 2) | (r & 3))];
            const float h = tf32_trunc(x);
            hv[k] = __float_as_uint(h);
            lv[k] = __float_as_uint(x - h);
          }
        }
        const uint32_t ta = tmem + kColA + 64u * (uint32_t)as + ((uint32_t)(32 * q) << 16);
        tmem_st32(ta, hv);
        tmem_st32(ta + 32, lv);
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
        tc_fence_before();
        if (++as == 2) {
          as = 0;
          aph ^= 1;
        }
      }
      __syncwarp();
      if (lane == 0) {
        mbar_arrive(&S.aempty[ast]);
        mbar_arrive(&S.conv[stage]);
      }
      if (flags & F_DONE) break;
      if (++stage == kStages) {
        stage = 0;
        phase ^= 1;
      }
      if (++ast == kAStages) {
        ast = 0;
        aphase ^= 1;
      }
    }
  } else if (warp >= 8 && warp < 4 + kSplitWarps) {
    // ------------------------------------------------------------ split B (smem)
    // Warp 8+q owns B block q (four 1 KiB swizzle atoms of 8 rows x 128 B, two
    // float4 per lane).  hi replaces the landed value in place, lo goes to the
    // stage's lo area.  The MN-major operand (B unless transposed) is re-laid
    // out for the 128-byte swizzle with 32-byte atoms (SWIZZLE_128B_BASE32B):
    // 16-byte chunk c of row r moves from c ^ (r&7) to ((c>>1 ^ (r&3))<<1 | (c&1))
    // — in place, after all lanes of the warp have read the atom.
    const int q = warp - 8;
    int stage = 0;
    uint32_t phase = 0;
    for (;;) {
      mbar_wait(&S.full[stage], phase);
      const int flags = S.hdr[stage].flags;
      if (!(flags & (F_END | F_DONE))) {
        float4* hi = reinterpret_cast<float4*>(data + (size_t)stage * kStageBytes + q * kBlkBytes);
        float4* lo = reinterpret_cast<float4*>(data + (size_t)stage * kStageBytes + kBloOff + q * kBlkBytes);
#pragma unroll 1
        for (int atom = 0; atom < 4; ++atom) {
          float4 x[2];
#pragma unroll
          for (int h = 0; h < 2; ++h) x[h] = hi[atom * 64 + lane + 32 * h];
          __syncwarp();
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int f = lane + 32 * h;
            int t = f;
            if (!kTB) {
              const int r = f >> 3, c16 = (f & 7) ^ r;
              t = r * 8 + ((((c16 >> 1) ^ (r & 3)) << 1) | (c16 & 1));
            }
            float4 hv, lv;
            hv.x = tf32_trunc(x[h].x);
            hv.y = tf32_trunc(x[h].y);
            hv.z = tf32_trunc(x[h].z);
            hv.w = tf32_trunc(x[h].w);
            lv.x = x[h].x - hv.x;  // exact: at most 13 significant bits
            lv.y = x[h].y - hv.y;
            lv.z = x[h].z - hv.z;
            lv.w = x[h].w - hv.w;
            hi[atom * 64 + t] = hv;
            lo[atom * 64 + t] = lv;
          }
        }
        fence_proxy_async();  // generic-proxy writes -> visible to the tensor core
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&S.conv[stage]);
      if (flags & F_DONE) break;
      if (++stage == kStages) {
        stage = 0;
        phase ^= 1;
      }
    }
  } else if (warp == kMmaWarp) {
    // ------------------------------------------------------------ MMA issuer
    // One thread runs the whole role (waits, MMAs, commits): no warp
    // synchronisation on the issue path; the other lanes go straight to the
    // final barrier.
    if (lane == 0) {
    int stage = 0;
    uint32_t phase = 0;
    int acc = 0;
    uint32_t acc_phase = 0;
    int as = 0;
    int ntiles_done = 0;  // tiles published to the epilogue (cross-accumulator uses)
    bool started = false;
    const uint32_t sbase = smem_u32(data);
    // B descriptors of stage 0, K-slice 0; a stage / K-slice only moves the
    // start-address field (address >> 4, < 2^14 for any shared address)
    const uint64_t bd_hi0 = kTB ? sdesc(sbase, 16, 1024, kSW128) : sdesc(sbase, 4096, 512, kSW128_32B);
    const uint64_t bd_lo0 = kTB ? sdesc(sbase + kBloOff, 16, 1024, kSW128) : sdesc(sbase + kBloOff, 4096, 512, kSW128_32B);
    for (;;) {
      mbar_wait(&S.conv[stage], phase);
      const int2 th = *reinterpret_cast<const int2*>(&S.hdr[stage]);  // (tile, flags) in one load
      const int tile = th.x, flags = th.y;
      if (flags & F_DONE) {
        mbar_wait(&S.tempty[acc], acc_phase ^ 1);
        S.acc_tile[acc] = -1;
        mbar_arrive(&S.tfull[acc]);
        mbar_arrive(&S.tfull[acc]);
        break;
      }
      if (flags & F_END) {
        // a tile whose tasks produce no block product has no data step: still
        // wait for the buffer before publishing its (empty) result
        if (!started) mbar_wait(&S.tempty[acc], acc_phase ^ 1);
        started = false;
        S.acc_tile[acc] = tile;
        tc_commit(&S.tfull[acc]);      // fires when every MMA of the tile is done
        mbar_arrive(&S.tfull[acc]);    // publishes acc_tile
        mbar_arrive(&S.empty[stage]);  // the marker stage carried no data
        ++ntiles_done;
        acc ^= 1;
        if (acc == 0) acc_phase ^= 1;
      } else {
        if (flags & F_FIRST) {
          mbar_wait(&S.tempty[acc], acc_phase ^ 1);
          // the cross accumulator is shared: the previous tile's epilogue must be done
          if (ntiles_done > 0) mbar_wait(&S.cfree, (uint32_t)((ntiles_done - 1) & 1));
          started = true;
        }
        tc_fence_after();
        {
          const uint64_t so = (uint64_t)(((uint32_t)stage * kStageBytes) >> 4);
          const uint32_t d_main = tmem + (uint32_t)acc * 128;  // hi*hi
          const uint32_t d_cross = tmem + kColCross;           // hi*lo + lo*hi
          const uint32_t a_slot = tmem + kColA + 64u * (uint32_t)as;
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            // A: TMEM, K-slice j = columns 8j..8j+7 of the slot's hi (+0) and lo (+32) halves.
            // B MN-major (4 blocks side by side along N, rows = K): 32-byte-atom
            // SW128, LBO 4096 B between the 32-wide atoms (= blocks), SBO 512 B
            // between 4-row K atoms, K-slice j (rows 8j..8j+7) at +1024 B;
            // K-major (transposed B): SW128, SBO 1024 B, K-slice j at +32 B.
            const uint64_t jo = (uint64_t)((kTB ? 32u * j : 1024u * j) >> 4);
            const uint64_t b_hi = bd_hi0 + so + jo;
            const uint64_t b_lo = bd_lo0 + so + jo;
            constexpr uint32_t kIdesc = idesc_tf32_ts<kTB>();
            const uint32_t acc_in = ((flags & F_FIRST) && j == 0) ? 0u : 1u;
            const uint32_t a_hi = a_slot + 8u * j, a_lo = a_hi + 32u;
            tc_mma_ts(d_cross, a_lo, b_hi, kIdesc, acc_in);
            tc_mma_ts(d_cross, a_hi, b_lo, kIdesc, 1u);
            tc_mma_ts(d_main, a_hi, b_hi, kIdesc, acc_in);
          }
          tc_commit(&S.empty[stage]);
          tc_commit(&S.afree[as]);
        }
        as ^= 1;
      }
      if (++stage == kStages) {
        stage = 0;
        phase ^= 1;
      }
    }
    }  // lane 0
  } else {
    // ------------------------------------------------------------ epilogue (warps 0-3)
    float* poolC = static_cast<float*>(a.poolC);
    int acc = 0;
    uint32_t acc_phase = 0;
    for (;;) {
      mbar_wait(&S.tfull[acc], acc_phase);
      const int tile = S.acc_tile[acc];
      if (tile < 0) break;
      tc_fence_after();
      const int4 q4 = a.childC2[tile];
      const int i1 = warp >> 1, i2 = warp & 1;  // C block row i = warp = 2*i1 + i2
#pragma unroll 1
      for (int j = 0; j < 4; ++j) {
        const int j1 = j >> 1, j2 = j & 1;
        const int qs = 2 * i1 + j1;
        const int quad = qs == 0 ? q4.x : qs == 1 ? q4.y : qs == 2 ? q4.z : q4.w;
        int cb = -1;
        if (quad >= 0) {
          const int4 c4 = a.childC1[quad];
          const int s = 2 * i2 + j2;
          cb = s == 0 ? c4.x : s == 1 ? c4.y : s == 2 ? c4.z : c4.w;
        }
        uint32_t v[32], w[32];
        const uint32_t lanes = (uint32_t)(warp * 32) << 16;
        tmem_ld32(tmem + (uint32_t)acc * 128 + lanes + 32u * j, v);  // hi*hi
        tmem_ld32(tmem + kColCross + lanes + 32u * j, w);            // cross terms
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
        for (int c = 0; c < 32; ++c) v[c] = __float_as_uint(__uint_as_float(w[c]) + __uint_as_float(v[c]));
        if (cb >= 0) {
          float* Cb = poolC + (size_t)cb * 1024;
          const int r = lane;  // row of the C block
#pragma unroll
          for (int c = 0; c < 8; ++c) {
            float4 w = make_float4(__uint_as_float(v[4 * c]), __uint_as_float(v[4 * c + 1]),
                                   __uint_as_float(v[4 * c + 2]), __uint_as_float(v[4 * c + 3]));
            *reinterpret_cast<float4*>(Cb + r * 32 + ((c ^ (r & 7)) << 2)) = w;
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        mbar_arrive(&S.tempty[acc]);
        mbar_arrive(&S.cfree);
      }
      acc ^= 1;
      if (acc == 0) acc_phase ^= 1;
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(kTmemCols)
                 : "memory");
  }
}

// Transposed copy of a pool of FP32 blocks (symmetric square): out(r,c) =
// in(c,r), both in the internal 128-byte swizzle (swz32).
__global__ void k_transpose_blocks_f32(const float* __restrict__ in, float* __restrict__ out, int64_t nb) {
  __shared__ float tile[32][33];
  for (int64_t b = blockIdx.x; b < nb; b += gridDim.x) {
    const float* src = in + b * 1024;
    float* dst = out + b * 1024;
    for (int r = threadIdx.x >> 5; r < 32; r += blockDim.x >> 5) {
      const int c = threadIdx.x & 31;
      tile[r][c] = src[swz32(r, c)];
    }
    __syncthreads();
    for (int r = threadIdx.x >> 5; r < 32; r += blockDim.x >> 5) {
      const int c = threadIdx.x & 31;
      dst[swz32(r, c)] = tile[c][r];
    }
    __syncthreads();
  }
}

}  // namespace

void launch_transpose_blocks_f32(qt_ctx ctx, const void* in, void* out, int64_t nb) {
  if (nb <= 0) return;
  const int grid = (int)std::min<int64_t>(nb, 8ll * ctx->num_sms);
  k_transpose_blocks_f32<<<grid, 256, 0, ctx->stream>>>(static_cast<const float*>(in), static_cast<float*>(out),
                                                         nb);
  QT_LAUNCH_CHECK(ctx);
}

template <bool TA, bool TB, bool SYM = false>
static void launch_f32_t(qt_ctx ctx, const NumericArgs32& a, int grid) {
  // the dynamic shared memory limit is a per-device function attribute: set
  // it once per device (bit d of `attr_set`; concurrent first calls only
  // repeat an idempotent call)
  static std::atomic<unsigned long long> attr_set{0};
  const unsigned long long bit = 1ull << (ctx->device & 63);
  if (!(attr_set.load(std::memory_order_acquire) & bit)) {
    QT_CUDA(cudaFuncSetAttribute(k_numeric_f32<TA, TB, SYM>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmemBytes));
    attr_set.fetch_or(bit, std::memory_order_release);
  }
  k_numeric_f32<TA, TB, SYM><<<grid, kThreads, kSmemBytes, a.stream ? a.stream : ctx->stream>>>(a);
}

void launch_numeric_f32(qt_ctx ctx, const NumericArgs32& a) {
  if (!a.counter_ready) QT_CUDA(cudaMemsetAsync(a.counter, 0, sizeof(int), a.stream ? a.stream : ctx->stream));
  const int grid = (int)std::min<int64_t>(a.ntiles, ctx->num_sms);
  if (a.trans & 4) {  // symmetric square
    launch_f32_t<false, false, true>(ctx, a, grid);
    QT_LAUNCH_CHECK(ctx);
    return;
  }
  switch (a.trans & 3) {
    case 0: launch_f32_t<false, false>(ctx, a, grid); break;
    case 1: launch_f32_t<true, false>(ctx, a, grid); break;
    case 2: launch_f32_t<false, true>(ctx, a, grid); break;
    default: launch_f32_t<true, true>(ctx, a, grid); break;
  }
  QT_LAUNCH_CHECK(ctx);
}

}  // namespace qt
