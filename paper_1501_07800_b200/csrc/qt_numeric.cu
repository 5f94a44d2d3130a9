// Numeric block-sparse multiply (K5): C(I,J) = sum_{k ascending} A(I,k) B(k,J)
// for every C block produced by the symbolic pass.
//
// Paper: the leaf multiply is a sum of outer products executed as cuBLAS
// batched GEMMs, one batch per inner index k (Fig.
// fig:block-sparse-mmul).  Here the same block products are instead grouped by
// OUTPUT: a work item ("tile") is a C node at level L-1, i.e. a 2x2 group of
// 32x32 C blocks, together with its ascending-k task list from the symbolic
// pass.  Each step of a tile stages the blocks among A(I0,k), A(I1,k),
// B(k,J0), B(k,J1) that take part in a product, in shared memory with 1-D TMA
// bulk copies (cp.async.bulk, mbarrier complete_tx); four consumer warps each
// own one 16x16 quadrant of all four C blocks and accumulate A(Ii,k)·B(k,Jj)
// in registers with FP64 tensor-core DMMA (mma.sync.m8n8k4.f64) — a staged
// block feeds up to two products.  Each C element is written exactly once: no
// atomics, no batch barriers, and a deterministic summation order (ascending
// k, reading C-5).
//
// CTA = 3 streams x (4 consumer warps + 1 producer warp), persistent (one CTA
// per SM), tiles handed out by an atomic counter in Morton order (L2
// locality); each stream stages through its own ring of 8 KiB block slots.
#include <atomic>

#include <cuda_runtime.h>

#include "qt_common.cuh"
#include "qt_internal.h"

namespace qt {

namespace {

// Independent tile streams per CTA (each: 4 consumer warps + 1 producer
// warp), so every SM sub-partition runs several consumer warps: while one is
// in its tile prologue/epilogue or waits on shared memory, the others keep the
// DMMA pipe busy.
//
// Each stream stages blocks through a ring of kSlotsPer 8 KiB block slots and
// describes its steps in a ring of kHdrPer step headers.  A step takes only
// the slots of the blocks it uses (1-4), so sparse steps (ES-like: 2.9 blocks
// per step on average, random: ~2) keep more steps in flight than fixed
// 4-block stages would.
//
// Three streams (three consumer warps per SM sub-partition: one stream's step
// boundary — header wait, dispatch, tile epilogue — is covered by the other
// two) with 9 slots each: 216 KiB of the 227 KiB of shared memory.  The
// consumers need <= 128 registers for 15 warps to fit one SM.
constexpr int kStreams = 3;
constexpr int kSlotsPer = 9;
constexpr int kHdrPer = 16;
constexpr int kConsumerWarps = 4;
constexpr int kNumThreads = kStreams * (kConsumerWarps + 1) * 32;
constexpr int kBlockElems = 1024;                // 32 x 32
constexpr int kBlockBytes = kBlockElems * 8;     // 8 KiB (FP64)

enum : int { F_COMPUTE = 1, F_STORE = 2, F_DONE = 4 };

struct __align__(16) StageHdr {
  int a[2];      // slot of A(I0,k), A(I1,k) in the stream's ring (-1: not staged)
  int b[2];      // slot of B(k,J0), B(k,J1)
  int c[4];      // F_STORE: C block indices of the tile (slot 2i+j; -1 = none)
  int flags;
  int sub;       // block size 16: quadrant masks of the staged blocks as read (op applied):
                 // bits 0-3 A(I0,k), 4-7 A(I1,k), 8-11 B(k,J0), 12-15 B(k,J1)
  int pmask;     // bit 2i+j: product A(i,k)*B(k,j) at this step
  int slot_end;  // producer bookkeeping: slots allocated up to and including this step
};

// a block product survives: both present and (screening) norms^2 product >= tau^2
// (block size 16: "screening" by the quadrant masks — a product whose
// quadrants never meet adds only zeros and is skipped, as in the BFS)
// kScreen: 0 none, 1 norms, 2 block-size-16 quadrant masks
// kScreen 3 (block size 16 + norm screening): make_step decides per 16-block
// product from the quadrant norms (the step's pair mask), prod_ok only checks presence
// (ta/tb: the block is read transposed — a symmetric square's reference into U)
template <bool kTA, bool kTB, int kScreen>
__device__ __forceinline__ bool prod_ok(int a, int b, const NumericArgs& na, int ta = 0, int tb = 0) {
  if (a < 0 || b < 0) return false;
  if (kScreen == 0 || kScreen == 3) return true;
  if (kScreen == 2) {
    int x = na.subA[a], y = na.subB[b];
    if (kTA || ta) x = mask_t(x);
    if (kTB || tb) y = mask_t(y);
    return mask_meet(x, y);
  }
  return __dmul_rn(na.normA[a], na.normB[b]) >= na.tau2;
}

// a level L-1 child entry -> (block index, transposed) ; plain indices unless symmetric
template <bool kSym>
__device__ __forceinline__ int blk(int ref, int& t) {
  if (!kSym) {
    t = 0;
    return ref;
  }
  t = ref >= 0 ? (ref & 1) : 0;
  return ref >= 0 ? (ref >> 2) : -1;
}

constexpr size_t kSmemBytes = (size_t)kStreams * kSlotsPer * kBlockBytes +
                              kStreams * kHdrPer * sizeof(StageHdr) +
                              2 * kStreams * kHdrPer * sizeof(uint64_t);

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
__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}
__device__ __forceinline__ int4 shfl_int4(int4 v, int src) {
  v.x = __shfl_sync(0xffffffffu, v.x, src);
  v.y = __shfl_sync(0xffffffffu, v.y, src);
  v.z = __shfl_sync(0xffffffffu, v.z, src);
  v.w = __shfl_sync(0xffffffffu, v.w, src);
  return v;
}

// Fragment offsets in the internal swizzled layout (qt_common.cuh swz64) for
// the mma.m8n8k4.f64 operand of row/column x = 16q + 8m + g at k-slice ks:
//   "x-major" element (x, 4ks+t4)  — A as stored, or B read transposed;
//   "k-major" element (4ks+t4, x)  — B as stored, or A read transposed.
// Both patterns hit every 8-byte bank pair exactly twice (the minimum).
__device__ __forceinline__ int off_x(int q, int m, int ks, int g, int t4) {
  return (16 * q + 8 * m + g) * 32 + (((ks ^ (g & 3)) << 2) | t4);
}
__device__ __forceinline__ int off_k(int q, int m, int ks, int g, int t4) {
  return (4 * ks + t4) * 32 + 16 * q + ((8 * m + g) ^ (t4 << 2));
}

// One step of a tile on one consumer warp: warp (qi, qj) accumulates the
// (qi, qj) 16x16 quadrant of C(Ii,Jj) += op(A(Ii,k))·op(B(k,Jj)) for every
// product p = 2i+j of the step (bit p of PM).  Every warp therefore does the
// same number of DMMAs whatever the step's product mask is, so the four SM
// sub-partitions stay balanced on sparse patterns (a step of a banded tile has
// 4 products, an ES-like one 2.2 on average, a random one ~1).  A fragments
// of A(Ii,k) are shared by the products of row i, B fragments of B(k,Jj) by
// those of column j.  PM is a template parameter so that only the step's own
// loads and DMMAs are issued (a predicated-off DMMA still occupies the pipe).
// tA/tB: per-block transposes (bit 0: block 0, bit 1: block 1).
// KS0/NKS: the k-slices [KS0, KS0+NKS) of 4 columns each — the whole block
// (0, 8), or one 16-column half (0, 4) / (4, 4) at block size 16, where the
// k-half h of a product is skipped when the A(Ii,k) quadrant (qi,h) or the
// B(k,Jj) quadrant (h,qj) is absent (reading C-27).
template <int PM, int KS0, int NKS>
__device__ __forceinline__ void warp_step_mma(double (&acc)[4][2][2][2], const double* __restrict__ A0,
                                              const double* __restrict__ A1, const double* __restrict__ B0,
                                              const double* __restrict__ B1, int tA, int tB, int qi,
                                              int qj, int lane) {
  constexpr bool ua0 = PM & 3, ua1 = PM & 12, ub0 = PM & 5, ub1 = PM & 10;
  const int g = lane >> 2, t4 = lane & 3;
#pragma unroll
  for (int ks = KS0; ks < KS0 + NKS; ++ks) {
    double af[2][2], bf[2][2];
#pragma unroll
    for (int m = 0; m < 2; ++m) {
      const int ox = off_x(qi, m, ks, g, t4), ok = off_k(qi, m, ks, g, t4);
      if (ua0) af[0][m] = A0[(tA & 1) ? ok : ox];
      if (ua1) af[1][m] = A1[(tA & 2) ? ok : ox];
    }
#pragma unroll
    for (int n = 0; n < 2; ++n) {
      const int ox = off_x(qj, n, ks, g, t4), ok = off_k(qj, n, ks, g, t4);
      if (ub0) bf[0][n] = B0[(tB & 1) ? ox : ok];
      if (ub1) bf[1][n] = B1[(tB & 2) ? ox : ok];
    }
#pragma unroll
    for (int p = 0; p < 4; ++p) {
      if (PM & (1 << p)) {
#pragma unroll
        for (int m = 0; m < 2; ++m)
#pragma unroll
          for (int n = 0; n < 2; ++n)
            dmma(acc[p][m][n][0], acc[p][m][n][1], af[p >> 1][m], bf[p & 1][n]);
      }
    }
  }
}

template <int KS0 = 0, int NKS = 8>
__device__ __forceinline__ void warp_step(double (&acc)[4][2][2][2], const double* A0, const double* A1,
                                          const double* B0, const double* B1, int pm, int tA, int tB,
                                          int qi, int qj, int lane) {
#define QT_STEP(P) warp_step_mma<P, KS0, NKS>(acc, A0, A1, B0, B1, tA, tB, qi, qj, lane)
  switch (pm) {
    case 0: break;
    case 1: QT_STEP(1); break;
    case 2: QT_STEP(2); break;
    case 3: QT_STEP(3); break;
    case 4: QT_STEP(4); break;
    case 5: QT_STEP(5); break;
    case 6: QT_STEP(6); break;
    case 7: QT_STEP(7); break;
    case 8: QT_STEP(8); break;
    case 9: QT_STEP(9); break;
    case 10: QT_STEP(10); break;
    case 11: QT_STEP(11); break;
    case 12: QT_STEP(12); break;
    case 13: QT_STEP(13); break;
    case 14: QT_STEP(14); break;
    default: QT_STEP(15); break;
  }
#undef QT_STEP
}

// Block size 16: the products p = 2i+j of the step's mask `pm` whose k-half h
// exists for this warp's quadrant (qi, qj): A(Ii,k) has quadrant (qi,h) and
// B(k,Jj) has quadrant (h,qj) (masks as read, bit 2r+c = quadrant (r,c)).
__device__ __forceinline__ int half_mask(int pm, int sub, int qi, int qj, int h) {
  int out = 0;
#pragma unroll
  for (int p = 0; p < 4; ++p) {
    const int i = p >> 1, j = p & 1;
    const int ma = (sub >> (4 * i)) & 15, mb = (sub >> (8 + 4 * j)) & 15;
    if (((pm >> p) & 1) && ((ma >> (2 * qi + h)) & 1) && ((mb >> (2 * h + qj)) & 1)) out |= 1 << p;
  }
  return out;
}

// The two steps (kb = 0, 1) of task p at level L-1: the staged blocks
// A(I0,k) A(I1,k) B(k,J0) B(k,J1) (-1 = not staged) and meta = product mask |
// transposes << 4, computed lane-parallel for 32 tasks at a time so that the
// producer's serial per-step path is only shuffles, the ring wait and the
// TMA issue.
struct StepDesc {
  int a0, a1, b0, b1, meta, sub;  // sub: block size 16 quadrant masks (StageHdr::sub)
};
template <bool kTA, bool kTB, bool kSym, int kScreen>
__device__ __forceinline__ StepDesc make_step(int4 A4, int4 B4, int kb, int keep, const NumericArgs& a) {
  // A child (i,kb) in slot 2i+kb ; B child (kb,j) in slot 2kb+j
  int ta0, ta1, tb0, tb1;
  const int a0 = blk<kSym>(kb ? A4.y : A4.x, ta0), a1 = blk<kSym>(kb ? A4.w : A4.z, ta1);
  const int b0 = blk<kSym>(kb ? B4.z : B4.x, tb0), b1 = blk<kSym>(kb ? B4.w : B4.y, tb1);
  // products of this step: both blocks present and, when screening,
  // ||A(i,k)||^2 * ||B(k,j)||^2 >= tau^2 (the symbolic pass's test)
  const int pm = ((prod_ok<kTA, kTB, kScreen>(a0, b0, a, ta0, tb0) ? 1 : 0) |
                  (prod_ok<kTA, kTB, kScreen>(a0, b1, a, ta0, tb1) ? 2 : 0) |
                  (prod_ok<kTA, kTB, kScreen>(a1, b0, a, ta1, tb0) ? 4 : 0) |
                  (prod_ok<kTA, kTB, kScreen>(a1, b1, a, ta1, tb1) ? 8 : 0)) &
                 keep;
  StepDesc d;
  d.a0 = (pm & 3) ? a0 : -1;
  d.a1 = (pm & 12) ? a1 : -1;
  d.b0 = (pm & 5) ? b0 : -1;
  d.b1 = (pm & 10) ? b1 : -1;
  d.meta = pm | ((ta0 | (ta1 << 1) | (tb0 << 2) | (tb1 << 3)) << 4);
  d.sub = 0;
  if (kScreen == 3) {  // per consumer warp (qi,qj), product p, k-half h: bit 8*(2qi+qj) + 2p + h
    int pm3 = 0;
#pragma unroll
    for (int p = 0; p < 4; ++p) {
      const int ai = (p >> 1) ? a1 : a0, bj = (p & 1) ? b1 : b0;
      if (!((pm >> p) & 1)) continue;
      const int x = a.subA[ai], y = a.subB[bj];
      const int m = screen16(x, y, a.norm16A + 4 * (int64_t)ai, a.norm16B + 4 * (int64_t)bj, a.tau2);
#pragma unroll
      for (int cq = 0; cq < 4; ++cq) {  // C quadrant (r,c) = the consumer warp's quadrant
        d.sub |= ((m >> (2 * cq)) & 3) << (8 * cq + 2 * p);
      }
      if (m) pm3 |= 1 << p;
    }
    d.a0 = (pm3 & 3) ? a0 : -1;
    d.a1 = (pm3 & 12) ? a1 : -1;
    d.b0 = (pm3 & 5) ? b0 : -1;
    d.b1 = (pm3 & 10) ? b1 : -1;
    d.meta = pm3 | (d.meta & ~15);
  }
  if (kScreen == 2) {  // the operands' quadrant masks as the consumers read them
    auto m = [&](const uint8_t* sub, int idx, bool tr) {
      if (idx < 0) return 0;
      const int x = sub[idx];
      return tr ? mask_t(x) : x;
    };
    d.sub = m(a.subA, d.a0, kTA || ta0) | (m(a.subA, d.a1, kTA || ta1) << 4) |
            (m(a.subB, d.b0, kTB || tb0) << 8) | (m(a.subB, d.b1, kTB || tb1) << 12);
  }
  return d;
}

template <bool kTA, bool kTB, bool kSym, int kScreen, bool kPhase, bool kProf = false, bool kMerge = false,
          bool kOut32 = false>
__global__ void __launch_bounds__(kNumThreads, 1) k_numeric_f64(NumericArgs a) {
  // kProf (QT_NUM_PROF=1, diagnostics): per-warp clock64 sums of where the time goes
  unsigned long long pf[5] = {0, 0, 0, 0, 0};
  extern __shared__ __align__(1024) uint8_t smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // warps [0, 4*kStreams): consumers, stream = warp / 4 ; then one producer per stream
  const bool producer = warp >= kStreams * kConsumerWarps;
  const int sid = producer ? warp - kStreams * kConsumerWarps : warp / kConsumerWarps;
  double* data = reinterpret_cast<double*>(smem) + (size_t)sid * kSlotsPer * kBlockElems;
  StageHdr* hdr_all = reinterpret_cast<StageHdr*>(smem + (size_t)kStreams * kSlotsPer * kBlockBytes);
  uint64_t* full_all = reinterpret_cast<uint64_t*>(hdr_all + kStreams * kHdrPer);
  uint64_t* empty_all = full_all + kStreams * kHdrPer;
  StageHdr* hdr = hdr_all + sid * kHdrPer;
  uint64_t* full = full_all + sid * kHdrPer;
  uint64_t* empty = empty_all + sid * kHdrPer;

  if (threadIdx.x == 0) {
    for (int s = 0; s < kStreams * kHdrPer; ++s) {
      mbar_init(&full_all[s], 1);
      mbar_init(&empty_all[s], kConsumerWarps);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  if (producer) {
    // ------------------------------------------------------------ producer
    const long long pf_t0 = kProf ? clock64() : 0;
    // Work is taken in groups of a.group consecutive tiles (one atomic per
    // group; for groups > 1 the next group's atomic is issued before the
    // current group is streamed, so its latency is hidden).  The tasks of a
    // group are a contiguous range of the level L-1 queue; they are streamed 32
    // at a time with lane-parallel metadata loads and step descriptors, across
    // tile boundaries, and a STORE marker is posted at every tile end.  Sparse
    // patterns (few tasks per tile) get large groups, banded/dense ones
    // group = 1 (fine-grained dynamic balance).
    const double* poolA = static_cast<const double*>(a.poolA);
    const double* poolB = static_cast<const double*>(a.poolB);
    const double* poolB2 = static_cast<const double*>(a.poolB2);
    // The metadata of the NEXT batch of 32 tasks (for a new group: the
    // scheduler atomic, the group's tile starts and C children, then the
    // tasks' node ids and child tables) is fetched by a small state machine
    // advanced once per posted step, so its four dependent round trips overlap
    // the ring waits instead of stalling the ring at every group start.  The
    // next group is grabbed when <= kGrabAhead tasks of the current one remain
    // (late enough to keep the dynamic balance of the tail).
    constexpr int kGrabAhead = 8;
    const int G = a.group;
    // phase launches of the multi-rank overlap (kPhase): work items map[t_off + i]
    // (a separate instantiation: the runtime checks cost the plain kernel 2-5 %
    // on sparse patterns)
    int ntiles = (int)a.ntiles, t_off = 0;
    if (a.ntiles_dev) ntiles = *a.ntiles_dev * (a.split ? 4 : 1);  // sync-free: the BFS's count
    if (kPhase) {
      const int ns = *a.nsel;
      const int nt = a.split ? (int)a.ntiles / 4 : (int)a.ntiles;
      t_off = a.phase == 1 ? 0 : ns;
      ntiles = (a.phase == 1 ? ns : nt - ns) * (a.split ? 4 : 1);
    }
    auto tile_of = [&](int i) { return kPhase ? a.tile_map[t_off + i] : i; };
    // current group: tiles [g_t0, g_t0+g_n), lane l: task start of tile g_t0+l (lane g_n: end), C children
    int g_n = 0, g_ts = 0, g_pend = 0;
    int4 g_cc = make_int4(-1, -1, -1, -1);
    // next batch
    int n_state = 0, n_tl = 0, n_t0 = 0, n_n = 0, n_ts = 0, n_pb0 = 0, n_pend = 0, n_pa = -1, n_pb = -1;
    int n_keep = 15, g_keep = 15;  // product mask of the work item (split mode: one C child)
    bool n_newgroup = true, n_valid = false;
    int4 n_cc = make_int4(-1, -1, -1, -1), n_ra = n_cc, n_rb = n_cc;
    StepDesc n_d0{-1, -1, -1, -1, 0, 0}, n_d1{-1, -1, -1, -1, 0, 0};
    auto issue_tasks = [&]() {  // node ids of the next batch
      const int p = n_pb0 + lane;
      n_pa = p < n_pend ? a.pa[p] : -1;
      n_pb = p < n_pend ? a.pb[p] : -1;
    };
    auto adv = [&]() {
      switch (n_state) {
        case 1: {  // scheduler atomic -> group metadata loads
          n_t0 = __shfl_sync(0xffffffffu, n_tl, 0);
          if (n_t0 >= ntiles) {
            n_valid = false;
            n_state = 5;
            break;
          }
          n_valid = true;
          if (a.split) {  // item = (tile, C child q): one product slot of the tile
            const int tile = tile_of(n_t0 >> 2), q = n_t0 & 3;
            n_n = 1;
            n_keep = 1 << q;
            n_ts = lane <= 1 ? a.tile_start[tile + lane] : 0;
            int4 c = make_int4(-1, -1, -1, -1);
            if (lane == 0) {
              const int4 t4 = a.childC[tile];
              if (q == 0) c.x = t4.x;
              if (q == 1) c.y = t4.y;
              if (q == 2) c.z = t4.z;
              if (q == 3) c.w = t4.w;
            }
            n_cc = c;
          } else {
            n_n = min(G, ntiles - n_t0);  // (G == 1 with a tile map)
            const int t0 = tile_of(n_t0);
            n_ts = lane <= n_n ? a.tile_start[t0 + lane] : 0;
            n_cc = lane < n_n ? a.childC[t0 + lane] : make_int4(-1, -1, -1, -1);
          }
          n_state = 2;
          break;
        }
        case 2: {  // group metadata -> first batch's node ids
          n_pb0 = __shfl_sync(0xffffffffu, n_ts, 0);
          n_pend = __shfl_sync(0xffffffffu, n_ts, n_n);
          issue_tasks();
          n_state = 3;
          break;
        }
        case 3: {  // node ids -> child tables
          const int4 nil = make_int4(-1, -1, -1, -1);
          n_ra = n_pa >= 0 ? a.childA[kSym ? (n_pa >> 2) : n_pa] : nil;
          n_rb = n_pb >= 0 ? a.childB[kSym ? (n_pb >> 2) : n_pb] : nil;
          n_state = 4;
          break;
        }
        case 4: {  // child tables -> step descriptors
          if (n_pa >= 0) {
            const int4 ca = op_xform(n_ra, n_pa, kTA, kSym);
            const int4 cb = op_xform(n_rb, n_pb, kTB, kSym);
            const int keep = n_newgroup ? n_keep : g_keep;
            n_d0 = make_step<kTA, kTB, kSym, kScreen>(ca, cb, 0, keep, a);
            n_d1 = make_step<kTA, kTB, kSym, kScreen>(ca, cb, 1, keep, a);
          } else {
            n_d0 = StepDesc{-1, -1, -1, -1, 0, 0};
            n_d1 = n_d0;
          }
          n_state = 5;
          break;
        }
        default: break;
      }
    };
    // Few equal work items (split mode: one C block each): a static
    // round-robin over the SMs — item b + G*(stream + 3*k) — so that no SM
    // holds more than ceil(items / SMs) of them (with the atomic, the CTAs
    // that start first take three items each and the others none).
    int n_grabs = 0;
    auto grab = [&]() {  // start fetching the next group
      n_newgroup = true;
      if (a.split && !kPhase)
        n_tl = blockIdx.x + gridDim.x * (sid + kStreams * n_grabs++);
      else if (lane == 0)
        n_tl = atomicAdd(a.counter, G);
      n_state = 1;
    };
    int posted = 0, released = 0;  // steps posted / known released by the consumers
    int head = 0, freed = 0;       // slots allocated / released (monotonic)
    int slot_pos = 0;              // head % kSlotsPer
    int hpos = 0;                  // posted % kHdrPer
    // wait until a header and n slots are free (consumers release steps in order)
    auto reserve = [&](int n) {
      const long long t0 = kProf ? clock64() : 0;
      while (posted - released >= kHdrPer || head + n - freed > kSlotsPer) {
        const int ri = released % kHdrPer;
        mbar_wait(&empty[ri], (released / kHdrPer) & 1);
        freed = *reinterpret_cast<volatile int*>(&hdr[ri].slot_end);
        ++released;
      }
      if (kProf) pf[0] += clock64() - t0;
    };
    auto post = [&](int flags, int4 cc) {
      adv();
      reserve(0);
      if (lane == 0) {
        StageHdr& h = hdr[hpos];
        h.c[0] = cc.x;
        h.c[1] = cc.y;
        h.c[2] = cc.z;
        h.c[3] = cc.w;
        h.flags = flags;
        h.slot_end = head;
        mbar_arrive(&full[hpos]);
      }
      __syncwarp();
      ++posted;
      if (++hpos == kHdrPer) hpos = 0;
    };
    // A completed tile's STORE rides on the next compute step's header (the
    // consumers store, then compute): one header and barrier round trip less
    // per tile — sparse patterns post about as many tiles as steps.  A tile
    // with no C block posts nothing unless a step accumulated into it (the
    // symmetric square's (1,0) products of a diagonal tile are computed and
    // discarded: the STORE still clears the accumulators).
    bool pend = false, dirty = false;
    int4 pend_cc = make_int4(-1, -1, -1, -1);
    // (kMerge: the instantiation for grouped grabs = sparse tiles only; the
    // dense-tile instantiation keeps the separate STORE headers)
    const bool merge = kMerge;
    auto defer_store = [&](int4 cc) {
      if (cc.x < 0 && cc.y < 0 && cc.z < 0 && cc.w < 0 && !dirty) return;
      if (pend) post(F_STORE, pend_cc);
      if (!merge) {
        post(F_STORE, cc);
        dirty = false;
        return;
      }
      pend = true;
      pend_cc = cc;
      dirty = false;
    };
    const double* poolT = static_cast<const double*>(a.poolT);
    auto asrc = [&](int la, int t) {
      return (kSym && t ? poolT : poolA) + (size_t)la * kBlockElems;
    };
    auto bsrc = [&](int lb) {
      return lb < a.splitB ? poolB + (size_t)lb * kBlockElems
                           : poolB2 + (size_t)(lb - a.splitB) * kBlockElems;
    };
    grab();
    while (n_state < 5) adv();
    int cur = 0, boundary = 0;
    while (n_valid) {
      // promote the prefetched batch
      if (n_newgroup) {
        g_n = n_n;
        g_keep = n_keep;
        g_ts = n_ts;
        g_cc = n_cc;
        g_pend = n_pend;
        cur = 0;
        boundary = __shfl_sync(0xffffffffu, g_ts, 1);
      }
      const int c_pb0 = n_pb0;
      const StepDesc c_d0 = n_d0, c_d1 = n_d1;
      const int c_nloc = max(0, min(32, g_pend - c_pb0));
      const bool last = c_pb0 + 32 >= g_pend;
      n_state = 0;
      if (!last) {  // next batch of the same group
        n_newgroup = false;
        n_pb0 = c_pb0 + 32;
        n_pend = g_pend;
        issue_tasks();
        n_state = 3;
      } else if (g_pend - c_pb0 <= kGrabAhead) {
        grab();
      }
      const long long tu = kProf ? clock64() : 0;
      // only the tasks with a product at one of their two steps (sparse
      // patterns: about half of the level L-1 tasks have none); the tiles
      // they pass are stored on the way
      unsigned live = __ballot_sync(0xffffffffu, lane < c_nloc && ((c_d0.meta | c_d1.meta) & 15));
      while (live) {
        const int u = __ffs(live) - 1;
        live &= live - 1;
        if (last && n_state == 0 && g_pend - (c_pb0 + u) <= kGrabAhead) grab();
        while (c_pb0 + u >= boundary) {  // tile `cur` is complete
          defer_store(shfl_int4(g_cc, cur));
          ++cur;
          boundary = __shfl_sync(0xffffffffu, g_ts, cur + 1);
        }
#pragma unroll
        for (int kb = 0; kb < 2; ++kb) {
          const StepDesc& d = kb ? c_d1 : c_d0;
          const int meta = __shfl_sync(0xffffffffu, d.meta, u);
          if (!(meta & 15)) continue;
          const int la0 = __shfl_sync(0xffffffffu, d.a0, u);
          const int la1 = __shfl_sync(0xffffffffu, d.a1, u);
          const int lb0 = __shfl_sync(0xffffffffu, d.b0, u);
          const int lb1 = __shfl_sync(0xffffffffu, d.b1, u);
          const int sub = kScreen >= 2 ? __shfl_sync(0xffffffffu, d.sub, u) : 0;
          long long ta = kProf ? clock64() : 0;
          adv();
          if (kProf) {
            const long long t1 = clock64();
            pf[1] += t1 - ta;
            ta = t1;
          }
          const int n = (la0 >= 0) + (la1 >= 0) + (lb0 >= 0) + (lb1 >= 0);
          reserve(n);
          if (kProf) ta = clock64();
          // (every lane computes the slots; lane 0 writes the header and the
          // transaction count, then lanes 0-3 issue one bulk copy each in
          // parallel — cfg4 12.37 -> 12.20 ms — except on sparse tiles)
          int sp = slot_pos;
          auto take = [&](int blkidx) {
            if (blkidx < 0) return -1;
            const int sl = sp;
            sp = sp + 1 == kSlotsPer ? 0 : sp + 1;
            return sl;
          };
          const int s0 = take(la0), s1 = take(la1), s2 = take(lb0), s3 = take(lb1);
          uint64_t* fb = &full[hpos];
          if (lane == 0) {
            StageHdr& h = hdr[hpos];
            h.a[0] = s0;
            h.a[1] = s1;
            h.b[0] = s2;
            h.b[1] = s3;
            h.flags = pend ? F_COMPUTE | F_STORE : F_COMPUTE;
            if (pend) {
              h.c[0] = pend_cc.x;
              h.c[1] = pend_cc.y;
              h.c[2] = pend_cc.z;
              h.c[3] = pend_cc.w;
            }
            h.sub = sub;
            h.pmask = meta & 15;
            h.slot_end = head + n;
            mbar_arrive_expect_tx(fb, (uint32_t)kBlockBytes * n);
          }
          if (!kMerge) __syncwarp();  // (sparse tiles: lane 0 issues all, measured faster there)
          if (kMerge ? lane == 0 : lane < 4) {
            // symmetric square: a block of U read transposed comes from the
            // transposed copy of the pool (meta bits 4..7), so the consumers
            // always read blocks as stored
            const int tb = meta >> 4;
            if (kMerge) {
              if (s0 >= 0) bulk_g2s(data + s0 * kBlockElems, asrc(la0, tb & 1), kBlockBytes, fb);
              if (s1 >= 0) bulk_g2s(data + s1 * kBlockElems, asrc(la1, tb & 2), kBlockBytes, fb);
              if (s2 >= 0) bulk_g2s(data + s2 * kBlockElems, bsrc(lb0), kBlockBytes, fb);
              if (s3 >= 0) bulk_g2s(data + s3 * kBlockElems, bsrc(lb1), kBlockBytes, fb);
            } else {
              const int sx = lane == 0 ? s0 : lane == 1 ? s1 : lane == 2 ? s2 : s3;
              if (sx >= 0) {
                const double* src = lane == 0   ? asrc(la0, tb & 1)
                                    : lane == 1 ? asrc(la1, tb & 2)
                                    : lane == 2 ? (kSym ? asrc(lb0, tb & 4) : bsrc(lb0))
                                                : (kSym ? asrc(lb1, tb & 8) : bsrc(lb1));
                bulk_g2s(data + sx * kBlockElems, src, kBlockBytes, fb);
              }
            }
          }
          __syncwarp();
          pend = false;
          dirty = true;
          if (kProf) pf[2] += clock64() - ta;
          head += n;
          slot_pos += n;
          if (slot_pos >= kSlotsPer) slot_pos -= kSlotsPer;
          ++posted;
          if (++hpos == kHdrPer) hpos = 0;
        }
      }
      if (kProf) pf[4] += clock64() - tu;
      if (last) {
        for (; cur < g_n; ++cur) defer_store(shfl_int4(g_cc, cur));
        if (n_state == 0) grab();
      }
      const long long tz = kProf ? clock64() : 0;
      while (n_state < 5) adv();
      if (kProf) pf[3] += clock64() - tz;
    }
    if (pend) post(F_STORE, pend_cc);
    post(F_DONE, make_int4(-1, -1, -1, -1));
    if (kProf && lane == 0) {
      atomicAdd(a.prof + 4, pf[0]);          // producer: waiting for ring space
      atomicAdd(a.prof + 6, (unsigned long long)(clock64() - pf_t0));
      atomicAdd(a.prof + 7, (unsigned long long)posted);
      atomicAdd(a.prof + 9, 1ull);
      atomicAdd(a.prof + 11, pf[1]);  // adv() of compute posts
      atomicAdd(a.prof + 12, pf[2]);  // lane-0 header + TMA issue
      atomicAdd(a.prof + 13, pf[3]);  // end-of-batch metadata completion
      atomicAdd(a.prof + 14, pf[4]);  // the task loop of the batches
    }
  } else {
    // ------------------------------------------------------------ consumers
    const int q = warp % kConsumerWarps;
    const int qi = q >> 1, qj = q & 1;  // this warp's quadrant of every C block
    double* poolC = static_cast<double*>(a.poolC);
    double acc[4][2][2][2];
#pragma unroll
    for (int p = 0; p < 4; ++p)
#pragma unroll
      for (int m = 0; m < 2; ++m)
#pragma unroll
        for (int n = 0; n < 2; ++n) acc[p][m][n][0] = acc[p][m][n][1] = 0.0;
    const int g = lane >> 2, t4 = lane & 3;
    int hi = 0;
    uint32_t phase = 0;
    const long long c_t0 = kProf ? clock64() : 0;
    for (;;) {
      long long tw = kProf ? clock64() : 0;
      mbar_wait(&full[hi], phase);
      if (kProf) {
        const long long t1 = clock64();
        pf[0] += t1 - tw;
        tw = t1;
      }
      const StageHdr& h = hdr[hi];
      const int flags = h.flags;
      if (flags & F_DONE) break;
      if (flags & F_STORE) {  // the tile that just ended (possibly before this header's compute step)
        int cb[4];
#pragma unroll
        for (int p = 0; p < 4; ++p) cb[p] = h.c[p];
        if (!kMerge || !(flags & F_COMPUTE)) {
          __syncwarp();
          if (lane == 0) mbar_arrive(&empty[hi]);
        }
#pragma unroll
        for (int p = 0; p < 4; ++p) {
          if (cb[p] >= 0) {
            if (kOut32) {  // FP32 C (reading C-30): round to nearest, the FP32 pool layout
              float* Cb = reinterpret_cast<float*>(poolC) + (size_t)cb[p] * kBlockElems;
#pragma unroll
              for (int m = 0; m < 2; ++m)
#pragma unroll
                for (int n = 0; n < 2; ++n) {
                  const int r = 16 * qi + 8 * m + g, c = 16 * qj + 8 * n + 2 * t4;
                  *reinterpret_cast<float2*>(Cb + swz32(r, c)) =
                      make_float2(__double2float_rn(acc[p][m][n][0]), __double2float_rn(acc[p][m][n][1]));
                }
            } else {
              double* Cb = poolC + (size_t)cb[p] * kBlockElems;
#pragma unroll
              for (int m = 0; m < 2; ++m)
#pragma unroll
                for (int n = 0; n < 2; ++n) {
                  const int r = 16 * qi + 8 * m + g, c = 16 * qj + 8 * n + 2 * t4;
                  *reinterpret_cast<double2*>(Cb + swz64(r, c)) =
                      make_double2(acc[p][m][n][0], acc[p][m][n][1]);
                }
            }
          }
#pragma unroll
          for (int m = 0; m < 2; ++m)
#pragma unroll
            for (int n = 0; n < 2; ++n) acc[p][m][n][0] = acc[p][m][n][1] = 0.0;
        }
        if (kProf) {
          const long long t1 = clock64();
          pf[2] += t1 - tw;
          tw = t1;
        }
      }
      if (kMerge ? (flags & F_COMPUTE) : !(flags & F_STORE)) {
        const int pm = h.pmask;
        const double* A0 = data + h.a[0] * kBlockElems;
        const double* A1 = data + h.a[1] * kBlockElems;
        const double* B0 = data + h.b[0] * kBlockElems;
        const double* B1 = data + h.b[1] * kBlockElems;
        const int tA = kTA ? 3 : 0, tB = kTB ? 3 : 0;
        if (kScreen == 2) {  // block size 16: only the k-halves whose quadrants exist
          const int sub = h.sub;
          warp_step<0, 4>(acc, A0, A1, B0, B1, half_mask(pm, sub, qi, qj, 0), tA, tB, qi, qj, lane);
          warp_step<4, 4>(acc, A0, A1, B0, B1, half_mask(pm, sub, qi, qj, 1), tA, tB, qi, qj, lane);
        } else if (kScreen == 3) {  // ... and pass the norm screen (this warp's 8 bits of the pair mask)
          const int w8 = (h.sub >> (8 * (2 * qi + qj))) & 255;
          int h0 = 0, h1 = 0;
#pragma unroll
          for (int p = 0; p < 4; ++p) {
            h0 |= ((w8 >> (2 * p)) & 1) << p;
            h1 |= ((w8 >> (2 * p + 1)) & 1) << p;
          }
          warp_step<0, 4>(acc, A0, A1, B0, B1, h0, tA, tB, qi, qj, lane);
          warp_step<4, 4>(acc, A0, A1, B0, B1, h1, tA, tB, qi, qj, lane);
        } else {
          warp_step(acc, A0, A1, B0, B1, pm, tA, tB, qi, qj, lane);
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[hi]);
        if (kProf) {
          pf[1] += clock64() - tw;
          pf[3] += 1;
        }
      }
      if (++hi == kHdrPer) {
        hi = 0;
        phase ^= 1;
      }
    }
    if (kProf && lane == 0) {
      atomicAdd(a.prof + 0, pf[0]);  // consumers: waiting for staged data
      atomicAdd(a.prof + 1, pf[1]);  // compute steps (issue of fragment loads + DMMAs)
      atomicAdd(a.prof + 2, pf[2]);  // tile epilogues (C stores)
      atomicAdd(a.prof + 3, pf[3]);  // compute steps
      atomicAdd(a.prof + 8, (unsigned long long)(clock64() - c_t0));
      atomicAdd(a.prof + 10, 1ull);
    }
  }
}

// Transposed copy of a pool of FP64 blocks (symmetric square: U(i,j)^T is
// read wherever the full matrix has its (j,i) block): out(r,c) = in(c,r), both
// in the internal swizzled layout.  One 32x32 block per 256-thread CTA
// iteration, staged through a padded shared tile.
__global__ void k_transpose_blocks(const double* __restrict__ in, double* __restrict__ out, int64_t nb) {
  __shared__ double tile[32][33];
  for (int64_t b = blockIdx.x; b < nb; b += gridDim.x) {
    const double* src = in + b * kBlockElems;
    double* dst = out + b * kBlockElems;
#pragma unroll
    for (int i = threadIdx.x; i < kBlockElems; i += blockDim.x) {
      const int r = i >> 5, c = (i & 31) ^ ((r & 3) << 2);  // i = swz64(r, c)
      tile[r][c] = src[i];
    }
    __syncthreads();
#pragma unroll
    for (int o = threadIdx.x; o < kBlockElems; o += blockDim.x) {
      const int r = o >> 5, c = (o & 31) ^ ((r & 3) << 2);  // o = swz64(r, c)
      dst[o] = tile[c][r];
    }
    __syncthreads();
  }
}

// ---------------------------------------------------------------- FP64 peaks

__global__ void k_peak_dmma(double* out, int iters) {
  double acc[16][2];
#pragma unroll
  for (int i = 0; i < 16; ++i) acc[i][0] = acc[i][1] = 0.0;
  const double av = 1.0 + threadIdx.x * 1e-9, bv = 1e-9;
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int i = 0; i < 16; ++i) dmma(acc[i][0], acc[i][1], av, bv);
  double s = 0;
#pragma unroll
  for (int i = 0; i < 16; ++i) s += acc[i][0] + acc[i][1];
  if (s == 123.456) out[0] = s;
}

__global__ void k_peak_dfma(double* out, int iters) {
  double x[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) x[i] = threadIdx.x * 1e-3 + i;
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int r = 0; r < 4; ++r)
#pragma unroll
      for (int i = 0; i < 8; ++i) x[i] = fma(x[i], 1.0000001, 1e-9);
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += x[i];
  if (s == 123.456) out[0] = s;
}

}  // namespace

template <bool TA, bool TB, bool SYM = false, int SCR = 0, bool PH = false, bool MG = false, bool O32 = false>
static void launch_numeric_t(qt_ctx ctx, const NumericArgs& a, int grid) {
  static const bool prof = getenv("QT_NUM_PROF") != nullptr;
  if (prof && !TA && !TB && (SCR == 0 || SCR == 2) && !PH && !O32) {  // diagnostics: the instrumented kernel
    static bool set = false;
    if (!set) {
      QT_CUDA(cudaFuncSetAttribute(k_numeric_f64<false, false, SYM, SCR, false, true, MG>,
                                   cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmemBytes));
      set = true;
    }
    cudaStream_t st = a.stream ? a.stream : ctx->stream;
    DevBuf pb(16 * 8, st);
    QT_CUDA(cudaMemsetAsync(pb.p, 0, 16 * 8, st));
    NumericArgs b = a;
    b.prof = pb.as<unsigned long long>();
    k_numeric_f64<false, false, SYM, SCR, false, true, MG><<<grid, kNumThreads, kSmemBytes, st>>>(b);
    unsigned long long h[16];
    QT_CUDA(cudaMemcpyAsync(h, pb.p, 16 * 8, cudaMemcpyDeviceToHost, st));
    QT_CUDA(cudaStreamSynchronize(st));
    const double nc = (double)h[10], np = (double)h[9];
    fprintf(stderr,
            "[qt numeric prof] consumer warps %.0f: total %.0f cyc, wait-data %.0f, compute %.0f, store %.0f, "
            "steps %.1f | producers %.0f: total %.0f, wait-ring %.0f, posts %.1f, adv %.0f, issue %.0f, "
            "batch-end %.0f, task-loop %.0f\n",
            nc, h[8] / nc, h[0] / nc, h[1] / nc, h[2] / nc, h[3] / nc, np, h[6] / np, h[4] / np, h[7] / np,
            h[11] / np, h[12] / np, h[13] / np, h[14] / np);
    return;
  }
  // the dynamic shared memory limit is a per-device function attribute: set
  // it once per device (bit d of `attr_set`; concurrent first calls only
  // repeat an idempotent call)
  static std::atomic<unsigned long long> attr_set{0};
  const unsigned long long bit = 1ull << (ctx->device & 63);
  if (!(attr_set.load(std::memory_order_acquire) & bit)) {
    QT_CUDA(cudaFuncSetAttribute(k_numeric_f64<TA, TB, SYM, SCR, PH, false, MG, O32>,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmemBytes));
    attr_set.fetch_or(bit, std::memory_order_release);
  }
  k_numeric_f64<TA, TB, SYM, SCR, PH, false, MG, O32>
      <<<grid, kNumThreads, kSmemBytes, a.stream ? a.stream : ctx->stream>>>(a);
}

void launch_numeric(qt_ctx ctx, qt_dtype dt, const NumericArgs& a0) {
  if (dt != QT_F64) fail(QT_EDTYPE, "launch_numeric is the FP64 kernel");
  if (!a0.counter_ready) QT_CUDA(cudaMemsetAsync(a0.counter, 0, sizeof(int), a0.stream ? a0.stream : ctx->stream));
  // Few tiles (fewer than half the tile streams of the GPU): every C block of
  // a tile becomes its own work item, so more streams share the work — a lone
  // stream per SM is latency bound (its 9-slot ring covers ~2 steps of TMA
  // latency).  Config 1 (64 tiles): numeric 60 -> 29 us.
  NumericArgs a = a0;
  if (a.ntiles * 2 < (int64_t)ctx->num_sms * kStreams) {
    a.split = 1;
    a.ntiles = 4 * a0.ntiles;
    a.group = 1;
  }
  const int grid = (int)std::min<int64_t>(a.ntiles, ctx->num_sms);
  // a.group: one tile per grab (dense/banded: finest dynamic balance) or
  // grouped grabs (sparse patterns: amortise the scheduler and metadata latency)
  if (a.out_f32) {  // FP32 C from FP64 operands (reading C-30): plain products, any transposes
    if (a.phase || (a.trans & 4) || a.normA || a.norm16A) fail(QT_EINVAL, "FP32 output: plain products only");
    if (a.subA) {
      switch (a.trans & 3) {
        case 0: launch_numeric_t<false, false, false, 2, false, false, true>(ctx, a, grid); break;
        case 1: launch_numeric_t<true, false, false, 2, false, false, true>(ctx, a, grid); break;
        case 2: launch_numeric_t<false, true, false, 2, false, false, true>(ctx, a, grid); break;
        default: launch_numeric_t<true, true, false, 2, false, false, true>(ctx, a, grid); break;
      }
    } else {
      switch (a.trans & 3) {
        case 0:
          if (a.group > 1)
            launch_numeric_t<false, false, false, 0, false, true, true>(ctx, a, grid);
          else
            launch_numeric_t<false, false, false, 0, false, false, true>(ctx, a, grid);
          break;
        case 1: launch_numeric_t<true, false, false, 0, false, false, true>(ctx, a, grid); break;
        case 2: launch_numeric_t<false, true, false, 0, false, false, true>(ctx, a, grid); break;
        default: launch_numeric_t<true, true, false, 0, false, false, true>(ctx, a, grid); break;
      }
    }
  } else if (a.phase) {  // multi-rank overlap phases: plain (or bs-16 masked) products only
    if (a.trans & 7) fail(QT_EINVAL, "overlap phases are built for the plain product");
    if (a.subA && a.norm16A)
      launch_numeric_t<false, false, false, 3, true>(ctx, a, grid);
    else if (a.subA)
      launch_numeric_t<false, false, false, 2, true>(ctx, a, grid);
    else if (a.normA)
      launch_numeric_t<false, false, false, 1, true>(ctx, a, grid);
    else
      launch_numeric_t<false, false, false, 0, true>(ctx, a, grid);
  } else if (a.trans & 4) {  // symmetric square (block size 16: k-halves by the quadrant masks)
    if (a.subA)
      launch_numeric_t<false, false, true, 2>(ctx, a, grid);
    else
      launch_numeric_t<false, false, true>(ctx, a, grid);
  } else if (a.subA && a.norm16A) {  // block size 16, norm-screened (plain product)
    if (a.trans & 3) fail(QT_EINVAL, "the screened product is built for the plain product");
    launch_numeric_t<false, false, false, 3>(ctx, a, grid);
  } else if (a.normA) {  // norm-screened product
    switch (a.trans & 3) {
      case 0: launch_numeric_t<false, false, false, 1>(ctx, a, grid); break;
      case 1: launch_numeric_t<true, false, false, 1>(ctx, a, grid); break;
      case 2: launch_numeric_t<false, true, false, 1>(ctx, a, grid); break;
      default: launch_numeric_t<true, true, false, 1>(ctx, a, grid); break;
    }
  } else if (a.subA) {  // block size 16: products whose quadrant masks never meet are skipped
    switch (a.trans & 3) {
      case 0: launch_numeric_t<false, false, false, 2>(ctx, a, grid); break;
      case 1: launch_numeric_t<true, false, false, 2>(ctx, a, grid); break;
      case 2: launch_numeric_t<false, true, false, 2>(ctx, a, grid); break;
      default: launch_numeric_t<true, true, false, 2>(ctx, a, grid); break;
    }
  } else {
    switch (a.trans & 3) {
      case 0:  // (grouped grabs: the STORE-merging instantiation)
        if (a.group > 1)
          launch_numeric_t<false, false, false, 0, false, true>(ctx, a, grid);
        else
          launch_numeric_t<false, false>(ctx, a, grid);
        break;
      case 1: launch_numeric_t<true, false>(ctx, a, grid); break;
      case 2: launch_numeric_t<false, true>(ctx, a, grid); break;
      default: launch_numeric_t<true, true>(ctx, a, grid); break;
    }
  }
  QT_LAUNCH_CHECK(ctx);
}

void launch_transpose_blocks(qt_ctx ctx, const void* in, void* out, int64_t nb) {
  if (nb <= 0) return;
  const int grid = (int)std::min<int64_t>(nb, 8ll * ctx->num_sms);
  k_transpose_blocks<<<grid, 256, 0, ctx->stream>>>(static_cast<const double*>(in),
                                                     static_cast<double*>(out), nb);
  QT_LAUNCH_CHECK(ctx);
}

// kind 0: DMMA (512 flop per mma per warp), kind 1: DFMA (2 flop per lane)
void launch_fp64_peak(qt_ctx ctx, int kind, int iters, int grid) {
  double* out = ctx->counters.as<double>() + 12;
  if (kind == 0)
    k_peak_dmma<<<grid, 256, 0, ctx->stream>>>(out, iters);
  else
    k_peak_dfma<<<grid, 256, 0, ctx->stream>>>(out, iters);
  QT_LAUNCH_CHECK(ctx);
}

}  // namespace qt
