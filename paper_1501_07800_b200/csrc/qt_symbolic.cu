// Symbolic multiply (K3/K4/K7): level-synchronous BFS over the quadtrees of A
// and B that produces, level by level, the compacted queue of multiply tasks.
//
// Paper: the task C = AB (§3.2) registers, for a non-leaf node
// pair, the child products A_ik * B_kj (i, k, j in {0,1}) and skips every
// product with a NIL operand; a C node is assembled from the sums over k of
// its child products.  Here one BFS level = one level of that
// recursion for all tasks at once:
//   frontier(l)  = the tasks (a_node, b_node) at level l, grouped by the C
//                  node they contribute to (C nodes in Morton order), inside a
//                  group sorted by ascending k;
//   frontier(l+1): task p of C node s expands to child tasks (A_{ik}, B_{kj})
//                  of C child q = (i,j); the new group of (s,q) lists, for
//                  every parent task in order, k = 0 then k = 1 — so groups
//                  stay sorted by ascending global k with no sort at all.
// |frontier(l)| is the paper's task count C_l.  C's quadtree falls
// out of the same pass: the non-empty groups (s,q) are C's nodes at level l+1
// and their indices are C's child table at level l (the "assemble" task,
// P:286-294).  The last transition (to the block level) only counts: the
// numeric kernel consumes the level L-1 queue directly, one 2x2-block C node
// (a "tile") per work item.
//
// Host synchronisation: the task count of every level is known before the BFS
// starts — C_l = sum_K colcount(A_l)[K] * rowcount(B_l)[K] from per-level
// occupancy histograms kept with each matrix — so all frontier buffers are
// sized exactly and the BFS runs without host round trips.  The top levels
// (frontiers up to 8K tasks) run in ONE single-CTA kernel with block-wide
// scans (plain products start at level <= 4 from dense node maps); the large
// levels in ONE persistent cooperative kernel whose phases are separated by
// grid-wide barriers.  One host sync remains for large products, before the
// numeric kernel (to size C's block pool); small products size C by an upper
// bound and run sync-free (multiply_local).
#include <atomic>
#include <chrono>
#include <cstdlib>
#include <cub/cub.cuh>

#include "qt_common.cuh"
#include "qt_internal.h"

namespace qt {

namespace {

constexpr int kSmallThreads = 1024;
constexpr int64_t kSmallMaxF = 1 << 13;



// C node on the block diagonal: in the symmetric square only its upper
// children exist (the (1,0) child is the transpose of (0,1), not computed)
__device__ __forceinline__ bool on_diagonal(uint64_t ckey) {
  return morton_row(ckey) == morton_col(ckey);
}

// C children (bit q = child (i,j), q = 2i+j) of C node `ck` at level l that
// are computed: not the (1,0) child of a diagonal node in the symmetric
// square's pruned levels, and only children whose block rows meet the row
// window [rlo, rhi) (a rank's strip in the multi-rank symmetric square)
// (the node key is loaded only when a rule needs it)
__device__ __forceinline__ int cmask(const uint64_t* __restrict__ ckp, int l, int L, bool prune, int32_t rlo,
                                     int32_t rhi) {
  const bool window = rlo > 0 || rhi < INT32_MAX;
  if (!prune && !window) return 0xF;
  const uint64_t ck = *ckp;
  int m = (prune && on_diagonal(ck)) ? 0xB : 0xF;
  if (window) {
    const int64_t r = morton_row(ck);
    const int sh = L - l - 1;
#pragma unroll
    for (int i = 0; i < 2; ++i) {
      const int64_t a0 = (2 * r + i) << sh, a1 = (2 * r + i + 1) << sh;
      if (a1 <= rlo || a0 >= rhi) m &= i ? ~0xC : ~0x3;
    }
  }
  return m;
}

// A child (i,k) sits in slot 2i+k, B child (k,j) in slot 2k+j, C child (i,j) in 2i+j.
// Norm screening (qt_multiply_screened): a child task (a, b) survives iff
// ||a||^2 * ||b||^2 >= tau^2, squared Frobenius norms of quadtree nodes.  A
// node's squared norm is the sum of its blocks', so a node pair below the
// threshold contains only block pairs below it: pruning at any level is exact
// with respect to the block-level test.  na == nullptr: no screening.
// Block size 16 (qt_bs16.cu): at the block level a pair whose quadrant masks
// never meet has no 16-block product and is skipped (ma/mb: the operands'
// masks, tr: transposed operands), so C gets no container without one.
struct Screen {
  const double* na;
  const double* nb;
  double tau2;
  const uint8_t* ma = nullptr;
  const uint8_t* mb = nullptr;
  int tr = 0;
  const double* n16a = nullptr;  // block size 16 + screening: squared 16-block norms [nb][4]
  const double* n16b = nullptr;
};
__device__ __forceinline__ bool pair_ok(int ar, int br, const Screen& sc, bool sym) {
  if (ar < 0 || br < 0) return false;
  if (sc.ma) {  // (symmetric square: references into U carry the transpose bit)
    int x = sc.ma[sym ? (ar >> 2) : ar], y = sc.mb[sym ? (br >> 2) : br];
    if (sym ? (ar & 1) : (sc.tr & 1)) x = mask_t(x);
    if (sym ? (br & 1) : (sc.tr & 2)) y = mask_t(y);
    // screened (plain product only): some 16-block product passes the test
    if (sc.n16a) return screen16(x, y, sc.n16a + 4 * (int64_t)ar, sc.n16b + 4 * (int64_t)br, sc.tau2) != 0;
    return mask_meet(x, y);
  }
  if (!sc.na) return true;
  const int ai = sym ? (ar >> 2) : ar, bi = sym ? (br >> 2) : br;
  return __dmul_rn(sc.na[ai], sc.nb[bi]) >= sc.tau2;
}
__device__ __forceinline__ void child_counts(int4 a, int4 b, int (&c)[4], const Screen& sc, bool sym) {
  c[0] = pair_ok(a.x, b.x, sc, sym) + pair_ok(a.y, b.z, sc, sym);  // (0,0)
  c[1] = pair_ok(a.x, b.y, sc, sym) + pair_ok(a.y, b.w, sc, sym);  // (0,1)
  c[2] = pair_ok(a.z, b.x, sc, sym) + pair_ok(a.w, b.z, sc, sym);  // (1,0)
  c[3] = pair_ok(a.z, b.y, sc, sym) + pair_ok(a.w, b.w, sc, sym);  // (1,1)
}

// Write the child tasks of task p (group s, local index loc) at the exclusive
// offsets `off` of its (s,q) slots; gidx maps (s,q) to the new group index.
__device__ __forceinline__ void emit_task(int4 a4, int4 b4, int64_t base, int32_t m, int32_t s,
                                          int cm, const Screen& sc, bool sym,
                                          const int32_t* __restrict__ off,
                                          const int32_t* __restrict__ gidx, int32_t* __restrict__ pa2,
                                          int32_t* __restrict__ pb2, int32_t* __restrict__ pc2) {
  const int a[4] = {a4.x, a4.y, a4.z, a4.w};
  const int b[4] = {b4.x, b4.y, b4.z, b4.w};
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    if (!((cm >> q) & 1)) continue;
    const int i = q >> 1, j = q & 1;
    int32_t pos = -1, newc = -1;
#pragma unroll
    for (int k = 0; k < 2; ++k) {
      const int ac = a[2 * i + k], bc = b[2 * k + j];
      if (pair_ok(ac, bc, sc, sym)) {
        if (pos < 0) {
          pos = off[base + (int64_t)q * m];
          newc = gidx[4 * s + q];
        }
        pa2[pos] = ac;
        pb2[pos] = bc;
        pc2[pos] = newc;
        ++pos;
      }
    }
  }
}

// ------------------------------------------------------------ small levels (one CTA)

struct SmallBfsArgs {
  int l_end;  // run transitions l -> l+1 for l < l_end
  int L;      // the block level: the transition L-1 -> L only counts (no emit)
  int trans;  // mode: bit 0 A transposed, bit 1 B transposed, bit 2 symmetric square
  const int4* childA[QT_MAX_LEVELS];
  const int4* childB[QT_MAX_LEVELS];
  int32_t* pa[2];
  int32_t* pb[2];
  int32_t* pc[2];
  int32_t* cstart[2];
  uint64_t* ckey[2];
  int32_t* off;     // 4 * max F scratch (counts, then exclusive offsets in place)
  int32_t* gidx;    // 4 * max ns scratch
  int32_t* ns_out;  // C groups per level
  int32_t* f_out;   // tasks per level
  const double* normA[QT_MAX_LEVELS];  // squared node norms per level (screening), or null
  const double* normB[QT_MAX_LEVELS];
  double tau2;
  int32_t row_lo, row_hi;  // C row window (block rows)
  const uint8_t* subA;     // block size 16: quadrant masks (pair test at the block level)
  const uint8_t* subB;
  const double* n16A;      // block size 16 + screening: squared 16-block norms, or null
  const double* n16B;
  unsigned long long* prof;  // QT_BFS_PROF: per-phase %globaltimer marks (diagnostics), or null
  int* zero;                 // the numeric kernel's scheduler counters, zeroed here (saves a memset launch)
  int tiny_cap;              // the tiny variant's shared-memory frontier capacity
  int32_t* host_counts;      // sync-free products: [ns(L+1) | F(L+1)] written to mapped host memory, or null
  int32_t nodesA[QT_MAX_LEVELS];  // child-table rows per level (L2 prefetch at kernel start)
  int32_t nodesB[QT_MAX_LEVELS];
  int l0 = 0;  // dense start: levels 1..l0 from the dense node maps (0: off)
  const int32_t* dmapA = nullptr;  // the operands' dense top-level node maps (qt_mat_s::dmap)
  const int32_t* dmapB = nullptr;
  int stage_cap = 0;  // dense start into global memory: tasks staged in shared memory (after the tiny area), or 0
};

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

// kExt: the block-size-16 pair test and the C row window (multi-rank
// symmetric square) are compiled in only for the launches that use them — the
// runtime checks cost the plain BFS ~10 % (cfg4)
// kSmem: the frontiers of the levels nobody reads after the kernel (all but
// level l_end, and level L-1 when the kernel runs to the block level), the
// scan scratch `off` and the (s,q) -> group map live in shared memory
// (dynamic, kTinyF tasks / groups per level), so a level costs the child-table
// gathers and block barriers only, not ~7 dependent round trips to L2.
constexpr int kTinyF = 2048;
// dynamic shared memory of the tiny variant for levels of <= cap tasks (the
// launch asks only for what the problem's levels need: a large carve-out
// costs the launch several microseconds)
__host__ __device__ inline size_t tiny_smem(int cap) {
  return 2 * (3 * 4 + 4 + 8) * (size_t)cap + 4 * 2 * (size_t)cap + 4 * 4 * (size_t)cap + 4 * 4 * (size_t)cap + 64;
}

// kMode — instantiations without the runtime mode branches: 1 plain or
// transposed products (kPlain: no symmetric references, no norm tests — the
// pair test is two NIL checks; dense start), 2 the symmetric square (symmetric
// references always, no norm tests), 3 screened plain products (norm tests,
// no symmetric references); 0 generic (runtime flags).  The tiny
// levels are latency and instruction-fetch bound, so the smaller code pays.
template <bool kExt, bool kSmem, int kMode>
__global__ void __launch_bounds__(kSmem ? 256 : kSmallThreads, 1) k_bfs_small(SmallBfsArgs a) {
  constexpr bool kPlain = kMode == 1, kNoNorms = kMode == 1 || kMode == 2;
  // the tiny variant runs 256 threads: its levels have <= kTinyF tasks and
  // its cost is the latency of block scans and barriers, cheaper with 8 warps
  constexpr int kT = kSmem ? 256 : kSmallThreads;
  using BS = cub::BlockScan<int, kT>;
  __shared__ typename BS::TempStorage tmp;
  __shared__ int s_F, s_ns;
  extern __shared__ __align__(16) uint8_t tiny[];
  const int tid = threadIdx.x;
  const bool sym = kMode == 2 || (kMode == 0 && (a.trans & 4));
  // per-level buffers: shared memory unless the level is read after the kernel
  uint64_t* ck0 = reinterpret_cast<uint64_t*>(tiny);
  const int T = a.tiny_cap;  // capacity (tasks / groups per level) of the shared-memory frontiers
  int32_t* base = reinterpret_cast<int32_t*>(ck0 + 2 * T);
  int32_t* off = kSmem ? base + 8 * T + 8 : a.off;
  int32_t* gidx_s = kSmem ? off + 4 * T : a.gidx;
  auto glob = [&](int l) { return !kSmem || l == a.l_end || (a.l_end == a.L && l == a.L - 1); };
  auto PA = [&](int l) { return glob(l) ? a.pa[l & 1] : base + (l & 1) * T; };
  auto PB = [&](int l) { return glob(l) ? a.pb[l & 1] : base + (2 + (l & 1)) * T; };
  auto PC = [&](int l) { return glob(l) ? a.pc[l & 1] : base + (4 + (l & 1)) * T; };
  auto CS = [&](int l) { return glob(l) ? a.cstart[l & 1] : base + 6 * T + (l & 1) * (T + 4); };
  auto CK = [&](int l) { return glob(l) ? a.ckey[l & 1] : ck0 + (l & 1) * T; };
  int np = 0;
  auto mark = [&]() {
    if (a.prof && tid == 0 && np < 40) a.prof[np] = gtimer();
    ++np;
  };
  mark();
  // one DRAM round trip for every child table the kernel will gather from
  // (they were evicted from L2 by the previous numeric pass), instead of one
  // per level
  // (the dense start's levels are read off the node maps, not gathered)
  for (int l = kPlain ? a.l0 : 0; l < a.l_end; ++l) {
    const char* ta = reinterpret_cast<const char*>(a.childA[l]);
    const char* tb = reinterpret_cast<const char*>(a.childB[l]);
    for (int i = tid; i < a.nodesA[l] / 8 + 1; i += kT)
      asm volatile("prefetch.global.L2 [%0];" ::"l"(ta + 128 * (size_t)i));
    if (tb != ta)
      for (int i = tid; i < a.nodesB[l] / 8 + 1; i += kT)
        asm volatile("prefetch.global.L2 [%0];" ::"l"(tb + 128 * (size_t)i));
  }
  // per-level table pointers copied to shared memory once: indexing the
  // (large) parameter block by the level is a constant-cache miss per level
  __shared__ const int4* s_cA[QT_MAX_LEVELS];
  __shared__ const int4* s_cB[QT_MAX_LEVELS];
  __shared__ const double* s_nA[QT_MAX_LEVELS];
  __shared__ const double* s_nB[QT_MAX_LEVELS];
  if (tid < QT_MAX_LEVELS && tid <= a.L) {
    s_cA[tid] = a.childA[tid];
    s_cB[tid] = a.childB[tid];
    if (!kNoNorms) {
      s_nA[tid] = a.normA[tid];
      s_nB[tid] = a.normB[tid];
    }
  }
  if (tid < 2) a.zero[tid] = 0;
  if (tid == 0) {
    PA(0)[0] = sym ? 2 : 0;  // the root (a diagonal node in the symmetric square)
    PB(0)[0] = sym ? 2 : 0;
    PC(0)[0] = 0;
    a.f_out[0] = 1;
    CS(0)[0] = 0;
    CS(0)[1] = 1;
    CK(0)[0] = 0;
    a.ns_out[0] = 1;
    s_F = 1;
    s_ns = 1;
  }
  __syncthreads();
  int l_start = 0;
  if (kPlain && a.l0 > 0) {
    // Dense start (plain and transposed products): the tasks of level l0 are
    // every pair (op(A)(i,k), op(B)(k,j)) of non-NIL level-l0 nodes — the
    // recursion of §3.2 registers exactly those, a NIL operand at
    // any coarser level having no non-NIL descendants — so the first l0
    // transitions are replaced by a lookup in the operands' dense
    // Morton-indexed node maps of the top l0 levels (4^l nodes at level l,
    // kept with each matrix: build_levels) and one block scan.
    // Order as the BFS: groups (C nodes) in Morton order, ascending k inside.
    constexpr int kDenseMax = 341;  // 1 + 4 + 16 + 64 + 256: levels 0..4
    __shared__ int32_t sDA[kDenseMax], sDB[kDenseMax];
    __shared__ int s_lf[8], s_lns[8];
    const int l0 = a.l0;
    const int nmap = ((4 << (2 * l0)) - 1) / 3;  // levels 0..l0
    for (int t = tid; t < nmap; t += kT) {
      sDA[t] = a.dmapA[t];
      sDB[t] = a.dmapB[t];
    }
    if (tid < 8) s_lf[tid] = s_lns[tid] = 0;
    __syncthreads();
    // tasks and C nodes of the levels 1..l0-1 (statistics) and of level l0
    // (emitted): C node m of level l pairs with k = 0 .. 2^l - 1
    const bool tA = a.trans & 1, tB = a.trans & 2;
    // Morton index of (r, c) at a level <= 4: the bits of r and c (< 16) interleaved
    auto sp4 = [](int x) { return (x & 1) | ((x & 2) << 1) | ((x & 4) << 2) | ((x & 8) << 3); };
    auto spread_rc = [&](int m, int& ri, int& cj) {  // m -> spread row / column bits
      ri = (m >> 1) & 0x55;
      cj = m & 0x55;
    };
    unsigned kmask = 0;
    int cnt0 = 0, rA0 = 0, rB0 = 0;
    for (int l = 1, o = 1; l <= l0; o += 1 << (2 * l), ++l) {
      const int K = 1 << l;
      for (int m = tid; m < K * K; m += kT) {
        int si, sj;
        spread_rc(m, si, sj);
        // op(A)(i,k) at Morton (i,k), or (k,i) transposed; op(B)(k,j) likewise
        const int ra = tA ? si : si << 1, ka = tA ? 1 : 0;
        const int rb = tB ? sj << 1 : sj, kb = tB ? 0 : 1;
        int c = 0;
        unsigned msk = 0;
        for (int k = 0; k < K; ++k) {
          const int sk = sp4(k);
          const int xa = sDA[o + (ra | (sk << ka))];
          const int xb = sDB[o + (rb | (sk << kb))];
          if (xa >= 0 && xb >= 0) {
            ++c;
            msk |= 1u << k;
          }
        }
        if (l == l0) {  // (K * K <= kT: one C node per thread)
          kmask = msk;
          cnt0 = c;
          rA0 = ra | (ka << 8);
          rB0 = rb | (kb << 8);
        } else if (c > 0) {
          atomicAdd(&s_lf[l], c);
          atomicAdd(&s_lns[l], 1);
        }
      }
    }
    // level l0: packed scan (tasks in the low 16 bits, groups above: <= 4096 / 256)
    int ex, agg;
    BS(tmp).ExclusiveSum(cnt0 + ((cnt0 > 0) << 16), ex, agg);
    const int o0 = ((1 << (2 * l0)) - 1) / 3;  // offset of level l0 in the dense maps
    // (a level l0 handed to the next kernel is written through a shared-memory
    // stage: each thread's tasks are contiguous, so direct stores would be
    // 32 scattered sectors per warp instruction)
    int32_t* stg = a.stage_cap > 0 ? reinterpret_cast<int32_t*>(tiny + tiny_smem(T)) : nullptr;
    if (cnt0 > 0) {
      int pos = ex & 0xFFFF;
      const int g = ex >> 16;
      CS(l0)[g] = pos;
      CK(l0)[g] = (uint64_t)tid;
      int32_t *pa0 = stg ? stg : PA(l0), *pb0 = stg ? stg + a.stage_cap : PB(l0),
              *pc0 = stg ? stg + 2 * a.stage_cap : PC(l0);
      for (unsigned msk = kmask; msk; msk &= msk - 1) {
        const int sk = sp4(__ffs(msk) - 1);
        pa0[pos] = sDA[o0 + ((rA0 & 0xFF) | (sk << (rA0 >> 8)))];
        pb0[pos] = sDB[o0 + ((rB0 & 0xFF) | (sk << (rB0 >> 8)))];
        pc0[pos] = g;
        ++pos;
      }
    }
    __syncthreads();
    if (stg) {
      const int F0 = agg & 0xFFFF;
      int32_t *pa0 = PA(l0), *pb0 = PB(l0), *pc0 = PC(l0);
      for (int i = tid; i < F0; i += kT) {
        pa0[i] = stg[i];
        pb0[i] = stg[a.stage_cap + i];
        pc0[i] = stg[2 * a.stage_cap + i];
      }
    }
    if (tid == 0) {
      const int F0 = agg & 0xFFFF, ns0 = agg >> 16;
      CS(l0)[ns0] = F0;
      for (int l = 1; l < l0; ++l) {
        a.f_out[l] = s_lf[l];
        a.ns_out[l] = s_lns[l];
      }
      a.f_out[l0] = F0;
      a.ns_out[l0] = ns0;
      s_F = F0;
      s_ns = ns0;
    }
    __syncthreads();
    l_start = l0;
    mark();
  }
  for (int l = l_start; l < a.l_end; ++l) {
    const bool prune = sym && l < (a.trans >> 8);  // C below the diagonal is not computed
    const int F = s_F, ns = s_ns;
    const int32_t* pa = PA(l);
    const int32_t* pb = PB(l);
    const int32_t* pc = PC(l);
    const int32_t* cs = CS(l);
    const uint64_t* ck = CK(l);
    int32_t* csn = CS(l + 1);
    uint64_t* ckn = CK(l + 1);
    // the group map of the last transition is C's child table when the kernel reaches the blocks
    int32_t* gidx = (!kSmem || (a.l_end == a.L && l == a.L - 1)) ? a.gidx : gidx_s;
    const int4* cA = s_cA[l];
    const int4* cB = s_cB[l];
    const bool lastl = kExt && l + 1 == a.L && a.subA;
    const Screen sc{kNoNorms ? nullptr : s_nA[l + 1], kNoNorms ? nullptr : s_nB[l + 1], a.tau2, lastl ? a.subA : nullptr, lastl ? a.subB : nullptr,
                    a.trans & 3, lastl ? a.n16A : nullptr, lastl ? a.n16B : nullptr};
    const int32_t rlo = kExt ? a.row_lo : 0, rhi = kExt ? a.row_hi : INT32_MAX;
    // 1. child-task counts per (task, C child), group-major
    auto count_task = [&](int p, int4 rA, int4 rB) {
      const int s = pc[p], c0 = cs[s], m = cs[s + 1] - c0;
      int c[4];
      child_counts(rA, rB, c, sc, sym);
      const int cm = cmask(ck + s, l, a.L, prune, rlo, rhi);
#pragma unroll
      for (int q = 0; q < 4; ++q)
        if (!((cm >> q) & 1)) c[q] = 0;
      const int64_t base = 4ll * c0 + (p - c0);
#pragma unroll
      for (int q = 0; q < 4; ++q) off[base + (int64_t)q * m] = c[q];
    };
    for (int p = tid; p < F; p += kT)
      count_task(p, op_children(cA, pa[p], a.trans & 1, sym), op_children(cB, pb[p], a.trans & 2, sym));
    __syncthreads();
    mark();
    // 2. exclusive scan in place (kIt consecutive entries per thread: a level
    // of F tasks takes 4F / (kT kIt) block scans, not 4F / kT)
    constexpr int kIt = 8;
    int carry = 0;
    for (int b0 = 0; b0 < 4 * F; b0 += kT * kIt) {
      const int i0 = b0 + tid * kIt;
      int v[kIt], ex[kIt];
#pragma unroll
      for (int j = 0; j < kIt; ++j) v[j] = i0 + j < 4 * F ? off[i0 + j] : 0;
      int agg;
      BS(tmp).ExclusiveSum(v, ex, agg);
#pragma unroll
      for (int j = 0; j < kIt; ++j)
        if (i0 + j < 4 * F) off[i0 + j] = carry + ex[j];
      carry += agg;
      __syncthreads();
    }
    const int Fn = carry;
    mark();
    // 3. new groups (non-empty (s,q)), their starts and keys
    int ncarry = 0;
    for (int b0 = 0; b0 < 4 * ns; b0 += kT * kIt) {
      const int x0 = b0 + tid * kIt;
      int flag[kIt], gst[kIt], ex[kIt];
#pragma unroll
      for (int j = 0; j < kIt; ++j) {
        const int x = x0 + j;
        flag[j] = 0;
        gst[j] = 0;
        if (x < 4 * ns) {
          const int s = x >> 2, q = x & 3, c0 = cs[s], m = cs[s + 1] - c0;
          const int lo = 4 * c0 + q * m, hi = lo + m;
          gst[j] = off[lo];
          const int en = hi < 4 * F ? off[hi] : Fn;
          flag[j] = en > gst[j];
        }
      }
      int agg;
      BS(tmp).ExclusiveSum(flag, ex, agg);
#pragma unroll
      for (int j = 0; j < kIt; ++j) {
        const int x = x0 + j;
        if (x < 4 * ns) {
          const int t = flag[j] ? ncarry + ex[j] : -1;
          gidx[x] = t;
          if (flag[j]) {
            csn[t] = gst[j];
            ckn[t] = (ck[x >> 2] << 2) | (uint64_t)(x & 3);
          }
        }
      }
      ncarry += agg;
      __syncthreads();
    }
    const int nsn = ncarry;
    if (tid == 0) {
      csn[nsn] = Fn;
      a.ns_out[l + 1] = nsn;
      a.f_out[l + 1] = Fn;
    }
    __syncthreads();
    mark();
    // 4. emit the child tasks (none below the block level)
    auto emit = [&](int p, int4 rA, int4 rB) {
      const int s = pc[p], c0 = cs[s], m = cs[s + 1] - c0;
      emit_task(rA, rB, 4ll * c0 + (p - c0), m, s, cmask(ck + s, l, a.L, prune, rlo, rhi), sc, sym, off, gidx,
                PA(l + 1), PB(l + 1), PC(l + 1));
    };
    for (int p = tid; p < F && l + 1 < a.L; p += kT)
      emit(p, op_children(cA, pa[p], a.trans & 1, sym), op_children(cB, pb[p], a.trans & 2, sym));
    __syncthreads();
    if (tid == 0) {
      s_F = Fn;
      s_ns = nsn;
    }
    __syncthreads();
    mark();
  }
  if (a.prof && tid == 0) a.prof[63] = np;
  if (a.host_counts && a.l_end == a.L) {  // (this kernel produced every level; one level per thread)
    __syncthreads();
    for (int l = tid; l <= a.L; l += kT) {
      a.host_counts[l] = a.ns_out[l];
      a.host_counts[a.L + 1 + l] = a.f_out[l];
    }
  }
}

// ------------------------------------------------------------ large levels (one persistent kernel)
//
// All transitions l -> l+1 for l in [l_begin, L) run in ONE cooperative launch
// (one 1024-thread CTA per SM, all resident), three phases per level separated
// by grid-wide barriers.  Work is split by groups (C nodes of level l): CTA b
// owns the groups whose first task lies in its 1/G share of the level's tasks,
// a warp walks one group's tasks at a time.
//   A count  per group and C child q: the number of child tasks T[4s+q]
//            (warp reduction over the group's tasks); CTA sums of T and of
//            the non-empty slots
//   B groups exclusive scans over the 4·ns slots (CTA prefix from the CTA
//            sums + block scans): new group index, its first task, its key;
//            the task and group counts of level l+1
//   C emit   the child tasks, slot by slot in (parent task, k) order (warp
//            scans place them), written at their group's start
// So the scans run over the 4·ns group slots, not the 4·F task slots, and a
// level costs two grid barriers (A | B C |): phase C of a CTA only reads the
// positions its own phase B computed.  The launch replaces ~8 kernel launches + 2
// device scans per level (the large levels were host-launch bound).
constexpr int kLargeThreads = 1024;
constexpr int kLargeWarps = kLargeThreads / 32;
static_assert(kLargeWarps <= 32, "the CTA sums reduce one warp's worth of warp partials");

struct LargeBfsArgs {
  int l_begin, L;
  int trans;  // bits 0-2: mode (A^T, B^T, symmetric); trans >> 8: symmetric prune levels
  double tau2;
  const int4* childA[QT_MAX_LEVELS];
  const int4* childB[QT_MAX_LEVELS];
  const double* normA[QT_MAX_LEVELS];  // squared node norms per level (screening), or null
  const double* normB[QT_MAX_LEVELS];
  int32_t* pa[QT_MAX_LEVELS];  // tasks of level l
  int32_t* pb[QT_MAX_LEVELS];
  int32_t* pc[QT_MAX_LEVELS];
  int32_t* cstart[QT_MAX_LEVELS];  // groups (C nodes) of level l: task starts (+ end)
  uint64_t* ckey[QT_MAX_LEVELS];
  int32_t* gidx[QT_MAX_LEVELS];  // transition l: (s,q) -> group of level l+1, or -1
  int32_t* slot_cnt;             // 4 * max ns: child tasks per (s,q)
  int32_t* slot_off;             // 4 * max ns: first child task of (s,q)
  int32_t* part;                 // 2 * gridDim
  int32_t* ns_out;               // groups per level
  int32_t* f_out;                // tasks per level
  unsigned* bar;                 // grid barrier: arrival count (self-resetting), generation
  unsigned long long* prof;      // QT_BFS_PROF: CTA 0's %globaltimer at each phase boundary, or null
  int32_t* host_counts;          // sync-free products: the level counts to mapped host memory, or null
  int32_t row_lo, row_hi;        // C row window (block rows)
  const uint8_t* subA;           // block size 16: quadrant masks (pair test at the block level)
  const uint8_t* subB;
  const double* n16A;            // block size 16 + screening: squared 16-block norms, or null
  const double* n16B;
};

__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
// Sense-reversing grid barrier (all CTAs are co-resident: cooperative launch).
__device__ __forceinline__ void grid_sync(unsigned* bar, unsigned& gen) {
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned g = gen;
    unsigned prev;
    asm volatile("atom.add.acq_rel.gpu.global.u32 %0, [%1], 1;" : "=r"(prev) : "l"(bar) : "memory");
    if (prev == gridDim.x - 1) {
      bar[0] = 0;
      asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(bar + 1), "r"(g + 1) : "memory");
    } else {
      while (ld_acquire(bar + 1) == g) {
      }
    }
    gen = g + 1;
  }
  __syncthreads();
}

// kMode: as k_bfs_small's (1 plain, 2 symmetric square, 3 screened, 0 generic) — the
// pair test of the count and emit phases without runtime mode branches
template <bool kExt, int kMode>
__global__ void __launch_bounds__(kLargeThreads, 1) k_bfs_large(LargeBfsArgs a) {
  constexpr bool kNoNorms = kMode == 1 || kMode == 2;
  using BS = cub::BlockScan<int, kLargeThreads>;
  __shared__ union {
    typename BS::TempStorage scan;
  } tmp;
  __shared__ int s_val[4];
  __shared__ int s_wsum[kLargeWarps][4];
  __shared__ int32_t s_g[2];
  unsigned gen = 0;
  if (threadIdx.x == 0) gen = ld_acquire(&a.bar[1]);
  const bool sym = kMode == 2 || (kMode == 0 && (a.trans & 4));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const unsigned FULL = 0xffffffffu;
  for (int l = a.l_begin; l < a.L; ++l) {
    const bool last = l == a.L - 1;
    const int mode = (a.trans & 7) | ((sym && l < (a.trans >> 8)) ? 8 : 0);
    const bool lastl = kExt && l + 1 == a.L && a.subA;
    const Screen sc{kNoNorms ? nullptr : a.normA[l + 1], kNoNorms ? nullptr : a.normB[l + 1], a.tau2, lastl ? a.subA : nullptr, lastl ? a.subB : nullptr,
                    a.trans & 3, lastl ? a.n16A : nullptr, lastl ? a.n16B : nullptr};
    const int32_t rlo = kExt ? a.row_lo : 0, rhi = kExt ? a.row_hi : INT32_MAX;
    const int32_t F = a.f_out[l], ns = a.ns_out[l];
    const int32_t* pa = a.pa[l];
    const int32_t* pb = a.pb[l];
    const int32_t* cs = a.cstart[l];
    const uint64_t* ck = a.ckey[l];
    const int4* cA = a.childA[l];
    const int4* cB = a.childB[l];
    auto pmark = [&](int k) {
      if (a.prof && blockIdx.x == 0 && threadIdx.x == 0 && l < 16) a.prof[8 * l + k] = gtimer();
    };
    pmark(0);
    // this CTA's groups: first task in [b F / G, (b+1) F / G) — the first
    // group starting at or after task p0 is the group of p0 (pc) if it starts
    // there, else the next one: two dependent loads, no search
    if (threadIdx.x < 2) {
      const int64_t p0 = (int64_t)F * (blockIdx.x + threadIdx.x) / gridDim.x;
      int32_t g = ns;
      if (p0 < F) {
        const int32_t s0 = a.pc[l][p0];
        g = cs[s0] == p0 ? s0 : s0 + 1;
      }
      s_g[threadIdx.x] = g;
    }
    __syncthreads();
    const int32_t g_lo = s_g[0], g_hi = s_g[1];
    pmark(1);
    // child counts of task p per C child q (0 for the pruned lower child of a diagonal node)
    auto counts_of = [&](int4 rA, int4 rB, int32_t sgrp, int (&c)[4]) {
      child_counts(rA, rB, c, sc, sym);
      const int cm = cmask(ck + sgrp, l, a.L, mode & 8, rlo, rhi);
#pragma unroll
      for (int q = 0; q < 4; ++q)
        if (!((cm >> q) & 1)) c[q] = 0;
    };
    auto counts = [&](int32_t p, int32_t sgrp, int (&c)[4]) {
      counts_of(op_children(cA, pa[p], mode & 1, sym), op_children(cB, pb[p], mode & 2, sym), sgrp, c);
    };
    // A. child tasks per (s,q).  A group is walked by W lanes (a power of two
    // near half the level's mean group size): random patterns have ~1-task
    // groups at the lower levels, banded ones ~17.
    int W = 1;
    {
      const int32_t half_mean = (F / max(ns, 1) + 1) / 2;
      while (W < 32 && W < half_mean) W <<= 1;
    }
    const int gpw = 32 / W;                 // groups per warp pass
    const int sub = lane / W, li = lane % W;
    {
      int vsum = 0, vflag = 0;  // this lane's sums over the groups it leads
      for (int32_t sg0 = g_lo + warp * gpw; sg0 < g_hi; sg0 += kLargeWarps * gpw) {
        const int32_t sg = sg0 + sub;
        int t[4] = {0, 0, 0, 0};
        if (sg < g_hi) {
          const int32_t c0 = cs[sg], c1 = cs[sg + 1];
          for (int32_t p = c0 + li; p < c1; p += W) {
            int c[4];
            counts(p, sg, c);
#pragma unroll
            for (int q = 0; q < 4; ++q) t[q] += c[q];
          }
        }
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          for (int d = W >> 1; d > 0; d >>= 1) t[q] += __shfl_xor_sync(FULL, t[q], d);
        }
        if (sg < g_hi && li == 0) {
          *reinterpret_cast<int4*>(a.slot_cnt + 4ll * sg) = make_int4(t[0], t[1], t[2], t[3]);
          vsum += t[0] + t[1] + t[2] + t[3];
          vflag += (t[0] > 0) + (t[1] > 0) + (t[2] > 0) + (t[3] > 0);
        }
      }
#pragma unroll
      for (int d = 16; d > 0; d >>= 1) {
        vsum += __shfl_xor_sync(FULL, vsum, d);
        vflag += __shfl_xor_sync(FULL, vflag, d);
      }
      if (lane == 0) {
        s_wsum[warp][0] = vsum;
        s_wsum[warp][1] = vflag;
      }
      __syncthreads();
      if (warp == 0) {
        int x0 = lane < kLargeWarps ? s_wsum[lane][0] : 0, x1 = lane < kLargeWarps ? s_wsum[lane][1] : 0;
#pragma unroll
        for (int d = 16; d > 0; d >>= 1) {
          x0 += __shfl_xor_sync(FULL, x0, d);
          x1 += __shfl_xor_sync(FULL, x1, d);
        }
        if (lane == 0) {
          a.part[blockIdx.x] = x0;
          a.part[gridDim.x + blockIdx.x] = x1;
        }
      }
    }
    pmark(2);
    grid_sync(a.bar, gen);
    pmark(3);
    // B. new groups: starts, keys, (s,q) -> group map
    int tpre, Fn, gpre, nsn;
    {
      int v[4] = {0, 0, 0, 0};
      for (int i = threadIdx.x; i < (int)gridDim.x; i += kLargeThreads) {
        const int x = a.part[i], y = a.part[gridDim.x + i];
        v[1] += x;
        v[3] += y;
        if (i < (int)blockIdx.x) {
          v[0] += x;
          v[2] += y;
        }
      }
      // the four CTA sums in one pass (warp shuffles, then warp 0 over the warps)
#pragma unroll
      for (int k = 0; k < 4; ++k)
#pragma unroll
        for (int d = 16; d > 0; d >>= 1) v[k] += __shfl_xor_sync(FULL, v[k], d);
      if (lane == 0)
#pragma unroll
        for (int k = 0; k < 4; ++k) s_wsum[warp][k] = v[k];
      __syncthreads();
      if (warp == 0) {
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          int x = lane < kLargeWarps ? s_wsum[lane][k] : 0;
#pragma unroll
          for (int d = 16; d > 0; d >>= 1) x += __shfl_xor_sync(FULL, x, d);
          if (lane == 0) s_val[k] = x;
        }
      }
      __syncthreads();
      tpre = s_val[0];
      Fn = s_val[1];
      gpre = s_val[2];
      nsn = s_val[3];
      __syncthreads();
    }
    int32_t* csn = a.cstart[l + 1];
    uint64_t* ckn = a.ckey[l + 1];
    int32_t* gx = a.gidx[l];
    for (int64_t b0 = 4ll * g_lo; b0 < 4ll * g_hi; b0 += kLargeThreads) {
      const int64_t x = b0 + threadIdx.x;
      const bool in = x < 4ll * g_hi;
      const int c = in ? a.slot_cnt[x] : 0;
      const int f = c > 0;
      int ex_t, agg_t, ex_f, agg_f;
      BS(tmp.scan).ExclusiveSum(c, ex_t, agg_t);
      __syncthreads();
      BS(tmp.scan).ExclusiveSum(f, ex_f, agg_f);
      if (in) {
        const int32_t start = tpre + ex_t;
        a.slot_off[x] = start;
        const int t = f ? gpre + ex_f : -1;
        gx[x] = t;
        if (f) {
          csn[t] = start;
          ckn[t] = (ck[x >> 2] << 2) | (uint64_t)(x & 3);
        }
      }
      tpre += agg_t;
      gpre += agg_f;
      __syncthreads();
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      csn[nsn] = Fn;
      a.ns_out[l + 1] = nsn;
      a.f_out[l + 1] = Fn;
    }
    pmark(4);
    if (last) break;
    // (no grid barrier here: phase C of this CTA reads only what its own
    // phase B wrote — the positions and group ids of its own slots — and the
    // level-l tasks; the barrier after C orders it before the next level's A)
    __syncthreads();
    pmark(5);
    // C. emit the child tasks of level l+1: slot (s,q) lists, for every parent
    // task in order, k = 0 then k = 1 (ascending global k inside the group)
    {
      int32_t* pa2 = a.pa[l + 1];
      int32_t* pb2 = a.pb[l + 1];
      int32_t* pc2 = a.pc[l + 1];
      for (int32_t sg0 = g_lo + warp * gpw; sg0 < g_hi; sg0 += kLargeWarps * gpw) {
        const int32_t sg = sg0 + sub;
        const bool live = sg < g_hi;
        int32_t c0 = 0, c1 = 0;
        int cm = 0xF;
        int pos[4] = {0, 0, 0, 0}, gq[4] = {-1, -1, -1, -1};
        if (live) {
          c0 = cs[sg];
          c1 = cs[sg + 1];
          cm = cmask(ck + sg, l, a.L, mode & 8, rlo, rhi);
          const int4 o4 = *reinterpret_cast<const int4*>(a.slot_off + 4ll * sg);
          const int4 g4 = *reinterpret_cast<const int4*>(gx + 4ll * sg);
          pos[0] = o4.x; pos[1] = o4.y; pos[2] = o4.z; pos[3] = o4.w;
          gq[0] = g4.x; gq[1] = g4.y; gq[2] = g4.z; gq[3] = g4.w;
        }
        // uniform trip count across the warp (the scans below shuffle)
        int iters = (c1 - c0 + W - 1) / W;
#pragma unroll
        for (int d = 16; d > 0; d >>= 1) iters = max(iters, __shfl_xor_sync(FULL, iters, d));
        for (int it = 0; it < iters; ++it) {
          const int32_t p = c0 + it * W + li;
          int4 A4 = make_int4(-1, -1, -1, -1), B4 = A4;
          if (p < c1) {
            A4 = op_children(cA, pa[p], mode & 1, sym);
            B4 = op_children(cB, pb[p], mode & 2, sym);
          }
          const int av[4] = {A4.x, A4.y, A4.z, A4.w};
          const int bv[4] = {B4.x, B4.y, B4.z, B4.w};
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const int i = q >> 1, j = q & 1;
            const bool on = (cm >> q) & 1;
            const bool k0 = on && pair_ok(av[2 * i], bv[j], sc, sym);
            const bool k1 = on && pair_ok(av[2 * i + 1], bv[2 + j], sc, sym);
            const int n = (int)k0 + (int)k1;
            int ex = n;
            for (int d = 1; d < W; d <<= 1) {
              const int y = __shfl_up_sync(FULL, ex, d, W);
              if (li >= d) ex += y;
            }
            const int tot = __shfl_sync(FULL, ex, W - 1, W);
            ex -= n;
            int w = pos[q] + ex;
            if (k0) {
              pa2[w] = av[2 * i];
              pb2[w] = bv[j];
              pc2[w] = gq[q];
              ++w;
            }
            if (k1) {
              pa2[w] = av[2 * i + 1];
              pb2[w] = bv[2 + j];
              pc2[w] = gq[q];
            }
            pos[q] += tot;
          }
        }
      }
    }
    pmark(6);
    grid_sync(a.bar, gen);
    pmark(7);
  }
  // (CTA 0 wrote the counts of this kernel's levels; the small kernel the others)
  if (a.host_counts && blockIdx.x == 0) {  // (one level per thread)
    __syncthreads();
    for (int l = threadIdx.x; l <= a.L; l += blockDim.x) {
      a.host_counts[l] = a.ns_out[l];
      a.host_counts[a.L + 1 + l] = a.f_out[l];
    }
  }
}

// the single-CTA BFS instantiation for (row-window/bs-16 extensions, tiny
// shared-memory frontiers, kMode)
const void* small_fn(bool ext, bool tiny, int mode) {
#define QT_SMALL(e, t)                                                                        \
  (mode == 0   ? (const void*)k_bfs_small<e, t, 0>                                            \
   : mode == 1 ? (const void*)k_bfs_small<e, t, 1>                                            \
   : mode == 2 ? (const void*)k_bfs_small<e, t, 2>                                            \
               : (const void*)k_bfs_small<e, t, 3>)
  return ext ? (tiny ? QT_SMALL(true, true) : QT_SMALL(true, false))
             : (tiny ? QT_SMALL(false, true) : QT_SMALL(false, false));
#undef QT_SMALL
}

// CTAs of the cooperative BFS launch: every CTA resident (occupancy x SMs)
int large_bfs_grid(qt_ctx ctx) {
  static int per_sm = -1;
  if (per_sm < 0) {
    int n = 1 << 30;
    for (const void* f : {(const void*)k_bfs_large<false, 0>, (const void*)k_bfs_large<true, 0>,
                          (const void*)k_bfs_large<false, 1>, (const void*)k_bfs_large<true, 1>,
                          (const void*)k_bfs_large<false, 2>, (const void*)k_bfs_large<true, 2>,
                          (const void*)k_bfs_large<false, 3>, (const void*)k_bfs_large<true, 3>}) {
      int m = 0;
      QT_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&m, f, kLargeThreads, 0));
      n = std::min(n, m);
    }
    if (n < 1) fail(QT_ECUDA, "k_bfs_large cannot be resident");
    per_sm = 1;
  }
  return per_sm * ctx->num_sms;
}


// Largest transient C pool (bytes) the sync-free mode may allocate by its upper bound.
size_t syncfree_cap() {
  static size_t cap = [] {
    const char* e = getenv("QT_SYNCFREE_MB");
    return (size_t)(e ? atoll(e) : 1024) << 20;
  }();
  return cap;
}

}  // namespace

// Optional host-side phase trace (QT_TRACE=1): wall-clock marks to stderr.
struct Trace {
  bool on;
  std::chrono::steady_clock::time_point t0;
  std::string buf;
  Trace() : on(getenv("QT_TRACE") != nullptr), t0(std::chrono::steady_clock::now()) {}
  void mark(const char* what) {
    if (!on) return;
    double us = std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - t0).count();
    char b[128];
    snprintf(b, sizeof b, " %s@%.0f", what, us);
    buf += b;
  }
  ~Trace() {
    mark("exit");
    if (on) fprintf(stderr, "[qt trace] multiply:%s\n", buf.c_str());
  }
};

// Task counts per level from the host copies of the occupancy histograms (no
// device work, no sync): exact for regular products, an upper bound for the
// symmetric square (its actual counts come from the BFS).
std::vector<int64_t> level_task_bounds(qt_mat A, qt_mat B, int trans) {
  const int L = A->L;
  const bool sym = trans & 4;
  std::vector<int64_t> F(L + 1, 0);
  if (A->nb == 0 || B->nb == 0) return F;
  const int64_t H = 2ll << L;
  const int32_t* hA = A->hist_host.data();
  const int32_t* hB = B->hist_host.data();
  for (int l = 0; l <= L; ++l) {
    const int64_t base = (1ll << l) - 1, m = 1ll << l;
    int64_t f = 0;
    for (int64_t K = 0; K < m; ++K) {
      if (sym) {
        const int64_t c = (int64_t)hA[base + K] + hA[H + base + K];
        f += c * c;
      } else {
        // cols(op(A)_l) . rows(op(B)_l); a transposed operand swaps its row/column histograms
        f += (int64_t)hA[((trans & 1) ? 0 : H) + base + K] * (int64_t)hB[((trans & 2) ? H : 0) + base + K];
      }
    }
    F[l] = f;
  }
  return F;
}

qt_mat multiply_local(qt_mat A, qt_mat B, qt_stats* stp, float* ms_sym, float* ms_num, int trans,
                      double tau, Overlap* ov, int32_t row_lo, int32_t row_hi, NumericPlan* plan,
                      bool out_f32) {
  const bool screen = tau >= 0.0;
  const double tau2 = tau * tau;
  if (screen) {
    ensure_norms(A);
    ensure_norms(B);
  }
  // trans: bit 0 A^T, bit 1 B^T, bit 2 symmetric square (A = B = U, C upper)
  const bool sym = trans & 4;
  Trace tr;
  qt_ctx ctx = A->ctx;
  cudaStream_t st = ctx->stream;
  const int L = A->L;
  qt_mat C = new qt_mat_s();
  C->ctx = ctx;
  C->n = A->n;
  C->leaf_dim = A->leaf_dim;
  C->bs = A->bs;
  C->dtype = out_f32 ? QT_F32 : A->dtype;
  if (out_f32 && (A->dtype != QT_F64 || (trans & 4) || ov || plan))
    fail(QT_EINVAL, "FP32 output of the FP64 kernel: plain FP64 operands only");
  C->L = L;
  C->leaf_level = A->leaf_level;
  C->nbr = A->nbr;
  C->row_lo = A->row_lo;
  C->row_hi = A->row_hi;
  C->bounds = A->bounds;
  C->ubs = A->ubs;
  // C's quadtree levels are (re)built from its block keys on first use
  // (ensure_levels): a task group whose child products are all NIL is a NIL
  // node of C (the recursion of §3.2 returns NIL for it), so the canonical
  // tree is the one spanned by the C blocks.
  C->levels_built = false;
  qt_stats& S = *stp;
  S.nlevels = L + 1;
  S.leaf_level = A->leaf_level;
  try {
    // (the timing events are skipped by qt_multiply_async and with the
    // context's timing off: ms_* are 0 then)
    const bool timed = !ctx->async_multiply && ctx->timing;
    if (timed) QT_CUDA(cudaEventRecord(ctx->ev[2], st));
    std::vector<int64_t> F = level_task_bounds(A, B, trans);
    if (A->nb > 0 && B->nb > 0) {
      tr.mark("counts");
      for (int l = 0; l <= L; ++l)
        if (F[l] >= (1ll << 31) / 4) fail(QT_EINVAL, "level %d has %lld tasks (> 2^29)", l, (long long)F[l]);
    }
    for (int l = 0; l <= L; ++l) S.level_tasks[l] = F[l];
    S.block_products = F[L];
    if (F[L] == 0) {
      // no block product at all: C is the NIL matrix
      C->nb = 0;
      if (timed) {
        QT_CUDA(cudaEventRecord(ctx->ev[3], st));
        QT_CUDA(cudaEventRecord(ctx->ev[4], st));
      }
    } else {
      // upper bounds of the group counts: ns_{l+1} <= min(4 ns_l, F_{l+1})
      std::vector<int64_t> nsb(L + 1, 1);
      for (int l = 0; l < L; ++l) nsb[l + 1] = std::min<int64_t>(4 * nsb[l], F[l + 1]);
      // Sync-free mode (small problems, where a host round trip between the
      // BFS and the numeric kernel is a large share of the call): C's pool is
      // sized by the upper bound nsb[L] (transient over-allocation <=
      // QT_SYNCFREE_MB, default 1024 MiB), the numeric kernel reads the tile
      // count from the device, and the last BFS kernel writes the level counts
      // straight into mapped host memory — the context's staging area (read
      // after the call's one final sync) or, for qt_multiply_async, a ring
      // slot read when C is first used (resolve).
      const size_t cbound = (size_t)nsb[L] * 1024 * elem_size(C->dtype);
      const bool syncfree =
          A->ubs != 16 && !ov && !plan && !B->pool2 && cbound <= syncfree_cap();
      int32_t* h_counts = static_cast<int32_t*>(ctx->pinned);  // [ns(L+1) | F(L+1)]
      int pend_slot = -1;
      int32_t* host_counts = nullptr;
      if (syncfree && ctx->async_multiply) {
        pend_slot = ctx->pend_next;
        ctx->pend_next = (pend_slot + 1) % qt_ctx_s::kPendRing;
        if (ctx->pend_owner[pend_slot]) resolve(ctx->pend_owner[pend_slot]);  // (ring full: the oldest first)
        host_counts = ctx->pend_host + 128 * pend_slot;
      } else {
        // (blocking sync-free product: read after the call's final sync;
        // otherwise right after the BFS — written by the last BFS kernel into
        // mapped memory either way, not by a copy that could queue behind a
        // bulk read-back on the copy engine)
        host_counts = h_counts;
      }
      DevBuf cnt_dev(8 * (L + 1), st);  // [ns(L+1) | F(L+1)]: one D2H copy
      int32_t* nsd = cnt_dev.as<int32_t>();
      int32_t* fd = nsd + (L + 1);
      // --- small levels in one CTA
      const bool f32 = A->dtype == QT_F32;  // the FP32 (tcgen05) kernel
      int l_end = 0;
      // (block size 16: the container level's mask tests make the single-CTA
      // kernel slower per task — 4096 measured best for it, 8192 for bs 32)
      static const int64_t small_env = getenv("QT_SMALL_MAXF") ? atoll(getenv("QT_SMALL_MAXF")) : 0;
      const int64_t small_max = small_env > 0 ? small_env : (A->ubs == 16 ? kSmallMaxF / 2 : kSmallMaxF);
      while (l_end < L - 1 && F[l_end + 1] <= small_max) ++l_end;
      // every level small (FP64): the single-CTA kernel also runs the last
      // transition and no cooperative launch is needed
      if (!f32 && l_end == L - 1 && F[L - 1] <= small_max) l_end = L;
      if (f32) l_end = std::min(l_end, L - 2);  // the FP32 tiles need the level L-2 queue
      int64_t maxF = 1, maxNS = 1, maxF4 = 1;
      for (int l = 0; l <= l_end; ++l) {
        maxF = std::max(maxF, F[l]);
        maxNS = std::max(maxNS, nsb[l]);
        if (l < l_end) maxF4 = std::max(maxF4, 4 * F[l]);
      }
      DevBuf sp[2], sb[2], sc[2], scs[2], sck[2];
      SmallBfsArgs sa;
      sa.l_end = l_end;
      sa.L = L;
      sa.trans = trans;
      sa.tau2 = tau2;
      sa.row_lo = row_lo;
      sa.row_hi = row_hi;
      // (bs 16: container pairs whose quadrant masks never meet are pruned)
      sa.subA = A->ubs == 16 ? A->sub.as<uint8_t>() : nullptr;
      sa.subB = A->ubs == 16 ? B->sub.as<uint8_t>() : nullptr;
      sa.n16A = A->ubs == 16 && screen ? A->norm16.as<double>() : nullptr;
      sa.n16B = A->ubs == 16 && screen ? B->norm16.as<double>() : nullptr;
      for (int l = 0; l <= L && l < QT_MAX_LEVELS; ++l) {
        sa.normA[l] = screen ? A->norm2[l].as<double>() : nullptr;
        sa.normB[l] = screen ? B->norm2[l].as<double>() : nullptr;
      }
      for (int l = 0; l < L; ++l) {
        sa.childA[l] = A->child[l].as<int4>();
        sa.childB[l] = B->child[l].as<int4>();
        sa.nodesA[l] = (int32_t)std::min<int64_t>(A->cnt[l], INT32_MAX);
        sa.nodesB[l] = (int32_t)std::min<int64_t>(B->cnt[l], INT32_MAX);
      }
      for (int b = 0; b < 2; ++b) {
        sp[b].alloc(4 * maxF, st);
        sb[b].alloc(4 * maxF, st);
        sc[b].alloc(4 * maxF, st);
        scs[b].alloc(4 * (maxNS + 1), st);
        sck[b].alloc(8 * maxNS, st);
        sa.pa[b] = sp[b].as<int32_t>();
        sa.pb[b] = sb[b].as<int32_t>();
        sa.pc[b] = sc[b].as<int32_t>();
        sa.cstart[b] = scs[b].as<int32_t>();
        sa.ckey[b] = sck[b].as<uint64_t>();
      }
      DevBuf soff(4 * maxF4, st), sg(16 * maxNS, st);
      sa.off = soff.as<int32_t>();
      sa.gidx = sg.as<int32_t>();
      sa.ns_out = nsd;
      sa.f_out = fd;
      sa.zero = ctx->counters.as<int>() + 16;  // the numeric kernels' scheduler counters (16, 17)
      sa.host_counts = host_counts;
      tr.mark("small_alloc");
      const bool ext = sa.subA || row_lo > 0 || row_hi < INT32_MAX;
      // dense start: plain and transposed products without screening (the
      // other modes prune by rules the dense maps do not carry)
      static const int dense_env = getenv("QT_DENSE_START") ? atoi(getenv("QT_DENSE_START")) : 4;
      // (block size 16: the quadrant-mask test applies only to the block-level
      // pairs, below any level the dense start produces; a row window does not)
      const bool plain = !sym && !screen;
      const int mode = screen ? (sym ? 0 : 3) : (sym ? 2 : 1);  // the BFS kernels' kMode
      const bool window = row_lo > 0 || row_hi < INT32_MAX;
      sa.l0 = (plain && !window && A->dmap.p && B->dmap.p)
                  ? std::min(std::min(std::min(dense_env, qt_mat_s::kDenseLevels), l_end), L - 1)
                  : 0;
      if (sa.l0 < 2) sa.l0 = 0;
      sa.dmapA = A->dmap.as<int32_t>();
      sa.dmapB = B->dmap.as<int32_t>();
      static const bool bfs_prof = getenv("QT_BFS_PROF") != nullptr;
      DevBuf profbuf;
      sa.prof = nullptr;
      if (bfs_prof) {
        profbuf.alloc(64 * 8, st);
        QT_CUDA(cudaMemsetAsync(profbuf.p, 0, 64 * 8, st));
        sa.prof = profbuf.as<unsigned long long>();
      }
      // the intermediate small levels in shared memory when every one fits
      bool tiny = true;
      int64_t tiny_max = 1;
      for (int l = 0; l < l_end; ++l) {
        tiny = tiny && F[l] <= kTinyF;
        tiny_max = std::max(tiny_max, F[l]);
      }
      sa.tiny_cap = (int)((tiny_max + 127) / 128 * 128);
      if (tiny) {
        static std::atomic<unsigned long long> attr_set{0};  // per device (bit d)
        const unsigned long long bit = 1ull << (ctx->device & 63);
        if (!(attr_set.load(std::memory_order_acquire) & bit)) {
          for (const void* f : {small_fn(false, true, 0), small_fn(false, true, 1), small_fn(false, true, 2),
                                small_fn(false, true, 3), small_fn(true, true, 0), small_fn(true, true, 1),
                                small_fn(true, true, 2), small_fn(true, true, 3)})
            QT_CUDA(cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)tiny_smem(kTinyF)));
          attr_set.fetch_or(bit, std::memory_order_release);
        }
        // dense start straight into the next kernel's level: staged (when it fits)
        size_t smem = tiny_smem(sa.tiny_cap);
        sa.stage_cap = 0;
        if (sa.l0 > 0 && sa.l0 == l_end && smem + 12 * (size_t)F[l_end] <= tiny_smem(kTinyF)) {
          sa.stage_cap = (int)F[l_end];
          smem += 12 * (size_t)F[l_end];
        }
        void* kargs[] = {&sa};
        QT_CUDA(cudaLaunchKernel(small_fn(ext, true, mode), dim3(1), dim3(256), kargs, smem, st));
      } else {
        void* kargs[] = {&sa};
        QT_CUDA(cudaLaunchKernel(small_fn(ext, false, mode), dim3(1), dim3(kSmallThreads), kargs, 0, st));
      }
      QT_LAUNCH_CHECK(ctx);
      if (bfs_prof) {
        unsigned long long h[64];
        QT_CUDA(cudaMemcpyAsync(h, profbuf.p, 64 * 8, cudaMemcpyDeviceToHost, st));
        QT_CUDA(cudaStreamSynchronize(st));
        fprintf(stderr, "[qt bfs_small] l_end=%d tiny=%d F:", l_end, (int)tiny);
        for (int l = 0; l <= l_end; ++l) fprintf(stderr, " %lld", (long long)F[l]);
        fprintf(stderr, " marks(ns):");
        for (int i = 1; i < (int)h[63] && i < 40; ++i) fprintf(stderr, " %llu", h[i] - h[i - 1]);
        fprintf(stderr, "\n");
      }
      const bool all_small = l_end == L;
      const int cb = (all_small ? L - 1 : l_end) & 1;
      DevBuf pa = std::move(sp[cb]), pb = std::move(sb[cb]), pc = std::move(sc[cb]);
      DevBuf cstart = std::move(scs[cb]), ckey = std::move(sck[cb]);
      // --- large levels: one persistent cooperative kernel, no host sync
      DevBuf cchild, t2_pa, t2_pb, t2_cstart, cchild2;
      tr.mark("small_launch");
      if (all_small) {
        // level L-1's queue and C's blocks (level L groups) came from the small kernel
        C->key = std::move(sck[L & 1]);
        cchild = std::move(sg);
      } else {
        // level l_end lives in the small kernel's buffers; levels l_end+1..L
        // alternate between two buffer sets (level L: groups only)
        int64_t mF = 1, mNS = 1, mNSg = 1;
        for (int l = l_end + 1; l < L; ++l) mF = std::max(mF, F[l]);
        for (int l = l_end + 1; l < L; ++l) mNS = std::max(mNS, nsb[l]);
        for (int l = l_end; l < L; ++l) mNSg = std::max(mNSg, 4 * nsb[l]);
        DevBuf qa[2], qb[2], qc[2], qcs[2], qck[2], qgx[2];
        for (int b = 0; b < 2; ++b) {
          if (l_end + 1 < L) {
            qa[b].alloc(4 * mF, st);
            qb[b].alloc(4 * mF, st);
            qc[b].alloc(4 * mF, st);
          }
          qcs[b].alloc(4 * (mNS + 1), st);
          qck[b].alloc(8 * mNS, st);
          qgx[b].alloc(4 * mNSg, st);
        }
        // level L (C's blocks): its own buffers — the ping-pong set of level L
        // is level L-2's, whose queue the FP32 kernel still needs
        DevBuf ckeyL(8 * std::max<int64_t>(nsb[L], 1), st), csL(4 * (nsb[L] + 1), st);
        DevBuf slot_cnt(4 * mNSg, st), slot_off(4 * mNSg, st);
        const int G = large_bfs_grid(ctx);
        DevBuf part(4 * 2 * G, st);
        LargeBfsArgs la;
        la.l_begin = l_end;
        la.L = L;
        la.trans = trans;
        la.tau2 = tau2;
        la.row_lo = row_lo;
        la.row_hi = row_hi;
        la.subA = sa.subA;
        la.subB = sa.subB;
        la.n16A = sa.n16A;
        la.n16B = sa.n16B;
        for (int l = 0; l < L && l < QT_MAX_LEVELS; ++l) {
          la.childA[l] = A->child[l].as<int4>();
          la.childB[l] = B->child[l].as<int4>();
        }
        for (int l = 0; l <= L && l < QT_MAX_LEVELS; ++l) {
          la.normA[l] = screen ? A->norm2[l].as<double>() : nullptr;
          la.normB[l] = screen ? B->norm2[l].as<double>() : nullptr;
        }
        auto set = [&](int l) { return (l - l_end) & 1; };
        for (int l = l_end; l <= L; ++l) {
          if (l == l_end) {
            la.pa[l] = pa.as<int32_t>();
            la.pb[l] = pb.as<int32_t>();
            la.pc[l] = pc.as<int32_t>();
            la.cstart[l] = cstart.as<int32_t>();
            la.ckey[l] = ckey.as<uint64_t>();
          } else {
            if (l < L) {
              la.pa[l] = qa[set(l)].as<int32_t>();
              la.pb[l] = qb[set(l)].as<int32_t>();
              la.pc[l] = qc[set(l)].as<int32_t>();
            }
            la.cstart[l] = l == L ? csL.as<int32_t>() : qcs[set(l)].as<int32_t>();
            la.ckey[l] = l == L ? ckeyL.as<uint64_t>() : qck[set(l)].as<uint64_t>();
          }
          if (l < L) la.gidx[l] = qgx[set(l)].as<int32_t>();
        }
        la.slot_cnt = slot_cnt.as<int32_t>();
        la.slot_off = slot_off.as<int32_t>();
        la.part = part.as<int32_t>();
        la.ns_out = nsd;
        la.f_out = fd;
        la.bar = reinterpret_cast<unsigned*>(ctx->counters.as<int>() + 40);
        la.host_counts = host_counts;
        DevBuf lprof;
        la.prof = nullptr;
        if (bfs_prof) {
          lprof.alloc(8 * 128, st);
          QT_CUDA(cudaMemsetAsync(lprof.p, 0, 8 * 128, st));
          la.prof = lprof.as<unsigned long long>();
        }
        void* kargs[] = {&la};
        const void* kfn = mode == 0   ? (ext ? (const void*)k_bfs_large<true, 0> : (const void*)k_bfs_large<false, 0>)
                          : mode == 1 ? (ext ? (const void*)k_bfs_large<true, 1> : (const void*)k_bfs_large<false, 1>)
                          : mode == 2 ? (ext ? (const void*)k_bfs_large<true, 2> : (const void*)k_bfs_large<false, 2>)
                                      : (ext ? (const void*)k_bfs_large<true, 3> : (const void*)k_bfs_large<false, 3>);
        QT_CUDA(cudaLaunchCooperativeKernel(kfn,
                                            dim3(G), dim3(kLargeThreads), kargs, 0,
                                            st));
        ctx->launches += 1;
        QT_LAUNCH_CHECK(ctx);
        if (bfs_prof) {
          unsigned long long h[128];
          QT_CUDA(cudaMemcpyAsync(h, lprof.p, 8 * 128, cudaMemcpyDeviceToHost, st));
          QT_CUDA(cudaStreamSynchronize(st));
          fprintf(stderr, "[qt bfs_large] per level (F): lbound A sync B sync C sync (ns)\n");
          for (int l = l_end; l < L && l < 16; ++l) {
            const unsigned long long* m = h + 8 * l;
            fprintf(stderr, "  l=%d (%lld):", l, (long long)F[l]);
            for (int k = 1; k < 8; ++k)
              if (m[k] && m[k - 1]) fprintf(stderr, " %llu", m[k] - m[k - 1]);
            if (l + 1 < L && h[8 * (l + 1)] && m[7]) fprintf(stderr, " | next %llu", h[8 * (l + 1)] - m[7]);
            fprintf(stderr, "\n");
          }
        }
        // hand the queues the numeric kernels consume over
        C->key = std::move(ckeyL);
        cchild = std::move(qgx[set(L - 1)]);
        if (f32) {  // the level L-2 queue: the FP32 work items (l_end <= L-2)
          cchild2 = std::move(qgx[set(L - 2)]);
          if (L - 2 > l_end) {
            t2_pa = std::move(qa[set(L - 2)]);
            t2_pb = std::move(qb[set(L - 2)]);
            t2_cstart = std::move(qcs[set(L - 2)]);
          } else {  // level l_end: the small kernel's buffers
            t2_pa = std::move(pa);
            t2_pb = std::move(pb);
            t2_cstart = std::move(cstart);
          }
        }
        if (L - 1 > l_end) {
          pa = std::move(qa[set(L - 1)]);
          pb = std::move(qb[set(L - 1)]);
          cstart = std::move(qcs[set(L - 1)]);
        }
      }
      // --- group counts of every level: C's block count (sync-free mode: above)
      tr.mark("levels_launched");
      std::vector<int32_t> ns(L + 1, 0), Fa(L + 1, 0);
      if (syncfree) {
        for (int l = 0; l <= L; ++l) ns[l] = (int32_t)nsb[l];  // upper bounds until the final sync
        C->nb = nsb[L];
        C->pool.alloc(cbound, st);
        tr.mark("c_alloc_bound");
      } else {
        QT_CUDA(cudaStreamSynchronize(st));  // (the BFS wrote h_counts)
        for (int l = 0; l <= L; ++l) {
          ns[l] = h_counts[l];
          Fa[l] = h_counts[L + 1 + l];
        }
        tr.mark("levels_done");
        for (int l = 0; l <= L; ++l) {
          S.level_c_nodes[l] = ns[l];
          S.level_tasks[l] = Fa[l];  // actual counts (== F for regular products)
          F[l] = Fa[l];
        }
        S.block_products = Fa[L];
        C->nb = ns[L];
        C->pool.alloc((size_t)C->nb * 1024 * elem_size(C->dtype), st);
        tr.mark("c_alloc");
      }
      // tiles per scheduler grab (FP64): ~32 tasks per grab, at most 16 tiles
      int group = 1;
      {
        const int64_t per_tile = std::max<int64_t>(1, F[L - 1] / std::max<int32_t>(1, ns[L - 1]));
        // (tiles with >= 8 tasks stream well one at a time: grouping only costs balance)
        int64_t g = per_tile >= 8 ? 1 : std::min<int64_t>(16, 32 / per_tile);
        // keep >= 8 grabs per tile stream (2 per CTA, one CTA per SM)
        g = std::min<int64_t>(g, ns[L - 1] / (16ll * ctx->num_sms));
        group = (int)std::max<int64_t>(1, g);
        if (tr.on) {
          char b[64];
          snprintf(b, sizeof b, "group=%d", group);
          tr.mark(b);
        }
      }
      // multi-rank overlap: the tiles that read only local B blocks run while
      // the payload is in flight, the rest behind it on ov->s2.  Partitioned
      // on the device (no host sync); FP64 only with one tile per grab (the
      // grouped grabs of sparse patterns need contiguous task ranges).
      const bool two_phase = ov && ov->s2 && B->pool2 && B->split < B->nb && C->nb > 0 && (f32 || group == 1);
      DevBuf tmap, tnsel;
      int64_t n_all = 0;
      if (two_phase) {
        n_all = f32 ? ns[L - 2] : ns[L - 1];
        tmap.alloc(4 * n_all, st);
        tnsel.alloc(4, st);
        if (f32)
          split_tiles(ctx, n_all, t2_cstart.as<int32_t>(), t2_pb.as<int32_t>(), B->child[L - 2].as<int4>(),
                      B->child[L - 1].as<int4>(), B->split, tmap.as<int32_t>(), tnsel.as<int32_t>());
        else
          split_tiles(ctx, n_all, cstart.as<int32_t>(), pb.as<int32_t>(), B->child[L - 1].as<int4>(), nullptr,
                      B->split, tmap.as<int32_t>(), tnsel.as<int32_t>());
        tr.mark("tile_split");
      }
      if (timed) QT_CUDA(cudaEventRecord(ctx->ev[3], st));
      NumericArgs na;
      na.ntiles = ns[L - 1];
      na.tile_start = cstart.as<int32_t>();
      na.pa = pa.as<int32_t>();
      na.pb = pb.as<int32_t>();
      na.childA = A->child[L - 1].as<int4>();
      na.childB = B->child[L - 1].as<int4>();
      na.childC = cchild.as<int4>();
      na.poolA = A->pool_ptr();
      na.poolB = B->pool_ptr();
      na.poolB2 = B->pool2;
      na.splitB = B->split;
      na.poolC = C->pool.p;
      na.counter = ctx->counters.as<int>() + 16;
      na.trans = trans & 7;  // bit 2: symmetric square (block refs carry transpose bits)
      // (block size 16: the 16-block test replaces the container norms, below)
      na.normA = screen && A->ubs != 16 ? A->norm2[L].as<double>() : nullptr;
      na.normB = screen && A->ubs != 16 ? B->norm2[L].as<double>() : nullptr;
      na.tau2 = tau2;
      if (A->ubs == 16 && !f32) {  // block size 16: only the 16-block products that exist (and pass the screen)
        na.subA = A->sub.as<uint8_t>();
        na.subB = B->sub.as<uint8_t>();
        if (screen) {
          na.norm16A = A->norm16.as<double>();
          na.norm16B = B->norm16.as<double>();
        }
      }
      na.group = group;
      na.counter_ready = true;  // zeroed by the small BFS kernel
      na.out_f32 = out_f32;
      if (syncfree) na.ntiles_dev = nsd + (L - 1);  // the actual tile count (na.ntiles: its bound)
      // symmetric square: blocks of U read transposed come from U^T's copy —
      // kept with U (handles are immutable) except for plans, whose execute
      // refreshes its own copy from U's current values
      DevBuf poolT;
      const void* poolTp = nullptr;
      if (C->nb > 0 && sym) {
        const size_t tb = (size_t)A->nb * 1024 * elem_size(C->dtype);
        auto transpose_into = [&](void* dst) {
          if (f32)
            launch_transpose_blocks_f32(ctx, A->pool_ptr(), dst, A->nb);
          else
            launch_transpose_blocks(ctx, A->pool_ptr(), dst, A->nb);
        };
        if (plan) {
          poolT.alloc(tb, st);
          transpose_into(poolT.p);
          poolTp = poolT.p;
        } else {
          if (!A->poolT_cache.p || A->poolT_src != A->pool_ptr()) {
            A->poolT_cache.alloc(tb, st);
            transpose_into(A->poolT_cache.p);
            A->poolT_src = A->pool_ptr();
          }
          poolTp = A->poolT_cache.p;
        }
        na.poolT = poolTp;
      }
      // phase launches: the local-only tiles on the ctx stream now, the rest
      // on ov->s2 behind the payload; the ctx stream joins s2 afterwards.
      // Phase 2's CTAs take over the SMs as phase 1's finish.
      auto phases = [&](auto args, auto launch) {
        args.tile_map = tmap.as<int32_t>();
        args.nsel = tnsel.as<int32_t>();
        QT_CUDA(cudaEventRecord(ctx->ov_ev[0], st));
        auto a1 = args;
        a1.phase = 1;
        launch(a1);
        QT_CUDA(cudaStreamWaitEvent(ov->s2, ctx->ov_ev[0], 0));
        auto a2 = args;
        a2.phase = 2;
        a2.counter = ctx->counters.as<int>() + 17;
        a2.stream = ov->s2;
        launch(a2);
        QT_CUDA(cudaEventRecord(ctx->ov_ev[1], ov->s2));
        QT_CUDA(cudaStreamWaitEvent(st, ctx->ov_ev[1], 0));
      };
      if (C->nb > 0 && !f32) {
        if (two_phase)
          phases(na, [&](const NumericArgs& x) { launch_numeric(ctx, A->dtype, x); });
        else
          launch_numeric(ctx, A->dtype, na);
      }
      if (C->nb > 0 && f32) {
        NumericArgs32 nb;
        nb.ntiles = ns[L - 2];
        nb.tile_start = t2_cstart.as<int32_t>();
        nb.pa = t2_pa.as<int32_t>();
        nb.pb = t2_pb.as<int32_t>();
        nb.childA2 = A->child[L - 2].as<int4>();
        nb.childA1 = A->child[L - 1].as<int4>();
        nb.childB2 = B->child[L - 2].as<int4>();
        nb.childB1 = B->child[L - 1].as<int4>();
        nb.childC2 = cchild2.as<int4>();
        nb.childC1 = cchild.as<int4>();
        nb.poolA = A->pool_ptr();
        nb.poolB = B->pool_ptr();
        nb.poolB2 = B->pool2;
        nb.splitB = B->split;
        nb.poolC = C->pool.p;
        nb.zeros = ctx->zeros.p;
        nb.counter = ctx->counters.as<int>() + 16;
        nb.counter_ready = true;
        if (syncfree) nb.ntiles_dev = nsd + (L - 2);  // the actual tile count (nb.ntiles: its bound)
        nb.trans = trans & 7;
        nb.poolT = poolTp;
        if (two_phase)
          phases(nb, [&](const NumericArgs32& x) { launch_numeric_f32(ctx, x); });
        else
          launch_numeric_f32(ctx, nb);
      }
      if (pend_slot >= 0) QT_CUDA(cudaEventRecord(ctx->pend_ev[pend_slot], st));  // (C's counts are in its ring slot)
      if (timed) QT_CUDA(cudaEventRecord(ctx->ev[4], st));
      tr.mark("numeric_launched");
      // (the frontier buffers go back to this stream's cache: stream-ordered reuse)
      if (timed)
        QT_CUDA(cudaEventSynchronize(ctx->ev[4]));
      else if (!ctx->async_multiply)
        QT_CUDA(cudaStreamSynchronize(st));
      tr.mark("numeric_done");
      if (pend_slot >= 0) {
        // (stats: the task counts are exact for regular products; C's block
        // and group counts are unknown until C is resolved)
        C->pend_slot = pend_slot;
        ctx->pend_owner[pend_slot] = C;
        for (int l = 0; l <= L; ++l) S.level_c_nodes[l] = 0;
      } else if (syncfree) {
        for (int l = 0; l <= L; ++l) {
          ns[l] = h_counts[l];
          Fa[l] = h_counts[L + 1 + l];
          S.level_c_nodes[l] = ns[l];
          S.level_tasks[l] = Fa[l];
          F[l] = Fa[l];
        }
        S.block_products = Fa[L];
        C->nb = ns[L];  // (the pool keeps its bound-sized allocation)
      }
      if (two_phase && !ctx->async_multiply) {
        int32_t h = 0;
        QT_CUDA(cudaMemcpyAsync(&h, tnsel.p, 4, cudaMemcpyDeviceToHost, st));
        QT_CUDA(cudaStreamSynchronize(st));
        ov->tiles_local = h;
        ov->tiles_remote = n_all - h;
      }
      void* const plan_pool_c = C->pool.p;  // (a bs-16 drop of empty containers would move C: no plan then)
      if (A->ubs == 16) {  // the 16-block pattern of C and the 16-block products (qt_bs16.cu)
        C->sub.alloc(std::max<int64_t>(C->nb, 1), st);
        int64_t r16[4];
        cmask16(ctx, ns[L - 1], cstart.as<int32_t>(), pa.as<int32_t>(), pb.as<int32_t>(), A->child[L - 1].as<int4>(),
                B->child[L - 1].as<int4>(), cchild.as<int4>(), A->sub.as<uint8_t>(), B->sub.as<uint8_t>(), trans & 7,
                C->key.as<uint64_t>(), C->sub.as<uint8_t>(), C->nb, r16, screen ? A->norm16.as<double>() : nullptr,
                screen ? B->norm16.as<double>() : nullptr, tau2);
        tr.mark("cmask16");
        if (sym) symm_finish16(C);
        C->nb16 = r16[1];
        S.level_tasks[L] = r16[3];  // all non-NIL container pairs (the BFS kept those with a 16-block product)
        S.level_tasks[L + 1] = r16[0];
        S.level_c_nodes[L + 1] = r16[1];
        S.block_products = r16[0];
        if (r16[2] > 0) {  // containers none of whose quadrants is a product: NIL at 16-granularity
          qt_mat D = drop_empty16(C);
          delete C;
          C = D;
          tr.mark("drop_empty16");
        }
      }
      if (plan && C->nb > 0 && !two_phase && C->pool.p == plan_pool_c) {  // keep the launch for qt_plan_execute
        plan->valid = true;
        plan->f32 = f32;
        if (f32) {
          NumericArgs32 nb;  // rebuilt as launched above
          nb.ntiles = ns[L - 2];
          nb.tile_start = t2_cstart.as<int32_t>();
          nb.pa = t2_pa.as<int32_t>();
          nb.pb = t2_pb.as<int32_t>();
          nb.childA2 = A->child[L - 2].as<int4>();
          nb.childA1 = A->child[L - 1].as<int4>();
          nb.childB2 = B->child[L - 2].as<int4>();
          nb.childB1 = B->child[L - 1].as<int4>();
          nb.childC2 = cchild2.as<int4>();
          nb.childC1 = cchild.as<int4>();
          nb.poolA = A->pool_ptr();
          nb.poolB = B->pool_ptr();
          nb.poolB2 = B->pool2;
          nb.splitB = B->split;
          nb.poolC = C->pool.p;
          nb.zeros = ctx->zeros.p;
          nb.counter = ctx->counters.as<int>() + 16;
          nb.trans = trans & 7;
          nb.poolT = poolTp;
          nb.counter_ready = false;  // re-executions zero the counter themselves
          plan->nb = nb;
          plan->keep[0] = std::move(t2_cstart);
          plan->keep[1] = std::move(t2_pa);
          plan->keep[2] = std::move(t2_pb);
          plan->keep[3] = std::move(cchild2);
          plan->keep[4] = std::move(cchild);
        } else {
          plan->na = na;
          plan->na.counter_ready = false;  // re-executions zero the counter themselves
          plan->keep[0] = std::move(cstart);
          plan->keep[1] = std::move(pa);
          plan->keep[2] = std::move(pb);
          plan->keep[3] = std::move(cchild);
        }
        if (sym) {
          plan->poolT = std::move(poolT);
          plan->tsrc = A->pool_ptr();
          plan->tnb = A->nb;
        }
      }
    }
    if (!ctx->async_multiply && ctx->timing) {
      QT_CUDA(cudaEventSynchronize(ctx->ev[4]));
      QT_CUDA(cudaEventElapsedTime(ms_sym, ctx->ev[2], ctx->ev[3]));
      QT_CUDA(cudaEventElapsedTime(ms_num, ctx->ev[3], ctx->ev[4]));
    }
    S.c_blocks = C->pend_slot >= 0 ? -1 : C->nb;  // (-1: a sync-free async product, not known yet)
    if (A->ubs == 16) S.nlevels = L + 2;  // + the 16-block level below the containers
    tr.mark("stats");
  } catch (...) {
    delete C;
    throw;
  }
  return C;
}

}  // namespace qt
