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
// scans; the large levels use grid-wide kernels + device scans.  One host sync
// remains, before the numeric kernel (to size C's block pool).
#include <chrono>
#include <cstdlib>
#include <cub/cub.cuh>

#include "qt_common.cuh"
#include "qt_internal.h"

namespace qt {

namespace {

constexpr int kThreads = 256;
constexpr int kSmallThreads = 1024;
constexpr int64_t kSmallMaxF = 1 << 13;

inline unsigned grid_for(int64_t n) {
  int64_t g = (n + kThreads - 1) / kThreads;
  return (unsigned)(g < 1 ? 1 : g);
}

// C_l for every level: one CTA per level
__global__ void k_level_tasks(const int32_t* __restrict__ histA, const int32_t* __restrict__ histB,
                              int64_t H, int trans, int64_t* __restrict__ out) {
  using BR = cub::BlockReduce<long long, kThreads>;
  __shared__ typename BR::TempStorage tmp;
  const int l = blockIdx.x;
  const int64_t base = (1ll << l) - 1, m = 1ll << l;
  long long s = 0;
  for (int64_t K = threadIdx.x; K < m; K += blockDim.x)
    // cols(op(A)_l) . rows(op(B)_l); a transposed operand swaps its row/column histograms
    s += (long long)histA[((trans & 1) ? 0 : H) + base + K] *
         (long long)histB[((trans & 2) ? H : 0) + base + K];
  s = BR(tmp).Sum(s);
  if (threadIdx.x == 0) out[l] = s;
}

// C node on the block diagonal: in the symmetric square only its upper
// children exist (the (1,0) child is the transpose of (0,1), not computed)
__device__ __forceinline__ bool on_diagonal(uint64_t ckey) {
  return morton_row(ckey) == morton_col(ckey);
}

// A child (i,k) sits in slot 2i+k, B child (k,j) in slot 2k+j, C child (i,j) in 2i+j.
// Norm screening (qt_multiply_screened): a child task (a, b) survives iff
// ||a||^2 * ||b||^2 >= tau^2, squared Frobenius norms of quadtree nodes.  A
// node's squared norm is the sum of its blocks', so a node pair below the
// threshold contains only block pairs below it: pruning at any level is exact
// with respect to the block-level test.  na == nullptr: no screening.
struct Screen {
  const double* na;
  const double* nb;
  double tau2;
};
__device__ __forceinline__ bool pair_ok(int ar, int br, const Screen& sc, bool sym) {
  if (ar < 0 || br < 0) return false;
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
                                          bool skip_lower, const Screen& sc, bool sym,
                                          const int32_t* __restrict__ off,
                                          const int32_t* __restrict__ gidx, int32_t* __restrict__ pa2,
                                          int32_t* __restrict__ pb2, int32_t* __restrict__ pc2) {
  const int a[4] = {a4.x, a4.y, a4.z, a4.w};
  const int b[4] = {b4.x, b4.y, b4.z, b4.w};
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    if (skip_lower && q == 2) continue;
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
};

__global__ void __launch_bounds__(kSmallThreads, 1) k_bfs_small(SmallBfsArgs a) {
  using BS = cub::BlockScan<int, kSmallThreads>;
  __shared__ typename BS::TempStorage tmp;
  __shared__ int s_F, s_ns;
  const int tid = threadIdx.x;
  const bool sym = a.trans & 4;
  if (tid == 0) {
    a.pa[0][0] = sym ? 2 : 0;  // the root (a diagonal node in the symmetric square)
    a.pb[0][0] = sym ? 2 : 0;
    a.pc[0][0] = 0;
    a.f_out[0] = 1;
    a.cstart[0][0] = 0;
    a.cstart[0][1] = 1;
    a.ckey[0][0] = 0;
    a.ns_out[0] = 1;
    s_F = 1;
    s_ns = 1;
  }
  __syncthreads();
  for (int l = 0; l < a.l_end; ++l) {
    const int cur = l & 1, nxt = cur ^ 1;
    const bool prune = sym && l < (a.trans >> 8);  // C below the diagonal is not computed
    const int F = s_F, ns = s_ns;
    const int32_t* pa = a.pa[cur];
    const int32_t* pb = a.pb[cur];
    const int32_t* pc = a.pc[cur];
    const int32_t* cs = a.cstart[cur];
    const uint64_t* ck = a.ckey[cur];
    const int4* cA = a.childA[l];
    const int4* cB = a.childB[l];
    const Screen sc{a.normA[l + 1], a.normB[l + 1], a.tau2};
    // 1. child-task counts per (task, C child), group-major
    for (int p = tid; p < F; p += kSmallThreads) {
      const int s = pc[p], c0 = cs[s], m = cs[s + 1] - c0;
      int c[4];
      child_counts(op_children(cA, pa[p], a.trans & 1, sym), op_children(cB, pb[p], a.trans & 2, sym), c,
                   sc, sym);
      if (prune && on_diagonal(ck[s])) c[2] = 0;
      const int64_t base = 4ll * c0 + (p - c0);
#pragma unroll
      for (int q = 0; q < 4; ++q) a.off[base + (int64_t)q * m] = c[q];
    }
    __syncthreads();
    // 2. exclusive scan in place
    int carry = 0;
    for (int b0 = 0; b0 < 4 * F; b0 += kSmallThreads) {
      const int i = b0 + tid;
      const int v = i < 4 * F ? a.off[i] : 0;
      int ex, agg;
      BS(tmp).ExclusiveSum(v, ex, agg);
      if (i < 4 * F) a.off[i] = carry + ex;
      carry += agg;
      __syncthreads();
    }
    const int Fn = carry;
    // 3. new groups (non-empty (s,q)), their starts and keys
    int ncarry = 0;
    for (int b0 = 0; b0 < 4 * ns; b0 += kSmallThreads) {
      const int x = b0 + tid;
      int flag = 0, gst = 0;
      if (x < 4 * ns) {
        const int s = x >> 2, q = x & 3, c0 = cs[s], m = cs[s + 1] - c0;
        const int lo = 4 * c0 + q * m, hi = lo + m;
        gst = a.off[lo];
        const int en = hi < 4 * F ? a.off[hi] : Fn;
        flag = en > gst;
      }
      int ex, agg;
      BS(tmp).ExclusiveSum(flag, ex, agg);
      if (x < 4 * ns) {
        const int t = flag ? ncarry + ex : -1;
        a.gidx[x] = t;
        if (flag) {
          a.cstart[nxt][t] = gst;
          a.ckey[nxt][t] = (ck[x >> 2] << 2) | (uint64_t)(x & 3);
        }
      }
      ncarry += agg;
      __syncthreads();
    }
    const int nsn = ncarry;
    if (tid == 0) {
      a.cstart[nxt][nsn] = Fn;
      a.ns_out[l + 1] = nsn;
      a.f_out[l + 1] = Fn;
    }
    __syncthreads();
    // 4. emit the child tasks
    for (int p = tid; p < F; p += kSmallThreads) {
      const int s = pc[p], c0 = cs[s], m = cs[s + 1] - c0;
      emit_task(op_children(cA, pa[p], a.trans & 1, sym), op_children(cB, pb[p], a.trans & 2, sym),
                4ll * c0 + (p - c0), m, s, prune && on_diagonal(ck[s]), sc, sym, a.off, a.gidx, a.pa[nxt],
                a.pb[nxt],
                a.pc[nxt]);
    }
    __syncthreads();
    if (tid == 0) {
      s_F = Fn;
      s_ns = nsn;
    }
    __syncthreads();
  }
}

// ------------------------------------------------------------ large levels (grid-wide)

// Launch sizes come from host-side bounds (exact for regular products); the
// actual task count of the level is read from f_dev.  Threads of "virtual"
// tasks p in [F, Fb) zero the count positions [4p, 4p+4), so the scan over
// 4*Fb positions is exact.
__global__ void k_count(int32_t Fb, const int32_t* __restrict__ f_dev, const int32_t* __restrict__ pa,
                        const int32_t* __restrict__ pb, const int32_t* __restrict__ pc,
                        const int32_t* __restrict__ cstart, const uint64_t* __restrict__ ckey,
                        const int4* __restrict__ childA, const int4* __restrict__ childB, int mode,
                        Screen sc, int32_t* __restrict__ cnt) {
  const int32_t p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= Fb) return;
  if (p >= *f_dev) {
    *reinterpret_cast<int4*>(cnt + 4ll * p) = make_int4(0, 0, 0, 0);
    return;
  }
  const bool sym = mode & 4;
  const int32_t s = pc[p], c0 = cstart[s], m = cstart[s + 1] - c0;
  int c[4];
  child_counts(op_children(childA, pa[p], mode & 1, sym), op_children(childB, pb[p], mode & 2, sym), c,
               sc, sym);
  if ((mode & 8) && on_diagonal(ckey[s])) c[2] = 0;
  const int64_t base = 4ll * c0 + (p - c0);
#pragma unroll
  for (int q = 0; q < 4; ++q) cnt[base + (int64_t)q * m] = c[q];
}

// per (s,q) slot: start of the new group and non-empty flag (0 beyond the real ns)
__global__ void k_segs(int32_t nsb, const int32_t* __restrict__ ns_dev, int64_t n4,
                       const int32_t* __restrict__ cstart, const int32_t* __restrict__ off,
                       const int32_t* __restrict__ cnt, int32_t* __restrict__ flag,
                       int32_t* __restrict__ gstart) {
  const int32_t x = blockIdx.x * blockDim.x + threadIdx.x;
  if (x >= 4 * nsb) return;
  const int32_t ns = *ns_dev;
  int32_t f = 0, st = 0;
  if (x < 4 * ns) {
    const int32_t s = x >> 2, q = x & 3, c0 = cstart[s], m = cstart[s + 1] - c0;
    const int64_t lo = 4ll * c0 + (int64_t)q * m, hi = lo + m;
    st = off[lo];
    const int32_t en = hi < n4 ? off[hi] : off[n4 - 1] + cnt[n4 - 1];
    f = en > st;
  }
  flag[x] = f;
  gstart[x] = st;
}

__global__ void k_newc(int32_t nsb, const int32_t* __restrict__ ns_dev, int64_t n4,
                       const int32_t* __restrict__ off, const int32_t* __restrict__ cnt,
                       const int32_t* __restrict__ flag, const int32_t* __restrict__ nex,
                       const int32_t* __restrict__ gstart, const uint64_t* __restrict__ ckey,
                       int32_t* __restrict__ cstart_next, uint64_t* __restrict__ ckey_next,
                       int32_t* __restrict__ gidx, int32_t* __restrict__ ns_next,
                       int32_t* __restrict__ f_next) {
  const int32_t x = blockIdx.x * blockDim.x + threadIdx.x;
  const int32_t ns = *ns_dev;
  if (x >= 4 * ns) return;
  if (x == 4 * ns - 1) {
    const int32_t nsn = nex[x] + flag[x];
    const int32_t Fn = off[n4 - 1] + cnt[n4 - 1];
    cstart_next[nsn] = Fn;
    *ns_next = nsn;
    *f_next = Fn;
  }
  if (flag[x]) {
    const int32_t t = nex[x];
    cstart_next[t] = gstart[x];
    ckey_next[t] = (ckey[x >> 2] << 2) | (uint64_t)(x & 3);
    gidx[x] = t;
  } else {
    gidx[x] = -1;
  }
}

__global__ void k_emit(int32_t Fb, const int32_t* __restrict__ f_dev, const int32_t* __restrict__ pa,
                       const int32_t* __restrict__ pb, const int32_t* __restrict__ pc,
                       const int32_t* __restrict__ cstart, const uint64_t* __restrict__ ckey,
                       const int4* __restrict__ childA, const int4* __restrict__ childB, int mode,
                       Screen sc, const int32_t* __restrict__ off, const int32_t* __restrict__ gidx,
                       int32_t* __restrict__ pa2, int32_t* __restrict__ pb2,
                       int32_t* __restrict__ pc2) {
  const int32_t p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= Fb || p >= *f_dev) return;
  const bool sym = mode & 4;
  const int32_t s = pc[p], c0 = cstart[s], m = cstart[s + 1] - c0;
  emit_task(op_children(childA, pa[p], mode & 1, sym), op_children(childB, pb[p], mode & 2, sym),
            4ll * c0 + (p - c0), m, s, (mode & 8) && on_diagonal(ckey[s]), sc, sym, off, gidx, pa2, pb2,
            pc2);
}

// Upper bound of the symmetric square's tasks per level: with the full
// matrix's column and row counts both bounded by rows(U) + cols(U).
__global__ void k_level_tasks_sym(const int32_t* __restrict__ hist, int64_t H,
                                  int64_t* __restrict__ out) {
  using BR = cub::BlockReduce<long long, kThreads>;
  __shared__ typename BR::TempStorage tmp;
  const int l = blockIdx.x;
  const int64_t base = (1ll << l) - 1, m = 1ll << l;
  long long s = 0;
  for (int64_t K = threadIdx.x; K < m; K += blockDim.x) {
    const long long c = (long long)hist[base + K] + hist[H + base + K];
    s += c * c;
  }
  s = BR(tmp).Sum(s);
  if (threadIdx.x == 0) out[l] = s;
}

template <class T>
void excl_sum(qt_ctx ctx, const T* in, T* out, int64_t n) {
  size_t tb = 0;
  QT_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tb, in, out, (int)n, ctx->stream));
  void* tmp = scratch(ctx, tb);
  QT_CUDA(cub::DeviceScan::ExclusiveSum(tmp, tb, in, out, (int)n, ctx->stream));
  ctx->launches += 2;
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
    if (on) fprintf(stderr, "[qt trace] multiply:%s\n", buf.c_str());
  }
};

qt_mat multiply_local(qt_mat A, qt_mat B, qt_stats* stp, float* ms_sym, float* ms_num, int trans,
                      double tau) {
  const bool screen = tau >= 0.0;
  const double tau2 = tau * tau;
  if (screen) {
    ensure_norms(A);
    ensure_norms(B);
  }
  auto screen_at = [&](int level) {
    return Screen{screen ? A->norm2[level].as<double>() : nullptr,
                  screen ? B->norm2[level].as<double>() : nullptr, tau2};
  };
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
  C->dtype = A->dtype;
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
    QT_CUDA(cudaEventRecord(ctx->ev[2], st));
    std::vector<int64_t> F(L + 1, 0);
    if (A->nb > 0 && B->nb > 0) {
      // task counts per level (one sync): exact for regular products, an upper
      // bound for the symmetric square (its actual counts come from the BFS)
      const int64_t H = 2ll << L;
      DevBuf dF(8 * (L + 1), st);
      if (sym)
        k_level_tasks_sym<<<L + 1, kThreads, 0, st>>>(A->hist.as<int32_t>(), H, dF.as<int64_t>());
      else
        k_level_tasks<<<L + 1, kThreads, 0, st>>>(A->hist.as<int32_t>(), B->hist.as<int32_t>(), H,
                                                 trans & 3, dF.as<int64_t>());
      QT_LAUNCH_CHECK(ctx);
      QT_CUDA(cudaMemcpyAsync(F.data(), dF.p, 8 * (L + 1), cudaMemcpyDeviceToHost, st));
      QT_CUDA(cudaStreamSynchronize(st));
      tr.mark("counts");
      for (int l = 0; l <= L; ++l)
        if (F[l] >= (1ll << 31) / 4) fail(QT_EINVAL, "level %d has %lld tasks (> 2^29)", l, (long long)F[l]);
    }
    for (int l = 0; l <= L; ++l) S.level_tasks[l] = F[l];
    S.block_products = F[L];
    if (F[L] == 0) {
      // no block product at all: C is the NIL matrix
      C->nb = 0;
      QT_CUDA(cudaEventRecord(ctx->ev[3], st));
      QT_CUDA(cudaEventRecord(ctx->ev[4], st));
    } else {
      // upper bounds of the group counts: ns_{l+1} <= min(4 ns_l, F_{l+1})
      std::vector<int64_t> nsb(L + 1, 1);
      for (int l = 0; l < L; ++l) nsb[l + 1] = std::min<int64_t>(4 * nsb[l], F[l + 1]);
      DevBuf ns_dev(4 * (L + 1), st), f_dev(4 * (L + 1), st);
      int32_t* nsd = ns_dev.as<int32_t>();
      int32_t* fd = f_dev.as<int32_t>();
      // --- small levels in one CTA
      const bool f32 = C->dtype == QT_F32;
      int l_end = 0;
      while (l_end < L - 1 && F[l_end + 1] <= kSmallMaxF) ++l_end;
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
      sa.trans = trans;
      sa.tau2 = tau2;
      for (int l = 0; l <= L && l < QT_MAX_LEVELS; ++l) {
        sa.normA[l] = screen ? A->norm2[l].as<double>() : nullptr;
        sa.normB[l] = screen ? B->norm2[l].as<double>() : nullptr;
      }
      for (int l = 0; l < L; ++l) {
        sa.childA[l] = A->child[l].as<int4>();
        sa.childB[l] = B->child[l].as<int4>();
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
      tr.mark("small_alloc");
      k_bfs_small<<<1, kSmallThreads, 0, st>>>(sa);
      QT_LAUNCH_CHECK(ctx);
      const int cb = l_end & 1;
      DevBuf pa = std::move(sp[cb]), pb = std::move(sb[cb]), pc = std::move(sc[cb]);
      DevBuf cstart = std::move(scs[cb]), ckey = std::move(sck[cb]);
      // --- large levels, grid-wide, no host sync
      DevBuf cchild, t2_pa, t2_pb, t2_cstart, cchild2;
      tr.mark("small_launch");
      for (int l = l_end; l < L; ++l) {
        const bool last = (l == L - 1);
        const int32_t Fb = (int32_t)F[l];  // launch bound (exact unless symmetric)
        // per-level mode: transposes, symmetric, bit 3 = prune C below the diagonal here
        const int mode_l = (trans & 7) | ((sym && l < (trans >> 8)) ? 8 : 0);
        const int64_t n4 = 4ll * Fb, s4 = 4ll * nsb[l];
        DevBuf cnt(4 * n4, st), off(4 * n4, st);
        k_count<<<grid_for(Fb), kThreads, 0, st>>>(Fb, fd + l, pa.as<int32_t>(), pb.as<int32_t>(),
                                                   pc.as<int32_t>(), cstart.as<int32_t>(),
                                                   ckey.as<uint64_t>(), A->child[l].as<int4>(),
                                                   B->child[l].as<int4>(), mode_l, screen_at(l + 1),
                                                   cnt.as<int32_t>());
        QT_LAUNCH_CHECK(ctx);
        excl_sum(ctx, cnt.as<int32_t>(), off.as<int32_t>(), n4);
        DevBuf flag(4 * s4, st), gstart(4 * s4, st), nex(4 * s4, st), gidx(4 * s4, st);
        k_segs<<<grid_for(s4), kThreads, 0, st>>>((int32_t)nsb[l], nsd + l, n4, cstart.as<int32_t>(),
                                                  off.as<int32_t>(), cnt.as<int32_t>(),
                                                  flag.as<int32_t>(), gstart.as<int32_t>());
        QT_LAUNCH_CHECK(ctx);
        excl_sum(ctx, flag.as<int32_t>(), nex.as<int32_t>(), s4);
        DevBuf cstart2(4 * (nsb[l + 1] + 1), st), ckey2(8 * std::max<int64_t>(nsb[l + 1], 1), st);
        k_newc<<<grid_for(s4), kThreads, 0, st>>>((int32_t)nsb[l], nsd + l, n4, off.as<int32_t>(),
                                                  cnt.as<int32_t>(), flag.as<int32_t>(),
                                                  nex.as<int32_t>(), gstart.as<int32_t>(),
                                                  ckey.as<uint64_t>(), cstart2.as<int32_t>(),
                                                  ckey2.as<uint64_t>(), gidx.as<int32_t>(), nsd + l + 1,
                                                  fd + l + 1);
        QT_LAUNCH_CHECK(ctx);
        if (last) {
          C->key = std::move(ckey2);
          cchild = std::move(gidx);
          break;
        }
        const int64_t Fnb = F[l + 1];
        DevBuf pa2(4 * Fnb, st), pb2(4 * Fnb, st), pc2(4 * Fnb, st);
        k_emit<<<grid_for(Fb), kThreads, 0, st>>>(Fb, fd + l, pa.as<int32_t>(), pb.as<int32_t>(),
                                                  pc.as<int32_t>(), cstart.as<int32_t>(),
                                                  ckey.as<uint64_t>(), A->child[l].as<int4>(),
                                                  B->child[l].as<int4>(), mode_l, screen_at(l + 1),
                                                  off.as<int32_t>(),
                                                  gidx.as<int32_t>(), pa2.as<int32_t>(),
                                                  pb2.as<int32_t>(), pc2.as<int32_t>());
        QT_LAUNCH_CHECK(ctx);
        if (f32 && l == L - 2) {  // keep the level L-2 queue: the FP32 work items
          t2_pa = std::move(pa);
          t2_pb = std::move(pb);
          t2_cstart = std::move(cstart);
          cchild2 = std::move(gidx);
        }
        pa = std::move(pa2);
        pb = std::move(pb2);
        pc = std::move(pc2);
        cstart = std::move(cstart2);
        ckey = std::move(ckey2);
      }
      // --- group counts of every level (the one remaining sync): C's block count
      tr.mark("levels_launched");
      std::vector<int32_t> ns(L + 1, 0), Fa(L + 1, 0);
      QT_CUDA(cudaMemcpyAsync(ns.data(), nsd, 4 * (L + 1), cudaMemcpyDeviceToHost, st));
      QT_CUDA(cudaMemcpyAsync(Fa.data(), fd, 4 * (L + 1), cudaMemcpyDeviceToHost, st));
      QT_CUDA(cudaStreamSynchronize(st));
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
      QT_CUDA(cudaEventRecord(ctx->ev[3], st));
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
      na.normA = screen ? A->norm2[L].as<double>() : nullptr;
      na.normB = screen ? B->norm2[L].as<double>() : nullptr;
      na.tau2 = tau2;
      // tiles per scheduler grab: ~32 tasks per grab, at most 16 tiles
      {
        const int64_t per_tile = std::max<int64_t>(1, F[L - 1] / std::max<int32_t>(1, ns[L - 1]));
        // (tiles with >= 8 tasks stream well one at a time: grouping only costs balance)
        int64_t g = per_tile >= 8 ? 1 : std::min<int64_t>(16, 32 / per_tile);
        // keep >= 8 grabs per tile stream (2 per CTA, one CTA per SM)
        g = std::min<int64_t>(g, ns[L - 1] / (16ll * ctx->num_sms));
        na.group = (int)std::max<int64_t>(1, g);
        if (tr.on) {
          char b[64];
          snprintf(b, sizeof b, "group=%d", na.group);
          tr.mark(b);
        }
      }
      DevBuf poolT;  // symmetric square: blocks of U read transposed come from U^T's copy
      if (C->nb > 0 && !f32 && sym) {
        poolT.alloc((size_t)A->nb * 1024 * 8, st);
        launch_transpose_blocks(ctx, A->pool_ptr(), poolT.p, A->nb);
        na.poolT = poolT.p;
      }
      if (C->nb > 0 && !f32) launch_numeric(ctx, C->dtype, na);
      if (C->nb > 0 && f32 && sym) fail(QT_EDTYPE, "the symmetric square is FP64-only in this build");
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
        nb.trans = trans & 7;
        launch_numeric_f32(ctx, nb);
      }
      QT_CUDA(cudaEventRecord(ctx->ev[4], st));
      tr.mark("numeric_launched");
      QT_CUDA(cudaEventSynchronize(ctx->ev[4]));  // frontier buffers are released after this
      tr.mark("numeric_done");
    }
    QT_CUDA(cudaEventSynchronize(ctx->ev[4]));
    QT_CUDA(cudaEventElapsedTime(ms_sym, ctx->ev[2], ctx->ev[3]));
    QT_CUDA(cudaEventElapsedTime(ms_num, ctx->ev[3], ctx->ev[4]));
    S.c_blocks = C->nb;
  } catch (...) {
    delete C;
    throw;
  }
  return C;
}

}  // namespace qt
