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
#include <cub/cub.cuh>

#include "qt_common.cuh"
#include "qt_internal.h"

namespace qt {

namespace {

constexpr int kThreads = 256;
inline unsigned grid_for(int64_t n) {
  int64_t g = (n + kThreads - 1) / kThreads;
  return (unsigned)(g < 1 ? 1 : g);
}

// counts of child tasks per (parent task, C child q), written group-major:
// position 4*start(s) + q*m(s) + local(p)
__global__ void k_count(int32_t F, const int32_t* __restrict__ pa, const int32_t* __restrict__ pb,
                        const int32_t* __restrict__ pc, const int32_t* __restrict__ cstart,
                        const int4* __restrict__ childA, const int4* __restrict__ childB,
                        int32_t* __restrict__ cnt) {
  int32_t p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= F) return;
  int32_t s = pc[p];
  int32_t c0 = cstart[s], m = cstart[s + 1] - c0, loc = p - c0;
  int4 a = childA[pa[p]];
  int4 b = childB[pb[p]];
  // A child (i,k) in slot 2i+k ; B child (k,j) in slot 2k+j
  int64_t base = 4ll * c0 + loc;
  cnt[base + 0ll * m] = (a.x >= 0 && b.x >= 0) + (a.y >= 0 && b.z >= 0);  // (0,0)
  cnt[base + 1ll * m] = (a.x >= 0 && b.y >= 0) + (a.y >= 0 && b.w >= 0);  // (0,1)
  cnt[base + 2ll * m] = (a.z >= 0 && b.x >= 0) + (a.w >= 0 && b.z >= 0);  // (1,0)
  cnt[base + 3ll * m] = (a.z >= 0 && b.y >= 0) + (a.w >= 0 && b.w >= 0);  // (1,1)
}

// per (s,q): start and size of the new group; flag = non-empty
__global__ void k_segs(int32_t ns, const int32_t* __restrict__ cstart,
                       const int32_t* __restrict__ incl, int32_t* __restrict__ flag,
                       int32_t* __restrict__ gstart) {
  int32_t x = blockIdx.x * blockDim.x + threadIdx.x;
  if (x >= 4 * ns) return;
  int32_t s = x >> 2, q = x & 3;
  int32_t c0 = cstart[s], m = cstart[s + 1] - c0;
  int64_t lo = 4ll * c0 + (int64_t)q * m, hi = lo + m;
  int32_t st = lo == 0 ? 0 : incl[lo - 1];
  int32_t en = incl[hi - 1];
  flag[x] = en > st;
  gstart[x] = st;
}

// C nodes of level l+1 (the non-empty groups) and the group -> node map of
// level l (C's child table at level l before pruning)
__global__ void k_newc(int32_t ns, const int32_t* __restrict__ flag,
                       const int32_t* __restrict__ nincl, const int32_t* __restrict__ gstart,
                       const uint64_t* __restrict__ ckey, const int32_t* __restrict__ incl,
                       int64_t n4, int32_t* __restrict__ cstart_next,
                       uint64_t* __restrict__ ckey_next, int32_t* __restrict__ cchild,
                       int32_t* __restrict__ sizes_out) {
  int32_t x = blockIdx.x * blockDim.x + threadIdx.x;
  if (x == 0) {
    int32_t nsn = nincl[4 * ns - 1];
    int32_t Fnext = incl[n4 - 1];
    cstart_next[nsn] = Fnext;
    sizes_out[0] = Fnext;
    sizes_out[1] = nsn;
  }
  if (x >= 4 * ns) return;
  if (flag[x]) {
    int32_t t = nincl[x] - 1;
    cstart_next[t] = gstart[x];
    ckey_next[t] = (ckey[x >> 2] << 2) | (uint64_t)(x & 3);
    cchild[x] = t;
  } else {
    cchild[x] = -1;
  }
}

__global__ void k_emit(int32_t F, const int32_t* __restrict__ pa, const int32_t* __restrict__ pb,
                       const int32_t* __restrict__ pc, const int32_t* __restrict__ cstart,
                       const int4* __restrict__ childA, const int4* __restrict__ childB,
                       const int32_t* __restrict__ incl, const int32_t* __restrict__ nincl,
                       int32_t* __restrict__ pa2, int32_t* __restrict__ pb2,
                       int32_t* __restrict__ pc2) {
  int32_t p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= F) return;
  int32_t s = pc[p];
  int32_t c0 = cstart[s], m = cstart[s + 1] - c0, loc = p - c0;
  int4 a4 = childA[pa[p]];
  int4 b4 = childB[pb[p]];
  int a[4] = {a4.x, a4.y, a4.z, a4.w};
  int b[4] = {b4.x, b4.y, b4.z, b4.w};
  int64_t base = 4ll * c0 + loc;
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    int i = q >> 1, j = q & 1;
    int64_t idx = base + (int64_t)q * m;
    int32_t pos = idx == 0 ? 0 : incl[idx - 1];
    int32_t newc = -1;
#pragma unroll
    for (int k = 0; k < 2; ++k) {
      int ac = a[2 * i + k], bc = b[2 * k + j];
      if (ac >= 0 && bc >= 0) {
        if (newc < 0) newc = nincl[4 * s + q] - 1;
        pa2[pos] = ac;
        pb2[pos] = bc;
        pc2[pos] = newc;
        ++pos;
      }
    }
  }
}

template <class T>
void incl_sum(qt_ctx ctx, const T* in, T* out, int64_t n) {
  size_t tb = 0;
  QT_CUDA(cub::DeviceScan::InclusiveSum(nullptr, tb, in, out, (int)n, ctx->stream));
  void* tmp = scratch(ctx, tb);
  QT_CUDA(cub::DeviceScan::InclusiveSum(tmp, tb, in, out, (int)n, ctx->stream));
  ctx->launches += 2;
}

}  // namespace

qt_mat multiply_local(qt_mat A, qt_mat B, qt_stats* stp, float* ms_sym, float* ms_num) {
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
    if (A->nb == 0 || B->nb == 0) {
      QT_CUDA(cudaEventRecord(ctx->ev[3], st));
      QT_CUDA(cudaEventRecord(ctx->ev[4], st));
    } else {
      int32_t* sizes = ctx->counters.as<int32_t>() + 8;  // [F', ns']
      int32_t* hsz = (int32_t*)ctx->pinned;
      // level 0: the single root task
      int32_t F = 1, ns = 1;
      DevBuf pa(4, st), pb(4, st), pc(4, st), cstart(8, st), ckey(8, st);
      {
        int32_t h0[4] = {0, 0, 0, 1};
        uint64_t k0 = 0;
        QT_CUDA(cudaMemsetAsync(pa.p, 0, 4, st));
        QT_CUDA(cudaMemsetAsync(pb.p, 0, 4, st));
        QT_CUDA(cudaMemsetAsync(pc.p, 0, 4, st));
        QT_CUDA(cudaMemcpyAsync(cstart.p, h0 + 2, 8, cudaMemcpyHostToDevice, st));
        QT_CUDA(cudaMemcpyAsync(ckey.p, &k0, 8, cudaMemcpyHostToDevice, st));
      }
      S.level_tasks[0] = 1;
      S.level_c_nodes[0] = 1;
      int64_t products = 0;
      for (int l = 0; l < L && F > 0; ++l) {
        bool last = (l == L - 1);
        int64_t n4 = 4ll * F;
        DevBuf cnt(n4 * 4, st), incl(n4 * 4, st);
        k_count<<<grid_for(F), kThreads, 0, st>>>(F, pa.as<int32_t>(), pb.as<int32_t>(),
                                                  pc.as<int32_t>(), cstart.as<int32_t>(),
                                                  A->child[l].as<int4>(), B->child[l].as<int4>(),
                                                  cnt.as<int32_t>());
        QT_LAUNCH_CHECK(ctx);
        incl_sum(ctx, cnt.as<int32_t>(), incl.as<int32_t>(), n4);
        DevBuf flag(16ll * ns, st), gstart(16ll * ns, st), nincl(16ll * ns, st);
        k_segs<<<grid_for(4ll * ns), kThreads, 0, st>>>(ns, cstart.as<int32_t>(), incl.as<int32_t>(),
                                                        flag.as<int32_t>(), gstart.as<int32_t>());
        QT_LAUNCH_CHECK(ctx);
        incl_sum(ctx, flag.as<int32_t>(), nincl.as<int32_t>(), 4ll * ns);
        // next-level C nodes (upper bound 4*ns) and the group -> node map
        DevBuf cstart2(4 * (4ll * ns + 1), st), ckey2(8 * 4ll * ns, st), cchild(16ll * ns, st);
        k_newc<<<grid_for(4ll * ns), kThreads, 0, st>>>(ns, flag.as<int32_t>(), nincl.as<int32_t>(),
                                                        gstart.as<int32_t>(), ckey.as<uint64_t>(),
                                                        incl.as<int32_t>(), n4, cstart2.as<int32_t>(),
                                                        ckey2.as<uint64_t>(), cchild.as<int32_t>(),
                                                        sizes);
        QT_LAUNCH_CHECK(ctx);
        QT_CUDA(cudaMemcpyAsync(hsz, sizes, 8, cudaMemcpyDeviceToHost, st));
        QT_CUDA(cudaStreamSynchronize(st));
        int32_t Fn = hsz[0], nsn = hsz[1];
        S.level_tasks[l + 1] = Fn;
        S.level_c_nodes[l + 1] = nsn;
        if (last) {
          products = Fn;
          // C blocks = level-L nodes; keys ascending (Morton order by construction)
          C->nb = nsn;
          C->key = std::move(ckey2);
          C->pool.alloc((size_t)nsn * 1024 * elem_size(C->dtype), st);
          QT_CUDA(cudaEventRecord(ctx->ev[3], st));
          NumericArgs na;
          na.ntiles = ns;
          na.tile_start = cstart.as<int32_t>();
          na.pa = pa.as<int32_t>();
          na.pb = pb.as<int32_t>();
          na.childA = A->child[l].as<int4>();
          na.childB = B->child[l].as<int4>();
          na.childC = cchild.as<int4>();
          na.poolA = A->pool_ptr();
          na.poolB = B->pool_ptr();
          na.poolB2 = B->pool2;
          na.splitB = B->split;
          na.poolC = C->pool.p;
          na.counter = ctx->counters.as<int>() + 16;
          if (nsn > 0) launch_numeric(ctx, C->dtype, na);
          QT_CUDA(cudaEventRecord(ctx->ev[4], st));
          break;
        }
        if (Fn == 0) break;
        DevBuf pa2(4ll * Fn, st), pb2(4ll * Fn, st), pc2(4ll * Fn, st);
        k_emit<<<grid_for(F), kThreads, 0, st>>>(F, pa.as<int32_t>(), pb.as<int32_t>(),
                                                 pc.as<int32_t>(), cstart.as<int32_t>(),
                                                 A->child[l].as<int4>(), B->child[l].as<int4>(),
                                                 incl.as<int32_t>(), nincl.as<int32_t>(),
                                                 pa2.as<int32_t>(), pb2.as<int32_t>(),
                                                 pc2.as<int32_t>());
        QT_LAUNCH_CHECK(ctx);
        pa = std::move(pa2);
        pb = std::move(pb2);
        pc = std::move(pc2);
        cstart = std::move(cstart2);
        ckey = std::move(ckey2);
        F = Fn;
        ns = nsn;
      }
      S.block_products = products;
      if (products == 0) {
        QT_CUDA(cudaEventRecord(ctx->ev[3], st));
        QT_CUDA(cudaEventRecord(ctx->ev[4], st));
      }
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
