// C ABI entry points of libqtmm (include/qt.h).  Argument checking, handle
// management and orchestration only; every step of the path runs in the
// kernels of qt_tree.cu, qt_symbolic.cu, qt_numeric.cu and qt_dist.cu.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>
#include <memory>
#include <mutex>
#include <new>
#include <unordered_map>

#include "qt_internal.h"

namespace qt {

static thread_local std::string g_last_error;
static std::mutex g_ctx_mu;
static std::unordered_map<cudaStream_t, int> g_stream_refs;

void fail(qt_status s, const char* fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  throw Error(s, buf);
}

static qt_status handle_exception() {
  try {
    throw;
  } catch (const Error& e) {
    g_last_error = e.what();
    return e.status;
  } catch (const std::bad_alloc&) {
    g_last_error = "host allocation failed";
    return QT_ENOMEM;
  } catch (const std::exception& e) {
    g_last_error = e.what();
    return QT_EINVAL;
  } catch (...) {
    g_last_error = "unknown error";
    return QT_EINVAL;
  }
}

// Multi-rank validation: a check or preparation that may fail on some ranks
// only (a block outside the rank's strip, a duplicate, a block below the
// diagonal, out of memory) must not leave the other ranks blocked in the next
// collective.  `local` runs on every rank; then one int64 allgather tells
// every rank whether any rank failed, and all of them fail with the same
// status (the failing rank keeps its own message).  `extra` (may be null) is
// sent along: the caller's per-rank payload of the same allgather.
template <class F>
static void collective_check(qt_ctx ctx, F&& local, int64_t* extra = nullptr, int64_t* extra_all = nullptr) {
  qt_status mine = QT_OK;
  std::string msg;
  try {
    local();
  } catch (const Error& e) {
    mine = e.status;
    msg = e.what();
  } catch (const std::bad_alloc&) {
    mine = QT_ENOMEM;
    msg = "host allocation failed";
  }
  if (ctx->world > 1) {
    int64_t send[2] = {(int64_t)mine, extra ? *extra : 0};
    std::vector<int64_t> all(2 * ctx->world);
    allgather_i64(ctx, send, all.data(), 2);
    if (extra_all)
      for (int g = 0; g < ctx->world; ++g) extra_all[g] = all[2 * g + 1];
    if (mine == QT_OK)
      for (int g = 0; g < ctx->world; ++g)
        if (all[2 * g] != QT_OK)
          fail((qt_status)all[2 * g], "rank %d failed (status %lld); see its qt_last_error()", g,
               (long long)all[2 * g]);
  }
  if (mine != QT_OK) throw Error(mine, msg);
}

// ---------------------------------------------------------------- allocator

namespace {
struct StreamCache {
  std::unordered_map<size_t, std::vector<void*>> free;
};
// Free lists are per (device, stream): the legacy default stream has the same
// handle (0) on every device, so the stream alone would let a block of one
// device be handed to a context of another.
struct CacheKey {
  int dev;
  cudaStream_t s;
  bool operator==(const CacheKey& o) const { return dev == o.dev && s == o.s; }
};
struct CacheKeyHash {
  size_t operator()(const CacheKey& k) const {
    return std::hash<const void*>()(k.s) ^ (size_t(k.dev) * 0x9E3779B97F4A7C15ull);
  }
};
std::mutex g_cache_mu;
std::unordered_map<CacheKey, StreamCache, CacheKeyHash> g_cache;

size_t size_class(size_t b) {
  if (b <= 512) return 512;
  if (b < (1u << 20)) {
    size_t c = 512;
    while (c < b) c <<= 1;
    return c;
  }
  const size_t g = 2u << 20;
  return (b + g - 1) / g * g;
}

int current_device() {
  int d = 0;
  cudaGetDevice(&d);
  return d;
}

void flush_device_caches(int dev) {
  // called on out-of-memory on `dev`: make sure no stream of that device still
  // uses a cached block, then return that device's cached blocks
  cudaDeviceSynchronize();
  for (auto it = g_cache.begin(); it != g_cache.end();) {
    if (it->first.dev != dev) {
      ++it;
      continue;
    }
    for (auto& fv : it->second.free)
      for (void* q : fv.second) cudaFree(q);
    it = g_cache.erase(it);
  }
}
}  // namespace

void* cache_alloc(size_t bytes, cudaStream_t s, int dev, size_t* granted) {
  const size_t c = size_class(bytes);
  *granted = c;
  {
    std::lock_guard<std::mutex> lk(g_cache_mu);
    auto it = g_cache.find(CacheKey{dev, s});
    if (it != g_cache.end()) {
      auto f = it->second.free.find(c);
      if (f != it->second.free.end() && !f->second.empty()) {
        void* q = f->second.back();
        f->second.pop_back();
        return q;
      }
    }
  }
  void* q = nullptr;
  cudaError_t e = cudaMalloc(&q, c);
  if (e == cudaErrorMemoryAllocation) {
    cudaGetLastError();
    std::lock_guard<std::mutex> lk(g_cache_mu);
    flush_device_caches(dev);
    e = cudaMalloc(&q, c);
  }
  if (e != cudaSuccess) {
    cudaGetLastError();
    fail(QT_ENOMEM, "device allocation of %zu bytes failed: %s", c, cudaGetErrorString(e));
  }
  return q;
}

void cache_free(void* p, size_t granted, cudaStream_t s, int dev) {
  std::lock_guard<std::mutex> lk(g_cache_mu);
  g_cache[CacheKey{dev, s}].free[granted].push_back(p);
}

void cache_release_stream(cudaStream_t s, int dev) {
  cudaStreamSynchronize(s);
  std::lock_guard<std::mutex> lk(g_cache_mu);
  auto it = g_cache.find(CacheKey{dev, s});
  if (it == g_cache.end()) return;
  for (auto& fv : it->second.free)
    for (void* q : fv.second) cudaFree(q);
  g_cache.erase(it);
}

int cache_device() { return current_device(); }

// Internal padding levels: the kernels need at least 4x4 32-blocks (the FP32
// kernel tiles 4x4 blocks), so a matrix of fewer block rows gets a quadtree
// of 2^L >= 4 blocks per side whose top levels are a chain of single nodes.
// The paper's quadtree (split "as far as possible") starts at the
// smallest 2^Lp >= the block rows; statistics and level counts are reported
// in that geometry, i.e. without the `pad` chain levels above its root.
static int pad_levels(const qt_mat_s* M) {
  int lp = 0;
  while ((1ll << lp) < M->nbr) ++lp;
  return M->L - lp;
}

static void shift_levels(qt_stats& S, int pad) {
  if (pad <= 0) return;
  for (int l = 0; l + pad < QT_MAX_LEVELS; ++l) {
    S.level_tasks[l] = S.level_tasks[l + pad];
    S.level_c_nodes[l] = S.level_c_nodes[l + pad];
  }
  for (int l = QT_MAX_LEVELS - pad; l < QT_MAX_LEVELS; ++l) S.level_tasks[l] = S.level_c_nodes[l] = 0;
  S.nlevels -= pad;
  S.leaf_level = std::max(0, S.leaf_level - pad);
}

// statistics at the caller's block size: for 64-blocks the 32-block level is
// internal (a 64-block product = one task at level L-1, 8 products of 32-blocks)
static void user_stats(qt_mat R, qt_stats& S) {
  if (R->ubs == 16) {  // levels and products at 16-block granularity were set by the multiply
    S.c_blocks = R->nb16;
  } else if (R->ubs == 64) {
    const int L = R->L;
    S.nlevels = L;  // levels 0 .. L-1
    S.block_products = S.level_tasks[L - 1];
    S.c_blocks = user_nblocks(R);
    S.level_tasks[L] = 0;
    S.level_c_nodes[L] = 0;
    if (S.leaf_level > L - 1) S.leaf_level = L - 1;
  }
  shift_levels(S, pad_levels(R));
}

static int ilog2(int64_t x) {
  int r = 0;
  while ((1ll << (r + 1)) <= x) ++r;
  return r;
}

void resolve_pending(qt_mat M) {
  qt_ctx ctx = M->ctx;
  const int slot = M->pend_slot;
  QT_CUDA(cudaEventSynchronize(ctx->pend_ev[slot]));
  M->nb = ctx->pend_host[128 * slot + M->L];  // the BFS's group count at the block level
  M->global_nb = user_nblocks(M);
  if (ctx->pend_owner[slot] == M) ctx->pend_owner[slot] = nullptr;
  M->pend_slot = -1;
}

}  // namespace qt

qt_mat_s::~qt_mat_s() {
  if (pend_slot >= 0 && ctx && ctx->pend_owner[pend_slot] == this) ctx->pend_owner[pend_slot] = nullptr;
}

using namespace qt;

// (a stale, non-sticky CUDA error left by an earlier call — already reported
// through that call's status — must not be attributed to this call's launches)
#define API_TRY \
  try {         \
    (void)cudaGetLastError();
#define API_CATCH              \
  }                            \
  catch (...) {                \
    return handle_exception(); \
  }                            \
  return QT_OK;

extern "C" {

const char* qt_last_error(void) { return g_last_error.c_str(); }

static void ctx_create(int device, void* cuda_stream, int rank, int world, const void* uid,
                       void* hub, qt_ctx* out) {
  if (!out) fail(QT_EINVAL, "out is NULL");
  *out = nullptr;
  if (world < 1 || rank < 0 || rank >= world) fail(QT_EINVAL, "bad rank %d / world %d", rank, world);
  int ndev = 0;
  QT_CUDA(cudaGetDeviceCount(&ndev));
  if (device < 0 || device >= ndev) fail(QT_EINVAL, "device %d not in [0,%d)", device, ndev);
  QT_CUDA(cudaSetDevice(device));
  qt_ctx c = new qt_ctx_s();
  try {
    c->device = device;
    c->stream = (cudaStream_t)cuda_stream;
    c->rank = rank;
    c->world = world;
    QT_CUDA(cudaDeviceGetAttribute(&c->num_sms, cudaDevAttrMultiProcessorCount, device));
    for (auto& e : c->ev) QT_CUDA(cudaEventCreate(&e));
    {
      std::lock_guard<std::mutex> lk(g_ctx_mu);
      ++g_stream_refs[c->stream];
    }
    c->counters.alloc(256, c->stream);
    QT_CUDA(cudaMemsetAsync(c->counters.p, 0, 256, c->stream));
    c->zeros.alloc(8192, c->stream);
    QT_CUDA(cudaMemsetAsync(c->zeros.p, 0, 8192, c->stream));
    c->pinned_bytes = 1024;  // small D2H staging (the sync-free multiply's level counts)
    // (mapped: the BFS kernels write the level counts of sync-free products straight into it)
    QT_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&c->pend_host), sizeof(int32_t) * 128 * qt_ctx_s::kPendRing,
                          cudaHostAllocMapped));
    for (auto& e : c->pend_ev) QT_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    QT_CUDA(cudaHostAlloc(&c->pinned, c->pinned_bytes, cudaHostAllocMapped));
    if (world > 1) {
      if (hub) dist_init_loopback(c, hub);
      else dist_init(c, uid);
    } else if (uid) {
      dist_init(c, uid);  // a one-rank NCCL communicator (the binding on one GPU; multiplies stay local)
    }
    QT_CUDA(cudaStreamSynchronize(c->stream));
  } catch (...) {
    if (c->pinned) cudaFreeHost(c->pinned);
    delete c;
    throw;
  }
  *out = c;
}

qt_status qt_ctx_create(int device, void* cuda_stream, int rank, int world,
                        const void* nccl_unique_id, qt_ctx* out) {
  API_TRY
  if (world > 1 && !nccl_unique_id) fail(QT_EINVAL, "nccl_unique_id is NULL with world > 1");
  ctx_create(device, cuda_stream, rank, world, nccl_unique_id, nullptr, out);
  API_CATCH
}

qt_status qt_ctx_info(qt_ctx ctx, int32_t* rank, int32_t* world, int32_t* comm_ranks, int32_t* transport) {
  API_TRY
  if (!ctx) fail(QT_EINVAL, "NULL context");
  int kind = 0;
  const int n = transport_info(ctx, &kind);
  if (rank) *rank = ctx->rank;
  if (world) *world = ctx->world;
  if (comm_ranks) *comm_ranks = n;
  if (transport) *transport = kind;
  API_CATCH
}

qt_status qt_ctx_set_timing(qt_ctx ctx, int32_t on) {
  API_TRY
  if (!ctx) fail(QT_EINVAL, "NULL context");
  ctx->timing = on != 0;
  API_CATCH
}

qt_status qt_loopback_hub_create(int32_t world, void** hub) {
  API_TRY
  if (!hub || world < 1) fail(QT_EINVAL, "bad arguments");
  *hub = loop_hub_create(world);
  API_CATCH
}

qt_status qt_loopback_hub_destroy(void* hub) {
  API_TRY
  if (hub) loop_hub_destroy(hub);
  API_CATCH
}

qt_status qt_ctx_create_loopback(int device, void* cuda_stream, int rank, int world, void* hub,
                                 qt_ctx* out) {
  API_TRY
  if (!hub) fail(QT_EINVAL, "hub is NULL");
  ctx_create(device, cuda_stream, rank, world, nullptr, hub, out);
  API_CATCH
}

qt_status qt_ctx_destroy(qt_ctx ctx) {
  API_TRY
  if (!ctx) return QT_OK;
  cudaSetDevice(ctx->device);
  cudaStreamSynchronize(ctx->stream);
  reap_pending(ctx, true);
  if (ctx->copy_stream) cudaStreamDestroy(ctx->copy_stream);
  if (ctx->h2d_stream) {
    cudaStreamSynchronize(ctx->h2d_stream);
    cache_release_stream(ctx->h2d_stream, ctx->device);
    cudaStreamDestroy(ctx->h2d_stream);
    cudaEventDestroy(ctx->h2d_done);
  }
  if (ctx->comm_stream) {
    cudaStreamSynchronize(ctx->comm_stream);
    cudaStreamDestroy(ctx->comm_stream);
    for (auto& e : ctx->ov_ev) cudaEventDestroy(e);
  }
  if (ctx->transport) dist_finalize(ctx);
  for (auto& e : ctx->ev) cudaEventDestroy(e);
  ctx->scratch.release();
  ctx->counters.release();
  ctx->zeros.release();
  cudaStreamSynchronize(ctx->stream);
  // cached blocks of this stream are freed only when no other context uses it
  {
    std::lock_guard<std::mutex> lk(g_ctx_mu);
    if (--g_stream_refs[ctx->stream] == 0) {
      g_stream_refs.erase(ctx->stream);
      cache_release_stream(ctx->stream, ctx->device);
    }
  }
  if (ctx->pinned) cudaFreeHost(ctx->pinned);
  if (ctx->pend_host) cudaFreeHost(ctx->pend_host);
  if (ctx->small_host) cudaFreeHost(ctx->small_host);
  for (auto& e : ctx->pend_ev)
    if (e) cudaEventDestroy(e);
  delete ctx;
  API_CATCH
}

qt_status qt_create(qt_ctx ctx, int64_t n, int32_t leaf_dim, int32_t block_size, qt_dtype dtype,
                    int64_t nblocks, const int32_t* brow, const int32_t* bcol, const void* values,
                    const int32_t* row_bounds, qt_mat* out) {
  API_TRY
  if (!ctx || !out) fail(QT_EINVAL, "ctx/out is NULL");
  *out = nullptr;
  QT_CUDA(cudaSetDevice(ctx->device));
  if (dtype != QT_F64 && dtype != QT_F32) fail(QT_EDTYPE, "unknown dtype %d", (int)dtype);
  if (block_size != 16 && block_size != 32 && block_size != 64)
    fail(QT_EINVAL, "block_size %d: 16, 32 and 64 are built", block_size);
  // (16-blocks are held in 32-blocks: n and leaf_dim multiples of 32, reading C-27)
  const int gran = std::max(block_size, 32);
  if (n <= 0 || n % gran != 0)
    fail(QT_EINVAL, "n=%lld must be a positive multiple of %d (block_size=%d, readings C-4, C-27)",
         (long long)n, gran, block_size);
  if (leaf_dim < gran || leaf_dim % gran != 0 || ((leaf_dim / gran) & (leaf_dim / gran - 1)) != 0)
    fail(QT_EINVAL, "leaf_dim=%d must be a power-of-two multiple of %d (block_size=%d)", leaf_dim, gran,
         block_size);
  if (nblocks < 0 || nblocks >= (1ll << 31)) fail(QT_EINVAL, "nblocks=%lld", (long long)nblocks);
  if (nblocks > 0 && (!brow || !bcol || !values)) fail(QT_EINVAL, "NULL block arrays");
  // 64-blocks are held as 2x2 quads of 32-blocks (the kernels' block size)
  const int f = block_size / 32;
  int64_t nbr = n / 32;
  if (nbr > (1 << 20)) fail(QT_EINVAL, "n too large (more than 2^20 block rows)");
  qt_mat M = new qt_mat_s();
  try {
    M->ctx = ctx;
    M->n = n;
    M->leaf_dim = leaf_dim;
    M->bs = 32;
    M->ubs = block_size;
    M->dtype = dtype;
    M->nbr = (int32_t)nbr;
    // at least 4x4 (caller) blocks (reading C-3): the FP32 kernel tiles 4x4 32-blocks
    int L = f == 2 ? 3 : 2;
    while ((1ll << L) < nbr) ++L;
    M->L = L;
    M->leaf_level = std::max(0, L - ilog2(leaf_dim / 32));
    // every rank validates its own blocks; all ranks learn whether any failed
    // (and each rank's block count) in one allgather, so a rank-local
    // QT_ERANGE / QT_EDUP / QT_ENOMEM never leaves the others blocked
    cudaStream_t st = ctx->stream;
    int64_t mine_nb = 0;
    std::vector<int64_t> all_nb(ctx->world, 0);
    collective_check(ctx, [&] {
      // block-row ownership
      M->bounds.assign(ctx->world + 1, 0);
      if (ctx->world == 1) {
        M->bounds[1] = (int32_t)nbr;
      } else if (row_bounds) {
        for (int g = 0; g <= ctx->world; ++g) {
          if (block_size == 16 && (row_bounds[g] & 1)) fail(QT_EINVAL, "block_size 16: row_bounds must be even");
          M->bounds[g] = rows_to_internal(row_bounds[g], block_size);
        }
        if (M->bounds[0] != 0 || M->bounds[ctx->world] != nbr)
          fail(QT_EINVAL, "row_bounds must start at 0 and end at %lld",
               (long long)rows_to_user((int32_t)nbr, block_size));
        for (int g = 0; g < ctx->world; ++g)
          if (M->bounds[g + 1] < M->bounds[g]) fail(QT_EINVAL, "row_bounds not non-decreasing");
      } else {
        const int64_t nu = std::max<int64_t>(1, nbr / std::max(f, 1)),
                      per = (nu + ctx->world - 1) / ctx->world;
        for (int g = 0; g <= ctx->world; ++g)
          M->bounds[g] = (int32_t)(std::min<int64_t>(nu, per * g) * std::max(f, 1));
      }
      M->row_lo = M->bounds[ctx->rank];
      M->row_hi = M->bounds[ctx->rank + 1];
      // inputs to the device (stream-ordered copies from host, pinned or pageable)
        size_t es = elem_size(dtype);
      DevBuf dr, dc, dv;
      const int32_t* pr = brow;
      const int32_t* pc = bcol;
      const void* pv = values;
      if (nblocks > 0) {
        if (!is_device_ptr(brow)) {
          dr.alloc(nblocks * 4, st);
          QT_CUDA(cudaMemcpyAsync(dr.p, brow, nblocks * 4, cudaMemcpyHostToDevice, st));
          pr = dr.as<int32_t>();
        }
        if (!is_device_ptr(bcol)) {
          dc.alloc(nblocks * 4, st);
          QT_CUDA(cudaMemcpyAsync(dc.p, bcol, nblocks * 4, cudaMemcpyHostToDevice, st));
          pc = dc.as<int32_t>();
        }
        const size_t vb = (size_t)nblocks * block_size * block_size * es;
        if (!is_device_ptr(values)) {
          // the values (the bulk) come in on the context's H2D stream, into a
          // staging buffer of that stream's cache: the copy can start while the
          // context stream still runs earlier work (e.g. the previous
          // qt_multiply_async); the build waits for it through an event
          if (!ctx->h2d_stream) {
            QT_CUDA(cudaStreamCreateWithFlags(&ctx->h2d_stream, cudaStreamNonBlocking));
            QT_CUDA(cudaEventCreateWithFlags(&ctx->h2d_done, cudaEventDisableTiming));
          }
          dv.alloc(vb, ctx->h2d_stream);
          QT_CUDA(cudaMemcpyAsync(dv.p, values, vb, cudaMemcpyHostToDevice, ctx->h2d_stream));
          QT_CUDA(cudaEventRecord(ctx->h2d_done, ctx->h2d_stream));
          QT_CUDA(cudaStreamWaitEvent(st, ctx->h2d_done, 0));
          pv = dv.p;
        }
      }
      if (block_size == 16) {
        build_from_blocks16(M, nblocks, pr, pc, pv, 2 * M->row_lo, 2 * M->row_hi);
      } else if (f == 2 && nblocks > 0) {
        DevBuf sr, sc, sv;
        split64(ctx, dtype, nblocks, pr, pc, pv, sr, sc, sv);
        build_from_blocks(M, 4 * nblocks, sr.as<int32_t>(), sc.as<int32_t>(), sv.p, M->row_lo, M->row_hi);
      } else {
        build_from_blocks(M, nblocks, pr, pc, pv, M->row_lo, M->row_hi);
      }
      mine_nb = user_nblocks(M);
    }, &mine_nb, all_nb.data());
    M->global_nb = mine_nb;
    if (ctx->world > 1) {
      M->global_nb = 0;
      for (auto v : all_nb) M->global_nb += v;
    }
    QT_CUDA(cudaStreamSynchronize(st));
  } catch (...) {
    delete M;
    throw;
  }
  *out = M;
  API_CATCH
}

// Reading C-30: the FP32 kernel computes whole 4x4-block tiles (16 block
// products per tile step, absent blocks as zeros); the FP64 kernel computes
// only the products that exist, at ~1/5 of the FP32 kernel's dense rate.  With
// steps <= 4 * (tasks at level L-2), the tile density is at least
// products / (64 * tasks_{L-2}); below QT_F32_DENSITY (default 0.2 = the rate
// ratio 35 / 178 TFLOP/s measured on B200) the FP64 path is faster.
static bool fp32_prefers_fp64(qt_mat A, qt_mat B, int trans) {
  if (A->L < 2 || (trans & 4)) return false;
  const char* e = getenv("QT_F32_DENSITY");
  const double thr = e ? atof(e) : 0.2;
  if (thr <= 0) return false;
  const std::vector<int64_t> F = level_task_bounds(A, B, trans);
  const int L = A->L;
  if (F[L] == 0 || F[L - 2] == 0) return false;
  return (double)F[L] / (64.0 * (double)F[L - 2]) < thr;
}

qt_status qt_multiply(qt_mat A, qt_mat B, qt_mat* C, qt_stats* st) {
  return qt_multiply_ex(A, B, 0, 0, C, st);
}

qt_status qt_multiply_ex(qt_mat A, qt_mat B, int32_t trans_a, int32_t trans_b, qt_mat* C,
                         qt_stats* st) {
  API_TRY
  resolve(A);
  resolve(B);
  if (!A || !B || !C) fail(QT_EINVAL, "NULL argument");
  *C = nullptr;
  if (A->ctx != B->ctx) fail(QT_ESTATE, "A and B belong to different contexts");
  if (A->n != B->n) fail(QT_EDIM, "dimension mismatch: %lld vs %lld", (long long)A->n, (long long)B->n);
  if (A->leaf_dim != B->leaf_dim || A->ubs != B->ubs)
    fail(QT_EBS, "leaf_dim/block_size mismatch: (%d,%d) vs (%d,%d)", A->leaf_dim, A->ubs,
         B->leaf_dim, B->ubs);
  if (A->dtype != B->dtype) fail(QT_EDTYPE, "dtype mismatch");
  qt_ctx ctx = A->ctx;
  QT_CUDA(cudaSetDevice(ctx->device));
  if ((trans_a | trans_b) & ~1) fail(QT_EINVAL, "trans_a / trans_b must be 0 or 1");
  const int trans = (trans_a ? 1 : 0) | (trans_b ? 2 : 0);
  if (trans && ctx->world > 1)
    fail(QT_EINVAL, "transposed operands are single-rank only (row strips of A^T are column strips of A)");
  ensure_levels(A);
  ensure_levels(B);
  qt_stats local;
  qt_stats& S = st ? *st : local;
  memset(&S, 0, sizeof(S));
  const bool timed = !ctx->async_multiply && ctx->timing;
  if (timed) QT_CUDA(cudaEventRecord(ctx->ev[0], ctx->stream));
  qt_mat R;
  if (ctx->world == 1 && A->dtype == QT_F32 && fp32_prefers_fp64(A, B, trans)) {
    // reading C-30: a sparse FP32 product whose 4x4-block tcgen05 tiles would
    // be mostly empty runs on FP64 copies through the FP64 kernel (which
    // skips absent blocks) and C is rounded to FP32
    float ms_sym = 0, ms_num = 0;
    R = multiply_local(f64_of(A), f64_of(B), &S, &ms_sym, &ms_num, trans, -1.0, nullptr, 0, INT32_MAX, nullptr,
                       /*out_f32=*/true);
    S.ms_symbolic = ms_sym;
    S.ms_numeric = ms_num;
  } else if (ctx->world == 1) {
    float ms_sym = 0, ms_num = 0;
    R = multiply_local(A, B, &S, &ms_sym, &ms_num, trans);
    S.ms_symbolic = ms_sym;
    S.ms_numeric = ms_num;
  } else {
    R = multiply_dist(A, B, &S);
  }
  if (ctx->world == 1 && A->ubs != 16 && timed) {
    // the numeric kernel's completion event (already waited for) ends the call:
    // no second record + host round trip
    QT_CUDA(cudaEventElapsedTime(&S.ms_total, ctx->ev[0], ctx->ev[4]));
  } else if (timed) {
    QT_CUDA(cudaEventRecord(ctx->ev[1], ctx->stream));
    QT_CUDA(cudaEventSynchronize(ctx->ev[1]));
    QT_CUDA(cudaEventElapsedTime(&S.ms_total, ctx->ev[0], ctx->ev[1]));
  } else if (!ctx->async_multiply && !(ctx->world == 1 && A->ubs != 16)) {
    QT_CUDA(cudaStreamSynchronize(ctx->stream));  // (timing off: the call still ends complete)
  }
  R->global_nb = user_nblocks(R);
  user_stats(R, S);
  *C = R;
  API_CATCH
}

// ------------------------------------------------------------ plan / execute

struct qt_plan_s {
  qt_ctx ctx = nullptr;
  qt_mat C = nullptr;  // the product the plan writes (owned by the caller)
  NumericPlan np;
};

qt_status qt_multiply_plan(qt_mat A, qt_mat B, int32_t trans_a, int32_t trans_b, qt_plan* plan, qt_mat* C,
                           qt_stats* st) {
  API_TRY
  resolve(A);
  resolve(B);
  if (!A || !B || !C || !plan) fail(QT_EINVAL, "NULL argument");
  *C = nullptr;
  *plan = nullptr;
  if (A->ctx != B->ctx) fail(QT_ESTATE, "A and B belong to different contexts");
  if (A->ctx->world != 1) fail(QT_EINVAL, "plans are single-rank");
  if (A->ctx->async_multiply) fail(QT_ESTATE, "plan inside qt_multiply_async");
  if (A->n != B->n) fail(QT_EDIM, "dimension mismatch");
  if (A->leaf_dim != B->leaf_dim || A->ubs != B->ubs) fail(QT_EBS, "leaf_dim/block_size mismatch");
  if (A->dtype != B->dtype) fail(QT_EDTYPE, "dtype mismatch");
  if ((trans_a | trans_b) & ~1) fail(QT_EINVAL, "trans_a / trans_b must be 0 or 1");
  qt_ctx ctx = A->ctx;
  QT_CUDA(cudaSetDevice(ctx->device));
  ensure_levels(A);
  ensure_levels(B);
  qt_stats local;
  qt_stats& S = st ? *st : local;
  memset(&S, 0, sizeof(S));
  auto* P = new qt_plan_s();
  try {
    P->ctx = ctx;
    QT_CUDA(cudaEventRecord(ctx->ev[0], ctx->stream));
    float ms_sym = 0, ms_num = 0;
    qt_mat R = multiply_local(A, B, &S, &ms_sym, &ms_num, (trans_a ? 1 : 0) | (trans_b ? 2 : 0), -1.0, nullptr, 0,
                              INT32_MAX, &P->np);
    S.ms_symbolic = ms_sym;
    S.ms_numeric = ms_num;
    QT_CUDA(cudaEventRecord(ctx->ev[1], ctx->stream));
    QT_CUDA(cudaEventSynchronize(ctx->ev[1]));
    QT_CUDA(cudaEventElapsedTime(&S.ms_total, ctx->ev[0], ctx->ev[1]));
    R->global_nb = user_nblocks(R);
    user_stats(R, S);
    P->C = R;
    *C = R;
  } catch (...) {
    delete P;
    throw;
  }
  *plan = P;
  API_CATCH
}

qt_status qt_symm_square_plan(qt_mat A, qt_plan* plan, qt_mat* C, qt_stats* st) {
  API_TRY
  resolve(A);
  if (!A || !C || !plan) fail(QT_EINVAL, "NULL argument");
  *C = nullptr;
  *plan = nullptr;
  qt_ctx ctx = A->ctx;
  if (ctx->world != 1) fail(QT_EINVAL, "plans are single-rank");
  if (ctx->async_multiply) fail(QT_ESTATE, "plan inside qt_multiply_async");
  if (A->ubs != 32) fail(QT_EBS, "symmetric-square plans are built for block_size 32");
  QT_CUDA(cudaSetDevice(ctx->device));
  check_upper(A);
  ensure_levels(A);
  qt_stats local;
  qt_stats& S = st ? *st : local;
  memset(&S, 0, sizeof(S));
  auto* P = new qt_plan_s();
  try {
    P->ctx = ctx;
    QT_CUDA(cudaEventRecord(ctx->ev[0], ctx->stream));
    float ms_sym = 0, ms_num = 0;
    qt_mat R = multiply_local(A, A, &S, &ms_sym, &ms_num, 4 | (A->L << 8), -1.0, nullptr, 0, INT32_MAX, &P->np);
    S.ms_symbolic = ms_sym;
    S.ms_numeric = ms_num;
    QT_CUDA(cudaEventRecord(ctx->ev[1], ctx->stream));
    QT_CUDA(cudaEventSynchronize(ctx->ev[1]));
    QT_CUDA(cudaEventElapsedTime(&S.ms_total, ctx->ev[0], ctx->ev[1]));
    R->global_nb = user_nblocks(R);
    P->C = R;
    *C = R;
  } catch (...) {
    delete P;
    throw;
  }
  *plan = P;
  API_CATCH
}

qt_status qt_plan_execute(qt_plan plan) {
  API_TRY
  if (!plan) fail(QT_EINVAL, "NULL plan");
  qt_ctx ctx = plan->ctx;
  QT_CUDA(cudaSetDevice(ctx->device));
  NumericPlan& np = plan->np;
  if (!np.valid) return QT_OK;  // an empty product: nothing to recompute
  if (np.tnb > 0) {             // symmetric square: U's transposed copy from its current values
    if (np.f32)
      launch_transpose_blocks_f32(ctx, np.tsrc, np.poolT.p, np.tnb);
    else
      launch_transpose_blocks(ctx, np.tsrc, np.poolT.p, np.tnb);
  }
  if (np.f32)
    launch_numeric_f32(ctx, np.nb);
  else
    launch_numeric(ctx, QT_F64, np.na);
  API_CATCH
}

qt_status qt_plan_destroy(qt_plan plan) {
  API_TRY
  if (!plan) return QT_OK;
  QT_CUDA(cudaSetDevice(plan->ctx->device));
  QT_CUDA(cudaStreamSynchronize(plan->ctx->stream));
  delete plan;
  API_CATCH
}

qt_status qt_update_values(qt_mat A, const void* values) {
  API_TRY
  resolve(A);
  if (!A) fail(QT_EINVAL, "NULL matrix");
  if (A->ubs != 32) fail(QT_EBS, "qt_update_values is built for block_size 32");
  if (A->nb > 0 && !values) fail(QT_EINVAL, "NULL values");
  QT_CUDA(cudaSetDevice(A->ctx->device));
  update_values(A, values);
  API_CATCH
}

qt_status qt_multiply_async(qt_mat A, qt_mat B, qt_mat* C, qt_stats* st) {
  if (!A) return qt_multiply(A, B, C, st);
  qt_ctx ctx = A->ctx;
  // single rank only (the multi-rank exchange synchronises anyway)
  const bool was = ctx->async_multiply;
  ctx->async_multiply = ctx->world == 1;
  const qt_status r = qt_multiply(A, B, C, st);
  ctx->async_multiply = was;
  return r;
}

qt_status qt_multiply_screened(qt_mat A, qt_mat B, double tau, qt_mat* C, qt_stats* st) {
  API_TRY
  resolve(A);
  resolve(B);
  if (!A || !B || !C) fail(QT_EINVAL, "NULL argument");
  *C = nullptr;
  if (!(tau >= 0)) fail(QT_EINVAL, "tau must be >= 0");
  if (A->ctx != B->ctx) fail(QT_ESTATE, "A and B belong to different contexts");
  if (A->n != B->n) fail(QT_EDIM, "dimension mismatch");
  if (A->leaf_dim != B->leaf_dim || A->ubs != B->ubs) fail(QT_EBS, "leaf_dim/block_size mismatch");
  if (A->dtype != B->dtype) fail(QT_EDTYPE, "dtype mismatch");
  if (A->ubs == 64) fail(QT_EBS, "norm screening is built for block_size 16 and 32");
  qt_ctx ctx = A->ctx;
  QT_CUDA(cudaSetDevice(ctx->device));
  ensure_levels(A);
  ensure_levels(B);
  // FP32 (reading C-29): a tcgen05 tile MMA cannot skip single block
  // products, so the screened FP32 product runs on FP64 copies of A and B
  // (exact conversion) through the FP64 kernel and C is rounded to FP32 —
  // the oracle is the double product of the same FP32 values
  qt_mat a = A, b = B;
  if (A->dtype == QT_F32) {  // (the FP64 copies are kept with the handles)
    a = f64_of(A);
    b = f64_of(B);
  }
  qt_stats local;
  qt_stats& S = st ? *st : local;
  memset(&S, 0, sizeof(S));
  QT_CUDA(cudaEventRecord(ctx->ev[0], ctx->stream));
  qt_mat R;
  if (ctx->world > 1) {  // the exchange of the full product, then the screened multiply on B_ext
    R = multiply_dist(a, b, &S, tau);
  } else {
    float ms_sym = 0, ms_num = 0;
    R = multiply_local(a, b, &S, &ms_sym, &ms_num, 0, tau);
    S.ms_symbolic = ms_sym;
    S.ms_numeric = ms_num;
  }
  if (A->dtype == QT_F32) {
    std::unique_ptr<qt_mat_s> R64(R);
    R = convert_dtype(R64.get(), QT_F32);
  }
  QT_CUDA(cudaEventRecord(ctx->ev[1], ctx->stream));
  QT_CUDA(cudaEventSynchronize(ctx->ev[1]));
  QT_CUDA(cudaEventElapsedTime(&S.ms_total, ctx->ev[0], ctx->ev[1]));
  R->global_nb = user_nblocks(R);
  user_stats(R, S);
  *C = R;
  API_CATCH
}

qt_status qt_symm_square(qt_mat A, qt_mat* C, qt_stats* st) {
  API_TRY
  resolve(A);
  if (!A || !C) fail(QT_EINVAL, "NULL argument");
  *C = nullptr;
  qt_ctx ctx = A->ctx;
  QT_CUDA(cudaSetDevice(ctx->device));
  if (ctx->world > 1 && A->ubs == 64) fail(QT_EBS, "the multi-rank symmetric square needs block_size 16 or 32");
  // rank-local checks (a block below the diagonal in this rank's strip, out
  // of memory preparing the completed copy) are agreed on by all ranks before
  // the first exchange step
  collective_check(ctx, [&] {
    if (A->ubs == 16)
      check_upper16(A);
    else
      check_upper(A);
    ensure_levels(A);
    if (ctx->world > 1 && A->ubs == 16 && !A->sym16) A->sym16.reset(symm_prepare16(A));
  });
  qt_stats local;
  qt_stats& S = st ? *st : local;
  memset(&S, 0, sizeof(S));
  QT_CUDA(cudaEventRecord(ctx->ev[0], ctx->stream));
  float ms_sym = 0, ms_num = 0;
  qt_mat R;
  if (ctx->world > 1) {
    // (block size 16: the exchange moves the completed containers of each
    // rank's copy, so received diagonal containers arrive complete)
    if (A->ubs == 16 && !A->sym16) A->sym16.reset(symm_prepare16(A));
    R = symm_square_dist(A->ubs == 16 ? A->sym16.get() : A, &S);
    ms_sym = S.ms_symbolic;
    ms_num = S.ms_numeric;
  } else if (A->ubs == 64) {
    // drop the (1,0) 32-sub-block of every diagonal 64-block (it is the
    // transpose of (0,1)); diagonal C 64-blocks are then completed by not
    // pruning at the last (32-block) level
    qt_mat U = upper32_view(A);
    try {
      R = multiply_local(U, U, &S, &ms_sym, &ms_num, 4 | ((A->L - 1) << 8));
    } catch (...) {
      delete U;
      throw;
    }
    delete U;
  } else if (A->ubs == 16) {
    // diagonal 32-containers completed with (1,0) = (0,1)^T: the symmetric
    // square of the 32-container matrix, the (1,0) 16-blocks of C's diagonal
    // containers left out (k_cmask16) and zeroed (symm_finish16); the
    // completed copy is kept with A for the next call
    if (!A->sym16) A->sym16.reset(symm_prepare16(A));
    R = multiply_local(A->sym16.get(), A->sym16.get(), &S, &ms_sym, &ms_num, 4 | (A->L << 8));
  } else {
    R = multiply_local(A, A, &S, &ms_sym, &ms_num, 4 | (A->L << 8));
  }
  S.ms_symbolic = ms_sym;
  S.ms_numeric = ms_num;
  QT_CUDA(cudaEventRecord(ctx->ev[1], ctx->stream));
  QT_CUDA(cudaEventSynchronize(ctx->ev[1]));
  QT_CUDA(cudaEventElapsedTime(&S.ms_total, ctx->ev[0], ctx->ev[1]));
  R->global_nb = user_nblocks(R);
  user_stats(R, S);
  *C = R;
  API_CATCH
}

qt_status qt_truncate(qt_mat A, double tau, qt_mat* out) {
  API_TRY
  resolve(A);
  if (!A || !out) fail(QT_EINVAL, "NULL argument");
  *out = nullptr;
  if (!(tau >= 0)) fail(QT_EINVAL, "tau must be >= 0");
  QT_CUDA(cudaSetDevice(A->ctx->device));
  qt_mat R;
  if (A->ctx->world > 1) {
    R = truncate_dist(A, tau);
  } else {
    R = truncate(A, tau);
    R->global_nb = user_nblocks(R);
  }
  QT_CUDA(cudaStreamSynchronize(A->ctx->stream));
  *out = R;
  API_CATCH
}

qt_status qt_info(qt_mat A, int64_t* n, int32_t* leaf_dim, int32_t* block_size, qt_dtype* dtype,
                  int64_t* local_nblocks, int64_t* global_nblocks, int32_t* row_lo,
                  int32_t* row_hi) {
  API_TRY
  resolve(A);
  if (!A) fail(QT_EINVAL, "NULL matrix");
  if (n) *n = A->n;
  if (leaf_dim) *leaf_dim = A->leaf_dim;
  if (block_size) *block_size = A->ubs;
  if (dtype) *dtype = A->dtype;
  if (local_nblocks) *local_nblocks = user_nblocks(A);
  if (global_nblocks) *global_nblocks = A->global_nb;
  if (row_lo) *row_lo = rows_to_user(A->row_lo, A->ubs);
  if (row_hi) *row_hi = rows_to_user(A->row_hi, A->ubs);
  API_CATCH
}

qt_status qt_level_nodes(qt_mat A, int64_t* counts, int32_t cap, int32_t* nlevels) {
  API_TRY
  if (!A) fail(QT_EINVAL, "NULL matrix");
  QT_CUDA(cudaSetDevice(A->ctx->device));
  ensure_levels(A);
  const int top = A->ubs == 64 ? A->L - 1 : A->ubs == 16 ? A->L + 1 : A->L;  // the caller's block level
  const int pad = pad_levels(A);  // chain levels above the paper's root (not reported)
  if (nlevels) *nlevels = top + 1 - pad;
  for (int l = pad; l <= top && l - pad < cap; ++l) counts[l - pad] = l <= A->L ? A->cnt[l] : A->nb16;
  API_CATCH
}

qt_status qt_read_back(qt_mat A, int32_t* brow, int32_t* bcol, void* values) {
  API_TRY
  resolve(A);
  if (!A) fail(QT_EINVAL, "NULL matrix");
  QT_CUDA(cudaSetDevice(A->ctx->device));
  read_back(A, brow, bcol, values);
  API_CATCH
}

qt_status qt_gather(qt_mat A, int32_t root, int32_t* brow, int32_t* bcol, void* values, int64_t* total) {
  API_TRY
  resolve(A);
  if (!A) fail(QT_EINVAL, "NULL matrix");
  qt_ctx ctx = A->ctx;
  if (root < 0 || root >= ctx->world) fail(QT_EINVAL, "root %d outside [0,%d)", root, ctx->world);
  QT_CUDA(cudaSetDevice(ctx->device));
  int64_t N;
  if (ctx->world == 1) {
    N = user_nblocks(A);
    if (brow || bcol || values) read_back(A, brow, bcol, values);
  } else {
    N = gather_dist(A, root, ctx->rank == root ? brow : nullptr, ctx->rank == root ? bcol : nullptr,
                    ctx->rank == root ? values : nullptr);
  }
  if (total) *total = N;
  API_CATCH
}

qt_status qt_read_back_async(qt_mat A, int32_t* brow, int32_t* bcol, void* values) {
  API_TRY
  resolve(A);
  if (!A) fail(QT_EINVAL, "NULL matrix");
  QT_CUDA(cudaSetDevice(A->ctx->device));
  read_back(A, brow, bcol, values, true);
  API_CATCH
}

qt_status qt_ctx_synchronize(qt_ctx ctx) {
  API_TRY
  if (!ctx) fail(QT_EINVAL, "NULL context");
  QT_CUDA(cudaSetDevice(ctx->device));
  QT_CUDA(cudaStreamSynchronize(ctx->stream));
  reap_pending(ctx, true);
  API_CATCH
}

qt_status qt_destroy(qt_mat A) {
  API_TRY
  if (!A) return QT_OK;
  cudaSetDevice(A->ctx->device);
  delete A;
  API_CATCH
}

qt_status qt_nccl_unique_id(void* out128) {
  API_TRY
  if (!out128) fail(QT_EINVAL, "out128 is NULL");
  nccl_unique_id(out128);
  API_CATCH
}

// ------------------------------------------------------------ row-strip plan (a3)

qt_status qt_plan_strips(qt_ctx ctx, int64_t n, int32_t block_size, int32_t align_rows, int64_t nb_a,
                         const int32_t* a_brow, const int32_t* a_bcol, int64_t nb_b, const int32_t* b_brow,
                         int32_t parts, int32_t* bounds, int64_t* strip_products) {
  API_TRY
  if (!bounds) fail(QT_EINVAL, "bounds is NULL");
  if (block_size != 16 && block_size != 32 && block_size != 64) fail(QT_EINVAL, "block_size %d", block_size);
  if (n <= 0 || n % block_size != 0) fail(QT_EINVAL, "n=%lld must be a positive multiple of block_size",
                                          (long long)n);
  if (parts < 1) fail(QT_EINVAL, "parts=%d", parts);
  if (align_rows < 1) fail(QT_EINVAL, "align_rows=%d", align_rows);
  if ((nb_a > 0 && (!a_brow || !a_bcol)) || (nb_b > 0 && !b_brow) || nb_a < 0 || nb_b < 0)
    fail(QT_EINVAL, "NULL or negative block arrays");
  const int64_t nbr = n / block_size;
  if (nbr > (1ll << 22)) fail(QT_EINVAL, "too many block rows");
  // B's blocks per row, then products per C row: prod(I) = sum over A(I,K) of nnz(B(K,:))
  std::vector<int64_t> rowB(nbr, 0), prod(nbr, 0);
  for (int64_t t = 0; t < nb_b; ++t) {
    const int32_t r = b_brow[t];
    if (r < 0 || r >= nbr) fail(QT_ERANGE, "B block %lld: brow=%d outside [0,%lld)", (long long)t, r, (long long)nbr);
    ++rowB[r];
  }
  const bool multi = ctx && ctx->world > 1;
  if (multi) {  // every rank passed its own blocks: sum the row counts over ranks
    std::vector<int64_t> all((size_t)nbr * ctx->world);
    allgather_i64(ctx, rowB.data(), all.data(), (int)nbr);
    for (int64_t r = 0; r < nbr; ++r) {
      int64_t v = 0;
      for (int q = 0; q < ctx->world; ++q) v += all[(size_t)q * nbr + r];
      rowB[r] = v;
    }
  }
  for (int64_t t = 0; t < nb_a; ++t) {
    const int32_t r = a_brow[t], c = a_bcol[t];
    if (r < 0 || r >= nbr || c < 0 || c >= nbr)
      fail(QT_ERANGE, "A block %lld at (brow=%d, bcol=%d) outside [0,%lld)", (long long)t, r, c, (long long)nbr);
    prod[r] += rowB[c];
  }
  if (multi) {
    std::vector<int64_t> all((size_t)nbr * ctx->world);
    allgather_i64(ctx, prod.data(), all.data(), (int)nbr);
    for (int64_t r = 0; r < nbr; ++r) {
      int64_t v = 0;
      for (int q = 0; q < ctx->world; ++q) v += all[(size_t)q * nbr + r];
      prod[r] = v;
    }
  }
  // chunks of align_rows rows; contiguous partition into `parts` strips
  // minimising the largest strip (binary search on the bound, greedy packing
  // from the top; every rank computes the same boundaries)
  const int64_t nch = (nbr + align_rows - 1) / align_rows;
  std::vector<int64_t> w(nch, 0);
  for (int64_t r = 0; r < nbr; ++r) w[r / align_rows] += prod[r];
  int64_t lo = 0, hi = 0;
  for (int64_t c = 0; c < nch; ++c) {
    lo = std::max(lo, w[c]);
    hi += w[c];
  }
  auto strips_for = [&](int64_t cap) {
    int64_t cnt = 1, cur = 0;
    for (int64_t c = 0; c < nch; ++c) {
      if (cur + w[c] > cap) {
        ++cnt;
        cur = 0;
      }
      cur += w[c];
    }
    return cnt;
  };
  while (lo < hi) {
    const int64_t mid = lo + (hi - lo) / 2;
    if (strips_for(mid) <= parts) hi = mid;
    else lo = mid + 1;
  }
  // boundaries of the greedy packing at the optimal bound; unused strips are empty at the end
  std::vector<int32_t> b(parts + 1, (int32_t)nbr);
  b[0] = 0;
  {
    int g = 1;
    int64_t cur = 0;
    for (int64_t c = 0; c < nch; ++c) {
      if (cur + w[c] > lo && g < parts) {
        b[g++] = (int32_t)std::min<int64_t>(c * align_rows, nbr);
        cur = 0;
      }
      cur += w[c];
    }
  }
  for (int g = 0; g <= parts; ++g) bounds[g] = b[g];
  if (strip_products) {
    for (int g = 0; g < parts; ++g) {
      int64_t v = 0;
      for (int64_t r = b[g]; r < b[g + 1]; ++r) v += prod[r];
      strip_products[g] = v;
    }
  }
  API_CATCH
}

qt_status qt_symm_square_virtual(qt_mat A, int32_t P, int32_t g, const int32_t* row_bounds, qt_mat* C,
                                 qt_stats* st) {
  API_TRY
  resolve(A);
  if (!A || !C || !row_bounds) fail(QT_EINVAL, "NULL argument");
  *C = nullptr;
  if (A->ctx->world != 1) fail(QT_ESTATE, "virtual ranks need a single-rank context");
  if (A->ubs == 64) fail(QT_EBS, "the multi-rank symmetric square needs block_size 16 or 32");
  if (P < 1 || g < 0 || g >= P) fail(QT_EINVAL, "bad P=%d / g=%d", P, g);
  std::vector<int32_t> b(P + 1);
  for (int q = 0; q <= P; ++q) {  // caller's block rows -> 32-rows
    if (A->ubs == 16 && (row_bounds[q] & 1)) fail(QT_EINVAL, "block_size 16: row_bounds must be even");
    b[q] = rows_to_internal(row_bounds[q], A->ubs);
  }
  if (b[0] != 0 || b[P] != A->nbr)
    fail(QT_EINVAL, "row_bounds must span [0,%d]", rows_to_user(A->nbr, A->ubs));
  for (int q = 0; q < P; ++q)
    if (b[q + 1] < b[q]) fail(QT_EINVAL, "row_bounds not non-decreasing");
  qt_ctx ctx = A->ctx;
  QT_CUDA(cudaSetDevice(ctx->device));
  if (A->ubs == 16) {
    check_upper16(A);
    if (!A->sym16) A->sym16.reset(symm_prepare16(A));
  } else {
    check_upper(A);
  }
  qt_stats local;
  qt_stats& S = st ? *st : local;
  memset(&S, 0, sizeof(S));
  QT_CUDA(cudaEventRecord(ctx->ev[0], ctx->stream));
  qt_mat R = symm_square_virtual(A->ubs == 16 ? A->sym16.get() : A, b.data(), P, g, &S);
  QT_CUDA(cudaEventRecord(ctx->ev[1], ctx->stream));
  QT_CUDA(cudaEventSynchronize(ctx->ev[1]));
  QT_CUDA(cudaEventElapsedTime(&S.ms_total, ctx->ev[0], ctx->ev[1]));
  R->global_nb = user_nblocks(R);
  R->bounds = b;
  user_stats(R, S);
  *C = R;
  API_CATCH
}

qt_status qt_multiply_virtual(qt_mat A, qt_mat B, int32_t P, int32_t g, const int32_t* row_bounds,
                              qt_mat* C, qt_stats* st) {
  API_TRY
  resolve(A);
  resolve(B);
  if (!A || !B || !C || !row_bounds) fail(QT_EINVAL, "NULL argument");
  *C = nullptr;
  if (A->ctx != B->ctx) fail(QT_ESTATE, "A and B belong to different contexts");
  if (A->ctx->world != 1) fail(QT_ESTATE, "virtual ranks need a single-rank context");
  if (A->n != B->n) fail(QT_EDIM, "dimension mismatch");
  if (A->leaf_dim != B->leaf_dim || A->bs != B->bs) fail(QT_EBS, "leaf_dim/block_size mismatch");
  if (A->dtype != B->dtype) fail(QT_EDTYPE, "dtype mismatch");
  if (P < 1 || g < 0 || g >= P) fail(QT_EINVAL, "bad P=%d / g=%d", P, g);
  if (A->ubs != B->ubs) fail(QT_EBS, "block_size mismatch");
  std::vector<int32_t> b32(P + 1);
  for (int q = 0; q <= P; ++q) {  // caller's block rows -> 32-rows
    if (A->ubs == 16 && (row_bounds[q] & 1)) fail(QT_EINVAL, "block_size 16: row_bounds must be even");
    b32[q] = rows_to_internal(row_bounds[q], A->ubs);
  }
  if (b32[0] != 0 || b32[P] != A->nbr)
    fail(QT_EINVAL, "row_bounds must span [0,%d]", rows_to_user(A->nbr, A->ubs));
  for (int q = 0; q < P; ++q)
    if (b32[q + 1] < b32[q]) fail(QT_EINVAL, "row_bounds not non-decreasing");
  qt_ctx ctx = A->ctx;
  QT_CUDA(cudaSetDevice(ctx->device));
  qt_stats local;
  qt_stats& S = st ? *st : local;
  memset(&S, 0, sizeof(S));
  QT_CUDA(cudaEventRecord(ctx->ev[0], ctx->stream));
  qt_mat R = multiply_virtual(A, B, b32.data(), P, g, &S);
  QT_CUDA(cudaEventRecord(ctx->ev[1], ctx->stream));
  QT_CUDA(cudaEventSynchronize(ctx->ev[1]));
  QT_CUDA(cudaEventElapsedTime(&S.ms_total, ctx->ev[0], ctx->ev[1]));
  R->global_nb = user_nblocks(R);
  R->bounds = b32;
  user_stats(R, S);
  *C = R;
  API_CATCH
}

int64_t qt_kernel_launches(qt_ctx ctx) { return ctx ? ctx->launches : 0; }

qt_status qt_fp64_peak(qt_ctx ctx, int kind, float ms, double* flops) {
  API_TRY
  if (!ctx || !flops || (kind != 0 && kind != 1)) fail(QT_EINVAL, "bad arguments");
  QT_CUDA(cudaSetDevice(ctx->device));
  const int grid = ctx->num_sms * 2, threads = 256;
  // calibrate: a short run, then one sized to `ms`
  int iters = 256;
  float t = 0;
  for (int rep = 0; rep < 2; ++rep) {
    launch_fp64_peak(ctx, kind, 16, grid);  // warm
    QT_CUDA(cudaEventRecord(ctx->ev[5], ctx->stream));
    launch_fp64_peak(ctx, kind, iters, grid);
    QT_CUDA(cudaEventRecord(ctx->ev[6], ctx->stream));
    QT_CUDA(cudaEventSynchronize(ctx->ev[6]));
    QT_CUDA(cudaEventElapsedTime(&t, ctx->ev[5], ctx->ev[6]));
    if (rep == 0) iters = std::max(16, (int)(iters * (ms / std::max(t, 1e-3f))));
  }
  double fl = kind == 0 ? (double)grid * (threads / 32) * iters * 16 * 512
                        : (double)grid * threads * iters * 4 * 8 * 2;
  *flops = fl / (t * 1e-3);
  API_CATCH
}

}  // extern "C"
