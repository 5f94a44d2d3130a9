// Internal declarations of libqtmm (not part of the ABI).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdarg>
#include <cstdio>
#include <stdexcept>
#include <string>
#include <memory>
#include <vector>

#include "../../include/qt.h"

namespace qt {

// ----------------------------------------------------------------- errors

struct Error : std::runtime_error {
  qt_status status;
  Error(qt_status s, const std::string& m) : std::runtime_error(m), status(s) {}
};

[[noreturn]] void fail(qt_status s, const char* fmt, ...);

#define QT_CUDA(x)                                                                  \
  do {                                                                              \
    cudaError_t e_ = (x);                                                           \
    if (e_ != cudaSuccess)                                                          \
      ::qt::fail(e_ == cudaErrorMemoryAllocation ? QT_ENOMEM : QT_ECUDA, "%s:%d %s: %s", \
                 __FILE__, __LINE__, #x, cudaGetErrorString(e_));                   \
  } while (0)

#define QT_LAUNCH_CHECK(ctx)                                                        \
  do {                                                                              \
    (ctx)->launches++;                                                              \
    cudaError_t e_ = cudaGetLastError();                                            \
    if (e_ != cudaSuccess)                                                          \
      ::qt::fail(QT_ECUDA, "%s:%d kernel launch: %s", __FILE__, __LINE__,          \
                 cudaGetErrorString(e_));                                           \
  } while (0)

// ----------------------------------------------------------------- memory

// Device memory: a caching allocator per CUDA stream.  Every kernel of a
// context runs on its one stream, so a block freed on that stream can be handed
// to the next allocation on the same stream with no synchronisation (stream
// order guarantees the previous user is done).  Sizes are rounded to classes
// (powers of two below 1 MiB, multiples of 2 MiB above) and matched exactly;
// misses call cudaMalloc, and on out-of-memory the caches are flushed and the
// allocation retried.  In steady state (repeated multiplies) no CUDA allocator
// call happens at all.
// Free lists are keyed by (device, stream); `dev` is the current device at
// allocation time (every entry point sets its context's device first).
void* cache_alloc(size_t bytes, cudaStream_t s, int dev, size_t* granted);
void cache_free(void* p, size_t granted, cudaStream_t s, int dev);
void cache_release_stream(cudaStream_t s, int dev);
int cache_device();

struct DevBuf {
  void* p = nullptr;
  size_t bytes = 0;
  size_t granted = 0;
  cudaStream_t s = nullptr;
  int dev = 0;
  DevBuf() = default;
  DevBuf(size_t b, cudaStream_t st) { alloc(b, st); }
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  DevBuf(DevBuf&& o) noexcept : p(o.p), bytes(o.bytes), granted(o.granted), s(o.s), dev(o.dev) {
    o.p = nullptr;
    o.bytes = o.granted = 0;
  }
  DevBuf& operator=(DevBuf&& o) noexcept {
    if (this != &o) {
      release();
      p = o.p;
      bytes = o.bytes;
      granted = o.granted;
      s = o.s;
      dev = o.dev;
      o.p = nullptr;
      o.bytes = o.granted = 0;
    }
    return *this;
  }
  ~DevBuf() { release(); }
  void alloc(size_t b, cudaStream_t st) {
    release();
    s = st;
    bytes = b;
    if (b == 0) return;
    dev = cache_device();
    p = cache_alloc(b, st, dev, &granted);
  }
  void release() {
    if (p) cache_free(p, granted, s, dev);
    p = nullptr;
    bytes = granted = 0;
  }
  template <class T> T* as() const { return static_cast<T*>(p); }
};

// ----------------------------------------------------------------- handles

struct NcclApi;  // dynamically loaded NCCL entry points (qt_dist.cu)

}  // namespace qt

struct qt_ctx_s {
  int device = 0;
  cudaStream_t stream = nullptr;
  int rank = 0, world = 1;
  void* transport = nullptr;  // qt::Transport (NCCL or loopback), world > 1
  int num_sms = 148;
  int64_t launches = 0;
  cudaEvent_t ev[8] = {};
  qt::DevBuf scratch;  // cub temp storage, grown on demand
  qt::DevBuf counters; // small device counters (scheduler, errors)
  qt::DevBuf zeros;    // one zero block (8 KiB) for absent tcgen05 operands
  void* pinned = nullptr;  // small pinned host staging area
  size_t pinned_bytes = 0;
  // mapped pinned buffer of read_small: small device-to-host reads written by a
  // kernel, not a copy-engine memcpy (which would queue behind a bulk
  // qt_read_back_async copy in flight on the same engine)
  void* small_host = nullptr;
  static constexpr size_t kSmallHostBytes = 256 << 10;
  cudaStream_t copy_stream = nullptr;  // device-to-host copies of qt_read_back_async
  cudaStream_t h2d_stream = nullptr;   // host-to-device value copies of qt_create
  cudaEvent_t h2d_done = nullptr;
  cudaStream_t comm_stream = nullptr;  // multi-rank: payload exchange + the remote tiles' numeric launch
  cudaEvent_t ov_ev[4] = {};           // overlap ordering (0, 1) and payload timing (2, 3)
  bool async_multiply = false;         // qt_multiply_async: no final synchronisation
  bool timing = true;                  // qt_ctx_set_timing: CUDA-event phase timings in qt_stats
  // sync-free qt_multiply_async (small products): the BFS's level counts of a
  // product still in flight land in a pinned ring slot; the product's block
  // count is read on first use (qt::resolve)
  static constexpr int kPendRing = 32;
  int32_t* pend_host = nullptr;        // [kPendRing][128] pinned
  cudaEvent_t pend_ev[kPendRing] = {};
  qt_mat_s* pend_owner[kPendRing] = {};
  int pend_next = 0;
  struct PendingCopy {
    cudaEvent_t done;
    qt::DevBuf bufs[3];  // staging buffers, released when `done` has completed
  };
  std::vector<PendingCopy*> pending;
};

struct qt_mat_s {
  qt_ctx ctx = nullptr;
  int64_t n = 0;
  int32_t leaf_dim = 0, bs = 0;  // bs: the internal block size (32)
  int32_t ubs = 32;    // the caller's block size: 32; 64 = stored as 2x2 quads of 32-blocks;
                       // 16 = held as the quadrants of 32-blocks (qt_bs16.cu)
  qt_dtype dtype = QT_F64;
  int L = 1;           // levels above the block level; level L = blocks
  int leaf_level = 0;
  int32_t nbr = 0;     // block rows (= block cols) of the matrix
  int64_t nb = 0;      // local blocks
  int64_t global_nb = 0;
  int32_t row_lo = 0, row_hi = 0;
  std::vector<int32_t> bounds;  // world+1 block-row boundaries
  qt::DevBuf key;      // uint64 [nb] Morton keys, ascending
  qt::DevBuf pool;     // [nb][bs*bs] values in the internal (swizzled) layout
  std::vector<int64_t> cnt;     // non-NIL nodes per level, l = 0..L (cnt[L] = nb)
  std::vector<qt::DevBuf> child; // child[l] : int32 [cnt[l]][4], l = 0..L-1 (-1 = NIL)
  bool levels_built = true;     // false for a fresh product: built on first use
  qt::DevBuf hist;     // int32 per-level node counts per row / per column (see build_levels)
  // dense Morton-indexed node maps of the top levels: int32 [kDenseNodes],
  // level l (l <= 4, l < L) at offset (4^l - 1) / 3, entry = node index or -1
  // (the symbolic pass's dense start reads the tasks of level l0 off them)
  qt::DevBuf dmap;
  static constexpr int kDenseLevels = 4, kDenseNodes = 341;
  std::vector<int32_t> hist_host;  // host copy of hist (per-level task counts without a sync)
  std::vector<qt::DevBuf> norm2;  // squared Frobenius norms per node, levels 0..L (screening; lazy)
  qt::DevBuf norm16;   // ubs == 16 screening: squared norms of the 16-blocks, double [nb][4] (0 if absent; lazy)
  qt::DevBuf rm_inv;   // pool index -> position in row-major (brow, bcol) order (qt_update_values; lazy)
  qt::DevBuf sub;      // ubs == 16: uint8 [nb] quadrant occupancy (bit 2i+j), indexed like the pool
  int64_t nb16 = 0;    // ubs == 16: the caller's blocks (set quadrants)
  // ubs == 16 symmetric square: the copy with completed diagonal containers
  // (symm_prepare16), made on the first call and kept (values never change
  // in place at bs 16: qt_update_values is bs 32 only)
  std::unique_ptr<qt_mat_s> sym16;
  // symmetric square: U^T's block pool (blocks read transposed), made on the
  // first call and kept with the immutable handle; poolT_src = the pool it was
  // made from (qt_update_values drops it)
  qt::DevBuf poolT_cache;
  const void* poolT_src = nullptr;
  // FP32 matrix: its FP64 copy for the products that run on the FP64 kernel
  // (readings C-29, C-30), made on first use and kept (qt_update_values drops it)
  std::unique_ptr<qt_mat_s> f64_copy;
  // B_ext of a multi-rank multiply: pool1 overrides pool.p (a borrowed view of
  // the local pool); block ids >= split live in pool2 (the received blocks).
  const void* pool1 = nullptr;
  const void* pool2 = nullptr;
  int64_t split = INT64_MAX;
  // a sync-free async product whose block count is still on its way (the
  // context's ring slot), or -1; nb is the BFS's upper bound until resolved
  int pend_slot = -1;
  ~qt_mat_s();
  const void* pool_ptr() const { return pool1 ? pool1 : pool.p; }
};

namespace qt {

inline size_t elem_size(qt_dtype d) { return d == QT_F64 ? 8 : 4; }

// memory kind of a pointer
bool is_device_ptr(const void* p);

// cub temp storage of at least `bytes` on the ctx
void* scratch(qt_ctx ctx, size_t bytes);

// Read `bytes` of device memory into host memory `dst` on the ctx stream and
// wait for it: a kernel stores them into the context's mapped pinned buffer
// (chunks of kSmallHostBytes), so the read never waits for a copy engine
// busy with a bulk transfer.
void read_small(qt_ctx ctx, void* dst, const void* src, size_t bytes);
template <class T>
T read_scalar(qt_ctx ctx, const T* d) {
  T h;
  read_small(ctx, &h, d, sizeof(T));
  return h;
}

// ----- kernels / host drivers (qt_tree.cu)
// keys from coordinates; validation; sort; duplicate check; swizzled pool fill.
void build_from_blocks(qt_mat M, int64_t nb, const int32_t* d_brow, const int32_t* d_bcol,
                       const void* d_vals, int32_t row_lo, int32_t row_hi);
// build levels L-1..0 from the sorted block keys in M->key.  leaf_ids (device,
// optional): the pool index of each sorted block, stored in the level L-1
// child table instead of the sorted position (used by the merged B_ext).
void build_levels(qt_mat M, const int32_t* leaf_ids = nullptr);
// a product of a sync-free qt_multiply_async: wait for its level counts and
// set its block count (every entry point does this before reading nb)
void resolve_pending(qt_mat M);
inline void resolve(qt_mat M) {
  if (M && M->pend_slot >= 0) resolve_pending(M);
}
inline void ensure_levels(qt_mat M) {
  resolve(M);
  if (!M->levels_built) { build_levels(M); M->levels_built = true; }
}
// QT_EINVAL unless every (caller-size) block has brow <= bcol (upper block triangle)
void check_upper(qt_mat M);
// 64-block matrix without the (1,0) 32-sub-blocks of its diagonal 64-blocks
qt_mat upper32_view(qt_mat M);
// row-major (brow, bcol) order and un-swizzle into caller buffers (caller's block size)
void read_back(qt_mat M, int32_t* brow, int32_t* bcol, void* vals, bool async = false);
void reap_pending(qt_ctx ctx, bool wait);
// new values for M's blocks, given in read-back (row-major brow, bcol) order, host or device
void update_values(qt_mat M, const void* values);
// 64-blocks (2x2 quads of 32-blocks): split inputs / user-level block count
void split64(qt_ctx ctx, qt_dtype dt, int64_t nb, const int32_t* brow, const int32_t* bcol,
             const void* vals, DevBuf& obrow, DevBuf& obcol, DevBuf& ovals);
inline int64_t user_nblocks(qt_mat M) { return M->ubs == 64 ? M->nb / 4 : M->ubs == 16 ? M->nb16 : M->nb; }
// the caller's block rows -> internal 32-block rows (16: must be even)
inline int32_t rows_to_internal(int32_t r, int ubs) { return ubs == 64 ? 2 * r : ubs == 16 ? r / 2 : r; }
inline int32_t rows_to_user(int32_t r, int ubs) { return ubs == 64 ? r / 2 : ubs == 16 ? 2 * r : r; }
// block size 16 (qt_bs16.cu)
void build_from_blocks16(qt_mat M, int64_t n, const int32_t* brow, const int32_t* bcol, const void* vals,
                         int32_t lo16, int32_t hi16);
void read_back16(qt_mat M, int32_t* brow, int32_t* bcol, void* vals);
void truncate_terms16(qt_mat A, DevBuf& nrm, DevBuf& rm);
qt_mat apply_keep16(qt_mat A, const uint8_t* keep_user);
int64_t compact_sub16(qt_ctx ctx, const uint8_t* keep, const int32_t* incl, const uint8_t* in, int64_t n,
                      int64_t kept, DevBuf& out);
// C's quadrant masks from the level L-1 task list; out = {16-block products, C 16-blocks, empty
// containers, non-NIL container pairs (the level-L task count)}
void cmask16(qt_ctx ctx, int64_t ntiles, const int32_t* ts, const int32_t* pa, const int32_t* pb, const int4* cA,
             const int4* cB, const int4* cC, const uint8_t* subA, const uint8_t* subB, int trans,
             const uint64_t* keyC, uint8_t* subC, int64_t nc, int64_t out[4], const double* n16A = nullptr,
             const double* n16B = nullptr, double tau2 = 0.0);
qt_mat drop_empty16(qt_mat C);
// symmetric square at bs 16: upper-storage check, U with completed diagonal
// containers, and C's lower quadrants of diagonal containers removed
void check_upper16(qt_mat M);
qt_mat symm_prepare16(qt_mat U);
void symm_finish16(qt_mat C);
// keep flags per user block -> per internal block
void expand_keep(qt_mat M, const uint8_t* keep_user, DevBuf& keep32);
// truncate (reading C-16): local terms, global decision, single-rank driver
void truncate_terms(qt_mat A, DevBuf& nrm, DevBuf& rm);
void truncate_decide(qt_ctx ctx, const double* nrm_all, const uint64_t* rm_all, const int64_t* id_all,
                     int64_t n_all, double tau2, int me, uint8_t* keep_local);
qt_mat truncate(qt_mat A, double tau);
qt_mat truncate_dist(qt_mat A, double tau);
// the same matrix with its values converted to `to` (FP32 <-> FP64; plain matrices)
qt_mat convert_dtype(qt_mat A, qt_dtype to);
// an FP32 matrix's FP64 copy, kept with the handle
inline qt_mat f64_of(qt_mat A) {
  if (!A->f64_copy) A->f64_copy.reset(convert_dtype(A, QT_F64));
  return A->f64_copy.get();
}
// copy `keep` flagged blocks (Morton order preserved) of A into a new matrix
qt_mat select_blocks(qt_mat A, const uint8_t* d_keep);

// ----- symbolic + numeric multiply (qt_symbolic.cu, qt_numeric.cu)
// trans: bit 0 = op(A) = A^T, bit 1 = op(B) = B^T  (C = op(A) op(B)),
// bit 2 = symmetric square, bits 8+ = its pruning depth.  tau >= 0: norm
// screening (block products with ||A_ik||*||B_kj|| < tau are skipped).
// Multi-rank overlap of the payload exchange with the numeric kernel
// (SURVEY §8(a) a4, §8(e)): when B is a B_ext with received blocks (ids >=
// B->split), the C tiles whose products read only local B blocks run on the
// ctx stream while the payload is still in flight; the other tiles are
// launched on `s2` behind the exchange (whatever was enqueued on s2 before the
// call) and the ctx stream joins s2 at the end.
struct Overlap {
  cudaStream_t s2 = nullptr;
  int64_t tiles_local = 0, tiles_remote = 0;  // out: C tiles per phase
};
// [row_lo, row_hi): only C blocks in these block rows are computed (the BFS
// prunes C nodes outside the window at every level).
struct NumericPlan;
// multiply tasks per level 0..L from the occupancy histograms (exact for
// regular products, an upper bound for the symmetric square)
std::vector<int64_t> level_task_bounds(qt_mat A, qt_mat B, int trans);
// out_f32: FP64 operands, C stored as FP32 by the FP64 kernel's epilogue (the
// FP32 products that run on the FP64 kernel, reading C-30)
qt_mat multiply_local(qt_mat A, qt_mat B, qt_stats* st, float* ms_sym, float* ms_num, int trans = 0,
                      double tau = -1.0, Overlap* ov = nullptr, int32_t row_lo = 0,
                      int32_t row_hi = INT32_MAX, NumericPlan* plan = nullptr, bool out_f32 = false);
// Tiles (C nodes of one level with CSR task ranges `ts` over the task array
// pb) partitioned on the device: map[0, *nsel) = the tiles whose B nodes hold
// only block ids < splitB (Morton order), map[*nsel, ntiles) = the rest.
// childB_t: B's child table at the tiles' level; childB_1: B's level L-1 table
// when the tiles sit at level L-2 (FP32), else null.  No host sync.
void split_tiles(qt_ctx ctx, int64_t ntiles, const int32_t* ts, const int32_t* pb, const int4* childB_t,
                 const int4* childB_1, int64_t splitB, int32_t* map, int32_t* nsel);
// squared Frobenius norms of every quadtree node (levels 0..L) into M->norm2;
// block size 16: also the 16-blocks' (M->norm16), a container's = the sum of its quadrants'
void ensure_norms(qt_mat M);

struct NumericArgs {
  int64_t ntiles;            // C nodes at level L-1
  const int32_t* tile_start; // [ntiles+1] pair ranges
  const int32_t* pa;         // A node (level L-1) per pair
  const int32_t* pb;         // B node (level L-1) per pair
  const int4* childA;        // A child table at level L-1 (block indices)
  const int4* childB;
  const int4* childC;        // C child table at level L-1 (C block indices)
  const void* poolA;
  const void* poolB;
  const void* poolB2;        // remote pool for B blocks >= splitB (or null)
  int64_t splitB;
  void* poolC;
  int* counter;              // tile scheduler counter (zeroed before launch)
  int group = 1;             // tiles per scheduler grab (1..31)
  int split = 0;             // 1: work item = (tile, C child q), ntiles = 4 x tiles (few-tile problems)
  int trans = 0;             // bit 0: A transposed, bit 1: B transposed, bit 2: symmetric square
  const void* poolT = nullptr;    // symmetric square: transposed copy of poolA (= poolB)
  const double* normA = nullptr;  // block squared norms (screening) or null
  const double* normB = nullptr;
  double tau2 = 0.0;
  const uint8_t* subA = nullptr;  // block size 16: quadrant masks (products whose quadrants never meet are skipped)
  const uint8_t* subB = nullptr;
  const double* norm16A = nullptr;  // block size 16 + screening: squared 16-block norms [nb][4]
  const double* norm16B = nullptr;
  cudaStream_t stream = nullptr;  // launch stream (null: the ctx stream)
  // overlap phases (split_tiles): phase 1 = tiles map[0, *nsel), phase 2 =
  // map[*nsel, ntiles); 0 = all tiles in order (tile_map unused).  group == 1.
  int phase = 0;
  const int32_t* tile_map = nullptr;
  const int32_t* nsel = nullptr;
  // sync-free multiply: the actual tile count on the device (ntiles is then an
  // upper bound used for the launch shape only)
  const int32_t* ntiles_dev = nullptr;
  bool counter_ready = false;  // the scheduler counter is already zero (no memset before the launch)
  unsigned long long* prof = nullptr;  // QT_NUM_PROF diagnostics (instrumented instantiation only)
  int out_f32 = 0;             // C pool is FP32 (swz32 layout): the epilogue rounds to nearest
};
void launch_numeric(qt_ctx ctx, qt_dtype dt, const NumericArgs& a);
void launch_transpose_blocks(qt_ctx ctx, const void* in, void* out, int64_t nb);
void launch_transpose_blocks_f32(qt_ctx ctx, const void* in, void* out, int64_t nb);

// FP32 (tcgen05 kind::tf32, 3xTF32): tiles are C nodes at level L-2 (4x4 blocks)
struct NumericArgs32 {
  int64_t ntiles;            // C nodes at level L-2
  const int32_t* tile_start; // [ntiles+1] task ranges at level L-2
  const int32_t* pa;         // A node (level L-2) per task
  const int32_t* pb;         // B node (level L-2) per task
  const int4* childA2;       // A child tables at levels L-2 and L-1
  const int4* childA1;
  const int4* childB2;
  const int4* childB1;
  const int4* childC2;       // C child tables: level L-2 -> quads, level L-1 -> blocks
  const int4* childC1;
  const void* poolA;
  const void* poolB;
  const void* poolB2;
  int64_t splitB;
  void* poolC;
  const void* zeros;         // one zero block (absent operands)
  int* counter;
  int trans = 0;             // bit 0: A transposed, bit 1: B transposed, bit 2: symmetric square
  const void* poolT = nullptr;  // symmetric square: transposed copy of poolA (= poolB)
  cudaStream_t stream = nullptr;  // launch stream (null: the ctx stream)
  int phase = 0;                   // overlap phases, as in NumericArgs
  const int32_t* tile_map = nullptr;
  const int32_t* nsel = nullptr;
  bool counter_ready = false;      // as in NumericArgs
  const int32_t* ntiles_dev = nullptr;  // as in NumericArgs (sync-free products)
};
void launch_numeric_f32(qt_ctx ctx, const NumericArgs32& a);

// The numeric launch of a multiply kept for re-execution (qt_multiply_plan):
// its arguments and the symbolic pass's buffers the kernel reads.
struct NumericPlan {
  bool valid = false, f32 = false;
  NumericArgs na;
  NumericArgs32 nb;
  DevBuf keep[6];
  DevBuf poolT;                   // symmetric square: U^T's pool, refreshed on execute
  const void* tsrc = nullptr;
  int64_t tnb = 0;
};
void launch_fp64_peak(qt_ctx ctx, int kind, int iters, int grid);

// ----- distributed (qt_dist.cu)
void dist_init(qt_ctx ctx, const void* uid);
void dist_init_loopback(qt_ctx ctx, void* hub);
void* loop_hub_create(int P);
void loop_hub_destroy(void* hub);
void nccl_unique_id(void* out128);
void dist_finalize(qt_ctx ctx);
// ranks of the context's communicator; *kind = 0 none (world 1), 1 NCCL, 2 loopback
int transport_info(qt_ctx ctx, int* kind);
// tau >= 0: the norm-screened product (B_ext's norms from both of its pools)
qt_mat multiply_dist(qt_mat A, qt_mat B, qt_stats* st, double tau = -1.0);
// the same path for virtual rank g of P on one device (D2D copies stand in for
// the NCCL transfers); A and B are whole matrices on this context.
qt_mat multiply_virtual(qt_mat A, qt_mat B, const int32_t* bounds, int P, int g, qt_stats* st);
void allgather_i64(qt_ctx ctx, const int64_t* send_host, int64_t* recv_host, int count);
// multi-rank symmetric square (32-blocks): U's rows [row_lo, row_hi) on this
// rank; C = its rows of A^2, upper triangle.  The virtual form runs rank g of P
// on one device from the whole U.
qt_mat symm_square_dist(qt_mat U, qt_stats* st);
// every rank's blocks to `root` in (brow, bcol) order (collective); returns the total count
int64_t gather_dist(qt_mat A, int root, int32_t* brow, int32_t* bcol, void* vals);
qt_mat symm_square_virtual(qt_mat U, const int32_t* bounds, int P, int g, qt_stats* st);

}  // namespace qt
