/*
 * qt.h — C ABI of libqtmm: block-sparse quadtree matrix multiply on B200.
 *
 * The operation (arXiv 1501.07800, Rubensson & Rudberg; P:nnn = line of
 * /root/reference/PAPER.md):
 *   C = A*B for block-sparse matrices held as sparse quadtrees whose leaves
 *   are block-sparse submatrices (abstract; §3.1; §4.1
 *   P:350-357).  Zero submatrices are NIL at every level and every operation
 *   on them is skipped (§3.2).  C's block pattern is the structural
 *   product of A's and B's patterns (reading C-1): nothing is dropped
 *   numerically; only qt_truncate removes blocks.
 *
 * Conventions for every entry point:
 *   - All functions return qt_status; on failure qt_last_error() names the
 *     problem (thread-local string, valid until the next failing call on the
 *     same thread).  No function aborts the process.
 *   - Pointers are plain host or device pointers; the library detects which
 *     (cudaPointerGetAttributes).  Host pointers may be pageable or pinned.
 *   - Sizes are element counts unless named *_bytes.
 *   - Ownership: the library copies every input array before returning (the
 *     caller keeps its buffers).  Each qt_mat owns its device memory until
 *     qt_destroy.  qt_mat handles are immutable after creation (chunks are
 *     read-only after registration), so A and B may be the same
 *     handle (C = A*A).
 *   - All device work runs on the stream given to qt_ctx_create, in stream
 *     order.  Functions that must know a size on the host (qt_create,
 *     qt_multiply, qt_truncate, qt_read_back) synchronise that stream.
 *   - Multi-rank: one process per GPU, one qt_ctx per process.  Functions
 *     marked "collective" must be called by every rank in the same order.
 */
#ifndef QT_H_
#define QT_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  QT_OK = 0,
  QT_EINVAL = 1,  /* invalid argument (null handle, bad size, bs does not divide leaf_dim, ...) */
  QT_ERANGE = 2,  /* a block coordinate is outside [0, ceil(n/bs)) */
  QT_EDUP = 3,    /* the same (brow, bcol) is listed twice */
  QT_EDIM = 4,    /* operand dimensions differ */
  QT_EBS = 5,     /* operand leaf_dim or block_size differ */
  QT_EDTYPE = 6,  /* operand dtypes differ, or dtype unsupported */
  QT_ENOMEM = 7,  /* device allocation failed */
  QT_ECUDA = 8,   /* a CUDA runtime call failed (message kept) */
  QT_ENCCL = 9,   /* an NCCL call failed or NCCL could not be loaded */
  QT_ESTATE = 10  /* handles from different contexts, or context misuse */
} qt_status;

typedef enum { QT_F64 = 0, QT_F32 = 1 } qt_dtype;

typedef struct qt_ctx_s* qt_ctx;  /* device, stream, rank/world, NCCL communicator */
typedef struct qt_mat_s* qt_mat;  /* immutable matrix (the rank-local part when world > 1) */

#define QT_MAX_LEVELS 40

/* Statistics of one qt_multiply (the paper's instrumentation, §5, §6.3). */
typedef struct {
  int32_t nlevels;           /* L+1: levels 0 (root) .. L (blocks) */
  int32_t leaf_level;        /* the quadtree level of the leaf matrices */
  int64_t level_tasks[QT_MAX_LEVELS]; /* multiply tasks per level: (A-node, B-node)
                                         pairs with both non-NIL (C_l) */
  int64_t level_c_nodes[QT_MAX_LEVELS]; /* C nodes the BFS created per level (task
                                           groups; a group whose child products
                                           all vanish is later pruned as NIL) */
  int64_t block_products;    /* = level_tasks[L]; effective flops = 2*bs^3 each */
  int64_t c_blocks;          /* local C blocks */
  int64_t bytes_recv_payload; /* bytes of A/B block values received */
  int64_t bytes_recv_meta;   /* request/reply metadata received */
  int64_t bytes_sent_payload;
  int64_t bytes_sent_meta;
  int64_t blocks_recv;       /* remote B blocks received */
  float ms_exchange;         /* device time of the exchange phase (0 when world == 1) */
  float ms_symbolic;         /* device time of the symbolic BFS (a5-a7) */
  float ms_numeric;          /* device time of the numeric kernel (a8) */
  float ms_total;            /* device time of the whole call */
  /* multi-rank overlap (world > 1, on unless QT_OVERLAP=0): the payload is
   * exchanged on a second stream while the symbolic pass and the C tiles
   * that read only local B blocks run; the other tiles follow it */
  int64_t tiles_overlapped;  /* numeric tiles run while the payload was in flight */
  int64_t tiles_after;       /* numeric tiles launched behind the payload */
  float ms_payload;          /* device time of the payload transfer (comm stream) */
} qt_stats;

/* ------------------------------------------------------------------ context */

/* Create a context on CUDA device `device`.  `cuda_stream` is a cudaStream_t
 * (NULL = the legacy default stream).  `rank`/`world`: this process's rank
 * and the number of ranks.  `nccl_unique_id`: the 128-byte ncclUniqueId made
 * by qt_nccl_unique_id() on rank 0 and broadcast by the caller; required
 * when world > 1.  With world == 1 it may be NULL (no communicator) or a fresh
 * id: the context then builds a one-rank NCCL communicator (qt_ctx_info
 * reports it) — the NCCL binding exercised on a single GPU; multiplies take
 * the single-GPU path either way.  Collective when world > 1 (ncclCommInitRank).
 * Errors: QT_EINVAL (bad rank/world/device), QT_ECUDA, QT_ENCCL. */
qt_status qt_ctx_create(int device, void* cuda_stream, int rank, int world,
                        const void* nccl_unique_id, qt_ctx* out);
qt_status qt_ctx_destroy(qt_ctx ctx);

/* Describe a context: this process's rank, the world size it was created
 * with, and the number of ranks of the communicator the library actually
 * built (NCCL: ncclCommCount on the library's own communicator; loopback: the
 * hub's rank count; 1 when world == 1), and the transport kind (0 none, 1
 * NCCL, 2 loopback).  Any output pointer may be NULL.  Errors: QT_EINVAL,
 * QT_ENCCL. */
qt_status qt_ctx_info(qt_ctx ctx, int32_t* rank, int32_t* world, int32_t* comm_ranks, int32_t* transport);

/* Per-phase device timings of the multiply calls (qt_stats.ms_symbolic,
 * ms_numeric, ms_total), measured with CUDA events on the context's stream:
 * on (1, the default) or off (0).  Off skips the event records and the
 * elapsed-time queries — about 10 us of driver calls per blocking call, a
 * large share of a small product — and reports 0 for them; results and every
 * other statistic are unchanged, and a blocking call still returns with its
 * work complete.  (Measurement only: no passage of the paper.)
 * Errors: QT_EINVAL (NULL context). */
qt_status qt_ctx_set_timing(qt_ctx ctx, int32_t on);

/* Write a fresh 128-byte ncclUniqueId into `out128` (loads NCCL on demand).
 * Errors: QT_ENCCL when libnccl.so.2 cannot be loaded. */
qt_status qt_nccl_unique_id(void* out128);

/* ------------------------------------------------------------------ matrices */

/* Create a quadtree matrix of dimension n (the matrix-parameters chunk,
 * §3.1: n, leaf dimension, leaf block size) from `nblocks` dense
 * blocks.  Block t has block coordinates (brow[t], bcol[t]) and values
 * values[t*bs*bs .. (t+1)*bs*bs) in row-major order, of type `dtype`
 * (double for QT_F64, float for QT_F32).  brow, bcol, values may be host or
 * device pointers; order of blocks is arbitrary.  Zero submatrices are never
 * stored: only the listed blocks exist, a listed all-zero block is
 * kept (reading C-2).
 * The quadtree is uniform: 2^L x 2^L blocks with 2^L the smallest power of
 * two >= ceil(n/bs) — the matrix is split "as far as possible" into a uniform
 * block size per level — padded children are NIL (reading C-3);
 * the leaf level is L - log2(leaf_dim/bs) clipped at 0 (leaves are
 * block-sparse submatrices, §4.1).  (Internally the kernels need at least
 * 4x4 32-blocks: smaller matrices get a chain of single-child levels above
 * the root, which statistics and qt_level_nodes do not report.)
 * Requirements: block_size 16, 32 or 64 (the leaf block size; P:378-379
 * "16-64").  A 64x64 block is held internally as a 2x2 quad of 32x32 blocks —
 * the kernels' block size — so the quadtree simply continues one level below
 * the caller's blocks.  16x16 blocks are held as the quadrants of 32x32
 * "containers" with a 4-bit occupancy mask (DESIGN reading C-27): n and
 * leaf_dim must then be multiples of 32 and multi-rank row_bounds even.
 * Statistics, read-back, truncation and info are reported in the caller's
 * blocks.  leaf_dim a power-of-two multiple of max(block_size, 32),
 * n % max(block_size, 32) == 0 (reading C-4), nblocks >= 0 (0 gives the NIL
 * matrix).
 * Multi-rank (world > 1): collective; each rank passes the blocks of its own
 * block-row range.  `row_bounds` (host, world+1 non-decreasing block-row
 * boundaries, first 0 and last ceil(n/bs)) gives the ranges; NULL means equal
 * strips of ceil(nbr/world) rows.  A block outside the rank's range is
 * QT_ERANGE.  Ignored when world == 1.
 * Errors: QT_EINVAL, QT_ERANGE (names the block), QT_EDUP (names the block),
 * QT_EDTYPE, QT_ENOMEM, QT_ECUDA. */
qt_status qt_create(qt_ctx ctx, int64_t n, int32_t leaf_dim, int32_t block_size,
                    qt_dtype dtype, int64_t nblocks, const int32_t* brow,
                    const int32_t* bcol, const void* values,
                    const int32_t* row_bounds, qt_mat* out);

/* C = A*B (§3.2).  A and B must share ctx, n, leaf_dim, block_size
 * and dtype.  Runs the symbolic multiply (level-synchronous BFS over the two
 * quadtrees, skipping NIL children at every level, emitting per level the
 * compacted queue of (A-node, B-node) tasks grouped by C node), then the
 * numeric block-sparse multiply (each C block = sum over k ascending of
 * A(I,k)*B(k,J), accumulated in registers, no atomics).  The result is a new
 * handle; A and B are unchanged.  `st` may be NULL.
 * Precision: QT_F64 computes in FP64 (DMMA); QT_F32 in 3xTF32 on tcgen05
 * (reading C-9), or — a sparse product whose 4x4-block tensor-core tiles
 * would be mostly empty — on FP64 copies with the result rounded to FP32
 * (reading C-30).  The FP32 tiles multiply absent blocks as zeros, so FP32
 * inputs must be finite (an Inf/NaN would reach C blocks the sparse product
 * leaves finite); FP64 never combines a present block with an absent one.
 * Multi-rank: collective.  C gets A's block-row ranges; each rank receives
 * from the owners exactly the B block rows its A rows reference (NCCL
 * send/recv) and reports the bytes in `st`.
 * Errors: QT_EINVAL, QT_EDIM, QT_EBS, QT_EDTYPE, QT_ESTATE, QT_ENOMEM,
 * QT_ECUDA, QT_ENCCL. */
qt_status qt_multiply(qt_mat A, qt_mat B, qt_mat* C, qt_stats* st);

/* C = op(A) op(B) with op(X) = X (0) or X^T (1): the transposed multiply task
 * types C = A^T B, A B^T, A^T B^T of §3.2.  A transposed operand
 * is read through its own quadtree with the off-diagonal children swapped and
 * each block transposed on the fly (no copy).  Same requirements, statistics
 * and errors as qt_multiply; world > 1 supports only trans_a = trans_b = 0
 * (QT_EINVAL otherwise). */
qt_status qt_multiply_ex(qt_mat A, qt_mat B, int32_t trans_a, int32_t trans_b, qt_mat* C,
                         qt_stats* st);

/* Norm-screened product (the norm-annotated quadtree of P:1294-1299):
 * C~ = sum over block products with ||A(I,K)||_F * ||B(K,J)||_F >= tau of
 * A(I,K) B(K,J).  Every quadtree node carries its squared Frobenius norm (sum
 * of its blocks', computed once per matrix); the symbolic pass drops a task
 * (a, b) as soon as ||a||^2 ||b||^2 < tau^2 — exact with respect to the
 * block-level test, since a node's norm bounds its blocks' — and the numeric
 * kernel skips the same block products.  ||C - C~||_F <= sum of the skipped
 * ||A(I,K)|| ||B(K,J)||.  tau = 0 gives qt_multiply's result.  Squared block
 * norms are summed row-major with separate multiply/add roundings (the
 * oracle's order, so both take identical decisions).
 * Block size 16 (the paper screens its S^2 runs at block size 16):
 * the test is per 16-block product with 16-block norms; a container's norm
 * is the sum of its quadrants' (pruning above stays exact), and the consumer
 * warps skip the k-halves whose 16-block product fails.  block_products
 * counts the surviving 16-block products.
 * FP32 (reading C-29): the screened product runs on FP64 copies of A and B
 * (exact conversion) through the FP64 kernel and C is rounded to FP32 — a
 * tcgen05 tile MMA cannot skip single block products.
 * Multi-rank (collective): each rank fetches the B rows of the full product
 * (qt_multiply's exchange) and screens its own strip; C is bitwise the
 * single-rank screened product's rows.  Errors: QT_EINVAL (tau < 0), QT_EDIM,
 * QT_EBS (block_size 64), QT_EDTYPE, QT_ENOMEM, QT_ECUDA, QT_ENCCL. */
qt_status qt_multiply_screened(qt_mat A, qt_mat B, double tau, qt_mat* C, qt_stats* st);

/* Symmetric matrix square C = A^2 (§3.3): A is symmetric and given
 * by its upper block triangle (every block of A has brow <= bcol; a diagonal
 * block is a full bs x bs block, used as stored); C is returned the same way
 * — only its upper block triangle is computed (about half of the products of
 * the full multiply).  The symbolic pass walks the quadtree of the
 * full matrix through references into U (diagonal nodes expose their (0,1)
 * child transposed as (1,0); transposed nodes swap and transpose their
 * children) and prunes C nodes below the diagonal at every level; blocks
 * read transposed come from a transposed copy of U's block pool made once
 * per call.  FP64 or FP32 (A's dtype).  Block size 16 (the paper's S^2 runs,
 * P:926-935): the 32-containers of U are the upper triangle at container
 * granularity; a diagonal container's (1,0) 16-block is below the diagonal
 * (QT_EINVAL) and is filled in as (0,1)^T on a copy of U, C's diagonal
 * containers are computed whole and their (1,0) 16-blocks dropped
 * (DESIGN reading C-28); block_products counts 16-block products.
 * Multi-rank (world > 1, block_size 16 or 32; collective): each rank passes its
 * block rows of U (the bounds given at create time) and gets its block rows
 * of C, upper triangle.  Rank g receives from the others every block of U
 * that a product of its C rows reads, and no other — the rows and columns its
 * strip references above it, and the parts (columns >= its first row) of the
 * rows below it that reach into it (DESIGN reading C-26; bytes in `st`,
 * oracle.exchange_plan_symm) — and runs the
 * symmetric-square BFS on its blocks + the received ones, pruned to its rows.
 * At block size 16 the exchange moves 32-containers (completed diagonal
 * ones) + one mask byte each.
 * Errors: QT_EINVAL (a block below the diagonal), QT_EBS (world > 1 with
 * block_size 64), QT_ENOMEM, QT_ECUDA, QT_ENCCL. */
qt_status qt_symm_square(qt_mat A, qt_mat* C, qt_stats* st);

/* Frobenius-norm truncation (reading C-16): remove the longest
 * prefix of blocks, sorted ascending by Frobenius norm with ties broken by
 * (brow, bcol), whose accumulated squared norm is < tau^2, so that
 * ||A - out||_F < tau (or nothing removed).  tau >= 0.  New handle; A
 * unchanged.  Multi-rank: collective — the prefix is global: every rank sends
 * its (norm^2, brow, bcol) terms (24 bytes per block) to all others and all
 * ranks take the same decision; each keeps its surviving local blocks.
 * Errors: QT_EINVAL, QT_ENOMEM, QT_ECUDA, QT_ENCCL. */
qt_status qt_truncate(qt_mat A, double tau, qt_mat* out);

/* Describe a matrix (the matrix-parameters chunk of §3.1: dimension,
 * leaf dimension, block size; plus this rank's block counts and rows).  Any
 * output pointer may be NULL.  local_nblocks: blocks
 * held by this rank; global_nblocks: over all ranks for created and truncated
 * matrices — for the product of a multi-rank multiply it is the local count
 * (summing would cost the multiply a collective; qt_gather's `total` gives
 * the global count); row_lo/row_hi: this rank's block-row range. */
qt_status qt_info(qt_mat A, int64_t* n, int32_t* leaf_dim, int32_t* block_size,
                  qt_dtype* dtype, int64_t* local_nblocks, int64_t* global_nblocks,
                  int32_t* row_lo, int32_t* row_hi);

/* Per-level non-NIL node counts of the quadtree (levels 0..L), written to
 * `counts` (host, capacity `cap`); *nlevels receives L+1. */
qt_status qt_level_nodes(qt_mat A, int64_t* counts, int32_t cap, int32_t* nlevels);

/* Copy this rank's blocks out, sorted by (brow, bcol), values row-major per
 * block — the to_triplets read-back of SPEC S:149-157 at block granularity
 * (a block list instead of element triplets).  brow/bcol: local_nblocks int32 each; values: local_nblocks*bs*bs
 * elements of the matrix dtype.  Host or device pointers; any may be NULL
 * to skip it.  Synchronises the stream before returning.
 * Errors: QT_EINVAL, QT_ECUDA. */
qt_status qt_read_back(qt_mat A, int32_t* brow, int32_t* bcol, void* values);

/* qt_multiply without the final synchronisation on the numeric kernel
 * (single rank; a multi-rank context behaves as qt_multiply): C is returned
 * as soon as its blocks are allocated and the numeric kernel is enqueued on
 * the context stream, so the caller can already enqueue the next step (e.g.
 * qt_create from host, whose value copy runs on the context's H2D stream).
 * The st->ms_* timings are 0; everything else in st is filled, except for
 * small products (C's pool sized by the symbolic pass's upper bound, at most
 * QT_SYNCFREE_MB): these return without any host synchronisation — C's block
 * count is not known yet, st->c_blocks is -1 and st->level_c_nodes 0 — and
 * C's count is read when C is first used by any entry point (qt_info,
 * qt_read_back, as an operand, ...), so back-to-back multiplies pipeline on
 * the device.  A and B may be destroyed right after the call (stream-ordered
 * reuse).  QT_F32 products are routed as by qt_multiply (reading C-30; the
 * FP64 copies of the operands are made stream-ordered on first use).
 * Errors: as qt_multiply. */
qt_status qt_multiply_async(qt_mat A, qt_mat B, qt_mat* C, qt_stats* st);

/* Distributed read-back: collective over the context's ranks.
 * `root` receives every rank's blocks in (brow, bcol) order — the ranks own
 * contiguous block-row strips, so this is the order of the whole matrix —
 * into brow/bcol/values (caller block size, host or device; the other ranks'
 * pointers are ignored).  *total (all ranks, may be NULL) = the number of
 * blocks of the whole matrix.  Call once with NULL buffers on the root to
 * learn the size, then with buffers.  world == 1: qt_read_back.
 * Errors: QT_EINVAL (root), QT_ECUDA, QT_ENCCL. */
qt_status qt_gather(qt_mat A, int32_t root, int32_t* brow, int32_t* bcol, void* values, int64_t* total);

/* qt_read_back without the final synchronisation, for pipelined host
 * transfers: the reorder/unpack kernels run on the context stream into a
 * device staging buffer, and the device-to-host copies run on the context's
 * COPY stream (PCIe is full duplex: they overlap the next step's host-to-device
 * input copy and its compute).  The host buffers (pinned, for real overlap)
 * are valid only after qt_ctx_synchronize(ctx); A may be destroyed right
 * after the call.  Device destination pointers are written on the context
 * stream (no copy stream involved).  Block sizes 16 and 64 complete the
 * read-back before returning (as qt_read_back).
 * Errors: QT_EINVAL, QT_ECUDA. */
qt_status qt_read_back_async(qt_mat A, int32_t* brow, int32_t* bcol, void* values);

/* Plans: a multiply whose numeric pass can be re-run.  qt_multiply_plan is
 * qt_multiply_ex (single rank; no overlap phases) that also keeps the numeric
 * launch and the symbolic pass's buffers it reads; C is returned as usual.
 * qt_plan_execute recomputes C's values from the CURRENT values of A and B
 * (the patterns are fixed: change values with qt_update_values) — the same
 * kernel and summation order, so the result is bitwise that of a fresh
 * qt_multiply.  It only enqueues work on the context stream (no host
 * synchronisation, no allocation), so it can be captured into a CUDA graph.
 * A, B and C must outlive the plan.  Errors: as qt_multiply_ex; QT_EINVAL
 * (world > 1). */
typedef struct qt_plan_s* qt_plan;
qt_status qt_multiply_plan(qt_mat A, qt_mat B, int32_t trans_a, int32_t trans_b, qt_plan* plan,
                           qt_mat* C, qt_stats* st);
/* The symmetric square's plan (qt_symm_square, single rank, block_size 32):
 * executing it refreshes U's transposed copy from U's current values and
 * recomputes C — the S^2 of density-matrix purification steps whose pattern
 * is fixed.  Errors: as qt_symm_square; QT_EBS (block_size != 32). */
qt_status qt_symm_square_plan(qt_mat A, qt_plan* plan, qt_mat* C, qt_stats* st);
qt_status qt_plan_execute(qt_plan plan);
qt_status qt_plan_destroy(qt_plan plan);

/* New values for A's blocks (same pattern): `values` holds nblocks blocks of
 * bs x bs row-major values in qt_read_back order (ascending brow, then bcol),
 * host or device memory; A's cached screening norms are dropped.  Stream
 * ordered on the context stream (a host source is copied before return).
 * block_size 32.  Errors: QT_EINVAL, QT_EBS, QT_ECUDA. */
qt_status qt_update_values(qt_mat A, const void* values);

/* Wait for everything this context has enqueued, including the copies of
 * qt_read_back_async, and release their staging buffers.  Errors: QT_ECUDA. */
qt_status qt_ctx_synchronize(qt_ctx ctx);

/* Release a matrix (stream-ordered; safe right after the last use).  The
 * paper's chunks are deleted by their owner when no longer referenced
 * (single assignment: a handle is never modified, only freed). */
qt_status qt_destroy(qt_mat A);

/* Message of the last failure on this thread ("" if none). */
const char* qt_last_error(void);

/* ---------------------------------------------------------------- diagnostics */

/* The multi-rank multiply of rank g out of P virtual ranks, on this single
 * (world == 1) context: A and B are whole matrices; the call restricts them
 * to rank g's block rows [row_bounds[g], row_bounds[g+1]) (A, B and C share
 * the bounds), determines the remote B rows as qt_multiply does, packs them
 * from B exactly as their owners would, and runs the same B_ext merge and
 * local multiply.  Only the NCCL transfers are replaced by device copies.
 * C holds rank g's block rows of A*B; `st` reports what rank g would receive.
 * Used to test the distributed path on one GPU. */
/* Row-strip plan (the locality-aware partition of P:82-97,
 * §5.2): `parts` contiguous block-row strips of C = A·B, boundaries
 * at multiples of `align_rows` block rows (a quadtree node row: leaf_dim /
 * block_size for leaf-aligned strips), balanced by block products — row I of
 * C costs sum over A(I,K) of nnz(B(K,:)) products — so that the largest strip
 * is as small as any contiguous aligned partition allows.  Host-only, O(nnz).
 * ctx: NULL or a single-rank context = the arrays are the whole A (block rows
 * and columns) and B (block rows); a multi-rank context = each rank passes its
 * own blocks and the counts are summed over ranks (collective; every rank gets
 * the same bounds).  Out: bounds[parts+1] (caller block rows, bounds[0] = 0,
 * bounds[parts] = n / block_size; trailing strips may be empty) and, if not
 * NULL, strip_products[parts].  Use the bounds as qt_create's row_bounds.
 * Errors: QT_EINVAL (sizes, NULL arrays), QT_ERANGE (a block outside the
 * grid), QT_ENCCL (multi-rank). */
qt_status qt_plan_strips(qt_ctx ctx, int64_t n, int32_t block_size, int32_t align_rows, int64_t nb_a,
                         const int32_t* a_brow, const int32_t* a_bcol, int64_t nb_b, const int32_t* b_brow,
                         int32_t parts, int32_t* bounds, int64_t* strip_products);

/* The multi-rank symmetric square of rank g out of P virtual ranks on this
 * single (world == 1) context: A is the whole upper-triangular U; rank g's
 * block rows are [row_bounds[g], row_bounds[g+1]); the blocks it would receive
 * are selected from U by the rule of qt_symm_square and the same pruned BFS
 * runs.  C holds rank g's rows of A^2 (upper triangle); `st` reports what
 * rank g would receive.  block_size 16 (even row_bounds) or 32.  Errors: as qt_multiply_virtual,
 * QT_EINVAL (a block below the diagonal), QT_EBS (block_size 64). */
qt_status qt_symm_square_virtual(qt_mat A, int32_t P, int32_t g, const int32_t* row_bounds, qt_mat* C,
                                 qt_stats* st);

qt_status qt_multiply_virtual(qt_mat A, qt_mat B, int32_t P, int32_t g,
                              const int32_t* row_bounds, qt_mat* C, qt_stats* st);

/* Loopback transport for testing the multi-rank path on ONE device: `world`
 * rank threads of one process each create a context with
 * qt_ctx_create_loopback on the same hub (and their own stream) and call the
 * collective functions concurrently.  Every NCCL send/recv of the exchange is
 * replaced by a device-to-device cudaMemcpyAsync ordered by CUDA events (no
 * kernel waits on another rank); allgathers go through host memory.  All other
 * code — partition, request lists, packing, B_ext merge, multiply — is the
 * multi-rank code of qt_multiply.  The hub must outlive its contexts. */
qt_status qt_loopback_hub_create(int32_t world, void** hub);
qt_status qt_loopback_hub_destroy(void* hub);
qt_status qt_ctx_create_loopback(int device, void* cuda_stream, int rank, int world, void* hub,
                                 qt_ctx* out);

/* Number of CUDA kernels this context has launched so far (bench accounting). */
int64_t qt_kernel_launches(qt_ctx ctx);

/* FP64 peak microbenchmark on the context's device (roofline denominator,
 * MEASURED_PEAKS.json has no FP64 entry): kind 0 = DMMA (mma.sync m8n8k4 f64),
 * kind 1 = DFMA.  Runs about `ms` milliseconds of back-to-back work and
 * returns the achieved FLOP/s in *flops. */
qt_status qt_fp64_peak(qt_ctx ctx, int kind, float ms, double* flops);

#ifdef __cplusplus
}
#endif
#endif /* QT_H_ */
