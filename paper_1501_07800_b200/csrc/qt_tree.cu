// Quadtree construction (K1/K2), read-back (K9) and truncation (K8).
//
// Matrix chunk = quadtree node (§3.1): every internal node has four
// child slots, NIL (-1) for a zero submatrix; zero submatrices are never
// stored.  On the device a level is an array of non-NIL nodes in Morton order
// and a child table int32[n_l][4]; the block level (l = L) is the block pool
// itself, sorted by Morton key.  The leaf matrices of the paper (block-sparse
// submatrices, §4.1) are the subtrees below the leaf level: their
// "two-dimensional array where only non-zero submatrices are allocated" is
// represented by the same child tables, which lets the symbolic multiply run
// the recursion of §3.2 straight through the leaves to block granularity
// ("merging several of the lowest levels").
#include <cub/cub.cuh>

#include "qt_common.cuh"
#include "qt_internal.h"

namespace qt {

namespace {

constexpr int kThreads = 256;
inline unsigned grid_for(int64_t n, int t = kThreads) {
  int64_t g = (n + t - 1) / t;
  return (unsigned)(g < 1 ? 1 : (g > (1 << 30) ? (1 << 30) : g));
}

__global__ void k_keys(const int32_t* __restrict__ brow, const int32_t* __restrict__ bcol,
                       int64_t nb, int32_t nbr, int32_t row_lo, int32_t row_hi,
                       uint64_t* __restrict__ key, int32_t* __restrict__ idx,
                       unsigned long long* __restrict__ err_range) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < nb;
       t += (int64_t)gridDim.x * blockDim.x) {
    int32_t r = brow[t], c = bcol[t];
    bool bad = r < 0 || c < 0 || r >= nbr || c >= nbr || r < row_lo || r >= row_hi;
    if (bad) atomicMin(err_range, (unsigned long long)t);
    key[t] = bad ? 0 : morton((uint32_t)r, (uint32_t)c);
    idx[t] = (int32_t)t;
  }
}

__global__ void k_dup(const uint64_t* __restrict__ key, int64_t nb,
                      unsigned long long* __restrict__ err_dup) {
  for (int64_t t = 1 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < nb;
       t += (int64_t)gridDim.x * blockDim.x)
    if (key[t] == key[t - 1]) atomicMin(err_dup, (unsigned long long)t);
}

// pool[t] = layout(vals[idx[t]]) ; one 32x32 block per 256 threads, 4 elements each
template <class T>
__global__ void k_fill_pool(const T* __restrict__ vals, const int32_t* __restrict__ idx,
                            int64_t nb, T* __restrict__ pool) {
  for (int64_t t = blockIdx.x; t < nb; t += gridDim.x) {
    const T* src = vals + (int64_t)idx[t] * 1024;
    T* dst = pool + t * 1024;
#pragma unroll
    for (int e = threadIdx.x; e < 1024; e += 256) {
      int r = e >> 5, c = e & 31;
      T v = src[e];
      if (sizeof(T) == 8) dst[swz64(r, c)] = v;
      else dst[swz32(r, c)] = v;
    }
  }
}

__global__ void k_parent_flags(const uint64_t* __restrict__ key, int64_t n,
                               int32_t* __restrict__ flag) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n;
       t += (int64_t)gridDim.x * blockDim.x)
    flag[t] = (t == 0 || (key[t] >> 2) != (key[t - 1] >> 2)) ? 1 : 0;
}

__global__ void k_link(const uint64_t* __restrict__ key, const int32_t* __restrict__ incl,
                       int64_t n, const int32_t* __restrict__ ids, int32_t* __restrict__ child,
                       uint64_t* __restrict__ pkey, int32_t* __restrict__ dmap) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n;
       t += (int64_t)gridDim.x * blockDim.x) {
    int32_t p = incl[t] - 1;
    uint64_t k = key[t];
    child[(int64_t)p * 4 + (int)(k & 3)] = ids ? ids[t] : (int32_t)t;
    if (t == 0 || (k >> 2) != (key[t - 1] >> 2)) {
      pkey[p] = k >> 2;
      if (dmap) dmap[k >> 2] = p;  // (top levels: the parent level's dense map)
    }
  }
}

// per-level occupancy histograms: rows at hist[(1<<l)-1 + r], columns at
// hist[H + (1<<l)-1 + c], H = 2^(L+1)
__global__ void k_level_hist(const uint64_t* __restrict__ key, int64_t n, int l, int64_t H,
                             int32_t* __restrict__ hist) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n;
       t += (int64_t)gridDim.x * blockDim.x) {
    uint64_t k = key[t];
    int64_t base = (1ll << l) - 1;
    atomicAdd(&hist[base + morton_row(k)], 1);
    atomicAdd(&hist[H + base + morton_col(k)], 1);
  }
}

__global__ void k_rowmajor_keys(const uint64_t* __restrict__ key, int64_t n,
                                uint64_t* __restrict__ rm, int32_t* __restrict__ iota) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n;
       t += (int64_t)gridDim.x * blockDim.x) {
    uint64_t k = key[t];
    rm[t] = ((uint64_t)morton_row(k) << 32) | morton_col(k);
    iota[t] = (int32_t)t;
  }
}

template <class T>
__global__ void k_unpack(const T* __restrict__ pool, const uint64_t* __restrict__ key,
                         const int32_t* __restrict__ order, int64_t nb,
                         int32_t* __restrict__ brow, int32_t* __restrict__ bcol,
                         T* __restrict__ out) {
  for (int64_t t = blockIdx.x; t < nb; t += gridDim.x) {
    int32_t s = order[t];
    if (threadIdx.x == 0) {
      uint64_t k = key[s];
      if (brow) brow[t] = (int32_t)morton_row(k);
      if (bcol) bcol[t] = (int32_t)morton_col(k);
    }
    if (!out) continue;
    const T* src = pool + (int64_t)s * 1024;
    T* dst = out + t * 1024;
#pragma unroll
    for (int e = threadIdx.x; e < 1024; e += 256) {
      int r = e >> 5, c = e & 31;
      dst[e] = (sizeof(T) == 8) ? src[swz64(r, c)] : src[swz32(r, c)];
    }
  }
}

template <class T>
__global__ void k_block_norm2(const T* __restrict__ pool, int64_t nb, double* __restrict__ out) {
  // one warp per block, fixed reduction order
  int lane = threadIdx.x & 31;
  int64_t w = blockIdx.x * (int64_t)(blockDim.x / 32) + threadIdx.x / 32;
  for (; w < nb; w += (int64_t)gridDim.x * (blockDim.x / 32)) {
    const T* b = pool + w * 1024;
    double s = 0.0;
    for (int e = lane; e < 1024; e += 32) {
      double v = (double)b[e];
      s += v * v;
    }
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) out[w] = s;
  }
}

__global__ void k_compact_blocks(const uint8_t* __restrict__ keep, const int32_t* __restrict__ incl,
                                 const uint64_t* __restrict__ key, const uint4* __restrict__ pool,
                                 int64_t n, int64_t vec_per_block, uint64_t* __restrict__ okey,
                                 uint4* __restrict__ opool) {
  for (int64_t t = blockIdx.x; t < n; t += gridDim.x) {
    if (!keep[t]) continue;
    int64_t d = incl[t] - 1;
    if (threadIdx.x == 0) okey[d] = key[t];
    for (int64_t e = threadIdx.x; e < vec_per_block; e += blockDim.x)
      opool[d * vec_per_block + e] = pool[t * vec_per_block + e];
  }
}

__global__ void k_u8_to_i32(const uint8_t* __restrict__ in, int64_t n, int32_t* __restrict__ out) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n;
       t += (int64_t)gridDim.x * blockDim.x)
    out[t] = in[t];
}

template <class T>
void cub_sort_pairs(qt_ctx ctx, const uint64_t* kin, uint64_t* kout, const T* vin, T* vout,
                    int64_t n, int end_bit) {
  size_t tb = 0;
  QT_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tb, kin, kout, vin, vout, (int)n, 0, end_bit,
                                          ctx->stream));
  void* tmp = scratch(ctx, tb);
  QT_CUDA(cub::DeviceRadixSort::SortPairs(tmp, tb, kin, kout, vin, vout, (int)n, 0, end_bit,
                                          ctx->stream));
  ctx->launches += 4;
}

template <class T>
void cub_incl_sum(qt_ctx ctx, const T* in, T* out, int64_t n) {
  size_t tb = 0;
  QT_CUDA(cub::DeviceScan::InclusiveSum(nullptr, tb, in, out, (int)n, ctx->stream));
  void* tmp = scratch(ctx, tb);
  QT_CUDA(cub::DeviceScan::InclusiveSum(tmp, tb, in, out, (int)n, ctx->stream));
  ctx->launches += 2;
}

__global__ void k_read_small(const uint8_t* __restrict__ src, uint8_t* __restrict__ dst, size_t n) {
  // (16-byte words where both ends allow it, bytes otherwise)
  const bool v16 = ((reinterpret_cast<uintptr_t>(src) | reinterpret_cast<uintptr_t>(dst)) & 15) == 0;
  const size_t nv = v16 ? n / 16 : 0;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < nv; i += (size_t)gridDim.x * blockDim.x)
    reinterpret_cast<uint4*>(dst)[i] = reinterpret_cast<const uint4*>(src)[i];
  for (size_t i = 16 * nv + blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n;
       i += (size_t)gridDim.x * blockDim.x)
    dst[i] = src[i];
}

}  // namespace

void read_small(qt_ctx ctx, void* dst, const void* src, size_t bytes) {
  if (bytes == 0) return;
  if (!ctx->small_host) {
    QT_CUDA(cudaHostAlloc(&ctx->small_host, qt_ctx_s::kSmallHostBytes, cudaHostAllocMapped));
  }
  for (size_t o = 0; o < bytes; o += qt_ctx_s::kSmallHostBytes) {
    const size_t n = std::min(bytes - o, qt_ctx_s::kSmallHostBytes);
    const unsigned grid = (unsigned)std::min<size_t>(32, (n + 4095) / 4096);
    k_read_small<<<grid, 256, 0, ctx->stream>>>(static_cast<const uint8_t*>(src) + o,
                                                 static_cast<uint8_t*>(ctx->small_host), n);
    QT_LAUNCH_CHECK(ctx);
    QT_CUDA(cudaStreamSynchronize(ctx->stream));
    memcpy(static_cast<uint8_t*>(dst) + o, ctx->small_host, n);
  }
}

void* scratch(qt_ctx ctx, size_t bytes) {
  if (ctx->scratch.bytes < bytes) {
    size_t want = bytes + bytes / 2 + 4096;
    ctx->scratch.alloc(want, ctx->stream);
  }
  return ctx->scratch.p;
}

bool is_device_ptr(const void* p) {
  if (!p) return false;
  cudaPointerAttributes a;
  cudaError_t e = cudaPointerGetAttributes(&a, p);
  if (e != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

void build_levels(qt_mat M, const int32_t* leaf_ids) {
  qt_ctx ctx = M->ctx;
  cudaStream_t st = ctx->stream;
  M->cnt.assign(M->L + 1, 0);
  M->child.clear();
  M->child.resize(M->L);
  M->cnt[M->L] = M->nb;
  const int64_t H = 2ll << M->L;
  M->hist.alloc(8 * H, st);
  QT_CUDA(cudaMemsetAsync(M->hist.p, 0, 8 * H, st));
  M->hist_host.assign(2 * H, 0);
  M->dmap.alloc(4 * qt_mat_s::kDenseNodes, st);
  QT_CUDA(cudaMemsetAsync(M->dmap.p, 0xff, 4 * qt_mat_s::kDenseNodes, st));
  if (M->nb == 0) return;
  DevBuf cur_keys(M->nb * 8, st);
  QT_CUDA(cudaMemcpyAsync(cur_keys.p, M->key.p, M->nb * 8, cudaMemcpyDeviceToDevice, st));
  k_level_hist<<<grid_for(M->nb), kThreads, 0, st>>>(cur_keys.as<uint64_t>(), M->nb, M->L, H,
                                                     M->hist.as<int32_t>());
  QT_LAUNCH_CHECK(ctx);
  for (int l = M->L - 1; l >= 0; --l) {
    int64_t n = M->cnt[l + 1];
    DevBuf flag(n * 4, st), incl(n * 4, st);
    k_parent_flags<<<grid_for(n), kThreads, 0, st>>>(cur_keys.as<uint64_t>(), n, flag.as<int32_t>());
    QT_LAUNCH_CHECK(ctx);
    cub_incl_sum(ctx, flag.as<int32_t>(), incl.as<int32_t>(), n);
    int32_t np = read_scalar(ctx, incl.as<int32_t>() + (n - 1));
    M->cnt[l] = np;
    M->child[l].alloc((size_t)np * 16, st);
    QT_CUDA(cudaMemsetAsync(M->child[l].p, 0xff, (size_t)np * 16, st));
    DevBuf pkey((size_t)np * 8, st);
    k_link<<<grid_for(n), kThreads, 0, st>>>(cur_keys.as<uint64_t>(), incl.as<int32_t>(), n,
                                             l == M->L - 1 ? leaf_ids : nullptr,
                                             M->child[l].as<int32_t>(), pkey.as<uint64_t>(),
                                             l <= qt_mat_s::kDenseLevels
                                                 ? M->dmap.as<int32_t>() + ((1 << (2 * l)) - 1) / 3
                                                 : nullptr);
    QT_LAUNCH_CHECK(ctx);
    cur_keys = std::move(pkey);
    k_level_hist<<<grid_for(np), kThreads, 0, st>>>(cur_keys.as<uint64_t>(), np, l, H,
                                                    M->hist.as<int32_t>());
    QT_LAUNCH_CHECK(ctx);
  }
  // host copy: qt_multiply derives its per-level task counts from it
  read_small(ctx, M->hist_host.data(), M->hist.p, 8 * H);
}

void build_from_blocks(qt_mat M, int64_t nb, const int32_t* d_brow, const int32_t* d_bcol,
                       const void* d_vals, int32_t row_lo, int32_t row_hi) {
  qt_ctx ctx = M->ctx;
  cudaStream_t st = ctx->stream;
  M->nb = nb;
  if (nb == 0) {
    build_levels(M);
    return;
  }
  DevBuf key0(nb * 8, st), idx0(nb * 4, st), idx1(nb * 4, st);
  M->key.alloc(nb * 8, st);
  unsigned long long* err = ctx->counters.as<unsigned long long>();
  QT_CUDA(cudaMemsetAsync(err, 0xff, 16, st));
  k_keys<<<grid_for(nb), kThreads, 0, st>>>(d_brow, d_bcol, nb, M->nbr, row_lo, row_hi,
                                            key0.as<uint64_t>(), idx0.as<int32_t>(), err);
  QT_LAUNCH_CHECK(ctx);
  cub_sort_pairs(ctx, key0.as<uint64_t>(), M->key.as<uint64_t>(), idx0.as<int32_t>(),
                 idx1.as<int32_t>(), nb, 2 * M->L);
  k_dup<<<grid_for(nb), kThreads, 0, st>>>(M->key.as<uint64_t>(), nb, err + 1);
  QT_LAUNCH_CHECK(ctx);
  unsigned long long e[2];
  read_small(ctx, e, err, 16);
  if (e[0] != ~0ull) {
    int32_t r, c;
    QT_CUDA(cudaMemcpy(&r, d_brow + e[0], 4, cudaMemcpyDeviceToHost));
    QT_CUDA(cudaMemcpy(&c, d_bcol + e[0], 4, cudaMemcpyDeviceToHost));
    const int f = M->ubs / 32;
    fail(QT_ERANGE, "block %llu at (brow=%d, bcol=%d) is outside the block grid [0,%d) or this "
         "rank's block rows [%d,%d)", e[0] / (f * f), r < 0 ? r : r / f, c < 0 ? c : c / f,
         M->nbr / f, row_lo / f, row_hi / f);
  }
  if (e[1] != ~0ull) {
    uint64_t k;
    QT_CUDA(cudaMemcpy(&k, M->key.as<uint64_t>() + e[1], 8, cudaMemcpyDeviceToHost));
    const int f = M->ubs / 32;
    fail(QT_EDUP, "block (brow=%u, bcol=%u) is listed twice", morton_row(k) / f, morton_col(k) / f);
  }
  size_t es = elem_size(M->dtype);
  M->pool.alloc(nb * 1024 * es, st);
  unsigned g = (unsigned)std::min<int64_t>(nb, 148 * 16);
  if (M->dtype == QT_F64)
    k_fill_pool<double><<<g, 256, 0, st>>>((const double*)d_vals, idx1.as<int32_t>(), nb,
                                           M->pool.as<double>());
  else
    k_fill_pool<float><<<g, 256, 0, st>>>((const float*)d_vals, idx1.as<int32_t>(), nb,
                                          M->pool.as<float>());
  QT_LAUNCH_CHECK(ctx);
  build_levels(M);
}

namespace {
__global__ void k_lower_count(const uint64_t* __restrict__ key, int64_t n, int f,
                              unsigned long long* bad) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n;
       t += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t k = key[t];
    if (morton_row(k) / f > morton_col(k) / f) atomicMin(bad, (unsigned long long)t);
  }
}
__global__ void k_keep_upper32(const uint64_t* __restrict__ key, int64_t n, uint8_t* __restrict__ keep) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n;
       t += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t k = key[t];
    keep[t] = morton_row(k) <= morton_col(k);
  }
}
}  // namespace

void check_upper(qt_mat M) {
  qt_ctx ctx = M->ctx;
  if (M->nb == 0) return;
  unsigned long long* bad = ctx->counters.as<unsigned long long>();
  QT_CUDA(cudaMemsetAsync(bad, 0xff, 8, ctx->stream));
  const int f = M->ubs / 32;
  k_lower_count<<<grid_for(M->nb), kThreads, 0, ctx->stream>>>(M->key.as<uint64_t>(), M->nb, f, bad);
  QT_LAUNCH_CHECK(ctx);
  const unsigned long long b = read_scalar(ctx, bad);
  if (b != ~0ull) {
    uint64_t k;
    QT_CUDA(cudaMemcpy(&k, M->key.as<uint64_t>() + b, 8, cudaMemcpyDeviceToHost));
    fail(QT_EINVAL, "symmetric square needs upper-triangular block storage; block (brow=%u, bcol=%u) "
         "is below the diagonal", morton_row(k) / f, morton_col(k) / f);
  }
}

qt_mat upper32_view(qt_mat M) {
  DevBuf keep(std::max<int64_t>(M->nb, 1), M->ctx->stream);
  if (M->nb > 0) {
    k_keep_upper32<<<grid_for(M->nb), kThreads, 0, M->ctx->stream>>>(M->key.as<uint64_t>(), M->nb,
                                                                     keep.as<uint8_t>());
    QT_LAUNCH_CHECK(M->ctx);
  }
  return select_blocks(M, keep.as<uint8_t>());
}

namespace {
template <class T>
__global__ void k_split64(const int32_t* __restrict__ brow, const int32_t* __restrict__ bcol,
                          const T* __restrict__ vals, int64_t nb, int32_t* __restrict__ obrow,
                          int32_t* __restrict__ obcol, T* __restrict__ ovals) {
  for (int64_t u = blockIdx.x; u < 4 * nb; u += gridDim.x) {
    const int64_t t = u >> 2;
    const int i = (u >> 1) & 1, j = u & 1;
    if (threadIdx.x == 0) {
      obrow[u] = 2 * brow[t] + i;
      obcol[u] = 2 * bcol[t] + j;
    }
    for (int e = threadIdx.x; e < 1024; e += blockDim.x) {
      const int r = e >> 5, c = e & 31;
      ovals[u * 1024 + e] = vals[t * 4096 + (32 * i + r) * 64 + 32 * j + c];
    }
  }
}

// quads (level L-1 nodes) of a 64-block matrix: row-major key and first child
__global__ void k_quad_keys(const int4* __restrict__ child, const uint64_t* __restrict__ key,
                            int64_t nq, uint64_t* __restrict__ rm, int32_t* __restrict__ iota) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < nq;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int4 c = child[t];
    const int any = c.x >= 0 ? c.x : c.y >= 0 ? c.y : c.z >= 0 ? c.z : c.w;
    const uint64_t q = key[any] >> 2;
    rm[t] = ((uint64_t)morton_row(q) << 32) | morton_col(q);
    iota[t] = (int32_t)t;
  }
}

template <class T>
__global__ void k_unpack64(const T* __restrict__ pool, const int4* __restrict__ child,
                           const uint64_t* __restrict__ rm_sorted, const int32_t* __restrict__ order,
                           int64_t nq, int32_t* __restrict__ brow, int32_t* __restrict__ bcol,
                           T* __restrict__ out) {
  for (int64_t u = blockIdx.x; u < nq; u += gridDim.x) {
    const int4 c4 = child[order[u]];
    if (threadIdx.x == 0) {
      if (brow) brow[u] = (int32_t)(rm_sorted[u] >> 32);
      if (bcol) bcol[u] = (int32_t)(rm_sorted[u] & 0xffffffffu);
    }
    if (!out) continue;
    for (int e = threadIdx.x; e < 4096; e += blockDim.x) {
      const int R = e >> 6, Cc = e & 63, i = R >> 5, j = Cc >> 5, r = R & 31, c = Cc & 31;
      const int s = 2 * i + j;
      const int b = s == 0 ? c4.x : s == 1 ? c4.y : s == 2 ? c4.z : c4.w;
      T v = 0;
      if (b >= 0) v = pool[(int64_t)b * 1024 + (sizeof(T) == 8 ? swz64(r, c) : swz32(r, c))];
      out[u * 4096 + e] = v;
    }
  }
}

__global__ void k_expand_keep(const uint8_t* __restrict__ in, int64_t n, uint8_t* __restrict__ out) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n;
       t += (int64_t)gridDim.x * blockDim.x)
    out[t] = in[t >> 2];
}

__global__ void k_quad_terms(const double* __restrict__ nrm32, const uint64_t* __restrict__ key,
                             int64_t nq, double* __restrict__ nrm, uint64_t* __restrict__ rm) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < nq;
       t += (int64_t)gridDim.x * blockDim.x) {
    // the four 32-blocks of a complete quad are consecutive in Morton order; the
    // squared norms are summed in the fixed sub-block order (0,0),(0,1),(1,0),(1,1)
    nrm[t] = ((nrm32[4 * t] + nrm32[4 * t + 1]) + nrm32[4 * t + 2]) + nrm32[4 * t + 3];
    const uint64_t q = key[4 * t] >> 2;
    rm[t] = ((uint64_t)morton_row(q) << 32) | morton_col(q);
  }
}
}  // namespace

namespace {
// squared Frobenius norm of each block: one thread, row-major order, separate
// multiply and add roundings (the oracle's loop, so both take the same
// screening decisions)
template <class T>
__global__ void k_block_norm2_seq(const T* __restrict__ pool, int64_t nb, double* __restrict__ out) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < nb;
       t += (int64_t)gridDim.x * blockDim.x) {
    const T* b = pool + t * 1024;
    double s = 0.0;
    for (int r = 0; r < 32; ++r)
      for (int c = 0; c < 32; ++c) {
        const double v = (double)b[sizeof(T) == 8 ? swz64(r, c) : swz32(r, c)];
        s = __dadd_rn(s, __dmul_rn(v, v));
      }
    out[t] = s;
  }
}
// node norm^2 = sum of its children's in slot order
__global__ void k_node_norm2(const int4* __restrict__ child, int64_t n, const double* __restrict__ below,
                             double* __restrict__ out) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int4 c = child[t];
    double s = 0.0;
    if (c.x >= 0) s = __dadd_rn(s, below[c.x]);
    if (c.y >= 0) s = __dadd_rn(s, below[c.y]);
    if (c.z >= 0) s = __dadd_rn(s, below[c.z]);
    if (c.w >= 0) s = __dadd_rn(s, below[c.w]);
    out[t] = s;
  }
}
// Block size 16: the squared norm of each present 16-block (row-major over its
// 16 x 16 entries with separate roundings: the oracle's order, so screening
// decisions agree), and the container's = the sum of its quadrants' — a sum of
// non-negative terms is >= each term under rounding, so container and node
// pruning stay exact with respect to the 16-block test.
__global__ void k_quad_norm2(const double* __restrict__ pool, const uint8_t* __restrict__ sub, int64_t nb,
                             double* __restrict__ out16, double* __restrict__ out32) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < nb; t += (int64_t)gridDim.x * blockDim.x) {
    const double* b = pool + t * 1024;
    const int m = sub[t];
    double tot = 0.0;
    for (int q = 0; q < 4; ++q) {
      double s = 0.0;
      if ((m >> q) & 1) {
        const int r0 = 16 * (q >> 1), c0 = 16 * (q & 1);
        for (int r = 0; r < 16; ++r)
          for (int c = 0; c < 16; ++c) {
            const double v = b[swz64(r0 + r, c0 + c)];
            s = __dadd_rn(s, __dmul_rn(v, v));
          }
      }
      out16[4 * t + q] = s;
      tot = __dadd_rn(tot, s);
    }
    out32[t] = tot;
  }
}
}  // namespace

void ensure_norms(qt_mat M) {
  if (!M->norm2.empty()) return;
  ensure_levels(M);
  qt_ctx ctx = M->ctx;
  cudaStream_t st = ctx->stream;
  std::vector<DevBuf> nv(M->L + 1);
  nv[M->L].alloc(8 * std::max<int64_t>(M->nb, 1), st);
  if (M->ubs == 16) {
    if (M->dtype != QT_F64) fail(QT_EDTYPE, "16-block norms are computed on FP64 pools");
    M->norm16.alloc(32 * std::max<int64_t>(M->nb, 1), st);
  }
  // block norms indexed like the pool ids (a multi-rank B_ext: ids < split in
  // the local pool, the rest in the received payload)
  const int64_t n1 = std::min<int64_t>(M->nb, M->split), n2 = M->nb - n1;
  const void* p1 = M->pool_ptr();
  for (int part = 0; part < 2; ++part) {
    const int64_t n = part ? n2 : n1;
    if (n <= 0) continue;
    const void* src = part ? M->pool2 : p1;
    double* out = nv[M->L].as<double>() + (part ? n1 : 0);
    if (M->ubs == 16)
      k_quad_norm2<<<grid_for(n), kThreads, 0, st>>>(static_cast<const double*>(src),
                                                      M->sub.as<uint8_t>() + (part ? n1 : 0), n,
                                                      M->norm16.as<double>() + 4 * (part ? n1 : 0), out);
    else if (M->dtype == QT_F64)
      k_block_norm2_seq<double><<<grid_for(n), kThreads, 0, st>>>(static_cast<const double*>(src), n, out);
    else
      k_block_norm2_seq<float><<<grid_for(n), kThreads, 0, st>>>(static_cast<const float*>(src), n, out);
    QT_LAUNCH_CHECK(ctx);
  }
  for (int l = M->L - 1; l >= 0; --l) {
    nv[l].alloc(8 * std::max<int64_t>(M->cnt[l], 1), st);
    if (M->cnt[l] > 0) {
      k_node_norm2<<<grid_for(M->cnt[l]), kThreads, 0, st>>>(M->child[l].as<int4>(), M->cnt[l],
                                                             nv[l + 1].as<double>(), nv[l].as<double>());
      QT_LAUNCH_CHECK(ctx);
    }
  }
  M->norm2 = std::move(nv);
}

void split64(qt_ctx ctx, qt_dtype dt, int64_t nb, const int32_t* brow, const int32_t* bcol,
             const void* vals, DevBuf& obrow, DevBuf& obcol, DevBuf& ovals) {
  cudaStream_t st = ctx->stream;
  obrow.alloc(16 * nb, st);
  obcol.alloc(16 * nb, st);
  ovals.alloc(4 * nb * 1024 * elem_size(dt), st);
  const unsigned g = (unsigned)std::min<int64_t>(4 * nb, 148 * 16);
  if (dt == QT_F64)
    k_split64<double><<<g, 256, 0, st>>>(brow, bcol, (const double*)vals, nb, obrow.as<int32_t>(),
                                         obcol.as<int32_t>(), ovals.as<double>());
  else
    k_split64<float><<<g, 256, 0, st>>>(brow, bcol, (const float*)vals, nb, obrow.as<int32_t>(),
                                        obcol.as<int32_t>(), ovals.as<float>());
  QT_LAUNCH_CHECK(ctx);
}

void expand_keep(qt_mat M, const uint8_t* keep_user, DevBuf& keep32) {
  keep32.alloc(std::max<int64_t>(M->nb, 1), M->ctx->stream);
  if (M->nb == 0) return;
  k_expand_keep<<<grid_for(M->nb), kThreads, 0, M->ctx->stream>>>(keep_user, M->nb, keep32.as<uint8_t>());
  QT_LAUNCH_CHECK(M->ctx);
}

static void read_back64(qt_mat M, int32_t* brow, int32_t* bcol, void* vals) {
  qt_ctx ctx = M->ctx;
  cudaStream_t st = ctx->stream;
  ensure_levels(M);
  const int64_t nq = M->cnt[M->L - 1];
  if (nq == 0 || M->nb == 0) return;
  const size_t es = elem_size(M->dtype);
  const int4* child = M->child[M->L - 1].as<int4>();
  DevBuf rm(nq * 8, st), rm2(nq * 8, st), iota(nq * 4, st), order(nq * 4, st);
  k_quad_keys<<<grid_for(nq), kThreads, 0, st>>>(child, M->key.as<uint64_t>(), nq, rm.as<uint64_t>(),
                                                 iota.as<int32_t>());
  QT_LAUNCH_CHECK(ctx);
  cub_sort_pairs(ctx, rm.as<uint64_t>(), rm2.as<uint64_t>(), iota.as<int32_t>(), order.as<int32_t>(),
                 nq, 64);
  bool dr = brow && is_device_ptr(brow), dc = bcol && is_device_ptr(bcol),
       dv = vals && is_device_ptr(vals);
  DevBuf sr, sc, sv;
  int32_t* obr = brow ? (dr ? brow : (sr.alloc(nq * 4, st), sr.as<int32_t>())) : nullptr;
  int32_t* obc = bcol ? (dc ? bcol : (sc.alloc(nq * 4, st), sc.as<int32_t>())) : nullptr;
  void* ov = vals ? (dv ? vals : (sv.alloc(nq * 4096 * es, st), sv.p)) : nullptr;
  const unsigned g = (unsigned)std::min<int64_t>(nq, 148 * 16);
  if (M->dtype == QT_F64)
    k_unpack64<double><<<g, 256, 0, st>>>(M->pool.as<double>(), child, rm2.as<uint64_t>(),
                                          order.as<int32_t>(), nq, obr, obc, (double*)ov);
  else
    k_unpack64<float><<<g, 256, 0, st>>>(M->pool.as<float>(), child, rm2.as<uint64_t>(),
                                         order.as<int32_t>(), nq, obr, obc, (float*)ov);
  QT_LAUNCH_CHECK(ctx);
  if (brow && !dr) QT_CUDA(cudaMemcpyAsync(brow, obr, nq * 4, cudaMemcpyDeviceToHost, st));
  if (bcol && !dc) QT_CUDA(cudaMemcpyAsync(bcol, obc, nq * 4, cudaMemcpyDeviceToHost, st));
  if (vals && !dv) QT_CUDA(cudaMemcpyAsync(vals, ov, nq * 4096 * es, cudaMemcpyDeviceToHost, st));
  QT_CUDA(cudaStreamSynchronize(st));
}

void reap_pending(qt_ctx ctx, bool wait) {
  auto& P = ctx->pending;
  size_t keep = 0;
  for (size_t i = 0; i < P.size(); ++i) {
    auto* pc = P[i];
    const cudaError_t e = wait ? cudaEventSynchronize(pc->done) : cudaEventQuery(pc->done);
    if (e == cudaSuccess) {
      cudaEventDestroy(pc->done);
      delete pc;  // releases the staging buffers
    } else if (e == cudaErrorNotReady) {
      P[keep++] = pc;
    } else {
      QT_CUDA(e);
    }
  }
  P.resize(keep);
}

void read_back(qt_mat M, int32_t* brow, int32_t* bcol, void* vals, bool async) {
  if (M->ubs == 16) {  // (async: completes before returning)
    read_back16(M, brow, bcol, vals);
    return;
  }
  if (M->ubs == 64) {  // (async: completes before returning)
    read_back64(M, brow, bcol, vals);
    return;
  }
  qt_ctx ctx = M->ctx;
  cudaStream_t st = ctx->stream;
  int64_t nb = M->nb;
  if (nb == 0) return;
  size_t es = elem_size(M->dtype);
  DevBuf rm(nb * 8, st), rm2(nb * 8, st), iota(nb * 4, st), order(nb * 4, st);
  k_rowmajor_keys<<<grid_for(nb), kThreads, 0, st>>>(M->key.as<uint64_t>(), nb, rm.as<uint64_t>(),
                                                     iota.as<int32_t>());
  QT_LAUNCH_CHECK(ctx);
  int bits = 32 + 32 - __builtin_clz((unsigned)std::max(M->nbr, 2));
  cub_sort_pairs(ctx, rm.as<uint64_t>(), rm2.as<uint64_t>(), iota.as<int32_t>(),
                 order.as<int32_t>(), nb, std::min(64, bits));
  bool dr = brow && is_device_ptr(brow), dc = bcol && is_device_ptr(bcol),
       dv = vals && is_device_ptr(vals);
  DevBuf sr, sc, sv;
  int32_t* obr = brow ? (dr ? brow : (sr.alloc(nb * 4, st), sr.as<int32_t>())) : nullptr;
  int32_t* obc = bcol ? (dc ? bcol : (sc.alloc(nb * 4, st), sc.as<int32_t>())) : nullptr;
  void* ov = vals ? (dv ? vals : (sv.alloc(nb * 1024 * es, st), sv.p)) : nullptr;
  unsigned g = (unsigned)std::min<int64_t>(nb, 148 * 16);
  if (M->dtype == QT_F64)
    k_unpack<double><<<g, 256, 0, st>>>(M->pool.as<double>(), M->key.as<uint64_t>(),
                                        order.as<int32_t>(), nb, obr, obc, (double*)ov);
  else
    k_unpack<float><<<g, 256, 0, st>>>(M->pool.as<float>(), M->key.as<uint64_t>(),
                                       order.as<int32_t>(), nb, obr, obc, (float*)ov);
  QT_LAUNCH_CHECK(ctx);
  if (async && ((brow && !dr) || (bcol && !dc) || (vals && !dv))) {
    // device-to-host copies on the copy stream after the unpack; the staging
    // buffers live until the copies are done (reap_pending)
    reap_pending(ctx, false);
    if (!ctx->copy_stream) QT_CUDA(cudaStreamCreateWithFlags(&ctx->copy_stream, cudaStreamNonBlocking));
    auto* pc = new qt_ctx_s::PendingCopy();
    cudaEvent_t ready;
    QT_CUDA(cudaEventCreateWithFlags(&ready, cudaEventDisableTiming));
    QT_CUDA(cudaEventCreateWithFlags(&pc->done, cudaEventDisableTiming));
    QT_CUDA(cudaEventRecord(ready, st));
    QT_CUDA(cudaStreamWaitEvent(ctx->copy_stream, ready, 0));
    cudaStream_t cs = ctx->copy_stream;
    if (brow && !dr) QT_CUDA(cudaMemcpyAsync(brow, obr, nb * 4, cudaMemcpyDeviceToHost, cs));
    if (bcol && !dc) QT_CUDA(cudaMemcpyAsync(bcol, obc, nb * 4, cudaMemcpyDeviceToHost, cs));
    if (vals && !dv) QT_CUDA(cudaMemcpyAsync(vals, ov, nb * 1024 * es, cudaMemcpyDeviceToHost, cs));
    QT_CUDA(cudaEventRecord(pc->done, cs));
    QT_CUDA(cudaEventDestroy(ready));  // destruction is deferred until the event completes
    pc->bufs[0] = std::move(sr);
    pc->bufs[1] = std::move(sc);
    pc->bufs[2] = std::move(sv);
    ctx->pending.push_back(pc);
    return;
  }
  if (brow && !dr) QT_CUDA(cudaMemcpyAsync(brow, obr, nb * 4, cudaMemcpyDeviceToHost, st));
  if (bcol && !dc) QT_CUDA(cudaMemcpyAsync(bcol, obc, nb * 4, cudaMemcpyDeviceToHost, st));
  if (vals && !dv) QT_CUDA(cudaMemcpyAsync(vals, ov, nb * 1024 * es, cudaMemcpyDeviceToHost, st));
  if (!async) QT_CUDA(cudaStreamSynchronize(st));
}

namespace {
__global__ void k_scatter_inv(const int32_t* __restrict__ order, int64_t n, int32_t* __restrict__ inv) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x)
    inv[order[t]] = (int32_t)t;
}
}  // namespace

void update_values(qt_mat M, const void* values) {
  qt_ctx ctx = M->ctx;
  cudaStream_t st = ctx->stream;
  const int64_t nb = M->nb;
  if (nb == 0) return;
  const size_t es = elem_size(M->dtype);
  if (!M->rm_inv.p) {  // pool index -> row-major position, once per matrix
    DevBuf rm(nb * 8, st), rm2(nb * 8, st), iota(nb * 4, st), order(nb * 4, st);
    k_rowmajor_keys<<<grid_for(nb), kThreads, 0, st>>>(M->key.as<uint64_t>(), nb, rm.as<uint64_t>(),
                                                       iota.as<int32_t>());
    QT_LAUNCH_CHECK(ctx);
    cub_sort_pairs(ctx, rm.as<uint64_t>(), rm2.as<uint64_t>(), iota.as<int32_t>(), order.as<int32_t>(), nb, 64);
    M->rm_inv.alloc(nb * 4, st);
    k_scatter_inv<<<grid_for(nb), kThreads, 0, st>>>(order.as<int32_t>(), nb, M->rm_inv.as<int32_t>());
    QT_LAUNCH_CHECK(ctx);
  }
  DevBuf dv;
  const void* src = values;
  if (!is_device_ptr(values)) {
    dv.alloc(nb * 1024 * es, st);
    QT_CUDA(cudaMemcpyAsync(dv.p, values, nb * 1024 * es, cudaMemcpyHostToDevice, st));
    src = dv.p;
  }
  const unsigned g = (unsigned)std::min<int64_t>(nb, 148 * 16);
  if (M->dtype == QT_F64)
    k_fill_pool<double><<<g, 256, 0, st>>>((const double*)src, M->rm_inv.as<int32_t>(), nb, M->pool.as<double>());
  else
    k_fill_pool<float><<<g, 256, 0, st>>>((const float*)src, M->rm_inv.as<int32_t>(), nb, M->pool.as<float>());
  QT_LAUNCH_CHECK(ctx);
  M->norm2.clear();  // (screening norms and U^T's cached pool follow the values)
  M->norm16.release();
  M->poolT_cache.release();
  M->poolT_src = nullptr;
  M->f64_copy.reset();
  if (!is_device_ptr(values)) QT_CUDA(cudaStreamSynchronize(st));  // the host buffer may be reused on return
}

static qt_mat clone_params(qt_mat A) {
  qt_mat M = new qt_mat_s();
  M->ctx = A->ctx;
  M->n = A->n;
  M->leaf_dim = A->leaf_dim;
  M->bs = A->bs;
  M->dtype = A->dtype;
  M->L = A->L;
  M->leaf_level = A->leaf_level;
  M->nbr = A->nbr;
  M->row_lo = A->row_lo;
  M->row_hi = A->row_hi;
  M->bounds = A->bounds;
  M->ubs = A->ubs;
  return M;
}

qt_mat select_blocks(qt_mat A, const uint8_t* d_keep) {
  qt_ctx ctx = A->ctx;
  cudaStream_t st = ctx->stream;
  qt_mat M = clone_params(A);
  try {
    int64_t n = A->nb;
    int64_t kept = 0;
    DevBuf k32, incl;
    if (n > 0) {
      k32.alloc(n * 4, st);
      incl.alloc(n * 4, st);
      k_u8_to_i32<<<grid_for(n), kThreads, 0, st>>>(d_keep, n, k32.as<int32_t>());
      QT_LAUNCH_CHECK(ctx);
      cub_incl_sum(ctx, k32.as<int32_t>(), incl.as<int32_t>(), n);
      kept = read_scalar(ctx, incl.as<int32_t>() + (n - 1));
    }
    M->nb = kept;
    if (A->ubs == 16) M->nb16 = n > 0 ? compact_sub16(ctx, d_keep, incl.as<int32_t>(), A->sub.as<uint8_t>(), n, kept, M->sub) : 0;
    if (kept > 0) {
      size_t es = elem_size(A->dtype);
      M->key.alloc(kept * 8, st);
      M->pool.alloc(kept * 1024 * es, st);
      int64_t vpb = 1024 * es / 16;
      unsigned g = (unsigned)std::min<int64_t>(n, 148 * 16);
      k_compact_blocks<<<g, 256, 0, st>>>(d_keep, incl.as<int32_t>(), A->key.as<uint64_t>(),
                                          A->pool.as<uint4>(), n, vpb, M->key.as<uint64_t>(),
                                          M->pool.as<uint4>());
      QT_LAUNCH_CHECK(ctx);
    }
    build_levels(M);
  } catch (...) {
    delete M;
    throw;
  }
  return M;
}

// Pool conversion between the FP32 layout (swz32) and the FP64 layout (swz64),
// element by element (float -> double is exact; double -> float rounds to
// nearest).  One 32x32 block per CTA iteration.
template <class Ti, class To>
__global__ void k_convert_pool(const Ti* __restrict__ in, To* __restrict__ out, int64_t nb) {
  for (int64_t b = blockIdx.x; b < nb; b += gridDim.x) {
    const Ti* src = in + b * 1024;
    To* dst = out + b * 1024;
    for (int i = threadIdx.x; i < 1024; i += blockDim.x) {
      const int r = i >> 5, c = i & 31;
      dst[sizeof(To) == 8 ? swz64(r, c) : swz32(r, c)] = (To)src[sizeof(Ti) == 8 ? swz64(r, c) : swz32(r, c)];
    }
  }
}

qt_mat convert_dtype(qt_mat A, qt_dtype to) {
  qt_ctx ctx = A->ctx;
  cudaStream_t st = ctx->stream;
  if (A->pool1 || A->split != INT64_MAX) fail(QT_ESTATE, "convert_dtype: a plain matrix is required");
  qt_mat M = clone_params(A);
  try {
    M->dtype = to;
    M->nb = A->nb;
    M->nb16 = A->nb16;
    M->global_nb = A->global_nb;
    if (A->nb > 0) {
      M->key.alloc(8 * A->nb, st);
      QT_CUDA(cudaMemcpyAsync(M->key.p, A->key.p, 8 * A->nb, cudaMemcpyDeviceToDevice, st));
      if (A->ubs == 16) {
        M->sub.alloc(A->nb, st);
        QT_CUDA(cudaMemcpyAsync(M->sub.p, A->sub.p, A->nb, cudaMemcpyDeviceToDevice, st));
      }
      M->pool.alloc((size_t)A->nb * 1024 * elem_size(to), st);
      const unsigned g = (unsigned)std::min<int64_t>(A->nb, 148 * 8);
      if (A->dtype == QT_F32 && to == QT_F64)
        k_convert_pool<float, double><<<g, 256, 0, st>>>(A->pool.as<float>(), M->pool.as<double>(), A->nb);
      else if (A->dtype == QT_F64 && to == QT_F32)
        k_convert_pool<double, float><<<g, 256, 0, st>>>(A->pool.as<double>(), M->pool.as<float>(), A->nb);
      else
        fail(QT_EDTYPE, "convert_dtype: F32 <-> F64 only");
      QT_LAUNCH_CHECK(ctx);
    }
    // the quadtree is the same: copy it (stream-ordered, no host sync) rather
    // than rebuilding it; a fresh product's levels stay unbuilt
    M->levels_built = A->levels_built;
    if (A->levels_built) {
      M->cnt = A->cnt;
      M->hist_host = A->hist_host;
      auto dup = [&](const DevBuf& src, DevBuf& dst) {
        dst.alloc(src.bytes, st);
        if (src.bytes) QT_CUDA(cudaMemcpyAsync(dst.p, src.p, src.bytes, cudaMemcpyDeviceToDevice, st));
      };
      dup(A->hist, M->hist);
      dup(A->dmap, M->dmap);
      M->child.resize(A->child.size());
      for (size_t l = 0; l < A->child.size(); ++l) dup(A->child[l], M->child[l]);
    }
  } catch (...) {
    delete M;
    throw;
  }
  return M;
}

// Frobenius norms^2 and row-major keys of the local blocks (truncation terms)
void truncate_terms(qt_mat A, DevBuf& nrm, DevBuf& rm) {
  if (A->ubs == 16) {
    truncate_terms16(A, nrm, rm);
    return;
  }
  qt_ctx ctx = A->ctx;
  cudaStream_t st = ctx->stream;
  const int64_t n = A->nb;
  nrm.alloc(8 * std::max<int64_t>(n, 1), st);
  rm.alloc(8 * std::max<int64_t>(n, 1), st);
  if (n == 0) return;
  DevBuf iota(n * 4, st);
  const int wpb = 8;
  const unsigned gr = (unsigned)std::min<int64_t>((n + wpb - 1) / wpb, 148 * 32);
  if (A->dtype == QT_F64)
    k_block_norm2<double><<<gr, 32 * wpb, 0, st>>>(A->pool.as<double>(), n, nrm.as<double>());
  else
    k_block_norm2<float><<<gr, 32 * wpb, 0, st>>>(A->pool.as<float>(), n, nrm.as<double>());
  QT_LAUNCH_CHECK(ctx);
  k_rowmajor_keys<<<grid_for(n), kThreads, 0, st>>>(A->key.as<uint64_t>(), n, rm.as<uint64_t>(),
                                                    iota.as<int32_t>());
  QT_LAUNCH_CHECK(ctx);
  if (A->ubs == 64) {  // terms of the caller's 64-blocks (complete quads of 32-blocks)
    const int64_t nq = n / 4;
    DevBuf n64(8 * std::max<int64_t>(nq, 1), st), r64(8 * std::max<int64_t>(nq, 1), st);
    k_quad_terms<<<grid_for(nq), kThreads, 0, st>>>(nrm.as<double>(), A->key.as<uint64_t>(), nq,
                                                    n64.as<double>(), r64.as<uint64_t>());
    QT_LAUNCH_CHECK(ctx);
    nrm = std::move(n64);
    rm = std::move(r64);
  }
}

namespace {
__global__ void k_iota64(int64_t* __restrict__ out, int64_t n) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n;
       t += (int64_t)gridDim.x * blockDim.x)
    out[t] = t;
}
__global__ void k_gather_bits(const double* __restrict__ nrm, const int64_t* __restrict__ ord,
                              int64_t n, uint64_t* __restrict__ bits) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n;
       t += (int64_t)gridDim.x * blockDim.x)
    bits[t] = (uint64_t)__double_as_longlong(nrm[ord[t]]);  // norms >= 0: bit order = value order
}
__global__ void k_gather_val(const double* __restrict__ nrm, const int64_t* __restrict__ ord,
                             int64_t n, double* __restrict__ out) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n;
       t += (int64_t)gridDim.x * blockDim.x)
    out[t] = nrm[ord[t]];
}
// the blocks of the dropped prefix that belong to rank `me` lose their keep flag
__global__ void k_mark_drop(const double* __restrict__ prefix, const int64_t* __restrict__ ord,
                            const int64_t* __restrict__ id, int64_t n, double tau2, int me,
                            uint8_t* __restrict__ keep) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n;
       t += (int64_t)gridDim.x * blockDim.x) {
    if (!(prefix[t] < tau2)) continue;
    const int64_t v = id[ord[t]];
    if ((int)(v >> 32) == me) keep[v & 0xffffffffll] = 0;
  }
}
}  // namespace

// Global truncation decision (reading C-16) over all terms of all ranks: order
// by (norm^2, brow, bcol) — a stable sort by the row-major key, then a stable
// sort by the norm — prefix sums of norm^2 in that order, and every term
// whose prefix is < tau^2 is dropped.  Every rank evaluates the same
// deterministic sort and scan on the same data, so all agree.
void truncate_decide(qt_ctx ctx, const double* nrm_all, const uint64_t* rm_all, const int64_t* id_all,
                     int64_t n_all, double tau2, int me, uint8_t* keep_local) {
  cudaStream_t st = ctx->stream;
  if (n_all == 0) return;
  DevBuf iota(8 * n_all, st), rm2(8 * n_all, st), ord1(8 * n_all, st), bits(8 * n_all, st),
      bits2(8 * n_all, st), ord2(8 * n_all, st), g(8 * n_all, st), pre(8 * n_all, st);
  k_iota64<<<grid_for(n_all), kThreads, 0, st>>>(iota.as<int64_t>(), n_all);
  QT_LAUNCH_CHECK(ctx);
  cub_sort_pairs(ctx, rm_all, rm2.as<uint64_t>(), iota.as<int64_t>(), ord1.as<int64_t>(), n_all, 64);
  k_gather_bits<<<grid_for(n_all), kThreads, 0, st>>>(nrm_all, ord1.as<int64_t>(), n_all,
                                                      bits.as<uint64_t>());
  QT_LAUNCH_CHECK(ctx);
  cub_sort_pairs(ctx, bits.as<uint64_t>(), bits2.as<uint64_t>(), ord1.as<int64_t>(),
                 ord2.as<int64_t>(), n_all, 64);
  k_gather_val<<<grid_for(n_all), kThreads, 0, st>>>(nrm_all, ord2.as<int64_t>(), n_all, g.as<double>());
  QT_LAUNCH_CHECK(ctx);
  cub_incl_sum(ctx, g.as<double>(), pre.as<double>(), n_all);
  k_mark_drop<<<grid_for(n_all), kThreads, 0, st>>>(pre.as<double>(), ord2.as<int64_t>(), id_all,
                                                    n_all, tau2, me, keep_local);
  QT_LAUNCH_CHECK(ctx);
}

qt_mat truncate(qt_mat A, double tau) {
  qt_ctx ctx = A->ctx;
  cudaStream_t st = ctx->stream;
  const int64_t n = user_nblocks(A);
  DevBuf keep(std::max<int64_t>(n, 1), st);
  if (n > 0) {
    QT_CUDA(cudaMemsetAsync(keep.p, 1, n, st));
    DevBuf nrm, rm, id(8 * n, st);
    truncate_terms(A, nrm, rm);
    k_iota64<<<grid_for(n), kThreads, 0, st>>>(id.as<int64_t>(), n);  // rank 0, local index
    QT_LAUNCH_CHECK(ctx);
    truncate_decide(ctx, nrm.as<double>(), rm.as<uint64_t>(), id.as<int64_t>(), n, tau * tau, 0,
                    keep.as<uint8_t>());
  }
  if (A->ubs == 64) {
    DevBuf k32;
    expand_keep(A, keep.as<uint8_t>(), k32);
    return select_blocks(A, k32.as<uint8_t>());
  }
  if (A->ubs == 16) return apply_keep16(A, keep.as<uint8_t>());
  return select_blocks(A, keep.as<uint8_t>());
}

}  // namespace qt
