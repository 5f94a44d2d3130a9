// Block size 16 (the paper's leaf block size "around 16-64",
// P:378-379, and its S^2 experiments' block size 16).
//
// A matrix of 16x16 blocks is held in the kernels' 32x32 blocks
// ("containers"): container (R, C) holds the caller's blocks (2R+i, 2C+j),
// i, j in {0,1}, as its quadrants, absent quadrants exactly zero, and an
// occupancy mask sub[t] (bit 2i+j) per container indexed like the pool.  The
// quadtree is the 16-block quadtree with its last level folded into the
// containers; every 32-block product of the numeric kernels computes all
// 16-block products between the two containers (the products with an absent
// quadrant add exact zeros), so each present C quadrant is the sum of its
// 16-block products.  The 16-block pattern of C (the symbolic product one
// level further down) is the boolean 2x2 product of the operand
// masks summed over each tile's tasks (k_cmask16).  At the container level the
// BFS and the FP64 kernel skip container pairs whose quadrants never meet (no
// 16-block product), so C holds no empty container; the task count of that
// level is still reported over all non-NIL pairs (the paper's C_l).  Reading
// C-27 in DESIGN.md.
#include <cub/cub.cuh>

#include "qt_common.cuh"
#include "qt_internal.h"

namespace qt {

namespace {

constexpr int kT = 256;
inline unsigned gfor(int64_t n, int t = kT) {
  int64_t g = (n + t - 1) / t;
  return (unsigned)(g < 1 ? 1 : (g > (1 << 30) ? (1 << 30) : g));
}

template <class T>
void sort_pairs(qt_ctx ctx, const uint64_t* kin, uint64_t* kout, const T* vin, T* vout, int64_t n, int bits) {
  size_t tb = 0;
  QT_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tb, kin, kout, vin, vout, (int)n, 0, bits, ctx->stream));
  void* tmp = scratch(ctx, tb);
  QT_CUDA(cub::DeviceRadixSort::SortPairs(tmp, tb, kin, kout, vin, vout, (int)n, 0, bits, ctx->stream));
  ctx->launches += 4;
}
void incl_sum(qt_ctx ctx, const int32_t* in, int32_t* out, int64_t n) {
  size_t tb = 0;
  QT_CUDA(cub::DeviceScan::InclusiveSum(nullptr, tb, in, out, (int)n, ctx->stream));
  void* tmp = scratch(ctx, tb);
  QT_CUDA(cub::DeviceScan::InclusiveSum(tmp, tb, in, out, (int)n, ctx->stream));
  ctx->launches += 2;
}


template <class T>
__device__ __forceinline__ int swz(int r, int c) {
  return sizeof(T) == 8 ? swz64(r, c) : swz32(r, c);
}

// boolean 2x2 product of quadrant masks, and the number of quadrant products
__device__ __forceinline__ int mask_mul(int a, int b, int& nprod, int keep = 15) {
  int out = 0;
#pragma unroll
  for (int r = 0; r < 2; ++r)
#pragma unroll
    for (int c = 0; c < 2; ++c) {
      if (!((keep >> (2 * r + c)) & 1)) continue;
      const int n = (((a >> (2 * r)) & 1) & ((b >> c) & 1)) + (((a >> (2 * r + 1)) & 1) & ((b >> (2 + c)) & 1));
      nprod += n;
      if (n) out |= 1 << (2 * r + c);
    }
  return out;
}

__global__ void k_keys16(const int32_t* __restrict__ brow, const int32_t* __restrict__ bcol, int64_t n,
                         int32_t nbr16, int32_t lo, int32_t hi, uint64_t* __restrict__ key,
                         int32_t* __restrict__ idx, unsigned long long* __restrict__ err) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x) {
    const int32_t r = brow[t], c = bcol[t];
    const bool bad = r < 0 || c < 0 || r >= nbr16 || c >= nbr16 || r < lo || r >= hi;
    if (bad) atomicMin(err, (unsigned long long)t);
    key[t] = bad ? 0 : morton((uint32_t)r, (uint32_t)c);
    idx[t] = (int32_t)t;
  }
}

__global__ void k_dup16(const uint64_t* __restrict__ key, int64_t n, unsigned long long* __restrict__ err) {
  for (int64_t t = 1 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x)
    if (key[t] == key[t - 1]) atomicMin(err, (unsigned long long)t);
}

__global__ void k_heads16(const uint64_t* __restrict__ key, int64_t n, int32_t* __restrict__ head) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x)
    head[t] = (t == 0 || (key[t] >> 2) != (key[t - 1] >> 2)) ? 1 : 0;
}

// container keys and masks (one thread per container head)
__global__ void k_containers16(const uint64_t* __restrict__ key, const int32_t* __restrict__ head,
                               const int32_t* __restrict__ incl, int64_t n, uint64_t* __restrict__ ckey,
                               uint8_t* __restrict__ sub) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x) {
    if (!head[t]) continue;
    const uint64_t c = key[t] >> 2;
    int m = 0;
    for (int64_t s = t; s < n && s < t + 4 && (key[s] >> 2) == c; ++s) m |= 1 << (int)(key[s] & 3);
    const int32_t d = incl[t] - 1;
    ckey[d] = c;
    sub[d] = (uint8_t)m;
  }
}

// the values of sorted 16-block s (caller index idx[s]) into quadrant key&3 of container incl[s]-1
template <class T>
__global__ void k_fill16(const T* __restrict__ vals, const uint64_t* __restrict__ key, const int32_t* __restrict__ idx,
                         const int32_t* __restrict__ incl, int64_t n, T* __restrict__ pool) {
  for (int64_t s = blockIdx.x; s < n; s += gridDim.x) {
    const int q = (int)(key[s] & 3), i = q >> 1, j = q & 1;
    const T* src = vals + (int64_t)idx[s] * 256;
    T* dst = pool + (int64_t)(incl[s] - 1) * 1024;
    const int e = threadIdx.x, r = e >> 4, c = e & 15;
    dst[swz<T>(16 * i + r, 16 * j + c)] = src[e];
  }
}

__global__ void k_popc(const uint8_t* __restrict__ sub, int64_t n, int32_t* __restrict__ cnt) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x)
    cnt[t] = __popc((unsigned)sub[t]);
}

// user-order terms: 16-block u = (container t, its k-th set quadrant), row-major key and source
__global__ void k_terms16(const uint64_t* __restrict__ key, const uint8_t* __restrict__ sub,
                          const int32_t* __restrict__ incl, int64_t n, uint64_t* __restrict__ rm,
                          int32_t* __restrict__ src) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x) {
    const int m = sub[t];
    int u = incl[t] - __popc((unsigned)m);
    const uint64_t R = morton_row(key[t]), C = morton_col(key[t]);
    for (int q = 0; q < 4; ++q) {
      if (!((m >> q) & 1)) continue;
      rm[u] = ((2 * R + (q >> 1)) << 32) | (2 * C + (q & 1));
      src[u] = (int32_t)(4 * t + q);
      ++u;
    }
  }
}

template <class T>
__global__ void k_unpack16(const T* __restrict__ pool, const uint64_t* __restrict__ rm, const int32_t* __restrict__ src,
                           int64_t n, int32_t* __restrict__ brow, int32_t* __restrict__ bcol, T* __restrict__ out) {
  for (int64_t u = blockIdx.x; u < n; u += gridDim.x) {
    const int32_t s = src[u];
    if (threadIdx.x == 0) {
      if (brow) brow[u] = (int32_t)(rm[u] >> 32);
      if (bcol) bcol[u] = (int32_t)(rm[u] & 0xffffffffu);
    }
    if (!out) continue;
    const int q = s & 3, i = q >> 1, j = q & 1, e = threadIdx.x, r = e >> 4, c = e & 15;
    out[u * 256 + e] = pool[(int64_t)(s >> 2) * 1024 + swz<T>(16 * i + r, 16 * j + c)];
  }
}

// squared Frobenius norm of each listed quadrant (one thread, row-major)
template <class T>
__global__ void k_norm16(const T* __restrict__ pool, const int32_t* __restrict__ src, int64_t n,
                         double* __restrict__ out) {
  for (int64_t u = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; u < n; u += (int64_t)gridDim.x * blockDim.x) {
    const int32_t s = src[u];
    const int q = s & 3, i = q >> 1, j = q & 1;
    const T* b = pool + (int64_t)(s >> 2) * 1024;
    double acc = 0.0;
    for (int r = 0; r < 16; ++r)
      for (int c = 0; c < 16; ++c) {
        const double v = (double)b[swz<T>(16 * i + r, 16 * j + c)];
        acc = __dadd_rn(acc, __dmul_rn(v, v));
      }
    out[u] = acc;
  }
}

// new masks after a truncation decision on the user-order terms
__global__ void k_newmask16(const uint8_t* __restrict__ sub, const int32_t* __restrict__ incl,
                            const uint8_t* __restrict__ keep_user, int64_t n, uint8_t* __restrict__ nsub,
                            uint8_t* __restrict__ keep) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x) {
    const int m = sub[t];
    int u = incl[t] - __popc((unsigned)m), nm = 0;
    for (int q = 0; q < 4; ++q) {
      if (!((m >> q) & 1)) continue;
      if (keep_user[u]) nm |= 1 << q;
      ++u;
    }
    nsub[t] = (uint8_t)nm;
    keep[t] = nm != 0;
  }
}

// zero the quadrants a container's mask does not list (one CTA per container)
template <class T>
__global__ void k_zero_absent16(T* __restrict__ pool, const uint8_t* __restrict__ sub, int64_t n) {
  for (int64_t t = blockIdx.x; t < n; t += gridDim.x) {
    const int m = sub[t];
    if (m == 15) continue;
    for (int e = threadIdx.x; e < 1024; e += blockDim.x) {
      const int r = e >> 5, c = e & 31, q = 2 * (r >> 4) + (c >> 4);
      if (!((m >> q) & 1)) pool[t * 1024 + swz<T>(r, c)] = T(0);
    }
  }
}

// one warp per C tile (level L-1 node): the 16-block pattern of its four C
// containers = OR over the tile's tasks and inner k of mask(op(A)) x mask(op(B))
__global__ void k_cmask16(const int32_t* __restrict__ ts, const int32_t* __restrict__ pa, const int32_t* __restrict__ pb,
                          int64_t ntiles, const int4* __restrict__ cA, const int4* __restrict__ cB,
                          const int4* __restrict__ cC, const uint8_t* __restrict__ subA,
                          const uint8_t* __restrict__ subB, int trans, const uint64_t* __restrict__ keyC,
                          uint8_t* __restrict__ subC, unsigned long long* __restrict__ counts,
                          const double* __restrict__ n16A, const double* __restrict__ n16B, double tau2) {
  // symmetric square (trans bit 2): node and block entries are references
  // into U (index << 2 | diagonal << 1 | transposed), see op_children; the
  // (1,0) quadrant of a diagonal C container, and every container below the
  // diagonal, are not part of C: none of their products counted
  const bool sym = trans & 4;
  const int lane = threadIdx.x & 31;
  const int64_t t = blockIdx.x * (int64_t)(blockDim.x / 32) + threadIdx.x / 32;
  if (t >= ntiles) return;
  int keep[4] = {15, 15, 15, 15};
  if (sym) {
    const int4 c4 = cC[t];
    const int c[4] = {c4.x, c4.y, c4.z, c4.w};
#pragma unroll
    for (int q = 0; q < 4; ++q)  // (a container below the diagonal of a diagonal tile is NIL in C)
      keep[q] = c[q] < 0 ? 0 : morton_row(keyC[c[q]]) == morton_col(keyC[c[q]]) ? 11 : 15;
  }
  int m[4] = {0, 0, 0, 0}, np = 0, npairs = 0;
  for (int32_t p = ts[t] + lane; p < ts[t + 1]; p += 32) {
    const int4 A4 = op_children(cA, pa[p], trans & 1, sym), B4 = op_children(cB, pb[p], trans & 2, sym);
    const int a[4] = {A4.x, A4.y, A4.z, A4.w}, b[4] = {B4.x, B4.y, B4.z, B4.w};
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int i = q >> 1, j = q & 1;
#pragma unroll
      for (int k = 0; k < 2; ++k) {
        const int x = a[2 * i + k], y = b[2 * k + j];
        if (x < 0 || y < 0) continue;
        ++npairs;
        int ma, mb;
        if (sym) {
          ma = subA[x >> 2];
          mb = subB[y >> 2];
          if (x & 1) ma = mask_t(ma);
          if (y & 1) mb = mask_t(mb);
        } else {
          ma = subA[x];
          mb = subB[y];
          if (trans & 1) ma = mask_t(ma);
          if (trans & 2) mb = mask_t(mb);
        }
        if (n16A) {  // norm screening (plain product): the 16-block products that pass
          const int pm = screen16(ma, mb, n16A + 4 * (int64_t)x, n16B + 4 * (int64_t)y, tau2);
#pragma unroll
          for (int cq = 0; cq < 4; ++cq) {
            const int nq = ((pm >> (2 * cq)) & 1) + ((pm >> (2 * cq + 1)) & 1);
            np += nq;
            if (nq) m[q] |= 1 << cq;
          }
        } else {
          m[q] |= mask_mul(ma, mb, np, keep[q]);
        }
      }
    }
  }
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) {
#pragma unroll
    for (int q = 0; q < 4; ++q) m[q] |= __shfl_xor_sync(0xffffffffu, m[q], d);
    np += __shfl_xor_sync(0xffffffffu, np, d);
    npairs += __shfl_xor_sync(0xffffffffu, npairs, d);
  }
  if (lane == 0) {
    const int4 c4 = cC[t];
    const int c[4] = {c4.x, c4.y, c4.z, c4.w};
    int n16 = 0, empty = 0;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      if (c[q] < 0) continue;
      subC[c[q]] = (uint8_t)m[q];
      n16 += __popc((unsigned)m[q]);
      empty += m[q] == 0;
    }
    atomicAdd(&counts[0], (unsigned long long)np);
    atomicAdd(&counts[1], (unsigned long long)n16);
    atomicAdd(&counts[2], (unsigned long long)empty);
    atomicAdd(&counts[3], (unsigned long long)npairs);
  }
}

// the first container holding a 16-block below the diagonal (R > C, or the
// (1,0) quadrant of a diagonal container)
__global__ void k_lower16(const uint64_t* __restrict__ key, const uint8_t* __restrict__ sub, int64_t n,
                          unsigned long long* __restrict__ bad) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t R = morton_row(key[t]), C = morton_col(key[t]);
    if (R > C || (R == C && (sub[t] & 4))) atomicMin(bad, (unsigned long long)t);
  }
}

// symmetric square at bs 16: a diagonal container of U gets its (1,0)
// quadrant = (0,1)^T, so it is the full symmetric 32-block the 32-level
// symmetric square uses as stored (reading C-23 one level down)
template <class T>
__global__ void k_complete_diag16(const uint64_t* __restrict__ key, uint8_t* __restrict__ sub, int64_t n,
                                  T* __restrict__ pool) {
  for (int64_t t = blockIdx.x; t < n; t += gridDim.x) {
    if (morton_row(key[t]) != morton_col(key[t]) || !(sub[t] & 2)) continue;
    T* b = pool + t * 1024;
    const int e = threadIdx.x, r = e >> 4, c = e & 15;  // (1,0)[r][c] = (0,1)[c][r]
    b[swz<T>(16 + r, c)] = b[swz<T>(c, 16 + r)];
    if (threadIdx.x == 0) sub[t] |= 4;
  }
}

// C of the bs-16 symmetric square: the (1,0) quadrant of a diagonal
// container is below the diagonal — not part of C (k_cmask16 left its mask
// bit clear); the numeric kernel computed it with the full 32-block: zero it
template <class T>
__global__ void k_drop_lower16(const uint64_t* __restrict__ key, int64_t n, T* __restrict__ pool) {
  for (int64_t t = blockIdx.x; t < n; t += gridDim.x) {
    if (morton_row(key[t]) != morton_col(key[t])) continue;
    T* b = pool + t * 1024;
    const int e = threadIdx.x, r = e >> 4, c = e & 15;
    b[swz<T>(16 + r, c)] = T(0);
  }
}

__global__ void k_compact_u8(const uint8_t* __restrict__ keep, const int32_t* __restrict__ incl,
                             const uint8_t* __restrict__ in, int64_t n, uint8_t* __restrict__ out) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x)
    if (keep[t]) out[incl[t] - 1] = in[t];
}

__global__ void k_nonempty(const uint8_t* __restrict__ sub, int64_t n, uint8_t* __restrict__ keep) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x)
    keep[t] = sub[t] != 0;
}

// per-container counts and their inclusive scan (the user order of 16-blocks)
int64_t user_scan16(qt_mat M, DevBuf& incl) {
  qt_ctx ctx = M->ctx;
  cudaStream_t st = ctx->stream;
  DevBuf cnt(4 * M->nb, st);
  incl.alloc(4 * M->nb, st);
  k_popc<<<gfor(M->nb), kT, 0, st>>>(M->sub.as<uint8_t>(), M->nb, cnt.as<int32_t>());
  QT_LAUNCH_CHECK(ctx);
  incl_sum(ctx, cnt.as<int32_t>(), incl.as<int32_t>(), M->nb);
  return read_scalar(ctx, incl.as<int32_t>() + (M->nb - 1));
}

}  // namespace

void build_from_blocks16(qt_mat M, int64_t n, const int32_t* brow, const int32_t* bcol, const void* vals,
                         int32_t lo16, int32_t hi16) {
  qt_ctx ctx = M->ctx;
  cudaStream_t st = ctx->stream;
  M->nb16 = n;
  if (n == 0) {
    M->nb = 0;
    build_levels(M);
    return;
  }
  DevBuf k0(8 * n, st), k1(8 * n, st), i0(4 * n, st), i1(4 * n, st), head(4 * n, st), incl(4 * n, st);
  unsigned long long* err = ctx->counters.as<unsigned long long>();
  QT_CUDA(cudaMemsetAsync(err, 0xff, 16, st));
  k_keys16<<<gfor(n), kT, 0, st>>>(brow, bcol, n, 2 * M->nbr, lo16, hi16, k0.as<uint64_t>(), i0.as<int32_t>(), err);
  QT_LAUNCH_CHECK(ctx);
  sort_pairs(ctx, k0.as<uint64_t>(), k1.as<uint64_t>(), i0.as<int32_t>(), i1.as<int32_t>(), n, 2 * (M->L + 1));
  k_dup16<<<gfor(n), kT, 0, st>>>(k1.as<uint64_t>(), n, err + 1);
  QT_LAUNCH_CHECK(ctx);
  unsigned long long e[2];
  read_small(ctx, e, err, 16);
  if (e[0] != ~0ull) {
    int32_t r, c;
    QT_CUDA(cudaMemcpy(&r, brow + e[0], 4, cudaMemcpyDeviceToHost));
    QT_CUDA(cudaMemcpy(&c, bcol + e[0], 4, cudaMemcpyDeviceToHost));
    fail(QT_ERANGE, "block %llu at (brow=%d, bcol=%d) is outside the block grid [0,%d) or this rank's block rows "
         "[%d,%d)", e[0], r, c, 2 * M->nbr, lo16, hi16);
  }
  if (e[1] != ~0ull) {
    uint64_t k;
    QT_CUDA(cudaMemcpy(&k, k1.as<uint64_t>() + e[1], 8, cudaMemcpyDeviceToHost));
    fail(QT_EDUP, "block (brow=%u, bcol=%u) is listed twice", morton_row(k), morton_col(k));
  }
  k_heads16<<<gfor(n), kT, 0, st>>>(k1.as<uint64_t>(), n, head.as<int32_t>());
  QT_LAUNCH_CHECK(ctx);
  incl_sum(ctx, head.as<int32_t>(), incl.as<int32_t>(), n);
  const int64_t nc = read_scalar(ctx, incl.as<int32_t>() + (n - 1));
  const size_t es = elem_size(M->dtype);
  M->nb = nc;
  M->key.alloc(8 * nc, st);
  M->sub.alloc(nc, st);
  M->pool.alloc(nc * 1024 * es, st);
  QT_CUDA(cudaMemsetAsync(M->pool.p, 0, nc * 1024 * es, st));
  k_containers16<<<gfor(n), kT, 0, st>>>(k1.as<uint64_t>(), head.as<int32_t>(), incl.as<int32_t>(), n,
                                         M->key.as<uint64_t>(), M->sub.as<uint8_t>());
  QT_LAUNCH_CHECK(ctx);
  const unsigned g = (unsigned)std::min<int64_t>(n, 148 * 32);
  if (M->dtype == QT_F64)
    k_fill16<double><<<g, 256, 0, st>>>((const double*)vals, k1.as<uint64_t>(), i1.as<int32_t>(), incl.as<int32_t>(),
                                        n, M->pool.as<double>());
  else
    k_fill16<float><<<g, 256, 0, st>>>((const float*)vals, k1.as<uint64_t>(), i1.as<int32_t>(), incl.as<int32_t>(), n,
                                       M->pool.as<float>());
  QT_LAUNCH_CHECK(ctx);
  build_levels(M);
}

void read_back16(qt_mat M, int32_t* brow, int32_t* bcol, void* vals) {
  qt_ctx ctx = M->ctx;
  cudaStream_t st = ctx->stream;
  if (M->nb == 0 || M->nb16 == 0) return;
  DevBuf incl;
  const int64_t n = user_scan16(M, incl);
  const size_t es = elem_size(M->dtype);
  DevBuf rm(8 * n, st), rm2(8 * n, st), src(4 * n, st), src2(4 * n, st);
  k_terms16<<<gfor(M->nb), kT, 0, st>>>(M->key.as<uint64_t>(), M->sub.as<uint8_t>(), incl.as<int32_t>(), M->nb,
                                        rm.as<uint64_t>(), src.as<int32_t>());
  QT_LAUNCH_CHECK(ctx);
  sort_pairs(ctx, rm.as<uint64_t>(), rm2.as<uint64_t>(), src.as<int32_t>(), src2.as<int32_t>(), n, 64);
  const bool dr = brow && is_device_ptr(brow), dc = bcol && is_device_ptr(bcol), dv = vals && is_device_ptr(vals);
  DevBuf sr, sc, sv;
  int32_t* obr = brow ? (dr ? brow : (sr.alloc(n * 4, st), sr.as<int32_t>())) : nullptr;
  int32_t* obc = bcol ? (dc ? bcol : (sc.alloc(n * 4, st), sc.as<int32_t>())) : nullptr;
  void* ov = vals ? (dv ? vals : (sv.alloc(n * 256 * es, st), sv.p)) : nullptr;
  const unsigned g = (unsigned)std::min<int64_t>(n, 148 * 32);
  if (M->dtype == QT_F64)
    k_unpack16<double><<<g, 256, 0, st>>>(M->pool.as<double>(), rm2.as<uint64_t>(), src2.as<int32_t>(), n, obr, obc,
                                          (double*)ov);
  else
    k_unpack16<float><<<g, 256, 0, st>>>(M->pool.as<float>(), rm2.as<uint64_t>(), src2.as<int32_t>(), n, obr, obc,
                                         (float*)ov);
  QT_LAUNCH_CHECK(ctx);
  if (brow && !dr) QT_CUDA(cudaMemcpyAsync(brow, obr, n * 4, cudaMemcpyDeviceToHost, st));
  if (bcol && !dc) QT_CUDA(cudaMemcpyAsync(bcol, obc, n * 4, cudaMemcpyDeviceToHost, st));
  if (vals && !dv) QT_CUDA(cudaMemcpyAsync(vals, ov, n * 256 * es, cudaMemcpyDeviceToHost, st));
  QT_CUDA(cudaStreamSynchronize(st));
}

void truncate_terms16(qt_mat A, DevBuf& nrm, DevBuf& rm) {
  qt_ctx ctx = A->ctx;
  cudaStream_t st = ctx->stream;
  const int64_t n = A->nb16;
  nrm.alloc(8 * std::max<int64_t>(n, 1), st);
  rm.alloc(8 * std::max<int64_t>(n, 1), st);
  if (n == 0 || A->nb == 0) return;
  DevBuf incl, src(4 * n, st);
  user_scan16(A, incl);
  k_terms16<<<gfor(A->nb), kT, 0, st>>>(A->key.as<uint64_t>(), A->sub.as<uint8_t>(), incl.as<int32_t>(), A->nb,
                                        rm.as<uint64_t>(), src.as<int32_t>());
  QT_LAUNCH_CHECK(ctx);
  if (A->dtype == QT_F64)
    k_norm16<double><<<gfor(n), kT, 0, st>>>(A->pool.as<double>(), src.as<int32_t>(), n, nrm.as<double>());
  else
    k_norm16<float><<<gfor(n), kT, 0, st>>>(A->pool.as<float>(), src.as<int32_t>(), n, nrm.as<double>());
  QT_LAUNCH_CHECK(ctx);
}

qt_mat apply_keep16(qt_mat A, const uint8_t* keep_user) {
  qt_ctx ctx = A->ctx;
  cudaStream_t st = ctx->stream;
  if (A->nb == 0) return select_blocks(A, nullptr);
  DevBuf incl, nsub(A->nb, st), keep(A->nb, st);
  user_scan16(A, incl);
  k_newmask16<<<gfor(A->nb), kT, 0, st>>>(A->sub.as<uint8_t>(), incl.as<int32_t>(), keep_user, A->nb,
                                          nsub.as<uint8_t>(), keep.as<uint8_t>());
  QT_LAUNCH_CHECK(ctx);
  // select the surviving containers with their new masks, then clear the dropped quadrants
  DevBuf old = std::move(A->sub);
  A->sub = std::move(nsub);
  qt_mat R;
  try {
    R = select_blocks(A, keep.as<uint8_t>());
  } catch (...) {
    A->sub = std::move(old);
    throw;
  }
  A->sub = std::move(old);
  if (R->nb > 0) {
    const unsigned g = (unsigned)std::min<int64_t>(R->nb, 148 * 16);
    if (R->dtype == QT_F64)
      k_zero_absent16<double><<<g, 256, 0, st>>>(R->pool.as<double>(), R->sub.as<uint8_t>(), R->nb);
    else
      k_zero_absent16<float><<<g, 256, 0, st>>>(R->pool.as<float>(), R->sub.as<uint8_t>(), R->nb);
    QT_LAUNCH_CHECK(ctx);
  }
  return R;
}

// masks of a selection (select_blocks): out[incl[t]-1] = in[t] for kept t; returns the 16-block count
int64_t compact_sub16(qt_ctx ctx, const uint8_t* keep, const int32_t* incl, const uint8_t* in, int64_t n, int64_t kept,
                      DevBuf& out) {
  cudaStream_t st = ctx->stream;
  out.alloc(std::max<int64_t>(kept, 1), st);
  if (kept == 0) return 0;
  k_compact_u8<<<gfor(n), kT, 0, st>>>(keep, incl, in, n, out.as<uint8_t>());
  QT_LAUNCH_CHECK(ctx);
  DevBuf cnt(4 * kept, st), inc(4 * kept, st);
  k_popc<<<gfor(kept), kT, 0, st>>>(out.as<uint8_t>(), kept, cnt.as<int32_t>());
  QT_LAUNCH_CHECK(ctx);
  incl_sum(ctx, cnt.as<int32_t>(), inc.as<int32_t>(), kept);
  return read_scalar(ctx, inc.as<int32_t>() + (kept - 1));
}

void cmask16(qt_ctx ctx, int64_t ntiles, const int32_t* ts, const int32_t* pa, const int32_t* pb, const int4* cA,
             const int4* cB, const int4* cC, const uint8_t* subA, const uint8_t* subB, int trans,
             const uint64_t* keyC, uint8_t* subC, int64_t nc, int64_t out[4], const double* n16A,
             const double* n16B, double tau2) {
  cudaStream_t st = ctx->stream;
  DevBuf cnt(32, st);
  QT_CUDA(cudaMemsetAsync(cnt.p, 0, 32, st));
  QT_CUDA(cudaMemsetAsync(subC, 0, std::max<int64_t>(nc, 1), st));
  if (ntiles > 0) {
    k_cmask16<<<(unsigned)((ntiles + 7) / 8), 256, 0, st>>>(ts, pa, pb, ntiles, cA, cB, cC, subA, subB, trans, keyC,
                                                           subC, cnt.as<unsigned long long>(), n16A, n16B, tau2);
    QT_LAUNCH_CHECK(ctx);
  }
  unsigned long long h[4];
  read_small(ctx, h, cnt.p, 32);
  for (int i = 0; i < 4; ++i) out[i] = (int64_t)h[i];
}

void check_upper16(qt_mat M) {
  qt_ctx ctx = M->ctx;
  if (M->nb == 0) return;
  unsigned long long* bad = ctx->counters.as<unsigned long long>();
  QT_CUDA(cudaMemsetAsync(bad, 0xff, 8, ctx->stream));
  k_lower16<<<gfor(M->nb), kT, 0, ctx->stream>>>(M->key.as<uint64_t>(), M->sub.as<uint8_t>(), M->nb, bad);
  QT_LAUNCH_CHECK(ctx);
  const unsigned long long b = read_scalar(ctx, bad);
  if (b != ~0ull) {
    uint64_t k;
    uint8_t m;
    QT_CUDA(cudaMemcpy(&k, M->key.as<uint64_t>() + b, 8, cudaMemcpyDeviceToHost));
    QT_CUDA(cudaMemcpy(&m, M->sub.as<uint8_t>() + b, 1, cudaMemcpyDeviceToHost));
    const uint32_t R = morton_row(k), C = morton_col(k);
    const int q = R > C ? __builtin_ctz(m) : 2;
    fail(QT_EINVAL, "symmetric square needs upper-triangular block storage; block (brow=%u, bcol=%u) is below "
         "the diagonal", 2 * R + (q >> 1), 2 * C + (q & 1));
  }
}

qt_mat symm_prepare16(qt_mat U) {
  qt_ctx ctx = U->ctx;
  DevBuf keep(std::max<int64_t>(U->nb, 1), ctx->stream);
  if (U->nb > 0) QT_CUDA(cudaMemsetAsync(keep.p, 1, U->nb, ctx->stream));
  qt_mat X = select_blocks(U, keep.as<uint8_t>());  // a copy (U itself stays as the caller gave it)
  if (X->nb > 0) {
    const unsigned g = (unsigned)std::min<int64_t>(X->nb, 148 * 16);
    if (X->dtype == QT_F64)
      k_complete_diag16<double><<<g, 256, 0, ctx->stream>>>(X->key.as<uint64_t>(), X->sub.as<uint8_t>(), X->nb,
                                                            X->pool.as<double>());
    else
      k_complete_diag16<float><<<g, 256, 0, ctx->stream>>>(X->key.as<uint64_t>(), X->sub.as<uint8_t>(), X->nb,
                                                           X->pool.as<float>());
    QT_LAUNCH_CHECK(ctx);
  }
  return X;
}

void symm_finish16(qt_mat C) {
  qt_ctx ctx = C->ctx;
  if (C->nb == 0) return;
  const unsigned g = (unsigned)std::min<int64_t>(C->nb, 148 * 16);
  if (C->dtype == QT_F64)
    k_drop_lower16<double><<<g, 256, 0, ctx->stream>>>(C->key.as<uint64_t>(), C->nb, C->pool.as<double>());
  else
    k_drop_lower16<float><<<g, 256, 0, ctx->stream>>>(C->key.as<uint64_t>(), C->nb, C->pool.as<float>());
  QT_LAUNCH_CHECK(ctx);
}

qt_mat drop_empty16(qt_mat C) {
  qt_ctx ctx = C->ctx;
  DevBuf keep(std::max<int64_t>(C->nb, 1), ctx->stream);
  if (C->nb > 0) {
    k_nonempty<<<gfor(C->nb), kT, 0, ctx->stream>>>(C->sub.as<uint8_t>(), C->nb, keep.as<uint8_t>());
    QT_LAUNCH_CHECK(ctx);
  }
  return select_blocks(C, keep.as<uint8_t>());
}

}  // namespace qt
