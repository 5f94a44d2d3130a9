// Device helpers shared by the libqtmm kernels (Morton keys, internal block
// layout).  Not shared with the oracle.
#pragma once
#include <stdint.h>

namespace qt {

// Morton key of a block: row bits at odd positions, column bits at even
// positions, so key >> 2 is the parent node and key & 3 = 2*rowbit + colbit is
// the child slot in row-major order (NW, NE, SW, SE) — the quadtree split of
// §3.1 addressed by coordinates.
__host__ __device__ inline uint64_t spread_bits(uint32_t x) {
  uint64_t v = x;
  v = (v | (v << 16)) & 0x0000FFFF0000FFFFull;
  v = (v | (v << 8)) & 0x00FF00FF00FF00FFull;
  v = (v | (v << 4)) & 0x0F0F0F0F0F0F0F0Full;
  v = (v | (v << 2)) & 0x3333333333333333ull;
  v = (v | (v << 1)) & 0x5555555555555555ull;
  return v;
}
__host__ __device__ inline uint32_t compact_bits(uint64_t v) {
  v &= 0x5555555555555555ull;
  v = (v | (v >> 1)) & 0x3333333333333333ull;
  v = (v | (v >> 2)) & 0x0F0F0F0F0F0F0F0Full;
  v = (v | (v >> 4)) & 0x00FF00FF00FF00FFull;
  v = (v | (v >> 8)) & 0x0000FFFF0000FFFFull;
  v = (v | (v >> 16)) & 0x00000000FFFFFFFFull;
  return (uint32_t)v;
}
__host__ __device__ inline uint64_t morton(uint32_t row, uint32_t col) {
  return (spread_bits(row) << 1) | spread_bits(col);
}
__host__ __device__ inline uint32_t morton_row(uint64_t k) { return compact_bits(k >> 1); }
__host__ __device__ inline uint32_t morton_col(uint64_t k) { return compact_bits(k); }

// Internal FP64 block layout (32x32): element (r, c) lives at
//   r*32 + (c ^ ((r & 3) << 2)),
// i.e. the eight 32-byte chunks of each 256-byte row are XOR-permuted by
// (r & 3).  With this layout the warp-wide fragment loads of
// mma.sync.m8n8k4.f64 — A: (row g, col t), B: (row t, col g), g = lane>>2,
// t = lane&3 — hit every 8-byte bank pair exactly twice (2 wavefronts, the
// minimum for 256 bytes), and the accumulator pairs stay 16-byte contiguous.
__host__ __device__ inline int swz64(int r, int c) { return r * 32 + (c ^ ((r & 3) << 2)); }

// Internal FP32 block layout (32x32): rows of 128 bytes, the eight 16-byte
// chunks of row r XOR-permuted by (r & 7) — the canonical 128-byte swizzle of
// the tcgen05 shared-memory descriptors.  A 4 KiB block copied unchanged to a
// 1024-byte-aligned smem address is then, at once, a K-major SW128 tile of the
// A operand (rows = M, 32 fp32 of K per row) and an MN-major SW128 tile of the
// B operand (rows = K, 32 fp32 of N per row): one pool serves both operands.
__host__ __device__ inline int swz32(int r, int c) {
  return r * 32 + ((((c >> 2) ^ (r & 7)) << 2) | (c & 3));
}

// Child slots of op(X): the transpose of a node has its off-diagonal children
// swapped (slot 1 <-> 2) and each child transposed in turn — so for a globally
// transposed operand (C = A^T B etc.) only the slot order changes.
__device__ __forceinline__ int4 ldchild(const int4* __restrict__ tab, int idx, bool trans) {
  int4 c = tab[idx];
  if (trans) {
    const int t = c.y;
    c.y = c.z;
    c.z = t;
  }
  return c;
}

// Symmetric square (§3.3): A = B = the symmetric matrix whose upper
// block triangle U is stored.  A node of the full matrix is a reference
// (U node index, diagonal?, transposed?) = idx*4 + diag*2 + t: the children of
// a diagonal node D are (D00 diag, D01, D01^T, D11 diag) — its stored (1,0)
// slot is NIL in upper storage — and the children of a transposed node are the
// slot-swapped transposes of its children.  NIL = -1.
__device__ __forceinline__ int sref(int idx, int diag, int t) {
  return idx < 0 ? -1 : ((idx << 2) | (diag << 1) | t);
}
// op_children split into the table load (row tab[ref >> 2] when symmetric,
// tab[ref] otherwise) and the transform of the loaded row, so a caller can
// issue the load early and transform later.
__device__ __forceinline__ int4 op_xform(int4 c, int ref, bool trans, bool sym) {
  if (!sym) {
    if (trans) {
      const int t = c.y;
      c.y = c.z;
      c.z = t;
    }
    return c;
  }
  const int diag = (ref >> 1) & 1, t = ref & 1;
  if (diag) return make_int4(sref(c.x, 1, 0), sref(c.y, 0, 0), sref(c.y, 0, 1), sref(c.w, 1, 0));
  if (t) return make_int4(sref(c.x, 0, 1), sref(c.z, 0, 1), sref(c.y, 0, 1), sref(c.w, 0, 1));
  return make_int4(sref(c.x, 0, 0), sref(c.y, 0, 0), sref(c.z, 0, 0), sref(c.w, 0, 0));
}
__device__ __forceinline__ int4 op_children(const int4* __restrict__ tab, int ref, bool trans,
                                            bool sym) {
  return op_xform(tab[sym ? (ref >> 2) : ref], ref, trans, sym);
}

// Block size 16 (qt_bs16.cu): quadrant masks of 32-blocks, bit 2i+j = 16-block (i,j).
// mask of the transposed 32-block: quadrant (i,j) -> (j,i)
__host__ __device__ __forceinline__ int mask_t(int m) { return (m & 9) | ((m & 2) << 1) | ((m & 4) >> 1); }
// some 16-block product x(r,s)·y(s,c) exists (column s of x meets row s of y)
__host__ __device__ __forceinline__ bool mask_meet(int x, int y) {
  return ((x & 5) && (y & 3)) || ((x & 10) && (y & 12));
}

// Block size 16 with norm screening: the 16-block products of the container
// pair (x, y) (masks as read) that exist and pass ||x_rh||^2 ||y_hc||^2 >= tau^2
// (squared 16-block norms n16x[2r+h], n16y[2h+c]).  bit 2*(2r+c)+h = product
// x(r,h)·y(h,c) of C quadrant (r,c).
__device__ __forceinline__ int screen16(int x, int y, const double* __restrict__ nx, const double* __restrict__ ny,
                                        double tau2) {
  int out = 0;
#pragma unroll
  for (int r = 0; r < 2; ++r)
#pragma unroll
    for (int c = 0; c < 2; ++c)
#pragma unroll
      for (int h = 0; h < 2; ++h)
        if (((x >> (2 * r + h)) & 1) && ((y >> (2 * h + c)) & 1) && __dmul_rn(nx[2 * r + h], ny[2 * h + c]) >= tau2)
          out |= 1 << (2 * (2 * r + c) + h);
  return out;
}

}  // namespace qt
