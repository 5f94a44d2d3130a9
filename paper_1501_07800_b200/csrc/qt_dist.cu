// Multi-GPU multiply (X1-X3): locality-aware row strips + NCCL point-to-point
// exchange of exactly the B block rows a rank's output needs.
//
// Paper: output work and data are kept where the data is (the quadtree keeps
// locality, P:82-97 Fig. fig:random_destruction, §5.2) and each
// process fetches the remote chunks its tasks need; "data received by each
// process" is the central measured quantity (§6.3).  CHT-MPI
// moves chunks by work stealing + MPI fetches; here the mapping
// is static: rank g owns block rows [b_g, b_{g+1}) of A, B and C (output
// subtrees aligned to quadtree rows), A stays put, and rank g receives from
// their owners the B block rows K in cols(A[rows_g, :]) outside its own range
// — one request/response round over NCCL send/recv (NVLink / NVSwitch).
//
// Protocol (all int32 unless noted):
//   0. allgather of the P x P matrix of requested-row counts (int64)
//   1. requester -> owner : the sorted list of requested block rows
//   2. owner -> requester : number of blocks in each requested row
//   3. owner -> requester : block columns, then the block values (internal
//      layout, 8 KiB per FP64 block) — the payload
// The requester merges the received blocks with its local B into B_ext (a
// quadtree over the union, Morton-sorted; the level L-1 child table stores
// pool ids, ids >= nb_local point into the received payload) and runs the
// single-GPU multiply A_local * B_ext.
#include <dlfcn.h>
#include <nccl.h>

#include <condition_variable>
#include <deque>
#include <memory>
#include <mutex>
#include <tuple>

#include <algorithm>
#include <cub/cub.cuh>

#include "qt_common.cuh"
#include "qt_internal.h"

namespace qt {

// ------------------------------------------------------------------ NCCL

struct NcclApi {
  bool ok = false;
  std::string why;
  void* h = nullptr;
  decltype(&ncclGetUniqueId) GetUniqueId = nullptr;
  decltype(&ncclCommInitRank) CommInitRank = nullptr;
  decltype(&ncclCommDestroy) CommDestroy = nullptr;
  decltype(&ncclSend) Send = nullptr;
  decltype(&ncclRecv) Recv = nullptr;
  decltype(&ncclGroupStart) GroupStart = nullptr;
  decltype(&ncclGroupEnd) GroupEnd = nullptr;
  decltype(&ncclAllGather) AllGather = nullptr;
  decltype(&ncclAllReduce) AllReduce = nullptr;
  decltype(&ncclGetErrorString) GetErrorString = nullptr;
  decltype(&ncclCommCount) CommCount = nullptr;
};

static NcclApi& nccl() {
  static NcclApi api;
  static bool tried = false;
  if (tried) {
    if (!api.ok) fail(QT_ENCCL, "NCCL unavailable: %s", api.why.c_str());
    return api;
  }
  tried = true;
  api.h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
  if (!api.h) api.h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
  if (!api.h) {
    api.why = dlerror() ? dlerror() : "dlopen failed";
    fail(QT_ENCCL, "cannot load libnccl.so.2: %s", api.why.c_str());
  }
#define LOAD(name)                                                       \
  api.name = (decltype(api.name))dlsym(api.h, "nccl" #name);             \
  if (!api.name) {                                                       \
    api.why = "missing symbol nccl" #name;                               \
    fail(QT_ENCCL, "%s", api.why.c_str());                               \
  }
  LOAD(GetUniqueId)
  LOAD(CommInitRank)
  LOAD(CommDestroy)
  LOAD(Send)
  LOAD(Recv)
  LOAD(GroupStart)
  LOAD(GroupEnd)
  LOAD(AllGather)
  LOAD(AllReduce)
  LOAD(GetErrorString)
  LOAD(CommCount)
#undef LOAD
  api.ok = true;
  return api;
}

#define NCCL_CALL(x)                                                                       \
  do {                                                                                     \
    ncclResult_t r_ = (x);                                                                 \
    if (r_ != ncclSuccess) fail(QT_ENCCL, "%s: %s", #x, nccl().GetErrorString(r_));        \
  } while (0)

// ------------------------------------------------------------------ transport
//
// The exchange talks to a Transport: NCCL in production (one process per GPU,
// NVLink / NVSwitch), or — for testing the same orchestration on a single GPU —
// a loopback between rank threads of one process, where a device-to-device
// cudaMemcpyAsync ordered by CUDA events stands in for each send/recv pair.
// Kernels never wait on other ranks in either transport.

struct Transport {
  virtual ~Transport() = default;
  virtual void allgather_i64(const int64_t* send_host, int64_t* recv_host, int count) = 0;
  virtual void group_start() = 0;
  virtual void send(const void* buf, size_t bytes, int peer) = 0;
  virtual void recv(void* buf, size_t bytes, int peer) = 0;
  virtual void group_end() = 0;
  // ranks of the underlying communicator (NCCL: ncclCommCount) and kind (1 NCCL, 2 loopback)
  virtual int comm_size() = 0;
  virtual int kind() const = 0;
  // stream the following send/recv groups are ordered on (null: the ctx stream)
  void set_stream(cudaStream_t s) { cur_ = s; }
  cudaStream_t cur(qt_ctx ctx) const { return cur_ ? cur_ : ctx->stream; }

 protected:
  cudaStream_t cur_ = nullptr;
};

struct NcclTransport : Transport {
  qt_ctx ctx;
  ncclComm_t comm = nullptr;
  NcclTransport(qt_ctx c, const void* uid) : ctx(c) {
    NcclApi& N = nccl();
    ncclUniqueId id;
    memcpy(&id, uid, sizeof(id));
    NCCL_CALL(N.CommInitRank(&comm, ctx->world, id, ctx->rank));
  }
  ~NcclTransport() override {
    if (comm) nccl().CommDestroy(comm);
  }
  void allgather_i64(const int64_t* send_host, int64_t* recv_host, int count) override {
    NcclApi& N = nccl();
    DevBuf s(8 * count, ctx->stream), r(8ll * count * ctx->world, ctx->stream);
    QT_CUDA(cudaMemcpyAsync(s.p, send_host, 8 * count, cudaMemcpyHostToDevice, ctx->stream));
    NCCL_CALL(N.AllGather(s.p, r.p, count, ncclInt64, comm, ctx->stream));
    read_small(ctx, recv_host, r.p, 8ll * count * ctx->world);
  }
  void group_start() override { NCCL_CALL(nccl().GroupStart()); }
  void send(const void* buf, size_t bytes, int peer) override {
    NCCL_CALL(nccl().Send(buf, bytes, ncclInt8, peer, comm, cur(ctx)));
  }
  void recv(void* buf, size_t bytes, int peer) override {
    NCCL_CALL(nccl().Recv(buf, bytes, ncclInt8, peer, comm, cur(ctx)));
  }
  void group_end() override { NCCL_CALL(nccl().GroupEnd()); }
  int comm_size() override {
    int n = 0;
    NCCL_CALL(nccl().CommCount(comm, &n));
    return n;
  }
  int kind() const override { return 1; }
};

// Shared state of the loopback ranks (one per process, created by the caller).
struct LoopHub {
  int P;
  std::mutex mu;
  std::condition_variable cv;
  struct Msg {
    const void* src;
    size_t bytes;
    cudaEvent_t ready;  // sender's data is complete
    cudaEvent_t done;   // receiver's copy is complete
    bool taken = false, copied = false;
  };
  std::vector<std::deque<std::shared_ptr<Msg>>> q;  // [src*P + dst]
  // allgather
  std::vector<int64_t> ag;
  int ag_count = 0, ag_arrived = 0, ag_left = 0;
  uint64_t ag_gen = 0;
  explicit LoopHub(int p) : P(p), q((size_t)p * p) {}
};

struct LoopTransport : Transport {
  qt_ctx ctx;
  LoopHub* hub;
  std::vector<std::shared_ptr<LoopHub::Msg>> posted;
  std::vector<std::tuple<void*, size_t, int>> pending;
  LoopTransport(qt_ctx c, LoopHub* h) : ctx(c), hub(h) {}
  int comm_size() override { return hub->P; }
  int kind() const override { return 2; }
  void allgather_i64(const int64_t* send_host, int64_t* recv_host, int count) override {
    std::unique_lock<std::mutex> lk(hub->mu);
    // wait until the previous allgather has been fully consumed
    hub->cv.wait(lk, [&] { return hub->ag_left == 0; });
    if (hub->ag_arrived == 0) {
      hub->ag.assign((size_t)count * hub->P, 0);
      hub->ag_count = count;
    }
    if (hub->ag_count != count) fail(QT_ESTATE, "loopback allgather size mismatch");
    for (int i = 0; i < count; ++i) hub->ag[(size_t)ctx->rank * count + i] = send_host[i];
    uint64_t gen = hub->ag_gen;
    if (++hub->ag_arrived == hub->P) {
      hub->ag_arrived = 0;
      hub->ag_left = hub->P;
      ++hub->ag_gen;
      hub->cv.notify_all();
    } else {
      hub->cv.wait(lk, [&] { return hub->ag_gen != gen; });
    }
    for (size_t i = 0; i < hub->ag.size(); ++i) recv_host[i] = hub->ag[i];
    if (--hub->ag_left == 0) hub->cv.notify_all();
  }
  void group_start() override {
    posted.clear();
    pending.clear();
  }
  void send(const void* buf, size_t bytes, int peer) override {
    auto m = std::make_shared<LoopHub::Msg>();
    m->src = buf;
    m->bytes = bytes;
    QT_CUDA(cudaEventCreateWithFlags(&m->ready, cudaEventDisableTiming));
    QT_CUDA(cudaEventCreateWithFlags(&m->done, cudaEventDisableTiming));
    QT_CUDA(cudaEventRecord(m->ready, cur(ctx)));
    {
      std::lock_guard<std::mutex> lk(hub->mu);
      hub->q[(size_t)ctx->rank * hub->P + peer].push_back(m);
    }
    hub->cv.notify_all();
    posted.push_back(m);
  }
  void recv(void* buf, size_t bytes, int peer) override { pending.emplace_back(buf, bytes, peer); }
  void group_end() override {
    // receives in program order per peer
    for (auto& [buf, bytes, peer] : pending) {
      std::shared_ptr<LoopHub::Msg> m;
      {
        std::unique_lock<std::mutex> lk(hub->mu);
        auto& dq = hub->q[(size_t)peer * hub->P + ctx->rank];
        hub->cv.wait(lk, [&] { return !dq.empty(); });
        m = dq.front();
        dq.pop_front();
      }
      if (m->bytes != bytes)
        fail(QT_ESTATE, "loopback size mismatch: rank %d expects %zu bytes from %d, got %zu",
             ctx->rank, bytes, peer, m->bytes);
      QT_CUDA(cudaStreamWaitEvent(cur(ctx), m->ready, 0));
      QT_CUDA(cudaMemcpyAsync(buf, m->src, bytes, cudaMemcpyDeviceToDevice, cur(ctx)));
      QT_CUDA(cudaEventRecord(m->done, cur(ctx)));
      {
        std::lock_guard<std::mutex> lk(hub->mu);
        m->copied = true;
      }
      hub->cv.notify_all();
    }
    pending.clear();
    // a send buffer may be reused only after the receiver's copy
    for (auto& m : posted) {
      {
        std::unique_lock<std::mutex> lk(hub->mu);
        hub->cv.wait(lk, [&] { return m->copied; });
      }
      QT_CUDA(cudaStreamWaitEvent(cur(ctx), m->done, 0));
    }
    QT_CUDA(cudaStreamSynchronize(cur(ctx)));
    for (auto& m : posted) {
      cudaEventDestroy(m->ready);
      cudaEventDestroy(m->done);
    }
    posted.clear();
  }
};

static Transport* T(qt_ctx ctx) { return static_cast<Transport*>(ctx->transport); }

void dist_init(qt_ctx ctx, const void* uid) { ctx->transport = new NcclTransport(ctx, uid); }

void dist_init_loopback(qt_ctx ctx, void* hub) {
  LoopHub* h = static_cast<LoopHub*>(hub);
  if (h->P != ctx->world) fail(QT_EINVAL, "hub for %d ranks, world is %d", h->P, ctx->world);
  ctx->transport = new LoopTransport(ctx, h);
}

void dist_finalize(qt_ctx ctx) {
  delete T(ctx);
  ctx->transport = nullptr;
}

int transport_info(qt_ctx ctx, int* kind) {
  if (!ctx->transport) {
    *kind = 0;
    return 1;
  }
  *kind = T(ctx)->kind();
  return T(ctx)->comm_size();
}

void* loop_hub_create(int P) { return new LoopHub(P); }
void loop_hub_destroy(void* h) { delete static_cast<LoopHub*>(h); }

void allgather_i64(qt_ctx ctx, const int64_t* send_host, int64_t* recv_host, int count) {
  T(ctx)->allgather_i64(send_host, recv_host, count);
}

// ------------------------------------------------------------------ kernels

namespace {

constexpr int kT = 256;
inline unsigned gfor(int64_t n) { return (unsigned)std::max<int64_t>(1, (n + kT - 1) / kT); }

// flag[K] = 1 for every block column K of A outside [lo, hi)
__global__ void k_mark_cols(const uint64_t* __restrict__ key, int64_t nb, int32_t lo, int32_t hi,
                            int32_t* __restrict__ flag) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < nb;
       t += (int64_t)gridDim.x * blockDim.x) {
    int32_t c = (int32_t)morton_col(key[t]);
    if (c < lo || c >= hi) flag[c] = 1;
  }
}

__global__ void k_scatter_flagged(const int32_t* __restrict__ flag, const int32_t* __restrict__ incl,
                                  int32_t n, int32_t* __restrict__ out) {
  int32_t t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t < n && flag[t]) out[incl[t] - 1] = t;
}

// flag[t] = 1 if block t's row is in [lo, hi)
__global__ void k_flag_rows(const uint64_t* __restrict__ key, int64_t nb, int32_t lo, int32_t hi,
                            uint8_t* __restrict__ keep) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < nb;
       t += (int64_t)gridDim.x * blockDim.x) {
    int32_t r = (int32_t)morton_row(key[t]);
    keep[t] = (r >= lo && r < hi) ? 1 : 0;
  }
}

__global__ void k_rm_keys(const uint64_t* __restrict__ key, int64_t nb, uint64_t* __restrict__ rm,
                          int32_t* __restrict__ iota) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < nb;
       t += (int64_t)gridDim.x * blockDim.x) {
    uint64_t k = key[t];
    rm[t] = ((uint64_t)morton_row(k) << 32) | morton_col(k);
    iota[t] = (int32_t)t;
  }
}

// row_cnt[row] += 1 per block (rows of the whole grid)
__global__ void k_row_hist(const uint64_t* __restrict__ rm_sorted, int64_t nb,
                           int32_t* __restrict__ row_cnt) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < nb;
       t += (int64_t)gridDim.x * blockDim.x)
    atomicAdd(&row_cnt[(int32_t)(rm_sorted[t] >> 32)], 1);
}

// counts of requested rows
__global__ void k_req_counts(const int32_t* __restrict__ rows, int32_t n,
                             const int32_t* __restrict__ row_cnt, int32_t* __restrict__ out) {
  int32_t t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t < n) out[t] = row_cnt[rows[t]];
}

// one warp per requested row: copy its blocks (columns + values) to the
// packed buffers at the row's offset
__global__ void k_pack(const int32_t* __restrict__ rows, int32_t n, const int32_t* __restrict__ offs,
                       const int32_t* __restrict__ row_ptr, const int32_t* __restrict__ order,
                       const uint64_t* __restrict__ rm_sorted, const uint4* __restrict__ pool,
                       int vec_per_block, int32_t* __restrict__ cols, uint4* __restrict__ payload,
                       const uint8_t* __restrict__ sub_in, uint8_t* __restrict__ sub_out) {
  int lane = threadIdx.x & 31;
  int64_t w = blockIdx.x * (int64_t)(blockDim.x / 32) + threadIdx.x / 32;
  if (w >= n) return;
  int32_t r = rows[w];
  int32_t s0 = row_ptr[r], s1 = row_ptr[r + 1];
  int32_t o = offs[w];
  for (int32_t s = s0; s < s1; ++s) {
    int32_t src = order[s];
    if (lane == 0) cols[o + (s - s0)] = (int32_t)(rm_sorted[s] & 0xffffffffu);
    if (lane == 0 && sub_in) sub_out[o + (s - s0)] = sub_in[src];
    const uint4* sp = pool + (int64_t)src * vec_per_block;
    uint4* dp = payload + (int64_t)(o + (s - s0)) * vec_per_block;
    for (int e = lane; e < vec_per_block; e += 32) dp[e] = sp[e];
  }
}

// Morton keys of the received blocks; ids continue after the local blocks
__global__ void k_remote_keys(const int32_t* __restrict__ rows, int32_t n,
                              const int32_t* __restrict__ offs, const int32_t* __restrict__ cols,
                              uint64_t* __restrict__ key, int32_t* __restrict__ ids, int64_t nb_local) {
  int lane = threadIdx.x & 31;
  int64_t w = blockIdx.x * (int64_t)(blockDim.x / 32) + threadIdx.x / 32;
  if (w >= n) return;
  int32_t r = rows[w];
  for (int32_t e = offs[w] + lane; e < offs[w + 1]; e += 32) {
    key[e] = morton((uint32_t)r, (uint32_t)cols[e]);
    ids[e] = (int32_t)(nb_local + e);
  }
}

__global__ void k_iota(int32_t* __restrict__ out, int64_t n) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n;
       t += (int64_t)gridDim.x * blockDim.x)
    out[t] = (int32_t)t;
}

// one warp per tile: local[t] = 0 if a task of tile t reads a received B
// block (block id >= split), through the B node's children (and, for tiles
// at level L-2, its children's children), else 1; ids[t] = t
__global__ void k_tile_local(const int32_t* __restrict__ ts, const int32_t* __restrict__ pb, int64_t ntiles,
                             const int4* __restrict__ cbt, const int4* __restrict__ cb1, int64_t split,
                             uint8_t* __restrict__ local, int32_t* __restrict__ ids) {
  const int lane = threadIdx.x & 31;
  const int64_t t = blockIdx.x * (int64_t)(blockDim.x / 32) + threadIdx.x / 32;
  if (t >= ntiles) return;
  auto far = [&](int4 c) { return c.x >= split || c.y >= split || c.z >= split || c.w >= split; };
  bool rem = false;
  for (int32_t p = ts[t] + lane; p < ts[t + 1] && !rem; p += 32) {
    const int4 c = cbt[pb[p]];
    if (!cb1) {
      rem = far(c);
    } else {
      const int n[4] = {c.x, c.y, c.z, c.w};
      for (int i = 0; i < 4; ++i)
        if (n[i] >= 0 && far(cb1[n[i]])) rem = true;
    }
  }
  rem = __any_sync(0xffffffffu, rem);
  if (lane == 0) {
    local[t] = rem ? 0 : 1;
    ids[t] = (int32_t)t;
  }
}

template <class T>
void excl_sum(qt_ctx ctx, const T* in, T* out, int64_t n) {
  size_t tb = 0;
  QT_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tb, in, out, (int)n, ctx->stream));
  void* tmp = scratch(ctx, tb);
  QT_CUDA(cub::DeviceScan::ExclusiveSum(tmp, tb, in, out, (int)n, ctx->stream));
  ctx->launches += 2;
}
template <class T>
void incl_sum(qt_ctx ctx, const T* in, T* out, int64_t n) {
  size_t tb = 0;
  QT_CUDA(cub::DeviceScan::InclusiveSum(nullptr, tb, in, out, (int)n, ctx->stream));
  void* tmp = scratch(ctx, tb);
  QT_CUDA(cub::DeviceScan::InclusiveSum(tmp, tb, in, out, (int)n, ctx->stream));
  ctx->launches += 2;
}
template <class V>
void sort_pairs(qt_ctx ctx, const uint64_t* kin, uint64_t* kout, const V* vin, V* vout, int64_t n,
                int bits) {
  size_t tb = 0;
  QT_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tb, kin, kout, vin, vout, (int)n, 0, bits,
                                          ctx->stream));
  void* tmp = scratch(ctx, tb);
  QT_CUDA(cub::DeviceRadixSort::SortPairs(tmp, tb, kin, kout, vin, vout, (int)n, 0, bits,
                                          ctx->stream));
  ctx->launches += 4;
}

// Row-major view of a matrix for the owner side: blocks sorted by (row, col)
// and a row pointer over the whole grid.
struct RowView {
  DevBuf rm_sorted, order, row_ptr;
};

void build_row_view(qt_mat B, RowView& v) {
  qt_ctx ctx = B->ctx;
  cudaStream_t st = ctx->stream;
  int64_t nb = B->nb;
  int32_t nbr = B->nbr;
  v.row_ptr.alloc(4ll * (nbr + 1), st);
  DevBuf cnt(4ll * (nbr + 1), st);
  QT_CUDA(cudaMemsetAsync(cnt.p, 0, 4ll * (nbr + 1), st));
  if (nb > 0) {
    DevBuf rm(nb * 8, st), iota(nb * 4, st);
    v.rm_sorted.alloc(nb * 8, st);
    v.order.alloc(nb * 4, st);
    k_rm_keys<<<gfor(nb), kT, 0, st>>>(B->key.as<uint64_t>(), nb, rm.as<uint64_t>(), iota.as<int32_t>());
    QT_LAUNCH_CHECK(ctx);
    sort_pairs(ctx, rm.as<uint64_t>(), v.rm_sorted.as<uint64_t>(), iota.as<int32_t>(),
               v.order.as<int32_t>(), nb, 64);
    k_row_hist<<<gfor(nb), kT, 0, st>>>(v.rm_sorted.as<uint64_t>(), nb, cnt.as<int32_t>());
    QT_LAUNCH_CHECK(ctx);
  }
  excl_sum(ctx, cnt.as<int32_t>(), v.row_ptr.as<int32_t>(), nbr + 1);
}

// The block rows a rank with rows [lo, hi) of A needs from others: sorted.
std::vector<int32_t> needed_rows(qt_mat A, int32_t lo, int32_t hi, DevBuf& d_rows) {
  qt_ctx ctx = A->ctx;
  cudaStream_t st = ctx->stream;
  int32_t nbr = A->nbr;
  DevBuf flag(4ll * nbr, st), incl(4ll * nbr, st);
  QT_CUDA(cudaMemsetAsync(flag.p, 0, 4ll * nbr, st));
  if (A->nb > 0) {
    k_mark_cols<<<gfor(A->nb), kT, 0, st>>>(A->key.as<uint64_t>(), A->nb, lo, hi, flag.as<int32_t>());
    QT_LAUNCH_CHECK(ctx);
  }
  incl_sum(ctx, flag.as<int32_t>(), incl.as<int32_t>(), nbr);
  int32_t n = 0;
  read_small(ctx, &n, incl.as<int32_t>() + nbr - 1, 4);
  d_rows.alloc(4ll * std::max(n, 1), st);
  std::vector<int32_t> h(n);
  if (n > 0) {
    k_scatter_flagged<<<gfor(nbr), kT, 0, st>>>(flag.as<int32_t>(), incl.as<int32_t>(), nbr,
                                                d_rows.as<int32_t>());
    QT_LAUNCH_CHECK(ctx);
    read_small(ctx, h.data(), d_rows.p, 4ll * n);
  }
  return h;
}

// Owner side, step 2: per requested row, its block count (device) -> counts
void pack_counts(qt_mat B, const RowView& v, const int32_t* d_rows, int32_t n, int32_t* d_counts) {
  qt_ctx ctx = B->ctx;
  if (n == 0) return;
  DevBuf rc(4ll * B->nbr, ctx->stream);
  // row_cnt[r] = row_ptr[r+1] - row_ptr[r]; computed on the fly by k_req_counts via row_ptr diff
  // (reuse k_req_counts on an explicit histogram for clarity)
  QT_CUDA(cudaMemsetAsync(rc.p, 0, 4ll * B->nbr, ctx->stream));
  if (B->nb > 0) {
    k_row_hist<<<gfor(B->nb), kT, 0, ctx->stream>>>(v.rm_sorted.as<uint64_t>(), B->nb, rc.as<int32_t>());
    QT_LAUNCH_CHECK(ctx);
  }
  k_req_counts<<<gfor(n), kT, 0, ctx->stream>>>(d_rows, n, rc.as<int32_t>(), d_counts);
  QT_LAUNCH_CHECK(ctx);
}

// Owner side, step 3: columns and values of the requested rows, packed at the
// exclusive-scan offsets of the counts.
void pack_blocks(qt_mat B, const RowView& v, const int32_t* d_rows, int32_t n, const int32_t* d_offs,
                 int32_t* d_cols, void* d_payload, uint8_t* d_sub = nullptr) {
  qt_ctx ctx = B->ctx;
  if (n == 0) return;
  int vpb = (int)(1024 * elem_size(B->dtype) / 16);
  unsigned g = (unsigned)((n + 7) / 8);
  k_pack<<<g, 256, 0, ctx->stream>>>(d_rows, n, d_offs, v.row_ptr.as<int32_t>(), v.order.as<int32_t>(),
                                     v.rm_sorted.as<uint64_t>(), static_cast<const uint4*>(B->pool_ptr()),
                                     vpb, d_cols, static_cast<uint4*>(d_payload),
                                     B->ubs == 16 ? B->sub.as<uint8_t>() : nullptr, d_sub);
  QT_LAUNCH_CHECK(ctx);
}

// What a requester ends up with after the exchange.
struct Received {
  int32_t nrows = 0;
  int64_t nblk = 0;
  DevBuf rows, counts, offs, cols, payload;
  DevBuf sub;  // block size 16: the received blocks' quadrant masks
};

qt_mat clone_shape(qt_mat A) {
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

// B_ext = local B rows + received rows; the received payload is owned by `rx`.
qt_mat make_b_ext(qt_mat B, Received& rx) {
  qt_ctx ctx = B->ctx;
  cudaStream_t st = ctx->stream;
  qt_mat X = clone_shape(B);
  try {
    int64_t nl = B->nb, nr = rx.nblk, nt = nl + nr;
    X->nb = nt;
    X->pool1 = B->pool_ptr();
    X->pool2 = rx.payload.p;
    X->split = nl;
    if (B->ubs == 16) {  // masks indexed like the pool ids: local, then received
      X->sub.alloc(std::max<int64_t>(nt, 1), st);
      if (nl > 0) QT_CUDA(cudaMemcpyAsync(X->sub.p, B->sub.p, nl, cudaMemcpyDeviceToDevice, st));
      if (nr > 0) QT_CUDA(cudaMemcpyAsync(X->sub.as<uint8_t>() + nl, rx.sub.p, nr, cudaMemcpyDeviceToDevice, st));
    }
    if (nt == 0) {
      build_levels(X);
      return X;
    }
    DevBuf keys(8 * nt, st), ids(4 * nt, st), sids(4 * nt, st);
    if (nl > 0) {
      QT_CUDA(cudaMemcpyAsync(keys.p, B->key.p, 8 * nl, cudaMemcpyDeviceToDevice, st));
      k_iota<<<gfor(nl), kT, 0, st>>>(ids.as<int32_t>(), nl);
      QT_LAUNCH_CHECK(ctx);
    }
    if (nr > 0) {
      unsigned g = (unsigned)((rx.nrows + 7) / 8);
      k_remote_keys<<<g, 256, 0, st>>>(rx.rows.as<int32_t>(), rx.nrows, rx.offs.as<int32_t>(),
                                       rx.cols.as<int32_t>(), keys.as<uint64_t>() + nl,
                                       ids.as<int32_t>() + nl, nl);
      QT_LAUNCH_CHECK(ctx);
    }
    X->key.alloc(8 * nt, st);
    sort_pairs(ctx, keys.as<uint64_t>(), X->key.as<uint64_t>(), ids.as<int32_t>(), sids.as<int32_t>(),
               nt, 2 * X->L);
    build_levels(X, sids.as<int32_t>());
  } catch (...) {
    delete X;
    throw;
  }
  return X;
}

qt_mat rows_of(qt_mat A, int32_t lo, int32_t hi) {
  qt_ctx ctx = A->ctx;
  DevBuf keep(std::max<int64_t>(A->nb, 1), ctx->stream);
  if (A->nb > 0) {
    k_flag_rows<<<gfor(A->nb), kT, 0, ctx->stream>>>(A->key.as<uint64_t>(), A->nb, lo, hi,
                                                     keep.as<uint8_t>());
    QT_LAUNCH_CHECK(ctx);
  }
  qt_mat M = select_blocks(A, keep.as<uint8_t>());
  M->row_lo = lo;
  M->row_hi = hi;
  return M;
}

void fill_exchange_stats(qt_stats* S, const Received& rx, size_t block_bytes, bool masks) {
  S->blocks_recv = rx.nblk;
  S->bytes_recv_payload = rx.nblk * (int64_t)block_bytes;
  S->bytes_recv_meta = 4ll * rx.nrows + 4ll * rx.nblk + (masks ? rx.nblk : 0);
  S->bytes_sent_meta = 4ll * rx.nrows;
}

}  // namespace

void split_tiles(qt_ctx ctx, int64_t ntiles, const int32_t* ts, const int32_t* pb, const int4* childB_t,
                 const int4* childB_1, int64_t splitB, int32_t* map, int32_t* nsel) {
  cudaStream_t st = ctx->stream;
  if (ntiles <= 0) return;
  DevBuf local(ntiles, st), ids(4 * ntiles, st);
  const unsigned gw = (unsigned)((ntiles + 7) / 8);  // 8 warps per 256-thread CTA
  k_tile_local<<<gw, 256, 0, st>>>(ts, pb, ntiles, childB_t, childB_1, splitB, local.as<uint8_t>(),
                                   ids.as<int32_t>());
  QT_LAUNCH_CHECK(ctx);
  // selected (local) tiles first in order, the rest after them (reversed)
  size_t tb = 0;
  QT_CUDA(cub::DevicePartition::Flagged(nullptr, tb, ids.as<int32_t>(), local.as<uint8_t>(), map, nsel,
                                        (int)ntiles, st));
  void* tmp = scratch(ctx, tb);
  QT_CUDA(cub::DevicePartition::Flagged(tmp, tb, ids.as<int32_t>(), local.as<uint8_t>(), map, nsel,
                                        (int)ntiles, st));
  ctx->launches += 2;
}

namespace {
qt_mat finish_multiply(qt_mat A_local, qt_mat Bx, qt_stats* S, Overlap* ov, double tau = -1.0) {
  float ms_sym = 0, ms_num = 0;
  qt_mat C = multiply_local(A_local, Bx, S, &ms_sym, &ms_num, 0, tau, ov);
  S->ms_symbolic = ms_sym;
  S->ms_numeric = ms_num;
  if (ov) {
    S->tiles_overlapped = ov->tiles_local;
    S->tiles_after = ov->tiles_remote;
  }
  return C;
}

// the overlap is on unless QT_OVERLAP=0
bool overlap_enabled() {
  const char* e = getenv("QT_OVERLAP");
  return !(e && e[0] == '0');
}

cudaStream_t comm_stream(qt_ctx ctx) {
  if (!ctx->comm_stream) {
    QT_CUDA(cudaStreamCreateWithFlags(&ctx->comm_stream, cudaStreamNonBlocking));
    QT_CUDA(cudaEventCreateWithFlags(&ctx->ov_ev[0], cudaEventDisableTiming));
    QT_CUDA(cudaEventCreateWithFlags(&ctx->ov_ev[1], cudaEventDisableTiming));
    QT_CUDA(cudaEventCreate(&ctx->ov_ev[2]));
    QT_CUDA(cudaEventCreate(&ctx->ov_ev[3]));
  }
  return ctx->comm_stream;
}
}  // namespace

// ------------------------------------------------------------------ NCCL path

qt_mat multiply_dist(qt_mat A, qt_mat B, qt_stats* S, double tau) {
  qt_ctx ctx = A->ctx;
  cudaStream_t st = ctx->stream;
  const int P = ctx->world, g = ctx->rank;
  if (A->bounds != B->bounds) fail(QT_EINVAL, "A and B must have the same block-row bounds");
  Transport* X = T(ctx);
  const size_t bb = 1024 * elem_size(A->dtype);
  QT_CUDA(cudaEventRecord(ctx->ev[5], st));
  const int32_t lo = A->row_lo, hi = A->row_hi;
  // 1. rows needed from others, split by owner (bounds are sorted, so is the list)
  DevBuf d_req;
  std::vector<int32_t> req = needed_rows(A, lo, hi, d_req);
  std::vector<int64_t> my_counts(P, 0), seg_off(P + 1, 0);
  for (int q = 0; q < P; ++q) {
    auto b = std::lower_bound(req.begin(), req.end(), A->bounds[q]);
    auto e = std::lower_bound(req.begin(), req.end(), A->bounds[q + 1]);
    seg_off[q] = b - req.begin();
    my_counts[q] = e - b;
  }
  seg_off[P] = (int64_t)req.size();
  // 0. P x P request matrix
  std::vector<int64_t> M((size_t)P * P);
  allgather_i64(ctx, my_counts.data(), M.data(), P);  // M[r*P+q] = rows r wants from q
  // 1. request lists
  std::vector<int64_t> in_off(P + 1, 0);
  for (int r = 0; r < P; ++r) in_off[r + 1] = in_off[r] + (r == g ? 0 : M[(size_t)r * P + g]);
  int64_t n_in = in_off[P];
  DevBuf d_in_rows(4 * std::max<int64_t>(n_in, 1), st);
  X->group_start();
  for (int q = 0; q < P; ++q) {
    if (q == g) continue;
    if (my_counts[q] > 0)
      X->send(d_req.as<int32_t>() + seg_off[q], 4 * my_counts[q], q);
    int64_t cnt = M[(size_t)q * P + g];
    if (cnt > 0)
      X->recv(d_in_rows.as<int32_t>() + in_off[q], 4 * cnt, q);
  }
  X->group_end();
  // 2. owner: block counts of the requested rows; requester: receive counts
  RowView v;
  build_row_view(B, v);
  DevBuf d_out_counts(4 * std::max<int64_t>(n_in, 1), st), d_out_offs(4 * (n_in + 1), st);
  pack_counts(B, v, d_in_rows.as<int32_t>(), (int32_t)n_in, d_out_counts.as<int32_t>());
  Received rx;
  rx.nrows = (int32_t)req.size();
  rx.rows = std::move(d_req);
  rx.counts.alloc(4 * std::max<int64_t>(rx.nrows, 1), st);
  rx.offs.alloc(4 * (rx.nrows + 1), st);
  X->group_start();
  for (int q = 0; q < P; ++q) {
    if (q == g) continue;
    int64_t cnt_out = M[(size_t)q * P + g];
    if (cnt_out > 0)
      X->send(d_out_counts.as<int32_t>() + in_off[q], 4 * cnt_out, q);
    if (my_counts[q] > 0)
      X->recv(rx.counts.as<int32_t>() + seg_off[q], 4 * my_counts[q], q);
  }
  X->group_end();
  // offsets on both sides (host copies decide the message sizes)
  std::vector<int32_t> h_out_counts(n_in), h_in_counts(rx.nrows);
  read_small(ctx, h_out_counts.data(), d_out_counts.p, 4 * n_in);
  read_small(ctx, h_in_counts.data(), rx.counts.p, 4ll * rx.nrows);
  QT_CUDA(cudaStreamSynchronize(st));
  std::vector<int32_t> h_out_offs(n_in + 1, 0), h_in_offs(rx.nrows + 1, 0);
  for (int64_t i = 0; i < n_in; ++i) h_out_offs[i + 1] = h_out_offs[i] + h_out_counts[i];
  for (int32_t i = 0; i < rx.nrows; ++i) h_in_offs[i + 1] = h_in_offs[i] + h_in_counts[i];
  QT_CUDA(cudaMemcpyAsync(d_out_offs.p, h_out_offs.data(), 4 * (n_in + 1), cudaMemcpyHostToDevice, st));
  QT_CUDA(cudaMemcpyAsync(rx.offs.p, h_in_offs.data(), 4ll * (rx.nrows + 1), cudaMemcpyHostToDevice, st));
  int64_t nblk_out = h_out_offs[n_in];
  rx.nblk = h_in_offs[rx.nrows];
  // 3. owner packs columns + values; exchange
  const bool m16 = B->ubs == 16;
  DevBuf d_out_cols(4 * std::max<int64_t>(nblk_out, 1), st), d_out_pay(bb * std::max<int64_t>(nblk_out, 1), st),
      d_out_sub(m16 ? std::max<int64_t>(nblk_out, 1) : 0, st);
  pack_blocks(B, v, d_in_rows.as<int32_t>(), (int32_t)n_in, d_out_offs.as<int32_t>(),
              d_out_cols.as<int32_t>(), d_out_pay.p, m16 ? d_out_sub.as<uint8_t>() : nullptr);
  if (m16) rx.sub.alloc(std::max<int64_t>(rx.nblk, 1), st);
  rx.cols.alloc(4 * std::max<int64_t>(rx.nblk, 1), st);
  rx.payload.alloc(bb * std::max<int64_t>(rx.nblk, 1), st);
  int64_t sent_payload = 0, sent_meta = 0;
  // 3a. block columns (ctx stream): B_ext's quadtree and the whole symbolic
  // multiply need only them
  X->group_start();
  for (int q = 0; q < P; ++q) {
    if (q == g) continue;
    int64_t r0 = in_off[q], r1 = in_off[q + 1];
    int64_t b0 = h_out_offs[r0], b1 = h_out_offs[r1];
    if (b1 > b0) X->send(d_out_cols.as<int32_t>() + b0, 4 * (b1 - b0), q);
    if (b1 > b0 && m16) X->send(d_out_sub.as<uint8_t>() + b0, b1 - b0, q);
    sent_meta += 4 * (r1 - r0) + (m16 ? 5 : 4) * (b1 - b0);
    int64_t i0 = h_in_offs[seg_off[q]], i1 = h_in_offs[seg_off[q] + my_counts[q]];
    if (i1 > i0) X->recv(rx.cols.as<int32_t>() + i0, 4 * (i1 - i0), q);
    if (i1 > i0 && m16) X->recv(rx.sub.as<uint8_t>() + i0, i1 - i0, q);
  }
  X->group_end();
  // 3b. values: on the comm stream (behind the packing) when overlapped, so
  // the symbolic pass and the local-only tiles run while they are in flight
  const bool ovl = overlap_enabled();
  cudaStream_t s2 = ovl ? comm_stream(ctx) : st;
  if (ovl) {
    QT_CUDA(cudaEventRecord(ctx->ov_ev[0], st));
    QT_CUDA(cudaStreamWaitEvent(s2, ctx->ov_ev[0], 0));
    QT_CUDA(cudaEventRecord(ctx->ov_ev[2], s2));
    X->set_stream(s2);
  }
  X->group_start();
  for (int q = 0; q < P; ++q) {
    if (q == g) continue;
    int64_t b0 = h_out_offs[in_off[q]], b1 = h_out_offs[in_off[q + 1]];
    if (b1 > b0) {
      X->send((char*)d_out_pay.p + b0 * bb, (b1 - b0) * bb, q);
      sent_payload += (b1 - b0) * bb;
    }
    int64_t i0 = h_in_offs[seg_off[q]], i1 = h_in_offs[seg_off[q] + my_counts[q]];
    if (i1 > i0) X->recv((char*)rx.payload.p + i0 * bb, (i1 - i0) * bb, q);
  }
  X->group_end();
  if (ovl) {
    X->set_stream(nullptr);
    QT_CUDA(cudaEventRecord(ctx->ov_ev[3], s2));
  }
  qt_mat Bx = make_b_ext(B, rx);
  QT_CUDA(cudaEventRecord(ctx->ev[6], st));
  fill_exchange_stats(S, rx, bb, m16);
  S->bytes_sent_payload = sent_payload;
  S->bytes_sent_meta += sent_meta;
  qt_mat C;
  Overlap ov;
  ov.s2 = s2;
  try {
    C = finish_multiply(A, Bx, S, ovl ? &ov : nullptr, tau);
  } catch (...) {
    if (ovl) cudaStreamSynchronize(s2);
    delete Bx;
    throw;
  }
  if (ovl) {
    // the send/receive buffers go back to the ctx stream's cache: join s2 first
    QT_CUDA(cudaStreamWaitEvent(st, ctx->ov_ev[3], 0));
    if (!ctx->async_multiply) {
      QT_CUDA(cudaEventSynchronize(ctx->ov_ev[3]));
      QT_CUDA(cudaEventElapsedTime(&S->ms_payload, ctx->ov_ev[2], ctx->ov_ev[3]));
    }
  }
  delete Bx;
  QT_CUDA(cudaEventElapsedTime(&S->ms_exchange, ctx->ev[5], ctx->ev[6]));
  return C;
}

// ------------------------------------------------------------ truncation (multi-rank)

namespace {
__global__ void k_ids(int64_t* __restrict__ out, int64_t n, int64_t rank) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n;
       t += (int64_t)gridDim.x * blockDim.x)
    out[t] = (rank << 32) | t;
}
}  // namespace

// Every rank sends its (norm^2, row-major key, id) terms to every other rank,
// then all ranks take the same global decision (truncate_decide) and keep
// their local survivors.  Moves 24 bytes per block to each peer (not on the
// multiply's hot path).
qt_mat truncate_dist(qt_mat A, double tau) {
  qt_ctx ctx = A->ctx;
  cudaStream_t st = ctx->stream;
  const int P = ctx->world, me = ctx->rank;
  Transport* X = T(ctx);
  const int64_t n = user_nblocks(A);
  std::vector<int64_t> counts(P);
  X->allgather_i64(&n, counts.data(), 1);
  std::vector<int64_t> off(P + 1, 0);
  for (int q = 0; q < P; ++q) off[q + 1] = off[q] + counts[q];
  const int64_t n_all = off[P];
  DevBuf nrm, rm;
  truncate_terms(A, nrm, rm);
  DevBuf ids(8 * std::max<int64_t>(n, 1), st);
  if (n > 0) {
    k_ids<<<gfor(n), kT, 0, st>>>(ids.as<int64_t>(), n, me);
    QT_LAUNCH_CHECK(ctx);
  }
  DevBuf nrm_all(8 * std::max<int64_t>(n_all, 1), st), rm_all(8 * std::max<int64_t>(n_all, 1), st),
      id_all(8 * std::max<int64_t>(n_all, 1), st);
  if (n > 0) {
    QT_CUDA(cudaMemcpyAsync(nrm_all.as<double>() + off[me], nrm.p, 8 * n, cudaMemcpyDeviceToDevice, st));
    QT_CUDA(cudaMemcpyAsync(rm_all.as<uint64_t>() + off[me], rm.p, 8 * n, cudaMemcpyDeviceToDevice, st));
    QT_CUDA(cudaMemcpyAsync(id_all.as<int64_t>() + off[me], ids.p, 8 * n, cudaMemcpyDeviceToDevice, st));
  }
  X->group_start();
  for (int q = 0; q < P; ++q) {
    if (q == me) continue;
    if (n > 0) {
      X->send(nrm.p, 8 * n, q);
      X->send(rm.p, 8 * n, q);
      X->send(ids.p, 8 * n, q);
    }
    if (counts[q] > 0) {
      X->recv(nrm_all.as<double>() + off[q], 8 * counts[q], q);
      X->recv(rm_all.as<uint64_t>() + off[q], 8 * counts[q], q);
      X->recv(id_all.as<int64_t>() + off[q], 8 * counts[q], q);
    }
  }
  X->group_end();
  DevBuf keep(std::max<int64_t>(n, 1), st);
  if (n > 0) QT_CUDA(cudaMemsetAsync(keep.p, 1, n, st));
  truncate_decide(ctx, nrm_all.as<double>(), rm_all.as<uint64_t>(), id_all.as<int64_t>(), n_all,
                  tau * tau, me, keep.as<uint8_t>());
  qt_mat R;
  if (A->ubs == 64) {
    DevBuf k32;
    expand_keep(A, keep.as<uint8_t>(), k32);
    R = select_blocks(A, k32.as<uint8_t>());
  } else if (A->ubs == 16) {
    R = apply_keep16(A, keep.as<uint8_t>());
  } else {
    R = select_blocks(A, keep.as<uint8_t>());
  }
  int64_t kept = user_nblocks(R), tot = 0;
  std::vector<int64_t> all(P);
  X->allgather_i64(&kept, all.data(), 1);
  for (auto v : all) tot += v;
  R->global_nb = tot;
  return R;
}

// ------------------------------------------------------------ virtual ranks

qt_mat multiply_virtual(qt_mat A, qt_mat B, const int32_t* bounds, int P, int g, qt_stats* S) {
  if (g < 0 || g >= P) fail(QT_EINVAL, "virtual rank %d not in [0,%d)", g, P);
  qt_ctx ctx = A->ctx;
  cudaStream_t st = ctx->stream;
  const size_t bb = 1024 * elem_size(A->dtype);
  const int32_t lo = bounds[g], hi = bounds[g + 1];
  qt_mat Al = rows_of(A, lo, hi);
  qt_mat Bl = nullptr, Bx = nullptr, C = nullptr;
  try {
    Bl = rows_of(B, lo, hi);
    QT_CUDA(cudaEventRecord(ctx->ev[5], st));
    DevBuf d_req;
    std::vector<int32_t> req = needed_rows(Al, lo, hi, d_req);
    Received rx;
    rx.nrows = (int32_t)req.size();
    rx.rows = std::move(d_req);
    rx.counts.alloc(4 * std::max<int64_t>(rx.nrows, 1), st);
    rx.offs.alloc(4 * (rx.nrows + 1), st);
    // every owner's rows are rows of the whole B: pack from B directly
    RowView v;
    build_row_view(B, v);
    pack_counts(B, v, rx.rows.as<int32_t>(), rx.nrows, rx.counts.as<int32_t>());
    std::vector<int32_t> hc(rx.nrows), ho(rx.nrows + 1, 0);
    read_small(ctx, hc.data(), rx.counts.p, 4ll * rx.nrows);
    QT_CUDA(cudaStreamSynchronize(st));
    for (int32_t i = 0; i < rx.nrows; ++i) ho[i + 1] = ho[i] + hc[i];
    QT_CUDA(cudaMemcpyAsync(rx.offs.p, ho.data(), 4ll * (rx.nrows + 1), cudaMemcpyHostToDevice, st));
    rx.nblk = ho[rx.nrows];
    rx.cols.alloc(4 * std::max<int64_t>(rx.nblk, 1), st);
    rx.payload.alloc(bb * std::max<int64_t>(rx.nblk, 1), st);
    if (B->ubs == 16) rx.sub.alloc(std::max<int64_t>(rx.nblk, 1), st);
    pack_blocks(B, v, rx.rows.as<int32_t>(), rx.nrows, rx.offs.as<int32_t>(), rx.cols.as<int32_t>(),
                rx.payload.p, B->ubs == 16 ? rx.sub.as<uint8_t>() : nullptr);
    Bx = make_b_ext(Bl, rx);
    QT_CUDA(cudaEventRecord(ctx->ev[6], st));
    fill_exchange_stats(S, rx, bb, B->ubs == 16);
    // the two-phase numeric launch of the NCCL path (here the payload is
    // already in place: the phases' split and stream ordering are what runs)
    Overlap ov;
    if (overlap_enabled()) ov.s2 = comm_stream(ctx);
    C = finish_multiply(Al, Bx, S, ov.s2 ? &ov : nullptr);
    QT_CUDA(cudaEventElapsedTime(&S->ms_exchange, ctx->ev[5], ctx->ev[6]));
    C->row_lo = lo;
    C->row_hi = hi;
  } catch (...) {
    delete Al;
    delete Bl;
    delete Bx;
    throw;
  }
  delete Bx;
  delete Bl;
  delete Al;
  return C;
}

// ------------------------------------------------------------ symmetric square (multi-rank)
//
// Rank g owns block rows [lo, hi) of the upper-triangular storage U and
// computes C = A^2 for its rows, upper triangle only (reading C-26).
// A(I,K) for I in the strip is U(I,K) (K >= I, local) or U(K,I)^T (K < I),
// and A(K,J) for J >= lo is U(K,J) (J >= K) or U(J,K)^T (lo <= J < K).  With
// R_g = the block columns >= hi of g's blocks, g receives every block (r,c) of
// another rank with
//   r >= hi and (r in R_g or c in R_g)       -- rows and columns above the strip
//   r <  lo, c >= lo and row r has a block in [lo,hi) -- rows reaching into it
// which is exactly the set of other ranks' blocks that some product of C's
// strip rows reads (oracle.exchange_plan_symm, pinned in tests/test_oracle.py
// against a brute-force enumeration of the products).  The symmetric-square BFS
// then runs on U_ext = local + received blocks, pruned to C rows [lo, hi).

namespace {
// flag[r] = 1 for every block row r with a block in columns [lo, hi)
__global__ void k_mark_rowhit(const uint64_t* __restrict__ key, int64_t nb, int32_t lo, int32_t hi,
                              int32_t* __restrict__ flag) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < nb;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int32_t c = (int32_t)morton_col(key[t]);
    if (c >= lo && c < hi) flag[morton_row(key[t])] = 1;
  }
}

__global__ void k_scatter_list(const int32_t* __restrict__ list, int64_t n, int32_t* __restrict__ flag) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n;
       t += (int64_t)gridDim.x * blockDim.x)
    flag[list[t]] = 1;
}

// the selection rule above for the strip [lo, hi); blocks inside the strip: keep_strip
__global__ void k_sym_keep(const uint64_t* __restrict__ key, int64_t nb, int32_t lo, int32_t hi,
                           const int32_t* __restrict__ inR, const int32_t* __restrict__ rowhit,
                           uint8_t keep_strip, uint8_t* __restrict__ keep) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < nb;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int32_t r = (int32_t)morton_row(key[t]), c = (int32_t)morton_col(key[t]);
    uint8_t k;
    if (r < lo)
      k = rowhit && rowhit[r] && c >= lo;
    else if (r >= hi)
      k = inR && (inR[r] || inR[c]);
    else
      k = keep_strip;
    keep[t] = k;
  }
}

// one warp per listed block: its key and values into the packed buffers
__global__ void k_pack_sel(const int32_t* __restrict__ ids, int64_t n, const uint64_t* __restrict__ key,
                           const uint4* __restrict__ pool, int vpb, uint64_t* __restrict__ okey,
                           uint4* __restrict__ opay, const uint8_t* __restrict__ sub, uint8_t* __restrict__ omask) {
  const int lane = threadIdx.x & 31;
  const int64_t w = blockIdx.x * (int64_t)(blockDim.x / 32) + threadIdx.x / 32;
  if (w >= n) return;
  const int32_t id = ids[w];
  if (lane == 0) okey[w] = key[id];
  if (lane == 0 && sub) omask[w] = sub[id];
  const uint4* sp = pool + (int64_t)id * vpb;
  uint4* dp = opay + w * vpb;
  for (int e = lane; e < vpb; e += 32) dp[e] = sp[e];
}

// U_ext = U's local blocks + nr received blocks (keys, values, block size
// 16: quadrant masks): one pool
qt_mat make_u_ext(qt_mat U, int64_t nr, const uint64_t* rkeys, const void* rpay, const uint8_t* rmask) {
  qt_ctx ctx = U->ctx;
  cudaStream_t st = ctx->stream;
  const size_t bb = 1024 * elem_size(U->dtype);
  qt_mat X = clone_shape(U);
  try {
    const int64_t nl = U->nb, nt = nl + nr;
    X->nb = nt;
    if (nt == 0) {
      build_levels(X);
      return X;
    }
    DevBuf keys(8 * nt, st), ids(4 * nt, st), sids(4 * nt, st);
    if (nl > 0) QT_CUDA(cudaMemcpyAsync(keys.p, U->key.p, 8 * nl, cudaMemcpyDeviceToDevice, st));
    if (nr > 0) QT_CUDA(cudaMemcpyAsync(keys.as<uint64_t>() + nl, rkeys, 8 * nr, cudaMemcpyDeviceToDevice, st));
    k_iota<<<gfor(nt), kT, 0, st>>>(ids.as<int32_t>(), nt);
    QT_LAUNCH_CHECK(ctx);
    X->key.alloc(8 * nt, st);
    sort_pairs(ctx, keys.as<uint64_t>(), X->key.as<uint64_t>(), ids.as<int32_t>(), sids.as<int32_t>(), nt,
               2 * X->L);
    X->pool.alloc(bb * nt, st);
    if (nl > 0) QT_CUDA(cudaMemcpyAsync(X->pool.p, U->pool_ptr(), bb * nl, cudaMemcpyDeviceToDevice, st));
    if (nr > 0)
      QT_CUDA(cudaMemcpyAsync((char*)X->pool.p + bb * nl, rpay, bb * nr, cudaMemcpyDeviceToDevice, st));
    if (U->ubs == 16) {  // (masks indexed like the pool)
      X->sub.alloc(nt, st);
      if (nl > 0) QT_CUDA(cudaMemcpyAsync(X->sub.p, U->sub.p, nl, cudaMemcpyDeviceToDevice, st));
      if (nr > 0) QT_CUDA(cudaMemcpyAsync(X->sub.as<uint8_t>() + nl, rmask, nr, cudaMemcpyDeviceToDevice, st));
    }
    build_levels(X, sids.as<int32_t>());
  } catch (...) {
    delete X;
    throw;
  }
  return X;
}

qt_mat symm_finish(qt_mat X, int32_t lo, int32_t hi, qt_stats* S) {
  float ms_sym = 0, ms_num = 0;
  qt_mat C = multiply_local(X, X, S, &ms_sym, &ms_num, 4 | (X->L << 8), -1.0, nullptr, lo, hi);
  S->ms_symbolic = ms_sym;
  S->ms_numeric = ms_num;
  C->row_lo = lo;
  C->row_hi = hi;
  return C;
}

// |R_q|: distinct block columns >= hi of the blocks in rows [lo, hi)
int64_t count_requests(qt_mat U, int32_t lo, int32_t hi) {
  qt_mat Uq = rows_of(U, lo, hi);
  DevBuf d;
  int64_t n = 0;
  try {
    n = (int64_t)needed_rows(Uq, lo, hi, d).size();
  } catch (...) {
    delete Uq;
    throw;
  }
  delete Uq;
  return n;
}
}  // namespace

qt_mat symm_square_dist(qt_mat U, qt_stats* S) {
  qt_ctx ctx = U->ctx;
  cudaStream_t st = ctx->stream;
  const int P = ctx->world, g = ctx->rank;
  Transport* X = T(ctx);
  const size_t bb = 1024 * elem_size(U->dtype);
  const int vpb = (int)(bb / 16);
  const int32_t lo = U->row_lo, hi = U->row_hi, nbr = U->nbr;
  const std::vector<int32_t>& b = U->bounds;
  const int64_t nb = U->nb;
  QT_CUDA(cudaEventRecord(ctx->ev[5], st));
  // 0. R_g (every local block has row in the strip) and the list sizes
  DevBuf d_req;
  const int64_t nreq = (int64_t)needed_rows(U, lo, hi, d_req).size();
  std::vector<int64_t> nr_all(P);
  X->allgather_i64(&nreq, nr_all.data(), 1);
  // 1. request lists go to the higher ranks (owners of rows >= hi)
  std::vector<DevBuf> rlist(P);
  for (int q = 0; q < g; ++q) rlist[q].alloc(4 * std::max<int64_t>(nr_all[q], 1), st);
  X->group_start();
  for (int q = 0; q < P; ++q) {
    if (q > g && nreq > 0) X->send(d_req.p, 4 * nreq, q);
    if (q < g && nr_all[q] > 0) X->recv(rlist[q].p, 4 * nr_all[q], q);
  }
  X->group_end();
  // 2. owner side: the blocks each other rank needs
  DevBuf iota(4 * std::max<int64_t>(nb, 1), st), keep(std::max<int64_t>(nb, 1), st),
      flag(4ll * nbr, st), cnt(4ll * P, st), rcnt(4ll * P, st);
  QT_CUDA(cudaMemsetAsync(cnt.p, 0, 4ll * P, st));
  QT_CUDA(cudaMemsetAsync(rcnt.p, 0, 4ll * P, st));
  if (nb > 0) {
    k_iota<<<gfor(nb), kT, 0, st>>>(iota.as<int32_t>(), nb);
    QT_LAUNCH_CHECK(ctx);
  }
  std::vector<DevBuf> sel(P);
  for (int q = 0; q < P && nb > 0; ++q) {
    if (q == g) continue;
    QT_CUDA(cudaMemsetAsync(flag.p, 0, 4ll * nbr, st));
    if (q > g) {  // my rows are below q's strip
      k_mark_rowhit<<<gfor(nb), kT, 0, st>>>(U->key.as<uint64_t>(), nb, b[q], b[q + 1], flag.as<int32_t>());
    } else if (nr_all[q] > 0) {  // my rows are above q's strip
      k_scatter_list<<<gfor(nr_all[q]), kT, 0, st>>>(rlist[q].as<int32_t>(), nr_all[q], flag.as<int32_t>());
    }
    QT_LAUNCH_CHECK(ctx);
    k_sym_keep<<<gfor(nb), kT, 0, st>>>(U->key.as<uint64_t>(), nb, b[q], b[q + 1],
                                        q < g ? flag.as<int32_t>() : nullptr,
                                        q > g ? flag.as<int32_t>() : nullptr, 0, keep.as<uint8_t>());
    QT_LAUNCH_CHECK(ctx);
    sel[q].alloc(4 * nb, st);
    size_t tb = 0;
    QT_CUDA(cub::DeviceSelect::Flagged(nullptr, tb, iota.as<int32_t>(), keep.as<uint8_t>(), sel[q].as<int32_t>(),
                                       cnt.as<int32_t>() + q, (int)nb, st));
    void* tmp = scratch(ctx, tb);
    QT_CUDA(cub::DeviceSelect::Flagged(tmp, tb, iota.as<int32_t>(), keep.as<uint8_t>(), sel[q].as<int32_t>(),
                                       cnt.as<int32_t>() + q, (int)nb, st));
    ctx->launches += 2;
  }
  // 3. counts
  X->group_start();
  for (int q = 0; q < P; ++q) {
    if (q == g) continue;
    X->send(cnt.as<int32_t>() + q, 4, q);
    X->recv(rcnt.as<int32_t>() + q, 4, q);
  }
  X->group_end();
  std::vector<int32_t> out_cnt(P), in_cnt(P);
  read_small(ctx, out_cnt.data(), cnt.p, 4ll * P);
  read_small(ctx, in_cnt.data(), rcnt.p, 4ll * P);
  std::vector<int64_t> out_off(P + 1, 0), in_off(P + 1, 0);
  for (int q = 0; q < P; ++q) {
    out_off[q + 1] = out_off[q] + (q == g ? 0 : out_cnt[q]);
    in_off[q + 1] = in_off[q] + (q == g ? 0 : in_cnt[q]);
  }
  // 4. keys + values
  const int64_t n_out = out_off[P], n_in = in_off[P];
  DevBuf okey(8 * std::max<int64_t>(n_out, 1), st), opay(bb * std::max<int64_t>(n_out, 1), st);
  DevBuf ikey(8 * std::max<int64_t>(n_in, 1), st), ipay(bb * std::max<int64_t>(n_in, 1), st);
  const bool m16 = U->ubs == 16;  // block size 16: one quadrant-mask byte per block travels too
  DevBuf omask(m16 ? std::max<int64_t>(n_out, 1) : 0, st), imask(m16 ? std::max<int64_t>(n_in, 1) : 0, st);
  for (int q = 0; q < P; ++q) {
    if (q == g || out_cnt[q] == 0) continue;
    k_pack_sel<<<(unsigned)((out_cnt[q] + 7) / 8), 256, 0, st>>>(
        sel[q].as<int32_t>(), out_cnt[q], U->key.as<uint64_t>(), static_cast<const uint4*>(U->pool_ptr()), vpb,
        okey.as<uint64_t>() + out_off[q], opay.as<uint4>() + out_off[q] * vpb,
        m16 ? U->sub.as<uint8_t>() : nullptr, m16 ? omask.as<uint8_t>() + out_off[q] : nullptr);
    QT_LAUNCH_CHECK(ctx);
  }
  X->group_start();
  for (int q = 0; q < P; ++q) {
    if (q == g) continue;
    if (out_cnt[q] > 0) {
      X->send(okey.as<uint64_t>() + out_off[q], 8ll * out_cnt[q], q);
      X->send((char*)opay.p + bb * out_off[q], bb * out_cnt[q], q);
      if (m16) X->send(omask.as<uint8_t>() + out_off[q], out_cnt[q], q);
    }
    if (in_cnt[q] > 0) {
      X->recv(ikey.as<uint64_t>() + in_off[q], 8ll * in_cnt[q], q);
      X->recv((char*)ipay.p + bb * in_off[q], bb * in_cnt[q], q);
      if (m16) X->recv(imask.as<uint8_t>() + in_off[q], in_cnt[q], q);
    }
  }
  X->group_end();
  qt_mat Ux = make_u_ext(U, n_in, ikey.as<uint64_t>(), ipay.p, m16 ? imask.as<uint8_t>() : nullptr);
  QT_CUDA(cudaEventRecord(ctx->ev[6], st));
  int64_t lists_in = 0;
  for (int q = 0; q < g; ++q) lists_in += nr_all[q];
  S->blocks_recv = n_in;
  S->bytes_recv_payload = n_in * (int64_t)bb;
  S->bytes_recv_meta = 8 * n_in + 4ll * (P - 1) + 4 * lists_in + (m16 ? n_in : 0);
  S->bytes_sent_payload = n_out * (int64_t)bb;
  S->bytes_sent_meta = 8 * n_out + 4ll * (P - 1) + 4 * nreq * (P - 1 - g) + (m16 ? n_out : 0);
  qt_mat C;
  try {
    C = symm_finish(Ux, lo, hi, S);
  } catch (...) {
    delete Ux;
    throw;
  }
  delete Ux;
  QT_CUDA(cudaEventElapsedTime(&S->ms_exchange, ctx->ev[5], ctx->ev[6]));
  return C;
}

qt_mat symm_square_virtual(qt_mat U, const int32_t* bounds, int P, int g, qt_stats* S) {
  qt_ctx ctx = U->ctx;
  cudaStream_t st = ctx->stream;
  const size_t bb = 1024 * elem_size(U->dtype);
  const int32_t lo = bounds[g], hi = bounds[g + 1], nbr = U->nbr;
  const int64_t nb = U->nb;
  qt_mat Ul = rows_of(U, lo, hi), Ux = nullptr, C = nullptr;
  try {
    QT_CUDA(cudaEventRecord(ctx->ev[5], st));
    DevBuf d_req;
    const int64_t nreq = (int64_t)needed_rows(Ul, lo, hi, d_req).size();
    DevBuf inR(4ll * nbr, st), rowhit(4ll * nbr, st), keep(std::max<int64_t>(nb, 1), st);
    QT_CUDA(cudaMemsetAsync(inR.p, 0, 4ll * nbr, st));
    QT_CUDA(cudaMemsetAsync(rowhit.p, 0, 4ll * nbr, st));
    if (nreq > 0) {
      k_scatter_list<<<gfor(nreq), kT, 0, st>>>(d_req.as<int32_t>(), nreq, inR.as<int32_t>());
      QT_LAUNCH_CHECK(ctx);
    }
    if (nb > 0) {
      k_mark_rowhit<<<gfor(nb), kT, 0, st>>>(U->key.as<uint64_t>(), nb, lo, hi, rowhit.as<int32_t>());
      QT_LAUNCH_CHECK(ctx);
      k_sym_keep<<<gfor(nb), kT, 0, st>>>(U->key.as<uint64_t>(), nb, lo, hi, inR.as<int32_t>(),
                                          rowhit.as<int32_t>(), 1, keep.as<uint8_t>());
      QT_LAUNCH_CHECK(ctx);
    }
    Ux = select_blocks(U, keep.as<uint8_t>());
    ensure_levels(Ux);
    QT_CUDA(cudaEventRecord(ctx->ev[6], st));
    int64_t lists_in = 0;
    for (int q = 0; q < g; ++q) lists_in += count_requests(U, bounds[q], bounds[q + 1]);
    const int64_t n_in = Ux->nb - Ul->nb;
    S->blocks_recv = n_in;
    S->bytes_recv_payload = n_in * (int64_t)bb;
    S->bytes_recv_meta = 8 * n_in + 4ll * (P - 1) + 4 * lists_in + (U->ubs == 16 ? n_in : 0);  // (+ mask bytes)
    S->bytes_sent_meta = 4 * nreq * (P - 1 - g);
    C = symm_finish(Ux, lo, hi, S);
    QT_CUDA(cudaEventElapsedTime(&S->ms_exchange, ctx->ev[5], ctx->ev[6]));
  } catch (...) {
    delete Ul;
    delete Ux;
    throw;
  }
  delete Ux;
  delete Ul;
  return C;
}

// ------------------------------------------------------------ gather (X4)

// Every rank's blocks to `root`, in (brow, bcol) order: the ranks own
// contiguous block-row strips in rank order, so the root concatenates the
// ranks' own sorted lists.  Collective; returns the total block count.
int64_t gather_dist(qt_mat A, int root, int32_t* brow, int32_t* bcol, void* vals) {
  qt_ctx ctx = A->ctx;
  cudaStream_t st = ctx->stream;
  const int P = ctx->world, g = ctx->rank;
  Transport* X = T(ctx);
  const int64_t n = user_nblocks(A);
  std::vector<int64_t> cnt(P);
  X->allgather_i64(&n, cnt.data(), 1);
  std::vector<int64_t> off(P + 1, 0);
  for (int q = 0; q < P; ++q) off[q + 1] = off[q] + cnt[q];
  const int64_t N = off[P];
  const bool want = brow || bcol || vals;
  int any = want ? 1 : 0;
  {  // every rank must take the same branch: the root decides (it owns the buffers)
    int64_t w = any;
    std::vector<int64_t> aw(P);
    X->allgather_i64(&w, aw.data(), 1);
    any = (int)aw[root];
  }
  if (!any || N == 0) return N;
  const size_t vb = (size_t)A->ubs * A->ubs * elem_size(A->dtype);
  DevBuf lr(4 * std::max<int64_t>(n, 1), st), lc(4 * std::max<int64_t>(n, 1), st),
      lv(vb * std::max<int64_t>(n, 1), st);
  if (n > 0) read_back(A, lr.as<int32_t>(), lc.as<int32_t>(), lv.p);
  if (g != root) {
    X->group_start();
    if (n > 0) {
      X->send(lr.p, 4 * n, root);
      X->send(lc.p, 4 * n, root);
      X->send(lv.p, vb * n, root);
    }
    X->group_end();
    return N;
  }
  DevBuf R(4 * N, st), Cc(4 * N, st), V(vb * N, st);
  if (n > 0) {
    QT_CUDA(cudaMemcpyAsync(R.as<int32_t>() + off[g], lr.p, 4 * n, cudaMemcpyDeviceToDevice, st));
    QT_CUDA(cudaMemcpyAsync(Cc.as<int32_t>() + off[g], lc.p, 4 * n, cudaMemcpyDeviceToDevice, st));
    QT_CUDA(cudaMemcpyAsync((char*)V.p + vb * off[g], lv.p, vb * n, cudaMemcpyDeviceToDevice, st));
  }
  X->group_start();
  for (int q = 0; q < P; ++q) {
    if (q == g || cnt[q] == 0) continue;
    X->recv(R.as<int32_t>() + off[q], 4 * cnt[q], q);
    X->recv(Cc.as<int32_t>() + off[q], 4 * cnt[q], q);
    X->recv((char*)V.p + vb * off[q], vb * cnt[q], q);
  }
  X->group_end();
  if (brow) QT_CUDA(cudaMemcpyAsync(brow, R.p, 4 * N, cudaMemcpyDefault, st));
  if (bcol) QT_CUDA(cudaMemcpyAsync(bcol, Cc.p, 4 * N, cudaMemcpyDefault, st));
  if (vals) QT_CUDA(cudaMemcpyAsync(vals, V.p, vb * N, cudaMemcpyDefault, st));
  QT_CUDA(cudaStreamSynchronize(st));
  return N;
}

}  // namespace qt

namespace qt {
void nccl_unique_id(void* out128) {
  NcclApi& N = nccl();
  ncclUniqueId id;
  NCCL_CALL(N.GetUniqueId(&id));
  memcpy(out128, &id, sizeof(id));
}
}  // namespace qt
