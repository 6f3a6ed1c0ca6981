// Slab-decomposed friends-of-friends across ranks (SURVEY §8 row e) — the
// device pipeline behind sp_fof_slabs (one process per GPU, NCCL) and
// sp_fof_slabs_multi (one process driving several contexts, peer copies).
//
// The reference has no distributed search; the paper's
// ArborX partitions FoF over MPI ranks.  Here every
// rank holds the rows [first, first + n) of the global point array and gets
// back the labels of exactly those rows: the smallest GLOBAL index of the
// point's cluster (-1 = noise), bit-identical to a single-GPU (and to the
// reference's) friends_of_friends over the whole array (dbscan.hpp:286-292).
//
// One step, all on the device except one host read of a G x 3G count matrix:
//   A  x-histogram of a strided sample (2^20 bins of the order-mapped float
//      bits), summed over ranks (all-reduce);
//   B  G-1 splitters at the histogram's quantiles (identical on every rank);
//      per point: owner slab d = #splitters <= x, ghost slabs = the slabs
//      meeting [x - w, x + w] (exact in double, w = eps (1 + 2^-20) covers
//      every pair the reference's distance test can accept); per-destination
//      counts of owned / ghost entries and of owned points that are ghosts
//      somewhere ("near"), all-gathered -> the host sizes every exchange;
//   C  pack (xyz, global id) per destination (warp-aggregated atomics),
//      remembering each row's return slot; all-to-all;
//   D  local FoF over owned + ghost points in global-id space (fof_cells
//      with ids: labels = smallest global id of the local piece);
//   E  (global id, local label) for every received ghost and every near owned
//      point, all-gathered: copies of one point link the labels of the
//      slabs that hold it;
//   F  every rank sorts the same pairs and unites the linked labels
//      (lock-free union-find, the smaller label wins, union_find.hpp:17-59);
//      a label's component minimum is the global cluster label;
//   G  owned entries relabelled and returned to their input rank
//      (all-to-all), scattered to input order; core = label >= 0.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>  // types only: the functions are resolved at run time (NcclApi)
#include <stdint.h>

#include <algorithm>
#include <cstring>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include "sp_common.cuh"
#include "sp_internal.hpp"
#include "sp_slabs.hpp"
#include "sp_traverse.cuh"

namespace spb {

// ---------------------------------------------------------------------------
// NCCL, bound at run time: the process's already-loaded libnccl.so.2 (e.g.
// torch's, so communicators made there are usable here) or the system one.
// ---------------------------------------------------------------------------
namespace {
struct NcclApi {
  decltype(&ncclGetUniqueId) GetUniqueId = nullptr;
  decltype(&ncclCommInitRank) CommInitRank = nullptr;
  decltype(&ncclCommDestroy) CommDestroy = nullptr;
  decltype(&ncclCommCount) CommCount = nullptr;
  decltype(&ncclCommUserRank) CommUserRank = nullptr;
  decltype(&ncclAllReduce) AllReduce = nullptr;
  decltype(&ncclAllGather) AllGather = nullptr;
  decltype(&ncclSend) Send = nullptr;
  decltype(&ncclRecv) Recv = nullptr;
  decltype(&ncclGroupStart) GroupStart = nullptr;
  decltype(&ncclGroupEnd) GroupEnd = nullptr;
  decltype(&ncclGetErrorString) GetErrorString = nullptr;
  std::string error;

  static NcclApi &get() {
    static NcclApi api;
    static std::once_flag once;
    std::call_once(once, [] { api.load(); });
    if (!api.error.empty()) throw NcclError(api.error);
    return api;
  }
  void load() {
    void *h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_LOCAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_LOCAL);
    if (!h) {
      error = "NCCL (libnccl.so.2) not found";
      return;
    }
#define SPB_NCCL_SYM(name)                                                         \
  name = reinterpret_cast<decltype(name)>(dlsym(h, "nccl" #name));                 \
  if (!name) {                                                                     \
    error = "NCCL symbol nccl" #name " missing";                                   \
    return;                                                                        \
  }
    SPB_NCCL_SYM(GetUniqueId)
    SPB_NCCL_SYM(CommInitRank)
    SPB_NCCL_SYM(CommDestroy)
    SPB_NCCL_SYM(CommCount)
    SPB_NCCL_SYM(CommUserRank)
    SPB_NCCL_SYM(AllReduce)
    SPB_NCCL_SYM(AllGather)
    SPB_NCCL_SYM(Send)
    SPB_NCCL_SYM(Recv)
    SPB_NCCL_SYM(GroupStart)
    SPB_NCCL_SYM(GroupEnd)
    SPB_NCCL_SYM(GetErrorString)
#undef SPB_NCCL_SYM
  }
};

void nccl_check(ncclResult_t r, const char *what) {
  if (r != ncclSuccess) throw NcclError(std::string(what) + ": " + NcclApi::get().GetErrorString(r));
}
}  // namespace

void nccl_unique_id(uint8_t out[128]) {
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId is 128 bytes");
  ncclUniqueId id;
  nccl_check(NcclApi::get().GetUniqueId(&id), "ncclGetUniqueId");
  std::memcpy(out, &id, 128);
}

// ---------------------------------------------------------------------------
// Exchanges: the collectives of one step over the ranks this host thread
// drives (one under NCCL, all of them in the single-process form).
// ---------------------------------------------------------------------------
struct SlabExchange {
  // host-mapped pinned scratch for the count matrix: written by a kernel, so
  // the read never queues on a copy engine behind a bulk transfer
  unsigned long long *host_mat = nullptr, *dev_mat = nullptr;
  unsigned long long *mapped(size_t count) {
    if (!host_mat) {
      SPB_CUDA(cudaHostAlloc(reinterpret_cast<void **>(&host_mat),
                             (size_t)3 * kMaxSlabRanks * kMaxSlabRanks * sizeof(unsigned long long),
                             cudaHostAllocMapped | cudaHostAllocPortable));
      SPB_CUDA(cudaHostGetDevicePointer(reinterpret_cast<void **>(&dev_mat), host_mat, 0));
    }
    (void)count;
    return dev_mat;
  }
  virtual ~SlabExchange() {
    if (host_mat) cudaFreeHost(host_mat);
  }
  virtual int size() const = 0;
  virtual int rank_of(int local) const = 0;
  // recv[l] (G * bytes) <- every rank's send (bytes); in place allowed when
  // send[l] == recv[l] + rank * bytes
  virtual void allgather(const std::vector<Ctx *> &c, const std::vector<const void *> &send,
                         const std::vector<void *> &recv, size_t bytes) = 0;
  // buf[l] <- sum over ranks (uint32, count elements)
  virtual void allreduce_u32(const std::vector<Ctx *> &c, const std::vector<uint32_t *> &buf, size_t count) = 0;
  // rank r's block for peer p: send[r] + soff[r][p], sbytes[r][p] bytes ->
  // peer p's recv + roff[p][r]
  virtual void alltoallv(const std::vector<Ctx *> &c, const std::vector<const void *> &send,
                         const std::vector<std::vector<size_t>> &soff, const std::vector<std::vector<size_t>> &sbytes,
                         const std::vector<void *> &recv, const std::vector<std::vector<size_t>> &roff,
                         const std::vector<std::vector<size_t>> &rbytes) = 0;
};

struct NcclExchange : SlabExchange {
  ncclComm_t comm = nullptr;
  bool owned = false;
  int G = 1, me = 0;
  ~NcclExchange() override {
    if (owned && comm) NcclApi::get().CommDestroy(comm);
  }
  int size() const override { return G; }
  int rank_of(int) const override { return me; }
  void allgather(const std::vector<Ctx *> &c, const std::vector<const void *> &send, const std::vector<void *> &recv,
                 size_t bytes) override {
    if (bytes == 0) return;
    nccl_check(NcclApi::get().AllGather(send[0], recv[0], bytes, ncclUint8, comm, c[0]->stream), "ncclAllGather");
  }
  void allreduce_u32(const std::vector<Ctx *> &c, const std::vector<uint32_t *> &buf, size_t count) override {
    nccl_check(NcclApi::get().AllReduce(buf[0], buf[0], count, ncclUint32, ncclSum, comm, c[0]->stream),
               "ncclAllReduce");
  }
  void alltoallv(const std::vector<Ctx *> &c, const std::vector<const void *> &send,
                 const std::vector<std::vector<size_t>> &soff, const std::vector<std::vector<size_t>> &sbytes,
                 const std::vector<void *> &recv, const std::vector<std::vector<size_t>> &roff,
                 const std::vector<std::vector<size_t>> &rbytes) override {
    (void)roff;
    const NcclApi &api = NcclApi::get();
    nccl_check(api.GroupStart(), "ncclGroupStart");
    for (int p = 0; p < G; ++p) {
      if (sbytes[0][p])
        nccl_check(api.Send(static_cast<const char *>(send[0]) + soff[0][p], sbytes[0][p], ncclUint8, p, comm,
                            c[0]->stream),
                   "ncclSend");
      if (rbytes[0][p])
        nccl_check(api.Recv(static_cast<char *>(recv[0]) + roff[0][p], rbytes[0][p], ncclUint8, p, comm,
                            c[0]->stream),
                   "ncclRecv");
    }
    nccl_check(api.GroupEnd(), "ncclGroupEnd");
  }
};

namespace {
__global__ void k_sum_slices_u32(uint32_t *dst, const uint32_t *slices, int G, size_t count) {
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < count; i += stride) {
    uint32_t s = 0;
    for (int g = 0; g < G; ++g) s += slices[(size_t)g * count + i];
    dst[i] = s;
  }
}
}  // namespace

// All ranks in this process: every exchange is a barrier (events), copies
// pulled by each destination on its own stream (cudaMemcpyPeerAsync, so the
// contexts may sit on one device or several), and a closing barrier so no
// source buffer is reused before every copy out of it has finished.
struct LocalExchange : SlabExchange {
  int G = 1;
  std::vector<cudaEvent_t> ev;
  explicit LocalExchange(const std::vector<Ctx *> &c) : G((int)c.size()), ev(c.size(), nullptr) {
    for (int r = 0; r < G; ++r) {
      ScopedDevice sd(c[r]->device);
      SPB_CUDA(cudaEventCreateWithFlags(&ev[r], cudaEventDisableTiming));
    }
  }
  ~LocalExchange() override {
    for (auto e : ev)
      if (e) cudaEventDestroy(e);
  }
  int size() const override { return G; }
  int rank_of(int local) const override { return local; }
  void barrier(const std::vector<Ctx *> &c) {
    for (int r = 0; r < G; ++r) {
      ScopedDevice sd(c[r]->device);
      SPB_CUDA(cudaEventRecord(ev[r], c[r]->stream));
    }
    for (int r = 0; r < G; ++r) {
      ScopedDevice sd(c[r]->device);
      for (int q = 0; q < G; ++q)
        if (q != r) SPB_CUDA(cudaStreamWaitEvent(c[r]->stream, ev[q], 0));
    }
  }
  void copy(Ctx *dst_c, void *dst, Ctx *src_c, const void *src, size_t bytes) {
    if (!bytes) return;
    ScopedDevice sd(dst_c->device);
    SPB_CUDA(cudaMemcpyPeerAsync(dst, dst_c->device, src, src_c->device, bytes, dst_c->stream));
  }
  void allgather(const std::vector<Ctx *> &c, const std::vector<const void *> &send, const std::vector<void *> &recv,
                 size_t bytes) override {
    if (bytes == 0) return;
    barrier(c);
    for (int r = 0; r < G; ++r)
      for (int q = 0; q < G; ++q) {
        char *dst = static_cast<char *>(recv[r]) + (size_t)q * bytes;
        if (dst != send[q]) copy(c[r], dst, c[q], send[q], bytes);
      }
    barrier(c);
  }
  void allreduce_u32(const std::vector<Ctx *> &c, const std::vector<uint32_t *> &buf, size_t count) override {
    std::vector<DevBuf<uint32_t>> tmp;
    std::vector<void *> recv;
    std::vector<const void *> send;
    for (int r = 0; r < G; ++r) {
      ScopedDevice sd(c[r]->device);
      tmp.emplace_back((size_t)G * count, c[r]->stream);
      recv.push_back(tmp.back().get());
      send.push_back(buf[r]);
    }
    allgather(c, send, recv, count * sizeof(uint32_t));
    for (int r = 0; r < G; ++r) {
      ScopedDevice sd(c[r]->device);
      k_sum_slices_u32<<<grid_for((int64_t)count, 256, 148 * 4), 256, 0, c[r]->stream>>>(buf[r], tmp[r].get(), G,
                                                                                        count);
      SPB_LAUNCHED();
    }
  }
  void alltoallv(const std::vector<Ctx *> &c, const std::vector<const void *> &send,
                 const std::vector<std::vector<size_t>> &soff, const std::vector<std::vector<size_t>> &sbytes,
                 const std::vector<void *> &recv, const std::vector<std::vector<size_t>> &roff,
                 const std::vector<std::vector<size_t>> &rbytes) override {
    barrier(c);
    for (int r = 0; r < G; ++r)
      for (int p = 0; p < G; ++p) {
        if (sbytes[r][p] != rbytes[p][r]) throw CudaError("slab exchange: inconsistent sizes");
        copy(c[p], static_cast<char *>(recv[p]) + roff[p][r], c[r], static_cast<const char *>(send[r]) + soff[r][p],
             sbytes[r][p]);
      }
    barrier(c);
  }
};

// ---------------------------------------------------------------------------
// kernels
// ---------------------------------------------------------------------------
namespace {

constexpr int kHistBits = 20;
constexpr uint32_t kHistBins = 1u << kHistBits;
constexpr uint32_t kNoId = 0xffffffffu;

__device__ __forceinline__ uint32_t ord_key(float x) {
  const uint32_t b = __float_as_uint(x);
  return (b & 0x80000000u) ? ~b : (b | 0x80000000u);
}
__device__ __forceinline__ float key_float(uint32_t u) {
  return __uint_as_float((u & 0x80000000u) ? (u & 0x7fffffffu) : ~u);
}

// Destination slabs of a point: owner d = #splitters <= x; ghost slabs are
// [lo, hi] \ {d} with lo/hi the owners of x -/+ w, computed exactly in double.
// The G - 1 splitters stay on the device (no host read); each block copies
// them to shared memory first (Route).
struct Splitters {
  const float *s;  // device, G - 1 values
  int G;
  double w;
};
struct Route {
  float s[kMaxSlabRanks];
  int G;
  double w;
  __device__ __forceinline__ void load(const Splitters &S) {
    if (threadIdx.x < kMaxSlabRanks) s[threadIdx.x] = threadIdx.x + 1 < (unsigned)S.G ? S.s[threadIdx.x] : 0.f;
    if (threadIdx.x == 0) {
      G = S.G;
      w = S.w;
    }
    __syncthreads();
  }
  __device__ __forceinline__ void route(float x, int &d, int &lo, int &hi) const {
    const double xd = (double)x, a = xd - w, b = xd + w;
    d = lo = hi = 0;
    for (int k = 0; k < G - 1; ++k) {
      const float sk = s[k];
      d += sk <= x;
      lo += (double)sk <= a;
      hi += (double)sk <= b;
    }
  }
};

__global__ void k_slab_hist(const float *__restrict__ pts, int64_t n, int64_t stride, uint32_t *hist) {
  const int64_t ns = (n + stride - 1) / stride;
  const int64_t st = (int64_t)gridDim.x * blockDim.x;
  for (int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; s < ns; s += st)
    atomicAdd(&hist[ord_key(pts[3 * (s * stride)]) >> (32 - kHistBits)], 1u);
}

// One block of 1024 threads: splitter k (1 <= k < G) is the lower edge of the
// bin after the first bin whose inclusive count reaches k * total / G.
__global__ void __launch_bounds__(1024) k_slab_splitters(const uint32_t *__restrict__ hist, int G, float *split) {
  __shared__ unsigned long long s[1024];
  const int t = threadIdx.x;
  constexpr int per = kHistBins / 1024;
  unsigned long long mine = 0;
  for (int i = 0; i < per; ++i) mine += hist[t * per + i];
  s[t] = mine;
  __syncthreads();
  for (int off = 1; off < 1024; off <<= 1) {  // inclusive scan
    const unsigned long long v = t >= off ? s[t - off] : 0ull;
    __syncthreads();
    s[t] += v;
    __syncthreads();
  }
  const unsigned long long total = s[1023], incl = s[t], excl = incl - mine;
  for (int k = 1; k < G; ++k) {
    const unsigned long long target = (unsigned long long)k * total / (unsigned long long)G;
    if (target == 0) {
      if (t == 0) split[k - 1] = -__int_as_float(0x7f800000);  // -inf: slab k-1 starts empty
      continue;
    }
    if (excl < target && target <= incl) {
      unsigned long long run = excl;
      int b = t * per;
      for (; b < (t + 1) * per; ++b) {
        run += hist[b];
        if (run >= target) break;
      }
      const uint32_t nb = (uint32_t)b + 1;
      split[k - 1] = nb >= kHistBins ? __int_as_float(0x7f800000) : key_float(nb << (32 - kHistBits));
    }
  }
}

// Warp-aggregated atomic add of 1 per active lane on cnt[key] (lanes with the
// same key share one atomic); returns the lane's slot among them.
template <class T>
__device__ __forceinline__ T agg_add(T *cnt, int key, bool active) {
  const int lane = threadIdx.x & 31;
  const unsigned act = __ballot_sync(0xffffffffu, active);
  const unsigned peers = __match_any_sync(0xffffffffu, active ? key : -1) & act;
  const int leader = peers ? __ffs(peers) - 1 : lane;
  T base = 0;
  if (active && lane == leader) base = atomicAdd(cnt + key, (T)__popc(peers));
  base = __shfl_sync(0xffffffffu, base, leader);
  return base + (T)__popc(peers & ((1u << lane) - 1u));
}

// per-destination counts: [0, G) owned, [G, 2G) ghost, [2G, 3G) near owned
__global__ void __launch_bounds__(256) k_slab_count(const float *__restrict__ pts, int64_t n, Splitters SP,
                                                    unsigned long long *counts) {
  __shared__ unsigned int sc[3 * kMaxSlabRanks];
  __shared__ Route S;
  for (int i = threadIdx.x; i < 3 * kMaxSlabRanks; i += blockDim.x) sc[i] = 0;
  S.load(SP);
  const int G = SP.G;
  const int64_t st = (int64_t)gridDim.x * blockDim.x;
  const int64_t t0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  for (int64_t wb = t0 - (threadIdx.x & 31); wb < n; wb += st) {
    const int64_t i = wb + (threadIdx.x & 31);
    const bool valid = i < n;
    int d = 0, lo = 0, hi = 0;
    if (valid) S.route(pts[3 * i], d, lo, hi);
    agg_add(sc, d, valid);
    const bool near = valid && (lo != d || hi != d);
    agg_add(sc, 2 * G + d, near);
    for (int t = lo;; ++t) {
      if (near && t == d) ++t;
      const bool more = near && t <= hi;
      if (!__any_sync(0xffffffffu, more)) break;
      agg_add(sc, G + t, more);
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < 3 * G; i += blockDim.x)
    if (sc[i]) atomicAdd(&counts[i], (unsigned long long)sc[i]);
}

struct PackLayout {
  int64_t owned_base[kMaxSlabRanks];  // send position of the owned block for peer d
  int64_t ghost_base[kMaxSlabRanks];  // send position of the ghost block for peer d
  int64_t ret_base[kMaxSlabRanks];    // where peer d's returned labels land
  // the self block -- rows this rank owns itself, then ghost copies of rows
  // it holds for slabs it owns -- skips the send buffer and the exchange: it
  // is written straight into the receive buffer at self_base (owned rows
  // never return)
  int me;
  int64_t self_base, self_owned;
  float *rxyz;
  int32_t *rid;
};

// warp-aggregated global slot (one atomic per key per warp)
__device__ __forceinline__ unsigned long long agg_slot(unsigned long long *ctr, int key, bool active) {
  return agg_add(ctr, key, active);
}

// Pack a tile of PK_ITEMS x 256 rows per block: slots are reserved per block
// (one global atomic per destination per block, not per warp) and handed out
// inside the block by warp-aggregated shared atomics, so the entries of one
// destination stay in runs of about a tile in input order.
constexpr int PK_ITEMS = 4;
__global__ void __launch_bounds__(256) k_slab_pack(const float *__restrict__ pts, int64_t n, int64_t first,
                                                   Splitters SP, PackLayout L, unsigned long long *cursor,
                                                   float *__restrict__ sxyz, int32_t *__restrict__ sid,
                                                   int32_t *__restrict__ slot_of_row) {
  __shared__ Route S;
  __shared__ unsigned int cnt[2 * kMaxSlabRanks], gcnt[kMaxSlabRanks];
  __shared__ unsigned long long base[2 * kMaxSlabRanks];
  const int G = SP.G;
  const int64_t tile = (int64_t)blockDim.x * PK_ITEMS;
  S.load(SP);
  for (int64_t t0 = (int64_t)blockIdx.x * tile; t0 < n; t0 += (int64_t)gridDim.x * tile) {
    if (threadIdx.x < 2 * kMaxSlabRanks) cnt[threadIdx.x] = 0;
    if (threadIdx.x < kMaxSlabRanks) gcnt[threadIdx.x] = 0;
    __syncthreads();
    float x[PK_ITEMS], y[PK_ITEMS], z[PK_ITEMS];
    int d[PK_ITEMS], lo[PK_ITEMS], hi[PK_ITEMS];
    unsigned off[PK_ITEMS];
#pragma unroll
    for (int j = 0; j < PK_ITEMS; ++j) {
      const int64_t i = t0 + (int64_t)j * blockDim.x + threadIdx.x;
      const bool valid = i < n;
      d[j] = lo[j] = 0;
      hi[j] = -1;  // no ghosts for an invalid row
      x[j] = y[j] = z[j] = 0.f;
      if (valid) {
        x[j] = pts[3 * i];
        y[j] = pts[3 * i + 1];
        z[j] = pts[3 * i + 2];
        S.route(x[j], d[j], lo[j], hi[j]);
      }
      off[j] = agg_add(cnt, d[j], valid);
      for (int t = lo[j];; ++t) {
        if (valid && t == d[j]) ++t;
        const bool more = valid && t <= hi[j];
        if (!__any_sync(0xffffffffu, more)) break;
        agg_add(cnt, G + t, more);
      }
    }
    __syncthreads();
    if (threadIdx.x < 2 * G) base[threadIdx.x] = cnt[threadIdx.x] ? atomicAdd(cursor + threadIdx.x,
                                                                              (unsigned long long)cnt[threadIdx.x])
                                                                  : 0ull;
    __syncthreads();
#pragma unroll
    for (int j = 0; j < PK_ITEMS; ++j) {
      const int64_t i = t0 + (int64_t)j * blockDim.x + threadIdx.x;
      const bool valid = i < n;
      if (valid) {
        const int64_t k = (int64_t)base[d[j]] + off[j];
        const bool self = d[j] == L.me;
        const int64_t pos = self ? L.self_base + k : L.owned_base[d[j]] + k;
        float *xyz = self ? L.rxyz : sxyz;
        xyz[3 * pos] = x[j];
        xyz[3 * pos + 1] = y[j];
        xyz[3 * pos + 2] = z[j];
        (self ? L.rid : sid)[pos] = (int32_t)(first + i);
        slot_of_row[i] = self ? -1 : (int32_t)(L.ret_base[d[j]] + k);
      }
      for (int t = lo[j];; ++t) {  // ghost copies: one round per target slab
        if (valid && t == d[j]) ++t;
        const bool more = valid && t <= hi[j];
        if (!__any_sync(0xffffffffu, more)) break;
        const unsigned g = agg_add(gcnt, t, more);
        if (more) {
          const bool self = t == L.me;
          const int64_t pos = (self ? L.self_base + L.self_owned : L.ghost_base[t]) + (int64_t)base[G + t] + g;
          float *xyz = self ? L.rxyz : sxyz;
          xyz[3 * pos] = x[j];
          xyz[3 * pos + 1] = y[j];
          xyz[3 * pos + 2] = z[j];
          (self ? L.rid : sid)[pos] = (int32_t)(first + i);
        }
      }
    }
    __syncthreads();
  }
}

// Received layout: per source rank p, [owned block | ghost block] from
// seg_start[p].
struct RecvLayout {
  int64_t seg_start[kMaxSlabRanks + 1];
  int64_t owned[kMaxSlabRanks];
  int64_t ret_off[kMaxSlabRanks];  // return-buffer position of p's owned block
  int G;
  __device__ __forceinline__ int seg(int64_t j) const {
    int p = 0;
    while (p + 1 < G && j >= seg_start[p + 1]) ++p;
    return p;
  }
};

// (global id, local label) of every received ghost and every near owned
// point with a label (noise points link nothing).
__global__ void __launch_bounds__(256) k_slab_pairs(const float *__restrict__ rxyz, const int32_t *__restrict__ rid,
                                                    const int32_t *__restrict__ rlab, int64_t nrecv, RecvLayout R,
                                                    Splitters SP, uint2 *pairs, unsigned long long *cursor) {
  __shared__ Route S;
  S.load(SP);
  const int64_t st = (int64_t)gridDim.x * blockDim.x;
  const int64_t t0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  for (int64_t wb = t0 - (threadIdx.x & 31); wb < nrecv; wb += st) {
    const int64_t j = wb + (threadIdx.x & 31);
    bool emit = false;
    int32_t lab = -1;
    if (j < nrecv) {
      lab = rlab[j];
      if (lab >= 0) {
        const int p = R.seg(j);
        if (j - R.seg_start[p] >= R.owned[p]) {
          emit = true;  // a ghost copy
        } else {
          int d, lo, hi;
          S.route(rxyz[3 * j], d, lo, hi);
          emit = lo != d || hi != d;  // an owned point shipped as a ghost
        }
      }
    }
    const unsigned long long slot = agg_slot(cursor, 0, emit);
    if (emit) pairs[slot] = make_uint2((uint32_t)rid[j], (uint32_t)lab);
  }
}

__device__ __forceinline__ int64_t lower_bound_u64(const uint64_t *a, int64_t m, uint64_t v) {
  int64_t lo = 0, hi = m;
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (a[mid] < v) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}

__global__ void k_pairs_split(const uint2 *__restrict__ pairs, int64_t m, uint64_t *gid, uint32_t *glab,
                              uint64_t *lab) {
  const int64_t st = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m; i += st) {
    const uint2 p = pairs[i];
    gid[i] = p.x;
    glab[i] = p.y;
    lab[i] = p.y;
  }
}

// Copies of one point (equal global ids, adjacent after the sort) link their
// labels; a label's vertex is its first position in the sorted label array.
__global__ void k_slab_unions(const uint64_t *__restrict__ gid, const uint32_t *__restrict__ glab, int64_t m,
                              const uint64_t *__restrict__ slab, int32_t *parent) {
  const int64_t st = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x + 1; i < m; i += st) {
    const uint64_t g = gid[i];
    if (g == kNoId || g != gid[i - 1]) continue;
    const int32_t a = (int32_t)lower_bound_u64(slab, m, glab[i - 1]);
    const int32_t b = (int32_t)lower_bound_u64(slab, m, glab[i]);
    if (a != b) uf_union(parent, a, b);
  }
}

__global__ void k_slab_comp(const uint64_t *__restrict__ slab, int64_t m, const int32_t *__restrict__ parent,
                            int32_t *__restrict__ comp) {
  const int64_t st = (int64_t)gridDim.x * blockDim.x;
  for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < m; v += st)
    comp[v] = (int32_t)slab[uf_root(parent, (int32_t)v)];
}

// Owned entries: final label (component minimum when the local label is
// linked, else the local label), written to the return block of its source.
__global__ void k_slab_relabel(const int32_t *__restrict__ rlab, const int32_t *__restrict__ rid, int64_t nrecv,
                               RecvLayout R, const uint64_t *__restrict__ slab, const int32_t *__restrict__ comp,
                               int64_t m, int32_t *__restrict__ ret, int me, int64_t first,
                               int32_t *__restrict__ labels, uint8_t *__restrict__ core) {
  const int64_t st = (int64_t)gridDim.x * blockDim.x;
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < nrecv; j += st) {
    const int p = R.seg(j);
    const int64_t k = j - R.seg_start[p];
    if (k >= R.owned[p]) continue;
    int32_t a = rlab[j];
    if (a >= 0 && m > 0) {
      const int64_t pos = lower_bound_u64(slab, m, (uint64_t)a);
      if (pos < m && slab[pos] == (uint64_t)a) a = comp[pos];
    }
    if (p == me) {  // this rank's own rows: final labels in input order
      const int64_t row = (int64_t)rid[j] - first;
      labels[row] = a;
      core[row] = a >= 0;
    } else {
      ret[R.ret_off[p] + k] = a;
    }
  }
}

__global__ void k_slab_unpack(const int32_t *__restrict__ slot_of_row, const int32_t *__restrict__ ret, int64_t n,
                              int32_t *__restrict__ labels, uint8_t *__restrict__ core) {
  const int64_t st = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += st) {
    const int32_t s = slot_of_row[i];
    if (s < 0) continue;  // a row this rank owns itself (k_slab_relabel wrote it)
    const int32_t l = ret[s];
    labels[i] = l;
    core[i] = l >= 0;
  }
}

// Labels of a rank that ran the single-GPU FoF in place: local smallest index
// -> global (first + local).
__global__ void k_slab_offset(int32_t *labels, int64_t n, int32_t first) {
  const int64_t st = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += st) {
    const int32_t l = labels[i];
    if (l >= 0) labels[i] = l + first;
  }
}

__global__ void k_copy_u64(const unsigned long long *__restrict__ src, unsigned long long *dst, int count) {
  for (int i = threadIdx.x; i < count; i += blockDim.x) dst[i] = src[i];
}

__global__ void k_iota_i32(int32_t *a, int64_t n) {
  const int64_t st = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += st) a[i] = (int32_t)i;
}

}  // namespace

// ---------------------------------------------------------------------------
// host driver
// ---------------------------------------------------------------------------
struct SlabRank {
  SlabInput in;
  int rank = 0;
  DevBuf<uint32_t> hist;
  DevBuf<float> split;
  DevBuf<unsigned long long> counts, cmat, cursor;
  DevBuf<float> sxyz, rxyz;
  DevBuf<int32_t> sid, rid, slot_of_row, rlab, ret_send, ret_recv;
  DevBuf<uint8_t> rcore;
  DevBuf<uint2> pairs;
  int64_t nrecv = 0;
  Splitters S{};
  std::vector<size_t> soff, sbytes, roff, rbytes;  // per peer
};

void fof_slabs(std::vector<SlabInput> &inputs, SlabExchange &ex, float eps) {
  const int L = (int)inputs.size();
  const int G = ex.size();
  if (G < 1 || G > kMaxSlabRanks) throw InvalidArgument("slab FoF: 1..32 ranks");
  if (!(eps > 0.f) || !std::isfinite(eps)) throw InvalidArgument("dbscan: eps must be positive and finite");
  std::vector<std::unique_ptr<SlabRank>> R;
  std::vector<Ctx *> ctx;
  for (int l = 0; l < L; ++l) {
    R.emplace_back(new SlabRank);
    R[l]->in = inputs[l];
    R[l]->rank = ex.rank_of(l);
    ctx.push_back(inputs[l].c);
    if (inputs[l].n < 0 || inputs[l].first < 0 || inputs[l].first + inputs[l].n > 0x7fffffffLL)
      throw InvalidArgument("slab FoF: global indices must fit int32");
  }
  auto each = [&](auto &&f) {
    for (int l = 0; l < L; ++l) {
      ScopedDevice sd(ctx[l]->device);
      f(l, *R[l], *ctx[l]);
    }
  };
  const double w = (double)eps * (1.0 + 1.0 / 1048576.0);

  // A: sampled x histogram, summed over ranks
  each([&](int l, SlabRank &r, Ctx &c) {
    if (G == 1) return;  // one slab: no splitters
    r.hist = DevBuf<uint32_t>(kHistBins, c.stream);
    SPB_CUDA(cudaMemsetAsync(r.hist.get(), 0, kHistBins * sizeof(uint32_t), c.stream));
    if (r.in.n > 0) {
      const int64_t stride = std::max<int64_t>(1, r.in.n >> 20);
      k_slab_hist<<<grid_for((r.in.n + stride - 1) / stride, 256, 148 * 8), 256, 0, c.stream>>>(r.in.pts, r.in.n,
                                                                                                   stride,
                                                                                                   r.hist.get());
      SPB_LAUNCHED();
    }
  });
  if (G > 1) {
    std::vector<uint32_t *> hb;
    for (auto &r : R) hb.push_back(r->hist.get());
    ex.allreduce_u32(ctx, hb, kHistBins);
  }
  // B: splitters, per-destination counts, all-gathered
  each([&](int l, SlabRank &r, Ctx &c) {
    r.split = DevBuf<float>(kMaxSlabRanks, c.stream);
    if (G > 1) {
      k_slab_splitters<<<1, 1024, 0, c.stream>>>(r.hist.get(), G, r.split.get());
      SPB_LAUNCHED();
    }
    r.counts = DevBuf<unsigned long long>(3 * G, c.stream);
    r.cmat = DevBuf<unsigned long long>((size_t)3 * G * G, c.stream);
    SPB_CUDA(cudaMemsetAsync(r.counts.get(), 0, 3 * G * sizeof(unsigned long long), c.stream));
    mark(c, "slab_split");
  });
  each([&](int l, SlabRank &r, Ctx &c) {
    (void)l;
    r.S = Splitters{r.split.get(), G, w};
    if (r.in.n > 0) {
      k_slab_count<<<grid_for(r.in.n, 256, 148 * 8), 256, 0, c.stream>>>(r.in.pts, r.in.n, r.S, r.counts.get());
      SPB_LAUNCHED();
    }
  });
  {
    std::vector<const void *> snd;
    std::vector<void *> rcv;
    for (auto &r : R) {
      snd.push_back(r->counts.get());
      rcv.push_back(r->cmat.get());
    }
    if (G > 1) {
      ex.allgather(ctx, snd, rcv, 3 * G * sizeof(unsigned long long));
    } else {
      ScopedDevice sd(ctx[0]->device);
      SPB_CUDA(cudaMemcpyAsync(rcv[0], snd[0], 3 * sizeof(unsigned long long), cudaMemcpyDeviceToDevice,
                               ctx[0]->stream));
    }
  }
  // the one host read that sizes everything: the G x 3G count matrix
  std::vector<unsigned long long> mat((size_t)3 * G * G);
  {
    ScopedDevice sd(ctx[0]->device);
    k_copy_u64<<<1, 256, 0, ctx[0]->stream>>>(R[0]->cmat.get(), ex.mapped(mat.size()), (int)mat.size());
    SPB_LAUNCHED();
    SPB_CUDA(cudaStreamSynchronize(ctx[0]->stream));
    std::memcpy(mat.data(), ex.host_mat, mat.size() * sizeof(unsigned long long));
  }
  auto owned = [&](int src, int dst) { return (int64_t)mat[(size_t)src * 3 * G + dst]; };
  auto ghost = [&](int src, int dst) { return (int64_t)mat[(size_t)src * 3 * G + G + dst]; };
  auto nearc = [&](int src, int dst) { return (int64_t)mat[(size_t)src * 3 * G + 2 * G + dst]; };
  int64_t pmax = 0;
  for (int r = 0; r < G; ++r) {
    int64_t p = 0;
    for (int s = 0; s < G; ++s) p += ghost(s, r) + nearc(s, r);
    pmax = std::max(pmax, p);
  }
  // An empty exchange (every rank's rows are its own, no point is a ghost
  // anywhere: one rank, or slabs further than eps apart) leaves each rank a
  // plain FoF over its own rows: run it in place, labels offset to global
  // indices.  The matrix is the same on every rank, so all ranks take this
  // branch together and no collective is left unmatched.
  bool exchange_empty = true;
  for (int a = 0; a < G; ++a)
    for (int b = 0; b < G; ++b)
      if (a != b && (owned(a, b) || ghost(a, b) || nearc(a, b))) exchange_empty = false;
  if (exchange_empty) {
    each([&](int l, SlabRank &r, Ctx &c) {
      (void)l;
      if (r.in.n > 0) {
        dbscan(c, r.in.pts, r.in.n, 3, eps, 2, 1, 64, r.in.labels, r.in.core, nullptr, nullptr);
        if (r.in.first != 0) {
          k_slab_offset<<<grid_for(r.in.n, 256, 148 * 8), 256, 0, c.stream>>>(r.in.labels, r.in.n,
                                                                             (int32_t)r.in.first);
          SPB_LAUNCHED();
        }
      }
      mark(c, "slab_local");
    });
    return;
  }

  // C: pack and exchange (xyz, global id)
  std::vector<PackLayout> PL(L);
  std::vector<RecvLayout> RL(L);
  for (int l = 0; l < L; ++l) {
    SlabRank &r = *R[l];
    const int me = r.rank;
    int64_t pos = 0, ret = 0;
    r.soff.assign(G, 0);
    r.sbytes.assign(G, 0);
    r.roff.assign(G, 0);
    r.rbytes.assign(G, 0);
    // send blocks per peer; the self block is written straight into the
    // receive buffer
    for (int d = 0; d < G; ++d) {
      const bool self = d == me;
      PL[l].owned_base[d] = pos;
      PL[l].ghost_base[d] = pos + (self ? 0 : owned(me, d));
      PL[l].ret_base[d] = ret;
      r.soff[d] = (size_t)pos;
      r.sbytes[d] = self ? 0 : (size_t)(owned(me, d) + ghost(me, d));
      pos += (int64_t)r.sbytes[d];
      ret += self ? 0 : owned(me, d);
    }
    int64_t rpos = 0, rret = 0;
    RL[l].G = G;
    for (int p = 0; p < G; ++p) {
      const bool self = p == me;
      RL[l].seg_start[p] = rpos;
      RL[l].owned[p] = owned(p, me);
      RL[l].ret_off[p] = rret;
      r.roff[p] = (size_t)rpos;
      r.rbytes[p] = self ? 0 : (size_t)(owned(p, me) + ghost(p, me));
      if (self) PL[l].self_base = rpos;
      rpos += owned(p, me) + ghost(p, me);
      rret += self ? 0 : owned(p, me);
    }
    RL[l].seg_start[G] = rpos;
    PL[l].me = me;
    PL[l].self_owned = owned(me, me);
    r.nrecv = rpos;
  }
  each([&](int l, SlabRank &r, Ctx &c) {
    int64_t nsend = 0;
    for (int d = 0; d < G; ++d) nsend += (int64_t)r.sbytes[d];
    r.sxyz = DevBuf<float>((size_t)std::max<int64_t>(nsend, 1) * 3, c.stream);
    r.sid = DevBuf<int32_t>((size_t)std::max<int64_t>(nsend, 1), c.stream);
    r.slot_of_row = DevBuf<int32_t>((size_t)std::max<int64_t>(r.in.n, 1), c.stream);
    r.rxyz = DevBuf<float>((size_t)std::max<int64_t>(r.nrecv, 1) * 3, c.stream);
    r.rid = DevBuf<int32_t>((size_t)std::max<int64_t>(r.nrecv, 1), c.stream);
    r.cursor = DevBuf<unsigned long long>(2 * G, c.stream);
    SPB_CUDA(cudaMemsetAsync(r.cursor.get(), 0, 2 * G * sizeof(unsigned long long), c.stream));
    PL[l].rxyz = r.rxyz.get();
    PL[l].rid = r.rid.get();
    if (r.in.n > 0) {
      k_slab_pack<<<grid_for((r.in.n + PK_ITEMS - 1) / PK_ITEMS, 256, 148 * 8), 256, 0, c.stream>>>(r.in.pts, r.in.n, r.in.first, r.S, PL[l],
                                                                         r.cursor.get(), r.sxyz.get(), r.sid.get(),
                                                                         r.slot_of_row.get());
      SPB_LAUNCHED();
    }
    mark(c, "slab_route");
  });
  {
    std::vector<const void *> sx, si;
    std::vector<void *> rx, ri;
    std::vector<std::vector<size_t>> so3(L), sb3(L), ro3(L), rb3(L), so4(L), sb4(L), ro4(L), rb4(L);
    for (int l = 0; l < L; ++l) {
      SlabRank &r = *R[l];
      sx.push_back(r.sxyz.get());
      si.push_back(r.sid.get());
      rx.push_back(r.rxyz.get());
      ri.push_back(r.rid.get());
      for (int p = 0; p < G; ++p) {
        so3[l].push_back(r.soff[p] * 12);
        sb3[l].push_back(r.sbytes[p] * 12);
        ro3[l].push_back(r.roff[p] * 12);
        rb3[l].push_back(r.rbytes[p] * 12);
        so4[l].push_back(r.soff[p] * 4);
        sb4[l].push_back(r.sbytes[p] * 4);
        ro4[l].push_back(r.roff[p] * 4);
        rb4[l].push_back(r.rbytes[p] * 4);
      }
    }
    ex.alltoallv(ctx, sx, so3, sb3, rx, ro3, rb3);
    ex.alltoallv(ctx, si, so4, sb4, ri, ro4, rb4);
  }
  // D: local FoF over owned + ghost points, labels in global-id space
  each([&](int l, SlabRank &r, Ctx &c) {
    r.sxyz.reset();
    r.sid.reset();
    mark(c, "slab_exchange");
    r.rlab = DevBuf<int32_t>((size_t)std::max<int64_t>(r.nrecv, 1), c.stream);
    r.rcore = DevBuf<uint8_t>((size_t)std::max<int64_t>(r.nrecv, 1), c.stream);
    if (r.nrecv > 0) dbscan(c, r.rxyz.get(), r.nrecv, 3, eps, 2, 1, 64, r.rlab.get(), r.rcore.get(), nullptr,
                            r.rid.get());
  });
  // E: (global id, label) pairs of every ghost copy and near owned point
  const int64_t M = pmax * G;
  each([&](int l, SlabRank &r, Ctx &c) {
    r.pairs = DevBuf<uint2>((size_t)std::max<int64_t>(M, 1), c.stream);
    if (M > 0) {
      SPB_CUDA(cudaMemsetAsync(r.pairs.get(), 0xff, (size_t)M * sizeof(uint2), c.stream));
      SPB_CUDA(cudaMemsetAsync(r.cursor.get(), 0, sizeof(unsigned long long), c.stream));
      if (r.nrecv > 0) {
        k_slab_pairs<<<grid_for(r.nrecv, 256, 148 * 8), 256, 0, c.stream>>>(
            r.rxyz.get(), r.rid.get(), r.rlab.get(), r.nrecv, RL[l], r.S, r.pairs.get() + (size_t)r.rank * pmax,
            r.cursor.get());
        SPB_LAUNCHED();
      }
    }
  });
  if (M > 0) {
    std::vector<const void *> snd;
    std::vector<void *> rcv;
    for (auto &r : R) {
      snd.push_back(r->pairs.get() + (size_t)r->rank * pmax);
      rcv.push_back(r->pairs.get());
    }
    ex.allgather(ctx, snd, rcv, (size_t)pmax * sizeof(uint2));
  }
  // F + G: unite linked labels, relabel owned entries, return them
  for (int l = 0; l < L; ++l) {
    SlabRank &r = *R[l];
    Ctx &c = *ctx[l];
    ScopedDevice sd(c.device);
    DevBuf<uint64_t> gk, gk2, lk, lk2;
    DevBuf<uint32_t> gv, gv2, lv, lv2;
    DevBuf<int32_t> parent, comp;
    uint64_t *slabels = nullptr;
    if (M > 0) {
      gk = DevBuf<uint64_t>((size_t)M, c.stream);
      gk2 = DevBuf<uint64_t>((size_t)M, c.stream);
      lk = DevBuf<uint64_t>((size_t)M, c.stream);
      lk2 = DevBuf<uint64_t>((size_t)M, c.stream);
      gv = DevBuf<uint32_t>((size_t)M, c.stream);
      gv2 = DevBuf<uint32_t>((size_t)M, c.stream);
      lv = DevBuf<uint32_t>((size_t)M, c.stream);
      lv2 = DevBuf<uint32_t>((size_t)M, c.stream);
      const unsigned g = grid_for(M, 256, 148 * 8);
      k_pairs_split<<<g, 256, 0, c.stream>>>(r.pairs.get(), M, gk.get(), gv.get(), lk.get());
      SPB_LAUNCHED();
      uint64_t *ka = gk.get(), *kb = gk2.get(), *la = lk.get(), *lb = lk2.get();
      uint32_t *va = gv.get(), *vb = gv2.get(), *wa = lv.get(), *wb = lv2.get();
      radix_sort_pairs(c, &ka, &va, &kb, &vb, M, 32, false);
      radix_sort_pairs(c, &la, &wa, &lb, &wb, M, 32, true);
      slabels = la;
      parent = DevBuf<int32_t>((size_t)M, c.stream);
      comp = DevBuf<int32_t>((size_t)M, c.stream);
      k_iota_i32<<<g, 256, 0, c.stream>>>(parent.get(), M);
      SPB_LAUNCHED();
      k_slab_unions<<<g, 256, 0, c.stream>>>(ka, va, M, la, parent.get());
      SPB_LAUNCHED();
      k_slab_comp<<<g, 256, 0, c.stream>>>(la, M, parent.get(), comp.get());
      SPB_LAUNCHED();
    }
    int64_t nret_send = 0;
    for (int p = 0; p < G; ++p) nret_send += p == r.rank ? 0 : RL[l].owned[p];
    r.ret_send = DevBuf<int32_t>((size_t)std::max<int64_t>(nret_send, 1), c.stream);
    if (r.nrecv > 0) {
      k_slab_relabel<<<grid_for(r.nrecv, 256, 148 * 8), 256, 0, c.stream>>>(
          r.rlab.get(), r.rid.get(), r.nrecv, RL[l], slabels, comp.get(), M, r.ret_send.get(), r.rank, r.in.first,
          r.in.labels, r.in.core);
      SPB_LAUNCHED();
    }
    r.ret_recv = DevBuf<int32_t>((size_t)std::max<int64_t>(r.in.n, 1), c.stream);
    r.rxyz.reset();
    r.rid.reset();
    r.rlab.reset();
    r.rcore.reset();
    r.pairs.reset();
    mark(c, "slab_merge");
  }
  {
    std::vector<const void *> snd;
    std::vector<void *> rcv;
    std::vector<std::vector<size_t>> so(L), sb(L), ro(L), rb(L);
    for (int l = 0; l < L; ++l) {
      SlabRank &r = *R[l];
      const int me = r.rank;
      snd.push_back(r.ret_send.get());
      rcv.push_back(r.ret_recv.get());
      for (int p = 0; p < G; ++p) {
        so[l].push_back((size_t)RL[l].ret_off[p] * 4);
        sb[l].push_back(p == me ? 0 : (size_t)owned(p, me) * 4);
        ro[l].push_back((size_t)PL[l].ret_base[p] * 4);
        rb[l].push_back(p == me ? 0 : (size_t)owned(me, p) * 4);
      }
    }
    ex.alltoallv(ctx, snd, so, sb, rcv, ro, rb);
  }
  each([&](int l, SlabRank &r, Ctx &c) {
    int64_t from_peers = 0;  // rows of this rank owned elsewhere
    for (int p = 0; p < G; ++p) from_peers += p == r.rank ? 0 : owned(r.rank, p);
    if (from_peers > 0) {
      k_slab_unpack<<<grid_for(r.in.n, 256, 148 * 8), 256, 0, c.stream>>>(r.slot_of_row.get(), r.ret_recv.get(),
                                                                           r.in.n, r.in.labels, r.in.core);
      SPB_LAUNCHED();
    }
    mark(c, "slab_return");
  });
}

// ---------------------------------------------------------------------------
// communicators
// ---------------------------------------------------------------------------
SlabExchange *nccl_exchange_create(int device, int nranks, int rank, const uint8_t id[128]) {
  if (nranks < 1 || nranks > kMaxSlabRanks || rank < 0 || rank >= nranks)
    throw InvalidArgument("slab communicator: bad rank / size");
  ScopedDevice sd(device);
  std::unique_ptr<NcclExchange> x(new NcclExchange);
  ncclUniqueId uid;
  std::memcpy(&uid, id, 128);
  nccl_check(NcclApi::get().CommInitRank(&x->comm, nranks, uid, rank), "ncclCommInitRank");
  x->owned = true;
  x->G = nranks;
  x->me = rank;
  return x.release();
}

SlabExchange *nccl_exchange_wrap(void *comm) {
  if (!comm) throw InvalidArgument("slab communicator: null ncclComm_t");
  std::unique_ptr<NcclExchange> x(new NcclExchange);
  x->comm = static_cast<ncclComm_t>(comm);
  nccl_check(NcclApi::get().CommCount(x->comm, &x->G), "ncclCommCount");
  nccl_check(NcclApi::get().CommUserRank(x->comm, &x->me), "ncclCommUserRank");
  if (x->G > kMaxSlabRanks) throw InvalidArgument("slab FoF: at most 32 ranks");
  return x.release();
}

int exchange_size(const SlabExchange *x) { return x->size(); }
int exchange_rank(const SlabExchange *x) { return x->rank_of(0); }
void exchange_destroy(SlabExchange *x) { delete x; }

void fof_slabs_multi(std::vector<SlabInput> &inputs, float eps) {
  std::vector<Ctx *> c;
  for (auto &i : inputs) c.push_back(i.c);
  LocalExchange ex(c);
  fof_slabs(inputs, ex, eps);
}

}  // namespace spb
