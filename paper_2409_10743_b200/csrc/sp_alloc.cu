// Stream-keyed caching allocator for the library's device temporaries.
//
// Every pipeline allocates its scratch (sort ping-pong buffers, trees, scan
// arrays, union-find state) per call.  cudaMallocAsync from the default pool
// costs ~1 ms per large block even when the pool has room, and occasionally
// tens to hundreds of milliseconds when the driver remaps pool memory: the GPU
// idles while the host waits (measured on C3, profiles/r01/README.md).  Blocks
// freed here go to a free list of the stream they were used on; a later
// request on the SAME stream may take a block immediately, because stream
// order guarantees the previous user's kernels have finished before the new
// user's kernels start (the caching-allocator model).  Blocks are returned to
// the driver when a context's stream is unregistered or an allocation fails.
#include <cuda_runtime.h>

#include <map>
#include <mutex>
#include <unordered_map>

#include "sp_internal.hpp"

namespace spb {

namespace {

struct Cache {
  std::mutex mu;
  std::unordered_map<cudaStream_t, std::multimap<size_t, void *>> free_blocks;
  std::unordered_map<void *, size_t> live;  // block -> rounded size
  std::unordered_map<cudaStream_t, int> registered;  // stream -> contexts using it
};

Cache &cache() {
  static Cache *c = new Cache;  // never destroyed: frees may run during process exit
  return *c;
}

size_t round_size(size_t bytes) {
  if (bytes <= (1u << 20)) return (bytes + 511) & ~(size_t)511;
  return (bytes + (2u << 20) - 1) & ~(size_t)((2u << 20) - 1);
}

// Free every cached block of every stream (caller holds the lock).
void drain_all(Cache &c) {
  for (auto &kv : c.free_blocks)
    for (auto &b : kv.second) cudaFreeAsync(b.second, kv.first);
  c.free_blocks.clear();
}

}  // namespace

void cache_register_stream(cudaStream_t s) {
  Cache &c = cache();
  std::lock_guard<std::mutex> g(c.mu);
  ++c.registered[s];
}

void cache_unregister_stream(cudaStream_t s) {
  Cache &c = cache();
  std::lock_guard<std::mutex> g(c.mu);
  auto r = c.registered.find(s);
  if (r == c.registered.end() || --r->second > 0) return;
  c.registered.erase(r);
  auto it = c.free_blocks.find(s);
  if (it != c.free_blocks.end()) {
    for (auto &b : it->second) cudaFreeAsync(b.second, s);
    c.free_blocks.erase(it);
  }
}

void *cache_alloc(size_t bytes, cudaStream_t s) {
  if (bytes == 0) return nullptr;
  const size_t want = round_size(bytes);
  Cache &c = cache();
  std::lock_guard<std::mutex> g(c.mu);
  if (c.registered.count(s)) {
    auto &fl = c.free_blocks[s];
    auto it = fl.lower_bound(want);
    // best fit with bounded waste (12.5% or 8 MB)
    if (it != fl.end() && (it->first - want <= want / 8 || it->first - want <= (8u << 20))) {
      void *p = it->second;
      c.live[p] = it->first;
      fl.erase(it);
      return p;
    }
  }
  void *p = nullptr;
  cudaError_t e = cudaMallocAsync(&p, want, s);
  if (e != cudaSuccess) {
    cudaGetLastError();
    drain_all(c);
    cudaDeviceSynchronize();
    e = cudaMallocAsync(&p, want, s);
    if (e != cudaSuccess) {
      cudaGetLastError();
      throw CudaError(std::string("device allocation of ") + std::to_string(bytes) +
                      " bytes failed: " + cudaGetErrorString(e));
    }
  }
  c.live[p] = want;
  return p;
}

// Return every cached block of every stream and the default pool's reserved
// but unused memory (sp_ctx_create keeps freed pool memory reserved) to the
// driver, so that cudaMalloc and other processes can have it.
void cache_drain() {
  Cache &c = cache();
  {
    std::lock_guard<std::mutex> g(c.mu);
    drain_all(c);
  }
  cudaDeviceSynchronize();
  int dev = 0;
  cudaMemPool_t pool;
  if (cudaGetDevice(&dev) == cudaSuccess && cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess)
    cudaMemPoolTrimTo(pool, 0);
}

void cache_free(void *p, cudaStream_t s) {
  if (!p) return;
  Cache &c = cache();
  std::lock_guard<std::mutex> g(c.mu);
  auto it = c.live.find(p);
  const size_t sz = it == c.live.end() ? 0 : it->second;
  if (it != c.live.end()) c.live.erase(it);
  if (sz && c.registered.count(s)) {
    c.free_blocks[s].emplace(sz, p);
  } else {
    cudaFree(p);  // the stream may be gone (a tree outliving its context)
  }
}


int sm_count(int device) {
  static std::mutex mu;
  static std::map<int, int> cache;
  std::lock_guard<std::mutex> g(mu);
  auto it = cache.find(device);
  if (it != cache.end()) return it->second;
  int v = 0;
  SPB_CUDA(cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, device));
  cache[device] = v;
  return v;
}

int resident_blocks(const void *kernel, int threads) {
  static std::mutex mu;
  static std::map<std::pair<const void *, int>, int> cache;
  std::lock_guard<std::mutex> g(mu);
  const auto key = std::make_pair(kernel, threads);
  auto it = cache.find(key);
  if (it != cache.end()) return it->second;
  int v = 0;
  SPB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&v, kernel, threads, 0));
  if (v < 1) v = 1;
  cache[key] = v;
  return v;
}

}  // namespace spb
