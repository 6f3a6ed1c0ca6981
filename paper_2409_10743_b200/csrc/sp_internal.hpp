// Host-side internals shared by the translation units of libspb200.so.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <initializer_list>
#include <string>
#include <utility>
#include <vector>

#include "sp_common.cuh"

namespace spb {

// A context: one device, one stream, stream-ordered allocations from the
// device's default memory pool (release threshold raised so freed blocks stay
// reserved — a caching allocator without host synchronisation).
struct Ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  bool owns_stream = false;
  std::string last_error;
  int64_t launches = 0;
  // Phase marks of the current call: events recorded on the stream between
  // pipeline stages; (name_i, ms_i) = time from mark i-1 to mark i.
  std::vector<cudaEvent_t> event_pool;
  std::vector<const char *> mark_names;
  size_t marks_used = 0;
  std::vector<std::pair<std::string, double>> phases;
  // SP_FLAG_ASYNC: calls only enqueue work (no host synchronisation); input
  // validity errors found on the device accumulate in d_err and are reported
  // by the next sp_ctx_synchronize.
  int flags = 0;
  int *d_err = nullptr;
  cudaStream_t h2d = nullptr, d2h = nullptr;  // copy streams for host buffers
  bool async() const { return (flags & 1) != 0; }
  // SP_FLAG_STATS: diagnostic kernels count traversal work into counters
  bool stats() const { return (flags & 2) != 0; }
  // Double-buffered device staging for host arrays (per call parity, per
  // argument position).  A slot is reused two calls later, after the event
  // recorded when its last consumer (kernels for inputs, the download for
  // outputs) finished — explicit, so copy streams never wait on unrelated
  // compute the way cross-stream pool reuse would make them.
  struct Staging {
    void *p = nullptr;
    size_t cap = 0;
    cudaEvent_t done = nullptr;  // last consumer of this slot
  };
  Staging in_stage[2][8], out_stage[2][8];
  int64_t calls = 0;
  int in_used = 0, out_used = 0;
  // diagnostic counters of the last call (e.g. "fof_cells": non-empty cells)
  std::vector<std::pair<std::string, int64_t>> counters;
  uint8_t *peek_buf = nullptr;  // host-mapped pinned scratch for peek()
  void count(const char *name, int64_t v) { counters.emplace_back(name, v); }
};

// Small device-to-host reads (sizes, flags, bounds) through host-mapped pinned
// memory written by a kernel, then a wait on the context stream.  No copy
// engine is involved, so the read never queues behind a bulk download on the
// same engine (with SP_FLAG_ASYNC the previous call's results are still
// streaming out while the next call needs its scene bounds).
struct PeekItem {
  const void *src;  // device
  void *dst;        // host
  uint32_t bytes;   // <= 64
};
void peek(Ctx &c, std::initializer_list<PeekItem> items);

// Record a phase boundary on the context stream (cheap; no host sync).
void mark(Ctx &c, const char *name);
// Resolve the marks of the finished call into c.phases (after a sync).
void resolve_marks(Ctx &c);
void reset_marks(Ctx &c);

// Stream-keyed caching allocator (sp_alloc.cpp): blocks freed on a registered
// stream are reused by later requests on that stream without driver calls.
void cache_register_stream(cudaStream_t s);
void cache_unregister_stream(cudaStream_t s);
void *cache_alloc(size_t bytes, cudaStream_t s);  // throws CudaError
void cache_free(void *p, cudaStream_t s);
void cache_drain();  // return every cached block of every stream to the driver

template <class T>
struct DevBuf {
  T *p = nullptr;
  size_t n = 0;
  cudaStream_t s = nullptr;
  DevBuf() = default;
  DevBuf(size_t count, cudaStream_t stream) : n(count), s(stream) {
    if (count) p = static_cast<T *>(cache_alloc(count * sizeof(T), stream));
  }
  DevBuf(const DevBuf &) = delete;
  DevBuf &operator=(const DevBuf &) = delete;
  DevBuf(DevBuf &&o) noexcept : p(o.p), n(o.n), s(o.s) { o.p = nullptr; o.n = 0; }
  DevBuf &operator=(DevBuf &&o) noexcept {
    reset();
    p = o.p; n = o.n; s = o.s;
    o.p = nullptr; o.n = 0;
    return *this;
  }
  ~DevBuf() { reset(); }
  void reset() {
    if (p) cache_free(p, s);
    p = nullptr;
    n = 0;
  }
  T *release() { T *q = p; p = nullptr; n = 0; return q; }
  T *get() const { return p; }
};

// A device-resident hierarchy (the B200 counterpart of Bvh<D>, bvh.hpp:43-86).
struct Tree {
  int64_t n = 0;
  int dim = 3;
  int width = 64;
  bool points = true;       // built over point boxes (min == max)
  float4 *nodes = nullptr;  // 2 float4 per node, 2n-1 nodes (NodeRef order)
  int32_t *perm = nullptr;  // leaf position -> object index
  float *scene = nullptr;   // device float[6]: min xyz, max xyz
  float4 *leafpt = nullptr; // point trees: leaf p as {x, y, z, rope} (16 B)
  cudaStream_t stream = nullptr;
  Tree() = default;
  Tree(const Tree &) = delete;
  Tree &operator=(const Tree &) = delete;
  ~Tree() { free_all(); }
  void free_all() {
    cache_free(nodes, stream);
    cache_free(perm, stream);
    cache_free(scene, stream);
    cache_free(leafpt, stream);
    leafpt = nullptr;
    nodes = nullptr;
    perm = nullptr;
    scene = nullptr;
  }
};

// ---- build stages (sp_build.cu) ----------------------------------------------
// objects: device float[n*dim] (points) or float[n*2*dim] (boxes).
// Computes the scene box into scene[6] and returns false (after a sync) if any
// coordinate is non-finite.
void scene_bounds(Ctx &c, const float *objects, int64_t n, int dim, bool points, float *scene, int *bad);
// codes[i] = code_of(centroid(object i), scene); vals[i] = i.
void morton_codes(Ctx &c, const float *objects, int64_t n, int dim, bool points, int width, const float *scene,
                  uint64_t *codes, uint32_t *vals);
// Stable LSD radix sort of (key, value) pairs over key bits [0, key_bits).
// Sorted output ends in (*keys, *vals); the alternate buffers are scratch and
// the pointers may be swapped.
void radix_sort_pairs(Ctx &c, uint64_t **keys, uint32_t **vals, uint64_t **keys_alt, uint32_t **vals_alt, int64_t n,
                      int key_bits, bool vals_iota);
// hist_in: the pass digit counts already accumulated by the kernel that wrote
// the keys (RS_HIST_ENTRIES(npass) entries, zeroed before that kernel; see
// hist_acc in sp_common.cuh), or nullptr to count them here.
void radix_sort_pairs(Ctx &c, uint32_t **keys, uint32_t **vals, uint32_t **keys_alt, uint32_t **vals_alt, int64_t n,
                      int key_bits, bool vals_iota, uint32_t *hist_in = nullptr);
void radix_sort_pairs_40(Ctx &c, const uint64_t *keys, uint32_t **vals, uint32_t **vals_alt, uint32_t *k32,
                         uint32_t *k32_alt, int64_t n, bool vals_iota, uint32_t *hist_in = nullptr);
constexpr int RS_HIST_ENTRIES(int npass) { return npass * 256 + npass; }
// Full Bvh::build into `t` (allocates t.nodes/perm/scene). Throws
// InvalidArgument on non-finite input.
void build_tree(Ctx &c, const float *objects, int64_t n, int dim, bool points, int width, Tree &t);
// LBVH over m objects already in key order (strictly increasing keys): leaf p
// is object p with box boxes[p] (2*dim floats); no sort, identity permutation.
// delta_in: the key-split array (m - 1 entries, k_delta's values) when the
// caller already computed it; keys are then not read.
void build_sorted_hierarchy(Ctx &c, const uint64_t *keys, int64_t m, int dim, const float *boxes, Tree &t,
                            DevBuf<int32_t> *delta_in = nullptr);
// sort_queries: the stable 64-bit Morton order of points against their scene.
void sort_points(Ctx &c, const float *pts, int64_t n, int dim, int32_t *order);


// Host side of the SM-affine schedule (SmSliceWalk, sp_common.cuh): one
// zeroed chunk counter per SM and a fully resident grid.  The SM count and
// each kernel's residency are queried once per process (device 0 of the pool
// and every B200 agree), not per call.
int sm_count(int device);
int resident_blocks(const void *kernel, int threads);
struct SmSlices {
  int nsm = 0;
  DevBuf<unsigned long long> ctr;
  explicit SmSlices(Ctx &c) {
    nsm = sm_count(c.device);
    ctr = DevBuf<unsigned long long>((size_t)nsm, c.stream);
    SPB_CUDA(cudaMemsetAsync(ctr.get(), 0, (size_t)nsm * sizeof(unsigned long long), c.stream));
  }
  template <class K>
  unsigned grid(K kernel, int threads) const {
    return (unsigned)(nsm * resident_blocks(reinterpret_cast<const void *>(kernel), threads));
  }
};
}  // namespace spb
