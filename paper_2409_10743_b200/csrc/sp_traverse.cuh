// Stackless rope traversal primitives and the lock-free union-find shared by
// the query and clustering kernels.
#pragma once

#include "sp_common.cuh"

namespace spb {

// Node field access for the unified 32-byte node layout (see sp_common.cuh).
__device__ __forceinline__ int32_t node_link(const float4 &lo) { return __float_as_int(lo.w); }  // left / object
__device__ __forceinline__ int32_t node_rope(const float4 &hi) { return __float_as_int(hi.w); }

// Sphere range-count walk from the root (traverse_range, traversal.hpp:45-60):
// on a leaf hit count it (stop once `cap` is reached, the kTerminateQuery of
// dbscan.hpp:165-166), then follow the rope; at an internal node descend left
// on a hit, else follow the rope.  `thr` is radius_threshold(r).
__device__ __forceinline__ int32_t count_sphere(const float4 *__restrict__ nodes, int64_t n, float cx, float cy,
                                                float cz, double thr, int32_t cap) {
  int32_t c = 0;
  int32_t cur = 0;  // root (bvh.hpp:67-71): internal 0, or leaf_ref(0) == 0 when n == 1
  const int64_t first_leaf = n - 1;
  while (cur != kSentinel) {
    const float4 lo = ld_node(nodes, 2 * (int64_t)cur);
    const float4 hi = ld_node(nodes, 2 * (int64_t)cur + 1);
    const bool hit = gap2(cx, cy, cz, lo, hi) <= thr;
    if (cur >= first_leaf) {
      if (hit && ++c == cap) break;
      cur = node_rope(hi);
    } else {
      cur = hit ? node_link(lo) : node_rope(hi);
    }
  }
  return c;
}

// ---- lock-free union-find (union_find.hpp:17-59) ------------------------------
// Invariant parent[x] <= x: the larger root is hooked under the smaller with a
// CAS that only succeeds on a root, so roots are set minima and every pointer
// only ever decreases.  find() shortens paths with plain stores; they are
// benign because each store writes an ancestor of the old value.
__device__ __forceinline__ int32_t uf_find(int32_t *parent, int32_t x) {
  int32_t p = parent[x];
  if (p != x) {
    int32_t prev = x, next;
    while (p > (next = parent[p])) {
      parent[prev] = next;
      prev = p;
      p = next;
    }
  }
  return p;
}

__device__ __forceinline__ void uf_union(int32_t *parent, int32_t a, int32_t b) {
  a = uf_find(parent, a);
  b = uf_find(parent, b);
  while (a != b) {
    if (a > b) {
      int32_t t = a;
      a = b;
      b = t;
    }
    int32_t old = atomicCAS(&parent[b], b, a);
    if (old == b) return;
    b = uf_find(parent, old);
    a = uf_find(parent, a);
  }
}

// Full root lookup without modification (after all unions are done).
__device__ __forceinline__ int32_t uf_root(const int32_t *parent, int32_t x) {
  int32_t p = parent[x];
  while (p != x) {
    x = p;
    p = parent[x];
  }
  return p;
}

}  // namespace spb
