// Stackless rope traversal primitives, the exact-with-fp32-filter distance
// predicates, and the lock-free union-find shared by the query and clustering
// kernels.
#pragma once

#include "sp_common.cuh"

namespace spb {

// Node field access for the unified 32-byte node layout (see sp_common.cuh).
__device__ __forceinline__ int32_t node_link(const float4 &lo) { return __float_as_int(lo.w); }  // left / object
__device__ __forceinline__ int32_t node_rope(const float4 &hi) { return __float_as_int(hi.w); }

// ---- the comparison rule of intersects(box, sphere) (geometry.hpp:116-119) --
// Exact decision: S <= thr with S the double-accumulated squared gap and thr =
// radius_threshold(r) (sp_common.cuh).  Hot loops first evaluate S in fp32
// (S32): every fp32 step is one correctly rounded operation, so with all
// relevant magnitudes normal |S32 - S| <= 6*2^-24 * S.  Hence
//   S32 <  lo32 = thr*(1 - 2^-20)  =>  exact hit,
//   S32 >  hi32 = thr*(1 + 2^-20)  =>  exact miss,
// and only the thin band between falls back to the exact f64 evaluation.
// Internal nodes need only a conservative superset (S32 <= hi32): a false
// positive costs one extra visit, never a wrong answer.  The filter is off
// (fast = false) when thr is outside [2^-90, 2^120], where subnormal or
// overflowing fp32 squares would break the bound (e.g. eps = 1e-30).
struct Radius {
  double thr;
  float lo32, hi32;
  int fast;
};

__host__ __device__ inline Radius make_radius(float r) {
  Radius R;
  R.thr = radius_threshold(r);
  R.fast = (R.thr >= 0x1p-90 && R.thr <= 0x1p120) ? 1 : 0;
  const double dlo = R.thr * (1.0 - 0x1p-20), dhi = R.thr * (1.0 + 0x1p-20);
  float flo = (float)dlo, fhi = (float)dhi;
#ifdef __CUDA_ARCH__
  if ((double)flo > dlo) flo = nextafterf(flo, 0.0f);
  if ((double)fhi < dhi) fhi = nextafterf(fhi, 3.4e38f);
#else
  if ((double)flo > dlo) flo = std::nextafter(flo, 0.0f);
  if ((double)fhi < dhi) fhi = std::nextafter(fhi, 3.4e38f);
#endif
  R.lo32 = flo;
  R.hi32 = fhi;
  return R;
}

__device__ __forceinline__ float sq3(float x, float y, float z) {
  return __fadd_rn(__fadd_rn(__fmul_rn(x, x), __fmul_rn(y, y)), __fmul_rn(z, z));
}

// Exact point-point test (a point box against a sphere centre).
__device__ __forceinline__ bool hit_point(const Radius &R, float cx, float cy, float cz, float qx, float qy,
                                          float qz) {
  if (R.fast) {
    const float s = sq3(__fsub_rn(qx, cx), __fsub_rn(qy, cy), __fsub_rn(qz, cz));
    if (s < R.lo32) return true;
    if (s > R.hi32) return false;
  }
  return dist2(cx, cy, cz, qx, qy, qz) <= R.thr;
}

__device__ __forceinline__ float gap32(float c, float lo, float hi) {
  return fmaxf(fmaxf(__fsub_rn(lo, c), __fsub_rn(c, hi)), 0.f);
}

// Exact box test (leaves of box trees).
__device__ __forceinline__ bool hit_box(const Radius &R, float cx, float cy, float cz, const float4 &lo,
                                        const float4 &hi) {
  if (R.fast) {
    const float s = sq3(gap32(cx, lo.x, hi.x), gap32(cy, lo.y, hi.y), gap32(cz, lo.z, hi.z));
    if (s < R.lo32) return true;
    if (s > R.hi32) return false;
  }
  return gap2(cx, cy, cz, lo, hi) <= R.thr;
}

// Conservative internal-node test: true whenever the exact test is true.
__device__ __forceinline__ bool maybe_box(const Radius &R, float cx, float cy, float cz, const float4 &lo,
                                          const float4 &hi) {
  if (R.fast) return sq3(gap32(cx, lo.x, hi.x), gap32(cy, lo.y, hi.y), gap32(cz, lo.z, hi.z)) <= R.hi32;
  return gap2(cx, cy, cz, lo, hi) <= R.thr;
}

// Sphere range-count walk from the root (traverse_range, traversal.hpp:45-60):
// on a leaf hit count it (stop once `cap` is reached, the kTerminateQuery of
// dbscan.hpp:165-166), then follow the rope; at an internal node descend left
// on a hit, else follow the rope.  For point trees `leafpt` holds each leaf as
// one float4 {x, y, z, rope}, so a leaf visit is a single 16-byte load.
__device__ __forceinline__ int32_t count_sphere(const float4 *__restrict__ nodes, const float4 *__restrict__ leafpt,
                                                int64_t n, float cx, float cy, float cz, const Radius &R,
                                                int32_t cap) {
  int32_t c = 0;
  int32_t cur = 0;  // root (bvh.hpp:67-71): internal 0, or leaf_ref(0) == 0 when n == 1
  const int64_t first_leaf = n - 1;
  while (cur != kSentinel) {
    if (cur >= first_leaf) {
      bool hit;
      int32_t next;
      if (leafpt) {
        const float4 L = ld_node(leafpt, cur - first_leaf);
        hit = hit_point(R, cx, cy, cz, L.x, L.y, L.z);
        next = __float_as_int(L.w);
      } else {
        float4 lo, hi;
        ld_node2(nodes, (int64_t)cur, lo, hi);
        hit = hit_box(R, cx, cy, cz, lo, hi);
        next = node_rope(hi);
      }
      // cap reached: end the walk through the loop test (a break here costs
      // the warp its per-iteration reconvergence)
      cur = (hit && ++c == cap) ? kSentinel : next;
    } else {
      float4 lo, hi;
      ld_node2(nodes, (int64_t)cur, lo, hi);
      cur = maybe_box(R, cx, cy, cz, lo, hi) ? node_link(lo) : node_rope(hi);
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

// Unite the sets of a and b; returns the root of the merged set as seen by
// this thread (a valid hint for later unions of either element).
__device__ __forceinline__ int32_t uf_union(int32_t *parent, int32_t a, int32_t b) {
  a = uf_find(parent, a);
  b = uf_find(parent, b);
  while (a != b) {
    if (a > b) {
      int32_t t = a;
      a = b;
      b = t;
    }
    int32_t old = atomicCAS(&parent[b], b, a);
    if (old == b) return a;
    b = uf_find(parent, old);
    a = uf_find(parent, a);
  }
  return a;
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
