// Query kernels over a device hierarchy: range counts (K5), CRS collection,
// pair enumeration and k-nearest neighbours (K10).
// Reference: traversal.hpp:23-266.
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>

#include "sp_common.cuh"
#include "sp_internal.hpp"
#include "sp_query.hpp"
#include "sp_traverse.cuh"

namespace spb {

// ---------------------------------------------------------------------------
// predicates
// ---------------------------------------------------------------------------
struct SpherePred {
  float x, y, z;
  double thr;
};

// Representatives for sort_queries (traversal.hpp:188-218): sphere centres, or
// box centroids (double midpoint rounded to float, geometry.hpp:130-137).
__global__ void k_representatives(const float *__restrict__ preds, int64_t nq, int dim, int kind,
                                  float *__restrict__ out) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < nq; q += stride) {
    for (int k = 0; k < dim; ++k) {
      float v;
      if (kind == 0) v = preds[q * (dim + 1) + k];
      else v = __double2float_rn(__dmul_rn(__dadd_rn((double)preds[q * 2 * dim + k], (double)preds[q * 2 * dim + dim + k]), 0.5));
      out[q * dim + k] = v;
    }
  }
}

void query_order(Ctx &c, const float *preds, int64_t nq, int dim, int kind, int32_t *order) {
  if (nq <= 0) return;
  DevBuf<float> reps((size_t)nq * dim, c.stream);
  k_representatives<<<grid_for(nq, 256, 148 * 16), 256, 0, c.stream>>>(preds, nq, dim, kind, reps.get());
  SPB_LAUNCHED();
  sort_points(c, reps.get(), nq, dim, order);
}

// mode 0: spheres of one radius over centres float[nq*dim]
// mode 1: spheres with per-query radius float[nq*(dim+1)]
// mode 2: boxes float[nq*2*dim]
// MODE 0: one radius; 1: per-query radius; 2: box queries; 3: one radius
// that admits the fp32 filter (compiled without the double box test).
template <int MODE>
__device__ __forceinline__ void range_count_one(const float4 *__restrict__ nodes, const float4 *__restrict__ leafpt,
                                                int64_t n, const float *__restrict__ preds, int dim,
                                                const int32_t *__restrict__ order, int64_t qi, Radius R0,
                                                int32_t cap, int32_t *__restrict__ counts) {
  const int64_t q = order ? order[qi] : qi;
  int32_t c;
  if (MODE != 2) {
    const int stride = MODE == 1 ? dim + 1 : dim;
    const float *p = preds + q * stride;
    float cx = p[0], cy = p[1], cz = dim == 3 ? p[2] : 0.f;
    Radius R = MODE == 1 ? make_radius(p[dim]) : R0;
    if (MODE == 3) R.fast = 1;
    c = count_sphere(nodes, leafpt, n, cx, cy, cz, R, cap);
  } else {
    float b[6] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
    for (int k = 0; k < dim; ++k) {
      b[k] = preds[q * 2 * dim + k];
      b[3 + k] = preds[q * 2 * dim + dim + k];
    }
    c = 0;
    int32_t cur = 0;
    while (cur != kSentinel) {
      float4 lo, hi;
      ld_node2(nodes, (int64_t)cur, lo, hi);
      const bool hit = box_touch(lo, hi, b);
      if (cur >= n - 1) {
        cur = (hit && ++c == cap) ? kSentinel : node_rope(hi);
      } else {
        cur = hit ? node_link(lo) : node_rope(hi);
      }
    }
  }
  counts[q] = c;
}

// Range counts, one query per thread on the SM-affine schedule (sp_common.cuh):
// C2 query 15.7 -> 12.8 ms at 2^24 (128-thread blocks in plain order: 15.7,
// 512-thread blocks alone: 14.0).
template <int MODE>
__global__ void __launch_bounds__(512, 1) k_range_count_sm(const float4 *__restrict__ nodes,
                                                           const float4 *__restrict__ leafpt, int64_t n,
                                                           const float *__restrict__ preds, int dim,
                                                           const int32_t *__restrict__ order, int64_t nq, Radius R0,
                                                           int32_t cap, int32_t *__restrict__ counts,
                                                           unsigned long long *slices, int nslices) {
  SmSliceWalk w(nq, slices, nslices);
  for (int64_t qi; w.next(qi);)
    if (qi >= 0) range_count_one<MODE>(nodes, leafpt, n, preds, dim, order, qi, R0, cap, counts);
}

void range_count(Ctx &c, const Tree &t, int kind, const float *preds, int64_t nq, float radius, int32_t cap,
                 int32_t *counts, const int32_t *order_in) {
  if (nq <= 0) return;
  if (t.n == 0) {
    SPB_CUDA(cudaMemsetAsync(counts, 0, (size_t)nq * sizeof(int32_t), c.stream));
    return;
  }
  DevBuf<int32_t> order;
  const int32_t *ord = order_in;
  if (!ord) {
    order = DevBuf<int32_t>((size_t)nq, c.stream);
    if (kind == RQ_RADIUS) {
      sort_points(c, preds, nq, t.dim, order.get());
    } else {
      query_order(c, preds, nq, t.dim, kind == RQ_SPHERES ? 0 : 1, order.get());
    }
    ord = order.get();
  }
  const Radius R = make_radius(radius);
  const int mode = kind == RQ_RADIUS ? (R.fast ? 3 : 0) : (kind == RQ_SPHERES ? 1 : 2);
  SmSlices sl(c);
  auto launch = [&](auto kern) {
    kern<<<sl.grid(kern, 512), 512, 0, c.stream>>>(t.nodes, t.leafpt, t.n, preds, t.dim, ord, nq, R, cap, counts,
                                                   sl.ctr.get(), sl.nsm);
  };
  switch (mode) {
    case 3: launch(k_range_count_sm<3>); break;
    case 0: launch(k_range_count_sm<0>); break;
    case 1: launch(k_range_count_sm<1>); break;
    default: launch(k_range_count_sm<2>); break;
  }
  SPB_LAUNCHED();
}

// ---------------------------------------------------------------------------
// exclusive scan int32 -> int64 (offsets[n+1]); three kernels
// ---------------------------------------------------------------------------
constexpr int SCAN_BLOCK = 1024;

__device__ __forceinline__ int64_t block_incl_scan(int64_t v, int64_t *wsum) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int d = 1; d < 32; d <<= 1) {
    int64_t y = __shfl_up_sync(0xffffffffu, v, d);
    if (lane >= d) v += y;
  }
  if (lane == 31) wsum[warp] = v;
  __syncthreads();
  if (warp == 0) {
    int64_t s = lane < (int)(blockDim.x >> 5) ? wsum[lane] : 0;
    for (int d = 1; d < 32; d <<= 1) {
      int64_t y = __shfl_up_sync(0xffffffffu, s, d);
      if (lane >= d) s += y;
    }
    wsum[lane] = s;
  }
  __syncthreads();
  if (warp > 0) v += wsum[warp - 1];
  return v;
}

__global__ void k_scan_blocks(const int32_t *__restrict__ in, int64_t n, int64_t *__restrict__ out,
                              int64_t *__restrict__ bsum) {
  __shared__ int64_t wsum[32];
  const int64_t i = (int64_t)blockIdx.x * SCAN_BLOCK + threadIdx.x;
  int64_t v = i < n ? in[i] : 0;
  int64_t incl = block_incl_scan(v, wsum);
  if (i < n) out[i + 1] = incl;
  if (threadIdx.x == SCAN_BLOCK - 1) bsum[blockIdx.x] = incl;
}

__global__ void k_scan_sums(int64_t *bsum, int64_t nb) {
  __shared__ int64_t wsum[32];
  __shared__ int64_t carry;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  for (int64_t base = 0; base < nb; base += SCAN_BLOCK) {
    int64_t i = base + threadIdx.x;
    int64_t v = i < nb ? bsum[i] : 0;
    int64_t incl = block_incl_scan(v, wsum);
    int64_t c0 = carry;
    if (i < nb) bsum[i] = c0 + incl - v;  // exclusive
    __syncthreads();
    if (threadIdx.x == SCAN_BLOCK - 1) carry = c0 + incl;
    __syncthreads();
  }
}

__global__ void k_scan_add(int64_t *out, int64_t n, const int64_t *__restrict__ bsum) {
  const int64_t i = (int64_t)blockIdx.x * SCAN_BLOCK + threadIdx.x;
  if (i < n) out[i + 1] += bsum[blockIdx.x];
  if (i == 0) out[0] = 0;
}

void exclusive_scan(Ctx &c, const int32_t *in, int64_t n, int64_t *out) {
  if (n <= 0) {
    SPB_CUDA(cudaMemsetAsync(out, 0, sizeof(int64_t), c.stream));
    return;
  }
  const int64_t nb = (n + SCAN_BLOCK - 1) / SCAN_BLOCK;
  DevBuf<int64_t> bsum((size_t)nb, c.stream);
  k_scan_blocks<<<(unsigned)nb, SCAN_BLOCK, 0, c.stream>>>(in, n, out, bsum.get());
  SPB_LAUNCHED();
  k_scan_sums<<<1, SCAN_BLOCK, 0, c.stream>>>(bsum.get(), nb);
  SPB_LAUNCHED();
  k_scan_add<<<(unsigned)nb, SCAN_BLOCK, 0, c.stream>>>(out, n, bsum.get());
  SPB_LAUNCHED();
}

// ---------------------------------------------------------------------------
// CRS fill (query_crs second pass, traversal.hpp:254-260) and row sort
// ---------------------------------------------------------------------------
template <int MODE>
__global__ void __launch_bounds__(128) k_range_fill(const float4 *__restrict__ nodes, int64_t n,
                                                    const float *__restrict__ preds, int dim,
                                                    const int32_t *__restrict__ order, int64_t nq,
                                                    const int64_t *__restrict__ offsets,
                                                    uint64_t *__restrict__ keyed, unsigned long long *slices,
                                                    int nslices) {
  SmSliceWalk sw(nq, slices, nslices);  // SM-affine schedule (sp_common.cuh)
  for (int64_t qi; sw.next(qi);) {
    if (qi < 0) continue;
    const int64_t q = order[qi];
    int64_t w = offsets[q];
    float b[6] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
    float cx = 0.f, cy = 0.f, cz = 0.f;
    Radius R{0.0, 0.f, 0.f, 0};
    if (MODE == 1) {
      const float *p = preds + q * (dim + 1);
      cx = p[0]; cy = p[1]; cz = dim == 3 ? p[2] : 0.f;
      R = make_radius(p[dim]);
    } else {
      for (int k = 0; k < dim; ++k) {
        b[k] = preds[q * 2 * dim + k];
        b[3 + k] = preds[q * 2 * dim + dim + k];
      }
    }
    int32_t cur = 0;
    while (cur != kSentinel) {
      float4 lo, hi;
      ld_node2(nodes, (int64_t)cur, lo, hi);
      const bool leaf = cur >= n - 1;
      const bool hit = MODE == 1 ? (leaf ? hit_box(R, cx, cy, cz, lo, hi) : maybe_box(R, cx, cy, cz, lo, hi))
                                 : box_touch(lo, hi, b);
      if (leaf) {
        // key = (query << 32) | object; sorting the keys orders each row by object
        if (hit) keyed[w++] = ((uint64_t)q << 32) | (uint32_t)node_link(lo);
        cur = node_rope(hi);
      } else {
        cur = hit ? node_link(lo) : node_rope(hi);
      }
    }
  }
}

__global__ void k_low_words(const uint64_t *__restrict__ keys, int64_t m, int32_t *__restrict__ out) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m; i += stride) out[i] = (int32_t)(uint32_t)keys[i];
}

int64_t range_crs(Ctx &c, const Tree &t, int kind, const float *preds, int64_t nq, int64_t *offsets, int32_t *values,
                  int64_t capacity) {
  if (nq <= 0) {
    SPB_CUDA(cudaMemsetAsync(offsets, 0, sizeof(int64_t), c.stream));
    return 0;
  }
  DevBuf<int32_t> order((size_t)nq, c.stream), counts((size_t)nq, c.stream);
  query_order(c, preds, nq, t.dim, kind == RQ_SPHERES ? 0 : 1, order.get());
  range_count(c, t, kind, preds, nq, 0.f, 0, counts.get(), order.get());
  exclusive_scan(c, counts.get(), nq, offsets);
  int64_t total = 0;
  peek(c, {{offsets + nq, &total, sizeof(int64_t)}});
  if (total > capacity) return total;
  if (total == 0 || t.n == 0) return total;
  DevBuf<uint64_t> k0((size_t)total, c.stream), k1((size_t)total, c.stream);
  DevBuf<uint32_t> v0((size_t)total, c.stream), v1((size_t)total, c.stream);
  SmSlices sl(c);
  if (kind == RQ_SPHERES)
    k_range_fill<1><<<sl.grid(k_range_fill<1>, 128), 128, 0, c.stream>>>(t.nodes, t.n, preds, t.dim, order.get(), nq,
                                                                         offsets, k0.get(), sl.ctr.get(), sl.nsm);
  else
    k_range_fill<2><<<sl.grid(k_range_fill<2>, 128), 128, 0, c.stream>>>(t.nodes, t.n, preds, t.dim, order.get(), nq,
                                                                         offsets, k0.get(), sl.ctr.get(), sl.nsm);
  SPB_LAUNCHED();
  int qbits = 1;
  while (qbits < 31 && (1LL << qbits) < nq) ++qbits;
  uint64_t *ka = k0.get(), *kb = k1.get();
  uint32_t *va = v0.get(), *vb = v1.get();
  radix_sort_pairs(c, &ka, &va, &kb, &vb, total, 32 + qbits, true);
  k_low_words<<<grid_for(total, 256, 148 * 16), 256, 0, c.stream>>>(ka, total, values);
  SPB_LAUNCHED();
  return total;
}

// ---------------------------------------------------------------------------
// pair_traversal (traversal.hpp:162-184): leaf p walks from its own rope, so
// only later leaves are examined and each close pair appears exactly once.
// ---------------------------------------------------------------------------
template <bool FILL>
__global__ void __launch_bounds__(128) k_pairs(const float4 *__restrict__ nodes, int64_t n, Radius R,
                                               int32_t *__restrict__ counts, const int64_t *__restrict__ offsets,
                                               int32_t *__restrict__ pairs) {
  const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= n) return;
  const int64_t self = n - 1 + p;
  const float4 me = ld_node(nodes, 2 * self);
  int32_t cur = node_rope(ld_node(nodes, 2 * self + 1));
  int64_t w = FILL ? offsets[p] : 0;
  int32_t c = 0;
  while (cur != kSentinel) {
    float4 lo, hi;
    ld_node2(nodes, (int64_t)cur, lo, hi);
    const bool leaf = cur >= n - 1;
    const bool hit = leaf ? hit_box(R, me.x, me.y, me.z, lo, hi) : maybe_box(R, me.x, me.y, me.z, lo, hi);
    if (leaf) {
      if (hit) {
        if (FILL) {
          pairs[2 * w] = node_link(me);
          pairs[2 * w + 1] = node_link(lo);
          ++w;
        } else {
          ++c;
        }
      }
      cur = node_rope(hi);
    } else {
      cur = hit ? node_link(lo) : node_rope(hi);
    }
  }
  if (!FILL) counts[p] = c;
}

int64_t pair_list(Ctx &c, const Tree &t, float eps, int32_t *pairs, int64_t capacity) {
  if (t.n < 2) return 0;
  const Radius thr = make_radius(eps);
  DevBuf<int32_t> counts((size_t)t.n, c.stream);
  DevBuf<int64_t> offsets((size_t)t.n + 1, c.stream);
  unsigned g = (unsigned)((t.n + 127) / 128);
  k_pairs<false><<<g, 128, 0, c.stream>>>(t.nodes, t.n, thr, counts.get(), nullptr, nullptr);
  SPB_LAUNCHED();
  exclusive_scan(c, counts.get(), t.n, offsets.get());
  int64_t total = 0;
  peek(c, {{offsets.get() + t.n, &total, sizeof(int64_t)}});
  if (total > capacity || total == 0) return total;
  k_pairs<true><<<g, 128, 0, c.stream>>>(t.nodes, t.n, thr, nullptr, offsets.get(), pairs);
  SPB_LAUNCHED();
  return total;
}

// ---------------------------------------------------------------------------
// k nearest neighbours (nearest_query, traversal.hpp:93-156).
// Results are the min(k, n) smallest (float distance, object) pairs, which any
// exact pruning order reproduces; this kernel keeps the reference's explicit
// stack (near child popped first) and its strict `dist > worst` pruning, with
// the candidate max-heap in local memory.
// ---------------------------------------------------------------------------
constexpr int KNN_STACK = 100;
#ifndef SPB_KNN_STACK2
#define SPB_KNN_STACK2 1
#endif  // tree depth <= 96 prefix bits + 1

__device__ __forceinline__ float box_dist(float x, float y, float z, const float4 &lo, const float4 &hi) {
  return __double2float_rn(__dsqrt_rn(gap2(x, y, z, lo, hi)));
}

// (distance, index) order; bitwise, so the compiler emits one predicate chain
// instead of a short-circuit branch per comparison
__device__ __forceinline__ bool cand_less(float da, int32_t ia, float db, int32_t ib) {
  return (da < db) | ((da == db) & (ia < ib));
}

template <int KMAX>
__global__ void __launch_bounds__(128) k_knn(const float4 *__restrict__ nodes, int64_t n,
                                             const float *__restrict__ origins, int dim,
                                             const int32_t *__restrict__ order, int64_t nq, int32_t k,
                                             float *__restrict__ gdist, int32_t *__restrict__ gidx,
                                             int32_t *__restrict__ out_idx, float *__restrict__ out_dist) {
  const int64_t qi = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (qi >= nq) return;
  const int64_t q = order[qi];
  const float x = origins[q * dim], y = origins[q * dim + 1], z = dim == 3 ? origins[q * dim + 2] : 0.f;
  const int32_t kk = (int32_t)((int64_t)k < n ? (int64_t)k : n);
  // heap storage: registers/local for KMAX > 0, else global scratch rows
  float hd_local[KMAX > 0 ? KMAX : 1];
  int32_t hi_local[KMAX > 0 ? KMAX : 1];
  float *hd = KMAX > 0 ? hd_local : gdist + qi * (int64_t)kk;
  int32_t *hx = KMAX > 0 ? hi_local : gidx + qi * (int64_t)kk;
  int32_t size = 0;
  // KMAX == 16: an ascending list in registers (worst = last real slot),
  // sentinels (-inf) before the kk real slots; else a max-heap
  constexpr bool REG = KMAX == 16;
  if (REG) {
#pragma unroll
    for (int j = 0; j < (REG ? KMAX : 1); ++j) {
      const bool real = j >= KMAX - kk;
      hd_local[j] = __int_as_float(real ? 0x7f800000 : (int)0xff800000);
      hi_local[j] = real ? 0x7fffffff : (int32_t)0x80000000;
    }
  }
  auto worst = [&]() -> float { return REG ? hd_local[KMAX > 0 ? KMAX - 1 : 0] : hd[0]; };

  // The node being visited lives in registers (d, ref); the nearer child of
  // an expanded node is visited next without a stack round trip, only the
  // farther one is pushed (same visiting order as push-both-pop-near).  An
  // entry carries what its node's box load already gave: ref = the left child
  // of an internal node, or ~object for a leaf, so a pop never re-reads the
  // node itself (42.6 -> 41.3 ms at C4).
#if SPB_KNN_STACK2
  // one 8-byte entry {distance bits, ref} per level: a push or pop is one
  // local access instead of two
  uint2 stk[KNN_STACK];
#else
  float sd[KNN_STACK];
  int32_t sr[KNN_STACK];
#endif
  int top = 0;
  float d;
  int32_t ref = 0;
  {
    const float4 lo = ld_node(nodes, 0), hi = ld_node(nodes, 1);
    d = box_dist(x, y, z, lo, hi);
    ref = n == 1 ? ~node_link(lo) : node_link(lo);
  }
  bool have = true;
  for (;;) {
    if (!have) {
      if (top == 0) break;
      --top;
#if SPB_KNN_STACK2
      const uint2 e = stk[top];
      d = __uint_as_float(e.x);
      ref = (int32_t)e.y;
#else
      d = sd[top];
      ref = sr[top];
#endif
    }
    have = false;
    if (size == kk && d > worst()) continue;
    if (ref < 0) {
      const int32_t obj = ~ref;
      if (REG) {
        constexpr int K = KMAX > 0 ? KMAX : 1;
        if (cand_less(d, obj, hd_local[K - 1], hi_local[K - 1])) {
          // one comparison per slot, then a select network that shifts the
          // tail right by one (no branches: 56.4 -> 44.3 ms at C4)
          bool lt[K];
#pragma unroll
          for (int j = 0; j < K; ++j) lt[j] = cand_less(d, obj, hd_local[j], hi_local[j]);
#pragma unroll
          for (int j = K - 1; j > 0; --j) {
            hd_local[j] = lt[j - 1] ? hd_local[j - 1] : (lt[j] ? d : hd_local[j]);
            hi_local[j] = lt[j - 1] ? hi_local[j - 1] : (lt[j] ? obj : hi_local[j]);
          }
          hd_local[0] = lt[0] ? d : hd_local[0];
          hi_local[0] = lt[0] ? obj : hi_local[0];
          if (size < kk) ++size;
        }
      } else if (size < kk) {  // push + sift up
        int32_t i = size++;
        while (i > 0) {
          int32_t pa = (i - 1) >> 1;
          if (!cand_less(hd[pa], hx[pa], d, obj)) break;
          hd[i] = hd[pa];
          hx[i] = hx[pa];
          i = pa;
        }
        hd[i] = d;
        hx[i] = obj;
      } else if (cand_less(d, obj, hd[0], hx[0])) {  // replace top + sift down
        int32_t i = 0;
        while (true) {
          int32_t l = 2 * i + 1, r = l + 1, m = i;
          float md = d;
          int32_t mi = obj;
          if (l < size && cand_less(md, mi, hd[l], hx[l])) { m = l; md = hd[l]; mi = hx[l]; }
          if (r < size && cand_less(md, mi, hd[r], hx[r])) { m = r; md = hd[r]; mi = hx[r]; }
          if (m == i) break;
          hd[i] = hd[m];
          hx[i] = hx[m];
          i = m;
        }
        hd[i] = d;
        hx[i] = obj;
      }
      continue;
    }
    const int32_t left = ref;
    float4 llo, lhi;
    ld_node2(nodes, (int64_t)left, llo, lhi);
    const int32_t right = node_rope(lhi);
    float4 rlo, rhi;
    ld_node2(nodes, (int64_t)right, rlo, rhi);
    float dn = box_dist(x, y, z, llo, lhi), df = box_dist(x, y, z, rlo, rhi);
    int32_t rn = left >= n - 1 ? ~node_link(llo) : node_link(llo);
    int32_t rf = right >= n - 1 ? ~node_link(rlo) : node_link(rlo);
    if (df < dn) {
      float td = dn; dn = df; df = td;
      int32_t tr = rn; rn = rf; rf = tr;
    }
    const bool full = size == kk;
    const float w = worst();
    const bool keep_f = !(full && df > w), keep_n = !(full && dn > w);
    if (keep_n) {
#if SPB_KNN_STACK2
      if (keep_f && top < KNN_STACK) { stk[top] = make_uint2(__float_as_uint(df), (uint32_t)rf); ++top; }
#else
      if (keep_f && top < KNN_STACK) { sd[top] = df; sr[top] = rf; ++top; }
#endif
      d = dn;
      ref = rn;
      have = true;
    } else if (keep_f) {  // not reached (dn <= df), kept as the general rule
      d = df;
      ref = rf;
      have = true;
    }
  }
  if (REG) {
    constexpr int K = KMAX > 0 ? KMAX : 1;
#pragma unroll
    for (int j = 0; j < K; ++j) {
      const int32_t r = j - (K - kk);
      if (r >= 0 && r < size) {
        const int64_t o = q * (int64_t)k + r;
        out_idx[o] = hi_local[j];
        if (out_dist) out_dist[o] = hd_local[j];
      }
    }
    for (int32_t j = size; j < k; ++j) {
      const int64_t o = q * (int64_t)k + j;
      out_idx[o] = -1;
      if (out_dist) out_dist[o] = __int_as_float(0x7f800000);
    }
    return;
  }
  // heap -> ascending order: repeatedly move the max to the end
  for (int32_t end = size - 1; end > 0; --end) {
    float td = hd[0]; int32_t tx = hx[0];
    float ld = hd[end]; int32_t lx = hx[end];
    int32_t i = 0;
    while (true) {
      int32_t l = 2 * i + 1, r = l + 1, m = i;
      float md = ld; int32_t mi = lx;
      if (l < end && cand_less(md, mi, hd[l], hx[l])) { m = l; md = hd[l]; mi = hx[l]; }
      if (r < end && cand_less(md, mi, hd[r], hx[r])) { m = r; md = hd[r]; mi = hx[r]; }
      if (m == i) break;
      hd[i] = hd[m]; hx[i] = hx[m];
      i = m;
    }
    hd[i] = ld; hx[i] = lx;
    hd[end] = td; hx[end] = tx;
  }
  for (int32_t j = 0; j < k; ++j) {
    const int64_t o = q * (int64_t)k + j;
    out_idx[o] = j < size ? hx[j] : -1;
    if (out_dist) out_dist[o] = j < size ? hd[j] : __int_as_float(0x7f800000);
  }
}

// k <= 16 with lower-bound keys.  The result set depends only on the exact
// leaf distances (float(sqrt(S)) with S the double-accumulated square, as
// box_dist computes them); the visiting order is free and a node may be
// pruned whenever its distance is certainly above the current k-th.  Every
// node -- internal or leaf -- is keyed by a fp32 LOWER bound: gaps, squares,
// sum and square root all rounded toward zero (__f*_rd), so key <= the real
// distance <= the exact float distance (a float within 2^-52 of the real value
// rounds to itself), and `key > worst` prunes only what the exact test would.
// The double-precision distance is computed once per leaf that survives the
// bound, at its visit, from its node (in L1: the parent's expansion loaded
// it); expansions are all fp32 and branch-free.  Leaves travel on the stack
// as ~(leaf node index).
#ifndef SPB_KNN_SQ
#define SPB_KNN_SQ 1
#endif
__device__ __forceinline__ float gap_rd(float c, float lo, float hi) {
  return fmaxf(fmaxf(__fsub_rd(lo, c), __fsub_rd(c, hi)), 0.f);
}
__device__ __forceinline__ float box_dist_lb(float x, float y, float z, const float4 &lo, const float4 &hi) {
  const float gx = gap_rd(x, lo.x, hi.x), gy = gap_rd(y, lo.y, hi.y), gz = gap_rd(z, lo.z, hi.z);
  const float s = __fadd_rd(__fadd_rd(__fmul_rd(gx, gx), __fmul_rd(gy, gy)), __fmul_rd(gz, gz));
#if SPB_KNN_SQ
  return s;  // keys are squared lower bounds, pruned against knn_sq_bound(worst)
#else
  return __fsqrt_rd(s);
#endif
}
// SPB_KNN_SQ: a node keyed by its squared lower bound s may be pruned when s >
// T = ru((w + ulp(w))^2): then the real distance exceeds w + ulp(w), which
// rounds (to nearest, through the double square root) to a float above w, so
// the exact test `distance > w` holds -- ties at w are never pruned.
__device__ __forceinline__ float knn_sq_bound(float w) {
  const float w1 = __fadd_ru(w, __fsub_ru(nextafterf(w, __int_as_float(0x7f800000)), w));
  return __fmul_ru(w1, w1);
}

#ifndef SPB_KNN_BLOCK
#define SPB_KNN_BLOCK 128
#endif
__global__ void __launch_bounds__(SPB_KNN_BLOCK) k_knn16lb(const float4 *__restrict__ nodes, int64_t n,
                                                 const float *__restrict__ origins, int dim,
                                                 const int32_t *__restrict__ order, int64_t nq, int32_t k,
                                                 int32_t *__restrict__ out_idx, float *__restrict__ out_dist) {
  constexpr int K = 16;
  const int64_t qi = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (qi >= nq) return;
  const int64_t q = order[qi];
  const float x = origins[q * dim], y = origins[q * dim + 1], z = dim == 3 ? origins[q * dim + 2] : 0.f;
  const int32_t kk = (int32_t)((int64_t)k < n ? (int64_t)k : n);
  float hd[K];
  int32_t hx[K];
#pragma unroll
  for (int j = 0; j < K; ++j) {
    const bool real = j >= K - kk;
    hd[j] = __int_as_float(real ? 0x7f800000 : (int)0xff800000);
    hx[j] = real ? 0x7fffffff : (int32_t)0x80000000;
  }
  int32_t size = 0;
  float wkey = __int_as_float(0x7f800000);  // prune keys above this (the k-th distance, or its squared bound)
  uint2 stk[KNN_STACK];
  int top = 0;
  const int32_t first_leaf = (int32_t)(n - 1);
  float d = 0.f;  // the root: always opened (or the single leaf)
  int32_t ref = n == 1 ? ~0 : node_link(ld_node(nodes, 0));  // the root's left child
  bool have = true;
  for (;;) {
    if (!have) {
      if (top == 0) break;
      --top;
      const uint2 e = stk[top];
      d = __uint_as_float(e.x);
      ref = (int32_t)e.y;
    }
    have = false;
    if (d > wkey) continue;  // wkey stays +inf until the list is full
    if (ref < 0) {  // a leaf: its exact distance decides
      const int32_t leaf = ~ref;
      const float4 lo = ld_node(nodes, 2 * ((int64_t)first_leaf + leaf));
      const float dx = __double2float_rn(__dsqrt_rn(dist2(x, y, z, lo.x, lo.y, lo.z)));
      const int32_t obj = node_link(lo);
      if (cand_less(dx, obj, hd[K - 1], hx[K - 1])) {
        bool lt[K];
#pragma unroll
        for (int j = 0; j < K; ++j) lt[j] = cand_less(dx, obj, hd[j], hx[j]);
#pragma unroll
        for (int j = K - 1; j > 0; --j) {
          hd[j] = lt[j - 1] ? hd[j - 1] : (lt[j] ? dx : hd[j]);
          hx[j] = lt[j - 1] ? hx[j - 1] : (lt[j] ? obj : hx[j]);
        }
        hd[0] = lt[0] ? dx : hd[0];
        hx[0] = lt[0] ? obj : hx[0];
        if (size < kk) ++size;
#if SPB_KNN_SQ
        if (size == kk) wkey = knn_sq_bound(hd[K - 1]);
#else
        if (size == kk) wkey = hd[K - 1];
#endif
      }
      continue;
    }
    // an internal node: ref is its left child
    const int32_t left = ref;
    float4 llo, lhi;
    ld_node2(nodes, (int64_t)left, llo, lhi);
    const int32_t right = node_rope(lhi);
    float4 rlo, rhi;
    ld_node2(nodes, (int64_t)right, rlo, rhi);
    float dn = box_dist_lb(x, y, z, llo, lhi), df = box_dist_lb(x, y, z, rlo, rhi);
    int32_t rn = left >= first_leaf ? ~(left - first_leaf) : node_link(llo);
    int32_t rf = right >= first_leaf ? ~(right - first_leaf) : node_link(rlo);
    if (df < dn) {
      const float td = dn; dn = df; df = td;
      const int32_t tr = rn; rn = rf; rf = tr;
    }
    const bool keep_f = !(df > wkey), keep_n = !(dn > wkey);
    if (keep_n) {
      // at most one entry per tree level: split lengths grow strictly down the
      // tree and stay below 64 + 32 (code bits + index tie-break), so the
      // stack never holds more than 95 < KNN_STACK entries
      if (keep_f) { stk[top] = make_uint2(__float_as_uint(df), (uint32_t)rf); ++top; }
      d = dn;
      ref = rn;
      have = true;
    } else if (keep_f) {
      d = df;
      ref = rf;
      have = true;
    }
  }
#pragma unroll
  for (int j = 0; j < K; ++j) {
    const int32_t r = j - (K - kk);
    if (r >= 0 && r < size) {
      const int64_t o = q * (int64_t)k + r;
      out_idx[o] = hx[j];
      if (out_dist) out_dist[o] = hd[j];
    }
  }
  for (int32_t j = size; j < k; ++j) {
    const int64_t o = q * (int64_t)k + j;
    out_idx[o] = -1;
    if (out_dist) out_dist[o] = __int_as_float(0x7f800000);
  }
}

#ifndef SPB_KNN_LB
#define SPB_KNN_LB 1
#endif

void knn(Ctx &c, const Tree &t, const float *origins, int64_t nq, int32_t k, int32_t *idx, float *dist) {
  if (nq <= 0 || k <= 0) return;
  if (t.n == 0) {
    SPB_CUDA(cudaMemsetAsync(idx, 0xff, (size_t)nq * k * sizeof(int32_t), c.stream));
    return;
  }
  DevBuf<int32_t> order((size_t)nq, c.stream);
  sort_points(c, origins, nq, t.dim, order.get());
  unsigned g = (unsigned)((nq + 127) / 128);
  const int64_t kk = std::min<int64_t>(k, t.n);
  if (kk <= 16 && SPB_KNN_LB) {
    k_knn16lb<<<(unsigned)((nq + SPB_KNN_BLOCK - 1) / SPB_KNN_BLOCK), SPB_KNN_BLOCK, 0, c.stream>>>(
        t.nodes, t.n, origins, t.dim, order.get(), nq, k, idx, dist);
  } else if (kk <= 16) {
    k_knn<16><<<g, 128, 0, c.stream>>>(t.nodes, t.n, origins, t.dim, order.get(), nq, k, nullptr, nullptr, idx, dist);
  } else if (kk <= 64) {
    k_knn<64><<<g, 128, 0, c.stream>>>(t.nodes, t.n, origins, t.dim, order.get(), nq, k, nullptr, nullptr, idx, dist);
  } else {
    if ((double)nq * (double)kk * 8.0 > 8e9) throw CapacityError();
    DevBuf<float> gd((size_t)(nq * kk), c.stream);
    DevBuf<int32_t> gi((size_t)(nq * kk), c.stream);
    k_knn<0><<<g, 128, 0, c.stream>>>(t.nodes, t.n, origins, t.dim, order.get(), nq, k, gd.get(), gi.get(), idx, dist);
  }
  SPB_LAUNCHED();
}

}  // namespace spb

namespace spb {

// Diagnostics: node visits of each leaf's pair walk (traversal.hpp:162-184).
__global__ void k_walk_lengths(const float4 *__restrict__ nodes, const float4 *__restrict__ leafpt, int64_t n,
                               Radius R, int32_t *__restrict__ steps, int32_t *__restrict__ hits) {
  const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= n) return;
  const float4 me = ld_node(leafpt, p);
  int32_t cur = __float_as_int(me.w), s = 0, h = 0;
  while (cur != kSentinel) {
    ++s;
    if (cur >= n - 1) {
      const float4 L = ld_node(leafpt, cur - (n - 1));
      h += hit_point(R, me.x, me.y, me.z, L.x, L.y, L.z);
      cur = __float_as_int(L.w);
    } else {
      float4 lo, hi;
      ld_node2(nodes, (int64_t)cur, lo, hi);
      cur = maybe_box(R, me.x, me.y, me.z, lo, hi) ? node_link(lo) : node_rope(hi);
    }
  }
  steps[p] = s;
  hits[p] = h;
}

void walk_lengths(Ctx &c, const Tree &t, float eps, int32_t *steps, int32_t *hits) {
  if (t.n == 0 || !t.leafpt) return;
  k_walk_lengths<<<(unsigned)((t.n + 127) / 128), 128, 0, c.stream>>>(t.nodes, t.leafpt, t.n, make_radius(eps), steps,
                                                                      hits);
  SPB_LAUNCHED();
}

}  // namespace spb

namespace spb {

// ---------------------------------------------------------------------------
// check_equivalence (verify.hpp:21-61) on the device.  violation codes:
// 1 core flag, 2 noise, 3 core partition (one reference cluster split),
// 4 core clusters merged, 5 border point without an in-cluster core point
// within eps.  The border test walks the point tree (early exit on the first
// qualifying core point) instead of the reference's O(n^2) scan.
// ---------------------------------------------------------------------------
__global__ void k_eq_flags(int64_t n, const int32_t *__restrict__ gl, const uint8_t *__restrict__ gc,
                           const int32_t *__restrict__ wl, const uint8_t *__restrict__ wc,
                           unsigned long long *__restrict__ first) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    if ((gc[i] != 0) != (wc[i] != 0)) atomicMin(&first[0], (unsigned long long)i);
    if ((gl[i] == -1) != (wl[i] == -1)) atomicMin(&first[1], (unsigned long long)i);
  }
}

// (want, got) label pairs of core points, packed for sorting
__global__ void k_eq_pairs(int64_t n, const int32_t *__restrict__ gl, const int32_t *__restrict__ wl,
                           const uint8_t *__restrict__ wc, uint64_t *__restrict__ fwd, uint64_t *__restrict__ rev,
                           uint32_t *__restrict__ idx) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    const bool c = wc[i] != 0;
    fwd[i] = c ? ((uint64_t)(uint32_t)wl[i] << 32) | (uint32_t)gl[i] : ~0ull;
    rev[i] = c ? ((uint64_t)(uint32_t)gl[i] << 32) | (uint32_t)wl[i] : ~0ull;
    idx[i] = (uint32_t)i;
  }
}

// sorted pairs: equal high words with different low words violate the map
__global__ void k_eq_bijective(int64_t n, const uint64_t *__restrict__ s, const uint32_t *__restrict__ idx,
                               unsigned long long *__restrict__ out) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i + 1 < n; i += stride) {
    const uint64_t a = s[i], b = s[i + 1];
    if (b == ~0ull) continue;
    if ((a >> 32) == (b >> 32) && (uint32_t)a != (uint32_t)b) {
      const uint32_t x = idx[i], y = idx[i + 1];
      atomicMin(out, (unsigned long long)(x > y ? x : y));
    }
  }
}

__global__ void __launch_bounds__(128) k_eq_border(const float4 *__restrict__ nodes, const float4 *__restrict__ leafpt,
                                                   const int32_t *__restrict__ perm, int64_t n, Radius R,
                                                   const int32_t *__restrict__ gl, const uint8_t *__restrict__ gc,
                                                   unsigned long long *__restrict__ out) {
  const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= n) return;
  const int32_t b = perm[p];
  if (gc[b] || gl[b] == -1) return;
  const float4 me = ld_node(leafpt, p);
  const int32_t lab = gl[b];
  int32_t cur = 0;
  bool ok = false;
  while (cur != kSentinel && !ok) {
    if (cur >= n - 1) {
      const float4 L = ld_node(leafpt, cur - (n - 1));
      if (hit_point(R, me.x, me.y, me.z, L.x, L.y, L.z)) {
        const int32_t c = perm[cur - (n - 1)];
        ok = gc[c] && gl[c] == lab;
      }
      cur = __float_as_int(L.w);
    } else {
      float4 lo, hi;
      ld_node2(nodes, (int64_t)cur, lo, hi);
      cur = maybe_box(R, me.x, me.y, me.z, lo, hi) ? node_link(lo) : node_rope(hi);
    }
  }
  if (!ok) atomicMin(out, (unsigned long long)b);
}

int64_t check_equivalence(Ctx &c, const float *pts, int64_t n, int dim, float eps, const int32_t *gl,
                          const uint8_t *gc, const int32_t *wl, const uint8_t *wc, int *kind) {
  *kind = 0;
  if (n <= 0) return -1;
  DevBuf<unsigned long long> first(5, c.stream);
  SPB_CUDA(cudaMemsetAsync(first.get(), 0xff, 5 * sizeof(unsigned long long), c.stream));
  const unsigned G = grid_for(n, 256, 148 * 16);
  k_eq_flags<<<G, 256, 0, c.stream>>>(n, gl, gc, wl, wc, first.get());
  SPB_LAUNCHED();
  {
    DevBuf<uint64_t> f0((size_t)n, c.stream), r0((size_t)n, c.stream), t((size_t)n, c.stream);
    DevBuf<uint32_t> i0((size_t)n, c.stream), i1((size_t)n, c.stream), j0((size_t)n, c.stream);
    k_eq_pairs<<<G, 256, 0, c.stream>>>(n, gl, wl, wc, f0.get(), r0.get(), i0.get());
    SPB_LAUNCHED();
    SPB_CUDA(cudaMemcpyAsync(j0.get(), i0.get(), (size_t)n * 4, cudaMemcpyDeviceToDevice, c.stream));
    for (int which = 0; which < 2; ++which) {
      uint64_t *ka = which ? r0.get() : f0.get(), *kb = t.get();
      uint32_t *va = which ? j0.get() : i0.get(), *vb = i1.get();
      radix_sort_pairs(c, &ka, &va, &kb, &vb, n, 64, false);
      k_eq_bijective<<<G, 256, 0, c.stream>>>(n, ka, va, first.get() + 2 + which);
      SPB_LAUNCHED();
    }
  }
  Tree t;
  build_tree(c, pts, n, dim, true, 64, t);
  k_eq_border<<<(unsigned)((n + 127) / 128), 128, 0, c.stream>>>(t.nodes, t.leafpt, t.perm, n, make_radius(eps), gl,
                                                                   gc, first.get() + 4);
  SPB_LAUNCHED();
  unsigned long long h[5];
  peek(c, {{first.get(), h, sizeof(h)}});
  for (int k = 0; k < 5; ++k)
    if (h[k] != ~0ull) {
      *kind = k + 1;
      return (int64_t)h[k];
    }
  return -1;
}

}  // namespace spb
