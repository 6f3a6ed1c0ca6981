// Clustering on sm_100a: FDBSCAN / friends-of-friends with the pair traversal
// fused with lock-free union-find (K6), capped core counting (K5 with early
// termination), the border claim latch, and label finalisation (K7).
// Reference: dbscan.hpp:72-292, union_find.hpp:17-82, traversal.hpp:162-184.
//
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <cmath>

#include "sp_common.cuh"
#include "sp_internal.hpp"
#include "sp_query.hpp"
#include "sp_traverse.cuh"

namespace spb {

// Union-find lives in SORTED-POSITION space: Morton neighbours are memory
// neighbours, so parent[] accesses stay local.  Canonical labels (the smallest
// ORIGINAL index of each set, finalize_labels, dbscan.hpp:72-98) are recovered
// in the finalisation pass.

__global__ void k_iota(int32_t *a, int64_t n) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) a[i] = (int32_t)i;
}

// Capped neighbour counts (detect_core_counts, dbscan.hpp:146-182); queries
// run in leaf order, which is the order sort_queries gives the same points
// (traversal.hpp:209-218).  Counts include the point itself and stop at
// min_pts, so count = min(hits, min_pts) whatever the visiting order.
template <bool FAST>
__global__ void __launch_bounds__(128, 1) k_core_flags(const float4 *__restrict__ nodes,
                                                    const float4 *__restrict__ leafpt, int64_t n, Radius R,
                                                    int32_t min_pts, uint8_t *__restrict__ corep,
                                                    unsigned long long *slices, int nslices) {
  R.fast = FAST ? 1 : 0;  // as the host checked: one form of the filters compiles
  SmSliceWalk w(n, slices, nslices);
  for (int64_t p; w.next(p);) {
    if (p < 0) continue;
    const float4 me = ld_node(leafpt, p);
    // Morton neighbours (leaf order) first; the walk from the root skips them.
    // Counts include the point itself and stop at min_pts.
    constexpr int W = 8;
    const int64_t w_lo = p - W > 0 ? p - W : 0, w_hi = p + W < n - 1 ? p + W : n - 1;
    int32_t c = 0;
    for (int64_t q = w_lo; q <= w_hi && c < min_pts; ++q) {
      const float4 L = ld_node(leafpt, q);
      c += hit_point(R, me.x, me.y, me.z, L.x, L.y, L.z);
    }
    if (c < min_pts) {
      const int64_t first_leaf = n - 1;
      int32_t cur = 0;  // root (a leaf when n == 1)
      while (cur != kSentinel) {
        if (cur >= first_leaf) {
          const int64_t q = cur - first_leaf;
          const float4 L = ld_node(leafpt, q);
          const bool counted = q >= w_lo && q <= w_hi;  // in the Morton window above
          if (!counted && hit_point(R, me.x, me.y, me.z, L.x, L.y, L.z) && ++c == min_pts) cur = kSentinel;
          else cur = __float_as_int(L.w);
        } else {
          float4 lo, hi;
          ld_node2(nodes, (int64_t)cur, lo, hi);
          cur = maybe_box(R, me.x, me.y, me.z, lo, hi) ? node_link(lo) : node_rope(hi);
        }
      }
    }
    corep[p] = c >= min_pts;
  }
}

// The merge rule for one close pair (p's leaf precedes q's).  FOF: every
// close pair unions (core <=> set size > 1 is derived at finalisation,
// dbscan.hpp:102-110, 259-263).  Otherwise merge_close_pair
// (dbscan.hpp:123-137): core-core unions; core-noncore unions iff the
// non-core side wins its one-shot claim latch (union_find.hpp:63-82).
// root_p is a hint for p's root: if q already points at it the pair is in one
// set (true even for a stale hint, which is still a member of p's set), else a
// union costs one find on q.
// SEQ (ExecMode::kSequential): core-core pairs only; border points are
// assigned afterwards by k_border_seq.
template <bool FOF, bool SEQ = false>
__device__ __forceinline__ void merge_pair(int32_t p, int32_t q, bool core_p, int32_t &root_p, int32_t *parent,
                                           const uint8_t *corep, uint32_t *claims) {
  if (FOF) {
    if (parent[q] == root_p) return;
    root_p = uf_union(parent, root_p, q);
    return;
  }
  const bool core_q = corep[q] != 0;
  if (core_p && core_q) {
    if (parent[q] == root_p) return;
    root_p = uf_union(parent, root_p, q);
  } else if (!SEQ && (core_p || core_q)) {
    const int32_t b = core_p ? q : p;  // the non-core side
    const uint32_t bit = 1u << (b & 31);
    if (!(atomicOr(&claims[b >> 5], bit) & bit)) root_p = uf_union(parent, root_p, q);
  }
}

// Pair traversal fused with the merge rule (traversal.hpp:162-184 +
// dbscan.hpp:252-263): leaf p walks the ropes from its own rope, so only later
// leaves are examined and each close pair is seen exactly once.  Leaves are
// read as one 16-byte {x,y,z,rope}; internal nodes take the conservative
// fp32 test, leaves the exact one.
template <bool FOF, bool FAST, bool SEQ = false>
__global__ void __launch_bounds__(128, 1) k_merge_pairs(const float4 *__restrict__ nodes,
                                                     const float4 *__restrict__ leafpt, int64_t n, Radius R,
                                                     int32_t *parent, const uint8_t *__restrict__ corep,
                                                     uint32_t *claims, unsigned long long *slices, int nslices) {
  R.fast = FAST ? 1 : 0;
  SmSliceWalk w(n, slices, nslices);
  for (int64_t p; w.next(p);) {
    if (p < 0) continue;
    const int64_t first_leaf = n - 1;
    const float4 me = ld_node(leafpt, p);
    int32_t cur = __float_as_int(me.w);
    int32_t root_p = (int32_t)p;
    const bool core_p = FOF ? true : corep[p] != 0;
    while (cur != kSentinel) {
      if (cur >= first_leaf) {
        const int32_t q = (int32_t)(cur - first_leaf);
        const float4 L = ld_node(leafpt, q);
        if (hit_point(R, me.x, me.y, me.z, L.x, L.y, L.z))
          merge_pair<FOF, SEQ>((int32_t)p, q, core_p, root_p, parent, corep, claims);
        cur = __float_as_int(L.w);
      } else {
        float4 lo, hi;
        ld_node2(nodes, (int64_t)cur, lo, hi);
        cur = maybe_box(R, me.x, me.y, me.z, lo, hi) ? node_link(lo) : node_rope(hi);
      }
    }
  }
}

// Border points of the sequential mode (ExecMode::kSequential, exec.hpp:12).
// The reference's sequential pair traversal (traversal.hpp:162-184 with
// parallel_for run in order) reports the pairs of leaf p before those of leaf
// p + 1, and each leaf's later partners in leaf order, so the first
// (core, border) pair of a border point y -- the one whose claim latch wins
// (dbscan.hpp:123-137) -- is the one with its core neighbour of SMALLEST leaf
// position: a partner x before y is reported in x's turn, before y's own,
// and among partners after y the rope walk meets the smallest first.  Here
// every non-core point walks the tree from the root in depth-first order,
// which meets the leaves in increasing position, stops at the first core
// leaf within eps and joins that point's set.  The labels are therefore the
// reference's sequential labels bit for bit.
template <bool FAST>
__global__ void __launch_bounds__(128) k_border_seq(const float4 *__restrict__ nodes,
                                                    const float4 *__restrict__ leafpt, int64_t n, Radius R,
                                                    int32_t *parent, const uint8_t *__restrict__ corep,
                                                    uint32_t *claims) {
  R.fast = FAST ? 1 : 0;
  const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= n || corep[p]) return;
  const float4 me = ld_node(leafpt, p);
  const int64_t first_leaf = n - 1;
  int32_t cur = 0, found = -1;
  while (cur != kSentinel) {
    if (cur >= first_leaf) {
      const int32_t q = (int32_t)(cur - first_leaf);
      const float4 L = ld_node(leafpt, q);
      const bool take = q != p && corep[q] && hit_point(R, me.x, me.y, me.z, L.x, L.y, L.z);
      found = take ? q : found;
      cur = take ? kSentinel : __float_as_int(L.w);
    } else {
      float4 lo, hi;
      ld_node2(nodes, (int64_t)cur, lo, hi);
      cur = maybe_box(R, me.x, me.y, me.z, lo, hi) ? node_link(lo) : node_rope(hi);
    }
  }
  if (found >= 0) {
    atomicOr(&claims[p >> 5], 1u << (p & 31));
    uf_union(parent, (int32_t)p, found);
  }
}

// FoF core flags: a point is core iff its set has another member, i.e. it is
// not a root, or it is a root somebody points at (mark_core_by_set_size,
// dbscan.hpp:102-110).  Compresses every point to its root.
__global__ void __launch_bounds__(256) k_fof_core(int64_t n, int32_t *parent, uint8_t *corep) {
  const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= n) return;
  const int32_t r = uf_root(parent, (int32_t)p);
  if (r != p) {
    parent[p] = r;
    corep[p] = 1;
    corep[r] = 1;
  }
}

__device__ __forceinline__ bool is_member(const uint8_t *corep, const uint32_t *claims, int64_t p) {
  return corep[p] != 0 || (claims && ((claims[p >> 5] >> (p & 31)) & 1u));
}

// Finalisation 1: compress every member to its root and fold the smallest
// original index into minobj[root] (warp-aggregated: Morton-adjacent members
// usually share a root).
__global__ void __launch_bounds__(256) k_final_roots(int64_t n, int32_t *parent, const uint8_t *__restrict__ corep,
                                                     const uint32_t *__restrict__ claims,
                                                     const int32_t *__restrict__ perm,
                                                     const int32_t *__restrict__ ids, int32_t *minobj) {
  const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  int32_t key = -1, v = 0x7fffffff;
  if (p < n && is_member(corep, claims, p)) {
    key = uf_root(parent, (int32_t)p);
    parent[p] = key;
    v = ids ? ids[perm[p]] : perm[p];
  }
  const uint32_t peers = __match_any_sync(0xffffffffu, key);
  const int32_t m = (int32_t)__reduce_min_sync(peers, (uint32_t)v);
  if (key >= 0 && (threadIdx.x & 31) == __ffs(peers) - 1) atomicMin(&minobj[key], m);
}

// Finalisation 2: scatter labels/core flags to original order; a point that
// is neither core nor claimed is a singleton and therefore noise.
__global__ void __launch_bounds__(256) k_final_labels(int64_t n, const int32_t *__restrict__ parent,
                                                      const uint8_t *__restrict__ corep,
                                                      const uint32_t *__restrict__ claims,
                                                      const int32_t *__restrict__ perm,
                                                      const int32_t *__restrict__ minobj, int32_t *__restrict__ labels,
                                                      uint8_t *__restrict__ core) {
  const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= n) return;
  const int32_t obj = perm[p];
  const bool member = is_member(corep, claims, p);
  labels[obj] = member ? minobj[parent[p]] : -1;
  core[obj] = corep[p];
}

void dbscan(Ctx &c, const float *points, int64_t n, int dim, float eps, int32_t min_pts, int algo, int width,
            int32_t *labels, uint8_t *core, DbscanResult *res, const int32_t *ids) {
  if (!(eps > 0.f) || !std::isfinite(eps)) throw InvalidArgument("dbscan: eps must be positive and finite");
  // algo: 0 fdbscan, 1 friends_of_friends, 2 fdbscan_densebox (sp_b200.h
  // SP_ALGO_*); 3 friends_of_friends by pair traversal over the point
  // hierarchy (the reference's own algorithm, no grid); 4 fdbscan_densebox
  // over the reference's mixed tree of dense cells and sparse points.
  // SP_ALGO_SEQUENTIAL (0x100): ExecMode::kSequential; deterministic border
  // assignment equal to the reference's sequential run.  Friends-of-friends
  // is deterministic in both modes.
  const bool seq = (algo & 0x100) != 0;
  algo &= 0xff;
  if (algo == 1 || algo == 3) min_pts = 2;
  if (min_pts < 2) throw InvalidArgument("dbscan: min_pts must be at least 2");
  if (n == 0) return;
  if (min_pts == 2 && (algo == 0 || algo == 1)) {
    // friends-of-friends over grid cells (the DenseBox shortcut)
    extern bool fof_cells(Ctx &, const float *, int64_t, int, float, int32_t *, uint8_t *, DbscanResult *,
                          const int32_t *);
    if (fof_cells(c, points, n, dim, eps, labels, core, res, ids)) return;
  }
  if (algo == 2 || algo == 4) {
    extern void densebox(Ctx &, const float *, int64_t, int, float, int32_t, int, int32_t *, uint8_t *,
                         DbscanResult *, bool, bool);
    densebox(c, points, n, dim, eps, min_pts, width, labels, core, res, algo == 2, seq);
    return;
  }
  cudaEvent_t ev[5];
  for (auto &e : ev) SPB_CUDA(cudaEventCreate(&e));
  struct EvGuard {
    cudaEvent_t *e;
    ~EvGuard() {
      for (int i = 0; i < 5; ++i) cudaEventDestroy(e[i]);
    }
  } guard{ev};
  SPB_CUDA(cudaEventRecord(ev[0], c.stream));
  Tree t;
  try {
    build_tree(c, points, n, dim, true, width, t);
  } catch (const InvalidArgument &) {
    throw InvalidArgument("dbscan: non-finite coordinate");
  }
  SPB_CUDA(cudaEventRecord(ev[1], c.stream));
  const Radius R = make_radius(eps);
  const bool count_phase = min_pts > 2;
  const unsigned g256 = (unsigned)((n + 255) / 256);
  DevBuf<uint8_t> corep((size_t)n, c.stream);
  DevBuf<int32_t> parent((size_t)n, c.stream), minobj((size_t)n, c.stream);
  DevBuf<uint32_t> claims(count_phase ? (size_t)((n + 31) / 32) : 0, c.stream);
  // both walks run on the SM-affine schedule (sp_common.cuh)
  if (count_phase) {
    SmSlices sl(c);
    auto kern = R.fast ? k_core_flags<true> : k_core_flags<false>;
    kern<<<sl.grid(kern, 128), 128, 0, c.stream>>>(t.nodes, t.leafpt, n, R, min_pts, corep.get(), sl.ctr.get(),
                                                   sl.nsm);
    SPB_LAUNCHED();
    mark(c, "core");
  } else {
    SPB_CUDA(cudaMemsetAsync(corep.get(), 0, (size_t)n, c.stream));
  }
  SPB_CUDA(cudaEventRecord(ev[2], c.stream));
  k_iota<<<grid_for(n, 256, 148 * 16), 256, 0, c.stream>>>(parent.get(), n);
  SPB_LAUNCHED();
  {
    SmSlices sl(c);
    if (count_phase) SPB_CUDA(cudaMemsetAsync(claims.get(), 0, claims.n * sizeof(uint32_t), c.stream));
    auto kern = count_phase ? (seq ? (R.fast ? k_merge_pairs<false, true, true> : k_merge_pairs<false, false, true>)
                                   : (R.fast ? k_merge_pairs<false, true> : k_merge_pairs<false, false>))
                            : (R.fast ? k_merge_pairs<true, true> : k_merge_pairs<true, false>);
    kern<<<sl.grid(kern, 128), 128, 0, c.stream>>>(t.nodes, t.leafpt, n, R, parent.get(), corep.get(),
                                                   count_phase ? claims.get() : nullptr, sl.ctr.get(), sl.nsm);
  }
  SPB_LAUNCHED();
  if (count_phase && seq) {
    auto kern = R.fast ? k_border_seq<true> : k_border_seq<false>;
    kern<<<(unsigned)((n + 127) / 128), 128, 0, c.stream>>>(t.nodes, t.leafpt, n, R, parent.get(), corep.get(),
                                                            claims.get());
    SPB_LAUNCHED();
  }
  SPB_CUDA(cudaEventRecord(ev[3], c.stream));
  mark(c, "merge");
  if (!count_phase) {
    k_fof_core<<<g256, 256, 0, c.stream>>>(n, parent.get(), corep.get());
    SPB_LAUNCHED();
  }
  SPB_CUDA(cudaMemsetAsync(minobj.get(), 0x7f, (size_t)n * sizeof(int32_t), c.stream));
  k_final_roots<<<g256, 256, 0, c.stream>>>(n, parent.get(), corep.get(), claims.get(), t.perm, ids, minobj.get());
  SPB_LAUNCHED();
  k_final_labels<<<g256, 256, 0, c.stream>>>(n, parent.get(), corep.get(), claims.get(), t.perm, minobj.get(), labels,
                                             core);
  SPB_LAUNCHED();
  SPB_CUDA(cudaEventRecord(ev[4], c.stream));
  mark(c, "finalize");
  if (c.async()) return;  // timings need a host wait; async calls skip them
  SPB_CUDA(cudaEventSynchronize(ev[4]));
  if (res) {
    for (int i = 0; i < 4; ++i) {
      float ms = 0.f;
      cudaEventElapsedTime(&ms, ev[i], ev[i + 1]);
      res->ms[i] = ms;
    }
  }
}

}  // namespace spb

namespace spb {

// ---------------------------------------------------------------------------
// adjacency_graph_dbscan (dbscan.hpp:456-504): the historical min_pts = 2
// baseline.  Materialises every point's eps-neighbourhood as CRS (query_crs,
// traversal.hpp:235-266; SP_ECAPACITY beyond max_adjacency, like its
// CapacityError), unions each point with every other member of its row, and
// marks a point core iff its row holds more than itself.  Union-find runs in
// original index space with min-index hooking, so a root is the label.
// ---------------------------------------------------------------------------
__global__ void k_point_spheres(const float *__restrict__ pts, int64_t n, int dim, float eps,
                                float *__restrict__ sph) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    for (int k = 0; k < dim; ++k) sph[i * (dim + 1) + k] = pts[i * dim + k];
    sph[i * (dim + 1) + dim] = eps;
  }
}

__global__ void k_adjacency_unions(int64_t n, const int64_t *__restrict__ off, const int32_t *__restrict__ val,
                                   int32_t *parent, uint8_t *__restrict__ core) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  int32_t root = (int32_t)i;
  for (int64_t e = off[i]; e < off[i + 1]; ++e) {
    const int32_t j = val[e];
    if (j != i) root = uf_union(parent, root, j);
  }
  core[i] = (off[i + 1] - off[i]) > 1;
}

__global__ void k_adjacency_labels(int64_t n, const int32_t *__restrict__ parent, const uint8_t *__restrict__ core,
                                   int32_t *__restrict__ labels) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride)
    labels[i] = core[i] ? uf_root(parent, (int32_t)i) : -1;
}

void adjacency_dbscan(Ctx &c, const float *points, int64_t n, int dim, float eps, int width, int64_t max_adjacency,
                      int32_t *labels, uint8_t *core, DbscanResult *res) {
  if (!(eps > 0.f) || !std::isfinite(eps)) throw InvalidArgument("dbscan: eps must be positive and finite");
  if (n == 0) return;
  cudaEvent_t ev[5];
  for (auto &e : ev) SPB_CUDA(cudaEventCreate(&e));
  struct EvGuard {
    cudaEvent_t *e;
    ~EvGuard() {
      for (int i = 0; i < 5; ++i) cudaEventDestroy(e[i]);
    }
  } guard{ev};
  SPB_CUDA(cudaEventRecord(ev[0], c.stream));
  Tree t;
  try {
    build_tree(c, points, n, dim, true, width, t);
  } catch (const InvalidArgument &) {
    throw InvalidArgument("dbscan: non-finite coordinate");
  }
  SPB_CUDA(cudaEventRecord(ev[1], c.stream));
  DevBuf<float> sph((size_t)n * (dim + 1), c.stream);
  k_point_spheres<<<grid_for(n, 256, 148 * 16), 256, 0, c.stream>>>(points, n, dim, eps, sph.get());
  SPB_LAUNCHED();
  DevBuf<int64_t> off((size_t)n + 1, c.stream);
  const int64_t total = range_crs(c, t, RQ_SPHERES, sph.get(), n, off.get(), nullptr, 0);
  if (total > max_adjacency) throw CapacityError();
  DevBuf<int32_t> val((size_t)std::max<int64_t>(total, 1), c.stream);
  range_crs(c, t, RQ_SPHERES, sph.get(), n, off.get(), val.get(), total);
  SPB_CUDA(cudaEventRecord(ev[2], c.stream));
  DevBuf<int32_t> parent((size_t)n, c.stream);
  k_iota<<<grid_for(n, 256, 148 * 16), 256, 0, c.stream>>>(parent.get(), n);
  SPB_LAUNCHED();
  k_adjacency_unions<<<(unsigned)((n + 127) / 128), 128, 0, c.stream>>>(n, off.get(), val.get(), parent.get(), core);
  SPB_LAUNCHED();
  SPB_CUDA(cudaEventRecord(ev[3], c.stream));
  k_adjacency_labels<<<grid_for(n, 256, 148 * 16), 256, 0, c.stream>>>(n, parent.get(), core, labels);
  SPB_LAUNCHED();
  SPB_CUDA(cudaEventRecord(ev[4], c.stream));
  SPB_CUDA(cudaEventSynchronize(ev[4]));
  if (res) {
    for (int i = 0; i < 4; ++i) {
      float ms = 0.f;
      cudaEventElapsedTime(&ms, ev[i], ev[i + 1]);
      res->ms[i] = ms;
    }
  }
}

}  // namespace spb

namespace spb {

// ---------------------------------------------------------------------------
// dbscan_reference (dbscan.hpp:188-222) on the device: brute-force O(n^2)
// neighbourhoods, exact core flags, core-core unions, and each border point
// claimed by one core neighbour.  Independent of the tree; the CLI's
// --verify / --algo oracle counterpart (intended for small n).
// ---------------------------------------------------------------------------
__global__ void k_bf_core(const float4 *__restrict__ p4, int64_t n, Radius R, int32_t min_pts,
                          uint8_t *__restrict__ core) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const float4 a = p4[i];
  int32_t c = 0;
  for (int64_t j = 0; j < n; ++j) {
    const float4 b = p4[j];
    c += hit_point(R, a.x, a.y, a.z, b.x, b.y, b.z);
  }
  core[i] = c >= min_pts;
}

__global__ void k_bf_merge(const float4 *__restrict__ p4, int64_t n, Radius R, const uint8_t *__restrict__ core,
                           int32_t *parent, uint32_t *claims) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n || !core[i]) return;
  const float4 a = p4[i];
  int32_t root = (int32_t)i;
  for (int64_t j = 0; j < n; ++j) {
    if (j == i) continue;
    const float4 b = p4[j];
    if (!hit_point(R, a.x, a.y, a.z, b.x, b.y, b.z)) continue;
    if (core[j]) {
      if (j > i) root = uf_union(parent, root, (int32_t)j);
    } else {
      const uint32_t bit = 1u << (j & 31);
      if (!(atomicOr(&claims[j >> 5], bit) & bit)) root = uf_union(parent, root, (int32_t)j);
    }
  }
}

__global__ void k_bf_points(const float *__restrict__ pts, int64_t n, int dim, float4 *__restrict__ p4) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride)
    p4[i] = make_float4(pts[i * dim], pts[i * dim + 1], dim == 3 ? pts[i * dim + 2] : 0.f, 0.f);
}

__global__ void k_bf_labels(int64_t n, const int32_t *__restrict__ parent, const uint8_t *__restrict__ core,
                            const uint32_t *__restrict__ claims, int32_t *__restrict__ labels) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    const bool member = core[i] || ((claims[i >> 5] >> (i & 31)) & 1u);
    labels[i] = member ? uf_root(parent, (int32_t)i) : -1;
  }
}

void bruteforce_dbscan(Ctx &c, const float *points, int64_t n, int dim, float eps, int32_t min_pts, int32_t *labels,
                       uint8_t *core) {
  if (!(eps > 0.f) || !std::isfinite(eps)) throw InvalidArgument("dbscan: eps must be positive and finite");
  if (min_pts < 2) throw InvalidArgument("dbscan: min_pts must be at least 2");
  if (n == 0) return;
  const Radius R = make_radius(eps);
  DevBuf<float4> p4((size_t)n, c.stream);
  DevBuf<int32_t> parent((size_t)n, c.stream);
  DevBuf<uint32_t> claims((size_t)((n + 31) / 32), c.stream);
  const unsigned G = grid_for(n, 256, 148 * 16), Gq = (unsigned)((n + 127) / 128);
  k_bf_points<<<G, 256, 0, c.stream>>>(points, n, dim, p4.get());
  SPB_LAUNCHED();
  SPB_CUDA(cudaMemsetAsync(claims.get(), 0, claims.n * sizeof(uint32_t), c.stream));
  k_iota<<<G, 256, 0, c.stream>>>(parent.get(), n);
  SPB_LAUNCHED();
  k_bf_core<<<Gq, 128, 0, c.stream>>>(p4.get(), n, R, min_pts, core);
  SPB_LAUNCHED();
  k_bf_merge<<<Gq, 128, 0, c.stream>>>(p4.get(), n, R, core, parent.get(), claims.get());
  SPB_LAUNCHED();
  k_bf_labels<<<G, 256, 0, c.stream>>>(n, parent.get(), core, claims.get(), labels);
  SPB_LAUNCHED();
}

}  // namespace spb
