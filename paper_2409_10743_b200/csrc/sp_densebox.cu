// FDBSCAN-DenseBox on sm_100a (fdbscan_densebox, dbscan.hpp:298-449;
// build_dense_grid, dense_grid.hpp:52-103).
//
//   K8  grid:   cell coordinates floor((p - anchor) / cell_length) in double,
//               Morton-interleaved into one sortable key; a stable radix sort
//               groups every cell's members contiguously in ascending index
//               order; segment heads give cell sizes; cells with >= min_pts
//               members are dense (none when coordinates could saturate).
//   objects:    dense cells ordered by smallest member (dbscan.hpp:312-320)
//               as tight boxes, then every sparse point as a point box in
//               index order (dbscan.hpp:322-339) -> the mixed hierarchy.
//   K9  core:   sparse points count self + sparse neighbours + dense-cell
//               members within eps, stopping at min_pts (dbscan.hpp:351-385).
//   K9  merge:  intra-dense-cell unions (dbscan.hpp:390-394), then every point
//               walks the mixed tree: own cell skipped, dense hits expand to
//               per-member checks with the i < j guard (counted as
//               distance_checks), sparse hits merge with i < j
//               (dbscan.hpp:398-440).
// Union-find runs in ORIGINAL index space with min-index hooking, so a root
// is already the canonical label (finalize_labels, dbscan.hpp:72-98).
#include <cuda_runtime.h>
#include <stdint.h>

#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "sp_common.cuh"
#include "sp_internal.hpp"
#include "sp_query.hpp"
#include "sp_traverse.cuh"

namespace spb {

#ifndef SPB_CORE_WINDOW
#define SPB_CORE_WINDOW 4
#endif

namespace {

// Host synchronisation point (the few phases that size a buffer from a
// device count).
void host_sync(Ctx &c, int line) {
  (void)line;
  SPB_CUDA(cudaStreamSynchronize(c.stream));
}

__device__ __forceinline__ uint64_t spread3_21(uint64_t v) {
  v &= 0x1fffffull;
  v = (v | (v << 32)) & 0x001f00000000ffffull;
  v = (v | (v << 16)) & 0x001f0000ff0000ffull;
  v = (v | (v << 8)) & 0x100f00f00f00f00full;
  v = (v | (v << 4)) & 0x10c30c30c30c30c3ull;
  v = (v | (v << 2)) & 0x1249249249249249ull;
  return v;
}
__device__ __forceinline__ uint64_t spread2_32(uint64_t v) {
  v &= 0xffffffffull;
  v = (v | (v << 16)) & 0x0000ffff0000ffffull;
  v = (v | (v << 8)) & 0x00ff00ff00ff00ffull;
  v = (v | (v << 4)) & 0x0f0f0f0f0f0f0f0full;
  v = (v | (v << 2)) & 0x3333333333333333ull;
  v = (v | (v << 1)) & 0x5555555555555555ull;
  return v;
}

// DenseGrid::coord_of (dense_grid.hpp:60-73) for one axis.
__host__ __device__ __forceinline__ int64_t cell_coord(float p, float anchor, float cell) {
  double f = floor(((double)p - (double)anchor) / (double)cell);
  if (f < -4.0e18) f = -4.0e18;
  if (f > 4.0e18) f = 4.0e18;
  return (int64_t)f;
}

// Morton key of the cell (axis 0 in the LSB), or per-axis coordinate keys
// when the coordinates need more than the interleave width.
__global__ void k_cell_keys(const float *__restrict__ pts, int64_t n, int dim, const float *__restrict__ scene,
                            float cell, int axis, uint64_t *__restrict__ keys) {
  const float a0 = scene[0], a1 = scene[1], a2 = scene[2];
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    const float *p = pts + i * dim;
    if (axis >= 0) {
      const float a = axis == 0 ? a0 : (axis == 1 ? a1 : a2);
      keys[i] = (uint64_t)cell_coord(p[axis], a, cell);
      continue;
    }
    const uint64_t c0 = (uint64_t)cell_coord(p[0], a0, cell), c1 = (uint64_t)cell_coord(p[1], a1, cell);
    if (dim == 3) {
      const uint64_t c2 = (uint64_t)cell_coord(p[2], a2, cell);
      keys[i] = spread3_21(c0) | (spread3_21(c1) << 1) | (spread3_21(c2) << 2);
    } else {
      keys[i] = spread2_32(c0) | (spread2_32(c1) << 1);
    }
  }
}

// 3-D points, 16-byte aligned: Morton cell keys, four points per step.
__global__ void __launch_bounds__(256) k_cell_keys_p3v(const float *__restrict__ pts, int64_t n,
                                                       const float *__restrict__ scene, float cell,
                                                       uint64_t *__restrict__ keys, uint32_t *ghist = nullptr) {
  __shared__ uint32_t s_hist[5 * 256];
  HistAcc<5> H;  // the 40-bit sort's five digits (radix_sort_pairs_40), when ghist is given
  H.init(s_hist, ghist);
  const float a0 = scene[0], a1 = scene[1], a2 = scene[2];
  const int64_t chunks = n / 4;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const int64_t t0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  auto key = [&](float x, float y, float z) -> uint64_t {
    return spread3_21((uint64_t)cell_coord(x, a0, cell)) | (spread3_21((uint64_t)cell_coord(y, a1, cell)) << 1) |
           (spread3_21((uint64_t)cell_coord(z, a2, cell)) << 2);
  };
  for (int64_t ch = t0; ch < chunks; ch += stride) {
    float x[4], y[4], z[4];
    load4pts(pts, ch, x, y, z);
    ulonglong2 k01, k23;
    k01.x = key(x[0], y[0], z[0]);
    k01.y = key(x[1], y[1], z[1]);
    k23.x = key(x[2], y[2], z[2]);
    k23.y = key(x[3], y[3], z[3]);
    reinterpret_cast<ulonglong2 *>(keys)[2 * ch] = k01;
    reinterpret_cast<ulonglong2 *>(keys)[2 * ch + 1] = k23;
    H.add(k01.x);
    H.add(k01.y);
    H.add(k23.x);
    H.add(k23.y);
  }
  for (int64_t i = chunks * 4 + t0; i < n; i += stride) {
    keys[i] = key(pts[3 * i], pts[3 * i + 1], pts[3 * i + 2]);
    H.add(keys[i]);
  }
  H.flush();
}

__global__ void k_gather_keys(const float *__restrict__ pts, int64_t n, int dim, const float *__restrict__ scene,
                              float cell, int axis, const uint32_t *__restrict__ order, uint64_t *__restrict__ keys) {
  const float a = scene[axis];
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride)
    keys[i] = (uint64_t)cell_coord(pts[(int64_t)order[i] * dim + axis], a, cell);
}

// Cell heads in the sorted order: head[i] = 1 where a new cell starts.  For
// the per-axis path the equality test needs all coordinates.
__global__ void k_heads(const uint64_t *__restrict__ keys, const uint32_t *__restrict__ order,
                        const float *__restrict__ pts, int dim, const float *__restrict__ scene, float cell,
                        int64_t n, bool exact_keys, int32_t *__restrict__ head) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    int32_t h;
    if (i == 0) {
      h = 1;
    } else if (exact_keys) {
      h = keys[i] != keys[i - 1];
    } else {
      const float *a = pts + (int64_t)order[i] * dim, *b = pts + (int64_t)order[i - 1] * dim;
      h = 0;
      for (int k = 0; k < dim; ++k) h |= cell_coord(a[k], scene[k], cell) != cell_coord(b[k], scene[k], cell);
    }
    head[i] = h;
  }
}

// Cell segmentation of the sorted keys in one pass (replaces heads + scan +
// starts): a stream compaction of the segment heads with a decoupled
// look-back over 4096-key tiles.  Writes cell_start[j] = first position of
// cell j, cell_of[i] = cell of sorted position i, and the number of cells.
#ifndef SPB_CC_ITEMS
#define SPB_CC_ITEMS 24  // 8 / 16 / 24 / 32: grid + hierarchy phase 7.74 / 7.64 / 7.42 / 8.05 ms at 2^27
#endif
constexpr int CC_THREADS = 256, CC_ITEMS = SPB_CC_ITEMS, CC_TILE = CC_THREADS * CC_ITEMS;
__global__ void __launch_bounds__(CC_THREADS) k_cell_compact(const uint64_t *__restrict__ keys, int64_t n,
                                                              int64_t *__restrict__ cell_start,
                                                              int32_t *__restrict__ cell_of,
                                                              unsigned long long *lookback, uint32_t *tile_ctr,
                                                              int64_t *total) {
  __shared__ uint32_t s_warp[CC_THREADS / 32];
  __shared__ uint32_t s_tile;
  __shared__ uint32_t s_excl;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) s_tile = atomicAdd(tile_ctr, 1u);
  __syncthreads();
  const int64_t tile = s_tile;
  const int64_t wbase = tile * CC_TILE + (int64_t)warp * (CC_ITEMS * 32);
  // striped items: item i of lane l is element wbase + i*32 + l
  uint32_t heads[CC_ITEMS];
  uint64_t prev_last = 0;
  {
    const int64_t pi = wbase - 1;
    prev_last = pi >= 0 && pi < n ? keys[pi] : ~0ull;
  }
  uint32_t wcount = 0;
#pragma unroll
  for (int i = 0; i < CC_ITEMS; ++i) {
    const int64_t idx = wbase + i * 32 + lane;
    const uint64_t k = idx < n ? keys[idx] : 0ull;
    uint64_t kp = __shfl_up_sync(0xffffffffu, k, 1);
    if (lane == 0) kp = prev_last;
    prev_last = __shfl_sync(0xffffffffu, k, 31);
    const bool h = idx < n && (idx == 0 || k != kp);
    heads[i] = __ballot_sync(0xffffffffu, h);
    wcount += __popc(heads[i]);
  }
  if (lane == 0) s_warp[warp] = wcount;
  __syncthreads();
  if (tid == 0) {
    uint32_t run = 0;
    for (int w = 0; w < CC_THREADS / 32; ++w) {
      const uint32_t c = s_warp[w];
      s_warp[w] = run;
      run += c;
    }
    // look-back over tiles (aggregate tag 1, inclusive tag 2)
    unsigned long long *mine = lookback + tile;
    uint32_t excl = 0;
    if (tile == 0) {
      st_volatile_u64(mine, (2ull << 32) | run);
    } else {
      st_volatile_u64(mine, (1ull << 32) | run);
      int64_t j = tile - 1;
      while (true) {
        const unsigned long long v = ld_volatile_u64(lookback + j);
        const unsigned long long st = v >> 32;
        if (st == 2) {
          excl += (uint32_t)v;
          break;
        }
        if (st == 1) {
          excl += (uint32_t)v;
          --j;
        }
      }
      st_volatile_u64(mine, (2ull << 32) | (excl + run));
    }
    s_excl = excl;
    if ((tile + 1) * (int64_t)CC_TILE >= n) *total = (int64_t)excl + run;
  }
  __syncthreads();
  uint32_t rank = s_excl + s_warp[warp];  // heads before this warp's slice
  const uint32_t lt = (1u << lane) - 1u;
#pragma unroll
  for (int i = 0; i < CC_ITEMS; ++i) {
    const int64_t idx = wbase + i * 32 + lane;
    const uint32_t r = rank + __popc(heads[i] & lt);  // heads before idx
    const bool h = (heads[i] >> lane) & 1u;
    if (idx < n) {
      cell_of[idx] = (int32_t)(r + (h ? 1u : 0u)) - 1;
      if (h) cell_start[r] = idx;
    }
    rank += __popc(heads[i]);
  }
}

// cell_start[c] = sorted position where cell c begins (c from the head scan).
__global__ void k_cell_starts(const int32_t *__restrict__ head, const int64_t *__restrict__ scan, int64_t n,
                              int64_t *__restrict__ cell_start) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride)
    if (head[i]) cell_start[scan[i]] = i;
}

// dense flag per cell; dense cells emit (min member, cell) for ordering.
__global__ void k_dense_flags(const int64_t *__restrict__ cell_start, int64_t m, int64_t n, int32_t min_pts,
                              bool no_dense, int32_t *__restrict__ dense) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; c < m; c += stride) {
    const int64_t len = (c + 1 < m ? cell_start[c + 1] : n) - cell_start[c];
    dense[c] = (!no_dense && len >= min_pts) ? 1 : 0;
  }
}

__global__ void k_dense_pack(const int32_t *__restrict__ dense, const int64_t *__restrict__ dscan,
                             const int64_t *__restrict__ cell_start, const uint32_t *__restrict__ order, int64_t m,
                             uint64_t *__restrict__ minkey, uint32_t *__restrict__ cellid) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; c < m; c += stride) {
    if (!dense[c]) continue;
    const int64_t d = dscan[c];
    minkey[d] = order[cell_start[c]];  // members ascend within a cell (stable sort)
    cellid[d] = (uint32_t)c;
  }
}

// One warp per dense object: member range, point_cell[], tight box
// (dense_grid.hpp / dbscan.hpp:326-333).
__global__ void k_dense_objects(const uint32_t *__restrict__ dense_cell, int64_t nd,
                                const int64_t *__restrict__ cell_start, int64_t m, int64_t n,
                                const uint32_t *__restrict__ order, const float *__restrict__ pts, int dim,
                                int32_t *__restrict__ point_cell, int64_t *__restrict__ dbeg, int32_t *__restrict__ dlen,
                                float *__restrict__ objects) {
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (warp >= nd) return;
  const int64_t c = dense_cell[warp];
  const int64_t s = cell_start[c], e = c + 1 < m ? cell_start[c + 1] : n;
  float lo[3] = {3.4028235e38f, 3.4028235e38f, 3.4028235e38f}, hi[3] = {-3.4028235e38f, -3.4028235e38f, -3.4028235e38f};
  for (int64_t i = s + lane; i < e; i += 32) {
    const uint32_t o = order[i];
    point_cell[o] = (int32_t)warp;
    for (int k = 0; k < dim; ++k) {
      const float v = pts[(int64_t)o * dim + k];
      lo[k] = fminf(lo[k], v);
      hi[k] = fmaxf(hi[k], v);
    }
  }
  for (int k = 0; k < dim; ++k) {
    for (int off = 16; off; off >>= 1) {
      lo[k] = fminf(lo[k], __shfl_xor_sync(0xffffffffu, lo[k], off));
      hi[k] = fmaxf(hi[k], __shfl_xor_sync(0xffffffffu, hi[k], off));
    }
  }
  if (lane == 0) {
    dbeg[warp] = s;
    dlen[warp] = (int32_t)(e - s);
    for (int k = 0; k < dim; ++k) {
      objects[warp * 2 * dim + k] = lo[k];
      objects[warp * 2 * dim + dim + k] = hi[k];
    }
  }
}

__global__ void k_sparse_flags(const int32_t *__restrict__ point_cell, int64_t n, int32_t *__restrict__ flag) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) flag[i] = point_cell[i] < 0;
}

__global__ void k_sparse_objects(const int32_t *__restrict__ point_cell, const int64_t *__restrict__ sscan, int64_t n,
                                 int64_t nd, const float *__restrict__ pts, int dim, int32_t *__restrict__ sparse_pts,
                                 float *__restrict__ objects) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    if (point_cell[i] >= 0) continue;
    const int64_t s = sscan[i];
    sparse_pts[s] = (int32_t)i;
    float *o = objects + (nd + s) * 2 * dim;
    for (int k = 0; k < dim; ++k) o[k] = o[dim + k] = pts[i * dim + k];
  }
}

struct DenseView {
  const float4 *nodes;
  int64_t nobj;
  int64_t nd;
  const int64_t *dbeg;
  const int32_t *dlen;
  const uint32_t *members;  // sorted-by-cell original indices
  const int32_t *sparse_pts;
  const float *pts;
  int dim;
  Radius R;
  const float4 *cpts;  // points in sorted-by-cell order {x, y, z, bits(original index)}
};

__global__ void k_cell_points(const uint32_t *__restrict__ order, const float *__restrict__ pts, int64_t n, int dim,
                              float4 *__restrict__ cpts) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < n; k += stride) {
    const uint32_t o = order[k];
    const float *q = pts + (int64_t)o * dim;
    cpts[k] = make_float4(q[0], q[1], dim == 3 ? q[2] : 0.f, __int_as_float((int)o));
  }
}

// 3-D, 16-byte aligned points: four sorted positions per thread with their
// random gathers in flight together, each point by one or two 16-byte loads
// (gather_pt3).
#ifndef SPB_CP_ILP
#define SPB_CP_ILP 2  // 2 / 4 / 8: grid + hierarchy phase 7.23 / 7.42 / 7.66 ms at 2^27
#endif
constexpr int CP_ILP = SPB_CP_ILP;
__global__ void __launch_bounds__(256) k_cell_points3v(const uint32_t *__restrict__ order,
                                                       const float *__restrict__ pts, int64_t n,
                                                       float4 *__restrict__ cpts) {
  const int64_t k0 = ((int64_t)blockIdx.x * blockDim.x) * CP_ILP + threadIdx.x;
  uint32_t o[CP_ILP];
  float x[CP_ILP], y[CP_ILP], z[CP_ILP];
#pragma unroll
  for (int u = 0; u < CP_ILP; ++u) {
    const int64_t k = k0 + (int64_t)u * blockDim.x;
    o[u] = k < n ? order[k] : 0u;
  }
#pragma unroll
  for (int u = 0; u < CP_ILP; ++u) gather_pt3(pts, n, o[u], x[u], y[u], z[u]);
#pragma unroll
  for (int u = 0; u < CP_ILP; ++u) {
    const int64_t k = k0 + (int64_t)u * blockDim.x;
    if (k < n) cpts[k] = make_float4(x[u], y[u], z[u], __int_as_float((int)o[u]));
  }
}

// The same gather, also writing each sorted point's Morton cell key (the
// 40-bit sort returns no keys: k_cell_keys_p3v's formula on the gathered point).
__global__ void __launch_bounds__(256) k_cell_points3v_keys(const uint32_t *__restrict__ order,
                                                            const float *__restrict__ pts, int64_t n,
                                                            const float *__restrict__ scene, float cell,
                                                            float4 *__restrict__ cpts, uint64_t *__restrict__ keys) {
  const float a0 = scene[0], a1 = scene[1], a2 = scene[2];
  const int64_t k0 = ((int64_t)blockIdx.x * blockDim.x) * CP_ILP + threadIdx.x;
  uint32_t o[CP_ILP];
  float x[CP_ILP], y[CP_ILP], z[CP_ILP];
#pragma unroll
  for (int u = 0; u < CP_ILP; ++u) {
    const int64_t k = k0 + (int64_t)u * blockDim.x;
    o[u] = k < n ? order[k] : 0u;
  }
#pragma unroll
  for (int u = 0; u < CP_ILP; ++u) gather_pt3(pts, n, o[u], x[u], y[u], z[u]);
#pragma unroll
  for (int u = 0; u < CP_ILP; ++u) {
    const int64_t k = k0 + (int64_t)u * blockDim.x;
    if (k >= n) continue;
    cpts[k] = make_float4(x[u], y[u], z[u], __int_as_float((int)o[u]));
    keys[k] = spread3_21((uint64_t)cell_coord(x[u], a0, cell)) | (spread3_21((uint64_t)cell_coord(y[u], a1, cell)) << 1) |
              (spread3_21((uint64_t)cell_coord(z[u], a2, cell)) << 2);
  }
}

void cell_points(Ctx &c, const uint32_t *order, const float *pts, int64_t n, int dim, float4 *cpts) {
  if (n <= 0) return;
  if (dim == 3 && aligned16(pts))
    k_cell_points3v<<<(unsigned)((n + 256 * CP_ILP - 1) / (256 * CP_ILP)), 256, 0, c.stream>>>(order, pts, n, cpts);
  else
    k_cell_points<<<grid_for(n, 256, 148 * 16), 256, 0, c.stream>>>(order, pts, n, dim, cpts);
  SPB_LAUNCHED();
}

__device__ __forceinline__ void load_pt(const float *pts, int dim, int64_t i, float &x, float &y, float &z) {
  x = pts[i * dim];
  y = pts[i * dim + 1];
  z = dim == 3 ? pts[i * dim + 2] : 0.f;
}

// Core detection for sparse points (dbscan.hpp:351-385).
__global__ void __launch_bounds__(128) k_db_core(DenseView v, const uint32_t *__restrict__ qorder, int64_t n,
                                                 const int32_t *__restrict__ point_cell, int32_t min_pts,
                                                 uint8_t *__restrict__ core) {
  const int64_t qi = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (qi >= n) return;
  const float4 me = v.cpts[qi];
  const int64_t i = __float_as_int(me.w);
  if (point_cell[i] >= 0) return;  // dense members are core already
  const float x = me.x, y = me.y, z = me.z;
  int32_t cnt = 0;
  int32_t cur = 0;
  while (cur != kSentinel) {
    const float4 lo = ld_node(v.nodes, 2 * (int64_t)cur);
    const float4 hi = ld_node(v.nodes, 2 * (int64_t)cur + 1);
    const bool leaf = cur >= v.nobj - 1;
    const bool hit = leaf ? hit_box(v.R, x, y, z, lo, hi) : maybe_box(v.R, x, y, z, lo, hi);
    if (cur >= v.nobj - 1) {
      if (hit) {
        const int32_t o = node_link(lo);
        if (o < v.nd) {
          const int64_t b = v.dbeg[o];
          const int32_t len = v.dlen[o];
          for (int32_t t = 0; t < len && cnt < min_pts; ++t) {
            const float4 q = v.cpts[b + t];
            if (hit_point(v.R, x, y, z, q.x, q.y, q.z)) ++cnt;
          }
        } else {
          ++cnt;
        }
        if (cnt >= min_pts) break;
      }
      cur = node_rope(hi);
    } else {
      cur = hit ? node_link(lo) : node_rope(hi);
    }
  }
  core[i] = cnt >= min_pts;
}

// Intra-cell unions: every member joins its cell's first (smallest) member.
__global__ void k_db_cell_unions(const int64_t *__restrict__ dbeg, const int32_t *__restrict__ dlen, int64_t nd,
                                 const uint32_t *__restrict__ members, int32_t *parent) {
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (warp >= nd) return;
  const int64_t b = dbeg[warp];
  const int32_t first = (int32_t)members[b];
  for (int32_t t = 1 + lane; t < dlen[warp]; t += 32) uf_union(parent, first, (int32_t)members[b + t]);
}

__device__ __forceinline__ bool cells_far(const Radius &R, const float4 &qlo, const float4 &qhi, const float4 &lo,
                                          const float4 &hi) {
  if (R.fast)
    return sq3(fmaxf(fmaxf(__fsub_rn(lo.x, qhi.x), __fsub_rn(qlo.x, hi.x)), 0.f),
               fmaxf(fmaxf(__fsub_rn(lo.y, qhi.y), __fsub_rn(qlo.y, hi.y)), 0.f),
               fmaxf(fmaxf(__fsub_rn(lo.z, qhi.z), __fsub_rn(qlo.z, hi.z)), 0.f)) > R.hi32;
  const double gx = fmax(fmax((double)lo.x - (double)qhi.x, (double)qlo.x - (double)hi.x), 0.0);
  const double gy = fmax(fmax((double)lo.y - (double)qhi.y, (double)qlo.y - (double)hi.y), 0.0);
  const double gz = fmax(fmax((double)lo.z - (double)qhi.z, (double)qlo.z - (double)hi.z), 0.0);
  return gx * gx + gy * gy + gz * gz > R.thr * (1.0 + 0x1p-30);
}

// ---- merge (dbscan.hpp:388-440), restated over objects ----------------------
// The reference walks every point and checks every member of every nearby dense
// cell.  Here the merge runs over OBJECTS (dense cells and sparse points, the
// leaves of the mixed tree) in two passes with the same result contract:
//  * core objects (dense cells -- all members core -- and core sparse points;
//    every sparse point for min_pts = 2): a rope walk from each object's leaf
//    over later leaves (pair traversal, traversal.hpp:162-184, so each object
//    pair once) unites two objects' sets at the first member pair within eps,
//    and skips objects already in its set.  The core partition therefore
//    equals the reference's (core-core pairs within eps, transitively).
//  * non-core sparse points (min_pts > 2): a walk from the root stops at the
//    first core point within eps and joins its set -- the reference's one-shot
//    claim latch (union_find.hpp:63-82) gives each border point to exactly one
//    adjacent cluster, which is all check_equivalence (verify.hpp:21-61)
//    requires.
// Union-find runs in original index space (root = smallest index).  A dense
// cell's set is represented by its first (smallest) member, pre-united with
// the others (dbscan.hpp:390-394).  distance_checks counts the member-pair
// distance evaluations this merge performs (dbscan.hpp:38-41).
struct ObjRef {
  int64_t beg;   // first member in cpts (dense cells)
  int32_t len;   // members (0: a sparse point)
  int32_t rep;   // set representative (original index)
  float x, y, z; // the point (sparse)
};

__device__ __forceinline__ ObjRef obj_ref(const DenseView &v, int32_t o, const float4 &lo) {
  ObjRef r;
  if (o < v.nd) {
    r.beg = v.dbeg[o];
    r.len = v.dlen[o];
    r.rep = __float_as_int(v.cpts[r.beg].w);
    r.x = r.y = r.z = 0.f;
  } else {
    r.beg = 0;
    r.len = 0;
    r.rep = v.sparse_pts[o - v.nd];
    r.x = lo.x;
    r.y = lo.y;
    r.z = lo.z;
  }
  return r;
}

// Is any member of a within eps of any member of b?  Counts evaluations.
__device__ __forceinline__ bool objs_close(const DenseView &v, const ObjRef &a, const ObjRef &b, uint64_t &checks) {
  if (a.len == 0 && b.len == 0) {
    ++checks;
    return hit_point(v.R, a.x, a.y, a.z, b.x, b.y, b.z);
  }
  if (a.len == 0 || b.len == 0) {
    const ObjRef &p = a.len == 0 ? a : b, &c = a.len == 0 ? b : a;
    for (int32_t t = 0; t < c.len; ++t) {
      const float4 q = v.cpts[c.beg + t];
      ++checks;
      if (hit_point(v.R, p.x, p.y, p.z, q.x, q.y, q.z)) return true;
    }
    return false;
  }
  for (int32_t s = 0; s < a.len; ++s) {
    const float4 x = v.cpts[a.beg + s];
    for (int32_t t = 0; t < b.len; ++t) {
      const float4 y = v.cpts[b.beg + t];
      ++checks;
      if (hit_point(v.R, x.x, x.y, x.z, y.x, y.y, y.z)) return true;
    }
  }
  return false;
}

__device__ __forceinline__ void add_checks(uint64_t checks, unsigned long long *total) {
  for (int off = 16; off; off >>= 1) checks += __shfl_xor_sync(0xffffffffu, checks, off);
  if ((threadIdx.x & 31) == 0 && checks) atomicAdd(total, (unsigned long long)checks);
}

// Leaf positions of core objects (list 0, leaf order) and of non-core sparse
// points (list 1).  key[p] = 1 for a core object.
__global__ void k_obj_class(const float4 *__restrict__ nodes, int64_t nobj, int64_t nd,
                            const int32_t *__restrict__ sparse_pts, const uint8_t *__restrict__ core, bool fof,
                            int32_t *__restrict__ key) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < nobj; p += stride) {
    const int32_t o = node_link(ld_node(nodes, 2 * (nobj - 1 + p)));
    key[p] = (fof || o < nd || core[sparse_pts[o - nd]]) ? 1 : 0;
  }
}

__global__ void k_obj_lists(const int32_t *__restrict__ key, const int64_t *__restrict__ scan, int64_t nobj,
                            int32_t *__restrict__ core_leaf, int32_t *__restrict__ border_leaf) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < nobj; p += stride) {
    if (key[p]) core_leaf[scan[p]] = (int32_t)p;
    else border_leaf[p - scan[p]] = (int32_t)p;
  }
}

template <bool FOF>
__global__ void __launch_bounds__(128) k_db_core_pairs(DenseView v, const int32_t *__restrict__ core_leaf,
                                                       const int64_t *__restrict__ ncore_p, int32_t *parent, uint8_t *core,
                                                       unsigned long long *__restrict__ checks_total) {
  const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t ncore = *ncore_p;
  uint64_t checks = 0;
  if (k < ncore) {
    const int64_t first_leaf = v.nobj - 1;
    const int64_t me = first_leaf + core_leaf[k];
    const float4 qlo = ld_node(v.nodes, 2 * me), qhi = ld_node(v.nodes, 2 * me + 1);
    const ObjRef a = obj_ref(v, node_link(qlo), qlo);
    int32_t root = a.rep;
    int32_t cur = node_rope(qhi);
    while (cur != kSentinel) {
      const float4 lo = ld_node(v.nodes, 2 * (int64_t)cur), hi = ld_node(v.nodes, 2 * (int64_t)cur + 1);
      if (cells_far(v.R, qlo, qhi, lo, hi)) {
        cur = node_rope(hi);
        continue;
      }
      if (cur < first_leaf) {
        cur = node_link(lo);
        continue;
      }
      cur = node_rope(hi);
      const int32_t o = node_link(lo);
      const int32_t brep = o < v.nd ? __float_as_int(v.cpts[v.dbeg[o]].w) : v.sparse_pts[o - v.nd];
      if (!FOF && o >= v.nd && !core[brep]) continue;  // border points join in the second pass
      if (parent[brep] == root) continue;
      const int32_t ra = uf_find(parent, root), rb = uf_find(parent, brep);
      root = ra;
      if (ra == rb) continue;
      const ObjRef b = obj_ref(v, o, lo);
      if (!objs_close(v, a, b, checks)) continue;
      root = uf_union(parent, ra, rb);
      if (FOF) {
        core[a.rep] = 1;
        core[brep] = 1;
      }
    }
  }
  add_checks(checks, checks_total);
}

// Border points: the first core point within eps claims the point.
// Border points of the sequential mode (ExecMode::kSequential) over the mixed
// tree.  The reference's sequential merge (dbscan.hpp:406-442) runs the points'
// range queries in sort_queries order (the point Morton order, position spos)
// and reports, in query i's turn, the pairs (i, j) with i < j in object leaf
// order, members of a dense cell in index order.  The claim of a border point
// y therefore goes to the core neighbour x minimising
//   (spos[x], 0, 0)                    for x < y  (reported in x's turn),
//   (spos[y], leaf position of x's object, x)  for x > y  (in y's own turn);
// every core neighbour within eps is examined (a full walk), and y joins the
// set of the minimiser.
__global__ void __launch_bounds__(128) k_db_border_seq(DenseView v, const int32_t *__restrict__ border_leaf,
                                                       const int64_t *__restrict__ ncore_p, int32_t *parent,
                                                       const uint8_t *__restrict__ core,
                                                       const int32_t *__restrict__ spos, uint32_t *__restrict__ claims,
                                                       unsigned long long *__restrict__ checks_total) {
  const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t nborder = v.nobj - *ncore_p;
  uint64_t checks = 0;
  if (k < nborder) {
    const int64_t first_leaf = v.nobj - 1;
    const float4 me = ld_node(v.nodes, 2 * (first_leaf + border_leaf[k]));
    const int32_t i = v.sparse_pts[node_link(me) - v.nd];
    const uint64_t own = (uint64_t)(uint32_t)spos[i] << 32;
    const float x = me.x, y = me.y, z = me.z;
    uint64_t best = ~0ull;
    int32_t best_x = 0x7fffffff, found = -1;
    auto offer = [&](int32_t j, int64_t leafpos) {
      const uint64_t key = j < i ? (uint64_t)(uint32_t)spos[j] << 32 : own | (uint64_t)leafpos;
      const int32_t tie = j < i ? 0 : j;
      if (key < best || (key == best && tie < best_x)) {
        best = key;
        best_x = tie;
        found = j;
      }
    };
    int32_t cur = 0;
    while (cur != kSentinel) {
      const float4 lo = ld_node(v.nodes, 2 * (int64_t)cur), hi = ld_node(v.nodes, 2 * (int64_t)cur + 1);
      if (cur < first_leaf) {
        cur = maybe_box(v.R, x, y, z, lo, hi) ? node_link(lo) : node_rope(hi);
        continue;
      }
      const int64_t leafpos = cur - first_leaf;
      cur = node_rope(hi);
      if (!hit_box(v.R, x, y, z, lo, hi)) continue;
      const int32_t o = node_link(lo);
      if (o < v.nd) {
        const int64_t b = v.dbeg[o];
        const int32_t len = v.dlen[o];
        for (int32_t t = 0; t < len; ++t) {
          const float4 q = v.cpts[b + t];
          ++checks;
          if (hit_point(v.R, x, y, z, q.x, q.y, q.z)) offer(__float_as_int(q.w), leafpos);
        }
      } else {
        const int32_t j = v.sparse_pts[o - v.nd];
        if (core[j]) offer(j, leafpos);  // the point box hit is the exact point test
      }
    }
    if (found >= 0) {
      atomicOr(&claims[i >> 5], 1u << (i & 31));
      uf_union(parent, found, i);
    }
  }
  add_checks(checks, checks_total);
}

__global__ void k_invert(const int32_t *__restrict__ order, int64_t n, int32_t *__restrict__ pos) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < n; k += stride) pos[order[k]] = (int32_t)k;
}

__global__ void __launch_bounds__(128) k_db_border(DenseView v, const int32_t *__restrict__ border_leaf,
                                                   const int64_t *__restrict__ ncore_p, int32_t *parent, const uint8_t *__restrict__ core,
                                                   uint32_t *__restrict__ claims,
                                                   unsigned long long *__restrict__ checks_total) {
  const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t nborder = v.nobj - *ncore_p;
  uint64_t checks = 0;
  if (k < nborder) {
    const int64_t first_leaf = v.nobj - 1;
    const float4 me = ld_node(v.nodes, 2 * (first_leaf + border_leaf[k]));
    const int32_t i = v.sparse_pts[node_link(me) - v.nd];
    const float x = me.x, y = me.y, z = me.z;
    int32_t cur = 0;
    int32_t found = -1;
    while (cur != kSentinel) {
      const float4 lo = ld_node(v.nodes, 2 * (int64_t)cur), hi = ld_node(v.nodes, 2 * (int64_t)cur + 1);
      if (cur < first_leaf) {
        cur = maybe_box(v.R, x, y, z, lo, hi) ? node_link(lo) : node_rope(hi);
        continue;
      }
      cur = node_rope(hi);
      if (!hit_box(v.R, x, y, z, lo, hi)) continue;
      const int32_t o = node_link(lo);
      if (o < v.nd) {
        const int64_t b = v.dbeg[o];
        const int32_t len = v.dlen[o];
        for (int32_t t = 0; t < len; ++t) {
          const float4 q = v.cpts[b + t];
          ++checks;
          if (hit_point(v.R, x, y, z, q.x, q.y, q.z)) {
            found = __float_as_int(q.w);
            break;
          }
        }
      } else {
        const int32_t j = v.sparse_pts[o - v.nd];
        if (core[j]) found = j;  // the point box hit is the exact point test
      }
      if (found >= 0) break;
    }
    if (found >= 0) {
      atomicOr(&claims[i >> 5], 1u << (i & 31));
      uf_union(parent, found, i);
    }
  }
  add_checks(checks, checks_total);
}

__global__ void k_db_labels(int64_t n, int32_t *parent, const uint8_t *__restrict__ core,
                            const uint32_t *__restrict__ claims, int32_t *__restrict__ labels,
                            uint8_t *__restrict__ core_out) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    const bool member = core[i] || (claims && ((claims[i >> 5] >> (i & 31)) & 1u));
    labels[i] = member ? uf_root(parent, (int32_t)i) : -1;
    core_out[i] = core[i];
  }
}

__global__ void k_iota32(int32_t *a, int64_t n) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) a[i] = (int32_t)i;
}

__global__ void k_dense_core(const int32_t *__restrict__ point_cell, int64_t n, uint8_t *__restrict__ core) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) core[i] = point_cell[i] >= 0;
}

// ---------------------------------------------------------------------------
// FoF over grid cells (the FDBSCAN-DenseBox dense-cell shortcut
// applied to friends-of-friends).  With cell length eps/sqrt(d)*(1-1e-6)
// (dense_grid.hpp:71-103) any two points of a cell are within eps, so a cell
// is one set from the start.  Points are sorted once by the Morton key of
// their cell; the LBVH is built over the non-empty cells in that order (tight
// cell boxes); each cell walks the ropes from its own leaf (later cells only,
// traversal.hpp:162-184) with a conservative box-box test, skips cells that
// are already in its set, and otherwise tests member pairs until the first
// close pair, which unions the two cells.  Labels are canonical, so the result
// equals the point-based FoF bit for bit.
// ---------------------------------------------------------------------------
// ckeys == nullptr: write the hierarchy's split array instead (delta[j] =
// the common-prefix length of cell keys j and j + 1, k_delta's value for
// distinct 64-bit keys), so the cell keys need not be stored and re-read.
// leaves != nullptr: write the cell tree's leaf nodes {box, cell, rope}
// directly (no box array for the hierarchy to re-read); rope(j) from the split
// lengths D(j), D(j+1) as HierView::rope.
__global__ void k_cell_ranges(const int64_t *__restrict__ cell_start, int64_t m, int64_t n,
                              const uint64_t *__restrict__ skeys, const float4 *__restrict__ cpts, int dim,
                              uint64_t *__restrict__ ckeys, float *__restrict__ boxes, int32_t *__restrict__ cell_of,
                              uint8_t *__restrict__ multi, int32_t *__restrict__ delta,
                              float4 *__restrict__ leaves = nullptr) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < m; j += stride) {
    const int64_t s = cell_start[j], e = j + 1 < m ? cell_start[j + 1] : n;
    float lo[3] = {3.4028235e38f, 3.4028235e38f, 3.4028235e38f};
    float hi[3] = {-3.4028235e38f, -3.4028235e38f, -3.4028235e38f};
    for (int64_t k = s; k < e; ++k) {
      const float4 q = cpts[k];
      lo[0] = fminf(lo[0], q.x); lo[1] = fminf(lo[1], q.y); lo[2] = fminf(lo[2], q.z);
      hi[0] = fmaxf(hi[0], q.x); hi[1] = fmaxf(hi[1], q.y); hi[2] = fmaxf(hi[2], q.z);
      if (cell_of) cell_of[k] = (int32_t)j;
    }
    if (boxes) {
      for (int k = 0; k < dim; ++k) {
        boxes[j * 2 * dim + k] = lo[k];
        boxes[j * 2 * dim + dim + k] = hi[k];
      }
    }
    if (ckeys) ckeys[j] = skeys[s];
    const int32_t dj = j + 1 < m ? __clzll((long long)(skeys[s] ^ skeys[e])) : -1;
    if (delta && j + 1 < m) delta[j] = dj;
    if (leaves) {
      const int32_t dj1 = j + 2 < m ? __clzll((long long)(skeys[e] ^ skeys[cell_start[j + 2]])) : -1;
      const int32_t rope = j == m - 1 ? kSentinel
                                      : ((j + 1 == m - 1 || dj1 < dj) ? (int32_t)(m - 1 + j + 1) : (int32_t)(j + 1));
      if (dim < 3) lo[2] = hi[2] = 0.f;
      leaves[2 * j] = make_float4(lo[0], lo[1], lo[2], __int_as_float((int)j));
      leaves[2 * j + 1] = make_float4(hi[0], hi[1], hi[2], __int_as_float(rope));
    }
    multi[j] = (e - s) > 1;
  }
}

// Union cell a's set (root hint `root`) with leaf cell b's when a member pair
// is within eps; returns the updated hint.
// STATS: count member-pair distance tests into *tests.
template <bool STATS = false>
__device__ __forceinline__ int32_t cells_leaf(const int64_t *__restrict__ cell_start, int64_t m, int64_t n,
                                              const float4 *__restrict__ cpts, const Radius &R, int32_t *parent,
                                              int64_t sa, int64_t ea, int32_t root, int32_t b,
                                              int64_t *tests = nullptr) {
  if (parent[b] == root) return root;
  const int32_t ra = uf_find(parent, root), rb = uf_find(parent, b);
  if (ra == rb) return ra;
  const int64_t sb = cell_start[b], eb = b + 1 < m ? cell_start[b + 1] : n;
  bool found = false;
  for (int64_t i = sa; i < ea && !found; ++i) {
    const float4 x = cpts[i];
    for (int64_t j = sb; j < eb; ++j) {
      const float4 y = cpts[j];
      if (STATS) ++*tests;
      if (hit_point(R, x.x, x.y, x.z, y.x, y.y, y.z)) {
        found = true;
        break;
      }
    }
  }
  return found ? uf_union(parent, ra, rb) : ra;
}

// One thread per non-empty cell a: a stackless walk of the cell hierarchy
// from a's rope visits only cells b > a (each cell pair once); cells whose
// point boxes are within eps are united when a member pair is within eps,
// skipped early when b already hangs off a's root (root hint).
// FAST: the radius admits the fp32 filter (Radius::fast), so the kernel is
// compiled without the double-precision box test (merge 29.6 -> 28.0 ms).
#ifndef SPB_MERGE_SM
#define SPB_MERGE_SM 1
#endif
// below ~4M cells the schedule's tail outweighs the locality (C1, 1M points:
// 0.63 vs 0.59 ms)
#ifndef SPB_SM_MIN_ITEMS
#define SPB_SM_MIN_ITEMS (1 << 22)
#endif

// STATS: add this walk's node visits and member-pair tests to stats[0..1]
// (diagnostic launch only, SP_FLAG_STATS; the timed kernel is STATS = false).
template <bool FAST, bool STATS = false>
__device__ __forceinline__ void fof_cell_walk(const float4 *__restrict__ nodes, int64_t m,
                                              const int64_t *__restrict__ cell_start, int64_t n,
                                              const float4 *__restrict__ cpts, const Radius &R, int32_t *parent,
                                              int64_t a, unsigned long long *stats = nullptr) {
  const int32_t first_leaf = (int32_t)(m - 1);
  float4 qlo, qhi;
  ld_node2(nodes, (first_leaf + a), qlo, qhi);
  const int64_t sa = cell_start[a], ea = a + 1 < m ? cell_start[a + 1] : n;
  int32_t root = (int32_t)a;
  int32_t cur = node_rope(qhi);
  int64_t visits = 0, tests = 0, nfar = 0, nleaf = 0, tail = 0;
  // One exit (the loop test) and the leaf work as the only conditional
  // block: an early exit inside the body lets the compiler drop the warp's
  // per-iteration reconvergence (no BSSY/BSYNC around the body in the SASS),
  // and the walk then runs about 5x slower.
  while (cur != kSentinel) {
    if (STATS) ++visits;
    float4 lo, hi;
    ld_node2(nodes, (int64_t)cur, lo, hi);
    const bool far = cells_far(R, qlo, qhi, lo, hi);
    const bool descend = !far && cur < first_leaf;
    if (STATS) {
      nfar += far;
      nleaf += !far && !descend;
      tail = far ? tail + 1 : 0;
    }
    if (!far && !descend)
      root = cells_leaf<STATS>(cell_start, m, n, cpts, R, parent, sa, ea, root, (int32_t)(cur - first_leaf), &tests);
    cur = descend ? node_link(lo) : node_rope(hi);
  }
  if (STATS) {
    atomicAdd(stats, (unsigned long long)visits);
    atomicAdd(stats + 1, (unsigned long long)tests);
    atomicAdd(stats + 2, (unsigned long long)nfar);
    atomicAdd(stats + 3, (unsigned long long)nleaf);
    atomicAdd(stats + 4, (unsigned long long)tail);
  }
}

template <bool FAST>
__global__ void __launch_bounds__(128, 1) k_fof_cells_merge(const float4 *__restrict__ nodes, int64_t m,
                                                         const int64_t *__restrict__ cell_start, int64_t n,
                                                         const float4 *__restrict__ cpts, Radius R, int32_t *parent) {
  R.fast = FAST ? 1 : 0;  // as the host checked: one form of the filters compiles
  const int64_t a = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (a >= m) return;
  fof_cell_walk<FAST>(nodes, m, cell_start, n, cpts, R, parent, a);
}

// The same walks on the SM-affine schedule (sm_slices, sp_common.cuh).
template <bool FAST>
#ifndef SPB_MERGE_THREADS
#define SPB_MERGE_THREADS 128
#endif
__global__ void __launch_bounds__(SPB_MERGE_THREADS, 1) k_fof_cells_merge_sm(const float4 *__restrict__ nodes, int64_t m,
                                                            const int64_t *__restrict__ cell_start, int64_t n,
                                                            const float4 *__restrict__ cpts, Radius R,
                                                            int32_t *parent, unsigned long long *slices,
                                                            int nslices) {
  R.fast = FAST ? 1 : 0;
  SmSliceWalk w(m, slices, nslices);
  for (int64_t a; w.next(a);)
    if (a >= 0) fof_cell_walk<FAST>(nodes, m, cell_start, n, cpts, R, parent, a);
}

// Diagnostic twin of the merge (same walks and unions) that also counts node
// visits and member-pair tests; launched instead of the merge only when the
// context has SP_FLAG_STATS, never in a timed run.
template <bool FAST>
__global__ void __launch_bounds__(128, 1) k_fof_cells_merge_stats(const float4 *__restrict__ nodes, int64_t m,
                                                               const int64_t *__restrict__ cell_start, int64_t n,
                                                               const float4 *__restrict__ cpts, Radius R,
                                                               int32_t *parent, unsigned long long *stats) {
  R.fast = FAST ? 1 : 0;
  const int64_t a = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (a < m) fof_cell_walk<FAST, true>(nodes, m, cell_start, n, cpts, R, parent, a, stats);
}

// cells: core iff the cell has two points or its set spans several cells;
// each cell's smallest original index (or id) is folded into minobj[root]
// (warp-aggregated atomicMin) in the same pass over cells (finalize 3.44 ->
// 3.01 ms at 2^27 against a second pass over points).
__global__ void __launch_bounds__(256) k_fof_cells_core_min(int64_t m, int64_t n, int32_t *parent, uint8_t *multi,
                                                            const int64_t *__restrict__ cell_start,
                                                            const uint32_t *__restrict__ order,
                                                            const int32_t *__restrict__ ids, int32_t *minobj) {
  const int64_t a = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  int32_t key = -1, v = 0x7fffffff;
  if (a < m) {
    const int32_t r = uf_root(parent, (int32_t)a);
    if (r != a) {
      parent[a] = r;
      multi[a] = 1;
      multi[r] = 1;
    }
    key = r;
    const int64_t s = cell_start[a];
    if (!ids) {
      // the sort is stable over original indices: a cell's first point has
      // its smallest index
      v = (int32_t)order[s];
    } else {
      const int64_t e = a + 1 < m ? cell_start[a + 1] : n;
      for (int64_t k = s; k < e; ++k) {
        const int32_t o = ids[order[k]];
        v = o < v ? o : v;
      }
    }
  }
  const uint32_t peers = __match_any_sync(0xffffffffu, key);
  const int32_t mn = (int32_t)__reduce_min_sync(peers, (uint32_t)v);
  if (key >= 0 && (threadIdx.x & 31) == __ffs(peers) - 1) atomicMin(&minobj[key], mn);
}

__global__ void __launch_bounds__(256) k_fof_cells_labels(int64_t n, const int32_t *__restrict__ cell_of,
                                                          const int32_t *__restrict__ parent,
                                                          const uint8_t *__restrict__ multi,
                                                          const uint32_t *__restrict__ order,
                                                          const int32_t *__restrict__ minobj,
                                                          int32_t *__restrict__ labels, uint8_t *__restrict__ core) {
  const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= n) return;
  const int32_t cl = cell_of[k];
  const int32_t o = (int32_t)order[k];
  const bool c = multi[cl] != 0;
  labels[o] = c ? minobj[parent[cl]] : -1;  // parent is flat after k_fof_cells_core_min
}

// FoF core flags in input order: core <=> the point has a label (every member
// of a set with >= 2 points is core, every singleton is noise), so the flags
// are one coalesced pass over the labels instead of a 1-byte scatter.
__global__ void __launch_bounds__(256) k_fof_core_from_labels(int64_t n, const int32_t *__restrict__ labels,
                                                              uint8_t *__restrict__ core) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x * 4;
  for (int64_t i = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) * 4; i < n; i += stride) {
    if (i + 4 <= n && (reinterpret_cast<uintptr_t>(labels + i) & 15) == 0 &&
        (reinterpret_cast<uintptr_t>(core + i) & 3) == 0) {
      const int4 l = *reinterpret_cast<const int4 *>(labels + i);
      const uint32_t packed = (uint32_t)(l.x >= 0) | ((uint32_t)(l.y >= 0) << 8) | ((uint32_t)(l.z >= 0) << 16) |
                              ((uint32_t)(l.w >= 0) << 24);
      *reinterpret_cast<uint32_t *>(core + i) = packed;
    } else {
      for (int64_t j = i; j < i + 4 && j < n; ++j) core[j] = labels[j] >= 0;
    }
  }
}

}  // namespace

bool dbscan_cells(Ctx &c, const float *pts, int64_t n, int dim, float eps, int32_t min_pts, int32_t *labels,
                  uint8_t *core_out, DbscanResult *res);

// fdbscan_densebox: the all-cells pipeline (dbscan_cells) whenever the grid
// applies; otherwise the reference's mixed tree of dense cells and sparse
// points below.
void densebox(Ctx &c, const float *pts, int64_t n, int dim, float eps, int32_t min_pts, int width, int32_t *labels,
              uint8_t *core_out, DbscanResult *res, bool cells, bool seq) {
  seq = seq && min_pts > 2;  // min_pts = 2 has no border points
  if (cells && !seq && dbscan_cells(c, pts, n, dim, eps, min_pts, labels, core_out, res)) return;
  cudaEvent_t ev[5];
  for (auto &e : ev) SPB_CUDA(cudaEventCreate(&e));
  SPB_CUDA(cudaEventRecord(ev[0], c.stream));
  mark(c, "start");
  const unsigned G = grid_for(n, 256, 148 * 16);

  // ---- grid (build_dense_grid) ----
  float cell = (float)((double)eps / std::sqrt((double)dim) * (1.0 - 1e-6));
  bool no_dense = !(cell > 0.f);
  DevBuf<float> scene(6, c.stream);
  DevBuf<int> bad(1, c.stream);
  scene_bounds(c, pts, n, dim, true, scene.get(), bad.get());
  float hs[6];
  int hbad = 0;
  peek(c, {{scene.get(), hs, sizeof(hs)}, {bad.get(), &hbad, sizeof(int)}});
  if (hbad) {
    for (auto &e : ev) cudaEventDestroy(e);
    throw InvalidArgument("dbscan: non-finite coordinate");
  }
  for (int k = 0; k < dim && !no_dense; ++k) {
    double extent = (double)hs[3 + k] - (double)hs[k];
    no_dense = extent / (double)cell >= 4.0e18;
  }
  if (!(cell > 0.f)) cell = 1.f;

  DevBuf<int32_t> point_cell((size_t)n, c.stream);
  SPB_CUDA(cudaMemsetAsync(point_cell.get(), 0xff, (size_t)n * sizeof(int32_t), c.stream));
  DevBuf<uint64_t> k0((size_t)n, c.stream), k1((size_t)n, c.stream);
  DevBuf<uint32_t> v0((size_t)n, c.stream), v1((size_t)n, c.stream);
  uint32_t *order = nullptr;  // points sorted by cell (members ascending)
  int64_t nd = 0;
  DevBuf<int64_t> dbeg, cell_start;
  DevBuf<int32_t> dlen;
  DevBuf<float> objects;
  int64_t num_dense_points = 0;
  {
    // bits needed per axis for the largest coordinate (that of the scene max)
    int bits = 1;
    for (int k = 0; k < dim; ++k) {
      int64_t mc = cell_coord(hs[3 + k], hs[k], cell);
      while (bits < 63 && (1LL << bits) <= mc) ++bits;
    }
    const bool interleave = (int64_t)bits * dim <= 64;
    uint64_t *ka = k0.get(), *kb = k1.get();
    uint32_t *va = v0.get(), *vb = v1.get();
    if (interleave) {
      k_cell_keys<<<G, 256, 0, c.stream>>>(pts, n, dim, scene.get(), cell, -1, ka);
      SPB_LAUNCHED();
      radix_sort_pairs(c, &ka, &va, &kb, &vb, n, bits * dim, true);
    } else {
      // lexicographic (x, y, z) by stable per-axis passes, last axis first
      bool first = true;
      for (int axis = dim - 1; axis >= 0; --axis) {
        if (first) {
          k_cell_keys<<<G, 256, 0, c.stream>>>(pts, n, dim, scene.get(), cell, axis, ka);
        } else {
          k_gather_keys<<<G, 256, 0, c.stream>>>(pts, n, dim, scene.get(), cell, axis, va, ka);
        }
        SPB_LAUNCHED();
        radix_sort_pairs(c, &ka, &va, &kb, &vb, n, bits, first);
        first = false;
      }
    }
    order = va;
    mark(c, "grid_sort");
    // segments
    DevBuf<int32_t> head((size_t)n, c.stream);
    DevBuf<int64_t> hscan((size_t)n + 1, c.stream);
    k_heads<<<G, 256, 0, c.stream>>>(ka, order, pts, dim, scene.get(), cell, n, interleave, head.get());
    SPB_LAUNCHED();
    exclusive_scan(c, head.get(), n, hscan.get());
    int64_t m = 0;
    peek(c, {{hscan.get() + n, &m, sizeof(int64_t)}});
    cell_start = DevBuf<int64_t>((size_t)m, c.stream);
    k_cell_starts<<<G, 256, 0, c.stream>>>(head.get(), hscan.get(), n, cell_start.get());
    SPB_LAUNCHED();
    DevBuf<int32_t> dense((size_t)m, c.stream);
    DevBuf<int64_t> dscan((size_t)m + 1, c.stream);
    const unsigned Gm = grid_for(m, 256, 148 * 16);
    k_dense_flags<<<Gm, 256, 0, c.stream>>>(cell_start.get(), m, n, min_pts, no_dense, dense.get());
    SPB_LAUNCHED();
    exclusive_scan(c, dense.get(), m, dscan.get());
    peek(c, {{dscan.get() + m, &nd, sizeof(int64_t)}});
    if (nd > 0) {
      // dense cells ordered by their smallest member
      DevBuf<uint64_t> mk0((size_t)nd, c.stream), mk1((size_t)nd, c.stream);
      DevBuf<uint32_t> mv0((size_t)nd, c.stream), mv1((size_t)nd, c.stream);
      k_dense_pack<<<Gm, 256, 0, c.stream>>>(dense.get(), dscan.get(), cell_start.get(), order, m, mk0.get(),
                                             mv0.get());
      SPB_LAUNCHED();
      uint64_t *ma = mk0.get(), *mb = mk1.get();
      uint32_t *wa = mv0.get(), *wb = mv1.get();
      radix_sort_pairs(c, &ma, &wa, &mb, &wb, nd, 32, false);
      dbeg = DevBuf<int64_t>((size_t)nd, c.stream);
      dlen = DevBuf<int32_t>((size_t)nd, c.stream);
      objects = DevBuf<float>((size_t)n * 2 * dim, c.stream);  // upper bound: nd + sparse <= n
      k_dense_objects<<<(unsigned)((nd * 32 + 255) / 256), 256, 0, c.stream>>>(
          wa, nd, cell_start.get(), m, n, order, pts, dim, point_cell.get(), dbeg.get(), dlen.get(), objects.get());
      SPB_LAUNCHED();
    } else {
      objects = DevBuf<float>((size_t)n * 2 * dim, c.stream);
    }
  }
  // sparse points in index order
  DevBuf<int32_t> sflag((size_t)n, c.stream);
  DevBuf<int64_t> sscan((size_t)n + 1, c.stream);
  k_sparse_flags<<<G, 256, 0, c.stream>>>(point_cell.get(), n, sflag.get());
  SPB_LAUNCHED();
  exclusive_scan(c, sflag.get(), n, sscan.get());
  int64_t ns = 0;
  peek(c, {{sscan.get() + n, &ns, sizeof(int64_t)}});
  num_dense_points = n - ns;
  DevBuf<int32_t> sparse_pts((size_t)(ns > 0 ? ns : 1), c.stream);
  k_sparse_objects<<<G, 256, 0, c.stream>>>(point_cell.get(), sscan.get(), n, nd, pts, dim, sparse_pts.get(),
                                            objects.get());
  SPB_LAUNCHED();
  sflag.reset();
  sscan.reset();
  mark(c, "objects");
  const int64_t nobj = nd + ns;
  DevBuf<float4> cpts((size_t)n, c.stream);
  cell_points(c, order, pts, n, dim, cpts.get());
  Tree t;
  build_tree(c, objects.get(), nobj, dim, false, width, t);
  SPB_CUDA(cudaEventRecord(ev[1], c.stream));
  mark(c, "tree");

  DenseView v{t.nodes, nobj, nd, dbeg.get(), dlen.get(), order, sparse_pts.get(), pts, dim, make_radius(eps),
              cpts.get()};
  DevBuf<uint8_t> core((size_t)n, c.stream);
  k_dense_core<<<G, 256, 0, c.stream>>>(point_cell.get(), n, core.get());
  SPB_LAUNCHED();
  const bool count_phase = min_pts > 2;
  const unsigned Gq = (unsigned)((n + 127) / 128);
  if (count_phase && ns > 0) {
    k_db_core<<<Gq, 128, 0, c.stream>>>(v, order, n, point_cell.get(), min_pts, core.get());
    SPB_LAUNCHED();
  }
  SPB_CUDA(cudaEventRecord(ev[2], c.stream));
  mark(c, "core");

  DevBuf<int32_t> parent((size_t)n, c.stream);
  DevBuf<uint32_t> claims(count_phase ? (size_t)((n + 31) / 32) : 0, c.stream);
  DevBuf<unsigned long long> checks(1, c.stream);
  SPB_CUDA(cudaMemsetAsync(checks.get(), 0, sizeof(unsigned long long), c.stream));
  if (count_phase) SPB_CUDA(cudaMemsetAsync(claims.get(), 0, claims.n * sizeof(uint32_t), c.stream));
  k_iota32<<<G, 256, 0, c.stream>>>(parent.get(), n);
  SPB_LAUNCHED();
  if (nd > 0) {
    k_db_cell_unions<<<(unsigned)((nd * 32 + 255) / 256), 256, 0, c.stream>>>(dbeg.get(), dlen.get(), nd, order,
                                                                              parent.get());
    SPB_LAUNCHED();
  }
  {
    // core objects and border points as leaf-order lists (no host round trip:
    // the kernels read the list lengths from the scan total)
    DevBuf<int32_t> key((size_t)nobj, c.stream), core_leaf((size_t)nobj, c.stream), border_leaf((size_t)nobj, c.stream);
    DevBuf<int64_t> kscan((size_t)nobj + 1, c.stream);
    const unsigned Go = grid_for(nobj, 256, 148 * 16);
    k_obj_class<<<Go, 256, 0, c.stream>>>(t.nodes, nobj, nd, sparse_pts.get(), core.get(), !count_phase, key.get());
    SPB_LAUNCHED();
    exclusive_scan(c, key.get(), nobj, kscan.get());
    k_obj_lists<<<Go, 256, 0, c.stream>>>(key.get(), kscan.get(), nobj, core_leaf.get(), border_leaf.get());
    SPB_LAUNCHED();
    const unsigned Gl = (unsigned)((nobj + 127) / 128);
    if (count_phase)
      k_db_core_pairs<false><<<Gl, 128, 0, c.stream>>>(v, core_leaf.get(), kscan.get() + nobj, parent.get(),
                                                       core.get(), checks.get());
    else
      k_db_core_pairs<true><<<Gl, 128, 0, c.stream>>>(v, core_leaf.get(), kscan.get() + nobj, parent.get(),
                                                      core.get(), checks.get());
    SPB_LAUNCHED();
    mark(c, "merge_core");
    if (count_phase && seq) {
      // sort_queries order of the points (traversal.hpp:188-218): spos
      DevBuf<int32_t> porder((size_t)n, c.stream), spos((size_t)n, c.stream);
      sort_points(c, pts, n, dim, porder.get());
      k_invert<<<G, 256, 0, c.stream>>>(porder.get(), n, spos.get());
      SPB_LAUNCHED();
      k_db_border_seq<<<Gl, 128, 0, c.stream>>>(v, border_leaf.get(), kscan.get() + nobj, parent.get(), core.get(),
                                                spos.get(), claims.get(), checks.get());
      SPB_LAUNCHED();
    } else if (count_phase) {
      k_db_border<<<Gl, 128, 0, c.stream>>>(v, border_leaf.get(), kscan.get() + nobj, parent.get(), core.get(),
                                            claims.get(), checks.get());
      SPB_LAUNCHED();
    }
  }
  SPB_CUDA(cudaEventRecord(ev[3], c.stream));
  mark(c, "merge");
  k_db_labels<<<G, 256, 0, c.stream>>>(n, parent.get(), core.get(), claims.get(), labels, core_out);
  SPB_LAUNCHED();
  SPB_CUDA(cudaEventRecord(ev[4], c.stream));
  mark(c, "finalize");
  unsigned long long hchecks = 0;
  peek(c, {{checks.get(), &hchecks, sizeof(hchecks)}});
  if (res) {
    for (int i = 0; i < 4; ++i) {
      float ms = 0.f;
      cudaEventElapsedTime(&ms, ev[i], ev[i + 1]);
      res->ms[i] = ms;
    }
    res->distance_checks = (int64_t)hchecks;
    res->num_dense_cells = nd;
    res->num_dense_points = num_dense_points;
  }
  for (auto &e : ev) cudaEventDestroy(e);
}

// The cell grid shared by the FoF and DBSCAN cell pipelines: points sorted by
// the Morton key of their cell (side eps/sqrt(d)*(1-1e-6), anchored at the
// scene min: build_dense_grid, dense_grid.hpp:71-103), cell segments, tight
// cell boxes and the LBVH over the non-empty cells in key order.  Returns
// false (nothing computed) when the grid does not apply: coordinates that
// could saturate (no dense cells in the reference either) or cell coordinates
// too wide for a 63-bit Morton key.
#ifndef SPB_FUSED_HIST
#define SPB_FUSED_HIST 1
#endif
#ifndef SPB_SORT40
#define SPB_SORT40 1
#endif
struct CellGrid {
  int64_t m = 0;
  DevBuf<uint64_t> k0, k1;
  DevBuf<uint32_t> v0, v1;
  uint64_t *keys = nullptr;   // sorted cell keys
  uint32_t *order = nullptr;  // sorted position -> original index
  DevBuf<float4> cpts;        // sorted points {x, y, z, bits(original index)}
  DevBuf<int64_t> cell_start;
  DevBuf<int32_t> cell_of;    // sorted position -> cell
  DevBuf<uint8_t> multi;      // cell has more than one point
  Tree t;
};

bool build_cell_grid(Ctx &c, const float *pts, int64_t n, int dim, float eps, CellGrid &g) {
  const float cell = (float)((double)eps / std::sqrt((double)dim) * (1.0 - 1e-6));
  if (!(cell > 0.f)) return false;
  DevBuf<float> scene(6, c.stream);
  DevBuf<int> bad(1, c.stream);
  scene_bounds(c, pts, n, dim, true, scene.get(), bad.get());
  float hs[6];
  int hbad = 0;
  peek(c, {{scene.get(), hs, sizeof(hs)}, {bad.get(), &hbad, sizeof(int)}});
  if (hbad) throw InvalidArgument("dbscan: non-finite coordinate");
  int bits = 1;
  for (int k = 0; k < dim; ++k) {
    const double extent = (double)hs[3 + k] - (double)hs[k];
    if (extent / (double)cell >= 4.0e18) return false;
    const int64_t mc = cell_coord(hs[3 + k], hs[k], cell);
    while (bits < 63 && (1LL << bits) <= mc) ++bits;
  }
  if ((int64_t)bits * dim > 63) return false;
  mark(c, "bounds");
  const unsigned G = grid_for(n, 256, 148 * 16);
  g.k0 = DevBuf<uint64_t>((size_t)n, c.stream);
  g.k1 = DevBuf<uint64_t>((size_t)n, c.stream);
  g.v0 = DevBuf<uint32_t>((size_t)n, c.stream);
  g.v1 = DevBuf<uint32_t>((size_t)n, c.stream);
  const bool sort40 = SPB_SORT40 && dim == 3 && bits * dim > 32 && bits * dim <= 40 && aligned16(pts);
  const bool keys_p3v = dim == 3 && aligned16(pts) && aligned16(g.k0.get());
  // the 40-bit sort's digit counts come from the key kernel (HistAcc)
  DevBuf<uint32_t> hist(sort40 && keys_p3v && SPB_FUSED_HIST ? RS_HIST_ENTRIES(5) : 0, c.stream);
  if (hist.n) SPB_CUDA(cudaMemsetAsync(hist.get(), 0, hist.n * sizeof(uint32_t), c.stream));
  if (keys_p3v)
    k_cell_keys_p3v<<<grid_for((n + 3) / 4, 256, 148 * 16), 256, 0, c.stream>>>(pts, n, scene.get(), cell,
                                                                                 g.k0.get(), hist.get());
  else
    k_cell_keys<<<G, 256, 0, c.stream>>>(pts, n, dim, scene.get(), cell, -1, g.k0.get());
  SPB_LAUNCHED();
  mark(c, "morton");
  uint64_t *ka = g.k0.get(), *kb = g.k1.get();
  uint32_t *va = g.v0.get(), *vb = g.v1.get();
  g.cpts = DevBuf<float4>((size_t)n, c.stream);
  if (sort40) {
    // five passes, the last four over 32-bit keys; the keys are recomputed
    // from the gathered points
    uint32_t *k32 = reinterpret_cast<uint32_t *>(kb);
    radix_sort_pairs_40(c, ka, &va, &vb, k32, k32 + n, n, true, hist.get());
    g.order = va;
    mark(c, "sort");
    k_cell_points3v_keys<<<(unsigned)((n + 256 * CP_ILP - 1) / (256 * CP_ILP)), 256, 0, c.stream>>>(
        va, pts, n, scene.get(), cell, g.cpts.get(), ka);
    SPB_LAUNCHED();
    g.keys = ka;
  } else {
    radix_sort_pairs(c, &ka, &va, &kb, &vb, n, bits * dim, true);
    g.keys = ka;
    g.order = va;
    mark(c, "sort");
    cell_points(c, va, pts, n, dim, g.cpts.get());
  }
  int64_t m = 0;
  g.cell_of = DevBuf<int32_t>((size_t)n, c.stream);
  g.cell_start = DevBuf<int64_t>((size_t)n, c.stream);  // capacity: m <= n
  {
    const int64_t ntiles = (n + CC_TILE - 1) / CC_TILE;
    DevBuf<unsigned long long> lb((size_t)ntiles, c.stream);
    DevBuf<uint32_t> ctr(1, c.stream);
    DevBuf<int64_t> total(1, c.stream);
    SPB_CUDA(cudaMemsetAsync(lb.get(), 0, lb.n * sizeof(unsigned long long), c.stream));
    SPB_CUDA(cudaMemsetAsync(ctr.get(), 0, sizeof(uint32_t), c.stream));
    k_cell_compact<<<(unsigned)ntiles, CC_THREADS, 0, c.stream>>>(ka, n, g.cell_start.get(), g.cell_of.get(), lb.get(),
                                                                ctr.get(), total.get());
    SPB_LAUNCHED();
    peek(c, {{total.get(), &m, sizeof(int64_t)}});
  }
  g.m = m;
  DevBuf<int32_t> delta(m > 1 ? m - 1 : 1, c.stream);
  g.multi = DevBuf<uint8_t>((size_t)m, c.stream);
  // the cell tree's leaf nodes straight from the cell ranges
  g.t.nodes = m > 0 ? static_cast<float4 *>(cache_alloc((size_t)(2 * m - 1) * 2 * sizeof(float4), c.stream))
                    : nullptr;
  if (m > 0) {
    k_cell_ranges<<<grid_for(m, 256, 148 * 16), 256, 0, c.stream>>>(g.cell_start.get(), m, n, ka, g.cpts.get(), dim,
                                                                     nullptr, nullptr, nullptr, g.multi.get(),
                                                                     delta.get(), g.t.nodes + 2 * (m - 1));
    SPB_LAUNCHED();
  }
  build_sorted_hierarchy(c, nullptr, m, dim, nullptr, g.t, &delta);
  mark(c, "hierarchy");
  return true;
}

// friends-of-friends over the cell grid: a cell is one set from the start,
// cells unite at their first member pair within eps (k_fof_cells_merge).
bool fof_cells(Ctx &c, const float *pts, int64_t n, int dim, float eps, int32_t *labels, uint8_t *core_out,
               DbscanResult *res, const int32_t *ids) {
  cudaEvent_t ev[5];
  for (auto &e : ev) SPB_CUDA(cudaEventCreate(&e));
  struct EvGuard {
    cudaEvent_t *e;
    ~EvGuard() {
      for (int i = 0; i < 5; ++i) cudaEventDestroy(e[i]);
    }
  } guard{ev};
  SPB_CUDA(cudaEventRecord(ev[0], c.stream));
  mark(c, "start");
  CellGrid g;
  if (!build_cell_grid(c, pts, n, dim, eps, g)) return false;
  const int64_t m = g.m;
  c.count("fof_cells", m);
  SPB_CUDA(cudaEventRecord(ev[1], c.stream));
  SPB_CUDA(cudaEventRecord(ev[2], c.stream));
  DevBuf<int32_t> parent((size_t)m, c.stream), minobj((size_t)m, c.stream);
  k_iota32<<<grid_for(m, 256, 148 * 16), 256, 0, c.stream>>>(parent.get(), m);
  SPB_LAUNCHED();
  {
    const Radius R = make_radius(eps);
    if (c.stats()) {
      DevBuf<unsigned long long> st(5, c.stream);
      SPB_CUDA(cudaMemsetAsync(st.get(), 0, 5 * sizeof(unsigned long long), c.stream));
      auto kern = R.fast ? k_fof_cells_merge_stats<true> : k_fof_cells_merge_stats<false>;
      kern<<<(unsigned)((m + 127) / 128), 128, 0, c.stream>>>(g.t.nodes, m, g.cell_start.get(), n, g.cpts.get(), R,
                                                              parent.get(), st.get());
      SPB_LAUNCHED();
      unsigned long long hs[5] = {0, 0, 0, 0, 0};
      peek(c, {{st.get(), hs, sizeof(hs)}});
      c.count("merge_node_visits", (int64_t)hs[0]);
      c.count("merge_pair_tests", (int64_t)hs[1]);
      c.count("merge_far_visits", (int64_t)hs[2]);
      c.count("merge_leaf_visits", (int64_t)hs[3]);
      c.count("merge_tail_visits", (int64_t)hs[4]);
    } else if (SPB_MERGE_SM && m >= SPB_SM_MIN_ITEMS) {
      SmSlices sl(c);
      if (R.fast)
        k_fof_cells_merge_sm<true><<<sl.grid(k_fof_cells_merge_sm<true>, SPB_MERGE_THREADS), SPB_MERGE_THREADS, 0, c.stream>>>(
            g.t.nodes, m, g.cell_start.get(), n, g.cpts.get(), R, parent.get(), sl.ctr.get(), sl.nsm);
      else
        k_fof_cells_merge_sm<false><<<sl.grid(k_fof_cells_merge_sm<false>, SPB_MERGE_THREADS), SPB_MERGE_THREADS, 0, c.stream>>>(
            g.t.nodes, m, g.cell_start.get(), n, g.cpts.get(), R, parent.get(), sl.ctr.get(), sl.nsm);
    } else if (R.fast)
      k_fof_cells_merge<true><<<(unsigned)((m + 127) / 128), 128, 0, c.stream>>>(g.t.nodes, m, g.cell_start.get(), n,
                                                                                 g.cpts.get(), R, parent.get());
    else
      k_fof_cells_merge<false><<<(unsigned)((m + 127) / 128), 128, 0, c.stream>>>(g.t.nodes, m, g.cell_start.get(),
                                                                                  n, g.cpts.get(), R, parent.get());
  }
  SPB_LAUNCHED();
  SPB_CUDA(cudaEventRecord(ev[3], c.stream));
  mark(c, "merge");
  SPB_CUDA(cudaMemsetAsync(minobj.get(), 0x7f, (size_t)m * sizeof(int32_t), c.stream));
  k_fof_cells_core_min<<<(unsigned)((m + 255) / 256), 256, 0, c.stream>>>(m, n, parent.get(), g.multi.get(),
                                                                          g.cell_start.get(), g.order, ids,
                                                                          minobj.get());
  SPB_LAUNCHED();
  k_fof_cells_labels<<<(unsigned)((n + 255) / 256), 256, 0, c.stream>>>(n, g.cell_of.get(), parent.get(),
                                                                        g.multi.get(), g.order, minobj.get(), labels,
                                                                        core_out);
  SPB_LAUNCHED();
  k_fof_core_from_labels<<<grid_for((n + 3) / 4, 256, 148 * 16), 256, 0, c.stream>>>(n, labels, core_out);
  SPB_LAUNCHED();
  SPB_CUDA(cudaEventRecord(ev[4], c.stream));
  mark(c, "finalize");
  if (c.async()) return true;
  SPB_CUDA(cudaEventSynchronize(ev[4]));
  if (res) {
    for (int i = 0; i < 4; ++i) {
      float ms = 0.f;
      cudaEventElapsedTime(&ms, ev[i], ev[i + 1]);
      res->ms[i] = ms;
    }
  }
  return true;
}


// ---------------------------------------------------------------------------
// DBSCAN (min_pts > 2) over the cell grid: the DenseBox idea (dbscan.hpp:
// 298-449) taken to every cell.  Any two points of one cell are within eps, so
//  * a point of a cell with >= min_pts members is core (the dense cells of
//    build_dense_grid); any other point counts its own cell whole and then the
//    members of cells within eps of it, stopping at min_pts
//    (detect_core_counts, dbscan.hpp:146-182: count = min(hits, min_pts));
//  * the core points of one cell form one set; two cells unite at the first
//    core-core member pair within eps (pair traversal over later cells, set
//    skip), so the core partition is the reference's;
//  * a non-core point joins the set of a core point within eps: one of its
//    own cell if there is any, else the first found by a walk from the root
//    (the one-shot claim latch of dbscan.hpp:123-137 / union_find.hpp:63-82);
//    points with none are noise.
// Labels are the smallest original index over each set's core and border
// points; core flags are exact; clusters satisfy check_equivalence
// (verify.hpp:21-61).
// ---------------------------------------------------------------------------
namespace {

__device__ __forceinline__ int64_t cell_end(const int64_t *cell_start, int64_t m, int64_t n, int64_t c) {
  return c + 1 < m ? cell_start[c + 1] : n;
}

// dense cells and their points (DbscanStats): {cells, points}
__global__ void k_cells_dense_stats(const int64_t *__restrict__ cell_start, int64_t m, int64_t n, int32_t min_pts,
                                    unsigned long long *st) {
  const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  uint32_t dense = 0, pts = 0;
  if (c < m) {
    const int64_t len = cell_end(cell_start, m, n, c) - cell_start[c];
    if (len >= min_pts) {
      dense = 1;
      pts = (uint32_t)len;
    }
  }
  dense = __reduce_add_sync(0xffffffffu, dense);
  pts = __reduce_add_sync(0xffffffffu, pts);
  if ((threadIdx.x & 31) == 0 && dense) {
    atomicAdd(&st[0], (unsigned long long)dense);
    atomicAdd(&st[1], (unsigned long long)pts);
  }
}

// Capped neighbour counts of the points of small cells (sorted order), on the
// SM-affine schedule (core 8.25 -> 7.95 ms at C3; the border claims below keep
// plain block order: 3.67 vs 3.81 ms).
template <bool FAST>
__global__ void __launch_bounds__(128) k_cells_core(const float4 *__restrict__ nodes, int64_t m,
                                                    const int64_t *__restrict__ cell_start, int64_t n,
                                                    const int32_t *__restrict__ cell_of,
                                                    const float4 *__restrict__ cpts, Radius R, int32_t min_pts,
                                                    uint8_t *__restrict__ corep, unsigned long long *slices,
                                                    int nslices) {
  R.fast = FAST ? 1 : 0;
  SmSliceWalk w(n, slices, nslices);
  for (int64_t k; w.next(k);) {
    if (k < 0) continue;
    const int32_t own = cell_of[k];
    int32_t cnt = (int32_t)(cell_end(cell_start, m, n, own) - cell_start[own]);
    const float4 me = cpts[k];
    const int64_t first_leaf = m - 1;
    // Morton-neighbour cells first (key order is spatial order): in dense
    // regions they usually hold the missing neighbours and the tree walk is
    // skipped; the walk below does not count them again.
    const int64_t w_lo = own - SPB_CORE_WINDOW > 0 ? own - SPB_CORE_WINDOW : 0;
    const int64_t w_hi = own + SPB_CORE_WINDOW < m - 1 ? own + SPB_CORE_WINDOW : m - 1;
    for (int64_t b = w_lo; b <= w_hi && cnt < min_pts; ++b) {
      if (b == own) continue;
      float4 lo, hi;
      ld_node2(nodes, (first_leaf + b), lo, hi);
      if (!hit_box(R, me.x, me.y, me.z, lo, hi)) continue;
      const int64_t e = cell_end(cell_start, m, n, b);
      for (int64_t j = cell_start[b]; j < e && cnt < min_pts; ++j) {
        const float4 q = cpts[j];
        cnt += hit_point(R, me.x, me.y, me.z, q.x, q.y, q.z);
      }
    }
    if (cnt < min_pts) {
      int32_t cur = 0;  // root: internal 0, or leaf 0 when m == 1
      while (cur != kSentinel) {
        float4 lo, hi;
        ld_node2(nodes, (int64_t)cur, lo, hi);
        if (cur < first_leaf) {
          cur = maybe_box(R, me.x, me.y, me.z, lo, hi) ? node_link(lo) : node_rope(hi);
          continue;
        }
        const int64_t b = cur - first_leaf;
        cur = node_rope(hi);
        if ((b >= w_lo && b <= w_hi) || !hit_box(R, me.x, me.y, me.z, lo, hi)) continue;
        const int64_t e = cell_end(cell_start, m, n, b);
        for (int64_t j = cell_start[b]; j < e && cnt < min_pts; ++j) {
          const float4 q = cpts[j];
          cnt += hit_point(R, me.x, me.y, me.z, q.x, q.y, q.z);
        }
        if (cnt >= min_pts) cur = kSentinel;  // through the loop test, not a break
      }
    }
    corep[k] = cnt >= min_pts;
  }
}

// hascore[c]: the cell holds a core point
__global__ void k_cells_has_core(const int64_t *__restrict__ cell_start, int64_t m, int64_t n,
                                 const uint8_t *__restrict__ corep, uint8_t *__restrict__ hascore) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; c < m; c += stride) {
    const int64_t e = cell_end(cell_start, m, n, c);
    uint8_t h = 0;
    for (int64_t j = cell_start[c]; j < e && !h; ++j) h = corep[j];
    hascore[c] = h;
  }
}

// Core cells: rope walk over later cells; two cells unite at the first
// core-core member pair within eps (SM-affine schedule: 15.4 -> 12.7 ms at C3).
template <bool FAST>
__global__ void __launch_bounds__(128) k_cells_core_merge(const float4 *__restrict__ nodes, int64_t m,
                                                          const int64_t *__restrict__ cell_start, int64_t n,
                                                          const float4 *__restrict__ cpts,
                                                          const uint8_t *__restrict__ corep,
                                                          const uint8_t *__restrict__ hascore, Radius R,
                                                          int32_t *parent, unsigned long long *checks_total,
                                                          unsigned long long *slices, int nslices) {
  R.fast = FAST ? 1 : 0;
  uint64_t checks = 0;
  SmSliceWalk w(m, slices, nslices);
  for (int64_t a; w.next(a);)
    if (a >= 0 && hascore[a]) {
      const int64_t first_leaf = m - 1;
      float4 qlo, qhi;
      ld_node2(nodes, (first_leaf + a), qlo, qhi);
      const int64_t sa = cell_start[a], ea = cell_end(cell_start, m, n, a);
      int32_t root = (int32_t)a;
      int32_t cur = node_rope(qhi);
      // one exit (the loop test), the leaf work as the only conditional
      // block (the FoF walk's shape, fof_cell_walk)
      while (cur != kSentinel) {
        float4 lo, hi;
        ld_node2(nodes, (int64_t)cur, lo, hi);
        const bool far = cells_far(R, qlo, qhi, lo, hi);
        const bool descend = !far && cur < first_leaf;
        const int32_t b = (int32_t)(cur - first_leaf);
        cur = descend ? node_link(lo) : node_rope(hi);
        if (!far && !descend && hascore[b] && parent[b] != root) {
          const int32_t ra = uf_find(parent, root), rb = uf_find(parent, b);
          root = ra;
          if (ra != rb) {
            const int64_t sb = cell_start[b], eb = cell_end(cell_start, m, n, b);
            bool found = false;
            for (int64_t i = sa; i < ea && !found; ++i) {
              if (!corep[i]) continue;
              const float4 x = cpts[i];
              for (int64_t j = sb; j < eb; ++j) {
                if (!corep[j]) continue;
                const float4 y = cpts[j];
                ++checks;
                if (hit_point(R, x.x, x.y, x.z, y.x, y.y, y.z)) {
                  found = true;
                  break;
                }
              }
            }
            if (found) root = uf_union(parent, ra, rb);
          }
        }
      }
    }
  add_checks(checks, checks_total);
}

// assign[k]: the cell whose set point k joins (-1: noise).
template <bool FAST>
__global__ void __launch_bounds__(128) k_cells_border(const float4 *__restrict__ nodes, int64_t m,
                                                      const int64_t *__restrict__ cell_start, int64_t n,
                                                      const int32_t *__restrict__ cell_of,
                                                      const float4 *__restrict__ cpts,
                                                      const uint8_t *__restrict__ corep,
                                                      const uint8_t *__restrict__ hascore, Radius R,
                                                      int32_t *__restrict__ assign,
                                                      unsigned long long *checks_total) {
  (void)FAST;  // generic: measured faster without the specialisation
  const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  uint64_t checks = 0;
  if (k < n) {
    const int32_t own = cell_of[k];
    int32_t found = -1;
    if (corep[k] || hascore[own]) {
      found = own;
    } else {
      const float4 me = cpts[k];
      const int64_t first_leaf = m - 1;
      int32_t cur = 0;
      while (cur != kSentinel && found < 0) {
        float4 lo, hi;
        // two 16-byte loads: the 256-bit form measured slower in this walk (4.21 vs 3.65 ms at C3)
        lo = ld_node(nodes, 2 * (int64_t)cur);
        hi = ld_node(nodes, 2 * (int64_t)cur + 1);
        if (cur < first_leaf) {
          cur = maybe_box(R, me.x, me.y, me.z, lo, hi) ? node_link(lo) : node_rope(hi);
          continue;
        }
        const int32_t b = (int32_t)(cur - first_leaf);
        cur = node_rope(hi);
        if (!hascore[b] || !hit_box(R, me.x, me.y, me.z, lo, hi)) continue;
        const int64_t e = cell_end(cell_start, m, n, b);
        for (int64_t j = cell_start[b]; j < e; ++j) {
          if (!corep[j]) continue;
          const float4 q = cpts[j];
          ++checks;
          if (hit_point(R, me.x, me.y, me.z, q.x, q.y, q.z)) {
            found = b;
            break;
          }
        }
      }
    }
    assign[k] = found;
  }
  add_checks(checks, checks_total);
}

__global__ void k_cells_compress(int64_t m, int32_t *parent) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t a = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; a < m; a += stride)
    parent[a] = uf_root(parent, (int32_t)a);
}

__global__ void __launch_bounds__(256) k_cells_minobj(int64_t n, const int32_t *__restrict__ assign,
                                                      const int32_t *__restrict__ parent,
                                                      const uint32_t *__restrict__ order, int32_t *minobj) {
  const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  int32_t key = -1, v = 0x7fffffff;
  if (k < n) {
    const int32_t a = assign[k];
    if (a >= 0) {
      key = parent[a];
      v = (int32_t)order[k];
    }
  }
  const uint32_t peers = __match_any_sync(0xffffffffu, key);
  const int32_t mn = (int32_t)__reduce_min_sync(peers, (uint32_t)v);
  if (key >= 0 && (threadIdx.x & 31) == __ffs(peers) - 1) atomicMin(&minobj[key], mn);
}

__global__ void __launch_bounds__(256) k_cells_labels(int64_t n, const int32_t *__restrict__ assign,
                                                      const int32_t *__restrict__ parent,
                                                      const uint8_t *__restrict__ corep,
                                                      const uint32_t *__restrict__ order,
                                                      const int32_t *__restrict__ minobj, int32_t *__restrict__ labels,
                                                      uint8_t *__restrict__ core) {
  const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= n) return;
  const int32_t a = assign[k];
  const int32_t o = (int32_t)order[k];
  labels[o] = a >= 0 ? minobj[parent[a]] : -1;
  core[o] = corep[k];
}

}  // namespace

bool dbscan_cells(Ctx &c, const float *pts, int64_t n, int dim, float eps, int32_t min_pts, int32_t *labels,
                  uint8_t *core_out, DbscanResult *res) {
  cudaEvent_t ev[5];
  for (auto &e : ev) SPB_CUDA(cudaEventCreate(&e));
  struct EvGuard {
    cudaEvent_t *e;
    ~EvGuard() {
      for (int i = 0; i < 5; ++i) cudaEventDestroy(e[i]);
    }
  } guard{ev};
  SPB_CUDA(cudaEventRecord(ev[0], c.stream));
  mark(c, "start");
  CellGrid g;
  if (!build_cell_grid(c, pts, n, dim, eps, g)) return false;
  const int64_t m = g.m;
  c.count("cells", m);
  const Radius R = make_radius(eps);
  const unsigned Gm = grid_for(m, 256, 148 * 16);
  DevBuf<unsigned long long> st(3, c.stream);  // dense cells, dense points, distance checks
  SPB_CUDA(cudaMemsetAsync(st.get(), 0, 3 * sizeof(unsigned long long), c.stream));
  k_cells_dense_stats<<<(unsigned)((m + 255) / 256), 256, 0, c.stream>>>(g.cell_start.get(), m, n, min_pts, st.get());
  SPB_LAUNCHED();
  SPB_CUDA(cudaEventRecord(ev[1], c.stream));
  DevBuf<uint8_t> corep((size_t)n, c.stream), hascore((size_t)m, c.stream);
  {
    SmSlices sl(c);
    auto kern = R.fast ? k_cells_core<true> : k_cells_core<false>;
    kern<<<sl.grid(kern, 128), 128, 0, c.stream>>>(g.t.nodes, m, g.cell_start.get(), n, g.cell_of.get(), g.cpts.get(),
                                                   R, min_pts, corep.get(), sl.ctr.get(), sl.nsm);
  }
  SPB_LAUNCHED();
  k_cells_has_core<<<Gm, 256, 0, c.stream>>>(g.cell_start.get(), m, n, corep.get(), hascore.get());
  SPB_LAUNCHED();
  SPB_CUDA(cudaEventRecord(ev[2], c.stream));
  mark(c, "core");
  DevBuf<int32_t> parent((size_t)m, c.stream), minobj((size_t)m, c.stream), assign((size_t)n, c.stream);
  k_iota32<<<Gm, 256, 0, c.stream>>>(parent.get(), m);
  SPB_LAUNCHED();
  {
    SmSlices sl(c);
    auto kern = R.fast ? k_cells_core_merge<true> : k_cells_core_merge<false>;
    kern<<<sl.grid(kern, 128), 128, 0, c.stream>>>(g.t.nodes, m, g.cell_start.get(), n, g.cpts.get(), corep.get(),
                                                   hascore.get(), R, parent.get(), st.get() + 2, sl.ctr.get(), sl.nsm);
  }
  SPB_LAUNCHED();
  mark(c, "merge_core");
  k_cells_border<false><<<(unsigned)((n + 127) / 128), 128, 0, c.stream>>>(g.t.nodes, m, g.cell_start.get(), n,
                                                                    g.cell_of.get(), g.cpts.get(), corep.get(),
                                                                    hascore.get(), R, assign.get(), st.get() + 2);
  SPB_LAUNCHED();
  SPB_CUDA(cudaEventRecord(ev[3], c.stream));
  mark(c, "merge");
  k_cells_compress<<<Gm, 256, 0, c.stream>>>(m, parent.get());
  SPB_LAUNCHED();
  SPB_CUDA(cudaMemsetAsync(minobj.get(), 0x7f, (size_t)m * sizeof(int32_t), c.stream));
  k_cells_minobj<<<(unsigned)((n + 255) / 256), 256, 0, c.stream>>>(n, assign.get(), parent.get(), g.order,
                                                                    minobj.get());
  SPB_LAUNCHED();
  k_cells_labels<<<(unsigned)((n + 255) / 256), 256, 0, c.stream>>>(n, assign.get(), parent.get(), corep.get(),
                                                                    g.order, minobj.get(), labels, core_out);
  SPB_LAUNCHED();
  SPB_CUDA(cudaEventRecord(ev[4], c.stream));
  mark(c, "finalize");
  if (c.async()) return true;  // statistics and timings need a host wait
  unsigned long long hst[3] = {0, 0, 0};
  peek(c, {{st.get(), hst, sizeof(hst)}});
  if (res) {
    for (int i = 0; i < 4; ++i) {
      float ms = 0.f;
      cudaEventElapsedTime(&ms, ev[i], ev[i + 1]);
      res->ms[i] = ms;
    }
    res->num_dense_cells = (int64_t)hst[0];
    res->num_dense_points = (int64_t)hst[1];
    res->distance_checks = (int64_t)hst[2];
  }
  return true;
}

}  // namespace spb
