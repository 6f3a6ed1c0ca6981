// Hierarchy construction on sm_100a: scene bounds (K1), Morton codes (K2), a
// stable onesweep LSD radix sort (K3) and a single bottom-up Apetrei pass that
// emits the reference's Karras-numbered nodes, exact union boxes and ropes in
// one sweep (K4).  Reference: Bvh<D>::build, bvh.hpp:100-261; morton.hpp:17-121.
#include <cuda_runtime.h>
#include <stdint.h>

#include <cstring>

#include <algorithm>
#include <climits>
#include <mutex>
#include <cstdlib>

#include "sp_common.cuh"
#include "sp_internal.hpp"

namespace spb {

thread_local int64_t *g_launch_counter = nullptr;

void mark(Ctx &c, const char *name) {
  if (c.marks_used == c.event_pool.size()) {
    cudaEvent_t e;
    SPB_CUDA(cudaEventCreate(&e));
    c.event_pool.push_back(e);
    c.mark_names.push_back(nullptr);
  }
  c.mark_names[c.marks_used] = name;
  SPB_CUDA(cudaEventRecord(c.event_pool[c.marks_used], c.stream));
  ++c.marks_used;
}

namespace {
struct PeekArgs {
  const uint8_t *src[8];
  uint32_t off[8];
  uint32_t bytes[8];
  int k;
};
__global__ void k_peek(PeekArgs a, uint8_t *dst) {
  for (int i = 0; i < a.k; ++i)
    for (uint32_t b = threadIdx.x; b < a.bytes[i]; b += blockDim.x) dst[a.off[i] + b] = a.src[i][b];
}
}  // namespace

void peek(Ctx &c, std::initializer_list<PeekItem> items) {
  if (!c.peek_buf) SPB_CUDA(cudaHostAlloc((void **)&c.peek_buf, 1024, cudaHostAllocMapped | cudaHostAllocPortable));
  PeekArgs a{};
  uint32_t off = 0;
  for (const PeekItem &it : items) {
    if (a.k == 8 || it.bytes > 64) throw CudaError("peek: too many or too large items");
    a.src[a.k] = static_cast<const uint8_t *>(it.src);
    a.off[a.k] = off;
    a.bytes[a.k] = it.bytes;
    off += (it.bytes + 7) & ~7u;
    ++a.k;
  }
  k_peek<<<1, 64, 0, c.stream>>>(a, c.peek_buf);
  SPB_LAUNCHED();
  SPB_CUDA(cudaStreamSynchronize(c.stream));
  off = 0;
  for (const PeekItem &it : items) {
    memcpy(it.dst, c.peek_buf + off, it.bytes);
    off += (it.bytes + 7) & ~7u;
  }
}

void reset_marks(Ctx &c) {
  c.marks_used = 0;
  c.phases.clear();
}

void resolve_marks(Ctx &c) {
  c.phases.clear();
  for (size_t i = 1; i < c.marks_used; ++i) {
    float ms = 0.f;
    if (cudaEventElapsedTime(&ms, c.event_pool[i - 1], c.event_pool[i]) != cudaSuccess) ms = -1.f;
    c.phases.emplace_back(c.mark_names[i], (double)ms);
  }
}

// ---------------------------------------------------------------------------
// K1: scene box + finiteness (bvh.hpp:247-254, geometry.hpp:58-69, 98-114)
// ---------------------------------------------------------------------------
__global__ void k_bounds_init(int32_t *ord6, int *bad) {
  int t = threadIdx.x;
  if (t < 3) ord6[t] = INT_MAX;
  else if (t < 6) ord6[t] = INT_MIN;
  if (t == 0) *bad = 0;
}

template <bool POINTS>
__global__ void __launch_bounds__(256) k_bounds(const float *__restrict__ obj, int64_t n, int dim,
                                                int32_t *__restrict__ ord6, int *__restrict__ bad) {
  int32_t mn[3] = {INT_MAX, INT_MAX, INT_MAX}, mx[3] = {INT_MIN, INT_MIN, INT_MIN};
  bool ok = true;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const int sz = POINTS ? dim : 2 * dim;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    const float *o = obj + i * sz;
    for (int k = 0; k < dim; ++k) {
      float lo = o[k];
      float hi = POINTS ? lo : o[dim + k];
      ok = ok && isfinite(lo) && isfinite(hi);
      mn[k] = min(mn[k], ord_of(lo));
      mx[k] = max(mx[k], ord_of(hi));
    }
  }
  for (int k = 0; k < 3; ++k) {
    mn[k] = __reduce_min_sync(0xffffffffu, mn[k]);
    mx[k] = __reduce_max_sync(0xffffffffu, mx[k]);
  }
  if ((threadIdx.x & 31) == 0) {
    for (int k = 0; k < dim; ++k) {
      atomicMin(&ord6[k], mn[k]);
      atomicMax(&ord6[3 + k], mx[k]);
    }
  }
  if (!__all_sync(0xffffffffu, ok) && (threadIdx.x & 31) == 0) *bad = 1;
}

// 3-D points, 16-byte aligned: four points per thread step (vector loads).
__global__ void __launch_bounds__(256) k_bounds_p3v(const float *__restrict__ pts, int64_t n,
                                                    int32_t *__restrict__ ord6, int *__restrict__ bad) {
  int32_t mn[3] = {INT_MAX, INT_MAX, INT_MAX}, mx[3] = {INT_MIN, INT_MIN, INT_MIN};
  bool ok = true;
  const int64_t chunks = n / 4;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  auto take = [&](float x, float y, float z) {
    ok = ok && isfinite(x) && isfinite(y) && isfinite(z);
    mn[0] = min(mn[0], ord_of(x)); mx[0] = max(mx[0], ord_of(x));
    mn[1] = min(mn[1], ord_of(y)); mx[1] = max(mx[1], ord_of(y));
    mn[2] = min(mn[2], ord_of(z)); mx[2] = max(mx[2], ord_of(z));
  };
  const int64_t t0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  for (int64_t ch = t0; ch < chunks; ch += stride) {
    float x[4], y[4], z[4];
    load4pts(pts, ch, x, y, z);
#pragma unroll
    for (int j = 0; j < 4; ++j) take(x[j], y[j], z[j]);
  }
  for (int64_t i = chunks * 4 + t0; i < n; i += stride) take(pts[3 * i], pts[3 * i + 1], pts[3 * i + 2]);
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    mn[k] = __reduce_min_sync(0xffffffffu, mn[k]);
    mx[k] = __reduce_max_sync(0xffffffffu, mx[k]);
  }
  if ((threadIdx.x & 31) == 0) {
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      atomicMin(&ord6[k], mn[k]);
      atomicMax(&ord6[3 + k], mx[k]);
    }
  }
  if (!__all_sync(0xffffffffu, ok) && (threadIdx.x & 31) == 0) *bad = 1;
}

// ord6 -> float scene[6]; axes beyond dim are 0 (2-D data lives at z = 0).
__global__ void k_bounds_final(const int32_t *ord6, int dim, int64_t n, float *scene) {
  int t = threadIdx.x;
  if (t < 6) {
    int k = t % 3;
    scene[t] = (k < dim && n > 0) ? float_of_ord(ord6[t]) : 0.f;
  }
}

__global__ void k_flag_or(const int *src, int *dst) {
  if (*src) *dst = 1;
}

void scene_bounds(Ctx &c, const float *objects, int64_t n, int dim, bool points, float *scene, int *bad) {
  DevBuf<int32_t> ord(6, c.stream);
  k_bounds_init<<<1, 32, 0, c.stream>>>(ord.get(), bad);
  SPB_LAUNCHED();
  if (n > 0) {
    unsigned g = grid_for(n, 256, 148 * 8);
    if (points && dim == 3 && aligned16(objects))
      k_bounds_p3v<<<grid_for((n + 3) / 4, 256, 148 * 8), 256, 0, c.stream>>>(objects, n, ord.get(), bad);
    else if (points) k_bounds<true><<<g, 256, 0, c.stream>>>(objects, n, dim, ord.get(), bad);
    else k_bounds<false><<<g, 256, 0, c.stream>>>(objects, n, dim, ord.get(), bad);
    SPB_LAUNCHED();
  }
  k_bounds_final<<<1, 32, 0, c.stream>>>(ord.get(), dim, n, scene);
  SPB_LAUNCHED();
}

// ---------------------------------------------------------------------------
// K2: Morton codes (morton.hpp:17-109; centroid geometry.hpp:130-137)
// ---------------------------------------------------------------------------
// Bit spreading: bit b of the input moves to bit b*stride.
__device__ __forceinline__ uint64_t spread_by3(uint64_t v) {  // 21 bits -> 63
  v &= 0x1fffffull;
  v = (v | (v << 32)) & 0x001f00000000ffffull;
  v = (v | (v << 16)) & 0x001f0000ff0000ffull;
  v = (v | (v << 8)) & 0x100f00f00f00f00full;
  v = (v | (v << 4)) & 0x10c30c30c30c30c3ull;
  v = (v | (v << 2)) & 0x1249249249249249ull;
  return v;
}
__device__ __forceinline__ uint64_t spread_by2(uint64_t v) {  // 32 bits -> 64
  v &= 0xffffffffull;
  v = (v | (v << 16)) & 0x0000ffff0000ffffull;
  v = (v | (v << 8)) & 0x00ff00ff00ff00ffull;
  v = (v | (v << 4)) & 0x0f0f0f0f0f0f0f0full;
  v = (v | (v << 2)) & 0x3333333333333333ull;
  v = (v | (v << 1)) & 0x5555555555555555ull;
  return v;
}

// Quantise one axis exactly as bin() does: floor((c - lo) / extent * 2^bits)
// in double, clamped; a non-positive extent gives bin 0.  The division is the
// IEEE-correct double division (a reciprocal multiply would not be bit-exact).
__device__ __forceinline__ uint32_t axis_bin(float c, float lo, float hi, double scale, uint32_t top) {
  double extent = __dsub_rn((double)hi, (double)lo);
  if (!(extent > 0.0)) return 0u;
  double t = __ddiv_rn(__dsub_rn((double)c, (double)lo), extent);
  double f = floor(__dmul_rn(t, scale));
  if (f <= 0.0) return 0u;
  if (f >= (double)top) return top;
  return (uint32_t)f;
}

__device__ __forceinline__ uint64_t encode_bins(uint32_t b0, uint32_t b1, uint32_t b2, int dim) {
  if (dim == 3) return spread_by3(b0) | (spread_by3(b1) << 1) | (spread_by3(b2) << 2);
  return spread_by2(b0) | (spread_by2(b1) << 1);
}

template <bool POINTS>
__global__ void __launch_bounds__(256) k_morton(const float *__restrict__ obj, int64_t n, int dim, int width,
                                                const float *__restrict__ scene, uint64_t *__restrict__ codes,
                                                uint32_t *__restrict__ vals) {
  const int bits = width / dim;
  const uint32_t top = bits >= 32 ? 0xffffffffu : ((1u << bits) - 1u);
  const double scale = (double)(1ull << bits);
  float slo[3], shi[3];
  for (int k = 0; k < 3; ++k) { slo[k] = scene[k]; shi[k] = scene[3 + k]; }
  const int sz = POINTS ? dim : 2 * dim;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    const float *o = obj + i * sz;
    uint32_t b[3] = {0u, 0u, 0u};
    for (int k = 0; k < dim; ++k) {
      float cen;
      if (POINTS) cen = o[k];
      else cen = __double2float_rn(__dmul_rn(__dadd_rn((double)o[k], (double)o[dim + k]), 0.5));
      b[k] = axis_bin(cen, slo[k], shi[k], scale, top);
    }
    codes[i] = encode_bins(b[0], b[1], b[2], dim);
    if (vals) vals[i] = (uint32_t)i;
  }
}

// 3-D points, 16-byte aligned: four codes per thread step (vector loads).
__global__ void __launch_bounds__(256) k_morton_p3v(const float *__restrict__ pts, int64_t n, int width,
                                                    const float *__restrict__ scene, uint64_t *__restrict__ codes,
                                                    uint32_t *__restrict__ vals) {
  const int bits = width / 3;
  const uint32_t top = bits >= 32 ? 0xffffffffu : ((1u << bits) - 1u);
  const double scale = (double)(1ull << bits);
  const float lo0 = scene[0], lo1 = scene[1], lo2 = scene[2], hi0 = scene[3], hi1 = scene[4], hi2 = scene[5];
  auto code = [&](float x, float y, float z) -> uint64_t {
    return encode_bins(axis_bin(x, lo0, hi0, scale, top), axis_bin(y, lo1, hi1, scale, top),
                       axis_bin(z, lo2, hi2, scale, top), 3);
  };
  const int64_t chunks = n / 4;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const int64_t t0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  for (int64_t ch = t0; ch < chunks; ch += stride) {
    float x[4], y[4], z[4];
    load4pts(pts, ch, x, y, z);
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      codes[4 * ch + j] = code(x[j], y[j], z[j]);
      if (vals) vals[4 * ch + j] = (uint32_t)(4 * ch + j);
    }
  }
  for (int64_t i = chunks * 4 + t0; i < n; i += stride) {
    codes[i] = code(pts[3 * i], pts[3 * i + 1], pts[3 * i + 2]);
    if (vals) vals[i] = (uint32_t)i;
  }
}

void morton_codes(Ctx &c, const float *objects, int64_t n, int dim, bool points, int width, const float *scene,
                  uint64_t *codes, uint32_t *vals) {
  if (n <= 0) return;
  unsigned g = grid_for(n, 256, 148 * 16);
  if (points && dim == 3 && aligned16(objects))
    k_morton_p3v<<<grid_for((n + 3) / 4, 256, 148 * 16), 256, 0, c.stream>>>(objects, n, width, scene, codes, vals);
  else if (points) k_morton<true><<<g, 256, 0, c.stream>>>(objects, n, dim, width, scene, codes, vals);
  else k_morton<false><<<g, 256, 0, c.stream>>>(objects, n, dim, width, scene, codes, vals);
  SPB_LAUNCHED();
}

// ---------------------------------------------------------------------------
// K3: stable onesweep LSD radix sort of (u64 key, u32 value), 8-bit digits.
// One upfront histogram pass for all digit positions, then one kernel per
// digit: each CTA ranks a 4096-key tile (warp match_any ranking keeps the
// original order within equal digits), obtains its global digit offsets by
// decoupled look-back over the preceding tiles, stages the tile in shared
// memory in digit order and writes it out coalesced.  Stability of every pass
// makes the final order equal std::stable_sort's (morton.hpp:113-121).
// ---------------------------------------------------------------------------
#ifndef SPB_RS_MINBLOCKS
#define SPB_RS_MINBLOCKS 3
#endif
constexpr int RS_BINS = 256;
#ifndef SPB_FUSED_HIST
#define SPB_FUSED_HIST 1  // digit counts accumulated by the key kernels (HistAcc)
#endif
constexpr int RS_WH = RS_BINS + 1;  // + one slot for out-of-range items

template <int ITEMS, int THREADS, class K>
constexpr size_t rs_smem_bytes() {
  return (size_t)THREADS * ITEMS * (sizeof(K) + 4) + (size_t)(THREADS / 32) * RS_WH * 4;
}

template <class K>
__global__ void __launch_bounds__(256) k_rs_hist(const K *__restrict__ keys, int64_t n, int npass,
                                                 uint32_t *__restrict__ ghist) {
  __shared__ uint32_t h[8 * RS_BINS];
  for (int i = threadIdx.x; i < npass * RS_BINS; i += blockDim.x) h[i] = 0;
  __syncthreads();
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    const uint64_t k = keys[i];
    for (int p = 0; p < npass; ++p) atomicAdd(&h[p * RS_BINS + ((k >> (8 * p)) & 0xff)], 1u);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < npass * RS_BINS; i += blockDim.x)
    if (h[i]) atomicAdd(&ghist[i], h[i]);
}

// Exclusive scan of each pass's 256 counts (one CTA per pass).
__global__ void k_rs_scan(uint32_t *ghist) {
  __shared__ uint32_t wsum[RS_BINS / 32];
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  uint32_t *h = ghist + blockIdx.x * RS_BINS;
  uint32_t v = h[t], x = v;
  for (int d = 1; d < 32; d <<= 1) {
    uint32_t y = __shfl_up_sync(0xffffffffu, x, d);
    if (lane >= d) x += y;
  }
  if (lane == 31) wsum[warp] = x;
  __syncthreads();
  uint32_t off = 0;
  for (int w = 0; w < warp; ++w) off += wsum[w];
  h[t] = off + x - v;
}


// THREADS threads, ITEMS keys each; threads [0, 256) own one digit each for
// the cross-warp prefix, the look-back and the tile-local digit scan.
#ifndef SPB_RS_MINBLOCKS32
#define SPB_RS_MINBLOCKS32 3
#endif
// KO / oshift: the keys are written out as (KO)(key >> oshift) (a pass that
// narrows 64-bit keys to their remaining 32 bits for the following passes).
template <int ITEMS, int THREADS, class K, class KO = K>
__global__ void __launch_bounds__(THREADS, (THREADS * ITEMS <= 2048) ? 4
                                           : (sizeof(K) == 4 ? SPB_RS_MINBLOCKS32 : SPB_RS_MINBLOCKS)) k_rs_onesweep(
    const K *__restrict__ kin, const uint32_t *__restrict__ vin, KO *__restrict__ kout,
    uint32_t *__restrict__ vout, int64_t n, int shift, const uint32_t *__restrict__ binbase,
    unsigned long long *lookback, uint32_t *tile_ctr, uint32_t tag, int oshift = 0) {
  constexpr int TILE = THREADS * ITEMS;
  constexpr int WARPS = THREADS / 32;
  // one thread per digit bin in the per-tile scans and the look-back (128
  // threads fault: measured)
  static_assert(THREADS >= RS_BINS, "onesweep needs at least one thread per digit bin");
  extern __shared__ __align__(16) unsigned char rs_smem[];
  K *skeys = reinterpret_cast<K *>(rs_smem);
  uint32_t *svals = reinterpret_cast<uint32_t *>(skeys + TILE);
  uint32_t *whist = svals + TILE;
  __shared__ uint32_t s_dstart[RS_BINS];
  __shared__ uint32_t s_gbase[RS_BINS];
  __shared__ uint32_t s_wsum[RS_BINS / 32];
  __shared__ uint32_t s_tile;

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int i = tid; i < WARPS * RS_WH; i += THREADS) whist[i] = 0;
  if (tid == 0) s_tile = atomicAdd(tile_ctr, 1u);
  __syncthreads();
  const uint32_t tile = s_tile;
  const int64_t base = (int64_t)tile * TILE;

  K key[ITEMS];
  uint32_t val[ITEMS];
  uint16_t rk[ITEMS];
  const int64_t wbase = base + (int64_t)warp * (ITEMS * 32);
  if (base + TILE <= n) {  // full tile: unconditional loads, all in flight together
#pragma unroll
    for (int i = 0; i < ITEMS; ++i) key[i] = kin[wbase + i * 32 + lane];
    if (vin) {
#pragma unroll
      for (int i = 0; i < ITEMS; ++i) val[i] = vin[wbase + i * 32 + lane];
    } else {
#pragma unroll
      for (int i = 0; i < ITEMS; ++i) val[i] = (uint32_t)(wbase + i * 32 + lane);
    }
  } else {
#pragma unroll
    for (int i = 0; i < ITEMS; ++i) {
      const int64_t idx = wbase + i * 32 + lane;
      key[i] = idx < n ? kin[idx] : (K)~(K)0;
      val[i] = idx < n ? (vin ? vin[idx] : (uint32_t)idx) : 0u;
    }
  }
  auto digit = [&](int i) -> uint32_t {
    return (wbase + i * 32 + lane < n) ? ((uint32_t)(key[i] >> shift) & 0xffu) : (uint32_t)RS_BINS;
  };
  // Warp-local stable ranks: items are visited in original order (item i of
  // lane l is element i*32 + l of the warp's slice).
  uint32_t *wh = whist + warp * RS_WH;
  const uint32_t lt = (1u << lane) - 1u;
#pragma unroll
  for (int i = 0; i < ITEMS; ++i) {
    const uint32_t d = digit(i);
    // peers by bit-sliced ballots over the 9 digit bits (256 = out of range);
    // measured faster than __match_any_sync on sm_100a (sort pass 1.45 ->
    // 1.30 ms at 2^27)
    uint32_t peers = 0xffffffffu;
#pragma unroll
    for (int bt = 0; bt < 9; ++bt) {
      const bool on = (d >> bt) & 1u;
      const uint32_t bal = __ballot_sync(0xffffffffu, on);
      peers &= on ? bal : ~bal;
    }
    // the lowest lane of each digit group advances the warp's counter; the
    // __syncwarp()s order the lanes' reads before the update and the update
    // before the next round's reads (memory-model clean: racecheck reports no
    // hazard; dropping them saved < 1% and relies on in-order warp execution)
    const uint32_t r = __popc(peers & lt);
    const uint32_t b = wh[d];
    __syncwarp();
    if (r == 0) wh[d] = b + __popc(peers);
    __syncwarp();
    rk[i] = (uint16_t)(b + r);
  }
  __syncthreads();

  // Thread t < 256 owns digit t: exclusive prefix over warps, then look-back.
  uint32_t tot = 0;
  if (tid < RS_BINS) {
#pragma unroll
    for (int w = 0; w < WARPS; ++w) {
      const uint32_t cw = whist[w * RS_WH + tid];
      whist[w * RS_WH + tid] = tot;
      tot += cw;
    }
    const unsigned long long agg_tag = (unsigned long long)tag << 32;
    const unsigned long long inc_tag = (unsigned long long)(tag + 1) << 32;
    unsigned long long *mine = lookback + (size_t)tile * RS_BINS + tid;
    uint32_t excl = 0;
    if (tile == 0) {
      st_volatile_u64(mine, inc_tag | tot);
    } else {
      st_volatile_u64(mine, agg_tag | tot);
      int64_t j = (int64_t)tile - 1;
      while (true) {
        const unsigned long long v = ld_volatile_u64(lookback + (size_t)j * RS_BINS + tid);
        const unsigned long long st = v & 0xffffffff00000000ull;
        if (st == inc_tag) {
          excl += (uint32_t)v;
          break;
        }
        if (st == agg_tag) {
          excl += (uint32_t)v;
          --j;
        }
      }
      st_volatile_u64(mine, inc_tag | (excl + tot));
    }
    s_gbase[tid] = binbase[tid] + excl;
    // tile-local digit starts: exclusive scan of tot over the 256 digits
    uint32_t x = tot;
    for (int d = 1; d < 32; d <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, x, d);
      if (lane >= d) x += y;
    }
    if (lane == 31) s_wsum[warp] = x;
    tot = x - tot;  // exclusive within the warp
  }
  __syncthreads();
  if (tid < RS_BINS) {
    uint32_t off = 0;
    for (int w = 0; w < warp; ++w) off += s_wsum[w];
    s_dstart[tid] = off + tot;
  }
  __syncthreads();

#pragma unroll
  for (int i = 0; i < ITEMS; ++i) {
    const uint32_t d = digit(i);
    if (d < RS_BINS) {
      const uint32_t pos = s_dstart[d] + wh[d] + rk[i];
      skeys[pos] = key[i];
      svals[pos] = val[i];
    }
  }
  __syncthreads();
  const int valid = (int)((n - base) < (int64_t)TILE ? (n - base) : (int64_t)TILE);
  for (int pos = tid; pos < valid; pos += THREADS) {
    const K k = skeys[pos];
    const uint32_t d = (uint32_t)(k >> shift) & 0xffu;
    const uint32_t o = s_gbase[d] + (uint32_t)pos - s_dstart[d];
    kout[o] = (KO)(k >> oshift);
    vout[o] = svals[pos];
  }
}

#ifndef SPB_RS_THREADS
#define SPB_RS_THREADS 256
#endif
#ifndef SPB_RS_ITEMS32
#define SPB_RS_ITEMS32 16  // keys per thread of the 32-bit-key passes
#endif
#ifndef SPB_RS_ITEMS
#define SPB_RS_ITEMS 12  // u64-key passes: 12 / 16 / 20 keys per thread: field build 16.18 / 16.24 / 16.34 ms
#endif

template <int ITEMS, int THREADS, class K>
void onesweep_passes(Ctx &c, K **keys, uint32_t **vals, K **keys_alt, uint32_t **vals_alt, int64_t n,
                     int npass, bool vals_iota, uint32_t *hist_in = nullptr) {
  constexpr int TILE = THREADS * ITEMS;
  constexpr size_t SMEM = rs_smem_bytes<ITEMS, THREADS, K>();
  // the dynamic shared-memory opt-in is per device (and per kernel)
  static std::mutex mu;
  static uint64_t opted = 0;  // bit d: set on device d
  {
    std::lock_guard<std::mutex> g(mu);
    if (c.device >= 64 || !((opted >> c.device) & 1)) {
      SPB_CUDA(cudaFuncSetAttribute(k_rs_onesweep<ITEMS, THREADS, K>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    (int)SMEM));
      if (c.device < 64) opted |= 1ull << c.device;
    }
  }
  const int64_t ntiles = (n + TILE - 1) / TILE;
  // hist_in: the digit counts already accumulated by the key kernel (fused
  // histogram, RS_HIST_ENTRIES(npass) zeroed entries), else counted here
  DevBuf<uint32_t> own;
  uint32_t *hist = hist_in;
  if (!hist) {
    own = DevBuf<uint32_t>((size_t)npass * RS_BINS + npass, c.stream);
    hist = own.get();
    SPB_CUDA(cudaMemsetAsync(hist, 0, own.n * sizeof(uint32_t), c.stream));
  }
  DevBuf<unsigned long long> lookback((size_t)ntiles * RS_BINS, c.stream);
  SPB_CUDA(cudaMemsetAsync(lookback.get(), 0, lookback.n * sizeof(unsigned long long), c.stream));
  if (!hist_in) {
    k_rs_hist<K><<<grid_for(n, 256, 148 * 4), 256, 0, c.stream>>>(*keys, n, npass, hist);
    SPB_LAUNCHED();
  }
  k_rs_scan<<<npass, RS_BINS, 0, c.stream>>>(hist);
  SPB_LAUNCHED();
  uint32_t *ctr = hist + (size_t)npass * RS_BINS;
  for (int p = 0; p < npass; ++p) {
    k_rs_onesweep<ITEMS, THREADS, K><<<(unsigned)ntiles, THREADS, SMEM, c.stream>>>(
        *keys, (p == 0 && vals_iota) ? nullptr : *vals, *keys_alt, *vals_alt, n, 8 * p,
        hist + (size_t)p * RS_BINS, lookback.get(), ctr + p, (uint32_t)(2 * p + 1));
    SPB_LAUNCHED();
    std::swap(*keys, *keys_alt);
    std::swap(*vals, *vals_alt);
  }
}

void radix_sort_pairs(Ctx &c, uint64_t **keys, uint32_t **vals, uint64_t **keys_alt, uint32_t **vals_alt, int64_t n,
                      int key_bits, bool vals_iota) {
  if (n <= 1) {
    if (n == 1 && vals_iota) SPB_CUDA(cudaMemsetAsync(*vals, 0, sizeof(uint32_t), c.stream));
    return;
  }
  const int npass = std::max(1, (key_bits + 7) / 8);
  onesweep_passes<SPB_RS_ITEMS, SPB_RS_THREADS, uint64_t>(c, keys, vals, keys_alt, vals_alt, n, npass, vals_iota);
}

// Stable sort of (u64 key < 2^40, u32 value) in five 8-bit passes: the first
// moves the 64-bit keys and writes key >> 8 as 32-bit keys, the other four
// move (u32, u32) pairs (16 instead of 24 bytes per element and pass).  Only
// the sorted values come back (*vals); the keys are consumed.  k32 and k32_alt
// hold n u32 each.
void radix_sort_pairs_40(Ctx &c, const uint64_t *keys, uint32_t **vals, uint32_t **vals_alt, uint32_t *k32,
                         uint32_t *k32_alt, int64_t n, bool vals_iota, uint32_t *hist_in) {
  if (n <= 1) {
    if (n == 1 && vals_iota) SPB_CUDA(cudaMemsetAsync(*vals, 0, sizeof(uint32_t), c.stream));
    return;
  }
  constexpr int ITEMS = SPB_RS_ITEMS, ITEMS32 = SPB_RS_ITEMS32, THREADS = SPB_RS_THREADS, TILE = ITEMS * THREADS,
                TILE32 = ITEMS32 * THREADS;
  constexpr size_t SMEM64 = rs_smem_bytes<ITEMS, THREADS, uint64_t>();
  constexpr size_t SMEM32 = rs_smem_bytes<ITEMS32, THREADS, uint32_t>();
  {
    static std::mutex mu;
    static uint64_t opted = 0;
    std::lock_guard<std::mutex> g(mu);
    if (c.device >= 64 || !((opted >> c.device) & 1)) {
      SPB_CUDA(cudaFuncSetAttribute(k_rs_onesweep<ITEMS, THREADS, uint64_t, uint32_t>,
                                    cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SMEM64));
      SPB_CUDA(cudaFuncSetAttribute(k_rs_onesweep<ITEMS32, THREADS, uint32_t>,
                                    cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SMEM32));
      if (c.device < 64) opted |= 1ull << c.device;
    }
  }
  constexpr int npass = 5;
  const int64_t ntiles = (n + TILE - 1) / TILE, ntiles32 = (n + TILE32 - 1) / TILE32;
  DevBuf<uint32_t> own;
  uint32_t *hist = hist_in;  // counts from the key kernel (fused histogram), else counted here
  if (!hist) {
    own = DevBuf<uint32_t>((size_t)npass * RS_BINS + npass, c.stream);
    hist = own.get();
    SPB_CUDA(cudaMemsetAsync(hist, 0, own.n * sizeof(uint32_t), c.stream));
  }
  DevBuf<unsigned long long> lookback((size_t)std::max(ntiles, ntiles32) * RS_BINS, c.stream);
  SPB_CUDA(cudaMemsetAsync(lookback.get(), 0, lookback.n * sizeof(unsigned long long), c.stream));
  if (!hist_in) {
    k_rs_hist<uint64_t><<<grid_for(n, 256, 148 * 4), 256, 0, c.stream>>>(keys, n, npass, hist);
    SPB_LAUNCHED();
  }
  k_rs_scan<<<npass, RS_BINS, 0, c.stream>>>(hist);
  SPB_LAUNCHED();
  uint32_t *ctr = hist + (size_t)npass * RS_BINS;
  k_rs_onesweep<ITEMS, THREADS, uint64_t, uint32_t><<<(unsigned)ntiles, THREADS, SMEM64, c.stream>>>(
      keys, vals_iota ? nullptr : *vals, k32, *vals_alt, n, 0, hist, lookback.get(), ctr, 1u, 8);
  SPB_LAUNCHED();
  std::swap(*vals, *vals_alt);
  uint32_t *ka = k32, *kb = k32_alt;
  for (int p = 1; p < npass; ++p) {
    k_rs_onesweep<ITEMS32, THREADS, uint32_t><<<(unsigned)ntiles32, THREADS, SMEM32, c.stream>>>(
        ka, *vals, kb, *vals_alt, n, 8 * (p - 1), hist + (size_t)p * RS_BINS, lookback.get(), ctr + p,
        (uint32_t)(2 * p + 1));
    SPB_LAUNCHED();
    std::swap(ka, kb);
    std::swap(*vals, *vals_alt);
  }
}

void radix_sort_pairs(Ctx &c, uint32_t **keys, uint32_t **vals, uint32_t **keys_alt, uint32_t **vals_alt, int64_t n,
                      int key_bits, bool vals_iota, uint32_t *hist_in) {
  if (n <= 1) {
    if (n == 1 && vals_iota) SPB_CUDA(cudaMemsetAsync(*vals, 0, sizeof(uint32_t), c.stream));
    return;
  }
  const int npass = std::max(1, std::min(4, (key_bits + 7) / 8));
  onesweep_passes<SPB_RS_ITEMS32, SPB_RS_THREADS, uint32_t>(c, keys, vals, keys_alt, vals_alt, n, npass, vals_iota,
                                                            hist_in);
}

// ---------------------------------------------------------------------------
// K4: hierarchy in one bottom-up pass (bvh.hpp:100-223).
// ---------------------------------------------------------------------------
// Adjacent prefix lengths of the augmented keys (code, object id): delta[i]
// compares sorted entries i and i+1 (bvh.hpp:106-115).
__global__ void __launch_bounds__(256) k_delta(const uint64_t *__restrict__ sk, const uint32_t *__restrict__ sv,
                                               int64_t n, int width, int32_t *__restrict__ delta) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i + 1 < n; i += stride) {
    uint64_t a = sk[i], b = sk[i + 1];
    int d;
    if (a != b) d = __clzll((long long)(a ^ b)) - (64 - width);
    else d = width + __clz((int)(sv ? sv[i] ^ sv[i + 1] : (uint32_t)(i ^ (i + 1))));
    delta[i] = d;
  }
}

#ifndef SPB_CLIMB_BLK
#define SPB_CLIMB_BLK 128  // 128 / 256 / 512: field build 15.83 / 16.13 / slower (hierarchy 6.23 vs 6.52 ms)
#endif
constexpr int CLIMB_BLK = SPB_CLIMB_BLK;
// Split lengths in 32-bit index arithmetic (n < 2^31: Karras indices are
// int32).  D(-1) = D(n-1) = -1 while every real split length is >= 0, which
// folds the range-end tests into the lengths themselves: a node [l, r] is its
// parent's left child iff D(r) > D(l-1) (l == 0 makes D(l-1) = -1; r == n-1
// makes D(r) = -1), it is the root iff both are -1, and its rope is the
// sentinel iff D(r) = -1, else leaf r+1 when D(r+1) < D(r) (bvh.hpp:176-222),
// else internal node r+1.
struct HierView {
  int32_t n;
  const int32_t *delta;
  // (reading D from the CTA's staged copy in shared memory instead measured
  // slower: hierarchy 8.8 -> 10.0 ms at 2^27)
  __device__ __forceinline__ int D(int32_t i) const {
    return (uint32_t)i < (uint32_t)(n - 1) ? __ldg(delta + i) : -1;
  }
};
__device__ __forceinline__ int32_t rope_of(int32_t n, int32_t r, int32_t dr, int32_t dr1) {
  return dr < 0 ? kSentinel : (dr1 < dr ? n + r : r + 1);
}

// The climb from leaf p (leaf box in lo/hi, already written): the first child
// to arrive at a parent records its far bound in flags[split] and stops; the
// second knows the parent's full range [l, r] and split, recovers its Karras
// index (r for a left child, l for a right child, 0 for the root), joins the
// two child boxes left-first and writes {box, left, rope}.
//
// Block-local hand-off (k_hierarchy): a CTA owns the leaves [B, B + BLK).
// When a parent lies inside, its two children meet in shared memory (box
// slots and a flag exchanged with CTA-scope acquire/release: no L2 round trip,
// no L1 invalidation); otherwise both use the global flag.  Both children must
// choose alike, so the choice is a property of the split: the parent at split
// a (the lowest common ancestor of leaves a and a + 1, prefix length D(a))
// spans [l'', r''] with l'' - 1 = max{j < a : D(j) < D(a)} and r'' = min{j > a
// : D(j) < D(a)} (D(-1) = D(n-1) = -1; equal lengths are always separated by a
// smaller one).  It lies inside the CTA iff the CTA holds a smaller split
// length on each side of a: prefix and suffix minima of the CTA's staged
// D(B-1 .. B+BLK-1), computed once per CTA.
struct LocalClimb {
  int32_t B;
  const uint8_t *in;  // [CLIMB_BLK] shared: the parent at split B + i lies inside
  unsigned long long *flag;  // [CLIMB_BLK][2] shared flag words {bound | lo.x, lo.y | lo.z}, bound -1 = empty
  unsigned long long *box;   // [2][CLIMB_BLK][2] shared words {hi.x | hi.y, hi.z | pass} per side (0 = left)
  __device__ __forceinline__ bool inside(int32_t a) const {
    return (uint32_t)(a - B) < (uint32_t)CLIMB_BLK && in[a - B];
  }
};

__device__ __forceinline__ int32_t exch_acq_rel_gpu(int32_t *p, int32_t v) {
  int32_t old;
  asm volatile("atom.acq_rel.gpu.global.exch.b32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
  return old;
}

__device__ __forceinline__ unsigned long long pack2(float a, float b) {
  return (unsigned long long)__float_as_uint(a) | ((unsigned long long)__float_as_uint(b) << 32);
}
__device__ __forceinline__ float lo32f(unsigned long long w) { return __uint_as_float((uint32_t)w); }
__device__ __forceinline__ float hi32f(unsigned long long w) { return __uint_as_float((uint32_t)(w >> 32)); }
__device__ __forceinline__ void exch128(unsigned long long *p, unsigned long long &x, unsigned long long &y,
                                        bool acq_rel) {
  const uint32_t a = (uint32_t)__cvta_generic_to_shared(p);
  if (acq_rel)
    asm volatile("{ .reg .b128 d, v; mov.b128 v, {%0, %1}; atom.acq_rel.cta.shared::cta.exch.b128 d, [%2], v;"
                 " mov.b128 {%0, %1}, d; }" : "+l"(x), "+l"(y) : "r"(a) : "memory");
  else
    asm volatile("{ .reg .b128 d, v; mov.b128 v, {%0, %1}; atom.relaxed.cta.shared::cta.exch.b128 d, [%2], v;"
                 " mov.b128 {%0, %1}, d; }" : "+l"(x), "+l"(y) : "r"(a) : "memory");
}

// One block-local hand-off at split a: publish this child's hi corner (and
// `pass`: its far-side split lengths) in its side's slot, then exchange the
// flag word {bound, lo.xyz} with CTA-scope acquire-release; returns the first
// arrival's bound (second arrival: sibling box in slo/shi, its lengths in
// *theirs) or -1 (first arrival).  Every shared access of the slots is a
// 128-bit atomic exchange: racecheck tracks barriers, not acquire/release
// (plain stores and loads were measured no faster).
__device__ __forceinline__ int32_t local_handoff(const LocalClimb &lc, int32_t a, bool L, int32_t bound,
                                                 const float lo[3], const float hi[3], float4 &slo, float4 &shi,
                                                 uint32_t pass, uint32_t &theirs) {
  const int32_t k = a - lc.B;
  unsigned long long h0 = pack2(hi[0], hi[1]), h1 = pack2(hi[2], __uint_as_float(pass));
  exch128(lc.box + ((L ? 0 : CLIMB_BLK) + k) * 2, h0, h1, false);
  unsigned long long w0 = (unsigned long long)(uint32_t)bound | ((unsigned long long)__float_as_uint(lo[0]) << 32);
  unsigned long long w1 = pack2(lo[1], lo[2]);
  exch128(lc.flag + 2 * k, w0, w1, true);
  const int32_t other = (int32_t)(uint32_t)w0;
  if (other < 0) return other;
  unsigned long long g0 = 0, g1 = 0;
  exch128(lc.box + ((L ? CLIMB_BLK : 0) + k) * 2, g0, g1, false);
  slo = make_float4(hi32f(w0), lo32f(w1), hi32f(w1), 0.f);
  shi = make_float4(lo32f(g0), hi32f(g0), lo32f(g1), 0.f);
  theirs = (uint32_t)(g1 >> 32);
  return other;
}

// One climb step of the node [l, r] (box lo/hi, split lengths dl1 = D(l-1),
// dr = D(r), dr1 = D(r+1)), already written: the first child to arrive at the
// parent records its far bound and stops; the second knows the parent's full
// range and split, joins the two child boxes left-first and writes the parent
// {box, left, rope} at its Karras index (r for a left child, l for a right
// child, 0 for the root).  Returns 0 when this thread stops (first arrival, or
// the root written), 1 when it now owns the parent after a block-local
// hand-off, 2 after a global exchange.
//
// Block-local hand-off (k_hierarchy): a CTA owns the leaves [B, B + BLK).
// When a parent lies inside, its two children meet in shared memory (no L2
// round trip, no L1 invalidation); otherwise both use the global flag.  Both
// children must choose alike, so the choice is a property of the split: the
// parent at split a (the lowest common ancestor of leaves a and a + 1, prefix
// length D(a)) spans [l'', r''] with l'' - 1 = max{j < a : D(j) < D(a)} and
// r'' = min{j > a : D(j) < D(a)} (equal lengths are always separated by a
// smaller one).  It lies inside the CTA iff the CTA holds a smaller split
// length on each side of a: prefix and suffix minima of the CTA's staged
// D(B-1 .. B+BLK-1), computed once per CTA.  A local hand-off passes the
// child's far-side lengths along with its box (a left child D(l-1), a right
// child D(r) and D(r+1), 16 bits each), so local levels read no split lengths
// from memory.
//
// Ordering: the global exchange is acquire-release -- the release half
// orders this node's stores before the flag changes hands, the acquire half
// orders the second arrival's reads of the sibling after the first arrival's
// stores (the PTX memory model gives no ordering through the address
// dependency alone); the sibling is read with L2-coherent loads.
template <bool LOCAL>
__device__ __forceinline__ int climb_step(const HierView &H, int32_t &l, int32_t &r, float lo[3], float hi[3],
                                          int32_t &dl1, int32_t &dr, int32_t &dr1, float4 *nodes, int32_t *flags,
                                          const LocalClimb &lc) {
  const int32_t n = H.n;
  const bool L = dr > dl1;
  const int32_t a = L ? r : l - 1;  // the parent's split position
  const int32_t bound = L ? l : r;
  const bool local = LOCAL && lc.inside(a);
  float4 slo, shi;
  if (local) {
    const uint32_t mine = L ? (uint32_t)(uint16_t)dl1 : ((uint32_t)(uint16_t)dr | ((uint32_t)(uint16_t)dr1 << 16));
    uint32_t theirs = 0;
    const int32_t other = local_handoff(lc, a, L, bound, lo, hi, slo, shi, mine, theirs);
    if (other < 0) return 0;
    if (L) {
      r = other;
      dr = (int16_t)(theirs & 0xffffu);
      dr1 = (int16_t)(theirs >> 16);
    } else {
      l = other;
      dl1 = (int16_t)(theirs & 0xffffu);
    }
  } else {
    const int32_t other = exch_acq_rel_gpu(flags + a, bound);
    if (other < 0) return 0;
    if (L) {
      r = other;
      dr = H.D(r);
      dr1 = H.D(r + 1);
    } else {
      l = other;
      dl1 = H.D(l - 1);
    }
    const int32_t sib = L ? ((a + 1 == r) ? n - 1 + r : a + 1) : ((a == l) ? n - 1 + l : a);
    slo = __ldcg(nodes + 2 * (int64_t)sib);
    shi = __ldcg(nodes + 2 * (int64_t)sib + 1);
  }
  if (L) {  // this node is the left child
    lo[0] = keep_min(lo[0], slo.x); lo[1] = keep_min(lo[1], slo.y); lo[2] = keep_min(lo[2], slo.z);
    hi[0] = keep_max(hi[0], shi.x); hi[1] = keep_max(hi[1], shi.y); hi[2] = keep_max(hi[2], shi.z);
  } else {
    lo[0] = keep_min(slo.x, lo[0]); lo[1] = keep_min(slo.y, lo[1]); lo[2] = keep_min(slo.z, lo[2]);
    hi[0] = keep_max(shi.x, hi[0]); hi[1] = keep_max(shi.y, hi[1]); hi[2] = keep_max(shi.z, hi[2]);
  }
  const int32_t left = (a == l) ? n - 1 + l : a;
  const int64_t k = dr > dl1 ? r : l;  // the root (both -1) lands at l = 0
  nodes[2 * k] = make_float4(lo[0], lo[1], lo[2], __int_as_float(left));
  nodes[2 * k + 1] = make_float4(hi[0], hi[1], hi[2], __int_as_float(rope_of(n, r, dr, dr1)));
  if ((dl1 & dr) < 0) return 0;  // the root
  return local ? 1 : 2;
}

// Climbs at most max_levels merges through the global flags; returns true
// when this thread still owns a node whose parent is not built yet (the state
// in l, r, lo, hi).
template <bool LOCAL>
__device__ __forceinline__ bool climb(const HierView &H, int32_t &l, int32_t &r, float lo[3], float hi[3],
                                      int32_t dl1, int32_t dr, int32_t dr1, float4 *nodes, int32_t *flags,
                                      int max_levels, const LocalClimb &lc) {
  for (int level = 0; level < max_levels;) {
    const int st = climb_step<LOCAL>(H, l, r, lo, hi, dl1, dr, dr1, nodes, flags, lc);
    if (st == 0) return false;
    if (st == 2) ++level;
  }
  return true;
}

// Climb state of a thread that outlived the first kernel: {l, r, lo xyz},
// {hi xyz, unused}.  The first kernel does the bottom levels for every leaf;
// the few threads still climbing continue here, packed densely, instead of
// holding mostly-finished warps for the whole height of the tree.
__global__ void __launch_bounds__(256) k_climb_rest(int32_t n, const int32_t *__restrict__ delta,
                                                    const float4 *__restrict__ queue,
                                                    const uint32_t *__restrict__ qcount, float4 *nodes,
                                                    int32_t *flags) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= (int64_t)*qcount) return;
  const HierView H{n, delta};
  const float4 s0 = queue[2 * i], s1 = queue[2 * i + 1];
  int32_t l = __float_as_int(s0.x), r = __float_as_int(s0.y);
  float lo[3] = {s0.z, s0.w, s1.x}, hi[3] = {s1.y, s1.z, s1.w};
  climb<false>(H, l, r, lo, hi, H.D(l - 1), H.D(r), H.D(r + 1), nodes, flags, 1 << 30,
               LocalClimb{0, nullptr, nullptr, nullptr});
}

template <bool POINTS>
__global__ void __launch_bounds__(CLIMB_BLK) k_hierarchy(int32_t n, const int32_t *__restrict__ delta,
                                                   const uint32_t *__restrict__ perm, const float *__restrict__ obj,
                                                   int dim, float4 *nodes, int32_t *flags,
                                                   int32_t *__restrict__ perm_out, float4 *__restrict__ leafpt,
                                                   int max_levels, float4 *__restrict__ queue,
                                                   uint32_t *__restrict__ qcount, const float4 *spts) {
  __shared__ int32_t s_D[CLIMB_BLK + 1], s_pre[CLIMB_BLK], s_suf[CLIMB_BLK + 1], s_wmin[2][CLIMB_BLK / 32];
  __shared__ uint8_t s_in[CLIMB_BLK];
  __shared__ __align__(16) unsigned long long s_box[2 * CLIMB_BLK * 2];
  __shared__ __align__(16) unsigned long long s_flag[2 * CLIMB_BLK];
  const HierView H{n, delta};
  const int32_t B = (int32_t)blockIdx.x * CLIMB_BLK;
  const int t = threadIdx.x, lane = t & 31, w = t >> 5;
  const int32_t p = B + t;
  const bool valid = p < n;
  // the leaf's box first: its load latency overlaps the staging below
  uint32_t oi = (uint32_t)p;
  float lo[3] = {0.f, 0.f, 0.f}, hi[3] = {0.f, 0.f, 0.f};
  if (!valid) {
  } else if (POINTS && spts) {  // sorted points from the top-bits sort (3-D): no gather
    const float4 q = spts[p];
    oi = __float_as_uint(q.w);
    lo[0] = hi[0] = q.x;
    lo[1] = hi[1] = q.y;
    lo[2] = hi[2] = q.z;
  } else if (!POINTS && !obj) {  // leaf nodes written by the caller (k_cell_ranges): read the box back
    const float4 a = nodes[2 * (int64_t)(n - 1 + p)], b = nodes[2 * (int64_t)(n - 1 + p) + 1];
    lo[0] = a.x; lo[1] = a.y; lo[2] = a.z;
    hi[0] = b.x; hi[1] = b.y; hi[2] = b.z;
  } else {
    oi = perm ? perm[p] : (uint32_t)p;
    const int sz = POINTS ? dim : 2 * dim;
    const float *o = obj + (int64_t)oi * sz;
    for (int k = 0; k < dim; ++k) {
      lo[k] = o[k];
      hi[k] = POINTS ? lo[k] : o[dim + k];
    }
  }
  s_flag[2 * t] = 0xffffffffull;  // bound -1
  s_flag[2 * t + 1] = 0;
  const int32_t dv = H.D(B - 1 + t);  // element t of D(B-1 .. B+BLK-1)
  s_D[t] = dv;
  if (t == 0) s_D[CLIMB_BLK] = H.D(B + CLIMB_BLK - 1);
  // inclusive prefix / suffix minima over the 256 elements (warp scans, then
  // the warp totals), suffix also over the last element s_D[BLK]
  int32_t pm = dv, sm = dv;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int32_t y = __shfl_up_sync(0xffffffffu, pm, o), z = __shfl_down_sync(0xffffffffu, sm, o);
    if (lane >= o) pm = min(pm, y);
    if (lane + o < 32) sm = min(sm, z);
  }
  if (lane == 31) s_wmin[0][w] = pm;
  if (lane == 0) s_wmin[1][w] = sm;
  __syncthreads();
  for (int k = 0; k < w; ++k) pm = min(pm, s_wmin[0][k]);
  for (int k = w + 1; k < CLIMB_BLK / 32; ++k) sm = min(sm, s_wmin[1][k]);
  s_pre[t] = pm;
  s_suf[t] = min(sm, s_D[CLIMB_BLK]);
  if (t == 0) s_suf[CLIMB_BLK] = s_D[CLIMB_BLK];
  __syncthreads();
  // split a = B + t: D(a) = s_D[t + 1]; left minimum over D(B-1 .. a-1) =
  // s_pre[t], right minimum over D(a+1 .. B+BLK-1) = s_suf[t + 2]
  s_in[t] = t + 1 < CLIMB_BLK && s_pre[t] < s_D[t + 1] && s_suf[t + 2] < s_D[t + 1];
  __syncthreads();
  if (!valid) return;
  // split lengths around the leaf: D(p-1), D(p), D(p+1)
  int32_t dl1 = dv, dr = s_D[t + 1], dr1 = t + 2 <= CLIMB_BLK ? s_D[t + 2] : H.D(p + 1);
  if (perm_out) perm_out[p] = (int32_t)oi;
  const int64_t leaf = n - 1 + p;
  const int32_t leaf_rope = rope_of(n, p, dr, dr1);
  if (POINTS || obj) {
    nodes[2 * leaf] = make_float4(lo[0], lo[1], lo[2], __int_as_float((int)oi));
    nodes[2 * leaf + 1] = make_float4(hi[0], hi[1], hi[2], __int_as_float(leaf_rope));
  }
  if (POINTS) leafpt[p] = make_float4(lo[0], lo[1], lo[2], __int_as_float(leaf_rope));
  if (n == 1) return;
  int32_t l = p, r = p;
  const LocalClimb lc{B, s_in, s_flag, s_box};
  if (climb<true>(H, l, r, lo, hi, dl1, dr, dr1, nodes, flags, max_levels, lc)) {
    const uint32_t slot = atomicAdd(qcount, 1u);
    queue[2 * (int64_t)slot] = make_float4(__int_as_float(l), __int_as_float(r), lo[0], lo[1]);
    queue[2 * (int64_t)slot + 1] = make_float4(lo[2], hi[0], hi[1], hi[2]);
  }
}

// The two-kernel climb: k_hierarchy climbs every block-local merge and at most
// `levels` merges through the global flags per leaf; the survivors (<= n /
// (levels + 1): their nodes are disjoint subtrees of >= levels + 1 leaves) are
// queued and finished by k_climb_rest.  With the block-local hand-off, one
// global level is best at 2^27 (hierarchy phase 13.1 -> 11.1 ms for point
// trees, 9.5 -> 9.1 ms for the FoF cell tree; 2, 4 and 8 levels are slower).
#ifndef SPB_CLIMB_LEVELS_POINTS
#define SPB_CLIMB_LEVELS_POINTS 1
#endif
#ifndef SPB_CLIMB_LEVELS_CELLS
#define SPB_CLIMB_LEVELS_CELLS 1
#endif
struct ClimbQueue {
  int levels = 8;
  int64_t cap = 0;
  DevBuf<float4> buf;
  DevBuf<uint32_t> count;
  ClimbQueue(Ctx &c, int64_t n, int lv) : levels(lv) {
    cap = n / (levels + 1) + 1;
    buf = DevBuf<float4>((size_t)(2 * cap), c.stream);
    count = DevBuf<uint32_t>(1, c.stream);
    SPB_CUDA(cudaMemsetAsync(count.get(), 0, sizeof(uint32_t), c.stream));
  }
  void finish(Ctx &c, int64_t n, const int32_t *delta, float4 *nodes, int32_t *flags) {
    if (n <= 1) return;
    k_climb_rest<<<(unsigned)((cap + 255) / 256), 256, 0, c.stream>>>(n, delta, buf.get(), count.get(), nodes, flags);
    SPB_LAUNCHED();
  }
};

// ---------------------------------------------------------------------------
// Point trees with 63-bit codes: sort by the top 32 code bits, then order the
// runs of equal top bits (morton.hpp:113-121 stable order = full code, then
// index).  Four 8-bit passes over (u32 key, u32 index) instead of eight over
// (u64, u32); the run fix-up gathers each point once (the gather the
// hierarchy needed anyway), recomputes its full code, and writes the sorted
// points for the hierarchy.  Runs longer than FIX_MAX_RUN (dense clumps,
// duplicates) make the host fall back to the full 63-bit sort.
// ---------------------------------------------------------------------------
constexpr int FIX_MAX_RUN = 512;
#ifndef SPB_FIX_ILP
#define SPB_FIX_ILP 4
#endif
constexpr int FIX_ILP = SPB_FIX_ILP;

__global__ void __launch_bounds__(256) k_morton_top32(const float *__restrict__ pts, int64_t n, int width,
                                                      const float *__restrict__ scene, uint32_t *__restrict__ key32,
                                                      uint32_t *ghist = nullptr) {
  __shared__ uint32_t s_hist[4 * 256];
  HistAcc<4> H;
  H.init(s_hist, ghist);
  const int bits = width / 3;
  const uint32_t top = bits >= 32 ? 0xffffffffu : ((1u << bits) - 1u);
  const double scale = (double)(1ull << bits);
  const int shift = 3 * bits - 32;
  const float lo0 = scene[0], lo1 = scene[1], lo2 = scene[2], hi0 = scene[3], hi1 = scene[4], hi2 = scene[5];
  auto code = [&](float x, float y, float z) -> uint32_t {
    return (uint32_t)(encode_bins(axis_bin(x, lo0, hi0, scale, top), axis_bin(y, lo1, hi1, scale, top),
                                  axis_bin(z, lo2, hi2, scale, top), 3) >> shift);
  };
  const int64_t chunks = n / 4;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const int64_t t0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  for (int64_t ch = t0; ch < chunks; ch += stride) {
    float x[4], y[4], z[4];
    load4pts(pts, ch, x, y, z);
    uint4 k;
    k.x = code(x[0], y[0], z[0]);
    k.y = code(x[1], y[1], z[1]);
    k.z = code(x[2], y[2], z[2]);
    k.w = code(x[3], y[3], z[3]);
    reinterpret_cast<uint4 *>(key32)[ch] = k;
    H.add(k.x);
    H.add(k.y);
    H.add(k.z);
    H.add(k.w);
  }
  for (int64_t i = chunks * 4 + t0; i < n; i += stride) {
    key32[i] = code(pts[3 * i], pts[3 * i + 1], pts[3 * i + 2]);
    H.add(key32[i]);
  }
  H.flush();
}

// Query ordering (sort_points): top 32 bits and the full code, both in input
// order; the run fix-up below reads full codes only for members of runs.
__global__ void __launch_bounds__(256) k_morton_top32_full(const float *__restrict__ pts, int64_t n, int width,
                                                           const float *__restrict__ scene,
                                                           uint32_t *__restrict__ key32, uint64_t *__restrict__ code,
                                                           uint32_t *ghist = nullptr) {
  __shared__ uint32_t s_hist[4 * 256];
  HistAcc<4> H;
  H.init(s_hist, ghist);
  const int bits = width / 3;
  const uint32_t top = bits >= 32 ? 0xffffffffu : ((1u << bits) - 1u);
  const double scale = (double)(1ull << bits);
  const int shift = 3 * bits - 32;
  const float lo0 = scene[0], lo1 = scene[1], lo2 = scene[2], hi0 = scene[3], hi1 = scene[4], hi2 = scene[5];
  auto full = [&](float x, float y, float z) -> uint64_t {
    return encode_bins(axis_bin(x, lo0, hi0, scale, top), axis_bin(y, lo1, hi1, scale, top),
                       axis_bin(z, lo2, hi2, scale, top), 3);
  };
  const int64_t chunks = n / 4;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const int64_t t0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  for (int64_t ch = t0; ch < chunks; ch += stride) {
    float x[4], y[4], z[4];
    load4pts(pts, ch, x, y, z);
    uint64_t c[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) c[j] = full(x[j], y[j], z[j]);
    reinterpret_cast<uint4 *>(key32)[ch] =
        make_uint4((uint32_t)(c[0] >> shift), (uint32_t)(c[1] >> shift), (uint32_t)(c[2] >> shift),
                   (uint32_t)(c[3] >> shift));
    reinterpret_cast<ulonglong2 *>(code)[2 * ch] = make_ulonglong2(c[0], c[1]);
    reinterpret_cast<ulonglong2 *>(code)[2 * ch + 1] = make_ulonglong2(c[2], c[3]);
#pragma unroll
    for (int j = 0; j < 4; ++j) H.add(c[j] >> shift);
  }
  for (int64_t i = chunks * 4 + t0; i < n; i += stride) {
    const uint64_t c = full(pts[3 * i], pts[3 * i + 1], pts[3 * i + 2]);
    key32[i] = (uint32_t)(c >> shift);
    code[i] = c;
    H.add(c >> shift);
  }
  H.flush();
}

// Runs of equal top bits ordered by (full code, index); singletons keep
// their place.  Writes the final order only.
__global__ void __launch_bounds__(256) k_fix_runs_order(const uint32_t *__restrict__ key32, int64_t n,
                                                        const uint32_t *__restrict__ idx,
                                                        const uint64_t *__restrict__ code, int32_t *__restrict__ order,
                                                        int *overflow) {
  const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= n) return;
  const uint32_t k = key32[p];
  int64_t s = p, e = p + 1;
  while (s > 0 && p - s < FIX_MAX_RUN && key32[s - 1] == k) --s;
  while (e < n && e - p <= FIX_MAX_RUN && key32[e] == k) ++e;
  const uint32_t i = idx[p];
  int64_t dst = p;
  if (e - s > 1) {
    if (e - s > FIX_MAX_RUN) {
      *overflow = 1;
      return;
    }
    const uint64_t c = code[i];
    int64_t r = 0;
    for (int64_t j = s; j < e; ++j) {
      const uint32_t ij = idx[j];
      const uint64_t cj = code[ij];
      r += (cj < c) | ((cj == c) & (ij < i));
    }
    dst = s + r;
  }
  order[dst] = (int32_t)i;
}

// Sorted position p: gather the point, recompute its full code.
__global__ void __launch_bounds__(256) k_fix_gather(const float *__restrict__ pts, int64_t n, int width,
                                                    const float *__restrict__ scene,
                                                    const uint32_t *__restrict__ idx, uint64_t *__restrict__ tcode,
                                                    float4 *__restrict__ tpt) {
  const int bits = width / 3;
  const uint32_t top = bits >= 32 ? 0xffffffffu : ((1u << bits) - 1u);
  const double scale = (double)(1ull << bits);
  const float lo0 = scene[0], lo1 = scene[1], lo2 = scene[2], hi0 = scene[3], hi1 = scene[4], hi2 = scene[5];
  // FIX_ILP sorted positions per thread, their random gathers all in flight
  // together (a gather is one DRAM round trip; one thread per position would
  // need the whole grid resident)
  const int64_t p0 = ((int64_t)blockIdx.x * blockDim.x) * FIX_ILP + threadIdx.x;
  uint32_t i[FIX_ILP];
  float x[FIX_ILP], y[FIX_ILP], z[FIX_ILP];
#pragma unroll
  for (int u = 0; u < FIX_ILP; ++u) {
    const int64_t p = p0 + (int64_t)u * blockDim.x;
    i[u] = p < n ? idx[p] : 0u;
  }
  // three 4-byte loads: measured faster here than gather_pt3's 16-byte
  // blocks (3.41 vs 3.66 ms at 2^27; a uniformly random gather costs ~128 B of
  // DRAM per point either way)
#pragma unroll
  for (int u = 0; u < FIX_ILP; ++u) {
    const float *q = pts + 3 * (int64_t)i[u];
    x[u] = __ldg(q);
    y[u] = __ldg(q + 1);
    z[u] = __ldg(q + 2);
  }
#pragma unroll
  for (int u = 0; u < FIX_ILP; ++u) {
    const int64_t p = p0 + (int64_t)u * blockDim.x;
    if (p >= n) break;
    tcode[p] = encode_bins(axis_bin(x[u], lo0, hi0, scale, top), axis_bin(y[u], lo1, hi1, scale, top),
                           axis_bin(z[u], lo2, hi2, scale, top), 3);
    tpt[p] = make_float4(x[u], y[u], z[u], __uint_as_float(i[u]));
  }
}

// Each element of a run of equal top bits [s, e) takes rank #{q in run :
// (code, index)(q) < (code, index)(p)} and moves to s + rank; singletons copy.
// The same in shared memory: a CTA stages the codes and indices of its
// FIX_CH positions and FIX_MAX_RUN more on each side (every run of at most
// FIX_MAX_RUN through a position of the chunk lies inside), so the run scans
// and the O(run) ranking read shared memory (clustered fields have runs of
// hundreds: the global-memory version took 20 ms at 2^27 on H(2^27)).
// The CTA also ranks the halo elements of the runs that reach into its chunk
// and keeps the sorted (code, index) of positions [c0, c0 + FIX_CH] in shared
// memory, so it writes the split lengths D(c0 .. c0 + FIX_CH - 1) of the
// hierarchy itself (k_delta's pass over the sorted codes and indices, and
// writing those, are gone); the sorted points go to spts.
#ifndef SPB_FIX_CH
#define SPB_FIX_CH 1024  // 1024 / 2048 / 4096: field build 16.10 / 16.17 / 16.69 ms
#endif
constexpr int FIX_CH = SPB_FIX_CH;
constexpr int FIX_WIN = FIX_CH + 2 * FIX_MAX_RUN;
constexpr size_t FIX_SMEM = (size_t)(FIX_WIN + FIX_CH + 1) * (sizeof(uint64_t) + sizeof(uint32_t));
template <int SHIFT>  // runs: equal code >> SHIFT (31: top 32 of 63 bits, 23: top 40)
__global__ void __launch_bounds__(256) k_fix_runs_win(int64_t n, const uint64_t *__restrict__ tcode,
                                                      const float4 *__restrict__ tpt, float4 *__restrict__ spts,
                                                      int32_t *__restrict__ delta, int *overflow) {
  extern __shared__ __align__(16) unsigned char fix_smem[];
  uint64_t *sc = reinterpret_cast<uint64_t *>(fix_smem);  // [FIX_WIN] window codes
  uint64_t *oc = sc + FIX_WIN;                              // [FIX_CH + 1] sorted codes at c0 ..
  uint32_t *si = reinterpret_cast<uint32_t *>(oc + FIX_CH + 1);  // [FIX_WIN] window indices
  uint32_t *ox = si + FIX_WIN;                                   // [FIX_CH + 1] sorted indices at c0 ..
  constexpr int M = FIX_MAX_RUN;  // window index of c0
  const int64_t c0 = (int64_t)blockIdx.x * FIX_CH, w0 = c0 - M;
  const int lo_lim = w0 < 0 ? (int)(-w0) : 0;
  const int hi_lim = (int)((n - w0) < FIX_WIN ? (n - w0) : FIX_WIN);
  for (int i = threadIdx.x; i < FIX_WIN; i += blockDim.x) {
    if (i >= lo_lim && i < hi_lim) {
      const int64_t q = w0 + i;
      sc[i] = tcode[q];
      si[i] = __float_as_uint(__ldg(&tpt[q].w));
    }
  }
  __syncthreads();
  const int last = min(M + FIX_CH, hi_lim - 1);  // the sorted positions kept: window [M, last]
  for (int li = threadIdx.x; li < FIX_WIN; li += blockDim.x) {
    if (li < lo_lim || li >= hi_lim || M > last) continue;
    const uint64_t c = sc[li], k = c >> SHIFT;
    // a halo element matters only if its run reaches the kept positions
    // (equal top bits are contiguous in sorted order)
    if (li < M ? (sc[M] >> SHIFT) != k : (li > last && (sc[last] >> SHIFT) != k)) continue;
    int s = li, e = li + 1;
    while (s > lo_lim && li - s < FIX_MAX_RUN && (sc[s - 1] >> SHIFT) == k) --s;
    while (e < hi_lim && e - li <= FIX_MAX_RUN && (sc[e] >> SHIFT) == k) ++e;
    const uint32_t i = si[li];
    int d = li;
    if (e - s > 1) {
      if (e - s > FIX_MAX_RUN) {
        *overflow = 1;
        continue;
      }
      int r = 0;
      for (int q = s; q < e; ++q) {
        const uint64_t cq = sc[q];
        r += (cq < c) | ((cq == c) & (si[q] < i));
      }
      d = s + r;
    }
    if (d >= M && d <= last) {
      oc[d - M] = c;
      ox[d - M] = i;
    }
    if (li >= M && li < M + FIX_CH) spts[w0 + d] = tpt[w0 + li];
  }
  __syncthreads();
  // D(p) of sorted positions p, p + 1 (k_delta with 64-bit codes)
  for (int j = threadIdx.x; j < FIX_CH; j += blockDim.x) {
    if (M + j + 1 > last) break;
    const uint64_t a = oc[j], b = oc[j + 1];
    delta[c0 + j] = a != b ? __clzll((long long)(a ^ b)) : 64 + __clz((int)(ox[j] ^ ox[j + 1]));
  }
}

#ifndef SPB_SORT_TOP32
#define SPB_SORT_TOP32 1
#endif

// Clustered inputs make long runs of equal top bits (halo cores: hundreds of
// points per top-32 cell on H(2^27)), for which a top-bits sort would end in
// the fallback after all its work.  A sample of n / 128 scattered points
// predicts them: a run of 3/4 FIX_MAX_RUN points leaves about 3 copies of its
// key in the sample.  The sample is sorted by its top 40 code bits once; no three
// equal top-32 keys choose the 32-bit sort (4 passes), else no three equal
// top-40 keys the 40-bit sort (5 passes), else the full 63-bit sort (on
// uniform points at 2^27 three equal sampled top-32 keys have probability
// ~1%; a miss only costs the fallback).
__global__ void __launch_bounds__(256) k_sample_top40(const float *__restrict__ pts, int64_t stride, int64_t ns,
                                                      const float *__restrict__ scene, uint64_t *__restrict__ key) {
  const int bits = 21;
  const uint32_t top = (1u << bits) - 1u;
  const double scale = (double)(1ull << bits);
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= ns) return;
  // scattered sample positions (a multiplicative hash): a fixed stride can
  // alias with the input's own structure (H(n) deals its halo points round
  // robin, and every 128th point falls into 96 of the 12288 halos at 2^27)
  const int64_t at = (int64_t)(((unsigned __int128)((uint64_t)i * 0x9E3779B97F4A7C15ull)) % (uint64_t)(ns * stride));
  const float *q = pts + 3 * at;
  key[i] = encode_bins(axis_bin(q[0], scene[0], scene[3], scale, top), axis_bin(q[1], scene[1], scene[4], scale, top),
                       axis_bin(q[2], scene[2], scene[5], scale, top), 3) >> 23;
}
__global__ void __launch_bounds__(256) k_sample_triples(const uint64_t *__restrict__ key, int64_t ns, int *found) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i + 2 >= ns) return;
  if ((key[i] >> 8) == (key[i + 2] >> 8)) found[0] = 1;  // three equal top-32 keys
  if (key[i] == key[i + 2]) found[1] = 1;                // three equal top-40 keys
}
int choose_top_bits(Ctx &c, const float *pts, int64_t n, const float *scene) {
  if (n < (1 << 18)) return 32;  // small: a fallback costs little
  const int64_t stride = 128, ns = n / stride;
  DevBuf<uint64_t> k0((size_t)ns, c.stream), k1((size_t)ns, c.stream);
  DevBuf<uint32_t> v0((size_t)ns, c.stream), v1((size_t)ns, c.stream);
  DevBuf<int> found(2, c.stream);
  SPB_CUDA(cudaMemsetAsync(found.get(), 0, 2 * sizeof(int), c.stream));
  k_sample_top40<<<(unsigned)((ns + 255) / 256), 256, 0, c.stream>>>(pts, stride, ns, scene, k0.get());
  SPB_LAUNCHED();
  uint64_t *ka = k0.get(), *kb = k1.get();
  uint32_t *va = v0.get(), *vb = v1.get();
  radix_sort_pairs(c, &ka, &va, &kb, &vb, ns, 40, true);
  k_sample_triples<<<(unsigned)((ns + 255) / 256), 256, 0, c.stream>>>(ka, ns, found.get());
  SPB_LAUNCHED();
  int h[2] = {0, 0};
  peek(c, {{found.get(), h, sizeof(h)}});
  return !h[0] ? 32 : (!h[1] ? 40 : 0);
}
__global__ void __launch_bounds__(256) k_morton_top40(const float *__restrict__ pts, int64_t n,
                                                      const float *__restrict__ scene, uint64_t *__restrict__ key,
                                                      uint32_t *ghist = nullptr) {
  __shared__ uint32_t s_hist[5 * 256];
  HistAcc<5> H;
  H.init(s_hist, ghist);
  const int bits = 21;
  const uint32_t top = (1u << bits) - 1u;
  const double scale = (double)(1ull << bits);
  const float lo0 = scene[0], lo1 = scene[1], lo2 = scene[2], hi0 = scene[3], hi1 = scene[4], hi2 = scene[5];
  auto code = [&](float x, float y, float z) -> uint64_t {
    return encode_bins(axis_bin(x, lo0, hi0, scale, top), axis_bin(y, lo1, hi1, scale, top),
                       axis_bin(z, lo2, hi2, scale, top), 3) >> 23;
  };
  const int64_t chunks = n / 4;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const int64_t t0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  for (int64_t ch = t0; ch < chunks; ch += stride) {
    float x[4], y[4], z[4];
    load4pts(pts, ch, x, y, z);
    const ulonglong2 a = make_ulonglong2(code(x[0], y[0], z[0]), code(x[1], y[1], z[1]));
    const ulonglong2 b = make_ulonglong2(code(x[2], y[2], z[2]), code(x[3], y[3], z[3]));
    reinterpret_cast<ulonglong2 *>(key)[2 * ch] = a;
    reinterpret_cast<ulonglong2 *>(key)[2 * ch + 1] = b;
    H.add(a.x);
    H.add(a.y);
    H.add(b.x);
    H.add(b.y);
  }
  for (int64_t i = chunks * 4 + t0; i < n; i += stride) {
    key[i] = code(pts[3 * i], pts[3 * i + 1], pts[3 * i + 2]);
    H.add(key[i]);
  }
  H.flush();
}

void build_tree(Ctx &c, const float *objects, int64_t n, int dim, bool points, int width, Tree &t) {
  t.n = n;
  t.dim = dim;
  t.width = width;
  t.points = points;
  t.stream = c.stream;
  t.scene = static_cast<decltype(t.scene)>(cache_alloc(6 * sizeof(float), c.stream));
  DevBuf<int> bad(1, c.stream);
  mark(c, "start");
  scene_bounds(c, objects, n, dim, points, t.scene, bad.get());
  mark(c, "bounds");
  if (c.async()) {
    // no host round trip: fold the flag into the context's deferred error
    k_flag_or<<<1, 1, 0, c.stream>>>(bad.get(), c.d_err);
    SPB_LAUNCHED();
  } else {
    int h_bad = 0;
    peek(c, {{bad.get(), &h_bad, sizeof(int)}});
    if (h_bad) throw InvalidArgument("bvh: non-finite object bounds");
  }
  if (n == 0) return;

  const int64_t num_nodes = 2 * n - 1;
  t.nodes = static_cast<decltype(t.nodes)>(cache_alloc((size_t)num_nodes * 2 * sizeof(float4), c.stream));
  t.perm = static_cast<decltype(t.perm)>(cache_alloc((size_t)n * sizeof(int32_t), c.stream));
  if (points) t.leafpt = static_cast<decltype(t.leafpt)>(cache_alloc((size_t)n * sizeof(float4), c.stream));

  DevBuf<uint64_t> k0(n, c.stream), k1(n, c.stream);
  DevBuf<uint32_t> v0(n, c.stream), v1(n, c.stream);
  DevBuf<int32_t> delta(n > 1 ? n - 1 : 1, c.stream), flags(n > 1 ? n - 1 : 1, c.stream);
  uint64_t *ka = k0.get(), *kb = k1.get();
  uint32_t *va = v0.get(), *vb = v1.get();
  const float4 *spts = nullptr;  // points in sorted order (the top-32 path writes them)
  const int topbits = (SPB_SORT_TOP32 && points && dim == 3 && width == 64 && n >= 2 && !c.async() &&
                       aligned16(objects))
                          ? choose_top_bits(c, objects, n, t.scene)
                          : 0;
  if (topbits) {
    if (topbits == 32) {
      uint32_t *k32a = reinterpret_cast<uint32_t *>(k0.get()), *k32b = k32a + n;
      DevBuf<uint32_t> hist(SPB_FUSED_HIST ? RS_HIST_ENTRIES(4) : 0, c.stream);
      if (SPB_FUSED_HIST) SPB_CUDA(cudaMemsetAsync(hist.get(), 0, hist.n * sizeof(uint32_t), c.stream));
      k_morton_top32<<<grid_for((n + 3) / 4, 256, 148 * 16), 256, 0, c.stream>>>(objects, n, width, t.scene, k32a,
                                                                                   hist.get());
      SPB_LAUNCHED();
      mark(c, "morton");
      radix_sort_pairs(c, &k32a, &va, &k32b, &vb, n, 32, /*vals_iota=*/true, hist.get());
    } else {
      DevBuf<uint32_t> hist(SPB_FUSED_HIST ? RS_HIST_ENTRIES(5) : 0, c.stream);
      if (SPB_FUSED_HIST) SPB_CUDA(cudaMemsetAsync(hist.get(), 0, hist.n * sizeof(uint32_t), c.stream));
      k_morton_top40<<<grid_for((n + 3) / 4, 256, 148 * 16), 256, 0, c.stream>>>(objects, n, t.scene, k0.get(),
                                                                                   hist.get());
      SPB_LAUNCHED();
      mark(c, "morton");
      uint32_t *k32 = reinterpret_cast<uint32_t *>(k1.get());
      radix_sort_pairs_40(c, k0.get(), &va, &vb, k32, k32 + n, n, /*vals_iota=*/true, hist.get());
    }
    // scratch in the node array (written by the hierarchy afterwards)
    float4 *tpt = reinterpret_cast<float4 *>(t.nodes);
    uint64_t *tcode = reinterpret_cast<uint64_t *>(tpt + n);
    DevBuf<int> ovf(1, c.stream);
    SPB_CUDA(cudaMemsetAsync(ovf.get(), 0, sizeof(int), c.stream));
    k_fix_gather<<<(unsigned)((n + 256 * FIX_ILP - 1) / (256 * FIX_ILP)), 256, 0, c.stream>>>(
        objects, n, width, t.scene, va, tcode, tpt);
    SPB_LAUNCHED();
    {
      static std::mutex mu;
      static uint64_t opted = 0;
      std::lock_guard<std::mutex> g(mu);
      if (c.device >= 64 || !((opted >> c.device) & 1)) {
        SPB_CUDA(cudaFuncSetAttribute(k_fix_runs_win<31>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)FIX_SMEM));
        SPB_CUDA(cudaFuncSetAttribute(k_fix_runs_win<23>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)FIX_SMEM));
        if (c.device < 64) opted |= 1ull << c.device;
      }
    }
    const unsigned gw = (unsigned)((n + FIX_CH - 1) / FIX_CH);
    if (topbits == 32)
      k_fix_runs_win<31><<<gw, 256, FIX_SMEM, c.stream>>>(n, tcode, tpt, t.leafpt, delta.get(), ovf.get());
    else
      k_fix_runs_win<23><<<gw, 256, FIX_SMEM, c.stream>>>(n, tcode, tpt, t.leafpt, delta.get(), ovf.get());
    SPB_LAUNCHED();
    int h_ovf = 0;
    peek(c, {{ovf.get(), &h_ovf, sizeof(int)}});
    c.count("sort_top_bits", topbits);
    c.count("sort_fallback", h_ovf);
    if (!h_ovf) {
      spts = t.leafpt;  // sorted points, their indices in .w, and D written
    } else {
      va = v0.get();  // a run longer than FIX_MAX_RUN: the full 63-bit sort below
      vb = v1.get();
    }
  }
  if (!spts) {
    morton_codes(c, objects, n, dim, points, width, t.scene, k0.get(), nullptr);
    mark(c, "morton");
    radix_sort_pairs(c, &ka, &va, &kb, &vb, n, (width / dim) * dim, /*vals_iota=*/true);
  }
  mark(c, "sort");
  if (n > 1) {
    if (!spts) {
      k_delta<<<grid_for(n, 256, 148 * 16), 256, 0, c.stream>>>(ka, va, n, width, delta.get());
      SPB_LAUNCHED();
    }
    SPB_CUDA(cudaMemsetAsync(flags.get(), 0xff, (size_t)(n - 1) * sizeof(int32_t), c.stream));
  }
  unsigned g = (unsigned)((n + CLIMB_BLK - 1) / CLIMB_BLK);
  ClimbQueue q(c, n, SPB_CLIMB_LEVELS_POINTS);
  if (points)
    k_hierarchy<true><<<g, CLIMB_BLK, 0, c.stream>>>(n, delta.get(), va, objects, dim, t.nodes, flags.get(), t.perm,
                                               t.leafpt, q.levels, q.buf.get(), q.count.get(), spts);
  else
    k_hierarchy<false><<<g, CLIMB_BLK, 0, c.stream>>>(n, delta.get(), va, objects, dim, t.nodes, flags.get(), t.perm,
                                                nullptr, q.levels, q.buf.get(), q.count.get(), nullptr);
  SPB_LAUNCHED();
  q.finish(c, n, delta.get(), t.nodes, flags.get());
  mark(c, "hierarchy");
}

void build_sorted_hierarchy(Ctx &c, const uint64_t *keys, int64_t m, int dim, const float *boxes, Tree &t,
                            DevBuf<int32_t> *delta_in) {
  t.n = m;
  t.dim = dim;
  t.width = 64;
  t.points = false;
  t.stream = c.stream;
  if (m == 0) return;
  // boxes == nullptr: the caller allocated t.nodes and wrote the leaf nodes
  if (boxes) t.nodes = static_cast<decltype(t.nodes)>(cache_alloc((size_t)(2 * m - 1) * 2 * sizeof(float4), c.stream));
  // leaves are the objects in order: no permutation array (t.perm stays null)
  DevBuf<int32_t> own_delta, flags(m > 1 ? m - 1 : 1, c.stream);
  DevBuf<int32_t> &delta = delta_in ? *delta_in : own_delta;
  if (!delta_in) own_delta = DevBuf<int32_t>(m > 1 ? m - 1 : 1, c.stream);
  if (m > 1) {
    if (!delta_in) {
      k_delta<<<grid_for(m, 256, 148 * 16), 256, 0, c.stream>>>(keys, nullptr, m, 64, delta.get());
      SPB_LAUNCHED();
    }
    SPB_CUDA(cudaMemsetAsync(flags.get(), 0xff, (size_t)(m - 1) * sizeof(int32_t), c.stream));
  }
  ClimbQueue q(c, m, SPB_CLIMB_LEVELS_CELLS);
  k_hierarchy<false><<<(unsigned)((m + CLIMB_BLK - 1) / CLIMB_BLK), CLIMB_BLK, 0, c.stream>>>(m, delta.get(), nullptr, boxes, dim, t.nodes,
                                                                        flags.get(), nullptr, nullptr, q.levels,
                                                                        q.buf.get(), q.count.get(), nullptr);
  SPB_LAUNCHED();
  q.finish(c, m, delta.get(), t.nodes, flags.get());
}

void sort_points(Ctx &c, const float *pts, int64_t n, int dim, int32_t *order) {
  if (n <= 0) return;
  DevBuf<float> scene(6, c.stream);
  DevBuf<int> bad(1, c.stream);
  scene_bounds(c, pts, n, dim, true, scene.get(), bad.get());
  DevBuf<uint64_t> k0(n, c.stream), k1(n, c.stream);
  DevBuf<uint32_t> v0(n, c.stream), v1(n, c.stream);
  if (SPB_SORT_TOP32 && dim == 3 && n >= 2 && !c.async() && aligned16(pts) &&
      choose_top_bits(c, pts, n, scene.get()) == 32) {
    // top 32 bits in four passes, runs ordered by the full codes (k1)
    uint32_t *k32a = reinterpret_cast<uint32_t *>(k0.get()), *k32b = k32a + n;
    uint32_t *va = v0.get(), *vb = v1.get();
    DevBuf<uint32_t> hist(SPB_FUSED_HIST ? RS_HIST_ENTRIES(4) : 0, c.stream);
    if (hist.n) SPB_CUDA(cudaMemsetAsync(hist.get(), 0, hist.n * sizeof(uint32_t), c.stream));
    k_morton_top32_full<<<grid_for((n + 3) / 4, 256, 148 * 16), 256, 0, c.stream>>>(pts, n, 64, scene.get(), k32a,
                                                                                   k1.get(), hist.get());
    SPB_LAUNCHED();
    radix_sort_pairs(c, &k32a, &va, &k32b, &vb, n, 32, /*vals_iota=*/true, hist.get());
    DevBuf<int> ovf(1, c.stream);
    SPB_CUDA(cudaMemsetAsync(ovf.get(), 0, sizeof(int), c.stream));
    k_fix_runs_order<<<(unsigned)((n + 255) / 256), 256, 0, c.stream>>>(k32a, n, va, k1.get(), order, ovf.get());
    SPB_LAUNCHED();
    int h_ovf = 0;
    peek(c, {{ovf.get(), &h_ovf, sizeof(int)}});
    if (!h_ovf) return;
  }
  morton_codes(c, pts, n, dim, true, 64, scene.get(), k0.get(), nullptr);
  uint64_t *ka = k0.get(), *kb = k1.get();
  uint32_t *va = v0.get(), *vb = v1.get();
  radix_sort_pairs(c, &ka, &va, &kb, &vb, n, (64 / dim) * dim, /*vals_iota=*/true);
  SPB_CUDA(cudaMemcpyAsync(order, va, (size_t)n * sizeof(int32_t), cudaMemcpyDeviceToDevice, c.stream));
}

}  // namespace spb
