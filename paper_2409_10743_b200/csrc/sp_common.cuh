// Shared device definitions for the B200 geometric-search path.
//
// Node layout (HBM): one unified array of 2n-1 nodes indexed by the
// reference's NodeRef numbering (bvh.hpp:20-28) — internal nodes [0, n-1)
// in Karras order, leaves [n-1, 2n-1) in Morton order — each node one 32-byte
// sector read as two float4:
//     lo = {min.x, min.y, min.z, bits(left child | object index)}
//     hi = {max.x, max.y, max.z, bits(rope)}
// 2-D data is stored with z = 0, which adds an exact 0.0 to every distance
// accumulation, so one set of kernels serves both dimensions; only the Morton
// stage and the dense grid look at `dim`.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>
#include <string.h>

#include <cmath>

#include <stdexcept>
#include <string>

namespace spb {

constexpr int32_t kSentinel = -1;
constexpr int kNumSMs = 148;

struct CudaError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct InvalidArgument : std::invalid_argument {
  using std::invalid_argument::invalid_argument;
};
struct NcclError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct CapacityError : std::runtime_error {
  CapacityError() : std::runtime_error("crs result exceeds capacity") {}
};

#define SPB_CUDA(expr)                                                                                   \
  do {                                                                                                   \
    cudaError_t _e = (expr);                                                                             \
    if (_e != cudaSuccess)                                                                               \
      throw ::spb::CudaError(std::string(#expr) + ": " + cudaGetErrorString(_e) + " (" + __FILE__ + ":" + \
                             std::to_string(__LINE__) + ")");                                            \
  } while (0)

// Launch bookkeeping: every kernel launch in the library goes through this
// macro so the context can report how many of OUR kernels ran.
extern thread_local int64_t *g_launch_counter;
#define SPB_LAUNCHED()                                 \
  do {                                                 \
    SPB_CUDA(cudaGetLastError());                      \
    if (::spb::g_launch_counter) ++*::spb::g_launch_counter; \
  } while (0)

inline unsigned grid_for(int64_t n, int block, int64_t cap = 148LL * 32) {
  int64_t g = (n + block - 1) / block;
  if (g < 1) g = 1;
  if (g > cap) g = cap;
  return (unsigned)g;
}

// ---- exact comparison arithmetic (geometry.hpp:73-96, 116-119) -------------
// The reference decides `float(sqrt(S)) <= r` with S the double-accumulated
// squared gap.  Since S -> float(sqrt_rn(S)) is monotone, that equals
// `S <= T(r)` for T(r) = the largest double with float(sqrt(T)) <= r.  T is
// found once per radius (a few ulps from (r + ulp/2)^2) and the hot loops
// never take a square root.  All arithmetic uses explicit _rn intrinsics so
// no FMA contraction can change a bit.
__host__ __device__ inline double next_up(double x) {
#ifdef __CUDA_ARCH__
  return __longlong_as_double(__double_as_longlong(x) + 1);
#else
  int64_t b;
  memcpy(&b, &x, 8);
  ++b;
  memcpy(&x, &b, 8);
  return x;
#endif
}
__host__ __device__ inline double next_down(double x) {
#ifdef __CUDA_ARCH__
  return __longlong_as_double(__double_as_longlong(x) - 1);
#else
  int64_t b;
  memcpy(&b, &x, 8);
  --b;
  memcpy(&x, &b, 8);
  return x;
#endif
}

__host__ __device__ __forceinline__ bool sqrt_le(double s, float r) {
#ifdef __CUDA_ARCH__
  return __double2float_rn(__dsqrt_rn(s)) <= r;
#else
  return (float)std::sqrt(s) <= r;  // IEEE sqrt, round-to-nearest cast
#endif
}

// T(r); negative/NaN r -> -1 (no squared gap qualifies); +inf -> +inf.
// Start from m^2, m = r + ulp(r)/2 (exact in double: m has <= 25 significant
// bits), then step the few ulps the double rounding of sqrt can move it.
__host__ __device__ inline double radius_threshold(float r) {
  if (!(r >= 0.f)) return -1.0;
  const double kInf = 1.0 / 0.0;
  if (r > 3.4028234663852886e38f) return kInf;
  double ulp;
  if (r == 3.4028234663852886e38f) {
    ulp = 20282409603651670423947251286016.0;  // 2^104
  } else {
#ifdef __CUDA_ARCH__
    ulp = (double)nextafterf(r, kInf) - (double)r;
#else
    ulp = (double)std::nextafter(r, (float)kInf) - (double)r;
#endif
  }
  double m = (double)r + 0.5 * ulp;
  double t = m * m;
  for (int i = 0; i < 64 && sqrt_le(next_up(t), r); ++i) t = next_up(t);
  for (int i = 0; i < 64 && t > 0.0 && !sqrt_le(t, r); ++i) t = next_down(t);
  return t;
}

// Squared distance from c to the box [lo, hi] accumulated exactly as
// min_distance does: gap_k = max(lo-c, c-hi, 0) in double, s = ((0+g0²)+g1²)+g2².
__device__ __forceinline__ double gap2(float cx, float cy, float cz, const float4 &lo, const float4 &hi) {
  double gx = fmax(fmax(__dsub_rn((double)lo.x, (double)cx), __dsub_rn((double)cx, (double)hi.x)), 0.0);
  double gy = fmax(fmax(__dsub_rn((double)lo.y, (double)cy), __dsub_rn((double)cy, (double)hi.y)), 0.0);
  double gz = fmax(fmax(__dsub_rn((double)lo.z, (double)cz), __dsub_rn((double)cz, (double)hi.z)), 0.0);
  double s = __dmul_rn(gx, gx);
  s = __dadd_rn(s, __dmul_rn(gy, gy));
  s = __dadd_rn(s, __dmul_rn(gz, gz));
  return s;
}

// Point-to-point squared distance (distance(), geometry.hpp:73-81).
__device__ __forceinline__ double dist2(float ax, float ay, float az, float bx, float by, float bz) {
  double dx = __dsub_rn((double)ax, (double)bx);
  double dy = __dsub_rn((double)ay, (double)by);
  double dz = __dsub_rn((double)az, (double)bz);
  double s = __dmul_rn(dx, dx);
  s = __dadd_rn(s, __dmul_rn(dy, dy));
  s = __dadd_rn(s, __dmul_rn(dz, dz));
  return s;
}

// Closed-interval box overlap (geometry.hpp:121-128).
__device__ __forceinline__ bool box_touch(const float4 &alo, const float4 &ahi, const float *b) {
  return !(alo.x > b[3] || b[0] > ahi.x || alo.y > b[4] || b[1] > ahi.y || alo.z > b[5] || b[2] > ahi.z);
}

// std::min/std::max tie semantics (keep the first unless the second is
// strictly smaller/larger) so unions reproduce the reference's signed zeros.
__host__ __device__ __forceinline__ float keep_min(float a, float b) { return b < a ? b : a; }
__host__ __device__ __forceinline__ float keep_max(float a, float b) { return a < b ? b : a; }

// Monotone int encoding of floats for atomicMin/atomicMax bounds.
__device__ __forceinline__ int32_t ord_of(float f) {
  int32_t i = __float_as_int(f);
  return i >= 0 ? i : (i ^ 0x7fffffff);
}
__host__ __device__ __forceinline__ float float_of_ord(int32_t i) {
  int32_t b = i >= 0 ? i : (i ^ 0x7fffffff);
#ifdef __CUDA_ARCH__
  return __int_as_float(b);
#else
  float f;
  memcpy(&f, &b, 4);
  return f;
#endif
}

// Fused radix histogram (radix_sort_pairs' hist_in): the kernel that writes
// the sort keys also counts their NPASS 8-bit digits in shared memory and adds
// the block's counts to the global ones once, so the sort skips its own
// counting pass over the keys.  Every thread of the block must call init and
// flush (no early return between them).
template <int NPASS>
struct HistAcc {
  uint32_t *sh;  // NPASS * 256 shared counters
  uint32_t *g;   // global counts (nullptr: no histogram)
  __device__ __forceinline__ void init(uint32_t *shared, uint32_t *global) {
    sh = shared;
    g = global;
    if (!g) return;
    for (int i = threadIdx.x; i < NPASS * 256; i += blockDim.x) sh[i] = 0;
    __syncthreads();
  }
  __device__ __forceinline__ void add(uint64_t k) {
    if (!g) return;
#pragma unroll
    for (int p = 0; p < NPASS; ++p) atomicAdd(&sh[p * 256 + (uint32_t)((k >> (8 * p)) & 0xffu)], 1u);
  }
  __device__ __forceinline__ void flush() {
    if (!g) return;
    __syncthreads();
    for (int i = threadIdx.x; i < NPASS * 256; i += blockDim.x)
      if (sh[i]) atomicAdd(&g[i], sh[i]);
  }
};

__device__ __forceinline__ float4 ld_node(const float4 *nodes, int64_t i) { return __ldg(nodes + i); }
// Both halves of node j (float4 2j and 2j + 1, one 32-byte sector) in one
// 256-bit read-only load (LDG.E.ENL2.256 on sm_100a): one L1 request per node
// visit instead of two -- the traversal walks are bound by L1 requests on
// L1-hot nodes, not by HBM.
#ifndef SPB_LD256
#define SPB_LD256 1
#endif
__device__ __forceinline__ void ld_node2(const float4 *nodes, int64_t j, float4 &lo, float4 &hi) {
#if SPB_LD256
  asm("ld.global.nc.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
      : "=f"(lo.x), "=f"(lo.y), "=f"(lo.z), "=f"(lo.w), "=f"(hi.x), "=f"(hi.y), "=f"(hi.z), "=f"(hi.w)
      : "l"(nodes + 2 * j));
#else
  lo = __ldg(nodes + 2 * j);
  hi = __ldg(nodes + 2 * j + 1);
#endif
}

// Four consecutive 3-D points (12 floats) as three 16-byte loads; the array
// must be 16-byte aligned.
__device__ __forceinline__ void load4pts(const float *__restrict__ pts, int64_t chunk, float x[4], float y[4],
                                         float z[4]) {
  const float4 *v = reinterpret_cast<const float4 *>(pts) + 3 * chunk;
  const float4 a = __ldg(v), b = __ldg(v + 1), d = __ldg(v + 2);
  x[0] = a.x; y[0] = a.y; z[0] = a.z;
  x[1] = a.w; y[1] = b.x; z[1] = b.y;
  x[2] = b.z; y[2] = b.w; z[2] = d.x;
  x[3] = d.y; y[3] = d.z; z[3] = d.w;
}
__host__ __device__ __forceinline__ bool aligned16(const void *p) {
  return (reinterpret_cast<uintptr_t>(p) & 15) == 0;
}

// Point i of a 16-byte aligned float[3n] array by one or two 16-byte loads of
// the aligned blocks holding its 12 bytes (three 4-byte loads would each go to
// L2 on their own: a random gather then costs ~4 sectors of DRAM traffic per
// point instead of ~2).  The tail stays inside the array.
__device__ __forceinline__ void gather_pt3(const float *__restrict__ pts, int64_t n, int64_t i, float &x, float &y,
                                           float &z) {
  const int64_t f = 3 * i, blk = f >> 2;
  const int off = (int)(f & 3);
  const float4 *v = reinterpret_cast<const float4 *>(pts);
  if (off >= 2 && blk + 1 > (3 * n - 1) >> 2) {
    x = __ldg(pts + f);
    y = __ldg(pts + f + 1);
    z = __ldg(pts + f + 2);
    return;
  }
  const float4 a = __ldg(v + blk);
  const float4 b = off >= 2 ? __ldg(v + blk + 1) : a;
  x = off == 0 ? a.x : (off == 1 ? a.y : (off == 2 ? a.z : a.w));
  y = off == 0 ? a.y : (off == 1 ? a.z : (off == 2 ? a.w : b.x));
  z = off == 0 ? a.z : (off == 1 ? a.w : (off == 2 ? b.x : b.y));
}

// Decoupled look-back status words (bypass L1: other CTAs publish them).
#ifndef SPB_LOOKBACK_GPU
#define SPB_LOOKBACK_GPU 1
#endif
// Look-back status words: relaxed GPU-scope loads and stores (L2-coherent;
// the status value itself carries the data, so no ordering is needed).
__device__ __forceinline__ void st_volatile_u64(unsigned long long *p, unsigned long long v) {
#if SPB_LOOKBACK_GPU
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
#else
  asm volatile("st.volatile.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
#endif
}
__device__ __forceinline__ unsigned long long ld_volatile_u64(const unsigned long long *p) {
  unsigned long long v;
#if SPB_LOOKBACK_GPU
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
#else
  asm volatile("ld.volatile.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
#endif
  return v;
}



// ---- SM-affine work schedule ---------------------------------------------------
// For items sorted in space-filling-curve order (queries, cells): [0, total)
// is cut into one contiguous slice per SM and every warp takes 32-item chunks
// from the slice of the SM it runs on, then (once that is drained) from the
// others.  All warps resident on an SM then walk the same neighbourhood of a
// tree and share its nodes in L1, instead of the 10-16 distant windows that
// round-robin block dispatch puts on one SM.  Launch a grid that is fully
// resident (SmSlices::grid); a lane's item is -1 past the end of a chunk.
__device__ __forceinline__ uint32_t sm_id() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(r));
  return r;
}

struct SmSliceWalk {
  int64_t total, per;
  unsigned long long *ctr;
  int nslices, own, t = 0;
  __device__ SmSliceWalk(int64_t total_, unsigned long long *ctr_, int nslices_)
      : total(total_), per((total_ + nslices_ - 1) / nslices_), ctr(ctr_), nslices(nslices_),
        own((int)(sm_id() % (uint32_t)nslices_)) {}
  // Next item of this lane (warp-uniform return: false when all are done).
  // The lanes probe 32 slices' counters at once, so finding work elsewhere
  // after the own slice is drained costs one round trip per 32 slices.
  __device__ bool next(int64_t &item) {
    const int lane = threadIdx.x & 31;
    __syncwarp();
    while (t < nslices) {
      const int tl = t + lane;
      bool avail = false;
      if (tl < nslices) {
        const int s = own + tl < nslices ? own + tl : own + tl - nslices;
        const int64_t lo = (int64_t)s * per, hi = lo + per < total ? lo + per : total;
        avail = lo < hi && (int64_t) * (volatile unsigned long long *)(ctr + s) < hi - lo;
      }
      const unsigned mask = __ballot_sync(0xffffffffu, avail);
      if (!mask) {
        t += 32;
        continue;
      }
      t += __ffs(mask) - 1;
      const int s = own + t < nslices ? own + t : own + t - nslices;
      const int64_t lo = (int64_t)s * per, hi = lo + per < total ? lo + per : total;
      unsigned long long base = 0;
      if (lane == 0) base = atomicAdd(ctr + s, 32ull);
      base = __shfl_sync(0xffffffffu, base, 0);
      if ((int64_t)base < hi - lo) {
        const int64_t i = lo + (int64_t)base + lane;
        item = i < hi ? i : -1;
        return true;
      }
      ++t;
    }
    return false;
  }
};

}  // namespace spb
