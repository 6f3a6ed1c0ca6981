// Synthetic inputs for benchmarks (no reference counterpart on the hot path):
// the SURVEY §8(d) HACC-like field shape — 25% uniform background plus
// Gaussian halos of 8192 points with sigma = 0.001*cbrt(2^26/n), clamped to
// the unit cube — from a counter-based Philox4x32-10 stream, so every slice of
// the global field can be produced independently on any rank.  (Parity tests
// use the reference's own mt19937_64 generator instead; see tests/.)
#include <cuda_runtime.h>
#include <stdint.h>

#include <cmath>

#include "sp_common.cuh"
#include "sp_internal.hpp"
#include "sp_query.hpp"

namespace spb {

__device__ __forceinline__ uint4 philox4x32_10(uint4 ctr, uint2 key) {
  const uint32_t M0 = 0xD2511F53u, M1 = 0xCD9E8D57u, W0 = 0x9E3779B9u, W1 = 0xBB67AE85u;
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    const uint32_t hi0 = __umulhi(M0, ctr.x), lo0 = M0 * ctr.x;
    const uint32_t hi1 = __umulhi(M1, ctr.z), lo1 = M1 * ctr.z;
    ctr = make_uint4(hi1 ^ ctr.y ^ key.x, lo1, hi0 ^ ctr.w ^ key.y, lo0);
    key.x += W0;
    key.y += W1;
  }
  return ctr;
}

// 24-bit uniform float in [0, 1)
__device__ __forceinline__ float u01(uint32_t x) { return (float)(x >> 8) * (1.0f / 16777216.0f); }
// 53-bit uniform double in (0, 1]
__device__ __forceinline__ double u01d(uint32_t a, uint32_t b) {
  return ((double)(((uint64_t)a << 21) ^ (uint64_t)(b >> 11)) + 1.0) * (1.0 / 9007199254740992.0);
}

__global__ void k_field(int64_t n_total, int64_t first, int64_t count, uint64_t seed, double sigma,
                        float *__restrict__ out) {
  const int64_t nbg = n_total / 4;
  const int64_t nh = n_total - nbg;
  int64_t nhalo = nh / 8192;
  if (nhalo < 1) nhalo = 1;
  const int64_t block = (nh + nhalo - 1) / nhalo;
  const uint2 key = make_uint2((uint32_t)seed, (uint32_t)(seed >> 32));
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < count; j += stride) {
    const int64_t i = first + j;
    float x, y, z;
    if (i < nbg) {
      uint4 r = philox4x32_10(make_uint4((uint32_t)i, (uint32_t)(i >> 32), 0u, 0x5eedu), key);
      x = u01(r.x); y = u01(r.y); z = u01(r.z);
    } else {
      int64_t h = (i - nbg) / block;
      if (h >= nhalo) h = nhalo - 1;
      uint4 cr = philox4x32_10(make_uint4((uint32_t)h, (uint32_t)(h >> 32), 1u, 0xce17u), key);
      const double cx = u01(cr.x), cy = u01(cr.y), cz = u01(cr.z);
      uint4 a = philox4x32_10(make_uint4((uint32_t)i, (uint32_t)(i >> 32), 2u, 0x9a55u), key);
      uint4 b = philox4x32_10(make_uint4((uint32_t)i, (uint32_t)(i >> 32), 3u, 0x9a55u), key);
      // Box-Muller: three normals from two pairs of uniforms
      const double r0 = sqrt(-2.0 * log(u01d(a.x, a.y))), t0 = 6.283185307179586 * u01d(a.z, a.w);
      const double r1 = sqrt(-2.0 * log(u01d(b.x, b.y))), t1 = 6.283185307179586 * u01d(b.z, b.w);
      double vx = cx + sigma * r0 * cos(t0), vy = cy + sigma * r0 * sin(t0), vz = cz + sigma * r1 * cos(t1);
      x = (float)fmin(fmax(vx, 0.0), 1.0);
      y = (float)fmin(fmax(vy, 0.0), 1.0);
      z = (float)fmin(fmax(vz, 0.0), 1.0);
    }
    out[3 * j] = x;
    out[3 * j + 1] = y;
    out[3 * j + 2] = z;
  }
}

__global__ void k_uniform(int64_t n, int dim, uint64_t seed, float *__restrict__ out) {
  const uint2 key = make_uint2((uint32_t)seed, (uint32_t)(seed >> 32));
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    uint4 r = philox4x32_10(make_uint4((uint32_t)i, (uint32_t)(i >> 32), 0u, 0x5eedu), key);
    out[i * dim] = u01(r.x);
    out[i * dim + 1] = u01(r.y);
    if (dim == 3) out[i * dim + 2] = u01(r.z);
  }
}

void generate_field(Ctx &c, int64_t n_total, int64_t first, int64_t count, uint64_t seed, float *out) {
  if (count <= 0) return;
  const double sigma = 0.001 * std::cbrt(67108864.0 / (double)n_total);
  k_field<<<grid_for(count, 256, 148 * 16), 256, 0, c.stream>>>(n_total, first, count, seed, sigma, out);
  SPB_LAUNCHED();
}

void generate_uniform(Ctx &c, int64_t n, int dim, uint64_t seed, float *out) {
  if (n <= 0) return;
  k_uniform<<<grid_for(n, 256, 148 * 16), 256, 0, c.stream>>>(n, dim, seed, out);
  SPB_LAUNCHED();
}

}  // namespace spb
