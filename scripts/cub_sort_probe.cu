// Off-product yardstick: CUB's onesweep DeviceRadixSort::SortPairs
// on the same (u64 key, u32 value) pairs the library sorts — 63-bit point
// Morton codes (Bvh::build) and 39-bit cell keys (FoF grid) at 2^27 — timed
// with events, median of 7 after 2 warm-ups.  Not linked into the product.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a scripts/cub_sort_probe.cu -o /tmp/cub_sort_probe
#include <cub/device/device_radix_sort.cuh>
#include <cstdio>
#include <algorithm>
#include <vector>
#include <cstdint>

__global__ void fill(uint64_t *k, uint32_t *v, int64_t n, int bits, uint64_t seed) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    uint64_t x = (uint64_t)i * 0x9E3779B97F4A7C15ull + seed;
    x ^= x >> 31; x *= 0xBF58476D1CE4E5B9ull; x ^= x >> 27; x *= 0x94D049BB133111EBull; x ^= x >> 33;
    k[i] = bits >= 64 ? x : (x & ((1ull << bits) - 1));
    v[i] = (uint32_t)i;
  }
}

int main(int argc, char **argv) {
  const int64_t n = argc > 1 ? atoll(argv[1]) : (1ll << 27);
  for (int bits : {63, 39}) {
    uint64_t *k0, *k1; uint32_t *v0, *v1;
    cudaMalloc(&k0, n * 8); cudaMalloc(&k1, n * 8); cudaMalloc(&v0, n * 4); cudaMalloc(&v1, n * 4);
    size_t tmp_bytes = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, k0, k1, v0, v1, (int)n, 0, bits);
    void *tmp; cudaMalloc(&tmp, tmp_bytes);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    std::vector<float> ms;
    for (int it = 0; it < 9; ++it) {
      fill<<<148 * 16, 256>>>(k0, v0, n, bits, 12345);
      cudaEventRecord(a);
      cub::DeviceRadixSort::SortPairs(tmp, tmp_bytes, k0, k1, v0, v1, (int)n, 0, bits);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float t; cudaEventElapsedTime(&t, a, b);
      if (it >= 2) ms.push_back(t);
    }
    std::sort(ms.begin(), ms.end());
    const double med = ms[ms.size() / 2];
    printf("{\"probe\": \"cub::DeviceRadixSort::SortPairs\", \"n\": %lld, \"key_bits\": %d, \"ms\": %.3f, "
           "\"gpairs_s\": %.2f, \"cub_version\": %d}\n", (long long)n, bits, med, n / med / 1e6, CUB_VERSION);
    cudaFree(k0); cudaFree(k1); cudaFree(v0); cudaFree(v1); cudaFree(tmp);
  }
  return cudaGetLastError() == cudaSuccess ? 0 : 1;
}
