// Host-side plumbing on the path's boundary: the reference's synthetic point
// generators (generate.cpp:17-66), reproduced with the same standard-library
// engine and distributions so `--generate` specs give identical bits.
#include <stdint.h>

#include <algorithm>
#include <cmath>
#include <random>
#include <thread>
#include <vector>

#include "../../include/sp_b200.h"

extern "C" {

// kind 0: uniform(n, dim, extent) — one uniform_real_distribution<double>(0,
// extent) draw per coordinate from mt19937_64(seed), cast to float.
// kind 1: gaussian_clusters(n, dim, k, sigma, extent, seed) — k centres drawn
// first, then every coordinate centre + N(0, sigma) clamped to [0, extent];
// point i belongs to cluster min(i / ceil(n/k), k-1).
int sp_generate_reference(int kind, int64_t n, int dim, int32_t k, double sigma, double extent, uint64_t seed,
                          float *out) {
  if (n < 0 || (dim != 2 && dim != 3) || !(extent > 0)) return SP_EINVAL;
  std::mt19937_64 rng(seed);
  std::uniform_real_distribution<double> unif(0.0, extent);
  if (kind == 0) {
    for (int64_t i = 0; i < n * dim; ++i) out[i] = static_cast<float>(unif(rng));
    return SP_OK;
  }
  if (k < 1 || !(sigma >= 0)) return SP_EINVAL;
  std::normal_distribution<double> gauss(0.0, sigma);
  std::vector<double> centre(static_cast<size_t>(k) * dim);
  for (double &c : centre) c = unif(rng);
  const int64_t per = (n + k - 1) / k;
  for (int64_t i = 0; i < n; ++i) {
    const int64_t c = std::min<int64_t>(i / per, k - 1);
    for (int d = 0; d < dim; ++d) {
      double v = centre[static_cast<size_t>(c * dim + d)] + gauss(rng);
      out[i * dim + d] = static_cast<float>(std::clamp(v, 0.0, extent));
    }
  }
  return SP_OK;
}

// Rows [first, first + count) of the SURVEY §8(d) field H(n_total) =
// uniform(n_total/4, 3, 1, seed 2409) ++ gaussian_clusters(n_total - n_total/4,
// 3, k = max((n_total - n_total/4)/8192, 1), 0.001*cbrt(2^26/n_total), 1,
// seed 2410), as the reference's generate() draws them (generate.cpp:17-66).
// The two generators are independent streams and run on two threads; each
// must still draw every value before `first`, but only the slice is stored,
// so a rank of the slab path holds its own share only.
int sp_generate_reference_field(int64_t n_total, int64_t first, int64_t count, float *out) {
  if (n_total < 0 || first < 0 || count < 0 || first + count > n_total || (count > 0 && !out)) return SP_EINVAL;
  const int64_t nbg = n_total / 4, nh = n_total - nbg;
  auto background = [&] {
    const int64_t lo = std::max<int64_t>(first, 0), hi = std::min<int64_t>(first + count, nbg);
    if (lo >= hi) return;
    std::mt19937_64 rng(2409);
    std::uniform_real_distribution<double> unif(0.0, 1.0);
    for (int64_t i = 0; i < hi * 3; ++i) {
      const float v = static_cast<float>(unif(rng));
      if (i >= lo * 3) out[i - first * 3] = v;
    }
  };
  auto halos = [&] {
    const int64_t lo = std::max<int64_t>(first, nbg) - nbg, hi = std::min<int64_t>(first + count, n_total) - nbg;
    if (lo >= hi) return;
    const int32_t k = (int32_t)std::max<int64_t>(nh / 8192, 1);
    const double sigma = 0.001 * std::cbrt(67108864.0 / (double)n_total);
    std::mt19937_64 rng(2410);
    std::uniform_real_distribution<double> unif(0.0, 1.0);
    std::normal_distribution<double> gauss(0.0, sigma);
    std::vector<double> centre(static_cast<size_t>(k) * 3);
    for (double &c : centre) c = unif(rng);
    const int64_t per = (nh + k - 1) / k;
    float *dst = out + (nbg + lo - first) * 3;
    for (int64_t i = 0; i < hi; ++i) {
      const int64_t c = std::min<int64_t>(i / per, k - 1);
      for (int d = 0; d < 3; ++d) {
        const double v = std::clamp(centre[static_cast<size_t>(c * 3 + d)] + gauss(rng), 0.0, 1.0);
        if (i >= lo) dst[(i - lo) * 3 + d] = static_cast<float>(v);
      }
    }
  };
  std::thread t(background);
  halos();
  t.join();
  return SP_OK;
}

}  // extern "C"
