// Host-side plumbing on the path's boundary: the reference's synthetic point
// generators (generate.cpp:17-66), reproduced with the same standard-library
// engine and distributions so `--generate` specs give identical bits.
#include <stdint.h>

#include <algorithm>
#include <random>
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

}  // extern "C"
