// Slab-decomposed friends-of-friends (sp_slabs.cu): the pipeline and its
// communicators, shared with the C ABI (sp_capi.cu).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <vector>

#include "sp_internal.hpp"
#include "sp_query.hpp"

namespace spb {

constexpr int kMaxSlabRanks = 32;

// Make `device` current for a scope (multi-device loops of one host thread).
struct ScopedDevice {
  int prev = -1;
  explicit ScopedDevice(int device) {
    cudaGetDevice(&prev);
    if (prev != device) cudaSetDevice(device);
  }
  ~ScopedDevice() {
    int cur = -1;
    cudaGetDevice(&cur);
    if (prev >= 0 && cur != prev) cudaSetDevice(prev);
  }
};

// One rank's part of a step: device rows [first, first + n) of the global
// point array (float[n*3]) and where its labels / core flags go.
struct SlabInput {
  Ctx *c = nullptr;
  const float *pts = nullptr;
  int64_t n = 0;
  int64_t first = 0;
  int32_t *labels = nullptr;
  uint8_t *core = nullptr;
};

struct SlabExchange;
void nccl_unique_id(uint8_t out[128]);
SlabExchange *nccl_exchange_create(int device, int nranks, int rank, const uint8_t id[128]);
SlabExchange *nccl_exchange_wrap(void *nccl_comm);
int exchange_size(const SlabExchange *x);
int exchange_rank(const SlabExchange *x);
void exchange_destroy(SlabExchange *x);

// The step over the ranks this thread drives (inputs[l] is rank
// x.rank_of(l)): one entry under NCCL, all ranks for fof_slabs_multi.
void fof_slabs(std::vector<SlabInput> &inputs, SlabExchange &x, float eps);
// All ranks in this process (contexts on one device or several).
void fof_slabs_multi(std::vector<SlabInput> &inputs, float eps);

}  // namespace spb
