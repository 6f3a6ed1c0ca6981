// The extern "C" boundary (include/sp_b200.h).  Translates host/device
// buffers, runs the device pipelines on the context stream, and maps C++
// exceptions to sp_status codes — nothing throws across the ABI.
#include <cuda_runtime.h>
#include <stdint.h>

#include <cstring>
#include <memory>
#include <mutex>
#include <new>
#include <string>
#include <vector>

#include "../../include/sp_b200.h"
#include "sp_common.cuh"
#include "sp_internal.hpp"
#include "sp_query.hpp"
#include "sp_slabs.hpp"

struct sp_ctx {
  spb::Ctx c;
};

struct sp_comm {
  spb::SlabExchange *x = nullptr;
};

struct sp_bvh {
  spb::Tree t;
  int device = 0;
};

namespace {

using spb::DevBuf;

// Host<->device copies run on the context's dedicated copy streams and are
// ordered against the compute stream with events, so with SP_FLAG_ASYNC the
// upload of call i+1 and the download of call i-1 overlap call i's kernels.
void stream_after(cudaStream_t waiter, cudaStream_t producer) {
  cudaEvent_t e;
  SPB_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  SPB_CUDA(cudaEventRecord(e, producer));
  SPB_CUDA(cudaStreamWaitEvent(waiter, e, 0));
  SPB_CUDA(cudaEventDestroy(e));
}

spb::Ctx::Staging &stage(spb::Ctx &c, bool input, size_t bytes) {
  const int parity = (int)(c.calls & 1);
  int &used = input ? c.in_used : c.out_used;
  if (used >= 8) throw spb::CudaError("too many host arrays in one call");
  spb::Ctx::Staging &s = (input ? c.in_stage : c.out_stage)[parity][used++];
  if (!s.done) SPB_CUDA(cudaEventCreateWithFlags(&s.done, cudaEventDisableTiming));
  if (s.cap < bytes) {
    // grow (rare): make sure nobody still uses the old block, then replace it
    SPB_CUDA(cudaEventSynchronize(s.done));
    if (s.p) SPB_CUDA(cudaFree(s.p));
    s.p = nullptr;
    s.cap = 0;
    if (cudaMalloc(&s.p, bytes) != cudaSuccess) {
      // out of memory: other streams' cached scratch blocks may hold it
      cudaGetLastError();
      spb::cache_drain();
      SPB_CUDA(cudaMalloc(&s.p, bytes));
    }
    s.cap = bytes;
  }
  return s;
}

// Input array: device pointer as-is, or a device copy of a host array in a
// double-buffered staging slot, uploaded on the H2D stream once the slot's
// previous consumer (two calls ago) has finished.
template <class T>
struct In {
  const T *p = nullptr;
  spb::Ctx::Staging *st = nullptr;
  spb::Ctx *ctx = nullptr;
  In(spb::Ctx &c, const T *src, size_t count, int mem) {
    if (!src || count == 0) return;
    if (mem == SP_MEM_DEVICE) {
      p = src;
      return;
    }
    st = &stage(c, true, count * sizeof(T));
    ctx = &c;
    SPB_CUDA(cudaStreamWaitEvent(c.h2d, st->done, 0));
    SPB_CUDA(cudaMemcpyAsync(st->p, src, count * sizeof(T), cudaMemcpyHostToDevice, c.h2d));
    stream_after(c.stream, c.h2d);
    p = static_cast<const T *>(st->p);
  }
  ~In() {
    if (st) cudaEventRecord(st->done, ctx->stream);  // consumed by this call's kernels
  }
};

// Output array: device pointer as-is, or a staging slot the kernels write
// (after its previous download finished) and flush() downloads on the D2H
// stream once the compute stream has produced it.
template <class T>
struct Out {
  T *p = nullptr;
  T *host = nullptr;
  size_t count = 0;
  spb::Ctx::Staging *st = nullptr;
  Out(spb::Ctx &c, T *dst, size_t n, int mem) : count(n) {
    if (!dst || n == 0) return;
    if (mem == SP_MEM_DEVICE) {
      p = dst;
      return;
    }
    st = &stage(c, false, n * sizeof(T));
    SPB_CUDA(cudaStreamWaitEvent(c.stream, st->done, 0));
    p = static_cast<T *>(st->p);
    host = dst;
  }
  void flush(spb::Ctx &c) {
    if (!host) return;
    stream_after(c.d2h, c.stream);
    SPB_CUDA(cudaMemcpyAsync(host, st->p, count * sizeof(T), cudaMemcpyDeviceToHost, c.d2h));
    SPB_CUDA(cudaEventRecord(st->done, c.d2h));
  }
};

struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    cudaGetDevice(&prev);
    if (prev != dev) cudaSetDevice(dev);
  }
  ~DeviceGuard() {
    int cur = -1;
    cudaGetDevice(&cur);
    if (prev >= 0 && cur != prev) cudaSetDevice(prev);
  }
};

// fresh = false (sp_ctx_synchronize): not a pipeline call, so the marks and
// counters of the last asynchronous call are kept and resolved.
template <class F>
int guarded(sp_ctx *ctx, F &&f, bool fresh = true) {
  if (!ctx) return SP_EINVAL;
  DeviceGuard dg(ctx->c.device);
  spb::g_launch_counter = &ctx->c.launches;
  if (fresh) {
    spb::reset_marks(ctx->c);
    ctx->c.in_used = ctx->c.out_used = 0;
    ctx->c.counters.clear();
    ++ctx->c.calls;
  }
  int rc = SP_OK;
  try {
    f(ctx->c);
    if (ctx->c.marks_used && (!ctx->c.async() || !fresh)) {
      SPB_CUDA(cudaStreamSynchronize(ctx->c.stream));
      spb::resolve_marks(ctx->c);
    }
  } catch (const spb::InvalidArgument &e) {
    ctx->c.last_error = e.what();
    rc = SP_EINVAL;
  } catch (const spb::CapacityError &e) {
    ctx->c.last_error = e.what();
    rc = SP_ECAPACITY;
  } catch (const spb::NcclError &e) {
    ctx->c.last_error = e.what();
    rc = SP_ENCCL;
  } catch (const spb::CudaError &e) {
    ctx->c.last_error = e.what();
    rc = strstr(e.what(), "allocation") ? SP_ENOMEM : SP_ECUDA;
  } catch (const std::bad_alloc &e) {
    ctx->c.last_error = "host allocation failed";
    rc = SP_ENOMEM;
  } catch (const std::exception &e) {
    ctx->c.last_error = e.what();
    rc = SP_ECUDA;
  }
  spb::g_launch_counter = nullptr;
  if (rc == SP_OK) ctx->c.last_error.clear();
  return rc;
}

void check_dim(int dim) {
  if (dim != 2 && dim != 3) throw spb::InvalidArgument("dimension must be 2 or 3");
}

void sync_all(spb::Ctx &c) {
  SPB_CUDA(cudaStreamSynchronize(c.stream));
  SPB_CUDA(cudaStreamSynchronize(c.h2d));
  SPB_CUDA(cudaStreamSynchronize(c.d2h));
}

void finish(spb::Ctx &c) {
  if (!c.async()) sync_all(c);
}

}  // namespace

extern "C" {

int sp_ctx_create(int device, void *stream, sp_ctx **out) {
  if (!out) return SP_EINVAL;
  *out = nullptr;
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || device < 0 || device >= ndev) return SP_ECUDA;
  DeviceGuard dg(device);
  sp_ctx *ctx = new (std::nothrow) sp_ctx;
  if (!ctx) return SP_ENOMEM;
  ctx->c.device = device;
  if (stream) {
    ctx->c.stream = (cudaStream_t)stream;
  } else {
    if (cudaStreamCreateWithFlags(&ctx->c.stream, cudaStreamNonBlocking) != cudaSuccess) {
      delete ctx;
      return SP_ECUDA;
    }
    ctx->c.owns_stream = true;
  }
  if (cudaStreamCreateWithFlags(&ctx->c.h2d, cudaStreamNonBlocking) != cudaSuccess ||
      cudaStreamCreateWithFlags(&ctx->c.d2h, cudaStreamNonBlocking) != cudaSuccess ||
      cudaMalloc(&ctx->c.d_err, sizeof(int)) != cudaSuccess || cudaMemset(ctx->c.d_err, 0, sizeof(int)) != cudaSuccess) {
    if (ctx->c.owns_stream) cudaStreamDestroy(ctx->c.stream);
    delete ctx;
    return SP_ECUDA;
  }
  spb::cache_register_stream(ctx->c.stream);
  // Keep freed stream-ordered allocations reserved: a caching allocator.
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
    uint64_t thr = UINT64_MAX;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
  }
  *out = ctx;
  return SP_OK;
}

int sp_ctx_destroy(sp_ctx *ctx) {
  if (!ctx) return SP_OK;
  {
    DeviceGuard dg(ctx->c.device);
    cudaStreamSynchronize(ctx->c.stream);
    for (cudaEvent_t e : ctx->c.event_pool) cudaEventDestroy(e);
    cudaStreamSynchronize(ctx->c.h2d);
    cudaStreamSynchronize(ctx->c.d2h);
    if (ctx->c.h2d) cudaStreamDestroy(ctx->c.h2d);
    if (ctx->c.d2h) cudaStreamDestroy(ctx->c.d2h);
    if (ctx->c.d_err) cudaFree(ctx->c.d_err);
    if (ctx->c.peek_buf) cudaFreeHost(ctx->c.peek_buf);
    for (auto *arr : {&ctx->c.in_stage, &ctx->c.out_stage})
      for (auto &row : *arr)
        for (auto &st : row) {
          if (st.p) cudaFree(st.p);
          if (st.done) cudaEventDestroy(st.done);
        }
    spb::cache_unregister_stream(ctx->c.stream);
    cudaStreamSynchronize(ctx->c.stream);
    if (ctx->c.owns_stream) cudaStreamDestroy(ctx->c.stream);
    // the pool keeps freed memory reserved while contexts run (release
    // threshold above); a destroyed context hands its share back
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, ctx->c.device) == cudaSuccess) cudaMemPoolTrimTo(pool, 0);
  }
  delete ctx;
  return SP_OK;
}

int sp_ctx_set_stream(sp_ctx *ctx, void *stream) {
  if (!ctx) return SP_EINVAL;
  DeviceGuard dg(ctx->c.device);
  cudaStreamSynchronize(ctx->c.stream);
  spb::cache_unregister_stream(ctx->c.stream);
  cudaStreamSynchronize(ctx->c.stream);
  if (ctx->c.owns_stream) cudaStreamDestroy(ctx->c.stream);
  ctx->c.owns_stream = false;
  if (stream) {
    ctx->c.stream = (cudaStream_t)stream;
  } else {
    if (cudaStreamCreateWithFlags(&ctx->c.stream, cudaStreamNonBlocking) != cudaSuccess) return SP_ECUDA;
    ctx->c.owns_stream = true;
  }
  spb::cache_register_stream(ctx->c.stream);
  return SP_OK;
}

int sp_ctx_synchronize(sp_ctx *ctx) {
  return guarded(ctx, [&](spb::Ctx &c) {
    sync_all(c);
    int err = 0;
    SPB_CUDA(cudaMemcpy(&err, c.d_err, sizeof(int), cudaMemcpyDeviceToHost));
    if (err) {
      SPB_CUDA(cudaMemset(c.d_err, 0, sizeof(int)));
      throw spb::InvalidArgument("non-finite coordinate in an asynchronous call");
    }
  }, /*fresh=*/false);
}

int sp_ctx_set_flags(sp_ctx *ctx, int flags) {
  if (!ctx) return SP_EINVAL;
  if (ctx->c.async() && !(flags & SP_FLAG_ASYNC)) {
    int rc = sp_ctx_synchronize(ctx);
    ctx->c.flags = flags;
    return rc;
  }
  ctx->c.flags = flags;
  return SP_OK;
}

const char *sp_last_error(const sp_ctx *ctx) { return ctx ? ctx->c.last_error.c_str() : "null context"; }

int64_t sp_ctx_kernel_launches(const sp_ctx *ctx) { return ctx ? ctx->c.launches : 0; }

int64_t sp_ctx_counter(const sp_ctx *ctx, const char *name) {
  if (!ctx || !name) return -1;
  for (const auto &kv : ctx->c.counters)
    if (kv.first == name) return kv.second;
  return -1;
}

int sp_ctx_phase_count(const sp_ctx *ctx) { return ctx ? (int)ctx->c.phases.size() : 0; }

const char *sp_ctx_phase_name(const sp_ctx *ctx, int i) {
  if (!ctx || i < 0 || i >= (int)ctx->c.phases.size()) return "";
  return ctx->c.phases[(size_t)i].first.c_str();
}

double sp_ctx_phase_ms(const sp_ctx *ctx, int i) {
  if (!ctx || i < 0 || i >= (int)ctx->c.phases.size()) return -1.0;
  return ctx->c.phases[(size_t)i].second;
}

int sp_bvh_build(sp_ctx *ctx, const float *objects, int64_t n, int dim, int is_points, int code_width, int mem,
                 sp_bvh **out) {
  if (out) *out = nullptr;
  return guarded(ctx, [&](spb::Ctx &c) {
    check_dim(dim);
    if (code_width != 32 && code_width != 64) throw spb::InvalidArgument("code width must be 32 or 64");
    if (n < 0 || n > (1LL << 30)) throw spb::InvalidArgument("object count out of range");
    if (!out) throw spb::InvalidArgument("null output handle");
    const size_t per = is_points ? dim : 2 * dim;
    In<float> obj(c, objects, (size_t)n * per, mem);
    sp_bvh *b = new sp_bvh;
    b->device = c.device;
    try {
      spb::build_tree(c, obj.p, n, dim, is_points != 0, code_width, b->t);
      finish(c);
    } catch (...) {
      delete b;
      throw;
    }
    *out = b;
  });
}

int sp_bvh_destroy(sp_bvh *bvh) {
  if (!bvh) return SP_OK;
  {
    DeviceGuard dg(bvh->device);
    cudaStreamSynchronize(bvh->t.stream);
    bvh->t.free_all();
    cudaStreamSynchronize(bvh->t.stream);
  }
  delete bvh;
  return SP_OK;
}

int64_t sp_bvh_size(const sp_bvh *bvh) { return bvh ? bvh->t.n : 0; }

int sp_bvh_export(sp_ctx *ctx, const sp_bvh *bvh, int32_t *internal_left, int32_t *internal_rope,
                  float *internal_boxes, int32_t *leaf_object, int32_t *leaf_rope, float *leaf_boxes, float *scene) {
  return guarded(ctx, [&](spb::Ctx &c) {
    if (!bvh) throw spb::InvalidArgument("null bvh");
    const spb::Tree &t = bvh->t;
    const int dim = t.dim;
    if (scene) {
      float s[6] = {0, 0, 0, 0, 0, 0};
      if (t.scene) SPB_CUDA(cudaMemcpyAsync(s, t.scene, sizeof(s), cudaMemcpyDeviceToHost, c.stream));
      finish(c);
      for (int k = 0; k < dim; ++k) {
        scene[k] = s[k];
        scene[dim + k] = s[3 + k];
      }
    }
    if (t.n == 0) return;
    const int64_t nn = 2 * t.n - 1;
    std::vector<float4> h((size_t)nn * 2);
    SPB_CUDA(cudaMemcpyAsync(h.data(), t.nodes, h.size() * sizeof(float4), cudaMemcpyDeviceToHost, c.stream));
    finish(c);
    auto bits = [](float f) {
      int32_t i;
      memcpy(&i, &f, 4);
      return i;
    };
    for (int64_t r = 0; r < nn; ++r) {
      const float4 &lo = h[(size_t)(2 * r)], &hi = h[(size_t)(2 * r + 1)];
      const float l3[3] = {lo.x, lo.y, lo.z}, h3[3] = {hi.x, hi.y, hi.z};
      const bool leaf = r >= t.n - 1;
      const int64_t i = leaf ? r - (t.n - 1) : r;
      int32_t *link = leaf ? leaf_object : internal_left;
      int32_t *rope = leaf ? leaf_rope : internal_rope;
      float *box = leaf ? leaf_boxes : internal_boxes;
      if (link) link[i] = bits(lo.w);
      if (rope) rope[i] = bits(hi.w);
      if (box)
        for (int k = 0; k < dim; ++k) {
          box[i * 2 * dim + k] = l3[k];
          box[i * 2 * dim + dim + k] = h3[k];
        }
    }
  });
}

int sp_range_count(sp_ctx *ctx, const sp_bvh *bvh, int pred_kind, const float *preds, int64_t nq, int32_t cap,
                   int32_t *counts, int mem) {
  return guarded(ctx, [&](spb::Ctx &c) {
    if (!bvh) throw spb::InvalidArgument("null bvh");
    if (nq < 0) throw spb::InvalidArgument("negative query count");
    const int dim = bvh->t.dim;
    const size_t per = pred_kind == SP_PRED_BOX ? 2 * dim : dim + 1;
    In<float> p(c, preds, (size_t)nq * per, mem);
    Out<int32_t> o(c, counts, (size_t)nq, mem);
    spb::range_count(c, bvh->t, pred_kind == SP_PRED_BOX ? spb::RQ_BOXES : spb::RQ_SPHERES, p.p, nq, 0.f, cap, o.p,
                     nullptr);
    o.flush(c);
    finish(c);
  });
}

int sp_range_count_radius(sp_ctx *ctx, const sp_bvh *bvh, const float *centres, int64_t nq, float radius, int32_t cap,
                          int32_t *counts, int mem) {
  return guarded(ctx, [&](spb::Ctx &c) {
    if (!bvh) throw spb::InvalidArgument("null bvh");
    if (nq < 0) throw spb::InvalidArgument("negative query count");
    In<float> p(c, centres, (size_t)nq * bvh->t.dim, mem);
    Out<int32_t> o(c, counts, (size_t)nq, mem);
    spb::range_count(c, bvh->t, spb::RQ_RADIUS, p.p, nq, radius, cap, o.p, nullptr);
    o.flush(c);
    finish(c);
  });
}

int sp_range_crs(sp_ctx *ctx, const sp_bvh *bvh, int pred_kind, const float *preds, int64_t nq, int64_t *offsets,
                 int32_t *values, int64_t capacity, int mem) {
  return guarded(ctx, [&](spb::Ctx &c) {
    if (!bvh) throw spb::InvalidArgument("null bvh");
    const int dim = bvh->t.dim;
    const size_t per = pred_kind == SP_PRED_BOX ? 2 * dim : dim + 1;
    In<float> p(c, preds, (size_t)nq * per, mem);
    Out<int64_t> off(c, offsets, (size_t)nq + 1, mem);
    // values: device scratch of `capacity` or the caller's device array
    DevBuf<int32_t> vbuf;
    int32_t *vdev = values;
    if (mem == SP_MEM_HOST && values && capacity > 0) {
      vbuf = DevBuf<int32_t>((size_t)capacity, c.stream);
      vdev = vbuf.get();
    }
    int64_t total = spb::range_crs(c, bvh->t, pred_kind == SP_PRED_BOX ? spb::RQ_BOXES : spb::RQ_SPHERES, p.p, nq,
                                   off.p, vdev, values ? capacity : 0);
    off.flush(c);
    if (total <= capacity && values && mem == SP_MEM_HOST && total > 0)
      SPB_CUDA(cudaMemcpyAsync(values, vdev, (size_t)total * sizeof(int32_t), cudaMemcpyDeviceToHost, c.stream));
    finish(c);
    if (total > capacity && values) throw spb::CapacityError();
  });
}

int sp_knn(sp_ctx *ctx, const sp_bvh *bvh, const float *origins, int64_t nq, int32_t k, int32_t *idx, float *dist,
           int mem) {
  return guarded(ctx, [&](spb::Ctx &c) {
    if (!bvh) throw spb::InvalidArgument("null bvh");
    if (k <= 0 || nq <= 0) return;
    In<float> o(c, origins, (size_t)nq * bvh->t.dim, mem);
    Out<int32_t> oi(c, idx, (size_t)nq * k, mem);
    Out<float> od(c, dist, (size_t)nq * k, mem);
    spb::knn(c, bvh->t, o.p, nq, k, oi.p, od.p);
    oi.flush(c);
    od.flush(c);
    finish(c);
  });
}

int sp_pair_list(sp_ctx *ctx, const sp_bvh *bvh, float eps, int32_t *pairs, int64_t capacity, int64_t *num_pairs,
                 int mem) {
  return guarded(ctx, [&](spb::Ctx &c) {
    if (!bvh) throw spb::InvalidArgument("null bvh");
    DevBuf<int32_t> pbuf;
    int32_t *pdev = pairs;
    if (mem == SP_MEM_HOST && pairs && capacity > 0) {
      pbuf = DevBuf<int32_t>((size_t)capacity * 2, c.stream);
      pdev = pbuf.get();
    }
    int64_t total = spb::pair_list(c, bvh->t, eps, pdev, pairs ? capacity : 0);
    if (num_pairs) *num_pairs = total;
    if (total <= capacity && pairs && mem == SP_MEM_HOST && total > 0)
      SPB_CUDA(cudaMemcpyAsync(pairs, pdev, (size_t)total * 2 * sizeof(int32_t), cudaMemcpyDeviceToHost, c.stream));
    finish(c);
    if (total > capacity && pairs) throw spb::CapacityError();
  });
}

int sp_check_equivalence(sp_ctx *ctx, const float *points, int64_t n, int dim, float eps, const int32_t *got_labels,
                         const uint8_t *got_core, const int32_t *want_labels, const uint8_t *want_core,
                         int64_t *violation, int *kind, int mem) {
  return guarded(ctx, [&](spb::Ctx &c) {
    check_dim(dim);
    In<float> p(c, points, (size_t)n * dim, mem);
    In<int32_t> gl(c, got_labels, (size_t)n, mem), wl(c, want_labels, (size_t)n, mem);
    In<uint8_t> gc(c, got_core, (size_t)n, mem), wc(c, want_core, (size_t)n, mem);
    int k = 0;
    const int64_t v = spb::check_equivalence(c, p.p, n, dim, eps, gl.p, gc.p, wl.p, wc.p, &k);
    if (violation) *violation = v;
    if (kind) *kind = k;
  });
}

// Diagnostics (not part of the reference surface): per-leaf node visits and
// close pairs of the pair walk, in leaf order.
int sp_debug_walk_lengths(sp_ctx *ctx, const sp_bvh *bvh, float eps, int32_t *steps, int32_t *hits, int mem) {
  return guarded(ctx, [&](spb::Ctx &c) {
    if (!bvh) throw spb::InvalidArgument("null bvh");
    Out<int32_t> os(c, steps, (size_t)bvh->t.n, mem), oh(c, hits, (size_t)bvh->t.n, mem);
    spb::walk_lengths(c, bvh->t, eps, os.p, oh.p);
    os.flush(c);
    oh.flush(c);
    finish(c);
  });
}

int sp_sort_queries(sp_ctx *ctx, const float *points, int64_t nq, int dim, int32_t *order, int mem) {
  return guarded(ctx, [&](spb::Ctx &c) {
    check_dim(dim);
    In<float> p(c, points, (size_t)nq * dim, mem);
    Out<int32_t> o(c, order, (size_t)nq, mem);
    spb::sort_points(c, p.p, nq, dim, o.p);
    o.flush(c);
    finish(c);
  });
}

int sp_morton_codes(sp_ctx *ctx, const float *objects, int64_t n, int dim, int is_points, int code_width,
                    uint64_t *codes, int mem) {
  return guarded(ctx, [&](spb::Ctx &c) {
    check_dim(dim);
    if (code_width != 32 && code_width != 64) throw spb::InvalidArgument("code width must be 32 or 64");
    const size_t per = is_points ? dim : 2 * dim;
    In<float> obj(c, objects, (size_t)n * per, mem);
    Out<uint64_t> o(c, codes, (size_t)n, mem);
    DevBuf<float> scene(6, c.stream);
    DevBuf<int> bad(1, c.stream);
    spb::scene_bounds(c, obj.p, n, dim, is_points != 0, scene.get(), bad.get());
    spb::morton_codes(c, obj.p, n, dim, is_points != 0, code_width, scene.get(), o.p, nullptr);
    o.flush(c);
    finish(c);
  });
}

int sp_dbscan(sp_ctx *ctx, const float *points, int64_t n, int dim, float eps, int32_t min_pts, int algo,
              int code_width, int32_t *labels, uint8_t *core, sp_timings *timings, sp_stats *stats, int mem) {
  return guarded(ctx, [&](spb::Ctx &c) {
    check_dim(dim);
    if ((algo & ~0x100) < 0 || (algo & ~0x100) > 4) throw spb::InvalidArgument("unknown algorithm");
    if (code_width != 32 && code_width != 64) throw spb::InvalidArgument("code width must be 32 or 64");
    if (n < 0 || n > (1LL << 30)) throw spb::InvalidArgument("point count out of range");
    In<float> p(c, points, (size_t)n * dim, mem);
    Out<int32_t> ol(c, labels, (size_t)n, mem);
    Out<uint8_t> oc(c, core, (size_t)n, mem);
    DevBuf<int32_t> lscratch;
    DevBuf<uint8_t> cscratch;
    int32_t *lp = ol.p;
    uint8_t *cp = oc.p;
    if (!lp && n) { lscratch = DevBuf<int32_t>((size_t)n, c.stream); lp = lscratch.get(); }
    if (!cp && n) { cscratch = DevBuf<uint8_t>((size_t)n, c.stream); cp = cscratch.get(); }
    spb::DbscanResult res;
    spb::dbscan(c, p.p, n, dim, eps, min_pts, algo, code_width, lp, cp, &res);
    ol.flush(c);
    oc.flush(c);
    finish(c);
    if (timings) {
      timings->build_ms = res.ms[0];
      timings->core_ms = res.ms[1];
      timings->merge_ms = res.ms[2];
      timings->finalize_ms = res.ms[3];
    }
    if (stats) {
      stats->distance_checks = res.distance_checks;
      stats->num_dense_cells = res.num_dense_cells;
      stats->num_dense_points = res.num_dense_points;
    }
  });
}

// ---- multi-GPU slab FoF (SURVEY §8 row e; sp_slabs.cu) -----------------------
int sp_comm_unique_id(uint8_t id[128]) {
  if (!id) return SP_EINVAL;
  try {
    spb::nccl_unique_id(id);
  } catch (const std::exception &) {
    return SP_ENCCL;
  }
  return SP_OK;
}

int sp_comm_create(sp_ctx *ctx, int nranks, int rank, const uint8_t id[128], sp_comm **out) {
  if (!out || !id) return SP_EINVAL;
  *out = nullptr;
  return guarded(ctx, [&](spb::Ctx &c) {
    sp_comm *cm = new sp_comm;
    try {
      cm->x = spb::nccl_exchange_create(c.device, nranks, rank, id);
    } catch (...) {
      delete cm;
      throw;
    }
    *out = cm;
  });
}

int sp_comm_wrap(sp_ctx *ctx, void *nccl_comm, sp_comm **out) {
  if (!out) return SP_EINVAL;
  *out = nullptr;
  return guarded(ctx, [&](spb::Ctx &) {
    sp_comm *cm = new sp_comm;
    try {
      cm->x = spb::nccl_exchange_wrap(nccl_comm);
    } catch (...) {
      delete cm;
      throw;
    }
    *out = cm;
  });
}

int sp_comm_destroy(sp_comm *comm) {
  if (!comm) return SP_EINVAL;
  spb::exchange_destroy(comm->x);
  delete comm;
  return SP_OK;
}

int sp_comm_size(const sp_comm *comm) { return comm ? spb::exchange_size(comm->x) : -1; }
int sp_comm_rank(const sp_comm *comm) { return comm ? spb::exchange_rank(comm->x) : -1; }

int sp_fof_slabs(sp_ctx *ctx, sp_comm *comm, const float *points, int64_t n_local, float eps, int64_t first_index,
                 int32_t *labels, uint8_t *core, int mem) {
  if (!comm) return SP_EINVAL;
  return guarded(ctx, [&](spb::Ctx &c) {
    if (n_local < 0 || n_local > (1LL << 30)) throw spb::InvalidArgument("point count out of range");
    if (n_local > 0 && (!points || !labels || !core)) throw spb::InvalidArgument("null array");
    In<float> p(c, points, (size_t)n_local * 3, mem);
    Out<int32_t> ol(c, labels, (size_t)n_local, mem);
    Out<uint8_t> oc(c, core, (size_t)n_local, mem);
    std::vector<spb::SlabInput> in(1);
    in[0] = spb::SlabInput{&c, p.p, n_local, first_index, ol.p, oc.p};
    spb::fof_slabs(in, *comm->x, eps);
    ol.flush(c);
    oc.flush(c);
    finish(c);
  });
}

int sp_fof_slabs_multi(sp_ctx *const *ctxs, int nranks, const float *const *points, const int64_t *n_local, float eps,
                       int32_t *const *labels, uint8_t *const *core, int mem) {
  if (!ctxs || nranks < 1 || !points || !n_local || !labels || !core) return SP_EINVAL;
  for (int r = 0; r < nranks; ++r)
    if (!ctxs[r]) return SP_EINVAL;
  return guarded(ctxs[0], [&](spb::Ctx &c0) {
    std::vector<std::unique_ptr<In<float>>> pin;
    std::vector<std::unique_ptr<Out<int32_t>>> pl;
    std::vector<std::unique_ptr<Out<uint8_t>>> pc;
    std::vector<spb::SlabInput> in((size_t)nranks);
    int64_t first = 0;
    for (int r = 0; r < nranks; ++r) {
      spb::Ctx &c = ctxs[r]->c;
      if (n_local[r] < 0 || n_local[r] > (1LL << 30)) throw spb::InvalidArgument("point count out of range");
      spb::ScopedDevice sd(c.device);
      if (r > 0) {
        spb::reset_marks(c);
        c.in_used = c.out_used = 0;
        c.counters.clear();
        ++c.calls;
      }
      pin.emplace_back(new In<float>(c, points[r], (size_t)n_local[r] * 3, mem));
      pl.emplace_back(new Out<int32_t>(c, labels[r], (size_t)n_local[r], mem));
      pc.emplace_back(new Out<uint8_t>(c, core[r], (size_t)n_local[r], mem));
      in[r] = spb::SlabInput{&c, pin[r]->p, n_local[r], first, pl[r]->p, pc[r]->p};
      first += n_local[r];
    }
    spb::fof_slabs_multi(in, eps);
    for (int r = 0; r < nranks; ++r) {
      spb::Ctx &c = ctxs[r]->c;
      spb::ScopedDevice sd(c.device);
      pl[r]->flush(c);
      pc[r]->flush(c);
      sync_all(c);
      if (r > 0 && c.marks_used) spb::resolve_marks(c);
    }
    (void)c0;
  });
}

int sp_fof_ids(sp_ctx *ctx, const float *points, int64_t n, int dim, float eps, const int32_t *ids,
               int32_t *labels, uint8_t *core, int mem) {
  return guarded(ctx, [&](spb::Ctx &c) {
    check_dim(dim);
    if (n < 0 || n > (1LL << 30)) throw spb::InvalidArgument("point count out of range");
    In<float> p(c, points, (size_t)n * dim, mem);
    In<int32_t> id(c, ids, (size_t)n, mem);
    Out<int32_t> ol(c, labels, (size_t)n, mem);
    Out<uint8_t> oc(c, core, (size_t)n, mem);
    if (n) spb::dbscan(c, p.p, n, dim, eps, 2, 1, 64, ol.p, oc.p, nullptr, id.p);
    ol.flush(c);
    oc.flush(c);
    finish(c);
  });
}

int sp_dbscan_adjacency(sp_ctx *ctx, const float *points, int64_t n, int dim, float eps, int code_width,
                        int64_t max_adjacency, int32_t *labels, uint8_t *core, sp_timings *timings, int mem) {
  return guarded(ctx, [&](spb::Ctx &c) {
    check_dim(dim);
    if (code_width != 32 && code_width != 64) throw spb::InvalidArgument("code width must be 32 or 64");
    if (n < 0 || n > (1LL << 30)) throw spb::InvalidArgument("point count out of range");
    In<float> p(c, points, (size_t)n * dim, mem);
    Out<int32_t> ol(c, labels, (size_t)n, mem);
    Out<uint8_t> oc(c, core, (size_t)n, mem);
    DevBuf<int32_t> ls;
    DevBuf<uint8_t> cs;
    int32_t *lp = ol.p;
    uint8_t *cp = oc.p;
    if (!lp && n) { ls = DevBuf<int32_t>((size_t)n, c.stream); lp = ls.get(); }
    if (!cp && n) { cs = DevBuf<uint8_t>((size_t)n, c.stream); cp = cs.get(); }
    spb::DbscanResult res;
    spb::adjacency_dbscan(c, p.p, n, dim, eps, code_width, max_adjacency, lp, cp, &res);
    ol.flush(c);
    oc.flush(c);
    finish(c);
    if (timings) {
      timings->build_ms = res.ms[0];
      timings->core_ms = res.ms[1];
      timings->merge_ms = res.ms[2];
      timings->finalize_ms = res.ms[3];
    }
  });
}

int sp_dbscan_bruteforce(sp_ctx *ctx, const float *points, int64_t n, int dim, float eps, int32_t min_pts,
                         int32_t *labels, uint8_t *core, int mem) {
  return guarded(ctx, [&](spb::Ctx &c) {
    check_dim(dim);
    In<float> p(c, points, (size_t)n * dim, mem);
    Out<int32_t> ol(c, labels, (size_t)n, mem);
    Out<uint8_t> oc(c, core, (size_t)n, mem);
    spb::bruteforce_dbscan(c, p.p, n, dim, eps, min_pts, ol.p, oc.p);
    ol.flush(c);
    oc.flush(c);
    finish(c);
  });
}

int sp_generate_field(sp_ctx *ctx, int64_t n_total, int64_t first, int64_t count, uint64_t seed, float *out,
                      int mem) {
  return guarded(ctx, [&](spb::Ctx &c) {
    if (n_total <= 0 || first < 0 || count < 0 || first + count > n_total)
      throw spb::InvalidArgument("generate_field: bad slice");
    Out<float> o(c, out, (size_t)count * 3, mem);
    spb::generate_field(c, n_total, first, count, seed, o.p);
    o.flush(c);
    finish(c);
  });
}

int sp_generate_uniform(sp_ctx *ctx, int64_t n, int dim, uint64_t seed, float *out, int mem) {
  return guarded(ctx, [&](spb::Ctx &c) {
    check_dim(dim);
    Out<float> o(c, out, (size_t)n * dim, mem);
    spb::generate_uniform(c, n, dim, seed, o.p);
    o.flush(c);
    finish(c);
  });
}

}  // extern "C"
