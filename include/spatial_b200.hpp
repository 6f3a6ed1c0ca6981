// spatial_b200.hpp — C++20 façade that restores the reference's
// `namespace spatial` signatures (/root/reference/proj/include/spatial/*.hpp)
// on top of the C ABI in sp_b200.h, so code written against the reference
// switches by changing the include and the namespace:
//
//   reference                                    here (spatial_b200::)
//   Bvh<D>::build(span<const Aabb<D>>, width)     same; tree lives on the GPU
//   bvh.internals / bvh.leaves / validate / dump  internals() / leaves() / validate() / dump()
//   range_query(bvh, preds, cb [, mode])          same (cb may return void or CallbackControl)
//   nearest_query(bvh, preds, cb [, mode])        same
//   pair_traversal(bvh, eps, cb [, mode])         same
//   sort_queries<D, P>(preds)                     same
//   query_crs(bvh, preds, mode, max_total)        same (throws CapacityError)
//   fdbscan / friends_of_friends /                same -> DbscanOutput
//   fdbscan_densebox
//
// Errors map back to the reference's exceptions: SP_EINVAL ->
// std::invalid_argument, SP_ECAPACITY -> CapacityError (a std::bad_alloc),
// anything else -> std::runtime_error.  The fused device paths (range counts,
// CRS, kNN, pairs, clustering) run entirely on the GPU; a *generic* host
// callback is served by replaying the device-computed matches per query in
// the reference's traversal (leaf) order, honouring kTerminateQuery.
#ifndef SPATIAL_B200_HPP
#define SPATIAL_B200_HPP

#include <algorithm>
#include <array>
#include <cstdint>
#include <cstdio>
#include <limits>
#include <memory>
#include <new>
#include <ostream>
#include <span>
#include <stdexcept>
#include <string>
#include <type_traits>
#include <variant>
#include <vector>

#include "sp_b200.h"

namespace spatial_b200 {

// ---- geometry types (geometry.hpp:15-51) ----------------------------------
template <int Dim>
struct Point {
  static_assert(Dim == 2 || Dim == 3, "only 2- and 3-dimensional data is supported");
  std::array<float, Dim> coords{};
  float &operator[](int k) { return coords[static_cast<std::size_t>(k)]; }
  float operator[](int k) const { return coords[static_cast<std::size_t>(k)]; }
  friend bool operator==(const Point &, const Point &) = default;
};

template <int Dim>
struct Aabb {
  Point<Dim> min_corner;
  Point<Dim> max_corner;
  constexpr Aabb() {
    for (int k = 0; k < Dim; ++k) {
      min_corner[k] = std::numeric_limits<float>::max();
      max_corner[k] = std::numeric_limits<float>::lowest();
    }
  }
  constexpr Aabb(const Point<Dim> &lo, const Point<Dim> &hi) : min_corner(lo), max_corner(hi) {}
  friend bool operator==(const Aabb &, const Aabb &) = default;
};

template <int Dim>
struct Sphere {
  Point<Dim> center;
  float radius = 0.f;
};

template <int Dim>
inline Aabb<Dim> point_box(const Point<Dim> &p) {
  return Aabb<Dim>(p, p);
}

enum class CodeWidth : int { k32 = 32, k64 = 64 };
// The GPU always runs in parallel; kSequential selects the deterministic
// border assignment of the reference's sequential run where results differ
// (fdbscan with min_pts > 2; friends_of_friends is deterministic anyway).
enum class ExecMode { kSequential, kParallel };
enum class CallbackControl { kContinue, kTerminateQuery };

struct NodeRef {
  std::int32_t value = -1;
  friend bool operator==(const NodeRef &, const NodeRef &) = default;
};
inline constexpr NodeRef kSentinel{-1};

template <int Dim>
struct RangePredicate {
  std::variant<Sphere<Dim>, Aabb<Dim>> geometry;
};

template <int Dim>
struct NearestPredicate {
  Point<Dim> origin;
  std::int32_t k = 1;
};

struct CapacityError : std::bad_alloc {
  const char *what() const noexcept override { return "crs result exceeds capacity"; }
};

struct CrsResult {
  std::vector<std::int64_t> offsets;
  std::vector<std::int32_t> values;
};

// ---- context: one per thread (sp_ctx = device + stream + allocator) --------
namespace detail {

inline void check(sp_ctx *ctx, int rc) {
  if (rc == SP_OK) return;
  std::string msg = sp_last_error(ctx);
  if (rc == SP_EINVAL) throw std::invalid_argument(msg);
  if (rc == SP_ECAPACITY) throw CapacityError{};
  throw std::runtime_error("sp_b200 status " + std::to_string(rc) + ": " + msg);
}

struct CtxHolder {
  sp_ctx *ctx = nullptr;
  CtxHolder() {
    if (sp_ctx_create(0, nullptr, &ctx) != SP_OK) throw std::runtime_error("sp_b200: no usable CUDA device");
  }
  ~CtxHolder() { sp_ctx_destroy(ctx); }
};

inline sp_ctx *context() {
  thread_local CtxHolder holder;
  return holder.ctx;
}

template <int Dim>
std::vector<float> flatten(std::span<const Aabb<Dim>> boxes) {
  std::vector<float> v(boxes.size() * 2 * Dim);
  for (std::size_t i = 0; i < boxes.size(); ++i)
    for (int k = 0; k < Dim; ++k) {
      v[i * 2 * Dim + k] = boxes[i].min_corner[k];
      v[i * 2 * Dim + Dim + k] = boxes[i].max_corner[k];
    }
  return v;
}

template <int Dim>
std::vector<float> flatten(std::span<const Point<Dim>> pts) {
  std::vector<float> v(pts.size() * Dim);
  for (std::size_t i = 0; i < pts.size(); ++i)
    for (int k = 0; k < Dim; ++k) v[i * Dim + k] = pts[i][k];
  return v;
}

}  // namespace detail

// ---- hierarchy (bvh.hpp:43-86) ----------------------------------------------
template <int Dim>
class Bvh {
 public:
  struct Leaf {
    Aabb<Dim> volume;
    std::int32_t object_index = -1;
    NodeRef rope = kSentinel;
  };
  struct Internal {
    Aabb<Dim> volume;
    NodeRef left_child;
    NodeRef rope = kSentinel;
  };

  static Bvh build(std::span<const Aabb<Dim>> objects, CodeWidth width = CodeWidth::k64) {
    Bvh b;
    b.width_ = width;
    auto flat = detail::flatten<Dim>(objects);
    sp_bvh *h = nullptr;
    detail::check(detail::context(), sp_bvh_build(detail::context(), flat.data(), (int64_t)objects.size(), Dim, 0,
                                                  static_cast<int>(width), SP_MEM_HOST, &h));
    b.h_.reset(h, [](sp_bvh *p) { sp_bvh_destroy(p); });
    return b;
  }

  std::int32_t size() const { return h_ ? static_cast<std::int32_t>(sp_bvh_size(h_.get())) : 0; }
  bool empty() const { return size() == 0; }
  CodeWidth width() const { return width_; }
  NodeRef root() const { return empty() ? kSentinel : NodeRef{size() == 1 ? 0 : 0}; }
  bool is_leaf(NodeRef ref) const { return ref.value >= size() - 1; }
  NodeRef leaf_ref(std::int32_t pos) const { return NodeRef{size() - 1 + pos}; }
  std::int32_t leaf_pos(NodeRef ref) const { return ref.value - (size() - 1); }
  const sp_bvh *handle() const { return h_.get(); }

  // The reference's public node arrays, copied back from the device.
  std::vector<Internal> internals() const {
    fetch();
    return cache_->internals;
  }
  std::vector<Leaf> leaves() const {
    fetch();
    return cache_->leaves;
  }

  // Bvh::validate (bvh.hpp:263-330) over the exported arrays.
  bool validate(std::string *violation = nullptr) const {
    fetch();
    const auto &in = cache_->internals;
    const auto &lf = cache_->leaves;
    const std::int32_t n = size();
    auto fail = [&](const std::string &m) {
      if (violation) *violation = m;
      return false;
    };
    if (n == 0) return in.empty() || fail("empty hierarchy has internal nodes");
    if ((std::int32_t)in.size() != n - 1) return fail("internal node count is not n-1");
    auto rope = [&](NodeRef r) { return is_leaf(r) ? lf[leaf_pos(r)].rope : in[r.value].rope; };
    auto vol = [&](NodeRef r) { return is_leaf(r) ? lf[leaf_pos(r)].volume : in[r.value].volume; };
    std::int32_t expected = 0;
    std::int64_t steps = 0;
    for (NodeRef cur = root(); cur != kSentinel;) {
      if (++steps > 2 * static_cast<std::int64_t>(n) + 1) return fail("rope walk does not terminate (cycle)");
      if (is_leaf(cur)) {
        if (leaf_pos(cur) != expected) return fail("rope walk out of leaf order");
        ++expected;
        cur = lf[leaf_pos(cur)].rope;
      } else {
        cur = in[cur.value].left_child;
      }
    }
    if (expected != n) return fail("rope walk does not cover every leaf");
    for (std::int32_t i = 0; i + 1 < n; ++i) {
      NodeRef left = in[i].left_child, right = rope(left);
      if (right == kSentinel) return fail("internal node has no reachable right child");
      Aabb<Dim> u = vol(left), r = vol(right);
      for (int k = 0; k < Dim; ++k) {
        u.min_corner[k] = std::min(u.min_corner[k], r.min_corner[k]);
        u.max_corner[k] = std::max(u.max_corner[k], r.max_corner[k]);
      }
      if (!(u == in[i].volume)) return fail("internal node volume is not the union of children");
    }
    return true;
  }

  // Bvh::dump text format (bvh.hpp:332-357).
  void dump(std::ostream &os) const {
    fetch();
    auto put = [&os](const Aabb<Dim> &b) {
      char buf[64];
      for (int k = 0; k < Dim; ++k) {
        std::snprintf(buf, sizeof(buf), " %.9g", static_cast<double>(b.min_corner[k]));
        os << buf;
      }
      for (int k = 0; k < Dim; ++k) {
        std::snprintf(buf, sizeof(buf), " %.9g", static_cast<double>(b.max_corner[k]));
        os << buf;
      }
    };
    os << "bvh n " << size() << " width " << static_cast<int>(width_) << '\n';
    for (std::size_t i = 0; i < cache_->internals.size(); ++i) {
      const auto &x = cache_->internals[i];
      os << "I " << i << " left " << x.left_child.value << " rope " << x.rope.value;
      put(x.volume);
      os << '\n';
    }
    for (std::size_t p = 0; p < cache_->leaves.size(); ++p) {
      const auto &x = cache_->leaves[p];
      os << "L " << p << " object " << x.object_index << " rope " << x.rope.value;
      put(x.volume);
      os << '\n';
    }
  }

  // leaf position of every object (inverse of the leaf permutation)
  std::vector<std::int32_t> leaf_rank() const {
    fetch();
    std::vector<std::int32_t> r(cache_->leaves.size());
    for (std::size_t p = 0; p < r.size(); ++p) r[(std::size_t)cache_->leaves[p].object_index] = (std::int32_t)p;
    return r;
  }

 private:
  struct Cache {
    std::vector<Internal> internals;
    std::vector<Leaf> leaves;
  };
  void fetch() const {
    if (cache_) return;
    auto c = std::make_shared<Cache>();
    const std::int32_t n = size();
    if (n > 0) {
      std::vector<std::int32_t> il(n - 1), ir(n - 1), lo(n), lr(n);
      std::vector<float> ib((std::size_t)(n - 1) * 2 * Dim), lb((std::size_t)n * 2 * Dim);
      detail::check(detail::context(), sp_bvh_export(detail::context(), h_.get(), il.data(), ir.data(), ib.data(),
                                                     lo.data(), lr.data(), lb.data(), nullptr));
      auto box = [](const float *f) {
        Aabb<Dim> b;
        for (int k = 0; k < Dim; ++k) {
          b.min_corner[k] = f[k];
          b.max_corner[k] = f[Dim + k];
        }
        return b;
      };
      c->internals.resize((std::size_t)(n - 1));
      for (std::int32_t i = 0; i + 1 < n; ++i)
        c->internals[i] = Internal{box(&ib[(std::size_t)i * 2 * Dim]), NodeRef{il[i]}, NodeRef{ir[i]}};
      c->leaves.resize((std::size_t)n);
      for (std::int32_t p = 0; p < n; ++p)
        c->leaves[p] = Leaf{box(&lb[(std::size_t)p * 2 * Dim]), lo[p], NodeRef{lr[p]}};
    }
    cache_ = c;
  }

  std::shared_ptr<sp_bvh> h_;
  CodeWidth width_ = CodeWidth::k64;
  mutable std::shared_ptr<Cache> cache_;
};

namespace detail {

// Split predicates into sphere and box batches (the C ABI takes one kind).
template <int Dim>
void split_preds(std::span<const RangePredicate<Dim>> preds, std::vector<float> &sph, std::vector<std::int32_t> &si,
                 std::vector<float> &box, std::vector<std::int32_t> &bi) {
  for (std::size_t q = 0; q < preds.size(); ++q) {
    if (const auto *s = std::get_if<Sphere<Dim>>(&preds[q].geometry)) {
      for (int k = 0; k < Dim; ++k) sph.push_back(s->center[k]);
      sph.push_back(s->radius);
      si.push_back((std::int32_t)q);
    } else {
      const auto &b = std::get<Aabb<Dim>>(preds[q].geometry);
      for (int k = 0; k < Dim; ++k) box.push_back(b.min_corner[k]);
      for (int k = 0; k < Dim; ++k) box.push_back(b.max_corner[k]);
      bi.push_back((std::int32_t)q);
    }
  }
}

template <int Dim>
CrsResult crs_of_kind(const Bvh<Dim> &bvh, int kind, const std::vector<float> &flat, std::int64_t nq) {
  CrsResult r;
  r.offsets.assign((std::size_t)nq + 1, 0);
  if (nq == 0) return r;
  sp_ctx *ctx = context();
  check(ctx, sp_range_crs(ctx, bvh.handle(), kind, flat.data(), nq, r.offsets.data(), nullptr, 0, SP_MEM_HOST));
  r.values.resize((std::size_t)r.offsets.back());
  check(ctx, sp_range_crs(ctx, bvh.handle(), kind, flat.data(), nq, r.offsets.data(), r.values.data(),
                          (std::int64_t)r.values.size(), SP_MEM_HOST));
  return r;
}

}  // namespace detail

// query_crs (traversal.hpp:235-266)
template <int Dim>
CrsResult query_crs(const Bvh<Dim> &bvh, std::span<const RangePredicate<Dim>> preds,
                    ExecMode = ExecMode::kParallel,
                    std::int64_t max_total_matches = std::numeric_limits<std::int64_t>::max()) {
  std::vector<float> sph, box;
  std::vector<std::int32_t> si, bi;
  detail::split_preds<Dim>(preds, sph, si, box, bi);
  CrsResult a = detail::crs_of_kind(bvh, SP_PRED_SPHERE, sph, (std::int64_t)si.size());
  CrsResult b = detail::crs_of_kind(bvh, SP_PRED_BOX, box, (std::int64_t)bi.size());
  CrsResult out;
  out.offsets.assign(preds.size() + 1, 0);
  std::vector<std::int64_t> cnt(preds.size(), 0);
  for (std::size_t j = 0; j < si.size(); ++j) cnt[(std::size_t)si[j]] = a.offsets[j + 1] - a.offsets[j];
  for (std::size_t j = 0; j < bi.size(); ++j) cnt[(std::size_t)bi[j]] = b.offsets[j + 1] - b.offsets[j];
  for (std::size_t q = 0; q < preds.size(); ++q) out.offsets[q + 1] = out.offsets[q] + cnt[q];
  if (out.offsets.back() > max_total_matches) throw CapacityError{};
  out.values.resize((std::size_t)out.offsets.back());
  for (std::size_t j = 0; j < si.size(); ++j)
    std::copy(a.values.begin() + a.offsets[j], a.values.begin() + a.offsets[j + 1],
              out.values.begin() + out.offsets[(std::size_t)si[j]]);
  for (std::size_t j = 0; j < bi.size(); ++j)
    std::copy(b.values.begin() + b.offsets[j], b.values.begin() + b.offsets[j + 1],
              out.values.begin() + out.offsets[(std::size_t)bi[j]]);
  return out;
}

// range_query (traversal.hpp:67-87): device-computed matches replayed per
// query in traversal (leaf) order; the callback may return void or
// CallbackControl, and kTerminateQuery stops only the emitting query.
template <int Dim, class Callback>
void range_query(const Bvh<Dim> &bvh, std::span<const RangePredicate<Dim>> preds, Callback &&callback,
                 ExecMode mode = ExecMode::kParallel) {
  if (bvh.empty()) return;
  CrsResult crs = query_crs<Dim>(bvh, preds, mode);
  std::vector<std::int32_t> rank = bvh.leaf_rank();
  for (std::size_t q = 0; q < preds.size(); ++q) {
    auto b = crs.values.begin() + crs.offsets[q], e = crs.values.begin() + crs.offsets[q + 1];
    std::sort(b, e, [&](std::int32_t x, std::int32_t y) { return rank[(std::size_t)x] < rank[(std::size_t)y]; });
    for (auto it = b; it != e; ++it) {
      if constexpr (std::is_void_v<decltype(callback(std::int32_t{}, std::int32_t{}))>) {
        callback(static_cast<std::int32_t>(q), *it);
      } else {
        if (callback(static_cast<std::int32_t>(q), *it) == CallbackControl::kTerminateQuery) break;
      }
    }
  }
}

// The fused counting path: counts[q] = min(matches, cap) (cap <= 0: uncapped).
template <int Dim>
std::vector<std::int32_t> range_count(const Bvh<Dim> &bvh, std::span<const Sphere<Dim>> spheres,
                                      std::int32_t cap = 0) {
  std::vector<float> flat;
  for (const auto &s : spheres) {
    for (int k = 0; k < Dim; ++k) flat.push_back(s.center[k]);
    flat.push_back(s.radius);
  }
  std::vector<std::int32_t> counts(spheres.size());
  detail::check(detail::context(), sp_range_count(detail::context(), bvh.handle(), SP_PRED_SPHERE, flat.data(),
                                                  (std::int64_t)spheres.size(), cap, counts.data(), SP_MEM_HOST));
  return counts;
}

// nearest_query (traversal.hpp:93-156): min(k, n) results per query in
// ascending (distance, index) order.
template <int Dim, class Callback>
void nearest_query(const Bvh<Dim> &bvh, std::span<const NearestPredicate<Dim>> preds, Callback &&callback,
                   ExecMode = ExecMode::kParallel) {
  if (bvh.empty() || preds.empty()) return;
  std::int32_t kmax = 0;
  for (const auto &p : preds) kmax = std::max(kmax, p.k);
  kmax = std::min<std::int32_t>(kmax, bvh.size());
  if (kmax <= 0) return;
  std::vector<float> org;
  for (const auto &p : preds)
    for (int k = 0; k < Dim; ++k) org.push_back(p.origin[k]);
  std::vector<std::int32_t> idx(preds.size() * (std::size_t)kmax);
  detail::check(detail::context(), sp_knn(detail::context(), bvh.handle(), org.data(), (std::int64_t)preds.size(),
                                          kmax, idx.data(), nullptr, SP_MEM_HOST));
  for (std::size_t q = 0; q < preds.size(); ++q) {
    const std::int32_t kq = std::min(std::max(preds[q].k, 0), kmax);
    for (std::int32_t j = 0; j < kq; ++j) callback(static_cast<std::int32_t>(q), idx[q * (std::size_t)kmax + j]);
  }
}

// pair_traversal (traversal.hpp:162-184): every close pair exactly once.
template <int Dim, class Callback>
void pair_traversal(const Bvh<Dim> &bvh, float eps, Callback &&callback, ExecMode = ExecMode::kParallel) {
  if (bvh.size() < 2) return;
  std::int64_t total = 0;
  sp_ctx *ctx = detail::context();
  detail::check(ctx, sp_pair_list(ctx, bvh.handle(), eps, nullptr, 0, &total, SP_MEM_HOST));
  std::vector<std::int32_t> pairs((std::size_t)total * 2);
  if (total) detail::check(ctx, sp_pair_list(ctx, bvh.handle(), eps, pairs.data(), total, &total, SP_MEM_HOST));
  for (std::int64_t i = 0; i < total; ++i) callback(pairs[(std::size_t)(2 * i)], pairs[(std::size_t)(2 * i + 1)]);
}

// sort_queries (traversal.hpp:209-218)
template <int Dim, class Predicate>
std::vector<std::int32_t> sort_queries(std::span<const Predicate> preds) {
  std::vector<float> reps;
  for (const auto &p : preds) {
    Point<Dim> c;
    if constexpr (std::is_same_v<Predicate, NearestPredicate<Dim>>) {
      c = p.origin;
    } else if (const auto *s = std::get_if<Sphere<Dim>>(&p.geometry)) {
      c = s->center;
    } else {
      const auto &b = std::get<Aabb<Dim>>(p.geometry);
      for (int k = 0; k < Dim; ++k)
        c[k] = static_cast<float>((static_cast<double>(b.min_corner[k]) + static_cast<double>(b.max_corner[k])) * 0.5);
    }
    for (int k = 0; k < Dim; ++k) reps.push_back(c[k]);
  }
  std::vector<std::int32_t> order(preds.size());
  if (!preds.empty())
    detail::check(detail::context(), sp_sort_queries(detail::context(), reps.data(), (std::int64_t)preds.size(), Dim,
                                                     order.data(), SP_MEM_HOST));
  return order;
}

// ---- clustering (dbscan.hpp:22-53, 277-301) --------------------------------
inline constexpr std::int32_t kNoiseLabel = -1;

struct DbscanParams {
  float eps = 0.f;
  std::int32_t min_pts = 2;
};

struct DbscanTimings {
  double build_ms = 0, core_ms = 0, merge_ms = 0, finalize_ms = 0;
  double total_ms() const { return build_ms + core_ms + merge_ms + finalize_ms; }
};

struct DbscanStats {
  std::int64_t distance_checks = 0, num_dense_cells = 0, num_dense_points = 0;
};

struct DbscanOutput {
  std::vector<std::int32_t> labels;
  std::vector<std::uint8_t> core_flags;
  DbscanTimings timings;
  DbscanStats stats;
};

namespace detail {
template <int Dim>
DbscanOutput run_dbscan(std::span<const Point<Dim>> pts, float eps, std::int32_t min_pts, int algo, CodeWidth w) {
  DbscanOutput out;
  auto flat = flatten<Dim>(pts);
  out.labels.resize(pts.size());
  out.core_flags.resize(pts.size());
  sp_timings t{};
  sp_stats s{};
  check(context(), sp_dbscan(context(), flat.data(), (std::int64_t)pts.size(), Dim, eps, min_pts, algo,
                             static_cast<int>(w), out.labels.data(), out.core_flags.data(), &t, &s, SP_MEM_HOST));
  out.timings = {t.build_ms, t.core_ms, t.merge_ms, t.finalize_ms};
  out.stats = {s.distance_checks, s.num_dense_cells, s.num_dense_points};
  return out;
}
}  // namespace detail

// ExecMode::kSequential: the reference's deterministic sequential labels
// (sp_b200.h SP_ALGO_SEQUENTIAL); kParallel: any valid border assignment.
template <int Dim>
DbscanOutput fdbscan(std::span<const Point<Dim>> points, const DbscanParams &params,
                     ExecMode mode = ExecMode::kParallel, CodeWidth width = CodeWidth::k64) {
  const int seq = mode == ExecMode::kSequential ? SP_ALGO_SEQUENTIAL : 0;
  return detail::run_dbscan<Dim>(points, params.eps, params.min_pts, SP_ALGO_FDBSCAN | seq, width);
}

template <int Dim>
DbscanOutput friends_of_friends(std::span<const Point<Dim>> points, float eps, ExecMode = ExecMode::kParallel,
                                CodeWidth width = CodeWidth::k64) {
  return detail::run_dbscan<Dim>(points, eps, 2, SP_ALGO_FOF, width);
}

template <int Dim>
DbscanOutput fdbscan_densebox(std::span<const Point<Dim>> points, const DbscanParams &params,
                              ExecMode mode = ExecMode::kParallel, CodeWidth width = CodeWidth::k64) {
  const int seq = mode == ExecMode::kSequential ? SP_ALGO_SEQUENTIAL : 0;
  return detail::run_dbscan<Dim>(points, params.eps, params.min_pts, SP_ALGO_DENSEBOX | seq, width);
}

}  // namespace spatial_b200

#endif  // SPATIAL_B200_HPP
