// ============================================================================
// ORACLE — TEST INFRASTRUCTURE ONLY.  Never linked into, loaded by, or called
// from the product path (paper_2409_10743_b200/).  Only tests/, the smoke()
// check in __graft_entry__.py and bench.py's cpu_baseline leg may use it, and
// only as the checker.
//
// A sequential CPU restatement of the reference's geometric-search and
// clustering semantics (/root/reference/proj/include/spatial/*.hpp).  It is
// written independently of the reference code paths it checks:
//   * the hierarchy is built TOP-DOWN by recursive arg-min splitting of the
//     adjacent augmented-key prefixes (the reference uses Karras' per-node
//     binary searches plus a skip table); the unique binary radix tree makes
//     both produce the same node arrays, numbering and ropes;
//   * range / kNN queries use an explicit-stack DFS and a best-first search
//     instead of the reference's rope walk;
//   * clustering enumerates within-eps neighbours and applies a sequential
//     union-find, then the reference's label/noise rules.
// Parity is PINNED: tests/golden/ holds outputs of the unmodified reference
// (compiled from /root/reference by oracle/Makefile into oracle/_ref/) and the
// FNV-1a-64 hashes SURVEY.md §8(c) recorded; tests/test_oracle.py checks this
// restatement against both.
//
// Every function cites the reference file:line whose semantics it restates.
// ============================================================================
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <limits>
#include <map>
#include <numeric>
#include <queue>
#include <random>
#include <array>
#include <vector>

namespace {

constexpr int32_t kNone = -1;

// ---- geometry (geometry.hpp:73-96, 116-128, 130-137) ------------------------
// Box stored as lo[3], hi[3]; 2-D data carries z = 0 which adds an exact 0.0
// to every double accumulation, so one 3-D routine serves both dimensions.
struct Box {
  float lo[3];
  float hi[3];
};

// min_distance: per-axis gap max(lo-p, p-hi, 0) squared and summed in double,
// sqrt in double, one rounding to float (geometry.hpp:86-96).
inline float gap_distance(const float p[3], const Box &b) {
  double acc = 0.0;
  for (int k = 0; k < 3; ++k) {
    double below = (double)b.lo[k] - (double)p[k];
    double above = (double)p[k] - (double)b.hi[k];
    double g = below > above ? below : above;
    if (g < 0.0) g = 0.0;
    acc = acc + g * g;
  }
  return (float)std::sqrt(acc);
}

// closed-interval overlap on every axis (geometry.hpp:121-128)
inline bool boxes_touch(const Box &a, const Box &b) {
  for (int k = 0; k < 3; ++k)
    if (a.lo[k] > b.hi[k] || b.lo[k] > a.hi[k]) return false;
  return true;
}

// std::min / std::max tie semantics: keep the first argument unless the second
// compares strictly smaller / larger (geometry.hpp:98-114).
inline float keep_min(float a, float b) { return b < a ? b : a; }
inline float keep_max(float a, float b) { return a < b ? b : a; }

inline Box join(const Box &a, const Box &b) {
  Box r;
  for (int k = 0; k < 3; ++k) {
    r.lo[k] = keep_min(a.lo[k], b.lo[k]);
    r.hi[k] = keep_max(a.hi[k], b.hi[k]);
  }
  return r;
}

inline Box empty_box() {
  Box b;
  for (int k = 0; k < 3; ++k) {
    b.lo[k] = std::numeric_limits<float>::max();
    b.hi[k] = std::numeric_limits<float>::lowest();
  }
  return b;
}

inline bool finite_box(const Box &b) {
  for (int k = 0; k < 3; ++k)
    if (!std::isfinite(b.lo[k]) || !std::isfinite(b.hi[k])) return false;
  return true;
}

std::vector<Box> boxes_from(const float *v, int64_t n, int dim, bool is_points) {
  std::vector<Box> out((size_t)n);
  for (int64_t i = 0; i < n; ++i) {
    Box &b = out[(size_t)i];
    for (int k = 0; k < 3; ++k) {
      if (k >= dim) {
        b.lo[k] = b.hi[k] = 0.f;
      } else if (is_points) {
        b.lo[k] = b.hi[k] = v[i * dim + k];
      } else {
        b.lo[k] = v[i * 2 * dim + k];
        b.hi[k] = v[i * 2 * dim + dim + k];
      }
    }
  }
  return out;
}

// ---- Morton codes (morton.hpp:17-109) ---------------------------------------
// Quantisation in double: floor((c - lo) / extent * 2^bits) clamped to
// [0, 2^bits - 1]; non-positive extent -> 0.  Interleave: bit b of axis k goes
// to code bit b*dim + k (restated with a plain bit loop, not magic masks).
uint64_t morton_code(const float c[3], const Box &scene, int dim, int width) {
  const int bits = width / dim;
  const uint32_t top = bits >= 32 ? 0xffffffffu : ((1u << bits) - 1u);
  const double scale = std::ldexp(1.0, bits);
  uint32_t bin[3] = {0, 0, 0};
  for (int k = 0; k < dim; ++k) {
    double extent = (double)scene.hi[k] - (double)scene.lo[k];
    if (!(extent > 0.0)) continue;
    double t = ((double)c[k] - (double)scene.lo[k]) / extent;
    double f = std::floor(t * scale);
    if (f <= 0.0) bin[k] = 0;
    else if (f >= (double)top) bin[k] = top;
    else bin[k] = (uint32_t)f;
  }
  uint64_t code = 0;
  for (int b = 0; b < bits; ++b)
    for (int k = 0; k < dim; ++k)
      code |= (uint64_t)((bin[k] >> b) & 1u) << (b * dim + k);
  return code;
}

// centroid: double midpoint rounded to float (geometry.hpp:130-137)
inline void centre_of(const Box &b, float c[3]) {
  for (int k = 0; k < 3; ++k) c[k] = (float)(((double)b.lo[k] + (double)b.hi[k]) * 0.5);
}

// ---- hierarchy (bvh.hpp:20-28, 45-55, 100-261) ------------------------------
struct Tree {
  int32_t n = 0;
  int width = 64;
  Box scene = empty_box();
  std::vector<int32_t> perm;        // leaf position -> object index
  std::vector<Box> leaf_box;        // n
  std::vector<int32_t> leaf_rope;   // n
  std::vector<Box> node_box;        // n-1 internals (Karras numbering)
  std::vector<int32_t> node_left;   // n-1
  std::vector<int32_t> node_rope;   // n-1
  int32_t root() const { return n == 0 ? kNone : (n == 1 ? 0 : 0); }
  bool is_leaf(int32_t ref) const { return ref >= n - 1; }
  int32_t leaf_ref(int32_t pos) const { return n - 1 + pos; }
  const Box &box(int32_t ref) const { return is_leaf(ref) ? leaf_box[ref - (n - 1)] : node_box[ref]; }
  int32_t rope(int32_t ref) const { return is_leaf(ref) ? leaf_rope[ref - (n - 1)] : node_rope[ref]; }
};

// Length of the common prefix of the augmented keys (code, object id) of two
// adjacent sorted entries (bvh.hpp:90-115).
inline int adjacent_prefix(uint64_t ca, uint64_t cb, int32_t ia, int32_t ib, int width) {
  if (ca != cb) {
    uint64_t x = ca ^ cb;
    int lz = 0;
    for (int b = width - 1; b >= 0 && !((x >> b) & 1ull); --b) ++lz;
    return lz;
  }
  uint32_t y = (uint32_t)ia ^ (uint32_t)ib;
  int lz = 0;
  for (int b = 31; b >= 0 && !((y >> b) & 1u); --b) ++lz;
  return width + (y == 0 ? 32 : lz);
}

// Bvh::build (bvh.hpp:243-261): finite check + scene fold, centroid codes,
// stable sort, radix-tree hierarchy with Karras numbering, exact union boxes
// (left child first), ropes.  Returns false on non-finite input.
bool build_tree(const std::vector<Box> &objs, int dim, int width, Tree &t) {
  t = Tree{};
  t.width = width;
  const int64_t n = (int64_t)objs.size();
  t.n = (int32_t)n;
  if (n == 0) return true;
  for (const Box &b : objs) {
    if (!finite_box(b)) return false;
    t.scene = join(t.scene, b);
  }
  std::vector<uint64_t> code((size_t)n);
  for (int64_t i = 0; i < n; ++i) {
    float c[3];
    centre_of(objs[(size_t)i], c);
    code[(size_t)i] = morton_code(c, t.scene, dim, width);
  }
  // Stable order by code == order by (code, index) because indices are unique.
  t.perm.resize((size_t)n);
  std::iota(t.perm.begin(), t.perm.end(), 0);
  std::sort(t.perm.begin(), t.perm.end(), [&](int32_t a, int32_t b) {
    return code[(size_t)a] != code[(size_t)b] ? code[(size_t)a] < code[(size_t)b] : a < b;
  });
  t.leaf_box.resize((size_t)n);
  t.leaf_rope.assign((size_t)n, kNone);
  for (int64_t p = 0; p < n; ++p) t.leaf_box[(size_t)p] = objs[(size_t)t.perm[(size_t)p]];
  if (n == 1) return true;

  std::vector<int> adj((size_t)(n - 1));
  for (int64_t i = 0; i + 1 < n; ++i)
    adj[(size_t)i] = adjacent_prefix(code[(size_t)t.perm[(size_t)i]], code[(size_t)t.perm[(size_t)i + 1]],
                                     t.perm[(size_t)i], t.perm[(size_t)i + 1], width);

  t.node_box.assign((size_t)(n - 1), empty_box());
  t.node_left.assign((size_t)(n - 1), kNone);
  t.node_rope.assign((size_t)(n - 1), kNone);
  std::vector<int32_t> node_right((size_t)(n - 1), kNone);

  // Top-down: a node covering [l, r] splits where the adjacent prefix over
  // [l, r-1] is smallest (unique for distinct augmented keys).  The left child
  // [l, s] carries Karras index s, the right child [s+1, r] index s+1.
  struct Item { int32_t l, r, idx, rope; };
  std::vector<Item> stack;
  std::vector<int32_t> order;  // internal nodes in pre-order
  order.reserve((size_t)(n - 1));
  stack.push_back({0, (int32_t)(n - 1), 0, kNone});
  while (!stack.empty()) {
    Item it = stack.back();
    stack.pop_back();
    int32_t s = it.l;
    for (int32_t i = it.l + 1; i < it.r; ++i)
      if (adj[(size_t)i] < adj[(size_t)s]) s = i;
    int32_t left = (s == it.l) ? t.leaf_ref(s) : s;
    int32_t right = (s + 1 == it.r) ? t.leaf_ref(s + 1) : s + 1;
    t.node_left[(size_t)it.idx] = left;
    node_right[(size_t)it.idx] = right;
    t.node_rope[(size_t)it.idx] = it.rope;
    order.push_back(it.idx);
    // rope(left) = right sibling; rope(right) = rope(parent)
    if (s == it.l) t.leaf_rope[(size_t)s] = right;
    else stack.push_back({it.l, s, s, right});
    if (s + 1 == it.r) t.leaf_rope[(size_t)(s + 1)] = it.rope;
    else stack.push_back({s + 1, it.r, s + 1, it.rope});
  }
  for (size_t q = order.size(); q-- > 0;) {
    int32_t i = order[q];
    t.node_box[(size_t)i] = join(t.box(t.node_left[(size_t)i]), t.box(node_right[(size_t)i]));
  }
  return true;
}

// ---- queries -----------------------------------------------------------------
// Range predicate: sphere (centre, radius) hit <=> gap_distance <= radius
// (geometry.hpp:116-119); box predicate hit <=> boxes_touch.
struct Pred {
  bool is_box;
  float c[3];
  float r;
  Box b;
};

inline bool pred_hits(const Pred &q, const Box &v) {
  return q.is_box ? boxes_touch(v, q.b) : (gap_distance(q.c, v) <= q.r);
}

// Number of stored objects hit, saturating at cap (cap <= 0: no cap).  With the
// reference's terminate-at-threshold callback the invocation count equals
// min(hits, cap) independent of visiting order (dbscan.hpp:146-170).
template <class Fn>
void dfs_hits(const Tree &t, const Pred &q, Fn &&on_object) {
  if (t.n == 0) return;
  std::vector<int32_t> st;
  st.push_back(t.n == 1 ? t.leaf_ref(0) : 0);
  while (!st.empty()) {
    int32_t ref = st.back();
    st.pop_back();
    if (!pred_hits(q, t.box(ref))) continue;
    if (t.is_leaf(ref)) {
      if (!on_object(t.perm[(size_t)(ref - (t.n - 1))])) return;
      continue;
    }
    int32_t left = t.node_left[(size_t)ref];
    st.push_back(t.rope(left));  // right child
    st.push_back(left);
  }
}

// ---- union-find (union_find.hpp:17-59), sequential -----------------------------
struct Sets {
  std::vector<int32_t> up;
  explicit Sets(int64_t n) : up((size_t)n) { std::iota(up.begin(), up.end(), 0); }
  int32_t root(int32_t i) {
    int32_t r = i;
    while (up[(size_t)r] != r) r = up[(size_t)r];
    while (up[(size_t)i] != r) { int32_t nx = up[(size_t)i]; up[(size_t)i] = r; i = nx; }
    return r;
  }
  void join(int32_t a, int32_t b) {
    a = root(a); b = root(b);
    if (a == b) return;
    if (a < b) up[(size_t)b] = a; else up[(size_t)a] = b;  // smaller index is the root
  }
};

// finalize_labels (dbscan.hpp:72-98): label = smallest member of the set, or
// -1 for a non-core point in a singleton set.
void finalize(Sets &s, const uint8_t *core, int64_t n, int32_t *labels) {
  std::vector<int32_t> least((size_t)n, std::numeric_limits<int32_t>::max());
  std::vector<int32_t> count((size_t)n, 0);
  for (int64_t i = 0; i < n; ++i) {
    int32_t r = s.root((int32_t)i);
    least[(size_t)r] = std::min(least[(size_t)r], (int32_t)i);
    ++count[(size_t)r];
  }
  for (int64_t i = 0; i < n; ++i) {
    int32_t r = s.root((int32_t)i);
    labels[i] = (!core[i] && count[(size_t)r] == 1) ? -1 : least[(size_t)r];
  }
}

// ---- dense grid (dense_grid.hpp:52-103) -------------------------------------
struct Grid {
  float cell = 0.f;
  bool no_dense = false;
  std::vector<std::array<int64_t, 3>> key;  // per point
};

Grid grid_keys(const std::vector<Box> &pts, int dim, float eps) {
  Grid g;
  g.cell = (float)((double)eps / std::sqrt((double)dim) * (1.0 - 1e-6));
  Box scene = empty_box();
  for (const Box &b : pts) scene = join(scene, b);
  g.no_dense = !(g.cell > 0.f);
  for (int k = 0; k < dim && !g.no_dense; ++k) {
    double extent = (double)scene.hi[k] - (double)scene.lo[k];
    g.no_dense = extent / (double)g.cell >= 4.0e18;
  }
  if (!(g.cell > 0.f)) g.cell = 1.f;
  g.key.resize(pts.size());
  for (size_t i = 0; i < pts.size(); ++i) {
    std::array<int64_t, 3> c = {0, 0, 0};
    for (int k = 0; k < dim; ++k) {
      double f = std::floor(((double)pts[i].lo[k] - (double)scene.lo[k]) / (double)g.cell);
      f = std::min(std::max(f, -4.0e18), 4.0e18);
      c[(size_t)k] = (int64_t)f;
    }
    g.key[i] = c;
  }
  return g;
}

}  // namespace

// ============================================================================
// C ABI (consumed by tests via ctypes)
// ============================================================================
extern "C" {

// FNV-1a-64 over raw bytes (the SURVEY §8(c) golden-hash definition).
uint64_t orc_fnv1a64(const void *data, int64_t nbytes) {
  const unsigned char *p = (const unsigned char *)data;
  uint64_t h = 1469598103934665603ull;
  for (int64_t i = 0; i < nbytes; ++i) h = (h ^ p[i]) * 1099511628211ull;
  return h;
}

// generate_uniform (src/generate.cpp:17-31): mt19937_64(seed), one
// uniform_real_distribution<double>(0, extent) draw per coordinate, cast to float.
int orc_generate_uniform(int64_t n, int dim, double extent, uint64_t seed, float *out) {
  if (n < 0 || (dim != 2 && dim != 3) || !(extent > 0)) return 1;
  std::mt19937_64 rng(seed);
  std::uniform_real_distribution<double> u(0.0, extent);
  for (int64_t i = 0; i < n * dim; ++i) out[i] = (float)u(rng);
  return 0;
}

// generate_gaussian_clusters (src/generate.cpp:33-66): centres first, then
// each point's coordinates centre + N(0, sigma), clamped to [0, extent];
// clusters own equal ceil(n/k) blocks (the last takes the rest).
int orc_generate_gaussian(int64_t n, int dim, int32_t k, double sigma, double extent, uint64_t seed,
                          float *out) {
  if (n < 0 || (dim != 2 && dim != 3) || k < 1 || !(sigma >= 0) || !(extent > 0)) return 1;
  std::mt19937_64 rng(seed);
  std::uniform_real_distribution<double> u(0.0, extent);
  std::normal_distribution<double> g(0.0, sigma);
  std::vector<double> ctr((size_t)k * (size_t)dim);
  for (double &c : ctr) c = u(rng);
  const int64_t block = (n + k - 1) / k;
  for (int64_t i = 0; i < n; ++i) {
    int64_t c = std::min<int64_t>(i / block, k - 1);
    for (int d = 0; d < dim; ++d) {
      double v = ctr[(size_t)(c * dim + d)] + g(rng);
      v = std::min(std::max(v, 0.0), extent);
      out[i * dim + d] = (float)v;
    }
  }
  return 0;
}

// The SURVEY §8(d) HACC-like field H(n): U(n/4, 2409) followed by
// gaussian(n - n/4, 3, (n - n/4)/8192 halos, 0.001*cbrt(2^26/n), 1.0, 2410).
int orc_generate_field(int64_t n, float *out) {
  int64_t nbg = n / 4, nh = n - nbg;
  if (orc_generate_uniform(nbg, 3, 1.0, 2409, out)) return 1;
  int32_t k = (int32_t)(nh / 8192);
  if (k < 1) k = 1;
  return orc_generate_gaussian(nh, 3, k, 0.001 * std::cbrt(67108864.0 / (double)n), 1.0, 2410,
                               out + nbg * 3);
}

// Morton codes of object centroids against the scene (morton.hpp:106-109).
int orc_morton_codes(const float *v, int64_t n, int dim, int is_points, int width, uint64_t *codes) {
  auto objs = boxes_from(v, n, dim, is_points != 0);
  Box scene = empty_box();
  for (const Box &b : objs) scene = join(scene, b);
  for (int64_t i = 0; i < n; ++i) {
    float c[3];
    centre_of(objs[(size_t)i], c);
    codes[i] = morton_code(c, scene, dim, width);
  }
  return 0;
}

// Bvh<D>::build node arrays.  internal_* hold n-1 entries, leaf_* n entries;
// boxes are (min xyz..., max xyz...) with `dim` coordinates each.
int orc_bvh_build(const float *v, int64_t n, int dim, int is_points, int width, int32_t *internal_left,
                  int32_t *internal_rope, float *internal_boxes, int32_t *leaf_object, int32_t *leaf_rope,
                  float *leaf_boxes) {
  Tree t;
  if (!build_tree(boxes_from(v, n, dim, is_points != 0), dim, width, t)) return 1;
  auto put = [dim](float *dst, const Box &b) {
    for (int k = 0; k < dim; ++k) { dst[k] = b.lo[k]; dst[dim + k] = b.hi[k]; }
  };
  for (int64_t i = 0; i + 1 < n; ++i) {
    internal_left[i] = t.node_left[(size_t)i];
    internal_rope[i] = t.node_rope[(size_t)i];
    put(internal_boxes + i * 2 * dim, t.node_box[(size_t)i]);
  }
  for (int64_t p = 0; p < n; ++p) {
    leaf_object[p] = t.perm[(size_t)p];
    leaf_rope[p] = t.leaf_rope[(size_t)p];
    put(leaf_boxes + p * 2 * dim, t.leaf_box[(size_t)p]);
  }
  return 0;
}

// range_query with a counting callback (traversal.hpp:67-87, dbscan.hpp:146-170).
// Objects: points or boxes.  Predicates: spheres (dim+1 floats: centre, radius)
// when pred_is_box == 0, else boxes (2*dim floats).  cap <= 0 means no cap.
int orc_range_count(const float *v, int64_t n, int dim, int is_points, const float *preds, int64_t nq,
                    int pred_is_box, int32_t cap, int32_t *counts) {
  Tree t;
  if (!build_tree(boxes_from(v, n, dim, is_points != 0), dim, 64, t)) return 1;
#pragma omp parallel for schedule(dynamic, 256)
  for (int64_t q = 0; q < nq; ++q) {
    Pred p{};
    p.is_box = pred_is_box != 0;
    if (p.is_box) {
      p.b = boxes_from(preds + q * 2 * dim, 1, dim, false)[0];
    } else {
      for (int k = 0; k < 3; ++k) p.c[k] = k < dim ? preds[q * (dim + 1) + k] : 0.f;
      p.r = preds[q * (dim + 1) + dim];
    }
    int32_t c = 0;
    dfs_hits(t, p, [&](int32_t) { ++c; return !(cap > 0 && c >= cap); });
    counts[q] = c;
  }
  return 0;
}

// CRS of matches (traversal.hpp:222-266): offsets[nq+1], values sorted per row.
// Pass values == nullptr to obtain only offsets.
int orc_range_crs(const float *v, int64_t n, int dim, int is_points, const float *spheres, int64_t nq,
                  int64_t *offsets, int32_t *values) {
  Tree t;
  if (!build_tree(boxes_from(v, n, dim, is_points != 0), dim, 64, t)) return 1;
  offsets[0] = 0;
  std::vector<int32_t> row;
  for (int64_t q = 0; q < nq; ++q) {
    Pred p{};
    for (int k = 0; k < 3; ++k) p.c[k] = k < dim ? spheres[q * (dim + 1) + k] : 0.f;
    p.r = spheres[q * (dim + 1) + dim];
    row.clear();
    dfs_hits(t, p, [&](int32_t o) { row.push_back(o); return true; });
    std::sort(row.begin(), row.end());
    if (values) std::copy(row.begin(), row.end(), values + offsets[q]);
    offsets[q + 1] = offsets[q] + (int64_t)row.size();
  }
  return 0;
}

// nearest_query (traversal.hpp:93-156): the min(k, n) objects smallest by
// (float distance to the object box, object index), ascending.  Best-first
// search; a node is skipped only if its distance is strictly worse than the
// current k-th, which keeps index tie-breaks exact.  idx/dist are nq*k,
// padded with -1 / +inf past min(k, n).
int orc_knn(const float *v, int64_t n, int dim, int is_points, const float *origins, int64_t nq, int32_t k,
            int32_t *idx, float *dist) {
  Tree t;
  if (!build_tree(boxes_from(v, n, dim, is_points != 0), dim, 64, t)) return 1;
  if (k <= 0) return 0;
#pragma omp parallel for schedule(dynamic, 64)
  for (int64_t q = 0; q < nq; ++q) {
    float o[3];
    for (int d = 0; d < 3; ++d) o[d] = d < dim ? origins[q * dim + d] : 0.f;
    typedef std::pair<float, int32_t> Cand;  // (dist, object) ordered lexicographically
    std::priority_queue<Cand> best;          // max-heap: top = worst kept
    typedef std::pair<float, int32_t> Item;  // (dist, node ref)
    std::priority_queue<Item, std::vector<Item>, std::greater<Item>> open;
    if (t.n > 0) {
      int32_t r = t.n == 1 ? t.leaf_ref(0) : 0;
      open.push({gap_distance(o, t.box(r)), r});
    }
    while (!open.empty()) {
      Item it = open.top();
      open.pop();
      if ((int64_t)best.size() == k && it.first > best.top().first) break;
      if (t.is_leaf(it.second)) {
        Cand c{it.first, t.perm[(size_t)(it.second - (t.n - 1))]};
        if ((int64_t)best.size() < k) best.push(c);
        else if (c < best.top()) { best.pop(); best.push(c); }
        continue;
      }
      int32_t left = t.node_left[(size_t)it.second];
      int32_t right = t.rope(left);
      open.push({gap_distance(o, t.box(left)), left});
      open.push({gap_distance(o, t.box(right)), right});
    }
    int64_t m = (int64_t)best.size();
    for (int64_t j = k - 1; j >= 0; --j) {
      if (j >= m) {
        idx[q * k + j] = -1;
        if (dist) dist[q * k + j] = std::numeric_limits<float>::infinity();
        continue;
      }
      idx[q * k + j] = best.top().second;
      if (dist) dist[q * k + j] = best.top().first;
      best.pop();
    }
  }
  return 0;
}

// DBSCAN family (dbscan.hpp:229-292, 298-449) on points.
//   min_pts == 2 : friends-of-friends; labels are unique (every close pair
//                  unions; core <=> set size > 1).
//   min_pts  > 2 : exact capped core counts; core-core pairs union; each
//                  border point joins the set of its first core neighbour in
//                  index order (the reference's claim latch picks any one —
//                  compare with orc_check_equivalence, not label identity).
// stats (may be null): [0] distance checks the DenseBox merge performs,
// [1] dense cells, [2] dense-cell points (dense_grid.hpp:71-103, dbscan.hpp:
// 344-345, 407-431) for the grid of cell length eps/sqrt(d)*(1-1e-6).
// Returns 1 for invalid params (dbscan.hpp:55-60) or non-finite points.
int orc_dbscan(const float *v, int64_t n, int dim, float eps, int32_t min_pts, int32_t *labels,
               uint8_t *core, int64_t *stats) {
  if (!(eps > 0) || !std::isfinite(eps) || min_pts < 2) return 1;
  auto pts = boxes_from(v, n, dim, true);
  for (const Box &b : pts)
    if (!finite_box(b)) return 1;
  if (n == 0) return 0;
  Tree t;
  build_tree(pts, dim, 64, t);
  auto ball = [&](int64_t i) {
    Pred p{};
    p.is_box = false;
    for (int k = 0; k < 3; ++k) p.c[k] = pts[(size_t)i].lo[k];
    p.r = eps;
    return p;
  };
  std::vector<int32_t> cnt((size_t)n, 0);
#pragma omp parallel for schedule(dynamic, 256)
  for (int64_t i = 0; i < n; ++i) {
    int32_t c = 0;
    dfs_hits(t, ball(i), [&](int32_t) { ++c; return c < min_pts; });
    cnt[(size_t)i] = c;
  }
  for (int64_t i = 0; i < n; ++i) core[i] = cnt[(size_t)i] >= min_pts;
  Sets s(n);
  std::vector<int32_t> nb;
  for (int64_t i = 0; i < n; ++i) {
    if (!core[i]) continue;
    nb.clear();
    dfs_hits(t, ball(i), [&](int32_t o) { nb.push_back(o); return true; });
    for (int32_t j : nb)
      if (j != i && core[j]) s.join((int32_t)i, j);
  }
  for (int64_t b = 0; b < n; ++b) {
    if (core[b]) continue;
    nb.clear();
    dfs_hits(t, ball(b), [&](int32_t o) { nb.push_back(o); return true; });
    std::sort(nb.begin(), nb.end());
    for (int32_t j : nb)
      if (j != b && core[j]) { s.join((int32_t)b, j); break; }
  }
  finalize(s, core, n, labels);

  if (stats) {
    // DenseBox bookkeeping: grid cells, dense cells (>= min_pts members, none
    // when coordinates could saturate), and the merge phase's per-member
    // distance checks: for every point i and every dense cell c != cell(i)
    // whose tight box is within eps of i, the members j > i of c.
    Grid g = grid_keys(pts, dim, eps);
    std::map<std::array<int64_t, 3>, std::vector<int32_t>> cells;
    for (int64_t i = 0; i < n; ++i) cells[g.key[(size_t)i]].push_back((int32_t)i);
    std::vector<Box> tight;
    std::vector<std::vector<int32_t>> members;
    std::vector<int32_t> cell_of((size_t)n, -1);
    for (auto &kv : cells) {
      if (g.no_dense || (int64_t)kv.second.size() < min_pts) continue;
      Box b = empty_box();
      for (int32_t i : kv.second) { b = join(b, pts[(size_t)i]); cell_of[(size_t)i] = (int32_t)tight.size(); }
      tight.push_back(b);
      members.push_back(kv.second);
    }
    int64_t dense_pts = 0;
    for (auto &m : members) dense_pts += (int64_t)m.size();
    int64_t checks = 0;
    if (!tight.empty()) {
      Tree ct;
      build_tree(tight, dim, 64, ct);
      std::vector<int32_t> id_of((size_t)0);
      for (int64_t i = 0; i < n; ++i) {
        Pred p = ball(i);
        dfs_hits(ct, p, [&](int32_t c) {
          if (c == cell_of[(size_t)i]) return true;
          const auto &m = members[(size_t)c];
          checks += (int64_t)(m.end() - std::upper_bound(m.begin(), m.end(), (int32_t)i));
          return true;
        });
      }
    }
    stats[0] = checks;
    stats[1] = (int64_t)tight.size();
    stats[2] = dense_pts;
  }
  return 0;
}

// check_equivalence (verify.hpp:21-61): core flags equal, noise sets equal,
// bijective label map on core points, and every border point's label names a
// cluster holding a core point within eps.  The border scan uses a tree
// instead of the reference's O(n^2) loop.  Returns -1 when equivalent, else
// the index of the first violating point (with *kind set to 1 core, 2 noise,
// 3 partition, 4 merged clusters, 5 border).
int64_t orc_check_equivalence(const float *v, int64_t n, int dim, float eps, const int32_t *got_labels,
                              const uint8_t *got_core, const int32_t *want_labels, const uint8_t *want_core,
                              int32_t *kind) {
  *kind = 0;
  for (int64_t i = 0; i < n; ++i)
    if ((got_core[i] != 0) != (want_core[i] != 0)) { *kind = 1; return i; }
  for (int64_t i = 0; i < n; ++i)
    if ((got_labels[i] == -1) != (want_labels[i] == -1)) { *kind = 2; return i; }
  std::map<int32_t, int32_t> fwd, rev;
  for (int64_t i = 0; i < n; ++i) {
    if (!want_core[i]) continue;
    auto f = fwd.emplace(want_labels[i], got_labels[i]);
    if (!f.second && f.first->second != got_labels[i]) { *kind = 3; return i; }
    auto r = rev.emplace(got_labels[i], want_labels[i]);
    if (!r.second && r.first->second != want_labels[i]) { *kind = 4; return i; }
  }
  auto pts = boxes_from(v, n, dim, true);
  Tree t;
  build_tree(pts, dim, 64, t);
  for (int64_t b = 0; b < n; ++b) {
    if (got_core[b] || got_labels[b] == -1) continue;
    Pred p{};
    for (int k = 0; k < 3; ++k) p.c[k] = pts[(size_t)b].lo[k];
    p.r = eps;
    bool ok = false;
    dfs_hits(t, p, [&](int32_t c) {
      if (got_core[c] && got_labels[c] == got_labels[b]) { ok = true; return false; }
      return true;
    });
    if (!ok) { *kind = 5; return b; }
  }
  return -1;
}

// float distance between two points as the reference computes it
// (geometry.hpp:73-81), for KAT tests.
float orc_distance(const float *a, const float *b, int dim) {
  Box pb;
  for (int k = 0; k < 3; ++k) pb.lo[k] = pb.hi[k] = k < dim ? b[k] : 0.f;
  float pa[3] = {a[0], a[1], dim > 2 ? a[2] : 0.f};
  return gap_distance(pa, pb);
}

}  // extern "C"
