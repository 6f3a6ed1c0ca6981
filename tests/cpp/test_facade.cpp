// Reference-style unit tests (proj/tests/test_bvh.cpp, test_traversal.cpp,
// test_dbscan.cpp) written against the C++ façade include/spatial_b200.hpp:
// the same calls and known answers, served by the sm_100a kernels.
#include <cmath>
#include <cstdio>
#include <random>
#include <set>
#include <sstream>

#include "spatial_b200.hpp"

using namespace spatial_b200;

static int g_fail = 0, g_checks = 0;
#define CHECK(c)                                                         \
  do {                                                                   \
    ++g_checks;                                                          \
    if (!(c)) {                                                          \
      ++g_fail;                                                          \
      std::fprintf(stderr, "%s:%d: CHECK(%s) failed\n", __FILE__, __LINE__, #c); \
    }                                                                    \
  } while (0)

template <int D>
static std::vector<Aabb<D>> boxes_of(const std::vector<Point<D>> &p) {
  std::vector<Aabb<D>> b;
  for (const auto &x : p) b.push_back(point_box(x));
  return b;
}

static float ref_distance(const Point<3> &a, const Point<3> &b) {
  double s = 0;
  for (int k = 0; k < 3; ++k) {
    double d = (double)a[k] - (double)b[k];
    s += d * d;
  }
  return (float)std::sqrt(s);
}

int main() {
  {  // test_bvh.cpp:193-205 golden serialization of a three-leaf tree
    std::vector<Point<2>> p{{{0.1f, 0.1f}}, {{0.9f, 0.9f}}, {{0.5f, 0.25f}}};
    auto bvh = Bvh<2>::build(boxes_of(p));
    std::ostringstream os;
    bvh.dump(os);
    CHECK(os.str() ==
          "bvh n 3 width 64\n"
          "I 0 left 1 rope -1 0.100000001 0.100000001 0.899999976 0.899999976\n"
          "I 1 left 2 rope 4 0.100000001 0.100000001 0.5 0.25\n"
          "L 0 object 0 rope 3 0.100000001 0.100000001 0.100000001 0.100000001\n"
          "L 1 object 2 rope 4 0.5 0.25 0.5 0.25\n"
          "L 2 object 1 rope -1 0.899999976 0.899999976 0.899999976 0.899999976\n");
    CHECK(bvh.validate());
  }
  {  // test_bvh.cpp:39-44, 188-191: empty tree; non-finite input is rejected
    auto bvh = Bvh<3>::build({});
    CHECK(bvh.empty() && bvh.root() == kSentinel);
    std::vector<Aabb<3>> bad{point_box(Point<3>{{0, 0, std::nanf("")}})};
    bool threw = false;
    try {
      Bvh<3>::build(bad);
    } catch (const std::invalid_argument &) {
      threw = true;
    }
    CHECK(threw);
  }
  std::mt19937 rng(42);
  std::uniform_real_distribution<float> u(0.f, 1.f);
  std::vector<Point<3>> pts(3000);
  for (auto &p : pts) p = Point<3>{{u(rng), u(rng), u(rng)}};
  auto bvh = Bvh<3>::build(boxes_of(pts));
  CHECK(bvh.validate());
  {  // test_traversal.cpp:71-95 range query == brute force (spheres and boxes)
    std::vector<RangePredicate<3>> preds;
    for (int q = 0; q < 200; ++q) {
      Point<3> c{{u(rng), u(rng), u(rng)}};
      if (q % 2) preds.push_back({Sphere<3>{c, 0.08f}});
      else preds.push_back({Aabb<3>(c, Point<3>{{c[0] + 0.1f, c[1] + 0.05f, c[2] + 0.07f}})});
    }
    std::vector<std::set<int>> got(preds.size());
    range_query<3>(bvh, preds, [&](std::int32_t q, std::int32_t o) { got[q].insert(o); });
    bool ok = true;
    for (std::size_t q = 0; q < preds.size(); ++q) {
      std::set<int> want;
      for (std::size_t i = 0; i < pts.size(); ++i) {
        bool hit;
        if (const auto *s = std::get_if<Sphere<3>>(&preds[q].geometry)) {
          hit = ref_distance(pts[i], s->center) <= s->radius;
        } else {
          const auto &b = std::get<Aabb<3>>(preds[q].geometry);
          hit = true;
          for (int k = 0; k < 3; ++k) hit = hit && pts[i][k] >= b.min_corner[k] && pts[i][k] <= b.max_corner[k];
        }
        if (hit) want.insert((int)i);
      }
      ok = ok && (want == got[q]);
    }
    CHECK(ok);
  }
  {  // test_traversal.cpp:97-126 early termination stops exactly the emitting query
    std::vector<RangePredicate<3>> preds(2, RangePredicate<3>{Sphere<3>{Point<3>{{0.5f, 0.5f, 0.5f}}, 10.f}});
    std::vector<int> calls(2, 0);
    range_query<3>(bvh, preds, [&](std::int32_t q, std::int32_t) {
      ++calls[q];
      return (q == 0 && calls[q] == 3) ? CallbackControl::kTerminateQuery : CallbackControl::kContinue;
    });
    CHECK(calls[0] == 3 && calls[1] == (int)pts.size());
  }
  {  // test_traversal.cpp:144-168 kNN at a stored point; k >= n
    std::vector<NearestPredicate<3>> preds{{pts[7], 1}, {pts[9], 5000}};
    std::vector<std::vector<int>> got(2);
    nearest_query<3>(bvh, preds, [&](std::int32_t q, std::int32_t o) { got[q].push_back(o); });
    CHECK(got[0].size() == 1 && got[0][0] == 7);
    CHECK(got[1].size() == pts.size() && got[1][0] == 9);
  }
  {  // test_traversal.cpp:232-281 pair traversal: each close pair exactly once
    std::set<std::pair<int, int>> seen;
    std::size_t calls = 0;
    pair_traversal<3>(bvh, 0.05f, [&](std::int32_t a, std::int32_t b) {
      ++calls;
      seen.insert({std::min(a, b), std::max(a, b)});
    });
    std::size_t want = 0;
    for (std::size_t i = 0; i < pts.size(); ++i)
      for (std::size_t j = i + 1; j < pts.size(); ++j) want += ref_distance(pts[i], pts[j]) <= 0.05f;
    CHECK(calls == want && seen.size() == want);
  }
  {  // test_traversal.cpp:369-379 CRS capacity overflow
    std::vector<RangePredicate<3>> preds(1, RangePredicate<3>{Sphere<3>{Point<3>{{0.5f, 0.5f, 0.5f}}, 10.f}});
    bool threw = false;
    try {
      query_crs<3>(bvh, preds, ExecMode::kParallel, 10);
    } catch (const CapacityError &) {
      threw = true;
    }
    CHECK(threw);
  }
  {  // test_dbscan.cpp:67-81 blob, border and noise with min_pts = 4
    std::vector<Point<2>> p{{{0.50f, 0.50f}}, {{0.52f, 0.50f}}, {{0.50f, 0.52f}},
                            {{0.59f, 0.50f}}, {{0.68f, 0.50f}}, {{0.95f, 0.95f}}};
    auto out = fdbscan<2>(p, DbscanParams{0.1f, 4});
    CHECK((out.core_flags == std::vector<std::uint8_t>{1, 1, 1, 1, 0, 0}));
    CHECK((out.labels == std::vector<std::int32_t>{0, 0, 0, 0, 0, kNoiseLabel}));
    auto db = fdbscan_densebox<2>(p, DbscanParams{0.1f, 4});
    CHECK(db.labels == out.labels);
  }
  {  // test_dbscan.cpp:284-293 FoF chains connect, singletons are noise
    std::vector<Point<2>> chain;
    for (int i = 0; i < 10; ++i) chain.push_back({{static_cast<float>(i) * 0.09f, 0.f}});
    chain.push_back({{5.f, 5.f}});
    auto out = friends_of_friends<2>(chain, 0.1f);
    bool ok = true;
    for (int i = 0; i < 10; ++i) ok = ok && out.labels[i] == 0;
    CHECK(ok && out.labels[10] == kNoiseLabel);
  }
  {  // test_dbscan.cpp:45-53 parameter validation
    std::vector<Point<3>> p(3);
    int threw = 0;
    try { fdbscan<3>(p, DbscanParams{0.f, 2}); } catch (const std::invalid_argument &) { ++threw; }
    try { fdbscan<3>(p, DbscanParams{0.1f, 1}); } catch (const std::invalid_argument &) { ++threw; }
    CHECK(threw == 2);
  }
  std::printf("%d checks, %d failed\n", g_checks, g_fail);
  return g_fail ? 1 : 0;
}
