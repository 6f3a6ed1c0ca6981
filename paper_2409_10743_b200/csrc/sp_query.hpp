// Host entry points of the query and clustering kernels.
#pragma once

#include <stdint.h>

#include "sp_internal.hpp"

namespace spb {

enum RangeKind { RQ_RADIUS = 0, RQ_SPHERES = 1, RQ_BOXES = 2 };

// sort_queries over predicate representatives (kind 0 spheres, 1 boxes).
void query_order(Ctx &c, const float *preds, int64_t nq, int dim, int kind, int32_t *order);
// counts[q] = min(hits, cap) (cap <= 0: uncapped).  order_in: an optional
// precomputed query order (e.g. the tree's own leaf order for self-queries).
void range_count(Ctx &c, const Tree &t, int kind, const float *preds, int64_t nq, float radius, int32_t cap,
                 int32_t *counts, const int32_t *order_in);
// Returns the total; values are written only if total <= capacity.
int64_t range_crs(Ctx &c, const Tree &t, int kind, const float *preds, int64_t nq, int64_t *offsets, int32_t *values,
                  int64_t capacity);
int64_t pair_list(Ctx &c, const Tree &t, float eps, int32_t *pairs, int64_t capacity);
void knn(Ctx &c, const Tree &t, const float *origins, int64_t nq, int32_t k, int32_t *idx, float *dist);
void exclusive_scan(Ctx &c, const int32_t *in, int64_t n, int64_t *out);
void walk_lengths(Ctx &c, const Tree &t, float eps, int32_t *steps, int32_t *hits);
// -1 if equivalent, else the first violating point (kind 1..5, see sp_b200.h)
int64_t check_equivalence(Ctx &c, const float *pts, int64_t n, int dim, float eps, const int32_t *gl,
                          const uint8_t *gc, const int32_t *wl, const uint8_t *wc, int *kind);

struct DbscanResult {
  double ms[4] = {0, 0, 0, 0};  // build, core, merge, finalize
  int64_t distance_checks = 0, num_dense_cells = 0, num_dense_points = 0;
};
// labels/core: device arrays of n entries (original point order).
// ids (optional, device, n entries): FoF labels become the smallest ids[i] of
// each cluster instead of the smallest index (the distributed FoF passes
// global indices).
void dbscan(Ctx &c, const float *points, int64_t n, int dim, float eps, int32_t min_pts, int algo, int width,
            int32_t *labels, uint8_t *core, DbscanResult *res, const int32_t *ids = nullptr);

void adjacency_dbscan(Ctx &c, const float *points, int64_t n, int dim, float eps, int width, int64_t max_adjacency,
                      int32_t *labels, uint8_t *core, DbscanResult *res);

void bruteforce_dbscan(Ctx &c, const float *points, int64_t n, int dim, float eps, int32_t min_pts, int32_t *labels,
                       uint8_t *core);

void generate_field(Ctx &c, int64_t n_total, int64_t first, int64_t count, uint64_t seed, float *out);
void generate_uniform(Ctx &c, int64_t n, int dim, uint64_t seed, float *out);

}  // namespace spb
