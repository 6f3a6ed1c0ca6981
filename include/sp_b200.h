/*
 * sp_b200.h — the drop-in C ABI of the B200-native geometric-search and
 * clustering path (arXiv 2409.10743, "Advances in ArborX ...").
 *
 * The reference (/root/reference/proj/include/spatial/) is a header-only C++20
 * template library with no ABI: callers instantiate Bvh<D>::build,
 * range_query/nearest_query/pair_traversal with compile-time callbacks, and
 * fdbscan / friends_of_friends / fdbscan_densebox.  This header is what a
 * foreign binding (ctypes / cgo / JNI / the C++ facade in spatial_b200.hpp)
 * links against instead.  Every entry point names the reference interface it
 * replaces (file:line, relative to /root/reference/proj/include/spatial/).
 *
 * Conventions
 *   - Plain pointers and sizes; no C++ or torch types; no exceptions cross
 *     the ABI.  Every call returns an sp_status; sp_last_error(ctx) holds the
 *     message of the last failure on that context.
 *   - `mem` says where ALL array arguments of a call live: SP_MEM_HOST
 *     (pageable or pinned host memory; the call copies in and out on the
 *     context stream) or SP_MEM_DEVICE (device pointers on the context's
 *     device; nothing crosses PCIe).
 *   - Points are interleaved float[n*dim]; boxes are float[n*2*dim] laid out
 *     (min_0..min_{dim-1}, max_0..max_{dim-1}) per object, i.e. Aabb<D>
 *     (geometry.hpp:29-45).  dim is 2 or 3.
 *   - One context per host thread; calls on one context are serialised on its
 *     stream and are synchronous on return unless SP_FLAG_ASYNC is given
 *     (device memory only; the call then only enqueues work).
 *   - Results are bit-identical to the reference: leaf permutation, node
 *     arrays, neighbour counts, kNN indices and FoF labels.
 */
#ifndef SP_B200_H
#define SP_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  SP_OK = 0,
  SP_EINVAL = 1,     /* std::invalid_argument in the reference (bvh.hpp:251-252, dbscan.hpp:55-67) */
  SP_ECAPACITY = 2,  /* CapacityError : std::bad_alloc (traversal.hpp:229-231, 250-251) */
  SP_ECUDA = 3,      /* a CUDA runtime error (no reference counterpart) */
  SP_ENOMEM = 4,     /* device allocation failure */
  SP_ENCCL = 5       /* an NCCL error (multi-GPU slab path) */
} sp_status;

enum { SP_MEM_HOST = 0, SP_MEM_DEVICE = 1 };
enum { SP_FLAG_ASYNC = 1, SP_FLAG_STATS = 2 };

/* DBSCAN family selector (dbscan.hpp:277-301, 456-504).  FDBSCAN and FOF
 * cluster over grid cells when min_pts = 2; FOF_POINTS is
 * friends_of_friends by pair traversal over the point hierarchy, the
 * reference's own algorithm (dbscan.hpp:229-292), with identical results;
 * DENSEBOX_MIXED is fdbscan_densebox over the reference's mixed tree of dense
 * cells and sparse points (dbscan.hpp:298-449), equivalent results. */
enum { SP_ALGO_FDBSCAN = 0, SP_ALGO_FOF = 1, SP_ALGO_DENSEBOX = 2, SP_ALGO_FOF_POINTS = 3, SP_ALGO_DENSEBOX_MIXED = 4 };
/* OR'ed into the selector: ExecMode::kSequential (exec.hpp:12).  FDBSCAN with
 * min_pts > 2 then assigns every border point to the cluster of its core
 * neighbour of smallest leaf position, which is the claim the reference's
 * sequential pair traversal makes (dbscan.hpp:123-137, traversal.hpp:162-184):
 * labels equal the reference's sequential labels bit for bit.  DENSEBOX and
 * DENSEBOX_MIXED with min_pts > 2 run over the reference's mixed tree and give
 * a border point to the core neighbour the reference's sequential merge
 * (dbscan.hpp:406-442) reports first: bit-identical labels too.  Friends-of-
 * friends is deterministic in both modes. */
enum { SP_ALGO_SEQUENTIAL = 0x100 };

/* Range predicate kinds (traversal.hpp:25-28: variant<Sphere, Aabb>). */
enum { SP_PRED_SPHERE = 0, SP_PRED_BOX = 1 };

typedef struct sp_ctx sp_ctx;
typedef struct sp_bvh sp_bvh;
typedef struct sp_comm sp_comm;

/* DbscanTimings (dbscan.hpp:29-36): device-event times per phase, ms. */
typedef struct {
  double build_ms;
  double core_ms;
  double merge_ms;
  double finalize_ms;
} sp_timings;

/* DbscanStats (dbscan.hpp:40-44). */
typedef struct {
  int64_t distance_checks;
  int64_t num_dense_cells;
  int64_t num_dense_points;
} sp_stats;

/* ---- context (replaces ExecMode / parallel_for, exec.hpp:12-26) ---------- */
/* stream: a cudaStream_t to run on, or NULL for a context-owned stream
 * (cudaStreamLegacy, (void *)1, selects the legacy default stream). */
int sp_ctx_create(int device, void *stream, sp_ctx **out);
int sp_ctx_destroy(sp_ctx *ctx);
int sp_ctx_set_stream(sp_ctx *ctx, void *stream);
/* Wait for all work on ctx; reports (SP_EINVAL) input errors that calls made
 * with SP_FLAG_ASYNC found on the device. */
int sp_ctx_synchronize(sp_ctx *ctx);
/* SP_FLAG_ASYNC: sp_dbscan / sp_bvh_build only ENQUEUE work on the context
 * stream (host<->device copies included) and return; host buffers must stay
 * valid and untouched until sp_ctx_synchronize.  Two contexts on two streams
 * then pipeline consecutive calls (one call's copies overlap the other's
 * kernels).  Timings are not collected in this mode.
 * SP_FLAG_STATS: diagnostic twins of the traversal kernels also count their
 * work into sp_ctx_counter ("merge_node_visits", "merge_pair_tests" for the
 * FoF cell merge); slower, for measurement only. */
int sp_ctx_set_flags(sp_ctx *ctx, int flags);
const char *sp_last_error(const sp_ctx *ctx);
/* Number of kernels this library launched on ctx since creation. */
int64_t sp_ctx_kernel_launches(const sp_ctx *ctx);
/* Device-event phase breakdown of the last call on ctx (StopWatch lap times,
 * exec.hpp:28-41, at kernel granularity): phase i ran for sp_ctx_phase_ms(i)
 * milliseconds, e.g. "bounds", "morton", "sort", "hierarchy", "core",
 * "merge", "finalize". */
int sp_ctx_phase_count(const sp_ctx *ctx);
/* Diagnostic counter of the last call, -1 if absent (e.g. "fof_cells": the
 * number of non-empty grid cells the FoF pipeline clustered). */
int64_t sp_ctx_counter(const sp_ctx *ctx, const char *name);
const char *sp_ctx_phase_name(const sp_ctx *ctx, int i);
double sp_ctx_phase_ms(const sp_ctx *ctx, int i);

/* ---- hierarchy (Bvh<D>::build, bvh.hpp:62, 243-261) ---------------------- */
/* objects: points (is_points=1, float[n*dim]) or boxes (float[n*2*dim]).
 * code_width: 32 or 64 (CodeWidth, bvh.hpp:18).  n == 0 gives an empty tree.
 * Non-finite input -> SP_EINVAL ("bvh: non-finite object bounds"). */
int sp_bvh_build(sp_ctx *ctx, const float *objects, int64_t n, int dim, int is_points, int code_width, int mem,
                 sp_bvh **out);
int sp_bvh_destroy(sp_bvh *bvh);
int64_t sp_bvh_size(const sp_bvh *bvh); /* Bvh::size (bvh.hpp:64) */

/* Bvh fields internals/leaves/scene (bvh.hpp:45-60) copied out to HOST arrays
 * in the reference's numbering: internal node i in [0, n-1), leaf p in [0, n);
 * NodeRef values (left, rope) use internal [0,n-1) / leaves [n-1,2n-1) /
 * sentinel -1 (bvh.hpp:20-28).  Any pointer may be NULL to skip that array.
 * Boxes are float[2*dim] per node; scene is float[2*dim]. */
int sp_bvh_export(sp_ctx *ctx, const sp_bvh *bvh, int32_t *internal_left, int32_t *internal_rope,
                  float *internal_boxes, int32_t *leaf_object, int32_t *leaf_rope, float *leaf_boxes, float *scene);

/* ---- queries --------------------------------------------------------------- */
/* range_query with a counting callback (traversal.hpp:67-87); with cap > 0 the
 * callback terminates a query once its count reaches cap, exactly as
 * detect_core_counts does (dbscan.hpp:146-170), so counts[q] = min(hits, cap).
 * preds: SP_PRED_SPHERE -> float[nq*(dim+1)] (centre, radius);
 *        SP_PRED_BOX    -> float[nq*2*dim].
 * Queries are Morton-sorted internally (sort_queries, traversal.hpp:209-218);
 * results are reported in the caller's query order. */
int sp_range_count(sp_ctx *ctx, const sp_bvh *bvh, int pred_kind, const float *preds, int64_t nq, int32_t cap,
                   int32_t *counts, int mem);

/* Same as sp_range_count for spheres of one radius centred on float[nq*dim]. */
int sp_range_count_radius(sp_ctx *ctx, const sp_bvh *bvh, const float *centres, int64_t nq, float radius, int32_t cap,
                          int32_t *counts, int mem);

/* query_crs (traversal.hpp:235-266): offsets[nq+1]; values (object indices,
 * ascending per query) written only if offsets[nq] <= capacity, else
 * SP_ECAPACITY with offsets still filled.  values may be NULL with
 * capacity 0 to size the result first. */
int sp_range_crs(sp_ctx *ctx, const sp_bvh *bvh, int pred_kind, const float *preds, int64_t nq, int64_t *offsets,
                 int32_t *values, int64_t capacity, int mem);

/* nearest_query (traversal.hpp:93-156): for each origin float[nq*dim] the
 * min(k, n) objects nearest by (float min_distance, object index), ascending;
 * idx/dist are [nq*k], padded with -1 / +inf beyond min(k, n).  dist may be
 * NULL.  k <= 0 writes nothing. */
int sp_knn(sp_ctx *ctx, const sp_bvh *bvh, const float *origins, int64_t nq, int32_t k, int32_t *idx, float *dist,
           int mem);

/* pair_traversal (traversal.hpp:162-184) over a point tree: every unordered
 * pair within eps exactly once as (object a, object b) with a's leaf before
 * b's.  *num_pairs receives the total; pairs[2*i] are written only if the
 * total fits capacity (else SP_ECAPACITY). */
int sp_pair_list(sp_ctx *ctx, const sp_bvh *bvh, float eps, int32_t *pairs, int64_t capacity, int64_t *num_pairs,
                 int mem);

/* sort_queries (traversal.hpp:209-218) for point representatives
 * float[nq*dim]: the stable Morton-order permutation (64-bit codes against the
 * representatives' own scene). */
int sp_sort_queries(sp_ctx *ctx, const float *points, int64_t nq, int dim, int32_t *order, int mem);

/* Diagnostics: node visits and close pairs of each leaf's pair walk (leaf
 * order) for a point tree.  Not part of the reference surface. */
int sp_debug_walk_lengths(sp_ctx *ctx, const sp_bvh *bvh, float eps, int32_t *steps, int32_t *hits, int mem);

/* code_of over object centroids against their scene (morton.hpp:106-109). */
int sp_morton_codes(sp_ctx *ctx, const float *objects, int64_t n, int dim, int is_points, int code_width,
                    uint64_t *codes, int mem);

/* ---- clustering (fdbscan / friends_of_friends / fdbscan_densebox,
 *      dbscan.hpp:277-301) ---------------------------------------------------- */
/* labels[n]: smallest original index of the cluster, or -1 for noise
 * (finalize_labels, dbscan.hpp:72-98); core[n]: 0/1.  SP_ALGO_FOF ignores
 * min_pts (uses 2).  timings/stats may be NULL. */
int sp_dbscan(sp_ctx *ctx, const float *points, int64_t n, int dim, float eps, int32_t min_pts, int algo,
              int code_width, int32_t *labels, uint8_t *core, sp_timings *timings, sp_stats *stats, int mem);

/* friends_of_friends with caller-supplied point ids (device or host per
 * `mem`, n entries, distinct, >= 0): labels[i] = the smallest id of i's
 * cluster (-1 = noise) instead of the smallest index — the building block of
 * the multi-GPU slab FoF, which passes global indices (distributed.py). */
int sp_fof_ids(sp_ctx *ctx, const float *points, int64_t n, int dim, float eps, const int32_t *ids,
               int32_t *labels, uint8_t *core, int mem);

/* ---- multi-GPU friends-of-friends over x-slabs (SURVEY §8 row e) ----------
 * The reference has no distributed search; this is the paper's
 * ArborX-style partitioned FoF with one process (or
 * context) per GPU.  Every rank passes the rows [first_index, first_index +
 * n_local) of one global float[n_total*3] point array (3-D only,
 * n_total < 2^31) and receives exactly those rows' labels: the smallest
 * GLOBAL index of the point's cluster, or -1 for noise, and core flags — bit-
 * identical to sp_dbscan(SP_ALGO_FOF) on the whole array (friends_of_friends,
 * dbscan.hpp:286-292).  Each call is collective over the communicator.
 * Steps: quantile x-splitters from an all-reduced sample histogram; one
 * all-to-all of (xyz, global id) to the owner slab plus eps ghost copies to
 * the neighbouring slabs; local FoF in global-id space; an all-gather of the
 * (global id, label) links of every ghost copy; the same union-find on every
 * rank; relabelled rows returned by a second all-to-all.  One host read (a
 * G x 3G count matrix) sizes the exchanges; when it shows an empty exchange
 * (no row changes rank, no ghost anywhere) every rank runs the single-GPU FoF
 * on its rows in place instead (labels offset by first_index). */
/* NCCL unique id for sp_comm_create: made by one rank, passed to all. */
int sp_comm_unique_id(uint8_t id[128]);
/* ncclCommInitRank over nranks processes (one GPU each) on ctx's device. */
int sp_comm_create(sp_ctx *ctx, int nranks, int rank, const uint8_t id[128], sp_comm **out);
/* Use the caller's ncclComm_t (not owned: sp_comm_destroy leaves it open). */
int sp_comm_wrap(sp_ctx *ctx, void *nccl_comm, sp_comm **out);
int sp_comm_destroy(sp_comm *comm);
int sp_comm_size(const sp_comm *comm);
int sp_comm_rank(const sp_comm *comm);
int sp_fof_slabs(sp_ctx *ctx, sp_comm *comm, const float *points, int64_t n_local, float eps, int64_t first_index,
                 int32_t *labels, uint8_t *core, int mem);
/* The same step with all nranks ranks in this process: ctxs[r] (one device
 * each, or several contexts on one device) holds points[r] (n_local[r]
 * rows; rank r's rows follow rank r-1's); exchanges are peer copies between
 * the contexts' streams.  Errors are reported on ctxs[0]. */
int sp_fof_slabs_multi(sp_ctx *const *ctxs, int nranks, const float *const *points, const int64_t *n_local, float eps,
                       int32_t *const *labels, uint8_t *const *core, int mem);

/* adjacency_graph_dbscan (dbscan.hpp:456-504): the legacy min_pts = 2
 * baseline that materialises the eps-neighbourhood CRS; SP_ECAPACITY when
 * the total exceeds max_adjacency (its CapacityError). */
int sp_dbscan_adjacency(sp_ctx *ctx, const float *points, int64_t n, int dim, float eps, int code_width,
                        int64_t max_adjacency, int32_t *labels, uint8_t *core, sp_timings *timings, int mem);

/* dbscan_reference (dbscan.hpp:188-222): brute-force O(n^2) DBSCAN on the
 * device, independent of the tree — the reference CLI's --verify / --algo
 * oracle counterpart, for small inputs. */
int sp_dbscan_bruteforce(sp_ctx *ctx, const float *points, int64_t n, int dim, float eps, int32_t min_pts,
                         int32_t *labels, uint8_t *core, int mem);

/* check_equivalence (verify.hpp:21-61): *violation = -1 when `got` is an
 * equivalent clustering of `want`, else the index of the first violating
 * point with *kind = 1 core flag, 2 noise, 3 core partition split, 4 core
 * clusters merged, 5 border point without an in-cluster core point within
 * eps.  The border test is a tree walk, not the reference's O(n^2) scan. */
int sp_check_equivalence(sp_ctx *ctx, const float *points, int64_t n, int dim, float eps, const int32_t *got_labels,
                         const uint8_t *got_core, const int32_t *want_labels, const uint8_t *want_core,
                         int64_t *violation, int *kind, int mem);

/* ---- synthetic input (for benchmarks; no reference counterpart) ---------- */
/* HACC-like clustered field of SURVEY §8(d) shape — 25% uniform background
 * plus Gaussian halos of 8192 points, sigma = 0.001*cbrt(2^26/n_total),
 * clamped to the unit cube — generated on the device with a counter-based
 * (Philox) stream so any slice [first, first+count) of the n_total-point field
 * can be produced independently (out: float[count*3], device or host). */
int sp_generate_field(sp_ctx *ctx, int64_t n_total, int64_t first, int64_t count, uint64_t seed, float *out,
                      int mem);
/* The reference's generators (generate.cpp:17-66) with the same engine and
 * distributions (std::mt19937_64, uniform_real / normal <double>), so specs
 * reproduce its bits: kind 0 uniform(n, dim, extent), kind 1
 * gaussian_clusters(n, dim, k, sigma, extent, seed).  Host memory. */
int sp_generate_reference(int kind, int64_t n, int dim, int32_t k, double sigma, double extent, uint64_t seed,
                          float *out);
/* Rows [first, first+count) of the SURVEY §8(d) field H(n_total): the
 * reference generator's uniform(n_total/4, 3, 1.0, seed 2409) followed by
 * gaussian_clusters(n_total - n_total/4, 3, max((n_total-n_total/4)/8192, 1),
 * 0.001*cbrt(2^26/n_total), 1.0, seed 2410), bit-identical to generate()
 * (generate.cpp:17-66).  Host memory, float[count*3]. */
int sp_generate_reference_field(int64_t n_total, int64_t first, int64_t count, float *out);
/* Uniform points in [0,1)^dim from the same Philox stream. */
int sp_generate_uniform(sp_ctx *ctx, int64_t n, int dim, uint64_t seed, float *out, int mem);

#ifdef __cplusplus
}
#endif

#endif /* SP_B200_H */
