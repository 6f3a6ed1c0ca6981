"""Regenerate the golden fixtures in tests/golden/ from the UNMODIFIED
reference (oracle/_ref/libref.so, built from /root/reference by
`make -C oracle ref`).  Run here, where /root/reference exists:

    python tests/golden/make_golden.py

Outputs (all small; committed):
  bvh_cases.npz     inputs + reference Bvh node arrays (bvh.hpp:243-261)
  query_cases.npz   range counts (traversal.hpp:67-87) and kNN indices
                    (traversal.hpp:93-156) for sphere/box/kNN predicates
  dbscan_cases.npz  friends_of_friends / fdbscan / fdbscan_densebox outputs
                    and DenseBox stats (dbscan.hpp:277-449)
  generator.json    FNV-1a-64 of reference generator outputs (generate.cpp)
golden_hashes.json (hand-maintained) holds the SURVEY §8(c) full-size hashes.
"""
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
from oracle_lib import Reference, Oracle  # noqa: E402


def bvh_cases(R):
    rng = np.random.default_rng(20240917)
    cases = []
    cases.append(("empty3", np.zeros((0, 3), np.float32), 3, 64, True))
    cases.append(("single3", np.array([[0.5, 0.5, 0.5]], np.float32), 3, 64, True))
    cases.append(("two2", np.array([[0.1, 0.1], [0.9, 0.9]], np.float32), 2, 64, True))
    cases.append(("golden3leaf2", np.array([[0.1, 0.1], [0.9, 0.9], [0.5, 0.25]], np.float32), 2, 64, True))
    cases.append(("collinear8", np.stack([np.arange(8, dtype=np.float32) / 7, np.zeros(8, np.float32),
                                          np.zeros(8, np.float32)], 1), 3, 64, True))
    cases.append(("identical257_32", np.tile(np.array([[0.25, 0.5, 0.75]], np.float32), (257, 1)), 3, 32, True))
    cases.append(("identical257_64", np.tile(np.array([[0.25, 0.5, 0.75]], np.float32), (257, 1)), 3, 64, True))
    clumps = np.array([[0.125 if i % 2 else 0.875] * 3 for i in range(500)], np.float32)
    clumps[:, 0] += rng.random(500, dtype=np.float32) * 1e-7
    cases.append(("clumps500_32", clumps, 3, 32, True))
    cases.append(("zero_extent_z", np.concatenate([rng.random((300, 2), dtype=np.float32),
                                                  np.full((300, 1), 0.5, np.float32)], 1), 3, 64, True))
    for dim in (2, 3):
        for width in (32, 64):
            cases.append(("rand%d_%d" % (dim, width), rng.random((777, dim), dtype=np.float32), dim, width, True))
            lo = rng.random((333, dim), dtype=np.float32)
            boxes = np.concatenate([lo, lo + rng.random((333, dim), dtype=np.float32) * 0.05], 1)
            cases.append(("boxes%d_%d" % (dim, width), boxes, dim, width, False))
            grid = (rng.integers(0, 6, (600, dim)) / 5).astype(np.float32)
            cases.append(("dups%d_%d" % (dim, width), grid, dim, width, True))
    # signed zeros and negative coordinates
    sz = rng.standard_normal((400, 3)).astype(np.float32)
    sz[::7, 1] = -0.0
    sz[::5, 1] = 0.0
    cases.append(("signed_zero", sz, 3, 64, True))
    out = {}
    names = []
    for name, objs, dim, width, pts in cases:
        r = R.bvh(objs, dim, width, pts)
        names.append(name)
        out[name + "/objects"] = objs
        out[name + "/meta"] = np.array([dim, width, int(pts)], np.int32)
        for k, v in r.items():
            out[name + "/" + k] = v
    out["names"] = np.array(names)
    np.savez_compressed(os.path.join(HERE, "bvh_cases.npz"), **out)


def query_cases(R, O):
    rng = np.random.default_rng(7)
    out = {}
    pts = rng.random((2000, 3), dtype=np.float32)
    # sphere range counts through the reference (Bvh::build + sort_queries + range_query)
    qs = rng.random((1500, 3), dtype=np.float32)
    counts, _ = R.range_count(pts, qs, 0.05)
    capped, _ = R.range_count(pts, qs, 0.05, cap=4)
    out.update({"rc/points": pts, "rc/centres": qs, "rc/radius": np.float32(0.05), "rc/counts": counts,
                "rc/capped4": capped})
    # kNN with ties (duplicated grid points) through nearest_query
    grid = (rng.integers(0, 8, (1200, 3)) / 7).astype(np.float32)
    org = (rng.integers(0, 15, (800, 3)) / 14).astype(np.float32)
    for k in (1, 5, 16, 32):
        idx, _ = R.knn(grid, org, k)
        out["knn/idx%d" % k] = idx
    out["knn/points"] = grid
    out["knn/origins"] = org
    idx, _ = R.knn(pts, qs, 16)
    out["knn/rand_idx16"] = idx
    np.savez_compressed(os.path.join(HERE, "query_cases.npz"), **out)


def dbscan_cases(R):
    rng = np.random.default_rng(11)
    out = {}
    names = []

    def add(name, pts, dim, eps, min_pts):
        names.append(name)
        out[name + "/points"] = pts
        out[name + "/meta"] = np.array([dim, min_pts], np.int32)
        out[name + "/eps"] = np.float32(eps)
        l, c = R.dbscan(pts, dim, eps, min_pts, "fof" if min_pts == 2 else "fdbscan")
        out[name + "/labels"] = l
        out[name + "/core"] = c
        l2, c2, st, _ = R.dbscan(pts, dim, eps, min_pts, "densebox", with_stats=True)
        out[name + "/db_labels"] = l2
        out[name + "/db_core"] = c2
        out[name + "/db_stats"] = st

    def clustered(n, dim, k, sigma, seed):
        r = np.random.default_rng(seed)
        centres = r.random((k, dim))
        pts = centres[r.integers(0, k, n)] + r.standard_normal((n, dim)) * sigma
        bg = r.random((n // 10, dim))
        return np.clip(np.concatenate([pts, bg]), 0, 1).astype(np.float32)

    add("uniform3_fof", rng.random((5000, 3), dtype=np.float32), 3, 0.02, 2)
    add("clustered3_fof", clustered(6000, 3, 12, 0.01, 1), 3, 0.01, 2)
    add("clustered3_m4", clustered(6000, 3, 12, 0.01, 2), 3, 0.01, 4)
    add("clustered3_m10", clustered(6000, 3, 12, 0.01, 3), 3, 0.012, 10)
    add("clustered2_fof", clustered(4000, 2, 8, 0.01, 4), 2, 0.01, 2)
    add("clustered2_m5", clustered(4000, 2, 8, 0.01, 5), 2, 0.01, 5)
    add("tiny_eps", rng.random((500, 3), dtype=np.float32), 3, 1e-30, 3)
    blob = np.array([[0, 0], [0.1, 0], [0, 0.1], [0.1, 0.1], [0.25, 0.05], [5, 5]], np.float32)
    add("blob_border_noise", blob, 2, 0.15, 4)
    dense = np.concatenate([np.full((40, 3), 0.5, np.float32), rng.random((200, 3), dtype=np.float32)])
    add("one_dense_cell", dense, 3, 0.05, 5)
    out["names"] = np.array(names)
    np.savez_compressed(os.path.join(HERE, "dbscan_cases.npz"), **out)


def generator_hashes(R, O):
    res = {}
    res["U(1000,3,2409)"] = "%016x" % O.fnv(R.uniform(1000, 3, 1.0, 2409))
    res["U(1000,2,7)"] = "%016x" % O.fnv(R.uniform(1000, 2, 1.0, 7))
    res["G(5000,3,7,0.01,1,5)"] = "%016x" % O.fnv(R.gaussian(5000, 3, 7, 0.01, 1.0, 5))
    res["H(65536)"] = "%016x" % O.fnv(R.field(65536))
    with open(os.path.join(HERE, "generator.json"), "w") as f:
        json.dump(res, f, indent=1, sort_keys=True)


if __name__ == "__main__":
    if not Reference.available():
        sys.exit("oracle/_ref/libref.so missing: run `make -C oracle ref` where /root/reference exists")
    R, O = Reference.get(), Oracle.get()
    bvh_cases(R)
    query_cases(R, O)
    dbscan_cases(R)
    generator_hashes(R, O)
    print("fixtures written to", HERE)
