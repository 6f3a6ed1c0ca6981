"""SURVEY §8(d) CPU baselines at the STATED sizes: the unmodified reference
(oracle/_ref) timed on this host's cores with OMP_PROC_BIND=close, median of
3 runs (C3: 1 run), the same calls the GPU configs time:
  C1 friends_of_friends, U(10^6)            (dbscan.hpp:286-292)
  C2 Bvh::build + sort_queries + range_query count, 2^24 x 2^24
                                            (bvh.hpp:243-261, traversal.hpp:67-87, 209-218)
  C3 fdbscan_densebox min_pts 5, H(2^26)    (dbscan.hpp:298-449)
  C4 Bvh::build + nearest_query k = 16, 2^24 x 2^24  (traversal.hpp:93-156)
Writes one JSON object (with nproc / lscpu) to OUT.  Baseline only.

    OMP_NUM_THREADS=$(nproc) OMP_PROC_BIND=close python scripts/cpu_baselines.py OUT.json [c1 c2 c3 c4]
"""
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np  # noqa: E402

from oracle_lib import Reference, eps_for  # noqa: E402

out_path = sys.argv[1]
which = sys.argv[2:] or ["c1", "c2", "c4", "c3"]
R = Reference.get()
res = json.load(open(out_path)) if os.path.exists(out_path) else {}
res["host"] = {"nproc": os.cpu_count(), "omp_num_threads": os.environ.get("OMP_NUM_THREADS"),
               "omp_proc_bind": os.environ.get("OMP_PROC_BIND"),
               "lscpu_model": subprocess.run("lscpu | grep 'Model name'", shell=True, capture_output=True,
                                             text=True).stdout.strip()}


def median_runs(fn, runs):
    secs, extra = [], None
    for _ in range(runs):
        t = time.perf_counter()
        extra = fn()
        secs.append(time.perf_counter() - t)
    return statistics.median(secs), secs, extra


for w in which:
    if w == "c1":
        n = 1000000
        p = R.uniform(n, 3, 1.0, 2409)
        med, secs, _ = median_runs(lambda: R.dbscan(p, 3, eps_for(n), 2, "fof"), 3)
        res[w] = {"call": "friends_of_friends", "n": n, "median_s": med, "runs_s": secs, "points_per_s": n / med}
    elif w == "c2":
        n = 1 << 24
        p = R.uniform(n, 3, 1.0, 2409)
        r = float(np.float32(np.cbrt(30.0 / (n * 4.18879020478639))))
        med, secs, last = median_runs(lambda: R.range_count(p, p, r), 3)
        counts, ms = last
        res[w] = {"call": "Bvh::build + sort_queries + range_query(count)", "n": n, "queries": n,
                  "median_s": med, "runs_s": secs, "queries_per_s": n / med,
                  "last_phase_ms": {"build": ms[0], "sort_queries": ms[1], "query": ms[2]},
                  "total_matches": int(counts.astype(np.int64).sum())}
    elif w == "c4":
        n = 1 << 24
        p = R.uniform(n, 3, 1.0, 2409)
        q = R.uniform(n, 3, 1.0, 2410)
        med, secs, last = median_runs(lambda: R.knn(p, q, 16), 3)
        res[w] = {"call": "Bvh::build + nearest_query(k=16)", "n": n, "queries": n, "median_s": med,
                  "runs_s": secs, "queries_per_s": n / med,
                  "last_phase_ms": {"build": last[1][0], "query": last[1][1]}}
    elif w == "c3":
        n = 1 << 26
        p = R.field(n)
        t = time.perf_counter()
        lab, core, stats, ms = R.dbscan(p, 3, eps_for(n), 5, "densebox", with_stats=True)
        dt = time.perf_counter() - t
        res[w] = {"call": "fdbscan_densebox(min_pts=5)", "n": n, "runs": 1, "seconds": dt, "points_per_s": n / dt,
                  "phase_ms": {"build": ms[0], "core": ms[1], "merge": ms[2], "finalize": ms[3]},
                  "dense_cells": int(stats[1]), "dense_points": int(stats[2]), "core": int(core.sum())}
    print(w, json.dumps(res[w]), flush=True)
    json.dump(res, open(out_path, "w"), indent=1)
