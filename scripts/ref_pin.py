"""Pin large configs to the UNMODIFIED reference (oracle/_ref/libref.so).

Runs the reference's friends_of_friends (dbscan.hpp:286-292) on the reference
generator's H(n) field with all host threads and writes the
labels / core-flag FNV-1a-64 hashes, the cluster / noise / core counts, the
bench checksum (bench.py:labels_checksum) and the run time to a JSON file.
Test infrastructure only: the output is committed into
tests/golden/golden_hashes.json by hand (keys "H_2^k").

    python scripts/ref_pin.py OUT.json LOG2N [LOG2N ...]
"""
import json
import os
import resource
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "tests"))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

from fixtures import summarize  # noqa: E402
from oracle_lib import Reference, eps_for, fnv1a64  # noqa: E402


def checksum(labels: np.ndarray) -> int:
    # must equal bench.py labels_checksum (computed on the device there)
    i = np.arange(labels.size, dtype=np.int64)
    w = (i % 65521) + 1
    return int(((labels.astype(np.int64) + 1) * w).sum() & ((1 << 63) - 1))


def main():
    out_path = sys.argv[1]
    res = {}
    if os.path.exists(out_path):
        with open(out_path) as f:
            res = json.load(f)
    R = Reference.get()
    for k in [int(a) for a in sys.argv[2:]]:
        n = 1 << k
        t = time.perf_counter()
        pts = R.field(n)
        tgen = time.perf_counter() - t
        eps = eps_for(n)
        t = time.perf_counter()
        lab, core, stats, ms = R.dbscan(pts, 3, eps, 2, "fof", with_stats=True)
        dt = time.perf_counter() - t
        c, noise, ncore = summarize(lab, core)
        res["H_2^%d" % k] = {
            "n": n, "eps_bits": "%08x" % np.float32(eps).view(np.uint32), "points_hash": fnv1a64(pts),
            "clusters": c, "noise": noise, "core": ncore, "core_hash": fnv1a64(core), "labels_hash": fnv1a64(lab),
            "labels_checksum": checksum(lab), "ref_seconds": round(dt, 2), "gen_seconds": round(tgen, 2),
            "ref_phase_ms": [round(float(x), 1) for x in ms], "threads": os.environ.get("OMP_NUM_THREADS"),
            "maxrss_gb": round(resource.getrusage(resource.RUSAGE_SELF).ru_maxrss / 1e6, 1)}
        print(json.dumps({k2: v for k2, v in res.items() if k2 == "H_2^%d" % k}), flush=True)
        del pts, lab, core
        with open(out_path, "w") as f:
            json.dump(res, f, indent=1)


if __name__ == "__main__":
    main()
