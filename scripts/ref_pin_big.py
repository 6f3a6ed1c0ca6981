"""Pin the FoF labels of the SURVEY §8(d) field H(2^k) to the UNMODIFIED
reference at sizes where Python-side copies would not fit host RAM (2^30:
~140 GB): oracle/_ref's ref_fof_field generates H(n) with the reference's
generate(), runs friends_of_friends (dbscan.hpp:286-292) and hashes the
outputs in one process.  Test infrastructure only; results go into
tests/golden/golden_hashes.json ("H_2^k").

    OMP_NUM_THREADS=$(nproc) OMP_PROC_BIND=close python scripts/ref_pin_big.py OUT.json K [K ...]
"""
import ctypes as C
import json
import os
import resource
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
L = C.CDLL(os.path.join(ROOT, "oracle", "_ref", "libref.so"))
L.ref_fof_field.argtypes = [C.c_int64, C.c_void_p, C.c_void_p, C.c_void_p]

out_path = sys.argv[1]
res = json.load(open(out_path)) if os.path.exists(out_path) else {}
for k in map(int, sys.argv[2:]):
    h = (C.c_uint64 * 4)()
    cnt = (C.c_int64 * 3)()
    secs = (C.c_double * 2)()
    assert L.ref_fof_field(1 << k, h, cnt, secs) == 0
    res["H_2^%d" % k] = {"n": 1 << k, "points_hash": "%016x" % h[0], "labels_hash": "%016x" % h[1],
                         "core_hash": "%016x" % h[2], "labels_checksum": int(h[3]), "clusters": cnt[0],
                         "noise": cnt[1], "core": cnt[2], "gen_seconds": round(secs[0], 2),
                         "ref_seconds": round(secs[1], 2), "threads": os.environ.get("OMP_NUM_THREADS"),
                         "maxrss_gb": round(resource.getrusage(resource.RUSAGE_SELF).ru_maxrss / 1e6, 1)}
    print(json.dumps(res["H_2^%d" % k]), flush=True)
    json.dump(res, open(out_path, "w"), indent=1)
