"""Golden fixtures for ExecMode::kSequential (exec.hpp:12) from the UNMODIFIED
reference (oracle/_ref/libref.so, `make -C oracle ref`): fdbscan and
fdbscan_densebox run sequentially, whose border assignment is deterministic
(dbscan.hpp:123-137, 406-442), so the labels are compared bit for bit.  Run
here, where /root/reference exists:

    python tests/golden/make_seq_golden.py        -> tests/golden/seq_cases.npz
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
from oracle_lib import Reference  # noqa: E402


def main():
    R = Reference.get()
    rng = np.random.default_rng(504)
    out, names = {}, []

    def add(name, pts, dim, eps, min_pts):
        names.append(name)
        out[name + "/points"] = pts
        out[name + "/meta"] = np.array([dim, min_pts], np.int32)
        out[name + "/eps"] = np.float32(eps)
        for algo, key in (("fdbscan_seq", "fd"), ("densebox_seq", "db")):
            l, c = R.dbscan(pts, dim, eps, min_pts, algo)
            l2, _ = R.dbscan(pts, dim, eps, min_pts, algo)
            assert np.array_equal(l, l2), "sequential run not repeatable"
            out[name + "/%s_labels" % key] = l
            out[name + "/%s_core" % key] = c

    def mixture(n, dim, k, sigma, seed):
        r = np.random.default_rng(seed)
        centres = r.random((k, dim))
        blobs = centres[r.integers(0, k, n // 2)] + r.standard_normal((n // 2, dim)) * sigma
        return np.clip(np.concatenate([blobs, r.random((n - n // 2, dim))]), 0, 1).astype(np.float32)

    add("mix3_m5", mixture(6000, 3, 12, 0.03, 1), 3, 0.05, 5)
    add("mix3_m8", mixture(8000, 3, 20, 0.02, 2), 3, 0.04, 8)
    add("mix3_m3", mixture(5000, 3, 8, 0.02, 3), 3, 0.03, 3)
    add("mix2_m6", mixture(5000, 2, 10, 0.02, 4), 2, 0.02, 6)
    add("mix2_m4", mixture(3000, 2, 6, 0.05, 5), 2, 0.03, 4)
    grid = (rng.integers(0, 12, (3000, 3)) / 11).astype(np.float32)  # duplicates and ties at eps
    add("dups3_m4", grid, 3, 1.0 / 11, 4)
    blob = np.array([[0, 0], [0.1, 0], [0, 0.1], [0.1, 0.1], [0.25, 0.05], [0.2, -0.05], [5, 5]], np.float32)
    add("blob_border", blob, 2, 0.15, 4)
    out["names"] = np.array(names)
    np.savez_compressed(os.path.join(HERE, "seq_cases.npz"), **out)
    for nm in names:
        c = out[nm + "/db_core"]
        print(nm, "core", int(c.sum()), "border", int(((out[nm + "/db_labels"] >= 0) & (c == 0)).sum()))


if __name__ == "__main__":
    main()
