"""Loaders for the committed golden fixtures (tests/golden/, made by
tests/golden/make_golden.py from the unmodified reference)."""
import json
import os

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def _cases(fname):
    z = np.load(os.path.join(GOLDEN, fname))
    names = [str(s) for s in z["names"]]
    out = {}
    for nm in names:
        pre = nm + "/"
        out[nm] = {k[len(pre):]: z[k] for k in z.files if k.startswith(pre)}
    return out


def bvh_cases():
    return _cases("bvh_cases.npz")


def dbscan_cases():
    return _cases("dbscan_cases.npz")


def query_cases():
    z = np.load(os.path.join(GOLDEN, "query_cases.npz"))
    return {k: z[k] for k in z.files}


def generator_hashes():
    with open(os.path.join(GOLDEN, "generator.json")) as f:
        return json.load(f)


def golden_hashes():
    with open(os.path.join(GOLDEN, "golden_hashes.json")) as f:
        return json.load(f)


BVH_KEYS = ("internal_left", "internal_rope", "internal_boxes", "leaf_object", "leaf_rope", "leaf_boxes")


def same_bits(a, b) -> bool:
    a, b = np.asarray(a), np.asarray(b)
    return a.shape == b.shape and np.array_equal(np.ascontiguousarray(a).view(np.uint8),
                                                 np.ascontiguousarray(b).view(np.uint8))


def summarize(labels, core):
    labels = np.asarray(labels)
    noise = int((labels == -1).sum())
    clusters = int(np.unique(labels[labels != -1]).size)
    return clusters, noise, int(np.asarray(core).sum())
