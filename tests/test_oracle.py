"""CPU: pin the oracle restatement (oracle/oracle.cpp) against the reference's
own outputs — the committed golden fixtures, the SURVEY §8(c) hashes, the
reference tests' known-answer values, and (when oracle/_ref was built here)
the unmodified reference itself on random instances."""
import numpy as np
import pytest

from fixtures import _cases, BVH_KEYS, bvh_cases, dbscan_cases, generator_hashes, golden_hashes, query_cases, same_bits, \
    summarize
from oracle_lib import Reference, eps_for, fnv1a64


def test_generator_matches_reference_hashes(oracle):
    g = generator_hashes()
    assert fnv1a64(oracle.uniform(1000, 3, 1.0, 2409)) == g["U(1000,3,2409)"]
    assert fnv1a64(oracle.uniform(1000, 2, 1.0, 7)) == g["U(1000,2,7)"]
    assert fnv1a64(oracle.gaussian(5000, 3, 7, 0.01, 1.0, 5)) == g["G(5000,3,7,0.01,1,5)"]
    assert fnv1a64(oracle.field(65536)) == g["H(65536)"]


@pytest.mark.parametrize("name", list(bvh_cases().keys()))
def test_bvh_node_arrays_match_reference(oracle, name):
    case = bvh_cases()[name]
    dim, width, pts = (int(v) for v in case["meta"])
    got = oracle.bvh(case["objects"], dim, width, bool(pts))
    for k in BVH_KEYS:
        assert same_bits(got[k], case[k]), (name, k)


def test_bvh_golden_three_leaf_dump(oracle):
    # test_bvh.cpp:193-205: the reference's golden serialization
    e = oracle.bvh(np.array([[0.1, 0.1], [0.9, 0.9], [0.5, 0.25]], np.float32), 2)
    assert e["internal_left"].tolist() == [1, 2] and e["internal_rope"].tolist() == [-1, 4]
    assert e["leaf_object"].tolist() == [0, 2, 1] and e["leaf_rope"].tolist() == [3, 4, -1]
    assert ["%.9g" % v for v in e["internal_boxes"][1]] == ["0.100000001", "0.100000001", "0.5", "0.25"]


def test_range_counts_match_reference(oracle):
    q = query_cases()
    r = float(q["rc/radius"])
    spheres = np.concatenate([q["rc/centres"], np.full((len(q["rc/centres"]), 1), r, np.float32)], 1)
    assert np.array_equal(oracle.range_count(q["rc/points"], 3, spheres), q["rc/counts"])
    assert np.array_equal(oracle.range_count(q["rc/points"], 3, spheres, cap=4), q["rc/capped4"])


@pytest.mark.parametrize("k", [1, 5, 16, 32])
def test_knn_matches_reference_with_ties(oracle, k):
    q = query_cases()
    idx, _ = oracle.knn(q["knn/points"], 3, q["knn/origins"], k)
    assert np.array_equal(idx, q["knn/idx%d" % k])


@pytest.mark.parametrize("name", list(dbscan_cases().keys()))
def test_dbscan_matches_reference(oracle, name):
    c = dbscan_cases()[name]
    dim, min_pts = (int(v) for v in c["meta"])
    eps = float(c["eps"])
    labels, core, stats = oracle.dbscan(c["points"], dim, eps, min_pts, with_stats=True)
    assert np.array_equal(core, c["core"])
    assert np.array_equal(core, c["db_core"])
    if min_pts == 2:
        assert np.array_equal(labels, c["labels"])
        assert np.array_equal(labels, c["db_labels"])
    else:
        assert oracle.check_equivalence(c["points"], dim, eps, (labels, core), (c["labels"], c["core"])) is None
        assert oracle.check_equivalence(c["points"], dim, eps, (labels, core), (c["db_labels"], c["db_core"])) is None
    assert stats.tolist() == c["db_stats"].tolist()


def test_equivalence_checker_flags_corruption(oracle):
    # test_dbscan.cpp:340-404: the checker must catch each kind of fault
    c = dbscan_cases()["clustered3_m4"]
    pts, eps = c["points"], float(c["eps"])
    want = (c["labels"], c["core"])
    core = want[1].copy()
    core[np.argmax(core)] ^= 1
    assert oracle.check_equivalence(pts, 3, eps, (want[0], core), want)[1] == 1
    lab = want[0].copy()
    i = int(np.argmax(lab == -1))
    lab[i] = 0
    assert oracle.check_equivalence(pts, 3, eps, (lab, want[1]), want)[1] in (2, 5)


def test_distance_kats(oracle):
    # test_geometry.cpp:11-15
    assert oracle.distance(np.array([0, 0, 0], np.float32), np.array([3, 4, 0], np.float32), 3) == 5.0
    assert oracle.distance(np.array([1, 2, 3], np.float32), np.array([1, 2, 3], np.float32), 3) == 0.0


def test_c1_full_size_hashes(oracle):
    g = golden_hashes()["C1"]
    p = oracle.uniform(g["n"], 3, 1.0, g["seed"])
    eps = eps_for(g["n"])
    assert "%08x" % np.float32(eps).view(np.uint32) == g["eps_bits"]
    e = oracle.bvh(p, 3)
    assert fnv1a64(e["leaf_object"]) == g["leaf_perm"]
    labels, core = oracle.dbscan(p, 3, eps, 2)
    assert fnv1a64(labels) == g["labels_hash"] and fnv1a64(core) == g["core_hash"]
    assert summarize(labels, core) == (g["clusters"], g["noise"], g["core"])


@pytest.mark.skipif(not Reference.available(), reason="oracle/_ref not built (no /root/reference here)")
def test_oracle_equals_reference_on_random_instances(oracle):
    R = Reference.get()
    rng = np.random.default_rng(99)
    for trial in range(60):
        n = int(rng.integers(1, 400))
        dim = int(rng.choice([2, 3]))
        width = int(rng.choice([32, 64]))
        pts = rng.random((n, dim), dtype=np.float32)
        if trial % 3 == 1:
            pts = np.round(pts * 4) / 4
        a, b = oracle.bvh(pts, dim, width), R.bvh(pts, dim, width)
        for k in BVH_KEYS:
            assert same_bits(a[k], b[k]), (trial, k)
        eps = float(rng.choice([0.05, 0.1, 0.2]))
        mp = int(rng.choice([2, 3, 5]))
        lab, core = oracle.dbscan(pts, dim, eps, mp)
        rl, rc = R.dbscan(pts, dim, eps, mp, "reference")
        assert np.array_equal(core, rc)
        assert oracle.check_equivalence(pts, dim, eps, (lab, core), (rl, rc)) is None


@pytest.mark.parametrize("name", list(_cases("seq_cases.npz").keys()))
def test_sequential_fixtures_pinned_by_oracle(oracle, name):
    # the sequential-mode fixtures (ExecMode::kSequential) against the
    # independent restatement: identical core flags, and clusters equivalent
    # to the oracle's under verify.hpp's contract
    c = _cases("seq_cases.npz")[name]
    dim, min_pts = (int(v) for v in c["meta"])
    eps = float(c["eps"])
    lab, core = oracle.dbscan(c["points"], dim, eps, min_pts)
    for key in ("fd", "db"):
        assert np.array_equal(c[key + "_core"], core), key
        assert oracle.check_equivalence(c["points"], dim, eps, (c[key + "_labels"], c[key + "_core"]),
                                        (lab, core)) is None, key
