"""GPU: Bvh<D>::build parity (bvh.hpp:243-261) — node arrays, numbering,
ropes and union boxes bit-identical to the reference fixtures and the oracle;
the reference's shape/KAT/fault tests (test_bvh.cpp) through the C ABI."""
import numpy as np
import pytest

from fixtures import BVH_KEYS, bvh_cases, golden_hashes, same_bits
from oracle_lib import fnv1a64

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("name", list(bvh_cases().keys()))
def test_node_arrays_match_reference_fixture(sp, name):
    case = bvh_cases()[name]
    dim, width, pts = (int(v) for v in case["meta"])
    objs = case["objects"]
    if not pts:
        objs = objs.reshape(len(objs), 2 * dim)
    b = sp.Bvh.build(objs if len(objs) else np.zeros((0, 2 * dim if not pts else dim), np.float32), width,
                     points=bool(pts))
    got = b.export()
    for k in BVH_KEYS:
        assert same_bits(got[k], case[k]), (name, k)
    assert b.validate()[0]


def test_random_trees_match_oracle(sp, oracle):
    rng = np.random.default_rng(5)
    for trial in range(120):
        n = int(rng.integers(1, 5000))
        dim = int(rng.choice([2, 3]))
        width = int(rng.choice([32, 64]))
        kind = trial % 4
        if kind == 0:
            objs, pts = rng.random((n, dim), dtype=np.float32), True
        elif kind == 1:
            objs, pts = (rng.integers(0, 5, (n, dim)) / 4).astype(np.float32), True
        elif kind == 2:
            lo = rng.random((n, dim), dtype=np.float32)
            objs, pts = np.concatenate([lo, lo + rng.random((n, dim), dtype=np.float32) * 0.1], 1), False
        else:
            objs, pts = (rng.standard_normal((n, dim)) * 10 ** rng.uniform(-6, 6)).astype(np.float32), True
        want = oracle.bvh(objs, dim, width, pts)
        got = sp.Bvh.build(objs, width, points=pts).export()
        for k in BVH_KEYS:
            assert same_bits(got[k], want[k]), (trial, n, dim, width, kind, k)


def test_golden_three_leaf_dump(sp):
    # test_bvh.cpp:193-205
    b = sp.Bvh.build(np.array([[0.1, 0.1], [0.9, 0.9], [0.5, 0.25]], np.float32))
    assert b.dump() == ("bvh n 3 width 64\n"
                        "I 0 left 1 rope -1 0.100000001 0.100000001 0.899999976 0.899999976\n"
                        "I 1 left 2 rope 4 0.100000001 0.100000001 0.5 0.25\n"
                        "L 0 object 0 rope 3 0.100000001 0.100000001 0.100000001 0.100000001\n"
                        "L 1 object 2 rope 4 0.5 0.25 0.5 0.25\n"
                        "L 2 object 1 rope -1 0.899999976 0.899999976 0.899999976 0.899999976\n")


def test_empty_single_two(sp):
    # test_bvh.cpp:39-67
    b = sp.Bvh.build(np.zeros((0, 3), np.float32))
    assert b.empty() and b.validate()[0]
    b = sp.Bvh.build(np.array([[0.5, 0.5, 0.5]], np.float32))
    e = b.export()
    assert b.size() == 1 and len(e["internal_left"]) == 0 and e["leaf_rope"].tolist() == [-1]
    b = sp.Bvh.build(np.array([[0.1, 0.1], [0.9, 0.9]], np.float32))
    e = b.export()
    assert e["internal_left"].tolist() == [1] and e["leaf_rope"].tolist() == [2, -1]


def test_identical_points_keep_original_order(sp):
    # test_bvh.cpp:159-171: stable tie-break
    objs = np.tile(np.array([[0.25, 0.5, 0.75]], np.float32), (257, 1))
    for width in (32, 64):
        b = sp.Bvh.build(objs, width)
        assert b.validate()[0]
        assert b.export()["leaf_object"].tolist() == list(range(257))


def test_non_finite_rejected(sp):
    # test_bvh.cpp:188-191
    for bad in (np.nan, np.inf, -np.inf):
        with pytest.raises(sp.InvalidArgument):
            sp.Bvh.build(np.array([[0, 0, bad], [1, 1, 1]], np.float32))


def test_fault_injection_detected_by_validate(sp):
    # test_bvh.cpp:126-147: a corrupted rope / shrunk volume must be caught
    rng = np.random.default_rng(3)
    b = sp.Bvh.build(rng.random((200, 3), dtype=np.float32))
    e = b.export()
    bad = dict(e)
    bad["leaf_rope"] = e["leaf_rope"].copy()
    bad["leaf_rope"][5] = e["leaf_rope"][7]
    assert not sp.validate_arrays(bad, 200, 3)[0]
    bad = dict(e)
    bad["internal_boxes"] = e["internal_boxes"].copy()
    bad["internal_boxes"][3, 0] += 0.01
    assert not sp.validate_arrays(bad, 200, 3)[0]


def test_morton_codes_match_oracle(sp, oracle):
    rng = np.random.default_rng(8)
    for dim in (2, 3):
        for width in (32, 64):
            p = rng.random((3000, dim), dtype=np.float32)
            assert np.array_equal(sp.morton_codes(p, width), oracle.morton(p, dim, width))
    # bin KATs (test_morton.cpp:12-22): scene corners and half-way
    p = np.array([[0, 0, 0], [1, 1, 1], [0.5, 0.5, 0.5]], np.float32)
    c = sp.morton_codes(p, 32)
    assert c[0] == 0 and c[1] == (1 << 30) - 1


def test_sort_queries_matches_leaf_order(sp, oracle):
    rng = np.random.default_rng(9)
    p = rng.random((50000, 3), dtype=np.float32)
    order = sp.sort_queries(p)
    assert np.array_equal(order, oracle.bvh(p, 3)["leaf_object"])


def test_c1_leaf_perm_and_node_arrays(sp, oracle):
    g = golden_hashes()["C1"]
    p = oracle.uniform(g["n"], 3, 1.0, g["seed"])
    e = sp.Bvh.build(p).export()
    assert fnv1a64(e["leaf_object"]) == g["leaf_perm"]
    blob = []
    m = len(e["internal_left"])
    ints = np.empty((m, 8), np.float32)
    ints[:, 0] = e["internal_left"].view(np.float32)
    ints[:, 1] = e["internal_rope"].view(np.float32)
    ints[:, 2:] = e["internal_boxes"]
    leaves = np.empty((g["n"], 8), np.float32)
    leaves[:, 0] = e["leaf_object"].view(np.float32)
    leaves[:, 1] = e["leaf_rope"].view(np.float32)
    leaves[:, 2:] = e["leaf_boxes"]
    assert fnv1a64(np.concatenate([ints.reshape(-1), leaves.reshape(-1)])) == g["node_arrays"]


def test_unaligned_device_points_take_the_scalar_path(sp):
    # the 3-D point kernels load four points as three float4 when the array is
    # 16-byte aligned; a view starting one point in is not, and must agree
    import torch
    rng = np.random.default_rng(41)
    base = torch.from_numpy(rng.random((40001, 3), dtype=np.float32)).cuda()
    view = base[1:]  # 12-byte offset
    dense = view.clone()  # aligned copy of the same points
    a = sp.Bvh.build(view).export()
    b = sp.Bvh.build(dense).export()
    for k in a:
        assert np.array_equal(np.asarray(a[k]).view(np.uint8), np.asarray(b[k]).view(np.uint8)), k
    eps = 0.01
    fa = sp.friends_of_friends(view, eps)
    fb = sp.friends_of_friends(dense, eps)
    assert torch.equal(fa.labels, fb.labels) and torch.equal(fa.core_flags, fb.core_flags)


@pytest.mark.parametrize("case", ["top40", "overflow", "top32_runs"])
def test_top_bits_sort_paths_match_oracle(sp, oracle, case):
    # Bvh::build sorts by the top 32 or 40 code bits and orders the runs of
    # equal top bits afterwards; a sample routes clumps to the wider sort, and
    # runs over 512 fall back to the full 63-bit sort.  Every path must give
    # the reference's tree bit for bit.
    rng = np.random.default_rng(4040)
    if case == "top40":  # dense enough for long top-32 runs, sparse at 40 bits
        pts = np.concatenate([rng.random((1 << 20, 3), dtype=np.float32),
                              (0.3 + rng.random((1 << 16, 3)) * 0.006).astype(np.float32)])
    elif case == "overflow":  # 1000 identical points below the sampling size: fix-up overflow
        pts = np.concatenate([rng.random((5000, 3), dtype=np.float32), np.full((1000, 3), 0.25, np.float32)])
    else:  # runs of tens of equal top-32 keys, handled in place
        pts = np.concatenate([rng.random((20000, 3), dtype=np.float32),
                              (0.6 + rng.random((3000, 3)) * 0.003).astype(np.float32)])
    ctx = sp.Context(0)
    tree = sp.Bvh.build(pts, ctx=ctx)
    path = (ctx.counter("sort_top_bits"), ctx.counter("sort_fallback"))
    got = tree.export()
    assert path == {"top40": (40, 0), "overflow": (32, 1), "top32_runs": (32, 0)}[case], path
    want = oracle.bvh(pts, 3)
    for key in BVH_KEYS:
        assert same_bits(got[key], want[key]), (case, key)
