"""GPU: range_query counts (traversal.hpp:67-87), early termination
(dbscan.hpp:146-170), query_crs (traversal.hpp:235-266), pair_traversal
(traversal.hpp:162-184) and nearest_query (traversal.hpp:93-156) parity."""
import numpy as np
import pytest

from fixtures import query_cases

pytestmark = pytest.mark.gpu


def spheres_of(c, r):
    return np.concatenate([c, np.full((len(c), 1), r, np.float32)], 1).astype(np.float32)


def test_range_counts_match_reference_fixture(sp):
    q = query_cases()
    b = sp.Bvh.build(q["rc/points"])
    r = float(q["rc/radius"])
    assert np.array_equal(sp.range_count(b, q["rc/centres"], radius=r), q["rc/counts"])
    assert np.array_equal(sp.range_count(b, spheres_of(q["rc/centres"], r)), q["rc/counts"])
    assert np.array_equal(sp.range_count(b, q["rc/centres"], radius=r, cap=4), q["rc/capped4"])


def test_range_counts_match_oracle_random(sp, oracle):
    rng = np.random.default_rng(12)
    for trial in range(30):
        dim = int(rng.choice([2, 3]))
        n = int(rng.integers(1, 20000))
        pts = rng.random((n, dim), dtype=np.float32)
        if trial % 3 == 0:
            pts = np.round(pts * 16) / 16
        nq = int(rng.integers(1, 5000))
        c = rng.random((nq, dim), dtype=np.float32)
        radii = rng.random(nq).astype(np.float32) * 0.1
        sph = np.concatenate([c, radii[:, None]], 1)
        b = sp.Bvh.build(pts)
        assert np.array_equal(sp.range_count(b, sph), oracle.range_count(pts, dim, sph)), trial
        cap = int(rng.integers(1, 6))
        assert np.array_equal(sp.range_count(b, sph, cap=cap), oracle.range_count(pts, dim, sph, cap=cap)), trial
        lo = rng.random((nq, dim), dtype=np.float32)
        boxes = np.concatenate([lo, lo + rng.random((nq, dim), dtype=np.float32) * 0.05], 1)
        assert np.array_equal(sp.range_count(b, boxes, kind="box"),
                              oracle.range_count(pts, dim, boxes, pred_is_box=True)), trial


def test_range_over_box_objects(sp, oracle):
    rng = np.random.default_rng(13)
    lo = rng.random((3000, 3), dtype=np.float32)
    objs = np.concatenate([lo, lo + rng.random((3000, 3), dtype=np.float32) * 0.02], 1)
    b = sp.Bvh.build(objs, points=False)
    sph = spheres_of(rng.random((2000, 3), dtype=np.float32), 0.03)
    assert np.array_equal(sp.range_count(b, sph), oracle.range_count(objs, 3, sph, is_points=False))


def test_boundary_exactness_at_eps(sp, oracle):
    # points placed exactly at / one ulp around the radius: the float(sqrt(double))
    # rule must be reproduced bit-for-bit (test_geometry.cpp:135-140)
    rng = np.random.default_rng(14)
    base = rng.random((4000, 3)).astype(np.float32)
    r = np.float32(0.01)
    d = rng.standard_normal((4000, 3))
    d /= np.linalg.norm(d, axis=1, keepdims=True)
    other = (base + d * float(r)).astype(np.float32)
    other = np.concatenate([other, np.nextafter(other, np.float32(2)), np.nextafter(other, np.float32(-1))])
    b = sp.Bvh.build(other)
    assert np.array_equal(sp.range_count(b, base, radius=float(r)),
                          oracle.range_count(other, 3, spheres_of(base, r)))
    for eps in (1e-30, 1e-38, 1e-45, 0.0):
        assert np.array_equal(sp.range_count(b, base, radius=eps), oracle.range_count(other, 3, spheres_of(base, eps)))


def test_empty_tree_and_covering_sphere(sp):
    b = sp.Bvh.build(np.zeros((0, 3), np.float32))
    assert sp.range_count(b, np.zeros((5, 4), np.float32)).tolist() == [0] * 5
    rng = np.random.default_rng(1)
    b = sp.Bvh.build(rng.random((1000, 3), dtype=np.float32))
    assert sp.range_count(b, np.array([[0.5, 0.5, 0.5, 10.0]], np.float32)).tolist() == [1000]


def test_crs_matches_oracle(sp, oracle):
    rng = np.random.default_rng(15)
    pts = rng.random((8000, 3), dtype=np.float32)
    sph = spheres_of(rng.random((3000, 3), dtype=np.float32), 0.04)
    b = sp.Bvh.build(pts)
    off, val = sp.query_crs(b, sph)
    woff, wval = oracle.range_crs(pts, 3, sph)
    assert np.array_equal(off, woff) and np.array_equal(val, wval)
    with pytest.raises(sp.CapacityError):
        sp.query_crs(b, sph, max_total_matches=int(woff[-1]) - 1)


def test_pair_traversal_exactly_once(sp, oracle):
    rng = np.random.default_rng(16)
    for dim in (2, 3):
        pts = rng.random((3000, dim), dtype=np.float32)
        eps = 0.03
        b = sp.Bvh.build(pts)
        pairs = sp.pair_traversal(b, eps)
        got = set(map(tuple, np.sort(pairs, axis=1).tolist()))
        assert len(got) == len(pairs)
        off, val = oracle.range_crs(pts, dim, spheres_of(pts, eps))
        want = set()
        for i in range(len(pts)):
            for j in val[off[i]:off[i + 1]]:
                if i < j:
                    want.add((i, int(j)))
        assert got == want
        # first element belongs to the earlier leaf
        rank = np.empty(len(pts), np.int64)
        rank[b.export()["leaf_object"]] = np.arange(len(pts))
        assert (rank[pairs[:, 0]] < rank[pairs[:, 1]]).all()


@pytest.mark.parametrize("k", [1, 5, 16, 32])
def test_knn_matches_reference_fixture(sp, k):
    q = query_cases()
    b = sp.Bvh.build(q["knn/points"])
    assert np.array_equal(sp.nearest_query(b, q["knn/origins"], k), q["knn/idx%d" % k])


def test_knn_random_and_large_k(sp, oracle):
    rng = np.random.default_rng(17)
    for trial in range(12):
        dim = int(rng.choice([2, 3]))
        n = int(rng.integers(1, 3000))
        pts = rng.random((n, dim), dtype=np.float32)
        if trial % 2:
            pts = np.round(pts * 8) / 8
        org = rng.random((700, dim), dtype=np.float32)
        for k in (1, 7, 16, 40, 100):
            idx, dist = sp.nearest_query(sp.Bvh.build(pts), org, k, with_distances=True)
            widx, wdist = oracle.knn(pts, dim, org, k)
            assert np.array_equal(idx, widx), (trial, k)
            assert same_float(dist, wdist)


def same_float(a, b):
    return np.array_equal(np.asarray(a).view(np.uint32), np.asarray(b).view(np.uint32))


def test_knn_k_at_least_n_and_degenerate(sp, oracle):
    # test_traversal.cpp:144-168: k >= n returns everything; k <= 0 nothing
    pts = np.array([[0, 0, 0], [1, 0, 0], [0, 2, 0], [0, 0, 3]], np.float32)
    b = sp.Bvh.build(pts)
    idx = sp.nearest_query(b, np.array([[0, 0, 0]], np.float32), 10)
    assert idx[0, :4].tolist() == [0, 1, 2, 3] and idx[0, 4:].tolist() == [-1] * 6
    assert sp.nearest_query(b, np.array([[0, 0, 0]], np.float32), 0).shape == (1, 0)
    idx = sp.nearest_query(b, np.array([[0, 0, 0]], np.float32), 1)
    assert idx.tolist() == [[0]]


@pytest.mark.parametrize("scale", [1e-30, 1e-18, 1e15, 1e30])
def test_knn_extreme_scales(sp, oracle, scale):
    # the fp32 pruning filter switches off where squared gaps leave the normal
    # range; results must stay exact at every scale
    rng = np.random.default_rng(23)
    pts = (rng.random((2000, 3)) * scale).astype(np.float32)
    pts[100:140] = pts[7]  # duplicates: worst distance 0
    org = np.concatenate([(rng.random((300, 3)) * scale).astype(np.float32), pts[:50]])
    for k in (1, 16, 50):
        idx, dist = sp.nearest_query(sp.Bvh.build(pts), org, k, with_distances=True)
        widx, wdist = oracle.knn(pts, 3, org, k)
        assert np.array_equal(idx, widx), k
        assert same_float(dist, wdist)


@pytest.mark.parametrize("n", [1, 2, 3, 5])
def test_knn_tiny_trees(sp, oracle, n):
    # root-is-a-leaf (n = 1) and trees whose children are all leaves; with
    # duplicated points every distance ties and the index decides
    rng = np.random.default_rng(100 + n)
    for dup in (False, True):
        pts = rng.random((n, 3), dtype=np.float32)
        if dup:
            pts[:] = pts[0]
        org = np.concatenate([rng.random((64, 3), dtype=np.float32), pts])
        b = sp.Bvh.build(pts)
        for k in (1, 2, 16, 17, 40):
            idx, dist = sp.nearest_query(b, org, k, with_distances=True)
            widx, wdist = oracle.knn(pts, 3, org, k)
            assert np.array_equal(idx, widx), (n, dup, k)
            assert same_float(dist, wdist)


def test_query_out_buffers(sp):
    # caller-supplied (pinned host or device) result buffers give the same
    # results as the allocated ones; wrong shape / dtype / memory space raise
    import torch
    rng = np.random.default_rng(31)
    pts = rng.random((5000, 3), dtype=np.float32)
    b = sp.Bvh.build(pts)
    want_c = sp.range_count(b, pts, radius=0.05)
    want_i, want_d = sp.nearest_query(b, pts, 8, with_distances=True)
    hc = torch.empty(5000, dtype=torch.int32, pin_memory=True)
    assert sp.range_count(b, pts, radius=0.05, out=hc) is hc
    assert np.array_equal(hc.numpy(), want_c)
    hi = torch.empty((5000, 8), dtype=torch.int32, pin_memory=True)
    hd = torch.empty((5000, 8), dtype=torch.float32, pin_memory=True)
    sp.nearest_query(b, pts, 8, with_distances=True, out=(hi, hd))
    assert np.array_equal(hi.numpy(), want_i) and np.array_equal(hd.numpy(), want_d)
    dpts = torch.from_numpy(pts).cuda()
    db = sp.Bvh.build(dpts)
    di = torch.empty((5000, 8), dtype=torch.int32, device="cuda")
    sp.nearest_query(db, dpts, 8, out=di)
    assert np.array_equal(di.cpu().numpy(), want_i)
    with pytest.raises(ValueError):
        sp.nearest_query(b, pts, 8, out=di)  # device buffer for host inputs
    with pytest.raises(ValueError):
        sp.range_count(b, pts, radius=0.05, out=np.empty(4999, np.int32))


@pytest.mark.parametrize("nq", [1, 31, 32, 33, 148 * 32 - 1, 148 * 32 + 5, 148 * 512 + 77])
def test_range_counts_every_query_once(sp, oracle, nq):
    # the SM-affine schedule (per-SM slices, 32-query chunks, stealing) must
    # write every count exactly once for totals around its chunk and slice sizes
    import torch
    rng = np.random.default_rng(nq)
    pts = rng.random((3000, 3), dtype=np.float32)
    qs = rng.random((nq, 3), dtype=np.float32)
    b = sp.Bvh.build(pts)
    want = oracle.range_count(pts, 3, spheres_of(qs, np.float32(0.06)))
    assert np.array_equal(sp.range_count(b, qs, radius=0.06), want)
    out = torch.full((nq,), -7, dtype=torch.int32, device="cuda")
    sp.range_count(sp.Bvh.build(torch.from_numpy(pts).cuda()), torch.from_numpy(qs).cuda(), radius=0.06, out=out)
    assert np.array_equal(out.cpu().numpy(), want)
