"""GPU: fdbscan / friends_of_friends parity (dbscan.hpp:229-292): FoF labels
bit-identical to the reference; minPts > 2 core flags identical and clusters
equivalent under the reference's check_equivalence contract (verify.hpp)."""
import numpy as np
import pytest

from fixtures import dbscan_cases, golden_hashes, summarize
from oracle_lib import eps_for, fnv1a64

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("name", list(dbscan_cases().keys()))
def test_fdbscan_matches_reference_fixture(sp, oracle, name):
    c = dbscan_cases()[name]
    dim, min_pts = (int(v) for v in c["meta"])
    eps = float(c["eps"])
    out = sp.fdbscan(c["points"], sp.DbscanParams(eps, min_pts))
    assert np.array_equal(out.core_flags, c["core"])
    if min_pts == 2:
        assert np.array_equal(out.labels, c["labels"])
        fof = sp.friends_of_friends(c["points"], eps)
        assert np.array_equal(fof.labels, c["labels"])
    else:
        assert oracle.check_equivalence(c["points"], dim, eps, (out.labels, out.core_flags),
                                        (c["labels"], c["core"])) is None


def test_fof_random_instances_match_oracle(sp, oracle):
    rng = np.random.default_rng(21)
    for trial in range(40):
        dim = int(rng.choice([2, 3]))
        n = int(rng.integers(1, 30000))
        pts = rng.random((n, dim), dtype=np.float32)
        if trial % 4 == 1:
            pts = np.round(pts * 32) / 32
        eps = float(rng.choice([0.002, 0.01, 0.03]))
        width = int(rng.choice([32, 64]))
        out = sp.friends_of_friends(pts, eps, width=width)
        lab, core = oracle.dbscan(pts, dim, eps, 2)
        assert np.array_equal(out.labels, lab) and np.array_equal(out.core_flags, core), trial


def test_minpts_random_instances_equivalent(sp, oracle):
    rng = np.random.default_rng(22)
    for trial in range(25):
        dim = int(rng.choice([2, 3]))
        n = int(rng.integers(1, 20000))
        centres = rng.random((8, dim))
        pts = np.clip(centres[rng.integers(0, 8, n)] + rng.standard_normal((n, dim)) * 0.02, 0, 1).astype(np.float32)
        eps = float(rng.choice([0.005, 0.01]))
        mp = int(rng.choice([3, 4, 5, 10]))
        out = sp.fdbscan(pts, sp.DbscanParams(eps, mp))
        lab, core = oracle.dbscan(pts, dim, eps, mp)
        assert np.array_equal(out.core_flags, core), trial
        assert oracle.check_equivalence(pts, dim, eps, (out.labels, out.core_flags), (lab, core)) is None, trial


def test_kats(sp):
    # test_dbscan.cpp:55-81: lone point is noise; a close pair is one cluster;
    # blob A..D + border E (through D) + noise F with min_pts 4
    out = sp.fdbscan(np.array([[0.5, 0.5]], np.float32), sp.DbscanParams(0.1, 2))
    assert out.labels.tolist() == [-1] and out.core_flags.tolist() == [0]
    out = sp.fdbscan(np.array([[0.5, 0.5], [0.55, 0.5]], np.float32), sp.DbscanParams(0.1, 2))
    assert out.labels.tolist() == [0, 0] and out.core_flags.tolist() == [1, 1]
    blob = np.array([[0.50, 0.50], [0.52, 0.50], [0.50, 0.52], [0.59, 0.50], [0.68, 0.50], [0.95, 0.95]],
                    np.float32)
    for algo in (sp.fdbscan, sp.fdbscan_densebox):
        out = algo(blob, sp.DbscanParams(0.1, 4))
        assert out.core_flags.tolist() == [1, 1, 1, 1, 0, 0]
        assert out.labels.tolist() == [0, 0, 0, 0, 0, -1]
    # test_dbscan.cpp:284-293: chains connect, singletons are noise
    chain = np.array([[i * 0.09, 0.0] for i in range(10)] + [[5.0, 5.0]], np.float32)
    out = sp.friends_of_friends(chain, 0.1)
    assert out.labels.tolist() == [0] * 10 + [-1]


def test_parameter_validation(sp):
    # test_dbscan.cpp:45-53
    p = np.zeros((3, 3), np.float32)
    for eps, mp in ((0.0, 2), (-1.0, 2), (float("inf"), 2), (float("nan"), 2), (0.1, 1)):
        with pytest.raises(sp.InvalidArgument):
            sp.fdbscan(p, sp.DbscanParams(eps, mp))
    with pytest.raises(sp.InvalidArgument):
        sp.friends_of_friends(np.array([[0, 0, np.nan]], np.float32), 0.1)


def test_empty_and_tiny_eps(sp, oracle):
    out = sp.fdbscan(np.zeros((0, 3), np.float32), sp.DbscanParams(0.1, 3))
    assert len(out.labels) == 0
    rng = np.random.default_rng(4)
    p = rng.random((500, 3), dtype=np.float32)
    p[100:110] = p[0]
    out = sp.fdbscan(p, sp.DbscanParams(1e-30, 3))
    lab, core = oracle.dbscan(p, 3, 1e-30, 3)
    assert np.array_equal(out.core_flags, core)
    assert oracle.check_equivalence(p, 3, 1e-30, (out.labels, out.core_flags), (lab, core)) is None


def test_permutation_invariance(sp):
    # test_dbscan.cpp:420-443: FoF labels map consistently under input permutation
    rng = np.random.default_rng(6)
    p = rng.random((20000, 3), dtype=np.float32)
    perm = rng.permutation(len(p))
    a = sp.friends_of_friends(p, 0.01).labels
    b = sp.friends_of_friends(p[perm], 0.01).labels
    inv = np.empty_like(perm)
    inv[perm] = np.arange(len(p))
    # same partition and noise set
    assert np.array_equal(a[perm] == -1, b == -1)
    ca = a[perm][b != -1]
    cb = b[b != -1]
    pairs = set(zip(ca.tolist(), cb.tolist()))
    assert len(pairs) == len(set(ca.tolist())) == len(set(cb.tolist()))


def test_repeatable_and_device_arrays(sp):
    import torch
    rng = np.random.default_rng(7)
    p = rng.random((100000, 3), dtype=np.float32)
    a = sp.friends_of_friends(p, 0.004)
    d = torch.from_numpy(p).cuda()
    b = sp.friends_of_friends(d, 0.004)
    assert np.array_equal(a.labels, b.labels.cpu().numpy())
    assert np.array_equal(a.core_flags, b.core_flags.cpu().numpy())


def test_c1_labels_hash(sp, oracle):
    g = golden_hashes()["C1"]
    p = oracle.uniform(g["n"], 3, 1.0, g["seed"])
    out = sp.friends_of_friends(p, eps_for(g["n"]))
    assert fnv1a64(out.labels) == g["labels_hash"]
    assert fnv1a64(out.core_flags) == g["core_hash"]
    assert summarize(out.labels, out.core_flags) == (g["clusters"], g["noise"], g["core"])


def test_adjacency_graph_dbscan_equals_fof_and_overflows(sp, oracle):
    # test_dbscan.cpp:306-338: legacy == FoF; the CRS cap raises CapacityError
    rng = np.random.default_rng(8)
    for dim in (2, 3):
        p = rng.random((20000, dim), dtype=np.float32)
        a = sp.adjacency_graph_dbscan(p, 0.01)
        b = sp.friends_of_friends(p, 0.01)
        assert np.array_equal(a.labels, b.labels) and np.array_equal(a.core_flags, b.core_flags)
    with pytest.raises(sp.CapacityError):
        sp.adjacency_graph_dbscan(p, 0.01, max_adjacency=100)
    c = dbscan_cases()["uniform3_fof"]
    out = sp.adjacency_graph_dbscan(c["points"], float(c["eps"]))
    assert np.array_equal(out.labels, c["labels"])


def test_context_on_torch_default_stream_is_ordered(sp, oracle):
    # stream handle 0 (torch's default stream) must mean the legacy default
    # stream, not "a context-owned stream": the FoF has to see points that
    # torch produces on that stream right before the call
    import torch
    pts = oracle.field(1 << 16)
    eps = eps_for(1 << 16)
    base = torch.from_numpy(pts).cuda()
    torch.cuda.synchronize()
    ctx = sp.Context(0, stream=torch.cuda.current_stream().cuda_stream)
    for _ in range(3):
        dst = torch.zeros_like(base)
        torch.cuda._sleep(50_000_000)  # ~25 ms of spinning on the default stream
        dst.copy_(base)
        out = sp.friends_of_friends(dst, eps, ctx=ctx)
        lab, core = oracle.dbscan(pts, 3, eps, 2)
        assert np.array_equal(out.labels.cpu().numpy(), lab)


def test_fof_ids_labels_are_min_id_per_cluster(sp, oracle):
    # sp_fof_ids: the same clusters, labelled by the smallest caller id
    import torch
    pts = oracle.field(1 << 16)
    eps = eps_for(1 << 16)
    lab, core = oracle.dbscan(pts, 3, eps, 2)
    rng = np.random.default_rng(5)
    ids = (rng.permutation(len(pts)) * 3 + 7).astype(np.int32)
    want = np.full(len(pts), -1, np.int64)
    members = lab >= 0
    mins = {}
    for i in np.nonzero(members)[0]:
        mins[lab[i]] = min(mins.get(lab[i], 1 << 40), ids[i])
    want[members] = [mins[l] for l in lab[members]]
    for mem in ("device", "host"):
        p = torch.from_numpy(pts).cuda() if mem == "device" else pts
        i = torch.from_numpy(ids).cuda() if mem == "device" else ids
        out = sp.friends_of_friends_ids(p, eps, i)
        got = out.labels.cpu().numpy() if mem == "device" else out.labels
        gc = out.core_flags.cpu().numpy() if mem == "device" else out.core_flags
        assert np.array_equal(got, want.astype(np.int32)), mem
        assert np.array_equal(gc, core), mem


@pytest.mark.parametrize("dim", [2, 3])
def test_fof_cells_boundary_and_degenerate_inputs(sp, oracle, dim):
    # The cell pipeline's shortcuts (a cell is one set; only cells <= 2 apart
    # can touch) must reproduce the exact predicate at the boundary: pairs at
    # float distance exactly eps and one ulp beyond, axis-aligned and
    # diagonal, on a lattice of spacing eps; identical points; negative and
    # large-magnitude coordinates.
    rng = np.random.default_rng(11 + dim)
    eps = np.float32(0.01)
    cases = []
    g = np.arange(12, dtype=np.float32) * eps  # spacing exactly eps
    grid = np.stack(np.meshgrid(*([g] * dim), indexing="ij"), -1).reshape(-1, dim)
    cases.append(grid)
    cases.append(grid * np.float32(1.0000001))  # just beyond eps
    diag = np.float32(eps / np.sqrt(dim))
    line = (np.arange(200, dtype=np.float32)[:, None] * diag) * np.ones((1, dim), np.float32)
    cases.append(line)
    same = np.tile(rng.random((1, dim), dtype=np.float32), (500, 1))
    cases.append(np.concatenate([same, rng.random((300, dim), dtype=np.float32)]))
    cases.append((rng.random((5000, dim), dtype=np.float32) - 0.5) * 0.3 - 7.0)  # negative coordinates
    cases.append(rng.random((5000, dim), dtype=np.float32) * 0.2 + 1000.0)  # large magnitude, coarse ulps
    for t, pts in enumerate(cases):
        pts = np.ascontiguousarray(pts, np.float32)
        out = sp.friends_of_friends(pts, float(eps))
        lab, core = oracle.dbscan(pts, dim, float(eps), 2)
        assert np.array_equal(out.labels, lab), (dim, t)
        assert np.array_equal(out.core_flags, core), (dim, t)
