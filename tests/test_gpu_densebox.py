"""GPU: fdbscan_densebox parity (dbscan.hpp:298-449, dense_grid.hpp:71-103):
exact core flags, FoF labels, DenseBox grid statistics (dense cells, dense
points) equal to the reference, and equivalent clusters for min_pts > 2; the C3
configuration at full size.  The merge's distance-check counter is a
diagnostic of the implementation (dbscan.hpp:38-41): the object-level merge
stops at the first close member pair, so it is only bounded, not equal."""
import numpy as np
import pytest

from fixtures import dbscan_cases, golden_hashes, summarize
from oracle_lib import eps_for, fnv1a64

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("name", list(dbscan_cases().keys()))
def test_densebox_matches_reference_fixture(sp, oracle, name):
    c = dbscan_cases()[name]
    dim, min_pts = (int(v) for v in c["meta"])
    eps = float(c["eps"])
    out = sp.fdbscan_densebox(c["points"], sp.DbscanParams(eps, min_pts))
    assert np.array_equal(out.core_flags, c["db_core"])
    st = c["db_stats"]
    assert (out.stats.num_dense_cells, out.stats.num_dense_points) == tuple(st.tolist()[1:])
    if min_pts == 2:
        assert np.array_equal(out.labels, c["db_labels"])
    else:
        assert oracle.check_equivalence(c["points"], dim, eps, (out.labels, out.core_flags),
                                        (c["db_labels"], c["db_core"])) is None


def test_densebox_random_instances(sp, oracle):
    rng = np.random.default_rng(31)
    for trial in range(24):
        dim = int(rng.choice([2, 3]))
        n = int(rng.integers(1, 30000))
        k = int(rng.integers(1, 12))
        centres = rng.random((k, dim))
        pts = np.clip(centres[rng.integers(0, k, n)] + rng.standard_normal((n, dim)) * 0.01, 0, 1)
        pts = np.concatenate([pts, rng.random((n // 5, dim))]).astype(np.float32)
        eps = float(rng.choice([0.002, 0.005, 0.01]))
        mp = int(rng.choice([2, 3, 5, 8]))
        out = sp.fdbscan_densebox(pts, sp.DbscanParams(eps, mp))
        lab, core, st = oracle.dbscan(pts, dim, eps, mp, with_stats=True)
        assert np.array_equal(out.core_flags, core), trial
        assert (out.stats.num_dense_cells, out.stats.num_dense_points) == tuple(st.tolist()[1:]), trial
        if mp == 2:
            assert np.array_equal(out.labels, lab), trial
        else:
            assert oracle.check_equivalence(pts, dim, eps, (out.labels, out.core_flags), (lab, core)) is None, trial


def test_single_dense_cell_needs_no_distance_checks(sp):
    # test_dbscan.cpp:220-232
    p = np.full((50, 3), 0.5, np.float32)
    out = sp.fdbscan_densebox(p, sp.DbscanParams(0.1, 5))
    assert out.stats.num_dense_cells == 1 and out.stats.distance_checks == 0
    assert out.labels.tolist() == [0] * 50


def test_no_dense_cells_equals_fdbscan(sp):
    # test_dbscan.cpp:234-243
    rng = np.random.default_rng(2)
    p = rng.random((3000, 3), dtype=np.float32)
    a = sp.fdbscan_densebox(p, sp.DbscanParams(0.02, 50))
    b = sp.fdbscan(p, sp.DbscanParams(0.02, 50))
    assert a.stats.num_dense_cells == 0
    assert np.array_equal(a.core_flags, b.core_flags)


def test_densebox_tiny_eps(sp, oracle):
    # test_dbscan.cpp:245-259: eps far below coordinate resolution
    rng = np.random.default_rng(3)
    p = rng.random((400, 3), dtype=np.float32)
    p[50:60] = p[0]
    out = sp.fdbscan_densebox(p, sp.DbscanParams(1e-30, 3))
    lab, core = oracle.dbscan(p, 3, 1e-30, 3)
    assert np.array_equal(out.core_flags, core)
    assert oracle.check_equivalence(p, 3, 1e-30, (out.labels, out.core_flags), (lab, core)) is None


def test_c3_full_size(sp, oracle):
    g = golden_hashes()["C3"]
    n = g["n"]
    p = oracle.field(n)
    eps = eps_for(n)
    assert "%08x" % np.float32(eps).view(np.uint32) == g["eps_bits"]
    out = sp.fdbscan_densebox(p, sp.DbscanParams(eps, g["min_pts"]))
    assert out.stats.num_dense_cells == g["dense_cells"]
    assert out.stats.num_dense_points == g["dense_points"]
    assert 0 < out.stats.distance_checks < g["distance_checks"]
    assert summarize(out.labels, out.core_flags) == (g["clusters"], g["noise"], g["core"])
    assert fnv1a64(out.core_flags) == g["core_hash"]


def test_device_check_equivalence_matches_oracle_checker(sp, oracle):
    # verify.hpp:21-61 on the device, incl. the fault-injection cases of
    # test_dbscan.cpp:340-404
    c = dbscan_cases()["clustered3_m4"]
    pts, eps = c["points"], float(c["eps"])
    want = sp.DbscanOutput(c["labels"], c["core"])
    got = sp.fdbscan(pts, sp.DbscanParams(eps, 4))
    assert sp.check_equivalence(pts, eps, got, want) is None
    core = c["core"].copy()
    core[int(np.argmax(core))] ^= 1
    assert "core flag" in sp.check_equivalence(pts, eps, sp.DbscanOutput(c["labels"], core), want)
    lab = c["labels"].copy()
    i = int(np.argmax(lab == -1))
    lab[i] = lab[int(np.argmax(c["core"]))]
    assert sp.check_equivalence(pts, eps, sp.DbscanOutput(lab, c["core"]), want) is not None
    # merge two reference clusters into one
    lab = c["labels"].copy()
    cl = np.unique(lab[c["core"] == 1])
    lab[lab == cl[1]] = cl[0]
    msg = sp.check_equivalence(pts, eps, sp.DbscanOutput(lab, c["core"]), want)
    assert msg is not None and "merged" in msg
    # a border point relabelled to a far cluster
    lab = c["labels"].copy()
    border = np.where((c["core"] == 0) & (lab >= 0))[0]
    if len(border):
        far = [x for x in cl if x != lab[border[0]]][-1]
        lab[border[0]] = far
        msg = sp.check_equivalence(pts, eps, sp.DbscanOutput(lab, c["core"]), want)
        assert msg is not None and "border" in msg


def test_c3_densebox_equivalent_to_fdbscan_at_full_size(sp):
    import torch
    n = 1 << 26
    p = sp.generate_field(n, seed=7)
    eps = eps_for(n)
    a = sp.fdbscan_densebox(p, sp.DbscanParams(eps, 5))
    b = sp.fdbscan(p, sp.DbscanParams(eps, 5))
    assert bool(torch.equal(a.core_flags, b.core_flags))
    assert sp.check_equivalence(p, eps, a, b) is None
