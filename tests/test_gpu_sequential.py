"""GPU: ExecMode::kSequential (exec.hpp:12).  The reference's sequential
fdbscan / fdbscan_densebox assign every border point deterministically
(dbscan.hpp:123-137, 406-442); the GPU's sequential mode reproduces those
labels bit for bit (tests/golden/seq_cases.npz, made by
tests/golden/make_seq_golden.py from the unmodified reference)."""
import numpy as np
import pytest

from fixtures import _cases

pytestmark = pytest.mark.gpu


def seq_cases():
    return _cases("seq_cases.npz")


@pytest.mark.parametrize("name", list(seq_cases().keys()))
def test_fdbscan_sequential_matches_reference(sp, name):
    c = seq_cases()[name]
    dim, min_pts = (int(v) for v in c["meta"])
    p = sp.DbscanParams(float(c["eps"]), min_pts)
    for _ in range(2):  # deterministic: repeated runs agree bit for bit
        out = sp.fdbscan(c["points"], p, mode="sequential")
        assert np.array_equal(out.core_flags, c["fd_core"])
        assert np.array_equal(out.labels, c["fd_labels"])


@pytest.mark.parametrize("algorithm", ["cells", "mixed"])
@pytest.mark.parametrize("name", list(seq_cases().keys()))
def test_densebox_sequential_matches_reference(sp, name, algorithm):
    c = seq_cases()[name]
    dim, min_pts = (int(v) for v in c["meta"])
    p = sp.DbscanParams(float(c["eps"]), min_pts)
    out = sp.fdbscan_densebox(c["points"], p, algorithm=algorithm, mode="sequential")
    assert np.array_equal(out.core_flags, c["db_core"])
    assert np.array_equal(out.labels, c["db_labels"])


def test_sequential_device_arrays_and_fof(sp):
    import torch
    c = seq_cases()["mix3_m5"]
    p = sp.DbscanParams(float(c["eps"]), int(c["meta"][1]))
    out = sp.fdbscan(torch.from_numpy(c["points"]).cuda(), p, mode="sequential")
    assert np.array_equal(out.labels.cpu().numpy(), c["fd_labels"])
    # min_pts = 2 is deterministic in both modes
    a = sp.fdbscan(c["points"], sp.DbscanParams(float(c["eps"]), 2), mode="sequential")
    b = sp.friends_of_friends(c["points"], float(c["eps"]))
    assert np.array_equal(a.labels, b.labels) and np.array_equal(a.core_flags, b.core_flags)
    with pytest.raises(ValueError):
        sp.fdbscan(c["points"], p, mode="serial")
