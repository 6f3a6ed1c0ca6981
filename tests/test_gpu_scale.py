"""GPU, full BASELINE sizes: parity against the SURVEY §8(c) hashes of the
unmodified reference at C2 (2^24 points + 2^24 range counts), C4 (2^24 x 2^24
kNN, k = 16) and the C5 proxies (FoF on the 2^24 / 2^26 clustered field),
plus size-independent properties at the bench size."""
import numpy as np
import pytest

from fixtures import golden_hashes, summarize
from oracle_lib import eps_for, fnv1a64

pytestmark = pytest.mark.gpu


def test_c2_leaf_perm_and_range_counts(sp, oracle):
    g = golden_hashes()["C2"]
    n = g["n"]
    p = oracle.uniform(n, 3, 1.0, g["seed"])
    r = np.float32(np.cbrt(30.0 / (n * 4.18879020478639)))
    assert "%08x" % r.view(np.uint32) == g["radius_bits"]
    b = sp.Bvh.build(p)
    e = b.export()
    assert fnv1a64(e["leaf_object"]) == g["leaf_perm"]
    counts = sp.range_count(b, p, radius=float(r))
    assert int(counts.sum()) == g["total_matches"]
    assert fnv1a64(counts) == g["counts_hash"]


def test_c4_knn(sp, oracle):
    g = golden_hashes()["C4"]
    n = g["n"]
    p = oracle.uniform(n, 3, 1.0, g["seeds"][0])
    q = oracle.uniform(n, 3, 1.0, g["seeds"][1])
    idx, dist = sp.nearest_query(sp.Bvh.build(p), q, 16, with_distances=True)
    assert fnv1a64(idx) == g["knn_idx"]
    assert abs(float(dist[:, 15].astype(np.float64).mean()) - g["mean_16th_dist"]) < 1e-9


@pytest.mark.parametrize("key", ["C5_2^24", "C5_2^26"])
def test_c5_proxy_fof_labels(sp, oracle, key):
    g = golden_hashes()[key]
    n = g["n"]
    p = oracle.field(n)
    out = sp.friends_of_friends(p, eps_for(n))
    assert summarize(out.labels, out.core_flags) == (g["clusters"], g["noise"], g["core"])
    assert fnv1a64(out.core_flags) == g["core_hash"]
    assert fnv1a64(out.labels) == g["labels_hash"]


def test_bench_field_properties(sp):
    # 2^27 points of the bench field: labels are canonical (label == min index
    # of its cluster, a core point's label is a member <= itself), noise
    # exactly the non-core points, and the run is repeatable.
    import torch
    n = 1 << 27
    p = sp.generate_field(n, seed=2409)
    eps = eps_for(n)
    a = sp.friends_of_friends(p, eps)
    lab = a.labels
    core = a.core_flags.bool()
    idx = torch.arange(n, device=lab.device, dtype=torch.int32)
    assert bool(((lab == -1) == ~core).all())
    assert bool((lab[core] <= idx[core]).all())
    assert bool((lab[lab[core].long()] == lab[core]).all())  # the label point is its own cluster's root
    b = sp.friends_of_friends(p, eps)
    assert bool((a.labels == b.labels).all())


@pytest.mark.parametrize("shape", ["uniform", "field", "plane", "line", "shell", "dups"])
@pytest.mark.parametrize("mult", [0.05, 0.3, 1.0, 3.0])
def test_fof_cells_equal_point_pipeline(sp, shape, mult):
    # Two independent exact FoF algorithms on the GPU: the grid-cell pipeline
    # (cells united at their first close member pair) and the point pipeline
    # (pair traversal over the point LBVH), on 2^20 points of several shapes
    # and eps from 0.05x to 3x the mean spacing: labels and core flags must be
    # bit-identical.
    import torch
    n = 1 << 20
    g = torch.Generator().manual_seed(["uniform", "field", "plane", "line", "shell", "dups"].index(shape) * 10 +
                                      [0.05, 0.3, 1.0, 3.0].index(mult))
    if shape == "uniform":
        p = torch.rand(n, 3, generator=g)
    elif shape == "field":
        p = sp.generate_field(n, seed=7).cpu()
    elif shape == "plane":
        p = torch.rand(n, 3, generator=g)
        p[:, 2] = 0.5
    elif shape == "line":
        p = torch.zeros(n, 3)
        p[:, 0] = torch.rand(n, generator=g)
    elif shape == "shell":
        v = torch.randn(n, 3, generator=g)
        p = v / v.norm(dim=1, keepdim=True) * 0.4 + 0.5
    else:
        p = torch.rand(n // 64, 3, generator=g).repeat_interleave(64, 0)
    p = p.float().contiguous().cuda()
    spacing = (1.0 / n) ** (1.0 / 3.0) if shape in ("uniform", "field", "shell", "dups") else \
        ((1.0 / n) ** 0.5 if shape == "plane" else 1.0 / n)
    eps = float(np.float32(mult * spacing))
    a = sp.friends_of_friends(p, eps)
    b = sp.friends_of_friends(p, eps, algorithm="points")
    assert torch.equal(a.labels, b.labels), (shape, mult)
    assert torch.equal(a.core_flags, b.core_flags), (shape, mult)


@pytest.mark.parametrize("key", ["H_2^27", "H_2^30"])
def test_field_fof_against_reference_pin(sp, key):
    # the SURVEY field H(n) at the bench size (2^27) and at C5's full size
    # (2^30, 1.07 B points, one GPU): labels, core flags and counts equal the
    # unmodified reference's friends_of_friends on the same input
    # (scripts/ref_pin*.py, run on the GPU host); then the same rows through
    # the slab pipeline at one rank (sp_fof_slabs_multi, the device path of
    # sp_fof_slabs) give the same labels.
    import torch
    from paper_2409_10743_b200.distributed import fof_slabs_multi
    g = golden_hashes()[key]
    n = g["n"]
    eps = eps_for(n)
    torch.cuda.empty_cache()
    pts = torch.from_numpy(sp.generate_reference_field(n)).cuda()
    lab = torch.empty(n, dtype=torch.int32, device="cuda")
    core = torch.empty(n, dtype=torch.uint8, device="cuda")
    ctx = sp.Context(0)
    sp.friends_of_friends(pts, eps, ctx=ctx, out=(lab, core))
    ctx.close()
    hl, hc = lab.cpu().numpy(), core.cpu().numpy()
    assert summarize(hl, hc) == (g["clusters"], g["noise"], g["core"])
    assert fnv1a64(hc) == g["core_hash"]
    assert fnv1a64(hl) == g["labels_hash"]
    del hl, hc
    lab.fill_(-2)
    core.fill_(2)
    ctx = sp.Context(0)
    fof_slabs_multi([pts], eps, ctxs=[ctx], out=[(lab, core)])
    ctx.close()
    assert fnv1a64(core.cpu().numpy()) == g["core_hash"]
    assert fnv1a64(lab.cpu().numpy()) == g["labels_hash"]
