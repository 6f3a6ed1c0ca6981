"""GPU: the native slab FoF (sp_fof_slabs_multi / sp_fof_slabs, csrc/sp_slabs.cu)
gives labels and core flags bit-identical to the single-GPU FoF over the whole
array (and so to the reference's friends_of_friends), for G = 1..8 ranks.

One box offers one GPU, so the G-rank runs put G contexts on that device
(sp_fof_slabs_multi: the same device pipeline, with peer copies in place of the
NCCL collectives); the NCCL form runs at world size 1 in a spawned process.
The field at 2^27 is checked against the unmodified reference's labels hash
(tests/golden/golden_hashes.json "H_2^27", scripts/ref_pin.py)."""
import os
import socket
import sys

import numpy as np
import pytest
import torch

from fixtures import golden_hashes, summarize
from oracle_lib import eps_for, fnv1a64

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _split(n, G, skew=None):
    if skew == "empty":  # G - 1 equal parts, then rank 1 holds nothing
        b = np.linspace(0, n, G).astype(np.int64)
        return np.concatenate([b[:2], b[1:]])
    return np.linspace(0, n, G + 1).astype(np.int64)


def _run_multi(sp, pts, eps, G, skew=None, host=False):
    n = len(pts)
    b = _split(n, G, skew)
    ctxs = [sp.Context(0) for _ in range(G)]
    if host:
        parts = [np.ascontiguousarray(pts[b[r]:b[r + 1]].cpu().numpy()) for r in range(G)]
    else:
        parts = [pts[b[r]:b[r + 1]].contiguous() for r in range(G)]
    from paper_2409_10743_b200.distributed import fof_slabs_multi
    res = fof_slabs_multi(parts, eps, ctxs=ctxs)
    lab = torch.cat([torch.as_tensor(r[0]).cpu() for r in res])
    core = torch.cat([torch.as_tensor(r[1]).cpu() for r in res])
    return lab, core


def _shape(kind, n, g):
    if kind == "field":
        import paper_2409_10743_b200 as sp
        return torch.from_numpy(sp.generate_reference_field(n)), eps_for(n)
    if kind == "uniform":
        return torch.rand(n, 3, generator=g), float(np.float32((1.0 / n) ** (1 / 3)))
    if kind == "wide_eps":  # eps wider than a slab: ghosts span several slabs
        return torch.rand(n, 3, generator=g), 0.3
    if kind == "chain":  # one cluster crossing every slab boundary along x
        t = torch.linspace(0, 1, n)
        p = torch.stack([t, torch.zeros(n), torch.zeros(n)], 1)
        return p, float(np.float32(1.0 / (n - 1) * 1.01))
    if kind == "same_x":  # all x equal: every point in one slab
        p = torch.rand(n, 3, generator=g)
        p[:, 0] = 0.25
        return p, float(np.float32((1.0 / n) ** 0.5))
    if kind == "dups":
        p = torch.rand(n // 16, 3, generator=g).repeat_interleave(16, 0)
        return p, float(np.float32((16.0 / n) ** (1 / 3) * 0.5))
    raise ValueError(kind)


@pytest.mark.parametrize("G", [1, 2, 3, 4, 8])
@pytest.mark.parametrize("kind", ["field", "uniform", "wide_eps", "chain", "same_x", "dups"])
def test_slabs_multi_equal_single_gpu(sp, G, kind):
    g = torch.Generator().manual_seed(G * 100 + len(kind))
    n = 1 << 18 if kind != "wide_eps" else 1 << 14
    p, eps = _shape(kind, n, g)
    p = p.float().contiguous().cuda()
    want = sp.friends_of_friends(p, eps)
    lab, core = _run_multi(sp, p, eps, G)
    assert torch.equal(lab, want.labels.cpu()), (kind, G)
    assert torch.equal(core, want.core_flags.cpu()), (kind, G)


@pytest.mark.parametrize("G", [3, 8])
def test_slabs_multi_empty_rank_and_host_buffers(sp, G):
    n = 1 << 18
    p, eps = _shape("field", n, None)
    p = p.cuda()
    want = sp.friends_of_friends(p, eps)
    lab, core = _run_multi(sp, p, eps, G, skew="empty")
    assert torch.equal(lab, want.labels.cpu()) and torch.equal(core, want.core_flags.cpu())
    lab, core = _run_multi(sp, p, eps, G, host=True)
    assert torch.equal(lab, want.labels.cpu()) and torch.equal(core, want.core_flags.cpu())


@pytest.mark.parametrize("G", [2, 4])
def test_slabs_multi_empty_exchange(sp, G):
    # each rank's rows fill their own x band, the bands further than eps
    # apart: no row moves and no point is a ghost anywhere, so every rank runs
    # the single-GPU FoF in place (labels offset to global indices)
    g = torch.Generator().manual_seed(7 + G)
    n = 1 << 16
    per = n // G
    p = torch.rand(n, 3, generator=g)
    band = torch.arange(n) // per
    p[:, 0] = (band.float() + 0.4 * p[:, 0]) / G
    eps = float(np.float32(0.02 / G))
    p = p.contiguous().cuda()
    want = sp.friends_of_friends(p, eps)
    lab, core = _run_multi(sp, p, eps, G)
    assert torch.equal(lab, want.labels.cpu()) and torch.equal(core, want.core_flags.cpu())
    assert int((want.labels >= per).sum()) > 0  # labels beyond the first rank's rows occur


def test_slabs_multi_h27_against_reference(sp):
    # 8 ranks x 2^24 rows of H(2^27): the labels of the unmodified reference
    g = golden_hashes()["H_2^27"]
    n = g["n"]
    p = torch.from_numpy(sp.generate_reference_field(n)).cuda()
    lab, core = _run_multi(sp, p, eps_for(n), 8)
    del p
    torch.cuda.empty_cache()
    lab, core = lab.numpy(), core.numpy()
    assert summarize(lab, core) == (g["clusters"], g["noise"], g["core"])
    assert fnv1a64(core) == g["core_hash"]
    assert fnv1a64(lab) == g["labels_hash"]


def test_slabs_invalid_arguments(sp):
    from paper_2409_10743_b200.distributed import fof_slabs_multi
    p = torch.rand(100, 3).cuda()
    with pytest.raises(sp.InvalidArgument):
        fof_slabs_multi([p, p], -1.0, ctxs=[sp.Context(0), sp.Context(0)])
    with pytest.raises(sp.InvalidArgument):
        fof_slabs_multi([torch.rand(10, 2).cuda()], 0.1, ctxs=[sp.Context(0)])


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _nccl_native_worker(rank, world, port, n, out_dir):
    sys.path.insert(0, ROOT)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    import torch.distributed as dist
    dist.init_process_group("nccl", rank=rank, world_size=world)
    import paper_2409_10743_b200 as sp
    from paper_2409_10743_b200.distributed import SlabComm, fof_slabs

    ctx = sp.Context(0, stream=torch.cuda.current_stream().cuda_stream)
    comm = SlabComm.create(ctx)
    host = sp.generate_reference_field(n)
    pts = torch.from_numpy(host).cuda()
    eps = eps_for(n)
    ok = [comm.size == world, comm.rank == rank]
    lab, core = fof_slabs(pts, eps, first_index=0, ctx=ctx, comm=comm)
    ref = sp.friends_of_friends(pts, eps, ctx=ctx)
    ok += [bool(torch.equal(lab, ref.labels)), bool(torch.equal(core, ref.core_flags))]
    hl, hc = fof_slabs(host, eps, first_index=0, ctx=ctx, comm=comm)  # host buffers through the C ABI
    ok += [bool(np.array_equal(hl.numpy(), ref.labels.cpu().numpy())),
           bool(np.array_equal(hc.numpy(), ref.core_flags.cpu().numpy()))]
    np.save(os.path.join(out_dir, "ok.npy"), np.array(ok))
    comm.close()
    dist.barrier()
    dist.destroy_process_group()


def test_slabs_nccl_world1_native(tmp_path):
    import torch.multiprocessing as mp
    mp.spawn(_nccl_native_worker, args=(1, _free_port(), 1 << 22, str(tmp_path)), nprocs=1, join=True)
    ok = np.load(tmp_path / "ok.npy")
    assert ok.all(), ok
