"""CPU, world_size 2/3 over gloo: the slab-decomposed FoF exchange and merge
(paper_2409_10743_b200/distributed.py) give labels identical to a single
FoF over the union of all slices.  The local per-slab FoF is replaced by the
oracle here (test infrastructure), so the test exercises exactly the
splitters / all-to-all / ghost / cross-slab merge / return logic the GPU run
uses."""
import os
import socket
import sys

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, pts, eps, out_dir):
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle_lib import Oracle
    from paper_2409_10743_b200.distributed import fof_slabs  # noqa: E402

    O = Oracle.get()

    def local(points, e):
        lab, core = O.dbscan(points.numpy(), 3, e, 2)
        return torch.from_numpy(lab.astype(np.int32)), torch.from_numpy(core)

    n = len(pts)
    bounds = np.linspace(0, n, world + 1).astype(int)
    lo, hi = bounds[rank], bounds[rank + 1]
    labels, core = fof_slabs(torch.from_numpy(pts[lo:hi]), eps, first_index=int(lo), local_fof=local, samples=64)
    np.save(os.path.join(out_dir, "lab%d.npy" % rank), labels.numpy())
    np.save(os.path.join(out_dir, "core%d.npy" % rank), core.numpy())
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world,kind", [(2, "field"), (3, "field"), (2, "uniform"), (3, "chain")])
def test_slab_fof_equals_single_run(oracle, tmp_path, world, kind):
    if kind == "field":
        pts = oracle.field(1 << 14)
        eps = float(np.float32(0.168 * np.cbrt(1.0 / (1 << 14))) * 3)
    elif kind == "uniform":
        pts = oracle.uniform(20000, 3, 1.0, 5)
        eps = 0.03
    else:  # a chain that crosses every slab boundary
        t = np.linspace(0, 1, 3000, dtype=np.float32)
        pts = np.stack([t, np.zeros_like(t), np.zeros_like(t)], 1).astype(np.float32)
        pts = np.concatenate([pts, oracle.uniform(500, 3, 1.0, 9)]).astype(np.float32)
        eps = float(1.0 / 2999 * 1.01)
    port = _free_port()
    mp.spawn(_worker, args=(world, port, pts, eps, str(tmp_path)), nprocs=world, join=True)
    labels = np.concatenate([np.load(tmp_path / ("lab%d.npy" % r)) for r in range(world)])
    core = np.concatenate([np.load(tmp_path / ("core%d.npy" % r)) for r in range(world)])
    want_l, want_c = oracle.dbscan(pts, 3, eps, 2)
    assert np.array_equal(core, want_c)
    assert np.array_equal(labels, want_l)


def test_label_components():
    from paper_2409_10743_b200.distributed import label_components
    keys = torch.tensor([5, 5, 7, 7, 9])
    labs = torch.tensor([10, 3, 3, 8, 11])
    u, f = label_components(keys, labs)
    m = dict(zip(u.tolist(), f.tolist()))
    assert m == {3: 3, 8: 3, 10: 3, 11: 11}


def test_label_components_long_chains():
    # chains of labels linked through shared keys in scrambled order: every
    # label must map to the minimum of its chain
    from paper_2409_10743_b200.distributed import label_components
    g = torch.Generator().manual_seed(3)
    labs = torch.randperm(5000, generator=g) * 7 + 11
    chains = torch.arange(5000) % 17
    keys, vals = [], []
    for c in range(17):
        members = labs[chains == c]
        for i in range(len(members) - 1):  # link consecutive members
            keys += [c * 100000 + i, c * 100000 + i]
            vals += [int(members[i]), int(members[i + 1])]
    perm = torch.randperm(len(keys), generator=g)
    u, f = label_components(torch.tensor(keys)[perm], torch.tensor(vals)[perm])
    m = dict(zip(u.tolist(), f.tolist()))
    for c in range(17):
        members = labs[chains == c]
        assert all(m[int(x)] == int(members.min()) for x in members)


def _gpu_worker(rank, world, port, pts, eps, out_dir):
    sys.path.insert(0, ROOT)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_2409_10743_b200 as sp
    from paper_2409_10743_b200.distributed import fof_slabs

    ctx = sp.Context(0)

    def local(points, e):  # the device FoF on this rank's slab (+ ghosts)
        out = sp.friends_of_friends(points.cuda(), e, ctx=ctx)
        return out.labels.cpu(), out.core_flags.cpu()

    n = len(pts)
    bounds = np.linspace(0, n, world + 1).astype(int)
    lo, hi = bounds[rank], bounds[rank + 1]
    labels, core = fof_slabs(torch.from_numpy(pts[lo:hi]), eps, first_index=int(lo), local_fof=local, samples=256)
    np.save(os.path.join(out_dir, "lab%d.npy" % rank), labels.numpy())
    np.save(os.path.join(out_dir, "core%d.npy" % rank), core.numpy())
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.gpu
@pytest.mark.parametrize("world", [2, 4])
def test_slab_fof_with_device_local_fof(oracle, tmp_path, world):
    n = 1 << 20
    pts = oracle.field(n)
    eps = float(np.float32(0.168 * np.cbrt(1.0 / n)))
    port = _free_port()
    mp.spawn(_gpu_worker, args=(world, port, pts, eps, str(tmp_path)), nprocs=world, join=True)
    labels = np.concatenate([np.load(tmp_path / ("lab%d.npy" % r)) for r in range(world)])
    core = np.concatenate([np.load(tmp_path / ("core%d.npy" % r)) for r in range(world)])
    want_l, want_c = oracle.dbscan(pts, 3, eps, 2)
    assert np.array_equal(core, want_c)
    assert np.array_equal(labels, want_l)


def _nccl_worker(rank, world, port, n, out_dir):
    # the production path: CUDA tensors, NCCL collectives, device FoF + device merge
    sys.path.insert(0, ROOT)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", rank=rank, world_size=world)
    import paper_2409_10743_b200 as sp
    from paper_2409_10743_b200.distributed import fof_slabs

    ctx = sp.Context(0)
    pts = sp.generate_field(n, seed=2409, ctx=ctx)
    eps = float(np.float32(0.168 * np.cbrt(1.0 / n)))
    labels, core = fof_slabs(pts, eps, first_index=0, ctx=ctx)
    ref = sp.friends_of_friends(pts, eps, ctx=ctx)
    np.save(os.path.join(out_dir, "ok.npy"), np.array([bool(torch.equal(labels, ref.labels)),
                                                       bool(torch.equal(core, ref.core_flags))]))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.gpu
def test_slab_fof_over_nccl_single_rank(tmp_path):
    # one GPU per rank is all a round's box offers: world_size 1 over NCCL runs
    # every collective of the slab path on CUDA tensors
    port = _free_port()
    mp.spawn(_nccl_worker, args=(1, port, 1 << 22, str(tmp_path)), nprocs=1, join=True)
    assert np.load(tmp_path / "ok.npy").all()
