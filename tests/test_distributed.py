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
    keys = np.array([5, 5, 7, 7, 9])
    labs = np.array([10, 3, 3, 8, 11])
    u, f = label_components(keys, labs)
    m = dict(zip(u.tolist(), f.tolist()))
    assert m == {3: 3, 8: 3, 10: 3, 11: 11}


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
