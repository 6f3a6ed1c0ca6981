"""Slab-decomposed friends-of-friends across ranks (SURVEY §8 row e).

The reference has no distributed search; the paper's
ArborX runs FoF per MPI rank.  This is the B200 form:
one process per GPU, `torch.distributed` (NCCL over NVLink on GPUs, gloo on
CPU for the tests) for the data exchange, the local FoF on the device.

    labels, core = fof_slabs(points, eps, first_index=...)

Every rank passes its slice of the global point array (rows
[first_index, first_index + n_local) in input order) and receives the labels
of exactly those rows: the smallest GLOBAL index of the point's cluster, or
-1 for noise — identical to a single-GPU run on the whole array.

Steps (each a collective over the default group):
  1. splitters  — all-gather per-rank x-quantiles; G-1 global x-splitters;
  2. partition  — all-to-all points + global indices to their slab owner;
  3. ghosts     — all-to-all copies of points within w = eps*(1+1e-6) of
                  another slab (a pair within eps has |dx| <= eps*(1+2^-24)
                  under the reference's rounding, so no cross pair is missed);
  4. local FoF  — owned + ghost points sorted by global index, so a local
                  min-index label IS the min global index of the local piece;
  5. merge      — all-gather (global index, local label) for every ghost copy
                  and its owner's label; labels sharing a global index are
                  connected; connected components over that small graph give
                  every rank the same label -> final label map;
  6. return     — all-to-all the owned labels back to the input layout.
Owned points see every neighbour within eps (owned or ghost), so core flags
and noise are exact locally.
"""
from __future__ import annotations

from typing import Callable, Optional, Tuple

import numpy as np
import torch
import torch.distributed as dist


def _all_to_all(t: torch.Tensor, send_counts: list, recv_counts: list, row: int = 1) -> torch.Tensor:
    out = torch.empty((sum(recv_counts) * row,), dtype=t.dtype, device=t.device)
    dist.all_to_all_single(out, t.reshape(-1).contiguous(), [c * row for c in recv_counts],
                           [c * row for c in send_counts])
    return out


def _exchange_counts(send: torch.Tensor, world: int) -> list:
    recv = torch.empty_like(send)
    dist.all_to_all_single(recv, send.contiguous())
    return recv.tolist()


def _all_gather_var(t: torch.Tensor, world: int) -> torch.Tensor:
    """All-gather tensors of different first dimensions."""
    n = torch.tensor([t.shape[0]], dtype=torch.int64, device=t.device)
    sizes = [torch.zeros_like(n) for _ in range(world)]
    dist.all_gather(sizes, n)
    sizes = [int(s.item()) for s in sizes]
    m = max(sizes) if sizes else 0
    pad = torch.zeros((m,) + tuple(t.shape[1:]), dtype=t.dtype, device=t.device)
    pad[: t.shape[0]] = t
    bufs = [torch.empty_like(pad) for _ in range(world)]
    dist.all_gather(bufs, pad)
    return torch.cat([b[:s] for b, s in zip(bufs, sizes)], dim=0)


def _device_fof(ctx):
    import paper_2409_10743_b200 as sp

    def run(points: torch.Tensor, eps: float):
        out = sp.friends_of_friends(points, eps, ctx=ctx)
        return out.labels, out.core_flags

    return run


def label_components(keys: np.ndarray, labels: np.ndarray) -> Tuple[np.ndarray, np.ndarray]:
    """Labels that share a key are connected; returns (unique labels, the
    minimum label of each one's component)."""
    from scipy.sparse import coo_matrix
    from scipy.sparse.csgraph import connected_components

    uniq, inv = np.unique(labels, return_inverse=True)
    if len(uniq) == 0:
        return uniq, uniq
    order = np.argsort(keys, kind="stable")
    k, v = keys[order], inv[order]
    same = k[1:] == k[:-1]
    a, b = v[:-1][same], v[1:][same]
    g = coo_matrix((np.ones(len(a), np.int8), (a, b)), shape=(len(uniq), len(uniq)))
    _, comp = connected_components(g, directed=False)
    comp_min = np.full(comp.max() + 1, np.iinfo(np.int64).max, np.int64)
    np.minimum.at(comp_min, comp, uniq)
    return uniq, comp_min[comp]


def fof_slabs(points: torch.Tensor, eps: float, first_index: int = 0, ctx=None,
              local_fof: Optional[Callable] = None, samples: int = 4096):
    """Friends-of-friends over all ranks' points; see the module docstring.

    points: (n_local, 3) float32 on this rank's device (CUDA for NCCL, CPU for
    gloo).  local_fof(points, eps) -> (labels int32, core uint8) with
    min-local-index labels; defaults to the device FoF (sp.friends_of_friends).
    Returns (labels int32, core uint8) for this rank's rows, input order."""
    world = dist.get_world_size()
    rank = dist.get_rank()
    dev = points.device
    run_local = local_fof or _device_fof(ctx)
    n_local = points.shape[0]
    gidx = torch.arange(first_index, first_index + n_local, dtype=torch.int64, device=dev)
    x = points[:, 0]

    # 1. splitters from gathered per-rank quantiles (identical on every rank)
    if n_local > 0:
        q = torch.linspace(0, 1, samples, device=dev, dtype=torch.float64)
        xs = torch.sort(x.double()).values
        local_q = xs[(q * (n_local - 1)).round().long()]
    else:
        local_q = torch.full((samples,), float("nan"), dtype=torch.float64, device=dev)
    allq = [torch.empty_like(local_q) for _ in range(world)]
    dist.all_gather(allq, local_q)
    allq = torch.cat(allq)
    allq = torch.sort(allq[~torch.isnan(allq)]).values
    if allq.numel() == 0:
        splitters = torch.zeros(max(world - 1, 0), dtype=torch.float32, device=dev)
    else:
        pos = (torch.arange(1, world, device=dev, dtype=torch.float64) / world * (allq.numel() - 1)).round().long()
        splitters = allq[pos].float()

    # 2. partition: rank d owns x in [splitters[d-1], splitters[d])
    dest = torch.bucketize(x, splitters, right=True)
    order = torch.argsort(dest, stable=True)
    send = torch.bincount(dest, minlength=world)
    recv = _exchange_counts(send, world)
    send = send.tolist()
    own_pts = _all_to_all(points[order], send, recv, 3).view(-1, 3)
    own_gidx = _all_to_all(gidx[order], send, recv)

    # 3. ghosts: copies to every other slab within w of the point
    w = float(eps) * (1.0 + 1e-6) + 1e-37
    ox = own_pts[:, 0]
    lo_r = torch.bucketize(ox - w, splitters, right=True)
    hi_r = torch.bucketize(ox + w, splitters, right=True)
    span = hi_r - lo_r + 1
    src = torch.repeat_interleave(torch.arange(own_pts.shape[0], device=dev), span)
    first = torch.repeat_interleave(lo_r, span)
    offs = torch.arange(src.numel(), device=dev) - torch.repeat_interleave(torch.cumsum(span, 0) - span, span)
    tgt = first + offs
    keep = tgt != rank
    src, tgt = src[keep], tgt[keep]
    gorder = torch.argsort(tgt, stable=True)
    src, tgt = src[gorder], tgt[gorder]
    gsend = torch.bincount(tgt, minlength=world)
    grecv = _exchange_counts(gsend, world)
    gsend = gsend.tolist()
    ghost_pts = _all_to_all(own_pts[src], gsend, grecv, 3).view(-1, 3)
    ghost_gidx = _all_to_all(own_gidx[src], gsend, grecv)
    sent_gidx = own_gidx[src]  # my points that live as ghosts elsewhere

    # 4. local FoF over owned + ghosts, in global-index order
    all_pts = torch.cat([own_pts, ghost_pts])
    all_gidx = torch.cat([own_gidx, ghost_gidx])
    perm = torch.argsort(all_gidx)
    lab, core = run_local(all_pts[perm].contiguous(), eps)
    lab = lab.to(torch.int64)
    sorted_gidx = all_gidx[perm]
    glab_sorted = torch.where(lab >= 0, sorted_gidx[lab.clamp(min=0)], torch.full_like(lab, -1))
    glab = torch.empty_like(glab_sorted)
    glab[perm] = glab_sorted
    core_all = torch.empty_like(core)
    core_all[perm] = core
    m_own = own_pts.shape[0]
    own_lab, own_core = glab[:m_own], core_all[:m_own]

    # 5. merge across slabs: (global index, label) of every ghost copy and of
    # the originals that were sent as ghosts
    pairs = torch.cat([torch.stack([ghost_gidx, glab[m_own:]], 1), torch.stack([sent_gidx, own_lab[src]], 1)])
    pairs = pairs[pairs[:, 1] >= 0]
    allpairs = _all_gather_var(pairs, world).cpu().numpy()
    uniq, final = label_components(allpairs[:, 0], allpairs[:, 1])
    if len(uniq):
        u = torch.from_numpy(uniq).to(dev)
        f = torch.from_numpy(final).to(dev)
        idx = torch.searchsorted(u, own_lab.clamp(min=0))
        idx = idx.clamp(max=len(uniq) - 1)
        hit = (own_lab >= 0) & (u[idx] == own_lab)
        own_lab = torch.where(hit, f[idx], own_lab)

    # 6. labels back to the input layout
    back_lab = _all_to_all(own_lab, recv, send)
    back_core = _all_to_all(own_core.to(torch.int32), recv, send)
    labels = torch.empty(n_local, dtype=torch.int64, device=dev)
    labels[order] = back_lab
    core_out = torch.empty(n_local, dtype=torch.int32, device=dev)
    core_out[order] = back_core
    return labels.to(torch.int32), core_out.to(torch.uint8)
