"""Slab-decomposed friends-of-friends across ranks (SURVEY §8 row e).

The reference has no distributed search; the paper's
ArborX runs FoF per MPI rank.  This is the B200 form:
one process per GPU.

    comm = SlabComm.create(ctx)                 # NCCL, over the default group
    labels, core = fof_slabs(points, eps, first_index=..., ctx=ctx, comm=comm)

Every rank passes its slice of the global point array (rows
[first_index, first_index + n_local) in input order) and receives the labels
of exactly those rows: the smallest GLOBAL index of the point's cluster, or
-1 for noise — identical to a single-GPU run on the whole array.

The product path is native: sp_fof_slabs (csrc/sp_slabs.cu) runs every step
on the device with NCCL collectives and one host read of the exchange sizes;
`fof_slabs_multi` drives several contexts from one process (sp_fof_slabs_multi,
peer copies instead of NCCL).  `fof_slabs_torch` restates the same algorithm
over torch.distributed collectives (any backend): with gloo and a CPU local
FoF it is the world-size-2/3 CPU model of the exchange and merge logic the
tests run without a GPU.

Steps of fof_slabs_torch (each a collective over the default group):
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
    """The device FoF with global ids: labels come back as the smallest global
    index of each local cluster directly (sp_fof_ids)."""
    import paper_2409_10743_b200 as sp

    def run(points: torch.Tensor, eps: float, gids: torch.Tensor):
        ids = gids.to(torch.int32).contiguous()
        c = ctx
        if c is None:
            # torch's current stream on the points' device: ordered after the
            # torch ops (and collectives) that produced points and ids
            c = sp.default_context(sp._device_of(points))
        elif points.is_cuda:
            cur = torch.cuda.current_stream(points.device)
            if getattr(c, "stream", None) is None or int(c.stream) != int(cur.cuda_stream):
                cur.synchronize()  # a context on another stream waits for them
        out = sp.friends_of_friends_ids(points, eps, ids, ctx=c)
        return out.labels, out.core_flags

    run.global_ids = True
    return run


def label_components(keys: torch.Tensor, labels: torch.Tensor) -> Tuple[torch.Tensor, torch.Tensor]:
    """Labels that share a key are connected; returns (unique labels, the
    minimum label of each one's component).  Runs where the tensors live (the
    GPU under NCCL): hook-to-min union-find over the compacted labels with
    pointer jumping, the same invariant as the device union-find (a root is
    the smallest member, union_find.hpp:15-16)."""
    keys = torch.as_tensor(keys)
    labels = torch.as_tensor(labels, device=keys.device)
    uniq, inv = torch.unique(labels, return_inverse=True)
    if uniq.numel() == 0:
        return uniq, uniq
    order = torch.argsort(keys, stable=True)
    k, v = keys[order], inv[order]
    same = k[1:] == k[:-1]
    a, b = v[:-1][same], v[1:][same]
    parent = torch.arange(uniq.numel(), device=uniq.device, dtype=torch.int64)
    while True:
        pa, pb = parent[a], parent[b]
        lo, hi = torch.minimum(pa, pb), torch.maximum(pa, pb)
        new = parent.clone()
        new.scatter_reduce_(0, hi, lo, reduce="amin")  # hook each root under the smaller one
        while True:  # pointer jumping to full compression
            nxt = new[new]
            if torch.equal(nxt, new):
                break
            new = nxt
        if torch.equal(new, parent):
            return uniq, uniq[parent]
        parent = new


def fof_slabs_torch(points: torch.Tensor, eps: float, first_index: int = 0, ctx=None,
                    local_fof: Optional[Callable] = None, samples: int = 4096):
    """Friends-of-friends over all ranks' points with torch.distributed
    collectives (the algorithm restated for any backend); see the module
    docstring.

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

    # 1. splitters from gathered per-rank quantiles of a strided sample
    #    (identical on every rank; they only balance the slabs)
    if n_local > 0:
        stride = max(1, n_local // (1 << 20))
        xs = torch.sort(x[::stride].double()).values
        q = torch.linspace(0, 1, samples, device=dev, dtype=torch.float64)
        local_q = xs[(q * (xs.numel() - 1)).round().long()]
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


    # 2. partition: rank d owns x in [splitters[d-1], splitters[d]); the stable
    #    argsort runs on 16-bit slab ids (a one/two-pass radix sort)
    if world > 1:
        dest = torch.bucketize(x, splitters, right=True)
        order = torch.argsort(dest.to(torch.int16), stable=True)
        send = torch.bincount(dest, minlength=world)
        recv = _exchange_counts(send, world)
        send = send.tolist()
        own_pts = _all_to_all(points[order], send, recv, 3).view(-1, 3)
        own_gidx = _all_to_all(gidx[order], send, recv)
    else:
        order, send, recv = None, [n_local], [n_local]
        own_pts, own_gidx = points, gidx


    # 3. ghosts: copies to every other slab within w of the point; only points
    #    within w of a splitter can have any
    w = float(eps) * (1.0 + 1e-6) + 1e-37
    m_own = own_pts.shape[0]
    if world > 1:
        ox = own_pts[:, 0]
        lo_r = torch.bucketize(ox - w, splitters, right=True)
        hi_r = torch.bucketize(ox + w, splitters, right=True)
        near = torch.nonzero(lo_r != hi_r).squeeze(1)
        lo_n, hi_n = lo_r[near], hi_r[near]
        span = hi_n - lo_n + 1
        src = torch.repeat_interleave(near, span)
        first = torch.repeat_interleave(lo_n, span)
        offs = torch.arange(src.numel(), device=dev) - torch.repeat_interleave(torch.cumsum(span, 0) - span, span)
        tgt = first + offs
        keep = tgt != rank
        src, tgt = src[keep], tgt[keep]
        gorder = torch.argsort(tgt.to(torch.int16), stable=True)
        src, tgt = src[gorder], tgt[gorder]
        gsend = torch.bincount(tgt, minlength=world)
        grecv = _exchange_counts(gsend, world)
        gsend = gsend.tolist()
        ghost_pts = _all_to_all(own_pts[src], gsend, grecv, 3).view(-1, 3)
        ghost_gidx = _all_to_all(own_gidx[src], gsend, grecv)
        all_pts = torch.cat([own_pts, ghost_pts])
        all_gidx = torch.cat([own_gidx, ghost_gidx])
    else:
        src = torch.empty(0, dtype=torch.int64, device=dev)
        ghost_gidx = torch.empty(0, dtype=torch.int64, device=dev)
        all_pts, all_gidx = own_pts, own_gidx
    sent_gidx = own_gidx[src]  # my points that live as ghosts elsewhere


    # 4. local FoF over owned + ghosts; the cluster label becomes the minimum
    #    GLOBAL index of its local members (a segmented min over the labels)
    if getattr(run_local, "global_ids", False):
        lab, core_all = run_local(all_pts.contiguous(), eps, all_gidx)
        glab = lab.to(torch.int64)
    else:
        lab, core_all = run_local(all_pts.contiguous(), eps)
        lab = lab.to(dev).to(torch.int64)
        member = lab >= 0
        gmin = torch.full((all_pts.shape[0],), torch.iinfo(torch.int64).max, dtype=torch.int64, device=dev)
        gmin.scatter_reduce_(0, lab[member], all_gidx[member], reduce="amin")
        glab = torch.where(member, gmin[lab.clamp(min=0)], torch.full_like(lab, -1))
    core_all = core_all.to(dev)
    own_lab, own_core = glab[:m_own], core_all[:m_own]


    # 5. merge across slabs: (global index, label) of every ghost copy and of
    # the originals that were sent as ghosts
    pairs = torch.cat([torch.stack([ghost_gidx, glab[m_own:]], 1), torch.stack([sent_gidx, own_lab[src]], 1)])
    pairs = pairs[pairs[:, 1] >= 0]
    allpairs = _all_gather_var(pairs, world)
    u, f = label_components(allpairs[:, 0], allpairs[:, 1])
    if u.numel():
        idx = torch.searchsorted(u, own_lab.clamp(min=0))
        idx = idx.clamp(max=u.numel() - 1)
        hit = (own_lab >= 0) & (u[idx] == own_lab)
        own_lab = torch.where(hit, f[idx], own_lab)


    # 6. labels back to the input layout
    if world > 1:
        back_lab = _all_to_all(own_lab, recv, send)
        back_core = _all_to_all(own_core.to(torch.int32), recv, send)
        labels = torch.empty(n_local, dtype=torch.int64, device=dev)
        labels[order] = back_lab
        core_out = torch.empty(n_local, dtype=torch.int32, device=dev)
        core_out[order] = back_core
    else:
        labels, core_out = own_lab, own_core
    return labels.to(torch.int32), core_out.to(torch.uint8)


# ---------------------------------------------------------------------------
# native path (sp_fof_slabs / sp_fof_slabs_multi)
# ---------------------------------------------------------------------------
class SlabComm:
    """An sp_comm: the NCCL communicator of the native slab FoF."""

    def __init__(self, handle, ctx):
        self.h = handle
        self.ctx = ctx

    @classmethod
    def create(cls, ctx, group=None) -> "SlabComm":
        """ncclCommInitRank over the ranks of `group` (default: the default
        process group); rank 0's unique id travels by a torch.distributed
        broadcast (any backend)."""
        import ctypes as C
        import paper_2409_10743_b200 as sp
        rank, world = dist.get_rank(group), dist.get_world_size(group)
        uid = (C.c_uint8 * 128)()
        if rank == 0 and sp._lib.sp_comm_unique_id(uid) != sp.SP_OK:
            raise sp.CudaError("sp_comm_unique_id failed (NCCL unavailable)")
        dev = torch.device("cuda", ctx.device) if dist.get_backend(group) == "nccl" else torch.device("cpu")
        t = torch.tensor(bytearray(bytes(uid)), dtype=torch.uint8, device=dev)
        dist.broadcast(t, src=dist.get_global_rank(group, 0) if group is not None else 0, group=group)
        uid = (C.c_uint8 * 128)(*t.cpu().tolist())
        h = C.c_void_p()
        ctx._check(sp._lib.sp_comm_create(ctx.h, world, rank, uid, C.byref(h)))
        return cls(h, ctx)

    @classmethod
    def from_process_group(cls, ctx, group=None) -> "SlabComm":
        return cls.create(ctx, group)

    @classmethod
    def wrap(cls, ctx, nccl_comm: int) -> "SlabComm":
        """Use an existing ncclComm_t (an integer handle; not owned)."""
        import ctypes as C
        import paper_2409_10743_b200 as sp
        h = C.c_void_p()
        ctx._check(sp._lib.sp_comm_wrap(ctx.h, C.c_void_p(nccl_comm), C.byref(h)))
        return cls(h, ctx)

    @property
    def size(self) -> int:
        import paper_2409_10743_b200 as sp
        return int(sp._lib.sp_comm_size(self.h))

    @property
    def rank(self) -> int:
        import paper_2409_10743_b200 as sp
        return int(sp._lib.sp_comm_rank(self.h))

    def close(self):
        import paper_2409_10743_b200 as sp
        if self.h:
            sp._lib.sp_comm_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


_comms: dict = {}


def _native_out(points, n, out, dev):
    import paper_2409_10743_b200 as sp
    if out is not None:
        lab, lp = sp._given_out(out[0], (n,), 4, dev)
        core, cp = sp._given_out(out[1], (n,), 1, dev)
        return lab, core, lp, cp
    kw = dict(device=points.device) if dev else dict(pin_memory=False)
    lab = torch.empty(n, dtype=torch.int32, **kw)
    core = torch.empty(n, dtype=torch.uint8, **kw)
    return lab, core, sp._ptr(lab), sp._ptr(core)


def fof_slabs(points, eps: float, first_index: int = 0, ctx=None, comm: Optional[SlabComm] = None, out=None,
              local_fof: Optional[Callable] = None, samples: int = 4096):
    """Friends-of-friends over all ranks' points; see the module docstring.

    With a SlabComm, or CUDA points under an NCCL default group, this is the
    native sp_fof_slabs (points: (n_local, 3) float32, device tensor or host
    array/pinned tensor; `out` = (labels int32, core uint8) in the same memory
    space).  With a custom `local_fof` or gloo/CPU tensors it is
    fof_slabs_torch.  Returns (labels int32, core uint8) for this rank's rows."""
    import ctypes as C
    import paper_2409_10743_b200 as sp
    native = comm is not None or (local_fof is None and sp._is_cuda(points) and dist.is_initialized() and
                                  dist.get_backend() == "nccl")
    if not native:
        return fof_slabs_torch(points, eps, first_index=first_index, ctx=ctx, local_fof=local_fof, samples=samples)
    if ctx is None:
        ctx = sp.default_context(sp._device_of(points))
    if comm is None:
        key = (ctx.device, id(dist.group.WORLD))
        if key not in _comms:
            _comms[key] = SlabComm.create(ctx)
        comm = _comms[key]
    if len(points.shape) != 2 or int(points.shape[1]) != 3:
        raise sp.InvalidArgument("points must have shape (n, 3)")
    n = int(points.shape[0])
    p, mem, keep = sp._in(points, np.float32)
    dev = mem == sp.SP_MEM_DEVICE
    lab, core, lp, cp = _native_out(points, n, out, dev)
    ctx._check(sp._lib.sp_fof_slabs(ctx.h, comm.h, p, n, C.c_float(eps), int(first_index), lp, cp, mem))
    return lab, core


def fof_slabs_multi(points: list, eps: float, ctxs: Optional[list] = None, out: Optional[list] = None):
    """All ranks in this process (sp_fof_slabs_multi): points[r] holds rank
    r's rows (rank r's rows follow rank r-1's), on ctxs[r]'s device (or all on
    the host).  Several contexts may share one device.  Returns
    [(labels, core)] per rank."""
    import ctypes as C
    import paper_2409_10743_b200 as sp
    G = len(points)
    if ctxs is None:
        ctxs = [sp.Context(sp._device_of(p)[0]) for p in points]
    if len(ctxs) != G:
        raise ValueError("one context per rank")
    arrs, keeps, mems, res = [], [], set(), []
    for r, pr in enumerate(points):
        if len(pr.shape) != 2 or int(pr.shape[1]) != 3:
            raise sp.InvalidArgument("points must have shape (n, 3)")
        p, mem, keep = sp._in(pr, np.float32)
        arrs.append(p)
        keeps.append(keep)
        mems.add(mem)
        res.append(_native_out(pr, int(pr.shape[0]), out[r] if out is not None else None, mem == sp.SP_MEM_DEVICE))
    if len(mems) != 1:
        raise ValueError("all ranks' points must live in the same memory space")
    mem = mems.pop()
    P = (C.c_void_p * G)(*[a.value for a in arrs])
    N = (C.c_int64 * G)(*[int(pr.shape[0]) for pr in points])
    LP = (C.c_void_p * G)(*[r_[2].value for r_ in res])
    CP = (C.c_void_p * G)(*[r_[3].value for r_ in res])
    H = (C.c_void_p * G)(*[c.h.value for c in ctxs])
    ctxs[0]._check(sp._lib.sp_fof_slabs_multi(H, G, P, N, C.c_float(eps), LP, CP, mem))
    return [(r_[0], r_[1]) for r_ in res]
