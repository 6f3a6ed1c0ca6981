"""B200-native geometric search and density clustering (arXiv 2409.10743).

Python host mirror of the reference's `namespace spatial` API
(/root/reference/proj/include/spatial/*.hpp) over the C ABI in
include/sp_b200.h (libspb200.so, sm_100a kernels).  Names, argument meaning
and error behaviour follow the reference:

  reference (C++)                          here
  ---------------------------------------  ----------------------------------
  Bvh<D>::build(objects, width)            Bvh.build(objects, width=64, points=...)
  range_query(bvh, preds, count-callback)  range_count(bvh, spheres|boxes, cap=0)
  query_crs(bvh, preds, ..., max_total)    query_crs(bvh, spheres, max_total_matches)
  nearest_query(bvh, preds, cb)            nearest_query(bvh, origins, k)
  pair_traversal(bvh, eps, cb)             pair_traversal(bvh, eps)
  sort_queries(preds)                      sort_queries(points)
  fdbscan / friends_of_friends /           fdbscan / friends_of_friends /
  fdbscan_densebox -> DbscanOutput         fdbscan_densebox -> DbscanOutput
  std::invalid_argument                    ValueError (InvalidArgument)
  CapacityError : std::bad_alloc           CapacityError (MemoryError)

Arrays may be numpy (host; copied through the call) or torch CUDA tensors
(device-resident; nothing crosses PCIe).  There is no CPU fallback: importing
this package on a machine where libspb200.so cannot be loaded raises, and
every call needs a CUDA device.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field
from typing import Optional

import numpy as np

from . import build as _build

__all__ = [
    "Bvh", "DbscanOutput", "DbscanParams", "DbscanTimings", "DbscanStats", "InvalidArgument", "CapacityError",
    "CudaError", "range_count", "query_crs", "nearest_query", "pair_traversal", "sort_queries", "morton_codes",
    "fdbscan", "friends_of_friends", "fdbscan_densebox", "adjacency_graph_dbscan", "dbscan_reference",
    "check_equivalence", "generate_reference_uniform", "generate_reference_gaussian", "generate_reference_field", "generate_field", "generate_uniform",
    "Context",
    "default_context", "library_path",
]

SP_OK, SP_EINVAL, SP_ECAPACITY, SP_ECUDA, SP_ENOMEM, SP_ENCCL = range(6)
SP_MEM_HOST, SP_MEM_DEVICE = 0, 1
SP_ALGO_FDBSCAN, SP_ALGO_FOF, SP_ALGO_DENSEBOX, SP_ALGO_FOF_POINTS, SP_ALGO_DENSEBOX_MIXED = 0, 1, 2, 3, 4
SP_ALGO_SEQUENTIAL = 0x100  # ExecMode::kSequential (exec.hpp:12)
SP_PRED_SPHERE, SP_PRED_BOX = 0, 1
kNoiseLabel = -1


class InvalidArgument(ValueError):
    """std::invalid_argument in the reference."""


class CapacityError(MemoryError):
    """spatial::CapacityError (a std::bad_alloc) in the reference."""


class CudaError(RuntimeError):
    pass


def library_path() -> str:
    return _build.LIB


def _load() -> C.CDLL:
    path = _build.LIB
    if not os.path.exists(path):
        # Build in-tree (nvcc cross-compiles for sm_100a); never fall back.
        _build.build()
    lib = C.CDLL(path)
    vp, i64, i32, f32 = C.c_void_p, C.c_int64, C.c_int32, C.c_float
    pp = C.POINTER(C.c_void_p)
    sig = {
        "sp_ctx_create": (C.c_int, [C.c_int, vp, pp]),
        "sp_ctx_destroy": (C.c_int, [vp]),
        "sp_ctx_set_stream": (C.c_int, [vp, vp]),
        "sp_ctx_synchronize": (C.c_int, [vp]),
        "sp_ctx_set_flags": (C.c_int, [vp, C.c_int]),
        "sp_last_error": (C.c_char_p, [vp]),
        "sp_ctx_kernel_launches": (i64, [vp]),
        "sp_ctx_phase_count": (C.c_int, [vp]),
        "sp_ctx_counter": (i64, [vp, C.c_char_p]),
        "sp_ctx_phase_name": (C.c_char_p, [vp, C.c_int]),
        "sp_ctx_phase_ms": (C.c_double, [vp, C.c_int]),
        "sp_bvh_build": (C.c_int, [vp, vp, i64, C.c_int, C.c_int, C.c_int, C.c_int, pp]),
        "sp_bvh_destroy": (C.c_int, [vp]),
        "sp_bvh_size": (i64, [vp]),
        "sp_bvh_export": (C.c_int, [vp, vp, vp, vp, vp, vp, vp, vp, vp]),
        "sp_range_count": (C.c_int, [vp, vp, C.c_int, vp, i64, i32, vp, C.c_int]),
        "sp_range_count_radius": (C.c_int, [vp, vp, vp, i64, f32, i32, vp, C.c_int]),
        "sp_range_crs": (C.c_int, [vp, vp, C.c_int, vp, i64, vp, vp, i64, C.c_int]),
        "sp_knn": (C.c_int, [vp, vp, vp, i64, i32, vp, vp, C.c_int]),
        "sp_pair_list": (C.c_int, [vp, vp, f32, vp, i64, C.POINTER(i64), C.c_int]),
        "sp_sort_queries": (C.c_int, [vp, vp, i64, C.c_int, vp, C.c_int]),
        "sp_morton_codes": (C.c_int, [vp, vp, i64, C.c_int, C.c_int, C.c_int, vp, C.c_int]),
        "sp_dbscan": (C.c_int, [vp, vp, i64, C.c_int, f32, i32, C.c_int, C.c_int, vp, vp, vp, vp, C.c_int]),
        "sp_dbscan_bruteforce": (C.c_int, [vp, vp, i64, C.c_int, f32, i32, vp, vp, C.c_int]),
        "sp_fof_ids": (C.c_int, [vp, vp, i64, C.c_int, f32, vp, vp, vp, C.c_int]),
        "sp_generate_reference": (C.c_int, [C.c_int, i64, C.c_int, i32, C.c_double, C.c_double, C.c_uint64, vp]),
        "sp_dbscan_adjacency": (C.c_int, [vp, vp, i64, C.c_int, f32, C.c_int, i64, vp, vp, vp, C.c_int]),
        "sp_check_equivalence": (C.c_int, [vp, vp, i64, C.c_int, f32, vp, vp, vp, vp, C.POINTER(i64),
                                           C.POINTER(C.c_int), C.c_int]),
        "sp_generate_reference_field": (C.c_int, [i64, i64, i64, vp]),
        "sp_comm_unique_id": (C.c_int, [vp]),
        "sp_comm_create": (C.c_int, [vp, C.c_int, C.c_int, vp, vp]),
        "sp_comm_wrap": (C.c_int, [vp, vp, vp]),
        "sp_comm_destroy": (C.c_int, [vp]),
        "sp_comm_size": (C.c_int, [vp]),
        "sp_comm_rank": (C.c_int, [vp]),
        "sp_fof_slabs": (C.c_int, [vp, vp, vp, i64, f32, i64, vp, vp, C.c_int]),
        "sp_fof_slabs_multi": (C.c_int, [vp, C.c_int, vp, vp, f32, vp, vp, C.c_int]),
        "sp_generate_field": (C.c_int, [vp, i64, i64, i64, C.c_uint64, vp, C.c_int]),
        "sp_generate_uniform": (C.c_int, [vp, i64, C.c_int, C.c_uint64, vp, C.c_int]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


_lib = _load()


class _Timings(C.Structure):
    _fields_ = [("build_ms", C.c_double), ("core_ms", C.c_double), ("merge_ms", C.c_double),
                ("finalize_ms", C.c_double)]


class _Stats(C.Structure):
    _fields_ = [("distance_checks", C.c_int64), ("num_dense_cells", C.c_int64), ("num_dense_points", C.c_int64)]


def _stream_arg(stream: Optional[int]):
    """None -> a context-owned stream; a cudaStream_t handle otherwise.  Handle
    0 (torch's default stream) is the legacy default stream, which the C ABI
    takes as cudaStreamLegacy ((void *)1) because NULL means "own stream"."""
    if stream is None:
        return None
    return C.c_void_p(stream if stream != 0 else 1)


class Context:
    """An sp_ctx: one device + one stream (exec.hpp's ExecMode analogue)."""

    def __init__(self, device: int = 0, stream: Optional[int] = None):
        h = C.c_void_p()
        rc = _lib.sp_ctx_create(device, _stream_arg(stream), C.byref(h))
        if rc != SP_OK:
            raise CudaError("sp_ctx_create(device=%d) failed (status %d): no usable CUDA device" % (device, rc))
        self.h = h
        self._flags = 0
        self.device = device
        self.stream = stream  # the caller's stream handle, or None (own stream)

    def close(self):
        if self.h:
            _lib.sp_ctx_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def set_stream(self, stream: Optional[int]):
        self._check(_lib.sp_ctx_set_stream(self.h, _stream_arg(stream)))
        self.stream = stream

    def synchronize(self):
        self._check(_lib.sp_ctx_synchronize(self.h))

    def set_async(self, on: bool = True):
        """SP_FLAG_ASYNC: calls only enqueue work; call synchronize() before
        reading outputs or reusing host buffers."""
        self._flags = (self._flags | 1) if on else (self._flags & ~1)
        self._check(_lib.sp_ctx_set_flags(self.h, self._flags))

    def set_stats(self, on: bool = True):
        """SP_FLAG_STATS: diagnostic kernels count traversal work into
        counter() ("merge_node_visits", "merge_pair_tests"); measurement only."""
        self._flags = (self._flags | 2) if on else (self._flags & ~2)
        self._check(_lib.sp_ctx_set_flags(self.h, self._flags))

    @property
    def kernel_launches(self) -> int:
        return int(_lib.sp_ctx_kernel_launches(self.h))

    def counter(self, name: str) -> int:
        """Diagnostic counter of the last call (-1 if absent)."""
        return int(_lib.sp_ctx_counter(self.h, name.encode()))

    def phases(self) -> list:
        """[(name, ms)] device-event phase times of the last call."""
        return [(_lib.sp_ctx_phase_name(self.h, i).decode(), float(_lib.sp_ctx_phase_ms(self.h, i)))
                for i in range(_lib.sp_ctx_phase_count(self.h))]

    def _check(self, rc: int):
        if rc == SP_OK:
            return
        msg = (_lib.sp_last_error(self.h) or b"").decode()
        if rc == SP_EINVAL:
            raise InvalidArgument(msg)
        if rc == SP_ECAPACITY:
            raise CapacityError(msg)
        raise CudaError("status %d: %s" % (rc, msg))


_defaults: dict = {}


def _device_of(a):
    """(device, stream) for the implicit context of a call on `a`: a CUDA
    tensor runs on its device and on torch's current stream there (so the call
    is ordered after the torch work that produced it); host arrays use device
    0 and a context-owned stream."""
    if _is_cuda(a):
        import torch
        d = int(a.device.index if a.device.index is not None else torch.cuda.current_device())
        return d, int(torch.cuda.current_stream(d).cuda_stream)
    return 0, None


def default_context(device=0, stream: Optional[int] = None) -> Context:
    """The process-wide context of (device, stream), made on first use;
    `device` may also be a (device, stream) pair from _device_of."""
    if isinstance(device, tuple):
        device, stream = device
    key = (device, stream)
    if key not in _defaults:
        _defaults[key] = Context(device, stream=stream)
    return _defaults[key]


# ---- array plumbing -----------------------------------------------------------
def _is_cuda(a) -> bool:
    return hasattr(a, "is_cuda") and bool(a.is_cuda)


def _is_torch(a) -> bool:
    return hasattr(a, "data_ptr") and hasattr(a, "is_contiguous")


def _ptr(a) -> C.c_void_p:
    return C.c_void_p(a.data_ptr() if _is_torch(a) else a.ctypes.data)


def _in(a, dtype):
    """(pointer, mem, keepalive) for an input array: numpy, a (pinned) CPU
    tensor, or a CUDA tensor (device-resident; no copy)."""
    if _is_torch(a):
        if not a.is_contiguous():
            a = a.contiguous()
        return C.c_void_p(a.data_ptr()), (SP_MEM_DEVICE if a.is_cuda else SP_MEM_HOST), a
    arr = np.ascontiguousarray(a, dtype=dtype)
    return arr.ctypes.data_as(C.c_void_p), SP_MEM_HOST, arr


def _out(like_device: bool, shape, np_dtype, torch_dtype=None, device=None):
    if like_device:
        import torch
        t = torch.empty(shape, dtype=torch_dtype, device=device)
        return t, C.c_void_p(t.data_ptr())
    arr = np.empty(shape, dtype=np_dtype)
    return arr, arr.ctypes.data_as(C.c_void_p)


def _given_out(a, shape, itemsize: int, dev: bool):
    """Pointer of a caller-supplied output buffer (numpy array or tensor, e.g.
    a reusable pinned host tensor): contiguous, in the inputs' memory space,
    with the expected shape and element size."""
    if _is_cuda(a) != dev:
        raise ValueError("out must live in the same memory space as the inputs")
    if tuple(a.shape) != tuple(shape):
        raise ValueError("out has shape %s, expected %s" % (tuple(a.shape), tuple(shape)))
    size = a.element_size() if _is_torch(a) else a.itemsize
    contiguous = a.is_contiguous() if _is_torch(a) else a.flags["C_CONTIGUOUS"]
    if size != itemsize or not contiguous:
        raise ValueError("out must be contiguous with %d-byte elements" % itemsize)
    return a, _ptr(a)


def _dim_of(a) -> int:
    s = tuple(a.shape)
    if len(s) != 2 or s[1] not in (2, 3):
        raise InvalidArgument("points must have shape (n, 2) or (n, 3)")
    return s[1]


# ---- hierarchy ------------------------------------------------------------------
class Bvh:
    """Device-resident Bvh<D> (bvh.hpp:43-86).  Immutable after build."""

    def __init__(self, handle, dim: int, width: int, ctx: Context):
        self.h = handle
        self.dim = dim
        self.width = width
        self.ctx = ctx

    @classmethod
    def build(cls, objects, width: int = 64, points: Optional[bool] = None, ctx: Optional[Context] = None) -> "Bvh":
        """Bvh<D>::build(objects, CodeWidth) (bvh.hpp:243-261).

        objects: (n, d) points (point boxes) or (n, 2, d) / (n, 2d) boxes with
        points=False.  Raises InvalidArgument on non-finite coordinates."""
        ctx = ctx or default_context(_device_of(objects))
        shape = tuple(objects.shape)
        if points is None:
            points = len(shape) == 2
        if points:
            dim = _dim_of(objects)
        else:
            dim = shape[-1] if len(shape) == 3 else shape[1] // 2
            if dim not in (2, 3):
                raise InvalidArgument("boxes must have shape (n, 2, d) or (n, 2d), d in {2, 3}")
        n = shape[0]
        p, mem, keep = _in(objects, np.float32)
        h = C.c_void_p()
        ctx._check(_lib.sp_bvh_build(ctx.h, p, n, dim, int(points), width, mem, C.byref(h)))
        return cls(h, dim, width, ctx)

    def __del__(self):
        try:
            if self.h:
                _lib.sp_bvh_destroy(self.h)
                self.h = None
        except Exception:
            pass

    def size(self) -> int:
        return int(_lib.sp_bvh_size(self.h))

    def empty(self) -> bool:
        return self.size() == 0

    def export(self) -> dict:
        """internals/leaves in the reference numbering (bvh.hpp:45-60)."""
        n, d = self.size(), self.dim
        m = max(n - 1, 0)
        out = dict(internal_left=np.empty(max(m, 1), np.int32), internal_rope=np.empty(max(m, 1), np.int32),
                   internal_boxes=np.empty((max(m, 1), 2 * d), np.float32),
                   leaf_object=np.empty(max(n, 1), np.int32), leaf_rope=np.empty(max(n, 1), np.int32),
                   leaf_boxes=np.empty((max(n, 1), 2 * d), np.float32), scene=np.empty(2 * d, np.float32))
        ptr = lambda a: a.ctypes.data_as(C.c_void_p)
        self.ctx._check(_lib.sp_bvh_export(self.ctx.h, self.h, ptr(out["internal_left"]), ptr(out["internal_rope"]),
                                           ptr(out["internal_boxes"]), ptr(out["leaf_object"]),
                                           ptr(out["leaf_rope"]), ptr(out["leaf_boxes"]), ptr(out["scene"])))
        for k in ("internal_left", "internal_rope", "internal_boxes"):
            out[k] = out[k][:m]
        for k in ("leaf_object", "leaf_rope", "leaf_boxes"):
            out[k] = out[k][:n]
        return out

    def dump(self) -> str:
        """Bvh::dump text format (bvh.hpp:332-357)."""
        e = self.export()
        d = self.dim
        lines = ["bvh n %d width %d" % (self.size(), self.width)]

        def box(b):
            return "".join(" %s" % _fmt9(float(v)) for v in b)

        for i in range(len(e["internal_left"])):
            lines.append("I %d left %d rope %d%s" % (i, e["internal_left"][i], e["internal_rope"][i],
                                                     box(e["internal_boxes"][i])))
        for p in range(len(e["leaf_object"])):
            lines.append("L %d object %d rope %d%s" % (p, e["leaf_object"][p], e["leaf_rope"][p],
                                                       box(e["leaf_boxes"][p])))
        return "\n".join(lines) + "\n"

    def validate(self) -> tuple:
        """Bvh::validate (bvh.hpp:263-330) on the exported arrays: (ok, violation)."""
        return validate_arrays(self.export(), self.size(), self.dim)


def _fmt9(v: float) -> str:
    s = "%.9g" % v
    return s


def validate_arrays(e: dict, n: int, dim: int) -> tuple:
    if n == 0:
        return True, ""
    il, ir, ib = e["internal_left"], e["internal_rope"], e["internal_boxes"]
    lo, lr, lb = e["leaf_object"], e["leaf_rope"], e["leaf_boxes"]
    if len(il) != n - 1:
        return False, "internal node count is not n-1"
    is_leaf = lambda r: r >= n - 1
    rope = lambda r: lr[r - (n - 1)] if is_leaf(r) else ir[r]
    vol = lambda r: lb[r - (n - 1)] if is_leaf(r) else ib[r]
    cur, expected, steps = (n - 1 if n == 1 else 0), 0, 0
    while cur != -1:
        steps += 1
        if steps > 2 * n + 1:
            return False, "rope walk does not terminate (cycle)"
        if is_leaf(cur):
            if cur - (n - 1) != expected:
                return False, "rope walk visits leaf %d expecting %d" % (cur - (n - 1), expected)
            expected += 1
            cur = rope(cur)
        else:
            cur = il[cur]
    if expected != n:
        return False, "rope walk covered %d of %d leaves" % (expected, n)
    for i in range(n - 1):
        left = il[i]
        right = rope(left)
        if right == -1:
            return False, "internal node %d has no reachable right child" % i
        a, b = vol(left), vol(right)
        u = np.concatenate([np.where(b[:dim] < a[:dim], b[:dim], a[:dim]), np.where(a[dim:] < b[dim:], b[dim:], a[dim:])])
        if not np.array_equal(u.view(np.uint32), np.asarray(ib[i], np.float32).view(np.uint32)):
            return False, "internal node %d volume is not the union of children" % i
    sentinels = int((ir == -1).sum() + (lr == -1).sum())
    length, cur = 0, (n - 1 if n == 1 else 0)
    while True:
        length += 1
        if is_leaf(cur):
            if rope(cur) != -1:
                return False, "right-most leaf rope is not the sentinel"
            break
        if ir[cur] != -1:
            return False, "right-most path internal node rope is not the sentinel"
        cur = rope(il[cur])
    if sentinels != length:
        return False, "sentinel ropes off the right-most path"
    return True, ""


# ---- queries ----------------------------------------------------------------------
def range_count(bvh: Bvh, predicates, kind: str = "sphere", cap: int = 0, radius: Optional[float] = None,
                out=None):
    """range_query with a counting callback (traversal.hpp:67-87).

    kind="sphere": predicates (nq, d+1) = centre, radius; or (nq, d) centres
    with a shared `radius`.  kind="box": (nq, 2d) boxes.  cap > 0 terminates a
    query at cap matches (detect_core_counts, dbscan.hpp:146-170).  out: an
    optional int32 (nq,) buffer to write the counts into (returned)."""
    ctx = bvh.ctx
    nq = int(predicates.shape[0])
    d = bvh.dim
    want = d if radius is not None else (2 * d if kind == "box" else d + 1)
    if len(predicates.shape) != 2 or int(predicates.shape[1]) != want:
        raise InvalidArgument("predicates must have shape (nq, %d) for kind=%r%s" %
                              (want, kind, " with radius" if radius is not None else ""))
    p, mem, keep = _in(predicates, np.float32)
    dev = mem == SP_MEM_DEVICE
    if out is not None:
        counts, cp = _given_out(out, (nq,), 4, dev)
    else:
        counts, cp = _out(dev, (nq,), np.int32, _torch_dtype("int32") if dev else None,
                          predicates.device if dev else None)
    if radius is not None:
        ctx._check(_lib.sp_range_count_radius(ctx.h, bvh.h, p, nq, float(radius), int(cap), cp, mem))
    else:
        k = SP_PRED_BOX if kind == "box" else SP_PRED_SPHERE
        ctx._check(_lib.sp_range_count(ctx.h, bvh.h, k, p, nq, int(cap), cp, mem))
    return counts


def query_crs(bvh: Bvh, predicates, kind: str = "sphere", max_total_matches: Optional[int] = None):
    """query_crs (traversal.hpp:235-266) -> (offsets int64[nq+1], values int32)."""
    ctx = bvh.ctx
    preds = np.ascontiguousarray(predicates, np.float32)
    nq = preds.shape[0]
    want = 2 * bvh.dim if kind == "box" else bvh.dim + 1
    if preds.ndim != 2 or preds.shape[1] != want:
        raise InvalidArgument("predicates must have shape (nq, %d) for kind=%r" % (want, kind))
    k = SP_PRED_BOX if kind == "box" else SP_PRED_SPHERE
    offsets = np.empty(nq + 1, np.int64)
    pv = preds.ctypes.data_as(C.c_void_p)
    ctx._check(_lib.sp_range_crs(ctx.h, bvh.h, k, pv, nq, offsets.ctypes.data_as(C.c_void_p), None, 0, SP_MEM_HOST))
    total = int(offsets[-1])
    cap = total if max_total_matches is None else int(max_total_matches)
    if total > cap:
        raise CapacityError("crs result exceeds capacity")
    values = np.empty(max(total, 1), np.int32)
    ctx._check(_lib.sp_range_crs(ctx.h, bvh.h, k, pv, nq, offsets.ctypes.data_as(C.c_void_p),
                                 values.ctypes.data_as(C.c_void_p), max(total, 1), SP_MEM_HOST))
    return offsets, values[:total]


def nearest_query(bvh: Bvh, origins, k: int, with_distances: bool = False, out=None):
    """nearest_query (traversal.hpp:93-156): (nq, k) object indices ascending
    by (distance, index), padded with -1 beyond min(k, n).  out: optional
    (nq, k) int32 index buffer, or (indices, distances) with with_distances."""
    ctx = bvh.ctx
    nq = int(origins.shape[0])
    if len(origins.shape) != 2 or int(origins.shape[1]) != bvh.dim:
        raise InvalidArgument("origins must have shape (nq, %d)" % bvh.dim)
    kk = max(int(k), 0)
    p, mem, keep = _in(origins, np.float32)
    dev = mem == SP_MEM_DEVICE
    out_idx, out_dist = (out if with_distances else (out, None)) if out is not None else (None, None)
    if out_idx is not None:
        idx, ip = _given_out(out_idx, (nq, kk), 4, dev)
    else:
        idx, ip = _out(dev, (nq, kk), np.int32, _torch_dtype("int32") if dev else None,
                       origins.device if dev else None)
    dist, dp = (None, None)
    if with_distances:
        if out_dist is not None:
            dist, dp = _given_out(out_dist, (nq, kk), 4, dev)
        else:
            dist, dp = _out(dev, (nq, kk), np.float32, _torch_dtype("float32") if dev else None,
                            origins.device if dev else None)
    if kk > 0 and nq > 0:
        ctx._check(_lib.sp_knn(ctx.h, bvh.h, p, nq, kk, ip, dp, mem))
    return (idx, dist) if with_distances else idx


def pair_traversal(bvh: Bvh, eps: float) -> np.ndarray:
    """pair_traversal (traversal.hpp:162-184): (m, 2) object index pairs, each
    close pair exactly once, first element from the earlier leaf."""
    ctx = bvh.ctx
    total = C.c_int64(0)
    ctx._check(_lib.sp_pair_list(ctx.h, bvh.h, float(eps), None, 0, C.byref(total), SP_MEM_HOST))
    m = int(total.value)
    pairs = np.empty((max(m, 1), 2), np.int32)
    if m:
        ctx._check(_lib.sp_pair_list(ctx.h, bvh.h, float(eps), pairs.ctypes.data_as(C.c_void_p), m, C.byref(total),
                                     SP_MEM_HOST))
    return pairs[:m]


def sort_queries(points, ctx: Optional[Context] = None):
    """sort_queries over point representatives (traversal.hpp:209-218)."""
    ctx = ctx or default_context(_device_of(points))
    dim = _dim_of(points)
    n = int(points.shape[0])
    p, mem, keep = _in(points, np.float32)
    dev = mem == SP_MEM_DEVICE
    order, op = _out(dev, (n,), np.int32, _torch_dtype("int32") if dev else None, points.device if dev else None)
    ctx._check(_lib.sp_sort_queries(ctx.h, p, n, dim, op, mem))
    return order


def morton_codes(objects, width: int = 64, points: bool = True, ctx: Optional[Context] = None):
    """code_of(centroid(object), scene) for every object (morton.hpp:106-109)."""
    ctx = ctx or default_context(_device_of(objects))
    arr = np.ascontiguousarray(objects, np.float32)
    n = arr.shape[0]
    dim = arr.shape[1] if points else arr.shape[1] // 2
    codes = np.empty(max(n, 1), np.uint64)
    ctx._check(_lib.sp_morton_codes(ctx.h, arr.ctypes.data_as(C.c_void_p), n, dim, int(points), width,
                                    codes.ctypes.data_as(C.c_void_p), SP_MEM_HOST))
    return codes[:n]


# ---- clustering ------------------------------------------------------------------
@dataclass
class DbscanParams:
    eps: float = 0.0
    min_pts: int = 2


@dataclass
class DbscanTimings:
    build_ms: float = 0.0
    core_ms: float = 0.0
    merge_ms: float = 0.0
    finalize_ms: float = 0.0

    def total_ms(self) -> float:
        return self.build_ms + self.core_ms + self.merge_ms + self.finalize_ms


@dataclass
class DbscanStats:
    distance_checks: int = 0
    num_dense_cells: int = 0
    num_dense_points: int = 0


@dataclass
class DbscanOutput:
    labels: object = None
    core_flags: object = None
    timings: DbscanTimings = field(default_factory=DbscanTimings)
    stats: DbscanStats = field(default_factory=DbscanStats)


def _dbscan(points, eps, min_pts, algo, width, ctx, out=None):
    ctx = ctx or default_context(_device_of(points))
    dim = _dim_of(points)
    n = int(points.shape[0])
    p, mem, keep = _in(points, np.float32)
    dev = mem == SP_MEM_DEVICE
    if out is not None:
        # one memory-space flag covers every pointer of the call (sp_b200.h)
        labels, lp = _given_out(out[0], (n,), 4, dev)
        core, cp = _given_out(out[1], (n,), 1, dev)
    else:
        labels, lp = _out(dev, (n,), np.int32, _torch_dtype("int32") if dev else None, points.device if dev else None)
        core, cp = _out(dev, (n,), np.uint8, _torch_dtype("uint8") if dev else None, points.device if dev else None)
    t, s = _Timings(), _Stats()
    ctx._check(_lib.sp_dbscan(ctx.h, p, n, dim, C.c_float(eps), int(min_pts), algo, int(width), lp, cp, C.byref(t),
                              C.byref(s), mem))
    return DbscanOutput(labels, core, DbscanTimings(t.build_ms, t.core_ms, t.merge_ms, t.finalize_ms),
                        DbscanStats(s.distance_checks, s.num_dense_cells, s.num_dense_points))


def fdbscan(points, params: DbscanParams, width: int = 64, ctx: Optional[Context] = None, out=None,
            mode: str = "parallel") -> DbscanOutput:
    """fdbscan (dbscan.hpp:277-282).  mode="sequential" (ExecMode::kSequential,
    exec.hpp:12) gives the reference's deterministic sequential labels: each
    border point joins the cluster of its core neighbour of smallest leaf
    position; "parallel" admits any valid border assignment."""
    if mode not in ("parallel", "sequential"):
        raise InvalidArgument("mode must be 'parallel' or 'sequential'")
    seq = SP_ALGO_SEQUENTIAL if mode == "sequential" else 0
    return _dbscan(points, params.eps, params.min_pts, SP_ALGO_FDBSCAN | seq, width, ctx, out)


def friends_of_friends(points, eps: float, width: int = 64, ctx: Optional[Context] = None, out=None,
                       algorithm: str = "cells") -> DbscanOutput:
    """friends_of_friends (dbscan.hpp:286-292): FDBSCAN with min_pts = 2.
    algorithm="cells" (default) clusters over grid cells;
    "points" runs the reference's own pair traversal over the point
    hierarchy.  Both give identical labels and core flags."""
    algo = {"cells": SP_ALGO_FOF, "points": SP_ALGO_FOF_POINTS}[algorithm]
    return _dbscan(points, eps, 2, algo, width, ctx, out)


def friends_of_friends_ids(points, eps: float, ids, ctx: Optional[Context] = None, out=None):
    """friends_of_friends whose labels are the smallest ids[i] of each
    cluster (-1 = noise) instead of the smallest index: the per-slab step of the
    multi-GPU FoF, which passes global indices (sp_fof_ids).  ids: int32, one
    per point, distinct, >= 0, in the same memory space as the points."""
    ctx = ctx or default_context(_device_of(points))
    dim = _dim_of(points)
    n = int(points.shape[0])
    p, mem, keep = _in(points, np.float32)
    dev = mem == SP_MEM_DEVICE
    if _is_cuda(ids) != dev:
        raise ValueError("ids must live in the same memory space as the points")
    if tuple(ids.shape) != (n,):
        raise InvalidArgument("ids must have shape (n,)")
    ip, _, keep_ids = _in(ids, np.int32)
    if out is not None:
        labels, lp = _given_out(out[0], (n,), 4, dev)
        core, cp = _given_out(out[1], (n,), 1, dev)
    else:
        labels, lp = _out(dev, (n,), np.int32, _torch_dtype("int32") if dev else None, points.device if dev else None)
        core, cp = _out(dev, (n,), np.uint8, _torch_dtype("uint8") if dev else None, points.device if dev else None)
    ctx._check(_lib.sp_fof_ids(ctx.h, p, n, dim, C.c_float(eps), ip, lp, cp, mem))
    return DbscanOutput(labels, core)


def fdbscan_densebox(points, params: DbscanParams, width: int = 64, ctx: Optional[Context] = None,
                     out=None, algorithm: str = "cells", mode: str = "parallel") -> DbscanOutput:
    """fdbscan_densebox (dbscan.hpp:298-449).  algorithm="cells" (default)
    runs the all-cells pipeline; "mixed" the reference's
    mixed tree of dense cells and sparse points.  Equivalent clusterings.
    mode="sequential" (ExecMode::kSequential) gives the reference's
    sequential labels bit for bit (over the mixed tree)."""
    if mode not in ("parallel", "sequential"):
        raise InvalidArgument("mode must be 'parallel' or 'sequential'")
    algo = {"cells": SP_ALGO_DENSEBOX, "mixed": SP_ALGO_DENSEBOX_MIXED}[algorithm]
    algo |= SP_ALGO_SEQUENTIAL if mode == "sequential" else 0
    return _dbscan(points, params.eps, params.min_pts, algo, width, ctx, out)


def adjacency_graph_dbscan(points, eps: float, width: int = 64, max_adjacency: Optional[int] = None,
                           ctx: Optional[Context] = None) -> DbscanOutput:
    """adjacency_graph_dbscan (dbscan.hpp:456-504): the historical baseline
    that materialises the neighbour CRS; raises CapacityError past
    max_adjacency."""
    ctx = ctx or default_context(_device_of(points))
    dim = _dim_of(points)
    n = int(points.shape[0])
    p, mem, keep = _in(points, np.float32)
    dev = mem == SP_MEM_DEVICE
    labels, lp = _out(dev, (n,), np.int32, _torch_dtype("int32") if dev else None, points.device if dev else None)
    core, cp = _out(dev, (n,), np.uint8, _torch_dtype("uint8") if dev else None, points.device if dev else None)
    t = _Timings()
    cap = (1 << 62) if max_adjacency is None else int(max_adjacency)
    ctx._check(_lib.sp_dbscan_adjacency(ctx.h, p, n, dim, C.c_float(eps), int(width), cap, lp, cp, C.byref(t), mem))
    return DbscanOutput(labels, core, DbscanTimings(t.build_ms, t.core_ms, t.merge_ms, t.finalize_ms))


def dbscan_reference(points, params: DbscanParams, ctx: Optional[Context] = None) -> DbscanOutput:
    """dbscan_reference (dbscan.hpp:188-222): brute-force O(n^2) DBSCAN on the
    device, independent of the tree (for verification of small inputs)."""
    ctx = ctx or default_context(_device_of(points))
    dim = _dim_of(points)
    n = int(points.shape[0])
    p, mem, keep = _in(points, np.float32)
    dev = mem == SP_MEM_DEVICE
    labels, lp = _out(dev, (n,), np.int32, _torch_dtype("int32") if dev else None, points.device if dev else None)
    core, cp = _out(dev, (n,), np.uint8, _torch_dtype("uint8") if dev else None, points.device if dev else None)
    ctx._check(_lib.sp_dbscan_bruteforce(ctx.h, p, n, dim, C.c_float(params.eps), int(params.min_pts), lp, cp, mem))
    return DbscanOutput(labels, core)


def generate_reference_uniform(n: int, dim: int = 3, extent: float = 1.0, seed: int = 0) -> np.ndarray:
    """generate(UniformSpec) (generate.cpp:17-31), bit-identical."""
    out = np.empty(max(n * dim, 1), np.float32)
    if _lib.sp_generate_reference(0, n, dim, 1, 0.0, extent, seed, out.ctypes.data_as(C.c_void_p)) != SP_OK:
        raise InvalidArgument("generate: bad uniform spec")
    return out[: n * dim].reshape(n, dim)


def generate_reference_gaussian(n: int, dim: int, k: int, sigma: float, extent: float, seed: int) -> np.ndarray:
    """generate(GaussianClustersSpec) (generate.cpp:33-66), bit-identical."""
    out = np.empty(max(n * dim, 1), np.float32)
    if _lib.sp_generate_reference(1, n, dim, k, sigma, extent, seed, out.ctypes.data_as(C.c_void_p)) != SP_OK:
        raise InvalidArgument("generate: bad gaussian_clusters spec")
    return out[: n * dim].reshape(n, dim)


def generate_reference_field(n_total: int, first: int = 0, count: Optional[int] = None, out=None):
    """Rows [first, first+count) of the SURVEY §8(d) field H(n_total), drawn
    exactly as the reference's generate() draws them (generate.cpp:17-66):
    25% uniform background (seed 2409) then Gaussian halos of 8192 points
    (seed 2410).  Host memory: a numpy array, or `out` (e.g. a pinned CPU
    tensor of shape (count, 3), float32)."""
    count = n_total - first if count is None else count
    if out is None:
        out = np.empty((max(count, 0), 3), np.float32)
    if tuple(out.shape) != (count, 3) or _is_cuda(out):
        raise ValueError("out must be a host (count, 3) float32 array")
    if _lib.sp_generate_reference_field(n_total, first, count, _ptr(out)) != SP_OK:
        raise InvalidArgument("generate: bad field slice")
    return out


def check_equivalence(points, eps: float, got: DbscanOutput, want: DbscanOutput, ctx: Optional[Context] = None):
    """check_equivalence (verify.hpp:21-61): None when equivalent, else a
    message naming the first violating point."""
    ctx = ctx or default_context(_device_of(points))
    dim = _dim_of(points)
    n = int(points.shape[0])
    p, mem, keep = _in(points, np.float32)
    arrs = []
    for a, dt in ((got.labels, np.int32), (got.core_flags, np.uint8), (want.labels, np.int32),
                  (want.core_flags, np.uint8)):
        if mem == SP_MEM_DEVICE:
            a = a if _is_torch(a) and a.is_cuda else _torch_from(a, points.device)
        else:
            a = np.ascontiguousarray(a.cpu().numpy() if _is_torch(a) else a, dtype=dt)
        arrs.append(a)
    v, k = C.c_int64(-1), C.c_int(0)
    ctx._check(_lib.sp_check_equivalence(ctx.h, p, n, dim, C.c_float(eps), _ptr(arrs[0]), _ptr(arrs[1]), _ptr(arrs[2]),
                                         _ptr(arrs[3]), C.byref(v), C.byref(k), mem))
    if v.value < 0:
        return None
    what = {1: "core flag mismatch", 2: "noise mismatch", 3: "core partition mismatch", 4: "core clusters merged",
            5: "border point has no in-cluster core point within eps"}[k.value]
    return "%s at point %d" % (what, v.value)


def _torch_from(a, device):
    import torch
    return torch.as_tensor(np.ascontiguousarray(a)).to(device)


# ---- synthetic inputs ---------------------------------------------------------------
def generate_field(n_total: int, first: int = 0, count: Optional[int] = None, seed: int = 2409, out=None,
                   ctx: Optional[Context] = None):
    """HACC-like clustered field slice [first, first+count) on the device."""
    ctx = ctx or default_context()
    count = n_total - first if count is None else count
    if out is None:
        import torch
        out = torch.empty((count, 3), dtype=torch.float32, device="cuda:%d" % ctx.device)
    ctx._check(_lib.sp_generate_field(ctx.h, n_total, first, count, seed, C.c_void_p(out.data_ptr()), SP_MEM_DEVICE))
    return out


def generate_uniform(n: int, dim: int = 3, seed: int = 2409, out=None, ctx: Optional[Context] = None):
    ctx = ctx or default_context()
    if out is None:
        import torch
        out = torch.empty((n, dim), dtype=torch.float32, device="cuda:%d" % ctx.device)
    ctx._check(_lib.sp_generate_uniform(ctx.h, n, dim, seed, C.c_void_p(out.data_ptr()), SP_MEM_DEVICE))
    return out


def _torch_dtype(name: str):
    import torch
    return getattr(torch, name)
