"""ctypes bindings to the test-only checkers under oracle/.

`Oracle` wraps oracle/liboracle.so (the CPU restatement, built from repo
sources); `Reference` wraps oracle/_ref/libref.so (the unmodified reference
compiled in place, present only where /root/reference existed at build time).
Both are TEST INFRASTRUCTURE: only tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / reference legs may load them.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ORACLE_DIR = os.path.join(ROOT, "oracle")
ORACLE_SO = os.path.join(ORACLE_DIR, "liboracle.so")
REF_SO = os.path.join(ORACLE_DIR, "_ref", "libref.so")

_f32p = np.ctypeslib.ndpointer(np.float32, flags="C_CONTIGUOUS")
_i32p = np.ctypeslib.ndpointer(np.int32, flags="C_CONTIGUOUS")
_i64p = np.ctypeslib.ndpointer(np.int64, flags="C_CONTIGUOUS")
_u8p = np.ctypeslib.ndpointer(np.uint8, flags="C_CONTIGUOUS")
_u64p = np.ctypeslib.ndpointer(np.uint64, flags="C_CONTIGUOUS")
_f64p = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")


def _f32(a):
    return np.ascontiguousarray(a, dtype=np.float32)


def fnv1a64(arr) -> str:
    """FNV-1a-64 over the raw little-endian bytes (SURVEY §8(c) golden hash)."""
    b = np.ascontiguousarray(arr).view(np.uint8)
    h = np.uint64(1469598103934665603)
    # vectorised in chunks would change nothing semantically; use the C helper
    return "%016x" % Oracle.get().fnv(b)


def eps_for(n: int) -> float:
    """eps(n) = float(0.168 * cbrt(1/n)) (report.cpp:12-16)."""
    return float(np.float32(0.168 * np.cbrt(1.0 / float(n))))


class Oracle:
    _inst = None

    @classmethod
    def get(cls) -> "Oracle":
        if cls._inst is None:
            if not os.path.exists(ORACLE_SO):
                subprocess.check_call(["make", "-s", "-C", ORACLE_DIR, "all"])
            cls._inst = cls(ORACLE_SO)
        return cls._inst

    def __init__(self, path):
        L = self.lib = C.CDLL(path)
        L.orc_fnv1a64.restype = C.c_uint64
        L.orc_fnv1a64.argtypes = [C.c_void_p, C.c_int64]
        L.orc_generate_uniform.argtypes = [C.c_int64, C.c_int, C.c_double, C.c_uint64, _f32p]
        L.orc_generate_gaussian.argtypes = [C.c_int64, C.c_int, C.c_int32, C.c_double, C.c_double, C.c_uint64, _f32p]
        L.orc_generate_field.argtypes = [C.c_int64, _f32p]
        L.orc_morton_codes.argtypes = [_f32p, C.c_int64, C.c_int, C.c_int, C.c_int, _u64p]
        L.orc_bvh_build.argtypes = [_f32p, C.c_int64, C.c_int, C.c_int, C.c_int, _i32p, _i32p, _f32p, _i32p, _i32p, _f32p]
        L.orc_range_count.argtypes = [_f32p, C.c_int64, C.c_int, C.c_int, _f32p, C.c_int64, C.c_int, C.c_int32, _i32p]
        L.orc_range_crs.argtypes = [_f32p, C.c_int64, C.c_int, C.c_int, _f32p, C.c_int64, _i64p, C.c_void_p]
        L.orc_knn.argtypes = [_f32p, C.c_int64, C.c_int, C.c_int, _f32p, C.c_int64, C.c_int32, _i32p, _f32p]
        L.orc_dbscan.argtypes = [_f32p, C.c_int64, C.c_int, C.c_float, C.c_int32, _i32p, _u8p, C.c_void_p]
        L.orc_check_equivalence.restype = C.c_int64
        L.orc_check_equivalence.argtypes = [_f32p, C.c_int64, C.c_int, C.c_float, _i32p, _u8p, _i32p, _u8p,
                                            C.POINTER(C.c_int32)]
        L.orc_distance.restype = C.c_float
        L.orc_distance.argtypes = [_f32p, _f32p, C.c_int]

    def fnv(self, b: np.ndarray) -> int:
        b = np.ascontiguousarray(b)
        return int(self.lib.orc_fnv1a64(b.ctypes.data, b.nbytes))

    def uniform(self, n, dim=3, extent=1.0, seed=0):
        out = np.empty(n * dim, np.float32)
        assert self.lib.orc_generate_uniform(n, dim, extent, seed, out) == 0
        return out.reshape(n, dim)

    def gaussian(self, n, dim, k, sigma, extent, seed):
        out = np.empty(n * dim, np.float32)
        assert self.lib.orc_generate_gaussian(n, dim, k, sigma, extent, seed, out) == 0
        return out.reshape(n, dim)

    def field(self, n):
        out = np.empty(n * 3, np.float32)
        assert self.lib.orc_generate_field(n, out) == 0
        return out.reshape(n, 3)

    def morton(self, objs, dim, width, is_points=True):
        objs = _f32(objs)
        n = objs.shape[0]
        codes = np.empty(n, np.uint64)
        self.lib.orc_morton_codes(objs.reshape(-1), n, dim, int(is_points), width, codes)
        return codes

    def bvh(self, objs, dim, width=64, is_points=True):
        """Node arrays: dict(internal_left, internal_rope, internal_boxes, leaf_object, leaf_rope, leaf_boxes)."""
        objs = _f32(objs)
        n = objs.shape[0]
        m = max(n - 1, 0)
        out = dict(internal_left=np.empty(m, np.int32), internal_rope=np.empty(m, np.int32),
                   internal_boxes=np.empty((m, 2 * dim), np.float32), leaf_object=np.empty(n, np.int32),
                   leaf_rope=np.empty(n, np.int32), leaf_boxes=np.empty((n, 2 * dim), np.float32))
        rc = self.lib.orc_bvh_build(objs.reshape(-1), n, dim, int(is_points), width, out["internal_left"],
                                    out["internal_rope"], out["internal_boxes"].reshape(-1), out["leaf_object"],
                                    out["leaf_rope"], out["leaf_boxes"].reshape(-1))
        if rc:
            raise ValueError("bvh: non-finite object bounds")
        return out

    def range_count(self, objs, dim, preds, pred_is_box=False, cap=0, is_points=True):
        objs, preds = _f32(objs), _f32(preds)
        nq = preds.shape[0]
        counts = np.empty(nq, np.int32)
        assert self.lib.orc_range_count(objs.reshape(-1), objs.shape[0], dim, int(is_points), preds.reshape(-1), nq,
                                        int(pred_is_box), cap, counts) == 0
        return counts

    def range_crs(self, objs, dim, spheres, is_points=True):
        objs, spheres = _f32(objs), _f32(spheres)
        nq = spheres.shape[0]
        off = np.empty(nq + 1, np.int64)
        self.lib.orc_range_crs(objs.reshape(-1), objs.shape[0], dim, int(is_points), spheres.reshape(-1), nq, off,
                               None)
        vals = np.empty(int(off[-1]), np.int32)
        self.lib.orc_range_crs(objs.reshape(-1), objs.shape[0], dim, int(is_points), spheres.reshape(-1), nq, off,
                               vals.ctypes.data)
        return off, vals

    def knn(self, objs, dim, origins, k, is_points=True):
        objs, origins = _f32(objs), _f32(origins)
        nq = origins.shape[0]
        kk = max(k, 0)
        idx = np.empty(max(nq * kk, 1), np.int32)
        dist = np.empty(max(nq * kk, 1), np.float32)
        assert self.lib.orc_knn(objs.reshape(-1), objs.shape[0], dim, int(is_points), origins.reshape(-1), nq, k,
                                idx, dist) == 0
        return idx[: nq * kk].reshape(nq, kk), dist[: nq * kk].reshape(nq, kk)

    def dbscan(self, pts, dim, eps, min_pts, with_stats=False):
        pts = _f32(pts)
        n = pts.shape[0]
        labels = np.empty(max(n, 1), np.int32)
        core = np.empty(max(n, 1), np.uint8)
        stats = np.zeros(3, np.int64)
        rc = self.lib.orc_dbscan(pts.reshape(-1), n, dim, eps, min_pts, labels, core,
                                 stats.ctypes.data if with_stats else None)
        if rc:
            raise ValueError("dbscan: invalid parameters or points")
        if with_stats:
            return labels[:n], core[:n], stats
        return labels[:n], core[:n]

    def check_equivalence(self, pts, dim, eps, got, want):
        pts = _f32(pts)
        kind = C.c_int32(0)
        i = self.lib.orc_check_equivalence(pts.reshape(-1), pts.shape[0], dim, eps,
                                           np.ascontiguousarray(got[0], np.int32),
                                           np.ascontiguousarray(got[1], np.uint8),
                                           np.ascontiguousarray(want[0], np.int32),
                                           np.ascontiguousarray(want[1], np.uint8), C.byref(kind))
        return None if i < 0 else (int(i), int(kind.value))

    def distance(self, a, b, dim):
        return float(self.lib.orc_distance(_f32(a), _f32(b), dim))


class Reference:
    """The unmodified reference (oracle/_ref/libref.so), if it was built."""

    _inst = None

    @classmethod
    def available(cls) -> bool:
        return os.path.exists(REF_SO)

    @classmethod
    def get(cls) -> "Reference":
        if cls._inst is None:
            cls._inst = cls(REF_SO)
        return cls._inst

    def __init__(self, path):
        L = self.lib = C.CDLL(path)
        L.ref_generate_uniform.argtypes = [C.c_int64, C.c_int, C.c_double, C.c_uint64, _f32p]
        L.ref_generate_gaussian.argtypes = [C.c_int64, C.c_int, C.c_int32, C.c_double, C.c_double, C.c_uint64, _f32p]
        L.ref_bvh_build.argtypes = [_f32p, C.c_int64, C.c_int, C.c_int, C.c_int, _i32p, _i32p, _f32p, _i32p, _i32p,
                                    _f32p]
        L.ref_dbscan.argtypes = [_f32p, C.c_int64, C.c_int, C.c_float, C.c_int32, C.c_int, C.c_void_p, C.c_void_p,
                                 C.c_void_p, C.c_void_p]
        L.ref_range_count.argtypes = [_f32p, C.c_int64, _f32p, C.c_int64, C.c_float, C.c_int32, _i32p, C.c_void_p]
        L.ref_knn.argtypes = [_f32p, C.c_int64, _f32p, C.c_int64, C.c_int32, _i32p, C.c_void_p]

    def uniform(self, n, dim=3, extent=1.0, seed=0):
        out = np.empty(max(n * dim, 1), np.float32)
        self.lib.ref_generate_uniform(n, dim, extent, seed, out)
        return out[: n * dim].reshape(n, dim)

    def gaussian(self, n, dim, k, sigma, extent, seed):
        out = np.empty(max(n * dim, 1), np.float32)
        self.lib.ref_generate_gaussian(n, dim, k, sigma, extent, seed, out)
        return out[: n * dim].reshape(n, dim)

    def field(self, n):
        nbg = n // 4
        nh = n - nbg
        bg = self.uniform(nbg, 3, 1.0, 2409)
        halos = self.gaussian(nh, 3, max(nh // 8192, 1), 0.001 * float(np.cbrt(67108864.0 / float(n))), 1.0, 2410)
        return np.concatenate([bg, halos], axis=0)

    def bvh(self, objs, dim, width=64, is_points=True):
        objs = _f32(objs)
        n = objs.shape[0]
        m = max(n - 1, 0)
        out = dict(internal_left=np.empty(max(m, 1), np.int32), internal_rope=np.empty(max(m, 1), np.int32),
                   internal_boxes=np.empty((max(m, 1), 2 * dim), np.float32), leaf_object=np.empty(max(n, 1), np.int32),
                   leaf_rope=np.empty(max(n, 1), np.int32), leaf_boxes=np.empty((max(n, 1), 2 * dim), np.float32))
        rc = self.lib.ref_bvh_build(objs.reshape(-1), n, dim, int(is_points), width, out["internal_left"],
                                    out["internal_rope"], out["internal_boxes"].reshape(-1), out["leaf_object"],
                                    out["leaf_rope"], out["leaf_boxes"].reshape(-1))
        if rc == 1:
            raise ValueError("bvh: non-finite object bounds")
        assert rc == 0, "reference validate() failed"
        for key in ("internal_left", "internal_rope", "internal_boxes"):
            out[key] = out[key][:m]
        for key in ("leaf_object", "leaf_rope", "leaf_boxes"):
            out[key] = out[key][:n]
        return out

    def dbscan(self, pts, dim, eps, min_pts, algo="fdbscan", with_stats=False):
        code = {"fdbscan": 0, "fof": 1, "densebox": 2, "reference": 3, "adjacency": 4, "fdbscan_seq": 5,
                "densebox_seq": 6}[algo]
        pts = _f32(pts)
        n = pts.shape[0]
        labels = np.empty(max(n, 1), np.int32)
        core = np.empty(max(n, 1), np.uint8)
        stats = np.zeros(3, np.int64)
        ms = np.zeros(4, np.float64)
        rc = self.lib.ref_dbscan(pts.reshape(-1), n, dim, eps, min_pts, code, labels.ctypes.data, core.ctypes.data,
                                 stats.ctypes.data, ms.ctypes.data)
        if rc:
            raise ValueError("dbscan: invalid parameters or points")
        if with_stats:
            return labels[:n], core[:n], stats, ms
        return labels[:n], core[:n]

    def range_count(self, pts, centres, radius, cap=0):
        pts, centres = _f32(pts), _f32(centres)
        counts = np.empty(centres.shape[0], np.int32)
        ms = np.zeros(3, np.float64)
        self.lib.ref_range_count(pts.reshape(-1), pts.shape[0], centres.reshape(-1), centres.shape[0], radius, cap,
                                 counts, ms.ctypes.data)
        return counts, ms

    def knn(self, pts, origins, k):
        pts, origins = _f32(pts), _f32(origins)
        idx = np.empty(origins.shape[0] * k, np.int32)
        ms = np.zeros(2, np.float64)
        self.lib.ref_knn(pts.reshape(-1), pts.shape[0], origins.reshape(-1), origins.shape[0], k, idx, ms.ctypes.data)
        return idx.reshape(-1, k), ms
