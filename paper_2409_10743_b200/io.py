"""Point-set files and label output (io.cpp:69-152, io.hpp:15-57).

ABXPTS01 binary: 8-byte magic "ABXPTS01", u32 dim, u64 count, then count*dim
little-endian fp32 values; CSV: one point per line, 2 or 3 comma-separated
coordinates.  Errors raise LoadError with the reference's messages; non-finite
coordinates are rejected at load time like the reference does.
"""
from __future__ import annotations

import numpy as np

MAGIC = b"ABXPTS01"


class LoadError(RuntimeError):
    """spatial::io::LoadError."""


def load_points(path: str, fmt: str = "csv") -> np.ndarray:
    return load_csv(path) if fmt == "csv" else load_binary(path)


def load_binary(path: str) -> np.ndarray:
    try:
        f = open(path, "rb")
    except OSError:
        raise LoadError(path + ": cannot open")
    with f:
        head = f.read(8)
        if head != MAGIC:
            raise LoadError(path + ": bad magic at byte 0")
        d = f.read(4)
        if len(d) < 4:
            raise LoadError(path + ": truncated header at byte 8")
        c = f.read(8)
        if len(c) < 8:
            raise LoadError(path + ": truncated header at byte 12")
        dim = int(np.frombuffer(d, "<u4")[0])
        count = int(np.frombuffer(c, "<u8")[0])
        if dim not in (2, 3):
            raise LoadError("%s: dimension %d out of range at byte 8" % (path, dim))
        payload = f.read(count * dim * 4)
    vals = np.frombuffer(payload, "<f4")
    if vals.size != count * dim:
        raise LoadError("%s: truncated payload at byte %d" % (path, 20 + len(payload)))
    bad = ~np.isfinite(vals)
    if bad.any():
        raise LoadError("%s: non-finite value at byte %d" % (path, 20 + 4 * int(np.argmax(bad))))
    return vals.reshape(count, dim).astype(np.float32)


def load_csv(path: str) -> np.ndarray:
    try:
        f = open(path)
    except OSError:
        raise LoadError(path + ": cannot open")
    rows, dim = [], 0
    with f:
        for no, line in enumerate(f, 1):
            line = line.rstrip("\n").rstrip("\r")
            if not line:
                continue
            vals = []
            for field in line.split(","):
                try:
                    v = np.float32(float(field.strip(" \t")))
                except ValueError:
                    raise LoadError("%s: malformed value at line %d" % (path, no))
                if not np.isfinite(v):
                    raise LoadError("%s: non-finite value at line %d" % (path, no))
                vals.append(v)
            if dim == 0:
                if len(vals) not in (2, 3):
                    raise LoadError("%s: line 1 has %d coordinates; only 2- and 3-dimensional data is supported"
                                    % (path, len(vals)))
                dim = len(vals)
            elif len(vals) != dim:
                raise LoadError("%s: line %d has %d coordinates, expected %d" % (path, no, len(vals), dim))
            rows.append(vals)
    return np.asarray(rows, np.float32).reshape(-1, dim or 3)


def save_points(path: str, points: np.ndarray, fmt: str = "csv") -> None:
    pts = np.ascontiguousarray(points, np.float32)
    if fmt == "csv":
        with open(path, "w") as f:
            for p in pts:
                f.write(",".join("%.9g" % float(v) for v in p) + "\n")
        return
    with open(path, "wb") as f:
        f.write(MAGIC)
        f.write(np.uint32(pts.shape[1]).tobytes())
        f.write(np.uint64(pts.shape[0]).tobytes())
        f.write(pts.astype("<f4").tobytes())


def write_labels(path: str, labels) -> None:
    """One label per line, -1 for noise (io.cpp:144-152)."""
    with open(path, "w") as f:
        f.write("".join("%d\n" % int(v) for v in np.asarray(labels)))
