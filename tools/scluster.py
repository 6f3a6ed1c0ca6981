#!/usr/bin/env python
"""GPU counterpart of the reference's batch driver (tools/scluster.cpp).

Same flags, stdout lines, report keys and exit codes (0 ok, 1 usage, 2 I/O or
capacity, 3 verification mismatch); the clustering runs on the B200 through
libspb200.so.  --sequential selects the sequential modes (ExecMode::kSequential):
fdbscan and densebox labels then equal the reference's sequential run bit for
bit (deterministic border assignment).  --verify compares against the device brute-force
dbscan_reference with check_equivalence (both on the GPU).
"""
from __future__ import annotations

import argparse
import math
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

EXIT_USAGE, EXIT_IO, EXIT_VERIFY = 1, 2, 3


class UsageError(Exception):
    pass


def derive_eps(b: float, v: float, n: float) -> float:
    """derive_eps (report.cpp:12-16): b * cbrt(V / n)."""
    if not (b > 0 and v > 0 and n > 0):
        raise UsageError("derive_eps: all inputs must be positive")
    return b * math.cbrt(v / n)


def parse_generate(spec: str, seed: int):
    """parse_generate_spec (generate.cpp:102-130)."""
    import paper_2409_10743_b200 as sp
    if "(" not in spec or not spec.endswith(")"):
        raise UsageError("generate: spec must be name(arg,...)")
    name, args = spec[: spec.index("(")], spec[spec.index("(") + 1: -1]
    try:
        vals = [float(x.strip()) for x in args.split(",")] if args else []
    except ValueError:
        raise UsageError("generate: malformed number in %s spec" % name)
    if name == "uniform":
        if len(vals) != 3:
            raise UsageError("generate: uniform expects 3 arguments")
        return sp.generate_reference_uniform(int(vals[0]), int(vals[1]), vals[2], seed)
    if name == "gaussian_clusters":
        if len(vals) != 6:
            raise UsageError("generate: gaussian_clusters expects 6 arguments")
        return sp.generate_reference_gaussian(int(vals[0]), int(vals[1]), int(vals[2]), vals[3], vals[4],
                                              int(vals[5]))
    raise UsageError("generate: unknown generator '%s'" % name)


def morton_stats(codes: np.ndarray):
    """compute_stats (morton.hpp:133-156)."""
    if len(codes) == 0:
        return 0, 0, 0
    _, counts = np.unique(codes, return_counts=True)
    return int((counts > 3).sum()), int(counts[counts > 1].sum()), int(counts.max())


def run(opt) -> int:
    import paper_2409_10743_b200 as sp
    from paper_2409_10743_b200 import io

    if opt.format not in ("csv", "binary"):
        raise UsageError("--format must be csv or binary")
    if opt.algo not in ("fdbscan", "densebox", "fof", "legacy", "oracle"):
        raise UsageError("--algo must be one of fdbscan, densebox, fof, legacy, oracle")
    if opt.code_width not in (32, 64):
        raise UsageError("--code-width must be 32 or 64")
    if opt.minpts < 2:
        raise UsageError("--minpts must be at least 2")
    if opt.algo in ("fof", "legacy") and opt.minpts != 2:
        raise UsageError("--algo %s requires --minpts 2" % opt.algo)
    eps = opt.eps
    if opt.derive_eps:
        parts = opt.derive_eps.split(",")
        if len(parts) != 3:
            raise UsageError("--derive-eps expects b,V,n")
        try:
            eps = derive_eps(*[float(x) for x in parts])
        except ValueError:
            raise UsageError("--derive-eps expects three numbers")
    if not (eps is not None and eps > 0 and math.isfinite(eps)):
        raise UsageError("eps must resolve to a positive finite value")
    pts = parse_generate(opt.generate, opt.seed) if opt.generate else io.load_points(opt.input, opt.format)
    n, dim = pts.shape
    if opt.verify and n > opt.oracle_ceiling:
        raise UsageError("--verify is limited to %d points (got %d)" % (opt.oracle_ceiling, n))
    params = sp.DbscanParams(float(np.float32(eps)), opt.minpts)
    mode = "sequential" if opt.sequential else "parallel"
    if opt.algo == "fdbscan":
        out = sp.fdbscan(pts, params, width=opt.code_width, mode=mode)
    elif opt.algo == "densebox":
        out = sp.fdbscan_densebox(pts, params, width=opt.code_width, mode=mode)
    elif opt.algo == "fof":
        out = sp.friends_of_friends(pts, params.eps, width=opt.code_width)
    elif opt.algo == "legacy":
        out = sp.adjacency_graph_dbscan(pts, params.eps, width=opt.code_width)
    else:
        out = sp.dbscan_reference(pts, params)
    labels, core = np.asarray(out.labels), np.asarray(out.core_flags)
    clusters = int(np.unique(labels[labels >= 0]).size)
    noise, ncore = int((labels == -1).sum()), int(core.sum())
    t = out.timings
    if opt.labels_out:
        io.write_labels(opt.labels_out, labels)
    m32 = m64 = None
    if opt.morton_report:
        m32 = morton_stats(sp.morton_codes(pts, 32))
        m64 = morton_stats(sp.morton_codes(pts, 64))
    if opt.report_out:
        with open(opt.report_out, "w") as f:
            f.write("n=%d\nd=%d\neps=%.9g\nmin_pts=%d\nalgorithm=%s\ncode_width=%d\n" %
                    (n, dim, eps, opt.minpts, opt.algo, opt.code_width))
            f.write("num_clusters=%d\nnum_noise=%d\nnum_core=%d\n" % (clusters, noise, ncore))
            for k, v in (("build", t.build_ms), ("core", t.core_ms), ("merge", t.merge_ms),
                         ("finalize", t.finalize_ms), ("total", t.total_ms())):
                f.write("time_%s_ms=%.9g\n" % (k, v))
            for name, st in (("morton32", m32), ("morton64", m64)):
                if st:
                    f.write("%s_codes_duplicated_gt3=%d\n%s_points_with_duplicate_code=%d\n"
                            "%s_max_same_code_duplicates=%d\n" % (name, st[0], name, st[1], name, st[2]))
    print("n=%d d=%d eps=%.9g min_pts=%d algo=%s code_width=%d%s" %
          (n, dim, eps, opt.minpts, opt.algo, opt.code_width, " sequential" if opt.sequential else ""))
    print("clusters=%d noise=%d core=%d" % (clusters, noise, ncore))
    if opt.algo == "densebox":
        s = out.stats
        print("dense_cells=%d dense_points=%d distance_checks=%d" %
              (s.num_dense_cells, s.num_dense_points, s.distance_checks))
    print("build=%.3fms core=%.3fms merge=%.3fms finalize=%.3fms total=%.3fms" %
          (t.build_ms, t.core_ms, t.merge_ms, t.finalize_ms, t.total_ms()))
    for name, st in (("morton32", m32), ("morton64", m64)):
        if st:
            print("%s: codes_dup_gt3=%d points_with_dup=%d max_dup=%d" % (name, st[0], st[1], st[2]))
    if opt.verify:
        ref = sp.dbscan_reference(pts, params)
        bad = sp.check_equivalence(pts, params.eps, out, ref)
        if bad:
            print("verify: MISMATCH: %s" % bad)
            return EXIT_VERIFY
        print("verify: OK")
    return 0


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(description="spatial clustering benchmark driver (B200)")
    src = ap.add_mutually_exclusive_group()
    src.add_argument("--input")
    src.add_argument("--generate")
    ap.add_argument("--format", default="csv")
    ap.add_argument("--algo", default="fdbscan")
    e = ap.add_mutually_exclusive_group()
    e.add_argument("--eps", type=float)
    e.add_argument("--derive-eps")
    ap.add_argument("--minpts", type=int, default=2)
    ap.add_argument("--code-width", type=int, default=64)
    ap.add_argument("--verify", action="store_true")
    ap.add_argument("--sequential", action="store_true")
    ap.add_argument("--labels-out")
    ap.add_argument("--report-out")
    ap.add_argument("--morton-report", action="store_true")
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--oracle-ceiling", type=int, default=20000)
    try:
        opt = ap.parse_args(argv)
    except SystemExit as ex:
        return 0 if ex.code == 0 else EXIT_USAGE
    if (opt.input is None) == (opt.generate is None):
        print("exactly one of --input or --generate is required", file=sys.stderr)
        return EXIT_USAGE
    if (opt.eps is None) == (opt.derive_eps is None):
        print("exactly one of --eps or --derive-eps is required", file=sys.stderr)
        return EXIT_USAGE
    try:
        return run(opt)
    except UsageError as ex:
        print(ex, file=sys.stderr)
        return EXIT_USAGE
    except Exception as ex:  # noqa: BLE001 - map like scluster.cpp:237-251
        from paper_2409_10743_b200 import CapacityError, InvalidArgument
        from paper_2409_10743_b200.io import LoadError
        print(ex, file=sys.stderr)
        if isinstance(ex, InvalidArgument):
            return EXIT_USAGE
        if isinstance(ex, (LoadError, CapacityError)):
            return EXIT_IO
        return EXIT_IO


if __name__ == "__main__":
    sys.exit(main())
