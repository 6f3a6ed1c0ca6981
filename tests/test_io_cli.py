"""Host plumbing of the path: ABXPTS01/CSV files, the
reference generators (bit-identical), derive_eps, and the scluster-compatible
CLI (tools/scluster.py) — the KATs of proj/tests/test_io_cli.cpp."""
import os
import subprocess
import sys

import numpy as np
import pytest

from fixtures import generator_hashes
from oracle_lib import fnv1a64

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CLI = [sys.executable, os.path.join(ROOT, "tools", "scluster.py")]


def run_cli(args, cwd=None):
    r = subprocess.run(CLI + args, capture_output=True, text=True, timeout=600, cwd=cwd)
    return r.returncode, r.stdout, r.stderr


def parse_report(path):
    kv = {}
    for line in open(path):
        k, v = line.rstrip("\n").split("=", 1)
        kv[k] = v
    return kv


def test_reference_generators_bit_identical(sp):
    g = generator_hashes()
    assert fnv1a64(sp.generate_reference_uniform(1000, 3, 1.0, 2409)) == g["U(1000,3,2409)"]
    assert fnv1a64(sp.generate_reference_uniform(1000, 2, 1.0, 7)) == g["U(1000,2,7)"]
    assert fnv1a64(sp.generate_reference_gaussian(5000, 3, 7, 0.01, 1.0, 5)) == g["G(5000,3,7,0.01,1,5)"]


def test_binary_and_csv_round_trip(tmp_path):
    from paper_2409_10743_b200 import io
    rng = np.random.default_rng(1)
    for dim in (2, 3):
        p = rng.random((257, dim), dtype=np.float32)
        io.save_points(str(tmp_path / "p.bin"), p, "binary")
        assert np.array_equal(io.load_points(str(tmp_path / "p.bin"), "binary"), p)
        io.save_points(str(tmp_path / "p.csv"), p, "csv")
        assert np.array_equal(io.load_points(str(tmp_path / "p.csv"), "csv"), p)


def test_file_errors(tmp_path):
    # io.cpp:69-102 / test_io_cli.cpp:71-131
    from paper_2409_10743_b200 import io
    (tmp_path / "bad.bin").write_bytes(b"NOTMAGIC" + b"\0" * 12)
    with pytest.raises(io.LoadError, match="bad magic"):
        io.load_points(str(tmp_path / "bad.bin"), "binary")
    (tmp_path / "short.bin").write_bytes(b"ABXPTS01\x03\0\0\0")
    with pytest.raises(io.LoadError, match="truncated header"):
        io.load_points(str(tmp_path / "short.bin"), "binary")
    (tmp_path / "dim.bin").write_bytes(b"ABXPTS01" + np.uint32(4).tobytes() + np.uint64(0).tobytes())
    with pytest.raises(io.LoadError, match="dimension 4"):
        io.load_points(str(tmp_path / "dim.bin"), "binary")
    (tmp_path / "trunc.bin").write_bytes(b"ABXPTS01" + np.uint32(3).tobytes() + np.uint64(2).tobytes() + b"\0" * 8)
    with pytest.raises(io.LoadError, match="truncated payload"):
        io.load_points(str(tmp_path / "trunc.bin"), "binary")
    (tmp_path / "nan.csv").write_text("0,0\nnan,1\n")
    with pytest.raises(io.LoadError, match="non-finite value at line 2"):
        io.load_points(str(tmp_path / "nan.csv"), "csv")
    (tmp_path / "mix.csv").write_text("0,0\n1,2,3\n")
    with pytest.raises(io.LoadError, match="line 2 has 3 coordinates, expected 2"):
        io.load_points(str(tmp_path / "mix.csv"), "csv")


def test_derive_eps():
    sys.path.insert(0, os.path.join(ROOT, "tools"))
    import scluster
    assert abs(scluster.derive_eps(0.168, 256.0 ** 3, 1024.0 ** 3) - 0.042) < 1e-12
    assert abs(scluster.derive_eps(0.2, 1000.0, 1000.0) - 0.2) < 1e-12
    with pytest.raises(scluster.UsageError):
        scluster.derive_eps(0.0, 1.0, 1.0)


def test_cli_usage_errors():
    # scluster.cpp:143-186, 226-233: exit code 1 before any device work
    assert run_cli(["--generate", "uniform(10,3,1)"])[0] == 1                       # no eps
    assert run_cli(["--eps", "1"])[0] == 1                                           # no input
    assert run_cli(["--generate", "uniform(10,3,1)", "--eps", "1", "--algo", "x"])[0] == 1
    assert run_cli(["--generate", "uniform(10,3,1)", "--eps", "1", "--algo", "fof", "--minpts", "3"])[0] == 1
    assert run_cli(["--generate", "uniform(10,3,1)", "--eps", "-1"])[0] == 1
    assert run_cli(["--generate", "bogus(1)", "--eps", "1"])[0] == 1


@pytest.mark.gpu
def test_cli_blobs_every_algorithm(tmp_path):
    # test_io_cli.cpp:226-249
    reports = {}
    for algo in ("fdbscan", "densebox", "fof", "legacy", "oracle"):
        rp = str(tmp_path / ("r_%s.txt" % algo))
        rc, out, err = run_cli(["--generate", "gaussian_clusters(200,3,2,0.001,100,42)", "--eps", "1", "--minpts", "2",
                                "--algo", algo, "--report-out", rp])
        assert rc == 0, out + err
        kv = parse_report(rp)
        assert kv["num_clusters"] == "2" and kv["num_noise"] == "0" and kv["n"] == "200"
        reports[algo] = kv
    for algo, kv in reports.items():
        assert kv["num_core"] == reports["fdbscan"]["num_core"]


@pytest.mark.gpu
def test_cli_verify_labels_and_binary(tmp_path):
    # test_io_cli.cpp:251-259, 314-322 and the 32-bit/binary case
    rc, out, err = run_cli(["--generate", "gaussian_clusters(5000,3,5,0.01,1,3)", "--eps", "0.01", "--minpts", "4",
                            "--verify"])
    assert rc == 0 and "verify: OK" in out, out + err
    csv = tmp_path / "pts.csv"
    csv.write_text("0,0\n0.05,0\n0.1,0\n5,5\n")
    lab = tmp_path / "labels.txt"
    rc, out, err = run_cli(["--input", str(csv), "--format", "csv", "--eps", "0.06", "--minpts", "2",
                            "--labels-out", str(lab)])
    assert rc == 0, out + err
    assert [int(x) for x in lab.read_text().split()] == [0, 0, 0, -1]
    from paper_2409_10743_b200 import io
    rng = np.random.default_rng(55)
    io.save_points(str(tmp_path / "p.bin"), rng.random((500, 3), dtype=np.float32), "binary")
    rc, out, err = run_cli(["--input", str(tmp_path / "p.bin"), "--format", "binary", "--eps", "0.05",
                            "--code-width", "32", "--verify"])
    assert rc == 0 and "verify: OK" in out, out + err
    rp = str(tmp_path / "m.txt")
    rc, out, err = run_cli(["--generate", "gaussian_clusters(10000,3,4,0.0001,1,8)", "--eps", "0.01",
                            "--morton-report", "--report-out", rp])
    kv = parse_report(rp)
    assert int(kv["morton64_points_with_duplicate_code"]) < int(kv["morton32_points_with_duplicate_code"])
