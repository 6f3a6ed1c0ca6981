"""The C++ façade (include/spatial_b200.hpp) compiles against the C ABI, and
(on a GPU) the reference-style unit tests in tests/cpp/test_facade.cpp pass."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "tests", "cpp", "test_facade.cpp")
OUT = os.path.join(ROOT, "tests", "cpp", "test_facade")


def build():
    import paper_2409_10743_b200 as sp
    libdir = os.path.dirname(sp.library_path())
    cmd = ["g++", "-std=c++20", "-O2", "-Wall", "-Wextra", "-I", os.path.join(ROOT, "include"), SRC, "-o", OUT,
           "-L", libdir, "-l:libspb200.so", "-Wl,-rpath," + libdir]
    subprocess.check_call(cmd)
    return OUT


def test_facade_compiles():
    assert os.path.exists(build())


@pytest.mark.gpu
def test_facade_reference_style_tests_pass():
    exe = build()
    r = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
