"""CPU: the drop-in boundary — libspb200.so builds for sm_100a, loads, and
exports every entry point include/sp_b200.h declares; the package imports
without a GPU and refuses to run without one (no CPU fallback)."""
import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    text = open(os.path.join(ROOT, "include", "sp_b200.h")).read()
    return sorted(set(re.findall(r"^\s*(?:const\s+)?\w+\s*\*?\s*(sp_\w+)\s*\(", text, re.M)))


def test_header_declares_the_reference_boundary():
    syms = declared_symbols()
    for s in ("sp_bvh_build", "sp_range_count", "sp_knn", "sp_dbscan", "sp_pair_list", "sp_range_crs",
              "sp_sort_queries", "sp_bvh_export"):
        assert s in syms
    text = open(os.path.join(ROOT, "include", "sp_b200.h")).read()
    for cite in ("bvh.hpp:62", "traversal.hpp:67-87", "traversal.hpp:93-156", "dbscan.hpp:277-301"):
        assert cite in text


def test_library_exports_every_declared_symbol(sp):
    lib = ctypes.CDLL(sp.library_path())
    missing = [s for s in declared_symbols() if not hasattr(lib, s)]
    assert not missing, missing


def test_library_is_sm100a_code(sp):
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", sp.library_path()], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


def test_no_gpu_means_loud_failure(sp):
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(sp.CudaError):
        sp.Context(0)


def test_product_does_not_reference_the_oracle():
    pkg = os.path.join(ROOT, "paper_2409_10743_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".hpp", ".h", ".cpp")):
                txt = open(os.path.join(dirpath, f), errors="ignore").read()
                for banned in ("liboracle", "libref", "oracle_lib", "orc_", "ref_dbscan"):
                    assert banned not in txt, (f, banned)
