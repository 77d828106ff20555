"""Host-side checks of the C-ABI library that need no GPU: it builds for sm_100a, loads, and
exports every symbol declared in include/rds.h; argument validation that precedes any CUDA
call returns the documented error codes."""
import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def lib():
    from paper_1807_11534_b200 import _build

    path = _build.build()
    return ctypes.CDLL(path), path


def _declared():
    src = open(os.path.join(ROOT, "include", "rds.h")).read()
    return sorted(set(re.findall(r"^\s*(?:int|const char \*)\s*(rds3?_\w+)\s*\(", src, re.M)))


def test_header_symbols_exported(lib):
    _, path = lib
    names = _declared()
    assert len(names) >= 20
    out = subprocess.run(["nm", "-D", "--defined-only", path], capture_output=True, text=True,
                         check=True).stdout
    exported = set(re.findall(r"\bT (rds3?_\w+)", out))
    missing = [n for n in names if n not in exported]
    assert not missing, missing
    from paper_1807_11534_b200 import rds

    assert sorted(rds.EXPORTS) == names


def test_sm100a_code_present(lib):
    _, path = lib
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", path],
                         capture_output=True, text=True, check=True).stdout
    assert "sm_100a" in out


def test_validation_without_gpu(lib):
    from paper_1807_11534_b200 import rds

    h = ctypes.c_void_p()
    assert rds._lib.rds_create(0, 5, ctypes.byref(h)) == rds.RDS_EINVAL
    assert "must be >= 1" in rds.rds_last_error()
    assert rds._lib.rds_create(5, -1, ctypes.byref(h)) == rds.RDS_EINVAL
    assert rds._lib.rds_create(1 << 20, 1 << 20, ctypes.byref(h)) == rds.RDS_EINVAL
    assert rds._lib.rds_create(4, 4, None) == rds.RDS_EINVAL
    assert rds._lib.rds_destroy(None) == rds.RDS_OK
    assert rds._lib.rds_solve(None, 1.0, 0.1, 0.125, 0.0, 1) == rds.RDS_EINVAL
    th, tw = rds.rds_tile_shape()
    assert (th, tw) == (32, 32)
    ks = rds.rds_kfuse_supported()
    assert 1 in ks and ks == sorted(ks)
    assert "sm_100a" in rds.rds_version()
