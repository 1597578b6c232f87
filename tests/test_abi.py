"""CPU tests of the C-ABI boundary: libgk_bfs.so loads, exports every symbol
include/gk_bfs.h declares, and refuses to compute without a device (there is
no CPU fallback).  No compute call needs a GPU here."""
import ctypes as C
import os
import re
import subprocess

import pytest

from conftest import HAS_GPU, ROOT

HDR = os.path.join(ROOT, "include", "gk_bfs.h")
LIB = os.path.join(ROOT, "paper_1508_03619_b200", "lib", "libgk_bfs.so")


@pytest.fixture(scope="module")
def lib():
    if not os.path.exists(LIB):
        subprocess.run(["make", "-C", ROOT, "lib"], check=True, capture_output=True)
    from paper_1508_03619_b200 import _lib
    return _lib.load()


def declared():
    txt = open(HDR).read()
    return sorted(set(re.findall(r"GK_API[^;(]*?\b(gk_\w+)\s*\(", txt)))


def test_header_declares_entry_points():
    names = declared()
    assert "gk_bfs" in names and "gk_graph_upload" in names and len(names) >= 14


def test_library_exports_every_declared_symbol(lib):
    out = subprocess.run(["nm", "-D", "--defined-only", LIB], capture_output=True, text=True).stdout
    exported = set(re.findall(r"\sT\s(gk_\w+)", out))
    missing = [n for n in declared() if n not in exported]
    assert not missing, missing
    for n in declared():
        assert hasattr(lib, n)


def test_python_binding_covers_header(lib):
    from paper_1508_03619_b200 import _lib
    assert set(_lib.EXPORTED) == set(declared())


def test_library_is_sm100a_only():
    out = subprocess.run(["cuobjdump", "--list-elf", LIB], capture_output=True, text=True).stdout
    arches = set(re.findall(r"sm_\d+a?", out))
    assert arches == {"sm_100a"}, arches


def test_abi_version(lib):
    assert lib.gk_abi_version() == 1


@pytest.mark.skipif(HAS_GPU, reason="checks the no-device path")
def test_no_cpu_fallback(lib):
    from paper_1508_03619_b200 import DeviceGraph, GapkitError
    assert lib.gk_device_count() == 0
    h = C.c_void_p()
    st = lib.gk_graph_generate(0, 10, 16, 24601, 1, 0, C.byref(h))
    assert st == 6  # GK_ERR_NO_DEVICE
    assert b"no CUDA device" in lib.gk_last_error()
    with pytest.raises(GapkitError, match="no CUDA device"):
        DeviceGraph.generate("kron", 10)


def test_null_arguments_are_errors_not_crashes(lib):
    assert lib.gk_graph_upload(None, 0, None) == 7  # GK_ERR_INVALID
    assert lib.gk_graph_info(None, None, None, None) == 7
    assert lib.gk_bfs(None, 0, 15, 18, 0, None, None, None) == 7


def test_vertex_count_limit_checked_before_any_device_work(lib):
    # parents are int32: more than 2^31 vertices is refused (no device needed)
    import ctypes as C
    from paper_1508_03619_b200._lib import CsrView
    off = (C.c_int64 * 2)(0, 0)
    v = CsrView((1 << 31) + 1, 0, 0, C.cast(off, C.c_void_p), None, None, None)
    h = C.c_void_p()
    assert lib.gk_graph_upload(C.byref(v), 0, C.byref(h)) == 7
    assert b"2^31" in lib.gk_last_error()
