"""CPU test of the host half of gk_bfs_batch's compact result transfer:
gk_expand.cpp (linked into libgk_bfs.so) against a direct restatement, built
from the object `make lib` leaves in build/ (tests/cpp/test_expand.cc)."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_expand_parents(tmp_path):
    obj = os.path.join(ROOT, "build", "gk_expand.o")
    if not os.path.exists(obj):
        pytest.skip("build/gk_expand.o missing: run make lib")
    exe = tmp_path / "test_expand"
    subprocess.run(["g++", "-O2", "-std=c++17", "-pthread", "-o", str(exe),
                    os.path.join(ROOT, "tests", "cpp", "test_expand.cc"), obj], check=True)
    out = subprocess.run([str(exe)], capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stdout + out.stderr
    lines = out.stdout.strip().splitlines()
    assert len(lines) == 24 and all(l.endswith("bad 0") for l in lines)
