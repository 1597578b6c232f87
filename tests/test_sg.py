"""Serialized-graph cache: the reference's .sg/.wsg
layout (io.hpp:328-456) loaded straight into HBM and written back from it.
Fixtures in tests/golden/*.sg were written by the reference's own
WriteSerialized (tests/golden/make_golden.py)."""
import os
import struct

import numpy as np
import pytest

from conftest import ROOT
from oracle import oracle as O

GOLD = os.path.join(ROOT, "tests", "golden")


def test_fixture_layout_is_the_pinned_reference_layout():
    # test_io.cc:174-203: BuildDirected({{0, 1}}) serialized byte for byte
    expected = b"GAPB" + bytes([1, 1]) + struct.pack("<QQ", 2, 1)
    expected += struct.pack("<QQQ", 0, 1, 1) + struct.pack("<I", 1)
    expected += struct.pack("<QQQ", 0, 0, 1) + struct.pack("<I", 0)
    assert open(os.path.join(GOLD, "directed_1edge.sg"), "rb").read() == expected


def _parse(path):
    b = open(path, "rb").read()
    n, m = struct.unpack_from("<QQ", b, 6)
    flags = b[5]
    off = np.frombuffer(b, np.uint64, n + 1, 22).astype(np.int64)
    nb = np.frombuffer(b, np.uint32, m, 22 + 8 * (n + 1))
    return n, m, flags, off, nb


def test_kron10_fixture_matches_oracle_build():
    n, m, flags, off, nb = _parse(os.path.join(GOLD, "kron10.sg"))
    g = O.build_csr(1 << 10, O.gen_kron(10))
    assert flags == 0 and n == g.n and m == g.m
    assert (off == g.off).all() and (nb == g.nb).all()


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["kron10.sg", "kron10.wsg", "dkron9.sg", "directed_1edge.sg"])
def test_load_matches_file(name):
    from paper_1508_03619_b200 import DeviceGraph
    path = os.path.join(GOLD, name)
    n, m, flags, off, nb = _parse(path)
    g = DeviceGraph.load_sg(path)
    assert (g.n, g.m, g.directed) == (n, m, bool(flags & 1))
    doff, dnb, dio, dinb = g.download()
    assert (doff == off).all() and (dnb == nb).all()
    if g.directed:
        b = open(path, "rb").read()
        base = 22 + 8 * (n + 1) + 4 * m + (4 * m if flags & 2 else 0)
        assert (dio == np.frombuffer(b, np.uint64, n + 1, base).astype(np.int64)).all()
        assert (dinb == np.frombuffer(b, np.uint32, m, base + 8 * (n + 1))).all()


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["kron10.sg", "dkron9.sg", "directed_1edge.sg"])
def test_save_is_byte_identical_to_reference(name, tmp_path):
    from paper_1508_03619_b200 import DeviceGraph
    g = DeviceGraph.load_sg(os.path.join(GOLD, name))
    out = tmp_path / name
    g.save_sg(str(out))
    assert out.read_bytes() == open(os.path.join(GOLD, name), "rb").read()


@pytest.mark.gpu
def test_loaded_graph_runs_bfs_with_parity(tmp_path):
    from paper_1508_03619_b200 import DeviceGraph
    g = DeviceGraph.load_sg(os.path.join(GOLD, "kron10.sg"))
    host = O.build_csr(1 << 10, O.gen_kron(10))
    for s in g.pick_sources(8):
        r = g.bfs(int(s), depth=True)
        assert (r.depth == O.bfs_depths(host, int(s))).all()
        assert O.verify_bfs(host, int(s), r.parent)[0]
    # device-generated -> .sg -> reload round trip at a larger scale
    big = DeviceGraph.generate("kron", 18)
    p = tmp_path / "kron18.sg"
    big.save_sg(str(p))
    again = DeviceGraph.load_sg(str(p))
    a, b = big.download(), again.download()
    assert (a[0] == b[0]).all() and (a[1] == b[1]).all()


@pytest.mark.gpu
def test_load_errors(tmp_path):
    from paper_1508_03619_b200 import GapkitError, LoadError, DeviceGraph
    good = open(os.path.join(GOLD, "kron10.sg"), "rb").read()
    bad_magic = tmp_path / "bad.sg"
    bad_magic.write_bytes(b"XXXX" + good[4:])
    with pytest.raises(LoadError, match="bad magic"):
        DeviceGraph.load_sg(str(bad_magic))
    bad_ver = tmp_path / "ver.sg"
    bad_ver.write_bytes(good[:4] + bytes([2]) + good[5:])
    with pytest.raises(LoadError, match="unsupported version 2"):
        DeviceGraph.load_sg(str(bad_ver))
    trunc = tmp_path / "trunc.sg"
    trunc.write_bytes(good[:-100])
    with pytest.raises(LoadError, match="shorter than its declared arrays"):
        DeviceGraph.load_sg(str(trunc))
    with pytest.raises(GapkitError, match="cannot open"):
        DeviceGraph.load_sg(str(tmp_path / "missing.sg"))
    # header past the int32 parent range: rejected before any size arithmetic
    huge = tmp_path / "huge.sg"
    huge.write_bytes(b"GAPB" + bytes([1, 0]) + struct.pack("<QQ", (1 << 31) + 1, 4) + bytes(64))
    with pytest.raises(GapkitError, match="more than 2\\^31 vertices"):
        DeviceGraph.load_sg(str(huge))
    arcs = tmp_path / "arcs.sg"
    arcs.write_bytes(b"GAPB" + bytes([1, 0]) + struct.pack("<QQ", 4, (1 << 62)) + bytes(64))
    with pytest.raises(LoadError, match="arc count out of range"):
        DeviceGraph.load_sg(str(arcs))
