"""Sharded (1D-partitioned) BFS: the host orchestrator
(paper_1508_03619_b200/dist.py) and exchange protocol.

CPU: P logical ranks in one process (LocalComm) and 2 real processes over
gloo (torchrun), both with the numpy engine, against the oracle: depths
exact, parents valid, schedule and counters equal to the reference replay.
GPU: the gk_shard_* kernels through the same orchestrator (P ranks on one
device, run sequentially -- no rank waits on another inside a kernel)."""
import os
import socket
import subprocess
import sys

import numpy as np
import pytest

from conftest import ROOT
from oracle import oracle as O

torch = pytest.importorskip("torch")

from np_engine import NpEngine  # noqa: E402
from paper_1508_03619_b200.dist import LocalComm, ShardedBfs, block_of  # noqa: E402


def check(g, res, src, strat=0, alpha=15, beta=18):
    d = O.bfs_depths(g, src)
    assert (res.depth == d).all()
    ok, msg = O.verify_bfs(g, src, res.parent)
    assert ok, msg
    rp = O.bfs_replay(g, src, alpha, beta, strat)
    assert res.schedule == rp.dirs
    assert [x[1] for x in res.steps] == rp.frontier
    assert [x[2] for x in res.steps] == rp.result
    assert [x[3] for x in res.steps] == rp.edges_to_check
    assert res.component_edges == O.component_edges(g, d)


GRAPHS = {
    "kron10p": lambda: O.make_graph("kron", 10),
    "urand10": lambda: O.make_graph("urand", 10),
    "grid30x40": lambda: O.make_graph("grid", rows=30, cols=40),
    "path8": lambda: O.build_csr(8, np.array([x for v in range(7) for x in (v, v + 1)], np.uint32)),
}


@pytest.mark.parametrize("P", [1, 2, 3, 4])
@pytest.mark.parametrize("name", list(GRAPHS))
def test_local_ranks_numpy(name, P):
    g = GRAPHS[name]()
    engines = [NpEngine(g, r, P) for r in range(P)]
    sb = ShardedBfs(engines, LocalComm(P))
    for src in O.pick_sources(g, 3):
        for strat in (0, 1, 2):
            check(g, sb.run(int(src), strategy=strat, want_depth=True, gather=True), int(src), strat)


def test_partition_blocks_are_word_aligned():
    for n in (1, 31, 32, 33, 1000, 1 << 20):
        for P in (1, 2, 3, 8):
            b = block_of(n, P)
            assert b % 32 == 0 and b * P >= n


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_two_processes_gloo():
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr=127.0.0.1", f"--master-port={_free_port()}", os.path.join(ROOT, "tests", "dist_worker.py")]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert "rank 0 ok" in r.stdout and "rank 1 ok" in r.stdout


# ------------------------------------------------------------------- GPU
def _gpu_engines(g, P):
    from paper_1508_03619_b200.dist import GpuEngine
    out = []
    for r in range(P):
        b = block_of(g.n, P)
        lo, hi = min(g.n, r * b), min(g.n, (r + 1) * b)
        out.append(GpuEngine.upload(g.n, r, P, g.off[lo:hi + 1] - g.off[lo], g.nb[g.off[lo]:g.off[hi]]))
    return out


@pytest.mark.gpu
@pytest.mark.parametrize("P", [1, 2, 4])
@pytest.mark.parametrize("name", ["kron10p", "urand10", "grid30x40", "path8"])
def test_local_ranks_gpu(name, P):
    g = GRAPHS[name]()
    sb = ShardedBfs(_gpu_engines(g, P), LocalComm(P))
    for src in O.pick_sources(g, 3):
        for strat in (0, 1, 2):
            check(g, sb.run(int(src), strategy=strat, want_depth=True, gather=True), int(src), strat)


@pytest.mark.gpu
@pytest.mark.parametrize("P", [2, 3])
def test_gpu_shard_generate_matches_single_device(P):
    from paper_1508_03619_b200 import DeviceGraph
    from paper_1508_03619_b200.dist import GpuEngine
    full = DeviceGraph.generate("kron", 16, 16, 24601, permute=True)
    off, nb, _, _ = full.download()
    g = O.Csr(full.n, off, nb)
    engines = [GpuEngine.generate("kron", 16, 16, 24601, True, r, P) for r in range(P)]
    for e in engines:
        assert e.m == int(off[e.hi] - off[e.lo])
    sb = ShardedBfs(engines, LocalComm(P))
    for src in full.pick_sources(4):
        check(g, sb.run(int(src), want_depth=True, gather=True), int(src))


@pytest.mark.gpu
def test_gpu_larger_shards():
    from paper_1508_03619_b200 import DeviceGraph
    from paper_1508_03619_b200.dist import GpuEngine
    full = DeviceGraph.generate("kron", 20, 16, 24601, permute=True)
    off, nb, _, _ = full.download()
    g = O.Csr(full.n, off, nb)
    P = 4
    sb = ShardedBfs([GpuEngine.generate("kron", 20, 16, 24601, True, r, P) for r in range(P)], LocalComm(P))
    for src in full.pick_sources(2):
        res = sb.run(int(src), want_depth=True, gather=True)
        check(g, res, int(src))


@pytest.mark.gpu
def test_gpu_shard_rejects_malformed_rows():
    from paper_1508_03619_b200 import GapkitError
    from paper_1508_03619_b200.dist import GpuEngine
    with pytest.raises(GapkitError, match="neighbour id out of range"):
        GpuEngine.upload(64, 0, 2, np.array([0, 1] + [1] * 31, np.int64), np.array([64], np.uint32))
    with pytest.raises(GapkitError, match="offsets not monotone"):
        GpuEngine.upload(64, 0, 2, np.array([0, 2, 1] + [2] * 30, np.int64), np.array([1, 2], np.uint32))
