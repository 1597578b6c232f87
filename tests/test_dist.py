"""Sharded (1D-partitioned) BFS: one persistent kernel per
rank, exchanges through peer memory, no host round trip per level
(csrc/gk_bfs_sharded.cu, paper_1508_03619_b200/dist.py).

CPU: the phase-for-phase model of the kernel (tests/shard_model.py) with P
ranks in one process and with 2 processes over gloo (torchrun), against the
oracle: exact depths, parents = first in-neighbour (ascending) one level up,
the reference's schedule and counters.
GPU: the kernel itself with P ranks emulated on one device (one cooperative
launch, cpr CTAs per rank -- ranks that wait on one another must not be
separate launches on one GPU): the same checks, parents valid (top-down
claimers store racy valid parents, as on one device)."""
import os
import socket
import subprocess
import sys

import numpy as np
import pytest

from conftest import ROOT
from oracle import oracle as O

import shard_model as M  # noqa: E402
from paper_1508_03619_b200.dist import block_of  # noqa: E402


def check(g, parent, depth, steps, src, strat=0, alpha=15, beta=18, min_parents=True):
    d = O.bfs_depths(g, src)
    assert (depth == d).all(), np.flatnonzero(depth != d)[:8]
    ok, msg = O.verify_bfs(g, src, parent)
    assert ok, msg
    if min_parents:  # the model resolves every parent as the first in-neighbour one level up
        assert (parent == M.min_parents(g, d)).all()
    rp = O.bfs_replay(g, src, alpha, beta, strat)
    assert "".join(s[0] for s in steps) == rp.dirs
    assert [s[1] for s in steps] == rp.frontier
    assert [s[2] for s in steps] == rp.result
    assert [s[3] for s in steps] == rp.edges_to_check


GRAPHS = {
    "kron10p": lambda: O.make_graph("kron", 10),
    "urand10": lambda: O.make_graph("urand", 10),
    "grid30x40": lambda: O.make_graph("grid", rows=30, cols=40),
    "path8": lambda: O.build_csr(8, np.array([x for v in range(7) for x in (v, v + 1)], np.uint32)),
}


@pytest.mark.parametrize("P", [1, 2, 3])
@pytest.mark.parametrize("name", list(GRAPHS))
def test_model_local_ranks(name, P):
    g = GRAPHS[name]()
    ranks = [M.Rank(g, r, P) for r in range(P)]
    for src in O.pick_sources(g, 2):
        for strat in (0, 1, 2):
            parent, depth, steps = M.run(ranks, M.LocalComm(), int(src), strategy=strat)
            check(g, np.concatenate(parent), np.concatenate(depth), steps, int(src), strat)


def test_partition_blocks_are_task_aligned():
    for n in (1, 31, 1024, 1025, 1 << 20, (1 << 27) + 5):
        for P in (1, 2, 3, 8):
            b = block_of(n, P)
            assert b % 1024 == 0 and b * P >= n


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_two_processes_gloo():
    pytest.importorskip("torch")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr=127.0.0.1", f"--master-port={_free_port()}", os.path.join(ROOT, "tests", "dist_worker.py")]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert "rank 0 ok" in r.stdout and "rank 1 ok" in r.stdout


# ------------------------------------------------------------------- GPU
@pytest.mark.gpu
@pytest.mark.parametrize("P", [1, 2, 4])
@pytest.mark.parametrize("name", list(GRAPHS))
def test_gpu_local_group(name, P):
    from paper_1508_03619_b200.dist import ShardGroup
    g = GRAPHS[name]()
    grp = ShardGroup.from_csr(g, P)
    for src in O.pick_sources(g, 3):
        for strat in (0, 1, 2):
            r = grp.run(int(src), strategy=strat, depth=True, counts=True)
            check(g, r.parent, r.depth, r.steps, int(src), strat, min_parents=False)
            assert r.component_edges == O.component_edges(g, r.depth)
            assert len(r.bytes_in) == P and (P == 1 or sum(r.bytes_in) > 0)


@pytest.mark.gpu
@pytest.mark.parametrize("P", [2, 3, 8])
def test_gpu_group_generate_matches_single_device(P):
    from paper_1508_03619_b200 import DeviceGraph
    from paper_1508_03619_b200.dist import ShardGroup, pick_sources
    full = DeviceGraph.generate("kron", 16, 16, 24601, permute=True)
    off, nb, _, _ = full.download()
    g = O.Csr(full.n, off, nb)
    grp = ShardGroup.generate("kron", 16, 16, 24601, True, P)
    for sh in grp.shards:
        assert sh.m == int(off[sh.hi] - off[sh.lo])
    deg = np.diff(off)
    srcs = pick_sources(lambda v: deg[v], g.n, 4)
    assert srcs == [int(s) for s in full.pick_sources(4)]
    for src in srcs:
        r = grp.run(src, depth=True)
        check(g, r.parent, r.depth, r.steps, src, min_parents=False)


@pytest.mark.gpu
def test_gpu_larger_group():
    from paper_1508_03619_b200 import DeviceGraph
    from paper_1508_03619_b200.dist import ShardGroup
    full = DeviceGraph.generate("kron", 20, 16, 24601, permute=True)
    off, nb, _, _ = full.download()
    g = O.Csr(full.n, off, nb)
    grp = ShardGroup.generate("kron", 20, 16, 24601, True, 4)
    for src in full.pick_sources(2):
        single = full.bfs(int(src), depth=True)
        r = grp.run(int(src), depth=True)
        assert (r.depth == single.depth).all() and r.schedule == single.schedule
        check(g, r.parent, r.depth, r.steps, int(src), min_parents=False)


@pytest.mark.gpu
def test_gpu_cross_device_protocol_one_rank(monkeypatch):
    """The multi-device path (gk_shard_export / connect / gather_dead /
    gk_shard_bfs) with its cross-rank barrier and counter reduction forced
    on for one rank (GK_SHARD_FORCE_X): several traversals in a row (the
    barrier count carries across them), exact depths, valid parents, the
    reference schedule."""
    monkeypatch.setenv("GK_SHARD_FORCE_X", "1")
    from paper_1508_03619_b200.dist import ShardedBfs, _Shard
    for name in ("kron10p", "grid30x40"):
        g = GRAPHS[name]()
        sb = ShardedBfs(_Shard.upload(g.n, 0, 1, g.off, g.nb), 1, allgather=lambda b: [b], barrier=lambda: None)
        for src in O.pick_sources(g, 4):
            for strat in (0, 1, 2):
                r = sb.run(int(src), strategy=strat, depth=True, counts=True)
                check(g, r.parent, r.depth, r.steps, int(src), strat, min_parents=False)
                assert r.reached == int((r.depth >= 0).sum()) and r.bytes_in == [0]


@pytest.mark.gpu
def test_gpu_shard_rejects_malformed_rows():
    from paper_1508_03619_b200 import GapkitError
    from paper_1508_03619_b200.dist import _Shard
    with pytest.raises(GapkitError, match="invalid shard rows"):
        _Shard.upload(2048, 0, 2, np.array([0, 1] + [1] * 1023, np.int64), np.array([4096], np.uint32))
