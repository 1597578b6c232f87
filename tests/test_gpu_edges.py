"""Edge cases of the device traversal's data-layout shortcuts against the
oracle: the never-reachable (dead) seed of visited, the per-vertex head
records of the bottom-up sweep, tiny-step claims, large-step bitmap claims
and their target-range passes, ragged vertex counts around bitmap words.

Bar as in test_gpu_bfs.py: depths bit-exact, parents valid (VerifyBfs
semantics), schedule and per-step counters equal to the reference's replay,
bottom-up parents equal to the reference's first-hit choice."""
import os

import numpy as np
import pytest

from oracle import oracle as O
from paper_1508_03619_b200 import Brandes, BfsStrategy, DeviceGraph

pytestmark = pytest.mark.gpu


def check(g, dg, s, alpha=15, beta=18, strategy=0):
    res = dg.bfs(int(s), alpha, beta, strategy, depth=True, counts=True)
    assert (res.depth == O.bfs_depths(g, int(s))).all()
    ok, msg = O.verify_bfs(g, int(s), res.parent)
    assert ok, msg
    rp = O.bfs_replay(g, int(s), alpha, beta, strategy)
    assert res.schedule == rp.dirs
    assert [x[2] for x in res.steps] == rp.result
    for i, c in enumerate(res.schedule):
        if c == "B" and res.steps[i][4] != "P":  # a pushed bottom-up step picks any valid parent
            sel = res.depth == i + 1
            assert (res.parent[sel] == rp.parent[sel]).all(), ("bottom-up parent", i)
    return res


@pytest.mark.parametrize("n", [1, 2, 31, 32, 33, 63, 65, 1000, 1025])
def test_ragged_vertex_counts(n, both_kernels):
    rng = np.random.default_rng(n)
    m = 3 * n
    e = rng.integers(0, n, size=2 * m, dtype=np.uint64).astype(np.uint32)
    g = O.build_csr(n, e)
    dg = DeviceGraph.from_csr(g)
    for s in {0, n - 1, n // 2}:
        for st in BfsStrategy:
            for a, b in ((15, 18), (1, 1)):
                check(g, dg, s, a, b, int(st))


def test_heavy_hub_small_graph(both_kernels):
    # one vertex of degree 6000 (> the 1024-edge chunk), plus a sparse ring:
    # heavy chunks, a large (bitmap) top-down step and head/list rounds
    n = 6001
    e = [x for v in range(1, n) for x in (0, v)] + [x for v in range(1, n - 1) for x in (v, v + 1)]
    g = O.build_csr(n, np.array(e, np.uint32))
    dg = DeviceGraph.from_csr(g)
    for s in (0, 1, 3000, n - 1):
        for a, b in ((15, 18), (1000, 1), (1, 1000)):
            check(g, dg, s, a, b)


def test_isolated_source_and_dead_vertices(both_kernels):
    # vertices 5..9 have no edges at all; BFS from one of them reaches only it
    e = np.array([0, 1, 1, 2, 2, 3, 3, 4], np.uint32)
    g = O.build_csr(10, e)
    dg = DeviceGraph.from_csr(g)
    r = dg.bfs(7, depth=True)
    assert r.parent.tolist() == [-1] * 7 + [7] + [-1] * 2
    assert r.depth.tolist() == [-1] * 7 + [0] + [-1] * 2
    check(g, dg, 0, 1, 1)


def test_directed_source_without_in_edges(both_kernels):
    # vertex 0 only has out-edges: it is "dead" for the bottom-up sweep but a
    # valid source; vertex 4 has in-edges only
    e = np.array([0, 1, 0, 2, 1, 3, 2, 3, 3, 4, 1, 4], np.uint32)
    g = O.build_csr(5, e, symmetrize=False, directed=True)
    dg = DeviceGraph.from_csr(g)
    for a, b in ((1, 1), (15, 18)):
        r = check(g, dg, 0, a, b)
        assert r.parent[0] == 0
    r = dg.bfs(4, depth=True)
    assert r.parent.tolist() == [-1, -1, -1, -1, 4]


@pytest.mark.parametrize("passes", ["2", "3", "7"])
def test_large_step_range_passes(passes, monkeypatch, grid_kernel):
    # GK_TD_PASSES forces the target-range passes of large top-down steps
    # that kick in by themselves only when the next bitmap exceeds 64 MB
    monkeypatch.setenv("GK_TD_PASSES", passes)
    g = O.make_graph("kron", 16, permute=True)
    dg = DeviceGraph.from_csr(g)
    for s in O.pick_sources(g, 6, 5):
        check(g, dg, int(s))
    gu = O.make_graph("urand", 15)
    dgu = DeviceGraph.from_csr(gu)
    for s in O.pick_sources(gu, 3, 5):
        check(gu, dgu, int(s))


def test_handle_state_across_kernels(both_kernels):
    # BFS, Brandes, BFS again on one handle: per-call state is re-initialised
    g = O.make_graph("kron", 12, permute=True)
    dg = DeviceGraph.from_csr(g)
    srcs = [int(s) for s in O.pick_sources(g, 3)]
    first = [dg.bfs(s, depth=True).depth.copy() for s in srcs]
    sc = Brandes(dg, srcs)
    assert np.abs(sc - O.brandes(g, srcs)).max() <= 1e-5
    for s, d in zip(srcs, first):
        r = check(g, dg, s)
        assert (r.depth == d).all()


def test_batch_matches_single_calls(both_kernels):
    # gk_bfs_batch: per-source results identical in depth, all parents valid,
    # copies overlapped with the next traversal
    from paper_1508_03619_b200 import ConfigError, PinnedBuffer
    g = O.make_graph("kron", 14, permute=True)
    dg = DeviceGraph.from_csr(g)
    srcs = [int(s) for s in O.pick_sources(g, 7)]
    outs = [np.empty(g.n, np.int32) for _ in srcs]
    ms = dg.bfs_batch(srcs, outs)
    assert ms.shape == (7,) and (ms > 0).all()
    for s, p in zip(srcs, outs):
        ok, msg = O.verify_bfs(g, s, p)
        assert ok, msg
    # repeated pinned buffers (the bench's use): the last result lands last
    pins = [PinnedBuffer(g.n), PinnedBuffer(g.n)]
    dg.bfs_batch(srcs, [pins[i & 1].array for i in range(len(srcs))])
    assert O.verify_bfs(g, srcs[-1], pins[0].array)[0] and O.verify_bfs(g, srcs[-2], pins[1].array)[0]
    # the handle's device parent is the last traversal's
    r = dg.bfs(srcs[0])
    assert O.verify_bfs(g, srcs[0], r.parent)[0]
    with pytest.raises(ConfigError, match="bfs source out of range"):
        dg.bfs_batch([0, g.n])
    assert dg.bfs_batch([]).size == 0


def _device_parent(dg, n):
    from cuda.bindings import runtime as rt
    out = np.empty(n, np.int32)
    err, = rt.cudaMemcpy(out.ctypes.data, dg.device_parent_ptr(), 4 * n, rt.cudaMemcpyKind.cudaMemcpyDeviceToHost)
    assert int(err) == 0
    return out


def _sparse_upload(n, m, seed):
    # mostly isolated vertices: a small reached set, so the result travels compact
    rng = np.random.default_rng(seed)
    e = rng.integers(0, n, size=2 * m, dtype=np.uint64).astype(np.uint32)
    g = O.build_csr(n, e)
    return g, DeviceGraph.from_csr(g)


@pytest.mark.parametrize("n", [1 << 22, (1 << 22) + 77])
def test_batch_compact_transfer(n):
    # gk_bfs_batch from 2^22 vertices ships each ParentArray compact (reached
    # bitmap + packed parents) and expands it on the host: every output must
    # equal the device result bit for bit, ragged last block included, and
    # the bytes moved must be the compact size
    from paper_1508_03619_b200 import PinnedBuffer
    g, dg = _sparse_upload(n, n, n)
    srcs = [int(s) for s in O.pick_sources(g, 5)]
    nblk = (n + 1023) // 1024
    for s in srcs:
        out = np.full(n, 7, np.int32)
        dg.bfs_batch([s], [out])
        ref = _device_parent(dg, n)
        assert (out == ref).all()
        ok, msg = O.verify_bfs(g, s, out)
        assert ok, msg
        total, packed = dg.batch_d2h_bytes()
        reached = int((ref >= 0).sum())
        # compact part (offsets, bitmap, packed parents) + the raw head blocks
        assert packed == 1 and 4 * (nblk + 1 + 32 * nblk) <= total <= 4 * (nblk + 1 + 32 * nblk + reached) + 4 * n // 4
    # several sources, repeated pinned outputs (the bench's use) and pageable ones
    pins = [PinnedBuffer(n), PinnedBuffer(n)]
    dg.bfs_batch(srcs, [pins[i & 1].array for i in range(len(srcs))])
    assert (pins[(len(srcs) - 1) & 1].array == _device_parent(dg, n)).all()
    assert O.verify_bfs(g, srcs[-2], pins[(len(srcs) - 2) & 1].array)[0]
    outs = [np.empty(n, np.int32) for _ in srcs]
    dg.bfs_batch(srcs, outs)
    for s, p in zip(srcs, outs):
        ok, msg = O.verify_bfs(g, s, p)
        assert ok, msg
    assert dg.batch_d2h_bytes()[1] == len(srcs)
    # every output the same array: the last source's result lands last
    same = np.empty(n, np.int32)
    dg.bfs_batch(srcs, [same] * len(srcs))
    assert (same == _device_parent(dg, n)).all()


def test_batch_raw_when_compact_is_larger():
    # a source reaching (nearly) every vertex gains nothing from the compact
    # form: it travels raw (n int32), GK_BATCH_PACK-independent results
    g = O.make_graph("urand", 22)
    dg = DeviceGraph.from_csr(g)
    srcs = [int(s) for s in O.pick_sources(g, 2)]
    outs = [np.empty(g.n, np.int32) for _ in srcs]
    dg.bfs_batch(srcs, outs)
    assert dg.batch_d2h_bytes() == (4 * g.n * len(srcs), 0)
    for s, p in zip(srcs, outs):
        ok, msg = O.verify_bfs(g, s, p)
        assert ok, msg


def test_malformed_csr_rejected():
    # every kernel indexes with off/nb: a malformed CSR is refused at creation
    from paper_1508_03619_b200 import GapkitError
    with pytest.raises(GapkitError, match="neighbour id out of range"):
        DeviceGraph.upload(3, np.array([0, 1, 2, 2], np.int64), np.array([1, 7], np.uint32))
    with pytest.raises(GapkitError, match="offsets not monotone"):
        DeviceGraph.upload(3, np.array([0, 2, 1, 2], np.int64), np.array([1, 0], np.uint32))
    with pytest.raises(GapkitError, match="offsets not monotone"):
        DeviceGraph.upload(2, np.array([1, 1, 2], np.int64), np.array([1, 0], np.uint32))
    # directed: the in-CSR is checked too
    with pytest.raises(GapkitError, match="neighbour id out of range"):
        DeviceGraph.upload(2, np.array([0, 1, 1], np.int64), np.array([1], np.uint32), directed=True,
                           in_offsets=np.array([0, 0, 1], np.int64), in_neighbors=np.array([5], np.uint32))
    ok = DeviceGraph.upload(3, np.array([0, 1, 2, 2], np.int64), np.array([1, 0], np.uint32))
    assert ok.bfs(0).parent.tolist() == [0, 0, -1]


@pytest.mark.parametrize("dmin", ["1", "40", "300"])
def test_owned_range_hub_expansion(dmin, monkeypatch, grid_kernel):
    # GK_OWN_DMIN makes small graphs' hubs take the owned-range expansion of
    # large top-down steps (td_own) that kron scale >= 21 uses by itself;
    # GK_NO_FRONT_SMEM keeps the bitmaps in global memory as at that size
    monkeypatch.setenv("GK_NO_FRONT_SMEM", "1")
    monkeypatch.setenv("GK_OWN_DMIN", dmin)
    seen = set()
    for kind, scale in (("kron", 16), ("urand", 14)):
        g = O.make_graph(kind, scale, permute=kind == "kron")
        dg = DeviceGraph.from_csr(g)
        for s in O.pick_sources(g, 6, 7):
            for a, b in ((15, 18), (2, 2)):
                check(g, dg, int(s), a, b)
                seen |= {t[0] for t in dg.trace()}
    assert "O" in seen  # the owned-range phase ran
    for n in (33, 1000, 1025):
        rng = np.random.default_rng(n)
        e = rng.integers(0, n, size=6 * n, dtype=np.uint64).astype(np.uint32)
        g = O.build_csr(n, e)
        dg = DeviceGraph.from_csr(g)
        for s in {0, n - 1}:
            check(g, dg, s, 1, 1)
            check(g, dg, s)


@pytest.mark.parametrize("no_head2", ["0", "1"])
def test_bottom_up_rounds_with_and_without_second_head(no_head2, monkeypatch, grid_kernel):
    # the second head record (in-neighbours 4..7) replaces the first in_nb
    # round; without it (GK_NO_HEAD2) round 2 reads in_off/in_nb as before.
    # Lists of every length around the 4/8 boundaries, bottom-up parents
    # must equal the reference's first hit.
    if no_head2 == "1":
        monkeypatch.setenv("GK_NO_HEAD2", "1")
    rng = np.random.default_rng(11)
    n = 3000
    deg = rng.integers(0, 14, size=n)
    e = np.array([x for v in range(n) for w in rng.integers(0, n, size=deg[v]) for x in (v, w)], np.uint32)
    g = O.build_csr(n, e)
    dg = DeviceGraph.from_csr(g)
    for s in O.pick_sources(g, 5, 3):
        for a, b in ((1000, 1000), (15, 18), (1, 1)):
            check(g, dg, int(s), a, b)
    gu = O.make_graph("urand", 14)
    dgu = DeviceGraph.from_csr(gu)
    for s in O.pick_sources(gu, 3, 5):
        check(gu, dgu, int(s))


def test_rescan_strategy_on_fresh_handle(both_kernels):
    # kTopDownRescan re-reads each new frontier's queue (bfs.hpp:161-167):
    # its large steps must write that queue even when no earlier traversal
    # on the handle left the same entries behind
    g = O.make_graph("kron", 16, permute=True)
    for s in O.pick_sources(g, 3, 9):
        dg = DeviceGraph.from_csr(g)
        check(g, dg, int(s), strategy=int(BfsStrategy.kTopDownRescan))


def test_sparse_sweeps_and_pulled_top_down(monkeypatch, grid_kernel):
    # Once few vertices are unreached, bottom-up steps scan a list of them
    # and a top-down step whose frontier outnumbers them runs as a pull
    # ('P' in the trace): same claimed set and counters as the reference's
    # top-down step (schedule and results equal the replay), bottom-up
    # parents still the reference's first hit.  Directed graphs pull over
    # in-edges and sum out-degrees.
    monkeypatch.setenv("GK_NO_FRONT_SMEM", "1")
    seen = set()
    graphs = [O.make_graph("kron", 16, permute=True), O.make_graph("urand", 15)]
    n = 4000
    rng = np.random.default_rng(5)
    e = rng.integers(0, n, size=2 * 8 * n, dtype=np.uint64).astype(np.uint32)
    graphs.append(O.build_csr(n, e, symmetrize=False, directed=True))
    for g in graphs:
        dg = DeviceGraph.from_csr(g)
        for s in O.pick_sources(g, 6, 13):
            check(g, dg, int(s))
            seen |= {t[0] for t in dg.trace()}
    assert "P" in seen


def test_pushed_bottom_up_step(monkeypatch, grid_kernel):
    # A bottom-up step entered with a frontier whose out-degree total is small
    # against the pending vertices runs as a push ('P' in the step log): the
    # same claimed set and awake count as the reference's bottom-up step, so
    # the schedule and every counter still equal the replay; parents valid.
    monkeypatch.setenv("GK_NO_FRONT_SMEM", "1")
    seen = set()
    g = O.make_graph("kron", 16, permute=True)
    dg = DeviceGraph.from_csr(g)
    for s in O.pick_sources(g, 8, 21):
        for a, b in ((15, 18), (2, 18), (60, 18)):  # small alpha: early switches from small frontiers
            res = check(g, dg, int(s), a, b)
            seen |= {st[4] for st in res.steps}
    assert "P" in seen
