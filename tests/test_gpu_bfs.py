"""GPU parity tests: the CUDA path (through the C ABI) against the oracle.

Bar (north_star): per-vertex depth bit-exact; every parent valid as
VerifyBfs checks it (verify.hpp:62-98); plus schedule parity -- the
direction sequence and per-step counters equal the reference's
(gkr_bfs_schedule / golden.json), and bottom-up parents equal the
reference's deterministic choice (bfs.hpp:55-60).
"""
import numpy as np
import pytest

from oracle import oracle as O
from paper_1508_03619_b200 import Bfs, BfsOptions, BfsStrategy, ConfigError, DeviceGraph

from test_oracle import build_case, small_graph

pytestmark = pytest.mark.gpu
SEED = 24601


def fnv(a):
    return f"{O.fnv1a(np.ascontiguousarray(a)):016x}"


@pytest.fixture(scope="module")
def hosts(golden):
    out = {}
    for name, ent in golden["graphs"].items():
        out[name] = build_case(name, ent) if ent["kind"] != "edges" else small_graph(name)
    return out


@pytest.fixture(scope="module")
def devs(hosts):
    return {name: DeviceGraph.from_csr(g) for name, g in hosts.items()}


def test_upload_roundtrip(hosts, devs):
    for name, g in hosts.items():
        off, nb, io, inb = devs[name].download()
        assert (off == g.off).all() and (nb == g.nb).all(), name
        if g.directed:
            assert (io == g.in_off).all() and (inb == g.in_nb).all()


@pytest.mark.parametrize("name,make", [
    ("kron10", lambda: DeviceGraph.generate("kron", 10, 16, SEED, permute=False)),
    ("urand10", lambda: DeviceGraph.generate("urand", 10, 16, SEED)),
    ("kron12_s7", lambda: DeviceGraph.generate("kron", 12, 16, 7, permute=False)),
    ("urand14", lambda: DeviceGraph.generate("urand", 14, 16, SEED)),
    ("kron16p", lambda: DeviceGraph.generate("kron", 16, 16, SEED, permute=True)),
    ("grid60x70", lambda: DeviceGraph.grid(60, 70, 0.15, 0.02, SEED)),
])
def test_device_generator_matches_reference(golden, name, make):
    ent = golden["graphs"][name]
    g = make()
    off, nb, _, _ = g.download()
    assert g.n == ent["n"] and g.m == ent["m"]
    assert fnv(off) == ent["off_fnv"] and fnv(nb) == ent["nb_fnv"]


def test_device_generator_larger_scales():
    for kind, scale, perm in (("kron", 18, True), ("urand", 17, False), ("kron", 17, False)):
        g = DeviceGraph.generate(kind, scale, 16, SEED, permute=perm)
        e = O.gen_kron(scale) if kind == "kron" else O.gen_urand(scale)
        if perm:
            e = O.permute_edges(e, scale, SEED)
        h = O.build_csr(1 << scale, e)
        off, nb, _, _ = g.download()
        assert (off == h.off).all() and (nb == h.nb).all(), (kind, scale)
    g = DeviceGraph.grid(300, 257, 0.15, 0.02, 99)
    h = O.make_graph("grid", rows=300, cols=257, seed=99)
    off, nb, _, _ = g.download()
    assert (off == h.off).all() and (nb == h.nb).all()


def test_pick_sources(golden, devs):
    for name, ent in golden["graphs"].items():
        assert devs[name].pick_sources(64, SEED).tolist() == ent["sources"], name


def test_bfs_parity_against_reference(golden, hosts, devs, both_kernels):
    """Every golden run: depths, parents, schedule and counters."""
    for name, ent in golden["graphs"].items():
        g, dg = hosts[name], devs[name]
        for r in ent["runs"]:
            s = r["source"]
            res = dg.bfs(s, r["alpha"], r["beta"], r["strategy"], depth=True, counts=True)
            key = (name, s, r["strategy"])
            assert fnv(res.depth) == r["depth_fnv"], key
            ok, msg = O.verify_bfs(g, s, res.parent)
            assert ok, (key, msg)
            assert res.schedule == r["dirs"], (key, res.schedule, r["dirs"])
            assert [x[1] for x in res.steps] == r["frontier"], key
            assert [x[2] for x in res.steps] == r["result"], key
            assert [x[3] for x in res.steps] == r["edges_to_check"], key
            assert res.reached == r["reached"], key
            rp = O.bfs_replay(g, s, r["alpha"], r["beta"], r["strategy"])
            for i, c in enumerate(res.schedule):
                if c == "B" and res.steps[i][4] != "P":  # pushed bottom-up steps pick any valid parent
                    sel = res.depth == i + 1
                    assert (res.parent[sel] == rp.parent[sel]).all(), (key, "bottom-up parent", i)


def test_known_answers(both_kernels):
    # test_kernels_source.cc:13-29
    path = DeviceGraph.from_csr(O.build_csr(3, np.array([0, 1, 1, 2], np.uint32)))
    assert Bfs(path, 0).tolist() == [0, 0, 1]
    iso = DeviceGraph.from_csr(O.build_csr(4, np.array([0, 1, 1, 2], np.uint32)))
    assert Bfs(iso, 0)[3] == -1
    with pytest.raises(ConfigError, match="bfs source out of range"):
        Bfs(path, 17)
    with pytest.raises(ConfigError, match="bfs alpha and beta must be positive"):
        Bfs(path, 0, BfsOptions(alpha=0))
    with pytest.raises(ConfigError, match="bfs alpha and beta must be positive"):
        Bfs(path, 0, BfsOptions(beta=-1))


def test_single_vertex_and_edgeless(both_kernels):
    one = DeviceGraph.upload(1, np.zeros(2, np.int64), np.zeros(0, np.uint32))
    assert Bfs(one, 0).tolist() == [0]
    none = DeviceGraph.upload(5, np.zeros(6, np.int64), np.zeros(0, np.uint32))
    assert Bfs(none, 3).tolist() == [-1, -1, -1, 3, -1]
    with pytest.raises(ConfigError, match="no edges"):
        none.pick_sources(1)


def test_strategies_agree(hosts, devs, both_kernels):
    # test_kernels_source.cc:42-53 on a larger graph
    g, dg = hosts["kron16p"], devs["kron16p"]
    for s in O.pick_sources(g, 6, 3):
        d = O.bfs_depths(g, int(s))
        for st in BfsStrategy:
            res = dg.bfs(int(s), strategy=int(st), depth=True)
            assert (res.depth == d).all(), st
            assert O.verify_bfs(g, int(s), res.parent)[0], st
            rp = O.bfs_replay(g, int(s), strategy=int(st))
            assert res.schedule == rp.dirs and [x[2] for x in res.steps] == rp.result


def test_directed_bottom_up_uses_in_edges(both_kernels):
    # test_kernels_source.cc:55-67 (alpha = beta = 1)
    e = O.gen_kron(12, 16, 11)
    g = O.build_csr(1 << 12, e, symmetrize=False, directed=True)
    dg = DeviceGraph.from_csr(g)
    seen_b = False
    for s in O.pick_sources(g, 16):
        s = int(s)
        for a, b in ((1, 1), (2, 1), (15, 18)):
            res = dg.bfs(s, a, b, depth=True)
            assert (res.depth == O.bfs_depths(g, s)).all()
            assert O.verify_bfs(g, s, res.parent)[0]
            rp = O.bfs_replay(g, s, a, b)
            assert res.schedule == rp.dirs and [x[2] for x in res.steps] == rp.result
            seen_b |= "B" in res.schedule
    assert seen_b


def test_launch_count(devs, both_kernels):
    """gk_bfs_launches counts one launch per traversal that never leaves its
    kernel (kron: no chain of tiny levels; the small-graph kernel is one
    launch by construction)."""
    dg = devs["kron16p"]
    l0 = dg.launches()
    srcs = [int(s) for s in dg.pick_sources(3, SEED)]
    for s in srcs:
        dg.bfs(s, parent=False)
    assert dg.launches() - l0 == 3
    dg.bfs_batch(srcs)
    assert dg.launches() - l0 == 6


def test_graph_untouched_and_repeatable(hosts, devs):
    # test_kernels_source.cc:69-85 + acceptance criterion 3 (determinism)
    g, dg = hosts["kron16p"], devs["kron16p"]
    s = int(O.pick_sources(g, 1)[0])
    a = dg.bfs(s, depth=True)
    b = dg.bfs(s, depth=True)
    off, nb, _, _ = dg.download()
    assert (off == g.off).all() and (nb == g.nb).all()
    assert (a.depth == b.depth).all() and a.steps == b.steps


def test_byte_model_matches_oracle(hosts, devs):
    for name in ("kron16p", "urand14", "grid60x70", "kron12_s7"):
        g, dg = hosts[name], devs[name]
        for s in O.pick_sources(g, 3):
            s = int(s)
            res = dg.bfs(s, depth=True)
            bs, bu = dg.byte_model(res.steps)
            obs, obu = O.byte_model(g, res.depth, res.schedule)
            assert bs == obs and bu == obu, (name, s)


def test_component_edges(hosts, devs):
    g, dg = hosts["kron16p"], devs["kron16p"]
    for s in O.pick_sources(g, 4):
        res = dg.bfs(int(s), counts=True, depth=True)
        assert res.component_edges == O.component_edges(g, res.depth)


def _check_bfs_properties(off, nb, src, depth, parent):
    """Size-independent certificate that depth is the exact BFS distance and
    parent a valid BFS tree: d(src)=0; every reached v != src has an edge
    (parent, v) with d(parent) = d(v)-1; every arc joins two reached or two
    unreached vertices and changes depth by at most 1."""
    n = off.size - 1
    reached = depth >= 0
    assert depth[src] == 0 and parent[src] == src
    assert ((parent >= 0) == reached).all()
    src_of = np.repeat(np.arange(n, dtype=np.int64), np.diff(off))
    du, dw = depth[src_of], depth[nb]
    assert (reached[src_of] == reached[nb]).all()
    both = reached[src_of]
    assert (np.abs(du[both].astype(np.int64) - dw[both]) <= 1).all()
    v = np.nonzero(reached)[0]
    v = v[v != src]
    p = parent[v].astype(np.int64)
    assert (depth[p] == depth[v] - 1).all()
    key = src_of * n + nb.astype(np.int64)  # CSR order is sorted by (u, w)
    q = p * n + v
    pos = np.searchsorted(key, q)
    assert (pos < key.size).all() and (key[np.minimum(pos, key.size - 1)] == q).all()


def test_small_graph_kernel_selected(devs, both_kernels):
    """Graphs with n <= 2^17 run in the single-cluster kernel (every step
    tagged 'S'); GK_NO_SMALL=1 sends them to the grid kernel."""
    dg = devs["kron16p"]
    for s in dg.pick_sources(3, SEED):
        pads = {x[4] for x in dg.bfs(int(s), parent=False).steps}
        assert pads == {"S"} if both_kernels == "small" else "S" not in pads


@pytest.mark.parametrize("kind,scale,perm", [("kron", 17, True), ("urand", 17, False), ("kron", 18, True)])
def test_small_kernel_size_limit(kind, scale, perm, both_kernels):
    """At the small kernel's limit (2^17 vertices: 256 bitmap words per CTA
    of a 16-CTA cluster) and just past it (2^18: grid kernel): depths,
    parents, schedule, counters and bottom-up parents against the oracle."""
    g = O.make_graph(kind, scale, permute=perm)
    dg = DeviceGraph.from_csr(g)
    for s in O.pick_sources(g, 4, 3):
        s = int(s)
        for st in (0, 1, 2):
            res = dg.bfs(s, strategy=st, depth=True, counts=True)
            assert (res.depth == O.bfs_depths(g, s)).all(), (s, st)
            assert O.verify_bfs(g, s, res.parent)[0], (s, st)
            rp = O.bfs_replay(g, s, strategy=st)
            assert res.schedule == rp.dirs and [x[2] for x in res.steps] == rp.result, (s, st)
            assert [x[3] for x in res.steps] == rp.edges_to_check, (s, st)
            for i, c in enumerate(res.schedule):
                if c == "B" and res.steps[i][4] != "P":
                    sel = res.depth == i + 1
                    assert (res.parent[sel] == rp.parent[sel]).all(), (s, st, i)
            if scale > 17:
                assert "S" not in {x[4] for x in res.steps}


@pytest.mark.parametrize("kind,scale", [("kron", 21), ("urand", 20)])
def test_medium_scale_against_oracle(kind, scale):
    dg = DeviceGraph.generate(kind, scale, 16, SEED)
    off, nb, _, _ = dg.download()
    g = O.Csr(dg.n, off, nb)
    for s in dg.pick_sources(4, SEED):
        s = int(s)
        res = dg.bfs(s, depth=True)
        assert (res.depth == O.bfs_depths(g, s)).all()
        assert O.verify_bfs(g, s, res.parent)[0]
        rp = O.bfs_replay(g, s)
        assert res.schedule == rp.dirs and [x[2] for x in res.steps] == rp.result


def test_large_scale_properties():
    dg = DeviceGraph.generate("kron", 23, 16, SEED)
    off, nb, _, _ = dg.download()
    for s in dg.pick_sources(2, SEED):
        s = int(s)
        res = dg.bfs(s, depth=True, counts=True)
        _check_bfs_properties(off, nb, s, res.depth, res.parent)
        assert res.reached == int((res.depth >= 0).sum())


def test_grid_high_diameter():
    dg = DeviceGraph.grid(700, 650, 0.15, 0.02, SEED)
    off, nb, _, _ = dg.download()
    g = O.Csr(dg.n, off, nb)
    for s in dg.pick_sources(2, SEED):
        s = int(s)
        res = dg.bfs(s, depth=True)
        assert (res.depth == O.bfs_depths(g, s)).all()
        assert O.verify_bfs(g, s, res.parent)[0]
        assert res.schedule == O.bfs_replay(g, s).dirs


@pytest.fixture(scope="module")
def chain_graphs():
    """High-diameter graphs whose traversals are long chains of tiny
    top-down levels (the cluster kernel's domain): a road-like grid and a
    path with a few branches."""
    out = {}
    h = O.make_graph("grid", rows=300, cols=257, seed=99)
    out["grid300x257"] = (h, DeviceGraph.from_csr(h))
    n = 6000
    e = [(i, i + 1) for i in range(n - 1)] + [(i, (i * 7919) % n) for i in range(0, n, 97)]
    p = O.build_csr(n, np.array(e, np.uint32).reshape(-1))
    out["path6000"] = (p, DeviceGraph.from_csr(p))
    return out


@pytest.mark.parametrize("strategy", [0, 1, 2])
def test_cluster_mode_parity(chain_graphs, strategy, grid_kernel):
    """Chains of tiny top-down levels run in the cluster kernel (steps tagged
    'K', gk_bfs_cluster.cu) and hand back to the grid kernel: depths exact,
    parents valid, schedule and every step counter equal the reference's."""
    for name, (g, dg) in chain_graphs.items():
        seen_k = False
        for s in O.pick_sources(g, 3, 5):
            s = int(s)
            l0 = dg.launches()
            res = dg.bfs(s, strategy=strategy, depth=True, counts=True)
            nl = dg.launches() - l0
            key = (name, s, strategy)
            assert (res.depth == O.bfs_depths(g, s)).all(), key
            assert O.verify_bfs(g, s, res.parent)[0], key
            rp = O.bfs_replay(g, s, strategy=strategy)
            assert res.schedule == rp.dirs, key
            assert [x[1] for x in res.steps] == rp.frontier, key
            assert [x[2] for x in res.steps] == rp.result, key
            assert [x[3] for x in res.steps] == rp.edges_to_check, key
            assert res.reached == int((res.depth >= 0).sum()), key
            k = any(x[4] == "K" for x in res.steps)
            assert nl >= (2 if k else 1), (key, nl)  # grid kernel + cluster kernel (+ resumptions)
            seen_k |= k
        assert seen_k, name  # the cluster kernel ran


@pytest.mark.parametrize("strategy", [0, 1, 2])
def test_chains_in_small_kernel(chain_graphs, strategy, both_kernels):
    """The same long chains of tiny levels through the single-cluster kernel
    (thousands of redundant levels without a cluster barrier, then the way
    back to cluster-wide levels) and through the grid kernel: depths,
    parents, schedule and counters against the oracle."""
    for name, (g, dg) in chain_graphs.items():
        for s in O.pick_sources(g, 2, 7):
            s = int(s)
            res = dg.bfs(s, strategy=strategy, depth=True, counts=True)
            key = (name, s, strategy, both_kernels)
            assert (res.depth == O.bfs_depths(g, s)).all(), key
            assert O.verify_bfs(g, s, res.parent)[0], key
            rp = O.bfs_replay(g, s, strategy=strategy)
            assert res.schedule == rp.dirs, key
            assert [x[2] for x in res.steps] == rp.result, key
            assert [x[3] for x in res.steps] == rp.edges_to_check, key
            if both_kernels == "small":
                assert {x[4] for x in res.steps} == {"S"}, key


def test_cluster_mode_batch(chain_graphs, grid_kernel):
    """gk_bfs_batch on a sparse graph checks for hand-offs after each trial:
    every parent array valid and equal-depth to the single-source call."""
    g, dg = chain_graphs["grid300x257"]
    srcs = [int(s) for s in O.pick_sources(g, 4, 9)]
    outs = [np.empty(g.n, np.int32) for _ in srcs]
    ms = dg.bfs_batch(srcs, outs)
    assert (ms > 0).all()
    for s, par in zip(srcs, outs):
        assert O.verify_bfs(g, s, par)[0], s


# ---------------------------------------------------------------- certificate
def _cuda_memcpy_h2d(dst_ptr, arr):
    """Tamper with a device array (test only) through the system CUDA runtime."""
    import ctypes
    import glob
    libs = glob.glob("/usr/local/cuda/lib64/libcudart.so*")
    rt = ctypes.CDLL(sorted(libs)[0])
    rt.cudaMemcpy.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int]
    assert rt.cudaMemcpy(dst_ptr, arr.ctypes.data, arr.nbytes, 1) == 0  # cudaMemcpyHostToDevice


def test_device_certificate_accepts(hosts, devs):
    for name in ("kron16p", "urand14", "grid60x70", "dkron10_s11", "star9", "path8"):
        g, dg = hosts[name], devs[name]
        dg.keep_depth(True)
        for s in O.pick_sources(g, 4):
            dg.bfs(int(s), parent=False)
            v = dg.verify(int(s))
            assert v["ok"], (name, s, v)
        dg.keep_depth(False)


def test_device_certificate_rejects_tampering():
    # acceptance.cc:392-405 / test_verify.cc:13-57 on the device checker
    g = O.build_csr(4, np.array([0, 1, 1, 2, 2, 3, 3, 0], np.uint32))  # square 0-1-2-3-0
    dg = DeviceGraph.from_csr(g)
    dg.keep_depth(True)
    dg.bfs(0, parent=False)
    assert dg.verify(0)["ok"]
    ptr = dg.device_parent_ptr()
    good = dg.bfs(0).parent.copy()
    for idx, val, slot in ((2, 0, 4), (1, 2, 3), (0, 1, 0), (2, -1, 1)):  # no edge / depth / source / unreached
        dg.bfs(0, parent=False)
        bad = good.copy()
        bad[idx] = val
        _cuda_memcpy_h2d(ptr, bad)
        v = dg.verify(0)
        assert not v["ok"], (idx, val)
    iso = DeviceGraph.from_csr(O.build_csr(3, np.array([0, 1], np.uint32)))
    iso.keep_depth(True)
    iso.bfs(0, parent=False)
    _cuda_memcpy_h2d(iso.device_parent_ptr(), np.array([0, 0, 1], np.int32))
    v = iso.verify(0)
    assert not v["ok"] and v["errors"][1] == 1 and v["first_bad"] == 2


def test_device_certificate_rejects_fake_root_directed():
    """Directed graph 0->1, 2->3 from source 0: vertex 3 claimed at depth 0
    with the unreached 2 as parent (depth[2] = -1 = 0 - 1) and no arc that
    leaves a reached vertex toward it -- accepted before the certificate
    required depth >= 1 off the source."""
    g = O.build_csr(4, np.array([0, 1, 2, 3], np.uint32), symmetrize=False, directed=True)
    dg = DeviceGraph.from_csr(g)
    dg.keep_depth(True)
    good = dg.bfs(0).parent.copy()
    assert dg.verify(0)["ok"]
    assert list(good) == [0, 0, -1, -1]
    bad_p = good.copy()
    bad_p[3] = 2
    bad_d = np.array([0, 1, -1, 0], np.int32)
    _cuda_memcpy_h2d(dg.device_parent_ptr(), bad_p)
    _cuda_memcpy_h2d(dg.device_depth_ptr(), bad_d)
    v = dg.verify(0)
    assert not v["ok"] and v["errors"][3] == 1 and v["first_bad"] == 3, v


@pytest.mark.parametrize("cfg", ["kron27", "urand27", "grid4900"])
def test_full_size_configs_certificate(cfg):
    """BASELINE configs 2-4 at full size: the size-independent certificate
    for several picked sources + schedule sanity."""
    if cfg == "grid4900":
        dg = DeviceGraph.grid(4900, 4900, 0.15, 0.02, SEED)
        nsrc = 2
    else:
        dg = DeviceGraph.generate(cfg[:-2], 27, 16, SEED)
        nsrc = 4
    dg.keep_depth(True)
    for s in dg.pick_sources(nsrc, SEED):
        r = dg.bfs(int(s), parent=False, counts=True)
        v = dg.verify(int(s))
        assert v["ok"], (cfg, s, v)
        assert r.reached > 0 and r.component_edges > 0
        if cfg != "grid4900":
            assert "B" in r.schedule
