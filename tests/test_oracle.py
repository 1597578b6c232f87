"""CPU tests: the C restatement (oracle/) against the reference's own outputs.

Pins the checker before anything is checked with it: the committed golden
fixtures (tests/golden/golden.json, written by make_golden.py from the
unmodified reference) and -- where oracle/_ref/libgapref.so exists -- the
live reference.  Mirrors the reference's BFS tests:
test_kernels_source.cc:13-67, test_verify.cc:13-57, test_benchmark.cc:15-38,
acceptance.cc:79-116 (criterion 1) and :392-405 (criterion 7).
"""
import numpy as np
import pytest

from oracle import oracle as O

SEED = 24601


def fnv(a):
    return f"{O.fnv1a(np.ascontiguousarray(a)):016x}"


def build_case(name, ent):
    kind, n = ent["kind"], ent["n"]
    if kind == "edges":
        return None
    if kind == "kron":
        seed = 7 if name.endswith("_s7") else (11 if name.endswith("_s11") else SEED)
        scale = n.bit_length() - 1
        e = O.gen_kron(scale, 16, seed)
    elif kind == "urand":
        e = O.gen_urand(n.bit_length() - 1, 16, SEED)
    elif kind == "kronp":
        scale = n.bit_length() - 1
        e = O.permute_edges(O.gen_kron(scale, 16, SEED), scale, SEED)
    elif kind == "grid":
        r, c = (int(x) for x in name[4:].split("x"))
        e = O.gen_grid(r, c, 0.15, 0.02, SEED)
    else:
        raise ValueError(kind)
    assert fnv(e) == ent["edges_fnv"], f"{name}: generator differs from the reference"
    return O.build_csr(n, e, symmetrize=not ent["directed"], directed=ent["directed"])


def small_graph(name):
    pairs = {
        "path8": [(v, v + 1) for v in range(7)],
        "star9": [(4, v) for v in range(9) if v != 4],
        "ring16": [(v, (v + 1) % 16) for v in range(16)],
        "k5": [(u, v) for u in range(5) for v in range(u + 1, 5)],
    }[name]
    n = {"path8": 8, "star9": 9, "ring16": 16, "k5": 5}[name]
    return O.build_csr(n, np.array([x for p in pairs for x in p], np.uint32))


@pytest.fixture(scope="module")
def graphs(golden):
    out = {}
    for name, ent in golden["graphs"].items():
        g = build_case(name, ent) if ent["kind"] != "edges" else small_graph(name)
        out[name] = g
    return out


def test_generators_and_builder_match_golden(golden, graphs):
    for name, ent in golden["graphs"].items():
        g = graphs[name]
        assert g.n == ent["n"] and g.m == ent["m"], name
        assert fnv(g.off) == ent["off_fnv"], name
        assert fnv(g.nb) == ent["nb_fnv"], name
        if ent["directed"]:
            assert fnv(g.in_off) == ent["in_off_fnv"] and fnv(g.in_nb) == ent["in_nb_fnv"], name


def test_pick_sources_match_golden(golden, graphs):
    for name, ent in golden["graphs"].items():
        assert O.pick_sources(graphs[name], 64, SEED).tolist() == ent["sources"], name


def test_depths_and_schedule_match_golden(golden, graphs):
    for name, ent in golden["graphs"].items():
        g = graphs[name]
        for r in ent["runs"]:
            d = O.bfs_depths(g, r["source"])
            assert fnv(d) == r["depth_fnv"], (name, r["source"])
            rp = O.bfs_replay(g, r["source"], r["alpha"], r["beta"], r["strategy"])
            assert rp.dirs == r["dirs"], (name, r["source"], r["strategy"])
            assert rp.frontier == r["frontier"] and rp.result == r["result"], (name, r["source"])
            assert rp.edges_to_check == r["edges_to_check"], (name, r["source"])
            ok, msg = O.verify_bfs(g, r["source"], rp.parent)
            assert ok, msg
            assert ((rp.parent >= 0) == (d >= 0)).all()


def test_known_answers(golden):
    g = O.build_csr(3, np.array([0, 1, 1, 2], np.uint32))
    assert O.bfs_replay(g, 0).parent.tolist() == golden["kat"]["path3_parent"] == [0, 0, 1]
    g = O.build_csr(4, np.array([0, 1, 1, 2], np.uint32))
    assert O.bfs_replay(g, 0).parent[3] == -1
    assert golden["kat"]["isolated_parent"][3] == -1
    assert [O.permute(v, 16, SEED) for v in range(8)] == golden["kat"]["perm_scale16_first8"]


def test_config_errors():
    g = O.build_csr(3, np.array([0, 1, 1, 2], np.uint32))
    with pytest.raises(ValueError, match="source out of range"):
        O.bfs_replay(g, 17)
    with pytest.raises(ValueError, match="alpha and beta"):
        O.bfs_replay(g, 0, alpha=0)


def test_verifier_rejects_tampering():
    # test_verify.cc:13-57 and acceptance.cc:392-405
    g = O.build_csr(3, np.array([0, 1, 1, 2], np.uint32))
    good = np.array([0, 0, 1], np.int32)
    assert O.verify_bfs(g, 0, good)[0]
    bad = good.copy(); bad[2] = 0
    ok, msg = O.verify_bfs(g, 0, bad)
    assert not ok and "no edge" in msg and "2" in msg
    bad = good.copy(); bad[2] = -1
    ok, msg = O.verify_bfs(g, 0, bad)
    assert not ok and "unreached" in msg
    h = O.build_csr(3, np.array([0, 1], np.uint32))
    assert not O.verify_bfs(h, 0, np.array([0, 0, 1], np.int32))[0]
    bad = good.copy(); bad[0] = 1
    assert not O.verify_bfs(g, 0, bad)[0]
    sq = O.build_csr(4, np.array([0, 1, 1, 2, 2, 3, 3, 0], np.uint32))
    tree = O.bfs_replay(sq, 0).parent
    assert O.verify_bfs(sq, 0, tree)[0]
    bad = tree.copy(); bad[1] = 2
    ok, msg = O.verify_bfs(sq, 0, bad)
    assert not ok and "depth" in msg


def test_picker_edge_cases():
    # test_benchmark.cc:15-38
    e = np.array([7, 8], np.uint32)
    g = O.build_csr(9, e, symmetrize=False, directed=True)
    assert O.pick_sources(g, 20, 123).tolist() == [7] * 20
    empty = O.build_csr(4, np.zeros(0, np.uint32))
    with pytest.raises(ValueError, match="no edges"):
        O.pick_sources(empty, 1)


def test_permutation_is_bijection():
    for scale in (1, 2, 5, 10, 16):
        keys = O.perm_keys(SEED, scale)
        import ctypes as C
        k = (C.c_uint64 * 8)(*[int(x) for x in keys])
        img = {O.lib().gko_permute(v, scale, k) for v in range(1 << scale)}
        assert img == set(range(1 << scale)), scale


def test_grid_generator_shape():
    g = O.make_graph("grid", rows=200, cols=300)
    deg = g.degree()
    base = 2 * 200 * 299 + 2 * 199 * 300
    # 15% deleted, ~2% diagonals: mean degree ~ (0.85*base + 2*0.02*199*300)/n
    expect = (0.85 * base + 2 * 0.02 * 199 * 300) / g.n
    assert abs(deg.mean() - expect) < 0.05
    assert deg.max() <= 6


def test_byte_model_small():
    # hand-checkable: path 0-1-2, source 0, all top-down
    g = O.build_csr(3, np.array([0, 1, 1, 2], np.uint32))
    rp = O.bfs_replay(g, 0, strategy=O.GKO_TD_ONLY)
    d = O.bfs_depths(g, 0)
    bs, bu = O.byte_model(g, d, rp.dirs)
    # 4n + TD0: (36+32)+36*1 + TD1: (36+32)+36*1 + TD2: (36+32)+0
    assert rp.dirs == "TTT"
    assert bs == 12 + (68 + 36) + (68 + 36) + 68
    assert bu == 12 + (12 + 4 + 4) + (12 + 8 + 4) + (12 + 4)


@pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")
def test_oracle_matches_live_reference():
    R = O.RefLib()
    for kind, scale in (("kron", 11), ("urand", 11)):
        e = O.gen_kron(scale) if kind == "kron" else O.gen_urand(scale)
        assert (e == R.gen(kind, scale)).all()
        g = O.build_csr(1 << scale, e)
        rg = R.wrap(g, check=True)
        for s in O.pick_sources(g, 8):
            s = int(s)
            assert (O.bfs_depths(g, s) == rg.depths(s)).all()
            ref = rg.schedule(s)
            rp = O.bfs_replay(g, s)
            assert (ref.dirs, ref.frontier, ref.result) == (rp.dirs, rp.frontier, rp.result)
            # bottom-up parents are deterministic: identical to the reference's
            d = O.bfs_depths(g, s)
            for i, c in enumerate(rp.dirs):
                if c == "B":
                    sel = d == i + 1
                    assert (rp.parent[sel] == ref.parent[sel]).all()


@pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")
def test_reference_arm_builder_matches_buildcsr():
    """ref_bench.cc's 64-bit OpenMP builder (the reference arm's, for graphs
    past BuildCsr's 2^32-arc limit, builder.hpp:71-73) is byte-identical to
    the reference's BuildCsr(el, false, true) where both run, and its
    bench-configuration graphs equal the restated generator + builder."""
    R = O.RefLib()
    for kind, scale in (("kron", 14), ("urand", 13)):
        e = R.gen(kind, scale, 16, SEED)
        a = R.build(1 << scale, e).csr()
        b = R.build64(1 << scale, e).csr()
        assert (a.off == b.off).all() and (a.nb == b.nb).all(), kind
    # with self-loops and duplicates in the input
    e = np.array([0, 0, 1, 2, 2, 1, 1, 2, 3, 3, 4, 0, 0, 4], np.uint32)
    a, b = R.build(6, e).csr(), R.build64(6, e).csr()
    assert (a.off == b.off).all() and (a.nb == b.nb).all()
    for kind, scale, permute in (("kron", 15, True), ("urand", 12, False)):
        g = R.bench_graph(kind, scale, 16, SEED, permute=permute).csr()
        h = O.make_graph(kind, scale, 16, SEED, permute=permute)
        assert (g.off == h.off).all() and (g.nb == h.nb).all(), kind
    g = R.bench_graph("grid", rows=40, cols=50).csr()
    h = O.make_graph("grid", rows=40, cols=50)
    assert (g.off == h.off).all() and (g.nb == h.nb).all()
    rg = R.bench_graph("kron", 12, 16, SEED, permute=True)
    src = rg.pick_sources(4, SEED)
    secs, mcc = rg.trials(src)
    assert (secs > 0).all()
    for s, m in zip(src, mcc):
        assert m == rg.component_edges(rg.bfs(int(s)))
