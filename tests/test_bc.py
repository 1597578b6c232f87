"""Brandes betweenness: the CUDA forward/backward pass
(gk_brandes) against the reference's scores.

The reference's Brandes (proj/include/gapkit/kernels/betweenness.hpp:84-145)
sums floating point; path counts are integers and exact in double, and the
per-vertex dependency sums run in a different order on the device for
vertices of degree > 32, so scores are compared within 1e-5 absolute
(normalised scores lie in [0, 1]); the reference's own VerifyBetweenness
tolerance is 1e-4 (verify.hpp:216-219).  Golden scores come from the
unmodified reference (tests/golden/make_golden.py); the CPU tests pin the C
restatement (oracle/gk_oracle.c gko_brandes) to them.
"""
import numpy as np
import pytest

from oracle import oracle as O

TOL = 1e-5
SEED = 24601


def bc_graph(name, ent):
    if name == "star5":
        return O.build_csr(5, np.array([x for v in range(4) for x in (4, v)], np.uint32))
    if name == "path2":
        return O.build_csr(2, np.array([0, 1], np.uint32))
    kind, scale, seed = {"kron10": ("kron", 10, SEED), "urand10": ("urand", 10, SEED),
                         "dkron9_s13": ("kron", 9, 13)}[name]
    e = O.gen_kron(scale, 16, seed) if kind == "kron" else O.gen_urand(scale, 16, seed)
    if ent["directed"]:
        return O.build_csr(1 << scale, e, symmetrize=False, directed=True)
    return O.build_csr(1 << scale, e)


def test_oracle_matches_reference_scores(golden):
    for name, ent in golden["bc"].items():
        g = bc_graph(name, ent)
        sc = O.brandes(g, ent["sources"])
        assert np.array_equal(sc, np.array(ent["scores"], np.float32)), name


def test_oracle_known_answers_and_errors():
    # test_kernels_source.cc:136-158
    star = O.build_csr(5, np.array([x for v in range(4) for x in (4, v)], np.uint32))
    sc = O.brandes(star, [0, 1, 2, 3, 4])
    assert sc[4] == pytest.approx(1.0) and np.all(sc[:4] == 0)
    assert np.all(O.brandes(O.build_csr(2, np.array([0, 1], np.uint32)), [0]) == 0)
    g = O.build_csr(3, np.array([0, 1], np.uint32))
    with pytest.raises(ValueError, match="requires at least one source"):
        O.brandes(g, [])
    with pytest.raises(ValueError, match="zero out-degree"):
        O.brandes(g, [2])
    with pytest.raises(ValueError, match="out of range"):
        O.brandes(g, [7])


@pytest.mark.skipif(not O.ref_available(), reason="needs oracle/_ref (reference compiled here)")
def test_oracle_passes_reference_verifier():
    R = O.RefLib()
    for kind in ("kron", "urand"):
        rg = R.build(1 << 12, R.gen(kind, 12, 16, 5))
        srcs = rg.pick_sources(8, SEED)
        ok, msg = rg.verify_bc(srcs, O.brandes(rg.csr(), srcs))
        assert ok, msg


@pytest.mark.gpu
def test_device_matches_reference_scores(golden):
    from paper_1508_03619_b200 import Brandes, DeviceGraph
    for name, ent in golden["bc"].items():
        g = bc_graph(name, ent)
        dg = DeviceGraph.from_csr(g)
        sc = Brandes(dg, ent["sources"])
        ref = np.array(ent["scores"], np.float32)
        assert sc.dtype == np.float32 and sc.shape == ref.shape
        assert np.abs(sc - ref).max() <= TOL, (name, np.abs(sc - ref).max())
        assert sc.min() >= 0 and sc.max() <= 1


@pytest.mark.gpu
def test_device_errors_follow_reference():
    from paper_1508_03619_b200 import Brandes, ConfigError, DeviceGraph
    dg = DeviceGraph.from_csr(O.build_csr(3, np.array([0, 1], np.uint32)))
    with pytest.raises(ConfigError, match="betweenness requires at least one source"):
        Brandes(dg, [])
    with pytest.raises(ConfigError, match="betweenness source out of range"):
        Brandes(dg, [3])
    with pytest.raises(ConfigError, match="betweenness source has zero out-degree"):
        Brandes(dg, [2])
    # the handle still works after the errors, and BFS after Brandes is clean
    assert np.all(Brandes(dg, [0]) == 0)
    r = dg.bfs(0, depth=True)
    assert r.parent.tolist() == [0, 0, -1] and r.depth.tolist() == [0, 1, -1]


@pytest.mark.gpu
@pytest.mark.parametrize("kind,scale,nsrc", [("kron", 14, 8), ("urand", 13, 8), ("kronp", 16, 4)])
def test_device_matches_oracle_larger(kind, scale, nsrc):
    from paper_1508_03619_b200 import Brandes, DeviceGraph
    if kind == "kronp":
        dg = DeviceGraph.generate("kron", scale, 16, SEED, permute=True)
        g = O.make_graph("kron", scale, permute=True)
    else:
        dg = DeviceGraph.generate(kind, scale, 16, SEED, permute=False)
        g = O.make_graph(kind, scale, permute=False)
    srcs = [int(s) for s in dg.pick_sources(nsrc, SEED)]
    sc = Brandes(dg, srcs)
    ref = O.brandes(g, srcs)
    assert np.abs(sc - ref).max() <= TOL, np.abs(sc - ref).max()


@pytest.mark.gpu
def test_device_high_diameter_and_directed():
    from paper_1508_03619_b200 import Brandes, DeviceGraph
    g = O.make_graph("grid", rows=60, cols=70, seed=SEED)
    dg = DeviceGraph.from_csr(g)
    srcs = [int(s) for s in O.pick_sources(g, 3)]
    assert np.abs(Brandes(dg, srcs) - O.brandes(g, srcs)).max() <= TOL
    e = O.gen_kron(11, 16, 3)
    gd = O.build_csr(1 << 11, e, symmetrize=False, directed=True)
    dgd = DeviceGraph.from_csr(gd)
    srcs = [int(s) for s in O.pick_sources(gd, 4)]
    assert np.abs(Brandes(dgd, srcs) - O.brandes(gd, srcs)).max() <= TOL


@pytest.mark.gpu
@pytest.mark.parametrize("no_pull", [False, True])
def test_device_forward_directions(no_pull, monkeypatch):
    # pulled (bottom-up) forward levels and the reference's top-down-only
    # forward give the same scores
    from paper_1508_03619_b200 import Brandes, DeviceGraph
    if no_pull:
        monkeypatch.setenv("GK_BC_NO_PULL", "1")
    for kind, scale in (("kron", 15), ("urand", 14)):
        dg = DeviceGraph.generate(kind, scale, 16, SEED, permute=kind == "kron")
        g = O.make_graph(kind, scale, permute=kind == "kron")
        srcs = [int(s) for s in dg.pick_sources(6, SEED)]
        assert np.abs(Brandes(dg, srcs) - O.brandes(g, srcs)).max() <= TOL
