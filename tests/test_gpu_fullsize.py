"""Full-size parity against the reference's own CPU oracle (BASELINE configs
2, 3 and 4; config 5's graph behind GK_FULLSIZE_KRON30=1).

north_star: "depth arrays bit-exact and parents valid versus the CPU oracle
on all five configs".  For each configuration at its full size:

* the reference arm's graph is built on the HOST, independently of the
  device: the reference's GenerateKronecker / GenerateUniform
  (generator.hpp:56-112) or the grid, the ID permutation and a 64-bit
  BuildCsr (oracle/ref_bench.cc, pinned byte-identical to BuildCsr in
  tests/test_oracle.py); the device graph must equal it array for array;
* PickSources (source_picker.hpp:47-54) on the host graph must give the
  device's sources;
* for two sources, the device depth array must equal the reference's
  detail::BfsDepths (verify.hpp:42-58) element for element, and the device
  ParentArray must pass the reference's VerifyBfs (verify.hpp:62-98).
The reference checks of the two sources run in parallel threads (each is a
serial BFS over billions of arcs).

Config 5's graph (kron30, 34 G arcs) cannot be rebuilt on a 196 GB host
next to its edge list, so that case checks the device graph downloaded into
the reference's CsrGraph (public constructor, graph.hpp:30-45); the device
builder itself is pinned to the reference generator + BuildCsr at scales
10-18 (test_gpu_bfs.py).
"""
import concurrent.futures
import os
import time

import numpy as np
import pytest

from oracle import oracle as O
from paper_1508_03619_b200 import DeviceGraph

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")]

SEED = 24601
NSRC = 2
CONFIGS = {
    "urand27": dict(kind="urand", scale=27, permute=False),
    "kron27": dict(kind="kron", scale=27, permute=True),
    "grid4900": dict(kind="grid", rows=4900, cols=4900),
}


def _device_graph(c):
    if c["kind"] == "grid":
        return DeviceGraph.grid(c["rows"], c["cols"], 0.15, 0.02, SEED)
    return DeviceGraph.generate(c["kind"], c["scale"], 16, SEED, permute=c["permute"])


def _check_sources(rg, g, sources, log):
    """Device depths == reference BfsDepths; device parents pass VerifyBfs."""
    dev = {}
    for s in sources:
        r = g.bfs(int(s), depth=True)
        dev[int(s)] = (r.depth, r.parent, r.schedule)
    t0 = time.time()
    with concurrent.futures.ThreadPoolExecutor(max_workers=2 * len(sources)) as ex:
        dfut = {s: ex.submit(rg.depths, s) for s in dev}
        vfut = {s: ex.submit(rg.verify, s, dev[s][1]) for s in dev}
        for s in dev:
            ref_depth = dfut[s].result()
            mism = np.flatnonzero(ref_depth != dev[s][0])
            assert mism.size == 0, f"source {s}: {mism.size} depths differ, first at {mism[:5]}"
            ok, msg = vfut[s].result()
            assert ok, f"source {s}: VerifyBfs: {msg}"
            reached = int((ref_depth >= 0).sum())
            log.append(f"src {s}: depths bit-exact vs BfsDepths ({reached} reached, max depth "
                       f"{int(ref_depth.max())}), VerifyBfs ok, schedule {dev[s][2][:40]}")
    log.append(f"reference checks {time.time() - t0:.0f} s")


@pytest.mark.parametrize("name", list(CONFIGS))
def test_full_size_parity_vs_reference(name):
    c = CONFIGS[name]
    R = O.RefLib()
    log = [name]
    t0 = time.time()
    if c["kind"] == "grid":
        rg = R.bench_graph("grid", seed=SEED, rows=c["rows"], cols=c["cols"])
    else:
        rg = R.bench_graph(c["kind"], c["scale"], 16, SEED, permute=c["permute"])
    log.append(f"host graph (reference generator + 64-bit BuildCsr) {time.time() - t0:.0f} s: "
               f"n={rg.n} arcs={rg.m}")
    g = _device_graph(c)
    assert (g.n, g.m) == (rg.n, rg.m)
    off_h, nb_h = rg.views()
    off_d, nb_d, _, _ = g.download()
    assert np.array_equal(off_d, off_h), "device offsets differ from the host build"
    assert np.array_equal(nb_d, nb_h), "device neighbours differ from the host build"
    del off_d, nb_d
    log.append("device CSR == host CSR (offsets and neighbours)")
    sources = rg.pick_sources(NSRC, SEED)
    assert (sources == g.pick_sources(NSRC, SEED)).all()
    _check_sources(rg, g, [int(s) for s in sources], log)
    print("\n".join(log))


@pytest.mark.skipif(os.environ.get("GK_FULLSIZE_KRON30") != "1",
                    reason="config 5's graph: ~30 min and ~160 GB of host RAM; GK_FULLSIZE_KRON30=1")
def test_kron30_parity_vs_reference():
    import ctypes as C
    g = DeviceGraph.generate("kron", 30, 16, SEED, permute=True)
    R = O.RefLib()
    po, pn, pio, pin = C.c_void_p(), C.c_void_p(), C.c_void_p(), C.c_void_p()
    h = R.L.gkr_graph_alloc(g.n, g.m, 0, C.byref(po), C.byref(pn), C.byref(pio), C.byref(pin))
    g.download_into(po.value, pn.value)
    err = C.create_string_buffer(256)
    assert R.L.gkr_graph_seal(h, 0, err, 256)
    rg = O.RefGraph(R, h)
    log = [f"kron30: n={rg.n} arcs={rg.m} (device graph in the reference's CsrGraph)"]
    # one source by default: the 145 GB graph, the reference's depth arrays
    # and VerifyBfs's own BFS share the host's ~196 GB
    ns = int(os.environ.get("GK_FULLSIZE_KRON30_NSRC", "1"))
    sources = rg.pick_sources(max(ns, 1), SEED)
    assert (sources == g.pick_sources(max(ns, 1), SEED)).all()
    _check_sources(rg, g, [int(s) for s in sources], log)
    print("\n".join(log))
