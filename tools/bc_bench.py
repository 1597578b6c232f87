"""Brandes betweenness timing (gk_brandes) on device-generated graphs, with
the reference's CPU Brandes (oracle/_ref, all host threads) on the same
graph and sources when it is available and the graph is small enough.

    python tools/bc_bench.py [--config kron20] [--sources 4] [--cpu]

Throughput = arcs traversed (forward + backward visit every stored arc of
the source's component) per second: 2 * m_cc_arcs * sources / time, also
reported as plain ms per source.
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import bench  # noqa: E402
from paper_1508_03619_b200 import DeviceGraph  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="kron20")
    ap.add_argument("--sources", type=int, default=4)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--cpu", action="store_true", help="also time the reference CPU Brandes")
    a = ap.parse_args()
    cfg = bench.parse_config(a.config)
    g, build_s = bench.build_graph(cfg, 0)
    srcs = [int(s) for s in g.pick_sources(a.sources, bench.SEED)]
    g.brandes(srcs)  # warm-up
    ms = []
    for _ in range(a.reps):
        _, t = g.brandes(srcs)
        ms.append(t)
    r = g.bfs(srcs[0], counts=True)
    arcs = 2 * r.component_edges  # stored arcs in the component (undirected)
    dev_ms = min(ms)
    out = {"config": a.config, "n": g.n, "arcs": g.m, "sources": a.sources, "device_ms": dev_ms,
           "ms_per_source": dev_ms / a.sources,
           "gteps_arcs": 2 * arcs * a.sources / (dev_ms * 1e-3) / 1e9}
    if a.cpu:
        from oracle import oracle as O
        if O.ref_available():
            off, nb, _, _ = g.download()
            R = O.RefLib()
            rg = R.wrap(O.Csr(g.n, off, nb))
            if rg is not None:
                t0 = time.perf_counter()
                ref = rg.brandes(srcs)
                cpu_s = time.perf_counter() - t0
                sc, _ = g.brandes(srcs)
                out.update({"cpu_ms": cpu_s * 1e3, "cpu_threads": R.L.gkr_max_threads(),
                            "max_abs_diff_vs_reference": float(np.abs(sc - ref).max())})
    print(json.dumps(out))


if __name__ == "__main__":
    main()
