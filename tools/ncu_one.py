"""Minimal driver for ncu captures: build one graph on the device and run a
few BFS calls (the first W are warm-up launches to skip with ncu -s).

    python tools/ncu_one.py [--config kron27] [--runs 2]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="kron27")
    ap.add_argument("--runs", type=int, default=2)
    a = ap.parse_args()
    cfg = bench.parse_config(a.config)
    g, _ = bench.build_graph(cfg, 0)
    srcs = [int(s) for s in g.pick_sources(a.runs, bench.SEED)]
    for s in srcs:
        r = g.bfs(s, parent=False)
        print(f"src {s} {r.device_ms:.3f} ms {r.schedule}", flush=True)


if __name__ == "__main__":
    main()
