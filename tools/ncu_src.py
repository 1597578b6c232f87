"""ncu driver: build one graph, run BFS from the given sources (W warm-up
calls first, skip them with ncu -s W).

    python tools/ncu_src.py --config kron27 --src 87211456 [--warm 2]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="kron27")
    ap.add_argument("--src", type=int, nargs="+", required=True)
    ap.add_argument("--warm", type=int, default=2)
    a = ap.parse_args()
    g, _ = bench.build_graph(bench.parse_config(a.config), 0)
    for _ in range(a.warm):
        g.bfs(a.src[0], parent=False)
    for s in a.src:
        r = g.bfs(s, parent=False)
        print(f"src {s} {r.device_ms:.3f} ms {r.schedule}", flush=True)


if __name__ == "__main__":
    main()
