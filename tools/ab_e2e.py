"""Device and end-to-end (gk_bfs_batch, parents to pinned host memory) times
of one library build on kron27's first K sources.

    GK_LIB_PATH=... python tools/ab_e2e.py [K]
"""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_1508_03619_b200 import PinnedBuffer  # noqa: E402


def main():
    k = int(sys.argv[1]) if len(sys.argv) > 1 else 16
    cfg = bench.parse_config("kron27")
    g, _ = bench.build_graph(cfg, 0)
    srcs = [int(s) for s in g.pick_sources(k, bench.SEED)]
    dev = [g.bfs(s, parent=False).device_ms for s in srcs]
    pins = [PinnedBuffer(g.n), PinnedBuffer(g.n)]
    g.bfs_batch(srcs[:2], [pins[i].array for i in range(2)])
    t0 = time.perf_counter()
    g.bfs_batch(srcs, [pins[i & 1].array for i in range(k)])
    t1 = time.perf_counter()
    print(f"mean device ms {np.mean(dev):.3f}  batch wall ms/BFS {(t1 - t0) * 1e3 / k:.3f}", flush=True)


if __name__ == "__main__":
    main()
