"""Small workload for compute-sanitizer runs (one tool per gpurun call):
BFS on Kronecker / grid graphs through both bottom-up front paths (shared
memory and global, with the large-graph step kinds forced on a small graph:
owned-range hubs, bitmap top-down steps, sparse sweeps), parity against the
oracle, and Brandes.

    compute-sanitizer --tool memcheck python tools/sanitize_one.py
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("GK_WATCHDOG_MS", "900000")  # sanitized kernels run 10-100x slower

from oracle import oracle as O  # noqa: E402
from paper_1508_03619_b200 import DeviceGraph  # noqa: E402

SEED = 24601


def check(dg, host, nsrc):
    for s in dg.pick_sources(nsrc, SEED):
        s = int(s)
        r = dg.bfs(s, depth=True)
        assert (r.depth == O.bfs_depths(host, s)).all(), f"depth mismatch from {s}"
        ok, msg = O.verify_bfs(host, s, r.parent)
        assert ok, msg
        print(f"  src {s}: ok {r.schedule}", flush=True)


def main():
    host = O.make_graph("kron", 13, 16, SEED)
    print("kron13, front in shared memory", flush=True)
    check(DeviceGraph.from_csr(host), host, 3)
    print("kron13, global front + forced large-graph steps", flush=True)
    os.environ.update(GK_NO_FRONT_SMEM="1", GK_OWN_DMIN="64", GK_BITMAP_TD_MIN="2048")
    dg = DeviceGraph.from_csr(host)
    check(dg, host, 3)
    for k in ("GK_NO_FRONT_SMEM", "GK_OWN_DMIN", "GK_BITMAP_TD_MIN"):
        del os.environ[k]
    grid = O.make_graph("grid", rows=40, cols=50)
    print("grid 40x50", flush=True)
    check(DeviceGraph.from_csr(grid), grid, 2)
    small = O.make_graph("kron", 10, 16, SEED)
    dg = DeviceGraph.from_csr(small)
    src = [int(s) for s in dg.pick_sources(4, SEED)]
    dev = dg.brandes(src)[0]
    ref = O.brandes(small, src)
    assert np.allclose(dev, ref, atol=1e-5), "brandes mismatch"
    print("brandes kron10 ok\nsanitize workload done", flush=True)


if __name__ == "__main__":
    main()
