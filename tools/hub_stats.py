"""Degree structure of the hub (heavy top-down) step: share of its edges by
frontier-vertex degree, and how many vertices exceed each degree threshold.

    python tools/hub_stats.py [--config kron27] [--sources 4]
"""
import argparse
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="kron27")
    ap.add_argument("--sources", type=int, default=4)
    a = ap.parse_args()
    g, _ = bench.build_graph(bench.parse_config(a.config), 0)
    off = torch.empty(g.n + 1, dtype=torch.int64, device="cuda")
    nb = torch.empty(g.m, dtype=torch.int32, device="cuda")
    g.download_into(off.data_ptr(), nb.data_ptr())
    torch.cuda.synchronize()
    deg = off[1:] - off[:-1]
    del nb
    ths = [1024, 2048, 4096, 9472, 16384, 65536, 262144]
    print("n", g.n, "m", g.m, "max deg", int(deg.max()))
    for t in ths:
        sel = deg >= t
        print(f"deg>={t}: vertices {int(sel.sum())}  arcs {int(deg[sel].sum())}")
    for s in g.pick_sources(a.sources, bench.SEED):
        r = g.bfs(int(s), depth=True, counts=True)
        d = torch.from_numpy(r.depth).cuda()
        for i, c in enumerate(r.schedule):
            fr = d == i
            e = int(deg[fr].sum())
            if c != "T" or e < g.m // 64:
                continue
            parts = " ".join(f">={t}:{int(deg[fr & (deg >= t)].sum()) / max(e, 1):.2f}/{int((fr & (deg >= t)).sum())}"
                             for t in ths)
            print(f"src {int(s)} step {i} {c}: frontier {int(fr.sum())} edges {e}  share(edges)/count {parts}")


if __name__ == "__main__":
    main()
