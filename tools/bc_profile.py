"""Per-phase breakdown of one Brandes source (gk_bfs_trace after gk_brandes).

    python tools/bc_profile.py [--config kron20] [--sources 2]
Tags: I init, T/H forward light/heavy per level, D/E backward level/chunks.
"""
import argparse
import os
import sys
from collections import defaultdict

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="kron20")
    ap.add_argument("--sources", type=int, default=2)
    a = ap.parse_args()
    cfg = bench.parse_config(a.config)
    g, _ = bench.build_graph(cfg, 0)
    srcs = [int(s) for s in g.pick_sources(a.sources, bench.SEED)]
    g.brandes(srcs[:1])
    for s in srcs:
        _, ms = g.brandes([s])
        tr = g.trace()
        tot = defaultdict(float)
        for i in range(1, len(tr)):
            tot[tr[i][0]] += tr[i][1] - tr[i - 1][1]
        print(f"src {s}: {ms:.3f} ms  kernel-span {tr[-1][1]:.3f}  phases " +
              " ".join(f"{k}{v:.3f}" for k, v in sorted(tot.items())) + f"  barriers {len(tr) - 1}")


if __name__ == "__main__":
    main()
