"""Per-phase breakdown of gk_bfs from the in-kernel barrier trace.

    python tools/phase_profile.py [--config kron27] [--sources 4]
"""
import argparse
import os
import sys
from collections import defaultdict

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="kron27")
    ap.add_argument("--sources", type=int, default=4)
    ap.add_argument("--warmup", type=int, default=2)
    ap.add_argument("--src", type=int, nargs="*", help="explicit sources instead of the first picked ones")
    a = ap.parse_args()
    cfg = bench.parse_config(a.config)
    g, bs = bench.build_graph(cfg, 0)
    print(f"{a.config}: n={g.n} arcs={g.m} build {bs:.2f}s")
    srcs = a.src or [int(s) for s in g.pick_sources(a.sources, bench.SEED)]
    for s in srcs[: a.warmup]:
        g.bfs(s, parent=False)
    tot = defaultdict(float)
    for s in srcs:
        r = g.bfs(s, parent=False, counts=True)
        tr = g.trace()
        parts = []
        for i in range(1, len(tr)):
            dt = tr[i][1] - tr[i - 1][1]
            tot[tr[i][0]] += dt
            parts.append(f"{tr[i][0]}{dt:.3f}")
        print(f"src {s}: {r.device_ms:.3f} ms  kernel-span {tr[-1][1]:.3f}  sched {r.schedule}  "
              f"m_cc {r.component_edges}  GTEPS {r.component_edges / r.device_ms / 1e6:.1f}")
        print("   " + " ".join(parts))
        for st in r.steps:
            print(f"     {st[0]}{st[4] or ' '} frontier {st[1]:>10} result {st[2]:>11} etc {st[3]}")
    print("mean per phase kind (ms):", {k: round(v / len(srcs), 4) for k, v in tot.items()})


if __name__ == "__main__":
    main()
