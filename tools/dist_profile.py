"""Per-operation wall time of the sharded BFS on one device (P logical ranks).

    GK_DIST_PROFILE=1 python tools/dist_profile.py [--config kron27] [--ranks 1] [--sources 3]
"""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("GK_DIST_PROFILE", "1")
import bench  # noqa: E402
from paper_1508_03619_b200.dist import GpuEngine, LocalComm, ShardedBfs, pick_sources_sharded  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="kron27")
    ap.add_argument("--ranks", type=int, default=1)
    ap.add_argument("--sources", type=int, default=3)
    a = ap.parse_args()
    cfg = bench.parse_config(a.config)
    E = [GpuEngine.generate(cfg["kind"], cfg["scale"], cfg["degree"], bench.SEED, cfg["permute"], r, a.ranks)
         for r in range(a.ranks)]
    sb = ShardedBfs(E, LocalComm(a.ranks))
    srcs = pick_sources_sharded(sb, a.sources, bench.SEED)
    sb.run(srcs[0])
    sb.prof.clear()
    t0 = time.perf_counter()
    for s in srcs:
        r = sb.run(s)
    dt = (time.perf_counter() - t0) / len(srcs)
    print(f"{a.config} P={a.ranks}: {dt * 1e3:.2f} ms/BFS (wall, profiled)  sched {r.schedule}")
    for k, v in sorted(sb.prof.items(), key=lambda kv: -kv[1]):
        print(f"  {k:12s} {v / len(srcs) * 1e3:8.3f} ms")


if __name__ == "__main__":
    main()
