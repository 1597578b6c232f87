"""The sharded traversal's cost on one GPU: the single-device kernel vs a
ShardGroup of P emulated ranks (one cooperative launch) on the same graph
and sources; prints mean ms, hmean GTEPS and the exchange bytes per BFS.

    python tools/shard_bench.py [--config kron27] [--ranks 1 2 4] [--sources 8]
"""
import argparse
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_1508_03619_b200.dist import ShardGroup  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="kron27")
    ap.add_argument("--ranks", type=int, nargs="*", default=[1, 2, 4])
    ap.add_argument("--sources", type=int, default=8)
    a = ap.parse_args()
    cfg = bench.parse_config(a.config)
    g, _ = bench.build_graph(cfg, 0)
    srcs = [int(s) for s in g.pick_sources(a.sources, bench.SEED)]
    m = {s: g.bfs(s, parent=False, counts=True).component_edges for s in srcs}
    ts = [g.bfs(s, parent=False).device_ms for s in srcs]
    print(f"{a.config} single-device: mean {statistics.mean(ts):.3f} ms  "
          f"hmean {bench.hmean([m[s] / t / 1e6 for s, t in zip(srcs, ts)]):.1f} GTEPS", flush=True)
    del g
    for P in a.ranks:
        grp = ShardGroup.generate(cfg["kind"], cfg["scale"], cfg["degree"], bench.SEED, cfg["permute"], P)
        grp.run(srcs[0], parent=False)
        res = [grp.run(s, parent=False) for s in srcs]
        ts = [r.device_ms for r in res]
        print(f"{a.config} sharded P={P} (emulated on one GPU): mean {statistics.mean(ts):.3f} ms  "
              f"hmean {bench.hmean([m[s] / t / 1e6 for s, t in zip(srcs, ts)]):.1f} GTEPS  "
              f"exchange bytes in / rank / BFS {statistics.mean(max(r.bytes_in) for r in res) / 1e6:.1f} MB  "
              f"schedule {res[0].schedule}", flush=True)
        grp.run(srcs[0], parent=False)
        tr = grp.trace()
        print("   " + " ".join(f"{tr[i][0]}{tr[i][1] - tr[i - 1][1]:.3f}" for i in range(1, len(tr))), flush=True)
        del grp


if __name__ == "__main__":
    main()
