"""Per-phase time of the sharded kernel at P=1 (emulated) vs the
single-device kernel on kron27, same sources (trace tags, ms per BFS)."""
import collections
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_1508_03619_b200.dist import ShardGroup  # noqa: E402


def agg(tr):
    d = collections.Counter()
    for (t0, a), (tag, b) in zip(tr, tr[1:]):
        d[tag] += b - a
    return d


def show(name, sums, k, sched):
    tot = sum(sums.values()) / k
    print(f"{name}: {tot:.3f} ms/BFS  " + "  ".join(f"{t}={v / k:.3f}" for t, v in sorted(sums.items())),
          f" schedules {sched}", flush=True)


cfg = bench.parse_config(sys.argv[1] if len(sys.argv) > 1 else "kron27")
g, _ = bench.build_graph(cfg, 0)
srcs = [int(s) for s in g.pick_sources(8, bench.SEED)]
os.environ["GK_TRACE_ALL"] = "1"
tot = collections.Counter()
sch = []
for s in srcs:
    r = g.bfs(s, parent=False)
    tot += agg(g.trace())
    sch.append("".join(x[0] for x in r.steps))
show("single", tot, len(srcs), sch[:3])
del g
grp = ShardGroup.generate(cfg["kind"], cfg["scale"], cfg["degree"], bench.SEED, cfg["permute"], 1)
grp.run(srcs[0], parent=False)
tot = collections.Counter()
sch = []
for s in srcs:
    r = grp.run(s, parent=False)
    tot += agg(grp.trace())
    sch.append(r.schedule)
show("sharded P=1", tot, len(srcs), sch[:3])

if len(sys.argv) > 2:  # one source's phase sequence, both kernels
    s = srcs[0]
    r = grp.run(s, parent=False)
    tr = grp.trace()
    print("sharded seq:", " ".join(f"{t}{(b - a) * 1e3:.0f}" for (_, a), (t, b) in zip(tr, tr[1:])))
    del grp
    g, _ = bench.build_graph(cfg, 0)
    g.bfs(s, parent=False)
    tr = g.trace()
    print("single  seq:", " ".join(f"{t}{(b - a) * 1e3:.0f}" for (_, a), (t, b) in zip(tr, tr[1:])))
