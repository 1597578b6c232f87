"""A/B library builds (GK_LIB_PATH) on chosen configs: mean device ms per
BFS over the first K picked sources (after one warm-up).

    python tools/ab_cfg.py --configs grid4900 kron16 --sources 4 LIB_A LIB_B ...
"""
import argparse
import os
import subprocess
import sys

CODE = r'''
import sys, statistics
sys.path.insert(0, ".")
import bench
for c, k in %s:
    cfg = bench.parse_config(c)
    g, _ = bench.build_graph(cfg, 0)
    srcs = [int(s) for s in g.pick_sources(k, bench.SEED)]
    g.bfs(srcs[0], parent=False)
    ts = [g.bfs(s, parent=False).device_ms for s in srcs]
    print(c, "mean ms", round(statistics.mean(ts), 4), "min", round(min(ts), 4), flush=True)
    del g
'''


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", nargs="+", default=["grid4900", "kron16"])
    ap.add_argument("--sources", type=int, default=4)
    ap.add_argument("libs", nargs="+")
    a = ap.parse_args()
    cfgs = [(c, a.sources if not c.startswith("kron1") else 16) for c in a.configs]
    for lib in a.libs:
        env = dict(os.environ, GK_LIB_PATH=os.path.abspath(lib))
        out = subprocess.run([sys.executable, "-c", CODE % repr(cfgs)], env=env, capture_output=True, text=True)
        for line in out.stdout.strip().splitlines():
            print(os.path.basename(lib), line, flush=True)
        if out.returncode:
            print(out.stderr[-800:])


if __name__ == "__main__":
    main()
