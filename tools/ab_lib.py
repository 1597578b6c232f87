"""A/B two builds of libgk_bfs.so on the same graphs and sources (GK_LIB_PATH).

    python tools/ab_lib.py LIB_A LIB_B [...]
"""
import os
import subprocess
import sys

CODE = r'''
import sys, statistics
sys.path.insert(0, ".")
import bench
for c in ("kron27", "urand27"):
    cfg = bench.parse_config(c)
    g, _ = bench.build_graph(cfg, 0)
    srcs = [int(s) for s in g.pick_sources(16 if c == "kron27" else 6, bench.SEED)]
    g.bfs(srcs[0], parent=False)
    ts = [g.bfs(s, parent=False).device_ms for s in srcs]
    m = g.bfs(srcs[0], parent=False, counts=True).component_edges
    print(c, round(statistics.mean(ts), 4), "hmean GTEPS", round(len(ts) / sum(t / (m / 1e6) for t in ts), 1),
          "max ms", round(max(ts), 3), flush=True)
    del g
'''
for lib in sys.argv[1:]:
    env = dict(os.environ, GK_LIB_PATH=os.path.abspath(lib))
    out = subprocess.run([sys.executable, "-c", CODE], env=env, capture_output=True, text=True)
    for line in out.stdout.strip().splitlines():
        print(os.path.basename(lib), line, flush=True)
    if out.returncode:
        print(out.stderr[-800:])
