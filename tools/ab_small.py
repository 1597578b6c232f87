import os, subprocess, sys
CODE = r'''
import sys, statistics
sys.path.insert(0, ".")
import bench
for c in ("kron16", "grid4900", "kron27"):
    cfg = bench.parse_config(c)
    g, _ = bench.build_graph(cfg, 0)
    srcs = [int(s) for s in g.pick_sources(32 if c != "grid4900" else 2, bench.SEED)]
    for s in srcs[:3]: g.bfs(s, parent=False)
    ts = [g.bfs(s, parent=False).device_ms for s in srcs]
    print(c, round(statistics.mean(ts), 4), flush=True)
    del g
'''
for lib in sys.argv[1:]:
    env = dict(os.environ, GK_LIB_PATH=os.path.abspath(lib))
    out = subprocess.run([sys.executable, "-c", CODE], env=env, capture_output=True, text=True)
    for line in out.stdout.strip().splitlines(): print(os.path.basename(lib), line, flush=True)
    if out.returncode: print(out.stderr[-500:])
