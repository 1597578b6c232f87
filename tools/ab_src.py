"""A/B library builds on chosen kron27 sources (GK_LIB_PATH), e.g. the slow ones.

    python tools/ab_src.py "SRC SRC ..." LIB_A LIB_B ...
"""
import os
import subprocess
import sys

CODE = r'''
import sys
sys.path.insert(0, ".")
import bench
cfg = bench.parse_config("kron27")
g, _ = bench.build_graph(cfg, 0)
srcs = [int(x) for x in sys.argv[1].split()]
g.bfs(srcs[0], parent=False)
for s in srcs:
    r = g.bfs(s, parent=False)
    print(s, round(r.device_ms, 3), r.schedule, flush=True)
'''
for lib in sys.argv[2:]:
    env = dict(os.environ, GK_LIB_PATH=os.path.abspath(lib))
    out = subprocess.run([sys.executable, "-c", CODE, sys.argv[1]], env=env, capture_output=True, text=True)
    print(os.path.basename(lib), " | ".join(out.stdout.strip().splitlines()), flush=True)
    if out.returncode:
        print(out.stderr[-800:])
