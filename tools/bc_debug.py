"""Brandes debugging aid: per-source device-vs-oracle score differences,
sources run back to back on one handle (state carried between launches)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from oracle import oracle as O  # noqa: E402
from paper_1508_03619_b200 import Brandes, DeviceGraph  # noqa: E402

for no_pull in (False, True):
    if no_pull:
        os.environ["GK_BC_NO_PULL"] = "1"
    for kind, scale in (("urand", 14), ("kron", 14), ("urand", 12)):
        dg = DeviceGraph.generate(kind, scale, 16, 24601, permute=kind == "kron")
        g = O.make_graph(kind, scale, permute=kind == "kron")
        srcs = [int(s) for s in dg.pick_sources(8, 24601)]
        worst = max(float(np.abs(Brandes(dg, [s]) - O.brandes(g, [s])).max()) for s in srcs)
        print("no_pull" if no_pull else "pull", kind, scale, f"{worst:.2e}", flush=True)
