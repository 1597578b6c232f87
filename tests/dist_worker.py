"""torchrun worker for tests/test_dist.py (gloo, CPU): each rank runs the
sharded orchestrator with the numpy engine and checks its owned parents and
depths against the oracle; rank 0 also checks the schedule."""
import os
import sys

import numpy as np
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

from np_engine import NpEngine  # noqa: E402
from oracle import oracle as O  # noqa: E402
from paper_1508_03619_b200.dist import ShardedBfs, TorchComm  # noqa: E402


def main():
    dist.init_process_group("gloo")
    rank, size = dist.get_rank(), dist.get_world_size()
    comm = TorchComm()
    for kind, scale in (("kron", 10), ("urand", 9)):
        g = O.make_graph(kind, scale)
        eng = NpEngine(g, rank, size)
        sb = ShardedBfs([eng], comm)
        for s in O.pick_sources(g, 4):
            s = int(s)
            for strat in (0, 1, 2):
                res = sb.run(s, strategy=strat, want_depth=True)
                d = O.bfs_depths(g, s)
                lo, hi = eng.lo, eng.hi
                assert (eng.depth == d[lo:hi]).all(), (kind, s, strat, "depth")
                par = eng.parent
                for r in range(hi - lo):
                    v = lo + r
                    if d[v] <= 0:
                        assert par[r] == (v if d[v] == 0 else -1)
                        continue
                    p = int(par[r])
                    assert d[p] == d[v] - 1, (kind, s, v, p)
                    assert p in g.nb[g.off[v]:g.off[v + 1]]
                if rank == 0:
                    rp = O.bfs_replay(g, s, strategy=strat)
                    assert res.schedule == rp.dirs, (res.schedule, rp.dirs)
                    assert [x[2] for x in res.steps] == rp.result
                    assert [x[1] for x in res.steps] == rp.frontier
                    assert res.component_edges == O.component_edges(g, d)
    dist.barrier()
    dist.destroy_process_group()
    print(f"rank {rank} ok")


if __name__ == "__main__":
    main()
