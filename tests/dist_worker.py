"""torchrun worker for tests/test_dist.py (gloo, CPU): each process runs one
rank of the sharded traversal's model (tests/shard_model.py) and checks its
owned depths and parents against the oracle; rank 0 also checks the
schedule."""
import os
import sys

import numpy as np
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import shard_model as M  # noqa: E402
from oracle import oracle as O  # noqa: E402


def main():
    dist.init_process_group("gloo")
    rank, size = dist.get_rank(), dist.get_world_size()
    for kind, scale in (("kron", 10), ("urand", 9)):
        g = O.make_graph(kind, scale)
        rk = M.Rank(g, rank, size)
        for s in O.pick_sources(g, 3):
            s = int(s)
            for strat in (0, 1, 2):
                (par,), (dep,), steps = M.run([rk], M.TorchComm(), s, strategy=strat)
                d = O.bfs_depths(g, s)
                assert (dep == d[rk.lo:rk.hi]).all(), (kind, s, strat)
                assert (par == M.min_parents(g, d)[rk.lo:rk.hi]).all(), (kind, s, strat)
                rp = O.bfs_replay(g, s, 15, 18, strat)
                assert "".join(x[0] for x in steps) == rp.dirs
                assert [x[2] for x in steps] == rp.result
    dist.barrier()
    print(f"rank {rank} ok", flush=True)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
