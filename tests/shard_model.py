"""CPU model of the sharded traversal (csrc/gk_bfs_sharded.cu), phase for
phase, for the multi-process tests: each rank holds its owned rows and
replicated n-bit bitmaps; the exchanges are the kernel's -- all-gather of
the owned slices of `next` after every step, OR-reduce of the top-down
claims bitmaps over each owner's words, counter sums at every barrier.

`LocalComm` runs P ranks inside one process in lockstep; `TorchComm` runs
one rank per process over torch.distributed (gloo in the CPU tests).  The
result must equal the device's: exact depths, parents = first in-neighbour
(ascending) in the previous level, the reference's schedule and counters.

Test infrastructure only (the device kernel is the product).
"""
from __future__ import annotations

import numpy as np

from paper_1508_03619_b200.dist import block_of


class Rank:
    def __init__(self, g, rank: int, P: int):
        self.g, self.r, self.P = g, rank, P
        self.n = g.n
        b = block_of(g.n, P)
        self.lo, self.hi = min(g.n, rank * b), min(g.n, (rank + 1) * b)
        deg = np.diff(g.off)
        self.dead_own = deg[self.lo:self.hi] == 0  # undirected: in-degree 0

    def deg(self, v: int) -> int:
        return int(self.g.off[v + 1] - self.g.off[v])

    def first_front_in(self, v: int, front: np.ndarray):
        for u in self.g.nb[self.g.off[v]:self.g.off[v + 1]]:
            if front[u]:
                return int(u)
        return None


class LocalComm:
    """All ranks in this process."""

    def sum(self, vals):
        t = int(sum(vals))
        return [t] * len(vals)

    def gather_owned(self, ranks, arrays):
        """Full-n bool arrays whose every owner slice comes from its owner."""
        full = np.zeros(ranks[0].n, bool)
        for rk, a in zip(ranks, arrays):
            full[rk.lo:rk.hi] = a[rk.lo:rk.hi]
        return [full.copy() for _ in ranks]

    def or_reduce_owned(self, ranks, arrays):
        """Per rank: OR over every rank's array, on its own slice."""
        tot = np.zeros(ranks[0].n, bool)
        for a in arrays:
            tot |= a
        return [tot[rk.lo:rk.hi].copy() for rk in ranks]


class TorchComm:
    """One rank per process (torch.distributed, any backend with CPU tensors)."""

    def __init__(self):
        import torch
        import torch.distributed as dist
        self.torch, self.dist = torch, dist

    def sum(self, vals):
        t = self.torch.tensor([int(sum(vals))], dtype=self.torch.int64)
        self.dist.all_reduce(t)
        return [int(t.item())] * len(vals)

    def _gather(self, a):
        t = self.torch.from_numpy(a.astype(np.uint8))
        parts = [self.torch.empty_like(t) for _ in range(self.dist.get_world_size())]
        self.dist.all_gather(parts, t)
        return [p.numpy().astype(bool) for p in parts]

    def gather_owned(self, ranks, arrays):
        (rk,), (a,) = ranks, arrays
        full = np.zeros(rk.n, bool)
        b = block_of(rk.n, rk.P)
        for q, part in enumerate(self._gather(a)):
            lo, hi = min(rk.n, q * b), min(rk.n, (q + 1) * b)
            full[lo:hi] = part[lo:hi]
        return [full]

    def or_reduce_owned(self, ranks, arrays):
        (rk,), (a,) = ranks, arrays
        tot = np.zeros(rk.n, bool)
        for part in self._gather(a):
            tot |= part
        return [tot[rk.lo:rk.hi].copy()]


def run(ranks, comm, src: int, alpha: int = 15, beta: int = 18, strategy: int = 0):
    """bfs_sharded's level loop over the local ranks.  Returns per local
    rank (parent, depth) of its owned vertices and the step log."""
    n = ranks[0].n
    dead = comm.gather_owned(ranks, [_dead_full(rk) for rk in ranks])
    vis = [d.copy() for d in dead]
    front = [np.zeros(n, bool) for _ in ranks]
    parent = [np.full(rk.hi - rk.lo, -1, np.int32) for rk in ranks]
    depth = [np.full(rk.hi - rk.lo, -1, np.int32) for rk in ranks]
    for i, rk in enumerate(ranks):
        vis[i][src] = front[i][src] = True
        if rk.lo <= src < rk.hi:
            parent[i][src - rk.lo] = src
            depth[i][src - rk.lo] = 0
    scout = comm.sum([rk.deg(src) if rk.lo <= src < rk.hi else 0 for rk in ranks])[0]
    etc = int(ranks[0].g.off[-1])
    gfront, lvl, steps = 1, 0, []
    while gfront > 0:
        if strategy == 0 and scout > etc // alpha:
            awake = gfront
            while True:
                old = awake
                nxt = []
                cnt = []
                for i, rk in enumerate(ranks):
                    foreign = np.ones(n, bool)
                    foreign[rk.lo:rk.hi] = False
                    vis[i] |= front[i] & foreign
                    nx = np.zeros(n, bool)
                    c = 0
                    for v in np.flatnonzero(~vis[i][rk.lo:rk.hi]) + rk.lo:
                        u = rk.first_front_in(int(v), front[i])
                        if u is not None:
                            parent[i][v - rk.lo] = u
                            depth[i][v - rk.lo] = lvl + 1
                            nx[v] = True
                            c += 1
                    vis[i][rk.lo:rk.hi] |= nx[rk.lo:rk.hi]
                    nxt.append(nx)
                    cnt.append(c)
                awake = comm.sum(cnt)[0]
                front = comm.gather_owned(ranks, nxt)
                steps.append(("B", old, awake, etc))
                lvl += 1
                if not (awake >= old or awake > n // beta):
                    break
            scout, gfront = 1, awake
        else:
            etc -= scout
            fsize = gfront
            claims = []
            for i, rk in enumerate(ranks):
                foreign = np.ones(n, bool)
                foreign[rk.lo:rk.hi] = False
                vis[i] |= front[i] & foreign
                cl = vis[i].copy()
                for u in np.flatnonzero(front[i][rk.lo:rk.hi]) + rk.lo:
                    cl[rk.g.nb[rk.g.off[u]:rk.g.off[u + 1]]] = True
                claims.append(cl)
            mine = comm.or_reduce_owned(ranks, claims)
            nxt, sc, cnt = [], [], []
            for i, rk in enumerate(ranks):
                new = mine[i] & ~vis[i][rk.lo:rk.hi]
                vis[i][rk.lo:rk.hi] |= new
                nx = np.zeros(n, bool)
                nx[rk.lo:rk.hi] = new
                s = c = 0
                for v in np.flatnonzero(new) + rk.lo:
                    parent[i][v - rk.lo] = rk.first_front_in(int(v), front[i])
                    depth[i][v - rk.lo] = lvl + 1
                    s += max(rk.deg(int(v)), 1)
                    c += 1
                nxt.append(nx)
                sc.append(s)
                cnt.append(c)
            scout = comm.sum(sc)[0]
            gfront = comm.sum(cnt)[0]
            front = comm.gather_owned(ranks, nxt)
            steps.append(("T", fsize, scout, etc))
            lvl += 1
    return parent, depth, steps


def _dead_full(rk: Rank) -> np.ndarray:
    a = np.zeros(rk.n, bool)
    a[rk.lo:rk.hi] = rk.dead_own
    return a


def min_parents(g, depth: np.ndarray) -> np.ndarray:
    """The deterministic parent of every reached vertex: its first
    in-neighbour (ascending id) one level up."""
    p = np.full(g.n, -1, np.int32)
    for v in np.flatnonzero(depth >= 0):
        if depth[v] == 0:
            p[v] = v
            continue
        for u in g.nb[g.off[v]:g.off[v + 1]]:
            if depth[u] == depth[v] - 1:
                p[v] = u
                break
    return p
