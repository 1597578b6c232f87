"""numpy stand-in for one rank's compute in the sharded BFS (TEST ONLY).

Implements the Engine interface of paper_1508_03619_b200/dist.py with the
same semantics as the gk_shard_* kernels (gk_shard.cu) so the orchestrator
and the exchange protocol can be exercised on CPU with gloo.  Exchanged
arrays are torch CPU tensors (slices: int32 words, pairs: int64 v<<32|u).
"""
from __future__ import annotations

import numpy as np
import torch

from paper_1508_03619_b200.dist import block_of


class NpEngine:
    def __init__(self, g, rank: int, nranks: int):
        self.n = g.n
        self.block = block_of(g.n, nranks)
        self.lo = min(g.n, rank * self.block)
        self.hi = min(g.n, self.lo + self.block)
        self.nloc = self.hi - self.lo
        self.off = (g.off[self.lo:self.hi + 1] - g.off[self.lo]).astype(np.int64)
        self.nb = g.nb[g.off[self.lo]:g.off[self.hi]].astype(np.uint32)
        self.m = int(self.nb.size)
        self.rank, self.nranks = rank, nranks
        self.slice = torch.zeros(self.block // 32, dtype=torch.int32)
        self.pairs = torch.empty(max(self.m, 1024), dtype=torch.int64)

    def _deg(self, v):
        r = v - self.lo
        return int(self.off[r + 1] - self.off[r])

    def owned_degree(self, v):
        return self._deg(v) if self.lo <= v < self.hi else 0

    def begin(self, src, strategy, want_depth):
        self.encode = strategy != 2
        self.parent = np.full(self.nloc, -1, np.int32)
        self.depth = np.full(self.nloc, -1, np.int32)
        self.visited = np.zeros(self.nloc, bool)
        self.queue = []
        if self.lo <= src < self.hi:
            r = src - self.lo
            self.parent[r] = src
            self.depth[r] = 0
            self.visited[r] = True
            self.queue.append(src)

    def tail(self):
        return len(self.queue)

    def _claim(self, v, u, lvl):
        r = v - self.lo
        if self.visited[r]:
            return False, 0
        self.visited[r] = True
        self.parent[r] = u
        self.depth[r] = lvl + 1
        self.queue.append(v)
        d = self._deg(v)
        return True, (max(d, 1) if self.encode else 1)

    def td_expand(self, qs, qe, lvl, dedup, P):
        claims = scout = 0
        out = [[] for _ in range(P)]
        sent = set()
        for u in list(self.queue[qs:qe]):
            r = u - self.lo
            for v in self.nb[self.off[r]:self.off[r + 1]]:
                v = int(v)
                o = v // self.block
                if o == self.rank:
                    won, s = self._claim(v, u, lvl)
                    claims += won
                    scout += s
                elif not dedup or v not in sent:
                    sent.add(v)
                    out[o].append((v << 32) | u)
        flat = [x for lst in out for x in lst]
        if flat:
            self.pairs[:len(flat)] = torch.tensor(flat, dtype=torch.int64)
        return claims, scout, [len(x) for x in out], self.pairs

    def td_apply(self, recv, nrecv, lvl):
        claims = scout = 0
        for pr in recv[:nrecv].tolist():
            pr &= 0xFFFFFFFFFFFFFFFF
            won, s = self._claim(pr >> 32, pr & 0xFFFFFFFF, lvl)
            claims += won
            scout += s
        return claims, scout

    def rescan(self, qs, qe):
        return sum(self._deg(u) for u in self.queue[qs:qe])

    def q2b(self, qs, qe):
        w = np.zeros(self.block // 32, np.uint32)
        for v in self.queue[qs:qe]:
            r = v - self.lo
            w[r >> 5] |= np.uint32(1 << (r & 31))
        self.slice = torch.from_numpy(w.view(np.int32).copy())
        return self.slice

    def bu(self, front, lvl):
        fw = front.numpy().view(np.uint32)
        nxt = np.zeros(self.block // 32, np.uint32)
        awake = 0
        for r in range(self.nloc):
            if self.visited[r]:
                continue
            for u in self.nb[self.off[r]:self.off[r + 1]]:
                u = int(u)
                if (fw[u >> 5] >> (u & 31)) & 1:
                    self.parent[r] = u
                    self.depth[r] = lvl + 1
                    self.visited[r] = True
                    nxt[r >> 5] |= np.uint32(1 << (r & 31))
                    awake += 1
                    break
        self.slice = torch.from_numpy(nxt.view(np.int32).copy())
        return awake, self.slice

    def b2q(self, own_slice):
        w = own_slice.numpy().view(np.uint32)
        for r in range(self.nloc):
            if (w[r >> 5] >> (r & 31)) & 1:
                self.queue.append(self.lo + r)

    def result(self, want_parent=True, want_depth=False):
        reached = self.parent >= 0
        degsum = int(np.diff(self.off)[reached].sum())
        return (self.parent.copy() if want_parent else None, self.depth.copy() if want_depth else None,
                int(reached.sum()), degsum)

    def own_slice_of(self, full, rank):
        w = self.block // 32
        return full[rank * w:(rank + 1) * w]
