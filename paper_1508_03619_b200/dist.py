"""1D-partitioned multi-GPU BFS: host orchestration.

Every rank owns the vertices [r*block, (r+1)*block) (block = ceil(n/P)
rounded up to a multiple of 32) and their CSR rows; the reference's level
loop (proj/include/gapkit/kernels/bfs.hpp:139-169) runs identically on every
rank from all-reduced counters, so the direction schedule equals the
single-GPU (and reference) schedule.  Per level:

* top-down  : each engine expands its owned frontier; owned targets are
              claimed in place, remote ones become (v, u) pairs bucketed by
              owner -> all-to-all -> the owner claims them;
* bottom-up : each engine sweeps its owned unvisited vertices against the
              replicated n-bit front bitmap -> all-gather of the owned slices
              of `next`;
* counters  : {scout, frontier, awake} all-reduced.

`Engine` = one rank's compute (GpuEngine over include/gk_bfs.h's gk_shard_*
entry points; the CPU tests plug in a numpy engine).  `Comm` = the exchange:
TorchComm (torch.distributed: NCCL on the GPU box, gloo in CPU tests, one
process per rank) or LocalComm (P engines inside one process, sequentially,
for single-device tests).  A process may drive several engines; collectives
span all engines of all processes.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from . import BfsStrategy, ConfigError, GapkitError

__all__ = ["GpuEngine", "TorchComm", "LocalComm", "ShardedBfs", "block_of", "owner_of"]


def block_of(n: int, nranks: int) -> int:
    b = (n + nranks - 1) // nranks
    return (b + 31) // 32 * 32


def owner_of(v: int, block: int) -> int:
    return v // block


def _tdiv(a: int, b: int) -> int:
    """C++ integer division (truncation toward zero), as in bfs.hpp:144,154."""
    q = abs(a) // abs(b)
    return q if (a >= 0) == (b > 0) else -q


def _check(st: int, what: str):
    if st == _lib.GK_OK:
        return
    msg = (_lib.load().gk_shard_last_error() or b"").decode()
    if st in (_lib.GK_ERR_SOURCE_RANGE, _lib.GK_ERR_BAD_PARAM):
        raise ConfigError(msg)
    raise GapkitError(f"{what}: {msg} (status {st})")


# --------------------------------------------------------------------- engines
class GpuEngine:
    """One rank's shard on a CUDA device (gk_shard_*)."""

    def __init__(self, handle, device: int):
        import torch
        self.torch = torch
        self._h = C.c_void_p(handle)
        self.device = device
        L = _lib.load()
        n, lo, hi, m, blk = (C.c_int64() for _ in range(5))
        _check(L.gk_shard_info(self._h, C.byref(n), C.byref(lo), C.byref(hi), C.byref(m), C.byref(blk)), "info")
        self.n, self.lo, self.hi, self.m, self.block = n.value, lo.value, hi.value, m.value, blk.value
        self.nloc = self.hi - self.lo
        dev = torch.device("cuda", device)
        self.stream = torch.cuda.current_stream(dev)
        _check(L.gk_shard_set_stream(self._h, C.c_void_p(self.stream.cuda_stream)), "set_stream")
        self.pairs = torch.empty(max(self.m, 1024), dtype=torch.int64, device=dev)
        self.slice = torch.zeros(self.block // 32, dtype=torch.int32, device=dev)

    @classmethod
    def generate(cls, kind: str, scale: int, degree: int, seed: int, permute: bool, rank: int, nranks: int,
                 device: int = 0) -> "GpuEngine":
        import torch
        torch.cuda.set_device(device)
        h = C.c_void_p()
        _check(_lib.load().gk_shard_generate({"kron": 0, "urand": 1}[kind], scale, degree, seed,
                                             1 if permute else 0, rank, nranks, device, C.byref(h)), "generate")
        return cls(h.value, device)

    @classmethod
    def upload(cls, n: int, rank: int, nranks: int, local_off: np.ndarray, nb: np.ndarray,
               device: int = 0) -> "GpuEngine":
        import torch
        torch.cuda.set_device(device)
        off = np.ascontiguousarray(local_off, np.int64)
        nbc = np.ascontiguousarray(nb, np.uint32)
        h = C.c_void_p()
        _check(_lib.load().gk_shard_upload(n, rank, nranks, off.ctypes.data, nbc.ctypes.data if nbc.size else None,
                                           device, C.byref(h)), "upload")
        return cls(h.value, device)

    def __del__(self):
        try:
            if self._h:
                _lib.load().gk_shard_free(self._h)
                self._h = None
        except Exception:
            pass

    # -- per-step operations --------------------------------------------
    def owned_degree(self, v: int) -> int:
        if not (self.lo <= v < self.hi):
            return 0
        d = C.c_int64()
        _check(_lib.load().gk_shard_degree(self._h, v, C.byref(d)), "degree")
        return d.value

    def begin(self, src: int, strategy: int, want_depth: bool):
        _check(_lib.load().gk_shard_begin(self._h, src, strategy, 1 if want_depth else 0), "begin")

    def tail(self) -> int:
        t = C.c_uint64()
        _check(_lib.load().gk_shard_tail(self._h, C.byref(t)), "tail")
        return t.value

    def td_expand(self, qs: int, qe: int, lvl: int, dedup: bool, nranks: int):
        local = (C.c_int64 * 2)()
        counts = (C.c_int64 * nranks)()
        _check(_lib.load().gk_shard_td_expand(self._h, qs, qe, lvl, 1 if dedup else 0, local, counts,
                                              C.c_void_p(self.pairs.data_ptr()), self.pairs.numel()), "td_expand")
        return local[0], local[1], list(counts), self.pairs

    def td_apply(self, recv, nrecv: int, lvl: int):
        out = (C.c_int64 * 2)()
        ptr = C.c_void_p(recv.data_ptr()) if nrecv else None
        _check(_lib.load().gk_shard_td_apply(self._h, ptr, nrecv, lvl, out), "td_apply")
        return out[0], out[1]

    def rescan(self, qs: int, qe: int) -> int:
        t = C.c_int64()
        _check(_lib.load().gk_shard_rescan(self._h, qs, qe, C.byref(t)), "rescan")
        return t.value

    def q2b(self, qs: int, qe: int):
        _check(_lib.load().gk_shard_q2b(self._h, qs, qe, C.c_void_p(self.slice.data_ptr())), "q2b")
        return self.slice

    def bu(self, front, lvl: int):
        a = C.c_int64()
        _check(_lib.load().gk_shard_bu(self._h, C.c_void_p(front.data_ptr()), C.c_void_p(self.slice.data_ptr()), lvl,
                                       C.byref(a)), "bu")
        return a.value, self.slice

    def b2q(self, own_slice):
        _check(_lib.load().gk_shard_b2q(self._h, C.c_void_p(own_slice.data_ptr())), "b2q")

    def result(self, want_parent: bool = True, want_depth: bool = False):
        if want_parent:
            if getattr(self, "_pin", None) is None:  # page-locked: the D2H runs at link speed
                from . import PinnedBuffer
                self._pin = PinnedBuffer(max(self.nloc, 1))
            parent = self._pin.array
        else:
            parent = None
        depth = np.empty(max(self.nloc, 1), np.int32) if want_depth else None
        counts = (C.c_int64 * 2)()
        _check(_lib.load().gk_shard_result(self._h, parent.ctypes.data if parent is not None else None,
                                           depth.ctypes.data if depth is not None else None, counts), "result")
        return (parent[: self.nloc] if parent is not None else None,
                depth[: self.nloc] if depth is not None else None, counts[0], counts[1])

    # -- array helpers used by the communicators ---------------------------
    def own_slice_of(self, full, rank: int):
        w = self.block // 32
        return full[rank * w:(rank + 1) * w]

    def launches(self) -> int:
        return int(_lib.load().gk_shard_launches(self._h))


# ----------------------------------------------------------------- communicators
class TorchComm:
    """Collectives over torch.distributed (NCCL for CUDA tensors, gloo for
    CPU tensors); one engine per process."""

    def __init__(self, group=None):
        import torch
        import torch.distributed as dist
        self.torch, self.dist, self.group = torch, dist, group
        self.rank = dist.get_rank(group)
        self.size = dist.get_world_size(group)

    def ranks_of(self, engines):
        assert len(engines) == 1
        return [self.rank]

    def allreduce(self, per_engine: list[list[int]], like) -> list[int]:
        t = self.torch.tensor(per_engine[0], dtype=self.torch.int64, device=like.device)
        self.dist.all_reduce(t, group=self.group)
        return [int(x) for x in t.tolist()]

    def alltoall(self, sends, counts_per_engine, like):
        torch, dist = self.torch, self.dist
        counts = counts_per_engine[0]
        sc = torch.tensor(counts, dtype=torch.int64, device=like.device)
        rc = torch.empty_like(sc)
        dist.all_to_all_single(rc, sc, group=self.group)
        rcounts = [int(x) for x in rc.tolist()]
        total_s, total_r = sum(counts), sum(rcounts)
        send = sends[0][:total_s]
        recv = torch.empty(max(total_r, 1), dtype=send.dtype, device=send.device)
        if self.size > 1:
            dist.all_to_all_single(recv[:total_r], send, output_split_sizes=rcounts, input_split_sizes=counts,
                                   group=self.group)
        else:
            recv[:total_r].copy_(send)
        return [recv], [total_r]

    def allgather(self, slices):
        torch, dist = self.torch, self.dist
        sl = slices[0]
        out = torch.empty(sl.numel() * self.size, dtype=sl.dtype, device=sl.device)
        if sl.device.type == "cuda":
            dist.all_gather_into_tensor(out, sl.contiguous(), group=self.group)
        else:
            parts = list(out.chunk(self.size))
            dist.all_gather(parts, sl.contiguous(), group=self.group)
            out = torch.cat(parts)
        return out


class LocalComm:
    """All P ranks' engines in this process (single-device tests)."""

    def __init__(self, size: int):
        import torch
        self.torch = torch
        self.rank = 0
        self.size = size

    def ranks_of(self, engines):
        assert len(engines) == self.size
        return list(range(self.size))

    def allreduce(self, per_engine, like):
        return [int(sum(v[i] for v in per_engine)) for i in range(len(per_engine[0]))]

    def alltoall(self, sends, counts_per_engine, like):
        torch = self.torch
        P = self.size
        offs = [np.concatenate([[0], np.cumsum(c)]) for c in counts_per_engine]
        recvs, nrecv = [], []
        for dst in range(P):
            parts = [sends[src][int(offs[src][dst]):int(offs[src][dst + 1])] for src in range(P)]
            r = torch.cat(parts) if parts else sends[dst][:0]
            recvs.append(r.clone() if r.numel() else torch.empty(1, dtype=sends[dst].dtype, device=sends[dst].device))
            nrecv.append(int(r.numel()))
        return recvs, nrecv

    def allgather(self, slices):
        return self.torch.cat([s.clone() for s in slices])


# ------------------------------------------------------------------ orchestrator
@dataclass
class ShardedResult:
    steps: list = field(default_factory=list)  # (dir, frontier, result, edges_to_check)
    parent: np.ndarray | None = None           # global (gathered) when requested
    depth: np.ndarray | None = None
    reached: int = 0
    component_edges: int = 0
    bytes_in: int = 0  # bytes received by this process's engines from other ranks

    @property
    def schedule(self) -> str:
        return "".join(s[0] for s in self.steps)


class ShardedBfs:
    """Runs bfs.hpp:139-169 over a set of engines + a communicator."""

    def __init__(self, engines, comm, alpha: int = 15, beta: int = 18):
        self.engines = engines
        self.comm = comm
        self.ranks = comm.ranks_of(engines)
        e0 = engines[0]
        self.n, self.block, self.P = e0.n, e0.block, comm.size
        self.alpha, self.beta = alpha, beta
        self.like = e0.slice
        import os
        self.profile = os.environ.get("GK_DIST_PROFILE") == "1"
        self.prof = {}
        self.m = comm.allreduce([[e.m] for e in engines], self.like)[0]

    def _ar(self, vals):
        return self._t("allreduce", self.comm.allreduce, vals, self.like)

    def _t(self, key, fn, *a):
        """Call fn(*a); with GK_DIST_PROFILE=1 accumulate its synchronized wall time."""
        if not self.profile:
            return fn(*a)
        import time
        import torch
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        out = fn(*a)
        torch.cuda.synchronize()
        self.prof[key] = self.prof.get(key, 0.0) + time.perf_counter() - t0
        return out

    def run(self, src: int, strategy: int = BfsStrategy.kDirectionOptimizing, want_depth: bool = False,
            gather: bool = False) -> ShardedResult:
        if src < 0 or src >= self.n:
            raise ConfigError("bfs source out of range")
        if self.alpha <= 0 or self.beta <= 0:
            raise ConfigError("bfs alpha and beta must be positive")
        E, P = self.engines, self.P
        for e in E:
            e.begin(src, int(strategy), want_depth)
        scout = self._ar([[e.owned_degree(src)] for e in E])[0]          # bfs.hpp:140
        etc = self.m                                                       # bfs.hpp:139
        qs = [0] * len(E)
        qe = [e.tail() for e in E]
        frontier = 1
        big_edges = max(4096, self.n // 16)
        front, front_valid, lvl = None, False, 0
        res = ShardedResult()
        slice_bytes = (P - 1) * (self.block // 8) * len(E)  # all-gather: every other rank's slice
        while frontier > 0:
            if strategy == BfsStrategy.kDirectionOptimizing and scout > _tdiv(etc, self.alpha):
                if not front_valid:                                        # QueueToBitmap
                    front = self._t("q2b+gather", lambda: self.comm.allgather([e.q2b(a, b) for e, a, b in zip(E, qs, qe)]))
                    res.bytes_in += slice_bytes
                awake = frontier
                qs = list(qe)
                while True:                                                # bfs.hpp:149-154
                    old = awake
                    outs = self._t("bu", lambda: [e.bu(front, lvl) for e in E])
                    awake = self._ar([[a] for a, _ in outs])[0]
                    front = self._t("allgather", lambda: self.comm.allgather([sl for _, sl in outs]))
                    res.bytes_in += slice_bytes
                    res.steps.append(("B", old, awake, etc))
                    lvl += 1
                    if not (awake >= old or awake > _tdiv(self.n, self.beta)):
                        break
                self._t("b2q", lambda: [e.b2q(e.own_slice_of(front, r)) for e, r in zip(E, self.ranks)])  # BitmapToQueue
                qe = [e.tail() for e in E]
                frontier = awake
                scout = 1                                                  # bfs.hpp:156
                front_valid = True
            else:
                etc -= scout                                               # bfs.hpp:158
                fsize = frontier
                dedup = scout > big_edges
                outs = self._t("td_expand", lambda: [e.td_expand(a, b, lvl, dedup, P) for e, a, b in zip(E, qs, qe)])
                recvs, nrecv = self._t("alltoall", self.comm.alltoall, [o[3] for o in outs], [o[2] for o in outs],
                                       self.like)
                res.bytes_in += 8 * sum(k - o[2][r] for k, o, r in zip(nrecv, outs, self.ranks))
                applied = self._t("td_apply", lambda: [e.td_apply(r, k, lvl) for e, r, k in zip(E, recvs, nrecv)])
                qs = list(qe)
                qe = [e.tail() for e in E]
                scout, frontier = self._ar([[o[1] + a[1], o[0] + a[0]] for o, a in zip(outs, applied)])
                if strategy == BfsStrategy.kTopDownRescan:                 # bfs.hpp:161-167
                    scout = self._ar([[e.rescan(a, b)] for e, a, b in zip(E, qs, qe)])[0]
                res.steps.append(("T", fsize, scout, etc))
                lvl += 1
                front_valid = False
        outs = [e.result(gather, want_depth and gather) for e in E]
        reached, degsum = self._ar([[o[2], o[3]] for o in outs])
        res.reached, res.component_edges = reached, degsum // 2
        if gather:
            res.parent = np.concatenate([o[0] for o in outs]) if len(E) == P else None
            if want_depth:
                res.depth = np.concatenate([o[1] for o in outs]) if len(E) == P else None
        return res


# ----------------------------------------------------------------- sources
def _mix64(x: int) -> int:
    M = (1 << 64) - 1
    x = (x + 0x9E3779B97F4A7C15) & M
    x = ((x ^ (x >> 30)) * 0xBF58476D1CE4E5B9) & M
    x = ((x ^ (x >> 27)) * 0x94D049BB133111EB) & M
    return x ^ (x >> 31)


def pick_sources_sharded(sb: ShardedBfs, count: int, seed: int = 24601) -> list[int]:
    """PickSources (source_picker.hpp:22-54) over a sharded graph: every rank
    draws the same Rng(seed) candidates; the owner reports the degree."""
    M = (1 << 64) - 1
    state = _mix64(seed) ^ _mix64(M)  # Rng(seed, stream=0): Mix64(seed) ^ Mix64(~0)
    n = sb.n
    mask = n - 1
    for sh in (1, 2, 4, 8, 16):
        mask |= mask >> sh
    out = []
    while len(out) < count:
        while True:
            state = (state + 0x9E3779B97F4A7C15) & M
            c = (_mix64((state - 0x9E3779B97F4A7C15) & M) >> 32) & mask
            if c < n:
                break
        if sb._ar([[e.owned_degree(c)] for e in sb.engines])[0] > 0:
            out.append(c)
    return out
