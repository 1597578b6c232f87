"""1D-partitioned BFS over several GPUs: Python drivers of
the device-driven sharded traversal (include/gk_bfs.h gk_shard_*,
csrc/gk_bfs_sharded.cu).

Rank r of P owns vertices [r*block, (r+1)*block) (block = ceil(n/P) rounded
up to 1024) and their CSR rows.  A traversal is one persistent kernel per
rank: the reference's level loop (proj/include/gapkit/kernels/bfs.hpp:
139-169) runs on the device, ranks exchange bitmap slices through peer
memory and meet at a device-side cross-rank barrier that also reduces the
direction heuristic's counters -- nothing crosses the host between levels.

* `ShardGroup`  -- every rank in this process on ONE device, all of them in
  one cooperative launch (the single-GPU emulation of the multi-device run;
  ranks that wait on one another must not be separate launches on one GPU).
* `ShardedBfs`  -- one process per GPU (torchrun): this rank's shard, wired
  to its peers with CUDA IPC handles exchanged through torch.distributed;
  every rank calls `run(source)` and the kernels meet on the device.

Parents: a vertex's parent is its first in-neighbour (ascending id) in the
previous level, for bottom-up and top-down levels alike (top-down claims are
resolved by their owner with that pull), so the sharded result is
deterministic; depths are exact BFS depths.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from . import BfsStrategy, ConfigError, GapkitError

__all__ = ["ShardGroup", "ShardedBfs", "ShardResult", "block_of", "owner_of", "pick_sources"]

_KINDS = {"kron": 0, "urand": 1}


def block_of(n: int, nranks: int) -> int:
    """Owned vertices per rank: ceil(n/P) rounded up to 1024 (whole 32-word
    bottom-up tasks never straddle two ranks)."""
    b = (n + nranks - 1) // nranks
    return (b + 1023) // 1024 * 1024


def owner_of(v: int, block: int) -> int:
    return v // block


def _check(st: int, what: str):
    if st == _lib.GK_OK:
        return
    msg = (_lib.load().gk_shard_last_error() or b"").decode()
    if st in (_lib.GK_ERR_SOURCE_RANGE, _lib.GK_ERR_BAD_PARAM):
        raise ConfigError(msg)
    raise GapkitError(f"{what}: {msg} (status {st})")


class _Shard:
    """One rank's rows + exchange buffers (gk_shard)."""

    def __init__(self, handle, device: int):
        self._h = handle
        self.device = device
        L = _lib.load()
        n, lo, hi, m, b = (C.c_int64() for _ in range(5))
        _check(L.gk_shard_info(self._h, C.byref(n), C.byref(lo), C.byref(hi), C.byref(m), C.byref(b)),
               "gk_shard_info")
        self.n, self.lo, self.hi, self.m, self.block = n.value, lo.value, hi.value, m.value, b.value
        self.nloc = self.hi - self.lo

    @classmethod
    def generate(cls, kind: str, scale: int, degree: int, seed: int, permute: bool, rank: int, nranks: int,
                 device: int = 0) -> "_Shard":
        h = C.c_void_p()
        _check(_lib.load().gk_shard_generate(_KINDS[kind], scale, degree, seed, int(permute), rank, nranks, device,
                                             C.byref(h)), "gk_shard_generate")
        return cls(h, device)

    @classmethod
    def upload(cls, n: int, rank: int, nranks: int, local_off: np.ndarray, nb: np.ndarray,
               device: int = 0) -> "_Shard":
        lo_ = np.ascontiguousarray(local_off, np.int64)
        nb_ = np.ascontiguousarray(nb, np.uint32)
        h = C.c_void_p()
        _check(_lib.load().gk_shard_upload(n, rank, nranks, lo_.ctypes.data, nb_.ctypes.data if nb_.size else None,
                                           device, C.byref(h)), "gk_shard_upload")
        return cls(h, device)

    def __del__(self):
        try:
            if self._h:
                _lib.load().gk_shard_free(self._h)
                self._h = None
        except Exception:
            pass

    def launches(self) -> int:
        return int(_lib.load().gk_shard_launches(self._h))

    def local_offsets(self) -> np.ndarray:
        off = np.empty(self.nloc + 1, np.int64)
        _check(_lib.load().gk_shard_download(self._h, off.ctypes.data, None), "gk_shard_download")
        return off


@dataclass
class ShardResult:
    parent: np.ndarray | None  # whole graph (ShardGroup) or this rank's owned range (ShardedBfs)
    depth: np.ndarray | None
    device_ms: float
    steps: list = field(default_factory=list)  # (dir, frontier, result, edges_to_check, '')
    reached: int = -1
    component_edges: int = -1
    bytes_in: list = field(default_factory=list)  # exchange bytes received per rank (NVLink)

    @property
    def schedule(self) -> str:
        return "".join(s[0] for s in self.steps)


def _steps(arr, k):
    return [(chr(arr[i].dir), arr[i].frontier, arr[i].result, arr[i].edges_to_check, "") for i in range(k)]


class ShardGroup:
    """P ranks of one graph on one device, run as one cooperative launch."""

    def __init__(self, shards: list[_Shard]):
        self.shards = shards
        self.P = len(shards)
        arr = (C.c_void_p * self.P)(*[s._h for s in shards])
        _check(_lib.load().gk_shard_join_local(arr, self.P), "gk_shard_join_local")
        self._arr = arr
        self.n = shards[0].n

    @classmethod
    def generate(cls, kind: str, scale: int, degree: int, seed: int, permute: bool, nranks: int,
                 device: int = 0) -> "ShardGroup":
        return cls([_Shard.generate(kind, scale, degree, seed, permute, r, nranks, device) for r in range(nranks)])

    @classmethod
    def from_csr(cls, g, nranks: int, device: int = 0) -> "ShardGroup":
        """Split a host CSR (n/off/nb, undirected) into nranks shards."""
        b = block_of(g.n, nranks)
        out = []
        for r in range(nranks):
            lo, hi = min(g.n, r * b), min(g.n, (r + 1) * b)
            out.append(_Shard.upload(g.n, r, nranks, g.off[lo:hi + 1] - g.off[lo], g.nb[g.off[lo]:g.off[hi]], device))
        return cls(out)

    def run(self, source: int, alpha: int = 15, beta: int = 18, strategy: int = BfsStrategy.kDirectionOptimizing,
            parent: bool = True, depth: bool = False, counts: bool = False, max_steps: int = 1 << 16) -> ShardResult:
        L = _lib.load()
        pa = [np.empty(s.nloc, np.int32) for s in self.shards] if parent else None
        da = [np.empty(s.nloc, np.int32) for s in self.shards] if depth else None
        pp = (C.c_void_p * self.P)(*[a.ctypes.data for a in pa]) if pa else None
        dp = (C.c_void_p * self.P)(*[a.ctypes.data for a in da]) if da else None
        steps = (_lib.Step * max_steps)()
        st = _lib.BfsStats(C.cast(steps, C.POINTER(_lib.Step)), max_steps, 1 if counts else 0, 0.0, 0, -1, -1)
        _check(L.gk_shard_group_bfs(self.shards[0]._h, int(source), alpha, beta, int(strategy), pp, dp, C.byref(st)),
               "gk_shard_group_bfs")
        k = min(st.num_steps, max_steps)
        bytes_in = []
        for r in range(self.P):
            b = C.c_int64()
            _check(L.gk_shard_bytes_in(self.shards[0]._h, r, steps, k, C.byref(b)), "gk_shard_bytes_in")
            bytes_in.append(b.value)
        return ShardResult(np.concatenate(pa) if pa else None, np.concatenate(da) if da else None, st.device_ms,
                           _steps(steps, k), st.reached, st.component_edges, bytes_in)

    def launches(self) -> int:
        return self.shards[0].launches()

    def trace(self):
        """[(tag, t_ms_since_kernel_start)] for the phases of the last run."""
        cap = 4096
        ts = (C.c_uint64 * cap)()
        tags = C.create_string_buffer(cap)
        cnt = C.c_int32()
        _check(_lib.load().gk_shard_trace(self.shards[0]._h, ts, tags, cap, C.byref(cnt)), "gk_shard_trace")
        k = min(cnt.value, cap)
        return [(tags.raw[i:i + 1].decode(), (ts[i] - ts[0]) * 1e-6) for i in range(k)]


class ShardConnectError(GapkitError):
    """The ranks could not map each other's buffers (peer access / CUDA IPC
    unavailable); raised on every rank of the group together."""


class ShardedBfs:
    """This process's rank of a multi-GPU group (one process per GPU;
    torch.distributed initialised).  The constructor wires the group: IPC
    handles all-gathered, peers mapped, the dead bitmap completed."""

    def __init__(self, shard: _Shard, nranks: int, group=None, allgather=None, barrier=None):
        """allgather(bytes) -> list of every rank's bytes and barrier() default
        to torch.distributed (tests wire a one-rank group without it)."""
        if allgather is None or barrier is None:
            import torch.distributed as dist

            def allgather(b):
                out = [None] * nranks
                dist.all_gather_object(out, b, group=group)
                return out

            def barrier():
                dist.barrier(group=group)
        self.shard, self.P = shard, nranks
        L = _lib.load()
        blob = C.create_string_buffer(int(L.gk_shard_handle_size()))
        _check(L.gk_shard_export(shard._h, blob), "gk_shard_export")
        joined = b"".join(allgather(bytes(blob.raw)))
        # every rank reports whether it mapped its peers before anyone acts on
        # it, so a rank that cannot (no peer access / IPC) fails the whole
        # group together instead of leaving the others in a collective
        st = L.gk_shard_connect(shard._h, joined)
        why = b"" if st == 0 else (_lib.last_error() or f"status {st}").encode()[:200]
        oks = allgather(b"ok" if st == 0 else b"fail:" + why)
        bad = [i for i, o in enumerate(oks) if o != b"ok"]
        if bad:
            raise ShardConnectError(f"gk_shard_connect failed on rank(s) {bad}: "
                                    + "; ".join(oks[i].decode(errors="replace") for i in bad))
        barrier()  # every rank has published its dead words (gk_shard_export)
        _check(L.gk_shard_gather_dead(shard._h), "gk_shard_gather_dead")
        barrier()
        self.n = shard.n

    @classmethod
    def generate(cls, kind: str, scale: int, degree: int, seed: int, permute: bool, rank: int, nranks: int,
                 device: int, group=None) -> "ShardedBfs":
        return cls(_Shard.generate(kind, scale, degree, seed, permute, rank, nranks, device), nranks, group)

    def run(self, source: int, alpha: int = 15, beta: int = 18, strategy: int = BfsStrategy.kDirectionOptimizing,
            parent: bool = True, depth: bool = False, counts: bool = False, max_steps: int = 1 << 16) -> ShardResult:
        L = _lib.load()
        s = self.shard
        pa = np.empty(s.nloc, np.int32) if parent else None
        da = np.empty(s.nloc, np.int32) if depth else None
        steps = (_lib.Step * max_steps)()
        st = _lib.BfsStats(C.cast(steps, C.POINTER(_lib.Step)), max_steps, 1 if counts else 0, 0.0, 0, -1, -1)
        b = C.c_int64()
        _check(L.gk_shard_bfs(s._h, int(source), alpha, beta, int(strategy), pa.ctypes.data if pa is not None else None,
                              da.ctypes.data if da is not None else None, C.byref(st), C.byref(b)), "gk_shard_bfs")
        k = min(st.num_steps, max_steps)
        return ShardResult(pa, da, st.device_ms, _steps(steps, k), st.reached, st.component_edges, [b.value])

    def launches(self) -> int:
        return self.shard.launches()


def pick_sources(degree_of, n: int, count: int, seed: int = 24601) -> list[int]:
    """PickSources (source_picker.hpp:22-54) over a degree oracle
    degree_of(v) -> int (e.g. a DeviceGraph's or a rank-owned lookup)."""
    mask64 = (1 << 64) - 1

    def mix(x):
        x = (x + 0x9E3779B97F4A7C15) & mask64
        x = ((x ^ (x >> 30)) * 0xBF58476D1CE4E5B9) & mask64
        x = ((x ^ (x >> 27)) * 0x94D049BB133111EB) & mask64
        return x ^ (x >> 31)

    state = mix(seed) ^ mix(mask64)
    bound = n
    m = bound - 1
    for sh in (1, 2, 4, 8, 16):
        m |= m >> sh
    out = []
    while len(out) < count:
        while True:
            state = (state + 0x9E3779B97F4A7C15) & mask64
            c = (mix((state - 0x9E3779B97F4A7C15) & mask64) >> 32) & m
            if c < bound:
                break
        if degree_of(c):
            out.append(c)
    return out
