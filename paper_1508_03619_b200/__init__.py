"""paper_1508_03619_b200 -- B200-native direction-optimizing BFS (GAP "gapkit" hot path).

Python mirror of the reference BFS surface over the C ABI (include/gk_bfs.h):

    Bfs(g, source, BfsOptions(alpha=15, beta=18, strategy=...)) -> parent array
                                   (reference: proj/include/gapkit/kernels/bfs.hpp:117-177)

``g`` is a :class:`DeviceGraph` (CSR resident in HBM).  Errors follow the
reference: ``ConfigError("bfs source out of range")`` and
``ConfigError("bfs alpha and beta must be positive")`` (bfs.hpp:120-123).
The compute path is libgk_bfs.so only; there is no CPU fallback.
"""
from __future__ import annotations

import ctypes as C
import enum
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from ._lib import BfsStats, CsrView, Step

__all__ = ["Bfs", "Brandes", "BfsOptions", "BfsStrategy", "BfsResult", "ConfigError", "GapkitError", "LoadError",
           "DeviceGraph", "PinnedBuffer", "device_count"]

kDefaultSeed = 24601  # types.hpp:33


class GapkitError(RuntimeError):
    """gapkit::Error (errors.hpp:13-15)."""


class ConfigError(GapkitError):
    """gapkit::ConfigError (errors.hpp:30-32)."""


class LoadError(GapkitError):
    """gapkit::LoadError (errors.hpp:35-46): bad magic / version / truncated."""


class BfsStrategy(enum.IntEnum):
    """gapkit::BfsStrategy (bfs.hpp:37)."""
    kDirectionOptimizing = 0
    kTopDownOnly = 1
    kTopDownRescan = 2


@dataclass
class BfsOptions:
    """gapkit::BfsOptions (bfs.hpp:39-43)."""
    alpha: int = 15
    beta: int = 18
    strategy: BfsStrategy = BfsStrategy.kDirectionOptimizing


@dataclass
class BfsResult:
    parent: np.ndarray | None
    depth: np.ndarray | None
    device_ms: float
    steps: list = field(default_factory=list)  # (dir, frontier, result, edges_to_check, executed-as)
    num_steps: int = 0
    reached: int = -1
    component_edges: int = -1

    @property
    def schedule(self) -> str:
        return "".join(s[0] for s in self.steps)


def device_count() -> int:
    return int(_lib.load().gk_device_count())


def _check(status: int, what: str):
    if status == _lib.GK_OK:
        return
    msg = _lib.last_error()
    if status in (_lib.GK_ERR_SOURCE_RANGE, _lib.GK_ERR_BAD_PARAM, _lib.GK_ERR_NO_EDGES):
        raise ConfigError(msg)
    if status == _lib.GK_ERR_LOAD:
        raise LoadError(msg)
    raise GapkitError(f"{what}: {msg} (status {status})")


class PinnedBuffer:
    """Page-locked host buffer (gk_host_alloc) viewed as a numpy array."""

    def __init__(self, count: int, dtype=np.int32):
        self.nbytes = int(count) * np.dtype(dtype).itemsize
        self._p = _lib.load().gk_host_alloc(max(self.nbytes, 16))
        if not self._p:
            raise GapkitError("gk_host_alloc failed: " + _lib.last_error())
        buf = (C.c_char * max(self.nbytes, 16)).from_address(self._p)
        self.array = np.frombuffer(buf, dtype=dtype, count=int(count))

    def __del__(self):
        try:
            if self._p:
                _lib.load().gk_host_free(self._p)
                self._p = None
        except Exception:
            pass


class DeviceGraph:
    """A CsrGraph resident in HBM (gk_graph handle)."""

    def __init__(self, handle: int, keepalive=None):
        self._h = C.c_void_p(handle)
        self._keep = keepalive
        L = _lib.load()
        n, m, d = C.c_int64(), C.c_int64(), C.c_int32()
        _check(L.gk_graph_info(self._h, C.byref(n), C.byref(m), C.byref(d)), "gk_graph_info")
        self.n, self.m, self.directed = n.value, m.value, bool(d.value)

    # ---- construction -------------------------------------------------
    @classmethod
    def upload(cls, num_nodes: int, out_offsets, out_neighbors, directed: bool = False,
               in_offsets=None, in_neighbors=None, device: int = 0) -> "DeviceGraph":
        off = np.ascontiguousarray(out_offsets, np.int64)
        nb = np.ascontiguousarray(out_neighbors, np.uint32)
        v = CsrView(num_nodes, 1 if directed else 0, 0, off.ctypes.data, nb.ctypes.data if nb.size else None,
                    None, None)
        keep = [off, nb]
        if directed:
            io = np.ascontiguousarray(in_offsets, np.int64)
            inb = np.ascontiguousarray(in_neighbors, np.uint32)
            v.in_offsets, v.in_neighbors = io.ctypes.data, (inb.ctypes.data if inb.size else None)
            keep += [io, inb]
        h = C.c_void_p()
        _check(_lib.load().gk_graph_upload(C.byref(v), device, C.byref(h)), "gk_graph_upload")
        return cls(h.value)

    @classmethod
    def from_csr(cls, csr, device: int = 0) -> "DeviceGraph":
        """Upload any object with n/off/nb(/directed/in_off/in_nb) attributes."""
        return cls.upload(csr.n, csr.off, csr.nb, bool(getattr(csr, "directed", False)),
                          getattr(csr, "in_off", None), getattr(csr, "in_nb", None), device)

    @classmethod
    def generate(cls, kind: str, scale: int, degree: int = 16, seed: int = kDefaultSeed,
                 permute: bool | None = None, device: int = 0) -> "DeviceGraph":
        """On-device GenerateKronecker/GenerateUniform + permute + BuildCsr(symmetrize)."""
        k = {"kron": 0, "urand": 1}[kind]
        if permute is None:
            permute = kind == "kron"
        h = C.c_void_p()
        _check(_lib.load().gk_graph_generate(k, scale, degree, seed, 1 if permute else 0, device,
                                             C.byref(h)), "gk_graph_generate")
        return cls(h.value)

    @classmethod
    def grid(cls, rows: int, cols: int, p_delete: float = 0.15, p_diag: float = 0.02,
             seed: int = kDefaultSeed, device: int = 0) -> "DeviceGraph":
        h = C.c_void_p()
        _check(_lib.load().gk_graph_generate_grid(rows, cols, p_delete, p_diag, seed, device, C.byref(h)),
               "gk_graph_generate_grid")
        return cls(h.value)

    @classmethod
    def load_sg(cls, path: str, device: int = 0) -> "DeviceGraph":
        """ReadSerialized (io.hpp:392-456) straight into HBM."""
        h = C.c_void_p()
        _check(_lib.load().gk_graph_load_sg(str(path).encode(), device, C.byref(h)), "gk_graph_load_sg")
        return cls(h.value)

    def save_sg(self, path: str):
        """WriteSerialized (io.hpp:364-389) from HBM."""
        _check(_lib.load().gk_graph_save_sg(self._h, str(path).encode()), "gk_graph_save_sg")

    def __del__(self):
        try:
            if self._h:
                _lib.load().gk_graph_free(self._h)
                self._h = None
        except Exception:
            pass

    # ---- accessors -----------------------------------------------------
    def download(self):
        off = np.empty(self.n + 1, np.int64)
        nb = np.empty(self.m, np.uint32)
        io = inb = None
        if self.directed:
            io = np.empty(self.n + 1, np.int64)
            inb = np.empty(self.m, np.uint32)
        _check(_lib.load().gk_graph_download(
            self._h, off.ctypes.data, nb.ctypes.data if self.m else None,
            io.ctypes.data if io is not None else None,
            inb.ctypes.data if (inb is not None and self.m) else None), "gk_graph_download")
        return off, nb, io, inb

    def download_into(self, off_ptr: int, nb_ptr: int):
        _check(_lib.load().gk_graph_download(self._h, off_ptr, nb_ptr if self.m else None, None, None),
               "gk_graph_download")

    def pick_sources(self, count: int, seed: int = kDefaultSeed) -> np.ndarray:
        out = np.empty(max(count, 1), np.uint32)
        _check(_lib.load().gk_pick_sources(self._h, count, seed, out.ctypes.data), "gk_pick_sources")
        return out[:count]

    def keep_depth(self, keep: bool = True):
        _check(_lib.load().gk_bfs_keep_depth(self._h, 1 if keep else 0), "gk_bfs_keep_depth")

    def bfs(self, source: int, alpha: int = 15, beta: int = 18,
            strategy: int = BfsStrategy.kDirectionOptimizing, parent: bool | np.ndarray = True,
            depth: bool | np.ndarray = False, counts: bool = False, max_steps: int = 1 << 16) -> BfsResult:
        """One gk_bfs call.  parent/depth: True -> fresh host array, ndarray ->
        caller buffer (n int32), False -> stay in HBM."""
        if source < 0 or source >= self.n:
            raise ConfigError("bfs source out of range")
        L = _lib.load()

        def outbuf(x):
            if x is False or x is None:
                return None, None
            a = np.empty(self.n, np.int32) if x is True else x
            assert a.dtype == np.int32 and a.size >= self.n and a.flags.c_contiguous
            return a, a.ctypes.data

        pa, pp = outbuf(parent)
        da, dp = outbuf(depth)
        # the step log is read into `sl` before returning, so one buffer per
        # handle serves every call (a fresh 1.5 MB ctypes array per call cost
        # ~0.1 ms of host time on small graphs)
        steps = self.__dict__.get("_steps_buf")
        if steps is None or len(steps) < max_steps:
            steps = self._steps_buf = (Step * max_steps)()
        st = BfsStats(C.cast(steps, C.POINTER(Step)), max_steps, 1 if counts else 0, 0.0, 0, -1, -1)
        _check(L.gk_bfs(self._h, int(source), int(alpha), int(beta), int(strategy), pp, dp, C.byref(st)),
               "gk_bfs")
        k = min(st.num_steps, max_steps)
        # (direction, frontier, result, edges_to_check, executed-as: '' or 'P' pushed
        # bottom-up / 'U' pulled top-down / 'K' top-down in the cluster kernel /
        # 'S' the whole traversal in the single-cluster small-graph kernel --
        # same claimed set and counters)
        sl = [(chr(steps[i].dir), steps[i].frontier, steps[i].result, steps[i].edges_to_check,
               chr(steps[i].pad) if steps[i].pad else "") for i in range(k)]
        return BfsResult(pa[: self.n] if pa is not None else None, da[: self.n] if da is not None else None,
                         st.device_ms, sl, st.num_steps, st.reached, st.component_edges)

    def byte_model(self, steps) -> tuple[float, float]:
        """(B_sec, B_use) of the last bfs (which must have recorded depths)."""
        arr = (Step * max(len(steps), 1))()
        for i, s in enumerate(steps):
            arr[i] = Step(ord(s[0]), 0, s[1], s[2], s[3])
        bs, bu = C.c_double(), C.c_double()
        _check(_lib.load().gk_bfs_byte_model(self._h, arr, len(steps), C.byref(bs), C.byref(bu)),
               "gk_bfs_byte_model")
        return bs.value, bu.value

    def verify(self, source: int) -> dict:
        """Device certificate of the last bfs (needs keep_depth or depth=...).
        Returns {'ok': bool, 'errors': [...7 counts], 'first_bad': v or -1}."""
        errs = (C.c_int64 * 8)()
        _check(_lib.load().gk_bfs_verify(self._h, int(source), errs), "gk_bfs_verify")
        e = list(errs)
        return {"ok": sum(e[:7]) == 0, "errors": e[:7], "first_bad": e[7]}

    def launches(self) -> int:
        """Traversal kernels launched on this graph so far (gk_bfs_launches)."""
        return int(_lib.load().gk_bfs_launches(self._h))

    def trace(self):
        """[(tag, t_ms_since_kernel_start)] for the phases of the last bfs."""
        cap = 4096
        ts = (C.c_uint64 * cap)()
        tags = C.create_string_buffer(cap)
        cnt = C.c_int32()
        _check(_lib.load().gk_bfs_trace(self._h, ts, tags, cap, C.byref(cnt)), "gk_bfs_trace")
        k = min(cnt.value, cap)
        return [(tags.raw[i:i + 1].decode(), (ts[i] - ts[0]) * 1e-6) for i in range(k)]

    def device_parent_ptr(self) -> int:
        return int(_lib.load().gk_bfs_device_parent(self._h) or 0)

    def device_depth_ptr(self) -> int:
        return int(_lib.load().gk_bfs_device_depth(self._h) or 0)

    def bfs_batch(self, sources, outs=None, alpha: int = 15, beta: int = 18, strategy: int = 0) -> np.ndarray:
        """gk_bfs_batch: one traversal per source, parent array i copied into
        outs[i] (host int32 arrays of length n, ideally PinnedBuffer views;
        entries may repeat or be None) while traversal i+1 runs.  Returns the
        per-source kernel times (ms)."""
        src = np.ascontiguousarray(np.asarray(sources, dtype=np.int64))
        if src.size and (src.min() < 0 or src.max() >= self.n):
            raise ConfigError("bfs source out of range")
        s32 = src.astype(np.uint32)
        k = int(s32.size)
        ptrs = (C.c_void_p * max(k, 1))()
        if outs is not None:
            if len(outs) != k:
                raise ValueError("outs must have one entry per source")
            for i, o in enumerate(outs):
                if o is None:
                    continue
                if o.dtype != np.int32 or o.size != self.n or not o.flags["C_CONTIGUOUS"]:
                    raise ValueError("each output must be a contiguous int32 array of length n")
                ptrs[i] = o.ctypes.data
        ms = np.zeros(max(k, 1), np.float32)
        _check(_lib.load().gk_bfs_batch(self._h, s32.ctypes.data if k else None, k, alpha, beta, strategy,
                                        ptrs, ms.ctypes.data), "gk_bfs_batch")
        return ms[:k]

    def batch_d2h_bytes(self) -> tuple[int, int]:
        """(device->host result bytes, sources sent compact) of the last
        bfs_batch (gk_bfs_batch_d2h_bytes)."""
        packed = C.c_int64(0)
        total = int(_lib.load().gk_bfs_batch_d2h_bytes(self._h, C.byref(packed)))
        return total, int(packed.value)

    def brandes(self, sources) -> tuple[np.ndarray, float]:
        """Betweenness scores over `sources` (gk_brandes) and the device ms."""
        src = np.ascontiguousarray(np.asarray(sources, dtype=np.int64))
        if src.size and (src.min() < 0 or src.max() > 0xFFFFFFFF):
            raise ConfigError("betweenness source out of range")
        s32 = src.astype(np.uint32)
        out = np.empty(self.n, np.float32)
        ms = C.c_double()
        _check(_lib.load().gk_brandes(self._h, s32.ctypes.data if s32.size else None, int(s32.size),
                                      out.ctypes.data, C.byref(ms)), "gk_brandes")
        return out, ms.value


def Brandes(g: DeviceGraph, sources) -> np.ndarray:
    """gapkit::Brandes (betweenness.hpp:84-145): approximate betweenness over
    `sources`, normalised so the maximum is 1 (float32 scores).  Raises
    ConfigError like the reference (no sources, source out of range, source
    with zero out-degree)."""
    return g.brandes(sources)[0]


def Bfs(g: DeviceGraph, source: int, opts: BfsOptions | None = None) -> np.ndarray:
    """gapkit::Bfs (bfs.hpp:117-177): parent array, parent[source] = source,
    unreachable = -1.  Raises ConfigError like the reference."""
    opts = opts or BfsOptions()
    if source < 0 or source >= g.n:
        raise ConfigError("bfs source out of range")
    if opts.alpha <= 0 or opts.beta <= 0:
        raise ConfigError("bfs alpha and beta must be positive")
    return g.bfs(source, opts.alpha, opts.beta, int(opts.strategy)).parent
