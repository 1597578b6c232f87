"""numpy/ctypes front-end of the CPU checker (TEST INFRASTRUCTURE ONLY).

Loads ``oracle/liboracle.so`` (the C restatement of the reference BFS path,
gk_oracle.c) and, when present, ``oracle/_ref/libgapref.so`` (the unmodified
reference headers behind ref_shim.cc).  Only tests/, ``__graft_entry__.smoke``
and bench.py's CPU-baseline legs may import this module; the product package
``paper_1508_03619_b200`` never does.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
_I64P = np.ctypeslib.ndpointer(np.int64, flags="C_CONTIGUOUS")
_U32P = np.ctypeslib.ndpointer(np.uint32, flags="C_CONTIGUOUS")
_I32P = np.ctypeslib.ndpointer(np.int32, flags="C_CONTIGUOUS")

GKO_DO, GKO_TD_ONLY, GKO_TD_RESCAN = 0, 1, 2


class _Step(C.Structure):
    _fields_ = [("dir", C.c_int32), ("pad", C.c_int32), ("frontier", C.c_int64),
                ("result", C.c_int64), ("edges_to_check", C.c_int64)]


def _load():
    path = os.path.join(HERE, "liboracle.so")
    if not os.path.exists(path):
        raise RuntimeError(f"{path} missing: run `make -C oracle` (or __graft_entry__.build())")
    lib = C.CDLL(path)
    lib.gko_gen_kron.argtypes = [C.c_int, C.c_int, C.c_uint64, _U32P]
    lib.gko_gen_kron.restype = C.c_int64
    lib.gko_gen_urand.argtypes = [C.c_int, C.c_int, C.c_uint64, _U32P]
    lib.gko_gen_urand.restype = C.c_int64
    lib.gko_permute_edges.argtypes = [_U32P, C.c_int64, C.c_int, C.c_uint64]
    lib.gko_perm_keys.argtypes = [C.c_uint64, C.c_int, C.POINTER(C.c_uint64)]
    lib.gko_permute.argtypes = [C.c_uint32, C.c_int, C.POINTER(C.c_uint64)]
    lib.gko_permute.restype = C.c_uint32
    lib.gko_grid_max_edges.argtypes = [C.c_int64, C.c_int64]
    lib.gko_grid_max_edges.restype = C.c_int64
    lib.gko_gen_grid.argtypes = [C.c_int64, C.c_int64, C.c_double, C.c_double, C.c_uint64, _U32P]
    lib.gko_gen_grid.restype = C.c_int64
    lib.gko_build_csr.argtypes = [C.c_int64, _U32P, C.c_int64, C.c_int, _I64P, _U32P]
    lib.gko_build_csr.restype = C.c_int64
    lib.gko_transpose.argtypes = [C.c_int64, _I64P, _U32P, _I64P, _U32P]
    lib.gko_pick_sources.argtypes = [C.c_int64, _I64P, C.c_int64, C.c_uint64, _U32P]
    lib.gko_pick_sources.restype = C.c_int
    lib.gko_bfs_depths.argtypes = [C.c_int64, _I64P, _U32P, C.c_uint32, _I32P]
    lib.gko_verify_bfs.argtypes = [C.c_int64, _I64P, _U32P, C.c_uint32, _I32P, C.c_char_p, C.c_int]
    lib.gko_verify_bfs.restype = C.c_int
    lib.gko_bfs_replay.argtypes = [C.c_int64, C.c_int64, _I64P, _U32P, _I64P, _U32P, C.c_uint32,
                                   C.c_int64, C.c_int64, C.c_int, _I32P, C.POINTER(_Step), C.c_int64]
    lib.gko_bfs_replay.restype = C.c_int64
    lib.gko_byte_model.argtypes = [C.c_int64, _I64P, _U32P, _I64P, _U32P, _I32P, C.c_char_p,
                                   C.c_int64, C.POINTER(C.c_double), C.POINTER(C.c_double)]
    lib.gko_component_edges.argtypes = [C.c_int64, _I64P, _I32P, C.c_int]
    lib.gko_component_edges.restype = C.c_int64
    lib.gko_fnv1a.argtypes = [C.c_void_p, C.c_int64]
    lib.gko_fnv1a.restype = C.c_uint64
    lib.gko_brandes.argtypes = [C.c_int64, _I64P, _U32P, _U32P, C.c_int64, C.POINTER(C.c_float)]
    lib.gko_brandes.restype = C.c_int
    return lib


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = _load()
    return _lib


@dataclass
class Csr:
    """Host CSR in the reference's layout (graph.hpp:26-183)."""
    n: int
    off: np.ndarray          # int64[n+1]
    nb: np.ndarray           # uint32[m]
    directed: bool = False
    in_off: np.ndarray | None = None
    in_nb: np.ndarray | None = None

    @property
    def m(self) -> int:
        return int(self.off[-1])

    def ins(self):
        return (self.in_off, self.in_nb) if self.directed else (self.off, self.nb)

    def degree(self) -> np.ndarray:
        return np.diff(self.off)


# --------------------------------------------------------------- generators
def gen_kron(scale: int, degree: int = 16, seed: int = 24601) -> np.ndarray:
    e = np.empty(2 * degree * (1 << scale), np.uint32)
    lib().gko_gen_kron(scale, degree, seed, e)
    return e


def gen_urand(scale: int, degree: int = 16, seed: int = 24601) -> np.ndarray:
    e = np.empty(2 * degree * (1 << scale), np.uint32)
    lib().gko_gen_urand(scale, degree, seed, e)
    return e


def permute_edges(edges: np.ndarray, scale: int, seed: int) -> np.ndarray:
    e = np.ascontiguousarray(edges, np.uint32).copy()
    lib().gko_permute_edges(e, e.size // 2, scale, seed)
    return e


def perm_keys(seed: int, scale: int) -> np.ndarray:
    k = (C.c_uint64 * 8)()
    lib().gko_perm_keys(seed, scale, k)
    return np.array(list(k), np.uint64)


def permute(v: int, scale: int, seed: int) -> int:
    k = (C.c_uint64 * 8)()
    lib().gko_perm_keys(seed, scale, k)
    return int(lib().gko_permute(v, scale, k))


def gen_grid(rows: int, cols: int, p_delete: float = 0.15, p_diag: float = 0.02,
             seed: int = 24601) -> np.ndarray:
    cap = lib().gko_grid_max_edges(rows, cols)
    e = np.empty(2 * max(cap, 1), np.uint32)
    cnt = lib().gko_gen_grid(rows, cols, p_delete, p_diag, seed, e)
    return e[: 2 * cnt].copy()


def build_csr(n: int, edges: np.ndarray, symmetrize: bool = True, directed: bool = False) -> Csr:
    e = np.ascontiguousarray(edges, np.uint32)
    m = e.size // 2
    off = np.empty(n + 1, np.int64)
    nb = np.empty(max((2 if symmetrize else 1) * m, 1), np.uint32)
    arcs = lib().gko_build_csr(n, e, m, 1 if symmetrize else 0, off, nb)
    if arcs < 0:
        raise ValueError("edge endpoint exceeds declared node count")
    g = Csr(n, off, nb[:arcs].copy(), directed=directed and not symmetrize)
    if g.directed:
        g.in_off = np.empty(n + 1, np.int64)
        g.in_nb = np.empty(max(arcs, 1), np.uint32)
        lib().gko_transpose(n, g.off, g.nb if g.nb.size else np.zeros(1, np.uint32), g.in_off, g.in_nb)
        g.in_nb = g.in_nb[:arcs].copy()
    return g


def _nbp(a: np.ndarray) -> np.ndarray:
    return a if a.size else np.zeros(1, np.uint32)


def pick_sources(g: Csr, count: int, seed: int = 24601) -> np.ndarray:
    out = np.empty(max(count, 1), np.uint32)
    if lib().gko_pick_sources(g.n, g.off, count, seed, out) != 0:
        raise ValueError("cannot pick sources: graph has no edges")
    return out[:count]


def bfs_depths(g: Csr, src: int) -> np.ndarray:
    d = np.empty(g.n, np.int32)
    lib().gko_bfs_depths(g.n, g.off, _nbp(g.nb), src, d)
    return d


_BC_ERRORS = {-1: "betweenness requires at least one source", -2: "betweenness source out of range",
              -3: "betweenness source has zero out-degree"}


def brandes(g: Csr, sources) -> np.ndarray:
    """Serial Brandes restatement (gko_brandes, betweenness.hpp:38-145);
    raises ValueError with the reference's ConfigError message."""
    src = np.ascontiguousarray(np.asarray(sources, dtype=np.uint32))
    out = np.empty(max(g.n, 1), np.float32)
    rc = lib().gko_brandes(g.n, g.off, _nbp(g.nb), src if src.size else np.zeros(1, np.uint32), src.size,
                           out.ctypes.data_as(C.POINTER(C.c_float)))
    if rc:
        raise ValueError(_BC_ERRORS[rc])
    return out[: g.n]


def verify_bfs(g: Csr, src: int, parent: np.ndarray) -> tuple[bool, str]:
    p = np.ascontiguousarray(parent, np.int32)
    if p.size != g.n:
        return False, "parent array has wrong length"
    buf = C.create_string_buffer(512)
    ok = lib().gko_verify_bfs(g.n, g.off, _nbp(g.nb), src, p, buf, 512)
    return bool(ok), buf.value.decode()


@dataclass
class Replay:
    parent: np.ndarray
    dirs: str
    frontier: list
    result: list
    edges_to_check: list


def bfs_replay(g: Csr, src: int, alpha: int = 15, beta: int = 18, strategy: int = GKO_DO,
               max_steps: int = 1 << 20) -> Replay:
    parent = np.empty(max(g.n, 1), np.int32)
    steps = (_Step * max_steps)()
    io, inb = g.ins()
    ns = lib().gko_bfs_replay(g.n, g.m, g.off, _nbp(g.nb), io, _nbp(inb), src, alpha, beta,
                              strategy, parent, steps, max_steps)
    if ns < 0:
        raise ValueError("bfs source out of range" if src >= g.n else "bfs alpha and beta must be positive")
    k = min(ns, max_steps)
    return Replay(parent[: g.n], "".join(chr(steps[i].dir) for i in range(k)),
                  [steps[i].frontier for i in range(k)], [steps[i].result for i in range(k)],
                  [steps[i].edges_to_check for i in range(k)])


def byte_model(g: Csr, depth: np.ndarray, dirs: str) -> tuple[float, float]:
    bs, bu = C.c_double(), C.c_double()
    io, inb = g.ins()
    lib().gko_byte_model(g.n, g.off, _nbp(g.nb), io, _nbp(inb), np.ascontiguousarray(depth, np.int32),
                         dirs.encode(), len(dirs), C.byref(bs), C.byref(bu))
    return bs.value, bu.value


def component_edges(g: Csr, depth_or_parent: np.ndarray) -> int:
    return int(lib().gko_component_edges(g.n, g.off, np.ascontiguousarray(depth_or_parent, np.int32),
                                         1 if g.directed else 0))


def fnv1a(a: np.ndarray) -> int:
    a = np.ascontiguousarray(a)
    return int(lib().gko_fnv1a(a.ctypes.data, a.nbytes))


# ------------------------------------------------------- canonical configs
def make_graph(kind: str, scale: int = 0, degree: int = 16, seed: int = 24601, permute: bool | None = None,
               rows: int = 0, cols: int = 0, p_delete: float = 0.15, p_diag: float = 0.02) -> Csr:
    """Graphs of BASELINE.json's configs at oracle-sized scales.

    kind 'kron' permutes by default (configs 1/3/5), 'urand' does not
    (config 2), 'grid' is the road-like generator (config 4)."""
    if kind == "grid":
        e = gen_grid(rows, cols, p_delete, p_diag, seed)
        return build_csr(rows * cols, e, True)
    if kind == "kron":
        e = gen_kron(scale, degree, seed)
        if permute is None or permute:
            e = permute_edges(e, scale, seed)
    elif kind == "urand":
        e = gen_urand(scale, degree, seed)
        if permute:
            e = permute_edges(e, scale, seed)
    else:
        raise ValueError(kind)
    return build_csr(1 << scale, e, True)


# -------------------------------------------------------- compiled reference
class RefLib:
    """The unmodified reference (oracle/_ref/libgapref.so)."""

    def __init__(self):
        path = os.path.join(HERE, "_ref", "libgapref.so")
        if not os.path.exists(path):
            raise RuntimeError(f"{path} missing (built by `make -C oracle` where /root/reference exists)")
        L = C.CDLL(path)
        vp = C.c_void_p
        L.gkr_max_threads.restype = C.c_int
        L.gkr_set_threads.argtypes = [C.c_int]
        L.gkr_gen.argtypes = [C.c_int, C.c_int, C.c_int, C.c_uint64, _U32P]
        L.gkr_gen.restype = C.c_int64
        L.gkr_build.argtypes = [C.c_int64, _U32P, C.c_int64, C.c_int, C.c_int, C.c_char_p, C.c_int]
        L.gkr_build.restype = vp
        L.gkr_graph_alloc.argtypes = [C.c_int64, C.c_int64, C.c_int, C.POINTER(vp), C.POINTER(vp),
                                      C.POINTER(vp), C.POINTER(vp)]
        L.gkr_graph_alloc.restype = vp
        L.gkr_graph_seal.argtypes = [vp, C.c_int, C.c_char_p, C.c_int]
        L.gkr_graph_seal.restype = C.c_int
        L.gkr_graph_free.argtypes = [vp]
        for f in ("gkr_graph_n", "gkr_graph_m"):
            getattr(L, f).argtypes = [vp]
            getattr(L, f).restype = C.c_int64
        L.gkr_graph_directed.argtypes = [vp]
        L.gkr_graph_directed.restype = C.c_int
        L.gkr_graph_arrays.argtypes = [vp, vp, vp, vp, vp]
        L.gkr_pick_sources.argtypes = [vp, C.c_int64, C.c_uint64, _U32P, C.c_char_p, C.c_int]
        L.gkr_pick_sources.restype = C.c_int
        L.gkr_bfs.argtypes = [vp, C.c_uint32, C.c_int64, C.c_int64, C.c_int, _I32P, C.c_char_p, C.c_int]
        L.gkr_bfs.restype = C.c_int
        L.gkr_bfs_timed.argtypes = [vp, _U32P, C.c_int, C.c_int64, C.c_int64,
                                    np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS"), vp]
        _I64 = np.ctypeslib.ndpointer(np.int64, flags="C_CONTIGUOUS")
        L.gkr_bfs_schedule.argtypes = [vp, C.c_uint32, C.c_int64, C.c_int64, C.c_int, _I32P, _I64, _I64, _I64,
                                       C.c_int64, _I32P]
        L.gkr_bfs_schedule.restype = C.c_int64
        L.gkr_bfs_depths.argtypes = [vp, C.c_uint32, _I32P]
        L.gkr_write_sg.argtypes = [vp, C.c_char_p, C.c_int, C.c_char_p, C.c_int]
        L.gkr_write_sg.restype = C.c_int
        L.gkr_read_sg.argtypes = [C.c_char_p, C.c_char_p, C.c_int]
        L.gkr_read_sg.restype = vp
        L.gkr_verify_bfs.argtypes = [vp, C.c_uint32, _I32P, C.c_char_p, C.c_int]
        L.gkr_verify_bfs.restype = C.c_int
        L.gkr_brandes.argtypes = [vp, _U32P, C.c_int64, C.POINTER(C.c_float), C.c_char_p, C.c_int]
        L.gkr_brandes.restype = C.c_int
        L.gkr_verify_bc.argtypes = [vp, _U32P, C.c_int64, C.POINTER(C.c_float), C.c_char_p, C.c_int]
        L.gkr_verify_bc.restype = C.c_int
        # ref_bench.cc: bench-configuration graphs, the 64-bit builder, trial loop
        L.gkr_bench_graph.argtypes = [C.c_int, C.c_int64, C.c_int64, C.c_uint64, C.c_int, C.c_double, C.c_double,
                                      C.c_char_p, C.c_int]
        L.gkr_bench_graph.restype = vp
        L.gkr_build64.argtypes = [C.c_int64, _U32P, C.c_int64]
        L.gkr_build64.restype = vp
        L.gkr_graph_views.argtypes = [vp, C.POINTER(vp), C.POINTER(vp)]
        L.gkr_component_edges.argtypes = [vp, _I32P]
        L.gkr_component_edges.restype = C.c_int64
        L.gkr_bfs_trials.argtypes = [vp, _U32P, C.c_int, C.c_int64, C.c_int64,
                                     np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS"), _I64]
        self.L = L

    def gen(self, kind: str, scale: int, degree: int = 16, seed: int = 24601) -> np.ndarray:
        e = np.empty(2 * degree * (1 << scale), np.uint32)
        self.L.gkr_gen(0 if kind == "kron" else 1, scale, degree, seed, e)
        return e

    def build(self, n: int, edges: np.ndarray, directed: bool = False, symmetrize: bool = True) -> "RefGraph":
        err = C.create_string_buffer(256)
        e = np.ascontiguousarray(edges, np.uint32)
        h = self.L.gkr_build(n, e if e.size else np.zeros(2, np.uint32), e.size // 2,
                             int(directed), int(symmetrize), err, 256)
        if not h:
            raise RuntimeError(err.value.decode())
        return RefGraph(self, h)

    def bench_graph(self, kind: str, scale: int = 0, degree: int = 16, seed: int = 24601, permute: bool = True,
                    rows: int = 0, cols: int = 0, p_delete: float = 0.15, p_diag: float = 0.02) -> "RefGraph":
        """A bench configuration's graph built on the host: the reference's
        generator (or the grid), the ID permutation, the 64-bit BuildCsr
        (ref_bench.cc)."""
        err = C.create_string_buffer(256)
        k = {"kron": 0, "urand": 1, "grid": 2}[kind]
        a, b = (rows, cols) if kind == "grid" else (scale, degree)
        h = self.L.gkr_bench_graph(k, a, b, seed, int(permute), p_delete, p_diag, err, 256)
        if not h:
            raise RuntimeError(err.value.decode())
        return RefGraph(self, h)

    def build64(self, n: int, edges: np.ndarray) -> "RefGraph":
        """ref_bench.cc's 64-bit OpenMP BuildCsr(el, false, true)."""
        e = np.ascontiguousarray(edges, np.uint32)
        return RefGraph(self, self.L.gkr_build64(n, e if e.size else np.zeros(2, np.uint32), e.size // 2))

    def read_sg(self, path: str) -> "RefGraph":
        err = C.create_string_buffer(256)
        h = self.L.gkr_read_sg(str(path).encode(), err, 256)
        if not h:
            raise RuntimeError(err.value.decode())
        return RefGraph(self, h)

    def wrap(self, g: Csr, check: bool = False) -> "RefGraph":
        """Public CsrGraph constructor (graph.hpp:30-45) over a host CSR."""
        po, pn, pio, pin = C.c_void_p(), C.c_void_p(), C.c_void_p(), C.c_void_p()
        h = self.L.gkr_graph_alloc(g.n, g.m, int(g.directed), C.byref(po), C.byref(pn), C.byref(pio), C.byref(pin))
        C.memmove(po.value, g.off.ctypes.data, g.off.nbytes)
        if g.m:
            C.memmove(pn.value, g.nb.ctypes.data, g.m * 4)
        if g.directed:
            C.memmove(pio.value, g.in_off.ctypes.data, g.in_off.nbytes)
            if g.m:
                C.memmove(pin.value, g.in_nb.ctypes.data, g.m * 4)
        err = C.create_string_buffer(256)
        ok = self.L.gkr_graph_seal(h, int(check), err, 256)
        rg = RefGraph(self, h)
        if not ok:
            raise RuntimeError(err.value.decode())
        return rg


class RefGraph:
    def __init__(self, ref: RefLib, h):
        self.ref, self.h = ref, h
        self.n = ref.L.gkr_graph_n(h)
        self.m = ref.L.gkr_graph_m(h)
        self.directed = bool(ref.L.gkr_graph_directed(h))

    def __del__(self):
        try:
            self.ref.L.gkr_graph_free(self.h)
        except Exception:
            pass

    def csr(self) -> Csr:
        off = np.empty(self.n + 1, np.int64)
        nb = np.empty(self.m, np.uint32)
        g = Csr(self.n, off, nb, directed=self.directed)
        if self.directed:
            g.in_off = np.empty(self.n + 1, np.int64)
            g.in_nb = np.empty(self.m, np.uint32)
            self.ref.L.gkr_graph_arrays(self.h, off.ctypes.data, nb.ctypes.data, g.in_off.ctypes.data,
                                        g.in_nb.ctypes.data)
        else:
            self.ref.L.gkr_graph_arrays(self.h, off.ctypes.data, nb.ctypes.data, None, None)
        return g

    def write_sg(self, path: str, weight_seed: int = -1):
        err = C.create_string_buffer(256)
        if not self.ref.L.gkr_write_sg(self.h, str(path).encode(), weight_seed, err, 256):
            raise RuntimeError(err.value.decode())

    def pick_sources(self, count: int, seed: int = 24601) -> np.ndarray:
        out = np.empty(max(count, 1), np.uint32)
        err = C.create_string_buffer(256)
        if not self.ref.L.gkr_pick_sources(self.h, count, seed, out, err, 256):
            raise RuntimeError(err.value.decode())
        return out[:count]

    def bfs(self, src: int, alpha: int = 15, beta: int = 18, strategy: int = 0) -> np.ndarray:
        p = np.empty(max(self.n, 1), np.int32)
        err = C.create_string_buffer(256)
        if not self.ref.L.gkr_bfs(self.h, src, alpha, beta, strategy, p, err, 256):
            raise ValueError(err.value.decode())
        return p[: self.n]

    def bfs_timed(self, sources, alpha: int = 15, beta: int = 18) -> np.ndarray:
        s = np.ascontiguousarray(sources, np.uint32)
        secs = np.empty(s.size, np.float64)
        self.ref.L.gkr_bfs_timed(self.h, s, s.size, alpha, beta, secs, None)
        return secs

    def trials(self, sources, alpha: int = 15, beta: int = 18) -> tuple[np.ndarray, np.ndarray]:
        """RunBenchmark's BFS trials: seconds per Bfs call and the component
        edges of each result."""
        s = np.ascontiguousarray(sources, np.uint32)
        secs = np.empty(s.size, np.float64)
        mcc = np.empty(s.size, np.int64)
        self.ref.L.gkr_bfs_trials(self.h, s, s.size, alpha, beta, secs, mcc)
        return secs, mcc

    def views(self) -> tuple[np.ndarray, np.ndarray]:
        """(offsets, neighbours) of the out-CSR as read-only numpy views of
        the reference's own vectors (valid while this object lives)."""
        po, pn = C.c_void_p(), C.c_void_p()
        self.ref.L.gkr_graph_views(self.h, C.byref(po), C.byref(pn))
        off = np.frombuffer((C.c_int64 * (self.n + 1)).from_address(po.value), np.int64)
        nb = np.frombuffer((C.c_uint32 * max(self.m, 1)).from_address(pn.value or po.value), np.uint32)[: self.m]
        return off, nb

    def component_edges(self, parent: np.ndarray) -> int:
        return int(self.ref.L.gkr_component_edges(self.h, np.ascontiguousarray(parent, np.int32)))

    def schedule(self, src: int, alpha: int = 15, beta: int = 18, strategy: int = 0,
                 max_steps: int = 1 << 16) -> Replay:
        """Step log from the reference's own detail:: step functions."""
        dirs = np.zeros(max_steps, np.int32)
        fr = np.zeros(max_steps, np.int64)
        rs = np.zeros(max_steps, np.int64)
        et = np.zeros(max_steps, np.int64)
        p = np.empty(max(self.n, 1), np.int32)
        ns = self.ref.L.gkr_bfs_schedule(self.h, src, alpha, beta, strategy, dirs, fr, rs, et, max_steps, p)
        k = min(ns, max_steps)
        return Replay(p[: self.n], "".join(chr(c) for c in dirs[:k]), fr[:k].tolist(), rs[:k].tolist(),
                      et[:k].tolist())

    def depths(self, src: int) -> np.ndarray:
        d = np.empty(max(self.n, 1), np.int32)
        self.ref.L.gkr_bfs_depths(self.h, src, d)
        return d[: self.n]

    def verify(self, src: int, parent: np.ndarray) -> tuple[bool, str]:
        msg = C.create_string_buffer(512)
        ok = self.ref.L.gkr_verify_bfs(self.h, src, np.ascontiguousarray(parent, np.int32), msg, 512)
        return bool(ok), msg.value.decode()

    def brandes(self, sources) -> np.ndarray:
        """The reference's Brandes; raises ValueError with its ConfigError text."""
        src = np.ascontiguousarray(np.asarray(sources, dtype=np.uint32))
        out = np.empty(max(self.n, 1), np.float32)
        err = C.create_string_buffer(256)
        if self.ref.L.gkr_brandes(self.h, src if src.size else np.zeros(1, np.uint32), src.size,
                                  out.ctypes.data_as(C.POINTER(C.c_float)), err, 256):
            raise ValueError(err.value.decode())
        return out[: self.n]

    def verify_bc(self, sources, scores: np.ndarray) -> tuple[bool, str]:
        """The reference's VerifyBetweenness (verify.hpp:216-270)."""
        src = np.ascontiguousarray(np.asarray(sources, dtype=np.uint32))
        sc = np.ascontiguousarray(scores, np.float32)
        msg = C.create_string_buffer(512)
        ok = self.ref.L.gkr_verify_bc(self.h, src, src.size, sc.ctypes.data_as(C.POINTER(C.c_float)), msg, 512)
        return bool(ok), msg.value.decode()


def ref_available() -> bool:
    return os.path.exists(os.path.join(HERE, "_ref", "libgapref.so"))
