"""ctypes binding of libgk_bfs.so (include/gk_bfs.h).

The library is the product: it must be built in-tree
(``make lib`` / ``__graft_entry__.build()``).  Loading fails loudly when it is
missing -- there is no Python or CPU fallback for the BFS path.
"""
from __future__ import annotations

import ctypes as C
import os

PKG_DIR = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("GK_LIB_PATH") or os.path.join(PKG_DIR, "lib", "libgk_bfs.so")  # override: A/B runs

GK_OK = 0
GK_ERR_SOURCE_RANGE = 1
GK_ERR_BAD_PARAM = 2
GK_ERR_CUDA = 3
GK_ERR_NCCL = 4
GK_ERR_OOM = 5
GK_ERR_NO_DEVICE = 6
GK_ERR_INVALID = 7
GK_ERR_TIMEOUT = 8
GK_ERR_NO_EDGES = 9
GK_ERR_LOAD = 10

# Exported symbols declared in include/gk_bfs.h (checked by the CPU tests).
EXPORTED = (
    "gk_last_error", "gk_abi_version", "gk_device_count", "gk_graph_upload",
    "gk_graph_generate", "gk_graph_generate_grid", "gk_graph_free", "gk_graph_info",
    "gk_graph_download", "gk_pick_sources", "gk_bfs", "gk_bfs_device_parent", "gk_bfs_device_depth",
    "gk_bfs_byte_model", "gk_bfs_keep_depth", "gk_host_alloc", "gk_host_free", "gk_bfs_trace",
    "gk_shard_last_error", "gk_shard_generate", "gk_shard_upload", "gk_shard_free", "gk_shard_info",
    "gk_shard_set_stream", "gk_shard_launches", "gk_shard_join_local", "gk_shard_handle_size",
    "gk_shard_export", "gk_shard_connect", "gk_shard_gather_dead", "gk_shard_group_bfs", "gk_shard_bfs",
    "gk_shard_bytes_in", "gk_shard_download", "gk_shard_trace", "gk_bfs_verify", "gk_graph_load_sg", "gk_graph_save_sg", "gk_brandes",
    "gk_bfs_batch", "gk_bfs_launches", "gk_bfs_batch_d2h_bytes",
)


class CsrView(C.Structure):
    _fields_ = [("num_nodes", C.c_int64), ("directed", C.c_int32), ("reserved", C.c_int32),
                ("out_offsets", C.c_void_p), ("out_neighbors", C.c_void_p),
                ("in_offsets", C.c_void_p), ("in_neighbors", C.c_void_p)]


class Step(C.Structure):
    _fields_ = [("dir", C.c_int32), ("pad", C.c_int32), ("frontier", C.c_int64),
                ("result", C.c_int64), ("edges_to_check", C.c_int64)]


class BfsStats(C.Structure):
    _fields_ = [("steps", C.POINTER(Step)), ("max_steps", C.c_int32), ("want_counts", C.c_int32),
                ("device_ms", C.c_float), ("num_steps", C.c_int32), ("reached", C.c_int64),
                ("component_edges", C.c_int64)]


_lib = None


class _Missing:
    """Stand-in for an entry point an older A/B build lacks (GK_LIB_PATH only)."""

    def __call__(self, *a, **k):
        raise RuntimeError("entry point missing from this A/B build of libgk_bfs.so")


class _Lenient(C.CDLL):
    def __getattr__(self, name):
        try:
            return super().__getattr__(name)
        except AttributeError:
            if name.startswith("gk_"):
                m = _Missing()
                setattr(self, name, m)
                return m
            raise


def load() -> C.CDLL:
    """Load libgk_bfs.so; raise if it has not been built."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(f"{LIB_PATH} is missing: build it with `make lib` or "
                           "`python -c 'import __graft_entry__ as g; g.build()'` (no CPU fallback exists)")
    L = (_Lenient if os.environ.get("GK_LIB_PATH") else C.CDLL)(LIB_PATH)
    vp, i64, i32, u32, u64 = C.c_void_p, C.c_int64, C.c_int32, C.c_uint32, C.c_uint64
    L.gk_last_error.restype = C.c_char_p
    L.gk_abi_version.restype = C.c_int
    L.gk_device_count.restype = C.c_int
    L.gk_graph_upload.argtypes = [C.POINTER(CsrView), C.c_int, C.POINTER(vp)]
    L.gk_graph_generate.argtypes = [C.c_int, C.c_int, C.c_int, u64, C.c_int, C.c_int, C.POINTER(vp)]
    L.gk_graph_generate_grid.argtypes = [i64, i64, C.c_double, C.c_double, u64, C.c_int, C.POINTER(vp)]
    L.gk_graph_load_sg.argtypes = [C.c_char_p, C.c_int, C.POINTER(vp)]
    L.gk_graph_save_sg.argtypes = [vp, C.c_char_p]
    L.gk_graph_free.argtypes = [vp]
    L.gk_graph_free.restype = None
    L.gk_graph_info.argtypes = [vp, C.POINTER(i64), C.POINTER(i64), C.POINTER(i32)]
    L.gk_graph_download.argtypes = [vp, vp, vp, vp, vp]
    L.gk_pick_sources.argtypes = [vp, i64, u64, vp]
    L.gk_bfs.argtypes = [vp, u32, i64, i64, i32, vp, vp, C.POINTER(BfsStats)]
    L.gk_bfs_device_parent.argtypes = [vp]
    L.gk_bfs_device_parent.restype = vp
    L.gk_bfs_device_depth.argtypes = [vp]
    L.gk_bfs_device_depth.restype = vp
    L.gk_bfs_byte_model.argtypes = [vp, C.POINTER(Step), i32, C.POINTER(C.c_double), C.POINTER(C.c_double)]
    L.gk_bfs_keep_depth.argtypes = [vp, i32]
    L.gk_bfs_verify.argtypes = [vp, u32, vp]
    L.gk_bfs_trace.argtypes = [vp, C.POINTER(C.c_uint64), C.c_char_p, i32, C.POINTER(i32)]
    L.gk_brandes.argtypes = [vp, vp, i64, vp, C.POINTER(C.c_double)]
    L.gk_bfs_batch.argtypes = [vp, vp, i32, i64, i64, i32, vp, vp]
    L.gk_bfs_launches.argtypes = [vp]
    L.gk_bfs_launches.restype = i64
    L.gk_bfs_batch_d2h_bytes.argtypes = [vp, C.POINTER(i64)]
    L.gk_bfs_batch_d2h_bytes.restype = i64
    L.gk_shard_last_error.restype = C.c_char_p
    L.gk_shard_generate.argtypes = [C.c_int, C.c_int, C.c_int, u64, C.c_int, C.c_int, C.c_int, C.c_int,
                                    C.POINTER(vp)]
    L.gk_shard_upload.argtypes = [i64, C.c_int, C.c_int, vp, vp, C.c_int, C.POINTER(vp)]
    L.gk_shard_free.argtypes = [vp]
    L.gk_shard_free.restype = None
    L.gk_shard_info.argtypes = [vp] + [C.POINTER(i64)] * 5
    L.gk_shard_set_stream.argtypes = [vp, vp]
    L.gk_shard_launches.argtypes = [vp]
    L.gk_shard_launches.restype = i64
    L.gk_shard_join_local.argtypes = [vp, C.c_int]
    L.gk_shard_download.argtypes = [vp, vp, vp]
    L.gk_shard_trace.argtypes = [vp, C.POINTER(C.c_uint64), C.c_char_p, i32, C.POINTER(i32)]
    L.gk_shard_handle_size.restype = i64
    L.gk_shard_export.argtypes = [vp, vp]
    L.gk_shard_connect.argtypes = [vp, vp]
    L.gk_shard_gather_dead.argtypes = [vp]
    L.gk_shard_group_bfs.argtypes = [vp, u32, i64, i64, i32, vp, vp, C.POINTER(BfsStats)]
    L.gk_shard_bfs.argtypes = [vp, u32, i64, i64, i32, vp, vp, C.POINTER(BfsStats), C.POINTER(i64)]
    L.gk_shard_bytes_in.argtypes = [vp, i32, C.POINTER(Step), i32, C.POINTER(i64)]
    L.gk_host_alloc.argtypes = [i64]
    L.gk_host_alloc.restype = vp
    L.gk_host_free.argtypes = [vp]
    L.gk_host_free.restype = None
    for f in EXPORTED:
        if f not in ("gk_last_error", "gk_abi_version", "gk_device_count", "gk_graph_free",
                     "gk_bfs_device_parent", "gk_bfs_device_depth", "gk_host_alloc", "gk_host_free", "gk_shard_last_error",
                     "gk_shard_free", "gk_shard_launches", "gk_shard_handle_size", "gk_bfs_launches",
                     "gk_bfs_batch_d2h_bytes"):
            getattr(L, f).restype = C.c_int
    _lib = L
    return L


def last_error() -> str:
    return (load().gk_last_error() or b"").decode()
