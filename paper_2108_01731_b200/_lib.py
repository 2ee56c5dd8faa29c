"""ctypes binding of the C ABI in ``include/lcc_b200.h`` (liblcc_b200.so).

The shared library is built in-tree by ``paper_2108_01731_b200/build.py``
(``__graft_entry__.build()``).  There is no fallback: if the library is
missing or fails to load, every call raises ``NativeLibraryError``.
"""
from __future__ import annotations

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
# LCC_LIB_PATH: an in-tree tuning build (A/B variants); default = the product
SO_PATH = os.environ.get("LCC_LIB_PATH") or os.path.join(_HERE, "_lib", "liblcc_b200.so")

LCC_OK, LCC_ERR_INVALID, LCC_ERR_CUDA, LCC_ERR_OOM = 0, 1, 2, 3
W_NONE, W_F32, W_F64, W_U32 = 0, 1, 2, 3
GRAPH_PARTIAL_ROWS = 1  # lcc_graph.flags: a rank's shard (only owned vertices carry rows)
SYNC, ASYNC = 0, 1
FRONTIER_ALL, FRONTIER_VERTEX_NBRS, FRONTIER_CLUSTER_NBRS = 0, 1, 2

# Every symbol include/lcc_b200.h declares (checked by tests/test_capi_symbols.py).
EXPORTS = (
    "lcc_abi_version", "lcc_last_error", "lcc_kernel_launches", "lcc_best_moves_round", "lcc_apply_moves",
    "lcc_compute_frontier", "lcc_par_best_moves", "lcc_par_compress", "lcc_par_flatten",
    "lcc_cc_objective", "lcc_parallel_cc", "lcc_gen_rmat", "lcc_gen_powerlaw_communities",
    "lcc_build_csr_from_pairs", "lcc_frontier_from_mask", "lcc_release_memory",
    "lcc_partition_scores", "lcc_avg_precision_recall", "lcc_cluster_stats", "lcc_weighted_degrees",
    "lcc_build_graph", "lcc_edge_id_range", "lcc_coo_merge",
)
ABI_VERSION = 3


class NativeLibraryError(RuntimeError):
    """The CUDA library is missing or a call failed inside CUDA."""


class LccGraph(ctypes.Structure):
    _fields_ = [("n", ctypes.c_int64), ("nnz", ctypes.c_int64), ("indptr", ctypes.c_void_p),
                ("indices", ctypes.c_void_p), ("weights", ctypes.c_void_p), ("wtype", ctypes.c_int32),
                ("flags", ctypes.c_int32), ("total_weight", ctypes.c_double)]


class LccParams(ctypes.Structure):
    _fields_ = [("k", ctypes.c_void_p), ("lam", ctypes.c_double)]


class LccOptions(ctypes.Structure):
    _fields_ = [("schedule", ctypes.c_int32), ("frontier_policy", ctypes.c_int32), ("refine", ctypes.c_int32),
                ("num_iter", ctypes.c_int32), ("seed", ctypes.c_uint64), ("degree_threshold", ctypes.c_int32),
                ("async_chunks", ctypes.c_int32)]


class LccStats(ctypes.Structure):
    _fields_ = [("rounds", ctypes.c_int64), ("levels", ctypes.c_int64), ("vertices", ctypes.c_int64),
                ("edges_scanned", ctypes.c_int64), ("moves", ctypes.c_int64),
                ("ms_best_moves", ctypes.c_double), ("ms_total", ctypes.c_double),
                ("ms_kernels", ctypes.c_double), ("kernel_launches", ctypes.c_int64)]

    def as_dict(self) -> dict:
        return {f: getattr(self, f) for f, _ in self._fields_}


_lib = None


def load() -> ctypes.CDLL:
    """Load (once) and type the library; raise loudly if it is absent."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(SO_PATH):
        raise NativeLibraryError(
            f"{SO_PATH} not found: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
            "(there is no CPU fallback)")
    try:
        L = ctypes.CDLL(SO_PATH)
    except OSError as e:  # pragma: no cover - depends on the box
        raise NativeLibraryError(f"cannot load {SO_PATH}: {e}") from e
    P, I32, I64, F64 = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_double
    G, PR, O, ST = (ctypes.POINTER(LccGraph), ctypes.POINTER(LccParams), ctypes.POINTER(LccOptions),
                    ctypes.POINTER(LccStats))
    pI64, pI32, pF64 = ctypes.POINTER(I64), ctypes.POINTER(I32), ctypes.POINTER(F64)
    sig = {
        "lcc_abi_version": (ctypes.c_int, []),
        "lcc_last_error": (ctypes.c_char_p, []),
        "lcc_kernel_launches": (ctypes.c_int64, []),
        "lcc_best_moves_round": (ctypes.c_int, [G, PR, P, P, P, I64, I32, I32, I32, P, P, P, pI64, ST, P]),
        "lcc_frontier_from_mask": (ctypes.c_int, [I64, P, P, pI64, P]),
        "lcc_release_memory": (ctypes.c_int, []),
        "lcc_apply_moves": (ctypes.c_int, [I64, P, I64, P, P, P, P]),
        "lcc_compute_frontier": (ctypes.c_int, [G, I32, P, P, P, P, pI64, P]),
        "lcc_par_best_moves": (ctypes.c_int, [G, PR, O, P, P, pI32, ST, P]),
        "lcc_par_compress": (ctypes.c_int, [G, PR, P, P, P, P, P, P, P, pI64, pI64, pF64, pF64, P]),
        "lcc_par_flatten": (ctypes.c_int, [I64, P, P, P, P, P, P]),
        "lcc_cc_objective": (ctypes.c_int, [G, PR, P, pF64, P]),
        "lcc_parallel_cc": (ctypes.c_int, [G, PR, O, P, ST, P]),
        "lcc_gen_rmat": (ctypes.c_int, [I32, I64, F64, F64, F64, ctypes.c_uint64, P, P, pI64, P]),
        "lcc_gen_powerlaw_communities": (ctypes.c_int, [I64, I64, F64, P, P, P, I64, ctypes.c_uint64, P, P, pI64, P]),
        "lcc_build_csr_from_pairs": (ctypes.c_int, [I64, I64, P, P, P, P, pI64, P]),
        "lcc_partition_scores": (ctypes.c_int, [I64, P, P, pF64, pF64, P]),
        "lcc_weighted_degrees": (ctypes.c_int, [G, P, P]),
        "lcc_build_graph": (ctypes.c_int, [I64, I64, P, P, P, P, P, P, pI64, pF64, pI32, P]),
        "lcc_edge_id_range": (ctypes.c_int, [I64, P, P, pI64, pI64, P]),
        "lcc_coo_merge": (ctypes.c_int, [I64, I64, P, P, P, I32, P, P, P, pI64, P]),
        "lcc_avg_precision_recall": (ctypes.c_int, [I64, P, I64, P, P, pF64, pF64, P]),
        "lcc_cluster_stats": (ctypes.c_int, [I64, P, pI64, pI64, pI64, pF64, P]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(L, name)
        fn.restype = res
        fn.argtypes = args
    ver = L.lcc_abi_version()
    if ver != ABI_VERSION:
        raise NativeLibraryError(f"ABI version mismatch: library {ver}, binding {ABI_VERSION}")
    _lib = L
    return L


def check(status: int) -> None:
    """Map an lcc_status to the reference's exception types (graph.py:19-20)."""
    if status == LCC_OK:
        return
    msg = (load().lcc_last_error() or b"").decode(errors="replace")
    if status == LCC_ERR_INVALID:
        from .graph import GraphError
        raise GraphError(msg)
    if status == LCC_ERR_OOM:
        raise MemoryError(msg)
    raise NativeLibraryError(msg)
