"""Device-resident CSR graph: the HBM image of the reference ``WeightedGraph``.

The reference stores an immutable symmetric CSR with ``indptr`` int64[n+1],
``indices`` int32[2m] (rows sorted) and ``weights`` float64[2m]
(``/root/reference/pkg/src/lambdacc/graph.py:23-61``).  ``DeviceGraph`` keeps
the same three arrays in HBM with two lossless layout choices:

* all-ones weights are not stored at all (``weights is None``): the kernels
  read 8 B per directed entry instead of 16 B;
* non-negative integer weights (multi-edge counts) with 2 * total weight
  < 2^31 are stored as int32 and summed in exact 32-bit integer tables
  (``LCC_W_U32``; shared-memory fp64 atomics are CAS loops on sm_100a);
* other weights exactly representable in float32 are stored as float32
  (the level-0 kNN config); the kernels widen them to fp64 on load, so the
  arithmetic is identical to fp64 storage.

Coarse levels produced by contraction carry integer weights when the input
is unweighted or integer-weighted, float64 weights otherwise.
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib


class GraphError(ValueError):
    """Malformed graph / parameter input (mirrors reference graph.py:19-20)."""


def _device() -> torch.device:
    if not torch.cuda.is_available():
        raise _lib.NativeLibraryError("no CUDA device: the LambdaCC kernels run on sm_100a only "
                                      "(there is no CPU fallback)")
    return torch.device("cuda", torch.cuda.current_device())


def _to_dev(a, dtype, dev) -> torch.Tensor:
    if isinstance(a, torch.Tensor):
        return a.to(device=dev, dtype=dtype).contiguous()
    arr = np.ascontiguousarray(np.asarray(a), dtype=torch.empty(0, dtype=dtype).numpy().dtype)
    t = torch.from_numpy(arr)
    if arr.nbytes >= (1 << 20):
        t = t.pin_memory()
    return t.to(dev, non_blocking=True)


@dataclass
class DeviceGraph:
    """Symmetric CSR in device memory (see module docstring)."""
    n: int
    m: int
    indptr: torch.Tensor            # int64 [n+1]
    indices: torch.Tensor           # int32 [2m]
    weights: torch.Tensor | None    # float32/float64/int32 [2m] or None (w == 1)
    total_weight: float

    @classmethod
    def from_graph(cls, g, *, keep_f64: bool = False) -> "DeviceGraph":
        """Upload anything with the reference WeightedGraph fields
        (n, indptr, indices, weights, total_weight); numpy or torch arrays."""
        if isinstance(g, DeviceGraph):
            return g
        dev = _device()
        n = int(g.n)
        indptr = _to_dev(g.indptr, torch.int64, dev)
        indices = _to_dev(g.indices, torch.int32, dev)
        if indptr.numel() != n + 1:
            raise GraphError("indptr must have n+1 entries")
        nnz = indices.numel()
        w = getattr(g, "weights", None)
        wt = None
        if isinstance(w, torch.Tensor) and w.dtype == torch.float32 and nnz:
            if w.numel() != nnz:
                raise GraphError("weights must have one entry per CSR index")
            wt = w.to(dev).contiguous()          # already the compact layout
            w = None
        if w is not None and nnz:
            wh = w.detach().cpu().numpy() if isinstance(w, torch.Tensor) else np.asarray(w)
            wh = np.asarray(wh, dtype=np.float64)
            if wh.size != nnz:
                raise GraphError("weights must have one entry per CSR index")
            if not np.all(wh == 1.0):
                w32 = wh.astype(np.float32)
                if (not keep_f64 and wh.min() >= 0 and 2 * wh.sum() < 2 ** 31
                        and np.array_equal(np.floor(wh), wh)):
                    wt = _to_dev(wh.astype(np.int32), torch.int32, dev)
                elif not keep_f64 and np.array_equal(w32.astype(np.float64), wh):
                    wt = _to_dev(w32, torch.float32, dev)
                else:
                    wt = _to_dev(wh, torch.float64, dev)
        tw = getattr(g, "total_weight", None)
        if tw is None:
            tw = float(nnz) / 2 if wt is None else float(wt.double().sum().item()) / 2
        m = int(getattr(g, "m", nnz // 2))
        return cls(n, m, indptr, indices, wt, float(tw))

    @property
    def nnz(self) -> int:
        return int(self.indices.numel())

    @property
    def device(self) -> torch.device:
        return self.indptr.device

    def degrees(self) -> torch.Tensor:
        return self.indptr[1:] - self.indptr[:-1]

    def weighted_degrees(self) -> torch.Tensor:
        """Per-vertex sum of incident weights (reference graph.py:57-61):
        ``lcc_weighted_degrees``, each row summed in CSR order like the
        reference's np.add.at, so the fp64 result is bit-identical."""
        out = torch.empty(max(self.n, 1), dtype=torch.float64, device=self.device)
        gs = self.c_struct()
        _lib.check(_lib.load().lcc_weighted_degrees(ctypes.byref(gs), out.data_ptr(), stream_ptr()))
        return out[:self.n]

    def c_struct(self) -> _lib.LccGraph:
        wtype = _lib.W_NONE
        wp = None
        if self.weights is not None:
            wtype = {torch.float32: _lib.W_F32, torch.int32: _lib.W_U32}.get(self.weights.dtype, _lib.W_F64)
            wp = self.weights.data_ptr()
        return _lib.LccGraph(self.n, self.nnz, self.indptr.data_ptr(),
                             self.indices.data_ptr() if self.nnz else None, wp, wtype, 0,
                             self.total_weight)

    def to_host(self):
        """(indptr, indices, weights-or-None) as numpy arrays."""
        return (self.indptr.cpu().numpy(), self.indices.cpu().numpy(),
                None if self.weights is None else self.weights.double().cpu().numpy())


def stream_ptr() -> int:
    return torch.cuda.current_stream().cuda_stream


# ---------------------------------------------------------------------------
# build_graph (reference graph.py:79-164) on the device
# ---------------------------------------------------------------------------

def _edge_arrays(edges):
    """The reference's ``_as_edge_arrays`` input forms (graph.py:62-76): a
    (u, v, w) tuple of arrays, or an iterable of (u, v, w) triples."""
    if isinstance(edges, tuple) and len(edges) == 3:
        return edges
    arr = np.asarray(list(edges) if not isinstance(edges, np.ndarray) else edges, dtype=np.float64)
    if arr.size == 0:
        return np.empty(0, np.int64), np.empty(0, np.int64), np.empty(0)
    if arr.ndim != 2 or arr.shape[1] != 3:
        raise GraphError("edge list must consist of (u, v, w) triples")
    return arr[:, 0].astype(np.int64), arr[:, 1].astype(np.int64), arr[:, 2]


def build_graph(edges, n: int | None = None) -> DeviceGraph:
    """SPEC build_graph (graph.py:79-95) on the device: see build_graph_arrays."""
    u, v, w = _edge_arrays(edges)
    return build_graph_arrays(u, v, w, n=n)


def build_graph_arrays(u, v, w=None, n: int | None = None) -> DeviceGraph:
    """build_graph_arrays (graph.py:98-164) as one device call
    (``lcc_build_graph``): self loops dropped, same-orientation parallel
    edges summed, the two orientations of a pair averaged, rows sorted --
    CSR, weights and total_weight bit-identical to the reference's (the
    kernels follow numpy's summation order).  ``w=None`` means every weight
    is 1.  Unit weights come back as ``weights=None`` (nothing to read)."""
    dev = _device()
    uu = _to_dev(u, torch.int64, dev).reshape(-1)
    vv = _to_dev(v, torch.int64, dev).reshape(-1)
    ww = None if w is None else _to_dev(w, torch.float64, dev).reshape(-1)
    if uu.numel() != vv.numel() or (ww is not None and ww.numel() != uu.numel()):
        raise GraphError("edge arrays must have equal length")
    ne = int(uu.numel())
    if ne == 0 and n is None:
        raise GraphError("empty graph")
    L = _lib.load()
    lo, hi = ctypes.c_int64(), ctypes.c_int64()
    _lib.check(L.lcc_edge_id_range(ne, uu.data_ptr() if ne else None, vv.data_ptr() if ne else None,
                                   ctypes.byref(lo), ctypes.byref(hi), stream_ptr()))
    if ne and lo.value < 0:
        raise GraphError("vertex ids must be non-negative")
    n_seen = hi.value + 1 if ne else 0
    if n is None:
        n = n_seen
    elif n < n_seen:
        raise GraphError(f"n={n} smaller than largest vertex id {n_seen - 1}")
    n = int(n)
    indptr = torch.empty(n + 1, dtype=torch.int64, device=dev)
    indices = torch.empty(max(2 * ne, 1), dtype=torch.int32, device=dev)
    weights = torch.empty(max(2 * ne, 1), dtype=torch.float64, device=dev)
    m, tw, unit = ctypes.c_int64(), ctypes.c_double(), ctypes.c_int32()
    _lib.check(L.lcc_build_graph(n, ne, uu.data_ptr() if ne else None, vv.data_ptr() if ne else None,
                                 None if ww is None or ne == 0 else ww.data_ptr(), indptr.data_ptr(),
                                 indices.data_ptr(), weights.data_ptr(), ctypes.byref(m), ctypes.byref(tw),
                                 ctypes.byref(unit), stream_ptr()))
    nnz = 2 * m.value
    wt = None if unit.value else weights[:nnz].clone()
    return DeviceGraph(n, m.value, indptr, indices[:nnz].clone(), wt, tw.value)
