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
        """Per-vertex sum of incident weights (reference graph.py:57-61)."""
        deg = self.degrees()
        if self.weights is None:
            return deg.to(torch.float64)
        rows = torch.repeat_interleave(torch.arange(self.n, device=self.device), deg)
        out = torch.zeros(self.n, dtype=torch.float64, device=self.device)
        return out.index_add_(0, rows, self.weights.to(torch.float64))

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
