"""LambdaCC objective module (``/root/reference/SPEC.md:84-174``).

``cc_objective`` runs on the device (``lcc_cc_objective``); the scalar
helpers ``rescaled_weight`` / ``move_delta`` are the SPEC's per-pair and
per-move formulas evaluated on the host for a single query.
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib
from .graph import DeviceGraph, GraphError, _device, _to_dev, stream_ptr


@dataclass
class ClusteringParams:
    """Resolution lambda and vertex weights k.
    ``k is None`` means k_v = 1 for every vertex."""
    lam: float
    k: torch.Tensor | None = None

    def __post_init__(self):
        lam = float(self.lam)
        # lambda = 0 is accepted as the degenerate test value
        if not (0.0 <= lam < 1.0):
            raise GraphError("lambda must lie in (0, 1)")
        self.lam = lam
        if self.k is not None:
            k = self.k if isinstance(self.k, torch.Tensor) else torch.as_tensor(np.asarray(self.k, np.float64))
            if (k < 0).any():
                raise GraphError("vertex weights must be non-negative")
            self.k = _to_dev(k, torch.float64, _device())

    @property
    def lam_(self) -> float:  # SPEC field name is `lambda` (a Python keyword)
        return self.lam

    def c_struct(self) -> _lib.LccParams:
        return _lib.LccParams(None if self.k is None else self.k.data_ptr(), self.lam)

    def check(self, g: DeviceGraph) -> None:
        if self.k is not None and self.k.numel() != g.n:
            raise GraphError("k length must match the graph's n")


@dataclass
class Clustering:
    """Vertex -> cluster assignment plus cluster masses K.
    ``assignment`` holds canonical labels (cluster id = smallest member id);
    ``cluster_mass[x]`` is K of the cluster labelled x (0 for unused ids)."""
    assignment: torch.Tensor        # int32 [n], device
    cluster_mass: torch.Tensor      # float64 [n], device
    meta: dict = field(default_factory=dict)

    @property
    def n(self) -> int:
        return int(self.assignment.numel())

    @property
    def num_clusters(self) -> int:
        if self.n == 0:
            return 0
        idx = torch.arange(self.n, device=self.assignment.device, dtype=torch.int32)
        return int((self.assignment == idx).sum().item())

    def labels(self) -> np.ndarray:
        return self.assignment.cpu().numpy()


def singletons(n: int, p: ClusteringParams) -> Clustering:
    dev = _device()
    a = torch.arange(n, dtype=torch.int32, device=dev)
    K = torch.ones(n, dtype=torch.float64, device=dev) if p.k is None else p.k.clone()
    return Clustering(a, K)


def clustering_from_labels(labels, p: ClusteringParams) -> Clustering:
    """Canonicalise arbitrary labels (< n) and compute masses on the device."""
    dev = _device()
    lab = _to_dev(labels, torch.int32, dev)
    n = lab.numel()
    C = torch.empty(n, dtype=torch.int32, device=dev)
    K = torch.empty(n, dtype=torch.float64, device=dev)
    if n:
        if int(lab.min().item()) < 0 or int(lab.max().item()) >= n:
            raise GraphError("cluster ids must lie in [0, n)")
        _lib.check(_lib.load().lcc_apply_moves(n, lab.data_ptr(), n,
                                               None if p.k is None else p.k.data_ptr(),
                                               C.data_ptr(), K.data_ptr(), stream_ptr()))
    return Clustering(C, K)


def rescaled_weight(g, p: ClusteringParams, u: int, v: int) -> float:
    """w'_uv: 0 if u == v; w_uv - lam k_u k_v on edges; -lam k_u k_v otherwise."""
    n = int(g.n)
    if not (0 <= u < n and 0 <= v < n):
        raise GraphError("vertex id out of range")
    if u == v:
        return 0.0
    indptr = np.asarray(g.indptr.cpu() if isinstance(g.indptr, torch.Tensor) else g.indptr)
    indices = np.asarray(g.indices.cpu() if isinstance(g.indices, torch.Tensor) else g.indices)
    s, e = int(indptr[u]), int(indptr[u + 1])
    row = indices[s:e]
    i = int(np.searchsorted(row, v))
    w = 0.0
    if i < row.size and row[i] == v:
        ws = g.weights
        if ws is None:
            w = 1.0
        else:
            ws = ws.cpu().numpy() if isinstance(ws, torch.Tensor) else np.asarray(ws)
            w = float(ws[s + i])
    ku = 1.0 if p.k is None else float(p.k[u])
    kv = 1.0 if p.k is None else float(p.k[v])
    return w - p.lam * ku * kv


def move_delta(p: ClusteringParams, k_v: float, K_current: float, K_target: float,
               s_current: float, s_target: float, same: bool = False) -> float:
    """Appendix delta, evaluated in the
    exact operation order the kernels use: (S_x - t K_x) - ((S_c - t K_c) + t k_v)."""
    if same:
        return 0.0
    t = p.lam * k_v
    return (s_target - t * K_target) - ((s_current - t * K_current) + t * k_v)


def cc_objective(g, p: ClusteringParams, c) -> float:
    """Unordered-pair LambdaCC objective, on the device."""
    dg = DeviceGraph.from_graph(g)
    p.check(dg)
    lab = c.assignment if isinstance(c, Clustering) else _to_dev(c, torch.int32, dg.device)
    if lab.numel() != dg.n:
        raise GraphError("clustering size does not match the graph")
    out = ctypes.c_double()
    gs, ps = dg.c_struct(), p.c_struct()
    _lib.check(_lib.load().lcc_cc_objective(ctypes.byref(gs), ctypes.byref(ps),
                                            lab.data_ptr() if dg.n else None, ctypes.byref(out), stream_ptr()))
    return out.value


def modularity_params(g, gamma: float) -> ClusteringParams:
    """k_v = weighted degree, lambda = gamma / (2 total_weight)."""
    dg = DeviceGraph.from_graph(g)
    if dg.n == 0 or dg.total_weight <= 0:
        raise GraphError("empty graph")
    lam = gamma / (2.0 * dg.total_weight)
    if not (0.0 < lam < 1.0):
        raise GraphError("resolution gamma/(2m) must lie in (0, 1)")
    return ClusteringParams(lam, dg.weighted_degrees())


def modularity_value(g, gamma: float, c) -> float:
    """Q = cc_objective / m with the modularity mapping (
    unordered-pair convention, see SURVEY.md §4 erratum 2)."""
    dg = DeviceGraph.from_graph(g)
    p = modularity_params(dg, gamma)
    return cc_objective(dg, p, c) / dg.total_weight
