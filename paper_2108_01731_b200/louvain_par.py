"""Parallel Louvain module (``/root/reference/SPEC.md:243-327``; Alg. 1).

The reference's clustering entry point and its options -- objective,
lambda / resolution, node weights, synchronous vs asynchronous moves, vertex
subsetting and multi-level refinement -- are kept as Python functions with
the SPEC names and argument meanings.  Behind them every operation is one
call into the sm_100a C-ABI library (``include/lcc_b200.h``); nothing here
computes on the CPU.
"""
from __future__ import annotations

import ctypes
import enum
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib
from .graph import DeviceGraph, GraphError, _device, _to_dev, stream_ptr
from .objective import Clustering, ClusteringParams, singletons


class Schedule(enum.IntEnum):
    """ParOptions.schedule (§3.2.1)."""
    Synchronous = _lib.SYNC
    Asynchronous = _lib.ASYNC


class FrontierPolicy(enum.IntEnum):
    """ParOptions.frontier_policy (§3.2.2)."""
    AllVertices = _lib.FRONTIER_ALL
    VertexNeighbors = _lib.FRONTIER_VERTEX_NBRS
    ClusterNeighbors = _lib.FRONTIER_CLUSTER_NBRS


_SCHED_ALIASES = {"sync": Schedule.Synchronous, "synchronous": Schedule.Synchronous,
                  "async": Schedule.Asynchronous, "asynchronous": Schedule.Asynchronous}
_FRONTIER_ALIASES = {"all": FrontierPolicy.AllVertices, "vertex-nbrs": FrontierPolicy.VertexNeighbors,
                     "vertex_neighbors": FrontierPolicy.VertexNeighbors,
                     "cluster-nbrs": FrontierPolicy.ClusterNeighbors,
                     "cluster_neighbors": FrontierPolicy.ClusterNeighbors}


@dataclass
class ParOptions:
    """SPEC.md:248-251.  Defaults = Asynchronous + VertexNeighbors + refine
    (§4.1 "overall optimal settings"), num_iter = 10.

    ``threads`` is recorded for compatibility (the GPU runs every frontier
    vertex concurrently).  ``degree_threshold`` is the degree above which a
    vertex's neighbour-cluster table is built by many CTAs in global memory
    instead of one CTA in shared memory (the GPU analogue of the paper's
    sequential-vs-parallel hash-table switch); it is clamped
    from below by the warp path (32) and from above by the shared-memory
    table capacity.  ``async_chunks``: the asynchronous schedule walks the
    frontier in this many ordered sub-rounds; later sub-rounds see the moves
    of earlier ones (symmetry breaking).  0 = auto (up to 64
    for small frontiers, one wave for frontiers of 4M+ vertices)."""
    schedule: Schedule = Schedule.Asynchronous
    frontier_policy: FrontierPolicy = FrontierPolicy.VertexNeighbors
    refine: bool = True
    num_iter: int = 10
    seed: int = 0
    threads: int = 0
    degree_threshold: int = 1000
    async_chunks: int = 0

    def __post_init__(self):
        if isinstance(self.schedule, str):
            self.schedule = _SCHED_ALIASES[self.schedule.lower()]
        if isinstance(self.frontier_policy, str):
            self.frontier_policy = _FRONTIER_ALIASES[self.frontier_policy.lower()]
        self.schedule = Schedule(self.schedule)
        self.frontier_policy = FrontierPolicy(self.frontier_policy)
        if int(self.num_iter) < 1:
            raise GraphError("num_iter must be >= 1")
        if int(self.threads) < 0:
            raise GraphError("threads must be >= 1 (0 = all)")
        if int(self.async_chunks) < 0:
            raise GraphError("async_chunks must be >= 0 (0 = auto)")

    def c_struct(self) -> _lib.LccOptions:
        return _lib.LccOptions(int(self.schedule), int(self.frontier_policy), 1 if self.refine else 0,
                               int(self.num_iter), int(self.seed) & ((1 << 64) - 1),
                               int(self.degree_threshold), int(self.async_chunks))


@dataclass
class MoveBuffer:
    """Alg. 1's D array plus the per-vertex moved flags."""
    desired: torch.Tensor   # int32 [n]; fresh-singleton targets are n + v
    moved: torch.Tensor     # uint8 [n]
    moved_count: int = 0


@dataclass
class Frontier:
    """Device vertex subset V' (sorted member ids)."""
    n: int
    ids: torch.Tensor       # int32, sorted

    @property
    def size(self) -> int:
        return int(self.ids.numel())

    def members(self) -> np.ndarray:
        return self.ids.cpu().numpy().astype(np.int64)


@dataclass
class CompressedLevel:
    """SPEC.md:181-184."""
    graph: DeviceGraph
    weights: torch.Tensor   # k' (float64 [n'])
    mapping: torch.Tensor   # int32 [n]
    internal_offset: float


@dataclass
class RunStats:
    rounds: int = 0
    levels: int = 0
    vertices: int = 0
    edges_scanned: int = 0
    moves: int = 0
    ms_best_moves: float = 0.0
    ms_total: float = 0.0
    ms_kernels: float = 0.0
    kernel_launches: int = 0
    extra: dict = field(default_factory=dict)


def _stats_from(st: _lib.LccStats) -> RunStats:
    d = st.as_dict()
    return RunStats(**d)


def _prep(g, p: ClusteringParams):
    dg = DeviceGraph.from_graph(g)
    p.check(dg)
    return dg, dg.c_struct(), p.c_struct()


def _labels_of(c, dg: DeviceGraph) -> torch.Tensor:
    lab = c.assignment if isinstance(c, Clustering) else _to_dev(c, torch.int32, dg.device)
    if lab.numel() != dg.n:
        raise GraphError("clustering size does not match the graph")
    return lab


# ---------------------------------------------------------------------------
# single iteration primitives
# ---------------------------------------------------------------------------

def best_moves_round(g, p: ClusteringParams, c: Clustering, frontier=None,
                     schedule: Schedule = Schedule.Synchronous, degree_threshold: int = 1000,
                     async_chunks: int = 0, nbr_mark: torch.Tensor | None = None) -> MoveBuffer:
    """One Alg. 1 iteration (lines 6-8).  Synchronous: returns D and moved
    flags, leaves ``c`` untouched.  Asynchronous: applies the moves to ``c``
    in place (labels may temporarily use ids n+v; call ``apply_moves``).
    ``nbr_mark`` (uint8 [n], optional): receives the fused VertexNeighbors
    frontier mask (see ``frontier_from_mask``)."""
    dg, gs, ps = _prep(g, p)
    schedule = Schedule(schedule)
    n = dg.n
    dev = dg.device
    moved = torch.empty(n, dtype=torch.uint8, device=dev)
    D = torch.empty(n, dtype=torch.int32, device=dev)
    cnt = ctypes.c_int64()
    fr = None if frontier is None else (frontier.ids if isinstance(frontier, Frontier)
                                        else _to_dev(frontier, torch.int32, dev))
    K = c.cluster_mass
    if schedule == Schedule.Asynchronous and K.numel() < 2 * n:
        K2 = torch.zeros(2 * n, dtype=torch.float64, device=dev)
        K2[:K.numel()] = K
        c.cluster_mass = K = K2
    _lib.check(_lib.load().lcc_best_moves_round(
        ctypes.byref(gs), ctypes.byref(ps), c.assignment.data_ptr(), K.data_ptr(),
        None if fr is None else fr.data_ptr(), n if fr is None else fr.numel(), int(schedule),
        int(degree_threshold), int(async_chunks), D.data_ptr(), moved.data_ptr(),
        None if nbr_mark is None else nbr_mark.data_ptr(), ctypes.byref(cnt), None, stream_ptr()))
    if schedule == Schedule.Asynchronous:
        D = c.assignment
    return MoveBuffer(D, moved, cnt.value)


def apply_moves(labels: torch.Tensor, label_range: int, p: ClusteringParams) -> Clustering:
    """Sync apply / async reconcile: canonical labels + rebuilt masses."""
    n = labels.numel()
    dev = labels.device
    C = torch.empty(n, dtype=torch.int32, device=dev)
    K = torch.empty(n, dtype=torch.float64, device=dev)
    _lib.check(_lib.load().lcc_apply_moves(n, labels.data_ptr(), int(label_range),
                                           None if p.k is None else p.k.data_ptr(), C.data_ptr(),
                                           K.data_ptr(), stream_ptr()))
    return Clustering(C, K)


def compute_frontier(policy, moved, g, c_old=None, c_new=None) -> Frontier:
    """SPEC.md:267-275.  ``moved``: uint8/bool device mask, or member ids."""
    dg = DeviceGraph.from_graph(g)
    if isinstance(policy, str):
        policy = _FRONTIER_ALIASES[policy.lower()]
    policy = FrontierPolicy(policy)
    dev = dg.device
    n = dg.n
    if isinstance(moved, torch.Tensor) and moved.dtype in (torch.uint8, torch.bool) and moved.numel() == n:
        mv = moved.to(device=dev, dtype=torch.uint8).contiguous()
    else:
        ids = np.unique(np.asarray(moved, dtype=np.int64))
        if ids.size and (ids[0] < 0 or ids[-1] >= n):
            raise GraphError("frontier member id out of range")
        mv = torch.zeros(n, dtype=torch.uint8, device=dev)
        if ids.size:
            mv[torch.as_tensor(ids, device=dev)] = 1
    co = None if c_old is None else _labels_of(c_old, dg)
    cn = None if c_new is None else _labels_of(c_new, dg)
    out = torch.empty(max(n, 1), dtype=torch.int32, device=dev)
    cnt = ctypes.c_int64()
    gs = dg.c_struct()
    _lib.check(_lib.load().lcc_compute_frontier(ctypes.byref(gs), int(policy), mv.data_ptr(),
                                                None if co is None else co.data_ptr(),
                                                None if cn is None else cn.data_ptr(), out.data_ptr(),
                                                ctypes.byref(cnt), None, stream_ptr()))
    return Frontier(n, out[:cnt.value].clone())


def release_memory() -> None:
    """Return the library's cached device scratch to the driver (calls keep
    up to LCC_POOL_KEEP_GB, default 64 GB, cached between them)."""
    _lib.check(_lib.load().lcc_release_memory())


def frontier_from_mask(mark: torch.Tensor) -> Frontier:
    """Compact a uint8 device mask (e.g. the ``nbr_mark`` of
    ``best_moves_round``) into a sorted Frontier."""
    n = mark.numel()
    out = torch.empty(max(n, 1), dtype=torch.int32, device=mark.device)
    cnt = ctypes.c_int64()
    _lib.check(_lib.load().lcc_frontier_from_mask(n, mark.data_ptr(), out.data_ptr(), ctypes.byref(cnt),
                                                  stream_ptr()))
    return Frontier(n, out[:cnt.value].clone())


# ---------------------------------------------------------------------------
# SPEC operations
# ---------------------------------------------------------------------------

def par_best_moves(g, p: ClusteringParams, c: Clustering | None = None, opts: ParOptions | None = None):
    """SPEC.md:258-266 -> (Clustering, any_moved).  ``c`` is updated in place
    (Clustering is caller-owned and mutable)."""
    opts = opts or ParOptions()
    dg, gs, ps = _prep(g, p)
    if c is None:
        c = singletons(dg.n, p)
    if c.assignment.numel() != dg.n:
        raise GraphError("clustering size does not match the graph")
    if c.cluster_mass.numel() < dg.n:
        raise GraphError("cluster_mass must have n entries")
    anym = ctypes.c_int32()
    st = _lib.LccStats()
    os_ = opts.c_struct()
    _lib.check(_lib.load().lcc_par_best_moves(ctypes.byref(gs), ctypes.byref(ps), ctypes.byref(os_),
                                              c.assignment.data_ptr() if dg.n else None,
                                              c.cluster_mass.data_ptr() if dg.n else None, ctypes.byref(anym),
                                              ctypes.byref(st), stream_ptr()))
    c.meta["stats"] = _stats_from(st)
    return c, bool(anym.value)


def per_vertex_best_target(g, p: ClusteringParams, c: Clustering, v: int, opts: ParOptions | None = None):
    """SPEC.md:296-304 -> (target, moves): target is the chosen cluster id
    (v's own id when staying; n+v denotes a fresh singleton)."""
    opts = opts or ParOptions()
    dg = DeviceGraph.from_graph(g)
    if not 0 <= v < dg.n:
        raise GraphError("vertex id out of range")
    mb = best_moves_round(dg, p, c, frontier=[v], schedule=Schedule.Synchronous,
                          degree_threshold=opts.degree_threshold)
    return int(mb.desired[v].item()), bool(mb.moved[v].item())


def par_compress(g, p, c: Clustering, lam: float | None = None) -> CompressedLevel:
    """SPEC.md:276-282 (same contract as compress).
    ``p`` is a ClusteringParams, or the vertex-weight array k (with ``lam``)."""
    if not isinstance(p, ClusteringParams):
        p = ClusteringParams(0.0 if lam is None else lam, p)
    dg, gs, ps = _prep(g, p)
    lab = _labels_of(c, dg)
    n, nnz = dg.n, dg.nnz
    dev = dg.device
    K = c.cluster_mass if isinstance(c, Clustering) else None
    if K is None or K.numel() < n:
        # raw labels: canonicalise (smallest-member ids) and build masses
        from .objective import clustering_from_labels
        c = clustering_from_labels(lab, p)
        lab, K = c.assignment, c.cluster_mass
    mapping = torch.empty(max(n, 1), dtype=torch.int32, device=dev)
    ck = torch.empty(max(n, 1), dtype=torch.float64, device=dev)
    cptr = torch.empty(n + 1, dtype=torch.int64, device=dev)
    cind = torch.empty(max(nnz, 1), dtype=torch.int32, device=dev)
    cw = torch.empty(max(nnz, 1), dtype=torch.float64, device=dev)
    cn, cnnz = ctypes.c_int64(), ctypes.c_int64()
    off, tot = ctypes.c_double(), ctypes.c_double()
    _lib.check(_lib.load().lcc_par_compress(ctypes.byref(gs), ctypes.byref(ps), lab.data_ptr(), K.data_ptr(),
                                            mapping.data_ptr(), ck.data_ptr(), cptr.data_ptr(), cind.data_ptr(),
                                            cw.data_ptr(), ctypes.byref(cn), ctypes.byref(cnnz),
                                            ctypes.byref(off), ctypes.byref(tot), stream_ptr()))
    cn, cnnz = cn.value, cnnz.value
    cg = DeviceGraph(cn, cnnz // 2, cptr[:cn + 1].clone(), cind[:cnnz].clone(), cw[:cnnz].clone(), tot.value)
    return CompressedLevel(cg, ck[:cn].clone(), mapping[:n].clone(), off.value)


def par_flatten(c: Clustering, c_prime, mapping, p: ClusteringParams | None = None) -> Clustering:
    """assignment[v] = c_prime[mapping[v]], canonicalised,
    masses recomputed (with p.k, or k = 1)."""
    lab = c.assignment if isinstance(c, Clustering) else torch.as_tensor(c)
    dev = _device()
    mapping = _to_dev(mapping, torch.int32, dev)
    cp = c_prime.assignment if isinstance(c_prime, Clustering) else _to_dev(c_prime, torch.int32, dev)
    n = mapping.numel()
    if lab.numel() != n:
        raise GraphError("dimension mismatch between clustering and mapping")
    if n and int(mapping.max().item()) >= cp.numel():
        raise GraphError("mapping refers past the coarse clustering")
    C = torch.empty(n, dtype=torch.int32, device=dev)
    K = torch.empty(n, dtype=torch.float64, device=dev)
    k = None if p is None or p.k is None else p.k
    _lib.check(_lib.load().lcc_par_flatten(n, mapping.data_ptr(), cp.data_ptr(), None if k is None else k.data_ptr(),
                                           C.data_ptr(), K.data_ptr(), stream_ptr()))
    return Clustering(C, K)


def parallel_cc(g, p: ClusteringParams, opts: ParOptions | None = None) -> Clustering:
    """SPEC.md:287-295; Alg. 1 Parallel-CC.  Accepts a reference
    WeightedGraph (host arrays; uploaded here) or a DeviceGraph."""
    opts = opts or ParOptions()
    dg, gs, ps = _prep(g, p)
    C = torch.empty(max(dg.n, 1), dtype=torch.int32, device=dg.device)
    st = _lib.LccStats()
    os_ = opts.c_struct()
    _lib.check(_lib.load().lcc_parallel_cc(ctypes.byref(gs), ctypes.byref(ps), ctypes.byref(os_),
                                           C.data_ptr(), ctypes.byref(st), stream_ptr()))
    C = C[:dg.n]
    from .objective import clustering_from_labels
    out = clustering_from_labels(C, p) if dg.n else Clustering(C, torch.zeros(0, dtype=torch.float64, device=dg.device))
    out.meta["stats"] = _stats_from(st)
    out.meta["seed"] = opts.seed
    return out
