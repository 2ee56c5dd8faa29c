"""Vertex-sharded multi-GPU LambdaCC.

One process per GPU.  Vertices are 1-D partitioned into contiguous ranges
balanced by degree sum; each rank keeps only the CSR rows of the vertices it
owns (edges co-located with their source) and a replica of the cluster
labels C and masses K.

Per best-move iteration (Alg. 1 lines 6-10, bulk-synchronous across ranks):
  1. every rank runs the best-move kernels over its owned frontier;
  2. the owned slices of the new labels are all-gathered over NCCL (padded
     equal chunks), so every rank holds the full new labelling; the moved
     flags follow locally (label changed);
  3. masses K are recomputed locally from the replicated labels (the apply /
     reconcile kernel) -- cheaper than all-reducing a dense fp64 K array, see
     SURVEY.md §8e step 3;
  4. every rank marks the neighbours of its owned movers, the marks are
     MAX-all-reduced, and each rank keeps its owned part as the next frontier.
Asynchronous mode is asynchronous inside a GPU and bulk-synchronous across
GPUs.  Synchronous mode gives labels identical to the single-GPU run (Jacobi
rounds do not depend on the partition).

Contraction: each rank compresses its owned rows with the device kernel
(renumbering is identical everywhere since labels are replicated); the
partial coarse CSRs are all-gathered and merged, the coarse levels run on
rank 0 (they are a small fraction of the work) and the coarse labels are
broadcast; flatten and the level-0 refinement run sharded again.

The per-rank compute goes through a backend object (``CudaBackend`` here:
the sm_100a C ABI).  Tests drive the same driver with a CPU backend over
``gloo`` to check the exchange logic without GPUs.
"""
from __future__ import annotations

import ctypes
import os
import sys
import time
from dataclasses import dataclass

import numpy as np
import torch
import torch.distributed as dist

from . import _lib
from .graph import DeviceGraph, stream_ptr


# ---------------------------------------------------------------------------
# partitioning
# ---------------------------------------------------------------------------

def partition_bounds(indptr: np.ndarray, parts: int) -> np.ndarray:
    """Contiguous vertex ranges with (vertex count + degree sum) balanced.
    Returns bounds[parts+1]; rank r owns [bounds[r], bounds[r+1])."""
    indptr = np.asarray(indptr, dtype=np.int64)
    n = indptr.size - 1
    # work(i) = indptr[i] + i (vertices + edges prefix) is increasing: bisect
    # it per target instead of materialising it (n is up to 65M on the host)
    total = int(indptr[-1]) + n
    targets = (total * np.arange(1, parts, dtype=np.float64) / parts).astype(np.int64)
    inner = []
    for t in targets.tolist():     # first i with work(i) >= t (searchsorted "left")
        lo, hi = 0, n + 1
        while lo < hi:
            mid = (lo + hi) // 2
            if int(indptr[mid]) + mid < t:
                lo = mid + 1
            else:
                hi = mid
        inner.append(lo)
    return np.asarray([0] + inner + [n], dtype=np.int64)


@dataclass
class PartGraph:
    """Owned rows of a symmetric CSR: indptr covers all n vertices (rows
    outside [lo, hi) are empty), indices/weights hold the owned rows only."""
    n: int
    lo: int
    hi: int
    indptr: torch.Tensor
    indices: torch.Tensor
    weights: torch.Tensor | None
    total_weight: float

    @property
    def m(self) -> int:
        return int(self.indices.numel()) // 2


def make_part(indptr, indices, weights, total_weight, lo: int, hi: int, device) -> PartGraph:
    """Build the owned-rows view from full host (numpy) or torch CSR arrays."""
    ip = indptr if isinstance(indptr, torch.Tensor) else torch.as_tensor(np.asarray(indptr, dtype=np.int64))
    n = ip.numel() - 1
    s, e = int(ip[lo]), int(ip[hi])
    # upload first (a pinned host indptr copies at full speed), clamp on the device
    pip = ip.to(device=device, dtype=torch.int64).clamp(min=s, max=e) - s
    ind = indices[s:e] if isinstance(indices, torch.Tensor) else torch.as_tensor(np.asarray(indices[s:e]))
    ind = ind.to(device=device, dtype=torch.int32).contiguous()
    w = None
    if weights is not None:
        ww = weights[s:e] if isinstance(weights, torch.Tensor) else torch.as_tensor(np.asarray(weights[s:e]))
        w = ww.to(device).contiguous()
    return PartGraph(n, lo, hi, pip, ind, w, float(total_weight))


# ---------------------------------------------------------------------------
# CUDA backend: the per-rank compute, all through the C ABI
# ---------------------------------------------------------------------------

class CudaBackend:
    fused_nbr_mark = True

    def __init__(self, device=None):
        self.device = torch.device("cuda", torch.cuda.current_device()) if device is None else torch.device(device)
        self.lib = _lib.load()

    def _g(self, part) -> _lib.LccGraph:
        wtype, wp = _lib.W_NONE, None
        if part.weights is not None:
            wtype = {torch.float32: _lib.W_F32, torch.int32: _lib.W_U32}.get(part.weights.dtype, _lib.W_F64)
            wp = part.weights.data_ptr()
        nnz = int(part.indices.numel())
        return _lib.LccGraph(part.n, nnz, part.indptr.data_ptr(), part.indices.data_ptr() if nnz else None, wp,
                             wtype, 0, part.total_weight)

    @staticmethod
    def _p(k, lam) -> _lib.LccParams:
        return _lib.LccParams(None if k is None else k.data_ptr(), float(lam))

    def round(self, part, k, lam, C, K, frontier, schedule, thr, chunks, nbr_mark=None):
        """Returns (labels, moved, count): sync -> D; async -> C updated in a
        copy with masses in a 2n copy of K.  ``nbr_mark`` (n bytes, optional)
        receives the VertexNeighbors marks of this rank's movers, fused into
        the round."""
        n = part.n
        g, p = self._g(part), self._p(k, lam)
        nm = None if nbr_mark is None else nbr_mark.data_ptr()
        moved = torch.empty(n, dtype=torch.uint8, device=self.device)
        cnt = ctypes.c_int64()
        fr = frontier.to(self.device, torch.int32).contiguous()
        if schedule == _lib.SYNC:
            D = torch.empty(n, dtype=torch.int32, device=self.device)
            _lib.check(self.lib.lcc_best_moves_round(ctypes.byref(g), ctypes.byref(p), C.data_ptr(), K.data_ptr(),
                                                     fr.data_ptr() if fr.numel() else None, fr.numel(),
                                                     _lib.SYNC, thr, chunks, D.data_ptr(), moved.data_ptr(), nm,
                                                     ctypes.byref(cnt), None, stream_ptr()))
            return D, moved, cnt.value
        Cw = C.clone()
        K2 = torch.zeros(2 * n, dtype=torch.float64, device=self.device)
        K2[:n] = K
        _lib.check(self.lib.lcc_best_moves_round(ctypes.byref(g), ctypes.byref(p), Cw.data_ptr(), K2.data_ptr(),
                                                 fr.data_ptr() if fr.numel() else None, fr.numel(),
                                                 _lib.ASYNC, thr, chunks, None, moved.data_ptr(), nm,
                                                 ctypes.byref(cnt), None, stream_ptr()))
        return Cw, moved, cnt.value

    def apply(self, labels, label_range, k):
        n = labels.numel()
        C = torch.empty(n, dtype=torch.int32, device=self.device)
        K = torch.empty(n, dtype=torch.float64, device=self.device)
        _lib.check(self.lib.lcc_apply_moves(n, labels.data_ptr(), int(label_range),
                                            None if k is None else k.data_ptr(), C.data_ptr(), K.data_ptr(),
                                            stream_ptr()))
        return C, K

    def frontier_mask(self, part, policy, moved, Cold, Cnew):
        n = part.n
        g = self._g(part)
        out = torch.empty(max(n, 1), dtype=torch.int32, device=self.device)
        cnt = ctypes.c_int64()
        _lib.check(self.lib.lcc_compute_frontier(ctypes.byref(g), int(policy), moved.data_ptr(), Cold.data_ptr(),
                                                 Cnew.data_ptr(), out.data_ptr(), ctypes.byref(cnt), None, stream_ptr()))
        mask = torch.zeros(n, dtype=torch.uint8, device=self.device)
        if cnt.value:
            mask[out[:cnt.value].long()] = 1
        return mask

    def compress(self, part, k, lam, C, K):
        n, nnz = part.n, int(part.indices.numel())
        d = self.device
        mapping = torch.empty(max(n, 1), dtype=torch.int32, device=d)
        ck = torch.empty(max(n, 1), dtype=torch.float64, device=d)
        cptr = torch.empty(n + 1, dtype=torch.int64, device=d)
        cind = torch.empty(max(nnz, 1), dtype=torch.int32, device=d)
        cw = torch.empty(max(nnz, 1), dtype=torch.float64, device=d)
        cn, cnnz, off, tot = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_double(), ctypes.c_double()
        g, p = self._g(part), self._p(k, lam)
        _lib.check(self.lib.lcc_par_compress(ctypes.byref(g), ctypes.byref(p), C.data_ptr(), K.data_ptr(),
                                             mapping.data_ptr(), ck.data_ptr(), cptr.data_ptr(), cind.data_ptr(),
                                             cw.data_ptr(), ctypes.byref(cn), ctypes.byref(cnnz), ctypes.byref(off),
                                             ctypes.byref(tot), stream_ptr()))
        cn, cnnz = cn.value, cnnz.value
        return cn, cptr[:cn + 1], cind[:cnnz], cw[:cnnz], ck[:cn], mapping[:n]

    def parallel_cc(self, indptr, indices, weights, total_weight, k, lam, opts):
        from .louvain_par import parallel_cc
        from .objective import ClusteringParams
        n = indptr.numel() - 1
        if weights is not None and weights.dtype != torch.int32:
            weights = weights.to(self.device, torch.float64)
            # integral coarse weights (multi-edge counts of an unweighted or
            # integer-weighted level 0) run on the exact uint32 tables, as in
            # the single-process driver
            if weights.numel() and bool((weights == weights.round()).all()) and \
                    float(weights.min()) >= 0 and float(weights.max()) < 2.0 ** 31:
                weights = weights.to(torch.int32)
        g = DeviceGraph(n, indices.numel() // 2, indptr.to(self.device), indices.to(self.device, torch.int32),
                        None if weights is None else weights.to(self.device), float(total_weight))
        p = ClusteringParams.__new__(ClusteringParams)
        p.lam, p.k = float(lam), k
        return parallel_cc(g, p, opts).assignment

    def flatten(self, mapping, Cc, k):
        n = mapping.numel()
        C = torch.empty(n, dtype=torch.int32, device=self.device)
        K = torch.empty(n, dtype=torch.float64, device=self.device)
        _lib.check(self.lib.lcc_par_flatten(n, mapping.data_ptr(), Cc.to(self.device, torch.int32).data_ptr(),
                                            None if k is None else k.data_ptr(), C.data_ptr(), K.data_ptr(),
                                            stream_ptr()))
        return C, K


# ---------------------------------------------------------------------------
# the sharded driver
# ---------------------------------------------------------------------------

def _max_(t: torch.Tensor, group):
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return t


def _sum_int(x: int, device, group) -> int:
    if dist.get_world_size(group) == 1:
        return int(x)
    t = torch.tensor([x], dtype=torch.int64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
    return int(t.item())


def _owned_sizes(part, group) -> list[int]:
    """Sizes of every rank's owned range (all-gathered once per PartGraph)."""
    sizes = getattr(part, "_sizes", None)
    if sizes is None:
        world = dist.get_world_size(group)
        dev = part.indptr.device
        t = torch.tensor([part.hi - part.lo], dtype=torch.int64, device=dev)
        outs = [torch.empty_like(t) for _ in range(world)]
        dist.all_gather(outs, t, group=group)
        sizes = [int(o.item()) for o in outs]
        part._sizes = sizes
    return sizes


def _allgather_owned(vals: torch.Tensor, part, group) -> torch.Tensor:
    """The owned slice of ``vals`` from every rank, concatenated in rank order
    (the ranges are contiguous and ordered, so this is the full array): one
    NCCL all-gather of padded equal-size chunks."""
    if dist.get_world_size(group) == 1:
        return vals
    sizes = _owned_sizes(part, group)
    mx = max(sizes)
    buf = torch.empty(mx, dtype=vals.dtype, device=vals.device)
    buf[:part.hi - part.lo] = vals[part.lo:part.hi]
    outs = [torch.empty_like(buf) for _ in sizes]
    dist.all_gather(outs, buf, group=group)
    return torch.cat([o[:sz] for o, sz in zip(outs, sizes)])


@dataclass
class ShardStats:
    rounds: int = 0
    edges_scanned: int = 0   # this rank's owned frontier edges
    moves: int = 0           # global movers


def sharded_best_moves(part: PartGraph, k, lam, C, K, opts, backend, group=None, stats: ShardStats | None = None):
    """par_best_moves over the owned vertices of every rank (module doc)."""
    from .louvain_par import FrontierPolicy
    dev = backend.device
    n = part.n
    owned = torch.arange(part.lo, part.hi, dtype=torch.int32, device=dev)
    F = owned                                   # V' <- V
    sched = int(opts.schedule)
    any_moved = False
    deg = (part.indptr[1:] - part.indptr[:-1])
    num_iter = int(opts.num_iter)
    policy = FrontierPolicy(opts.frontier_policy)
    # VertexNeighbors: the round marks its movers' neighbours itself (the
    # fused nbr_mark of lcc_best_moves_round); backends without it (the test
    # oracle) fall back to frontier_mask
    fused = policy == FrontierPolicy.VertexNeighbors and getattr(backend, "fused_nbr_mark", False)
    for it in range(num_iter):
        if _sum_int(int(F.numel()), dev, group) == 0:
            break
        # passed on the last iteration too: the round-1 async call measured
        # 10.7 ms with the marks and 11.9 ms without (tools/round_ab.py)
        mark = torch.empty(n, dtype=torch.uint8, device=dev) if fused else None
        if mark is None:
            labels, moved, cnt = backend.round(part, k, lam, C, K, F, sched, int(opts.degree_threshold),
                                               int(opts.async_chunks))
        else:
            labels, moved, cnt = backend.round(part, k, lam, C, K, F, sched, int(opts.degree_threshold),
                                               int(opts.async_chunks), nbr_mark=mark)
        if stats is not None:
            stats.rounds += 1
            stats.edges_scanned += int(deg.index_select(0, F).sum().item()) if F.numel() else 0
        total = _sum_int(int(cnt), dev, group)
        if stats is not None:
            stats.moves += total
        if total == 0:
            break                               # Alg. 1 line 9
        any_moved = True
        # owners' labels to every rank (one all-gather of the owned slices).
        # The moved flags need no exchange: a vertex moved iff its label
        # changed (a mover's target differs from its cluster; fresh ids n+v).
        lab = _allgather_owned(labels, part, group)
        Cn, Kn = backend.apply(lab, 2 * n, k)   # canonical labels + masses, replicated
        if it + 1 < num_iter:  # the next frontier is only needed by a next iteration
            if policy == FrontierPolicy.AllVertices:
                F = owned
            elif mark is not None:
                _max_(mark, group)
                F = (torch.nonzero(mark[part.lo:part.hi]).flatten() + part.lo).to(torch.int32)
            else:
                mv = (lab != C).to(torch.uint8)
                mask = backend.frontier_mask(part, int(policy), mv, C, Cn)
                _max_(mask, group)
                F = (torch.nonzero(mask[part.lo:part.hi]).flatten() + part.lo).to(torch.int32)
        C, K = Cn, Kn
    return C, K, any_moved


def _gather_coarse(cn, cptr, cind, cw, device, group, integral=False):
    """Gather the partial coarse CSRs on rank 0 (NCCL gather, not an
    all-gather: only rank 0 runs the coarse levels); rank 0 merges duplicate
    (a, b) entries and returns the coarse CSR (other ranks return None).
    Ids travel as int32 (cn < 2^31) and, when the level-0 weights are
    integral (unweighted or LCC_W_U32), weights as int32 too: 12 bytes per
    entry instead of 24."""
    world = dist.get_world_size(group)
    if world == 1:
        return cptr, cind, cw, float(cw.sum().item()) / 2.0
    rank = dist.get_rank(group)
    rows = torch.repeat_interleave(torch.arange(cn, device=device, dtype=torch.int32), cptr[1:] - cptr[:-1])
    local = torch.stack([rows, cind.to(torch.int32)]).contiguous()
    size = torch.tensor([local.shape[1]], dtype=torch.int64, device=device)
    sizes = [torch.zeros_like(size) for _ in range(world)]
    dist.all_gather(sizes, size, group=group)
    sizes = [int(x.item()) for x in sizes]
    mx = max(sizes)
    wdt = torch.int32 if integral else torch.float64
    pad_i = torch.full((2, mx), -1, dtype=torch.int32, device=device)
    pad_i[:, :local.shape[1]] = local
    pad_w = torch.zeros(mx, dtype=wdt, device=device)
    pad_w[:cw.numel()] = cw.to(wdt)
    gi = [torch.empty_like(pad_i) for _ in range(world)] if rank == 0 else None
    gw = [torch.empty_like(pad_w) for _ in range(world)] if rank == 0 else None
    dist.gather(pad_i, gi, dst=0, group=group)
    dist.gather(pad_w, gw, dst=0, group=group)
    if rank != 0:
        return None  # the coarse levels run on rank 0 only
    ab = torch.cat([g[:, :sz] for g, sz in zip(gi, sizes)], dim=1).to(torch.int64)
    w = torch.cat([g[:sz] for g, sz in zip(gw, sizes)])
    del gi, gw
    key = ab[0] * max(cn, 1) + ab[1]
    del ab
    key, order = torch.sort(key, stable=True)
    w = w[order].to(torch.int64 if integral else torch.float64)
    uk, inv = torch.unique_consecutive(key, return_inverse=True)
    ws = torch.zeros(uk.numel(), dtype=w.dtype, device=device).index_add_(0, inv, w).to(torch.float64)
    a, b = uk // max(cn, 1), uk % max(cn, 1)
    indptr = torch.zeros(cn + 1, dtype=torch.int64, device=device)
    indptr[1:] = torch.cumsum(torch.bincount(a, minlength=cn), 0)
    return indptr, b.to(torch.int32), ws, float(ws.sum().item()) / 2.0


class _Trace:
    """Per-phase wall times of the sharded driver on stderr (LCC_TRACE=1)."""

    def __init__(self, rank, dev):
        self.on = os.environ.get("LCC_TRACE", "0") not in ("", "0")
        self.rank, self.dev = rank, dev
        self.t = time.perf_counter()

    def __call__(self, what):
        if not self.on:
            return
        torch.cuda.synchronize(self.dev)
        t = time.perf_counter()
        print(f"[lcc dist r{self.rank}] {what}: {1e3 * (t - self.t):.1f} ms", file=sys.stderr, flush=True)
        self.t = t


def sharded_parallel_cc(indptr, indices, weights, total_weight, k, lam, opts, backend=None, group=None,
                        stats: ShardStats | None = None) -> torch.Tensor:
    """parallel_cc with level 0 sharded over the process
    group.  ``indptr``/``indices``/``weights`` are the full graph (host or
    device); ``k`` the full vertex weights (or None).  Returns the canonical
    labels (replicated on every rank)."""
    backend = backend or CudaBackend()
    dev = backend.device
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    tr = _Trace(rank, dev)
    ip = np.asarray(indptr.cpu() if isinstance(indptr, torch.Tensor) else indptr, dtype=np.int64)
    bounds = partition_bounds(ip, world)
    part = make_part(indptr, indices, weights, total_weight, int(bounds[rank]), int(bounds[rank + 1]), dev)
    n = part.n
    if k is not None:
        k = torch.as_tensor(k, dtype=torch.float64).to(dev)
    C = torch.arange(n, dtype=torch.int32, device=dev)
    K = torch.ones(n, dtype=torch.float64, device=dev) if k is None else k.clone()
    tr("upload")
    C, K, moved = sharded_best_moves(part, k, lam, C, K, opts, backend, group, stats)
    tr("level 0")
    if not moved:
        return C
    cn, cptr, cind, cw, ck, mapping = backend.compress(part, k, lam, C, K)
    tr("compress")
    if cn == n:
        return C                                      # no size reduction
    integral = part.weights is None or part.weights.dtype == torch.int32
    merged = _gather_coarse(cn, cptr, cind, cw, dev, group, integral)
    tr("gather coarse")
    Cc = torch.empty(cn, dtype=torch.int32, device=dev)
    if rank == 0:
        c_indptr, c_ind, c_w, c_tot = merged
        Cc = backend.parallel_cc(c_indptr, c_ind, c_w, c_tot, ck, lam, opts).to(torch.int32)
    tr("coarse levels")
    dist.broadcast(Cc, src=0, group=group)
    C, K = backend.flatten(mapping, Cc, k)
    if opts.refine:
        C, K, _ = sharded_best_moves(part, k, lam, C, K, opts, backend, group, stats)
    tr("flatten + refine")
    return C

