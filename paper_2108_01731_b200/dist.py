"""Vertex-sharded multi-GPU LambdaCC.

One process per GPU.  Vertices are 1-D partitioned into contiguous ranges
balanced by degree sum; each rank keeps only the CSR rows of the vertices it
owns (edges co-located with their source) and a replica of the cluster
labels C and masses K.

Per best-move iteration (Alg. 1 lines 6-10, bulk-synchronous across ranks):
  1. every rank runs the best-move kernels over its owned frontier (an empty
     owned frontier is an empty round: no call);
  2. the mover counts are all-gathered (termination, Alg. 1 line 9); the
     changed labels follow -- as (vertex, label) pairs while movers are
     sparse (< n/64), else as the owned slices of the label array (padded
     equal chunks) -- so every rank holds the full new labelling;
  3. masses K are recomputed locally from the replicated labels (the apply /
     reconcile kernel) -- cheaper than all-reducing a dense fp64 K array, see
     SURVEY.md §8e step 3;
  4. every rank marks the neighbours of its owned movers; the marks are
     MAX-reduce-scattered so each rank receives its owned part, the next
     frontier.
Asynchronous mode is asynchronous inside a GPU and bulk-synchronous across
GPUs.  Synchronous mode gives labels identical to the single-GPU run (Jacobi
rounds do not depend on the partition).

Contraction repartitions the supervertex graph (SURVEY.md
§8e): every rank renumbers identically (labels are replicated), compresses
its owned rows into partial coarse rows, and sends each partial row to the
coarse row's owner (one all-to-all; coarse ranges balanced on the summed
partial row lengths); the owner merges duplicate (a, b) entries with the
device COO merge (lcc_coo_merge) into its shard of the coarse CSR.  Coarse
levels stay sharded until the coarse graph has fewer than ``gather_below``
entries; that remainder is merged on rank 0, clustered there by the
single-GPU driver, and its labels broadcast.  Flatten and refinement run
sharded on every level while unwinding.

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
                             wtype, _lib.GRAPH_PARTIAL_ROWS, part.total_weight)

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
        cw = cw[:cnnz]
        if part.weights is None or part.weights.dtype == torch.int32:
            # integer sums: keep them as int32 (the uint32 tables of the next
            # level) and drop the fp64 buffer (8 -> 4 bytes per entry)
            cw = cw.to(torch.int32)
        return cn, cptr[:cn + 1], cind[:cnnz], cw, ck[:cn], mapping[:n]

    def parallel_cc(self, indptr, indices, weights, total_weight, k, lam, opts):
        from .louvain_par import parallel_cc
        from .objective import ClusteringParams
        n = indptr.numel() - 1
        if weights is not None and weights.dtype not in (torch.int32, torch.float64):
            weights = weights.to(self.device, torch.float64)
        if weights is not None and weights.dtype == torch.float64:
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

    def merge(self, n, rows, cols, w, integral):
        """COO (row, col, w) -> CSR with duplicates summed (lcc_coo_merge);
        integral weights as int32 (exact uint32 sums), else fp64."""
        d = self.device
        nnz = int(rows.numel())
        ip = torch.empty(n + 1, dtype=torch.int64, device=d)
        ind = torch.empty(max(nnz, 1), dtype=torch.int32, device=d)
        wo = torch.empty(max(nnz, 1), dtype=torch.int32 if integral else torch.float64, device=d)
        wi = w.to(d, torch.int32 if integral else torch.float64).contiguous() if nnz else None
        cnt = ctypes.c_int64()
        _lib.check(self.lib.lcc_coo_merge(n, nnz, rows.data_ptr() if nnz else None, cols.data_ptr() if nnz else None,
                                          None if wi is None else wi.data_ptr(),
                                          _lib.W_U32 if integral else _lib.W_F64, ip.data_ptr(), ind.data_ptr(),
                                          wo.data_ptr(), ctypes.byref(cnt), stream_ptr()))
        r = cnt.value
        return ip, ind[:r], wo[:r]

    def flatten(self, mapping, Cc, k):
        n = mapping.numel()
        C = torch.empty(n, dtype=torch.int32, device=self.device)
        K = torch.empty(n, dtype=torch.float64, device=self.device)
        _lib.check(self.lib.lcc_par_flatten(n, mapping.data_ptr(), Cc.to(self.device, torch.int32).data_ptr(),
                                            None if k is None else k.data_ptr(), C.data_ptr(), K.data_ptr(),
                                            stream_ptr()))
        return C, K


# ---------------------------------------------------------------------------
# collectives (NCCL in production; gloo stages CUDA tensors through the host
# for the collectives it has no CUDA path for)
# ---------------------------------------------------------------------------

def _gloo(group) -> bool:
    return dist.get_backend(group) == "gloo"


def _all_gather_ints(vals: list[int], device, group) -> list[list[int]]:
    """Every rank's small int vector (one all-gather, one host read)."""
    world = dist.get_world_size(group)
    if world == 1:
        return [list(vals)]
    dev = torch.device("cpu") if _gloo(group) else device
    t = torch.tensor(vals, dtype=torch.int64, device=dev)
    outs = [torch.empty_like(t) for _ in range(world)]
    dist.all_gather(outs, t, group=group)
    return torch.stack(outs).cpu().tolist()


def _owned_sizes(part, group) -> list[int]:
    """Sizes of every rank's owned range (all-gathered once per PartGraph)."""
    sizes = getattr(part, "_sizes", None)
    if sizes is None:
        sizes = [r[0] for r in _all_gather_ints([part.hi - part.lo], part.indptr.device, group)]
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


def _sparse(movers: int, n: int) -> bool:
    """(vertex, label) pairs cost 8 bytes per mover against 4n for the dense
    slices: pairs below n / LCC_DIST_SPARSE_DIV movers (default 64)."""
    return movers * int(os.environ.get("LCC_DIST_SPARSE_DIV", "64")) < n


def _exchange_labels(labels, moved, part, counts, group) -> torch.Tensor:
    """Full new labelling on every rank.  Sparse rounds (movers < n/64) send
    (vertex, label) pairs of the owned movers; dense rounds all-gather the
    owned slices."""
    world = dist.get_world_size(group)
    if world == 1:
        return labels
    n = part.n
    total = sum(counts)
    if not _sparse(total, n):
        return _allgather_owned(labels, part, group)
    ids = torch.nonzero(moved[part.lo:part.hi]).flatten().to(torch.int32) + part.lo
    mx = max(max(counts), 1)
    buf = torch.full((2, mx), -1, dtype=torch.int32, device=labels.device)
    c = int(ids.numel())
    buf[0, :c] = ids
    buf[1, :c] = labels[ids.long()]
    outs = [torch.empty_like(buf) for _ in range(world)]
    dist.all_gather(outs, buf, group=group)
    pairs = torch.cat([o[:, :k] for o, k in zip(outs, counts)], dim=1)
    lab = labels.clone()
    lab[pairs[0].long()] = pairs[1]
    return lab


def _owned_max(mark: torch.Tensor, part, group) -> torch.Tensor:
    """This rank's slice of the MAX over ranks of ``mark`` (the neighbour
    marks): an NCCL reduce-scatter of padded equal chunks; gloo has no
    reduce-scatter, so it all-reduces."""
    world = dist.get_world_size(group)
    if world == 1:
        return mark[part.lo:part.hi]
    if _gloo(group):
        dist.all_reduce(mark, op=dist.ReduceOp.MAX, group=group)
        return mark[part.lo:part.hi]
    sizes = _owned_sizes(part, group)
    mx = max(sizes)
    inp = torch.zeros(world * mx, dtype=mark.dtype, device=mark.device)
    off = 0
    for r, sz in enumerate(sizes):
        inp[r * mx:r * mx + sz] = mark[off:off + sz]
        off += sz
    out = torch.empty(mx, dtype=mark.dtype, device=mark.device)
    dist.reduce_scatter_tensor(out, inp, op=dist.ReduceOp.MAX, group=group)
    return out[:part.hi - part.lo]


def _all_to_all(inp: torch.Tensor, send: list[int], recv: list[int], group) -> torch.Tensor:
    dev = inp.device
    stage = _gloo(group) and inp.is_cuda
    x = inp.cpu() if stage else inp
    out = torch.empty(sum(recv), dtype=inp.dtype, device=x.device)
    dist.all_to_all_single(out, x.contiguous(), recv, send, group=group)
    return out.to(dev) if stage else out


# ---------------------------------------------------------------------------
# the sharded driver
# ---------------------------------------------------------------------------

@dataclass
class ShardStats:
    rounds: int = 0
    edges_scanned: int = 0   # this rank's owned frontier edges
    moves: int = 0           # global movers
    sharded_levels: int = 0  # levels whose best moves ran sharded (level 0 included)
    gathered_levels: int = 0  # levels merged on rank 0 and clustered there
    sparse_exchanges: int = 0  # iterations that exchanged (vertex, label) pairs


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
    edges = torch.zeros((), dtype=torch.int64, device=dev)  # summed on the device, read once
    num_iter = int(opts.num_iter)
    policy = FrontierPolicy(opts.frontier_policy)
    # VertexNeighbors: the round marks its movers' neighbours itself (the
    # fused nbr_mark of lcc_best_moves_round); backends without it (the test
    # oracle) fall back to frontier_mask
    fused = policy == FrontierPolicy.VertexNeighbors and getattr(backend, "fused_nbr_mark", False)
    for it in range(num_iter):
        nF = int(F.numel())
        mark = torch.zeros(n, dtype=torch.uint8, device=dev) if fused else None
        if nF == 0:
            # empty owned frontier: an empty round, no call (a NULL frontier
            # would mean V' = V); still take part in the collectives
            labels = C if sched == SYNC_ else C.clone()
            moved = torch.zeros(n, dtype=torch.uint8, device=dev)
        elif mark is None:
            labels, moved, _ = backend.round(part, k, lam, C, K, F, sched, int(opts.degree_threshold),
                                             int(opts.async_chunks))
        else:
            # passed on the last iteration too: the round-1 async call measured
            # 10.7 ms with the marks and 11.9 ms without (tools/round_ab.py)
            labels, moved, _ = backend.round(part, k, lam, C, K, F, sched, int(opts.degree_threshold),
                                             int(opts.async_chunks), nbr_mark=mark)
        cnt = int(moved[part.lo:part.hi].sum().item()) if nF else 0
        rows = _all_gather_ints([nF, cnt], dev, group)
        if sum(r[0] for r in rows) == 0:
            break                               # global frontier empty
        counts = [r[1] for r in rows]
        total = sum(counts)
        if stats is not None:
            stats.rounds += 1
            if nF:
                edges += deg.index_select(0, F.long()).sum()
            stats.moves += total
        if total == 0:
            break                               # Alg. 1 line 9
        any_moved = True
        # owners' labels to every rank.  The moved flags need no exchange: a
        # vertex moved iff its label changed (a mover's target differs from
        # its cluster; fresh ids n+v).
        if stats is not None and _sparse(total, n) and dist.get_world_size(group) > 1:
            stats.sparse_exchanges += 1
        lab = _exchange_labels(labels, moved, part, counts, group)
        Cn, Kn = backend.apply(lab, 2 * n, k)   # canonical labels + masses, replicated
        if it + 1 < num_iter:  # the next frontier is only needed by a next iteration
            if policy == FrontierPolicy.AllVertices:
                F = owned
            else:
                if mark is None:
                    mark = backend.frontier_mask(part, int(policy), (lab != C).to(torch.uint8), C, Cn)
                mine = _owned_max(mark, part, group)
                F = (torch.nonzero(mine).flatten() + part.lo).to(torch.int32)
        C, K = Cn, Kn
    if stats is not None:
        stats.edges_scanned += int(edges.item())
    return C, K, any_moved


SYNC_ = 0  # lcc_schedule LCC_SYNC


def _coarse_bounds(cn, cptr, dev, group) -> list[int]:
    """Coarse owner ranges: contiguous, balanced on (vertices + summed
    partial row lengths) like partition_bounds on the coarse graph."""
    world = dist.get_world_size(group)
    lens = (cptr[1:] - cptr[:-1]).to(torch.int64)
    stage = _gloo(group) and lens.is_cuda
    x = lens.cpu() if stage else lens
    dist.all_reduce(x, op=dist.ReduceOp.SUM, group=group)
    lens = x.to(dev) if stage else x
    P = torch.zeros(cn + 1, dtype=torch.int64, device=dev)
    torch.cumsum(lens + 1, 0, out=P[1:])
    total = int(P[-1].item())
    targets = torch.tensor([total * r // world for r in range(1, world)], dtype=torch.int64, device=dev)
    inner = torch.searchsorted(P, targets, right=False).cpu().tolist()
    return [0] + inner + [cn]


def _redistribute(cn, cptr, cind, cw, bounds, integral, backend, group):
    """Send every partial coarse row to its owner (bounds[r]..bounds[r+1]
    belong to rank r) and merge what arrives: (local indptr over the owned
    range, indices, weights).  One all-to-all per array; ids int32, weights
    int32 when integral (12 bytes per entry), else fp64."""
    rank = dist.get_rank(group)
    dev = backend.device
    world = len(bounds) - 1
    starts = cptr[torch.tensor(bounds, dtype=torch.long, device=cptr.device)].cpu().tolist()
    send = [starts[r + 1] - starts[r] for r in range(world)]
    recv = _all_to_all(torch.tensor(send, dtype=torch.int64, device=dev), [1] * world, [1] * world,
                       group).cpu().tolist()
    lens = cptr[1:] - cptr[:-1]
    rows = torch.repeat_interleave(torch.arange(cn, dtype=torch.int32, device=cptr.device), lens)
    wdt = torch.int32 if integral else torch.float64
    r_rows = _all_to_all(rows, send, recv, group)
    r_cols = _all_to_all(cind.to(torch.int32), send, recv, group)
    r_w = _all_to_all(cw.to(wdt), send, recv, group)
    lo, hi = bounds[rank], bounds[rank + 1]
    return backend.merge(hi - lo, (r_rows - lo).to(dev), r_cols.to(dev), r_w.to(dev), integral)


def _full_indptr(lptr, lo, cn, dev):
    """Owned-range indptr -> full-length indptr with empty non-owned rows."""
    nnz = lptr[-1:]
    return torch.cat([torch.zeros(lo, dtype=torch.int64, device=dev), lptr.to(dev),
                      nnz.to(dev).expand(cn - lo - (lptr.numel() - 1))])


def _sum_f64(x: float, dev, group) -> float:
    if dist.get_world_size(group) == 1:
        return float(x)
    t = torch.tensor([x], dtype=torch.float64, device=torch.device("cpu") if _gloo(group) else dev)
    dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
    return float(t.item())


class _Trace:
    """Per-phase wall times of the sharded driver on stderr (LCC_TRACE=1)."""

    def __init__(self, rank, dev):
        self.on = os.environ.get("LCC_TRACE", "0") not in ("", "0")
        self.rank, self.dev = rank, dev
        self.t = time.perf_counter()

    def __call__(self, what):
        if not self.on:
            return
        if self.dev.type == "cuda":
            torch.cuda.synchronize(self.dev)
        t = time.perf_counter()
        print(f"[lcc dist r{self.rank}] {what}: {1e3 * (t - self.t):.1f} ms", file=sys.stderr, flush=True)
        self.t = t


GATHER_BELOW = 64 << 20  # coarse graphs with fewer entries are clustered on rank 0


def sharded_parallel_cc(indptr, indices, weights, total_weight, k, lam, opts, backend=None, group=None,
                        stats: ShardStats | None = None, gather_below: int | None = None) -> torch.Tensor:
    """parallel_cc with every level vertex-sharded over the
    process group until the coarse graph has fewer than ``gather_below``
    entries (default 64M; 0 = never gather).  ``indptr``/``indices``/
    ``weights`` are the full graph (host or device); ``k`` the full vertex
    weights (or None).  Returns the canonical labels (replicated on every
    rank)."""
    backend = backend or CudaBackend()
    dev = backend.device
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    if gather_below is None:
        gather_below = int(os.environ.get("LCC_DIST_GATHER_NNZ", GATHER_BELOW))
    tr = _Trace(rank, dev)
    ip = np.asarray(indptr.cpu() if isinstance(indptr, torch.Tensor) else indptr, dtype=np.int64)
    bounds = partition_bounds(ip, world)
    part = make_part(indptr, indices, weights, total_weight, int(bounds[rank]), int(bounds[rank + 1]), dev)
    if k is not None:
        k = torch.as_tensor(k, dtype=torch.float64).to(dev)
    tr("upload")
    stack = []            # (part, k, mapping) of every contracted level
    cur, kcur = part, k
    level = 0
    while True:
        n = cur.n
        C = torch.arange(n, dtype=torch.int32, device=dev)
        K = torch.ones(n, dtype=torch.float64, device=dev) if kcur is None else kcur.clone()
        C, K, moved = sharded_best_moves(cur, kcur, lam, C, K, opts, backend, group, stats)
        if stats is not None:
            stats.sharded_levels += 1
        tr(f"level {level} best moves")
        if not moved:
            break                                     # Alg. 1 line 13
        cn, cptr, cind, cw, ck, mapping = backend.compress(cur, kcur, lam, C, K)
        tr(f"level {level} compress")
        if cn == n:
            break                                     # no size reduction
        integral = cur.weights is None or cur.weights.dtype == torch.int32
        stack.append((cur, kcur, mapping))
        gnnz = int(round(_sum_f64(float(cind.numel()), dev, group)))
        # (world size 1 runs the coarse levels in the single-GPU driver unless
        # gather_below == 0 asks for the sharded path: tests of the NCCL code)
        if gnnz < gather_below or (world == 1 and gather_below > 0):
            # the remainder on rank 0: single-GPU driver, labels broadcast
            Cc = torch.empty(cn, dtype=torch.int32, device=dev)
            if world == 1:
                Cc = backend.parallel_cc(cptr, cind, cw, float(cw.sum().item()) / 2.0, ck, lam, opts).to(torch.int32)
            else:
                lptr, lind, lw = _redistribute(cn, cptr, cind, cw, [0] + [cn] * world, integral, backend, group)
                if rank == 0:
                    Cc = backend.parallel_cc(lptr, lind, lw, float(lw.to(torch.float64).sum().item()) / 2.0, ck,
                                             lam, opts).to(torch.int32)
                dist.broadcast(Cc, src=0, group=group)
            if stats is not None:
                stats.gathered_levels += 1
            C = Cc
            tr(f"levels {level + 1}+ on rank 0")
            break
        # repartition the supervertex graph and stay sharded
        cb = _coarse_bounds(cn, cptr, dev, group)
        lptr, lind, lw = _redistribute(cn, cptr, cind, cw, cb, integral, backend, group)
        del cptr, cind, cw
        tw = _sum_f64(float(lw.to(torch.float64).sum().item()), dev, group) / 2.0
        cur = PartGraph(cn, cb[rank], cb[rank + 1], _full_indptr(lptr, cb[rank], cn, dev), lind, lw, tw)
        kcur = ck
        level += 1
        tr(f"level {level} repartition")
    # unwind: flatten + refine level by level (Alg. 1 lines 17-18)
    for lvl, kl, mapping in reversed(stack):
        C, K = backend.flatten(mapping, C, kl)
        if opts.refine:
            C, K, _ = sharded_best_moves(lvl, kl, lam, C, K, opts, backend, group, stats)
        tr(f"unwind n={lvl.n}")
    return C
