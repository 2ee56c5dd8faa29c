"""bench.py's CPU legs on the host (no GPU): the vertex sample the CPU
baseline and the reference arm time (every stride-th vertex keeps its full
row, all other rows empty) and the phase timer."""
import numpy as np
import torch

import bench
from oracle import oracle as O
from paper_2108_01731_b200.gen import csr_from_pairs, rmat_pairs_host


class _G:
    pass


def _graph():
    u, v = rmat_pairs_host(11, 8 << 11, 0.57, 0.19, 0.19, 5)
    return csr_from_pairs(1 << 11, u, v)


def test_sample_rows_keeps_full_rows():
    hg = _graph()
    g = _G()
    g.n, g.m = hg.n, hg.indices.size // 2
    g.indptr, g.indices = torch.from_numpy(hg.indptr), torch.from_numpy(hg.indices)
    for stride in (1, 3, 8):
        ip, ix, nF, edges = bench.sample_rows(g, stride)
        assert nF == (hg.n + stride - 1) // stride and ix.size == edges == ip[-1]
        for v in range(hg.n):
            row = ix[ip[v]:ip[v + 1]]
            want = hg.indices[hg.indptr[v]:hg.indptr[v + 1]] if v % stride == 0 else hg.indices[:0]
            assert np.array_equal(row, want), (stride, v)


def test_cpu_round_on_sample_equals_full_graph_round():
    """The sampled rows are all a round over the sample reads (singleton
    start: neighbour labels are their ids), so the sample's sync round
    equals the full graph's round restricted to the sample."""
    hg = _graph()
    g = O.as_graph(hg)
    n, stride = hg.n, 4
    keep = np.zeros(n, bool)
    keep[::stride] = True
    deg = np.diff(hg.indptr)
    ip = np.zeros(n + 1, np.int64)
    np.cumsum(np.where(keep, deg, 0), out=ip[1:])
    ix = hg.indices[np.repeat(keep, deg)]
    sg = bench.sample_graph(ip, np.ascontiguousarray(ix, np.int32), n, hg.indices.size // 2)
    F = np.arange(0, n, stride, dtype=np.int32)
    D1, m1, c1 = O.sync_round(sg, None, 0.85, np.arange(n, dtype=np.int32), np.ones(n), F)
    D2, m2, c2 = O.sync_round(g, None, 0.85, np.arange(n, dtype=np.int32), np.ones(n), F)
    assert c1 == c2 and np.array_equal(D1, D2) and np.array_equal(m1, m2)
    ph = bench.cpu_phases(sg, None, 0.85, "async", stride)
    assert ph["objective_entries"] == ix.size and ph["apply_s"] >= 0 and ph["compress_entries"] <= ix.size
