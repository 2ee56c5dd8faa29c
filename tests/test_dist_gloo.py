"""Sharded multi-GPU driver (dist.py) on CPU: world_size 2 over gloo with the
oracle as the per-rank compute.  Synchronous mode must reproduce the
single-process clustering exactly (Jacobi rounds are partition independent);
asynchronous mode must produce a valid clustering of comparable objective."""
import os
import socket
import tempfile

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

from oracle import oracle as O
from paper_2108_01731_b200.dist import ShardStats, partition_bounds, sharded_parallel_cc
from paper_2108_01731_b200.gen import csr_from_pairs, lfr_like, rmat_pairs_host, sbm
from paper_2108_01731_b200.louvain_par import ParOptions

from tests.dist_helpers import OracleBackend, run_rank


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _cluster(rank, world, indptr, indices, k, lam, opts_kw):
    opts = ParOptions(**opts_kw)
    st = ShardStats()
    C = sharded_parallel_cc(indptr, indices, None, float(indices.size // 2), k, lam, opts,
                            backend=OracleBackend(), stats=st)
    return {"C": C.numpy(), "rounds": st.rounds}


def run_world(world, fn, *args):
    out = tempfile.mktemp(suffix=".pt")
    mp.spawn(run_rank, args=(world, free_port(), fn, args, out), nprocs=world, join=True)
    res = torch.load(out, weights_only=False)
    os.remove(out)
    return res


def test_partition_bounds_balanced():
    hg, _ = lfr_like(n=20_000, seed=3)
    b = partition_bounds(hg.indptr, 4)
    assert b[0] == 0 and b[-1] == hg.n and np.all(np.diff(b) > 0)
    work = hg.indptr[b[1:]] - hg.indptr[b[:-1]] + np.diff(b)
    assert work.max() < 1.2 * work.mean()


def test_partition_bounds_matches_prefix_search():
    """The bisection over work(i) = indptr[i] + i equals a searchsorted over
    the materialised prefix, including empty graphs, more parts than
    vertices and runs of isolated vertices."""
    rng = np.random.default_rng(7)
    for n in [0, 1, 3, 100, 5000]:
        for parts in [1, 2, 3, 8]:
            deg = rng.integers(0, 20, n) * (rng.random(n) < 0.7)
            ip = np.concatenate([[0], np.cumsum(deg)]).astype(np.int64)
            work = ip + np.arange(n + 1)
            t = (work[-1] * np.arange(1, parts, dtype=np.float64) / parts).astype(np.int64)
            ref = np.concatenate([[0], np.searchsorted(work, t, side="left"), [n]])
            assert np.array_equal(partition_bounds(ip, parts), ref), (n, parts)


@pytest.mark.parametrize("policy", ["vertex-nbrs", "all", "cluster-nbrs"])
def test_sharded_sync_equals_single_process(policy):
    hg, _ = sbm(seed=1)
    g = O.as_graph(hg)
    pol = {"vertex-nbrs": O.VERTEX_NBRS, "all": O.ALL, "cluster-nbrs": O.CLUSTER_NBRS}[policy]
    ref = O.parallel_cc(g, None, 0.85, O.Opts(schedule=O.SYNC, frontier=pol))
    res = run_world(2, _cluster, hg.indptr, hg.indices, None, 0.85,
                    dict(schedule="sync", frontier_policy=policy))
    assert np.array_equal(res["C"], ref)


def test_sharded_sync_modularity_rmat():
    u, v = rmat_pairs_host(12, 16 << 12, 0.57, 0.19, 0.19, 8)
    hg = csr_from_pairs(1 << 12, u, v)
    g = O.as_graph(hg)
    k, lam = O.modularity_params(g, 1.0)
    ref = O.parallel_cc(g, k, lam, O.Opts(schedule=O.SYNC))
    res = run_world(2, _cluster, hg.indptr, hg.indices, torch.from_numpy(k), lam, dict(schedule="sync"))
    assert np.array_equal(res["C"], ref)


def test_sharded_async_valid_and_close():
    u, v = rmat_pairs_host(12, 16 << 12, 0.57, 0.19, 0.19, 9)
    hg = csr_from_pairs(1 << 12, u, v)
    g = O.as_graph(hg)
    ref = O.objective(g, None, 0.85, O.parallel_cc(g, None, 0.85, O.Opts(schedule=O.ASYNC)))
    res = run_world(2, _cluster, hg.indptr, hg.indices, None, 0.85, dict(schedule="async"))
    C = res["C"]
    assert C.min() >= 0 and C.max() < g.n and np.all(C[C] == C)
    got = O.objective(g, None, 0.85, C)
    assert got >= ref - 0.005 * abs(ref), (got, ref)
