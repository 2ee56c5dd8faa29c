"""Sharded driver with the CUDA backend.  Only one GPU is available, so two
ranks share it over gloo (collectives on the host; no kernel ever waits on
another rank), and a single-rank NCCL group exercises the NCCL code path."""
import os
import tempfile

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

from oracle import oracle as O
from paper_2108_01731_b200.gen import csr_from_pairs, rmat_pairs_host, sbm

from tests.test_dist_gloo import free_port

pytestmark = pytest.mark.gpu


def _rank_main(rank, world, port, backend_name, indptr, indices, lam, opts_kw, out, gather_below=None,
               level0=False):
    import torch.distributed as dist
    from paper_2108_01731_b200.dist import CudaBackend, ShardStats, sharded_parallel_cc
    from paper_2108_01731_b200.louvain_par import ParOptions
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group(backend_name, rank=rank, world_size=world)
    try:
        st = ShardStats()
        if level0:  # level 0 alone (sharded_best_moves)
            from paper_2108_01731_b200.dist import make_part, partition_bounds, sharded_best_moves
            b = partition_bounds(indptr, world)
            part = make_part(indptr, indices, None, float(indices.size // 2), int(b[rank]), int(b[rank + 1]),
                             torch.device("cuda", 0))
            n = part.n
            C, _, _ = sharded_best_moves(part, None, lam, torch.arange(n, dtype=torch.int32, device="cuda"),
                                         torch.ones(n, dtype=torch.float64, device="cuda"), ParOptions(**opts_kw),
                                         CudaBackend(), None, st)
        else:
            C = sharded_parallel_cc(indptr, indices, None, float(indices.size // 2), None, lam,
                                    ParOptions(**opts_kw), backend=CudaBackend(), stats=st, gather_below=gather_below)
        if rank == 0:
            torch.save({"C": C.cpu().numpy(), "rounds": st.rounds, "moves": st.moves,
                        "sharded_levels": st.sharded_levels}, out)
    finally:
        dist.destroy_process_group()


def run(world, backend_name, hg, lam, opts_kw, gather_below=None, level0=False):
    out = tempfile.mktemp(suffix=".pt")
    mp.spawn(_rank_main, args=(world, free_port(), backend_name, hg.indptr, hg.indices, lam, opts_kw, out,
                               gather_below, level0),
             nprocs=world, join=True)
    r = torch.load(out, weights_only=False)
    os.remove(out)
    return r


@pytest.mark.parametrize("world,backend_name", [(2, "gloo"), (1, "nccl")])
@pytest.mark.parametrize("policy", ["vertex", "cluster"])
def test_sharded_cuda_sync_exact(world, backend_name, policy):
    """VertexNeighbors runs the fused neighbour marks of the round,
    ClusterNeighbors the separate compute_frontier; both bit-exact."""
    from paper_2108_01731_b200.louvain_par import FrontierPolicy
    fp = FrontierPolicy.VertexNeighbors if policy == "vertex" else FrontierPolicy.ClusterNeighbors
    hg, _ = sbm(seed=1)
    g = O.as_graph(hg)
    ref = O.parallel_cc(g, None, 0.85, O.Opts(schedule=O.SYNC, frontier=int(fp)))
    r = run(world, backend_name, hg, 0.85, dict(schedule="sync", frontier_policy=fp))
    assert np.array_equal(r["C"], ref)


def test_sharded_cuda_async_objective():
    u, v = rmat_pairs_host(13, 16 << 13, 0.57, 0.19, 0.19, 10)
    hg = csr_from_pairs(1 << 13, u, v)
    g = O.as_graph(hg)
    ref = O.objective(g, None, 0.85, O.parallel_cc(g, None, 0.85, O.Opts(schedule=O.ASYNC)))
    r = run(2, "gloo", hg, 0.85, dict(schedule="async"))
    got = O.objective(g, None, 0.85, r["C"])
    assert got >= ref - 0.005 * abs(ref), (got, ref)


@pytest.mark.parametrize("world,backend_name", [(2, "gloo"), (1, "nccl")])
def test_sharded_cuda_levels_exact(world, backend_name):
    """Every coarse level repartitioned (gather_below=0): the all-to-all of
    partial coarse rows and the device COO merge (lcc_coo_merge) on each
    owner; labels bit-identical to the single-process oracle."""
    u, v = rmat_pairs_host(13, 16 << 13, 0.57, 0.19, 0.19, 14)
    hg = csr_from_pairs(1 << 13, u, v)
    g = O.as_graph(hg)
    ref = O.parallel_cc(g, None, 0.85, O.Opts(schedule=O.SYNC))
    r = run(world, backend_name, hg, 0.85, dict(schedule="sync"), gather_below=0)
    assert np.array_equal(r["C"], ref)
    assert r["sharded_levels"] >= 2


def test_sharded_cuda_idle_rank():
    """ADVICE (round 1): a rank whose owned frontier empties runs an empty
    round (no NULL-frontier call, which would mean V' = V) -- level-0 mover
    counts and labels equal the single-rank run."""
    from tests.test_dist_gloo import NCLQ, _split_graph
    hg = _split_graph()
    two = run(2, "gloo", hg, 0.85, dict(schedule="sync"), level0=True)
    one = run(1, "gloo", hg, 0.85, dict(schedule="sync"), level0=True)
    assert two["moves"] == one["moves"] and two["rounds"] == one["rounds"]
    assert np.array_equal(two["C"], one["C"])
    g = O.as_graph(hg)
    full = run(2, "gloo", hg, 0.85, dict(schedule="sync"))
    assert np.array_equal(full["C"], O.parallel_cc(g, None, 0.85, O.Opts(schedule=O.SYNC)))
    assert np.all(full["C"][:NCLQ].reshape(-1, 4) == full["C"][:NCLQ:4, None])
