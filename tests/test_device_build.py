"""Device graph build, weighted degrees / modularity mapping, the COO merge
of the sharded contraction, and the round's edge cases -- all through the C
ABI, against the reference's own outputs (golden) or the oracle.

* ``build_graph_arrays`` (lcc_build_graph) vs the reference's
  build_graph_arrays (graph.py:98-164): bit-exact CSR, weights and
  total_weight, including groups of hundreds of parallel edges (numpy's
  pairwise summation order) -- tests/golden/build_heavy.npz;
* ``weighted_degrees`` (lcc_weighted_degrees) vs graph.py:57-61 (np.add.at
  order): bit-exact;
* ``modularity_params`` / ``modularity_value`` vs the
  oracle: bit-exact unweighted, <= 1e-12 relative weighted;
* K rebuild with non-integral k: identical bits across runs;
* empty frontier: an empty round (SPEC "moved = {} -> empty frontier").
"""
import numpy as np
import pytest
import torch

import paper_2108_01731_b200 as L
from oracle import oracle as O
from paper_2108_01731_b200 import _lib
from paper_2108_01731_b200.gen import csr_from_pairs, rmat_pairs_host
from paper_2108_01731_b200.graph import build_graph, build_graph_arrays

from tests.test_gpu_parity import rand_weighted

pytestmark = pytest.mark.gpu


def test_build_heavy_groups_bit_exact(golden):
    z = golden("build_heavy.npz")
    for t in z["cases"]:
        p = f"b{t}_"
        g = build_graph_arrays(z[p + "u"], z[p + "v"], z[p + "w"], n=int(z[p + "n"][0]))
        ip, ind, w = g.to_host()
        assert g.m == int(z[p + "m"][0])
        assert np.array_equal(ip, z[p + "indptr"]) and np.array_equal(ind, z[p + "indices"])
        assert np.array_equal(w, z[p + "weights"]), t
        assert g.total_weight == float(z[p + "total"][0]), (t, g.total_weight, float(z[p + "total"][0]))


def test_build_errors_and_edge_cases():
    with pytest.raises(L.GraphError, match="equal length"):
        build_graph_arrays([0, 1], [1], [1.0, 1.0])
    with pytest.raises(L.GraphError, match="empty graph"):
        build_graph_arrays([], [], [])
    with pytest.raises(L.GraphError, match="non-negative"):
        build_graph_arrays([0, -1], [1, 2], [1.0, 1.0])
    with pytest.raises(L.GraphError, match="smaller than largest vertex id 4"):
        build_graph_arrays([0, 4], [1, 2], [1.0, 1.0], n=3)
    with pytest.raises(L.GraphError, match="triples"):
        build_graph([(0, 1)])
    g = build_graph_arrays([], [], [], n=5)  # isolated vertices only
    assert g.n == 5 and g.m == 0 and g.indptr.cpu().tolist() == [0] * 6 and g.total_weight == 0.0
    g = build_graph([(2, 2, 1.0), (3, 3, 5.0)])  # self loops only
    assert g.n == 4 and g.m == 0
    g = build_graph([(0, 1, 2.0), (1, 0, 4.0), (0, 1, 1.0), (5, 4, 1.0)])
    ip, ind, w = g.to_host()
    assert ip.tolist() == [0, 1, 2, 2, 2, 3, 4] and ind.tolist() == [1, 0, 5, 4]
    assert w.tolist() == [3.5, 3.5, 1.0, 1.0] and g.total_weight == 4.5


def test_weighted_degrees_bit_exact():
    rng = np.random.default_rng(5)
    for fp32 in (True, False):
        hg = rand_weighted(rng, 3000, 0.01, fp32=fp32, lo=0.1, hi=3.0)
        # a hub with a long row: the per-row sum order matters
        got = L.DeviceGraph.from_graph(hg).weighted_degrees().cpu().numpy()
        assert np.array_equal(got, O.weighted_degrees(O.as_graph(hg))), fp32
    u, v = rmat_pairs_host(12, 16 << 12, 0.57, 0.19, 0.19, 3)
    hg = csr_from_pairs(1 << 12, u, v)
    got = L.DeviceGraph.from_graph(hg).weighted_degrees().cpu().numpy()
    assert np.array_equal(got, np.diff(hg.indptr).astype(np.float64))


def test_modularity_params_and_value():
    u, v = rmat_pairs_host(12, 16 << 12, 0.57, 0.19, 0.19, 4)
    hg = csr_from_pairs(1 << 12, u, v)
    g = O.as_graph(hg)
    for gamma in (0.5, 1.0, 2.0):
        p = L.modularity_params(hg, gamma)
        k, lam = O.modularity_params(g, gamma)
        assert p.lam == lam and np.array_equal(p.k.cpu().numpy(), k)
        C = O.parallel_cc(g, k, lam, O.Opts(schedule=O.SYNC))
        q = L.modularity_value(hg, gamma, C)
        assert q == O.objective(g, k, lam, C) / g.total_weight
    rng = np.random.default_rng(6)
    hw = rand_weighted(rng, 2000, 0.01, fp32=False, lo=0.2, hi=2.0)
    gw = O.as_graph(hw)
    p = L.modularity_params(hw, 1.0)
    k, lam = O.modularity_params(gw, 1.0)
    assert np.array_equal(p.k.cpu().numpy(), k)
    assert abs(p.lam - lam) <= 1e-12 * lam
    C = O.parallel_cc(gw, k, lam, O.Opts(schedule=O.SYNC))
    ref = O.objective(gw, k, lam, C) / gw.total_weight
    assert abs(L.modularity_value(hw, 1.0, C) - ref) <= 1e-12 * max(1.0, abs(ref))


def test_mass_rebuild_nonintegral_k_deterministic():
    rng = np.random.default_rng(7)
    n = 200_000
    labels = torch.as_tensor(rng.integers(0, 5000, n).astype(np.int32), device="cuda")
    k = torch.as_tensor(rng.random(n) * 10.0 ** rng.uniform(-4, 4, n), device="cuda")
    p = L.ClusteringParams(0.5, k)
    runs = [L.apply_moves(labels, n, p) for _ in range(3)]
    for c in runs[1:]:
        assert torch.equal(c.assignment, runs[0].assignment)
        assert torch.equal(c.cluster_mass.view(torch.int64), runs[0].cluster_mass.view(torch.int64))
    C, K = O.canonicalize(n, labels.cpu().numpy(), n, k.cpu().numpy())
    assert np.array_equal(runs[0].assignment.cpu().numpy(), C)
    np.testing.assert_allclose(runs[0].cluster_mass.cpu().numpy(), K, rtol=1e-12, atol=0)


def test_empty_frontier_is_an_empty_round():
    u, v = rmat_pairs_host(10, 8 << 10, 0.57, 0.19, 0.19, 1)
    hg = csr_from_pairs(1 << 10, u, v)
    p = L.ClusteringParams(0.85)
    for sched in (L.Schedule.Synchronous, L.Schedule.Asynchronous):
        c = L.singletons(hg.n, p)
        mark = torch.ones(hg.n, dtype=torch.uint8, device="cuda")
        mb = L.best_moves_round(hg, p, c, frontier=[], schedule=sched, nbr_mark=mark)
        assert mb.moved_count == 0 and int(mb.moved.sum()) == 0 and int(mark.sum()) == 0
        assert torch.equal(mb.desired.cpu(), torch.arange(hg.n, dtype=torch.int32))
        # frontier=None is V' = V
        mb = L.best_moves_round(hg, p, L.singletons(hg.n, p), frontier=None, schedule=sched)
        assert mb.moved_count > 0


def test_coo_merge_sums_duplicates():
    import ctypes
    rng = np.random.default_rng(8)
    n, nnz = 3000, 200_000
    rows = rng.integers(0, n, nnz).astype(np.int32)
    cols = rng.integers(0, 5 * n, nnz).astype(np.int32)
    for wt in ("none", "u32", "f64"):
        w = None if wt == "none" else (rng.integers(1, 50, nnz).astype(np.uint32) if wt == "u32"
                                       else rng.random(nnz))
        key = rows.astype(np.int64) * (1 << 32) + cols
        uk, inv = np.unique(key, return_inverse=True)
        ref_w = np.bincount(inv, weights=None if w is None else w.astype(np.float64), minlength=uk.size)
        ref_ptr = np.zeros(n + 1, np.int64)
        np.cumsum(np.bincount(uk >> 32, minlength=n), out=ref_ptr[1:])
        d = {x: torch.as_tensor(y, device="cuda") for x, y in (("r", rows), ("c", cols))}
        wd = None if w is None else torch.as_tensor(w.astype(np.int32) if wt == "u32" else w, device="cuda")
        ip = torch.empty(n + 1, dtype=torch.int64, device="cuda")
        ind = torch.empty(nnz, dtype=torch.int32, device="cuda")
        wo = torch.empty(nnz, dtype=torch.float64 if wt == "f64" else torch.int32, device="cuda")
        cnt = ctypes.c_int64()
        wtype = {"none": _lib.W_NONE, "u32": _lib.W_U32, "f64": _lib.W_F64}[wt]
        _lib.check(_lib.load().lcc_coo_merge(n, nnz, d["r"].data_ptr(), d["c"].data_ptr(),
                                             None if wd is None else wd.data_ptr(), wtype, ip.data_ptr(),
                                             ind.data_ptr(), wo.data_ptr(), ctypes.byref(cnt),
                                             torch.cuda.current_stream().cuda_stream))
        R = cnt.value
        assert R == uk.size
        assert np.array_equal(ip.cpu().numpy(), ref_ptr)
        assert np.array_equal(ind[:R].cpu().numpy(), (uk & 0xffffffff).astype(np.int32))
        got = wo[:R].cpu().numpy().astype(np.float64)
        if wt == "f64":
            np.testing.assert_allclose(got, ref_w, rtol=1e-12)
        else:
            assert np.array_equal(got, ref_w)
