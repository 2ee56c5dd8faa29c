"""Pin the CPU oracle (oracle/) before trusting it as the parity checker.

* SPEC known-answer examples (SPEC.md:107-145, 202-213, 264-275, 302-304,
  221, 294) with the SURVEY.md §4 errata applied;
* golden vectors produced by the reference's own graph.py
  (tests/golden/make_golden.py): contraction via build_graph_arrays and
  vertex-neighbour frontiers via frontier_from_members;
* brute-force pair enumeration for the objective and the move delta;
* an independent pure-Python Jacobi round against the C round.
"""
import numpy as np
import pytest

from oracle import oracle as O


def graph(edges, n=None):
    """Small symmetric CSR from an edge list (unique unordered pairs)."""
    if n is None:
        n = 1 + max(max(u, v) for u, v, _ in edges) if edges else 0
    adj = [[] for _ in range(n)]
    for u, v, w in edges:
        if u != v:
            adj[u].append((v, w))
            adj[v].append((u, w))
    indptr = np.zeros(n + 1, np.int64)
    indices, weights = [], []
    for v in range(n):
        row = sorted(adj[v])
        indptr[v + 1] = indptr[v] + len(row)
        indices += [u for u, _ in row]
        weights += [w for _, w in row]
    w = np.array(weights, np.float64)
    g = O.Graph(n, indptr, np.array(indices, np.int32), None if np.all(w == 1.0) else w, float(w.sum() / 2))
    return g, adj


def rand_graph(rng, n, p, weighted):
    edges = []
    for i in range(n):
        for j in range(i + 1, n):
            if rng.random() < p:
                edges.append((i, j, float(rng.uniform(-1, 2)) if weighted else 1.0))
    return edges


# ---------------------------------------------------------------- KATs ----

def test_objective_kats():
    # SPEC.md:116-118
    g, _ = graph([(0, 1, 1.0), (0, 2, 1.0), (1, 2, -3.0)])
    assert O.objective(g, None, 0.0, np.arange(3, dtype=np.int32)) == 0.0
    assert O.objective(g, None, 0.0, np.zeros(3, np.int32)) == -1.0
    t, _ = graph([(0, 1, 1.0), (1, 2, 1.0), (0, 2, 1.0)])
    assert O.objective(t, None, 0.2, np.zeros(3, np.int32)) == pytest.approx(2.4, abs=1e-12)


def test_modularity_kats():
    t, _ = graph([(0, 1, 1.0), (1, 2, 1.0), (0, 2, 1.0)])
    k, lam = O.modularity_params(t, 1.0)
    assert lam == pytest.approx(1 / 6) and np.all(k == 2.0)
    assert O.objective(t, k, lam, np.zeros(3, np.int32)) / t.total_weight == pytest.approx(1 / 3)  # :144
    p2, _ = graph([(0, 1, 1.0)])
    k, lam = O.modularity_params(p2, 0.5)
    assert lam == pytest.approx(0.25) and np.all(k == 1.0)
    with pytest.raises(ValueError):
        O.modularity_params(p2, 2.0)
    # two disjoint edges: cc/m = 0.75 under the SPEC's own i != j definition
    # (SURVEY.md §4 erratum 2; SPEC.md:145 quotes Newman's 1/2)
    d, _ = graph([(0, 1, 1.0), (2, 3, 1.0)])
    k, lam = O.modularity_params(d, 1.0)
    q = O.objective(d, k, lam, np.array([0, 0, 2, 2], np.int32)) / d.total_weight
    assert q == pytest.approx(0.75)
    # Newman conversion: Q_newman = cc/m - gamma*sum d^2/(4 m^2)
    assert q - 1.0 * np.sum(k ** 2) / (4 * d.total_weight ** 2) == pytest.approx(0.5)


def test_figure1_sync_and_async():
    """SPEC.md:264-265, acceptance #4 with erratum 1."""
    g, _ = graph([(0, 1, 1.0), (0, 2, 1.0), (1, 2, -3.0)])
    C, K = O.singletons(3, None)
    # V' = {b, c}: both join {a}, objective -1
    D, mv, cnt = O.sync_round(g, None, 0.0, C, K, F=np.array([1, 2]))
    assert list(D) == [0, 0, 0] and cnt == 2
    Cn, _ = O.canonicalize(3, D, 6, None)
    assert O.objective(g, None, 0.0, Cn) == -1.0
    # V' = V: a moves too (tie -> lowest id), giving {a},{b,c}, objective -3
    D, mv, cnt = O.sync_round(g, None, 0.0, C, K)
    assert list(D) == [1, 0, 0]
    Cn, _ = O.canonicalize(3, D, 6, None)
    assert O.objective(g, None, 0.0, Cn) == -3.0
    # single-thread async: b joins a, c then declines -> objective 1 > -1
    C2 = C.copy()
    K2 = np.zeros(6); K2[:3] = 1
    O.async_round(g, None, 0.0, C2, K2, F=np.array([1, 2]))
    Cn, _ = O.canonicalize(3, C2, 6, None)
    assert O.objective(g, None, 0.0, Cn) == 1.0


def test_no_positive_pairs_no_moves():
    g, _ = graph([(0, 1, 0.1), (1, 2, 0.2)])
    C, K = O.singletons(3, None)
    _, _, cnt = O.sync_round(g, None, 0.5, C, K)
    assert cnt == 0


def test_isolated_vertex_stays_and_leaves():
    # isolated singleton stays
    g, _ = graph([(0, 1, 1.0)], n=3)
    C, K = O.singletons(3, None)
    D, _, _, gains = O.sync_round(g, None, 0.3, C, K, F=np.array([2]), with_gains=True)
    assert D[2] == 2 and gains[2] == 0.0
    # isolated vertex inside a bigger cluster takes the fresh singleton
    C = np.array([0, 0, 0], np.int32)
    K = np.array([3.0, 0, 0])
    D, _, _ = O.sync_round(g, None, 0.3, C, K, F=np.array([2]))
    assert D[2] == 3 + 2


def test_compress_kats():
    # SPEC.md:202-204
    g, _ = graph([(0, 1, 1.0), (0, 2, 2.0), (1, 2, 3.0)])
    C, K = O.canonicalize(3, np.array([0, 0, 2], np.int32), 3, None)
    lvl = O.compress(g, None, 0.0, C, K)
    assert lvl.graph.n == 2 and lvl.graph.m == 1 and list(lvl.graph.weights) == [5.0, 5.0]
    assert lvl.internal_offset == 1.0
    C, K = O.canonicalize(3, np.zeros(3, np.int32), 3, None)
    lvl = O.compress(g, None, 0.0, C, K)
    assert lvl.graph.n == 1 and lvl.graph.m == 0 and list(lvl.k) == [3.0]
    C, K = O.singletons(3, None)
    lvl = O.compress(g, None, 0.0, C, K)
    assert lvl.graph.n == 3 and np.array_equal(lvl.graph.indices, g.indices) and lvl.internal_offset == 0.0


def test_flatten_kats():
    # SPEC.md:211-213
    mapping = np.array([0, 0, 1], np.int32)
    C, _ = O.flatten(3, mapping, np.array([0, 1], np.int32), None)
    assert list(C) == [0, 0, 2]
    C, _ = O.flatten(3, mapping, np.array([0, 0], np.int32), None)
    assert list(C) == [0, 0, 0]


def test_frontier_kats():
    # SPEC.md:273-275
    p, _ = graph([(0, 1, 1.0), (1, 2, 1.0), (3, 4, 1.0)])
    none = np.zeros(5, np.uint8)
    C = np.arange(5, dtype=np.int32)
    assert O.frontier(p, O.VERTEX_NBRS, none, C, C).size == 0
    mv = np.array([0, 1, 0, 0, 0], np.uint8)
    assert list(O.frontier(p, O.VERTEX_NBRS, mv, C, C)) == [0, 2]
    Cold = np.array([0, 1, 2, 1, 4], np.int32)  # 1 moves from {1,3} into {0}
    Cnew = np.array([0, 0, 2, 3, 4], np.int32)
    assert list(O.frontier(p, O.CLUSTER_NBRS, mv, Cold, Cnew)) == [0, 1, 2, 4]


def test_two_cliques_sync_and_async():
    """two 4-cliques + bridge at lambda 0.4 -> the cliques (value 7.2)."""
    edges = [(b + i, b + j, 1.0) for b in (0, 4) for i in range(4) for j in range(i + 1, 4)] + [(3, 4, 1.0)]
    g, _ = graph(edges)
    _, best = O.py_brute_force_best(8, edges, None, 0.4)
    for sched in (O.SYNC, O.ASYNC):
        C = O.parallel_cc(g, None, 0.4, O.Opts(schedule=sched))
        assert list(C) == [0] * 4 + [4] * 4
        assert O.objective(g, None, 0.4, C) == pytest.approx(best, abs=1e-9)


# ------------------------------------------------------- golden vectors ----

def test_contraction_matches_reference_build_graph(golden):
    z = golden("contraction.npz")
    for t in z["cases"]:
        p = f"c{t}_"
        w = z[p + "weights"]
        g = O.Graph(int(z[p + "indptr"].size - 1), z[p + "indptr"], z[p + "indices"],
                    None if np.all(w == 1.0) else w, float(w.sum() / 2))
        C = z[p + "C"]
        K = np.bincount(C, minlength=g.n).astype(np.float64)
        lvl = O.compress(g, None, 0.3, C, K)
        assert np.array_equal(lvl.mapping, z[p + "mapping"])
        assert np.array_equal(lvl.graph.indptr, z[p + "cindptr"])
        assert np.array_equal(lvl.graph.indices, z[p + "cindices"])
        np.testing.assert_allclose(lvl.graph.weights, z[p + "cweights"], rtol=1e-12, atol=1e-12)
        assert lvl.graph.total_weight == pytest.approx(float(z[p + "ctotal"][0]), rel=1e-12, abs=1e-12)


def test_frontier_matches_reference(golden):
    z = golden("frontier.npz")
    for t in z["cases"]:
        p = f"f{t}_"
        n = z[p + "indptr"].size - 1
        g = O.Graph(n, z[p + "indptr"], z[p + "indices"], None, 0.0)
        mv = np.zeros(n, np.uint8)
        mv[z[p + "moved"]] = 1
        C = np.arange(n, dtype=np.int32)
        got = O.frontier(g, O.VERTEX_NBRS, mv, C, C)
        assert np.array_equal(got, z[p + "frontier"])


# ------------------------------------------------------------ properties ---

@pytest.mark.parametrize("seed", range(6))
def test_objective_equals_pair_enumeration(seed):
    rng = np.random.default_rng(seed)
    n = int(rng.integers(2, 12))
    edges = rand_graph(rng, n, 0.4, weighted=True)
    g, _ = graph(edges, n)
    k = rng.integers(0, 4, n).astype(np.float64)
    lam = float(rng.uniform(0, 0.9))
    C = rng.integers(0, n, n).astype(np.int32)
    assert O.objective(g, k, lam, C) == pytest.approx(O.py_objective_pairs(n, edges, k, lam, C), abs=1e-9)


@pytest.mark.parametrize("seed", range(6))
def test_move_delta_equals_objective_difference(seed):
    """SPEC.md:157 / acceptance #2."""
    rng = np.random.default_rng(100 + seed)
    n = int(rng.integers(3, 10))
    edges = rand_graph(rng, n, 0.5, weighted=True)
    g, adj = graph(edges, n)
    k = rng.integers(1, 3, n).astype(np.float64)
    lam = float(rng.uniform(0, 0.9))
    C, K = O.canonicalize(n, rng.integers(0, n, n).astype(np.int32), n, k)
    before = O.objective(g, k, lam, C)
    D, mv, cnt, gains = O.sync_round(g, k, lam, C, K, with_gains=True)
    for v in range(n):
        if mv[v]:
            lab = C.astype(np.int64).copy()
            lab[v] = D[v]  # fresh ids n+v stay unique
            C2, _ = O.canonicalize(n, lab.astype(np.int32), 2 * n, k)
            assert O.objective(g, k, lam, C2) - before == pytest.approx(gains[v], abs=1e-9)


@pytest.mark.parametrize("seed", range(8))
def test_c_round_equals_python_round(seed):
    rng = np.random.default_rng(200 + seed)
    n = int(rng.integers(2, 40))
    weighted = seed % 2 == 1
    edges = rand_graph(rng, n, 0.2, weighted)
    g, adj = graph(edges, n)
    k = None if seed % 3 else rng.integers(1, 5, n).astype(np.float64)
    lam = float(rng.uniform(0, 0.9))
    C, K = O.canonicalize(n, rng.integers(0, n, n).astype(np.int32), n, k)
    D, _, _ = O.sync_round(g, k, lam, C, K)
    assert list(D) == O.py_sync_round(n, adj, k, lam, list(C), list(K))


@pytest.mark.parametrize("seed", range(4))
def test_compression_conservation(seed):
    """SPEC.md:226 / acceptance #5: cc(G, flatten(C, C'')) = cc(G', C'') + offset."""
    rng = np.random.default_rng(300 + seed)
    n = int(rng.integers(3, 32))
    edges = rand_graph(rng, n, 0.3, weighted=True)
    g, _ = graph(edges, n)
    k = rng.integers(1, 4, n).astype(np.float64)
    lam = float(rng.uniform(0.01, 0.5))
    C, K = O.canonicalize(n, rng.integers(0, max(1, n // 2), n).astype(np.int32), n, k)
    lvl = O.compress(g, k, lam, C, K)
    Ccc = rng.integers(0, lvl.graph.n, lvl.graph.n).astype(np.int32)
    Cf, _ = O.flatten(n, lvl.mapping, Ccc, k)
    lhs = O.objective(g, k, lam, Cf)
    rhs = O.objective(lvl.graph, lvl.k, lam, Ccc) + lvl.internal_offset
    assert lhs == pytest.approx(rhs, abs=1e-9)


def test_sync_determinism_across_threads():
    """sync results identical across thread counts."""
    rng = np.random.default_rng(7)
    edges = rand_graph(rng, 300, 0.03, weighted=True)
    g, _ = graph(edges, 300)
    outs = [O.parallel_cc(g, None, 0.3, O.Opts(schedule=O.SYNC, threads=t)) for t in (1, 2, 8)]
    assert all(np.array_equal(outs[0], o) for o in outs[1:])


def test_async_mass_conservation():
    """SPEC.md:308 / acceptance #11 for the parallel (atomic) async round."""
    from paper_2108_01731_b200.gen import rmat_pairs_host, csr_from_pairs
    u, v = rmat_pairs_host(12, 16 << 12, 0.57, 0.19, 0.19, 5)
    hg = csr_from_pairs(1 << 12, u, v)
    g = O.as_graph(hg)
    C, K = O.singletons(g.n, None)
    K2 = np.zeros(2 * g.n); K2[:g.n] = K
    D = C.copy()
    O.async_round(g, None, 0.85, D, K2, parallel=True, threads=8)
    assert K2.sum() == pytest.approx(g.n, rel=1e-12)
    Cn, Kn = O.canonicalize(g.n, D, 2 * g.n, None)
    assert Kn.sum() == g.n
