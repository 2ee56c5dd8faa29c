"""Sequential Louvain comparator (louvain-seq; SURVEY.md §8f
row 4) -- an oracle-side CPU comparator, single-threaded by design
(SPEC.md:231).  CPU: the SPEC examples and acceptance #1 (micro-scale
optimality against brute force).  GPU: acceptance #7 (parallel quality
parity: the device ``parallel_cc`` within [0.95, 1.10] x the sequential
convergence-mode objective)."""
import time

import numpy as np
import pytest

from oracle import oracle as O
from tests.test_oracle import graph, rand_graph


def test_seq_spec_examples():
    g, _ = graph([(0, 1, 1.0)])
    C = O.sequential_cc(g, None, 0.25, converge=True)
    assert list(C) == [0, 0] and O.objective(g, None, 0.25, C) == pytest.approx(0.75)
    g, _ = graph([], n=5)  # empty-edge graph -> singletons
    assert list(O.sequential_cc(g, None, 0.5)) == list(range(5))
    g, _ = graph([(0, 1, -1.0), (1, 2, -0.5)], n=4)  # every w' < 0 -> no move
    assert list(O.sequential_cc(g, None, 0.3, converge=True)) == [0, 1, 2, 3]
    edges = [(b + i, b + j, 1.0) for b in (0, 4) for i in range(4) for j in range(i + 1, 4)] + [(3, 4, 1.0)]
    g, _ = graph(edges)
    for seed in range(5):
        C = O.sequential_cc(g, None, 0.4, seed=seed)
        assert list(C) == [0] * 4 + [4] * 4


def test_acceptance_1_micro_optimality():
    """200 random graphs (n <= 8, mixed-sign weights, lambda in
    {0.05, 0.3, 0.6}); best of 5 seeds >= 95% of brute force on >= 90%;
    never above it."""
    rng = np.random.default_rng(454)
    good = 0
    t_seq = 0.0
    for i in range(200):
        n = int(rng.integers(2, 9))
        lam = (0.05, 0.3, 0.6)[i % 3]
        edges = rand_graph(rng, n, float(rng.uniform(0.2, 0.8)), weighted=True)
        g, _ = graph(edges, n=n)
        _, best = O.py_brute_force_best(n, edges, None, lam)
        t0 = time.perf_counter()
        vals = [O.objective(g, None, lam, O.sequential_cc(g, None, lam, converge=True, seed=s)) for s in range(5)]
        t_seq += time.perf_counter() - t0
        got = max(vals)
        assert got <= best + 1e-9
        assert min(vals) >= -1e-9  # the objective never drops below the start (0)
        if got >= 0.95 * best - 1e-12:
            good += 1
    assert good >= 180, good
    assert t_seq < 10.0


@pytest.mark.gpu
def test_acceptance_7_parallel_quality_parity():
    """parallel_cc (defaults) objective within [0.95, 1.10] x
    sequential-converge, on 10 planted-partition graphs (500 vertices, 10
    planted clusters) and R-MAT scale 14, 5 seeds each."""
    import paper_2108_01731_b200 as L
    from paper_2108_01731_b200.gen import csr_from_pairs, rmat_pairs_host, sbm
    graphs = [sbm(n=500, communities=10, p_in=0.3, p_out=0.02, seed=100 + i)[0] for i in range(10)]
    u, v = rmat_pairs_host(14, 16 << 14, 0.5, 0.1, 0.1, 14)
    graphs.append(csr_from_pairs(1 << 14, u, v))
    lam = 0.3
    ratios = []
    for g in graphs:
        og = O.as_graph(g)
        for seed in range(5):
            want = O.objective(og, None, lam, O.sequential_cc(og, None, lam, converge=True, seed=seed))
            c = L.parallel_cc(g, L.ClusteringParams(lam), L.ParOptions(seed=seed))
            got = L.cc_objective(g, L.ClusteringParams(lam), c)
            ratios.append(got / want)
    ratios = np.array(ratios)
    assert ratios.min() >= 0.95 and ratios.max() <= 1.10, (ratios.min(), ratios.max())
