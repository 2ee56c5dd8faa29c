"""Eval module.

CPU: the oracle restatements against the SPEC known-answer examples and
sklearn (the SPEC's "standard formula").  GPU (-m gpu): the device metrics
(``csrc/eval.cu`` through the C ABI) against the oracle and sklearn.
"""
import numpy as np
import pytest
from sklearn.metrics import adjusted_rand_score, normalized_mutual_info_score

from oracle import oracle as O


def _nmi(a, b):
    return normalized_mutual_info_score(a, b, average_method="arithmetic")


# ---------------------------------------------------------------- CPU: oracle
def test_oracle_precision_recall_spec_examples():
    # SPEC.md:350-352
    lab = [0, 1, 1, 2, 2]  # vertices 0..4; clusters {1,2},{3,4}; vertex 0 alone
    assert O.py_avg_precision_recall(lab, [[1, 2, 3]]) == pytest.approx((1.0, 2 / 3))
    one = [0, 0, 0, 0, 0]
    assert O.py_avg_precision_recall(one, [[1, 2], [3, 4]]) == pytest.approx((0.4, 1.0))
    lab4 = [9, 9, 9, 9]  # SPEC literal: vertices {1,2,3,4} -> here ids 0..3 all in one cluster
    assert O.py_avg_precision_recall(lab4, [[0, 1], [2, 3]]) == pytest.approx((0.5, 1.0))
    part = [0, 0, 1, 1, 1]
    assert O.py_avg_precision_recall(part, [[0, 1], [2, 3, 4]]) == pytest.approx((1.0, 1.0))
    with pytest.raises(ValueError):
        O.py_avg_precision_recall(part, [])


def test_oracle_ari_nmi_against_sklearn():
    # SPEC.md:356-358 and 361-364
    a = [0, 0, 0, 1, 1, 1]
    b = [0, 0, 1, 1, 1, 1]
    assert O.py_ari_pairs(a, b) == pytest.approx(adjusted_rand_score(a, b), abs=1e-15)
    assert O.py_ari_pairs(a, a) == 1.0
    sing, one = list(range(8)), [0] * 8
    assert adjusted_rand_score(sing, one) == 0.0
    assert _nmi(one, sing) == 0.0
    rng = np.random.default_rng(5)
    for _ in range(20):
        x = rng.integers(0, 5, 40)
        y = rng.integers(0, 7, 40)
        assert O.py_ari_pairs(list(x), list(y)) == pytest.approx(adjusted_rand_score(x, y), abs=1e-12)


def test_oracle_cluster_stats():
    # SPEC.md:366-367
    assert O.py_cluster_stats([0, 1, 2, 3, 4]) == (5, 1, 1, 1.0)
    assert O.py_cluster_stats([7] * 5) == (1, 5, 5, 5.0)
    assert O.py_cluster_stats([0, 0, 1, 1, 1]) == (2, 2, 3, 2.5)


# ---------------------------------------------------------------- GPU parity
@pytest.mark.gpu
def test_gpu_ari_nmi_matches_sklearn():
    import paper_2108_01731_b200.eval as E
    rng = np.random.default_rng(11)
    cases = [
        (np.arange(10), np.arange(10)),                     # identical (all singletons)
        (np.zeros(10, int), np.zeros(10, int)),             # both one cluster
        (np.arange(12), np.zeros(12, int)),                 # singletons vs one cluster
        (np.array([0, 0, 0, 1, 1, 1]), np.array([0, 0, 1, 1, 1, 1])),
        (np.array([-5, -5, 3, 3, 7]), np.array([2, 2, 2, -1, -1])),  # arbitrary int32 ids
        (np.array([1]), np.array([4])),                     # one sample
    ]
    for n, ka, kb in [(1000, 10, 30), (100_000, 1000, 50), (2_000_000, 100_000, 5000)]:
        cases.append((rng.integers(0, ka, n), rng.integers(0, kb, n)))
    x = rng.integers(0, 3000, 500_000)
    cases.append((x, np.where(rng.random(x.size) < 0.9, x, rng.integers(0, 3000, x.size))))  # correlated
    for a, b in cases:
        ga, gn = E.ari_nmi(a.astype(np.int32), b.astype(np.int32))
        assert ga == pytest.approx(adjusted_rand_score(a, b), rel=1e-9, abs=1e-12), (a[:5], b[:5])
        assert gn == pytest.approx(_nmi(a, b), rel=1e-9, abs=1e-12), (a[:5], b[:5])
        # symmetric, permutation invariant
        assert E.ari(b.astype(np.int32), a.astype(np.int32)) == pytest.approx(ga, rel=1e-12, abs=1e-14)
        perm = rng.permutation(max(a.max(), 0) + 1)
        if a.min() >= 0:
            assert E.nmi(perm[a].astype(np.int32), b.astype(np.int32)) == pytest.approx(gn, rel=1e-12, abs=1e-14)


@pytest.mark.gpu
def test_gpu_precision_recall_matches_oracle():
    import paper_2108_01731_b200.eval as E
    from paper_2108_01731_b200.graph import GraphError
    # SPEC examples
    gt = E.GroundTruth.from_sets([[1, 2, 3]])
    assert E.avg_precision_recall(np.array([0, 1, 1, 2, 2], np.int32), gt) == pytest.approx((1.0, 2 / 3))
    gt2 = E.GroundTruth.from_sets([[0, 1], [2, 3]])
    assert E.avg_precision_recall(np.array([9, 9, 9, 9], np.int32), gt2) == pytest.approx((0.5, 1.0))
    rng = np.random.default_rng(3)
    for n, k, nc, size in [(200, 7, 15, 20), (50_000, 400, 800, 60), (1_000_000, 20_000, 5000, 300)]:
        lab = rng.integers(0, k, n).astype(np.int32)
        comms = [rng.choice(n, size=int(rng.integers(1, size)), replace=False) for _ in range(nc)]  # overlapping
        gt = E.GroundTruth.from_sets(comms)
        want = O.py_avg_precision_recall(lab, gt.communities())
        got = E.avg_precision_recall(lab, gt)
        assert got == pytest.approx(want, rel=1e-12)
    # ties to the lowest cluster id: {0,1} split 1/1 between clusters 5 and 3 -> 3 (size 3)
    lab = np.array([5, 3, 3, 3, 5], np.int32)
    assert E.avg_precision_recall(lab, E.GroundTruth.from_sets([[0, 1]])) == pytest.approx((1 / 3, 0.5))
    with pytest.raises(GraphError):
        E.avg_precision_recall(lab, E.GroundTruth(np.zeros(1, np.int64), np.zeros(0, np.int32)))
    with pytest.raises(GraphError):
        E.avg_precision_recall(lab, E.GroundTruth.from_sets([[0, 9]]))


@pytest.mark.gpu
def test_gpu_cluster_stats_and_parallel_cc_eval():
    import paper_2108_01731_b200 as L
    import paper_2108_01731_b200.eval as E
    from paper_2108_01731_b200.gen import sbm
    assert E.cluster_stats(np.arange(5, dtype=np.int32)) == (5, 1, 1, 1.0)
    assert E.cluster_stats(np.full(5, 7, np.int32)) == (1, 5, 5, 5.0)
    assert E.cluster_stats(np.array([0, 0, 1, 1, 1], np.int32)) == (2, 2, 3, 2.5)
    rng = np.random.default_rng(8)
    lab = rng.integers(-1000, 1000, 300_000).astype(np.int32)
    assert E.cluster_stats(lab) == pytest.approx(O.py_cluster_stats(lab))
    # SPEC.md:461 ground-truth recovery: planted partition p_in 0.5 / p_out 0.01, lambda 0.05
    g, truth = sbm(n=2000, communities=20, p_in=0.5, p_out=0.01, seed=7)
    c = L.parallel_cc(g, L.ClusteringParams(0.05), L.ParOptions(schedule=L.Schedule.Synchronous))
    gt = E.GroundTruth.from_sets([np.flatnonzero(truth == t) for t in range(20)])
    p, r = E.avg_precision_recall(c, gt)
    assert p >= 0.95 and r >= 0.95
    assert E.ari(c, truth.astype(np.int32)) > 0.9
