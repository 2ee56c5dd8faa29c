"""Host-side generators and CSR builder against the reference builder's
golden output (tests/golden/make_golden.py ran graph.py build_graph*)."""
import numpy as np

from paper_2108_01731_b200.gen import csr_from_pairs, lfr_like, rmat_pairs_host, sbm


def test_sbm_cfg1_matches_reference_csr(golden):
    z = golden("sbm_cfg1.npz")
    g, comm = sbm(seed=1)
    assert g.n == 10_000
    assert np.array_equal(g.indptr, z["indptr"])
    assert np.array_equal(g.indices, z["indices"])
    assert np.all(z["weights"] == 1.0)
    assert g.m == int(z["m"][0])
    assert np.array_equal(comm, z["community"])
    # shape sanity: ~24.75K intra + ~24.75K inter edges (BASELINE configs[0])
    assert 45_000 < g.m < 54_000


def test_rmat_host_stream_matches_reference_csr(golden):
    z = golden("rmat_s10.npz")
    u, v = rmat_pairs_host(10, 16 << 10, 0.57, 0.19, 0.19, 24)
    g = csr_from_pairs(1 << 10, u, v)
    assert np.array_equal(g.indptr, z["indptr"])
    assert np.array_equal(g.indices, z["indices"])


def test_csr_invariants_small_lfr():
    g, comm = lfr_like(n=20_000, seed=3)
    deg = np.diff(g.indptr)
    assert g.indptr[-1] == 2 * g.m
    src = np.repeat(np.arange(g.n), deg)
    assert np.all(src != g.indices)                    # no self loops
    key = src * g.n + g.indices
    assert np.all(np.diff(key) > 0)                    # rows sorted, no duplicates
    rev = np.sort(g.indices.astype(np.int64) * g.n + src)
    assert np.array_equal(np.sort(key), rev)           # symmetric
    assert 4.0 < deg.mean() < 8.0                      # avg degree ~6
    intra = np.mean(comm[src] == comm[g.indices])
    assert 0.55 < intra < 0.85                         # mixing mu ~0.3


def test_rmat_quadrant_a_fraction():
    """SPEC.md:429 (scaled): first-descent quadrant-a fraction ~ a."""
    u, v = rmat_pairs_host(1, 200_000, 0.57, 0.19, 0.19, 9)
    frac = np.mean((u == 0) & (v == 0))
    assert abs(frac - 0.57) < 0.01
