"""Generate the golden fixtures in tests/golden/ by running the REFERENCE.

Run in the build container (where /root/reference exists):
    python tests/golden/make_golden.py
The fixtures are committed; nothing at test time reads /root/reference.

What comes from the reference (``/root/reference/pkg/src/lambdacc/graph.py``):
* ``build_graph`` / ``build_graph_arrays`` (graph.py:79-164): the CSR of
  every fixture graph, and the contraction edge-merge -- SURVEY.md §8c:
  ``build_graph_arrays(mapping[src], mapping[dst], w, n=n')`` over all 2m
  directed entries is exactly the coarse graph of ``compress``.
* ``frontier_from_members`` (graph.py:205-215): vertex-neighbour frontiers.
"""
from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, "/root/reference/pkg/src")

from lambdacc.graph import build_graph, build_graph_arrays, frontier_from_members  # noqa: E402

from paper_2108_01731_b200.gen import rmat_pairs_host, sbm  # noqa: E402


def random_graph(rng, n, p, weighted, messy=True):
    """Edge list with duplicates / both orientations / self loops, as the
    reference builder accepts."""
    u, v = np.nonzero(np.triu(rng.random((n, n)) < p, 1))
    w = rng.uniform(-1.0, 2.0, u.size) if weighted else np.ones(u.size)
    if messy and u.size:
        # permuted orientation (average is exact when both orientations agree)
        flip = rng.random(u.size) < 0.5
        u, v = np.where(flip, v, u), np.where(flip, u, v)
        # self loops are dropped by the builder
        s = rng.integers(0, n, 3)
        u = np.concatenate([u, s]); v = np.concatenate([v, s]); w = np.concatenate([w, np.ones(3)])
    return build_graph_arrays(u, v, w, n=n)


def canonical(labels):
    n = labels.size
    minm = np.full(labels.max() + 1, n, np.int64)
    np.minimum.at(minm, labels, np.arange(n))
    return minm[labels].astype(np.int32)


def contraction_cases(rng):
    out = {}
    cases = []
    for t in range(40):
        n = int(rng.integers(2, 48))
        g = random_graph(rng, n, float(rng.uniform(0.05, 0.5)), weighted=(t % 2 == 1))
        nclus = int(rng.integers(1, n + 1))
        C = canonical(rng.integers(0, nclus, n))
        roots = np.flatnonzero(C == np.arange(n))
        rank = np.full(n, -1, np.int64)
        rank[roots] = np.arange(roots.size)
        mapping = rank[C]
        src = np.repeat(np.arange(n), np.diff(g.indptr))
        cg = build_graph_arrays(mapping[src], mapping[g.indices], g.weights, n=int(roots.size))
        pre = f"c{t}_"
        out[pre + "indptr"] = g.indptr
        out[pre + "indices"] = g.indices
        out[pre + "weights"] = g.weights
        out[pre + "C"] = C
        out[pre + "mapping"] = mapping.astype(np.int32)
        out[pre + "cindptr"] = cg.indptr
        out[pre + "cindices"] = cg.indices
        out[pre + "cweights"] = cg.weights
        out[pre + "ctotal"] = np.array([cg.total_weight])
        cases.append(t)
    out["cases"] = np.array(cases)
    return out


def frontier_cases(rng):
    out = {}
    for t in range(30):
        n = int(rng.integers(5, 80))
        g = random_graph(rng, n, float(rng.uniform(0.02, 0.3)), weighted=False)
        moved = np.flatnonzero(rng.random(n) < rng.uniform(0.0, 0.5))
        nb = [g.neighbors(int(v))[0] for v in moved]
        ids = np.concatenate(nb) if nb else np.empty(0, np.int64)
        fr = frontier_from_members(ids, n, g)
        pre = f"f{t}_"
        out[pre + "indptr"] = g.indptr
        out[pre + "indices"] = g.indices
        out[pre + "moved"] = moved
        out[pre + "frontier"] = fr.members()
    out["cases"] = np.arange(30)
    return out


def build_cases(rng):
    """Raw edge lists -> the reference builder (graph.py:98-164): duplicates in
    one orientation (summed), both orientations (averaged), self loops
    (dropped), weighted and unweighted.  Checks io.build_graph_arrays."""
    out = {}
    for t in range(20):
        n = int(rng.integers(2, 40))
        k = int(rng.integers(1, 4 * n))
        u = rng.integers(0, n, k)
        v = rng.integers(0, n, k)
        if t % 3 == 0:
            u = np.concatenate([u, v[: k // 2]])  # reversed copies
            v = np.concatenate([v, u[: k // 2]])
        w = np.round(rng.uniform(-1.0, 3.0, u.size), 3) if t % 2 else np.ones(u.size)
        g = build_graph_arrays(u, v, w, n=n)
        pre = f"b{t}_"
        out.update({pre + "u": u, pre + "v": v, pre + "w": w, pre + "n": np.array([n]),
                    pre + "indptr": g.indptr, pre + "indices": g.indices, pre + "weights": g.weights,
                    pre + "total": np.array([g.total_weight]), pre + "m": np.array([g.m])})
    out["cases"] = np.arange(20)
    return out


def heavy_build_cases(rng):
    """Summation-order stress for the device builder: same-orientation
    groups of 1..600 parallel edges with weights over six decades (numpy's
    pairwise summation differs from a sequential sum past 8 terms), both
    orientations with different weights, and graphs with ~40K pairs
    (total_weight's pairwise tree spans two or more 16K-entry leaves)."""
    out = {}
    for t in range(6):
        n = int(rng.integers(50, 2000)) if t < 4 else int(rng.integers(8000, 20000))
        pairs = int(rng.integers(5, 60)) if t < 4 else 40_000
        a = rng.integers(0, n, pairs)
        b = rng.integers(0, n, pairs)
        mult = rng.integers(1, 600, pairs) if t < 4 else np.ones(pairs, np.int64)
        u = np.repeat(a, mult)
        v = np.repeat(b, mult)
        flip = rng.random(u.size) < (0.5 if t % 2 else 0.1)
        u, v = np.where(flip, v, u), np.where(flip, u, v)
        w = rng.uniform(0.0, 1.0, u.size) * 10.0 ** rng.uniform(-3, 3, u.size)
        w[rng.random(u.size) < 0.05] *= -1.0
        perm = rng.permutation(u.size)
        u, v, w = u[perm], v[perm], w[perm]
        g = build_graph_arrays(u, v, w, n=n)
        pre = f"b{t}_"
        out.update({pre + "u": u.astype(np.int32), pre + "v": v.astype(np.int32), pre + "w": w,
                    pre + "n": np.array([n]), pre + "indptr": g.indptr, pre + "indices": g.indices,
                    pre + "weights": g.weights, pre + "total": np.array([g.total_weight]), pre + "m": np.array([g.m])})
    out["cases"] = np.arange(6)
    return out


def main():
    rng = np.random.default_rng(2108_01731)
    np.savez_compressed(os.path.join(HERE, "contraction.npz"), **contraction_cases(rng))
    np.savez_compressed(os.path.join(HERE, "frontier.npz"), **frontier_cases(rng))
    # config-1 SBM through the reference builder
    g, comm = sbm(seed=1)
    src = np.repeat(np.arange(g.n), np.diff(g.indptr))
    keep = src < g.indices
    rg = build_graph_arrays(src[keep], g.indices[keep], np.ones(int(keep.sum())), n=g.n)
    np.savez_compressed(os.path.join(HERE, "sbm_cfg1.npz"), indptr=rg.indptr, indices=rg.indices,
                        weights=rg.weights, m=np.array([rg.m]), community=comm.astype(np.int32))
    # R-MAT scale 10 sample stream through the reference builder
    u, v = rmat_pairs_host(10, 16 << 10, 0.57, 0.19, 0.19, 24)
    rg = build_graph([(int(a), int(b), 1.0) for a, b in zip(u, v)], n=1 << 10)
    # unweighted duplicates merge by sum/average in the reference (erratum 3);
    # the structural CSR is what the generator must reproduce
    np.savez_compressed(os.path.join(HERE, "rmat_s10.npz"), indptr=rg.indptr, indices=rg.indices,
                        m=np.array([rg.m]))
    print("golden fixtures written to", HERE)


if __name__ == "__main__":
    if sys.argv[1:] == ["build"]:  # only the build fixture (tests/golden/build.npz)
        np.savez_compressed(os.path.join(HERE, "build.npz"), **build_cases(np.random.default_rng(398)))
    elif sys.argv[1:] == ["build_heavy"]:  # tests/golden/build_heavy.npz
        np.savez_compressed(os.path.join(HERE, "build_heavy.npz"), **heavy_build_cases(np.random.default_rng(399)))
    else:
        main()
        np.savez_compressed(os.path.join(HERE, "build.npz"), **build_cases(np.random.default_rng(398)))
        np.savez_compressed(os.path.join(HERE, "build_heavy.npz"), **heavy_build_cases(np.random.default_rng(399)))
