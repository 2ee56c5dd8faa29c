"""Packed asynchronous rounds (LCC_PACK32, csrc/best_moves.cu): (label, mass)
in one 32-bit word per vertex; joins by compare-and-swap on the target's word.

An asynchronous round is deterministic when the frontier's vertices cannot
interact (one vertex per connected component), so on such frontiers the packed
round must leave exactly the state of the interleaved 64-bit image
(LCC_PACK32=0).  A second test narrows the mass field (LCC_PACK32_BITS) until
joins are refused, and checks the SPEC's async invariant (mass conservation,
SPEC.md:306-311) and the field bound.
"""
import os

import numpy as np
import pytest
import torch

import paper_2108_01731_b200 as L
from paper_2108_01731_b200 import _lib
from paper_2108_01731_b200.gen import csr_from_pairs

pytestmark = pytest.mark.gpu


def _async_round(d, p, C, K2, frontier, packed, bits=None):
    """One asynchronous round on copies of (C, K2) under LCC_PACK32=packed;
    returns labels, masses (2n) and the library's launch count for the call."""
    os.environ["LCC_PACK32"] = "1" if packed else "0"
    if bits is None:
        os.environ.pop("LCC_PACK32_BITS", None)
    else:
        os.environ["LCC_PACK32_BITS"] = str(bits)
    try:
        c = L.Clustering(C.clone(), K2.clone())
        lib = _lib.load()
        l0 = lib.lcc_kernel_launches()
        L.best_moves_round(d, p, c, frontier=frontier, schedule=L.Schedule.Asynchronous)
        torch.cuda.synchronize()
        return c.assignment, c.cluster_mass, lib.lcc_kernel_launches() - l0
    finally:
        os.environ.pop("LCC_PACK32", None)
        os.environ.pop("LCC_PACK32_BITS", None)


def _components_graph(rng, comps, size, p_edge):
    us, vs = [], []
    for q in range(comps):
        base = q * size
        for i in range(size):
            for j in range(i + 1, size):
                if rng.random() < p_edge:
                    us.append(base + i); vs.append(base + j)
        for i in range(size - 1):  # connected
            us.append(base + i); vs.append(base + i + 1)
    return csr_from_pairs(comps * size, np.array(us), np.array(vs))


@pytest.mark.parametrize("lam", [0.85, 0.3])
def test_packed_round_equals_interleaved_on_independent_frontiers(lam):
    rng = np.random.default_rng(7)
    # 8 components of 8 vertices: a frontier of one vertex per component is
    # n/8 vertices (the integer-mass images need at least that) and its
    # vertices cannot interact, so the round is deterministic
    comps, size = 8, 8
    hg = _components_graph(rng, comps, size, 0.5)
    n = hg.n
    d = L.DeviceGraph.from_graph(hg)
    p = L.ClusteringParams(lam)
    C = torch.arange(n, dtype=torch.int32, device="cuda")
    K2 = torch.zeros(2 * n, dtype=torch.float64, device="cuda")
    K2[:n] = 1.0
    took_packed = False
    for sweep in range(3):
        for i in range(size):
            F = [q * size + (i + q) % size for q in range(comps)]
            a = _async_round(d, p, C, K2, F, packed=True)
            b = _async_round(d, p, C, K2, F, packed=False)
            assert torch.equal(a[0], b[0]), (sweep, i)
            assert torch.equal(a[1], b[1]), (sweep, i)
            took_packed |= (b[2] - a[2]) == 1   # pack + unpack vs labels in + masses out + labels out
            C, K2 = a[0], a[1]
            # mass conservation: K2[x] = number of vertices labelled x (k = 1)
            cnt = torch.bincount(C.long(), minlength=2 * n).double()
            assert torch.equal(cnt, K2)
            # reconcile (canonical labels, rebuilt masses) and go on
            cl = L.apply_moves(C, 2 * n, p)
            C = cl.assignment
            K2 = torch.zeros(2 * n, dtype=torch.float64, device="cuda")
            K2[:n] = cl.cluster_mass
    assert took_packed, "the packed path never ran"
    assert int(torch.unique(C).numel()) < n  # something merged


def test_packed_round_refuses_joins_beyond_the_mass_field():
    # one 40-clique, lambda small: every vertex wants the same cluster.  A
    # 28-bit label field leaves 4 bits of mass (15): joins stop at 14.
    n = 40
    iu, ju = np.triu_indices(n, 1)
    hg = csr_from_pairs(n, iu, ju)
    d = L.DeviceGraph.from_graph(hg)
    p = L.ClusteringParams(0.01)
    C = torch.arange(n, dtype=torch.int32, device="cuda")
    K2 = torch.zeros(2 * n, dtype=torch.float64, device="cuda")
    K2[:n] = 1.0
    a = _async_round(d, p, C, K2, None, packed=True, bits=28)
    b = _async_round(d, p, C, K2, None, packed=False)
    assert (b[2] - a[2]) == 1, "the packed path did not run"
    lab, mass = a[0], a[1]
    cnt = torch.bincount(lab.long(), minlength=2 * n).double()
    assert torch.equal(cnt, mass)             # mass conservation
    assert float(mass.max().item()) <= 14.0   # the field bound held
    assert float(mass.max().item()) >= 2.0    # and joins did happen
    # the interleaved image conserves mass too
    assert torch.equal(torch.bincount(b[0].long(), minlength=2 * n).double(), b[1])
