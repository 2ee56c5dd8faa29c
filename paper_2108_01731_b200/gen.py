"""Seeded synthetic inputs for the five BASELINE.json configs.

The paper's SNAP / UCI inputs are absent, so each config is
a seeded synthetic stand-in with the stated shape.  Generators are input
plumbing, not the hot path:

* ``sbm``      -- config 1, planted-partition SBM (numpy, host).
* ``lfr_like`` -- config 2, power-law degrees + power-law community sizes
  with mixing mu, configuration-model pairing (numpy, host).
* ``knn_mixture`` -- config 3, weighted cosine kNN of a Gaussian mixture
  (torch on the device when present; fp32 weights in (0, 1]).
* ``rmat_device`` -- config 4, R-MAT on the device (``lcc_gen_rmat``):
  counter-based splitmix64 draws, so ``rmat_pairs_host`` reproduces the same
  sample stream on the host for small scales (tests).

All return undirected, deduplicated, self-loop-free graphs; the unweighted
ones deduplicate pairs before the CSR build (SURVEY.md §4 erratum 3), so
every edge weighs exactly 1.
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .graph import DeviceGraph, _device, stream_ptr


@dataclass
class HostGraph:
    """Host CSR with the reference WeightedGraph fields (graph.py:33-38)."""
    n: int
    m: int
    indptr: np.ndarray
    indices: np.ndarray
    weights: np.ndarray | None
    total_weight: float


def csr_from_pairs(n: int, u: np.ndarray, v: np.ndarray) -> HostGraph:
    """Symmetric CSR from undirected unweighted pairs: drop self loops,
    dedupe unordered pairs, emit both directions, rows sorted (the
    reference build_graph_arrays contract for w = 1, graph.py:117-164)."""
    u = np.asarray(u, np.int64)
    v = np.asarray(v, np.int64)
    keep = u != v
    lo = np.minimum(u[keep], v[keep])
    hi = np.maximum(u[keep], v[keep])
    key = np.unique(lo * n + hi)
    lo, hi = key // n, key % n
    src = np.concatenate([lo, hi])
    dst = np.concatenate([hi, lo])
    order = np.lexsort((dst, src))
    src, dst = src[order], dst[order]
    indptr = np.zeros(n + 1, np.int64)
    np.cumsum(np.bincount(src, minlength=n), out=indptr[1:])
    m = int(key.size)
    return HostGraph(n, m, indptr, dst.astype(np.int32), None, float(m))


def sbm(n: int = 10_000, communities: int = 100, p_in: float = 0.05, p_out: float = 0.0005,
        seed: int = 1):
    """Config 1: planted partition, equal communities, independent pairs.
    Returns (graph, ground-truth community of each vertex)."""
    rng = np.random.Generator(np.random.PCG64(seed))
    size = n // communities
    comm = np.arange(n) // size
    # intra: every pair inside each community, Bernoulli(p_in)
    iu, ju = np.triu_indices(size, 1)
    reps = communities
    base = (np.arange(reps) * size)[:, None]
    pu = (base + iu[None, :]).ravel()
    pv = (base + ju[None, :]).ravel()
    hit = rng.random(pu.size) < p_in
    eu, ev = [pu[hit]], [pv[hit]]
    # inter: Binomial(#inter pairs, p_out) distinct uniformly random pairs
    n_inter_pairs = n * (n - 1) // 2 - reps * size * (size - 1) // 2
    k = int(rng.binomial(n_inter_pairs, p_out))
    got = np.empty(0, np.int64)
    while got.size < k:
        a = rng.integers(0, n, size=2 * (k - got.size) + 16)
        b = rng.integers(0, n, size=a.size)
        ok = comm[a] != comm[b]
        lo, hi = np.minimum(a[ok], b[ok]), np.maximum(a[ok], b[ok])
        got = np.unique(np.concatenate([got, lo * n + hi]))
    got = rng.permutation(got)[:k]
    eu.append(got // n)
    ev.append(got % n)
    g = csr_from_pairs(n, np.concatenate(eu), np.concatenate(ev))
    return g, comm


def _powerlaw_int(rng, size, exponent, xmin, xmax):
    # continuous power law on [xmin, xmax] by inverse CDF, floored
    a = 1.0 - exponent
    u = rng.random(size)
    x = (xmin ** a + u * (xmax ** a - xmin ** a)) ** (1.0 / a)
    return np.floor(x).astype(np.int64)


def lfr_like(n: int = 1_200_000, avg_degree: float = 6.0, deg_exponent: float = 2.5,
             comm_exponent: float = 1.5, mu: float = 0.3, min_comm: int = 20, max_comm: int = 5000,
             max_degree: int = 1000, seed: int = 2):
    """Config 2: LFR-style planted communities.
    Degrees ~ power law (exponent 2.5) on [d_min, max_degree] with d_min set
    so the mean is ~avg_degree; community sizes ~ power law (exponent 1.5)
    on [min_comm, max_comm]; a fraction 1-mu of each vertex's stubs pair
    inside its community, the rest globally (configuration model); self
    loops and duplicates are dropped.  Returns (graph, community)."""
    rng = np.random.Generator(np.random.PCG64(seed))
    # choose d_min so that the truncated mean matches avg_degree
    dmin = 1.0
    for _ in range(60):
        probe = _powerlaw_int(np.random.Generator(np.random.PCG64(12345)), 200_000, deg_exponent, dmin, max_degree + 1)
        if probe.mean() < avg_degree:
            dmin *= 1.05
        else:
            break
    deg = np.clip(_powerlaw_int(rng, n, deg_exponent, dmin, max_degree + 1), 1, max_degree)
    sizes = []
    tot = 0
    while tot < n:
        s = int(_powerlaw_int(rng, 1, comm_exponent, min_comm, max_comm + 1)[0])
        s = min(s, n - tot)
        sizes.append(s)
        tot += s
    sizes = np.array(sizes, np.int64)
    perm = rng.permutation(n)
    comm = np.empty(n, np.int64)
    comm[perm] = np.repeat(np.arange(sizes.size), sizes)
    csize = sizes[comm]
    k_in = np.minimum(np.rint((1.0 - mu) * deg).astype(np.int64), csize - 1)
    k_out = deg - k_in
    # intra stubs: shuffle within community, pair consecutive
    stub_v = np.repeat(np.arange(n), k_in)
    stub_c = comm[stub_v]
    order = np.lexsort((rng.random(stub_v.size), stub_c))
    stub_v, stub_c = stub_v[order], stub_c[order]
    starts = np.searchsorted(stub_c, np.arange(sizes.size))
    pos = np.arange(stub_v.size) - starts[stub_c]
    first = (pos % 2 == 0)
    has_pair = np.zeros(stub_v.size, bool)
    has_pair[:-1] = first[:-1] & (stub_c[1:] == stub_c[:-1])
    idx = np.flatnonzero(has_pair)
    iu, iv = stub_v[idx], stub_v[idx + 1]
    # inter stubs: global configuration model
    ostub = rng.permutation(np.repeat(np.arange(n), k_out))
    if ostub.size % 2:
        ostub = ostub[:-1]
    ou, ov = ostub[0::2], ostub[1::2]
    g = csr_from_pairs(n, np.concatenate([iu, ou]), np.concatenate([iv, ov]))
    return g, comm


# ---------------------------------------------------------------------------
# R-MAT
# ---------------------------------------------------------------------------
_GOLD = np.uint64(0x9E3779B97F4A7C15)


def _splitmix64(z: np.ndarray) -> np.ndarray:
    with np.errstate(over="ignore"):
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        return z ^ (z >> np.uint64(31))


def rmat_pairs_host(scale: int, samples: int, a: float, b: float, c: float, seed: int):
    """Host replica of the device sample stream (gen.cu k_rmat)."""
    t1, t2, t3 = a, a + b, a + b + c
    i = np.arange(samples, dtype=np.uint64)
    src = np.zeros(samples, np.uint64)
    dst = np.zeros(samples, np.uint64)
    with np.errstate(over="ignore"):
        for l in range(scale):
            ctr = i * np.uint64(scale) + np.uint64(l) + np.uint64(1)
            z = _splitmix64(np.uint64(seed) + _GOLD * ctr)
            r = (z >> np.uint64(11)).astype(np.float64) * (2.0 ** -53)
            bs = (r >= t2).astype(np.uint64)
            bd = (((r >= t1) & (r < t2)) | (r >= t3)).astype(np.uint64)
            src = (src << np.uint64(1)) | bs
            dst = (dst << np.uint64(1)) | bd
    return src.astype(np.int64), dst.astype(np.int64)


def rmat_device(scale: int = 24, edge_factor: int = 16, a: float = 0.57, b: float = 0.19, c: float = 0.19,
                seed: int = 24, samples: int | None = None) -> DeviceGraph:
    """Config 4 (BASELINE.json configs[3]): Graph500 R-MAT, symmetrised,
    deduplicated, self-loops removed, no vertex permutation.  ``samples``
    (directed draws) overrides ``edge_factor * 2^scale``."""
    dev = _device()
    n = 1 << scale
    if samples is None:
        samples = edge_factor * n
    indptr = torch.empty(n + 1, dtype=torch.int64, device=dev)
    indices = torch.empty(max(2 * samples, 1), dtype=torch.int32, device=dev)
    nnz = ctypes.c_int64()
    _lib.check(_lib.load().lcc_gen_rmat(scale, samples, a, b, c, seed, indptr.data_ptr(), indices.data_ptr(),
                                        ctypes.byref(nnz), stream_ptr()))
    nnz = nnz.value
    indices = indices[:nnz].clone()
    return DeviceGraph(n, nnz // 2, indptr, indices, None, float(nnz // 2))


def device_csr_from_pairs(n: int, u, v) -> DeviceGraph:
    dev = _device()
    ut = torch.as_tensor(np.asarray(u, np.int32)).to(dev)
    vt = torch.as_tensor(np.asarray(v, np.int32)).to(dev)
    indptr = torch.empty(n + 1, dtype=torch.int64, device=dev)
    indices = torch.empty(max(2 * ut.numel(), 1), dtype=torch.int32, device=dev)
    nnz = ctypes.c_int64()
    _lib.check(_lib.load().lcc_build_csr_from_pairs(n, ut.numel(), ut.data_ptr(), vt.data_ptr(), indptr.data_ptr(),
                                                    indices.data_ptr(), ctypes.byref(nnz), stream_ptr()))
    nnz = nnz.value
    return DeviceGraph(n, nnz // 2, indptr, indices[:nnz].clone(), None, float(nnz // 2))


# ---------------------------------------------------------------------------
# config 3: weighted kNN similarity graph (BASELINE.json configs[2])
# ---------------------------------------------------------------------------

def knn_mixture(n: int = 4_000_000, dim: int = 64, components: int = 10_000, k: int = 10, sigma: float = 1.0,
                seed: int = 3, device=None, batch: int = 512):
    """Seeded stand-in for the paper's ScaNN k-NN graphs.

    Points: a Gaussian mixture in R^dim -- component means ~ N(0, I), points
    mean + sigma * N(0, I), component sizes multinomial with equal weights,
    ids grouped by component (no permutation).  Neighbours: exact top-k by
    cosine similarity inside each component (the mixture components are far
    apart, so this is the component-neighbourhood kNN of SURVEY.md §8d).
    Symmetrised: an unordered pair is an edge if either endpoint lists the
    other; its weight is the fp32 cosine recomputed once per pair, so both
    orientations carry identical values.  Pairs with cosine <= 0 are dropped
    and weights are clamped to (0, 1].  Returns (HostGraph with fp32-exact
    fp64 weights, component of each vertex)."""
    dev = torch.device(device) if device is not None else (torch.device("cuda") if torch.cuda.is_available()
                                                              else torch.device("cpu"))
    gen = torch.Generator().manual_seed(seed)
    sizes = torch.multinomial(torch.full((components,), 1.0 / components), n, replacement=True,
                              generator=gen).bincount(minlength=components)
    comp = torch.repeat_interleave(torch.arange(components), sizes)
    means = torch.randn(components, dim, generator=gen)
    pts = means[comp] + sigma * torch.randn(n, dim, generator=gen)
    pts = torch.nn.functional.normalize(pts, dim=1).to(dev)
    starts = torch.zeros(components + 1, dtype=torch.int64)
    starts[1:] = torch.cumsum(sizes, 0)
    us, vs = [], []
    smax = int(sizes.max())
    kk = min(k, max(smax - 1, 1))
    for c0 in range(0, components, batch):
        c1 = min(components, c0 + batch)
        nb = c1 - c0
        X = torch.zeros(nb, smax, dim, device=dev)
        valid = torch.zeros(nb, smax, dtype=torch.bool, device=dev)
        for j, c in enumerate(range(c0, c1)):
            s, e = int(starts[c]), int(starts[c + 1])
            X[j, :e - s] = pts[s:e]
            valid[j, :e - s] = True
        S = torch.bmm(X, X.transpose(1, 2))
        S.masked_fill_(~valid[:, None, :], -2.0)
        idx = torch.arange(smax, device=dev)
        S[:, idx, idx] = -2.0
        top = torch.topk(S, kk, dim=2)
        base = starts[c0:c1].to(dev)[:, None, None]
        src = (base + idx[None, :, None]).expand(nb, smax, kk)
        dst = base + top.indices
        ok = valid[:, :, None] & (top.values > -1.5)
        us.append(src[ok].cpu())
        vs.append(dst[ok].cpu())
    u = torch.cat(us).numpy()
    v = torch.cat(vs).numpy()
    lo, hi = np.minimum(u, v), np.maximum(u, v)
    key = np.unique(lo * n + hi)
    lo, hi = key // n, key % n
    P = pts.cpu()
    w = (P[torch.from_numpy(lo)] * P[torch.from_numpy(hi)]).sum(1).numpy().astype(np.float32)
    keep = w > 0
    lo, hi, w = lo[keep], hi[keep], np.minimum(w[keep], np.float32(1.0))
    src = np.concatenate([lo, hi])
    dst = np.concatenate([hi, lo])
    ww = np.concatenate([w, w]).astype(np.float64)
    order = np.lexsort((dst, src))
    src, dst, ww = src[order], dst[order], ww[order]
    indptr = np.zeros(n + 1, np.int64)
    np.cumsum(np.bincount(src, minlength=n), out=indptr[1:])
    m = int(lo.size)
    return HostGraph(n, m, indptr, dst.astype(np.int32), ww, float(w.astype(np.float64).sum())), comp.numpy()


# ---------------------------------------------------------------------------
# config 5: large power-law planted-community graph (BASELINE.json configs[4])
# ---------------------------------------------------------------------------

def powerlaw_communities_device(n: int = 65_000_000, m_target: int = 1_800_000_000, deg_exponent: float = 2.2,
                                mu: float = 0.4, max_degree: int = 5214, comm_exponent: float = 1.5,
                                min_comm: int = 20, max_comm: int = 5000, seed: int = 5,
                                oversample: float = 1.34) -> DeviceGraph:
    """Seeded stand-in for friendster (65.6M vertices, 1.8B
    edges; max degree 5,214 per PAPER.md:594).  Expected degrees follow a
    power law (exponent 2.2) capped at max_degree and scaled to mean
    2*m_target/n; community sizes follow a power law (exponent 1.5) on
    [min_comm, max_comm], contiguous ids; Chung-Lu draws (lcc_gen_powerlaw_
    communities) with mixing mu, then deduplicated and symmetrised on the
    device.  Host numpy builds the weight prefixes only."""
    dev = _device()
    rng = np.random.Generator(np.random.PCG64(seed))
    a = 1.0 - deg_exponent
    u = rng.random(n)
    theta = (1.0 + u * (float(max_degree) ** a - 1.0)) ** (1.0 / a)   # power law on [1, max_degree]
    theta *= (2.0 * m_target / n) / theta.mean()
    sizes = []
    tot = 0
    while tot < n:
        k = max(1, (n - tot) // 200)
        ua = rng.random(k)
        b = 1.0 - comm_exponent
        s = np.floor((min_comm ** b + ua * ((max_comm + 1) ** b - min_comm ** b)) ** (1.0 / b)).astype(np.int64)
        s = s[np.cumsum(s) <= n - tot] if s.sum() > n - tot else s
        if s.size == 0:
            s = np.array([n - tot], np.int64)
        sizes.append(s)
        tot += int(s.sum())
    sizes = np.concatenate(sizes)
    cstart = np.zeros(sizes.size + 1, np.int64)
    np.cumsum(sizes, out=cstart[1:])
    vw = np.zeros(n + 1, np.float64)
    np.cumsum(theta, out=vw[1:])
    cwp = vw[cstart]
    cw = cwp - cwp[0]
    samples = int(m_target * oversample)
    d_vw = torch.from_numpy(vw).to(dev)
    d_cs = torch.from_numpy(cstart).to(dev)
    d_cw = torch.from_numpy(cw).to(dev)
    indptr = torch.empty(n + 1, dtype=torch.int64, device=dev)
    indices = torch.empty(2 * samples, dtype=torch.int32, device=dev)
    nnz = ctypes.c_int64()
    _lib.check(_lib.load().lcc_gen_powerlaw_communities(n, samples, mu, d_vw.data_ptr(), d_cs.data_ptr(),
                                                        d_cw.data_ptr(), sizes.size, seed, indptr.data_ptr(),
                                                        indices.data_ptr(), ctypes.byref(nnz), stream_ptr()))
    del d_vw, d_cs, d_cw
    nnz = nnz.value
    out = indices[:nnz].clone()
    del indices
    torch.cuda.empty_cache()
    return DeviceGraph(n, nnz // 2, indptr, out, None, float(nnz // 2))
