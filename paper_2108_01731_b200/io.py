"""File ingestion and output (the reference's ``io-gen-cli`` module,
``SPEC.md:390-450``).

* ``read_edge_list(path, weighted)`` -- "u v" / "u v w" lines, '#' comments;
  non-integer ids are remapped densely (first appearance order) and the
  mapping is returned; the graph is built with the reference's
  ``build_graph_arrays`` semantics (``graph.py:98-164``): self loops dropped,
  parallel same-orientation edges summed, the two orientations of a pair
  averaged, rows sorted.  Unit weights are stored implicitly (``weights is
  None``) so the device path reads no weight array.
* ``read_ground_truth(path, id_map)`` -- one community per line.
* ``read_clustering`` / ``write_clustering`` -- "vertex_id cluster_id" lines
  in original ids; ``write_metrics`` -- one JSON object with the EvalReport
  keys (``SPEC.md:419``).

This is host-side plumbing around the device path (file parsing and the
CSR build of a file's edge list); the clustering itself and every metric
run in the sm_100a library.
"""
from __future__ import annotations

import json
import os
from dataclasses import dataclass

import numpy as np

from .eval import EvalReport, GroundTruth
from .graph import GraphError


@dataclass
class WeightedGraph:
    """Host CSR with the reference's ``WeightedGraph`` fields (graph.py:33-38)."""
    n: int
    m: int
    indptr: np.ndarray          # int64 [n+1]
    indices: np.ndarray         # int32 [2m]
    weights: np.ndarray | None  # float64 [2m], None when every weight is 1
    total_weight: float


def build_graph_arrays(u, v, w, n: int | None = None) -> WeightedGraph:
    """Restatement of the reference builder (graph.py:98-164)."""
    u = np.asarray(u, dtype=np.int64)
    v = np.asarray(v, dtype=np.int64)
    w = np.asarray(w, dtype=np.float64)
    if not (u.shape == v.shape == w.shape):
        raise GraphError("edge arrays must have equal length")
    if u.size == 0 and n is None:
        raise GraphError("empty graph")
    if u.size and (u.min() < 0 or v.min() < 0):
        raise GraphError("vertex ids must be non-negative")
    n_seen = int(max(u.max(), v.max())) + 1 if u.size else 0
    if n is None:
        n = n_seen
    elif n < n_seen:
        raise GraphError(f"n={n} smaller than largest vertex id {n_seen - 1}")
    n = int(n)
    keep = u != v
    u, v, w = u[keep], v[keep], w[keep]
    if u.size == 0:
        return WeightedGraph(n, 0, np.zeros(n + 1, np.int64), np.empty(0, np.int32), None, 0.0)
    lo, hi = np.minimum(u, v), np.maximum(u, v)
    orient = (u > v).astype(np.int8)
    order = np.lexsort((w, orient, hi, lo))  # weight last: order-independent sums
    lo, hi, orient, w = lo[order], hi[order], orient[order], w[order]
    grp = np.empty(lo.size, bool)
    grp[0] = True
    grp[1:] = (lo[1:] != lo[:-1]) | (hi[1:] != hi[:-1]) | (orient[1:] != orient[:-1])
    st = np.flatnonzero(grp)
    gsum = np.add.reduceat(w, st)
    glo, ghi = lo[st], hi[st]
    pair = np.empty(glo.size, bool)
    pair[0] = True
    pair[1:] = (glo[1:] != glo[:-1]) | (ghi[1:] != ghi[:-1])
    ps = np.flatnonzero(pair)
    cnt = np.diff(np.append(ps, glo.size))
    ew = np.add.reduceat(gsum, ps) / cnt
    eu, ev = glo[ps], ghi[ps]
    src = np.concatenate([eu, ev])
    dst = np.concatenate([ev, eu])
    ww = np.concatenate([ew, ew])
    order = np.lexsort((dst, src))
    src, dst, ww = src[order], dst[order], ww[order]
    indptr = np.zeros(n + 1, np.int64)
    np.cumsum(np.bincount(src, minlength=n), out=indptr[1:])
    weights = None if bool(np.all(ww == 1.0)) else ww
    return WeightedGraph(n, int(eu.size), indptr, dst.astype(np.int32), weights, float(ew.sum()))


def _parse_id(tok: str):
    try:
        return int(tok)
    except ValueError:
        return tok


def read_edge_list(path: str, weighted: bool = False):
    """SPEC.md:398-406.  Returns ``(graph, id_map)``; ``id_map[i]`` is the
    original id of vertex i, or None when the file's ids are non-negative
    integers (kept as they are)."""
    if not os.path.exists(path):
        raise FileNotFoundError(path)
    us, vs, ws = [], [], []
    with open(path) as f:
        for ln, line in enumerate(f, 1):
            s = line.strip()
            if not s or s.startswith("#"):
                continue
            tok = s.split()
            if len(tok) < 2 or len(tok) > 3 or (len(tok) == 3 and not weighted):
                raise GraphError(f"{path}:{ln}: malformed line {s!r}")
            us.append(_parse_id(tok[0]))
            vs.append(_parse_id(tok[1]))
            if weighted:
                if len(tok) == 3:
                    try:
                        ws.append(float(tok[2]))
                    except ValueError:
                        raise GraphError(f"{path}:{ln}: bad weight {tok[2]!r}") from None
                else:
                    ws.append(1.0)
    ids = us + vs
    id_map = None
    if all(isinstance(x, int) and x >= 0 for x in ids):
        u = np.asarray(us, np.int64)
        v = np.asarray(vs, np.int64)
    else:
        pos: dict = {}
        order = []
        for a, b in zip(us, vs):
            for x in (a, b):
                if x not in pos:
                    pos[x] = len(order)
                    order.append(x)
        u = np.asarray([pos[x] for x in us], np.int64)
        v = np.asarray([pos[x] for x in vs], np.int64)
        id_map = order
    w = np.asarray(ws, np.float64) if weighted else np.ones(u.size)
    n = None if u.size else 0
    return build_graph_arrays(u, v, w, n=n), id_map


def _index(id_map):
    return None if id_map is None else {x: i for i, x in enumerate(id_map)}


def read_ground_truth(path: str, id_map=None, n: int | None = None) -> GroundTruth:
    """one community per line, member ids whitespace separated."""
    idx = _index(id_map)
    comms = []
    with open(path) as f:
        for ln, line in enumerate(f, 1):
            tok = line.split()
            if not tok or tok[0].startswith("#"):
                continue
            mem = []
            for t in tok:
                x = _parse_id(t)
                if idx is not None:
                    if x not in idx:
                        raise GraphError(f"{path}:{ln}: unknown vertex id {t!r}")
                    x = idx[x]
                elif not isinstance(x, int) or x < 0 or (n is not None and x >= n):
                    raise GraphError(f"{path}:{ln}: unknown vertex id {t!r}")
                mem.append(x)
            comms.append(mem)
    return GroundTruth.from_sets(comms)


def _orig(i: int, id_map):
    return i if id_map is None else id_map[i]


def write_clustering(path: str, c, id_map=None) -> None:
    """lines "vertex_id cluster_id" in original ids; the
    cluster id is the original id of the cluster's smallest member."""
    lab = c.labels() if hasattr(c, "labels") else np.asarray(c)
    with open(path, "w") as f:
        if id_map is None:
            np.savetxt(f, np.stack([np.arange(lab.size), lab], 1), fmt="%d")
        else:
            for i, x in enumerate(lab.tolist()):
                f.write(f"{_orig(i, id_map)} {_orig(int(x), id_map)}\n")


def read_clustering(path: str, id_map=None, n: int | None = None) -> np.ndarray:
    """Inverse of ``write_clustering``: labels[n] (internal ids; any int values)."""
    idx = _index(id_map)
    pairs = []
    with open(path) as f:
        for ln, line in enumerate(f, 1):
            tok = line.split()
            if not tok or tok[0].startswith("#"):
                continue
            if len(tok) != 2:
                raise GraphError(f"{path}:{ln}: malformed line {line.strip()!r}")
            a, b = _parse_id(tok[0]), _parse_id(tok[1])
            if idx is not None:
                if a not in idx or b not in idx:
                    raise GraphError(f"{path}:{ln}: unknown vertex id")
                a, b = idx[a], idx[b]
            pairs.append((a, b))
    if not pairs:
        return np.zeros(0 if n is None else n, np.int32)
    arr = np.asarray(pairs, np.int64)
    size = int(arr[:, 0].max()) + 1 if n is None else n
    if arr[:, 0].min() < 0 or arr[:, 0].max() >= size:
        raise GraphError(f"{path}: vertex id out of range")
    lab = np.full(size, -1, np.int64)
    lab[arr[:, 0]] = arr[:, 1]
    if (lab < 0).any():
        raise GraphError(f"{path}: some vertices have no cluster")
    return lab.astype(np.int32)


def write_metrics(path: str, report: EvalReport) -> None:
    """one JSON object with the EvalReport keys (missing -> null)."""
    with open(path, "w") as f:
        f.write(report.to_json() + "\n")


def read_metrics(path: str) -> EvalReport:
    d = json.load(open(path))
    known = {k: d.pop(k) for k in list(d) if k in EvalReport.__dataclass_fields__ and k != "extra"}
    return EvalReport(**known, extra=d)
